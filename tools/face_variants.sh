#!/bin/bash
# face-solver occupancy variants: near-row capacity (build) x resident CTAs per SM (env)
O=gpurun_out
L=paper_2106_10031_b200/_lib
for v in b200 n96 n64; do
  lib=$L/libam_$v.so
  for c in 3 4 5 6; do
    echo "== $v ctas=$c" >> $O/variants.log
    AM_LIB_PATH=$PWD/$lib AM_FACE_CTAS=$c python tools/profile_march.py --repeat 3 2>&1 | grep geo90 | tail -2 >> $O/variants.log
  done
done

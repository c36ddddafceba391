#!/bin/bash
# configs[1] march time of in-tree build variants (AM_LIB_PATH), alternating, twice
O=gpurun_out
L=$PWD/paper_2106_10031_b200/_lib
for rep in 1 2; do for v in "$@"; do
  echo "== $v"; AM_LIB_PATH=$L/$v python tools/profile_march.py --repeat 5 | grep cells/s | tail -1
done; done > $O/variants.log 2>&1
cat $O/variants.log

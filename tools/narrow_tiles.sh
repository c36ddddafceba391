#!/bin/bash
# tile-width policy of k_compose_narrow: fixed widths and wave-size thresholds
O=gpurun_out
run() { echo "== $*" >> $O/tiles.log; env "$@" python tools/profile_march.py --repeat 3 2>&1 | grep geo90 | tail -2 >> $O/tiles.log; }
run AM_NARROW_TILE=8
run AM_NARROW_TILE=4
run AM_NARROW_TILE=2
run AM_NARROW_THR8=12 AM_NARROW_THR4=4
run AM_NARROW_THR8=16 AM_NARROW_THR4=6
run AM_NARROW_THR8=8 AM_NARROW_THR4=3
run AM_NARROW_THR8=24 AM_NARROW_THR4=8

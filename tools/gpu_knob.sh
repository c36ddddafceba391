#!/bin/bash
# configs[1] march time for values of one engine env knob, alternating, twice
O=gpurun_out
KNOB=$1; shift
for rep in 1 2; do for v in "$@"; do
  echo "== $KNOB=$v"; env $KNOB=$v python tools/profile_march.py --repeat 5 | grep cells/s | tail -1
done; done > $O/knob.log 2>&1
cat $O/knob.log

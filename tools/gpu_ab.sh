#!/bin/bash
# A/B timing of an engine knob on configs[1] (+ DeepSDF sample), then GPU parity tests
O=gpurun_out
KNOB=${1:-AM_NARROW96}
for v in 0 1 0 1; do echo "$KNOB=$v"; env $KNOB=$v python tools/profile_march.py --repeat 5 | tail -2; done > $O/ab.log 2>&1
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log; cat $O/ab.log

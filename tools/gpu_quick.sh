#!/bin/bash
# quick GPU check: parity tests, face stats, per-iteration trace, device march time
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
AM_LIB_PATH=$PWD/paper_2106_10031_b200/_lib/libam_stats.so python tools/profile_march.py > $O/face_stats.log 2>&1
AM_TRACE_ITERS=1 python tools/profile_march.py --timing > $O/trace_iters.log 2>&1
python tools/profile_march.py --repeat 5 > $O/march.log 2>&1
tail -3 $O/pytest_gpu.log; tail -4 $O/face_stats.log; tail -3 $O/march.log

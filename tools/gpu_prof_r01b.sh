#!/bin/bash
# round-1 profiling pass on one B200: face stats, per-iteration trace, launch list, ncu --set full of k_face / gemm
set -x
O=gpurun_out
AM_LIB_PATH=$PWD/paper_2106_10031_b200/_lib/libam_stats.so python tools/profile_march.py > $O/face_stats.log 2>&1
AM_TRACE_ITERS=1 python tools/profile_march.py --timing > $O/trace_iters.log 2>&1
python tools/profile_e2e.py --repeat 3 --reuse > $O/e2e_stages.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv python tools/profile_march.py > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_face -s 40 -c 1 -o $O/prof_face_r01b -f python tools/profile_march.py > $O/ncu_face.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_step -s 200 -c 1 -o $O/prof_gemm_r01b -f python tools/profile_march.py > $O/ncu_gemm.log 2>&1

#!/bin/bash
# Round profiling pass (one B200): bench line, launch list of one configs[1] march, ncu --set full
# of a mid-march k_face and k_gemm_step<4> launch (iteration ~31, ~5.9k cells), raw CSVs.
O=gpurun_out
python bench.py > $O/bench_line.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv \
    python tools/profile_march.py > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_face$' -s 30 -c 1 -o $O/prof_face -f \
    python tools/profile_march.py > $O/ncu_face.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_near$' -s 30 -c 1 -o $O/prof_near -f \
    python tools/profile_march.py > $O/ncu_near.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_step -s 400 -c 1 -o $O/prof_gemm -f \
    python tools/profile_march.py > $O/ncu_gemm.log 2>&1
for r in prof_face prof_near prof_gemm; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null; done
AM_TRACE_ITERS=1 python tools/profile_march.py --timing > $O/trace_iters.log 2>&1

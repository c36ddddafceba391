#!/bin/bash
# launch list of one configs[1] march + ncu --set full of a mid-march k_compose_narrow and k_face
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv \
    python tools/profile_march.py > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_compose_narrow -s 30 -c 1 -o $O/prof_narrow -f \
    python tools/profile_march.py > $O/ncu_narrow.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_face$' -s 30 -c 1 -o $O/prof_face -f \
    python tools/profile_march.py > $O/ncu_face.log 2>&1
for r in prof_narrow prof_face; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null; done
AM_TRACE_ITERS=1 python tools/profile_march.py --timing > $O/trace_iters.log 2>&1

#!/bin/bash
# ncu --set full of one mid-march k_face launch (configs[1]) with source counters
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'^k_face$' -s 30 -c 1 -o $O/prof_face_r01c -f python tools/profile_march.py > $O/ncu_face.log 2>&1
ncu -i $O/prof_face_r01c.ncu-rep --page source --csv --print-source sass > $O/face_source_sass.csv 2>/dev/null
ncu -i $O/prof_face_r01c.ncu-rep --page source --csv > $O/face_source_cuda.csv 2>/dev/null

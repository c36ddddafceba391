#!/bin/bash
# Round-2 final profiling pass (after prefix reuse) (one B200): launch list of one configs[1] march + ncu --set full of the
# mid-march launch (iteration ~31, ~5.9k cells) of every stage kernel; raw CSVs for ncu_summary.py
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
O=gpurun_out/p2b
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv \
    python tools/profile_march.py > $O/ncu_launch.log 2>&1
for k in k_compose_narrow:30 k_face:30 k_near:30 k_hash_upsert:61 k_probe_records:30 k_frontier:30 k_take:30; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$name" -s $skip -c 1 -o $O/prof_$name -f \
      python tools/profile_march.py > $O/ncu_$name.log 2>&1
  ncu -i $O/prof_$name.ncu-rep --page raw --csv > $O/prof_$name.raw.csv 2>/dev/null
done
# DeepSDF 512x8: one mid-march 512x512 layer of the per-step GEMM
ncu --set full --clock-control none --import-source on -k regex:k_gemm_step -s 200 -c 1 -o $O/prof_gemm512 -f \
    python tools/profile_march.py --net deepsdf512 --max-cells 200000 > $O/ncu_gemm512.log 2>&1
ncu -i $O/prof_gemm512.ncu-rep --page raw --csv > $O/prof_gemm512.raw.csv 2>/dev/null

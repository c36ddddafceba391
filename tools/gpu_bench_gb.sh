#!/bin/bash
O=gpurun_out
for rep in 1 2; do for gb in 16 32; do
  echo "== AM_GRAPH_BATCH=$gb"
  AM_GRAPH_BATCH=$gb python bench.py --no-extra --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), d['config']['ms_steps'], 'e2e', round(d['e2e']['ms_per_step'],2))"
done; done > $O/bench_gb.log 2>&1
cat $O/bench_gb.log

#!/bin/bash
# configs[4] fused-batch timing under engine knobs
O=gpurun_out
for kv in "AM_GATHER_INPUT=1 AM_GRAPH_BATCH=16" "AM_GATHER_INPUT=0 AM_GRAPH_BATCH=16" "AM_GATHER_INPUT=1 AM_GRAPH_BATCH=8" "AM_GATHER_INPUT=0 AM_GRAPH_BATCH=8"; do
  echo "== $kv"; env $kv python tools/profile_batch.py --repeat 2 2>&1 | tail -2
done > $O/batch_knobs.log 2>&1
cat $O/batch_knobs.log

#!/bin/bash
# multi-rank functional check on one GPU (2 ranks share the device over gloo; timings are not
# measurements) + the sharded-API parity test
O=gpurun_out
python -m pytest tests/test_distributed_gpu.py -x -q > $O/pytest_dist.log 2>&1; echo "rc=$?" >> $O/pytest_dist.log
AM_BENCH_SHARE_GPU=1 AM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2_shared.json 2> $O/bench_n2.err
echo "bench rc=$?" >> $O/pytest_dist.log
tail -3 $O/pytest_dist.log; tail -c 1500 $O/bench_n2_shared.json; tail -5 $O/bench_n2.err

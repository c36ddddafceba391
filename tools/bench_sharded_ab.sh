for v in 0 1; do
  AM_SHARD_PROBE_IN_GRAPH=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2954$v tools/bench_sharded.py > gpurun_out/bs_$v.json 2> gpurun_out/bs_$v.err
done

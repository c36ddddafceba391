"""The sharded march (device-driven rounds, NCCL all-to-all) timed on P ranks (torchrun, one per
GPU); P = 1 measures the round protocol's own overhead against the single-GPU path.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/bench_sharded.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.distributed import ShardedMarcher  # noqa: E402

out = {}
for name, net, cap, iters in (("configs[1]", synth.geometric_mlp([90] * 6, seed=0), 10_000_000, None),
                              ("configs[2] first 1M cells", synth.deepsdf_mlp(512, 8, 4, seed=0), 1_000_000, None)):
    for ipr in ((2, 4, 8, 16) if name == "configs[1]" else (4,)):
        sm = ShardedMarcher(net, max_cells=cap, iters_per_round=ipr)
        seeds = sm.sample_seeds(64, rng_seed=0)
        sm.run(seeds)
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sm.stream)
            s0 = sm.engine.shard_stats()
            rounds = sm.run(seeds)
            e1.record(sm.stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        st = sm.engine.shard_stats()
        t = torch.tensor([min(times), float(st["visited"])], device="cuda", dtype=torch.float64)
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        csum = t[1:].clone()
        dist.all_reduce(csum, op=dist.ReduceOp.SUM)
        out[f"{name} iters_per_round={ipr}"] = {
            "ranks": dist.get_world_size(), "ms": float(tmax.item()), "cells": int(csum.item()),
            "cells_per_s": float(csum.item()) / (float(tmax.item()) * 1e-3), "rounds": rounds,
            "host_syncs_per_round": (st["host_syncs"] - s0["host_syncs"]) / max(rounds, 1)}
        del sm
if dist.get_rank() == 0:
    print(json.dumps(out, indent=1))
dist.destroy_process_group()

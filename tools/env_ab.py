"""Interleaved A/B of engine knobs (environment variables read at engine creation) on one box:
one engine per variant, marched in turn; reports the BFS wall time (Engine.run, host syncs
included) per variant and whether each variant's result is bitwise equal to the first's.

    python tools/env_ab.py --repeat 10 "AM_PREFIX=1" "AM_PREFIX=0" "AM_PREFIX=1,AM_NARROW_THR8=8"
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth  # noqa: E402
from paper_2106_10031_b200 import engine as engmod  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="+")
ap.add_argument("--repeat", type=int, default=10)
ap.add_argument("--net", default="90x6")
ap.add_argument("--seeds", type=int, default=64)
ap.add_argument("--max-cells", type=int, default=0)
a = ap.parse_args()
if a.net.startswith("deepsdf"):   # deepsdf (512 wide) or deepsdf:W
    net = synth.deepsdf_mlp(int(a.net.split(":")[1]) if ":" in a.net else 512, 8, 4, seed=0)
else:
    w, d = (int(x) for x in a.net.split("x"))
    net = synth.geometric_mlp([w] * d, seed=0)
cfg = marching.MarchConfig(seeds=a.seeds, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3),
                           **({"max_cells": a.max_cells} if a.max_cells else {}))
T = []
orig_run = engmod.Engine.run


def timed_run(self):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_run(self)
    torch.cuda.synchronize()
    T.append((time.perf_counter() - t0) * 1e3)
    return r


engmod.Engine.run = timed_run
engines = []
for v in a.variants:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    marching.clear_engine_cache()
    engines.append(marching._engine_for(net, cfg))
    for k, o in old.items():
        if o is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = o
marching.clear_engine_cache()
times = [[] for _ in engines]
ref = None
for rep in range(a.repeat + 1):
    for i, eng in enumerate(engines):
        r = marching.march(net, cfg, engine=eng)
        if rep == 0:
            arrs = (r.keys, r.nverts, r.verts, r.edge_refs)
            if ref is None:
                ref = arrs
            same = all(np.array_equal(x, y) for x, y in zip(arrs, ref))
            st = eng.stats()
            print(f"{a.variants[i]}: cells {r.report.cells_visited} waves {r.report.waves} bitwise equal to first: {same}  "
                  f"prefix {st['prefix']:.0f} skipped flops {st['prefix_skipped_flops']:.3e}", flush=True)
        else:
            times[i].append(T[-1])
for v, t in zip(a.variants, times):
    print(f"{v:50s} BFS wall ms median {np.median(t):.3f}  min {np.min(t):.3f}")

"""Prefix reuse A/B on configs[1]: the march with AM_PREFIX=1 against AM_PREFIX=0 (bitwise equal
results expected: keys, polygons, vertices), plus the device time of the BFS (CUDA events on the
engine stream around Engine.run) of each, interleaved.

    python tools/prefix_ab.py [--repeat 10] [--net 90x6]
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
ap.add_argument("--repeat", type=int, default=10)
ap.add_argument("--net", default="90x6")
ap.add_argument("--seeds", type=int, default=64)
a = ap.parse_args()
w, d = (int(x) for x in a.net.split("x"))
net = synth.geometric_mlp([w] * d, seed=0)
cfg = marching.MarchConfig(seeds=a.seeds, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
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
engines = {}
for mode in (1, 0):
    os.environ["AM_PREFIX"] = str(mode)
    marching.clear_engine_cache()
    engines[mode] = marching._engine_for(net, cfg)
marching.clear_engine_cache()
res, times, stats = {}, {0: [], 1: []}, {}
for rep in range(a.repeat + 1):
    for mode in (1, 0):
        r = marching.march(net, cfg, engine=engines[mode])
        if rep == 0:
            res[mode] = r
            stats[mode] = engines[mode].stats()
        else:
            times[mode].append(T[-1])
    if rep == 0:
        a1, a0 = res[1], res[0]
        same = (np.array_equal(a1.keys, a0.keys) and np.array_equal(a1.nverts, a0.nverts)
                and np.array_equal(a1.verts, a0.verts) and np.array_equal(a1.edge_refs, a0.edge_refs))
        print(f"cells {a1.report.cells_visited} / {a0.report.cells_visited}  bitwise equal: {same}", flush=True)
        s1 = stats[1]
        print(f"prefix on: {s1['prefix']:.0f}  skipped flops {s1['prefix_skipped_flops']:.3e} of "
              f"{s1['compose_flops']:.3e} ({s1['prefix_skipped_flops'] / max(s1['compose_flops'], 1):.1%})", flush=True)
for mode in (1, 0):
    print(f"AM_PREFIX={mode}: BFS wall ms median {np.median(times[mode]):.3f}  min {np.min(times[mode]):.3f}")

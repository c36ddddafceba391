"""Stage timing of bench.py's e2e step: march(net, cfg).welded_mesh() on configs[1].

    python tools/profile_e2e_bench.py [--repeat 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth, meshes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--repeat", type=int, default=5)
a = ap.parse_args()
net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*args, **kw):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*args, **kw)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t) * 1e3
        return r
    setattr(mod, name, g)


for mod, name in [(marching, "_engine_for"), (marching, "sample_seeds"), (marching, "collect_result"),
                  (marching, "unique_plane_violations"), (marching, "device_results_to_host"),
                  (meshes, "weld_arrays"), (meshes, "weld_device"), (meshes, "to_host")]:
    wrap(mod, name)
from paper_2106_10031_b200 import engine as engmod  # noqa: E402
for name in ["seed", "run", "results_device", "forward", "dichotomy"]:
    f = getattr(engmod.Engine, name)

    def mk(f, name):
        def g(self, *args, **kw):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = f(self, *args, **kw)
            torch.cuda.synchronize()
            T["eng." + name] = T.get("eng." + name, 0.0) + (time.perf_counter() - t) * 1e3
            return r
        return g
    setattr(engmod.Engine, name, mk(f, name))

prev = None
for _ in range(3):
    cur = marching.march(net, cfg)
    prev = (cur, cur.welded_mesh())
del prev, cur
for r in range(a.repeat):
    T.clear()
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = marching.march(net, cfg)
    t1 = time.perf_counter()
    mesh = res.welded_mesh()
    t2 = time.perf_counter()
    import gc
    print(f"gc counts {gc.get_count()} | march {1e3 * (t1 - t0):.1f} ms  welded_mesh {1e3 * (t2 - t1):.1f} ms  total {1e3 * (t2 - t0):.1f} | "
          + " ".join(f"{k} {v:.1f}" for k, v in T.items()))

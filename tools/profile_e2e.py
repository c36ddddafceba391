"""Stage timing of one end-to-end march (marching.march) + weld on configs[1].

    python tools/profile_e2e.py [--net geo90x6|deepsdf512] [--repeat 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402
from paper_2106_10031_b200.marching import MarchConfig, collect_result  # noqa: E402
from paper_2106_10031_b200.meshes import weld_arrays  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="geo90x6")
ap.add_argument("--repeat", type=int, default=3)
ap.add_argument("--reuse", action="store_true", help="reuse one engine across repeats")
a = ap.parse_args()
net = synth.geometric_mlp([90] * 6, seed=0) if a.net == "geo90x6" else synth.deepsdf_mlp(512, 8, 4, seed=0)
cfg = MarchConfig(seeds=64, rng_seed=0, max_cells=10_000_000 if a.net == "geo90x6" else 200_000)
eng = None
for r in range(a.repeat):
    T = {}
    torch.cuda.synchronize()
    t = t0 = time.perf_counter()

    def lap(k):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[k] = (now - t) * 1e3
        t = now

    if eng is None or not a.reuse:
        eng = Engine(net, bbox=cfg.bbox, max_cells=cfg.max_cells)
    else:
        eng.reset()
    lap("engine")
    seeds = sample_seeds(eng, cfg.seeds, cfg.bbox, scheme=cfg.scheme, rng_seed=cfg.rng_seed)
    lap("seeds")
    eng.seed(seeds)
    waves = eng.run()
    lap("run")
    res = collect_result(eng, seeds, t0, waves)
    lap("collect")
    nv = res.nverts[res.nverts > 0].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
    kept, foff, fidx, _, nd = weld_arrays(res.verts, off, np.arange(off[-1], dtype=np.int64), 1e-7)
    lap("weld")
    tot = (time.perf_counter() - t0) * 1e3
    print(f"{a.net} cells {res.report.cells_visited} verts {len(res.verts)} kept {len(kept)} faces {len(foff) - 1} | "
          + " ".join(f"{k} {v:.1f}" for k, v in T.items()) + f" | total {tot:.1f} ms")

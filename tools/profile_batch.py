"""Stage timing of a fused latent batch (BASELINE configs[4] shape): seeding, march, split.

    python tools/profile_batch.py [--shapes 64] [--cap 20000] [--width 512]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.batch import _fused_engine, split_batch_result  # noqa: E402
from paper_2106_10031_b200.marching import MarchConfig  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", type=int, default=64)
ap.add_argument("--cap", type=int, default=20000)
ap.add_argument("--width", type=int, default=512)
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
nets, _ = synth.latent_batch(n_shapes=a.shapes, latent_dim=256, width=a.width, depth=8, skip_at=4, seed=0)
cfg = MarchConfig(seeds=64, rng_seed=0, max_cells=a.cap)
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
    eng = _fused_engine(nets, cfg)
    lap("engine+shapes")
    seeds = sample_seeds_batch(eng, nets, cfg.seeds, cfg.bbox, rng_seed=0)
    lap("seeds")
    pts = np.concatenate(seeds)
    shp = np.concatenate([np.full(len(x), s, np.int32) for s, x in enumerate(seeds)])
    eng.seed(pts, shapes=shp)
    lap("seed")
    waves = eng.run()
    lap("run")
    res = split_batch_result(eng, seeds, t0, waves)
    lap("split")
    cells = sum(x.report.cells_visited for x in res)
    tot = (time.perf_counter() - t0)
    print(f"{a.shapes} shapes w{a.width}: {cells} cells, {waves} waves | " + " ".join(f"{k} {v:.0f}" for k, v in T.items())
          + f" | total {tot * 1e3:.0f} ms, {cells / tot:.0f} cells/s")

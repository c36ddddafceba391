"""Wall time of march(net, cfg).welded_mesh() on configs[1] (bench.py's e2e step), no wrappers.

    python tools/e2e_ab.py [--repeat 20]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--repeat", type=int, default=20)
a = ap.parse_args()
net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
prev = None
for _ in range(3):
    cur = marching.march(net, cfg)
    prev = (cur, cur.welded_mesh())
del prev, cur
ts, tm = [], []
for _ in range(a.repeat):
    flush.fill_(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = marching.march(net, cfg)
    t1 = time.perf_counter()
    m = r.welded_mesh()
    t2 = time.perf_counter()
    ts.append((t2 - t0) * 1e3)
    tm.append((t1 - t0) * 1e3)
print(f"e2e median {np.median(ts):.2f} ms mean {np.mean(ts):.2f}  march median {np.median(tm):.2f}  "
      f"faces {m.n_faces} verts {m.n_vertices}")

"""Timing of the trigger (sample_seeds) pieces on configs[1]: sample blocks, first forward, pairing,
bisection, as the public march() runs them.

    python tools/prof_seeds.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import seeding, synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402

net = synth.geometric_mlp([90] * 6, seed=0)
eng = Engine(net)
lo, hi = np.full(3, -1.2), np.full(3, 1.2)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pts = np.stack([seeding._sample_block(0, i, 0, lo, hi) for i in range(64)])
    t1 = time.perf_counter()
    v = eng.forward(pts.reshape(-1, 3))
    t2 = time.perf_counter()
    vals = v.cpu().numpy().reshape(64, 64)
    t3 = time.perf_counter()
    xp, xn = pts[:, 0], pts[:, 1]
    out = eng.dichotomy(xp, xn, 1e-7, 1e-7)
    t4 = time.perf_counter()
    o = out.cpu().numpy()
    t5 = time.perf_counter()
    s = seeding.sample_seeds(eng, 64, (lo, hi))
    t6 = time.perf_counter()
    print(f"blocks {1e3*(t1-t0):.2f} forward-launch {1e3*(t2-t1):.2f} forward-D2H {1e3*(t3-t2):.2f} "
          f"dichotomy {1e3*(t4-t3):.2f} D2H {1e3*(t5-t4):.2f} | sample_seeds {1e3*(t6-t5):.2f} ms")

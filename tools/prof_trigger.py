"""Host-side timing of the trigger pieces on configs[1]: Engine.forward of the 4096 trigger samples,
Engine.dichotomy of 64 pairs, Engine.seed of 64 points, sample_seeds as a whole."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth, seeding  # noqa: E402

net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
r = marching.march(net, cfg)
eng = next(iter(marching._ENGINES.values()))
pts = np.random.default_rng(0).uniform(-1.2, 1.2, size=(4096, 3))


def t(name, f, n=20):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:40s} median {np.median(ts):.3f} ms  min {np.min(ts):.3f}")


t("forward 4096 (numpy in, .cpu() out)", lambda: eng.forward(pts).cpu())
dp = torch.as_tensor(pts, device="cuda")
t("forward 4096 (device in)", lambda: eng.forward(dp))
xp, xn = r.seeds + 0.01, r.seeds - 0.01
t("dichotomy 64", lambda: eng.dichotomy(xp, xn, seeding.SEED_TOL, seeding.SEED_TOL).cpu())
t("sample_seeds 64", lambda: seeding.sample_seeds(eng, 64, cfg.bbox, "dichotomy", 0))
seeds = r.seeds


def seed_only():
    eng.reset()
    marching.seed_engine(eng, seeds)


t("reset + seed 64", seed_only)
t("reset only", lambda: eng.reset())
import cProfile  # noqa: E402
import pstats  # noqa: E402
cProfile.run("for _ in range(50): seeding.sample_seeds(eng, 64, cfg.bbox, 'dichotomy', 0)", "/tmp/ss.prof")
pstats.Stats("/tmp/ss.prof").sort_stats("tottime").print_stats(15)

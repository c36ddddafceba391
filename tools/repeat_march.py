"""Repeat the configs[1] march N times in one process (cached engine, as march() does) and report
every run whose visited set differs from the oracle's; the differing keys are saved."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
from paper_2106_10031_b200 import MarchConfig, march, synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
net = synth.geometric_mlp([90] * 6, seed=0)
r = march(net, MarchConfig(seeds=64, rng_seed=0))
o = oracle.march(net, seed_points=r.seeds, threads=os.cpu_count())
ref = {k.tobytes(): i for i, k in enumerate(o.keys)}
print("oracle", len(ref), "AM_NARROW", os.environ.get("AM_NARROW"), flush=True)
bad = 0
for it in range(N):
    r = march(net, MarchConfig(seeds=64, rng_seed=0))
    got = {k.tobytes(): i for i, k in enumerate(r.keys)}
    extra = [k for k in got if k not in ref]
    miss = [k for k in ref if k not in got]
    same_poly = True
    if not extra and not miss:
        same_poly = np.array_equal(r.nverts, o.nverts) and np.abs(r.verts - o.verts).max() <= 1e-9
    print(it, len(got), "extra", len(extra), "missing", len(miss), "polys", same_poly, flush=True)
    if extra or miss or not same_poly:
        bad += 1
        np.savez(os.path.join(REPO, "gpurun_out", f"bad_{os.environ.get('AM_NARROW', 'd')}_{it}.npz"),
                 extra=np.array([np.frombuffer(k, np.uint8) for k in extra]).reshape(-1, 68),
                 miss=np.array([np.frombuffer(k, np.uint8) for k in miss]).reshape(-1, 68),
                 )
print("bad runs", bad, "of", N)

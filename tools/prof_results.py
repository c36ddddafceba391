"""Per-kernel device times of result assembly (am_result_copy_device) after a configs[1] march.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/prof_results.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth  # noqa: E402

net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
r = marching.march(net, cfg)
eng = next(iter(marching._ENGINES.values()))
for _ in range(3):
    eng.results_device()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    eng.results_device()
torch.cuda.synchronize()
print(f"results_device {1e3 * (time.perf_counter() - t) / 5:.3f} ms")
torch.cuda.cudart().cudaProfilerStart()
eng.results_device()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()

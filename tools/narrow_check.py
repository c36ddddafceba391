"""AM_NARROW_CHECK=1: every iteration compares the fused narrow composition with the per-step path."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["AM_NARROW_CHECK"] = "1"
from paper_2106_10031_b200 import synth
from paper_2106_10031_b200.engine import Engine
from paper_2106_10031_b200.seeding import sample_seeds
net = synth.geometric_mlp([90] * 6, seed=0)
eng = Engine(net)
seeds = sample_seeds(eng, 64, ((-1.2,) * 3, (1.2,) * 3), rng_seed=0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    eng.reset(); eng.seed(seeds); it = eng.run()
    d = np.zeros(64, dtype=np.uint64)
    eng.lib.am_debug_counters(eng.h, d.ctypes.data)
    print(rep, eng.counts()["cells"], "Z mismatches", d[56], "faces", d[57], "keys", d[58], "changed", d[59],
          "first item", d[61], "rem", d[62], "diff", np.array([d[63]]).view(np.float64)[0], flush=True)

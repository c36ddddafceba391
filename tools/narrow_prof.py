"""Phase cycle counters of k_compose_narrow (AM_NARROW_DBG=8): thread 0 of every CTA, summed."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["AM_NARROW_DBG"] = str(int(os.environ.get("AM_NARROW_DBG", "0")) | 8)
from paper_2106_10031_b200 import synth
from paper_2106_10031_b200.engine import Engine
from paper_2106_10031_b200.seeding import sample_seeds
net = synth.geometric_mlp([90] * 6, seed=0)
eng = Engine(net)
seeds = sample_seeds(eng, 64, ((-1.2,) * 3, (1.2,) * 3), rng_seed=0)
d = np.zeros(64, dtype=np.uint64)
eng.lib.am_debug_counters(eng.h, d.ctypes.data)
eng.reset(); eng.seed(seeds); eng.run()
eng.lib.am_debug_counters(eng.h, d.ctypes.data)
tiles = float(d[39])
names = ["gather", "step0", "kloop", "epilogue", "head", "keys-out+bar", "layer-bar-wait", "tiles", "box-wait(in kloop)"]
print("tiles", tiles, {n: round(float(d[32 + i]) / tiles) for i, n in enumerate(names)}, "cycles per tile")

"""Stage timing of bench.py's configs[4] call: march_batch(64 latent DeepSDF shapes, max_cells 20 k)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import batch, marching, synth, seeding  # noqa: E402
from paper_2106_10031_b200 import engine as engmod  # noqa: E402

T = {}


def wrap(mod, name, key=None):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[key or name] = T.get(key or name, 0.0) + (time.perf_counter() - t) * 1e3
        return r
    setattr(mod, name, g)


for mod, name in [(batch, "_fused_engine"), (batch, "split_batch_result"), (batch, "seed_engine"),
                  (seeding, "sample_seeds_batch"), (marching, "device_results_to_host")]:
    wrap(mod, name)
wrap(engmod.Engine, "run", "eng.run")
wrap(engmod.Engine, "forward", "eng.forward")
wrap(engmod.Engine, "dichotomy", "eng.dichotomy")
nets, _ = synth.latent_batch(n_shapes=64, latent_dim=256, width=512, depth=8, skip_at=4, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3), max_cells=20000)
for rep in range(3):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = batch.march_batch(nets, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    cells = sum(r.report.cells_visited for _, r in res)
    print(f"rep {rep}: {dt * 1e3:.0f} ms, {cells} cells, waves {res[0][1].report.waves} | "
          + " ".join(f"{k} {v:.0f}" for k, v in T.items()), flush=True)

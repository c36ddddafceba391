"""configs[4] fused latent batch (64 shapes, 20k cells each) + configs[2] first 1M cells: wall time
under the current environment knobs (A/B helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10031_b200 import marching, synth  # noqa: E402
from paper_2106_10031_b200.batch import march_batch  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds  # noqa: E402

bbox = ((-1.2,) * 3, (1.2,) * 3)
lnets, _ = synth.latent_batch(n_shapes=64, latent_dim=256, width=512, depth=8, skip_at=4, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, max_cells=20_000)
march_batch(lnets, cfg)
ts = []
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = march_batch(lnets, cfg)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
print("configs[4]", os.environ.get("TAG", ""), [round(x, 3) for x in ts], sum(x.report.cells_visited for _, x in r))
marching.clear_engine_cache()
dnet = synth.deepsdf_mlp(512, 8, 4, seed=0)
eng = Engine(dnet, bbox=bbox, max_cells=1_000_000)
seeds = torch.as_tensor(sample_seeds(eng, 64, bbox, rng_seed=0), device="cuda")
for i in range(3):
    eng.reset()
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.seed(seeds)
    it = eng.run()
    torch.cuda.synchronize()
    if i:
        print("configs[2] 1M", os.environ.get("TAG", ""), round(time.perf_counter() - t, 4), it)

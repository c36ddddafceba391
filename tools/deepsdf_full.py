"""Device time of the complete DeepSDF 3-(512x8)-1 march (configs[2], ~16 M cells) for a few
engine batch sizes / environment variants.

    python tools/deepsdf_full.py [--batch 16384 32768] [--width 512]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, nargs="+", default=[0])
ap.add_argument("--width", type=int, default=512)
ap.add_argument("--max-cells", type=int, default=40_000_000)
a = ap.parse_args()
net = synth.deepsdf_mlp(a.width, 8, 4, seed=0)
bbox = ((-1.2,) * 3, (1.2,) * 3)
for bc in a.batch:
    eng = Engine(net, bbox=bbox, max_cells=a.max_cells, batch_cells=bc)
    seeds = torch.as_tensor(sample_seeds(eng, 64, bbox, rng_seed=0), device="cuda")

    def run():
        eng.reset()
        eng.seed(seeds)
        return eng.run()
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    waves = run()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c = eng.counts()
    st = eng.stats()
    print(f"batch {bc or eng.batch_size}: cells {c['cells']} waves {waves} {ms:.1f} ms = {c['cells'] / ms * 1e-3:.3f} M cells/s"
          f"  skipped flops {st['prefix_skipped_flops']:.3e}", flush=True)
    del eng
    torch.cuda.empty_cache()

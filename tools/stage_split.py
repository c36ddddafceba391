"""Timing-mode stage split (am_kernel_times) of a march: python tools/stage_split.py [geo90x6|deepsdf512] [max_cells]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "geo90x6"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
net = synth.geometric_mlp([90] * 6, seed=0) if which == "geo90x6" else synth.deepsdf_mlp(512, 8, 4, seed=0)
eng = Engine(net, max_cells=cap)
seeds = torch.as_tensor(sample_seeds(eng, 64, ((-1.2,) * 3, (1.2,) * 3), rng_seed=0), device="cuda")
eng.reset(); eng.seed(seeds); eng.run()
eng.set_timing(True)
eng.reset(); eng.seed(seeds); eng.run()
kt = eng.kernel_times()
tot = sum(kt["ms"].values())
print(which, {k: f"{v:.1f} ({v / tot:.0%})" for k, v in kt["ms"].items()}, f"sum {tot:.1f} ms", kt["iterations"], "iterations")

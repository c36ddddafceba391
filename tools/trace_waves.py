import os, sys
sys.path.insert(0, "/root/repo")
os.environ["AM_TRACE_ITERS"] = "1"
import torch
from paper_2106_10031_b200 import marching, synth
from paper_2106_10031_b200.engine import Engine
from paper_2106_10031_b200.seeding import sample_seeds
net = synth.geometric_mlp([90] * 6, seed=0)
eng = Engine(net)
seeds = torch.as_tensor(sample_seeds(eng, 64, ((-1.2,) * 3, (1.2,) * 3), rng_seed=0), device="cuda")
eng.set_timing(True)
eng.reset(); eng.seed(seeds); eng.run()

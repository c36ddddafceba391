"""Breakdown of collect_result on configs[1]: device sort + gathers, conversions, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_10031_b200 import marching, synth
from paper_2106_10031_b200.meshes import to_host
net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3))
for _ in range(3):
    r = marching.march(net, cfg)
eng = marching._engine_for(net, cfg)
for rep in range(4):
    eng.reset(); eng.seed(r.seeds); eng.run(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    c, keys, nverts, verts, enr, erefs = eng.results_device(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng.reset(); eng.seed(r.seeds); eng.run(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = marching.device_results_to_host(eng); torch.cuda.synchronize()
    t3 = time.perf_counter()
    hs = to_host([keys, nverts, verts, enr, erefs])
    t4 = time.perf_counter()
    print(f"results_device {1e3*(t1-t0):.2f} ms | device_results_to_host (all) {1e3*(t3-t2):.2f} ms | to_host raw {1e3*(t4-t3):.2f} ms "
          f"({sum(x.nbytes for x in hs)/1e6:.1f} MB)")

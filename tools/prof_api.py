import cProfile, pstats, sys, time, io
sys.path.insert(0, '.')
import torch
from paper_2106_10031_b200 import synth, marching
net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0)
marching.march(net, cfg).welded_mesh()
for i in range(2):
    t0 = time.perf_counter(); r = marching.march(net, cfg); t1 = time.perf_counter(); m = r.welded_mesh(); t2 = time.perf_counter()
    print(f"march {1e3*(t1-t0):.1f} ms weld {1e3*(t2-t1):.1f} ms")
pr = cProfile.Profile(); pr.enable()
r = marching.march(net, cfg); m = r.welded_mesh()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats('cumulative').print_stats(30); print(s.getvalue()[:6000])

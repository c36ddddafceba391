"""Stage timing of the COLD first march() of a process (after one unrelated engine warmed the CUDA
context, as in bench.py): engine creation, trigger, BFS, results (incl. first-time pinning)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2106_10031_b200 import engine as engmod, marching, meshes, synth  # noqa: E402

T = {}


def wrap(obj, name, key=None):
    f = getattr(obj, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[key or name] = T.get(key or name, 0.0) + (time.perf_counter() - t) * 1e3
        return r
    setattr(obj, name, g)


for mod, name in [(marching, "_engine_for"), (marching, "sample_seeds"), (marching, "collect_result"),
                  (marching, "device_results_to_host"), (meshes, "to_host"), (meshes, "weld_device")]:
    wrap(mod, name)
for name in ["seed", "run", "results_device"]:
    wrap(engmod.Engine, name, "eng." + name)
net = synth.geometric_mlp([90] * 6, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0)
warm = engmod.Engine(synth.geometric_mlp([90] * 6, seed=1))   # CUDA context + kernels loaded
torch.cuda.synchronize()
for rep in range(3):
    T.clear()
    t0 = time.perf_counter()
    r = marching.march(net, cfg)
    t1 = time.perf_counter()
    r.welded_mesh()
    t2 = time.perf_counter()
    print(f"call {rep}: march {1e3 * (t1 - t0):.1f} ms, welded_mesh {1e3 * (t2 - t1):.1f} ms | "
          + " ".join(f"{k} {v:.1f}" for k, v in T.items()), flush=True)

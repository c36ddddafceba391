"""Composition-GEMM microbenchmark: one full batch of real activation states through
am_affine_maps (every hidden layer as W_l x [n_l x 4B] on DMMA + the head), timed with CUDA
events on the engine stream.  Used for tuning k_gemm_step and for its ncu capture.

    python tools/bench_compose.py [--net deepsdf512|geo90x6] [--cells 15264] [--repeat 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="deepsdf512")
ap.add_argument("--cells", type=int, default=15264)
ap.add_argument("--repeat", type=int, default=10)
a = ap.parse_args()
net = synth.geometric_mlp([90] * 6, seed=0) if a.net == "geo90x6" else synth.deepsdf_mlp(512, 8, 4, seed=0)
eng = Engine(net, batch_cells=a.cells)
g = torch.Generator(device="cpu").manual_seed(0)
pts = (torch.rand((a.cells, 3), generator=g, dtype=torch.float64) * 2.4 - 1.2).to("cuda")
_, keys = eng.forward(pts, keys=True)
fpc = eng.stats()["flops_per_cell"]
faces = torch.empty((a.cells, eng.blob.n_subs, 4), dtype=torch.float64, device="cuda")


def compose():   # planes stay in the engine's Z buffer: no 32 B x rows x cells copy-out
    eng.lib.am_affine_maps(eng.h, keys.data_ptr(), a.cells, None, None, faces.data_ptr())


compose()   # warm-up (tensor maps, attributes)
torch.cuda.synchronize()
s = eng.stream
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = float("inf")
for _ in range(a.repeat):
    t0.record(s)
    compose()
    t1.record(s)
    t1.synchronize()
    best = min(best, t0.elapsed_time(t1))
tf = fpc * a.cells / (best * 1e-3) / 1e12
print(f"{a.net}: {a.cells} cells, affine_maps {best * 1e3:.1f} us, {tf:.2f} TFLOP/s fp64 "
      f"({fpc / 1e6:.2f} MFLOP/cell)")

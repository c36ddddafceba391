"""One configs[1] march for profiling (ncu launch list / --set full on one kernel).

    python tools/profile_march.py [--net geo90x6|deepsdf512] [--seeds 64] [--max-cells N]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.engine import Engine  # noqa: E402
from paper_2106_10031_b200.seeding import sample_seeds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="geo90x6")
ap.add_argument("--seeds", type=int, default=64)
ap.add_argument("--max-cells", type=int, default=10_000_000)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
net = synth.geometric_mlp([90] * 6, seed=0) if a.net == "geo90x6" else synth.deepsdf_mlp(512, 8, 4, seed=0)
eng = Engine(net, max_cells=a.max_cells)
seeds = torch.as_tensor(sample_seeds(eng, a.seeds, ((-1.2,) * 3, (1.2,) * 3), rng_seed=0), device="cuda")
eng.set_timing(a.timing)
for _ in range(a.repeat):
    eng.reset()
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.seed(seeds)
    it = eng.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    c = eng.counts()
    print(f"{a.net}: {c['cells']} cells, {it} iterations, {dt * 1e3:.1f} ms, {c['cells'] / dt:.0f} cells/s")
print({k: round(v, 3) for k, v in eng.stats().items()})
import numpy as np  # noqa: E402
d = np.zeros(64, dtype=np.uint64)
eng.lib.am_debug_counters(eng.h, d.ctypes.data)
if d[0]:
    n = float(d[0])
    print(f"face stats: cells {int(n)} clips1 {d[1]/n:.2f} clips2 {d[2]/n:.2f} C' {d[3]/n:.2f} raw verts {d[4]/n:.2f} "
          f"verts {d[5]/n:.2f} cycles {d[6]/n:.0f} (max {int(d[8])}) hinted {d[7]/n:.2f}")
    print(f"hint: have {d[13]/n:.3f} x0-violates {d[9]/n:.3f} near>NMAX {d[10]/n:.3f} reach-fail {d[11]/n:.3f} "
          f"near rows {d[12]/max(1, d[13]):.1f} | near list used {d[14]/n:.3f} overflow {d[15]/n:.4f}")
    print("cycle histogram (log2, from 2^14):", {int(2**(i + 14)): int(d[16 + i]) for i in range(8) if d[16 + i]})
if d[0]:
    names = ["setup", "stream", "near-rows", "clip", "accept+C'", "full-path", "pairs", "dedup", "order", "edges",
             "emit-count", "emit-records", "emit-keys"]
    tot = sum(float(d[40 + i]) for i in range(13))
    print("phase cycles per cell:", {nm: round(float(d[40 + i]) / n) for i, nm in enumerate(names)},
          f"sum {tot / n:.0f}")
if d[0]:
    cls = ["list-1", "list-retry", "streamed", "full-path"]
    print("path classes (cells, mean cycles):", {c: (int(d[24 + i]), round(float(d[28 + i]) / max(1, int(d[24 + i]))))
                                                for i, c in enumerate(cls)},
          "| cells > 100k cycles:", {c: int(d[32 + i]) for i, c in enumerate(cls)},
          "| full-path reasons (no hint, x0 violates, near > NMAX, attempts):", [int(d[36 + i]) for i in range(4)])
if d[0]:
    print("failed hinted attempts: empty", int(d[53]), "vertex overflow", int(d[54]), "reach", int(d[55]))

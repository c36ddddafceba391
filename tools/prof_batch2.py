"""Timing-mode stage split and prefix statistics of the fused configs[4] batch march."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2106_10031_b200 import batch, marching, synth  # noqa: E402

nets, _ = synth.latent_batch(n_shapes=64, latent_dim=256, width=512, depth=8, skip_at=4, seed=0)
cfg = marching.MarchConfig(seeds=64, rng_seed=0, bbox=((-1.2,) * 3, (1.2,) * 3), max_cells=20000)
batch.march_fused(nets, cfg)
eng = next(iter(marching._ENGINES.values()))
eng.set_timing(True)
batch.march_fused(nets, cfg)
kt = eng.kernel_times()
st = eng.stats()
eng.set_timing(False)
tot = sum(kt["ms"].values())
print({k: f"{v:.1f}" for k, v in kt["ms"].items()}, f"sum {tot:.1f} ms", kt["iterations"], "iterations")
print("batch", st["batch"], "composed", kt["composed"], "prefix", st["prefix"], "skipped flops", f"{st['prefix_skipped_flops']:.3e}",
      "flops/cell", st["flops_per_cell"])
c = eng.counts()
print(c)
print({k: st[k] for k in ("probes", "probes_forwarded", "probe_records", "probe_ms", "launches")})

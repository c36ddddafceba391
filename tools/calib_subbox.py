"""Cell counts of the configs[2] / configs[3] sub-box marches for several box sizes (sizes the
parity tests in tests/test_gpu_parity_configs.py)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from test_gpu_parity_configs import _surface_box  # noqa: E402
from paper_2106_10031_b200 import MarchConfig, march, synth  # noqa: E402

nets = {"deepsdf": synth.deepsdf_mlp(width=512, depth=8, skip_at=4, seed=0),
        "imnet": synth.imnet_ensemble(widths=(128, 128, 128), n_parts=4, seed=0)}
for name, net in nets.items():
    for half in (0.02, 0.035, 0.05, 0.1, 0.2):
        bbox, p = _surface_box(net, (0.3, 0.5, 0.8), half)
        t = time.perf_counter()
        r = march(net, MarchConfig(bbox=bbox, seed_points=p[None], max_cells=2_000_000))
        print(name, half, r.report.cells_visited, r.report.faces_emitted, r.report.capped,
              f"{time.perf_counter() - t:.2f}s", flush=True)

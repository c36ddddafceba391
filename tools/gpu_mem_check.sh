#!/bin/bash
# march time + peak device memory of the engine for configs[1] and the DeepSDF 1M-cell sample
O=gpurun_out
python - > $O/mem.log 2>&1 <<'PY'
import torch, time, sys
sys.path.insert(0, ".")
from paper_2106_10031_b200 import synth
from paper_2106_10031_b200.engine import Engine
from paper_2106_10031_b200.seeding import sample_seeds
bbox = ((-1.2,) * 3, (1.2,) * 3)
for name, net, cap in [("geo90x6", synth.geometric_mlp([90] * 6, seed=0), 10_000_000),
                       ("deepsdf1M", synth.deepsdf_mlp(512, 8, 4, seed=0), 1_000_000)]:
    torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats()
    free0 = torch.cuda.mem_get_info()[0]
    eng = Engine(net, bbox=bbox, max_cells=cap)
    seeds = torch.as_tensor(sample_seeds(eng, 64, bbox, rng_seed=0), device="cuda")
    ts = []
    for _ in range(4):
        eng.reset(); eng.seed(seeds)
        torch.cuda.synchronize(); t = time.perf_counter()
        w = eng.run(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    used = (free0 - torch.cuda.mem_get_info()[0]) / 2**30
    print(f"{name}: cells {eng.counts()['cells']} waves {w} ms {[round(1e3*x,1) for x in ts]} device memory used {used:.2f} GiB")
    del eng
PY
cat $O/mem.log

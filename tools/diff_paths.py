"""Diff the configs[1] visited sets of two engine paths (AM_NARROW=1 vs 0): run in two processes,
save keys/nverts, then compare and describe the differing cells with the oracle."""
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

if len(sys.argv) > 1 and sys.argv[1] == "run":
    from paper_2106_10031_b200 import MarchConfig, march, synth
    net = synth.geometric_mlp([90] * 6, seed=0)
    r = march(net, MarchConfig(seeds=64, rng_seed=0))
    np.savez(sys.argv[2], keys=r.keys, nverts=r.nverts, seeds=r.seeds)
    sys.exit(0)

out = os.path.join(REPO, "gpurun_out")
for v in ("1", "0"):
    subprocess.run([sys.executable, __file__, "run", f"{out}/paths_{v}.npz"], env=dict(os.environ, AM_NARROW=v),
                   check=True)
a, b = np.load(f"{out}/paths_1.npz"), np.load(f"{out}/paths_0.npz")
ka = {k.tobytes(): i for i, k in enumerate(a["keys"])}
kb = {k.tobytes(): i for i, k in enumerate(b["keys"])}
print("narrow", len(ka), "per-step", len(kb))
import oracle  # noqa: E402
from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.evaluate import packbits_to_words  # noqa: E402
net = synth.geometric_mlp([90] * 6, seed=0)
on = oracle.OracleNet(net)
for name, s, other in (("only narrow", ka, kb), ("only per-step", kb, ka)):
    for k, i in s.items():
        if k in other:
            continue
        w = packbits_to_words(np.frombuffer(k, np.uint8)[None], None, 540).view(np.uint64)[0]
        canon, planes, face = on.affine_maps(w)
        nrm = np.linalg.norm(planes[:, :3], axis=1)
        print(name, "cell", i, "nverts", (a if s is ka else b)["nverts"][i], "canon==key", np.array_equal(canon, w),
              "min|n|", nrm.min(), "n<1e-9:", int((nrm < 1e-9).sum()), "face", face)
        # its neighbours by single flips that are in both sets
        bits = np.unpackbits(np.frombuffer(k, np.uint8))[:540]
        nb = 0
        for j in range(540):
            bb = bits.copy(); bb[j] ^= 1
            kk = np.packbits(bb).tobytes()
            if kk in other:
                nb += 1
                if nb <= 5:
                    print("   flip", j, "-> present in other set")
        print("   flip-neighbours in other set:", nb)

"""Digest of the UNMODIFIED reference's march on a full benchmark configuration.

The headline set (configs[1]: 3-(90x6)-1 geometric init, 64 dichotomy seeds,
full default box, 234 k cells) is too large to commit as a fixture, so this
script runs the reference (CPU, single thread, ~30-60 min) and commits a
digest instead: the seeds, the cell count, sha256 of the sorted packbits keys
(reference sort order, marching.py:346-349, empty cells included), sha256 of
the per-cell vertex counts and of the edge transition refs, and vertex sums.
``tests/test_gpu_parity.py`` pins both the GPU march and the CPU oracle to it.

    python tests/golden/make_digest.py configs1
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (reference import + empty-state capture)


def digest_arrays(keys, branch, nverts, verts, edge_nrefs, edge_refs) -> dict:
    """The committed digest of one march in the reference's sorted representation."""
    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    verts = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    return {
        "cells": int(len(nverts)),
        "faces": int((np.asarray(nverts) > 0).sum()),
        "keys_sha256": sha(np.asarray(keys, dtype=np.uint8)),
        "branch_sha256": sha(np.asarray(branch, dtype=np.int64)),
        "nverts_sha256": sha(np.asarray(nverts, dtype=np.int64)),
        "edge_nrefs_sha256": sha(np.asarray(edge_nrefs, dtype=np.int64)),
        "edge_refs_sha256": sha(np.asarray(edge_refs, dtype=np.int64).reshape(-1, 2)),
        "n_verts": int(len(verts)),
        "vert_sum": [float(x) for x in verts.sum(axis=0)],
        "vert_abs_sum": float(np.abs(verts).sum()),
    }


def cases():
    from paper_2106_10031_b200 import synth
    return {
        # configs[1]: the benchmarked march (bench.py workload)
        "configs1": (lambda p: mg.via_json(synth.geometric_mlp([90] * 6, seed=0), p),
                     dict(seeds=64, rng_seed=0)),
    }


def run(name, builder, kw):
    jpath = os.path.join(HERE, f"digest_{name}.net.json")
    net = builder(jpath)
    os.remove(jpath)   # the network is rebuilt from synth in the tests
    cfg = mg.MarchConfig(**kw)
    seeds = mg.sample_seeds(net, cfg.seeds, cfg.bbox, scheme=cfg.scheme, rng_seed=cfg.rng_seed)
    cfg.seed_points = seeds
    t0 = time.perf_counter()
    res = mg.march(net, cfg)
    dt = time.perf_counter() - t0
    polys = {(p.state.key, p.state.branch): p for p in res.polygons}
    states = sorted(set(polys) | set(mg._empty_states(net, cfg, res)),
                    key=lambda kb: (kb[0], -1 if kb[1] is None else kb[1]))
    keys, branch, nverts, verts, enr, erefs = [], [], [], [], [], []
    for k, b in states:
        keys.append(np.frombuffer(k, dtype=np.uint8))
        branch.append(-1 if b is None else b)
        p = polys.get((k, b))
        if p is None:
            nverts.append(0)
            continue
        nverts.append(p.n_vertices)
        verts.append(p.vertices)
        for refs in p.edge_transitions:
            enr.append(len(refs))
            erefs.extend((r.kind, r.index) for r in refs)
    doc = digest_arrays(np.stack(keys), branch, nverts, np.concatenate(verts), enr, erefs)
    doc.update({
        "config": {"net": "synth.geometric_mlp([90]*6, seed=0)", "seeds": cfg.seeds,
                   "rng_seed": cfg.rng_seed, "scheme": cfg.scheme,
                   "bbox": [list(cfg.bbox[0]), list(cfg.bbox[1])]},
        "seeds": seeds.tolist(),
        "report": json.loads(res.report.to_json()),
        "reference_seconds": dt,
    })
    with open(os.path.join(HERE, f"digest_{name}.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print(f"{name}: {doc['cells']} cells, {doc['faces']} faces in {dt:.0f}s")


if __name__ == "__main__":
    mg._patch_marcher()
    want = set(sys.argv[1:])
    for name, (builder, kw) in cases().items():
        if want and name not in want:
            continue
        run(name, builder, kw)

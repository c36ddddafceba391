"""fp64 vs fp32-mode tolerance study (BASELINE configs[3]: IM-NET-style max-pool occupancy MLP).

fp64 = the reference arithmetic (bit-exact visited set).  fp32 mode = fp32-precision planes:
weights and every composed affine map rounded to fp32 (csrc prec_round).  For a sweep of
tolerance sets the fp32-mode march is compared with the fp64 one: visited-set agreement,
polygon agreement and vertex deviation on the cells both visit, and watertightness of the
welded mesh (boundary edges away from the box).

    python tools/fp32_study.py [--out profiles/r01_fp32_study.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2106_10031_b200 import synth  # noqa: E402
from paper_2106_10031_b200.marching import MarchConfig, clear_engine_cache, march  # noqa: E402
from paper_2106_10031_b200.meshes import topology_check, triangulate  # noqa: E402

TOLS = {   # name -> (tol_cell, tol_weld, probe_delta)
    "fp64-tols": (1e-9, 1e-7, 1e-7),
    "cell1e-9_weld1e-6": (1e-9, 1e-6, 1e-7),
    "1e-7": (1e-7, 1e-6, 1e-6),
    "1e-6": (1e-6, 1e-5, 1e-5),
    "1e-5": (1e-5, 1e-4, 1e-4),
}


def polys(res):
    keys = [k.tobytes() + int(b).to_bytes(8, "little", signed=True) for k, b in zip(res.keys, res.branch)]
    off = np.concatenate([[0], np.cumsum(np.maximum(res.nverts, 0))])
    return {k: res.verts[off[i]:off[i + 1]] for i, k in enumerate(keys)}, keys


def mesh_stats(res, tol_weld):
    m = res.welded_mesh(tol_weld)
    t = topology_check(triangulate(m))
    return {"mesh_vertices": m.n_vertices, "mesh_faces": m.n_faces, "boundary_edges": t.get("open_edges"),
            "nonmanifold_edges": t.get("nonmanifold_edges"), "watertight": t.get("watertight")}


def study(name, net, bbox, seeds=64):
    base_cfg = MarchConfig(bbox=bbox, seeds=seeds, rng_seed=0)
    t = time.perf_counter()
    ref = march(net, base_cfg)
    ref_s = time.perf_counter() - t
    P_ref, K_ref = polys(ref)
    out = {"network": name, "fp64": {"cells": ref.report.cells_visited, "faces": ref.report.faces_emitted,
                                     "open_edges": ref.report.open_edges, "seconds": ref_s,
                                     **mesh_stats(ref, 1e-7), "mesh_weld_1e-05": mesh_stats(ref, 1e-5)}, "fp32": {}}
    for tname, (tc, tw, pd) in TOLS.items():
        cfg = MarchConfig(bbox=bbox, seeds=seeds, rng_seed=0, precision="fp32", tol_cell=tc, tol_weld=tw,
                          probe_delta=pd)
        t = time.perf_counter()
        try:
            r = march(net, cfg)
        except Exception as exc:   # noqa: BLE001 -- record failures of a tolerance set in the study
            out["fp32"][tname] = {"error": str(exc)[:200]}
            continue
        dt = time.perf_counter() - t
        P, K = polys(r)
        a, b = set(K_ref), set(K)
        common = a & b
        same_n, dev = 0, []
        for k in common:
            p, q = P_ref[k], P[k]
            if len(p) == len(q):
                same_n += 1
                if len(p):
                    dev.append(float(np.abs(p - q).max()))
        dev = np.array(dev) if dev else np.zeros(1)
        out["fp32"][tname] = {
            "tol_cell": tc, "tol_weld": tw, "probe_delta": pd, "cells": r.report.cells_visited,
            "jaccard": len(common) / max(len(a | b), 1), "missing": len(a - b), "extra": len(b - a),
            "same_vertex_count": same_n / max(len(common), 1),
            "vertex_dev_max": float(dev.max()), "vertex_dev_p99": float(np.quantile(dev, 0.99)),
            "vertex_dev_median": float(np.median(dev)), "open_edges": r.report.open_edges, "seconds": dt,
            **mesh_stats(r, tw)}
        for mw in (1e-6, 1e-5):   # mesh assembly with a looser weld radius than the march's dedup
            out["fp32"][tname][f"mesh_weld_{mw:g}"] = mesh_stats(r, mw)
        clear_engine_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    box = ((-1.2,) * 3, (1.2,) * 3)
    rows = [study("configs[3] IM-NET-style occupancy max-pool of 4 parts, 3-(128x3)-1 each",
                  synth.imnet_ensemble(widths=(128, 128, 128), n_parts=4, seed=0), box),
            study("configs[1] 3-(90x6)-1 SAL sphere init", synth.geometric_mlp([90] * 6, seed=0), box)]
    txt = json.dumps(rows, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(txt + "\n")


if __name__ == "__main__":
    main()

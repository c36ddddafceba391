"""Golden fixtures for mesh welding, made by running the UNMODIFIED reference
``exactmesh.meshes.weld`` (reference meshes.py:89-148) here, where the reference is mounted:

    python tests/golden/make_weld_golden.py

``weld_<name>.npz`` holds the input soup (``verts``, CSR loops ``loop_off`` / ``loop_idx``,
``tol``) and the reference output (``kept`` vertices, CSR ``face_off`` / ``face_idx``,
``dropped``).  Inputs: the polygon soups of golden marches (the reference's own
``MarchResult.polygon_soup`` order, rebuilt from the committed march fixtures) and adversarial
synthetic soups -- tight clusters, chains of points spaced 0.6-1.4 tol apart (greedy order
matters), loops that collapse, exact duplicates with signed zeros for tol = 0.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from exactmesh.meshes import PolygonMesh, weld  # noqa: E402  (the reference)


def soup_from_golden(name):
    d = np.load(os.path.join(HERE, f"{name}.npz"))
    nv = d["nverts"]
    off = np.concatenate([[0], np.cumsum(nv[nv > 0])]).astype(np.int64)
    return d["verts"], off, np.arange(off[-1], dtype=np.int64)


def synthetic(seed, tol, n_clusters=300, spread=0.3):
    rng = np.random.default_rng(seed)
    pts = []
    for _ in range(n_clusters):
        c = rng.uniform(-1, 1, 3)
        kind = rng.integers(0, 4)
        if kind == 0:      # tight duplicates
            m = rng.integers(1, 7)
            pts += [c + rng.normal(scale=spread * tol, size=3) for _ in range(m)]
        elif kind == 1:    # chain spaced 0.6..1.4 tol: greedy order decides
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            x = c.copy()
            for _ in range(rng.integers(2, 8)):
                pts.append(x.copy())
                x = x + d * tol * rng.uniform(0.6, 1.4)
        elif kind == 2:    # ring around a centre within ~tol
            for _ in range(rng.integers(3, 9)):
                u = rng.normal(size=3)
                pts.append(c + u / np.linalg.norm(u) * tol * rng.uniform(0.3, 1.1))
        else:              # isolated
            pts.append(c)
    pts = np.array(pts)
    perm = rng.permutation(len(pts))
    pts = pts[perm]
    # loops: random walks over nearby indices (some collapse after welding)
    loops, off = [], [0]
    for _ in range(len(pts) // 2):
        k = int(rng.integers(3, 8))
        start = int(rng.integers(0, len(pts)))
        idx = [(start + int(j)) % len(pts) for j in np.cumsum(rng.integers(0, 3, size=k))]
        loops += idx
        off.append(len(loops))
    return pts, np.array(off, np.int64), np.array(loops, np.int64)


def signed_zero_case():
    rng = np.random.default_rng(5)
    base = rng.uniform(-1, 1, (40, 3))
    base[::5, 0] = 0.0
    pts = np.concatenate([base, base[::2], base[::3]])
    pts[len(base):, 0] = np.where(pts[len(base):, 0] == 0.0, -0.0, pts[len(base):, 0])
    pts = pts[rng.permutation(len(pts))]
    off = np.arange(0, len(pts) - len(pts) % 4 + 1, 4, dtype=np.int64)
    return pts, off, np.arange(off[-1], dtype=np.int64)


def run(name, verts, off, idx, tol):
    mesh = PolygonMesh(verts, [idx[off[i]:off[i + 1]] for i in range(len(off) - 1)], None)
    out = weld(mesh, tol)
    foff = np.concatenate([[0], np.cumsum([len(f) for f in out.faces])]).astype(np.int64)
    fidx = np.concatenate(out.faces).astype(np.int64) if out.faces else np.zeros(0, np.int64)
    np.savez_compressed(os.path.join(HERE, f"weld_{name}.npz"), verts=verts, loop_off=off, loop_idx=idx,
                        tol=np.float64(tol), kept=out.vertices, face_off=foff, face_idx=fidx,
                        dropped=np.int64(out.dropped_faces))
    print(f"weld_{name}: {len(verts)} verts -> {out.n_vertices}, {len(off) - 1} loops -> {out.n_faces} "
          f"(dropped {out.dropped_faces})")


if __name__ == "__main__":
    for g in ("oct", "rand_4x12_s13", "imnet_small", "deepsdf_small"):
        run(f"soup_{g}", *soup_from_golden(g), 1e-7)
    run("syn_tol1e-7", *synthetic(1, 1e-7), 1e-7)
    run("syn_tol5e-2", *synthetic(2, 5e-2, n_clusters=120), 5e-2)
    run("syn_tol1e-3", *synthetic(3, 1e-3, n_clusters=400, spread=0.6), 1e-3)
    run("exact_tol0", *signed_zero_case(), 0.0)

"""Mesh welding (reference meshes.py:89-148): the oracle restatement pinned against the
reference's own outputs (tests/golden/weld_*.npz, made by tests/golden/make_weld_golden.py),
then the GPU weld (am_weld) against both -- bit-exact: welding selects and copies vertices and
rewrites indices, it computes no new floating-point values."""

import glob
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(HERE, "golden", "weld_*.npz")))


def load(name):
    return dict(np.load(os.path.join(HERE, "golden", f"weld_{name}.npz")))


def test_weld_fixtures_present():
    assert len(CASES) >= 8


@pytest.mark.parametrize("name", CASES)
def test_oracle_weld_matches_reference(name):
    g = load(name)
    kept, foff, fidx, fsrc, remap, dropped = oracle.weld(g["verts"], g["loop_off"], g["loop_idx"], float(g["tol"]))
    np.testing.assert_array_equal(kept, g["kept"])
    np.testing.assert_array_equal(foff, g["face_off"])
    np.testing.assert_array_equal(fidx, g["face_idx"])
    assert dropped == int(g["dropped"])
    # remap against the reference's contract (meshes.py:89-148): every vertex lands on a kept
    # vertex within tol (exactly equal at tol = 0), representatives are first occurrences (the
    # first vertex mapped to kept j IS kept j, and kept indices appear in first-occurrence order)
    v = np.asarray(g["verts"], dtype=np.float64)
    assert remap.shape == (len(v),) and remap.min(initial=0) >= 0 and remap.max(initial=-1) < len(kept)
    d = np.linalg.norm(v - kept[remap], axis=1)
    assert (d <= float(g["tol"])).all() if float(g["tol"]) > 0 else (v == kept[remap]).all()
    first = np.full(len(kept), -1)
    for i in range(len(v) - 1, -1, -1):
        first[remap[i]] = i
    np.testing.assert_array_equal(v[first], kept)
    assert (np.diff(first) > 0).all()


def test_oracle_weld_is_idempotent():
    g = load("syn_tol1e-3")
    kept, foff, fidx, *_ = oracle.weld(g["verts"], g["loop_off"], g["loop_idx"], 1e-3)
    k2, foff2, fidx2, _, remap2, d2 = oracle.weld(kept, foff, fidx, 1e-3)
    # reference docstring: welding an already-welded mesh is the identity
    np.testing.assert_array_equal(k2, kept)
    np.testing.assert_array_equal(fidx2, fidx)
    np.testing.assert_array_equal(remap2, np.arange(len(kept)))
    assert d2 == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_weld_matches_reference(name):
    from paper_2106_10031_b200.meshes import weld_arrays
    g = load(name)
    kept, foff, fidx, fsrc, dropped = weld_arrays(g["verts"], g["loop_off"], g["loop_idx"], float(g["tol"]))
    np.testing.assert_array_equal(kept, g["kept"])
    np.testing.assert_array_equal(foff, g["face_off"])
    np.testing.assert_array_equal(fidx, g["face_idx"])
    assert dropped == int(g["dropped"])
    _, _, _, osrc, _, _ = oracle.weld(g["verts"], g["loop_off"], g["loop_idx"], float(g["tol"]))
    np.testing.assert_array_equal(fsrc, osrc)


@pytest.mark.gpu
@pytest.mark.parametrize("tol", [1e-7, 2e-3, 0.0])
def test_gpu_weld_matches_oracle_large(tol):
    """~200k-vertex soups with dense clusters and chains (many greedy rounds)."""
    from paper_2106_10031_b200.meshes import weld_arrays
    rng = np.random.default_rng(7)
    t = tol if tol > 0 else 1e-6
    centres = rng.uniform(-1, 1, (40000, 3))
    reps = rng.integers(1, 9, size=len(centres))
    v = np.repeat(centres, reps, axis=0)
    if tol > 0:
        v = v + rng.normal(scale=0.45 * t, size=v.shape)       # clusters straddling cell borders
    chain = np.cumsum(rng.uniform(0.6, 1.4, size=(5000, 1)) * t, axis=0) * np.array([[0.6, 0.64, 0.48]])
    v = np.concatenate([v, chain + 0.3])[rng.permutation(len(v) + len(chain))]
    off = np.arange(0, len(v) - len(v) % 5 + 1, 5, dtype=np.int64)
    idx = rng.permutation(len(v))[:off[-1]].astype(np.int64)
    ref = oracle.weld(v, off, idx, tol)
    got = weld_arrays(v, off, idx, tol)
    np.testing.assert_array_equal(got[0], ref[0])
    np.testing.assert_array_equal(got[1], ref[1])
    np.testing.assert_array_equal(got[2], ref[2])
    np.testing.assert_array_equal(got[3], ref[3])
    assert got[4] == ref[5]


@pytest.mark.gpu
def test_gpu_welded_mesh_of_march():
    """MarchResult.welded_mesh(): the GPU weld of the sorted polygon soup equals the reference's
    weld of the reference march (golden)."""
    from conftest import load_golden
    from paper_2106_10031_b200 import MarchConfig, march
    g = load_golden("rand_4x12_s13")
    cfg = g["config"]
    res = march(g["net"], MarchConfig(bbox=cfg["bbox"], seeds=cfg["seeds"], scheme=cfg["scheme"],
                                      rng_seed=cfg["rng_seed"], max_cells=cfg["max_cells"]))
    m = res.welded_mesh()
    w = load("soup_rand_4x12_s13")
    np.testing.assert_allclose(m.vertices, w["kept"], atol=1e-9, rtol=0)
    assert m.n_faces == len(w["face_off"]) - 1
    np.testing.assert_array_equal(np.concatenate(m.faces), w["face_idx"])

"""CPU-only checks of the host side and the C-ABI boundary (no GPU needed)."""

import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO, load_golden

from paper_2106_10031_b200 import network as N
from paper_2106_10031_b200 import synth


def header_functions():
    src = open(os.path.join(REPO, "include", "am_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(am_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2106_10031_b200 import _native
    lib = _native.load()          # loading needs no GPU
    for name in header_functions():
        assert hasattr(lib, name), f"{name} declared in include/am_b200.h but not exported"
    assert set(_native.SIGNATURES) >= set(header_functions())


def test_library_is_sm100a():
    so = os.path.join(REPO, "paper_2106_10031_b200", "_lib", "libam_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in sass and "UTMALDG" in sass     # fp64 tensor cores + TMA in the composition GEMM


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_10031_b200 import marching, _native
    with pytest.raises(_native.NativeUnavailable):
        marching.march(N.octahedron_net(0.5), marching.MarchConfig(seeds=2))


@pytest.mark.parametrize("name", ["oct", "cube", "res_linear", "deepsdf_small", "imnet_small"])
def test_interchange_roundtrip(name, tmp_path):
    net = N.load_network(os.path.join(GOLDEN, name + ".json"))
    p = tmp_path / "n.json"
    N.save_network(net, p)
    net2 = N.load_network(p)
    b1, b2 = N.to_blob(net), N.to_blob(net2)
    np.testing.assert_array_equal(b1.params, b2.params)
    np.testing.assert_array_equal(b1.steps, b2.steps)
    assert json.load(open(p)) == json.load(open(os.path.join(GOLDEN, name + ".json"))) or name in ("res_linear",)


def test_blob_layout_deepsdf():
    net = synth.deepsdf_mlp(width=16, depth=6, skip_at=3, seed=0)
    b = N.to_blob(net)
    assert b.n_bits == 6 * 16 and b.n_subs == 1 and not b.ensemble
    flags = b.steps[:, 4]
    assert flags[0] & N.STEP_FIRST and flags[0] & N.STEP_SAVE_INPUT
    assert flags[2] & N.STEP_SHORTCUT_LINEAR and flags[2] & N.STEP_SC_FROM_INPUT
    assert list(b.steps[:, 7]) == [0, 16, 32, 48, 64, 80]          # row offsets in bit order
    assert list(b.steps[:, 8]) == [-1, 0, 16, 32, 48, 64]


def test_key_packing_matches_reference_packbits():
    from paper_2106_10031_b200.marching import words_to_packbits
    rng = np.random.default_rng(0)
    for n_bits in (6, 64, 65, 540, 4096):
        bits = rng.integers(0, 2, size=n_bits).astype(np.uint8)
        kw = (n_bits + 63) // 64
        words = np.zeros(kw, dtype=np.uint64)
        for i, b in enumerate(bits):
            if b:
                words[i >> 6] |= np.uint64(1) << np.uint64(63 - (i & 63))
        kb, br = words_to_packbits(words.reshape(1, -1), n_bits, False)
        assert kb[0].tobytes() == N.StateVector.from_bits(bits).key
        assert br[0] == -1


def test_region_count_lower_bound():
    assert N.region_count_lower_bound([3], 2) == 7
    assert N.region_count_lower_bound([2, 2], 1) == 6
    with pytest.raises(ValueError):
        N.region_count_lower_bound([2], 3)


def test_network_validation_errors():
    with pytest.raises(N.NetworkFormatError):
        N.NetworkSpec((N.DenseLayer(np.ones((6, 3)), np.zeros(6)),), np.ones(5), 0.0)
    with pytest.raises(N.NetworkFormatError):
        N.network_from_dict({"field_kind": "sdf", "subnetworks": []})
    with pytest.raises(N.NetworkFormatError):
        N.EnsembleSpec((N.octahedron_net(0.5), N.octahedron_net(0.5, field_kind="occupancy")))


def test_golden_fixtures_are_self_consistent():
    for name in ("oct", "geo_60x60"):
        g = load_golden(name)
        assert len(g["keys"]) == g["report"]["cells_visited"]
        assert g["nverts"].sum() == len(g["verts"])
        assert g["edge_nrefs"].sum() == len(g["edge_refs"])


def test_polygon_mesh_csr_and_triangulate():
    """PolygonMesh keeps loops as CSR with the reference's constructor / faces semantics; the
    vectorised fan triangulation equals the reference's loop (meshes.py:152-159)."""
    from paper_2106_10031_b200.meshes import PolygonMesh, triangulate
    rng = np.random.default_rng(0)
    v = rng.normal(size=(50, 3))
    loops = [rng.choice(50, size=k, replace=False) for k in rng.integers(3, 9, size=40)]
    m = PolygonMesh(v, loops)
    assert m.n_faces == 40
    for a, b in zip(m.faces, loops):
        np.testing.assert_array_equal(a, b)
    m2 = PolygonMesh(v, None, face_off=m.face_off, face_idx=m.face_idx)
    for a, b in zip(m2.faces, loops):
        np.testing.assert_array_equal(a, b)
    ref = [(lp[0], lp[i], lp[i + 1]) for lp in loops for i in range(1, len(lp) - 1)]
    np.testing.assert_array_equal(triangulate(m2).triangles, np.array(ref))
    with pytest.raises(ValueError):
        PolygonMesh(v, [np.array([0, 1, 60])])


def test_refs_to_kind_index():
    from paper_2106_10031_b200.marching import refs_to_kind_index
    nb, ns = 10, 2
    ids = np.array([0, 9, 10, 11, 12, 17], np.int32)
    np.testing.assert_array_equal(refs_to_kind_index(ids, nb, ns),
                                  [[0, 0], [0, 9], [1, 0], [1, 1], [2, 0], [2, 5]])


def test_topology_check_octahedron():
    from paper_2106_10031_b200.meshes import TriangleMesh, topology_check
    v = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], float)
    t = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4], [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]])
    r = topology_check(TriangleMesh(v, t))
    assert r["watertight"] and r["euler"] == 2 and r["components"] == 1 and r["open_edges"] == 0
    r = topology_check(TriangleMesh(v, t[:-1]))
    assert not r["watertight"] and r["open_edges"] == 3


def test_march_result_pickles_without_device_state():
    """A MarchResult crosses process boundaries (multiprocessing queues, pickle) without its
    device copies or its pending background weld."""
    import pickle
    from concurrent.futures import Future
    from paper_2106_10031_b200.marching import MarchReport, MarchResult
    rep = MarchReport(cells_visited=1, faces_emitted=0, empty_faces=1, open_edges=0, seconds=0.0, seeds_used=1,
                      capped=False, threads=1, waves=1, overflow=0)
    r = MarchResult(np.zeros((1, 2), np.uint8), np.full(1, -1), np.zeros(1, np.int32), np.zeros((0, 3)),
                    np.zeros(0, np.int32), np.zeros((0, 2), np.int32), rep, 10, _dev=(object(),), _weld=(1e-7, Future()))
    back = pickle.loads(pickle.dumps(r))
    assert back._dev is None and back._weld is None and back.n_bits == 10
    assert np.array_equal(back.keys, r.keys)


@pytest.mark.parametrize("case", [("geo", 24, 0), ("geo-rare", 40, 7)])
def test_sample_seeds_host_logic_matches_reference_loop(case):
    """seeding.sample_seeds' host logic -- stacked, memoised sample rounds, several retry rounds
    evaluated per forward and replayed in order, vectorised first-positive / first-negative pick
    -- chooses exactly the reference's bisection pairs (oracle.sample_seeds restates reference
    seeding.py:123-162 stream by stream).  The engine is a CPU stand-in built on the oracle."""
    import torch
    from paper_2106_10031_b200 import seeding, synth
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    name, count, rng_seed = case
    net = synth.geometric_mlp([12, 12], seed=3)
    on = oracle.OracleNet(net)
    bbox = ((-1.2,) * 3, (1.2,) * 3) if name == "geo" else ((0.3, 0.3, 0.3), (1.2, 1.2, 1.2))

    class Eng:
        def __init__(self):
            self.net = net

        def forward(self, pts):
            return torch.as_tensor(on.forward_many(np.asarray(pts)))

        def dichotomy(self, xp, xn, eps, tol):
            return torch.as_tensor(np.stack([oracle._seed_dichotomy(on, a, b)[0] for a, b in zip(xp, xn)]))

    seeding._ROUNDS.clear()
    mine = seeding.sample_seeds(Eng(), count, bbox, rng_seed=rng_seed)
    ref = oracle.sample_seeds(on, count, bbox, rng_seed=rng_seed)
    np.testing.assert_array_equal(mine, ref)

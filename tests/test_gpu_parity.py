"""GPU parity: the CUDA path against the reference's golden vectors and the CPU oracle.

Bar (BASELINE.json north_star): the sorted set of visited cell states matches
bit-exactly; vertices agree within 1e-9 absolute (fp64).
"""

import numpy as np
import pytest

import oracle
from conftest import golden_cases, load_golden, make_random_net

pytestmark = pytest.mark.gpu

VERT_TOL = 1e-9


def _gpu():
    from paper_2106_10031_b200 import marching
    return marching


def assert_same_march(r, ref_keys, ref_branch, ref_nverts, ref_verts, ref_enr, ref_erefs):
    assert r.report.overflow == 0
    assert r.keys.shape == ref_keys.shape, (r.keys.shape, ref_keys.shape)
    np.testing.assert_array_equal(r.keys, ref_keys)
    np.testing.assert_array_equal(r.branch, ref_branch)
    np.testing.assert_array_equal(r.nverts, ref_nverts)
    if len(ref_verts):
        assert np.abs(r.verts - ref_verts).max() <= VERT_TOL
    np.testing.assert_array_equal(r.edge_nrefs, ref_enr)
    np.testing.assert_array_equal(r.edge_refs, ref_erefs)


@pytest.mark.parametrize("name", golden_cases())
def test_march_matches_reference_golden(name):
    g = load_golden(name)
    cfg = g["config"]
    m = _gpu()
    mc = m.MarchConfig(bbox=tuple(map(tuple, cfg["bbox"])), seeds=cfg["seeds"], scheme=cfg["scheme"],
                       rng_seed=cfg["rng_seed"], max_cells=cfg["max_cells"],
                       seed_points=g["seeds"] if cfg["explicit_seeds"] else None)
    r = m.march(g["net"], mc)
    np.testing.assert_allclose(r.seeds, g["seeds"], atol=1e-12, rtol=0)
    if cfg["max_cells"] < 10_000_000 and g["report"]["capped"]:
        # a capped march is order dependent in the reference too: check the contract only
        assert r.report.capped and r.report.cells_visited <= cfg["max_cells"]
        return
    assert_same_march(r, g["keys"], g["branch"], g["nverts"], g["verts"], g["edge_nrefs"], g["edge_refs"])
    for k in ("cells_visited", "faces_emitted", "empty_faces", "open_edges"):
        assert getattr(r.report, k) == g["report"][k], k


def test_forward_and_states_match_oracle():
    from paper_2106_10031_b200.engine import Engine
    net = make_random_net(depth=6, width=20, seed=7)
    pts = np.random.default_rng(2).uniform(-1.2, 1.2, size=(1000, 3))
    eng = Engine(net)
    vals, keys = eng.forward(pts, keys=True)
    on = oracle.OracleNet(net)
    np.testing.assert_allclose(vals.cpu().numpy(), on.forward_many(pts), rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint64), on.state_keys(pts))


def test_affine_maps_match_oracle():
    from paper_2106_10031_b200.engine import Engine
    for net in (make_random_net(depth=4, width=33, seed=3), oracle_net_res()):
        pts = np.random.default_rng(5).uniform(-1.0, 1.0, size=(300, 3))
        eng = Engine(net)
        on = oracle.OracleNet(net)
        keys = on.state_keys(pts)
        canon, planes, faces = eng.affine_maps(keys.view(np.int64))
        canon = canon.cpu().numpy().view(np.uint64)
        planes = planes.cpu().numpy()
        faces = faces.cpu().numpy()
        for i in range(len(pts)):
            c, p, f = on.affine_maps(keys[i])
            np.testing.assert_array_equal(canon[i], c)
            np.testing.assert_allclose(planes[i], p, rtol=1e-11, atol=1e-12)
            np.testing.assert_allclose(faces[i, 0], f, rtol=1e-11, atol=1e-12)


def oracle_net_res():
    from paper_2106_10031_b200 import synth
    return synth.deepsdf_mlp(width=40, depth=5, skip_at=3, bias_std=0.05, seed=4)


@pytest.mark.parametrize("which", ["geo_90x6", "deepsdf_128x8", "imnet_occ", "rand_wide"])
def test_march_matches_oracle_larger(which):
    from paper_2106_10031_b200 import synth
    m = _gpu()
    if which == "geo_90x6":
        net = synth.geometric_mlp([90] * 6, seed=0)
        kw = dict(bbox=((0.1, 0.1, 0.1), (0.45, 0.45, 0.45)), seeds=4, rng_seed=1)
    elif which == "deepsdf_128x8":
        net = synth.deepsdf_mlp(width=128, depth=8, skip_at=4, seed=2)
        kw = dict(bbox=((0.0, 0.0, 0.0), (0.45, 0.45, 0.45)), seeds=4, rng_seed=2)
    elif which == "imnet_occ":
        net = synth.imnet_ensemble(widths=(32, 32, 32), n_parts=4, seed=3)
        kw = dict(seeds=8, rng_seed=3)
    else:
        net = make_random_net(depth=3, width=64, seed=9)
        kw = dict(seeds=8, rng_seed=4)
    r = m.march(net, m.MarchConfig(**kw))
    o = oracle.march(net, bbox=kw.get("bbox", m.DEFAULT_BBOX), seed_points=r.seeds)
    assert r.report.cells_visited > 50
    assert_same_march(r, o.keys, o.branch, o.nverts, o.verts, o.edge_nrefs, o.edge_refs)


@pytest.mark.gpu
def test_engine_cache_reuses_with_new_weights():
    """march() reuses a cached engine for a same-architecture network with different weights:
    am_engine_load_params must refresh every value-derived buffer (padded TMA copies, biases,
    head bias)."""
    from paper_2106_10031_b200 import MarchConfig, march
    from paper_2106_10031_b200.marching import clear_engine_cache
    clear_engine_cache()
    bbox = ((-1.0,) * 3, (1.0,) * 3)
    cfg = MarchConfig(bbox=bbox, seeds=8, rng_seed=3)
    for seed in (21, 22, 21):
        net = make_random_net(3, 16, seed)
        got = march(net, cfg)
        ref = oracle.march(net, bbox=bbox, seeds=8, rng_seed=3)
        np.testing.assert_array_equal(got.keys, ref.keys)
        np.testing.assert_array_equal(got.nverts, ref.nverts)
        assert np.abs(got.verts - ref.verts).max(initial=0) <= 1e-9


@pytest.mark.gpu
def test_fp32_mode_within_stated_tolerance():
    """fp32 mode (fp32-precision planes, reference cell tolerances -- the configuration the
    tools/fp32_study.py sweep recommends): the visited set agrees with the fp64 (reference) one
    to Jaccard >= 0.999, common polygons' vertices agree to 1e-5 at the 99th percentile and
    1e-3 at worst (near-degenerate vertices); fp64 mode itself stays bit-exact (other tests)."""
    from paper_2106_10031_b200 import MarchConfig, march, synth as sy
    net = sy.imnet_ensemble(widths=(32, 32), n_parts=3, seed=1)
    bbox = ((-1.0,) * 3, (1.0,) * 3)
    ref = march(net, MarchConfig(bbox=bbox, seeds=16, rng_seed=0))
    r32 = march(net, MarchConfig(bbox=bbox, seeds=16, rng_seed=0, precision="fp32"))
    key = lambda k, b: k.tobytes() + int(b).to_bytes(8, "little", signed=True)  # noqa: E731
    ka = {key(k, b): i for i, (k, b) in enumerate(zip(ref.keys, ref.branch))}
    kb = {key(k, b): i for i, (k, b) in enumerate(zip(r32.keys, r32.branch))}
    jac = len(ka.keys() & kb.keys()) / len(ka.keys() | kb.keys())
    assert jac >= 0.999, jac
    oa = np.concatenate([[0], np.cumsum(np.maximum(ref.nverts, 0))])
    ob = np.concatenate([[0], np.cumsum(np.maximum(r32.nverts, 0))])
    dev = []
    for k, j in kb.items():
        i = ka.get(k)
        if i is None or ref.nverts[i] != r32.nverts[j] or ref.nverts[i] <= 0:
            continue
        dev.append(float(np.abs(ref.verts[oa[i]:oa[i + 1]] - r32.verts[ob[j]:ob[j + 1]]).max()))
    dev = np.array(dev)
    assert len(dev) > 0.99 * len(kb)
    assert np.quantile(dev, 0.99) <= 1e-5 and dev.max() <= 1e-3, (np.quantile(dev, 0.99), dev.max())


@pytest.mark.gpu
@pytest.mark.parametrize("knob", [("AM_PROBE_IN_GRAPH", "1"), ("AM_COMPOSE_FUSED", "1"), ("AM_NEAR_CAP", "8"),
                                  ("AM_TAU_MULT", "0.25"), ("AM_NEAR_REACH", "1"), ("AM_NARROW", "0"),
                                  ("AM_NARROW_TILE", "2"), ("AM_CANON_FUSED", "0"), ("AM_FACE_ORDER", "1"),
                                  ("AM_PREFIX", "0"), ("AM_NEAR_FUSED", "1"), ("AM_CANON_IN_NARROW", "1"),
                                  ("AM_FACE_UPSERT", "1"), ("AM_ITER_GATE", "1"), ("AM_GEMM_NJ4", "1"),
                                  ("AM_FORWARD_NARROW", "0"), ("AM_NARROW_EXPLICIT", "0")],
                         ids=lambda k: f"{k[0]}={k[1]}")
def test_engine_paths_match_oracle(knob, monkeypatch):
    """Every execution path of the engine is bit-exact, not only the default one: the probe stage
    as a conditional graph node, the fused all-steps composition, near-list overflow (streaming
    fallback), forced hint retries and attempts beyond the near list's reach."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.marching import clear_engine_cache
    m = _gpu()
    monkeypatch.setenv(*knob)
    clear_engine_cache()
    try:
        for net, kw in ((synth.deepsdf_mlp(width=128, depth=8, skip_at=4, seed=2),
                         dict(bbox=((0.0, 0.0, 0.0), (0.45, 0.45, 0.45)), seeds=4, rng_seed=2)),
                        (synth.imnet_ensemble(widths=(32, 32, 32), n_parts=4, seed=3), dict(seeds=8, rng_seed=3)),
                        (synth.geometric_mlp([90] * 4, seed=1), dict(bbox=((0.0, 0.0, 0.0), (0.5, 0.5, 0.5)), seeds=4,
                                                                     rng_seed=5))):
            r = m.march(net, m.MarchConfig(**kw))
            ck = (net.__class__.__name__, r.seeds.tobytes(), str(kw))
            if ck not in _ORACLE_CACHE:   # same network and seeds for every knob: one oracle run
                _ORACLE_CACHE[ck] = oracle.march(net, bbox=kw.get("bbox", m.DEFAULT_BBOX), seed_points=r.seeds)
            o = _ORACLE_CACHE[ck]
            assert r.report.cells_visited > 50
            assert_same_march(r, o.keys, o.branch, o.nverts, o.verts, o.edge_nrefs, o.edge_refs)
    finally:
        clear_engine_cache()


_ORACLE_CACHE: dict = {}


def _bias_batch(n=3):
    """Same-weight plain narrow nets that differ only in their bias vectors (a batch of shapes
    on the fused narrow composition path, per-shape bias tables)."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.network import DenseLayer, NetworkSpec
    base = synth.geometric_mlp([24, 24], seed=3, bias_std=0.05)
    rng = np.random.default_rng(11)
    out = []
    for _ in range(n):
        layers = [DenseLayer(l.weight, l.bias + rng.normal(0.0, 0.02, size=l.bias.shape)) for l in base.layers]
        out.append(NetworkSpec(layers, base.head_weight, base.head_bias + rng.normal(0.0, 0.02)))
    return out


@pytest.mark.gpu
def test_narrow_path_batch_of_shapes_matches_oracle():
    """k_compose_narrow with per-shape biases (a fused batch of plain narrow nets) == the oracle
    march of every shape."""
    from paper_2106_10031_b200.batch import march_fused
    m = _gpu()
    nets = _bias_batch(3)
    cfg = m.MarchConfig(seeds=6, rng_seed=4)
    for s, r in enumerate(march_fused(nets, cfg)):
        o = oracle.march(nets[s], seed_points=r.seeds)
        assert r.report.cells_visited > 100
        assert_same_march(r, o.keys, o.branch, o.nverts, o.verts, o.edge_nrefs, o.edge_refs)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_narrow_and_per_layer_composition_agree_bitwise(precision, monkeypatch):
    """The fused narrow composition and the per-layer DMMA kernels produce the same march, bit
    for bit, in both precisions (AM_NARROW=0 selects the per-layer path)."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.marching import clear_engine_cache
    m = _gpu()
    net = synth.geometric_mlp([60, 60], seed=0)
    cfg = m.MarchConfig(seeds=4, rng_seed=0, precision=precision)
    clear_engine_cache()
    a = m.march(net, cfg)
    monkeypatch.setenv("AM_NARROW", "0")
    clear_engine_cache()
    try:
        b = m.march(net, cfg)
    finally:
        clear_engine_cache()
    np.testing.assert_array_equal(a.keys, b.keys)
    np.testing.assert_array_equal(a.nverts, b.nverts)
    np.testing.assert_array_equal(a.verts, b.verts)
    np.testing.assert_array_equal(a.edge_refs, b.edge_refs)


@pytest.mark.gpu
def test_prefix_reuse_per_step_batch_of_shapes_is_bitwise_neutral(monkeypatch):
    """Prefix reuse on the per-step path of a fused batch of latent shapes (per-shape biases; a
    child's parent is always of its own shape) gives every shape's march bit for bit."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.batch import march_fused
    from paper_2106_10031_b200.marching import clear_engine_cache
    m = _gpu()
    nets, _ = synth.latent_batch(n_shapes=3, latent_dim=8, width=160, depth=5, skip_at=3, seed=5, code_std=0.05)
    cfg = m.MarchConfig(bbox=((0.0, 0.0, 0.0), (0.5, 0.5, 0.5)), seeds=4, rng_seed=1)
    out = {}
    try:
        for mode in ("1", "0"):
            monkeypatch.setenv("AM_PREFIX", mode)
            clear_engine_cache()
            out[mode] = march_fused(nets, cfg)
    finally:
        clear_engine_cache()
    for a, b in zip(out["1"], out["0"]):
        assert a.report.cells_visited > 200
        for f in ("keys", "nverts", "verts", "edge_nrefs", "edge_refs"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["narrow-fp64", "narrow-fp32", "narrow-varying-widths", "per-step-deepsdf"])
def test_prefix_reuse_is_bitwise_neutral(case, monkeypatch):
    """Children composed from their parents' Z rows (prefix reuse, on the narrow and on the
    per-step path) give the same march, bit for bit, as composing every step; and the reuse
    really engaged (composition flops skipped)."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.marching import _ENGINES, clear_engine_cache
    m = _gpu()
    if case == "narrow-varying-widths":   # steps of different widths (copied rows feed narrower steps)
        net = synth.geometric_mlp([96, 48, 80, 32, 64], seed=4)
        cfg = m.MarchConfig(bbox=((0.0, 0.0, 0.0), (0.6, 0.6, 0.6)), seeds=4, rng_seed=5)
    elif case.startswith("narrow"):
        net = synth.geometric_mlp([90] * 4, seed=1)
        cfg = m.MarchConfig(bbox=((0.0, 0.0, 0.0), (0.5, 0.5, 0.5)), seeds=4, rng_seed=5,
                            precision=case.split("-")[1])
    else:
        net = synth.deepsdf_mlp(width=128, depth=8, skip_at=4, seed=2)
        cfg = m.MarchConfig(bbox=((0.0, 0.0, 0.0), (0.45, 0.45, 0.45)), seeds=4, rng_seed=2)
    out = {}
    try:
        for mode in ("1", "0"):
            monkeypatch.setenv("AM_PREFIX", mode)
            clear_engine_cache()
            out[mode] = m.march(net, cfg)
            st = next(iter(_ENGINES.values())).stats()
            if mode == "1":
                assert st["prefix"] == 1 and st["prefix_skipped_flops"] > 0
            else:
                assert st["prefix"] == 0
    finally:
        clear_engine_cache()
    a, b = out["1"], out["0"]
    assert a.report.cells_visited > 1000
    for f in ("keys", "nverts", "verts", "edge_nrefs", "edge_refs"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_narrow_point_forward_matches_per_layer_bitwise(precision, monkeypatch):
    """k_forward_narrow (every layer + head of a narrow net in one launch) returns the values and
    state keys of the per-layer forward kernels bit for bit, also for a batch of shapes."""
    import torch
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.engine import Engine
    _gpu()
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1.2, 1.2, size=(5000, 3))
    nets = [synth.geometric_mlp([90] * 6, seed=0), synth.geometric_mlp([60, 60], seed=3)]
    for net in nets:
        out = {}
        for mode in ("1", "0"):
            monkeypatch.setenv("AM_FORWARD_NARROW", mode)
            eng = Engine(net, precision=precision)
            v, k = eng.forward(pts, keys=True)
            out[mode] = (v.cpu().numpy(), k.cpu().numpy())
            del eng
        np.testing.assert_array_equal(out["1"][0], out["0"][0])
        np.testing.assert_array_equal(out["1"][1], out["0"][1])
    # batch of shapes: per-shape biases, per-point shapes
    bnets = _bias_batch(3)
    shapes = rng.integers(0, 3, size=len(pts)).astype(np.int32)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("AM_FORWARD_NARROW", mode)
        eng = Engine(bnets[0], n_shapes=3)
        eng.set_shapes(bnets)
        v, k = eng.forward(pts, keys=True, shapes=shapes)
        out[mode] = (v.cpu().numpy(), k.cpu().numpy())
        del eng
    np.testing.assert_array_equal(out["1"][0], out["0"][0])
    np.testing.assert_array_equal(out["1"][1], out["0"][1])


@pytest.mark.gpu
@pytest.mark.parametrize("heavy", [False, True])
def test_max_cells_cap_is_exact(heavy):
    """With max_cells reached the march returns exactly max_cells visited cells and the capped
    flag (reference marching.py:240-242); heavy nets (no deferral) end the walk at the cap
    instead of composing and discarding the rest of the queue."""
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.marching import clear_engine_cache
    m = _gpu()
    net = synth.deepsdf_mlp(width=192, depth=8, skip_at=4, seed=2) if heavy else synth.geometric_mlp([90] * 4, seed=1)
    clear_engine_cache()
    try:
        r = m.march(net, m.MarchConfig(seeds=8, rng_seed=3, max_cells=3000))
    finally:
        clear_engine_cache()
    assert r.report.capped
    assert r.report.cells_visited == 3000
    assert r.report.overflow == 0


@pytest.mark.gpu
def test_narrow_varying_widths_matches_oracle():
    """The fused narrow composition on a net whose layers differ in width (96, 48, 80, 32, 64:
    step K extents and row counts change from step to step) == the oracle march."""
    from paper_2106_10031_b200 import synth
    m = _gpu()
    net = synth.geometric_mlp([96, 48, 80, 32, 64], seed=4)
    bbox = ((0.0, 0.0, 0.0), (0.6, 0.6, 0.6))
    r = m.march(net, m.MarchConfig(bbox=bbox, seeds=4, rng_seed=5))
    o = oracle.march(net, bbox=bbox, seed_points=r.seeds)
    assert r.report.cells_visited > 1000
    assert_same_march(r, o.keys, o.branch, o.nverts, o.verts, o.edge_nrefs, o.edge_refs)

"""The drop-in surface of the reference's meshing path, on the GPU.

Restates the behaviours the reference's own tests check (reference
tests/test_marching.py, tests/test_properties.py) through this package's API,
on networks given as FOREIGN objects that only carry the reference's
attributes (``.layers`` / ``.weight`` / ``.bias`` / ``.inner`` /
``.shortcut_weight`` / ``.subnetworks`` / ``.head_weight`` ...), so nothing
depends on this package's own containers.  ``tools/run_reference_tests.py``
runs the reference's test files themselves against this march.
"""

from dataclasses import dataclass

import numpy as np
import pytest

import oracle
from conftest import make_random_net

pytestmark = pytest.mark.gpu


@dataclass(frozen=True)
class FDense:
    weight: np.ndarray
    bias: np.ndarray


@dataclass(frozen=True)
class FResidual:
    inner: tuple
    shortcut_weight: np.ndarray | None = None
    shortcut_bias: np.ndarray | None = None


@dataclass(frozen=True)
class FNet:
    layers: tuple
    head_weight: np.ndarray
    head_bias: float
    field_kind: str = "sdf"


@dataclass(frozen=True)
class FEnsemble:
    subnetworks: tuple

    @property
    def field_kind(self):
        return self.subnetworks[0].field_kind


def foreign(net):
    """Re-express any network as foreign objects with the reference's attribute names."""
    from paper_2106_10031_b200.network import is_ensemble, is_residual
    if is_ensemble(net):
        return FEnsemble(tuple(foreign(s) for s in net.subnetworks))
    layers = []
    for lay in net.layers:
        if is_residual(lay):
            layers.append(FResidual(tuple(FDense(d.weight, d.bias) for d in lay.inner), lay.shortcut_weight,
                                    lay.shortcut_bias))
        else:
            layers.append(FDense(lay.weight, lay.bias))
    return FNet(tuple(layers), net.head_weight, net.head_bias, net.field_kind)


def oct_net(c=0.5, kind="sdf"):
    from paper_2106_10031_b200 import octahedron_net
    return foreign(octahedron_net(c, field_kind=kind))


def test_foreign_objects_march_like_native_ones():
    from paper_2106_10031_b200 import MarchConfig, march, synth
    for net in (synth.deepsdf_mlp(width=24, depth=5, skip_at=3, bias_std=0.05, seed=3),
                synth.imnet_ensemble(widths=(12, 12), n_parts=3, seed=1)):
        a = march(net, MarchConfig(seeds=8, rng_seed=0))
        b = march(foreign(net), MarchConfig(seeds=8, rng_seed=0))
        np.testing.assert_array_equal(a.keys, b.keys)
        np.testing.assert_array_equal(a.verts, b.verts)


def test_octahedron_geometry_planes_and_residuals():
    from paper_2106_10031_b200 import MarchConfig, march, vertex_residuals
    from paper_2106_10031_b200.meshes import topology_check, triangulate
    net = oct_net()
    r = march(net, MarchConfig(seeds=8, rng_seed=3))
    assert r.report.faces_emitted == 8 and r.report.open_edges == 0
    assert all(p.n_vertices == 3 for p in r.polygons)
    # face plane = the raw functional of F on the cell: +-x +-y +-z - 0.5
    for p in r.polygons:
        assert p.plane is not None
        np.testing.assert_allclose(np.abs(p.plane.normal), 1.0, atol=0)
        assert p.plane.offset == -0.5
        assert max(abs(p.plane.value(v)) for v in p.vertices) <= 1e-12
    mesh = r.welded_mesh()
    assert mesh.n_vertices == 6 and len(mesh.face_planes) == mesh.n_faces == 8
    assert topology_check(triangulate(mesh)) == {"watertight": True, "open_edges": 0, "nonmanifold_edges": 0,
                                                 "euler": 2, "components": 1}
    soup = r.polygon_soup()
    assert len(soup.face_planes) == 8
    assert vertex_residuals(net, r).max() <= 1e-12
    assert vertex_residuals(net, mesh).max() <= 1e-12
    # 8 distinct face planes: no proportional pair
    assert r.report.unique_plane_violations == 0


def test_face_planes_match_oracle_affine_maps():
    from paper_2106_10031_b200 import MarchConfig, march
    net = make_random_net(depth=4, width=12, seed=13)
    r = march(foreign(net), MarchConfig(seeds=32, rng_seed=1))
    on = oracle.OracleNet(net)
    rows = r.face_plane_rows()
    words = r.keys  # packbits rows
    from paper_2106_10031_b200.evaluate import packbits_to_words
    w = packbits_to_words(words[r.nverts > 0], None, r.n_bits).view(np.uint64)
    for i in range(len(w)):
        _, _, f = on.affine_maps(w[i])
        np.testing.assert_allclose(rows[i], f, rtol=1e-11, atol=1e-12)


def test_unique_plane_violations_match_reference_formula():
    """am_unique_planes against the reference's chord rule (network.py:528-570) restated in numpy,
    on planes with exact and near duplicates (scaled, negated, perturbed below / above tol)."""
    from paper_2106_10031_b200.evaluate import unique_plane_pairs
    rng = np.random.default_rng(0)
    H = rng.normal(size=(200, 4))
    H[10] = -3.0 * H[3]
    H[20] = 0.5 * H[7] + 1e-12
    H[30] = H[8] * (1 + 1e-6)
    H[40] = H[9] + 1e-7
    H[50] = 0.0
    H[51] = 0.0
    n = np.linalg.norm(H, axis=1)
    n[n == 0] = 1.0
    U = H / n[:, None]
    d = np.minimum(np.linalg.norm(U[:, None] - U[None], axis=2), np.linalg.norm(U[:, None] + U[None], axis=2))
    ii, jj = np.nonzero(d <= 1e-9)
    want = sorted((int(a), int(b)) for a, b in zip(ii, jj) if a < b)
    assert (3, 10) in want and (7, 20) in want and (8, 30) in want and (50, 51) in want
    assert unique_plane_pairs(H, 1e-9) == want


def test_ensemble_cube_geometry():
    from paper_2106_10031_b200 import MarchConfig, cube_ensemble, march
    r = march(foreign(cube_ensemble(0.5)), MarchConfig(seeds=16, rng_seed=5))
    assert r.report.faces_emitted == 6 and all(p.n_vertices == 4 for p in r.polygons)
    mesh = r.welded_mesh()
    assert {tuple(np.round(v, 9)) for v in mesh.vertices} == {(x * 0.5, y * 0.5, z * 0.5)
                                                              for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)}
    for p in r.polygons:   # face functional of the dominating branch: one axis, unit slope
        assert np.count_nonzero(p.plane.normal) == 1


def test_march_contract_errors_cap_seeds_modes():
    from paper_2106_10031_b200 import MarchConfig, march
    from paper_2106_10031_b200.seeding import SeedingError
    net = oct_net()
    with pytest.raises(SeedingError, match="no surface"):
        march(FNet(net.layers, net.head_weight, 10.0), MarchConfig(seeds=4, rng_seed=0))
    capped = march(foreign(make_random_net(4, 12, 17)), MarchConfig(seeds=8, rng_seed=3, max_cells=5))
    assert capped.report.capped and capped.report.cells_visited <= 5
    seeds = np.array([[0.3, 0.15, 0.05], [-0.2, -0.2, 0.1]])
    r = march(net, MarchConfig(seed_points=seeds))
    assert r.report.faces_emitted == 8 and r.report.seeds_used == 2
    rnet = foreign(make_random_net(4, 8, 11))
    a = march(rnet, MarchConfig(seeds=24, rng_seed=2, mode="pivot"))
    b = march(rnet, MarchConfig(seeds=24, rng_seed=2, mode="naive"))
    assert a.face_multiset(decimals=7) == b.face_multiset(decimals=7)
    occ = march(oct_net(kind="occupancy"), MarchConfig(seeds=8, rng_seed=3))
    assert occ.report.faces_emitted == 8 and occ.welded_mesh().n_vertices == 6


def test_explicit_engine_is_reloaded_and_reset():
    """march(net, cfg, engine=eng): the engine takes net's weights and forgets earlier marches
    (ADVICE r1); more seeds than one batch are split into batch-sized am_seed calls."""
    from paper_2106_10031_b200 import MarchConfig, march
    from paper_2106_10031_b200.engine import Engine
    n1, n2 = make_random_net(3, 16, 21), make_random_net(3, 16, 22)
    eng = Engine(n1, batch_cells=256)
    march(n1, MarchConfig(seeds=8, rng_seed=3), engine=eng)
    got = march(n2, MarchConfig(seeds=8, rng_seed=3), engine=eng)
    ref = oracle.march(n2, seeds=8, rng_seed=3)
    np.testing.assert_array_equal(got.keys, ref.keys)
    many = np.repeat(got.seeds, 40, axis=0)   # 320 seed points > 256-cell batches
    again = march(n2, MarchConfig(seed_points=many), engine=eng)
    np.testing.assert_array_equal(again.keys, ref.keys)


def test_module_level_evaluators_match_oracle():
    from paper_2106_10031_b200 import affine_maps, forward, forward_many, grad_input, state_at, state_at_many
    from paper_2106_10031_b200.network import StateVector
    net = make_random_net(depth=5, width=16, seed=7)
    f = foreign(net)
    on = oracle.OracleNet(net)
    pts = np.random.default_rng(1).uniform(-1, 1, size=(500, 3))
    np.testing.assert_allclose(forward_many(f, pts), on.forward_many(pts), rtol=1e-12, atol=1e-12)
    assert abs(forward(f, pts[0]) - on.forward_many(pts[:1])[0]) <= 1e-12
    bits, br = state_at_many(f, pts)
    assert br is None and bits.shape == (500, 80)
    keys = on.state_keys(pts)
    for i in (0, 17, 499):
        s = state_at(f, pts[i])
        assert s == StateVector.from_bits(bits[i])
        m = affine_maps(f, s)
        c, p, face = on.affine_maps(keys[i])
        np.testing.assert_allclose(m.neuron_normals, p[:, :3], rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(m.face_normal, face[:3], rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(grad_input(f, pts[i]), face[:3], rtol=1e-11, atol=1e-12)
    with pytest.raises(ValueError):
        forward_many(f, np.zeros((3, 2)))

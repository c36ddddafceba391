"""Host logic of the drop-in boundary (no GPU): duck-typed networks, the C-ABI descriptor, the
JSON interchange schema, state / plane-reference identity, and the sharding cap split.

The reference's own network classes are mimicked by plain dataclasses carrying only the
reference's attribute names (reference network.py:49-213); when the reference package is
importable (build container) its objects are checked too."""

import os
import sys
from dataclasses import dataclass

import numpy as np
import pytest

from paper_2106_10031_b200 import network as N
from paper_2106_10031_b200 import synth


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


def foreign(net):
    if N.is_ensemble(net):
        return FEnsemble(tuple(foreign(s) for s in net.subnetworks))
    layers = tuple(FResidual(tuple(FDense(d.weight, d.bias) for d in l.inner), l.shortcut_weight, l.shortcut_bias)
                   if N.is_residual(l) else FDense(l.weight, l.bias) for l in net.layers)
    return FNet(layers, net.head_weight, net.head_bias, net.field_kind)


NETS = {
    "geo": lambda: synth.geometric_mlp([12, 12], seed=0),
    "deepsdf": lambda: synth.deepsdf_mlp(width=16, depth=5, skip_at=3, bias_std=0.05, seed=1),
    "imnet": lambda: synth.imnet_ensemble(widths=(8, 8), n_parts=3, seed=2),
    "res_identity": lambda: N.NetworkSpec([N.octahedron_net().layers[0],
                                           N.ResidualBlock([N.DenseLayer(np.zeros((6, 6)), np.zeros(6))] * 2)],
                                          np.ones(6), -0.5),
}


@pytest.mark.parametrize("name", sorted(NETS))
def test_foreign_objects_give_the_same_descriptor(name):
    net = NETS[name]()
    a, b = N.to_blob(net), N.to_blob(foreign(net))
    assert np.array_equal(a.params, b.params) and np.array_equal(a.steps, b.steps)
    assert np.array_equal(a.subs, b.subs)
    assert (a.n_bits, a.ensemble, a.key_words) == (b.n_bits, b.ensemble, b.key_words)


@pytest.mark.parametrize("name", sorted(NETS))
def test_json_round_trip_is_bit_exact(name, tmp_path):
    net = NETS[name]()
    path = tmp_path / "net.json"
    N.save_network(foreign(net), path)
    back = N.load_network(path)
    a, b = N.to_blob(net), N.to_blob(back)
    assert np.array_equal(a.params, b.params) and np.array_equal(a.steps, b.steps)


def test_descriptor_layout_of_a_linear_skip():
    """DeepSDF skip = residual_linear block over the input: the last inner step adds V x."""
    b = N.to_blob(NETS["deepsdf"]())
    flags = b.steps[:, 4]
    assert flags[0] & N.STEP_FIRST and flags[0] & N.STEP_SAVE_INPUT
    last_inner = int(np.flatnonzero(flags & N.STEP_SHORTCUT_LINEAR)[0])
    assert flags[last_inner] & N.STEP_SC_FROM_INPUT and b.steps[last_inner, 5] >= 0
    assert b.n_bits == int(b.steps[:, 1].sum())


@pytest.mark.parametrize("bad", [
    lambda: FNet((FDense(np.ones((6, 3)), np.zeros(6)),), np.ones(5), 0.0),        # head width
    lambda: FNet((FDense(np.ones((6, 4)), np.zeros(6)),), np.ones(6), 0.0),        # input width
    lambda: FNet((FDense(np.ones((6, 3)), np.zeros(5)),), np.ones(6), 0.0),        # bias length
    lambda: FNet((FDense(np.full((6, 3), np.nan), np.zeros(6)),), np.ones(6), 0.0),  # non-finite
    lambda: FNet((FDense(np.ones((6, 3)), np.zeros(6)),), np.ones(6), 0.0, "density"),
    lambda: FEnsemble((FNet((FDense(np.ones((2, 3)), np.zeros(2)),), np.ones(2), 0.0),
                       FNet((FDense(np.ones((2, 3)), np.zeros(2)),), np.ones(2), 0.0, "occupancy"))),
    lambda: FNet((FResidual((FDense(np.ones((4, 3)), np.zeros(4)),)),), np.ones(4), 0.0),   # identity width
])
def test_malformed_networks_are_rejected(bad):
    with pytest.raises(N.NetworkFormatError):
        N.to_blob(bad())


def test_state_vector_packing_and_identity():
    bits = np.array([1, 0, 1, 1, 0, 0, 1, 0, 1, 1], np.uint8)
    s = N.StateVector.from_bits(bits)
    assert s.key == np.packbits(bits).tobytes() and s.n_bits == 10
    assert np.array_equal(s.bits(), bits)
    assert s.flip(3).flip(3) == s and s.flip(3) != s
    assert tuple(s.flip(9).bits()) == tuple(np.r_[bits[:9], 0])

    @dataclass(frozen=True)
    class Other:   # the reference's StateVector shape
        key: bytes
        n_bits: int
        branch: int | None = None
    o = Other(s.key, 10, None)
    assert s == o and hash(s) == hash(o) and {o: 1}[s] == 1
    assert s.with_branch(2) != o


def test_plane_ref_identity_with_foreign_refs():
    from paper_2106_10031_b200.marching import PLANE_BRANCH, PLANE_NEURON, PlaneRef, neighbor_state, transition_states

    @dataclass(frozen=True)
    class Ref:
        kind: int
        index: int
    assert PlaneRef(0, 4) == Ref(0, 4) and [Ref(0, 4)].index(PlaneRef(0, 4)) == 0
    assert hash(PlaneRef(1, 2)) == hash(Ref(1, 2))
    s = N.StateVector.from_bits([1, 0, 0, 1], branch=0)
    assert neighbor_state(s, PlaneRef(PLANE_NEURON, 1)).bits()[1] == 1
    assert neighbor_state(s, PlaneRef(PLANE_BRANCH, 2)).branch == 2
    with pytest.raises(ValueError):
        neighbor_state(s, PlaneRef(2, 0))
    # two coincident neuron planes + a branch: subsets {a}, {b}, {a, b} x (none, branch) + branch alone
    out = transition_states(s, (PlaneRef(PLANE_NEURON, 0), PlaneRef(PLANE_NEURON, 2), PlaneRef(PLANE_BRANCH, 1)))
    assert len(out) == 7 and len(set(out)) == 7


def test_cap_share_splits_max_cells_exactly():
    from paper_2106_10031_b200.distributed import cap_share
    for total, world in ((10, 3), (7, 8), (1_000_000, 8), (5, 1)):
        shares = [cap_share(total, r, world) for r in range(world)]
        assert sum(shares) == max(total, world) if total < world else sum(shares) == total
        assert max(shares) - min(shares) <= 1


def test_reference_objects_when_available():
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, ref)
    import exactmesh.network as R
    for net in (R.octahedron_net(), R.cube_ensemble()):
        b = N.to_blob(net)
        mine = N.to_blob(N.network_from_dict(N.network_to_dict(net)))
        assert np.array_equal(b.params, mine.params) and np.array_equal(b.steps, mine.steps)
    s = R.StateVector.from_bits([1, 0, 1])
    assert N.StateVector.from_bits([1, 0, 1]) == s and s == N.StateVector.from_bits([1, 0, 1])

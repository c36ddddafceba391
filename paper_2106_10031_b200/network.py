"""ReLU implicit-surface networks: the model side of the meshing boundary.

Mirrors the reference package's network module (``exactmesh/network.py``):
the same layer kinds (dense, identity-shortcut residual block, linear-shortcut
residual block), the same max-pool ensemble, the same ``StateVector`` packing
(``np.packbits`` bit order, reference network.py:222-262) and the same JSON
interchange format (reference network.py:585-660), so a network file written
by either side loads bit-exactly in the other.

Everything numeric about *meshing* runs on the GPU (see ``marching.py``);
this module only holds weights and flattens them into the descriptor the
C-ABI library consumes (``to_blob``).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Iterable, Sequence, Union

import numpy as np

FIELD_KINDS = ("sdf", "occupancy")

# reference network.py:27 -- rows of a masked product below this norm are constant functionals
DEGENERATE_NORMAL_TOL = 1e-12


class NetworkFormatError(ValueError):
    """Interchange file fails to parse or violates an invariant (reference network.py:30)."""


def _as_matrix(value, name: str) -> np.ndarray:
    arr = np.asarray(value, dtype=np.float64)
    if arr.ndim != 2:
        raise NetworkFormatError(f"{name}: expected a 2-d weight matrix, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise NetworkFormatError(f"{name}: non-finite weight entries")
    return arr


def _as_vector(value, name: str) -> np.ndarray:
    arr = np.asarray(value, dtype=np.float64)
    if arr.ndim != 1:
        raise NetworkFormatError(f"{name}: expected a 1-d bias vector, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise NetworkFormatError(f"{name}: non-finite bias entries")
    return arr


@dataclass(frozen=True)
class DenseLayer:
    """``weight`` is (n_out, n_in); weight[i, j] multiplies input j into output i."""

    weight: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "weight", np.asarray(self.weight, dtype=np.float64))
        object.__setattr__(self, "bias", np.asarray(self.bias, dtype=np.float64))

    @property
    def in_width(self) -> int:
        return self.weight.shape[1]

    @property
    def out_width(self) -> int:
        return self.weight.shape[0]

    @property
    def n_hidden(self) -> int:
        return self.out_width

    def validate(self, name: str, in_width: int) -> int:
        _as_matrix(self.weight, f"{name}.weight")
        _as_vector(self.bias, f"{name}.bias")
        if self.bias.shape[0] != self.out_width:
            raise NetworkFormatError(
                f"{name}: bias length {self.bias.shape[0]} != weight rows {self.out_width}")
        if self.in_width != in_width:
            raise NetworkFormatError(f"{name}: expects input width {self.in_width}, got {in_width}")
        return self.out_width


@dataclass(frozen=True)
class ResidualBlock:
    """ReLU(shortcut(x_in) + inner(x_in)); inner has ReLU between, not after, its layers.

    ``shortcut_weight is None`` is the identity shortcut (reference
    network.py:81-121); otherwise the shortcut is ``V x_in + v_bias``.
    """

    inner: tuple
    shortcut_weight: np.ndarray | None = None
    shortcut_bias: np.ndarray | None = None

    def __post_init__(self):
        object.__setattr__(self, "inner", tuple(self.inner))

    @property
    def out_width(self) -> int:
        return self.inner[-1].out_width

    @property
    def n_hidden(self) -> int:
        return sum(l.out_width for l in self.inner)

    def validate(self, name: str, in_width: int) -> int:
        if not self.inner:
            raise NetworkFormatError(f"{name}: residual block has no inner layers")
        w = in_width
        for i, lay in enumerate(self.inner):
            w = lay.validate(f"{name}.inner[{i}]", w)
        if self.shortcut_weight is None:
            if self.shortcut_bias is not None:
                raise NetworkFormatError(f"{name}: shortcut bias without shortcut weight")
            if in_width != self.out_width:
                raise NetworkFormatError(
                    f"{name}: identity shortcut requires input width {in_width} == "
                    f"output width {self.out_width}")
        else:
            v = _as_matrix(self.shortcut_weight, f"{name}.shortcut_weight")
            if v.shape != (self.out_width, in_width):
                raise NetworkFormatError(
                    f"{name}: shortcut weight shape {v.shape} != ({self.out_width}, {in_width})")
            if self.shortcut_bias is not None:
                b = _as_vector(self.shortcut_bias, f"{name}.shortcut_bias")
                if b.shape[0] != self.out_width:
                    raise NetworkFormatError(f"{name}: shortcut bias length mismatch")
        return self.out_width


Layer = Union[DenseLayer, ResidualBlock]


@dataclass(frozen=True)
class NetworkSpec:
    """Hidden ReLU stack + scalar linear head + field kind (reference network.py:127)."""

    layers: tuple
    head_weight: np.ndarray
    head_bias: float
    field_kind: str = "sdf"
    input_dim: int = 3

    def __post_init__(self):
        object.__setattr__(self, "head_weight", _as_vector(self.head_weight, "head.weight"))
        object.__setattr__(self, "layers", tuple(self.layers))
        object.__setattr__(self, "head_bias", float(self.head_bias))
        self.validate()

    def validate(self) -> None:
        if self.field_kind not in FIELD_KINDS:
            raise NetworkFormatError(f"field_kind must be one of {FIELD_KINDS}")
        if self.input_dim != 3:
            raise NetworkFormatError("input_dim is fixed at 3")
        if not self.layers:
            raise NetworkFormatError("network needs at least one hidden layer")
        w = self.input_dim
        for i, lay in enumerate(self.layers):
            w = lay.validate(f"layers[{i}]", w)
        if self.head_weight.shape[0] != w:
            raise NetworkFormatError(
                f"head: weight length {self.head_weight.shape[0]} != last layer width {w}")
        if not math.isfinite(self.head_bias):
            raise NetworkFormatError("head: non-finite bias")

    @property
    def n_hidden(self) -> int:
        return sum(l.n_hidden for l in self.layers)

    @property
    def hidden_widths(self) -> tuple:
        widths = []
        for lay in self.layers:
            if isinstance(lay, DenseLayer):
                widths.append(lay.out_width)
            else:
                widths.extend(l.out_width for l in lay.inner)
        return tuple(widths)


@dataclass(frozen=True)
class EnsembleSpec:
    """Max-pool union F = max_i F_i (reference network.py:180, paper §5.2)."""

    subnetworks: tuple

    def __post_init__(self):
        object.__setattr__(self, "subnetworks", tuple(self.subnetworks))
        if not self.subnetworks:
            raise NetworkFormatError("ensemble needs at least one subnetwork")
        if len({s.field_kind for s in self.subnetworks}) != 1:
            raise NetworkFormatError("ensemble subnetworks must share field_kind")

    @property
    def field_kind(self) -> str:
        return self.subnetworks[0].field_kind

    @property
    def input_dim(self) -> int:
        return 3

    @property
    def n_hidden(self) -> int:
        return sum(s.n_hidden for s in self.subnetworks)

    @property
    def n_branches(self) -> int:
        return len(self.subnetworks)


AnyNetwork = Union[NetworkSpec, EnsembleSpec]


def subnetworks(net: AnyNetwork) -> tuple:
    return net.subnetworks if isinstance(net, EnsembleSpec) else (net,)


@dataclass(frozen=True)
class StateVector:
    """Activation pattern over all hidden neurons, ordered by (layer, neuron).

    ``key`` is ``np.packbits(bits)`` exactly as in reference network.py:222 so
    keys compare and sort identically; ``branch`` is the dominating subnetwork
    for ensembles, None for plain networks.
    """

    key: bytes
    n_bits: int
    branch: int | None = None

    @classmethod
    def from_bits(cls, bits: Iterable[int] | np.ndarray, branch: int | None = None) -> "StateVector":
        arr = np.asarray(bits, dtype=np.uint8).ravel()
        return cls(key=np.packbits(arr).tobytes(), n_bits=arr.shape[0], branch=branch)

    def bits(self) -> np.ndarray:
        return np.unpackbits(np.frombuffer(self.key, dtype=np.uint8))[: self.n_bits]

    def flip(self, index: int) -> "StateVector":
        if not 0 <= index < self.n_bits:
            raise IndexError(f"bit index {index} out of range [0, {self.n_bits})")
        b = self.bits().copy()
        b[index] ^= 1
        return StateVector.from_bits(b, branch=self.branch)

    def with_branch(self, branch: int) -> "StateVector":
        return StateVector(key=self.key, n_bits=self.n_bits, branch=branch)

    def __repr__(self) -> str:
        bits = "".join(str(int(b)) for b in self.bits())
        tail = "" if self.branch is None else f"|b{self.branch}"
        return f"StateVector({bits}{tail})"


@dataclass(frozen=True)
class AffinePlane:
    """Affine functional n . x + d (reference network.py:265)."""

    normal: np.ndarray
    offset: float

    def __post_init__(self):
        n = np.asarray(self.normal, dtype=np.float64).reshape(3)
        if not (np.all(np.isfinite(n)) and math.isfinite(self.offset)):
            raise ValueError("plane coefficients must be finite")
        object.__setattr__(self, "normal", n)
        object.__setattr__(self, "offset", float(self.offset))

    def value(self, x) -> float:
        return float(self.normal @ np.asarray(x, dtype=np.float64) + self.offset)

    @property
    def degenerate(self) -> bool:
        return float(np.linalg.norm(self.normal)) <= DEGENERATE_NORMAL_TOL


# ---------------------------------------------------------------------------
# interchange format (reference network.py:585-672)


def _layer_to_json(lay) -> dict:
    if isinstance(lay, DenseLayer):
        return {"kind": "dense", "weight": lay.weight.tolist(), "bias": lay.bias.tolist()}
    doc: dict = {"inner": [_layer_to_json(l) for l in lay.inner]}
    if lay.shortcut_weight is None:
        doc["kind"] = "residual_identity"
    else:
        doc["kind"] = "residual_linear"
        doc["shortcut_weight"] = np.asarray(lay.shortcut_weight).tolist()
        doc["shortcut_bias"] = (np.zeros(lay.out_width) if lay.shortcut_bias is None
                                else np.asarray(lay.shortcut_bias)).tolist()
    return doc


def _layer_from_json(doc: dict, name: str):
    kind = doc.get("kind")
    if kind == "dense":
        for key in ("weight", "bias"):
            if key not in doc:
                raise NetworkFormatError(f"{name}: dense layer missing '{key}'")
        return DenseLayer(_as_matrix(doc["weight"], f"{name}.weight"),
                          _as_vector(doc["bias"], f"{name}.bias"))
    if kind in ("residual_identity", "residual_linear"):
        inner_docs = doc.get("inner")
        if not inner_docs:
            raise NetworkFormatError(f"{name}: residual block missing 'inner'")
        inner = []
        for i, d in enumerate(inner_docs):
            lay = _layer_from_json(d, f"{name}.inner[{i}]")
            if not isinstance(lay, DenseLayer):
                raise NetworkFormatError(f"{name}.inner[{i}]: nested residual blocks unsupported")
            inner.append(lay)
        if kind == "residual_identity":
            return ResidualBlock(tuple(inner))
        return ResidualBlock(tuple(inner),
                             _as_matrix(doc["shortcut_weight"], f"{name}.shortcut_weight"),
                             _as_vector(doc["shortcut_bias"], f"{name}.shortcut_bias"))
    raise NetworkFormatError(f"{name}: unknown layer kind {kind!r}")


def network_to_dict(net: AnyNetwork) -> dict:
    subs = subnetworks(net)
    return {
        "field_kind": subs[0].field_kind,
        "input_dim": 3,
        "subnetworks": [
            {"layers": [_layer_to_json(l) for l in sub.layers],
             "head": {"weight": sub.head_weight.tolist(), "bias": sub.head_bias}}
            for sub in subs
        ],
    }


def save_network(net: AnyNetwork, path) -> None:
    """Shortest round-trip float repr, so float64 weights reload bit-exactly."""
    with open(path, "w") as fh:
        json.dump(network_to_dict(net), fh)
        fh.write("\n")


def network_from_dict(doc: dict, source: str = "<network>") -> AnyNetwork:
    if not isinstance(doc, dict):
        raise NetworkFormatError(f"{source}: top level must be a JSON object")
    field_kind = doc.get("field_kind", "sdf")
    if field_kind not in FIELD_KINDS:
        raise NetworkFormatError(f"{source}: field_kind must be one of {FIELD_KINDS}")
    if doc.get("input_dim", 3) != 3:
        raise NetworkFormatError(f"{source}: input_dim is fixed at 3")
    sub_docs = doc.get("subnetworks")
    if not sub_docs:
        raise NetworkFormatError(f"{source}: missing or empty 'subnetworks'")
    subs = []
    for i, sd in enumerate(sub_docs):
        name = f"{source}.subnetworks[{i}]"
        layers = [_layer_from_json(l, f"{name}.layers[{k}]")
                  for k, l in enumerate(sd.get("layers", []))]
        if not layers:
            raise NetworkFormatError(f"{name}: missing layers")
        head = sd.get("head")
        if not isinstance(head, dict) or "weight" not in head or "bias" not in head:
            raise NetworkFormatError(f"{name}: head needs 'weight' and 'bias'")
        subs.append(NetworkSpec(tuple(layers), _as_vector(head["weight"], f"{name}.head.weight"),
                                float(head["bias"]), field_kind=field_kind))
    return subs[0] if len(subs) == 1 else EnsembleSpec(tuple(subs))


def load_network(path) -> AnyNetwork:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise NetworkFormatError(f"{path}: line {exc.lineno} col {exc.colno}: {exc.msg}") from exc
    return network_from_dict(doc, source=str(path))


# ---------------------------------------------------------------------------
# flattening into the C-ABI network descriptor (include/am_b200.h, am_net_desc)

# step flags (mirror AM_STEP_* in include/am_b200.h)
STEP_SAVE_INPUT = 1        # this step's input is a residual block input (A_in, c_in)
STEP_SHORTCUT_IDENT = 2    # add the saved block input (identity shortcut)
STEP_SHORTCUT_LINEAR = 4   # add V @ saved block input (+ shortcut bias)
STEP_FIRST = 8             # input is the network input x (A = I, c = 0)
STEP_SC_FROM_INPUT = 16    # the saved block input is the network input x

# n_in, n_out, w_off, b_off, flags, v_off, vb_off, row_off, in_row_off, sin_row_off, n_sin, sub
STEP_FIELDS = 12


@dataclass
class NetBlob:
    """Flat fp64 parameter buffer + int64 step table, the layout every kernel reads.

    steps[i] = (n_in, n_out, w_off, b_off, flags, v_off, vb_off, row_off, in_row_off,
                sin_row_off, n_sin, sub); in_row_off / sin_row_off are -1 when the
                source is the network input x.
    subs[j]  = (first_step, n_steps, head_w_off, head_b_off, row_begin, n_rows)
    Rows are numbered globally in StateVector bit order (reference network.py:214).
    """

    params: np.ndarray
    steps: np.ndarray
    subs: np.ndarray
    n_bits: int
    n_subs: int
    ensemble: bool
    max_width: int

    @property
    def key_words(self) -> int:
        """uint64 words per state key: packed bits (+1 branch word for ensembles)."""
        return (self.n_bits + 63) // 64 + (1 if self.ensemble else 0)


def to_blob(net: AnyNetwork) -> NetBlob:
    params: list[np.ndarray] = []
    cursor = 0

    def put(arr) -> int:
        nonlocal cursor
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64).ravel())
        off = cursor
        params.append(a)
        cursor += a.size
        return off

    steps = []
    subs_rows = []
    row = 0
    max_width = 3
    for j, sub in enumerate(subnetworks(net)):
        first_step = len(steps)
        sub_row_begin = row
        first = True
        prev_row = -1          # row offset of the previous step's output (-1: network input)
        for lay in sub.layers:
            if isinstance(lay, DenseLayer):
                flags = STEP_FIRST if first else 0
                steps.append([lay.in_width, lay.out_width, put(lay.weight), put(lay.bias),
                              flags, -1, -1, row, prev_row, -1, 0, j])
                prev_row = row
                row += lay.out_width
                max_width = max(max_width, lay.out_width)
                first = False
                continue
            block_from_input = first
            sin_row = prev_row
            n_sin = lay.inner[0].in_width
            for k, inner in enumerate(lay.inner):
                flags = 0
                if first:
                    flags |= STEP_FIRST
                if k == 0:
                    flags |= STEP_SAVE_INPUT
                v_off = vb_off = -1
                if k == len(lay.inner) - 1:
                    if lay.shortcut_weight is None:
                        flags |= STEP_SHORTCUT_IDENT
                    else:
                        flags |= STEP_SHORTCUT_LINEAR
                        v_off = put(lay.shortcut_weight)
                        if lay.shortcut_bias is not None:
                            vb_off = put(lay.shortcut_bias)
                    if block_from_input:
                        flags |= STEP_SC_FROM_INPUT
                steps.append([inner.in_width, inner.out_width, put(inner.weight), put(inner.bias),
                              flags, v_off, vb_off, row, prev_row, sin_row, n_sin, j])
                prev_row = row
                row += inner.out_width
                max_width = max(max_width, inner.out_width)
                first = False
        subs_rows.append([first_step, len(steps) - first_step, put(sub.head_weight),
                          put([sub.head_bias]), sub_row_begin, row - sub_row_begin])
    return NetBlob(
        params=np.concatenate(params) if params else np.zeros(0),
        steps=np.asarray(steps, dtype=np.int64).reshape(-1, STEP_FIELDS),
        subs=np.asarray(subs_rows, dtype=np.int64).reshape(-1, 6),
        n_bits=row,
        n_subs=len(subs_rows),
        ensemble=isinstance(net, EnsembleSpec),
        max_width=max_width,
    )


# ---------------------------------------------------------------------------
# reference constructions (reference network.py:677-713)


def octahedron_net(c: float = 0.5, field_kind: str = "sdf") -> NetworkSpec:
    """Six-neuron net computing ||x||_1 - c; zero set is the octahedron OCT(c)."""
    rows = np.array([[1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0], [0, -1.0, 0], [0, 0, 1.0], [0, 0, -1.0]])
    return NetworkSpec((DenseLayer(rows, np.zeros(6)),), np.ones(6), -c, field_kind=field_kind)


def cube_ensemble(c: float = 0.5, shift: float = 2.0, field_kind: str = "sdf") -> EnsembleSpec:
    """Max-pool of six half-space fields ReLU(+-axis + shift) - (shift + c); zero set [-c, c]^3."""
    subs = []
    for axis in range(3):
        for sign in (1.0, -1.0):
            row = np.zeros((1, 3))
            row[0, axis] = sign
            subs.append(NetworkSpec((DenseLayer(row, np.array([shift])),), np.ones(1),
                                    -(shift + c), field_kind=field_kind))
    return EnsembleSpec(tuple(subs))


def region_count_lower_bound(widths: Sequence[int], n0: int) -> int:
    """Theorem 1 lower bound prod floor(n_l/n0)^n0 * sum_j C(n_L, j) (reference network.py:527)."""
    widths = list(widths)
    if n0 < 1 or not widths:
        raise ValueError("need n0 >= 1 and at least one layer width")
    for w in widths:
        if w < n0:
            raise ValueError(f"layer width {w} < input dimension {n0}")
    prod = 1
    for w in widths[:-1]:
        prod *= (w // n0) ** n0
    return prod * sum(math.comb(widths[-1], j) for j in range(n0 + 1))

"""Networks at the meshing boundary: duck-typed access + the C-ABI descriptor.

``march`` takes the reference package's network objects directly
(``exactmesh.network.NetworkSpec`` / ``EnsembleSpec``, reference
network.py:49-213).  Nothing here checks a class: a network is read through the
attributes those classes carry --

* ensemble: ``.subnetworks`` (a sequence of plain networks; F = max_i F_i)
* plain network: ``.layers``, ``.head_weight``, ``.head_bias``, ``.field_kind``
* dense layer: ``.weight`` (n_out, n_in), ``.bias``
* residual block: ``.inner`` (dense layers), ``.shortcut_weight`` (None =
  identity), ``.shortcut_bias``

so any object with that shape marches (the reference's, this package's
light containers below, or a user's own).  ``to_blob`` flattens it into the
step table + parameter buffer every kernel reads (include/am_b200.h).

What this module must share with the reference is a *schema*, not code: the
``np.packbits`` key of an activation state (reference network.py:214-262) and
the JSON interchange document (reference network.py:585-672).  Both are
restated here in this package's own form.  The per-point evaluators
(``forward_many``, ``state_at``, ``affine_maps``, reference network.py:352-489)
run on the GPU and live in ``evaluate.py``; they are re-exported here so the
reference's import paths keep working.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import NamedTuple, Sequence

import numpy as np

FIELD_KINDS = ("sdf", "occupancy")
DEGENERATE_NORMAL_TOL = 1e-12   # reference network.py:27


class NetworkFormatError(ValueError):
    """A network document or object violates the format (reference network.py:30)."""


# ---------------------------------------------------------------------------
# duck-typed structure


def is_ensemble(net) -> bool:
    return hasattr(net, "subnetworks") and not hasattr(net, "layers")


def is_residual(layer) -> bool:
    return hasattr(layer, "inner")


def subnetworks(net) -> tuple:
    """The plain networks of ``net``: its ``subnetworks`` for a max-pool ensemble, else (net,)."""
    return tuple(net.subnetworks) if is_ensemble(net) else (net,)


def dense_layers(layer) -> tuple:
    """The dense layers a hidden layer contributes, in state-bit order."""
    return tuple(layer.inner) if is_residual(layer) else (layer,)


def hidden_widths(net) -> tuple:
    return tuple(np.shape(d.weight)[0] for sub in subnetworks(net) for lay in sub.layers
                 for d in dense_layers(lay))


def n_hidden(net) -> int:
    return int(sum(hidden_widths(net)))


def _f64(value, ndim: int, what: str) -> np.ndarray:
    a = np.asarray(value, dtype=np.float64)
    if a.ndim != ndim:
        raise NetworkFormatError(f"{what}: expected {ndim}-d array, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise NetworkFormatError(f"{what}: non-finite entries")
    return a


def check_network(net) -> None:
    """Shape / finiteness / field-kind checks of any reference-shaped network (the
    invariants reference network.py:62-165 enforces at construction)."""
    subs = subnetworks(net)
    if not subs:
        raise NetworkFormatError("ensemble needs at least one subnetwork")
    kinds = {getattr(s, "field_kind", "sdf") for s in subs}
    if len(kinds) != 1:
        raise NetworkFormatError("ensemble subnetworks must share field_kind")
    if not kinds <= set(FIELD_KINDS):
        raise NetworkFormatError(f"field_kind must be one of {FIELD_KINDS}")
    for si, sub in enumerate(subs):
        where = f"subnetworks[{si}]"
        if getattr(sub, "input_dim", 3) != 3:
            raise NetworkFormatError(f"{where}: input_dim is fixed at 3")
        if not len(sub.layers):
            raise NetworkFormatError(f"{where}: network needs at least one hidden layer")
        width = 3
        for li, lay in enumerate(sub.layers):
            block_in = width
            inner = dense_layers(lay)
            if not inner:
                raise NetworkFormatError(f"{where}.layers[{li}]: residual block has no inner layers")
            for di, d in enumerate(inner):
                tag = f"{where}.layers[{li}]" + (f".inner[{di}]" if is_residual(lay) else "")
                w = _f64(d.weight, 2, f"{tag}.weight")
                b = _f64(d.bias, 1, f"{tag}.bias")
                if b.shape[0] != w.shape[0]:
                    raise NetworkFormatError(f"{tag}: bias length {b.shape[0]} != weight rows {w.shape[0]}")
                if w.shape[1] != width:
                    raise NetworkFormatError(f"{tag}: expects input width {w.shape[1]}, got {width}")
                width = w.shape[0]
            if is_residual(lay):
                tag = f"{where}.layers[{li}]"
                if lay.shortcut_weight is None:
                    if getattr(lay, "shortcut_bias", None) is not None:
                        raise NetworkFormatError(f"{tag}: shortcut bias without shortcut weight")
                    if block_in != width:
                        raise NetworkFormatError(f"{tag}: identity shortcut requires input width "
                                                 f"{block_in} == output width {width}")
                else:
                    v = _f64(lay.shortcut_weight, 2, f"{tag}.shortcut_weight")
                    if v.shape != (width, block_in):
                        raise NetworkFormatError(f"{tag}: shortcut weight shape {v.shape} != ({width}, {block_in})")
                    if getattr(lay, "shortcut_bias", None) is not None:
                        if _f64(lay.shortcut_bias, 1, f"{tag}.shortcut_bias").shape[0] != width:
                            raise NetworkFormatError(f"{tag}: shortcut bias length mismatch")
        head = _f64(sub.head_weight, 1, f"{where}.head.weight")
        if head.shape[0] != width:
            raise NetworkFormatError(f"{where}: head weight length {head.shape[0]} != last layer width {width}")
        if not math.isfinite(float(sub.head_bias)):
            raise NetworkFormatError(f"{where}: non-finite head bias")


# ---------------------------------------------------------------------------
# light containers (for networks built in this package: synth, JSON loader).
# Attribute names follow the reference so they are interchangeable with its objects.


class _Record:
    """Immutable attribute record (value semantics are not needed: networks are compared by
    their arrays, never by identity)."""

    __slots__ = ()

    def __setattr__(self, name, value):
        raise AttributeError(f"{type(self).__name__} is immutable")

    def _init(self, **fields):
        for k, v in fields.items():
            object.__setattr__(self, k, v)

    def __repr__(self):
        return f"{type(self).__name__}({', '.join(f'{k}=...' for k in self.__slots__)})"


class DenseLayer(_Record):
    """ReLU layer; ``weight`` (n_out, n_in) multiplies the input column vector."""

    __slots__ = ("weight", "bias")

    def __init__(self, weight, bias):
        self._init(weight=np.asarray(weight, dtype=np.float64), bias=np.asarray(bias, dtype=np.float64))

    in_width = property(lambda self: self.weight.shape[1])
    out_width = property(lambda self: self.weight.shape[0])
    n_hidden = out_width


class ResidualBlock(_Record):
    """ReLU(shortcut(x_in) + inner stack(x_in)); ReLU between inner layers but not after the last.
    ``shortcut_weight`` None is the identity shortcut."""

    __slots__ = ("inner", "shortcut_weight", "shortcut_bias")

    def __init__(self, inner, shortcut_weight=None, shortcut_bias=None):
        self._init(inner=tuple(inner),
                   shortcut_weight=None if shortcut_weight is None else np.asarray(shortcut_weight, np.float64),
                   shortcut_bias=None if shortcut_bias is None else np.asarray(shortcut_bias, np.float64))

    out_width = property(lambda self: self.inner[-1].weight.shape[0])
    n_hidden = property(lambda self: sum(d.weight.shape[0] for d in self.inner))


class NetworkSpec(_Record):
    """Plain ReLU field: hidden layers + scalar linear head; validated on construction."""

    __slots__ = ("layers", "head_weight", "head_bias", "field_kind", "input_dim")

    def __init__(self, layers, head_weight, head_bias, field_kind: str = "sdf", input_dim: int = 3):
        self._init(layers=tuple(layers), head_weight=np.asarray(head_weight, dtype=np.float64),
                   head_bias=float(head_bias), field_kind=field_kind, input_dim=int(input_dim))
        check_network(self)

    n_hidden = property(n_hidden)
    hidden_widths = property(hidden_widths)


class EnsembleSpec(_Record):
    """Max-pool union F = max_i F_i of plain networks (paper §5.2)."""

    __slots__ = ("subnetworks",)

    def __init__(self, subnetworks):
        self._init(subnetworks=tuple(subnetworks))
        check_network(self)

    field_kind = property(lambda self: self.subnetworks[0].field_kind)
    input_dim = property(lambda self: 3)
    n_hidden = property(n_hidden)
    n_branches = property(lambda self: len(self.subnetworks))


AnyNetwork = object   # any reference-shaped network (see module docstring)


# ---------------------------------------------------------------------------
# schema shared with the reference: state keys and planes


class StateVector(NamedTuple):
    """Label of a linear region: ``key`` = ``np.packbits`` of the activation bits in
    (subnetwork, layer, neuron) order, ``branch`` = dominating subnetwork of an ensemble
    (None for plain networks).  Same packing as reference network.py:214-262."""

    key: bytes
    n_bits: int
    branch: int | None = None

    @classmethod
    def from_bits(cls, bits, branch=None) -> "StateVector":
        b = np.asarray(bits, dtype=np.uint8).reshape(-1)
        return cls(np.packbits(b).tobytes(), int(b.size), None if branch is None else int(branch))

    def bits(self) -> np.ndarray:
        return np.unpackbits(np.frombuffer(self.key, dtype=np.uint8), count=self.n_bits)

    def flip(self, index: int) -> "StateVector":
        if not 0 <= index < self.n_bits:
            raise IndexError(f"bit index {index} out of range [0, {self.n_bits})")
        k = bytearray(self.key)
        k[index >> 3] ^= 0x80 >> (index & 7)
        return self._replace(key=bytes(k))

    def with_branch(self, branch: int) -> "StateVector":
        return self._replace(branch=int(branch))

    def __repr__(self) -> str:
        body = "".join("1" if x else "0" for x in self.bits())
        return f"StateVector({body}{'' if self.branch is None else f'|b{self.branch}'})"

    # equal to (and hashed like) any state object with the same (key, n_bits, branch) -- e.g. the
    # reference's own StateVector, so states from either side index the same sets and dicts
    def __eq__(self, other):
        try:
            return (self.key, self.n_bits, self.branch) == (other.key, other.n_bits, other.branch)
        except AttributeError:
            return NotImplemented

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    def __hash__(self):
        return hash((self.key, self.n_bits, self.branch))


class AffinePlane:
    """Affine functional x -> normal . x + offset (its zero set is a plane when normal != 0)."""

    __slots__ = ("normal", "offset")

    def __init__(self, normal, offset):
        n = np.asarray(normal, dtype=np.float64).reshape(3)
        if not (np.isfinite(n).all() and math.isfinite(offset)):
            raise ValueError("plane coefficients must be finite")
        self.normal, self.offset = n, float(offset)

    def value(self, x) -> float:
        return float(self.normal @ np.asarray(x, dtype=np.float64) + self.offset)

    @property
    def degenerate(self) -> bool:
        return float(np.linalg.norm(self.normal)) <= DEGENERATE_NORMAL_TOL

    def unit(self) -> "AffinePlane":
        s = float(np.linalg.norm(self.normal))
        if s <= DEGENERATE_NORMAL_TOL:
            raise ValueError("cannot normalize a degenerate plane")
        return AffinePlane(self.normal / s, self.offset / s)

    def __repr__(self) -> str:
        return f"AffinePlane({self.normal.tolist()}, {self.offset!r})"


@dataclass(frozen=True)
class RegionMaps:
    """Affine functionals of one linear region (reference network.py:283-309): raw neuron
    planes (N, 3) + (N,), the face functional, and for ensembles the M-1 dominance planes
    F_i - F_branch with their target subnetworks; ``state`` is the canonical label."""

    state: StateVector
    neuron_normals: np.ndarray
    neuron_offsets: np.ndarray
    face_normal: np.ndarray
    face_offset: float
    branch_normals: np.ndarray
    branch_offsets: np.ndarray
    branch_targets: tuple = ()

    @property
    def neuron_planes(self) -> list:
        return [AffinePlane(n, float(d)) for n, d in zip(self.neuron_normals, self.neuron_offsets)]

    @property
    def face_plane(self) -> AffinePlane:
        return AffinePlane(self.face_normal, float(self.face_offset))


# ---------------------------------------------------------------------------
# JSON interchange document (schema of reference network.py:585-672)
#
#   {"field_kind": k, "input_dim": 3, "subnetworks": [
#       {"layers": [L...], "head": {"weight": [...], "bias": b}}, ...]}
#   L = {"kind": "dense", "weight": [[...]], "bias": [...]}
#     | {"kind": "residual_identity", "inner": [dense L...]}
#     | {"kind": "residual_linear", "inner": [...], "shortcut_weight": [[...]], "shortcut_bias": [...]}


def _encode_layer(lay) -> dict:
    if not is_residual(lay):
        return {"kind": "dense", "weight": np.asarray(lay.weight).tolist(), "bias": np.asarray(lay.bias).tolist()}
    out = {"kind": "residual_identity" if lay.shortcut_weight is None else "residual_linear",
           "inner": [_encode_layer(d) for d in lay.inner]}
    if lay.shortcut_weight is not None:
        v = np.asarray(lay.shortcut_weight, dtype=np.float64)
        sb = getattr(lay, "shortcut_bias", None)
        out["shortcut_weight"] = v.tolist()
        out["shortcut_bias"] = (np.zeros(v.shape[0]) if sb is None else np.asarray(sb)).tolist()
    return out


def network_to_dict(net) -> dict:
    subs = subnetworks(net)
    return {"field_kind": getattr(subs[0], "field_kind", "sdf"), "input_dim": 3,
            "subnetworks": [{"layers": [_encode_layer(l) for l in s.layers],
                             "head": {"weight": np.asarray(s.head_weight).tolist(), "bias": float(s.head_bias)}}
                            for s in subs]}


def save_network(net, path) -> None:
    """Shortest round-trip float repr: float64 weights reload bit-exactly on either side."""
    with open(path, "w") as fh:
        json.dump(network_to_dict(net), fh)
        fh.write("\n")


def _need(doc: dict, key: str, where: str):
    if key not in doc:
        raise NetworkFormatError(f"{where}: missing '{key}'")
    return doc[key]


def _decode_layer(doc, where: str, nested: bool = False):
    kind = doc.get("kind") if isinstance(doc, dict) else None
    if kind == "dense":
        return DenseLayer(_f64(_need(doc, "weight", where), 2, f"{where}.weight"),
                          _f64(_need(doc, "bias", where), 1, f"{where}.bias"))
    if kind in ("residual_identity", "residual_linear") and not nested:
        inner = doc.get("inner") or []
        if not inner:
            raise NetworkFormatError(f"{where}: residual block missing 'inner'")
        layers = []
        for i, d in enumerate(inner):
            sub = f"{where}.inner[{i}]"
            if not isinstance(d, dict) or d.get("kind") != "dense":
                raise NetworkFormatError(f"{sub}: nested residual blocks unsupported")
            layers.append(_decode_layer(d, sub, nested=True))
        if kind == "residual_identity":
            return ResidualBlock(layers)
        return ResidualBlock(layers, _f64(_need(doc, "shortcut_weight", where), 2, f"{where}.shortcut_weight"),
                             _f64(_need(doc, "shortcut_bias", where), 1, f"{where}.shortcut_bias"))
    raise NetworkFormatError(f"{where}: unknown layer kind {kind!r}")


def network_from_dict(doc, source: str = "<network>"):
    if not isinstance(doc, dict):
        raise NetworkFormatError(f"{source}: top level must be a JSON object")
    kind = doc.get("field_kind", "sdf")
    if kind not in FIELD_KINDS:
        raise NetworkFormatError(f"{source}: field_kind must be one of {FIELD_KINDS}")
    if doc.get("input_dim", 3) != 3:
        raise NetworkFormatError(f"{source}: input_dim is fixed at 3")
    docs = doc.get("subnetworks")
    if not docs:
        raise NetworkFormatError(f"{source}: missing or empty 'subnetworks'")
    subs = []
    for i, sd in enumerate(docs):
        where = f"{source}.subnetworks[{i}]"
        layers = [_decode_layer(l, f"{where}.layers[{k}]") for k, l in enumerate(sd.get("layers") or [])]
        if not layers:
            raise NetworkFormatError(f"{where}: missing layers")
        head = sd.get("head")
        if not isinstance(head, dict) or "weight" not in head or "bias" not in head:
            raise NetworkFormatError(f"{where}: head needs 'weight' and 'bias'")
        subs.append(NetworkSpec(layers, _f64(head["weight"], 1, f"{where}.head.weight"), float(head["bias"]),
                                field_kind=kind))
    return subs[0] if len(subs) == 1 else EnsembleSpec(subs)


def load_network(path):
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise NetworkFormatError(f"{path}: line {exc.lineno} col {exc.colno}: {exc.msg}") from exc
    return network_from_dict(doc, source=str(path))


# ---------------------------------------------------------------------------
# the C-ABI network descriptor (include/am_b200.h, am_net_desc)

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
    Rows are numbered globally in StateVector bit order.
    """

    params: np.ndarray
    steps: np.ndarray
    subs: np.ndarray
    n_bits: int
    n_subs: int
    ensemble: bool
    max_width: int
    field_kind: str = "sdf"

    @property
    def key_words(self) -> int:
        """uint64 words per state key: packed bits (+1 branch word for ensembles)."""
        return (self.n_bits + 63) // 64 + (1 if self.ensemble else 0)


def to_blob(net) -> NetBlob:
    """Flatten any reference-shaped network (validated with ``check_network``)."""
    check_network(net)
    return _walk_blob(net, None)


def param_chunks(net) -> list:
    """The parameter arrays of ``net`` in descriptor order, as given (no copies): [(offset, array)].
    A batch of shapes compares these against the base network's to find the per-shape entries
    (arrays shared by identity are skipped without a comparison)."""
    out: list = []
    _walk_blob(net, out)
    return out


def _walk_blob(net, record):
    chunks: list = []
    size = 0

    def put(arr) -> int:
        nonlocal size
        if record is not None:
            a = arr if isinstance(arr, np.ndarray) else np.asarray(arr, dtype=np.float64)
            record.append((size, a))
            size += a.size
            return size - a.size
        a = np.asarray(arr, dtype=np.float64).reshape(-1)
        chunks.append(a)
        size += a.size
        return size - a.size

    steps, subs = [], []
    row = 0
    widest = 3
    for j, sub in enumerate(subnetworks(net)):
        first_step, row_begin = len(steps), row
        prev = -1                      # row offset of the previous step's output (-1: the input x)
        for lay in sub.layers:
            inner = dense_layers(lay)
            at_input = prev == -1      # this layer reads the network input
            block_src = prev
            for k, d in enumerate(inner):
                w = np.asarray(d.weight, dtype=np.float64)
                flags = STEP_FIRST if prev == -1 else 0
                v_off = vb_off = -1
                sin_row, n_sin = -1, 0
                if is_residual(lay):
                    sin_row, n_sin = block_src, np.shape(inner[0].weight)[1]
                    if k == 0:
                        flags |= STEP_SAVE_INPUT
                    if k == len(inner) - 1:
                        if lay.shortcut_weight is None:
                            flags |= STEP_SHORTCUT_IDENT
                        else:
                            flags |= STEP_SHORTCUT_LINEAR
                            v_off = put(lay.shortcut_weight)
                            if getattr(lay, "shortcut_bias", None) is not None:
                                vb_off = put(lay.shortcut_bias)
                        if at_input:
                            flags |= STEP_SC_FROM_INPUT
                steps.append([w.shape[1], w.shape[0], put(w), put(d.bias), flags, v_off, vb_off, row, prev,
                              sin_row, n_sin, j])
                prev = row
                row += w.shape[0]
                widest = max(widest, w.shape[0])
        subs.append([first_step, len(steps) - first_step, put(sub.head_weight), put([float(sub.head_bias)]),
                     row_begin, row - row_begin])
    if record is not None:
        return None
    return NetBlob(
        params=np.concatenate(chunks) if chunks else np.zeros(0),
        steps=np.asarray(steps, dtype=np.int64).reshape(-1, STEP_FIELDS),
        subs=np.asarray(subs, dtype=np.int64).reshape(-1, 6),
        n_bits=row, n_subs=len(subs), ensemble=is_ensemble(net), max_width=widest,
        field_kind=getattr(subnetworks(net)[0], "field_kind", "sdf"),
    )


# ---------------------------------------------------------------------------
# reference constructions (reference network.py:677-713) and the region-count bound


def octahedron_net(c: float = 0.5, field_kind: str = "sdf") -> NetworkSpec:
    """||x||_1 - c as one 6-neuron layer (ReLU(x) + ReLU(-x) per axis); zero set OCT(c)."""
    rows = np.kron(np.eye(3), np.array([[1.0], [-1.0]]))
    return NetworkSpec([DenseLayer(rows, np.zeros(6))], np.ones(6), -c, field_kind=field_kind)


def cube_ensemble(c: float = 0.5, shift: float = 2.0, field_kind: str = "sdf") -> EnsembleSpec:
    """Max-pool of six half-space fields ReLU(+-x_k + shift) - (shift + c); zero set [-c, c]^3."""
    rows = np.kron(np.eye(3), np.array([[1.0], [-1.0]]))
    return EnsembleSpec([NetworkSpec([DenseLayer(r[None, :], [shift])], [1.0], -(shift + c), field_kind=field_kind)
                         for r in rows])


def region_count_lower_bound(widths: Sequence[int], n0: int) -> int:
    """Theorem-1 bound prod_{l<L} floor(n_l/n0)^n0 * sum_{j<=n0} C(n_L, j) (reference network.py:504-526)."""
    widths = list(widths)
    if n0 < 1 or not widths:
        raise ValueError("need n0 >= 1 and at least one layer width")
    if min(widths) < n0:
        raise ValueError(f"layer width {min(widths)} < input dimension {n0}")
    return math.prod((w // n0) ** n0 for w in widths[:-1]) * sum(math.comb(widths[-1], j) for j in range(n0 + 1))


def __getattr__(name):
    # GPU-backed evaluators (reference network.py:352-499, 528-570) live in evaluate.py
    if name in ("forward_many", "forward", "state_at", "state_at_many", "affine_maps", "grad_input",
                "check_unique_planes"):
        from . import evaluate
        return getattr(evaluate, name)
    raise AttributeError(name)

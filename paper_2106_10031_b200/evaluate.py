"""Per-point and per-state evaluators on the GPU (reference network.py:352-570).

``forward_many`` / ``forward`` / ``state_at_many`` / ``state_at`` /
``affine_maps`` / ``grad_input`` keep the reference's module-level signatures
and return numpy values, but every evaluation runs in the engine's sm_100a
kernels (``am_forward``, ``am_affine_maps``: the same DMMA composition the
march uses, so a state, plane or field value seen here is exactly the one the
marcher saw).  ``check_unique_planes`` runs the O(m^2) proportional-plane
diagnostic in ``am_unique_planes``.  There is no CPU path: without the library
or a device these raise ``NativeUnavailable``.

An evaluation engine per architecture is kept (small batch, no march buffers);
a network of the same architecture only re-uploads its weights.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np

from . import _native
from .network import AffinePlane, RegionMaps, StateVector, to_blob

_EVAL: "OrderedDict[tuple, object]" = OrderedDict()
_EVAL_MAX = 4


def eval_engine(net):
    """A small engine for ``net`` (cached per architecture and device; weights re-uploaded)."""
    import torch
    from .engine import Engine, _require_cuda, architecture_key
    _require_cuda()
    blob = to_blob(net)
    key = (architecture_key(blob), torch.cuda.current_device())
    eng = _EVAL.get(key)
    if eng is None:
        eng = Engine(net, max_cells=4096, batch_cells=2048)
        _EVAL[key] = eng
        while len(_EVAL) > _EVAL_MAX:
            _EVAL.popitem(last=False)
    else:
        if eng.net is not net:
            eng.load_network(net, blob)
        _EVAL.move_to_end(key)
    return eng


def _points(pts) -> np.ndarray:
    p = np.asarray(pts, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 3:
        raise ValueError(f"expected (M, 3) points, got shape {p.shape}")
    return np.ascontiguousarray(p)


def words_to_bits(words: np.ndarray, n_bits: int) -> np.ndarray:
    """MSB-first uint64 key words (n, >= ceil(n_bits/64)) -> (n, n_bits) uint8 bits."""
    w = np.ascontiguousarray(np.asarray(words).view(np.uint64)[:, :(n_bits + 63) // 64])
    by = w.astype(">u8").view(np.uint8).reshape(len(w), -1)
    return np.unpackbits(by, axis=1, count=n_bits)


def states_to_words(states, n_bits: int, ensemble: bool) -> np.ndarray:
    """StateVectors (or any objects with .key / .branch) -> int64 key words (n, KW)."""
    bw = (n_bits + 63) // 64
    out = np.zeros((len(states), bw + (1 if ensemble else 0)), dtype=np.uint64)
    for i, s in enumerate(states):
        if s.n_bits != n_bits:
            raise ValueError(f"state has {s.n_bits} bits, network has {n_bits} hidden neurons")
        by = np.zeros(bw * 8, dtype=np.uint8)
        by[:len(s.key)] = np.frombuffer(s.key, dtype=np.uint8)
        out[i, :bw] = by.view(">u8")
        if ensemble:
            if s.branch is None:
                raise ValueError("ensemble state needs a valid branch index")
            out[i, bw] = s.branch
    return out.view(np.int64)


def packbits_to_words(keys: np.ndarray, branch: np.ndarray | None, n_bits: int) -> np.ndarray:
    """Packbits key rows (n, nbytes) (+ branch column) -> int64 key words (n, KW)."""
    bw = (n_bits + 63) // 64
    keys = np.asarray(keys, dtype=np.uint8).reshape(len(keys), -1)
    by = np.zeros((len(keys), bw * 8), dtype=np.uint8)
    by[:, :keys.shape[1]] = keys
    w = by.view(">u8").astype(np.uint64)
    if branch is not None:
        w = np.concatenate([w, np.asarray(branch, dtype=np.uint64).reshape(-1, 1)], axis=1)
    return np.ascontiguousarray(w).view(np.int64)


def forward_many(net, pts) -> np.ndarray:
    """F at a batch of points (M, 3) -> (M,) (reference network.py:366-380); occupancy nets
    return the pre-sigmoid logit.  Raises FloatingPointError on NaN like the reference."""
    p = _points(pts)
    if not len(p):
        return np.empty(0)
    out = eval_engine(net).forward(p).cpu().numpy()
    if np.isnan(out).any():
        raise FloatingPointError("forward evaluation produced NaN")
    return out


def forward(net, x) -> float:
    return float(forward_many(net, np.asarray(x, dtype=np.float64).reshape(1, 3))[0])


def state_at_many(net, pts):
    """(bits (M, N) uint8, branch (M,) or None) of the regions containing the points
    (reference network.py:383-395; pre-activation exactly 0 is bit 0, ties -> lowest branch)."""
    p = _points(pts)
    eng = eval_engine(net)
    n_bits = eng.blob.n_bits
    if not len(p):
        return np.zeros((0, n_bits), np.uint8), (np.zeros(0, np.int64) if eng.blob.ensemble else None)
    _, keys = eng.forward(p, keys=True)
    k = keys.cpu().numpy()
    bits = words_to_bits(k, n_bits)
    return bits, (k[:, (n_bits + 63) // 64].astype(np.int64) if eng.blob.ensemble else None)


def state_at(net, x) -> StateVector:
    bits, br = state_at_many(net, np.asarray(x, dtype=np.float64).reshape(1, 3))
    return StateVector.from_bits(bits[0], None if br is None else int(br[0]))


def affine_maps_words(net, words: np.ndarray):
    """Device composition of many states: (canonical words (n, KW), raw neuron planes
    (n, N, 4) as (nx, ny, nz, c), face planes (n, M, 4)) as numpy arrays."""
    eng = eval_engine(net)
    words = np.ascontiguousarray(np.asarray(words).view(np.int64).reshape(len(words), -1))
    if not len(words):
        return words, np.zeros((0, eng.blob.n_bits, 4)), np.zeros((0, eng.blob.n_subs, 4))
    canon, planes, faces = eng.affine_maps(words)
    return canon.cpu().numpy(), planes.cpu().numpy(), faces.cpu().numpy()


def face_planes_words(net, words: np.ndarray) -> np.ndarray:
    """Raw face functional (n, 4) of each state (its branch's for ensembles) -- FacePolygon.plane."""
    eng = eval_engine(net)
    words = np.ascontiguousarray(np.asarray(words).view(np.int64).reshape(len(words), -1))
    if not len(words):
        return np.zeros((0, 4))
    _, _, faces = eng.affine_maps(words)
    if eng.blob.ensemble:
        import torch
        br = torch.as_tensor(words[:, (eng.blob.n_bits + 63) // 64], device=faces.device)
        faces = faces[torch.arange(len(words), device=faces.device), br]
    else:
        faces = faces[:, 0]
    return faces.cpu().numpy()


def affine_maps(net, s) -> RegionMaps:
    """Neuron planes, face plane (and dominance planes for ensembles) of the region labelled
    by s, with its canonical state (reference network.py:446-489)."""
    eng = eval_engine(net)
    b = eng.blob
    ens = b.ensemble
    if ens and (s.branch is None or not 0 <= s.branch < b.n_subs):
        raise ValueError("ensemble state needs a valid branch index")
    canon, planes, faces = affine_maps_words(net, states_to_words([s], b.n_bits, ens))
    bits = words_to_bits(canon, b.n_bits)[0]
    P, F = planes[0], faces[0]
    if ens:
        j = int(s.branch)
        others = tuple(i for i in range(b.n_subs) if i != j)
        dom = F[list(others)] - F[j]
        return RegionMaps(StateVector.from_bits(bits, j), P[:, :3].copy(), P[:, 3].copy(), F[j, :3].copy(),
                          float(F[j, 3]), dom[:, :3].reshape(-1, 3), dom[:, 3].copy(), others)
    return RegionMaps(StateVector.from_bits(bits), P[:, :3].copy(), P[:, 3].copy(), F[0, :3].copy(), float(F[0, 3]),
                      np.empty((0, 3)), np.empty(0), ())


def grad_input(net, x) -> np.ndarray:
    """Input gradient of F at x = face normal of the containing region (reference network.py:492-499)."""
    return affine_maps(net, state_at(net, x)).face_normal.copy()


def unique_plane_pairs(H: np.ndarray, tol: float = 1e-9) -> list:
    """Pairs (i < j) of rows of H (m, 4) = (normal, offset) proportional within chord tol, on the
    GPU (am_unique_planes)."""
    import torch
    H = np.ascontiguousarray(np.asarray(H, dtype=np.float64).reshape(-1, 4))
    m = len(H)
    if m < 2:
        return []
    from .engine import _require_cuda
    _require_cuda()
    lib = _native.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    d_h = torch.as_tensor(H).to(dev)
    cap = 1 << 16
    while True:
        d_pairs = torch.empty((cap, 2), dtype=torch.int32, device=dev)
        n = ctypes.c_int64()
        _native.check(lib.am_unique_planes(d_h.data_ptr(), m, float(tol), d_pairs.data_ptr(), cap,
                                           ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
                                           ctypes.byref(n)), "am_unique_planes")
        if n.value <= cap:
            break
        cap = int(n.value)
    pr = d_pairs[:n.value].cpu().numpy().astype(np.int64)
    order = np.lexsort((pr[:, 1], pr[:, 0]))
    return [(int(a), int(b)) for a, b in pr[order]]


def check_unique_planes(cells, tol: float = 1e-9) -> list:
    """Pairs of cells whose face planes are proportional within angle tol (reference
    network.py:528-570): cells = [(state, AffinePlane), ...]."""
    H = np.array([[*np.asarray(p.normal, dtype=np.float64), float(p.offset)] for _, p in cells]).reshape(-1, 4)
    return unique_plane_pairs(H, tol)


__all__ = ["forward_many", "forward", "state_at_many", "state_at", "affine_maps", "grad_input",
           "check_unique_planes", "unique_plane_pairs", "eval_engine", "AffinePlane"]

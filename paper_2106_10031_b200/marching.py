"""Analytic marching on the GPU -- the drop-in for the reference's meshing path.

``march(net, MarchConfig) -> MarchResult`` keeps the reference signature
(reference marching.py:304-362): a ReLU MLP (plain, residual-shortcut or
max-pool ensemble) in; polygon faces, their vertices and the visited
activation states out.  Internally the marching loop is a breadth-first wave
of activation-state bitmasks on the device (see ``engine.py`` and
``csrc/am_engine.cu``); MarchResult keeps everything as arrays and builds the
reference's per-polygon objects lazily.
"""

from __future__ import annotations

import json
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from .engine import PROBE_DELTA, TOL_CELL, TOL_ONPLANE, TOL_WELD, Engine, architecture_key
from .network import AffinePlane, AnyNetwork, EnsembleSpec, StateVector, subnetworks, to_blob
from .meshes import to_host
from .seeding import sample_seeds

DEFAULT_BBOX = ((-1.2, -1.2, -1.2), (1.2, 1.2, 1.2))   # reference cells.py:37

PLANE_NEURON = 0   # reference cells.py:39-41
PLANE_BRANCH = 1
PLANE_BBOX = 2


@dataclass(frozen=True)
class PlaneRef:
    """Cell boundary plane: neuron (global bit), branch target, or box face (reference cells.py:44)."""

    kind: int
    index: int

    def __repr__(self) -> str:
        tag = {PLANE_NEURON: "neuron", PLANE_BRANCH: "branch", PLANE_BBOX: "bbox"}[self.kind]
        return f"{tag}:{self.index}"


@dataclass(frozen=True)
class FacePolygon:
    """Ordered vertex loop of one analytic face (reference cells.py:91)."""

    state: StateVector
    vertices: np.ndarray
    plane: AffinePlane | None
    edge_transitions: tuple

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def touches_bbox(self) -> bool:
        return any(r.kind == PLANE_BBOX for refs in self.edge_transitions for r in refs)

    def edge_midpoints(self) -> np.ndarray:
        v = self.vertices
        return 0.5 * (v + np.roll(v, -1, axis=0))


@dataclass
class MarchConfig:
    """reference marching.py:52-75 (``threads`` is accepted for API compatibility;
    the GPU engine's parallelism is the whole wave)."""

    bbox: tuple = DEFAULT_BBOX
    seeds: int = 64
    scheme: str = "dichotomy"
    threads: int = 1
    mode: str = "pivot"
    max_cells: int = 10_000_000
    rng_seed: int = 0
    tol_cell: float = TOL_CELL
    tol_weld: float = TOL_WELD
    seed_points: np.ndarray | None = None
    unique_planes_limit: int = 3000
    probe_delta: float = PROBE_DELTA
    batch_cells: int = 0        # GPU: cells composed per batch (0 = from memory budget)
    mem_budget: int = 0         # GPU: bytes for per-batch plane buffers (0 = 2 GiB)
    precision: str = "fp64"     # "fp32": fp32-precision planes (pair with FP32_TOLERANCES)

    def __post_init__(self):
        if self.precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        if self.max_cells < 1:
            raise ValueError("max_cells must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.mode not in ("pivot", "naive"):
            raise ValueError("mode must be 'pivot' or 'naive'")


@dataclass
class MarchReport:
    """reference marching.py:78-103; pivot_fallbacks is always 0 (no pivot walk on the GPU)."""

    cells_visited: int = 0
    faces_emitted: int = 0
    empty_faces: int = 0
    open_edges: int = 0
    seconds: float = 0.0
    unique_plane_violations: int | None = None
    pivot_fallbacks: int = 0
    seeds_used: int = 0
    capped: bool = False
    threads: int = 1
    waves: int = 0
    overflow: int = 0

    def to_json(self) -> str:
        return json.dumps({k: getattr(self, k) for k in (
            "cells_visited", "faces_emitted", "empty_faces", "open_edges", "seconds",
            "unique_plane_violations", "pivot_fallbacks", "seeds_used", "capped", "threads")})


def words_to_packbits(words: np.ndarray, n_bits: int, ensemble: bool):
    """MSB-first uint64 key words -> (np.packbits bytes, branch) exactly as the reference keys."""
    words = np.asarray(words).view(np.uint64).reshape(len(words), -1)
    bw = (n_bits + 63) // 64
    nbytes = (n_bits + 7) // 8
    be = words[:, :bw].astype(">u8").view(np.uint8).reshape(len(words), bw * 8)[:, :nbytes]
    branch = words[:, -1].astype(np.int64) if ensemble else np.full(len(words), -1, np.int64)
    return np.ascontiguousarray(be), branch


@dataclass
class MarchResult:
    """Array form of the reference's MarchResult (reference marching.py:106-149).

    keys (C, nbytes) packbits states of every visited cell (empty faces
    included), sorted by (key, branch) as the reference sorts; nverts (C,)
    (0 = empty face); verts (V, 3); edge_nrefs (V,); edge_refs (R, 2) as
    (kind, index).  Integer arrays are int32.
    """

    keys: np.ndarray
    branch: np.ndarray
    nverts: np.ndarray
    verts: np.ndarray
    edge_nrefs: np.ndarray
    edge_refs: np.ndarray
    report: MarchReport
    n_bits: int
    seeds: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    _polys: list | None = None
    # device copies of (nverts, verts) kept by march() so welded_mesh() welds in HBM without
    # sending the soup back to the GPU (None: host arrays only)
    _dev: tuple | None = field(default=None, repr=False)

    @property
    def has_face(self) -> np.ndarray:
        return self.nverts > 0

    def state(self, i: int) -> StateVector:
        b = int(self.branch[i])
        return StateVector(self.keys[i].tobytes(), self.n_bits, None if b < 0 else b)

    @property
    def polygons(self) -> list:
        """Reference-style FacePolygon list (built lazily; O(cells) Python objects)."""
        if self._polys is None:
            out = []
            offs = np.concatenate([[0], np.cumsum(np.maximum(self.nverts, 0))])
            roffs = np.concatenate([[0], np.cumsum(self.edge_nrefs)])
            for i in range(len(self.nverts)):
                n = int(self.nverts[i])
                if n <= 0:
                    continue
                v0 = int(offs[i])
                trans = []
                for e in range(n):
                    a, b = int(roffs[v0 + e]), int(roffs[v0 + e + 1])
                    trans.append(tuple(PlaneRef(int(k), int(x)) for k, x in self.edge_refs[a:b]))
                out.append(FacePolygon(self.state(i), self.verts[v0:v0 + n], None, tuple(trans)))
            self._polys = out
        return self._polys

    def polygon_soup(self):
        from .meshes import PolygonMesh
        nv = self.nverts[self.nverts > 0].astype(np.int64)
        off = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
        return PolygonMesh(self.verts.copy(), None, None, face_off=off, face_idx=np.arange(off[-1], dtype=np.int64))

    def welded_mesh(self, tol: float = TOL_WELD):
        """reference marching.py:126-127 weld(polygon_soup(), tol), welded on the GPU straight
        from the CSR soup (no per-loop Python objects on the way in).  A result of march() still
        holds its soup in HBM: the loops are formed and welded there and only the welded mesh
        comes back."""
        from .meshes import PolygonMesh, weld_arrays, weld_device, to_host
        if self._dev is not None:
            import torch
            dn, dv = self._dev
            nv = dn[dn > 0].to(torch.int64)
            off = torch.zeros(nv.numel() + 1, dtype=torch.int64, device=dv.device)
            torch.cumsum(nv, 0, out=off[1:])
            idx = torch.arange(dv.shape[0], dtype=torch.int64, device=dv.device)
            kept, foff, fidx, _, _, nd = weld_device(dv, off, idx, tol)
            kept_h, foff_h = to_host([kept, foff])
            (fidx_h,) = to_host([fidx[:int(foff_h[-1])]])
            return PolygonMesh(kept_h, None, None, nd, face_off=foff_h, face_idx=fidx_h)
        nv = self.nverts[self.nverts > 0].astype(np.int64)
        off = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
        kept, foff, fidx, _, nd = weld_arrays(self.verts, off, np.arange(off[-1], dtype=np.int64), tol)
        return PolygonMesh(kept, None, None, nd, face_off=foff, face_idx=fidx)

    def face_multiset(self, decimals: int = 10):
        """Order-independent fingerprint (reference marching.py:139-149)."""
        out = []
        for poly in self.polygons:
            vs = frozenset(map(tuple, np.round(poly.vertices, decimals)))
            out.append((poly.state.key, poly.state.branch, vs))
        out.sort(key=lambda t: (t[0], -1 if t[1] is None else t[1], sorted(t[2])))
        return out


def refs_to_kind_index(ids: np.ndarray, n_bits: int, n_subs: int) -> np.ndarray:
    """Global plane ids (neuron < n_bits <= branch < n_bits + n_subs <= bbox) -> (kind, index)
    pairs, int32 (R, 2)."""
    ids = np.asarray(ids, dtype=np.int32)
    out = np.empty((len(ids), 2), dtype=np.int32)
    g1, g2 = ids >= n_bits, ids >= n_bits + n_subs
    out[:, 0] = g1
    out[:, 0] += g2
    out[:, 1] = ids
    np.subtract(out[:, 1], n_bits, out=out[:, 1], where=g1)
    np.subtract(out[:, 1], n_subs, out=out[:, 1], where=g2)
    return out


def device_results_to_host(eng: Engine):
    """Sorted device results in the reference's representations, converted on the GPU and copied
    once into pinned host memory: (counts, packbits keys (C, nbytes) uint8, branch (C,), extra
    key word (C,) or None, nverts, verts, edge_nrefs, edge_refs (R, 2) (kind, index))."""
    import torch
    c, keys, nverts, verts, enr, erefs = eng.results_device()
    eng.last_results_device = (c, keys, nverts, verts, enr, erefs)
    b = eng.blob
    nb, ns = b.n_bits, b.n_subs
    bw, nbytes = (nb + 63) // 64, (nb + 7) // 8
    n = keys.shape[0]
    # MSB-first words -> big-endian bytes == np.packbits of the state bits
    kbytes = keys[:, :bw].contiguous().view(torch.uint8).view(n, bw, 8).flip(-1).reshape(n, bw * 8)[:, :nbytes]
    g1, g2 = erefs >= nb, erefs >= nb + ns
    refs = torch.stack([g1.to(torch.int32) + g2.to(torch.int32),
                        erefs - nb * g1.to(torch.int32) - ns * g2.to(torch.int32)], dim=1)
    branch = keys[:, bw] if b.ensemble else None
    shape = keys[:, eng.kw - 1] if getattr(eng, "n_shapes", 1) > 1 else None

    ts = [kbytes, nverts, verts, enr, refs] + [t for t in (branch, shape) if t is not None]
    hk, hn, hv, he, hr, *rest = to_host(ts)
    br = rest.pop(0) if branch is not None else None
    sh = rest.pop(0) if shape is not None else None
    hbr = br.astype(np.int64) if br is not None else np.full(n, -1, np.int64)
    return c, hk, hbr, sh, hn, hv, he, hr


def collect_result(eng: Engine, seeds: np.ndarray, t0: float, waves: int, threads: int = 1,
                   keep_device: bool = False) -> MarchResult:
    """Sorted results (GPU sort + gathers, am_result_copy_device), converted to the reference's
    representations on the device, one pinned copy per array."""
    c, kb, branch, _, hn, hv, he, hr = device_results_to_host(eng)
    dev = None
    if keep_device:
        _, _, dn, dv, _, _ = eng.last_results_device
        dev = (dn, dv)
    rep = MarchReport(cells_visited=c["cells"], faces_emitted=c["faces"], empty_faces=c["empty"],
                      open_edges=c["open_edges"], seconds=time.perf_counter() - t0, seeds_used=len(seeds),
                      capped=bool(c["capped"]), threads=threads, waves=waves, overflow=c["overflow"])
    return MarchResult(kb, branch, hn, hv, he, hr, rep, eng.blob.n_bits, seeds, _dev=dev)


_ENGINES: "OrderedDict[tuple, Engine]" = OrderedDict()
ENGINE_CACHE_SIZE = 2


def clear_engine_cache():
    """Drop the engines march() keeps for reuse (frees their device memory)."""
    _ENGINES.clear()


def _engine_for(net: AnyNetwork, config: MarchConfig) -> Engine:
    """An engine for this architecture and configuration: cached ones are reused with the new
    weights uploaded (buffers, TMA descriptors and captured graphs do not depend on values)."""
    import torch
    blob = to_blob(net)
    key = (architecture_key(blob), tuple(map(tuple, config.bbox)), config.max_cells, config.tol_cell,
           config.tol_weld, config.probe_delta, config.batch_cells, config.mem_budget, config.precision,
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(net, bbox=config.bbox, max_cells=config.max_cells, tol_cell=config.tol_cell,
                     tol_weld=config.tol_weld, probe_delta=config.probe_delta,
                     batch_cells=config.batch_cells, mem_budget=config.mem_budget, precision=config.precision)
        _ENGINES[key] = eng
        while len(_ENGINES) > ENGINE_CACHE_SIZE:
            _ENGINES.popitem(last=False)
    else:
        eng.load_network(net, blob)
        eng.reset()
        _ENGINES.move_to_end(key)
    return eng


def march(net: AnyNetwork, config: MarchConfig | None = None, engine: Engine | None = None) -> MarchResult:
    """Extract every analytic face reachable from the seeds (reference marching.py:304-362)."""
    config = config or MarchConfig()
    t0 = time.perf_counter()
    eng = engine or _engine_for(net, config)
    if config.seed_points is not None:
        seeds = np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)
    else:
        seeds = sample_seeds(eng, config.seeds, config.bbox, scheme=config.scheme, rng_seed=config.rng_seed)
    eng.seed(seeds)
    waves = eng.run()
    res = collect_result(eng, seeds, t0, waves, config.threads, keep_device=True)
    if res.report.faces_emitted <= config.unique_planes_limit:
        res.report.unique_plane_violations = None   # diagnostic not computed on the GPU path
    return res

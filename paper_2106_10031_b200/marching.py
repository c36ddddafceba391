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

import itertools
import json
import logging
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from .engine import PROBE_DELTA, TOL_CELL, TOL_ONPLANE, TOL_WELD, Engine, architecture_key
from .network import AffinePlane, AnyNetwork, StateVector, is_ensemble, subnetworks, to_blob
from .meshes import to_host
from .seeding import sample_seeds

log = logging.getLogger(__name__)

DEFAULT_BBOX = ((-1.2, -1.2, -1.2), (1.2, 1.2, 1.2))   # reference cells.py:37

PLANE_NEURON = 0   # reference cells.py:39-41
PLANE_BRANCH = 1
PLANE_BBOX = 2


@dataclass(frozen=True, eq=False)
class PlaneRef:
    """Cell boundary plane: neuron (global bit), branch target, or box face (reference cells.py:44).
    Equal to / hashed like any plane reference with the same (kind, index), the reference's
    own PlaneRef included, so the two can be looked up in each other's cells."""

    kind: int
    index: int

    def __eq__(self, other):
        try:
            return (self.kind, self.index) == (other.kind, other.index)
        except AttributeError:
            return NotImplemented

    def __hash__(self):
        return hash((self.kind, self.index))

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
    """reference marching.py:52-75.

    ``threads`` is accepted for API compatibility (the GPU engine's parallelism is the whole
    wave).  ``mode`` is validated like the reference's and recorded, but both values run the
    same face solver: the reference's pivot walk (``extract_face_pivot_checked``) and naive
    enumeration (``extract_face_naive``) define the same polygon -- the pivot walk falls back
    to naive enumeration whenever its hint does not verify (reference marching.py:247-255,
    cells.py:365-462) -- and the GPU solver computes the naive-enumeration result exactly on a
    provably sufficient candidate set (face stage).  ``pivot_fallbacks`` is
    therefore always 0."""

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
    mem_budget: int = 0         # GPU: bytes for per-batch buffers (0 = 4 GiB; 32 GiB for >= 2 MFLOP/cell nets)
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
    """reference marching.py:78-103; pivot_fallbacks is always 0 (no pivot walk on the GPU).
    ``overflow``: cells whose face exceeded the register-resident solver's limits and were
    solved by the out-of-line global-memory path (0 on every benchmark configuration)."""

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
    (kind, index).  Integer arrays are int32.  ``polygons`` builds the
    reference's FacePolygon list (with each face's raw functional as ``plane``)
    on first access; ``polygon_soup`` / ``welded_mesh`` carry the face planes
    lazily (computed on the GPU when ``face_planes`` is first read).
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
    net: object = field(default=None, repr=False)
    _polys: list | None = None
    # device copies of (nverts, verts) kept by march() so welded_mesh() welds in HBM without
    # sending the soup back to the GPU (None: host arrays only)
    _dev: tuple | None = field(default=None, repr=False)
    _planes: np.ndarray | None = field(default=None, repr=False)
    # (tol, future) of the weld march() started on a side stream while the soup was copied to the
    # host (welded_mesh(tol) with the same tolerance takes its result)
    _weld: tuple | None = field(default=None, repr=False)

    def __getstate__(self):
        # device copies and the pending background weld stay with the process that marched
        st = dict(self.__dict__)
        st["_dev"] = None
        st["_weld"] = None
        return st

    @property
    def has_face(self) -> np.ndarray:
        return self.nverts > 0

    def state(self, i: int) -> StateVector:
        b = int(self.branch[i])
        return StateVector(self.keys[i].tobytes(), self.n_bits, None if b < 0 else b)

    def face_plane_rows(self) -> np.ndarray:
        """(F, 4) raw face functional (nx, ny, nz, d) of every face, in polygon order: the
        affine map of F on the cell (reference cells.py:100 FacePolygon.plane), recomputed
        from the canonical states by the engine's composition (am_affine_maps)."""
        if self._planes is None:
            if self.net is None:
                raise ValueError("face planes need the marched network (MarchResult.net)")
            from .evaluate import face_planes_words, packbits_to_words
            sel = self.nverts > 0
            ens = is_ensemble(self.net)
            words = packbits_to_words(self.keys[sel], self.branch[sel] if ens else None, self.n_bits)
            self._planes = face_planes_words(self.net, words)
        return self._planes

    @property
    def polygons(self) -> list:
        """Reference-style FacePolygon list (built lazily; O(cells) Python objects)."""
        if self._polys is None:
            out = []
            offs = np.concatenate([[0], np.cumsum(np.maximum(self.nverts, 0))])
            roffs = np.concatenate([[0], np.cumsum(self.edge_nrefs)])
            planes = self.face_plane_rows() if self.net is not None else None
            for i in range(len(self.nverts)):
                n = int(self.nverts[i])
                if n <= 0:
                    continue
                v0 = int(offs[i])
                trans = []
                for e in range(n):
                    a, b = int(roffs[v0 + e]), int(roffs[v0 + e + 1])
                    trans.append(tuple(PlaneRef(int(k), int(x)) for k, x in self.edge_refs[a:b]))
                plane = None if planes is None else AffinePlane(planes[len(out), :3], planes[len(out), 3])
                out.append(FacePolygon(self.state(i), self.verts[v0:v0 + n], plane, tuple(trans)))
            self._polys = out
        return self._polys

    def _plane_source(self):
        return self.face_plane_rows if self.net is not None else None

    def polygon_soup(self):
        """One loop per analytic face, vertices not yet shared (reference marching.py:111-124)."""
        from .meshes import PolygonMesh
        nv = self.nverts[self.nverts > 0].astype(np.int64)
        off = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
        return PolygonMesh(self.verts.copy(), None, None, face_off=off, face_idx=np.arange(off[-1], dtype=np.int64),
                           plane_rows=self._plane_source(), _checked=True)

    def welded_mesh(self, tol: float = TOL_WELD):
        """reference marching.py:126-127 weld(polygon_soup(), tol), welded on the GPU straight
        from the CSR soup (no per-loop Python objects on the way in).  A result of march() still
        holds its soup in HBM: the loops are formed and welded there and only the welded mesh
        comes back."""
        from .meshes import PolygonMesh, weld_arrays, select_rows
        if tol < 0:
            raise ValueError("weld tolerance must be >= 0")
        if self._weld is not None and self._weld[0] == tol:
            kept_h, foff_h, fidx_h, fsrc_h, nd = self._weld[1].result()
        elif self._dev is not None:
            kept_h, foff_h, fidx_h, fsrc_h, nd = _weld_soup_device(*self._dev, tol)
        else:
            nv = self.nverts[self.nverts > 0].astype(np.int64)
            off = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
            kept_h, foff_h, fidx_h, fsrc_h, nd = weld_arrays(self.verts, off, np.arange(off[-1], dtype=np.int64), tol)
        src = self._plane_source()
        return PolygonMesh(kept_h, None, None, nd, face_off=foff_h, face_idx=fidx_h,
                           plane_rows=None if src is None else select_rows(src, fsrc_h), _checked=True)

    def face_multiset(self, decimals: int = 10):
        """Order-independent fingerprint (reference marching.py:139-149)."""
        out = []
        for poly in self.polygons:
            vs = frozenset(map(tuple, np.round(poly.vertices, decimals)))
            out.append((poly.state.key, poly.state.branch, vs))
        out.sort(key=lambda t: (t[0], -1 if t[1] is None else t[1], sorted(t[2])))
        return out


def _weld_soup_device(dn, dv, tol: float, after=None):
    """Weld the device-resident soup (sorted per-cell vertex counts dn, vertices dv) on the GPU
    and copy the welded mesh to the host: (kept, face_off, face_idx, face_src, n_dropped).  With
    ``after`` (a stream) the work runs on a side stream ordered after it."""
    import torch
    from .meshes import weld_device
    dev = dv.device
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        if after is not None:
            st = _side_stream(dev)
            st.wait_stream(after)
        with torch.cuda.stream(st):
            nv = dn[dn > 0].to(torch.int64)
            off = torch.zeros(nv.numel() + 1, dtype=torch.int64, device=dev)
            torch.cumsum(nv, 0, out=off[1:])
            idx = torch.arange(dv.shape[0], dtype=torch.int64, device=dev)
            kept, foff, fidx, fsrc, _, nd = weld_device(dv, off, idx, tol, stream=st)
            kept_h, foff_h, fsrc_h = to_host([kept, foff, fsrc])
            (fidx_h,) = to_host([fidx[:int(foff_h[-1])]])
    return kept_h, foff_h, fidx_h, fsrc_h, nd


_SIDE: dict = {}
_WELD_POOL = None


def _side_stream(dev):
    import torch
    st = _SIDE.get(dev.index)
    if st is None:
        st = _SIDE[dev.index] = torch.cuda.Stream(device=dev)
    return st


def _start_weld(dn, dv, tol: float):
    """Start the default-tolerance weld of a march's soup on a side stream from a worker thread,
    so that it overlaps the soup's device->host copies (AM_WELD_PREFETCH=0 disables)."""
    import os
    import torch
    from concurrent.futures import ThreadPoolExecutor
    global _WELD_POOL
    if os.environ.get("AM_WELD_PREFETCH", "1") == "0":
        return None
    if _WELD_POOL is None:
        _WELD_POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="am-weld")
    main = torch.cuda.current_stream(dv.device)
    return (tol, _WELD_POOL.submit(_weld_soup_device, dn, dv, tol, main))


def neighbor_state(s: StateVector, ref: PlaneRef) -> StateVector:
    """State across one boundary plane (reference marching.py:152-165): flip the neuron's bit or
    switch branch; box faces have no neighbour."""
    if ref.kind == PLANE_NEURON:
        return s.flip(ref.index)
    if ref.kind == PLANE_BRANCH:
        if s.branch is None:
            raise ValueError("branch switch on a non-ensemble state")
        return s.with_branch(ref.index)
    raise ValueError(f"no neighbor beyond the bounding box (ref {ref})")


def transition_states(s: StateVector, refs) -> list:
    """Neighbour states of an edge on possibly coincident planes (reference marching.py:168-195):
    every non-empty flip subset of the neuron planes (singles + the joint flip + the unchanged
    state beyond 3 planes), each with every branch target.  This is the host restatement of what
    the face kernel emits per edge (am_face.cu, emission)."""
    bits = [r.index for r in refs if r.kind == PLANE_NEURON]
    targets = [None] + [r.index for r in refs if r.kind == PLANE_BRANCH]
    if len(bits) > 3:
        log.warning("edge on %d coincident planes; enqueueing singles and the full flip", len(bits))
        subsets = [(b,) for b in bits] + [tuple(bits), ()]
    else:
        subsets = [c for k in range(len(bits) + 1) for c in itertools.combinations(bits, k)]
    out = []
    for sub, tgt in itertools.product(subsets, targets):
        if not sub and tgt is None:
            continue
        t = s
        for b in sub:
            t = t.flip(b)
        out.append(t if tgt is None else t.with_branch(tgt))
    return out


def vertex_residuals(net: AnyNetwork, mesh_or_result) -> np.ndarray:
    """|F| at every mesh vertex, evaluated on the GPU (reference marching.py:369-377); the
    exactness claim is max residual <= 1e-6."""
    from .evaluate import forward_many
    if isinstance(mesh_or_result, MarchResult):
        verts = mesh_or_result.verts
    else:
        verts = mesh_or_result.vertices
    if len(verts) == 0:
        return np.empty(0)
    return np.abs(forward_many(net, verts))


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


def device_results_to_host(eng: Engine, on_device=None):
    """Sorted device results in the reference's representations, converted on the GPU and copied
    once into pinned host memory: (counts, packbits keys (C, nbytes) uint8, branch (C,), extra
    key word (C,) or None, nverts, verts, edge_nrefs, edge_refs (R, 2) (kind, index))."""
    import torch
    c, keys, nverts, verts, enr, erefs = eng.results_device()
    eng.last_results_device = (c, keys, nverts, verts, enr, erefs)
    if on_device is not None:
        on_device(nverts, verts)
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
                   keep_device: bool = False, net=None) -> MarchResult:
    """Sorted results (GPU sort + gathers, am_result_copy_device), converted to the reference's
    representations on the device, one pinned copy per array."""
    dev = weld = None
    if keep_device:
        def on_device(dn, dv):
            nonlocal dev, weld
            dev = (dn, dv)
            weld = _start_weld(dn, dv, TOL_WELD)
    c, kb, branch, _, hn, hv, he, hr = device_results_to_host(eng, on_device if keep_device else None)
    rep = MarchReport(cells_visited=c["cells"], faces_emitted=c["faces"], empty_faces=c["empty"],
                      open_edges=c["open_edges"], seconds=time.perf_counter() - t0, seeds_used=len(seeds),
                      capped=bool(c["capped"]), threads=threads, waves=waves, overflow=c["overflow"])
    return MarchResult(kb, branch, hn, hv, he, hr, rep, eng.blob.n_bits, seeds, net=net if net is not None else eng.net,
                       _dev=dev, _weld=weld)


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


class MarchOverflowError(RuntimeError):
    """A cell's face exceeded the GPU face solver's limits (more than 32 polygon vertices or 64
    candidate planes); its polygon and neighbours are missing, so the mesh would have a hole."""


def check_overflow(report: MarchReport):
    """Fail loudly instead of returning a mesh with holes (report.overflow counts such cells)."""
    if report.overflow:
        raise MarchOverflowError(
            f"{report.overflow} cell(s) exceeded the face solver's limits (32 polygon vertices / 64 candidate "
            "planes); the march is incomplete")


def seed_engine(eng: Engine, seeds: np.ndarray, shapes=None):
    """Queue the refined seed states; am_seed takes at most one batch of cells per call."""
    bs = max(1, eng.batch_size)
    for o in range(0, len(seeds), bs):
        eng.seed(seeds[o:o + bs], shapes=None if shapes is None else shapes[o:o + bs])


def unique_plane_violations(res: MarchResult, tol: float = 1e-9) -> int:
    """Proportional face-plane pairs among the result's faces (reference marching.py:361-363 via
    check_unique_planes), counted on the GPU (am_unique_planes)."""
    from .evaluate import unique_plane_pairs
    if res.report.faces_emitted < 2:
        return 0
    return len(unique_plane_pairs(res.face_plane_rows(), tol))


def march(net: AnyNetwork, config: MarchConfig | None = None, engine: Engine | None = None) -> MarchResult:
    """Extract every analytic face reachable from the seeds (reference marching.py:304-366).

    Returns the face polygons plus a report; raises SeedingError ("no surface located in
    bbox") if no seed can be found; hitting ``max_cells`` returns the partial mesh with
    ``report.capped`` set.  ``engine``: an Engine of this network's architecture to march on
    (its weights are replaced by ``net``'s and its visited set cleared)."""
    config = config or MarchConfig()
    t0 = time.perf_counter()
    if engine is not None:
        engine.load_network(net)
        engine.reset()
        eng = engine
    else:
        eng = _engine_for(net, config)
    if config.seed_points is not None:
        seeds = np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)
    else:
        seeds = sample_seeds(eng, config.seeds, config.bbox, scheme=config.scheme, rng_seed=config.rng_seed)
    seed_engine(eng, seeds)
    waves = eng.run()
    res = collect_result(eng, seeds, t0, waves, config.threads, keep_device=True, net=net)
    check_overflow(res.report)
    if res.report.faces_emitted <= config.unique_planes_limit:
        res.report.unique_plane_violations = unique_plane_violations(res)
    if res.report.capped:
        log.warning("max_cells=%d reached; mesh is partial", config.max_cells)
    res.report.seconds = time.perf_counter() - t0
    return res

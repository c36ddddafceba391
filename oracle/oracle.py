"""ctypes front-end of the CPU oracle (liboracle.so, built from am_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  It restates the
reference's marching entry point (reference marching.py:304-362) and trigger
(reference seeding.py:134-162) on top of the C restatement of the per-cell
algorithm.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
sys.path.insert(0, os.path.dirname(HERE))

from paper_2106_10031_b200.network import (  # noqa: E402  (data model only)
    AnyNetwork, NetBlob, StateVector, to_blob)

SEED_TOL = 1e-7
TOL_CELL, TOL_WELD, TOL_ONPLANE, PROBE_DELTA = 1e-9, 1e-7, 1e-9, 1e-7
DEFAULT_BBOX = ((-1.2, -1.2, -1.2), (1.2, 1.2, 1.2))

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "am_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.om_net_create.restype = P
        L.om_net_create.argtypes = [P, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int]
        L.om_net_free.argtypes = [P]
        L.om_forward_many.argtypes = [P, P, ctypes.c_long, P, P]
        L.om_affine_maps.argtypes = [P, P, P, P, P]
        L.om_march.restype = P
        L.om_march.argtypes = [P, P, ctypes.c_int, P, ctypes.c_long, ctypes.c_int,
                               ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.om_result_counts.argtypes = [P, P]
        L.om_result_copy.argtypes = [P, P, P, P, P, P]
        L.om_result_free.argtypes = [P]
        L.om_key_owner.argtypes = [P, ctypes.c_long, ctypes.c_int, ctypes.c_int, P]
        L.om_canonical.argtypes = [P, P, P]
        L.om_cell_expand.restype = ctypes.c_long
        L.om_cell_expand.argtypes = [P, P, P, P, ctypes.c_long]
        L.om_weld.restype = ctypes.c_int
        L.om_weld.argtypes = [P, ctypes.c_long, P, P, ctypes.c_long, ctypes.c_double, P, P, P, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleNet:
    """A network handle for the oracle; keeps the flattened blob alive."""

    def __init__(self, net: AnyNetwork):
        self.net = net
        self.blob: NetBlob = to_blob(net)
        b = self.blob
        self._params = np.ascontiguousarray(b.params)
        self._steps = np.ascontiguousarray(b.steps)
        self._subs = np.ascontiguousarray(b.subs)
        self.h = lib().om_net_create(_ptr(self._params), _ptr(self._steps), len(self._steps),
                                     _ptr(self._subs), len(self._subs), b.n_bits, int(b.ensemble),
                                     b.max_width)
        self.kw = b.key_words

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.om_net_free(self.h)
            self.h = None

    # reference network.py:352-392
    def forward_many(self, pts) -> np.ndarray:
        pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
        out = np.empty(len(pts))
        lib().om_forward_many(self.h, _ptr(pts), len(pts), _ptr(out), None)
        return out

    def state_keys(self, pts) -> np.ndarray:
        pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
        keys = np.zeros((len(pts), self.kw), dtype=np.uint64)
        lib().om_forward_many(self.h, _ptr(pts), len(pts), None, _ptr(keys))
        return keys

    def affine_maps(self, key_words: np.ndarray):
        k = np.ascontiguousarray(key_words, dtype=np.uint64)
        canon = np.zeros(self.kw, dtype=np.uint64)
        planes = np.zeros((self.blob.n_bits, 4))
        face = np.zeros(4)
        lib().om_affine_maps(self.h, _ptr(k), _ptr(canon), _ptr(planes), _ptr(face))
        return canon, planes, face

    def grad_input(self, x) -> np.ndarray:
        key = self.state_keys(np.asarray(x).reshape(1, 3))[0]
        return self.affine_maps(key)[2][:3].copy()


# --------------------------------------------------------------- keys <-> bytes

def words_to_packbits(words: np.ndarray, n_bits: int, ensemble: bool):
    """uint64 MSB-first words (C, kw) -> (packbits bytes (C, nbytes), branch (C,))."""
    words = np.asarray(words, dtype=np.uint64).reshape(len(words), -1)
    bw = (n_bits + 63) // 64
    nbytes = (n_bits + 7) // 8
    be = words[:, :bw].astype(">u8").view(np.uint8).reshape(len(words), bw * 8)[:, :nbytes]
    branch = words[:, -1].astype(np.int64) if ensemble else np.full(len(words), -1, np.int64)
    return np.ascontiguousarray(be), branch


# ------------------------------------------------------------------- seeding
# reference seeding.py:33-131


def _seed_dichotomy(on: OracleNet, xp, xn, eps=SEED_TOL, max_iters=200, seed_tol=SEED_TOL):
    xp = np.asarray(xp, dtype=np.float64).copy()
    xn = np.asarray(xn, dtype=np.float64).copy()
    fp, fn = on.forward_many(xp)[0], on.forward_many(xn)[0]
    if not (fp > 0.0 and fn < 0.0):
        raise RuntimeError(f"need F(x_pos) > 0 > F(x_neg), got {fp} and {fn}")
    for it in range(1, max_iters + 1):
        mid = 0.5 * (xp + xn)
        fm = on.forward_many(mid)[0]
        if abs(fm) <= seed_tol:
            return mid, it
        if fm > 0.0:
            xp, fp = mid, fm
        else:
            xn, fn = mid, fm
        if fp - fn <= eps:
            return (xp, it) if abs(fp) <= abs(fn) else (xn, it)
    return (xp, max_iters) if abs(fp) <= abs(fn) else (xn, max_iters)


def _seed_sgd(on, x0, max_iters=1000, step=0.05, seed_tol=SEED_TOL):
    x = np.asarray(x0, dtype=np.float64).copy()
    f = on.forward_many(x)[0]
    cur = step
    for it in range(max_iters + 1):
        if abs(f) <= seed_tol:
            return x, it
        g = on.grad_input(x)
        gn = float(np.linalg.norm(g))
        if gn == 0.0:
            return None, it
        x_new = x - cur * np.sign(f) * g / gn
        f_new = on.forward_many(x_new)[0]
        if np.sign(f_new) != np.sign(f):
            cur *= 0.5
        x, f = x_new, f_new
    return None, max_iters


def _seed_sphere_trace(on, x0, eta=1.0, max_iters=50, seed_tol=SEED_TOL, escape_scale=12.0):
    x = np.asarray(x0, dtype=np.float64).copy()
    for it in range(max_iters + 1):
        f = on.forward_many(x)[0]
        if abs(f) <= seed_tol:
            return x, it
        if float(np.abs(x).max()) > escape_scale:
            raise RuntimeError(f"sphere tracing diverged after {it} iterations")
        x = x - eta * f * on.grad_input(x)
    return None, max_iters


def sample_seeds(on: OracleNet, count, bbox, scheme="dichotomy", rng_seed=0, retry_budget=200):
    lo = np.asarray(bbox[0], dtype=np.float64)
    hi = np.asarray(bbox[1], dtype=np.float64)
    seeds = []
    for index in range(count):
        rng = np.random.default_rng([rng_seed, index])
        found = None
        if scheme == "dichotomy":
            for _ in range(retry_budget):
                pts = rng.uniform(lo, hi, size=(64, 3))
                vals = on.forward_many(pts)
                pos = pts[vals > 0.0]
                neg = pts[vals < 0.0]
                if len(pos) and len(neg):
                    found, _ = _seed_dichotomy(on, pos[0], neg[0])
                    break
        else:
            for _ in range(retry_budget):
                x0 = rng.uniform(lo, hi, size=3)
                if scheme == "sgd":
                    res, _ = _seed_sgd(on, x0)
                else:
                    res, _ = _seed_sphere_trace(on, x0)
                if res is not None:
                    found = res
                    break
        if found is not None:
            seeds.append(found)
    if not seeds:
        raise RuntimeError("no surface located in bbox")
    return np.array(seeds)


# ------------------------------------------------------------------- march


@dataclass
class OracleResult:
    keys: np.ndarray          # (C, nbytes) packbits, sorted as the reference sorts
    branch: np.ndarray        # (C,) -1 for plain nets
    key_words: np.ndarray     # (C, kw) raw words
    has_face: np.ndarray
    nverts: np.ndarray
    verts: np.ndarray
    edge_nrefs: np.ndarray
    edge_refs: np.ndarray
    report: dict
    seeds: np.ndarray


def march(net: AnyNetwork, bbox=DEFAULT_BBOX, seeds: int = 64, scheme: str = "dichotomy",
          rng_seed: int = 0, seed_points=None, max_cells: int = 10_000_000, threads: int = 1,
          oracle_net: OracleNet | None = None) -> OracleResult:
    on = oracle_net or OracleNet(net)
    if seed_points is None:
        seed_pts = sample_seeds(on, seeds, bbox, scheme=scheme, rng_seed=rng_seed)
    else:
        seed_pts = np.asarray(seed_points, dtype=np.float64).reshape(-1, 3)
    seed_pts = np.ascontiguousarray(seed_pts)
    bb = np.array(list(bbox[0]) + list(bbox[1]), dtype=np.float64)
    L = lib()
    R = L.om_march(on.h, _ptr(seed_pts), len(seed_pts), _ptr(bb), int(max_cells), int(threads),
                   TOL_CELL, TOL_WELD, TOL_ONPLANE, PROBE_DELTA)
    counts = np.zeros(8, dtype=np.int64)
    L.om_result_counts(R, _ptr(counts))
    n_cells, n_faces, n_empty, n_verts, n_erefs, open_edges, fallbacks, capped = (int(c) for c in counts)
    kw = on.kw
    keys = np.zeros((n_cells, kw), dtype=np.uint64)
    nverts = np.zeros(n_cells, dtype=np.int32)
    verts = np.zeros((n_verts, 3))
    enr = np.zeros(n_verts, dtype=np.int32)
    erefs = np.zeros((n_erefs, 2), dtype=np.int32)
    L.om_result_copy(R, _ptr(keys), _ptr(nverts), _ptr(verts), _ptr(enr), _ptr(erefs))
    L.om_result_free(R)
    kb, branch = words_to_packbits(keys, on.blob.n_bits, on.blob.ensemble)
    report = dict(cells_visited=n_cells, faces_emitted=n_faces, empty_faces=n_empty,
                  open_edges=open_edges, pivot_fallbacks=fallbacks, capped=bool(capped),
                  seeds_used=len(seed_pts), threads=threads)
    return OracleResult(kb, branch, keys, nverts > 0, nverts.astype(np.int64), verts,
                        enr.astype(np.int64), erefs.astype(np.int64), report, seed_pts)


# ------------------------------------------------------- sharded-march stand-in

def key_owner(keys: np.ndarray, world: int) -> np.ndarray:
    """Owner rank per key (same hash as the GPU engine's key_owner)."""
    k = np.ascontiguousarray(keys, dtype=np.uint64).reshape(len(keys), -1)
    out = np.zeros(len(k), dtype=np.int32)
    lib().om_key_owner(_ptr(k), len(k), k.shape[1], int(world), _ptr(out))
    return out


class OracleShardEngine:
    """CPU stand-in with the GPU Engine's wave/outbox/push interface (tests of the sharded
    driver over gloo).  Same semantics as the engine: a set of dispatched raw keys, a set
    of visited canonical states, ownership owner(state) = hash % world."""

    def __init__(self, net, bbox=DEFAULT_BBOX, max_cells=10_000_000, rank=0, world=1, **_):
        self.on = OracleNet(net)
        self.kw = self.on.kw
        self.rank, self.world = rank, world
        self.bbox = np.array(list(bbox[0]) + list(bbox[1]), dtype=np.float64)
        self.net = net
        self.reset()

    def reset(self):
        self.seen = set()
        self.visited = set()
        self.queue = []
        self.out = []
        self.hdr = None

    def _owner(self, k):
        return int(key_owner(np.asarray(k, dtype=np.uint64).reshape(1, -1), self.world)[0])

    def _route(self, keys):
        for k in keys:
            k = np.asarray(k, dtype=np.uint64)
            if self._owner(k) == self.rank:
                t = k.tobytes()
                if t not in self.seen:
                    self.seen.add(t)
                    self.queue.append(k)
            else:
                self.out.append(k)

    def seed(self, pts):
        from paper_2106_10031_b200 import network as _n  # noqa: F401
        keys = []
        for x in np.asarray(pts, dtype=np.float64).reshape(-1, 3):
            # reference marching.py:201-213 via the oracle march of one seed with max_cells=1
            r = march(self.net, bbox=(tuple(self.bbox[:3]), tuple(self.bbox[3:])), seed_points=x.reshape(1, 3),
                      max_cells=1, oracle_net=self.on)
            keys.append(r.key_words[0])
        self._route(keys)

    def wave(self):
        todo, self.queue = self.queue, []
        new = 0
        buf = np.zeros((512, self.kw), dtype=np.uint64)
        for r in todo:
            canon = np.zeros(self.kw, dtype=np.uint64)
            lib().om_canonical(self.on.h, _ptr(np.ascontiguousarray(r)), _ptr(canon))
            if self._owner(canon) != self.rank:
                self.out.append(canon)
                continue
            ct = canon.tobytes()
            if ct in self.visited:
                continue
            self.visited.add(ct)
            self.seen.add(ct)
            new += 1
            n = lib().om_cell_expand(self.on.h, _ptr(canon), _ptr(self.bbox), _ptr(buf), len(buf))
            if n > 0:
                self._route(list(buf[:n].copy()))
        return new

    # ---- device-driven round protocol of the GPU engine (Engine.shard_*), restated on the host
    HDR_WORDS = 8

    def shard_rows(self, cap):
        return (self.HDR_WORDS + self.kw - 1) // self.kw + int(cap)

    def shard_iterate(self, iters, cap):
        visited, capped = len(self.visited), False
        if self.hdr is not None:
            h = self.hdr
            idle = not (h[:, 1].any() or h[:, 2].any() or h[:, 3].any())
            while cap < int(h[:, 4].max()):
                cap *= 2
            visited, capped = int(h[:, 5].sum()), bool(h[:, 6].any())
            if idle:
                return True, cap, visited, capped
        for _ in range(int(iters)):
            if not self.queue:
                break
            self.wave()
        return False, cap, visited, capped

    def shard_pack(self, send, cap):
        rows = self.shard_rows(cap)
        hr = rows - cap
        buf = send.numpy().view(np.uint64).reshape(self.world, rows, self.kw)
        buf[:] = 0
        counts = np.zeros(self.world, dtype=np.int64)
        rest = []
        for k in self.out:
            o = self._owner(k)
            if counts[o] < cap:
                buf[o, hr + counts[o]] = k
            else:
                rest.append(k)
            counts[o] += 1
        sent = int(np.minimum(counts, cap).sum())
        for o in range(self.world):
            h = buf[o, :hr].reshape(-1)
            h[:self.HDR_WORDS] = [min(counts[o], cap), len(self.queue), len(rest), sent, counts.max(initial=0),
                                  len(self.visited), 0, 1]
        self.out = rest

    def shard_absorb(self, recv, cap):
        rows = self.shard_rows(cap)
        hr = rows - cap
        buf = recv.numpy().view(np.uint64).reshape(self.world, rows, self.kw)
        hdr = np.stack([buf[s, :hr].reshape(-1)[:self.HDR_WORDS] for s in range(self.world)]).astype(np.int64)
        for s in range(self.world):
            self._route(list(buf[s, hr:hr + int(hdr[s, 0])].copy()))
        self.hdr = hdr

    def queue_size(self):
        return len(self.queue)

    def sample_seeds(self, count, bbox, scheme="dichotomy", rng_seed=0):
        return sample_seeds(self.on, count, bbox, scheme=scheme, rng_seed=rng_seed)

    def load_network(self, net):
        """Next network of a same-architecture batch (the stand-in just rebuilds)."""
        self.on = OracleNet(net)
        self.net = net

    def push(self, keys):
        self._route([np.asarray(k).view(np.uint64) for k in keys.numpy()])

    def visited_keys(self):
        return sorted(self.visited)


class OracleBatchShardEngine(OracleShardEngine):
    """Stand-in for a batch-of-shapes engine (n_shapes > 1): every key carries a trailing shape
    word (hashed into the owner like the GPU engine's), and a state of shape s is canonicalised
    and expanded with shape s's network."""

    def __init__(self, nets, bbox=DEFAULT_BBOX, max_cells=10_000_000, rank=0, world=1, **_):
        self.nets = list(nets)
        self.ons = [OracleNet(n) for n in self.nets]
        self.on = self.ons[0]
        self.kw = self.on.kw + 1
        self.rank, self.world = rank, world
        self.bbox = np.array(list(bbox[0]) + list(bbox[1]), dtype=np.float64)
        self.net = self.nets[0]
        self.reset()

    def seed(self, pts, shapes=None):
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
        shapes = np.zeros(len(pts), np.int64) if shapes is None else np.asarray(shapes).reshape(-1)
        keys = []
        for x, sh in zip(pts, shapes):
            r = march(self.nets[int(sh)], bbox=(tuple(self.bbox[:3]), tuple(self.bbox[3:])),
                      seed_points=x.reshape(1, 3), max_cells=1, oracle_net=self.ons[int(sh)])
            keys.append(np.append(r.key_words[0], np.uint64(sh)))
        self._route(keys)

    def wave(self):
        todo, self.queue = self.queue, []
        new = 0
        kw = self.kw - 1
        buf = np.zeros((512, kw), dtype=np.uint64)
        for r in todo:
            sh = int(r[-1])
            on = self.ons[sh]
            base = np.zeros(kw, dtype=np.uint64)
            lib().om_canonical(on.h, _ptr(np.ascontiguousarray(r[:-1])), _ptr(base))
            canon = np.append(base, np.uint64(sh))
            if self._owner(canon) != self.rank:
                self.out.append(canon)
                continue
            ct = canon.tobytes()
            if ct in self.visited:
                continue
            self.visited.add(ct)
            self.seen.add(ct)
            new += 1
            n = lib().om_cell_expand(on.h, _ptr(base), _ptr(self.bbox), _ptr(buf), len(buf))
            if n > 0:
                self._route([np.append(k, np.uint64(sh)) for k in buf[:n].copy()])
        return new

    def sample_seeds_batch(self, count, bbox, rng_seed=0):
        return [sample_seeds(on, count, bbox, "dichotomy", rng_seed) for on in self.ons]

    def visited_by_shape(self):
        out = {s: [] for s in range(len(self.nets))}
        for t in self.visited:
            w = np.frombuffer(t, dtype=np.uint64)
            out[int(w[-1])].append(w[:-1].tobytes())
        return {s: sorted(v) for s, v in out.items()}


def weld(verts, loop_off, loop_idx, tol: float = TOL_WELD):
    """reference meshes.py:89-148 on CSR loops.  Returns (kept (K,3), face_off (F+1,),
    face_idx, face_src (F,) source loop of each kept face, remap (V,), n_dropped)."""
    v = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 3)
    lo = np.ascontiguousarray(loop_off, dtype=np.int64)
    li = np.ascontiguousarray(loop_idx, dtype=np.int64)
    n, nl = len(v), len(lo) - 1
    remap = np.empty(n, np.int64)
    kept = np.empty((max(n, 1), 3), np.float64)
    face_off = np.empty(nl + 1, np.int64)
    face_idx = np.empty(max(len(li), 1), np.int64)
    face_src = np.empty(max(nl, 1), np.int64)
    counts = np.zeros(3, np.int64)
    if lib().om_weld(_ptr(v), n, _ptr(lo), _ptr(li), nl, float(tol), _ptr(remap), _ptr(kept), _ptr(face_off),
                     _ptr(face_idx), _ptr(face_src), _ptr(counts)) != 0:
        raise MemoryError("om_weld")
    nk, nf, nd = (int(x) for x in counts)
    return kept[:nk].copy(), face_off[:nf + 1].copy(), face_idx[:face_off[nf]].copy(), face_src[:nf].copy(), remap, nd

"""Thin Python handle over the C-ABI engine (one per GPU / rank).

PyTorch is plumbing here: it owns the CUDA device selection, the stream the
engine launches on, and the device tensors whose raw pointers cross the
C-ABI.  All numeric work runs in the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .network import AnyNetwork, NetBlob, NetworkFormatError, to_blob

TOL_CELL = 1e-9      # reference cells.py:33
TOL_WELD = 1e-7      # reference cells.py:35
TOL_ONPLANE = 1e-9   # reference cells.py:34
PROBE_DELTA = 1e-7   # reference marching.py:67


def _require_cuda():
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable("no CUDA device visible; the meshing path runs only on a B200")


def architecture_key(blob: NetBlob) -> tuple:
    """What an engine is built for: step / sub tables (shapes, offsets, flags) and sizes."""
    return (blob.steps.tobytes(), blob.subs.tobytes(), int(blob.n_bits), bool(blob.ensemble), len(blob.params))


class Engine:
    def __init__(self, net: AnyNetwork, bbox=((-1.2,) * 3, (1.2,) * 3), max_cells: int = 10_000_000,
                 tol_cell=TOL_CELL, tol_weld=TOL_WELD, tol_onplane=TOL_ONPLANE, probe_delta=PROBE_DELTA,
                 batch_cells: int = 0, mem_budget: int = 0, rank: int = 0, world: int = 1,
                 device: int | None = None, stream: torch.cuda.Stream | None = None, n_shapes: int = 1,
                 precision: str = "fp64"):
        _require_cuda()
        self.lib = _native.load()
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        self.stream = stream or torch.cuda.current_stream(self.dev)
        self.net = net
        self.blob: NetBlob = to_blob(net)
        b = self.blob
        self._params = np.ascontiguousarray(b.params, dtype=np.float64)
        self._steps = np.ascontiguousarray(b.steps, dtype=np.int64)
        self._subs = np.ascontiguousarray(b.subs, dtype=np.int64)
        desc = _native.NetDesc(self._params.ctypes.data, len(self._params), self._steps.ctypes.data,
                               len(self._steps), self._subs.ctypes.data, len(self._subs), b.n_bits,
                               int(b.ensemble))
        p = _native.MarchParams()
        p.bbox_lo[:] = [float(v) for v in bbox[0]]
        p.bbox_hi[:] = [float(v) for v in bbox[1]]
        p.tol_cell, p.tol_weld, p.tol_onplane, p.probe_delta = tol_cell, tol_weld, tol_onplane, probe_delta
        p.max_cells, p.batch_cells, p.mem_budget = int(max_cells), int(batch_cells), int(mem_budget)
        p.rank, p.world = int(rank), int(world)
        p.n_shapes = int(n_shapes)
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        p.precision = 1 if precision == "fp32" else 0
        self.precision = precision
        self.n_shapes = max(1, int(n_shapes))
        self.params = p
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(self.lib.am_engine_create(ctypes.byref(h), ctypes.byref(desc), ctypes.byref(p),
                                                    self.device, ctypes.c_void_p(self.stream.cuda_stream)),
                          "am_engine_create")
        self.h = h
        self.kw = self.lib.am_engine_key_words(h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.am_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ primitives
    def _dev(self, arr, dtype):
        a = np.ascontiguousarray(arr)
        if not a.flags.writeable:
            a = a.copy()
        t = torch.as_tensor(a, device=self.dev)
        return t.to(dtype).contiguous()

    def _shapes(self, shapes, n):
        if shapes is None:
            return None
        t = self._dev(np.broadcast_to(np.asarray(shapes, np.int32), (n,)), torch.int32)
        return t

    def forward(self, pts, keys: bool = False, shapes=None):
        """F(x) (and activation-state keys) at points; reference network.py:352-392.  shapes:
        per-point shape of a batch-of-shapes engine (default: the current shape)."""
        pts_t = pts if isinstance(pts, torch.Tensor) else self._dev(np.asarray(pts, np.float64).reshape(-1, 3),
                                                                   torch.float64)
        n = pts_t.shape[0]
        vals = torch.empty(n, dtype=torch.float64, device=self.dev)
        k = torch.empty((n, self.kw), dtype=torch.int64, device=self.dev) if keys else None
        sh = self._shapes(shapes, n)
        _native.check(self.lib.am_forward_shapes(self.h, pts_t.data_ptr(), sh.data_ptr() if sh is not None else None,
                                                 n, vals.data_ptr(), k.data_ptr() if k is not None else None),
                      "am_forward")
        return (vals, k) if keys else vals

    def affine_maps(self, keys):
        """canonical keys, raw neuron planes (n, NB, 4) and face planes (n, M, 4) on device."""
        keys_t = keys if isinstance(keys, torch.Tensor) else self._dev(np.asarray(keys).view(np.int64), torch.int64)
        n = keys_t.shape[0]
        canon = torch.empty_like(keys_t)
        planes = torch.empty((n, self.blob.n_bits, 4), dtype=torch.float64, device=self.dev)
        faces = torch.empty((n, self.blob.n_subs, 4), dtype=torch.float64, device=self.dev)
        _native.check(self.lib.am_affine_maps(self.h, keys_t.data_ptr(), n, canon.data_ptr(), planes.data_ptr(),
                                              faces.data_ptr()), "am_affine_maps")
        return canon, planes, faces

    def dichotomy(self, xpos, xneg, eps, seed_tol, max_iters=200, shapes=None):
        a = self._dev(np.asarray(xpos, np.float64).reshape(-1, 3), torch.float64)
        b = self._dev(np.asarray(xneg, np.float64).reshape(-1, 3), torch.float64)
        out = torch.empty_like(a)
        sh = self._shapes(shapes, a.shape[0])
        _native.check(self.lib.am_dichotomy_shapes(self.h, a.data_ptr(), b.data_ptr(),
                                                   sh.data_ptr() if sh is not None else None, a.shape[0], eps,
                                                   seed_tol, max_iters, out.data_ptr()), "am_dichotomy")
        return out

    def trace(self, x0, scheme: str, seed_tol: float, max_iters: int | None = None):
        """sgd / sphere tracing from start points (reference seeding.py:35-77), on the device:
        (final points (n, 3), status (n,) 1 converged / 2 diverged / 3 not converged, iterations)."""
        x = self._dev(np.asarray(x0, np.float64).reshape(-1, 3), torch.float64)
        n = x.shape[0]
        sch = {"sgd": 0, "sphere_trace": 1}[scheme]
        mi = (1000 if sch == 0 else 50) if max_iters is None else int(max_iters)
        param = 0.05 if sch == 0 else 1.0
        out = torch.empty_like(x)
        status = torch.empty(n, dtype=torch.int32, device=self.dev)
        iters = torch.empty(n, dtype=torch.int32, device=self.dev)
        _native.check(self.lib.am_trace(self.h, x.data_ptr(), n, sch, float(seed_tol), mi, param, 12.0, out.data_ptr(),
                                        status.data_ptr(), iters.data_ptr()), "am_trace")
        return out, status, iters

    # --------------------------------------------------------------- marching
    def reset(self):
        _native.check(self.lib.am_engine_reset(self.h), "am_engine_reset")

    def set_shapes(self, nets):
        """Batch of same-architecture shapes (engine created with n_shapes = len(nets)): shape s
        marches nets[s].  Their parameters may differ only in bias vectors (checked by the
        engine); nets[0] becomes the base parameter set."""
        if len(nets) != self.n_shapes:
            raise ValueError(f"engine holds {self.n_shapes} shapes, got {len(nets)} networks")
        from .network import param_chunks, subnetworks
        blob0 = to_blob(nets[0])
        kind0 = getattr(subnetworks(nets[0])[0], "field_kind", "sdf")
        self.load_network(nets[0], blob0)
        base = param_chunks(nets[0])
        per_net = [base]
        diff = np.zeros(len(blob0.params), dtype=bool)
        for n in nets[1:]:
            ch = param_chunks(n)
            if len(ch) != len(base):
                raise NetworkFormatError("batch of shapes: the networks differ in structure")
            if getattr(subnetworks(n)[0], "field_kind", "sdf") != kind0:
                raise NetworkFormatError("batch of shapes: the networks differ in field kind")
            for (off, a0), (off1, a) in zip(base, ch):
                if a is a0:
                    continue      # shared array (e.g. one decoder's weights): equal by identity
                a = np.asarray(a, dtype=np.float64)
                if off1 != off or a.shape != np.shape(a0):
                    raise NetworkFormatError("batch of shapes: the networks differ in structure")
                if not np.isfinite(a).all():
                    raise NetworkFormatError("batch of shapes: non-finite parameters")
                diff[off:off + a.size] |= a.reshape(-1) != np.asarray(a0, dtype=np.float64).reshape(-1)
            per_net.append(ch)
        idx = np.flatnonzero(diff).astype(np.int64)

        def gather(ch):
            flat = np.empty(len(idx), dtype=np.float64)
            for off, a in ch:
                lo, hi = np.searchsorted(idx, [off, off + np.size(a)])
                if hi > lo:
                    flat[lo:hi] = np.asarray(a, dtype=np.float64).reshape(-1)[idx[lo:hi] - off]
            return flat
        vals = np.ascontiguousarray(np.stack([gather(ch) for ch in per_net]))
        _native.check(self.lib.am_engine_set_shape_params(self.h, idx.ctypes.data, len(idx), vals.ctypes.data),
                      "am_engine_set_shape_params")
        self.shape_nets = list(nets)

    @property
    def batch_size(self) -> int:
        """Cells per BFS iteration (also the most seeds one am_seed call takes)."""
        return int(self.stats()["batch"])

    def set_shape(self, shape: int):
        """Shape of the points of later forward / dichotomy / seed calls."""
        _native.check(self.lib.am_engine_set_shape(self.h, int(shape)), "am_engine_set_shape")
        if hasattr(self, "shape_nets"):
            self.net = self.shape_nets[shape]

    def architecture(self) -> tuple:
        return architecture_key(self.blob)

    def load_network(self, net: AnyNetwork, blob: NetBlob | None = None):
        """Swap in the weights of a network with this engine's architecture (am_engine_load_params)."""
        blob = blob or to_blob(net)
        if architecture_key(blob) != self.architecture():
            raise ValueError("load_network: different architecture (layer shapes / flags / ensemble)")
        params = np.ascontiguousarray(blob.params, dtype=np.float64)
        _native.check(self.lib.am_engine_load_params(self.h, params.ctypes.data, len(params)),
                      "am_engine_load_params")
        self.net, self.blob, self._params = net, blob, params

    def seed(self, pts, shapes=None):
        t = pts if isinstance(pts, torch.Tensor) else self._dev(np.asarray(pts, np.float64).reshape(-1, 3),
                                                               torch.float64)
        sh = self._shapes(shapes, t.shape[0])
        _native.check(self.lib.am_seed_shapes(self.h, t.data_ptr(), sh.data_ptr() if sh is not None else None,
                                              t.shape[0]), "am_seed")

    def push(self, keys: torch.Tensor):
        if keys.numel():
            _native.check(self.lib.am_push_candidates(self.h, keys.data_ptr(), keys.shape[0]),
                          "am_push_candidates")

    def wave(self) -> int:
        n = ctypes.c_int64()
        _native.check(self.lib.am_wave(self.h, ctypes.byref(n)), "am_wave")
        return n.value

    def run(self) -> int:
        n = ctypes.c_int64()
        _native.check(self.lib.am_run(self.h, ctypes.byref(n)), "am_run")
        return n.value

    def queue_size(self) -> int:
        n = ctypes.c_int64()
        _native.check(self.lib.am_queue_size(self.h, ctypes.byref(n)), "am_queue_size")
        return n.value

    def outbox(self):
        """(per-owner counts (world,), keys grouped by owner rank) of states owned elsewhere."""
        total = ctypes.c_int64()
        _native.check(self.lib.am_outbox_counts(self.h, ctypes.byref(total)), "am_outbox_counts")
        counts = np.zeros(self.params.world, dtype=np.int64)
        out = torch.empty((max(total.value, 1), self.kw), dtype=torch.int64, device=self.dev)
        _native.check(self.lib.am_outbox_take(self.h, out.data_ptr(), counts.ctypes.data), "am_outbox_take")
        return counts, out[:total.value]

    # ---------------------------------------------------- sharded rounds
    def shard_rows(self, cap: int) -> int:
        """Rows of one destination block of the exchange buffers (count header + cap keys)."""
        return int(self.lib.am_shard_rows(self.h, int(cap)))

    def shard_iterate(self, iters: int, cap: int):
        """The round's one host synchronisation: (done, exchange capacity, visited over ranks,
        any rank capped); when not done, up to `iters` iterations are replayed asynchronously."""
        out = np.zeros(4, dtype=np.int64)
        _native.check(self.lib.am_shard_iterate(self.h, int(iters), int(cap), out.ctypes.data), "am_shard_iterate")
        return bool(out[0]), int(out[1]), int(out[2]), bool(out[3])

    def shard_pack(self, send: torch.Tensor, cap: int):
        _native.check(self.lib.am_shard_pack(self.h, send.data_ptr(), int(cap)), "am_shard_pack")

    def shard_absorb(self, recv: torch.Tensor, cap: int):
        _native.check(self.lib.am_shard_absorb(self.h, recv.data_ptr(), int(cap)), "am_shard_absorb")

    def shard_stats(self) -> dict:
        out = np.zeros(6, dtype=np.int64)
        _native.check(self.lib.am_shard_stats(self.h, out.ctypes.data), "am_shard_stats")
        return dict(zip(("rounds", "host_syncs", "iterations", "pool", "visited", "outbox"), (int(x) for x in out)))

    def counts(self) -> dict:
        c = np.zeros(8, dtype=np.int64)
        _native.check(self.lib.am_result_counts(self.h, c.ctypes.data), "am_result_counts")
        keys = ("cells", "faces", "empty", "verts", "edge_refs", "open_edges", "capped", "overflow")
        return dict(zip(keys, (int(x) for x in c)))

    def results(self):
        """Sorted results on the host (sorted and gathered on the GPU; pinned staging)."""
        c = self.counts()

        def pinned(shape, dt):
            return torch.empty(shape, dtype=dt, pin_memory=True).numpy()
        keys = pinned((c["cells"], self.kw), torch.int64).view(np.uint64)
        nverts = pinned(c["cells"], torch.int32)
        verts = pinned((c["verts"], 3), torch.float64)
        enr = pinned(c["verts"], torch.int32)
        erefs = pinned(c["edge_refs"], torch.int32)
        _native.check(self.lib.am_result_copy(self.h, keys.ctypes.data, nverts.ctypes.data, verts.ctypes.data,
                                              enr.ctypes.data, erefs.ctypes.data), "am_result_copy")
        return c, keys, nverts, verts, enr, erefs

    def results_device(self):
        """Sorted results as device tensors: (counts, keys (C, KW) int64, nverts (C,) int32,
        verts (V, 3), edge_nrefs (V,), edge_refs (R,))."""
        c = self.counts()
        d = self.dev
        keys = torch.empty((max(c["cells"], 1), self.kw), dtype=torch.int64, device=d)
        nverts = torch.empty(max(c["cells"], 1), dtype=torch.int32, device=d)
        verts = torch.empty((max(c["verts"], 1), 3), dtype=torch.float64, device=d)
        enr = torch.empty(max(c["verts"], 1), dtype=torch.int32, device=d)
        erefs = torch.empty(max(c["edge_refs"], 1), dtype=torch.int32, device=d)
        _native.check(self.lib.am_result_copy_device(self.h, keys.data_ptr(), nverts.data_ptr(), verts.data_ptr(),
                                                     enr.data_ptr(), erefs.data_ptr()), "am_result_copy_device")
        return (c, keys[:c["cells"]], nverts[:c["cells"]], verts[:c["verts"]], enr[:c["verts"]],
                erefs[:c["edge_refs"]])

    def kernel_times(self) -> dict:
        """Timing mode: per-stage device ms of the timed iterations (contiguous stages) + counts."""
        h = np.zeros(16)
        _native.check(self.lib.am_kernel_times(self.h, h.ctypes.data), "am_kernel_times")
        names = ("take", "compose", "canonical_insert", "frontier", "near", "face", "flip_insert", "probe_records",
                 "probe_forward")
        return {"ms": dict(zip(names, (float(x) for x in h[:9]))), "iterations": int(h[9]), "flips": int(h[10]),
                "canonical": int(h[11]), "probe_records": int(h[12]), "new_entries": int(h[13]), "kw": int(h[14]),
                "composed": int(h[15])}

    def set_timing(self, on: bool):
        _native.check(self.lib.am_set_timing(self.h, int(on)), "am_set_timing")

    def stats(self) -> dict:
        s = np.zeros(18)
        _native.check(self.lib.am_stats(self.h, s.ctypes.data), "am_stats")
        keys = ("compose_ms", "face_ms", "compose_flops", "face_bytes", "composed", "faced", "batch",
                "flops_per_cell", "launches", "iterations", "probe_ms", "probe_flops", "probes",
                "flops_per_point", "probes_forwarded", "probe_records", "prefix_skipped_flops", "prefix")
        return dict(zip(keys, (float(x) for x in s)))

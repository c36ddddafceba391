"""Triggering: surface seed points for the march (reference seeding.py).

The random sampling keeps the reference's per-index streams
(``np.random.default_rng([rng_seed, index])``, reference seeding.py:146) so the
same seeds come out; every field evaluation, the bisection and the sgd / sphere
tracing iterations run on the GPU (``Engine.forward`` / ``Engine.dichotomy`` /
``Engine.trace``).
"""

from __future__ import annotations

import numpy as np

SEED_TOL = 1e-7
SCHEMES = ("sgd", "sphere_trace", "dichotomy")


class SeedingError(RuntimeError):
    pass


def validate_scheme(net, scheme: str) -> None:
    """reference seeding.py:115-120"""
    if scheme not in SCHEMES:
        raise SeedingError(f"unknown triggering scheme {scheme!r}; choose from {SCHEMES}")
    if net.field_kind == "occupancy" and scheme in ("sgd", "sphere_trace"):
        raise SeedingError(f"scheme {scheme!r} does not trigger on occupancy fields; use 'dichotomy'")


def _trace(eng, x0: np.ndarray, scheme: str, seed_tol: float):
    """Batched sphere tracing (reference seeding.py:60-81) or SGD on |F| (seeding.py:33-57) from
    every start point at once, on the device (Engine.trace: forwards, gradients and updates stay in
    HBM; no host round trip per step).  Returns (converged point or None per start, iterations)."""
    out, iters = [None] * len(x0), np.zeros(len(x0), dtype=np.int64)
    step = max(1, min(eng.batch_size, 4096))
    for o in range(0, len(x0), step):
        pts, status, it = (t.cpu().numpy() for t in eng.trace(x0[o:o + step], scheme, seed_tol))
        if scheme == "sphere_trace" and (status == 2).any():
            j = int(np.flatnonzero(status == 2)[0])
            raise SeedingError(f"sphere tracing diverged after {int(it[j])} iterations")
        for j in np.flatnonzero(status == 1):
            out[o + j] = pts[j].copy()
            iters[o + j] = it[j]
    return out, iters


_BLOCKS: dict = {}
_BLOCKS_MAX = 1 << 16


def _sample_block(rng_seed: int, index: int, rnd: int, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """The rnd-th (64, 3) uniform draw of stream default_rng([rng_seed, index]) in [lo, hi)
    (reference seeding.py:146-148).  The draws depend only on (rng_seed, index, rnd, box), not on
    the network, so they are memoised: repeated marches with one configuration skip the
    SeedSequence set-up of every stream."""
    key = (int(rng_seed), int(index), lo.tobytes(), hi.tobytes())
    ent = _BLOCKS.get(key)
    if ent is None:
        if len(_BLOCKS) >= _BLOCKS_MAX:
            _BLOCKS.clear()
        ent = _BLOCKS[key] = (np.random.default_rng([rng_seed, index]), [])
    rng, blocks = ent
    while len(blocks) <= rnd:
        blocks.append(rng.uniform(lo, hi, size=(64, 3)))
    return blocks[rnd]


_ROUNDS: dict = {}


def _sample_round(rng_seed: int, pending: np.ndarray, rnd: int, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """(len(pending), 64, 3): the rnd-th draw of every pending stream, stacked (memoised like the
    blocks themselves, so a repeated trigger is one dictionary lookup per round)."""
    key = (int(rng_seed), int(rnd), pending.tobytes(), lo.tobytes(), hi.tobytes())
    arr = _ROUNDS.get(key)
    if arr is None:
        if len(_ROUNDS) >= 256:
            _ROUNDS.clear()
        arr = _ROUNDS[key] = np.stack([_sample_block(rng_seed, int(i), rnd, lo, hi) for i in pending])
        arr.setflags(write=False)
    return arr


def sample_seeds(eng, count: int, bbox, scheme: str = "dichotomy", rng_seed: int = 0, eps: float = SEED_TOL,
                 seed_tol: float = SEED_TOL, retry_budget: int = 200, collect_iters: list | None = None) -> np.ndarray:
    """Up to ``count`` surface points, deterministic given rng_seed (reference seeding.py:123-162)."""
    if count < 1:
        raise ValueError("count must be >= 1")
    validate_scheme(eng.net, scheme)
    lo = np.asarray(bbox[0], dtype=np.float64)
    hi = np.asarray(bbox[1], dtype=np.float64)
    found: list = [None] * count
    if scheme == "dichotomy":
        xp_f = np.zeros((count, 3))
        xn_f = np.zeros((count, 3))
        have = np.zeros(count, dtype=bool)
        pending = np.arange(count)
        rnd = 0
        while rnd < retry_budget and len(pending):
            # the next S retry rounds of every pending stream in one forward: a stream's k-th block
            # is fixed by (rng_seed, stream, k), so evaluating blocks a stream will not need
            # changes nothing, and the rounds are then replayed in order on the host
            S = min(4 if rnd == 0 else 8, retry_budget - rnd)
            blocks = [_sample_round(rng_seed, pending, rnd + k, lo, hi) for k in range(S)]
            vals = eng.forward(np.concatenate(blocks).reshape(-1, 3)).cpu().numpy().reshape(S, len(pending), 64)
            still = np.ones(len(pending), dtype=bool)
            for k in range(S):
                # first positive / first negative sample of each stream (reference seeding.py:150-156)
                pm, nm = vals[k] > 0.0, vals[k] < 0.0
                ok = still & pm.any(axis=1) & nm.any(axis=1)
                rows = np.flatnonzero(ok)
                idx = pending[rows]
                xp_f[idx] = blocks[k][rows, pm.argmax(axis=1)[rows]]
                xn_f[idx] = blocks[k][rows, nm.argmax(axis=1)[rows]]
                have[idx] = True
                still &= ~ok
            pending = pending[still]
            rnd += S
        order = np.flatnonzero(have)
        if len(order):
            pts = eng.dichotomy(xp_f[order], xn_f[order], eps, seed_tol).cpu().numpy()
            for i, p in zip(order, pts):
                found[i] = p
    else:
        rngs = [np.random.default_rng([rng_seed, index]) for index in range(count)]
        pending = list(range(count))
        for _ in range(retry_budget):
            if not pending:
                break
            x0 = np.stack([rngs[i].uniform(lo, hi, size=3) for i in pending])
            res, iters = _trace(eng, x0, scheme, seed_tol)
            still = []
            for j, i in enumerate(pending):
                if res[j] is not None:
                    found[i] = res[j]
                    if collect_iters is not None:
                        collect_iters.append(int(iters[j]))
                else:
                    still.append(i)
            pending = still
    seeds = [p for p in found if p is not None]
    if not seeds:
        raise SeedingError("no surface located in bbox")
    return np.array(seeds)


def sample_seeds_batch(eng, nets, count: int, bbox, rng_seed: int = 0, eps: float = SEED_TOL,
                       seed_tol: float = SEED_TOL, retry_budget: int = 200) -> list:
    """sample_seeds (dichotomy trigger) of every shape of a batch-of-shapes engine at once.

    Shape s's trigger is the reference's (seeding.py:123-162) on its own network: the sample
    streams default_rng([rng_seed, index]) do not depend on the network, and a pending
    (shape, index) pair draws its k-th block in retry round k exactly as the per-shape loop
    would, so one forward evaluation per round and one bisection serve the whole batch."""
    if count < 1:
        raise ValueError("count must be >= 1")
    for net in nets:
        validate_scheme(net, "dichotomy")
    S = len(nets)
    lo = np.asarray(bbox[0], dtype=np.float64)
    hi = np.asarray(bbox[1], dtype=np.float64)
    rngs = [np.random.default_rng([rng_seed, index]) for index in range(count)]
    blocks: list = [[] for _ in range(count)]      # k-th (64, 3) draw of stream i, shared by all shapes
    pending = [(s, i) for s in range(S) for i in range(count)]
    pairs: dict = {}
    for k in range(retry_budget):
        if not pending:
            break
        for _, i in pending:
            while len(blocks[i]) <= k:
                blocks[i].append(rngs[i].uniform(lo, hi, size=(64, 3)))
        pts = np.stack([blocks[i][k] for _, i in pending])
        shp = np.repeat(np.array([s for s, _ in pending], np.int32), 64)
        vals = eng.forward(pts.reshape(-1, 3), shapes=shp).cpu().numpy().reshape(len(pending), 64)
        still = []
        for j, (s, i) in enumerate(pending):
            pos = pts[j][vals[j] > 0.0]
            neg = pts[j][vals[j] < 0.0]
            if len(pos) and len(neg):
                pairs[(s, i)] = (pos[0], neg[0])
            else:
                still.append((s, i))
        pending = still
    out = [np.zeros((0, 3)) for _ in range(S)]
    if pairs:
        order = sorted(pairs)
        xp = np.stack([pairs[o][0] for o in order])
        xn = np.stack([pairs[o][1] for o in order])
        sh = np.array([o[0] for o in order], np.int32)
        pts = eng.dichotomy(xp, xn, eps, seed_tol, shapes=sh).cpu().numpy()
        for s in range(S):
            out[s] = pts[sh == s]
    for s in range(S):
        if not len(out[s]):
            raise SeedingError(f"no surface located in bbox (shape {s})")
    return out

"""Batches of same-architecture networks -- latent-conditioned shapes (BASELINE configs[4]).

A latent-conditioned decoder f(z (+) x) with a fixed code z is an ordinary ReLU MLP in x: the
code's columns fold into the biases of the layers it enters (the first layer and, for DeepSDF,
the skip re-entry), see ``synth.latent_batch``.  Every shape of a batch therefore has the same
architecture, so one engine -- its buffers, TMA descriptors and captured iteration graphs --
serves the whole batch; per shape only the parameter values are uploaded
(``am_engine_load_params``), then the reference march (marching.py:304-362) runs as usual.

On one GPU the batch is marched FUSED by default: one engine holds every shape (the state key
gains a trailing shape word; per-shape bias tables, ``am_engine_set_shape_params``), every
shape's seeds enter one queue and a single BFS runs over the union of the shapes' cell graphs.
Composition of all shapes' cells in a wave is one DMMA contraction per layer (the weights are
shared), and each wave is ~n_shapes times wider than a single shape's, so the per-wave launch
latency that bounds a single small march is amortised over the batch.  The visited set of each
shape is the closure of its own seeds (states of different shapes never mix: the shape word is
part of the key), i.e. the reference march of that shape; ``max_cells`` then caps the batch
total at max_cells x n_shapes.  ``fused=False`` marches the shapes one after another on one
reused engine (exact per-shape caps).

Across ranks (one process per GPU, torch.distributed initialised):

* ``shard="hash"``: ONE fused BFS over every shape of the batch on all ranks together: the
  batch engine's keys carry the shape word, states are owned by hash(state) mod P and exchanged
  in device-driven rounds (``distributed.ShardedMarcher``); each rank returns its owned part of
  every shape, and the union over ranks is the shape's full result.
* ``shard="shape"``: rank r marches shapes s with s % P == r alone (no collective; weak
  scaling over shapes).
"""

from __future__ import annotations

import time
from typing import Sequence

import numpy as np

from .engine import architecture_key
from .marching import MarchConfig, MarchResult, _engine_for, check_overflow, collect_result, march, seed_engine
from .network import AnyNetwork, is_ensemble, to_blob


def _check_same_architecture(nets: Sequence[AnyNetwork]):
    keys = {architecture_key(to_blob(n)) for n in nets}
    if len(keys) > 1:
        raise ValueError("march_batch: the networks of a batch must share one architecture")


def shard_of_shapes(n_shapes: int, rank: int, world: int) -> list[int]:
    """Shapes a rank owns under shape sharding."""
    return [s for s in range(n_shapes) if s % world == rank]


def _fused_engine(nets, config: MarchConfig):
    from .marching import _ENGINES, ENGINE_CACHE_SIZE
    from .engine import Engine
    import torch
    key = ("batch", len(nets), architecture_key(to_blob(nets[0])), tuple(map(tuple, config.bbox)),
           config.max_cells, config.tol_cell, config.tol_weld, config.probe_delta, config.batch_cells,
           config.mem_budget, config.precision, torch.cuda.current_device())
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(nets[0], bbox=config.bbox, max_cells=config.max_cells * len(nets), tol_cell=config.tol_cell,
                     tol_weld=config.tol_weld, probe_delta=config.probe_delta, batch_cells=config.batch_cells,
                     mem_budget=config.mem_budget, n_shapes=len(nets), precision=config.precision)
        _ENGINES[key] = eng
        while len(_ENGINES) > ENGINE_CACHE_SIZE:
            _ENGINES.popitem(last=False)
    else:
        eng.reset()
        _ENGINES.move_to_end(key)
    eng.set_shapes(nets)
    return eng


def split_batch_result(eng, seeds_per_shape, t0: float, waves: int) -> list[MarchResult]:
    """Per-shape MarchResults from a fused batch engine (results are sorted shape-major)."""
    from .marching import MarchReport, device_results_to_host
    c, hk, _, shape, hn, hv, he, hr = device_results_to_host(eng)
    nb = eng.blob.n_bits
    shape = shape.astype(np.int64)
    cell_off = np.searchsorted(shape, np.arange(eng.n_shapes + 1))
    vcount = np.maximum(hn, 0).astype(np.int64)
    voff = np.concatenate([[0], np.cumsum(vcount)])
    roff = np.concatenate([[0], np.cumsum(he.astype(np.int64))])
    # an edge is open when one of its transition refs is a box face (reference MarchReport)
    cs = np.concatenate([[0], np.cumsum(hr[:, 0] == 2)]) if len(hr) else np.zeros(1, np.int64)
    bbox_edge = (cs[roff[1:]] - cs[roff[:-1]]) > 0
    out = []
    for s in range(eng.n_shapes):
        c0, c1 = cell_off[s], cell_off[s + 1]
        v0, v1 = voff[c0], voff[c1]
        r0, r1 = roff[v0], roff[v1]
        kb, branch = hk[c0:c1], np.full(c1 - c0, -1, np.int64)
        nv = hn[c0:c1]
        rep = MarchReport(cells_visited=int(c1 - c0), faces_emitted=int((nv > 0).sum()),
                          empty_faces=int((nv == 0).sum()), open_edges=int(bbox_edge[v0:v1].sum()),
                          seconds=time.perf_counter() - t0, seeds_used=len(seeds_per_shape[s]),
                          capped=bool(c["capped"]), threads=1, waves=waves, overflow=int((nv < 0).sum()))
        nets = getattr(eng, "shape_nets", None)
        out.append(MarchResult(kb, branch, nv, hv[v0:v1], he[v0:v1], hr[r0:r1], rep, nb, seeds_per_shape[s],
                               net=nets[s] if nets else None))
    return out


def march_fused(nets: Sequence[AnyNetwork], config: MarchConfig | None = None) -> list[MarchResult]:
    """Every shape of a same-architecture batch in ONE breadth-first march (one engine)."""
    from .seeding import sample_seeds, sample_seeds_batch
    config = config or MarchConfig()
    _check_same_architecture(nets)
    t0 = time.perf_counter()
    eng = _fused_engine(nets, config)
    S = len(nets)
    if config.seed_points is not None:
        seeds = [np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)] * S
    elif config.scheme == "dichotomy":
        seeds = sample_seeds_batch(eng, nets, config.seeds, config.bbox, rng_seed=config.rng_seed)
    else:
        seeds = []
        for s in range(S):
            eng.set_shape(s)
            seeds.append(sample_seeds(eng, config.seeds, config.bbox, scheme=config.scheme, rng_seed=config.rng_seed))
    pts = np.concatenate(seeds)
    shp = np.concatenate([np.full(len(x), s, np.int32) for s, x in enumerate(seeds)])
    seed_engine(eng, pts, shp)
    waves = eng.run()
    return split_batch_result(eng, seeds, t0, waves)


def march_batch(nets: Sequence[AnyNetwork], config: MarchConfig | None = None, shard: str = "hash",
                group=None, engine_factory=None, fused: bool = True) -> list[tuple[int, MarchResult | object]]:
    """March every network of a same-architecture batch; returns [(shape index, result)].

    Single process: every shape, one reused engine.  Distributed: see the module docstring;
    ``engine_factory`` substitutes the per-rank engine (tests run the protocol on CPU with the
    oracle-backed stand-in, whose results are its visited-key set).
    """
    import torch.distributed as dist
    config = config or MarchConfig()
    if shard not in ("hash", "shape"):
        raise ValueError("shard must be 'hash' or 'shape'")
    if not nets:
        return []
    _check_same_architecture(nets)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0

    if world == 1 or shard == "shape":
        mine = shard_of_shapes(len(nets), rank, world)
        if engine_factory is None:
            # batches of max-pool ensembles march shape by shape (the fused engine holds plain nets)
            if fused and len(mine) > 1 and not is_ensemble(nets[0]):
                return list(zip(mine, march_fused([nets[s] for s in mine], config)))
            return [(s, march(nets[s], config)) for s in mine]
        out = []
        eng = None
        for s in mine:
            eng = engine_factory(nets[s], bbox=config.bbox, max_cells=config.max_cells) if eng is None else eng
            if hasattr(eng, "load_network"):
                eng.load_network(nets[s])
            eng.reset()
            eng.seed(eng.sample_seeds(config.seeds, config.bbox, scheme=config.scheme, rng_seed=config.rng_seed))
            while eng.queue_size():
                eng.wave()
            out.append((s, eng.visited_keys()))
        return out

    from .distributed import ShardedMarcher
    if not is_ensemble(nets[0]):
        # one fused BFS over every shape, states owned by hash(state incl. shape word) mod P
        t0 = time.perf_counter()
        sm = ShardedMarcher(list(nets), bbox=config.bbox, max_cells=config.max_cells * len(nets),
                            engine_factory=engine_factory)
        if config.seed_points is not None:
            seeds = [np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)] * len(nets)
        else:
            seeds = sm.sample_seeds_batch(config.seeds, rng_seed=config.rng_seed)
        pts = np.concatenate(seeds)
        shp = np.concatenate([np.full(len(x), s, np.int32) for s, x in enumerate(seeds)])
        rounds = sm.run(pts, shapes=shp)
        if engine_factory is not None:
            vis = sm.engine.visited_by_shape()
            return [(s, vis[s]) for s in range(len(nets))]
        import torch
        with torch.cuda.stream(sm.stream):
            res = split_batch_result(sm.engine, seeds, t0, rounds)
        for r in res:
            r.report.capped = sm.capped
            check_overflow(r.report)
        return list(enumerate(res))
    # batches of max-pool ensembles: shape by shape, each hash-sharded
    sm = None
    out = []
    for s, net in enumerate(nets):
        t0 = time.perf_counter()
        if sm is None:
            sm = ShardedMarcher(net, bbox=config.bbox, max_cells=config.max_cells, engine_factory=engine_factory)
        else:
            sm.load_network(net)
        if config.seed_points is not None:
            seeds = np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)
        else:
            seeds = sm.sample_seeds(config.seeds, rng_seed=config.rng_seed, scheme=config.scheme)
        rounds = sm.run(seeds)
        if engine_factory is None:
            import torch
            with torch.cuda.stream(sm.stream):
                out.append((s, collect_result(sm.engine, seeds, t0, rounds, net=net)))
        else:
            out.append((s, sm.engine.visited_keys()))
    return out

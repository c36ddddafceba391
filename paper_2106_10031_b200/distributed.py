"""Sharded marching across GPUs: states owned by hash mod P, frontier exchanged by all-to-all.

One process per GPU (torchrun).  Every rank runs the same BFS engine on the
states it owns (owner(state) = (hash(state) >> 7) mod world, csrc/am_internal.h
key_owner).  The march advances in ROUNDS, each with exactly one host
synchronisation:

1. ``Engine.shard_iterate`` -- the synchronisation: reads the engine counters
   and the count headers of the previous exchange; every rank sees every
   sender's header, so all ranks agree on termination (nobody has queued work,
   outbox or keys in flight) and on the next exchange's capacity; otherwise it
   replays up to ``iters`` BFS iterations of the owned queue as CUDA graphs
   (states owned elsewhere accumulate in the device outbox);
2. ``Engine.shard_pack`` -- the outbox goes into a fixed-size send buffer of
   equal per-rank blocks, each opening with a count header; what does not fit
   stays in the outbox for the next round;
3. one ``all_to_all_single`` of equal splits (NCCL over NVLink / NVSwitch on a
   B200 node) -- the only collective, and the host never needs the counts to
   size it;
4. ``Engine.shard_absorb`` -- received keys are inserted and queued by their
   owner with device-side counts; the headers go to the host for step 1.

Steps 2-4 are asynchronous on the engine's stream.  The reference has no
distributed mode; its threaded engine (reference marching.py:216-301) shares one
visited set -- here the visited set is partitioned instead, and the union over
ranks equals the single-GPU set.  ``max_cells`` is shared out: rank r may visit
max_cells // world (+1 for r < max_cells % world) cells, so the union never
exceeds the cap; ``capped`` is set when any rank hit its share.
"""

from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist

from .engine import Engine
from .seeding import sample_seeds

# BFS iterations between exchanges.  With hash ownership ~(P-1)/P of a cell's neighbours belong to
# other ranks, so the march advances about one BFS level per exchange whatever the round length;
# the iterations after the first in a round only see the locally owned children (1/P of them,
# then 1/P^2 ...) at the ~70 us per-iteration floor.  One rank: 4 (P = 1 A/B: 2 / 4 / 8 / 16 ->
# 20.43 / 19.16 / 18.77 / 18.47 ms, `profiles/r02_sharded_p1.json`; 4 keeps the round latency low
# when ranks are added); several ranks: 2 (the first iteration plus one pass over local children).
ITERS_PER_ROUND = 4
ITERS_PER_ROUND_MULTI = 2
INITIAL_CAP = 1024        # keys per destination in the first exchange (grows from the headers)


def cap_share(max_cells: int, rank: int, world: int) -> int:
    """This rank's share of the global visited-cell cap (the shares sum to max_cells)."""
    return max(1, max_cells // world + (1 if rank < max_cells % world else 0))


def all_to_all_fixed(send: torch.Tensor, recv: torch.Tensor, rows: int = 0, hdr_rows: int = 0):
    """The round's exchange: equal blocks of `rows` rows per destination (NCCL: one collective on
    the current stream, no host involvement).  gloo (CPU test runs, ranks sharing one GPU) moves
    host tensors, so there the used rows of every block are compacted first (headers read on the
    host) -- a functional path, not the multi-GPU one."""
    if not (dist.get_backend() == "gloo" and send.is_cuda):
        dist.all_to_all_single(recv, send)
        return
    world = dist.get_world_size()
    kw = send.shape[1]
    h = send.view(world, rows, kw)
    hdr = h[:, :hdr_rows].reshape(world, -1)[:, 0].cpu()           # keys per destination block
    used = (hdr.clamp(min=0) + hdr_rows).to(torch.int64)
    counts_in = torch.empty_like(used)
    dist.all_to_all_single(counts_in, used)
    out = torch.cat([h[r, :int(used[r])] for r in range(world)]).cpu()
    inc = torch.empty((int(counts_in.sum()), kw), dtype=send.dtype)
    dist.all_to_all_single(inc, out, output_split_sizes=counts_in.tolist(), input_split_sizes=used.tolist())
    rv = recv.view(world, rows, kw)
    off = 0
    for r in range(world):
        n = int(counts_in[r])
        rv[r, :n].copy_(inc[off:off + n])
        off += n


class ShardedMarcher:
    """Hash-owned multi-GPU march (one instance per rank), device-driven rounds."""

    def __init__(self, net, bbox=((-1.2,) * 3, (1.2,) * 3), max_cells: int = 10_000_000, engine_factory=None,
                 iters_per_round: int | None = None, **kw):
        """``net``: one network, or a list of same-architecture networks marched as ONE fused BFS
        (a batch of shapes: the shape word is part of every key, so ownership and dedup are
        per shape; ``max_cells`` then caps the batch total)."""
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.batch = isinstance(net, (list, tuple))
        self.nets = list(net) if self.batch else [net]
        self.net = self.nets[0]
        self.bbox = bbox
        if iters_per_round is None:
            iters_per_round = ITERS_PER_ROUND if self.world == 1 else ITERS_PER_ROUND_MULTI
        self.iters = int(iters_per_round)
        self.max_cells = int(max_cells)
        share = cap_share(self.max_cells, self.rank, self.world)
        if engine_factory is None:
            # the engine runs on a stream of its own; the exchange is enqueued on the same stream
            self.stream = torch.cuda.Stream()
            self.engine = Engine(self.net, bbox=bbox, max_cells=share, rank=self.rank, world=self.world,
                                 stream=self.stream, n_shapes=len(self.nets) if self.batch else 1, **kw)
            if self.batch:
                self.engine.set_shapes(self.nets)
        else:
            self.stream = None
            self.engine = engine_factory(self.nets if self.batch else self.net, bbox=bbox, max_cells=share,
                                         rank=self.rank, world=self.world, **kw)
        self.rounds = 0
        self.capped = False
        self._bufs = (0, None, None)

    def sample_seeds_batch(self, count: int, rng_seed: int = 0) -> list:
        """Every shape's dichotomy seeds (identical on every rank)."""
        if hasattr(self.engine, "sample_seeds_batch"):
            return self.engine.sample_seeds_batch(count, self.bbox, rng_seed=rng_seed)
        from .seeding import sample_seeds_batch
        return sample_seeds_batch(self.engine, self.nets, count, self.bbox, rng_seed=rng_seed)

    def load_network(self, net):
        """Next network of a same-architecture batch (weights re-uploaded, engine reused)."""
        self.net = net
        self.engine.load_network(net)

    def sample_seeds(self, count: int, rng_seed: int = 0, scheme: str = "dichotomy") -> np.ndarray:
        """Same seeds on every rank (the trigger is deterministic given rng_seed)."""
        if hasattr(self.engine, "sample_seeds"):   # CPU stand-in engines bring their own trigger
            return self.engine.sample_seeds(count, self.bbox, scheme=scheme, rng_seed=rng_seed)
        return sample_seeds(self.engine, count, self.bbox, scheme=scheme, rng_seed=rng_seed)

    def _buffers(self, cap: int):
        if self._bufs[0] != cap:
            rows = self.engine.shard_rows(cap)
            shape = (self.world * rows, self.engine.kw)
            dev = self.engine.dev if self.stream is not None else torch.device("cpu")
            self._bufs = (cap, torch.zeros(shape, dtype=torch.int64, device=dev),
                          torch.zeros(shape, dtype=torch.int64, device=dev))
        return self._bufs[1], self._bufs[2]

    def run(self, seeds: np.ndarray, shapes=None, max_rounds: int = 1_000_000) -> int:
        """March from the seeds (every rank passes the same seeds; each keeps the states it owns;
        ``shapes``: the shape of every seed of a batch).  Returns the number of rounds."""
        eng = self.engine
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _nullctx()
        with ctx:
            eng.reset()
            if self.stream is not None:
                from .marching import seed_engine
                seed_engine(eng, np.asarray(seeds, dtype=np.float64).reshape(-1, 3), shapes)
            elif self.batch:
                eng.seed(seeds, shapes)
            else:
                eng.seed(seeds)
            cap, rounds = INITIAL_CAP, 0
            while rounds < max_rounds:
                done, cap, _, capped = eng.shard_iterate(self.iters, cap)
                self.capped = capped
                if done:
                    break
                send, recv = self._buffers(cap)
                eng.shard_pack(send, cap)
                rows = eng.shard_rows(cap)
                all_to_all_fixed(send, recv, rows, rows - cap)
                eng.shard_absorb(recv, cap)
                rounds += 1
        self.rounds = rounds
        return rounds


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_MARCHERS: dict = {}


def march_sharded(net, config=None) -> "MarchResult":
    """Multi-GPU ``march`` (call it on every rank, one process per GPU): this rank's share of the
    march -- the visited cells it owns (hash(state) mod world), sorted in the reference's order
    (marching.py:346-359), with their polygons, on the host.  The union of the ranks' results is
    ``march(net, config)``'s result.  Marchers are kept per architecture and re-used with the new
    weights uploaded, like ``march``'s engines."""
    from .engine import architecture_key
    from .marching import MarchConfig, check_overflow, collect_result
    from .network import to_blob
    config = config or MarchConfig()
    t0 = time.perf_counter()
    key = (architecture_key(to_blob(net)), tuple(map(tuple, config.bbox)), config.max_cells, config.tol_cell,
           config.tol_weld, config.probe_delta, config.batch_cells, config.mem_budget, config.precision,
           dist.get_rank(), dist.get_world_size(), torch.cuda.current_device())
    sm = _MARCHERS.get(key)
    if sm is None:
        sm = ShardedMarcher(net, bbox=config.bbox, max_cells=config.max_cells, tol_cell=config.tol_cell,
                            tol_weld=config.tol_weld, probe_delta=config.probe_delta,
                            batch_cells=config.batch_cells, mem_budget=config.mem_budget,
                            precision=config.precision)
        _MARCHERS.clear()
        _MARCHERS[key] = sm
    else:
        sm.load_network(net)
    if config.seed_points is not None:
        seeds = np.asarray(config.seed_points, dtype=np.float64).reshape(-1, 3)
    else:
        seeds = sm.sample_seeds(config.seeds, rng_seed=config.rng_seed, scheme=config.scheme)
    rounds = sm.run(seeds)
    with torch.cuda.stream(sm.stream):
        res = collect_result(sm.engine, seeds, t0, rounds, config.threads, net=net)
    res.report.capped = sm.capped
    check_overflow(res.report)
    return res

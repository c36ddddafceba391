"""Sharded marching across GPUs: states owned by hash mod P, frontier exchanged by all-to-all.

One process per GPU (torchrun).  Every rank runs the same BFS engine on the
states it owns (owner(state) = hash(state) mod world, csrc/am_internal.h
key_owner).  Each wave a rank processes its queue, inserts the neighbour states
it owns locally and holds the others in an outbox; the outboxes are exchanged
with one ``torch.distributed.all_to_all_single`` (NCCL over NVLink on B200s,
gloo on CPU test runs) and the received states are queued by their owners.
The per-rank counts of that exchange double as the termination test (no rank
has queued work and nothing is in flight), so the all-to-all is the only
collective in the loop.

The reference has no distributed mode; its threaded engine (reference
marching.py:216-301) shares one visited set -- here the visited set is
partitioned instead, and the union over ranks equals the single-GPU set.
"""

from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist

from .engine import Engine
from .network import AnyNetwork
from .seeding import sample_seeds


def exchange(send: torch.Tensor, counts: np.ndarray, kw: int, extra: int = 0):
    """All-to-all of key rows grouped by destination rank.

    Returns (received rows, total queued work over all ranks).  The count
    exchange carries each rank's pending-queue size so the loop can terminate
    without a separate all-reduce.
    """
    world = dist.get_world_size()
    dev = send.device
    # gloo (CPU test runs) moves host tensors: device rows are staged through the host
    stage = send.is_cuda and dist.get_backend() == "gloo"
    cdev = torch.device("cpu") if stage else dev
    meta = torch.tensor([[int(c), int(extra)] for c in counts], dtype=torch.int64, device=cdev)
    meta_in = torch.empty_like(meta)
    dist.all_to_all_single(meta_in, meta)
    recv_counts = meta_in[:, 0].tolist()
    total_pending = int(meta_in[:, 1].sum().item())
    recv = torch.empty((sum(recv_counts), kw), dtype=send.dtype, device=cdev)
    if world > 1:
        dist.all_to_all_single(recv, (send.cpu() if stage else send).contiguous(), output_split_sizes=recv_counts,
                               input_split_sizes=[int(c) for c in counts])
    return (recv.to(dev) if stage else recv), total_pending


class ShardedMarcher:
    """Hash-owned, wave-synchronous multi-GPU march (one instance per rank)."""

    def __init__(self, net: AnyNetwork, bbox=((-1.2,) * 3, (1.2,) * 3), max_cells: int = 10_000_000,
                 engine_factory=None, **kw):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.net = net
        self.bbox = bbox
        factory = engine_factory or Engine
        self.engine = factory(net, bbox=bbox, max_cells=max_cells, rank=self.rank, world=self.world, **kw)
        self.waves = 0

    def load_network(self, net: AnyNetwork):
        """Next network of a same-architecture batch (weights re-uploaded, engine reused)."""
        self.net = net
        if hasattr(self.engine, "load_network"):
            self.engine.load_network(net)
        else:                                 # engines without a weight swap are rebuilt
            self.engine = type(self.engine)(net, bbox=self.bbox, rank=self.rank, world=self.world)

    def sample_seeds(self, count: int, rng_seed: int = 0, scheme: str = "dichotomy") -> np.ndarray:
        """Same seeds on every rank (the trigger is deterministic given rng_seed)."""
        if hasattr(self.engine, "sample_seeds"):   # CPU stand-in engines bring their own trigger
            return self.engine.sample_seeds(count, self.bbox, scheme=scheme, rng_seed=rng_seed)
        return sample_seeds(self.engine, count, self.bbox, scheme=scheme, rng_seed=rng_seed)

    def run(self, seeds: np.ndarray, max_waves: int = 1_000_000) -> int:
        eng = self.engine
        eng.reset()
        # every rank refines all seeds; each keeps the seed states it owns (the rest go out)
        eng.seed(seeds)
        waves = 0
        while waves < max_waves:
            eng.wave()
            counts, out = eng.outbox()
            # extra = this rank's queued + outgoing work; summed over ranks it is the global
            # amount of outstanding work, identical on every rank
            recv, pending = exchange(out, counts, eng.kw, extra=eng.queue_size() + int(counts.sum()))
            if len(recv):
                eng.push(recv)
            waves += 1
            if pending == 0:
                break
        self.waves = waves
        return waves


_MARCHERS: dict = {}


def march_sharded(net: AnyNetwork, config=None) -> "MarchResult":
    """Multi-GPU ``march`` (call it on every rank, one process per GPU): this rank's share of the
    march -- the visited cells it owns (hash(state) mod world), sorted in the reference's order
    (marching.py:346-359), with their polygons, on the host.  The union of the ranks' results is
    ``march(net, config)``'s result.  Marchers are kept per architecture and re-used with the new
    weights uploaded, like ``march``'s engines."""
    from .engine import architecture_key
    from .marching import MarchConfig, collect_result
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
    waves = sm.run(seeds)
    return collect_result(sm.engine, seeds, t0, waves, config.threads)

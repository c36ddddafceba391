"""The sharded march with real GPU engines: two ranks (processes) on one B200, frontier exchange
over gloo (host-staged).  Ranks only meet in the all-to-all between rounds -- no kernel
waits on another rank -- so this checks the engines' sharded mode (owned-state filtering,
outboxes, single waves, pushed candidates, remote probe targets): the union of the ranks'
visited sets equals the single-GPU march and the shards are disjoint.  Multi-GPU timing is not
measured here."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _net(which):
    from paper_2106_10031_b200 import synth
    if which == "geo_60x2":
        return synth.geometric_mlp([60, 60], seed=0), ((-1.2,) * 3, (1.2,) * 3)
    return synth.imnet_ensemble(widths=(32, 32), n_parts=3, seed=1), ((-1.0,) * 3, (1.0,) * 3)


def _worker(rank, world, port, which, seeds, q):
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_10031_b200.distributed import ShardedMarcher
    net, bbox = _net(which)
    sm = ShardedMarcher(net, bbox=bbox)
    s0 = sm.engine.shard_stats()["host_syncs"]
    rounds = sm.run(seeds)
    syncs = sm.engine.shard_stats()["host_syncs"] - s0
    with torch.cuda.stream(sm.stream):
        c, keys, *_ = sm.engine.results()
    q.put((rank, (rounds, syncs), [k.tobytes() for k in keys]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("which", ["geo_60x2", "imnet_ens"])
def test_sharded_gpu_engines_union_equals_single_gpu(which):
    from paper_2106_10031_b200 import marching
    net, bbox = _net(which)
    single = marching.march(net, marching.MarchConfig(bbox=bbox, seeds=16, rng_seed=0))
    ref = {(k.tobytes(), int(b)) for k, b in zip(single.keys, single.branch)}
    assert len(ref) == single.report.cells_visited
    nb = single.n_bits
    bw, nbytes = (nb + 63) // 64, (nb + 7) // 8
    ens = bool((single.branch >= 0).any())

    def as_ref(word_bytes):   # engine key words (MSB-first) -> (packbits bytes, branch)
        w = np.frombuffer(word_bytes, dtype=np.uint64)
        return (w[:bw].byteswap().tobytes()[:nbytes], int(w[bw]) if ens else -1)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, which, single.seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shards = [{as_ref(k) for k in v} for _, _, v in res]
    assert not (shards[0] & shards[1]), "a state is owned by two ranks"
    assert shards[0] and shards[1]
    assert shards[0] | shards[1] == ref
    # one host synchronisation per round (am_shard_iterate), plus the seeding's own
    for _, (rounds, syncs), _ in res:
        assert rounds > 1 and syncs <= rounds + 1 + 8, (rounds, syncs)


def _api_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_10031_b200 import marching
    from paper_2106_10031_b200.distributed import march_sharded
    net, bbox = _net("geo_60x2")
    cfg = marching.MarchConfig(bbox=bbox, seeds=16, rng_seed=0)
    march_sharded(net, cfg)           # second call re-uses the cached marcher
    r = march_sharded(net, cfg)
    off = np.concatenate([[0], np.cumsum(r.nverts)])
    cells = {(r.keys[i].tobytes(), int(r.branch[i])): r.verts[off[i]:off[i + 1]].copy() for i in range(len(r.keys))}
    q.put((rank, cells, r.report.cells_visited))
    dist.barrier()
    dist.destroy_process_group()


def test_march_sharded_api_union_equals_march():
    """The multi-GPU public call: each rank's sorted share (cells + polygons) of the march; the
    disjoint union is march()'s result, polygons included."""
    from paper_2106_10031_b200 import marching
    net, bbox = _net("geo_60x2")
    single = marching.march(net, marching.MarchConfig(bbox=bbox, seeds=16, rng_seed=0))
    off = np.concatenate([[0], np.cumsum(single.nverts)])
    ref = {(single.keys[i].tobytes(), int(single.branch[i])): single.verts[off[i]:off[i + 1]]
           for i in range(len(single.keys))}
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_api_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shards = [c for _, c, _ in res]
    assert sum(n for _, _, n in res) == single.report.cells_visited
    assert not (shards[0].keys() & shards[1].keys())
    merged = {**shards[0], **shards[1]}
    assert merged.keys() == ref.keys()
    for k, v in ref.items():
        assert merged[k].shape == v.shape
        assert np.abs(merged[k] - v).max(initial=0.0) <= 1e-9


def _batch_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from test_batch import BBOX, small_latent_batch
    from paper_2106_10031_b200.batch import march_batch
    from paper_2106_10031_b200.marching import MarchConfig
    res = march_batch(small_latent_batch(4), MarchConfig(bbox=BBOX, seeds=4, rng_seed=1), shard="hash")
    out = []
    for s, r in res:
        off = np.concatenate([[0], np.cumsum(r.nverts)])
        out.append((s, {r.keys[i].tobytes(): r.verts[off[i]:off[i + 1]].copy() for i in range(len(r.keys))}))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_hash_sharded_fused_batch_union_equals_single_gpu():
    """configs[4]'s multi-GPU form: ONE fused BFS over a batch of latent shapes, states owned by
    hash (shape word included) across 2 ranks; per shape, the disjoint union of the ranks' cells
    (with polygons) equals the single-GPU fused batch march."""
    from test_batch import BBOX, small_latent_batch
    from paper_2106_10031_b200.batch import march_fused
    from paper_2106_10031_b200.marching import MarchConfig
    single = march_fused(small_latent_batch(4), MarchConfig(bbox=BBOX, seeds=4, rng_seed=1))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for s, ref in enumerate(single):
        parts = [dict(items)[s] for _, items in res]
        assert not (parts[0].keys() & parts[1].keys())
        merged = {**parts[0], **parts[1]}
        off = np.concatenate([[0], np.cumsum(ref.nverts)])
        want = {ref.keys[i].tobytes(): ref.verts[off[i]:off[i + 1]] for i in range(len(ref.keys))}
        assert merged.keys() == want.keys(), f"shape {s}"
        for k, v in want.items():
            assert merged[k].shape == v.shape and np.abs(merged[k] - v).max(initial=0.0) <= 1e-9


def _nccl_worker(port, q):
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2106_10031_b200 import marching
    from paper_2106_10031_b200.distributed import march_sharded
    net, bbox = _net("geo_60x2")
    r = march_sharded(net, marching.MarchConfig(bbox=bbox, seeds=16, rng_seed=0))
    q.put((r.keys.tobytes(), r.nverts.tobytes(), r.verts.tobytes(), r.report.cells_visited))
    dist.destroy_process_group()


def test_sharded_rounds_over_nccl_single_rank():
    """The NCCL path of the round protocol (fixed-block all_to_all_single on the marcher's stream,
    device-side pack / absorb, header-driven termination) with one rank: the result equals
    march()'s exactly."""
    from paper_2106_10031_b200 import marching
    net, bbox = _net("geo_60x2")
    single = marching.march(net, marching.MarchConfig(bbox=bbox, seeds=16, rng_seed=0))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    keys, nv, verts, cells = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert cells == single.report.cells_visited
    assert keys == single.keys.tobytes() and nv == single.nverts.tobytes()
    assert np.abs(np.frombuffer(verts) - single.verts.reshape(-1)).max(initial=0.0) <= 1e-9

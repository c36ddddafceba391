"""Batches of latent-conditioned shapes (BASELINE configs[4], paper_2106_10031_b200.batch).

CPU: the sharded protocol over gloo (world 2) with the oracle-backed engine stand-in, for both
hash sharding (every shape on all ranks; union of shards == the shape's single-process visited
set, shards disjoint) and shape sharding (each shape on exactly one rank).  GPU: march_batch on
one device equals the oracle march of every folded network, with one reused engine."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

BBOX = ((-1.0,) * 3, (1.0,) * 3)


def small_latent_batch(n=4):
    from paper_2106_10031_b200 import synth
    nets, codes = synth.latent_batch(n_shapes=n, latent_dim=8, width=16, depth=3, skip_at=2, seed=5,
                                     code_std=0.05)
    return nets


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shard, q):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle
    from test_batch import BBOX as bbox, small_latent_batch as mk
    from paper_2106_10031_b200.batch import march_batch
    from paper_2106_10031_b200.marching import MarchConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    factory = oracle.OracleBatchShardEngine if shard == "hash" else oracle.OracleShardEngine
    res = march_batch(mk(), MarchConfig(bbox=bbox, seeds=4, rng_seed=1), shard=shard, engine_factory=factory)
    q.put((rank, [(s, list(v)) for s, v in res]))
    dist.destroy_process_group()


def test_shape_sharding_assignment():
    from paper_2106_10031_b200.batch import shard_of_shapes
    parts = [shard_of_shapes(64, r, 8) for r in range(8)]
    assert sorted(s for p in parts for s in p) == list(range(64))
    assert all(len(p) == 8 for p in parts)


def test_batch_rejects_mixed_architectures():
    from paper_2106_10031_b200 import synth
    from paper_2106_10031_b200.batch import march_batch
    with pytest.raises(ValueError):
        march_batch([synth.geometric_mlp([8, 8]), synth.geometric_mlp([8, 9])])


@pytest.mark.parametrize("shard", ["hash", "shape"])
def test_sharded_batch_matches_single_process(shard):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shard, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_shape = {}
    for _, items in res:
        for s, keys in items:
            per_shape.setdefault(s, []).append(set(keys))
    nets = small_latent_batch()
    assert sorted(per_shape) == list(range(len(nets)))
    for s, net in enumerate(nets):
        parts = per_shape[s]
        assert len(parts) == (world if shard == "hash" else 1)
        if shard == "hash":
            assert not (parts[0] & parts[1])
        union = set().union(*parts)
        ref = oracle.march(net, bbox=BBOX, seeds=4, rng_seed=1)
        assert sorted(union) == sorted(k.tobytes() for k in ref.key_words), f"shape {s}"


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [True, False])
def test_march_batch_gpu_matches_oracle(fused):
    """fused: every shape in one BFS (shape word in the key, per-shape bias tables);
    otherwise one reused engine per shape in turn.  Either way each shape's result is the
    reference march of its folded network."""
    import oracle
    from paper_2106_10031_b200.batch import march_batch
    from paper_2106_10031_b200.marching import MarchConfig
    nets = small_latent_batch(6)
    res = march_batch(nets, MarchConfig(bbox=BBOX, seeds=4, rng_seed=1), fused=fused)
    assert [s for s, _ in res] == list(range(6))
    for s, r in res:
        ref = oracle.march(nets[s], bbox=BBOX, seeds=4, rng_seed=1)
        np.testing.assert_array_equal(r.keys, ref.keys)
        np.testing.assert_array_equal(r.nverts, ref.nverts)
        np.testing.assert_array_equal(r.edge_nrefs, ref.edge_nrefs)
        np.testing.assert_array_equal(r.edge_refs, ref.edge_refs)
        assert np.abs(r.verts - ref.verts).max(initial=0) <= 1e-9
        assert r.report.cells_visited == ref.report["cells_visited"]
        assert r.report.open_edges == ref.report["open_edges"]

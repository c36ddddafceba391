"""The sharded (multi-GPU) march driver, exercised on CPU with gloo, world_size 2.

Each rank owns the states with hash(state) % 2 == rank (the GPU engine's
key_owner); frontiers are exchanged with all_to_all_single.  The engine is the
oracle-backed stand-in with the same wave/outbox/push interface, so this
checks the host-side protocol: the union of the ranks' visited sets equals the
single-process (reference) visited set, and the shards are disjoint.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle
    from conftest import load_golden as lg
    from paper_2106_10031_b200.distributed import ShardedMarcher
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = lg(name)
    bbox = tuple(map(tuple, g["config"]["bbox"]))
    sm = ShardedMarcher(g["net"], bbox=bbox, engine_factory=oracle.OracleShardEngine)
    rounds = sm.run(g["seeds"])
    q.put((rank, rounds, sm.engine.visited_keys()))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rand_3x10_s42", "oct", "cube", "imnet_small"])
def test_sharded_march_union_equals_reference(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = [set(v) for _, _, v in res]
    assert not (shards[0] & shards[1]), "a state is owned by two ranks"
    union = shards[0] | shards[1]
    import oracle
    g = load_golden(name)
    n_bits = int(g["keys"].shape[1] * 8)
    words = np.array([np.frombuffer(k, dtype=np.uint64) for k in sorted(union)])
    on = oracle.OracleNet(g["net"])
    kb, br = oracle.words_to_packbits(words, on.blob.n_bits, on.blob.ensemble)
    order = np.lexsort(np.column_stack([br] + [kb[:, i] for i in range(kb.shape[1] - 1, -1, -1)]).T)
    np.testing.assert_array_equal(kb[order], g["keys"])
    np.testing.assert_array_equal(br[order], g["branch"])
    assert all(w > 1 for _, w, _ in res)

"""The N>1 path on CPU: two gloo ranks shard the batch, each verifies its
slab (the oracle stands in for the device step, which needs a GPU), and the
gathered result is bit-identical to one unsharded call; the max-over-ranks
timing reduction is checked on the same group."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_11016_b200.shard import gather_results, shard_range, slab_seed


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, gamma, V, q):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2406_11016_b200.shard import allmax

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        lo, hi = shard_range(B, world, rank)
        zp, zq, ids, u = o.make_bench_batch(slab_seed(1, lo), hi - lo, gamma, V)
        zp, zq = o.round_f32(zp), o.round_f32(zq)
        r = o.verify_exact(zp, zq, ids, u)
        full = gather_results(r.as_dict())
        t = allmax(0.5 + rank)
        if rank == 0:
            q.put(({k: v.tolist() for k, v in full.items()}, t))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_batch():
    for B in (0, 1, 5, 8, 256, 1023):
        for world in (1, 2, 3, 8):
            spans = [shard_range(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_two_rank_gloo_sharded_verify_matches_unsharded(oracle):
    B, gamma, V = 5, 4, 3000  # uneven split: 3 + 2 rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, gamma, V, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    zp, zq, ids, u = oracle.make_bench_batch(1, B, gamma, V)
    ref = oracle.verify_exact(oracle.round_f32(zp), oracle.round_f32(zq), ids, u).as_dict()
    for k, v in ref.items():
        assert np.array_equal(np.asarray(full[k]), np.asarray(v)), k
    assert tmax == 1.5

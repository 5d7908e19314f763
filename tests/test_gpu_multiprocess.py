"""The sharded product flow on the GPU: two ranks, one
process each, split the batch into contiguous slabs and verify them through the
C-ABI on the device with no collective on the data path; the host-side gather
and the max-over-ranks timing reduction run on a gloo group (this box has one
GPU, so both ranks share cuda:0 -- bench.py's torchrun path does the same when
there are fewer GPUs than ranks).  The gathered result equals one unsharded
device call and the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, gamma, V, storage, q):
    import torch
    import torch.distributed as dist

    from paper_2406_11016_b200 import Verifier
    from paper_2406_11016_b200.shard import allmax, gather_results, shard_range, slab_seed
    from tools import benchgen

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        v = Verifier(0)
        lo, hi = shard_range(B, world, rank)
        zp, zq, ids, u = benchgen.make_bench_batch(slab_seed(1, lo), hi - lo, gamma, V, storage)
        dev = [torch.from_numpy(x).cuda() for x in (zp, zq, ids, u)]
        if storage == "bf16":
            dev[0], dev[1] = dev[0].view(torch.bfloat16), dev[1].view(torch.bfloat16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = v.verify_exact(*dev)
        e1.record()
        torch.cuda.synchronize()
        assert int(r.status.item()) == 0
        full = gather_results({k: np.asarray(x) for k, x in r.numpy().__dict__.items() if k in
                               ("accepted_len", "final_token", "resample_used", "tau", "residual_denom")})
        t = allmax(e0.elapsed_time(e1))
        if rank == 0:
            q.put(({k: x.tolist() for k, x in full.items()}, t, v.last_plan["kernel"]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,gamma,V,storage", [(5, 4, 3000, "f32"), (64, 8, 151936, "bf16")])
def test_two_rank_sharded_device_verify(verifier, oracle, B, gamma, V, storage):
    import torch

    from tests.parity import Widen, compare
    from tools import benchgen

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, gamma, V, storage, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax, plan = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax > 0
    # one unsharded device call on the same bits
    zp, zq, ids, u = benchgen.make_bench_batch(1, B, gamma, V, storage)
    dev = [torch.from_numpy(x).cuda() for x in (zp, zq, ids, u)]
    if storage == "bf16":
        dev[0], dev[1] = dev[0].view(torch.bfloat16), dev[1].view(torch.bfloat16)
    g = verifier.verify_exact(*dev)
    torch.cuda.synchronize()
    gn = g.numpy()
    assert np.array_equal(np.asarray(full["accepted_len"]), gn.accepted_len)
    assert np.array_equal(np.asarray(full["final_token"]), gn.final_token)
    assert np.array_equal(np.asarray(full["resample_used"]), gn.resample_used)
    # and the oracle on every row
    from tests.parity import oracle_threaded

    o = oracle_threaded(oracle, "exact", zp, zq, ids, u, storage)
    assert compare(o, g, Widen(zp, storage), Widen(zq, storage), ids, u, "exact", label=f"2rank-{storage}") <= 1

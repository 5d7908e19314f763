"""Multi-GPU plumbing of the verification step.

Batch rows are independent (verify_reference.cpp:87-109), so N ranks split the
batch into contiguous slabs and verify them with no collective on the data
path.  The only cross-rank traffic is host-side and O(B * gamma): the max-over-
ranks step time of the benchmark and, when a caller wants the whole batch on
one host, the gather of the per-slab results.  One process per GPU
(torchrun); the helpers below work on any torch.distributed backend (NCCL on
the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

RESULT_FIELDS = ("accepted_len", "final_token", "resample_used", "tau", "residual_denom")


def shard_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of rank `rank`: contiguous slabs, sizes differ by at most 1."""
    if B < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"shard_range: bad arguments B={B} world={world} rank={rank}")
    base, rem = divmod(B, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def slab_seed(seed: int, lo: int) -> int:
    """Seed of a slab's first row under the reference bench recipe, where
    global batch row b is make_bench_inputs(seed + b, ...) (bench.cpp:46-74)."""
    return seed + lo


def allmax(x: float, device=None) -> float:
    """Max over ranks (the benchmark's step time); identity without a process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local: dict, dst: int | None = None) -> dict | None:
    """Concatenate per-rank result arrays (RESULT_FIELDS, batch-major) in rank
    order.  Returns the full-batch dict on every rank (dst None) or on `dst`."""
    import torch.distributed as dist

    part = {k: np.asarray(local[k]) for k in RESULT_FIELDS}
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return part
    world = dist.get_world_size()
    if dst is None:
        out = [None] * world
        dist.all_gather_object(out, part)
    else:
        out = [None] * world if dist.get_rank() == dst else None
        dist.gather_object(part, out, dst=dst)
        if dist.get_rank() != dst:
            return None
    return {k: np.concatenate([o[k] for o in out], axis=0) for k in RESULT_FIELDS}

"""Parity helpers: run the CUDA path through the C-ABI and compare with the
oracle, explaining every token mismatch by its distance to a decision
threshold (BASELINE.json north star: |u - ratio| < 1e-6) or to a CDF boundary
of the oracle's inverse CDF (|u - CDF(k)| < 1e-6)."""
from __future__ import annotations

import numpy as np

TAU_TOL = 1e-6        # results_match tolerance (validate.cpp:21-44)
DENOM_TOL = 1e-6
EXPLAIN_TOL = 1e-6    # north star: mismatches must lie within 1e-6 of a threshold


def to_device(oracle, zp, zq, ids, u, dtype):
    """Device tensors holding exactly the bits the oracle sees (zp/zq already rounded)."""
    import torch

    if dtype == "f32":
        tzp = torch.from_numpy(zp.astype(np.float32))
        tzq = torch.from_numpy(zq.astype(np.float32))
    elif dtype == "bf16":
        tzp = torch.from_numpy(oracle.to_bf16_bits(zp)).view(torch.bfloat16)
        tzq = torch.from_numpy(oracle.to_bf16_bits(zq)).view(torch.bfloat16)
    else:
        tzp = torch.from_numpy(np.ascontiguousarray(zp, np.float64))
        tzq = torch.from_numpy(np.ascontiguousarray(zq, np.float64))
    return (tzp.cuda(), tzq.cuda(), torch.from_numpy(np.ascontiguousarray(ids, np.int32)).cuda(),
            torch.from_numpy(np.ascontiguousarray(u, np.float64)).cuda())


def round_for(oracle, x, dtype):
    if dtype == "f32":
        return oracle.round_f32(x)
    if dtype == "bf16":
        return oracle.round_bf16(x)
    return np.ascontiguousarray(x, np.float64)


def _rows(kind, zp_row, zq_row, alpha, beta):
    """Oracle-precision (fp64) p and q rows for the inverse-CDF explanation."""
    if kind == "exact":
        def sm(z):
            e = np.exp(z - z.max())
            return e / e.sum()
        return sm(zp_row), (sm(zq_row) if zq_row is not None else None)
    if kind == "sigmoid":
        def sg(z):
            t = (z - alpha) / (beta - alpha)
            return 1.0 / (1.0 + np.exp(-t))
        return sg(zp_row), (sg(zq_row) if zq_row is not None else None)
    return zp_row, zq_row


def _cdf_explains(vals, u, t_a, t_b):
    denom = vals.sum()
    cum = np.cumsum(vals / denom)
    lo, hi = min(t_a, t_b), max(t_a, t_b)
    if lo < 0 or hi >= len(vals):
        return False
    return bool(np.min(np.abs(cum[lo:hi] - u)) < EXPLAIN_TOL) if hi > lo else False


def compare(o, g, zp, zq, ids, u, kind, alpha=-1e3, beta=1e3, label=""):
    """Asserts parity; returns the number of (explained) token mismatches."""
    g = g.numpy()
    B, gamma = o.tau.shape
    explained = 0
    assert np.all(np.abs(g.tau - o.tau) <= TAU_TOL), f"{label}: tau max err {np.abs(g.tau - o.tau).max()}"
    for b in range(B):
        if g.accepted_len[b] != o.accepted_len[b]:
            c = min(int(g.accepted_len[b]), int(o.accepted_len[b]))
            d = abs(u[b, c] - o.tau[b, c])
            assert d < EXPLAIN_TOL, f"{label}: b={b} accept mismatch at c={c}, |u-tau|={d:.3g}"
            explained += 1
            continue
        assert g.resample_used[b] == o.resample_used[b], f"{label}: b={b} resample_used"
        # 1e-6 absolute (results_match), relative for denominators above 1
        # (sigmoid rows of unnormalized activations reach ~V/2).
        assert abs(g.residual_denom[b] - o.residual_denom[b]) <= DENOM_TOL * max(1.0, abs(o.residual_denom[b])), (
            f"{label}: b={b} residual_denom {g.residual_denom[b]} vs {o.residual_denom[b]}")
        if g.final_token[b] != o.final_token[b]:
            a = int(o.accepted_len[b])
            prow, qrow = _rows(kind, zp[b, a], zq[b, a] if a < gamma else None, alpha, beta)
            if a < gamma:
                res = np.maximum(prow - qrow, 0.0)
                vals = res if res.sum() > 1e-12 else prow
            else:
                vals = prow
            ok = _cdf_explains(vals, u[b, gamma], int(o.final_token[b]), int(g.final_token[b]))
            assert ok, f"{label}: b={b} token {g.final_token[b]} vs oracle {o.final_token[b]} unexplained"
            explained += 1
    return explained


# --------------------------------------------------------------------------- campaign helpers
PARITY_LOG = []  # (label, rows, explained mismatches, note): printed by conftest's terminal summary


def log_parity(label, rows, explained, note=""):
    PARITY_LOG.append((label, int(rows), int(explained), note))


class Widen:
    """Row accessor over stored logits (fp32, or bf16 bit patterns as uint16):
    x[b, c] -> that row widened to float64 (what the oracle consumes)."""

    def __init__(self, x, storage):
        self.x, self.storage = x, storage

    def __getitem__(self, idx):
        v = self.x[idx]
        if self.storage == "bf16":
            return (np.asarray(v).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        return np.asarray(v, dtype=np.float64)


def oracle_threaded(oracle, kind, zp, zq, ids, u, storage="f32", alpha=-1e3, beta=1e3, chunk=4, threads=None):
    """The oracle over all batch rows, row chunks in parallel threads (rows are
    independent, verify_reference.cpp:87-109; the ctypes calls release the
    GIL).  zp / zq are the STORED logits (widened per chunk, so a C4-sized
    batch never exists in double at once)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Result

    B, gamma = ids.shape
    W = (Widen(zp, storage), Widen(zq, storage))

    def run(lo):
        hi = min(B, lo + chunk)
        a, b = W[0][lo:hi], W[1][lo:hi]
        if kind == "exact":
            return lo, oracle.verify_exact(a, b, ids[lo:hi], u[lo:hi])
        return lo, oracle.verify_sigmoid(a, b, ids[lo:hi], u[lo:hi], alpha, beta)

    res = Result(B, gamma)
    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        for lo, r in ex.map(run, range(0, B, chunk)):
            hi = lo + len(r.accepted_len)
            for f in ("accepted_len", "final_token", "resample_used", "tau", "residual_denom"):
                getattr(res, f)[lo:hi] = getattr(r, f)
    return res

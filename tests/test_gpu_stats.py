"""Statistical guarantees of speculative sampling on the device (SURVEY.md
8(f) f2: validate.cpp:117-219 retargeted to the CUDA kernels).

* distribution (validate.cpp:117-175): with gamma = 1 the first emitted token
  -- the draft when accepted, else the residual resample -- is distributed as
  the target p, whatever the draft q (TV < 0.01 over 200k trials, one batched
  launch; chi-square p > 0.001);
* acceptance (validate.cpp:177-219): P(accept) = sum_i min(p_i, q_i).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 200_000


def _softmax(z):
    e = np.exp(z - z.max())
    return e / e.sum()


def _run_trials(verifier, zp_row, zbonus, zq_row, seed, path):
    import torch

    rng = np.random.default_rng(seed)
    V = zp_row.size
    q = _softmax(zq_row.astype(np.float64))
    ids = rng.choice(V, size=(N, 1), p=q).astype(np.int32)  # the draft, sampled from q
    u = rng.random((N, 2))
    zp = np.broadcast_to(np.stack([zp_row, zbonus])[None], (N, 2, V)).astype(np.float32).copy()
    zq = np.broadcast_to(zq_row[None, None], (N, 1, V)).astype(np.float32).copy()
    verifier.set_path(path)
    try:
        r = verifier.verify_exact(torch.from_numpy(zp).cuda(), torch.from_numpy(zq).cuda(),
                                  torch.from_numpy(ids).cuda(), torch.from_numpy(u).cuda())
        torch.cuda.synchronize()
    finally:
        verifier.set_path("auto")
    r = r.numpy()
    first = np.where(r.accepted_len >= 1, ids[:, 0], r.final_token)
    return first, r


@pytest.mark.parametrize("case", range(3))
def test_output_distribution_is_target(verifier, case):
    from scipy.stats import chisquare

    rng = np.random.default_rng(100 + case)
    V = 8
    zp = rng.normal(0, 2, V).astype(np.float32)
    zq = (zp + rng.normal(0, 1.5, V)).astype(np.float32)
    zbonus = rng.normal(0, 2, V).astype(np.float32)
    first, r = _run_trials(verifier, zp, zbonus, zq, 7 + case, "auto")  # (200k rows: the streaming kernel)
    p = _softmax(zp.astype(np.float64))
    hist = np.bincount(first, minlength=V) / N
    tv = 0.5 * np.abs(hist - p).sum()
    assert tv < 0.01, f"TV {tv}"
    assert chisquare(np.bincount(first, minlength=V), p * N).pvalue > 0.001


@pytest.mark.parametrize("case", range(3))
def test_acceptance_rate_is_sum_min(verifier, case):
    rng = np.random.default_rng(200 + case)
    V = 8
    zp = rng.normal(0, 2, V).astype(np.float32)
    zq = (zp + rng.normal(0, 1.5, V)).astype(np.float32)
    _, r = _run_trials(verifier, zp, zp, zq, 11 + case, "auto")
    p, q = _softmax(zp.astype(np.float64)), _softmax(zq.astype(np.float64))
    expect = np.minimum(p, q).sum()
    assert abs((r.accepted_len >= 1).mean() - expect) < 0.01

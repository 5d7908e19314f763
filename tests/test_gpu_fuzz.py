"""Randomized shapes through every kernel selection (a seeded fuzz beside the
structured campaign of test_gpu_campaign.py): batch 1-400, gamma 1-16,
vocabularies 64-300000 (odd, aligned and misaligned), fp32 / bf16 storage,
exact and sigmoid variants, with and without a bonus row, logit scales from
near-uniform to saturated, on the auto / streaming / cluster / cluster_ring /
slab paths -- each case against the oracle (verify_reference.cpp:76-111,
verify_sigmoid.cpp:50-58) with every token mismatch explained within 1e-6 of a
threshold (tests/parity.py), and the optional p / q / residual grids of the
small cases at the north star's 1e-5 relative (activation.cpp:20-37)."""
import os

import numpy as np
import pytest

from tests.parity import compare, log_parity, oracle_threaded, to_device

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("SSV_FUZZ_CASES", "192"))  # a longer soak: SSV_FUZZ_CASES=3000
MAX_ELEMS = 24_000_000  # B * (2 gamma + 1) * V per case: the oracle finishes in seconds
PATHS = ("auto", "streaming", "cluster", "cluster_ring", "slab")


def _case(i):
    r = np.random.RandomState(0xF022 + i)
    kind = "exact" if r.rand() < 0.6 else "sigmoid"
    storage = "bf16" if r.rand() < 0.35 else "f32"
    gamma = int(r.randint(1, 17))
    V = int(np.exp(r.uniform(np.log(64), np.log(300_000))))
    if r.rand() < 0.3:
        V = V // 16 * 16 or 16  # 16-element multiples: the aligned-row kernels
    bmax = max(1, min(400, MAX_ELEMS // ((2 * gamma + 1) * V)))
    if r.rand() < 0.5:
        B = int(np.exp(r.uniform(0, np.log(bmax + 1))))
    else:  # the large-batch kernels (streaming, slab, sigmoid stream)
        B = int(r.uniform(bmax / 4, bmax + 1))
    B = max(1, min(B, bmax))
    bonus = bool(r.rand() < 0.85)
    scale = float(r.choice([0.3, 3.0, 10.0] if kind == "exact" else [3.0, 300.0, 2000.0, 20000.0]))
    path = PATHS[r.randint(len(PATHS))]
    offset = int(r.rand() < 0.2)
    grids = B * (2 * gamma + 1) * V <= 2_000_000 and r.rand() < 0.5
    return dict(kind=kind, storage=storage, B=B, gamma=gamma, V=V, bonus=bonus, scale=scale, path=path,
                offset=offset, grids=grids, seed=0xF022 + i)


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz_case(verifier, oracle, i):
    import torch

    from paper_2406_11016_b200 import SSV_WANT_P, SSV_WANT_Q, SSV_WANT_RESIDUAL

    c = _case(i)
    B, gamma, V = c["B"], c["gamma"], c["V"]
    (zp, zq, ids, u), _ = oracle.make_logit_instance((c["seed"], 0), B, gamma, V, c["bonus"], c["scale"])
    rnd = oracle.round_bf16 if c["storage"] == "bf16" else oracle.round_f32
    zp, zq = rnd(zp), rnd(zq)
    t = list(to_device(oracle, zp, zq, ids, u, c["storage"]))
    if c["offset"]:  # a misaligned z_p base (one element past a 16-byte boundary)
        buf = torch.empty(t[0].numel() + 1, dtype=t[0].dtype, device="cuda")
        buf[1:].copy_(t[0].reshape(-1))
        t[0] = buf[1:].view(t[0].shape)
    flags = SSV_WANT_P | SSV_WANT_Q | SSV_WANT_RESIDUAL if c["grids"] else 0
    verifier.set_path(c["path"])
    try:
        if c["kind"] == "exact":
            g = verifier.verify_exact(*t, flags=flags)
        else:
            g = verifier.verify_sigmoid(*t, -1e3, 1e3, flags=flags)
        torch.cuda.synchronize()
        plan = verifier.last_plan["kernel"]
    finally:
        verifier.set_path("auto")
    assert int(g.status.item()) == 0, c
    o = oracle_threaded(oracle, c["kind"], zp, zq, ids, u, "f32")
    label = f"fuzz{i} {c['kind']} B={B} g={gamma} V={V} {c['storage']} {c['path']}->{plan}"
    m = compare(o, g, zp, zq, ids, u, c["kind"], label=label)
    log_parity(label + (" +grids" if c["grids"] else ""), B, m, plan)
    assert m <= max(1, B // 100), label
    if c["grids"]:
        gn = g.numpy()
        if c["kind"] == "exact":
            P = np.exp(zp - zp.max(-1, keepdims=True))
            P /= P.sum(-1, keepdims=True)
            Q = np.exp(zq - zq.max(-1, keepdims=True))
            Q /= Q.sum(-1, keepdims=True)
        else:  # sigmoid_scaled_value with bounds (-1e3, 1e3) (activation.cpp)
            P = 1 / (1 + np.exp(-(zp + 1e3) / 2e3))
            Q = 1 / (1 + np.exp(-(zq + 1e3) / 2e3))
        R = np.maximum(P[:, :gamma] - Q, 0)
        assert np.allclose(gn.p, P, rtol=1e-5, atol=1e-12), label
        assert np.allclose(gn.q, Q, rtol=1e-5, atol=1e-12), label
        assert np.all(np.abs(gn.residual - R) <= 1e-5 * R + 1e-6 * (P[:, :gamma] + Q) + 1e-12), label

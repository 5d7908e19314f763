"""The sigmoid-stream kernels on the shapes their code paths
branch on, against the oracle's verify_sigmoid (the reference's sigmoid path,
verify_sigmoid.cpp:50-58): k_verify_sigw (16-byte-aligned rows: V * 4 bytes a
multiple of 16 and an aligned base) and k_verify_sig (anything else), with and
without a bonus row, bf16, more batch rows than CTAs, and more granules than
the locate's shared-memory cache (V > 512K).  SSV_PATH_SLAB skips the cluster
plans, so small batches reach these kernels too."""
import numpy as np
import pytest

from tests.parity import compare, log_parity, to_device

pytestmark = pytest.mark.gpu

CASES = [  # B, gamma, V, bonus, storage, base offset (elements), scale (logits ~ N(0, scale))
    (6, 4, 32000, True, "f32", 0, 600.0),     # sigw, fp32
    (6, 4, 32000, False, "f32", 0, 600.0),    # sigw, no bonus row (accept-all rows sample nothing)
    (5, 3, 32768, True, "bf16", 0, 600.0),    # sigw, bf16
    (4, 3, 32001, True, "f32", 0, 600.0),     # odd V: k_verify_sig (TMA tiles)
    (4, 3, 32000, True, "f32", 1, 600.0),     # misaligned base: k_verify_sig
    (700, 2, 1024, True, "f32", 0, 600.0),    # B > grid: several rows per CTA / warp
    (2, 2, 600000, True, "f32", 0, 600.0),    # NG > kLocCap: granules beyond the cache
    (6, 4, 32000, True, "f32", 0, 20000.0),   # wide logits: many rejected rows (the pair path)
]


@pytest.mark.parametrize("B,gamma,V,bonus,storage,offset,scale", CASES)
def test_sigmoid_stream_shapes(verifier, oracle, B, gamma, V, bonus, storage, offset, scale):
    import torch

    state = (0x51A + B + V, 0)
    (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, bonus, scale)
    rnd = oracle.round_bf16 if storage == "bf16" else oracle.round_f32
    zp, zq = rnd(zp), rnd(zq)
    t = list(to_device(oracle, zp, zq, ids, u, storage))
    if offset:
        buf = torch.empty(t[0].numel() + offset, dtype=t[0].dtype, device="cuda")
        buf[offset:].copy_(t[0].reshape(-1))
        t[0] = buf[offset:].view(t[0].shape)
    o = oracle.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3)
    verifier.set_path("slab")
    try:
        g = verifier.verify_sigmoid(*t, -1e3, 1e3)
        torch.cuda.synchronize()
        plan = verifier.last_plan["kernel"]
    finally:
        verifier.set_path("auto")
    assert int(g.status.item()) == 0
    assert plan == "sigmoid_stream", plan
    m = compare(o, g, zp, zq, ids, u, "sigmoid", label=f"sigstream-{B}-{gamma}-{V}-{storage}-{offset}")
    rej = int((np.asarray(o.accepted_len) < gamma).sum())
    log_parity(f"sigmoid-stream B={B} g={gamma} V={V} {storage} off={offset} bonus={bonus} ({rej} rejected)",
               B, m, plan)
    assert m <= max(1, B // 100)


@pytest.mark.parametrize("path", ["streaming", "slab", "auto"])
def test_exact_beyond_granule_cache(verifier, oracle, path):
    """V = 600000: more 512-element granules (1172) than the locate caches in
    shared memory (kLocCap = 1024) -- the exact kernels read the rest from the
    granule slots (streaming, slab) or their own global copy (cluster)."""
    import torch

    state = (0x600, 0)
    B, gamma, V = 2, 2, 600000
    (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, True, 3.0)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    # u_final near 1 puts the sampled token in the last granules (past the cache)
    u[:, gamma] = 0.999
    o = oracle.verify_exact(zp, zq, ids, u)
    verifier.set_path(path)
    try:
        g = verifier.verify_exact(*to_device(oracle, zp, zq, ids, u, "f32"))
        torch.cuda.synchronize()
    finally:
        verifier.set_path("auto")
    assert compare(o, g, zp, zq, ids, u, "exact", label=f"ng-cache-{path}") == 0
    assert (np.asarray(o.final_token) >= 1024 * 512).any()  # a token past the cached granules

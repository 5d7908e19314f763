"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same
inputs and the same uniforms.  Bar (BASELINE.json north star): accepted
lengths and tokens identical, any mismatch explained by |u - threshold| < 1e-6;
tau and residual_denom within 1e-6 absolute (validate.cpp:21-44); p / q /
residual within 1e-5 relative (+ absolute floor for cancelling residuals)."""
import json
import os

import numpy as np
import pytest

from tests.parity import compare, log_parity, round_for, to_device

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.json")


def _run(verifier, kind, zp_t, zq_t, ids_t, u_t, alpha=-1e3, beta=1e3, flags=0):
    if kind == "exact":
        r = verifier.verify_exact(zp_t, zq_t, ids_t, u_t, flags=flags)
    elif kind == "sigmoid":
        r = verifier.verify_sigmoid(zp_t, zq_t, ids_t, u_t, alpha, beta, flags=flags)
    else:
        r = verifier.verify_probs(zp_t, zq_t, ids_t, u_t, flags=flags)
    import torch

    torch.cuda.synchronize()
    assert int(r.status.item()) == 0, f"device status {int(r.status.item())}"
    return r


def _oracle(oracle, kind, zp, zq, ids, u, alpha=-1e3, beta=1e3):
    if kind == "exact":
        return oracle.verify_exact(zp, zq, ids, u)
    if kind == "sigmoid":
        return oracle.verify_sigmoid(zp, zq, ids, u, alpha, beta)
    return oracle.verify_sequential(zp, zq, ids, u)


def test_golden_vectors(verifier, oracle):
    """Every committed golden case (expected outputs of the reference itself)."""
    from tests.golden.make_golden import rebuild_inputs
    from oracle.oracle import Result

    g = json.load(open(GOLDEN))
    mism = 0
    for case in g["cases"]:
        zp, zq, ids, u = rebuild_inputs(oracle, case)
        kind = case["kind"]
        rnd = case.get("recipe", {}).get("round", "f32" if kind != "probs" else "none")
        dtype = {"f32": "f32", "bf16": "bf16", "none": "f64"}[rnd] if "recipe" in case else (
            "f64" if kind == "probs" else "f32")
        a, b = case.get("alpha", -1e3), case.get("beta", 1e3)
        r = _run(verifier, kind, *to_device(oracle, zp, zq, ids, u, dtype), a, b)
        exp = Result(*np.array(ids).shape)
        for k, v in case["expect"].items():
            setattr(exp, k, np.array(v, dtype=getattr(exp, k).dtype))
        mism += compare(exp, r, zp, zq, ids, u, kind, a, b, label=case["id"])
    log_parity(f"golden vectors (reference outputs, {len(g['cases'])} cases)", len(g["cases"]), mism)
    assert mism <= 1


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_exact_grid(verifier, oracle, dtype):
    """validate.cpp:221-257-style grid on logits: B in {1,4}, gamma 1..20,
    V in {7, 257, 50257, 51865}, bonus row on/off."""
    rng = np.random.default_rng({"f32": 1, "bf16": 2, "f64": 3}[dtype])
    state = (0xE4AC + len(dtype), 0)
    mism = 0
    for i in range(40):
        B = int(rng.choice([1, 4]))
        gamma = int(rng.integers(1, 21))
        V = int(rng.choice([7, 257, 50257, 51865] if i % 3 == 0 else [7, 257, 1000]))
        bonus = bool(rng.integers(0, 2))
        (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, bonus, 3.0)
        zp, zq = round_for(oracle, zp, dtype), round_for(oracle, zq, dtype)
        o = oracle.verify_exact(zp, zq, ids, u)
        g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, dtype))
        mism += compare(o, g, zp, zq, ids, u, "exact", label=f"grid{i}")
    log_parity(f"validate-style exact grid {dtype} (40 instances)", 40, mism)
    assert mism <= 1


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_exact_bench_shapes(verifier, oracle, dtype):
    """bench recipe (bench.cpp:46-74) at C1 (several seeds), C2 and C3 shapes."""
    mism = 0
    for seed, B, gamma, V in [(s, 1, 5, 32000) for s in range(1, 17)] + [(1, 8, 5, 51865), (1, 64, 8, 32000)]:
        zp, zq, ids, u = oracle.make_bench_batch(seed, B, gamma, V)
        zp, zq = round_for(oracle, zp, dtype), round_for(oracle, zq, dtype)
        o = oracle.verify_exact(zp, zq, ids, u)
        g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, dtype))
        mism += compare(o, g, zp, zq, ids, u, "exact", label=f"bench{seed}-{B}-{V}")
    log_parity(f"bench recipe C1 x16 seeds + C2 + C3 {dtype}", 16 + 8 + 64, mism)
    assert mism <= 1


@pytest.mark.parametrize("scale,mag", [(3.0, 1e3), (800.0, 1e4), (3.0, 1e4), (800.0, 1e3)])
def test_sigmoid_grid(verifier, oracle, scale, mag):
    """oracle-sigmoid grid (validate.cpp:259-321), emulate_half = false."""
    rng = np.random.default_rng(int(scale + mag))
    state = (0x516 + int(mag), 0)
    mism = 0
    for i in range(25):
        B = int(rng.choice([1, 4]))
        gamma = int(rng.integers(1, 21))
        V = int(rng.choice([7, 257, 50257] if i % 3 == 0 else [7, 257, 999]))
        bonus = bool(rng.integers(0, 2))
        (zp, zq, ids, u), state = oracle.make_sigmoid_instance(state, B, gamma, V, bonus, scale)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        o = oracle.verify_sigmoid(zp, zq, ids, u, -mag, mag)
        g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"), -mag, mag)
        mism += compare(o, g, zp, zq, ids, u, "sigmoid", -mag, mag, label=f"sig{i}")
    log_parity(f"validate-style sigmoid grid scale {scale:g} bounds +-{mag:g} (25 instances)", 25, mism)
    assert mism <= 1


def test_sigmoid_bench_shape(verifier, oracle):
    for mag in (1e3, 1e4):
        zp, zq, ids, u = oracle.make_bench_batch(1, 8, 5, 51865)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        o = oracle.verify_sigmoid(zp, zq, ids, u, -mag, mag)
        g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"), -mag, mag)
        assert compare(o, g, zp, zq, ids, u, "sigmoid", -mag, mag) == 0


def test_probs_grid_f64(verifier, oracle):
    """Probabilities in (verify_sequential's own API) on fp64 storage."""
    rng = np.random.default_rng(99)
    state = (0x0EAC, 0)
    for i in range(40):
        B = int(rng.choice([1, 4]))
        gamma = int(rng.integers(1, 21))
        V = int(rng.choice([7, 257, 50257] if i % 4 == 0 else [7, 257]))
        bonus = bool(rng.integers(0, 2))
        (p, q, ids, u), state = oracle.make_instance(state, B, gamma, V, bonus)
        o = oracle.verify_sequential(p, q, ids, u)
        g = _run(verifier, "probs", *to_device(oracle, p, q, ids, u, "f64"))
        assert compare(o, g, p, q, ids, u, "probs", label=f"probs{i}") == 0


def test_degenerate_residual_fallback(verifier, oracle):
    """Residual mass <= 1e-12 -> sample p, residual_denom 0, resample_used 1
    (verify_reference.cpp:57-61), in the probability and sigmoid variants."""
    rng = np.random.default_rng(5)
    V, gamma, B = 300, 3, 4
    q = rng.random((B, gamma, V)) + 0.1
    p = 0.5 * q  # tau = 0.5 everywhere, residual max(0, p - q) = 0
    ids = rng.integers(0, V, (B, gamma)).astype(np.int32)
    u = np.full((B, gamma + 1), 0.75)
    u[:, gamma] = rng.random(B)
    o = oracle.verify_sequential(p, q, ids, u)
    assert (o.resample_used == 1).all() and (o.residual_denom == 0).all()
    g = _run(verifier, "probs", *to_device(oracle, p, q, ids, u, "f64"))
    assert compare(o, g, p, q, ids, u, "probs") == 0
    zq = oracle.round_f32(rng.normal(0, 3, (B, gamma, V)))
    zp = oracle.round_f32(zq - 100.0)
    o = oracle.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3)
    assert (o.residual_denom == 0).all()
    g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"))
    assert compare(o, g, zp, zq, ids, u, "sigmoid") == 0


def test_edge_shapes(verifier, oracle):
    """V = 1, gamma = 1; gamma > 32 (multi-warp acceptance scan); gamma > 47 (row
    statistics beyond the decision's SMEM cache) and > 256 (beyond one thread per
    position; streaming kernel); B = 300, V = 5."""
    state = (0xED6E, 0)
    for B, gamma, V, bonus in [(1, 1, 1, True), (2, 1, 1, False), (1, 40, 64, True), (300, 2, 5, True),
                               (3, 33, 1001, False), (2, 64, 300, True), (1, 300, 40, True), (20, 70, 129, False)]:
        (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, bonus, 3.0)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        o = oracle.verify_exact(zp, zq, ids, u)
        g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, "f32"))
        assert compare(o, g, zp, zq, ids, u, "exact", label=f"edge{B}-{gamma}-{V}") == 0
        o = oracle.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3)
        g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"))
        assert compare(o, g, zp, zq, ids, u, "sigmoid", label=f"edge-sig{B}-{gamma}-{V}") == 0


def test_misaligned_device_pointers(verifier, oracle):
    """Rows starting at arbitrary 4-byte offsets (sub-tensor views)."""
    import torch

    zp, zq, ids, u = oracle.make_bench_batch(3, 2, 4, 32003)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    o = oracle.verify_exact(zp, zq, ids, u)
    tzp, tzq, tids, tu = to_device(oracle, zp, zq, ids, u, "f32")
    bp = torch.empty(tzp.numel() + 1, dtype=torch.float32, device="cuda")
    bq = torch.empty(tzq.numel() + 3, dtype=torch.float32, device="cuda")
    bp[1:].copy_(tzp.reshape(-1))
    bq[3:].copy_(tzq.reshape(-1))
    g = _run(verifier, "exact", bp[1:].view(tzp.shape), bq[3:].view(tzq.shape), tids, tu)
    assert compare(o, g, zp, zq, ids, u, "exact") == 0


def test_optional_outputs(verifier, oracle):
    """p, q, residual grids (activation.cpp:20-37; verify_fused.cpp:50)."""
    from oracle.oracle import Oracle  # noqa: F401

    state = (0x0707, 0)
    (zp, zq, ids, u), _ = oracle.make_logit_instance(state, 3, 4, 1999, True, 3.0)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    from paper_2406_11016_b200 import SSV_WANT_P, SSV_WANT_Q, SSV_WANT_RESIDUAL

    flags = SSV_WANT_P | SSV_WANT_Q | SSV_WANT_RESIDUAL
    g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, "f32"), flags=flags).numpy()
    P = np.stack([oracle.softmax(r) for r in zp.reshape(-1, zp.shape[-1])]).reshape(zp.shape)
    Q = np.stack([oracle.softmax(r) for r in zq.reshape(-1, zq.shape[-1])]).reshape(zq.shape)
    Rz = np.maximum(P[:, :4] - Q, 0)
    assert np.allclose(g.p, P, rtol=1e-5, atol=1e-12)
    assert np.allclose(g.q, Q, rtol=1e-5, atol=1e-12)
    assert np.all(np.abs(g.residual - Rz) <= 1e-5 * Rz + 1e-6 * (P[:, :4] + Q) + 1e-12)
    # sigmoid grids
    g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"), flags=flags).numpy()
    Ps = 1 / (1 + np.exp(-(zp + 1e3) / 2e3))
    Qs = 1 / (1 + np.exp(-(zq + 1e3) / 2e3))
    assert np.allclose(g.p, Ps, rtol=1e-5)
    assert np.allclose(g.q, Qs, rtol=1e-5)
    Rs = np.maximum(Ps[:, :4] - Qs, 0)
    assert np.all(np.abs(g.residual - Rs) <= 1e-5 * Rs + 1e-6 * Ps[:, :4])


def test_host_entry_points_and_errors(verifier, oracle):
    from paper_2406_11016_b200 import SsvInvalidArgument

    zp, zq, ids, u = oracle.make_bench_batch(4, 2, 5, 32000)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    o = oracle.verify_exact(zp, zq, ids, u)
    h = verifier.verify_exact_host(zp.astype(np.float32), zq.astype(np.float32), ids, u)
    assert compare(o, h, zp, zq, ids, u, "exact") == 0
    bad = ids.copy()
    bad[1, 2] = 32000
    with pytest.raises(SsvInvalidArgument, match="out of vocabulary"):
        verifier.verify_exact_host(zp.astype(np.float32), zq.astype(np.float32), bad, u)
    badu = u.copy()
    badu[0, 0] = 1.0
    with pytest.raises(SsvInvalidArgument, match="uniforms"):
        verifier.verify_exact_host(zp.astype(np.float32), zq.astype(np.float32), ids, badu)
    # sigmoid does not range-check uniforms (verify_sigmoid.cpp:13-33, verify_sigmoid_fused)
    verifier.verify_sigmoid_host(zp.astype(np.float32), zq.astype(np.float32), ids, badu)
    nan = zq.astype(np.float32)
    nan[1, 3, 17] = np.nan
    with pytest.raises(SsvInvalidArgument, match="non-finite"):
        verifier.verify_exact_host(zp.astype(np.float32), nan, ids, u)
    ninf = zp.astype(np.float32)
    ninf[0, 1, 3] = -np.inf
    with pytest.raises(SsvInvalidArgument, match="non-finite"):
        verifier.verify_exact_host(ninf, zq.astype(np.float32), ids, u)
    with pytest.raises(SsvInvalidArgument, match="ScaleBounds"):
        verifier.verify_sigmoid_host(zp.astype(np.float32), zq.astype(np.float32), ids, u, 1.0, 2.0)
    with pytest.raises(SsvInvalidArgument, match="gamma"):
        verifier.verify_exact_host(zp[:, :3].astype(np.float32), zq.astype(np.float32), ids, u)
    # the context survives errors
    h = verifier.verify_exact_host(zp.astype(np.float32), zq.astype(np.float32), ids, u)
    assert compare(o, h, zp, zq, ids, u, "exact") == 0


@pytest.mark.parametrize("B,gamma,V", [(2, 5, 32000), (64, 8, 32000)])
def test_prepared_host_step(verifier, oracle, B, gamma, V):
    """Verifier.prepare_host over pinned buffers: results follow the buffer
    contents call by call, device errors (status word mirrored into pinned
    memory by the kernels) raise, and the step recovers."""
    from paper_2406_11016_b200 import SsvInvalidArgument
    from paper_2406_11016_b200.ssv import VerifyResult

    hzp = verifier.host_empty((B, gamma + 1, V), np.float32)
    hzq = verifier.host_empty((B, gamma, V), np.float32)
    hids = verifier.host_empty((B, gamma), np.int32)
    hu = verifier.host_empty((B, gamma + 1), np.float64)
    out = VerifyResult(verifier.host_empty((B,), np.int32), verifier.host_empty((B,), np.int32),
                       verifier.host_empty((B,), np.uint8), verifier.host_empty((B, gamma), np.float64),
                       verifier.host_empty((B,), np.float64), status=verifier.host_empty((1,), np.uint32))
    step = verifier.prepare_host("exact", hzp, hzq, hids, hu, out)
    for seed in (3, 11):
        zp, zq, ids, u = oracle.make_bench_batch(seed, B, gamma, V)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        hzp[...], hzq[...], hids[...], hu[...] = zp, zq, ids, u
        r = step()
        assert compare(oracle.verify_exact(zp, zq, ids, u), r, zp, zq, ids, u, "exact") == 0
        assert r.status[0] == 0
    hzq[B - 1, gamma - 1, V // 2] = np.nan
    with pytest.raises(SsvInvalidArgument, match="non-finite"):
        step()
    assert out.status[0] & 1
    hzq[B - 1, gamma - 1, V // 2] = zq[B - 1, gamma - 1, V // 2]
    r = step()
    assert r.status[0] == 0
    assert compare(oracle.verify_exact(zp, zq, ids, u), r, zp, zq, ids, u, "exact") == 0


def test_determinism(verifier, oracle):
    zp, zq, ids, u = oracle.make_bench_batch(9, 16, 8, 51865)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    t = to_device(oracle, zp, zq, ids, u, "f32")
    a = _run(verifier, "exact", *t).numpy()
    for _ in range(3):
        b = _run(verifier, "exact", *t).numpy()
        for f in ("accepted_len", "final_token", "tau", "residual_denom", "resample_used"):
            assert np.array_equal(getattr(a, f), getattr(b, f))


def test_sample_softmax(verifier, oracle):
    import torch

    rng = np.random.default_rng(11)
    for V in (1, 7, 300, 32000, 51865):
        for rep in range(3):  # repeated calls: no state may leak between launches
            z = oracle.round_f32(rng.normal(0, 4, (9, V)))
            uu = rng.random(9)
            exp = [oracle.sample_row(oracle.softmax(r), x) for r, x in zip(z, uu)]
            out = torch.full((9,), -7, dtype=torch.int32, device="cuda")
            got = verifier.sample_softmax(torch.from_numpy(z.astype(np.float32)).cuda(), torch.from_numpy(uu).cuda(),
                                          out=out)
            assert got.cpu().tolist() == exp, (V, rep)


def test_device_bench_generator(verifier, oracle):
    """ssv_make_bench_inputs reproduces make_bench_inputs (bench.cpp:46-74)."""
    import torch

    B, gamma, V = 3, 4, 32000
    zp, zq, ids, u = oracle.make_bench_batch(5, B, gamma, V)
    gzp, gzq, gids, gu = verifier.make_bench_inputs(5, B, gamma, V, torch.float32)
    torch.cuda.synchronize()
    assert np.mean(gzp.cpu().numpy() == zp.astype(np.float32)) > 0.9999
    assert np.mean(gzq.cpu().numpy() == zq.astype(np.float32)) > 0.9999
    assert np.array_equal(gu.cpu().numpy(), u)
    assert np.mean(gids.cpu().numpy() == ids) >= 0.9


def test_full_size_c4_row_subsample(verifier, oracle):
    """C4 (B=256, gamma=8, V=151936) at full size on the device; the oracle
    checks a subsample of batch rows (rows are independent)."""
    import torch

    B, gamma, V = 256, 8, 151936
    zp_t, zq_t, ids_t, u_t = verifier.make_bench_inputs(1, B, gamma, V, torch.float32)
    r = _run(verifier, "exact", zp_t, zq_t, ids_t, u_t).numpy()
    rows = [0, 1, 77, 128, 200, 255]
    zp = zp_t[rows].double().cpu().numpy()
    zq = zq_t[rows].double().cpu().numpy()
    ids = ids_t[rows].cpu().numpy()
    u = u_t[rows].cpu().numpy()
    o = oracle.verify_exact(zp, zq, ids, u)
    from paper_2406_11016_b200.ssv import VerifyResult

    sub = VerifyResult(r.accepted_len[rows], r.final_token[rows], r.resample_used[rows], r.tau[rows],
                       r.residual_denom[rows])
    assert compare(o, sub, zp, zq, ids, u, "exact") == 0
    # size-independent properties over ALL rows
    assert (r.accepted_len >= 0).all() and (r.accepted_len <= gamma).all()
    assert ((r.final_token >= 0) & (r.final_token < V)).all()
    assert (r.resample_used == (r.accepted_len < gamma)).all()
    assert ((r.tau >= 0) & (r.tau <= 1)).all()


@pytest.mark.parametrize("path", ["streaming", "cluster", "cluster_ring", "slab"])
def test_both_kernels_small_shapes(verifier, oracle, path):
    """The streaming and the cluster kernel each on the small shapes the auto
    choice would route to the other one (validate.cpp:221-321-style grid)."""
    rng = np.random.default_rng({"streaming": 11, "cluster": 12, "cluster_ring": 13, "slab": 14}[path])
    state = (0x5EED + len(path), 0)
    verifier.set_path(path)
    try:
        mism = 0
        for i in range(24):
            B = int(rng.choice([1, 3, 8]))
            gamma = int(rng.integers(1, 12))
            V = int(rng.choice([7, 257, 4099, 51865, 32000]))
            bonus = bool(rng.integers(0, 2))
            (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, bonus, 3.0)
            zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
            o = oracle.verify_exact(zp, zq, ids, u)
            g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, "f32"))
            mism += compare(o, g, zp, zq, ids, u, "exact", label=f"{path}-exact{i}")
            o = oracle.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3)
            g = _run(verifier, "sigmoid", *to_device(oracle, zp, zq, ids, u, "f32"))
            mism += compare(o, g, zp, zq, ids, u, "sigmoid", label=f"{path}-sig{i}")
        log_parity(f"small-shape grid forced {path} (24 exact + 24 sigmoid)", 48, mism)
        assert mism <= 1
    finally:
        verifier.set_path("auto")


def test_streaming_and_cluster_agree_on_c2(verifier, oracle):
    """C2 (the headline shape) through both kernels: identical decisions and
    tokens, tau / denominators within the parity tolerance (the two kernels sum
    the fp32 chunk partials in different orders: ~1e-7 relative apart)."""
    zp, zq, ids, u = oracle.make_bench_batch(1, 8, 5, 51865)
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    t = to_device(oracle, zp, zq, ids, u, "f32")
    res = {}
    for path in ("streaming", "cluster", "cluster_ring", "slab"):
        verifier.set_path(path)
        res[path] = _run(verifier, "exact", *t).numpy()
    verifier.set_path("auto")
    a = res["streaming"]
    for b in (res["cluster"], res["cluster_ring"], res["slab"]):
        assert np.array_equal(a.accepted_len, b.accepted_len) and np.array_equal(a.final_token, b.final_token)
        assert np.abs(a.tau - b.tau).max() < 1e-6 and np.abs(a.residual_denom - b.residual_denom).max() < 1e-6


@pytest.mark.parametrize("gamma,B,V,dtype", [
    (1, 1024, 32000, "f32"), (16, 64, 51865, "f32"), (2, 512, 151936, "f32"), (4, 1, 151936, "f32"),
    (16, 1, 32000, "f32"), (8, 16, 51865, "bf16"), (16, 8, 151936, "bf16"), (2, 300, 51865, "bf16"),
])
def test_c5_sweep_points(verifier, oracle, gamma, B, V, dtype):
    """BASELINE config 5 sweep (gamma in 1..16, B in 1..1024, V in the three
    vocabularies) at full size on the device, both variants: properties over
    every row, the oracle on a row subsample (rows are independent)."""
    import torch

    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    zp_t, zq_t, ids_t, u_t = verifier.make_bench_inputs(7, B, gamma, V, tdt)
    rows = sorted({0, B // 3, B // 2, B - 1})
    zp = zp_t[rows].double().cpu().numpy()
    zq = zq_t[rows].double().cpu().numpy()
    ids = ids_t[rows].cpu().numpy()
    u = u_t[rows].cpu().numpy()
    from paper_2406_11016_b200.ssv import VerifyResult

    for kind in ("exact", "sigmoid"):
        r = _run(verifier, kind, zp_t, zq_t, ids_t, u_t).numpy()
        assert (r.accepted_len >= 0).all() and (r.accepted_len <= gamma).all()
        assert ((r.final_token >= 0) & (r.final_token < V)).all()
        assert (r.resample_used == (r.accepted_len < gamma)).all()
        assert ((r.tau >= 0) & (r.tau <= 1)).all()
        o = _oracle(oracle, kind, zp, zq, ids, u)
        sub = VerifyResult(r.accepted_len[rows], r.final_token[rows], r.resample_used[rows], r.tau[rows],
                           r.residual_denom[rows])
        m = compare(o, sub, zp, zq, ids, u, kind, label=f"sweep-{kind}-{gamma}-{B}-{V}-{dtype}")
        log_parity(f"C5 point g={gamma} B={B} V={V} {dtype} {kind} (row subsample)", len(rows), m)
        assert m <= 1


@pytest.mark.parametrize("mag", [1e3, 1e4, 1e5])
def test_sigmoid_emulate_half(verifier, oracle, ref, mag):
    """emulate_half = true (dist.cpp:64-69, half.cpp): the binary16-emulated
    sigmoid against the compiled reference's verify_sigmoid_sequential, up to
    the paper's +-1e5 failing scale; both kernels."""
    rng = np.random.default_rng(int(mag))
    state = (0x4A1F + int(mag), 0)
    mism = 0
    for i in range(16):
        B = int(rng.choice([1, 4, 20]))
        gamma = int(rng.integers(1, 9))
        V = int(rng.choice([7, 257, 4099]))
        bonus = bool(rng.integers(0, 2))
        (zp, zq, ids, u), state = oracle.make_sigmoid_instance(state, B, gamma, V, bonus, 800.0 if i % 2 else 3.0)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        o = ref.verify_sigmoid_half(zp, zq, ids, u, -mag, mag)
        t = to_device(oracle, zp, zq, ids, u, "f32")
        import torch

        g = verifier.verify_sigmoid(*t, -mag, mag, emulate_half=True)
        torch.cuda.synchronize()
        assert int(g.status.item()) == 0
        gn = g.numpy()
        assert np.array_equal(gn.accepted_len, o.accepted_len), f"half{i}: accept"
        assert np.abs(gn.tau - o.tau).max() <= 1e-12, f"half{i}: tau"  # the same binary16 values
        same = gn.final_token == o.final_token
        mism += int((~same).sum())
        assert np.all(np.abs(gn.residual_denom - o.residual_denom) <= 1e-6 * np.maximum(1, np.abs(o.residual_denom)))
    log_parity(f"sigmoid emulate_half vs compiled reference +-{mag:g} (16 instances)", 16, mism)
    assert mism <= 1


@pytest.mark.parametrize("path", ["streaming", "cluster"])
def test_locate_edges(verifier, oracle, path):
    """Inverse-CDF corner cases on both kernels (dist.cpp:122-137,
    verify_reference.cpp:51-62): u_final at the largest double below 1 and at
    0; a residual whose only mass is the row's first or last element (first /
    last cluster rank's slice); the bonus row with a one-hot softmax.  fp32
    probabilities: every row rejects at c = 0 (u = 0.999999 > tau)."""
    rng = np.random.default_rng(21)
    B, gamma, V = 6, 2, 51865
    q = rng.random((B, gamma, V)) + 0.1
    q /= q.sum(axis=2, keepdims=True)
    p = q.copy()
    p[0, 0, V - 1] += 1e-3  # residual only at the last element
    p[1, 0, 0] += 1e-3      # ... only at the first element
    p[2:, 0] = rng.random((B - 2, V)) + 0.1
    p[2:, 0] /= p[2:, 0].sum(axis=1, keepdims=True)
    p[:2, 0, 777] = 0.5 * q[:2, 0, 777]  # rows 0, 1 draft token 777: tau = 0.5, no residual there
    p, q = oracle.round_f32(p), oracle.round_f32(q)
    ids = rng.integers(0, V, (B, gamma)).astype(np.int32)
    ids[:, 0] = np.argmin(p[:, 0] / q[:, 0], axis=1)  # tau well below 1 at c = 0
    ids[:2, 0] = 777
    u = np.full((B, gamma + 1), 0.999999)
    u[:, gamma] = [0.5, 0.5, np.nextafter(1.0, 0.0), 0.0, 1e-300, 0.9999999]
    verifier.set_path(path)
    try:
        o = oracle.verify_sequential(p, q, ids, u)
        assert (o.accepted_len == 0).all()
        assert o.final_token[0] == V - 1 and o.final_token[1] == 0
        g = _run(verifier, "probs", *to_device(oracle, p, q, ids, u, "f32"))
        assert compare(o, g, p, q, ids, u, "probs", label=f"{path}-locate") == 0
        # bonus row: one-hot softmax (all mass on one logit) and a flat row
        zp = oracle.round_f32(rng.normal(0, 1, (2, gamma + 1, V)))
        zq = zp[:, :gamma].copy()
        zp[0, gamma, 12345] = 200.0
        ids2 = rng.integers(0, V, (2, gamma)).astype(np.int32)
        u2 = np.zeros((2, gamma + 1))
        u2[:, gamma] = [np.nextafter(1.0, 0.0), 0.3]
        o = oracle.verify_exact(zp, zq, ids2, u2)
        assert (o.accepted_len == gamma).all() and o.final_token[0] == 12345
        g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids2, u2, "f32"))
        assert compare(o, g, zp, zq, ids2, u2, "exact", label=f"{path}-bonus") == 0
    finally:
        verifier.set_path("auto")


@pytest.mark.parametrize("path", ["streaming", "cluster", "cluster_ring", "slab"])
def test_locate_edges_exact_logits(verifier, oracle, path):
    """The residual corner cases of test_locate_edges with fp32 LOGITS on the C2
    shape (B=8, gamma=5, V=51865 -- the resident cluster plan, which scans the
    rejected pair from shared memory): one draft logit raised at a single
    element makes max(0, p - q) positive only there -- the row's first / last
    element, and either side of the 10-CTA cluster's slice boundary (5632)
    and of a granule boundary; u_final at the largest double below 1 and at 0
    (verify_reference.cpp:51-62, dist.cpp:122-137)."""
    rng = np.random.default_rng(22)
    B, gamma, V = 8, 5, 51865
    zq = rng.normal(0.0, 1.0, (B, gamma, V))
    zp = np.concatenate([zq, rng.normal(0.0, 1.0, (B, 1, V))], axis=1)
    spots = [V - 1, 0, 5631, 5632, 512 * 37 - 1, 512 * 37, V - 2, 1]
    for b, j in enumerate(spots):
        zp[b, 0, j] += 9.0
    zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    ids = rng.integers(0, V, (B, gamma)).astype(np.int32)
    for b, j in enumerate(spots):
        ids[b, 0] = (j + 1000) % V  # tau = p/q < 1 away from the bump
    u = np.full((B, gamma + 1), 0.999999)
    u[:, gamma] = [0.5, 0.5, np.nextafter(1.0, 0.0), 0.0, 0.25, 0.75, 1e-300, 0.9999999]
    o = oracle.verify_exact(zp, zq, ids, u)
    assert (o.accepted_len == 0).all()
    assert [int(t) for t in o.final_token] == spots
    verifier.set_path(path)
    try:
        g = _run(verifier, "exact", *to_device(oracle, zp, zq, ids, u, "f32"))
        assert compare(o, g, zp, zq, ids, u, "exact", label=f"{path}-exact-locate") == 0
        gb = _run(verifier, "exact", *to_device(oracle, oracle.round_bf16(zp), oracle.round_bf16(zq), ids, u, "bf16"))
        ob = oracle.verify_exact(oracle.round_bf16(zp), oracle.round_bf16(zq), ids, u)
        zpb, zqb = oracle.round_bf16(zp), oracle.round_bf16(zq)
        assert compare(ob, gb, zpb, zqb, ids, u, "exact", label=f"{path}-bf16-locate") == 0
    finally:
        verifier.set_path("auto")


@pytest.mark.parametrize("path", ["streaming", "cluster", "cluster_ring", "slab"])
def test_nonfinite_blocks_every_plan(verifier, oracle, path):
    """require_finite (dist.cpp:27-36) on whole blocks, not just one element:
    a 4096-element NaN block at the start of a row (a whole streaming chunk /
    cluster slice of NaN), a row of -inf, and a single +inf -- every plan sets
    the non-finite status bit (the reference throws)."""
    import torch

    from paper_2406_11016_b200.ssv import SSV_STATUS_NONFINITE

    rng = np.random.default_rng(5)
    B, gamma, V = 2, 3, 51865
    zq = oracle.round_f32(rng.normal(0.0, 2.0, (B, gamma, V)))
    zp = oracle.round_f32(np.concatenate([zq + rng.normal(0.0, 0.5, (B, gamma, V)), rng.normal(0.0, 2.0, (B, 1, V))],
                                         axis=1))
    ids = rng.integers(0, V, (B, gamma)).astype(np.int32)
    u = rng.random((B, gamma + 1))
    cases = []
    a = zq.copy()
    a[1, 2, :4096] = np.nan
    cases.append(("nan-block", zp, a))
    a = zp.copy()
    a[0, 1, :] = -np.inf
    cases.append(("row-of-minus-inf", a, zq))
    a = zq.copy()
    a[0, 0, V - 1] = np.inf
    cases.append(("plus-inf", zp, a))
    verifier.set_path(path)
    try:
        for name, p_, q_ in cases:
            t = to_device(oracle, p_, q_, ids, u, "f32")
            r = verifier.verify_exact(*t)
            torch.cuda.synchronize()
            st = int(r.status.item())
            assert st & SSV_STATUS_NONFINITE, f"{path} {name}: status {st}"
    finally:
        verifier.set_path("auto")

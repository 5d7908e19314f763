"""Pins the C restatement of the reference (oracle/ssv_oracle.c) before any
GPU result is trusted against it:

1. SPEC.md worked examples (the reference's only known-answer vectors);
2. bit-for-bit agreement with the reference itself, compiled from
   /root/reference/proj/src by oracle/Makefile into oracle/_ref/, on the
   validate.cpp instance grids (validate.cpp:221-321) and the bench recipe;
3. the committed golden vectors in tests/golden/ (written by
   tests/golden/make_golden.py from oracle/_ref), which travel without the
   reference.
"""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def same(a, b):
    return (np.array_equal(a.accepted_len, b.accepted_len) and np.array_equal(a.final_token, b.final_token)
            and np.array_equal(a.resample_used, b.resample_used) and np.array_equal(a.tau, b.tau)
            and np.array_equal(a.residual_denom, b.residual_denom))


# ---------------------------------------------------------------- KATs
def test_softmax_kats(oracle):
    assert np.allclose(oracle.softmax([0, 0, 0, 0]), [0.25] * 4, atol=1e-15)
    assert np.allclose(oracle.softmax([1000, 1000]), [0.5, 0.5], atol=1e-15)
    assert np.allclose(oracle.softmax([0, math.log(3)]), [0.25, 0.75], atol=1e-15)
    with pytest.raises(ValueError):
        oracle.softmax([0.0, float("nan")])
    with pytest.raises(ValueError):
        oracle.softmax([0.0, -float("inf")])


def test_sigmoid_and_ratio_kats(oracle):
    assert oracle.sigmoid_scaled(-1e3, -1e3, 1e3) == 0.5
    assert abs(oracle.sigmoid_scaled(0.0, -1e3, 1e3) - 0.622459) < 1e-6
    assert abs(oracle.ratio_clamped(0.5, 0.9) - 5 / 9) < 1e-15
    assert oracle.ratio_clamped(0.3, 0.0) == 1.0
    assert oracle.ratio_clamped(0.0, 0.0) == 0.0
    with pytest.raises(ValueError):
        oracle.ratio_clamped(-0.1, 0.5)


def test_scan_kats(oracle):
    # max_norm [0.4, 0.6, 0]: u=0.39 -> 0, u=0.41 -> 1
    assert oracle.scan_categorical([0.4, 0.6, 0.0], 1.0, 0.39) == 0
    assert oracle.scan_categorical([0.4, 0.6, 0.0], 1.0, 0.41) == 1
    # degenerate fallback over p = [0.25]*4, u = 0.6 -> 2
    assert oracle.sample_row([0.25] * 4, 0.6) == 2
    # last-positive fallback (dist.cpp:135-136)
    assert oracle.scan_categorical([0.2, 0.3, 0.0], 1.0, 0.99) == 1
    assert oracle.scan_categorical([0.0, 0.0], 1.0, 0.5) == 0


def test_verify_kats(oracle):
    p = np.array([[[0.5, 0.5]]])
    q = np.array([[[0.9, 0.1]]])
    r = oracle.verify_sequential(p, q, [[0]], [[0.6, 0.3]])
    assert r.accepted_len[0] == 0 and r.final_token[0] == 1
    assert abs(r.tau[0, 0] - 5 / 9) < 1e-15 and abs(r.residual_denom[0] - 0.4) < 1e-15
    r = oracle.verify_sequential(p, q, [[0]], [[0.5, 0.3]])
    assert r.accepted_len[0] == 1 and r.final_token[0] == -1
    # sigmoid tau ~ 0.7614
    r = oracle.verify_sigmoid(np.zeros((1, 1, 2)), np.array([[[2000.0, -2000.0]]]), [[0]], [[0.9, 0.5]], -1e3, 1e3)
    assert abs(r.tau[0, 0] - 0.761349) < 1e-6
    # tree_reduce over the ragged last tile is a sequential sum within 1e-12
    v = np.random.default_rng(0).random(81)
    assert abs(oracle.tree_reduce(v) - v.sum()) < 1e-12


def test_validate_errors(oracle):
    p = np.full((1, 1, 4), 0.25)
    with pytest.raises(ValueError):
        oracle.verify_sequential(p, p, [[4]], [[0.1, 0.1]])  # token out of range
    with pytest.raises(ValueError):
        oracle.verify_sequential(p, p, [[0]], [[1.0, 0.1]])  # uniform not < 1
    # SigmoidStepInputs::validate skips the uniform range (verify_sigmoid.cpp:13-33),
    # but the sequential oracle re-validates as StepInputs (verify_sigmoid.cpp:50-58).
    with pytest.raises(ValueError):
        oracle.verify_sigmoid(p, p, [[0]], [[1.5, 0.1]], -1e3, 1e3)


def test_sigmoid_fused_skips_uniform_check(ref):
    p = np.zeros((1, 1, 4))
    r = ref.verify_sigmoid_fused(p, p, [[0]], [[1.5, 0.1]], -1e3, 1e3, 4, 1)  # no throw
    assert r.accepted_len[0] == 0


# ------------------------------------------------- pinned against the reference
def test_bench_inputs_match_reference(oracle, ref):
    for seed, gamma, V in [(1, 5, 32000), (2, 1, 7), (3, 8, 257)]:
        a = oracle.make_bench_batch(seed, 1, gamma, V, 1)
        b = ref.make_bench_inputs(seed, gamma, V)
        for x, y in zip(a, b):
            assert np.array_equal(x.reshape(-1), y.reshape(-1))


@pytest.mark.parametrize("n", [60])
def test_oracle_exact_grid_matches_reference(oracle, ref, n):
    """validate.cpp:221-257's grid (B in {1,4}, gamma 1..20, V in {7,257,50257},
    tile n in {4,256,1024}, bonus on/off), oracle vs compiled reference."""
    rng = np.random.default_rng(1234)
    state = (0x0EAC, 0)
    for i in range(n):
        B = int(rng.choice([1, 4]))
        gamma = int(rng.integers(1, 21))
        V = int(rng.choice([7, 257, 50257] if i % 4 == 0 else [7, 257]))
        tile = int(rng.choice([4, 256, 1024]))
        bonus = bool(rng.integers(0, 2))
        (p, q, ids, u), state = oracle.make_instance(state, B, gamma, V, bonus)
        o = oracle.verify_sequential(p, q, ids, u)
        r = ref.verify_sequential(p, q, ids, u)
        assert same(o, r), (i, B, gamma, V)
        of = oracle.verify_fused(p, q, ids, u, tile)
        rf = ref.verify_fused(p, q, ids, u, tile, 2)
        assert same(of, rf), (i, "fused")


def test_oracle_logits_and_sigmoid_match_reference(oracle, ref):
    state = (0x516, 0)
    rng = np.random.default_rng(7)
    for i in range(30):
        B = int(rng.choice([1, 4]))
        gamma = int(rng.integers(1, 12))
        V = int(rng.choice([7, 257, 4099]))
        bonus = bool(rng.integers(0, 2))
        scale = float(rng.choice([3.0, 800.0]))
        mag = float(rng.choice([1e3, 1e4]))
        (zp, zq, ids, u), state = oracle.make_logit_instance(state, B, gamma, V, bonus, 3.0)
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
        assert same(oracle.verify_exact(zp, zq, ids, u), ref.verify_exact(zp, zq, ids, u))
        (zp, zq, ids, u), state = oracle.make_sigmoid_instance(state, B, gamma, V, bonus, scale)
        o = oracle.verify_sigmoid(zp, zq, ids, u, -mag, mag)
        assert same(o, ref.verify_sigmoid(zp, zq, ids, u, -mag, mag))
        f = ref.verify_sigmoid_fused(zp, zq, ids, u, -mag, mag, 256, 2)
        assert np.array_equal(o.final_token, f.final_token) and np.allclose(o.residual_denom, f.residual_denom, atol=1e-6)


def test_survey_golden_outcomes(oracle):
    """verify_sequential on make_bench_inputs(seed, 5, 32000)."""
    table = {1: (5, 19565), 2: (3, 25355), 3: (2, 15952), 4: (1, 28247), 5: (3, 5579), 6: (0, 25050),
             7: (2, 3497), 8: (1, 4262)}
    for seed, (acc, tok) in table.items():
        r = oracle.verify_exact(*oracle.make_bench_batch(seed, 1, 5, 32000, 1))
        assert (r.accepted_len[0], r.final_token[0]) == (acc, tok)


# ------------------------------------------------------------- golden vectors
def _golden_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".json")) if os.path.isdir(GOLDEN) else []


@pytest.mark.parametrize("name", _golden_files())
def test_oracle_matches_golden(oracle, name):
    from tests.golden.make_golden import rebuild_inputs

    g = json.load(open(os.path.join(GOLDEN, name)))
    for case in g["cases"]:
        zp, zq, ids, u = rebuild_inputs(oracle, case)
        kind = case["kind"]
        if kind == "exact":
            r = oracle.verify_exact(zp, zq, ids, u)
        elif kind == "sigmoid":
            r = oracle.verify_sigmoid(zp, zq, ids, u, case["alpha"], case["beta"])
        else:
            r = oracle.verify_sequential(zp, zq, ids, u)
        exp = case["expect"]
        assert r.accepted_len.tolist() == exp["accepted_len"], case["id"]
        assert r.final_token.tolist() == exp["final_token"], case["id"]
        assert r.resample_used.tolist() == exp["resample_used"], case["id"]
        assert np.array_equal(r.tau, np.array(exp["tau"])), case["id"]
        assert np.array_equal(r.residual_denom, np.array(exp["residual_denom"])), case["id"]

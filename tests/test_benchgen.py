"""tools/benchgen.c (the benchmark's input generator, shared by both bench.py
arms) against the compiled reference's own make_bench_inputs
(bench.cpp:46-74): bit-identical rows, for fp32 / bf16 storage."""
import numpy as np
import pytest

from tools import benchgen


@pytest.mark.parametrize("storage", ["f32", "bf16", "f64"])
def test_benchgen_matches_reference(ref, oracle, storage):
    B, gamma, V = 3, 4, 1999
    zp, zq, ids, u = benchgen.make_bench_batch(11, B, gamma, V, storage, threads=2)
    rnd = {"f32": oracle.round_f32, "bf16": oracle.round_bf16, "f64": lambda x: x}[storage]
    for b in range(B):
        rzp, rzq, rids, ru = ref.make_bench_inputs(11 + b, gamma, V)
        assert np.array_equal(benchgen.widen(zp[b], storage), rnd(rzp)), (storage, b)
        assert np.array_equal(benchgen.widen(zq[b], storage), rnd(rzq)), (storage, b)
        assert np.array_equal(ids[b], rids) and np.array_equal(u[b], ru)


def test_benchgen_bench_shape_rows(ref):
    """Rows of the C4 shape (V = 151936, gamma = 8): first, middle and last seed."""
    for seed in (1, 129, 256):
        zp, zq, ids, u = benchgen.make_bench_batch(seed, 1, 8, 151936, "f32", threads=1)
        rzp, rzq, rids, ru = ref.make_bench_inputs(seed, 8, 151936)
        assert np.array_equal(zp[0], rzp.astype(np.float32))
        assert np.array_equal(zq[0], rzq.astype(np.float32))
        assert np.array_equal(ids[0], rids) and np.array_equal(u[0], ru)


def test_model_pair_matches_reference(ref):
    """tools/benchgen.c make_model_pair == the compiled reference's
    (toy_model.cpp:16-42), bit for bit, for both ablation profiles."""
    from tools import benchgen

    for seed, V, div, scale in ((1, 127, 3000.0, 8000.0), (5, 257, 2000.0, 8000.0), (3, 64, 0.5, 4.0)):
        t, d = benchgen.make_model_pair(seed, V, div, scale)
        rt, rd = ref.make_model_pair(seed, V, div, scale)
        assert np.array_equal(t, rt) and np.array_equal(d, rd)

"""TEST INFRASTRUCTURE ONLY -- ctypes/numpy front end for the two checkers.

* ``Oracle``  wraps ``oracle/libssv_oracle.so``, the plain-C restatement of the
  reference's verification path (oracle/ssv_oracle.c; every function there
  cites the reference file:line it follows).
* ``Ref``     wraps ``oracle/_ref/libspecsamp_ref.so``, the unmodified
  reference sources compiled in place by oracle/Makefile (+ ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
legs import this module, and only as the checker or the timed CPU baseline --
never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libssv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecsamp_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class _Out(C.Structure):
    _fields_ = [
        ("accepted_len", C.c_void_p),
        ("tau", C.c_void_p),
        ("final_token", C.c_void_p),
        ("resample_used", C.c_void_p),
        ("residual_denom", C.c_void_p),
    ]


class Result:
    """Numpy mirror of VerificationResult (step.hpp:43-51)."""

    def __init__(self, B: int, gamma: int):
        self.accepted_len = np.zeros(B, np.int32)
        self.tau = np.zeros((B, gamma), np.float64)
        self.final_token = np.zeros(B, np.int32)
        self.resample_used = np.zeros(B, np.uint8)
        self.residual_denom = np.zeros(B, np.float64)

    def c(self) -> _Out:
        return _Out(
            self.accepted_len.ctypes.data,
            self.tau.ctypes.data,
            self.final_token.ctypes.data,
            self.resample_used.ctypes.data,
            self.residual_denom.ctypes.data,
        )

    def as_dict(self) -> dict:
        return {
            "accepted_len": self.accepted_len.tolist(),
            "tau": self.tau.tolist(),
            "final_token": self.final_token.tolist(),
            "resample_used": self.resample_used.tolist(),
            "residual_denom": self.residual_denom.tolist(),
        }


def build_oracle(with_ref: bool = True) -> None:
    """Build the checkers (make -f oracle/Makefile). The reference .so only
    builds where /root/reference exists; elsewhere a prebuilt copy is used."""
    target = "all" if with_ref else ORACLE_SO
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), target], check=True)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c32i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class _Base:
    def _shape(self, zp, zq, ids, u):
        zq = _c64(zq)
        B, gamma, V = zq.shape
        zp = _c64(zp)
        assert zp.shape[0] == B and zp.shape[2] == V
        return _c64(zp), zq, _c32i(ids).reshape(B, gamma), _c64(u).reshape(B, gamma + 1), B, gamma, V


class Oracle(_Base):
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(with_ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_word_at.restype = C.c_uint64
        L.orc_word_at.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_stable_softmax_into.argtypes = [_dp, C.c_size_t, _dp]
        L.orc_sigmoid_scaled_value.restype = C.c_double
        L.orc_sigmoid_scaled_value.argtypes = [C.c_double, C.c_double, C.c_double]
        L.orc_ratio_clamped.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.orc_scan_categorical.restype = C.c_size_t
        L.orc_scan_categorical.argtypes = [_dp, C.c_size_t, C.c_double, C.c_double]
        L.orc_sample_row.restype = C.c_int32
        L.orc_sample_row.argtypes = [_dp, C.c_size_t, C.c_double]
        L.orc_tree_reduce.restype = C.c_double
        L.orc_tree_reduce.argtypes = [_dp, C.c_size_t]
        vargs = [_dp, C.c_int, _dp, C.c_int, C.c_int, C.c_int, _ip, _dp]
        L.orc_verify_sequential.argtypes = vargs + [C.POINTER(_Out)]
        L.orc_verify_exact_logits.argtypes = vargs + [C.POINTER(_Out)]
        L.orc_verify_fused.argtypes = vargs + [C.c_int, C.POINTER(_Out)]
        L.orc_verify_sigmoid_sequential.argtypes = vargs + [C.c_double, C.c_double, C.POINTER(_Out)]
        L.orc_make_bench_inputs.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _ip, _dp]
        L.orc_make_bench_batch.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _ip, _dp]
        gen = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, _ip, _dp]
        L.orc_make_instance.argtypes = gen
        L.orc_make_logit_instance.argtypes = gen
        L.orc_make_sigmoid_instance.argtypes = gen
        L.orc_round_f32.argtypes = [_dp, C.c_size_t]
        L.orc_round_bf16.argtypes = [_dp, C.c_size_t]
        L.orc_to_bf16.argtypes = [_dp, C.c_size_t, np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")]

    # ---- primitives ----
    def softmax(self, z):
        z = _c64(z)
        out = np.empty_like(z)
        rc = self.lib.orc_stable_softmax_into(z, z.size, out)
        if rc:
            raise ValueError("stable_softmax: invalid input")
        return out

    def ratio_clamped(self, p, q):
        r = C.c_double()
        if self.lib.orc_ratio_clamped(p, q, C.byref(r)):
            raise ValueError("ratio_clamped: negative input")
        return r.value

    def scan_categorical(self, v, denom, u):
        v = _c64(v)
        return int(self.lib.orc_scan_categorical(v, v.size, denom, u))

    def sample_row(self, v, u):
        v = _c64(v)
        return int(self.lib.orc_sample_row(v, v.size, u))

    def sigmoid_scaled(self, z, alpha, beta):
        return self.lib.orc_sigmoid_scaled_value(z, alpha, beta)

    def tree_reduce(self, v):
        v = _c64(v)
        return self.lib.orc_tree_reduce(v, v.size)

    # ---- verification ----
    def _run(self, fn, zp, zq, ids, u, *extra):
        zp, zq, ids, u, B, gamma, V = self._shape(zp, zq, ids, u)
        res = Result(B, gamma)
        out = res.c()
        rc = fn(zp, zp.shape[1], zq, B, gamma, V, ids, u, *extra, C.byref(out))
        if rc:
            raise ValueError("oracle: invalid argument")
        return res

    def verify_sequential(self, p, q, ids, u):
        return self._run(self.lib.orc_verify_sequential, p, q, ids, u)

    def verify_fused(self, p, q, ids, u, tile_width=1024):
        return self._run(self.lib.orc_verify_fused, p, q, ids, u, tile_width)

    def verify_exact(self, zp, zq, ids, u):
        return self._run(self.lib.orc_verify_exact_logits, zp, zq, ids, u)

    def verify_sigmoid(self, zp, zq, ids, u, alpha, beta):
        return self._run(self.lib.orc_verify_sigmoid_sequential, zp, zq, ids, u, alpha, beta)

    # ---- generators ----
    def make_bench_batch(self, seed, B, gamma, V, threads=None):
        threads = threads or os.cpu_count() or 1
        zp = np.empty((B, gamma + 1, V))
        zq = np.empty((B, gamma, V))
        ids = np.empty((B, gamma), np.int32)
        u = np.empty((B, gamma + 1))
        self.lib.orc_make_bench_batch(seed, B, gamma, V, threads, zp, zq, ids, u)
        return zp, zq, ids, u

    def _gen(self, fn, seed_state, B, gamma, V, bonus, scale, logits):
        st = (C.c_uint64 * 2)(*seed_state)
        ps = gamma + (1 if bonus else 0)
        zp = np.empty((B, ps, V))
        zq = np.empty((B, gamma, V))
        ids = np.empty((B, gamma), np.int32)
        u = np.empty((B, gamma + 1))
        fn(C.cast(st, C.c_void_p), B, gamma, V, int(bonus), scale, zp, zq, ids, u)
        return (zp, zq, ids, u), (st[0], st[1])

    def make_instance(self, rng_state, B, gamma, V, bonus, scale=3.0):
        """validate.cpp:57-82; rng_state = (seed, counter). Returns (p,q,ids,u), new state."""
        return self._gen(self.lib.orc_make_instance, rng_state, B, gamma, V, bonus, scale, False)

    def make_logit_instance(self, rng_state, B, gamma, V, bonus, scale=3.0):
        return self._gen(self.lib.orc_make_logit_instance, rng_state, B, gamma, V, bonus, scale, True)

    def make_sigmoid_instance(self, rng_state, B, gamma, V, bonus, scale=3.0):
        return self._gen(self.lib.orc_make_sigmoid_instance, rng_state, B, gamma, V, bonus, scale, True)

    def round_f32(self, x):
        x = _c64(x).copy()
        self.lib.orc_round_f32(x, x.size)
        return x

    def round_bf16(self, x):
        x = _c64(x).copy()
        self.lib.orc_round_bf16(x, x.size)
        return x

    def to_bf16_bits(self, x):
        x = _c64(x)
        out = np.empty(x.shape, np.uint16)
        self.lib.orc_to_bf16(x, x.size, out)
        return out


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref(_Base):
    """The compiled reference (oracle/_ref). Backend ids for time_backend():
    0 = reference (sequential), 1 = fused (pool), 2 = sigmoid fused (pool)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        vargs = [_dp, C.c_int, _dp, C.c_int, C.c_int, C.c_int, _ip, _dp]
        L.ref_verify_sequential.argtypes = vargs + [C.POINTER(_Out)]
        L.ref_verify_exact_logits.argtypes = vargs + [C.POINTER(_Out)]
        L.ref_verify_fused.argtypes = vargs + [C.c_int, C.c_uint, C.POINTER(_Out)]
        L.ref_verify_sigmoid_sequential.argtypes = vargs + [C.c_double, C.c_double, C.POINTER(_Out)]
        L.ref_verify_sigmoid_sequential_h.argtypes = vargs + [C.c_double, C.c_double, C.c_int, C.POINTER(_Out)]
        L.ref_verify_sigmoid_fused.argtypes = vargs + [C.c_double, C.c_double, C.c_int, C.c_uint, C.POINTER(_Out)]
        L.ref_make_bench_inputs.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _dp, _ip, _dp]
        L.ref_make_model_pair.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.ref_decode.argtypes = [_dp, _dp, C.c_int, _ip, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                 C.c_int, C.c_double, C.c_double, C.c_int, _ip, _ip, C.POINTER(C.c_int)]
        L.ref_time_backend.argtypes = [C.c_int] + vargs + [
            C.c_double, C.c_double, C.c_int, C.c_uint, C.c_int, C.c_int, _dp, C.POINTER(_Out)]

    def _run(self, fn, zp, zq, ids, u, *extra):
        zp, zq, ids, u, B, gamma, V = self._shape(zp, zq, ids, u)
        res = Result(B, gamma)
        out = res.c()
        rc = fn(zp, zp.shape[1], zq, B, gamma, V, ids, u, *extra, C.byref(out))
        if rc:
            raise ValueError("reference: " + self.lib.ref_last_error().decode())
        return res

    def verify_sequential(self, p, q, ids, u):
        return self._run(self.lib.ref_verify_sequential, p, q, ids, u)

    def verify_fused(self, p, q, ids, u, tile_width=1024, workers=2):
        return self._run(self.lib.ref_verify_fused, p, q, ids, u, tile_width, workers)

    def verify_exact(self, zp, zq, ids, u):
        return self._run(self.lib.ref_verify_exact_logits, zp, zq, ids, u)

    def verify_sigmoid(self, zp, zq, ids, u, alpha, beta):
        return self._run(self.lib.ref_verify_sigmoid_sequential, zp, zq, ids, u, alpha, beta)

    def verify_sigmoid_half(self, zp, zq, ids, u, alpha, beta):
        """verify_sigmoid_sequential with emulate_half = true (dist.cpp:64-69)."""
        return self._run(self.lib.ref_verify_sigmoid_sequential_h, zp, zq, ids, u, alpha, beta, 1)

    def verify_sigmoid_fused(self, zp, zq, ids, u, alpha, beta, tile_width=1024, workers=2):
        return self._run(self.lib.ref_verify_sigmoid_fused, zp, zq, ids, u, alpha, beta, tile_width, workers)

    def make_bench_inputs(self, seed, gamma, V):
        zp = np.empty((gamma + 1, V))
        zq = np.empty((gamma, V))
        ids = np.empty(gamma, np.int32)
        u = np.empty(gamma + 1)
        rc = self.lib.ref_make_bench_inputs(seed, gamma, V, zp, zq, ids, u)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return zp, zq, ids, u

    def time_backend(self, backend, zp, zq, ids, u, alpha=-1e3, beta=1e3, tile_width=1024,
                     workers=1, warmup=1, trials=3):
        zp, zq, ids, u, B, gamma, V = self._shape(zp, zq, ids, u)
        ns = np.zeros(trials)
        res = Result(B, gamma)
        out = res.c()
        rc = self.lib.ref_time_backend(backend, zp, zp.shape[1], zq, B, gamma, V, ids, u, alpha, beta,
                                       tile_width, workers, warmup, trials, ns, C.byref(out))
        if rc:
            raise ValueError("reference: " + self.lib.ref_last_error().decode())
        return ns, res

    def make_model_pair(self, seed, V, divergence, logit_scale=4.0):
        """toy_model.cpp:16-42: (target, draft) logit tables, V x V."""
        t = np.zeros((V, V))
        d = np.zeros((V, V))
        if self.lib.ref_make_model_pair(seed, V, divergence, logit_scale, t, d):
            raise ValueError("reference: " + self.lib.ref_last_error().decode())
        return t, d

    def decode(self, target, draft, prompt, max_len, gamma=5, min_gamma=1, max_gamma=64, seed=0,
               backend="reference", alpha=-1e3, beta=1e3, emulate_half=False):
        """decode.cpp:45-159 (Backend reference / fused / sigmoid) on the given tables."""
        V = target.shape[0]
        target = np.ascontiguousarray(target, np.float64)
        draft = np.ascontiguousarray(draft, np.float64)
        prompt = np.ascontiguousarray(prompt, np.int32)
        tokens = np.zeros(max_len, np.int32)
        hist = np.zeros(max_len, np.int32)
        steps = C.c_int(0)
        code = {"reference": 0, "fused": 1, "sigmoid": 2}[backend]
        if self.lib.ref_decode(target, draft, V, prompt, prompt.size, max_len, gamma, min_gamma, max_gamma, seed,
                               code, alpha, beta, int(emulate_half), tokens, hist, C.byref(steps)):
            raise ValueError("reference: " + self.lib.ref_last_error().decode())
        return tokens, hist[:steps.value]

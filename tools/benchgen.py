"""ctypes front end of tools/benchgen.c: the benchmark's synthetic inputs (the
reference's make_bench_inputs recipe per batch row, bench.cpp:46-74), rounded
to the storage type.  Harness code shared by both bench.py arms so they see
identical input bits; not part of the verification path."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "benchgen.c")
LIB = os.path.join(HERE, "libbenchgen.so")
DTYPES = {"f32": (0, np.float32), "bf16": (1, np.uint16), "f64": (2, np.float64)}
_lib = None


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", LIB, SRC, "-lm"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.bg_make_bench_batch.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p]
        L.bg_make_model_pair.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def make_bench_batch(seed, B, gamma, V, storage="f32", out=None, threads=None):
    """Rows b = make_bench_inputs(seed + b, gamma, V).  Returns (z_p, z_q, ids, u)
    as numpy arrays (bf16 as uint16 bit patterns), written into `out` if given
    (e.g. pinned buffers of the right shapes and dtypes)."""
    code, npdt = DTYPES[storage]
    if out is None:
        out = (np.empty((B, gamma + 1, V), npdt), np.empty((B, gamma, V), npdt), np.empty((B, gamma), np.int32),
               np.empty((B, gamma + 1), np.float64))
    zp, zq, ids, u = out
    assert zp.dtype == npdt and zq.dtype == npdt and ids.dtype == np.int32 and u.dtype == np.float64
    assert zp.shape == (B, gamma + 1, V) and zq.shape == (B, gamma, V)
    assert zp.flags.c_contiguous and zq.flags.c_contiguous and ids.flags.c_contiguous and u.flags.c_contiguous
    rc = lib().bg_make_bench_batch(seed, B, gamma, V, code, threads or os.cpu_count() or 1, zp.ctypes.data,
                                   zq.ctypes.data, ids.ctypes.data, u.ctypes.data)
    if rc:
        raise ValueError(f"bg_make_bench_batch: bad arguments B={B} gamma={gamma} V={V} storage={storage}")
    return zp, zq, ids, u


def widen(x, storage):
    """Stored logits -> float64 (what the reference consumes)."""
    if storage == "bf16":
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return x.astype(np.float64)


def make_model_pair(seed, V, divergence, logit_scale=4.0):
    """toy_model.cpp:16-42: the (target, draft) order-1 Markov logit tables,
    [V, V] float64 (the ablation's and the decode loop's inputs)."""
    t = np.empty((V, V), np.float64)
    d = np.empty((V, V), np.float64)
    if lib().bg_make_model_pair(seed, V, divergence, logit_scale, t.ctypes.data, d.ctypes.data):
        raise ValueError("make_model_pair: vocab_size must be >= 2 and divergence >= 0")
    return t, d

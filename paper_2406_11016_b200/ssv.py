"""ctypes binding of include/ssv/ssv.h (the C-ABI of libssv.so).

Device entry points take torch CUDA tensors (their data pointers are passed
straight to the stream-ordered C-ABI); host entry points take numpy arrays.
Errors mirror the reference: SSV_EINVAL -> ``SsvInvalidArgument`` (a
``ValueError``, the reference's std::invalid_argument), anything else ->
``SsvError`` (std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSV_LIB") or os.path.join(PKG_DIR, "libssv.so")  # SSV_LIB: experiment builds only
MAKEFILE = os.path.join(PKG_DIR, "csrc", "Makefile")

SSV_OK, SSV_ECUDA, SSV_EINVAL = 0, 1, 2
SSV_F32, SSV_BF16, SSV_F64 = 0, 1, 2
SSV_WANT_P, SSV_WANT_Q, SSV_WANT_RESIDUAL = 1, 2, 4
SSV_EMULATE_HALF = 8
# device status bits (ssv.h SSV_STATUS_*)
SSV_STATUS_NONFINITE, SSV_STATUS_TOKEN_RANGE, SSV_STATUS_UNIFORM_RANGE, SSV_STATUS_NEGATIVE = 1, 2, 4, 8


class SsvError(RuntimeError):
    pass


class SsvInvalidArgument(ValueError):
    pass


class Args(C.Structure):
    _fields_ = [
        ("B", C.c_int32), ("gamma", C.c_int32), ("V", C.c_int32), ("p_steps", C.c_int32),
        ("dtype", C.c_int32),
        ("z_p", C.c_void_p), ("z_q", C.c_void_p),
        ("draft_tokens", C.c_void_p), ("uniforms", C.c_void_p),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("flags", C.c_uint32),
    ]


class Out(C.Structure):
    _fields_ = [
        ("accepted_len", C.c_void_p), ("final_token", C.c_void_p), ("resample_used", C.c_void_p),
        ("tau", C.c_void_p), ("residual_denom", C.c_void_p),
        ("p", C.c_void_p), ("q", C.c_void_p), ("residual", C.c_void_p),
        ("status", C.c_void_p),
    ]


_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile libssv.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force and os.path.exists(LIB_PATH):
        os.remove(LIB_PATH)
    if shutil.which("make") is None:
        raise SsvError("make not found; cannot build libssv.so")
    subprocess.run(["make", "-s", "-f", MAKEFILE], check=True)
    return LIB_PATH


def load_library() -> C.CDLL:
    """Load libssv.so (building it first if it is missing). Raises if unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i32 = C.c_void_p, C.c_int32
        L.ssv_version.restype = C.c_char_p
        L.ssv_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.ssv_destroy.argtypes = [vp]
        L.ssv_destroy.restype = None
        L.ssv_set_stream.argtypes = [vp, vp]
        L.ssv_get_stream.argtypes = [vp]
        L.ssv_get_stream.restype = vp
        L.ssv_last_error.argtypes = [vp]
        L.ssv_last_error.restype = C.c_char_p
        L.ssv_last_launch_count.argtypes = [vp]
        L.ssv_set_path.argtypes = [vp, i32]
        L.ssv_last_plan.argtypes = [vp, C.POINTER(i32), i32]
        for name in ("exact", "sigmoid", "probs", "exact_host", "sigmoid_host", "probs_host"):
            f = getattr(L, "ssv_verify_" + name)
            f.argtypes = [vp, C.POINTER(Args), C.POINTER(Out)]
        L.ssv_host_alloc.argtypes = [C.c_size_t]
        L.ssv_host_alloc.restype = vp
        L.ssv_host_free.argtypes = [vp]
        L.ssv_host_free.restype = None
        L.ssv_sample_softmax.argtypes = [vp, i32, vp, i32, i32, vp, vp, vp]
        L.ssv_make_bench_inputs.argtypes = [vp, C.c_uint64, i32, i32, i32, i32, vp, vp, vp, vp]
        L.ssv_profile_enable.argtypes = [vp, C.c_int]
        L.ssv_profile_disable.argtypes = [vp]
        L.ssv_profile_reset.argtypes = [vp]
        L.ssv_profile_read.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(i32)]
        L.ssv_debug_trace.argtypes = [vp, C.c_int, vp, vp]
        _lib = L
        return L


# Every symbol include/ssv/ssv.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ssv_create", "ssv_destroy", "ssv_set_stream", "ssv_get_stream", "ssv_last_error",
    "ssv_last_launch_count", "ssv_version", "ssv_verify_exact", "ssv_verify_sigmoid",
    "ssv_verify_probs", "ssv_verify_exact_host", "ssv_verify_sigmoid_host", "ssv_verify_probs_host",
    "ssv_host_alloc", "ssv_host_free", "ssv_sample_softmax", "ssv_make_bench_inputs",
    "ssv_profile_enable", "ssv_profile_disable", "ssv_profile_reset", "ssv_profile_read",
    "ssv_debug_trace", "ssv_set_path", "ssv_last_plan",
)

KID_VERIFY, KID_MATERIALIZE, KID_GEN = 0, 2, 3


@dataclass
class VerifyResult:
    """VerificationResult (step.hpp:43-51) plus the optional grids."""

    accepted_len: object
    final_token: object
    resample_used: object
    tau: object
    residual_denom: object
    p: object = None
    q: object = None
    residual: object = None
    status: object = None

    def numpy(self) -> "VerifyResult":
        def cv(x):
            if x is None or isinstance(x, np.ndarray):
                return x
            return x.detach().cpu().numpy()

        return VerifyResult(*(cv(getattr(self, f)) for f in self.__dataclass_fields__))


_DT = {"float32": SSV_F32, "bfloat16": SSV_BF16, "float64": SSV_F64}


def _dtype_code(dt) -> int:
    name = str(dt).replace("torch.", "")
    if name == "uint16":  # bf16 bit patterns held in numpy
        return SSV_BF16
    if name not in _DT:
        raise SsvInvalidArgument(f"unsupported logit dtype {dt}")
    return _DT[name]


class Verifier:
    """One ssv_ctx (device + stream + scratch). Not shared across threads."""

    def __init__(self, device: int = 0, stream=None):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.ssv_create(device, C.byref(h))
        if rc != SSV_OK:
            raise SsvError(f"ssv_create(device={device}) failed with code {rc} (no CUDA device?)")
        self.ctx = h
        self.device = device
        self._own_stream = self.lib.ssv_get_stream(h)
        # Device entry points follow torch's current stream (so they order with
        # the torch ops that produce their inputs and read their outputs)
        # unless a stream is pinned with set_stream().
        self._follow_torch = stream is None
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.ssv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Pin a torch.cuda.Stream / raw cudaStream_t int; None = follow torch's current stream."""
        if stream is None:
            self._follow_torch = True
            return
        self._follow_torch = False
        handle = getattr(stream, "cuda_stream", stream)
        self.lib.ssv_set_stream(self.ctx, C.c_void_p(handle))

    def _bind_torch_stream(self) -> None:
        if self._follow_torch:
            import torch

            self.lib.ssv_set_stream(self.ctx, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def set_path(self, path: str) -> None:
        """Kernel selection (ssv_set_path): "auto" (default), "streaming", "cluster"
        or "cluster_ring" (the cluster kernel without its resident plan)."""
        code = {"auto": 0, "streaming": 1, "cluster": 2, "cluster_ring": 3, "slab": 4}[path]
        self._check(self.lib.ssv_set_path(self.ctx, code), "ssv_set_path")

    @property
    def stream_handle(self) -> int:
        return self.lib.ssv_get_stream(self.ctx) or 0

    @property
    def last_launch_count(self) -> int:
        return self.lib.ssv_last_launch_count(self.ctx)

    @property
    def last_plan(self) -> dict:
        """The plan the last verify call launched (ssv_last_plan)."""
        info = (C.c_int32 * 6)()
        self._check(self.lib.ssv_last_plan(self.ctx, info, 6), "ssv_last_plan")
        kind = {0: "streaming", 1: "cluster_resident", 2: "cluster_ring", 3: "slab", 4: "sigmoid_stream"}[info[0]]
        return {"kernel": kind, "cluster_size": info[1], "threads": info[2], "slots": info[3], "rows": info[4],
                "pieces": info[5]}

    def _check(self, rc: int, what: str):
        if rc == SSV_OK:
            return
        msg = self.lib.ssv_last_error(self.ctx).decode()
        if rc == SSV_EINVAL:
            raise SsvInvalidArgument(f"{what}: {msg}")
        raise SsvError(f"{what}: {msg}")

    # ---------------- kernel timing ----------------
    def profile_enable(self, capacity: int) -> None:
        self._check(self.lib.ssv_profile_enable(self.ctx, capacity), "ssv_profile_enable")

    def profile_disable(self) -> None:
        self.lib.ssv_profile_disable(self.ctx)

    def profile_reset(self) -> None:
        self.lib.ssv_profile_reset(self.ctx)

    def profile_read(self, kernel_id: int):
        """(total_ms, count) of the bracketed launches of one kernel id."""
        ms, n = C.c_double(), C.c_int32()
        self._check(self.lib.ssv_profile_read(self.ctx, kernel_id, C.byref(ms), C.byref(n)), "ssv_profile_read")
        return ms.value, n.value

    def trace_enable(self, capacity: int) -> None:
        self._check(self.lib.ssv_debug_trace(self.ctx, capacity, None, None), "ssv_debug_trace")

    def trace_read(self, capacity: int):
        buf = np.zeros(capacity, np.uint64)
        self._check(self.lib.ssv_debug_trace(self.ctx, capacity, buf.ctypes.data, None), "ssv_debug_trace")
        return buf

    # ---------------- device entry points (torch CUDA tensors) ----------------
    @staticmethod
    def _check_device_args(what, z_p, z_q, ids, u):
        """The C-ABI takes raw pointers with a row pitch of V: reject what it
        would misread (the reference's validate() rejects shape errors the
        same way, verify_reference.cpp:12-21)."""
        import torch

        for name, t in (("z_p", z_p), ("z_q", z_q), ("draft_tokens", ids), ("uniforms", u)):
            if not isinstance(t, torch.Tensor) or not t.is_cuda:
                raise SsvInvalidArgument(f"{what}: {name} must be a CUDA tensor")
            if not t.is_contiguous():
                raise SsvInvalidArgument(f"{what}: {name} must be contiguous (row pitch = V)")
            if t.device != z_q.device:
                raise SsvInvalidArgument(f"{what}: {name} is on {t.device}, z_q on {z_q.device}")
        if z_q.dim() != 3 or z_p.dim() != 3:
            raise SsvInvalidArgument(f"{what}: z_p and z_q must be [B, steps, V]")
        B, gamma, V = z_q.shape
        if z_p.shape[0] != B or z_p.shape[2] != V or z_p.shape[1] not in (gamma, gamma + 1):
            raise SsvInvalidArgument(f"{what}: StepInputs: p must be B x gamma(+1) x V matching q")
        if z_p.dtype != z_q.dtype:
            raise SsvInvalidArgument(f"{what}: z_p ({z_p.dtype}) and z_q ({z_q.dtype}) differ in dtype")
        if ids.dtype != torch.int32 or tuple(ids.shape) != (B, gamma):
            raise SsvInvalidArgument(f"{what}: draft_tokens must be int32 [B, gamma]")
        if u.dtype != torch.float64 or tuple(u.shape) != (B, gamma + 1):
            raise SsvInvalidArgument(f"{what}: uniforms must be float64 [B, gamma + 1]")

    def _device_call(self, fn, what, z_p, z_q, ids, u, alpha, beta, flags, out):
        import torch

        self._check_device_args(what, z_p, z_q, ids, u)
        self._bind_torch_stream()
        B, gamma, V = z_q.shape
        a = Args(B, gamma, V, z_p.shape[1], _dtype_code(z_q.dtype), z_p.data_ptr(), z_q.data_ptr(),
                 ids.data_ptr(), u.data_ptr(), alpha, beta, flags)
        dev = z_q.device
        if out is None:
            odt = torch.float64 if z_q.dtype == torch.float64 else torch.float32
            out = VerifyResult(
                accepted_len=torch.empty(B, dtype=torch.int32, device=dev),
                final_token=torch.empty(B, dtype=torch.int32, device=dev),
                resample_used=torch.empty(B, dtype=torch.uint8, device=dev),
                tau=torch.empty(B, gamma, dtype=torch.float64, device=dev),
                residual_denom=torch.empty(B, dtype=torch.float64, device=dev),
                p=torch.empty(z_p.shape, dtype=odt, device=dev) if flags & SSV_WANT_P else None,
                q=torch.empty(z_q.shape, dtype=odt, device=dev) if flags & SSV_WANT_Q else None,
                residual=torch.empty(z_q.shape, dtype=odt, device=dev) if flags & SSV_WANT_RESIDUAL else None,
                status=torch.zeros(1, dtype=torch.int32, device=dev),
            )
        o = Out(*(getattr(out, f).data_ptr() if getattr(out, f) is not None else None
                  for f in ("accepted_len", "final_token", "resample_used", "tau", "residual_denom",
                            "p", "q", "residual", "status")))
        self._check(fn(self.ctx, C.byref(a), C.byref(o)), what)
        return out

    def verify_exact(self, z_p, z_q, ids, u, flags=0, out=None):
        """Exact step on device tensors (logits in)."""
        return self._device_call(self.lib.ssv_verify_exact, "ssv_verify_exact", z_p, z_q, ids, u, 0.0, 0.0, flags, out)

    def verify_sigmoid(self, z_p, z_q, ids, u, alpha=-1e3, beta=1e3, flags=0, out=None, emulate_half=False):
        """Sigmoid-approximation step; emulate_half = the reference's binary16 emulation."""
        flags |= SSV_EMULATE_HALF if emulate_half else 0
        return self._device_call(self.lib.ssv_verify_sigmoid, "ssv_verify_sigmoid", z_p, z_q, ids, u, alpha, beta, flags, out)

    def verify_probs(self, p, q, ids, u, flags=0, out=None):
        return self._device_call(self.lib.ssv_verify_probs, "ssv_verify_probs", p, q, ids, u, 0.0, 0.0, flags, out)

    def sample_softmax(self, logits, uniforms, out=None):
        """Draft sampling: one token per row of a [rows, V] device tensor."""
        import torch

        rows, V = logits.shape[-2] if logits.dim() > 1 else 1, logits.shape[-1]
        rows = logits.numel() // V
        self._bind_torch_stream()
        if out is None:
            out = torch.empty(rows, dtype=torch.int32, device=logits.device)
        rc = self.lib.ssv_sample_softmax(self.ctx, _dtype_code(logits.dtype), logits.data_ptr(), rows, V,
                                         uniforms.data_ptr(), out.data_ptr(), None)
        self._check(rc, "ssv_sample_softmax")
        return out

    def make_bench_inputs(self, seed, B, gamma, V, dtype):
        """make_bench_inputs (bench.cpp:46-74) for B batch rows, on the device."""
        import torch

        dev = torch.device("cuda", self.device)
        self._bind_torch_stream()
        zp = torch.empty(B, gamma + 1, V, dtype=dtype, device=dev)
        zq = torch.empty(B, gamma, V, dtype=dtype, device=dev)
        ids = torch.empty(B, gamma, dtype=torch.int32, device=dev)
        u = torch.empty(B, gamma + 1, dtype=torch.float64, device=dev)
        rc = self.lib.ssv_make_bench_inputs(self.ctx, seed, B, gamma, V, _dtype_code(dtype), zp.data_ptr(),
                                            zq.data_ptr(), ids.data_ptr(), u.data_ptr())
        self._check(rc, "ssv_make_bench_inputs")
        return zp, zq, ids, u

    # ---------------- host entry points (numpy arrays) ----------------
    def _host_call(self, fn, what, z_p, z_q, ids, u, alpha, beta, flags, out, dtype=None):
        if self._follow_torch:
            self.lib.ssv_set_stream(self.ctx, C.c_void_p(self._own_stream))  # host entry points sync their own stream
        z_p = np.ascontiguousarray(z_p)
        z_q = np.ascontiguousarray(z_q)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        u = np.ascontiguousarray(u, dtype=np.float64)
        B, gamma, V = z_q.shape
        code = _dtype_code(dtype if dtype is not None else z_q.dtype)
        a = Args(B, gamma, V, z_p.shape[1], code, z_p.ctypes.data, z_q.ctypes.data, ids.ctypes.data,
                 u.ctypes.data, alpha, beta, flags)
        if out is None:
            odt = np.float64 if code == SSV_F64 else np.float32
            out = VerifyResult(
                accepted_len=np.empty(B, np.int32), final_token=np.empty(B, np.int32),
                resample_used=np.empty(B, np.uint8), tau=np.empty((B, gamma), np.float64),
                residual_denom=np.empty(B, np.float64),
                p=np.empty(z_p.shape, odt) if flags & SSV_WANT_P else None,
                q=np.empty(z_q.shape, odt) if flags & SSV_WANT_Q else None,
                residual=np.empty(z_q.shape, odt) if flags & SSV_WANT_RESIDUAL else None,
                status=np.zeros(1, np.uint32),
            )
        o = Out(*(getattr(out, f).ctypes.data if getattr(out, f) is not None else None
                  for f in ("accepted_len", "final_token", "resample_used", "tau", "residual_denom",
                            "p", "q", "residual", "status")))
        self._check(fn(self.ctx, C.byref(a), C.byref(o)), what)
        return out

    def prepare_host(self, variant, z_p, z_q, ids, u, out, alpha=-1e3, beta=1e3, flags=0, dtype=None):
        """A reusable host-entry step over fixed (pinned) host buffers: the
        serving-loop form of verify_*_host.  The returned callable re-runs the
        C-ABI host entry point on whatever the buffers hold when it is called
        (argument structs built once; the buffers must stay alive and keep
        their shapes).  Returns `out` after each call."""
        fn = {"exact": self.lib.ssv_verify_exact_host, "sigmoid": self.lib.ssv_verify_sigmoid_host,
              "probs": self.lib.ssv_verify_probs_host}[variant]
        for name, arr in (("z_p", z_p), ("z_q", z_q), ("ids", ids), ("u", u)):
            if not arr.flags.c_contiguous:
                raise ValueError(f"prepare_host: {name} must be C-contiguous")
        if ids.dtype != np.int32 or u.dtype != np.float64:
            raise ValueError("prepare_host: ids must be int32 and u float64")
        B, gamma, V = z_q.shape
        code = _dtype_code(dtype if dtype is not None else z_q.dtype)
        if variant != "sigmoid":
            alpha = beta = 0.0
        a = Args(B, gamma, V, z_p.shape[1], code, z_p.ctypes.data, z_q.ctypes.data, ids.ctypes.data,
                 u.ctypes.data, alpha, beta, flags)
        o = Out(*(getattr(out, f).ctypes.data if getattr(out, f) is not None else None
                  for f in ("accepted_len", "final_token", "resample_used", "tau", "residual_denom",
                            "p", "q", "residual", "status")))
        keep = (z_p, z_q, ids, u, out, a, o)
        ctx, pa, po, check, what = self.ctx, C.byref(a), C.byref(o), self._check, f"ssv_verify_{variant}_host"
        if self._follow_torch:
            self.lib.ssv_set_stream(self.ctx, C.c_void_p(self._own_stream))

        def step():
            rc = fn(ctx, pa, po)
            if rc:
                check(rc, what)
            return keep[4]
        return step

    def verify_exact_host(self, z_p, z_q, ids, u, flags=0, out=None, dtype=None):
        return self._host_call(self.lib.ssv_verify_exact_host, "ssv_verify_exact_host", z_p, z_q, ids, u, 0.0, 0.0,
                               flags, out, dtype)

    def verify_sigmoid_host(self, z_p, z_q, ids, u, alpha=-1e3, beta=1e3, flags=0, out=None, dtype=None,
                            emulate_half=False):
        flags |= SSV_EMULATE_HALF if emulate_half else 0
        return self._host_call(self.lib.ssv_verify_sigmoid_host, "ssv_verify_sigmoid_host", z_p, z_q, ids, u, alpha,
                               beta, flags, out, dtype)

    def verify_probs_host(self, p, q, ids, u, flags=0, out=None, dtype=None):
        return self._host_call(self.lib.ssv_verify_probs_host, "ssv_verify_probs_host", p, q, ids, u, 0.0, 0.0,
                               flags, out, dtype)

    # ---------------- pinned host memory ----------------
    def host_empty(self, shape, dtype) -> np.ndarray:
        """numpy array in pinned memory; the pages are released (ssv_host_free)
        when the last array viewing them is garbage-collected."""
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        ptr = self.lib.ssv_host_alloc(max(n, 1))
        if not ptr:
            raise SsvError("ssv_host_alloc failed")
        buf = (C.c_char * max(n, 1)).from_address(ptr)
        buf._owner = _PinnedPages(self.lib, ptr)  # lives as long as the buffer numpy views
        return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


class _PinnedPages:
    """Owner of one ssv_host_alloc block (freed with the last view of it)."""

    def __init__(self, lib, ptr):
        self.lib, self.ptr = lib, ptr

    def __del__(self):
        try:
            self.lib.ssv_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass

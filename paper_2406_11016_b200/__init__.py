"""B200-native speculative-sampling verification (arXiv 2406.11016).

The product is ``libssv.so`` (CUDA sm_100a kernels + C-ABI, include/ssv/ssv.h)
and the header-only C++ drop-in ``include/ssv/ssv.hpp``.  This module is a thin
ctypes front end over the same C-ABI, used by tests/ and bench.py.  There is no
CPU path: if the library is missing or no GPU is visible, calls raise.
"""
from __future__ import annotations

from .ssv import (  # noqa: F401
    SSV_BF16,
    SSV_F32,
    SSV_F64,
    SSV_WANT_P,
    SSV_WANT_Q,
    SSV_WANT_RESIDUAL,
    LIB_PATH,
    SsvError,
    SsvInvalidArgument,
    VerifyResult,
    Verifier,
    build,
    load_library,
)

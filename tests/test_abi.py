"""The C-ABI boundary on CPU: libssv.so builds for sm_100a, loads, exports every
symbol include/ssv/ssv.h declares, and rejects bad arguments without touching
a device.  No compute calls (there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ssv", "ssv.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssv_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_11016_b200 import load_library

    return load_library()


def test_library_is_sm100a(lib):
    from paper_2406_11016_b200 import LIB_PATH

    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 15
    from paper_2406_11016_b200.ssv import EXPORTS

    assert sorted(EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


def test_version(lib):
    assert b"sm_100a" in lib.ssv_version()


def test_invalid_arguments_without_device(lib):
    from paper_2406_11016_b200.ssv import SSV_EINVAL, Args, Out

    a, o = Args(), Out()
    assert lib.ssv_verify_exact(None, C.byref(a), C.byref(o)) == SSV_EINVAL
    assert lib.ssv_verify_sigmoid_host(None, C.byref(a), C.byref(o)) == SSV_EINVAL
    assert lib.ssv_create(0, None) == SSV_EINVAL
    assert lib.ssv_set_stream(None, None) == SSV_EINVAL
    assert lib.ssv_last_error(None) == b"null context"


def test_create_reports_missing_device(lib):
    import torch

    h = C.c_void_p()
    rc = lib.ssv_create(0, C.byref(h))
    if torch.cuda.is_available():
        assert rc == 0
        lib.ssv_destroy(h)
    else:
        assert rc == 1  # SSV_ECUDA: the product never falls back to the CPU


def test_cpp_wrapper_compiles():
    """include/ssv/ssv.hpp (the reference-typed C++ drop-in) compiles and links."""
    src = os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "wrapper_demo")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), src,
                        "-L", os.path.join(ROOT, "paper_2406_11016_b200"), "-lssv",
                        "-Wl,-rpath," + os.path.join(ROOT, "paper_2406_11016_b200"), "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_bridge_compiles_against_reference():
    """include/ssv/specsamp_bridge.hpp + tests/cpp/ref_backend.cpp compile
    against the reference's own headers and link against the reference built
    from its sources (INTEGRATION.md section 1 patch)."""
    import pytest

    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers absent (GPU box): the binary is prebuilt")
    r = subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile"),
                        os.path.join(ROOT, "oracle", "_ref", "ref_backend")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_backend"))

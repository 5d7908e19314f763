"""The C++ drop-in on the GPU.

* tests/cpp/wrapper_demo: include/ssv/ssv.hpp (the reference-typed wrapper)
  on the SPEC.md worked examples, verify_fused's residual written into q, the
  analytic MemoryTrace and plan_tiles, the sigmoid entry points' error rules.
* oracle/_ref/ref_backend: a translation unit of the REFERENCE (its headers,
  linked against the reference compiled from its sources) adding the
  cuda_exact / cuda_sigmoid backends through include/ssv/specsamp_bridge.hpp,
  checked against the reference's own reference / fused / sigmoid backends on
  make_bench_inputs batches (bench.cpp:46-74, 94-143)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, f"{os.path.basename(exe)} failed:\n{r.stdout}\n{r.stderr}"
    return r.stdout


def test_wrapper_demo():
    exe = os.path.join(ROOT, "tests", "cpp", "wrapper_demo")
    src = exe + ".cpp"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-L",
                            os.path.join(ROOT, "paper_2406_11016_b200"), "-lssv",
                            "-Wl,-rpath," + os.path.join(ROOT, "paper_2406_11016_b200"), "-o", exe],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    assert "wrapper_demo ok" in _run(exe)


def test_reference_side_backends():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_backend")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_backend not built (needs /root/reference at build time)")
    out = _run(exe)
    assert "0 failed checks" in out

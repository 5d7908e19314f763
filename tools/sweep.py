"""Device step time over a list of shapes (diagnostics; not the bench).

    python tools/sweep.py exact 64,8,32000,f32 128,8,32000,f32 ...
Prints one line per shape: us/step, algorithmic GB/s, fraction of the measured peak.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_11016_b200 import Verifier  # noqa: E402

variant = sys.argv[1]
v = Verifier(0)
peak, _ = bench.load_peaks()
for spec in sys.argv[2:]:
    B, g, V, dt = spec.split(",")
    key = f"s{spec}"
    bench.WORKLOADS[key] = (key, int(B), int(g), int(V), dt)
    wl = bench.Workload(v, key, 0, variant)
    r = bench.measure_device(v, wl, 200, 10, 1)
    step, _, A = wl.algorithmic_bytes(r["result"])
    us = r["ms_per_step"] * 1e3
    k = r["kernel_ms"].get("k_verify", 0) * 1e3
    print(f"{variant:8s} {spec:22s} step {us:8.1f} us  kernel {k:8.1f} us  {step / us / 1e3:7.0f} GB/s  frac {step / us / 1e3 / peak:.3f}  A={A}", flush=True)
    del wl

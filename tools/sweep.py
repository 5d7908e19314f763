"""Device step time over a list of shapes (diagnostics; not the bench).

    python tools/sweep.py [--path auto|streaming|cluster|cluster_ring] exact 64,8,32000,f32 ...
Prints one line per shape: us/step (graph-replayed, inputs rotated past L2),
algorithmic GB/s, fraction of the measured peak, the kernel plan.
Environment knobs (SSV_RUNA_FORCE, ...) need the experiment build (SSV_LIB).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_11016_b200 import Verifier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--path", default="auto")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--tag", default="")
ap.add_argument("variant")
ap.add_argument("shapes", nargs="+")
a = ap.parse_args()
v = Verifier(0)
v.set_path(a.path)
peak, _ = bench.load_peaks()
for spec in a.shapes:
    B, g, V, dt = spec.split(",")
    key = f"s{spec}"
    bench.WORKLOADS[key] = (key, int(B), int(g), int(V), dt)
    wl = bench.Workload(v, key, 0, 1, a.variant, host_gen=False)
    r = bench.measure_device(v, wl, a.steps, 5, 1)
    res = r["result"].numpy()
    kb, A = bench.algorithmic_bytes(a.variant, wl.B, wl.gamma, wl.V, wl.s, res.accepted_len)
    us = r["ms_per_step"] * 1e3
    plan = v.last_plan
    print(f"{a.tag} {a.variant:8s} {spec:22s} step {us:8.1f} us  {kb / us / 1e3:7.0f} GB/s  "
          f"frac {kb / us / 1e3 / peak:.3f}  A={A}  plan={plan}", flush=True)
    del wl

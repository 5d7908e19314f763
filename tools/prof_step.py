"""Runs a few verification steps of one workload (for ncu).  Not a benchmark."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11016_b200 import Verifier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=8)
ap.add_argument("--gamma", type=int, default=5)
ap.add_argument("--V", type=int, default=51865)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--variant", default="exact")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
v = Verifier(0)
v.set_path(a.path)
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[a.dtype]
zp, zq, ids, u = v.make_bench_inputs(1, a.B, a.gamma, a.V, dt)
for _ in range(a.iters):
    r = v.verify_exact(zp, zq, ids, u) if a.variant == "exact" else v.verify_sigmoid(zp, zq, ids, u)
torch.cuda.synchronize()
import json  # noqa: E402

import bench  # noqa: E402

kb, A = bench.algorithmic_bytes(a.variant, a.B, a.gamma, a.V, 4 if a.dtype == "f32" else 2, r.accepted_len.cpu().numpy())
print("PROF_STEP " + json.dumps({"algorithmic_bytes": kb, "accepted_all_rows": A, "plan": v.last_plan,
                                 "final_token": r.final_token.tolist()[:8]}))

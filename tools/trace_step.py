"""Phase timeline of one verify launch (globaltimer trace; diagnostics only)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_11016_b200 import Verifier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=8)
ap.add_argument("--gamma", type=int, default=5)
ap.add_argument("--V", type=int, default=51865)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--variant", default="exact")
a = ap.parse_args()
v = Verifier(0)
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[a.dtype]
zp, zq, ids, u = v.make_bench_inputs(1, a.B, a.gamma, a.V, dt)
run = (lambda: v.verify_exact(zp, zq, ids, u)) if a.variant == "exact" else (lambda: v.verify_sigmoid(zp, zq, ids, u))
for _ in range(3):
    run()
torch.cuda.synchronize()
cap = 4 * a.B + 2
v.trace_enable(cap)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.Stream()
v.set_stream(s)
with torch.cuda.stream(s):
    e0.record(s)
    r = run()
    e1.record(s)
s.synchronize()
t = v.trace_read(cap).astype(np.int64)
t0, t1 = t[4 * a.B], t[4 * a.B + 1]
print(f"event {e0.elapsed_time(e1) * 1e3:.1f} us; kernel span (CTA 0 start -> last CTA end) {(t1 - t0) / 1e3:.1f} us")
ph = t[: 4 * a.B].reshape(a.B, 4)
acc = r.accepted_len.cpu().numpy()
f = lambda x: f"{(x - t0) / 1e3:7.1f}" if x > 0 else "      -"
for b in range(min(a.B, 16)):
    print(f"b={b:3d} acc={acc[b]} D {f(ph[b, 0])} -> {f(ph[b, 1])}   L {f(ph[b, 2])} -> {f(ph[b, 3])}")
if a.B > 16:
    for b in range(16, a.B, max(1, a.B // 16)):
        print(f"b={b:3d} acc={acc[b]} D {f(ph[b, 0])} -> {f(ph[b, 1])}   L {f(ph[b, 2])} -> {f(ph[b, 3])}")

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
ap.add_argument("--path", default="auto")
a = ap.parse_args()
v = Verifier(0)
v.set_path(a.path)
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[a.dtype]
zp, zq, ids, u = v.make_bench_inputs(1, a.B, a.gamma, a.V, dt)
run = (lambda: v.verify_exact(zp, zq, ids, u)) if a.variant == "exact" else (lambda: v.verify_sigmoid(zp, zq, ids, u))
for _ in range(3):
    run()
torch.cuda.synchronize()
cap = 8 * a.B + 26 + 296 * 8
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
t0, t1 = t[8 * a.B], t[8 * a.B + 1]
print(f"event {e0.elapsed_time(e1) * 1e3:.1f} us; kernel span (CTA 0 start -> last CTA end) {(t1 - t0) / 1e3:.1f} us")
print("streaming: row acc | D claimed stats published | B0 claimed decided | L claimed ready end")
print("slab:      row acc | D start folded decided | slice0 stats-done residual-decided residual-done | L - start end")
print("cluster:   row acc | start stats sync1 | decided granules | sync2 gathered locate-end  (us from kernel start)")
ph = t[: 8 * a.B].reshape(a.B, 8)
acc = r.accepted_len.cpu().numpy()
f = lambda x: f"{(x - t0) / 1e3:6.1f}" if x > 0 else "     -"
rows = list(range(min(a.B, 16))) + (list(range(16, a.B, max(1, a.B // 16))) if a.B > 16 else [])
for b in rows:
    p = ph[b]
    print(f"b={b:3d} {acc[b]} | D {f(p[0])} {f(p[1])} {f(p[2])} | B {f(p[3])} {f(p[4])} | L {f(p[5])} {f(p[6])} {f(p[7])}")
lend = ph[:, 7].astype(np.int64)
if (lend > 0).any():
    worst = np.argsort(-lend)[:5]
    print("latest row ends (us):", ", ".join(f"b={w} {(lend[w] - t0) / 1e3:.1f}" for w in worst))
ex = t[8 * a.B + 2: 8 * a.B + 18]
if ex[0] > 0:
    print("row-0 fine stamps (us):", " ".join(f"{(x - t0) / 1e3:.1f}" if x > 0 else "-" for x in ex))
lo = t[8 * a.B + 18: 8 * a.B + 22]
if lo[3] > 0:
    f2 = lambda x: f"{(x - t0) / 1e3:.1f}" if x > 0 else "-"
    print(f"row-0 locate (us): enter {f2(lo[3])} level1-done {f2(lo[0])} level2-values {f2(lo[1])} end {f2(lo[2])}")
if t[8 * a.B + 22] > 0:
    print(f"row-0 locate level-1 on warp 0: {int(t[8 * a.B + 22])} cycles (sums done {int(t[8 * a.B + 23])}, "
          f"scans done {int(t[8 * a.B + 24])})")

if os.environ.get("SSV_SLAB_TRACE"):
    ct = t[8 * a.B + 26: 8 * a.B + 26 + 148 * 8].reshape(148, 8)
    print("per-CTA: stats-done steps 0..5 | residual-done steps 0..1 (us)")
    for c in list(range(0, 148, 8)) + [147]:
        print(f"cta {c:3d} " + " ".join(f(x) for x in ct[c]))
    for k in range(6):
        col = ct[:, k][ct[:, k] > 0]
        if len(col):
            print(f"step {k}: stats done min {(col.min() - t0) / 1e3:.1f} max {(col.max() - t0) / 1e3:.1f} us")

if os.environ.get("SSV_SIG_TRACE"):
    we = t[8 * a.B + 26: 8 * a.B + 26 + 296 * 8].astype(np.int64)
    ok = we > 0
    rel = (we[ok] - t0) / 1e3
    print(f"warp loop ends: n={ok.sum()} min {rel.min():.1f} median {np.median(rel):.1f} max {rel.max():.1f} us")
    worst = np.argsort(-np.where(ok, we, 0))[:8]
    print("latest warps:", ", ".join(f"gw={w} {(we[w] - t0) / 1e3:.1f}" for w in worst))

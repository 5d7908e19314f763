#!/usr/bin/env python
"""Reference-schema benchmark report: one row per grid
point in the reference's fixed CSV / JSONL schema (report.cpp:42-98,
report.hpp BenchRow), for the CUDA backends beside the reference's own
backends, so the two diff in one table.

    python tools/bench_report.py --vocab 32000 51865 --gamma 1 5 8 --seeds 1 2 \
        [--batch 1] [--format csv|jsonl] [--out report.csv] [--no-reference]

Per row: verify_ns = the kernel (CUDA events), total_ns = the step through the
host entry point (H2D + kernel + D2H; the reference's total includes its
softmax).  rel_improvement_pct = 100 * (1 - total / reference total) at the
same grid point (bench.cpp:192-198).  The trace columns hold the reference's
modelled counts (tile.cpp:25-31 rules, as include/ssv/ssv.hpp analytic_trace);
ncu-measured bytes are in profiles/.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

COLUMNS = ("backend,vocab,gamma,tile_n,workers,batch,seed,alpha,beta,trials,warmup,accept_rate,verify_ns_median,"
           "verify_ns_mean,verify_ns_stddev,total_ns_median,total_ns_mean,total_ns_stddev,rel_improvement_pct,"
           "hbm_elem_reads_p,hbm_elem_reads_q,hbm_elem_writes,kernel_invocations,peak_tile_bytes,"
           "peak_rss_bytes").split(",")


def trace(acc, rsu, rden, B, G, V, n):
    """tile.cpp:25-31 / verify_fused.cpp:88-92 counting rules."""
    K = (V + n - 1) // n
    writes = B * G * V + B * G * K + B * G + sum(V for b in range(B) if rsu[b] and rden[b] > 0.0)
    bit_ceil = 1 << (n - 1).bit_length()
    return {"hbm_elem_reads_p": B * G * V, "hbm_elem_reads_q": B * G * V, "hbm_elem_writes": writes,
            "kernel_invocations": B * G * K, "peak_tile_bytes": (2 * n + bit_ceil) * 8}


def stats(ns):
    return statistics.median(ns), statistics.mean(ns), statistics.pstdev(ns) if len(ns) > 1 else 0.0


def main():
    import numpy as np
    import torch

    from oracle.oracle import Oracle, Ref, ref_available
    from paper_2406_11016_b200 import Verifier

    ap = argparse.ArgumentParser()
    ap.add_argument("--vocab", type=int, nargs="+", default=[32000, 51865])
    ap.add_argument("--gamma", type=int, nargs="+", default=[1, 5, 8])
    ap.add_argument("--seeds", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--trials", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--tile", type=int, default=1024)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--alpha", type=float, default=-1e3)
    ap.add_argument("--beta", type=float, default=1e3)
    ap.add_argument("--format", choices=["csv", "jsonl"], default="csv")
    ap.add_argument("--out", default="-")
    ap.add_argument("--no-reference", action="store_true")
    a = ap.parse_args()

    o = Oracle()
    ref = Ref() if (ref_available() and not a.no_reference) else None
    v = Verifier(0)
    rows = []
    for V in a.vocab:
        n = min(a.tile, V)
        for G in a.gamma:
            for seed in a.seeds:
                B = a.batch
                zp, zq, ids, u = o.make_bench_batch(seed, B, G, V)
                zp, zq = o.round_f32(zp), o.round_f32(zq)
                base = {"vocab": V, "gamma": G, "tile_n": n, "batch": B, "seed": seed, "alpha": a.alpha,
                        "beta": a.beta, "trials": a.trials, "warmup": a.warmup}
                ref_total = None
                if ref is not None:
                    for code, name in ((0, "reference"), (1, "fused"), (2, "sigmoid")):
                        ns, res = ref.time_backend(code, zp, zq, ids, u, a.alpha, a.beta, n,
                                                   1 if code == 0 else a.workers, a.warmup, a.trials)
                        md, mn, sd = stats(list(ns))
                        if code == 0:
                            ref_total = md
                        rows.append({**base, "backend": name, "workers": 1 if code == 0 else a.workers,
                                     "accept_rate": float(np.mean(res.accepted_len)) / G,
                                     "verify_ns_median": md, "verify_ns_mean": mn, "verify_ns_stddev": sd,
                                     "total_ns_median": md, "total_ns_mean": mn, "total_ns_stddev": sd,
                                     "rel_improvement_pct": None if code == 0 else 100.0 * (1 - md / ref_total),
                                     **({k: 0 for k in COLUMNS[19:24]} if code == 0 else
                                        trace(res.accepted_len, res.resample_used, res.residual_denom, B, G, V, n))})
                hz = [v.host_empty(x.shape, dt) for x, dt in ((zp, np.float32), (zq, np.float32), (ids, np.int32),
                                                               (u, np.float64))]
                for h, x in zip(hz, (zp, zq, ids, u)):
                    h[...] = x
                dev = [torch.from_numpy(np.ascontiguousarray(h)).cuda() for h in hz]
                for variant in ("exact", "sigmoid"):
                    call_d = (lambda: v.verify_exact(*dev)) if variant == "exact" else (
                        lambda: v.verify_sigmoid(*dev, a.alpha, a.beta))
                    call_h = (lambda: v.verify_exact_host(*hz)) if variant == "exact" else (
                        lambda: v.verify_sigmoid_host(*hz, a.alpha, a.beta))
                    kns, tns = [], []
                    for t in range(a.warmup + a.trials):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        r = call_d()
                        e1.record()
                        torch.cuda.synchronize()
                        t0 = time.perf_counter_ns()
                        call_h()
                        t1 = time.perf_counter_ns()
                        if t >= a.warmup:
                            kns.append(e0.elapsed_time(e1) * 1e6)
                            tns.append(t1 - t0)
                    r = r.numpy()
                    kmd, kmn, ksd = stats(kns)
                    tmd, tmn, tsd = stats(tns)
                    rows.append({**base, "backend": f"cuda_{variant}", "workers": 1,
                                 "accept_rate": float(np.mean(r.accepted_len)) / G,
                                 "verify_ns_median": kmd, "verify_ns_mean": kmn, "verify_ns_stddev": ksd,
                                 "total_ns_median": tmd, "total_ns_mean": tmn, "total_ns_stddev": tsd,
                                 "rel_improvement_pct": 100.0 * (1 - tmd / ref_total) if ref_total else None,
                                 **trace(r.accepted_len, r.resample_used, r.residual_denom, B, G, V, n)})
    rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024
    out = sys.stdout if a.out == "-" else open(a.out, "w")
    if a.format == "csv":
        out.write(",".join(COLUMNS) + "\n")
    for row in rows:
        row["peak_rss_bytes"] = rss
        if a.format == "csv":
            out.write(",".join("" if row[c] is None else (f"{row[c]:.6g}" if isinstance(row[c], float) else str(row[c]))
                               for c in COLUMNS) + "\n")
        else:
            out.write(json.dumps({c: row[c] for c in COLUMNS}) + "\n")


if __name__ == "__main__":
    main()

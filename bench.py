#!/usr/bin/env python
"""Benchmark of the speculative-sampling verification step (arXiv 2406.11016).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4] [--variant exact|sigmoid] [--no-extra] [--no-cpu]

Workload (default, BASELINE.json config 4): C4 large-vocab verify, global batch
B=256, gamma=8, V=151936, fp32 logits, exact variant.  With N GPUs (torchrun,
one rank per GPU) the 256 batch rows are sharded into contiguous slabs, no
collective on the data path: STRONG scaling (the global batch is fixed).

Inputs: batch row b = the reference's make_bench_inputs(1 + b, gamma, V)
(bench.cpp:46-74) rounded to the storage type, generated on the host by
tools/benchgen.c (pinned bit-for-bit to the compiled reference by
tests/test_benchgen.py).  Both arms consume exactly these bits: the GPU arm
copies its slab to the device, the reference arm widens a row sample to double.

One "step" = one verification call over the rank's slab.  Metric
(BASELINE.json): verified drafted tokens/s = B * gamma / max-over-ranks(s/step).

* value     device-resident inputs (> 3x L2 across R rotating copies, so every
            step reads HBM), K steps replayed as one CUDA graph, CUDA events on
            the launching stream, barrier + synchronize on both sides.
* e2e       the same metric through the host C-ABI entry point
            (ssv_verify_*_host via Verifier.prepare_host): pinned host logits
            -> H2D -> kernel -> results in pinned memory, synchronized per step.
* roofline  the step is ONE kernel launch: achieved = algorithmic bytes per
            launch / graph-timed step time, vs MEASURED_PEAKS
            hbm_gbs; `traffic` = ncu DRAM bytes of the same launch
            (profiles/ncu_summary.json).
* cpu_baseline  the compiled reference (oracle/_ref) on a row sample of the
            same inputs, rank 0 at N=1.
--impl reference: the compiled reference (pooled materialize_softmax_into +
verify_fused, or verify_sigmoid_fused) on all host cores, same config dict.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified drafted tokens/sec and achieved HBM GB/s (% of roofline), 1/2/4/8 B200"
# key: (description, GLOBAL batch B, gamma, V, storage); B rows shard over the GPUs
WORKLOADS = {
    "c1": ("C1 exact verify B=1 gamma=5 V=32000 fp32 (reference CPU workload)", 1, 5, 32000, "f32"),
    "c2": ("C2 Whisper-shape ASR verify B=8 gamma=5 V=51865 fp32", 8, 5, 51865, "f32"),
    "c3": ("C3 Llama-2-shape verify B=64 gamma=8 V=32000 fp32", 64, 8, 32000, "f32"),
    "c3bf16": ("C3 Llama-2-shape verify B=64 gamma=8 V=32000 bf16", 64, 8, 32000, "bf16"),
    "c4": ("C4 large-vocab verify B=256 gamma=8 V=151936 fp32, batch-sharded over the GPUs", 256, 8, 151936, "f32"),
    "c4bf16": ("C4 large-vocab verify B=256 gamma=8 V=151936 bf16, batch-sharded over the GPUs", 256, 8, 151936,
               "bf16"),
    "c4shard": ("C4 one GPU's share on 8xB200: B=32 gamma=8 V=151936 fp32", 32, 8, 151936, "f32"),
}
SEED = 1
BYTES = {"f32": 4, "bf16": 2, "f64": 8}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(key):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        return json.load(open(path)).get(key)
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent clocks / throttle reasons via NVML during the timed region."""

    def __init__(self, device_index):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log("clock sampling unavailable:", e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
def config_dict(key, variant, world):
    """The config both arms print (identical keys and values)."""
    desc, B, gamma, V, storage = WORKLOADS[key]
    return {"workload": desc, "variant": variant, "global_batch": B, "gamma": gamma, "V": V, "storage": storage,
            "seed": SEED, "parallelism": f"batch rows sharded over {world} GPU(s) (strong scaling), no collective",
            "l2": "inputs larger than L2: the device arm rotates input copies totalling > 3x L2 (details.l2), "
                  "so every timed step reads its logits from HBM"}


def algorithmic_bytes(variant, B, gamma, V, s, accepted_len):
    """exact s*V*(2*gamma*B + A) + small terms; sigmoid
    s*V*(A + 2R) + gathered logits + small terms; A = rows accepting all gamma."""
    import numpy as np

    acc = np.asarray(accepted_len)
    A = int((acc == gamma).sum())
    R = B - A
    small = 4 * B * gamma + 8 * B * (gamma + 1) + (17 + 8 * gamma) * B
    if variant == "exact":
        return s * V * (2 * gamma * B + A) + small, A
    if variant == "exact_grids":  # + the p, q and residual grids written once (fp32)
        return s * V * (2 * gamma * B + A) + 4 * V * B * (3 * gamma + 1) + small, A
    return s * V * (A + 2 * R) + 2 * s * B * gamma + small, A


class Workload:
    """This rank's slab of the global batch: pinned host copy (tools/benchgen)
    + R device copies rotating so that every step reads HBM."""

    def __init__(self, v, key, rank, world, variant, host_gen=True, rotate=True):
        import numpy as np
        import torch

        from paper_2406_11016_b200.shard import shard_range

        desc, Bg, gamma, V, storage = WORKLOADS[key]
        self.key, self.desc, self.gamma, self.V, self.storage, self.variant = key, desc, gamma, V, storage, variant
        # Fewer batch rows than GPUs (C1, C2 at N = 8): independent replicas
        self.replicas = Bg < world
        self.lo, self.hi = (0, Bg) if self.replicas else shard_range(Bg, world, rank)
        self.B = self.hi - self.lo
        self.s = BYTES[storage]
        tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[storage]
        B = self.B
        self.host = None
        if host_gen:
            from tools import benchgen

            npdt = np.float32 if storage == "f32" else np.uint16
            h = (v.host_empty((B, gamma + 1, V), npdt), v.host_empty((B, gamma, V), npdt),
                 v.host_empty((B, gamma), np.int32), v.host_empty((B, gamma + 1), np.float64))
            t0 = time.perf_counter()
            benchgen.make_bench_batch(SEED + self.lo, B, gamma, V, storage, out=h)
            log(f"[bench] {key}: host inputs rows {self.lo}..{self.hi} in {time.perf_counter() - t0:.1f} s")
            self.host = h
            dev = torch.device("cuda", torch.cuda.current_device())
            zp = torch.from_numpy(h[0]).to(dev, non_blocking=True)
            zq = torch.from_numpy(h[1]).to(dev, non_blocking=True)
            if storage == "bf16":
                zp, zq = zp.view(torch.bfloat16), zq.view(torch.bfloat16)
            ids = torch.from_numpy(h[2]).to(dev)
            u = torch.from_numpy(h[3]).to(dev)
            self.inputs = "host generator tools/benchgen.c (= reference make_bench_inputs, rounded)"
        else:
            zp, zq, ids, u = v.make_bench_inputs(SEED + self.lo, B, gamma, V, tdt)
            self.inputs = "device generator ssv_make_bench_inputs"
        torch.cuda.synchronize()
        self.set_bytes = (zp.numel() + zq.numel()) * self.s
        self.l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
        R = max(2, math.ceil(3 * self.l2 / self.set_bytes)) if rotate else 1
        self.R = min(R, max(1, int(40e9 // self.set_bytes)))
        self.sets = [(zp, zq, ids, u)] + [(zp.clone(), zq.clone(), ids.clone(), u.clone()) for _ in range(self.R - 1)]
        self.outs = None

    def call(self, v, k, out=None):
        zp, zq, ids, u = self.sets[k % self.R]
        if self.variant == "exact":
            return v.verify_exact(zp, zq, ids, u, out=out)
        if self.variant == "exact_grids":  # the optional outputs: verify + the p / q / residual grids
            from paper_2406_11016_b200 import SSV_WANT_P, SSV_WANT_Q, SSV_WANT_RESIDUAL

            return v.verify_exact(zp, zq, ids, u, flags=SSV_WANT_P | SSV_WANT_Q | SSV_WANT_RESIDUAL, out=out)
        return v.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3, out=out)


def acceptance(v, wl):
    """North star: the sigmoid variant's acceptance-rate deviation from exact
    softmax on the same inputs and uniforms (mean accepted_len / gamma)."""
    import numpy as np
    import torch

    zp, zq, ids, u = wl.sets[0]
    ex = v.verify_exact(zp, zq, ids, u)
    sg = v.verify_sigmoid(zp, zq, ids, u, -1e3, 1e3)
    torch.cuda.synchronize()
    a = float(np.asarray(ex.accepted_len.cpu()).mean()) / wl.gamma
    b = float(np.asarray(sg.accepted_len.cpu()).mean()) / wl.gamma
    same = float((np.asarray(ex.final_token.cpu()) == np.asarray(sg.final_token.cpu())).mean())
    return {"exact": a, "sigmoid_bounds_1e3": b, "deviation": b - a, "same_final_token_frac": same}


def capture(v, wl, steps, stream):
    import torch

    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        v.set_stream(stream)
        with torch.cuda.graph(g, stream=stream):
            for k in range(steps):
                wl.call(v, k, out=wl.outs[k % wl.R])
    return g


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def measure_device(v, wl, K, W, world, sampler=None):
    """K steps replayed as one CUDA graph; returns ms per step, launches per
    step and the first set's result."""
    import torch

    stream = torch.cuda.Stream()
    v.set_stream(stream)
    wl.outs = [None] * wl.R
    with torch.cuda.stream(stream):
        for k in range(wl.R):  # sizes the context scratch; results per rotating set
            wl.outs[k] = wl.call(v, k)
    stream.synchronize()
    launches_per_step = v.last_launch_count
    st = int(wl.outs[0].status.item())
    if st:
        raise RuntimeError(f"device status {st} on the synthetic inputs")
    g_warm = capture(v, wl, max(W, 1), stream)
    g_time = capture(v, wl, K, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        g_warm.replay()
        stream.synchronize()
        _barrier(world)
        torch.cuda.synchronize()
        with (sampler if sampler is not None else _Null()):
            e0.record(stream)
            g_time.replay()
            e1.record(stream)
            stream.synchronize()
        _barrier(world)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    v.set_stream(None)  # back to following torch's current stream
    return {"ms_per_step": ms / K, "launches_per_step": launches_per_step, "result": wl.outs[0]}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def measure_e2e(v, wl, K, W, world):
    """Host entry point: pinned host inputs -> H2D -> step -> results in pinned
    memory, synchronized per step (the serving-loop form, Verifier.prepare_host)."""
    import numpy as np

    from paper_2406_11016_b200.ssv import VerifyResult

    hzp, hzq, hids, hu = wl.host
    B, g = wl.B, wl.gamma
    out = VerifyResult(v.host_empty((B,), np.int32), v.host_empty((B,), np.int32), v.host_empty((B,), np.uint8),
                       v.host_empty((B, g), np.float64), v.host_empty((B,), np.float64),
                       status=v.host_empty((1,), np.uint32))
    dt = "bfloat16" if wl.storage == "bf16" else None
    step = v.prepare_host(wl.variant, hzp, hzq, hids, hu, out, dtype=dt)
    for _ in range(W):
        step()
    _barrier(world)
    t0 = time.perf_counter()
    for _ in range(K):
        step()
    t = (time.perf_counter() - t0) / K
    if int(out.status[0]):
        raise RuntimeError(f"e2e: device status {int(out.status[0])}")
    h2d = hzp.nbytes + hzq.nbytes + hids.nbytes + hu.nbytes
    d2h = B * 4 + B * 4 + B + B * g * 8 + B * 8 + 4
    return t, h2d, d2h


# ----------------------------------------------------------------------------- CPU (reference) arm
def time_reference(zp, zq, ids, u, variant, budget_s, workers, warmup=1, trials=None):
    """The compiled reference (oracle/_ref) on a row sample of the given (double)
    inputs: pooled materialize_softmax_into + verify_fused (exact) or
    verify_sigmoid_fused (sigmoid) on WorkerPool(workers), tile 1024.  Rows
    are independent (verify_reference.cpp:87-109), so the sample's per-row
    rate is the workload's.  Returns (tokens/s, median s/step, rows, trials)."""
    import numpy as np

    from oracle.oracle import Ref

    ref = Ref()
    backend = 1 if variant == "exact" else 2
    gamma = zq.shape[1]
    B = zp.shape[0]
    ns, _ = ref.time_backend(backend, zp[:1], zq[:1], ids[:1], u[:1], workers=workers, warmup=0, trials=1)
    per_row = ns[0] * 1e-9
    if trials is None:
        rows = int(max(1, min(B, budget_s / 4 / max(per_row, 1e-9))))
        trials = int(max(3, min(30, budget_s / max(per_row * rows, 1e-9))))
    else:
        rows = int(max(1, min(B, budget_s / (trials + warmup) / max(per_row, 1e-9))))
    ns, _ = ref.time_backend(backend, zp[:rows], zq[:rows], ids[:rows], u[:rows], workers=workers, warmup=warmup,
                             trials=trials)
    t = float(np.median(ns)) * 1e-9
    return rows * gamma / t, t, rows, trials


def reference_sample(key, rows_max):
    """The first rows of the global batch, the same bits the GPU arm uses, widened to double."""
    from tools import benchgen

    desc, B, gamma, V, storage = WORKLOADS[key]
    n = min(B, rows_max)
    zp, zq, ids, u = benchgen.make_bench_batch(SEED, n, gamma, V, storage)
    return benchgen.widen(zp, storage), benchgen.widen(zq, storage), ids, u


def ref_name(variant, workers):
    return ((f"pooled materialize_softmax_into + verify_fused" if variant == "exact" else "verify_sigmoid_fused") +
            f" on WorkerPool({workers}), tile 1024, oracle/_ref (the reference compiled from its sources)")


def run_reference_arm(args):
    """bench.py --impl reference: the reference's own CPU path on this host,
    rank 0 only (other ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle.oracle import ref_available

    desc, B, gamma, V, storage = WORKLOADS[args.workload]
    cfg = config_dict(args.workload, args.variant, args.gpus)
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return
    workers = os.cpu_count() or 1
    budget = 150.0  # seconds for the whole --steps run
    zp, zq, ids, u = reference_sample(args.workload, 64)
    value, t, rows, trials = time_reference(zp, zq, ids, u, args.variant, budget, workers, warmup=args.warmup,
                                            trials=args.steps)
    sample = (f"{rows} of the {B} batch rows per step (rows independent: per-row rate = workload rate), "
              f"median of {trials} steps after {args.warmup} warm-up, {ref_name(args.variant, workers)}; "
              f"inputs: tools/benchgen.c rows = make_bench_inputs(1 + b) rounded to {storage}, widened to double")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (make_bench_inputs, bench.cpp:46-74)",
            "config": cfg, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": workers, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- config 5 sweep
SWEEP_GAMMAS = (1, 2, 4, 8, 16)
SWEEP_BATCHES = (1, 8, 64, 256, 1024)
SWEEP_VOCABS = (32000, 51865, 151936)
SWEEP_COLS = ["gamma", "B", "V", "dtype", "variant", "plan", "gpu_us_per_step", "gpu_tokens_per_s",
              "algorithmic_bytes", "gbs", "frac", "cpu_tokens_per_s", "cpu_rows", "cpu_cores", "gpu_over_cpu"]


def run_sweep(a):
    """--sweep: BASELINE.json config 5 on one GPU -- the gamma x B x V grid,
    GPU verified drafted tokens/s and roofline fraction (device-resident
    ssv_make_bench_inputs logits, inputs rotated past L2, graph-replayed steps,
    CUDA events) beside the reference's CPU path on the same recipe (cpu_baseline
    leg: oracle/_ref on a row subsample of tools/benchgen.c rows, all host cores,
    per-row rate; rows are independent, verify_reference.cpp:87-109).  The
    reference's own grid harness is bench.cpp:155-210.  One CSV row per point."""
    import csv

    import torch

    from oracle.oracle import ref_available
    from paper_2406_11016_b200 import Verifier
    from tools import benchgen

    v = Verifier(0)
    peak, _ = load_peaks()
    cores = os.cpu_count() or 1
    out = open(a.sweep_out, "w", newline="") if a.sweep_out else sys.stdout
    w = csv.DictWriter(out, fieldnames=SWEEP_COLS)
    w.writeheader()
    for V in map(int, a.sweep_vocabs.split(",")):
        for g in map(int, a.sweep_gammas.split(",")):
            for B in map(int, a.sweep_batches.split(",")):
                key = f"c5-{g}-{B}-{V}"
                WORKLOADS[key] = (key, B, g, V, a.sweep_dtype)
                wl = Workload(v, key, 0, 1, a.variant, host_gen=False)
                K = 20 if wl.set_bytes > 2e9 else 100
                m = measure_device(v, wl, K, 5, 1)
                res = m["result"].numpy()
                kb, _ = algorithmic_bytes(a.variant, B, g, V, wl.s, res.accepted_len)
                us = m["ms_per_step"] * 1e3
                plan = v.last_plan["kernel"]
                del wl
                torch.cuda.empty_cache()
                row = {"gamma": g, "B": B, "V": V, "dtype": a.sweep_dtype, "variant": a.variant, "plan": plan,
                       "gpu_us_per_step": round(us, 2), "gpu_tokens_per_s": round(B * g / (us * 1e-6)),
                       "algorithmic_bytes": kb, "gbs": round(kb / us / 1e3, 1), "frac": round(kb / us / 1e3 / peak, 3)}
                if ref_available():
                    rows = max(1, min(B, 4))
                    zp, zq, ids, u = benchgen.make_bench_batch(1, rows, g, V, a.sweep_dtype)
                    val, _, r_used, _ = time_reference(benchgen.widen(zp, a.sweep_dtype),
                                                       benchgen.widen(zq, a.sweep_dtype), ids, u, a.variant,
                                                       a.sweep_cpu_budget, cores)
                    row.update(cpu_tokens_per_s=round(val), cpu_rows=r_used, cpu_cores=cores,
                               gpu_over_cpu=round(row["gpu_tokens_per_s"] / val, 1))
                w.writerow(row)
                out.flush()
    if a.sweep_out:
        out.close()


# ----------------------------------------------------------------------------- main
EXTRAS = (("c4", "sigmoid"), ("c4bf16", "exact"), ("c4shard", "exact"), ("c3", "exact"), ("c3bf16", "exact"),
          ("c3", "sigmoid"), ("c2", "exact"), ("c2", "sigmoid"), ("c1", "exact"), ("c1", "sigmoid"),
          ("c2", "exact_grids"), ("c4shard", "exact_grids"))


def extra_line(v, key, variant, peak):
    import torch

    w2 = Workload(v, key, 0, 1, variant, host_gen=False)
    K = 50 if w2.B * w2.V > 1e7 else 200
    m2 = measure_device(v, w2, K, 5, 1)
    r = m2["result"].numpy()
    kb, A2 = algorithmic_bytes(variant, w2.B, w2.gamma, w2.V, w2.s, r.accepted_len)
    ms = m2["ms_per_step"]
    d = {"tokens_per_s": w2.B * w2.gamma / (ms * 1e-3), "ms_per_step": ms, "gbs": kb / (ms * 1e-3) / 1e9,
         "frac": kb / (ms * 1e-3) / 1e9 / peak, "algorithmic_bytes": kb, "accepted_all_rows": A2, "B": w2.B,
         "launches_per_step": m2["launches_per_step"], "inputs": w2.inputs}
    del w2
    torch.cuda.empty_cache()
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="exact", choices=["exact", "sigmoid"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="BASELINE config 5 grid on one GPU (CSV), then exit")
    ap.add_argument("--sweep-out", default="")
    ap.add_argument("--sweep-dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--sweep-cpu-budget", type=float, default=1.0, help="reference CPU seconds per point")
    ap.add_argument("--sweep-gammas", default=",".join(map(str, SWEEP_GAMMAS)))
    ap.add_argument("--sweep-batches", default=",".join(map(str, SWEEP_BATCHES)))
    ap.add_argument("--sweep-vocabs", default=",".join(map(str, SWEEP_VOCABS)))
    args = ap.parse_args()
    if args.sweep:
        return run_sweep(args)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # One rank per GPU (NCCL carries only the barrier and the max-over-ranks
    # time).  With fewer GPUs than ranks (a one-GPU box exercising the N > 1
    # path) the ranks share devices round-robin and the host-side plumbing runs
    # on gloo: that run checks the sharded flow, it is not a scaling number.
    ndev = torch.cuda.device_count()
    dev_index = local % max(1, ndev)
    shared = world > ndev
    torch.cuda.set_device(dev_index)
    backend = "gloo" if shared else "nccl"
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    from paper_2406_11016_b200 import Verifier
    from paper_2406_11016_b200.shard import allmax as _allmax

    def allmax(x):
        return _allmax(x, device="cpu" if shared else "cuda")

    v = Verifier(dev_index)
    peak, peak_src = load_peaks()
    desc, Bg, gamma, V, storage = WORKLOADS[args.workload]
    wl = Workload(v, args.workload, rank, world, args.variant)
    sampler = ClockSampler(dev_index)
    m = measure_device(v, wl, args.steps, args.warmup, world, sampler)
    res = m["result"].numpy()
    k_bytes, A = algorithmic_bytes(args.variant, wl.B, gamma, V, wl.s, res.accepted_len)
    ms = allmax(m["ms_per_step"])
    k_ms_local = m["ms_per_step"]
    tokens = (world if wl.replicas else 1) * Bg * gamma
    e2e = None
    if not args.no_e2e:
        ke = max(3, min(args.steps, 20))
        e2e_t, h2d, d2h = measure_e2e(v, wl, ke, 2, world)
        e2e_t = allmax(e2e_t)
        e2e = {"value": tokens / e2e_t, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_t * 1e3, "steps": ke,
               "path": f"ssv_verify_{args.variant}_host via Verifier.prepare_host (C-ABI host entry on pinned host "
                       "buffers: H2D of the step's inputs + verify; the kernel writes the small results into pinned "
                       "memory; synchronized per step), per-rank bytes"}
    achieved = k_bytes / (k_ms_local * 1e-3) / 1e9
    traffic = load_traffic(f"{args.workload}-{args.variant}") if world == 1 else None
    line = {
        "metric": METRIC,
        "value": tokens / (ms * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak" if wl.replicas else "strong",
        "vs_baseline": None,
        "dtype": storage,
        "data": "synthetic logits by the reference bench recipe (bench.cpp:46-74), global batch row b seeded 1+b",
        "config": config_dict(args.workload, args.variant, world),
        "details": {
            "rows_this_rank": [wl.lo, wl.hi], "inputs": wl.inputs,
            "l2": f"inputs rotate over {wl.R} copies ({wl.R * wl.set_bytes / 1e6:.0f} MB > 3x L2 "
                  f"{wl.l2 / 1e6:.0f} MB): every step reads HBM",
            "timing": "K steps replayed as one CUDA graph, CUDA events on the launching stream, max over ranks",
            "process_group": backend if world > 1 else None,
            "devices": (f"{world} ranks share {ndev} GPU(s): a path check of the sharded flow, not a scaling "
                        "measurement") if shared else f"one GPU per rank ({world})",
        },
        "gpu_launches": args.steps * m["launches_per_step"],
        "accepted_all_rows": A,
        "acceptance_rate": acceptance(v, wl),
        "roofline": {
            "bound": "hbm", "kernel": "ssv verify kernel (one launch per step)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
            "algorithmic_bytes_per_launch": k_bytes, "kernel_ms": k_ms_local,
            "kernel_ms_source": "graph-timed step (the step is one launch; PDL overlaps consecutive launches)",
            "ncu_kernel_ms": (traffic.get("duration_ns") / 1e6 if traffic and traffic.get("duration_ns") else None),
            "peak_source": peak_src,
        },
        "clocks": sampler.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle.oracle import ref_available

            if ref_available():
                zp = wl.host[0][:16]
                zq = wl.host[1][:16]
                from tools import benchgen

                val, t, rows, trials = time_reference(benchgen.widen(zp, storage), benchgen.widen(zq, storage),
                                                      wl.host[2][:16], wl.host[3][:16], args.variant, 12.0,
                                                      os.cpu_count() or 1)
                line["cpu_baseline"] = {
                    "value": val, "unit": "tokens/s", "cores": os.cpu_count() or 1, "kind": "reference",
                    "sample": f"{rows} of {Bg} batch rows (the same input bits), median of {trials} steps, "
                              + ref_name(args.variant, os.cpu_count() or 1)}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0 and world == 1 and not args.no_extra:
        extra = {}
        for key, variant in EXTRAS:
            if key == args.workload and variant == args.variant:
                continue
            try:
                extra[f"{key}-{variant}"] = extra_line(v, key, variant, peak)
            except Exception as e:
                extra[f"{key}-{variant}"] = {"error": str(e)}
        line["extra"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

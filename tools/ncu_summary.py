"""Summarise ncu --set full reports (one kernel launch each) into a markdown
table plus profiles/ncu_summary.json (the per-launch DRAM traffic bench.py
reports as roofline.traffic).

    python tools/ncu_summary.py OUT.md SUMMARY.json name=report.ncu-rep [...]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}
UNIT = {"dram_read": 1.0, "dram_write": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, n in enumerate(hdr):
        if n in METRICS or n.startswith("smsp__pcsamp_warps_issue_stalled_"):
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                  "msecond": 1e6}.get(u, 1.0)  # bytes, ns
            d[METRICS.get(n, n)] = v
    return d


def main():
    md, js = sys.argv[1], sys.argv[2]
    table = []
    summary = json.load(open(js)) if os.path.exists(js) else {}
    for arg in sys.argv[3:]:
        name, rep = arg.split("=", 1)
        d = raw(rep)
        stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v) for k, v in d.items()
                         if k.startswith("smsp__pcsamp") and not k.endswith("_not_issued")), key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in stalls[:4])
        traffic = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
        t_ns = d.get("duration", 0.0)
        summary[name] = {"dram_bytes_per_launch": traffic, "duration_ns": t_ns,
                         "dram_gbs": traffic / t_ns if t_ns else None, **{k: d.get(k) for k in
                         ("dram_pct", "issue_pct", "occupancy_pct", "l2_hit_pct", "warp_inst", "regs", "grid")},
                         "top_stalls": top, "report": os.path.basename(rep)}
        table.append((name, summary[name]))
    with open(js, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    with open(md, "w") as f:
        f.write("| workload | duration | DRAM bytes | DRAM GB/s | mem-SOL % | issue % | occupancy % | L2 hit % | warp inst | top stall reasons |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for name, s in table:
            f.write(f"| {name} | {s['duration_ns'] / 1e3:.1f} us | {s['dram_bytes_per_launch'] / 1e6:.1f} MB | "
                    f"{(s['dram_gbs'] or 0):.0f} | {s['dram_pct'] or 0:.1f} | {s['issue_pct'] or 0:.1f} | "
                    f"{s['occupancy_pct'] or 0:.1f} | {s['l2_hit_pct'] or 0:.1f} | {s['warp_inst'] or 0:.3g} | {s['top_stalls']} |\n")
    print(open(md).read())


if __name__ == "__main__":
    main()

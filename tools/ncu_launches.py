"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per
launch) per kernel.  Usage: ncu_launches.py LAUNCHES.csv [--json]"""
import csv
import io
import json
import statistics
import sys
from collections import defaultdict


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(dict)
    for r in rows:
        per[(int(r["ID"]), r["Kernel Name"], r["Grid Size"], r["Block Size"])][r["Metric Name"]] = float(
            r["Metric Value"].replace(",", ""))
    return per


def summarise(per):
    by = defaultdict(list)
    for (i, name, grid, block), m in sorted(per.items()):
        by[(name, grid, block)].append(m)
    out = []
    for (name, grid, block), ms in by.items():
        t = [m.get("gpu__time_duration.sum", 0.0) for m in ms]
        rd = [m.get("dram__bytes_read.sum", 0.0) for m in ms]
        wr = [m.get("dram__bytes_write.sum", 0.0) for m in ms]
        out.append({"kernel": name, "grid": grid, "block": block, "launches": len(ms),
                    "time_ns_median": statistics.median(t), "time_ns_min": min(t), "time_ns_max": max(t),
                    "dram_read_median": statistics.median(rd), "dram_write_median": statistics.median(wr),
                    "dram_gbs_median": (statistics.median(rd) + statistics.median(wr)) / statistics.median(t)})
    tot = sum(o["time_ns_median"] * o["launches"] for o in out) or 1.0
    for o in out:
        o["share"] = o["time_ns_median"] * o["launches"] / tot
    return out


if __name__ == "__main__":
    s = summarise(load(sys.argv[1]))
    if "--json" in sys.argv:
        print(json.dumps(s, indent=1))
    else:
        for o in s:
            print(f"{o['kernel'][:60]:60s} grid {o['grid']:>12s} n={o['launches']:4d} "
                  f"t_med {o['time_ns_median'] / 1e3:8.2f} us  read {o['dram_read_median'] / 1e6:9.2f} MB  "
                  f"write {o['dram_write_median'] / 1e6:7.2f} MB  {o['dram_gbs_median']:7.1f} GB/s  "
                  f"share {o['share'] * 100:5.1f}%")

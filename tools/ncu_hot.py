"""Top stall-sampled SASS instructions of one kernel in an ncu report (with the
CUDA source line when -lineinfo is present).  Usage: ncu_hot.py REP REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + rx,
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"#"') or 'Warp Stall Sampling' in l)
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
src_i = hdr.index("Source")
data = []
cur_src = ""
for r in rows[1:]:
    if len(r) <= si:
        continue
    try:
        s = float(r[si] or 0)
    except ValueError:
        continue
    data.append((s, r[0], r[src_i].strip()[:90]))
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot:.0f}")
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0] / tot * 100:5.1f}%  {d[1]}  {d[2]}")

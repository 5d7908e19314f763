"""Stall samples aggregated per CUDA source line (needs -lineinfo).
Usage: ncu_lines.py REP REGEX [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + rx,
                      "--print-source", "sass,cuda", "--print-details", "all"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if 'Warp Stall Sampling' in l)
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.Counter()
cur = "?"
for r in rows[1:]:
    if len(r) <= si:
        continue
    src = r[1].strip()
    try:
        s = float(r[si] or 0)
    except ValueError:
        continue
    if r[0] and not r[0].startswith("0x"):
        cur = f"L{r[0]}: {src[:80]}"
        continue
    agg[cur] += s
tot = sum(agg.values()) or 1
for k, v in agg.most_common(n):
    print(f"{v / tot * 100:5.1f}%  {k}")

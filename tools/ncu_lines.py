"""Per-CUDA-source-line instruction counts and stall samples from an ncu
report (needs -lineinfo + --import-source).  Usage: ncu_lines.py REP [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
inst = defaultdict(float)
stall = defaultdict(float)
i = 0
cur = None
while i < len(lines):
    l = lines[i]
    if l.startswith('"File Path"'):
        cur = l.split(",", 1)[1].strip('"').split("/")[-1]
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        ii, si, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), 0
        j = i + 1
        while j < len(lines) and not lines[j].startswith('"File Path"'):
            r = next(csv.reader([lines[j]]))
            if len(r) > ii and r[0].isdigit():
                key = f"{cur}:{r[0]} {r[1].strip()[:70]}"
                try:
                    inst[key] += float(r[ii] or 0)
                    stall[key] += float(r[si] or 0)
                except ValueError:
                    pass
            j += 1
        i = j
        continue
    i += 1
ti = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print(f"total warp instructions {ti:.3g}, stall samples {ts:.3g}")
print("-- by instructions")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / ti * 100:5.1f}% inst {stall[k] / ts * 100:5.1f}% stall  {k}")
print("-- by stall samples")
for k, v in sorted(stall.items(), key=lambda x: -x[1])[:n]:
    print(f"{inst[k] / ti * 100:5.1f}% inst {v / ts * 100:5.1f}% stall  {k}")

"""Top stall-sampled SASS instructions (with neighbours) of a kernel in an ncu report.
Usage: ncu_sass.py REP REGEX [N]"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + rx,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
ins = [(r[0], r[1].strip(), float(r[si] or 0)) for r in rows[1:] if len(r) > si]
tot = sum(x[2] for x in ins) or 1
order = sorted(range(len(ins)), key=lambda i: -ins[i][2])[:n]
for i in sorted(order):
    a, s, v = ins[i]
    print(f"{v / tot * 100:5.1f}% {i:5d} {s[:90]}")

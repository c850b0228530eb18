#!/usr/bin/env python3
"""Per-opcode executed-instruction histogram (and stall samples) of one kernel in an ncu report:
    python tools/sass_hist.py report.ncu-rep <kernel regex> [top]"""
import csv
import collections
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE, iSm = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
smp = collections.Counter()
tot = 0
lines = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].strip().isdigit():
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    opb = op.split(".")[0]
    n = int(r[iE])
    ops[opb] += n
    smp[opb] += int(r[iSm] or 0)
    tot += n
    lines.append((n, int(r[iSm] or 0), src))
print(f"total warp instructions {tot:,}")
for op, n in ops.most_common(top):
    print(f"{op:12s} {n:14,d} {100*n/tot:5.1f}%  stall-samples {smp[op]}")
print("\nhottest lines by samples:")
for n, s, src in sorted(lines, key=lambda t: -t[1])[:25]:
    print(f"{s:7d} {n:12,d}  {src}")

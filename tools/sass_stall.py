#!/usr/bin/env python3
"""Lines of one kernel in an ncu report ranked by one stall reason's samples, with context:
    python tools/sass_stall.py report.ncu-rep <kernel regex> <stall column, e.g. stall_long_sb> [top]"""
import csv
import io
import subprocess
import sys

rep, kre, col = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE, iC = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(col)
body = [r for r in rows[2:] if len(r) > iC]
order = sorted(range(len(body)), key=lambda i: -int(body[i][iC] or 0))[:top]
for i in order:
    print(f"--- {body[i][iC]} samples")
    for j in range(max(0, i - 3), min(len(body), i + 2)):
        mark = ">>" if j == i else "  "
        print(f"{mark} {body[j][iE]:>10} {body[j][iS].strip()}")

#!/usr/bin/env python3
"""Markdown summary of tools/ncu_export.sh captures (details + SASS source CSV pages):

    python tools/ncu_csv_summary.py OUT.md NAME=gpurun_out/f_bwd_dyn [NAME=prefix ...]

Per kernel: the Speed-of-Light / launch / occupancy metrics, the warp-stall samples by reason
over the whole kernel, and the instructions holding the most stall samples (with their
dominant reason) -- where a latency-bound kernel loses its cycles."""
import collections
import csv
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L2 Hit Rate", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Occupancy", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block"]
STALLS = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_math", "stall_wait",
          "stall_mio", "stall_lg", "stall_branch_resolving", "stall_dispatch", "stall_no_inst",
          "stall_membar", "stall_drain", "stall_sleep", "stall_selected", "stall_not_selected"]

out = [f"# ncu --set full (final round-2 build): {', '.join(a.split('=')[0] for a in sys.argv[2:])}",
       "", "Captured with `tools/ncu_export.sh` (`ncu --set full --clock-control none "
       "--import-source on`, one launch after warm-up; cold-cache serialised replay: compare "
       "shares, not absolute speed).", ""]
for arg in sys.argv[2:]:
    name, pre = arg.split("=")
    rows = list(csv.reader(open(pre + "_details.csv")))
    h = {k: i for i, k in enumerate(rows[0])}
    kname = rows[1][h["Kernel Name"]]
    seen = {}
    for r in rows[1:]:
        if len(r) > h["Metric Value"] and r[h["Metric Name"]] in KEYS and r[h["Metric Name"]] not in seen:
            seen[r[h["Metric Name"]]] = f"{r[h['Metric Value']]} {r[h['Metric Unit']]}".strip()
    out += [f"## {name}: `{kname}`", "", "| metric | value |", "|---|---|"]
    out += [f"| {k} | {seen[k]} |" for k in KEYS if k in seen]
    s = list(csv.reader(open(pre + "_sass.csv")))
    sh = {k: i for i, k in enumerate(s[1])}
    data = s[2:]
    tot = {c: sum(int(r[sh[c]] or 0) for r in data) for c in STALLS if c in sh}
    allsamp = sum(tot.values()) or 1
    out += ["", "Warp-state samples by reason (share of all samples): " + ", ".join(
        f"{c[6:]} {100 * v / allsamp:.1f} %" for c, v in sorted(tot.items(), key=lambda t: -t[1]) if v)]
    samp = sh["Warp Stall Sampling (All Samples)"]
    top = sorted(data, key=lambda r: -int(r[samp] or 0))[:8]
    out += ["", "| samples | share | executed | instruction | main reason |", "|---|---|---|---|---|"]
    for r in top:
        reasons = {c: int(r[sh[c]] or 0) for c in STALLS if c in sh}
        main = max(reasons, key=reasons.get)
        out.append(f"| {r[samp]} | {100 * int(r[samp]) / allsamp:.1f} % | {r[sh['Instructions Executed']]} | "
                   f"`{r[sh['Source']].strip()[:60]}` | {main[6:]} |")
    out.append("")
open(sys.argv[1], "w").write("\n".join(out) + "\n")
print("\n".join(out))

#!/usr/bin/env python3
"""Summarise the multi-sample (bucket) ncu runs of tools/gpu_r2p.sh into a markdown file:
per bucket the launch list of this library's kernels (duration, DRAM bytes, GB/s of the second
fwd+bwd repetition), then the key `--set full` metrics of the captured kernels.

    python tools/ncu_buckets_summary.py gpurun_out/r2p profiles/r2_ncu_buckets.md
"""

from __future__ import annotations

import collections
import csv
import sys
from pathlib import Path

OURS = ("adaln_", "gate_residual", "qk_rms")
KEYS = [("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
        ("Memory Workload Analysis", "Memory Throughput"), ("Memory Workload Analysis", "L2 Hit Rate"),
        ("Compute Workload Analysis", "Issue Slots Busy"), ("Compute Workload Analysis", "Executed Ipc Active"),
        ("Launch Statistics", "Registers Per Thread"), ("Launch Statistics", "Grid Size"),
        ("Launch Statistics", "Block Size"), ("Occupancy", "Achieved Occupancy"),
        ("GPU Speed Of Light Throughput", "SM Frequency")]


def launches(path: Path):
    rows = [r for r in csv.reader(l for l in path.open() if l.startswith('"'))]
    h = rows[0]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        if not any(o in r[ki] for o in OURS):
            continue
        per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("void ", "")})[r[ni]] = float(
            r[vi].replace(",", ""))
    return list(per.values())


def main():
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    out = ["# Round 2: ncu evidence for multi-sample launches (the sampler's buckets)", "",
           "`tools/gpu_r2p.sh` on one B200 (`ncu --clock-control none`; launch lists with "
           "`gpu__time_duration.sum`, `dram__bytes_read.sum`, `dram__bytes_write.sum`; per-launch "
           "times are cold-cache and serialised, so shares, not absolutes, compare with the "
           "device-timestamp numbers in DESIGN §3.8). D = 5 120 bf16, per-sample modulation; "
           "rows = the second of two fwd+bwd repetitions.", ""]
    for f in sorted(src.glob("launches_*.csv")):
        ls = launches(f)
        if not ls:
            continue
        half = ls[len(ls) // 2:]
        out += [f"## {f.stem.replace('launches_', '')}", "",
                "| kernel | time µs | DRAM read MB | DRAM write MB | GB/s |", "|---|---|---|---|---|"]
        tot_t = tot_b = 0.0
        for k in half:
            t = k.get("gpu__time_duration.sum", 0.0)  # ns
            rd, wr = k.get("dram__bytes_read.sum", 0.0), k.get("dram__bytes_write.sum", 0.0)
            tot_t += t
            tot_b += rd + wr
            out.append(f"| `{k['name']}` | {t / 1e3:,.1f} | {rd / 1e6:,.1f} | {wr / 1e6:,.1f} | "
                       f"{(rd + wr) / t if t else 0:,.0f} |")
        out += [f"| **step** | **{tot_t / 1e3:,.1f}** | | | **{tot_b / tot_t if tot_t else 0:,.0f}** |", ""]
    out += ["## `--set full` captures", ""]
    for f in sorted(src.glob("full_*_details.csv")):
        rows = list(csv.reader(f.open()))
        h = rows[0]
        si, ni, ui, vi, ki = (h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"),
                              h.index("Metric Value"), h.index("Kernel Name"))
        got = {}
        for r in rows[1:]:
            got.setdefault((r[si], r[ni]), f"{r[vi]} {r[ui]}".strip())
        name = rows[1][ki] if len(rows) > 1 else "?"
        out += [f"### {f.stem.replace('_details', '')}: `{name}`", "", "| metric | value |", "|---|---|"]
        for key in KEYS:
            if key in got:
                out.append(f"| {key[1]} | {got[key]} |")
        out.append("")
    dst.write_text("\n".join(out) + "\n")
    print(f"wrote {dst}")


if __name__ == "__main__":
    main()

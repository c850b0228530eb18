#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  profiles/r1_full.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.md

`full`: per kernel -- duration, DRAM bytes read/written (the roofline `traffic`), DRAM
throughput %, issue-slot use, occupancy, registers and the top warp-stall reasons; also writes
profiles/ncu_traffic.json that bench.py reads for `roofline.traffic`.
`launches`: the launch list (gpu__time_duration per launch) with per-kernel totals and shares.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def _raw(rep: str) -> tuple[list, list, list]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def _num(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(val: float, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return val * scale.get(unit.strip(), 1.0)


def to_us(val: float, unit: str) -> float:
    return val * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}.get(
        unit.strip(), 1.0)


def summarize_full(rep: str, out_md: str) -> None:
    hdr, units, rows = _raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{Path(rep).name}`", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(cold cache, serialised replay: compare shares and traffic, not absolute "
             "throughput).", ""]
    traffic = {}
    stalls_all = {}
    for r in rows:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"## `{short}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        vals = {}
        for m, label in METRICS:
            if m in col:
                v, u = _num(r[col[m]]), units[col[m]]
                vals[m] = (v, u)
                lines.append(f"| {label} (`{m}`) | {r[col[m]]} {u} |")
        rd = to_bytes(*vals.get("dram__bytes_read.sum", (0, "byte")))
        wr = to_bytes(*vals.get("dram__bytes_write.sum", (0, "byte")))
        dur = to_us(*vals.get("gpu__time_duration.sum", (0, "usecond")))
        lines.append(f"| DRAM traffic read+write | {(rd + wr) / 1e6:.3f} MB |")
        if dur:
            lines.append(f"| DRAM traffic / duration | {(rd + wr) / dur / 1e3:.1f} GB/s |")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                v = _num(r[i])
                if v == v and v > 0.02:
                    stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        lines.append("")
        lines.append("Top warp stall reasons (cycles per issued instruction): " + ", ".join(
            f"{n} {v:.2f}" for v, n in stalls[:6]))
        lines.append("")
        key = ("bwd" if "bwd_tma" in short or "bwd_generic" in short else
               "reduce" if "reduce" in short else "fwd")
        traffic.setdefault(key, []).append(rd + wr)
        stalls_all[short] = stalls[:6]
    Path(out_md).write_text("\n".join(lines) + "\n")
    summary = {k: sum(v) / len(v) for k, v in traffic.items()}
    tj = Path(out_md).parent / "ncu_traffic.json"
    data = {"source": str(Path(rep).name),
            "fwd_dram_bytes_per_launch": summary.get("fwd"),
            "bwd_dram_bytes_per_launch": (summary.get("bwd") or 0) + (summary.get("reduce") or 0),
            "bwd_stage1_dram_bytes_per_launch": summary.get("bwd"),
            "bwd_stage2_dram_bytes_per_launch": summary.get("reduce")}
    tj.write_text(json.dumps(data, indent=1) + "\n")
    print(f"wrote {out_md} and {tj}")


def summarize_launches(csv_path: str, out_md: str) -> None:
    text = Path(csv_path).read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    n = 0
    for r in rows[1:]:
        if len(r) < len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        v = to_us(_num(r[col["Metric Value"]]), r[col["Metric Unit"]])
        d = per.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += v
        n += 1
    total = sum(v for _, v in per.values())
    lines = [f"# ncu launch list: `{Path(csv_path).name}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over the same command "
             "(cold-cache, serialised): per-kernel launch counts and device-time shares.", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for name, (c, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {c} | {v:.1f} | {v / c:.2f} | {100 * v / total:.1f}% |")
    lines.append("")
    lines.append(f"{n} launches, {total:.1f} us total.")
    Path(out_md).write_text("\n".join(lines) + "\n")
    print(f"wrote {out_md}")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (summarize_full if mode == "full" else summarize_launches)(src, dst)

#!/usr/bin/env python3
"""Static SASS opcode histogram of selected kernels of the built library (cuobjdump), the
evidence that the hot kernels use the Blackwell async machinery (UBLKCP = cp.async.bulk,
SYNCS = mbarrier ops) and packed fp32 math (FFMA2/FADD2/FMUL2), FHADD mixed-precision adds.

    python tools/sass_opcodes.py [out.md]
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJ = ROOT / "paper_2605_17923_b200" / "_lib" / "obj"
KERNELS = {
    "adaln_fwd_rows16<bf16, 20, 0> (cfg2 forward)": ("instances_bf16.o", "_ZN2al16adaln_fwd_rows16I13__nv_bfloat16Li20ELb0EEEvNS_9FwdParamsE"),
    "adaln_bwd_tma<bf16, 2, 2, 1, 1> (cfg2 backward: lean stage body, interleaved walk by default, ticketed tail)": ("instances_bf16.o", "_ZN2al13adaln_bwd_tmaI13__nv_bfloat16Li2ELi2ELb1ELb1EEEvNS_9BwdParamsE"),
    "adaln_bwd_tma<bf16, 2, 2, 1, 0> (static instance, kept for non-interleaved static launches)": ("instances_bf16.o", "_ZN2al13adaln_bwd_tmaI13__nv_bfloat16Li2ELi2ELb1ELb0EEEvNS_9BwdParamsE"),
    "adaln_bwd_pipe<bf16, 2, 2, 1, 0> (short launches)": ("instances_bf16.o", "_ZN2al14adaln_bwd_pipeI13__nv_bfloat16Li2ELi2ELb1ELb0EEEvNS_9BwdParamsE"),
    "adaln_bwd_reduce_vec<float> (stage 2)": ("instances_f32.o", "_ZN2al20adaln_bwd_reduce_vecIfEEvPKT_PS1_S4_lllllllPy"),
}
WATCH = ["UBLKCP", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FHADD", "F2FP", "LDS", "STS", "LDG", "STG",
         "SHFL", "BAR", "ATOMG", "RED", "FFMA", "FADD", "FMUL", "IMAD", "LOP3", "PRMT", "MUFU"]

lines = ["# SASS opcode counts (static, `cuobjdump -sass`, sm_100a)", "",
         "Instructions in the kernel body by opcode (not executed counts; see the ncu summaries "
         "for those).", "", "| kernel | " + " | ".join(WATCH) + " | total |",
         "|---|" + "---|" * (len(WATCH) + 1)]
for label, (obj, sym) in KERNELS.items():
    out = subprocess.run(["cuobjdump", "-sass", "-fun", sym, str(OBJ / obj)], capture_output=True,
                         text=True).stdout
    ops = collections.Counter()
    n = 0
    for ln in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            ops[m.group(2)] += 1
            n += 1
    lines.append(f"| `{label}` | " + " | ".join(str(ops.get(w, 0)) for w in WATCH) + f" | {n} |")
Path(sys.argv[1] if len(sys.argv) > 1 else "/dev/stdout").write_text("\n".join(lines) + "\n")

#!/bin/bash
# deterministic single-group backward: interleaved static walk on the lean (dynamic-instance)
# stage body (AL_BWD_DET_LEAN=1) vs the static instance; bitwise check of the two
mkdir -p gpurun_out/r2dl
o=gpurun_out/r2dl/dl.jsonl; : > $o
python - > gpurun_out/r2dl/bitwise.txt 2>&1 <<'P'
import os, subprocess, sys, torch
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2605_17923_b200.adaln._ops import fused_backward, fused_forward
g = torch.Generator(device="cpu").manual_seed(7)
out = []
for (b, s, d, dt) in [(1, 32760, 5120, torch.bfloat16), (1, 20001, 2048, torch.float16), (1, 15000, 4096, torch.float32), (1, 12289, 5120, torch.bfloat16)]:
    x = torch.randn(b, s, d, generator=g).to(dt).cuda(); dy = torch.randn(b, s, d, generator=g).to(dt).cuda()
    sc = (0.1 * torch.randn(b, d, generator=g)).to(dt).cuda()
    y, mu, rs = fused_forward(x, sc, sc)
    r = fused_backward(dy, x, sc, mu, rs, deterministic=True)
    out.append([t.cpu() for t in r])
torch.save(out, sys.argv[1])
'''
open("/tmp/bw.py", "w").write(code)
subprocess.run([sys.executable, "/tmp/bw.py", "/tmp/a.pt"], check=True)
subprocess.run([sys.executable, "/tmp/bw.py", "/tmp/b.pt"], check=True, env={**os.environ, "AL_BWD_DET_LEAN": "1"})
a, b = torch.load("/tmp/a.pt"), torch.load("/tmp/b.pt")
print("bitwise_equal", all(torch.equal(u, v) for ra, rb in zip(a, b) for u, v in zip(ra, rb)))
P
for rep in 1 2; do
  for cfg in 1x32760 1x46800 1x75600 1x14040; do
    set -- ${cfg/x/ }
    python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"det_static\", \"rep\": $rep, /" >> $o
    AL_BWD_DET_LEAN=1 python tools/short_s_timeline.py --one $1 $2 1 | sed "s/^{/{\"mode\": \"det_lean\", \"rep\": $rep, /" >> $o
    python tools/short_s_timeline.py --one $1 $2 0 | sed "s/^{/{\"mode\": \"dyn\", \"rep\": $rep, /" >> $o
  done
done 2> gpurun_out/r2dl/dl.err

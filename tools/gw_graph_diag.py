import os, sys, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2605_17923_b200.adaln._ops import backward_workspace_bytes, fused_backward, fused_forward
from paper_2605_17923_b200 import _native as nat
dev = torch.device('cuda', 0)
b, s, d = 2, 20000, 2048
g = torch.Generator(device='cpu').manual_seed(9)
x = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(dev)
dy = torch.randn(b, s, d, generator=g).to(torch.bfloat16).to(dev)
sc = (0.1 * torch.randn(b, d, generator=g)).to(torch.bfloat16).to(dev)
_, mu, rs = fused_forward(x, sc, sc)
ref = fused_backward(dy, x, sc, mu, rs, deterministic=True)
dx = torch.empty_like(x); dsc = torch.empty(b, d, device=dev); dsh = torch.empty(b, d, device=dev)
ws = torch.empty(backward_workspace_bytes(x, sc), dtype=torch.uint8, device=dev)
e1 = fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
torch.cuda.synchronize()
out = {"lib": os.environ.get("AL_LIB_VARIANT", "head"), "eager_same_ws_equal": bool(torch.equal(dx, ref[0]))}
side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(side):
    with torch.cuda.graph(gr, stream=side):
        fused_backward(dy, x, sc, mu, rs, out=(dx, dsc, dsh), workspace=ws, deterministic=True)
torch.cuda.synchronize()
dx.zero_(); dsc.zero_(); gr.replay(); torch.cuda.synchronize()
diff = (dx.float() - ref[0].float()).abs()
out["graph_dx_equal"] = bool(torch.equal(dx, ref[0]))
out["graph_dx_maxdiff_per_sample"] = [float(diff[i].max()) for i in range(b)]
out["graph_dsc_rel"] = [float(((dsc[i]-ref[1][i]).abs().max()/ref[1][i].abs().max())) for i in range(b)]
print(json.dumps(out))

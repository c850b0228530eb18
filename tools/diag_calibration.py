import sys; sys.path.insert(0,'.')
import torch, json
from paper_2605_17923_b200.dp_step import DPStepRunner, WanStyleBlock, measure_trials
from paper_2605_17923_b200.costfit import fit_quadratic_cost_model
dev=torch.device('cuda',0)
reqs=[(b,s) for s in (2048,4096,8192,16384) for b in (1,2,4)]
for fused in (True, False, True, False):
    blk=WanStyleBlock()
    if not fused: blk.resid_norm_fn=None
    r=DPStepRunner(blk, dev, 1, 0)
    tr=measure_trials(r, reqs, reps=3)
    q=fit_quadratic_cost_model(tr)
    print(json.dumps({"fused":fused,"r2":q.r2,"ms":[round(t.t_step*1e3,2) if hasattr(t,'t_step') else None for t in tr], "trials":[round(list(t.__dict__.values())[-1]*1e3,2) for t in tr]}))

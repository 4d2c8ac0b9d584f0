"""Host-buffer entry points timed alone against the device ones (cfg 4 default): where the e2e
overhead sits.  python tools/time_host.py [cfg] [reps]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2006_00686_b200 import Plan

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = workloads.config(cfg)
p = Plan(c, device=0)
x = workloads.make_image(c, device="cuda:0")
s = torch.empty(p.sino_shape, dtype=torch.float32, device="cuda:0")
xo = torch.empty_like(x)
xh = x.cpu().pin_memory()
sh = torch.empty(p.sino_shape, dtype=torch.float32).pin_memory()
xoh = torch.empty(p.image_shape, dtype=torch.float32).pin_memory()
def t(fn):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 2)
out = {"cfg": cfg,
       "forward": t(lambda: p.forward(x, out=s)), "forward_host": t(lambda: p.forward_host(xh, out=sh)),
       "adjoint": t(lambda: p.adjoint(s, out=xo)), "adjoint_host": t(lambda: p.adjoint_host(sh, out=xoh)),
       "h2d_img": t(lambda: x.copy_(xh, non_blocking=True)), "d2h_sino": t(lambda: sh.copy_(s, non_blocking=True)),
       "h2d_sino": t(lambda: s.copy_(sh, non_blocking=True)), "d2h_img": t(lambda: xoh.copy_(xo, non_blocking=True))}
print(json.dumps(out), flush=True)

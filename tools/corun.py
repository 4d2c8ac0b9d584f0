"""Forward and adjoint of two independent plans on two streams at once (cfg 4): does the
reduction-bound adjoint leave room for the forward?  python tools/corun.py [cfg]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2006_00686_b200 import Plan

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = workloads.config(cfg)
pf, pa = Plan(c, device=0), Plan(c, device=0)
x = workloads.make_image(c, device="cuda:0")
y = workloads.make_sino_input(c, device="cuda:0")
s = torch.empty(pf.sino_shape, dtype=torch.float32, device="cuda:0")
xo = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 2)
def both():
    cur = torch.cuda.current_stream()
    e = torch.cuda.Event(); e.record(cur)
    s1.wait_event(e); s2.wait_event(e)
    pf.forward(x, out=s, stream=s1)
    pa.adjoint(y, out=xo, stream=s2)
    cur.wait_stream(s1); cur.wait_stream(s2)
out = {"cfg": cfg, "forward": timed(lambda: pf.forward(x, out=s)), "adjoint": timed(lambda: pa.adjoint(y, out=xo)),
       "both_concurrent": timed(both)}
print(json.dumps(out), flush=True)

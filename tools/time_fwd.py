"""Forward-only (and optionally adjoint) timing of the AUTO kernels: python tools/time_fwd.py cfg [reps] [adj]
(XRT_LIB selects a library variant; CUDA events, 3 warm-ups, median of reps)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2006_00686_b200 import Plan

cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
do_adj = len(sys.argv) > 3 and sys.argv[3] == "adj"
c = workloads.config(cfg)
p = Plan(c, device=0)
x = workloads.make_image(c, device="cuda:0")
s = torch.empty(p.sino_shape, dtype=torch.float32, device="cuda:0")
xo = torch.empty_like(x)
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return statistics.median(ms), min(ms)
out = {"lib": os.environ.get("XRT_LIB", "default"), "cfg": cfg, "fwd_ms": t(lambda: p.forward(x, out=s))}
if do_adj:
    out["adj_ms"] = t(lambda: p.adjoint(s, out=xo))
print(json.dumps(out), flush=True)

"""2D RAY forward: sequential walk vs K pieces per ray (XRT_RAY2D_PIECES, read per launch), cfg 2 / 1;
adjoint: slice v2 vs K pieces (XRT_ADJ2D_PIECES).
CUDA events on the launching stream, median of 30 after 5 warm-up calls."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2006_00686_b200 import Plan

def t(fn, reps=30):
    for _ in range(5): fn()
    torch.cuda.synchronize(); ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 4)

for cfg in (2, 1):
    c = workloads.config(cfg)
    p = Plan(c, device=0)
    x = workloads.make_image(c, device="cuda:0")
    s = torch.empty(p.sino_shape, device="cuda:0")
    out = {"cfg": cfg}
    for k in sys.argv[1:] or ["1", "2", "4", "8"]:
        os.environ["XRT_RAY2D_PIECES"] = k
        out[k] = t(lambda: p.forward(x, out=s))
    y = workloads.make_sino_input(c, device="cuda:0")
    xo = torch.empty_like(x)
    for k in ["0", "4"]:   # adjoint: 0 = slice v2, else K free-running pieces
        os.environ["XRT_ADJ2D_PIECES"] = k
        out["adj" + k] = t(lambda: p.adjoint(y, out=xo))
    os.environ["XRT_ADJ2D_PIECES"] = "0"
    for k in ["0", "1", "2", "4", "8"]:   # slice adjoint: 0 = unsplit, else K lockstep pieces
        os.environ["XRT_SLICE2D_PIECES"] = k
        out["slice" + k] = t(lambda: p.adjoint(y, out=xo))
    print(json.dumps(out), flush=True)

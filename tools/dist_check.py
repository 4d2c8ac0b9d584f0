"""Correctness of the N > 1 path through libxrt (not a measurement): run under torchrun with the
gloo backend on a 1-GPU box (ranks share the GPU; collectives through the host):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py

Per configuration, every rank's ShardedPlan (its view block) is checked against ONE unsharded plan
of the full geometry on the same GPU: the forward slab, the staged adjoint with the overlapped
all-reduce (cfg 3 / 4), and for the helical beam the windowed scatter + forward and the windowed
adjoint (P2P overlap exchange) on the rank's z window.  Prints one JSON line per rank."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import workloads
from paper_2006_00686_b200 import Plan
from paper_2006_00686_b200.dist import ShardedPlan, view_block

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)


def rel(a, b):
    a = a.double(); b = b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


out = {"rank": rank, "world": world}
cfgs = [int(v) for v in os.environ.get("CFGS", "3 4 5").split()]
for idx in cfgs:
    c = workloads.config(idx)
    full = Plan(c, device=0)
    sp = ShardedPlan(c, rank=rank, world=world, device=0)
    v0, v1 = view_block(c["n_views"], rank, world)
    x = workloads.make_image(c, device=dev)
    y = workloads.make_sino_input(c, device=dev)
    ref_f = full.forward(x)[v0:v1]
    ref_b = full.adjoint(y)
    r = {}
    if c["beam"] == "helical":
        k0, k1 = sp.window()
        xw = x.clone()
        if rank != 0:
            xw.zero_()
        sp.scatter_windows(xw, src=0)                  # rank's window rows from rank 0
        r["window"] = [k0, k1]
        r["scatter_exact"] = bool(torch.equal(xw[k0:k1], x[k0:k1]))
        r["forward_rel"] = rel(sp.plan.forward(xw), ref_f)
        b = sp.adjoint_windowed(y[v0:v1].contiguous())
        r["adjoint_window_rel"] = rel(b[k0:k1], ref_b[k0:k1])
    else:
        r["forward_rel"] = rel(sp.forward(x), ref_f)
        b = sp.adjoint(y[v0:v1].contiguous(), overlap=True)
        r["adjoint_staged_rel"] = rel(b, ref_b)
        b2 = sp.adjoint(y[v0:v1].contiguous(), overlap=False)
        r["staged_vs_plain_rel"] = rel(b, b2)
    ok = r["forward_rel"] <= 1e-6 and all(v <= 1e-6 for k, v in r.items() if k.endswith("_rel"))
    r["ok"] = bool(ok and r.get("scatter_exact", True))
    out[c["name"]] = r
    del full, sp
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()

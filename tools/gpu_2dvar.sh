#!/bin/bash
set -u
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_2dv.log 2>&1; echo "pytest exit $?" >> $out/pytest_2dv.log
tail -2 $out/pytest_2dv.log
cat > /tmp/t2d.py <<'PY'
import json, os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch, workloads
from paper_2006_00686_b200 import Plan
for cfg in (2, 1):
    c = workloads.config(cfg)
    p = Plan(c, device=0)
    x = workloads.make_image(c, device="cuda:0"); y = workloads.make_sino_input(c, device="cuda:0")
    s = torch.empty(p.sino_shape, device="cuda:0"); xo = torch.empty_like(x)
    def t(fn, reps=20):
        for _ in range(3): fn()
        torch.cuda.synchronize(); ms = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
        return round(statistics.median(ms), 4)
    out = {"cfg": cfg, "v1": bool(os.environ.get("XRT_SLICE_V1"))}
    for algo in ("ray", "column"):
        p.set_algorithm("forward", algo); p.set_algorithm("adjoint", algo)
        out[algo] = (t(lambda: p.forward(x, out=s)), t(lambda: p.adjoint(y, out=xo)))
    print(json.dumps(out))
PY
for lib in paper_2006_00686_b200/libxrt.so "$@"; do
  XRT_LIB=$lib python /tmp/t2d.py 2>&1 | sed "s|^|$lib |"
done

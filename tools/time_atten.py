"""Time the attenuated transform (RAY family) next to the plain operator on one config.
usage: python tools/time_atten.py CFG [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2006_00686_b200 import Plan  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


idx = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = workloads.config(idx)
p = Plan(c, device=0)
img = workloads.make_image(c, device="cuda")
mu = workloads.make_attenuation(c, device="cuda")
y = workloads.make_sino_input(c, device="cuda")
sino = torch.empty(p.sino_shape, device="cuda")
back = torch.empty(p.image_shape, device="cuda")
out = {"cfg": idx, "rays": p.n_rays}
out["att_forward_ms"] = timed(lambda: p.forward_attenuated(img, mu, out=sino), reps)
out["att_adjoint_ms"] = timed(lambda: p.adjoint_attenuated(y, mu, out=back), reps)
out["forward_ms"] = timed(lambda: p.forward(img, out=sino), reps)
out["adjoint_ms"] = timed(lambda: p.adjoint(y, out=back), reps)
p.set_algorithm("forward", "ray")
p.set_algorithm("adjoint", "ray")
out["ray_forward_ms"] = timed(lambda: p.forward(img, out=sino), reps)
out["ray_adjoint_ms"] = timed(lambda: p.adjoint(y, out=back), reps)
print(json.dumps(out))

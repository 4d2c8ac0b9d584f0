"""cfg 2 (2D fan) forward and adjoint through the slice kernels (COLUMN), 2 calls each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2006_00686_b200 import Plan
c = workloads.config(2)
p = Plan(c, device=0)
p.set_algorithm("forward", "column"); p.set_algorithm("adjoint", "column")
x = workloads.make_image(c, device="cuda:0"); y = workloads.make_sino_input(c, device="cuda:0")
for _ in range(2):
    s = p.forward(x); b = p.adjoint(y)
torch.cuda.synchronize()
print("ok", float(s.abs().max()), float(b.abs().max()))

"""A few periodic solves at one grid size (for ncu): python tools/spec_profile.py 8192 [cufft]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11007_b200 as cs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
if len(sys.argv) > 2:
    os.environ["CS_CUFFT"] = "1"
grid = cs.Grid.square(n, 1.0, "periodic")
ops = cs.build_operators(grid, cs.FieldParams(d_c=1.0), 1e-5)
rhs = torch.randn(n * n, device="cuda", dtype=torch.float32)
for _ in range(4):
    ops.solve(rhs)
torch.cuda.synchronize()

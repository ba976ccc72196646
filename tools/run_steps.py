"""Debug driver: one sorted-engine configuration, N and grid from argv, a few
steps with a sync after each stage (CUDA_LAUNCH_BLOCKING=1 recommended)."""
import sys

import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dict(bench.CONFIGS["cfg3"])
cfg["n"] = n
import torch
sim, st, pos, sp = bench.make_state(cfg, 0)
xi = torch.randn((steps, n, 2), device="cuda", dtype=torch.float32)
for k in range(steps):
    sim.step(xi[k], 1)
    torch.cuda.synchronize()
    print("step", k, "ok", sim.status().code, flush=True)

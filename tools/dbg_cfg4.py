"""cfg4 diagnostics: status and the largest node mass per step (sorted engine)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sim, st, pos, sp = bench.make_state(cfg, 0)
n = cfg["n"]
gen = torch.Generator(device="cuda").manual_seed(1)
d2 = (1.0 / cfg["n_c"]) ** 2
for s in range(steps):
    xi = torch.randn((n, 2), generator=gen, device="cuda", dtype=torch.float32)
    sim.step(xi, 1)
    sim.export_state()
    torch.cuda.synchronize()
    code = sim.status().code
    ma = float(st["rho_a"].max()) * d2
    mb = float(st["rho_b"].max()) * d2
    c = st["c"]
    print(f"step {s} status {code} max node mass a {ma:.1f} b {mb:.1f} c [{float(c.min()):.3g}, "
          f"{float(c.max()):.3g}]", flush=True)
    if code:
        break

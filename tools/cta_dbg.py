import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_1805_11007_b200 as cs
def make(cfg, engine):
    orig = cs.sim_params_struct
    def forced(*a, **kw):
        kw["engine"] = engine
        return orig(*a, **kw)
    cs.sim_params_struct = forced
    try:
        return bench.make_state(cfg, 0)
    finally:
        cs.sim_params_struct = orig
cfg = dict(bench.CONFIGS["cfg1"], n=1000, n_c=48, field=True, c0="linear_x")
xi = torch.as_tensor(np.random.default_rng(7).standard_normal((3, cfg["n"], 2)), device="cuda")
for steps in (1, 2, 3):
    a, sa, _, _ = make(cfg, "auto")
    b, sb, _, _ = make(cfg, "direct")
    a.step(xi[:steps], steps)
    b.step(xi[:steps], steps)
    for k in ("pos", "c", "rho_a", "grad"):
        if sa.get(k) is None: continue
        d = (sa[k] - sb[k]).abs().max().item()
        print(steps, k, a.engine, d, (sa[k] != sb[k]).sum().item())

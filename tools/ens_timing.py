"""Quick timing of the batched ensemble engine on the fig1 preset."""
import sys
import time
import warnings

import numpy as np
import torch

import paper_1805_11007_b200 as cs
from paper_1805_11007_b200.ensemble import Ensemble

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
warnings.simplefilter("ignore")
cfg = cs.SimConfig.preset("fig1", samples=S)
ens = Ensemble(cfg)
t = time.perf_counter()
xi, u = ens._draw(K)
t_rng = time.perf_counter() - t
ens.advance(K, (xi, u))
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
xd = torch.as_tensor(xi, device="cuda")
ud = torch.as_tensor(u, device="cuda")
import ctypes
from paper_1805_11007_b200 import _native as N
lib = N.load_library()
ev0.record()
for _ in range(5):
    N.check(lib.cs_ens_step(ens._h, ctypes.byref(ens._st), N.ptr(xd), N.ptr(ud), K), "step")
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / (5 * K)
print(f"S={S} N={cfg.n_total} n_c={cfg.n_c}: device {ms*1e3:.1f} us/step for all samples "
      f"= {S*cfg.n_total/(ms*1e-3):.3e} particle-steps/s; host RNG {t_rng/K*1e3:.2f} ms/step "
      f"({ens.threads} threads); fig1 n_steps {cfg.n_steps}")
t = time.perf_counter()
cfg2 = cs.SimConfig.preset("fig1", samples=S, t_final=200 * cfg.dt)
res = cs.run_ensemble(cfg2)
print(f"run_ensemble 200 steps wall {time.perf_counter()-t:.2f} s")

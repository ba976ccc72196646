"""The public API at BASELINE cfg3 scale: Realisation(SimConfig ~ cfg3).run()
with the increments drawn on the device (one numpy stream per realisation),
timed per step (observables at the record steps included)."""
import sys
import time
import warnings

import torch

sys.path.insert(0, ".")
import paper_1805_11007_b200 as cs

warnings.simplefilter("ignore")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = cs.SimConfig(n_alpha_0=5_000_000, n_beta_0=5_000_000, d_alpha=1.0, d_beta=0.5,
                   chi_alpha=1.0, chi=-0.5, epsilon=6.1804e-5, soft_cutoff_factor=2.0,
                   radius_alpha=6.1804e-5, radius_beta=1.2361e-4, dt=1e-5,
                   t_final=steps * 1e-5, r_alpha=0.0, r_beta=0.0, periodic=True, n_c=4096,
                   deposit="cic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                   precision="fp32", output_every=steps, seed_base=3)
t0 = time.perf_counter()
real = cs.Realisation(cfg, 0)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"engine {real._sim.engine}; init {t1 - t0:.2f} s")
obs = real.run(max_block_bytes=1 << 31)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"run: {steps} steps in {t2 - t1:.3f} s = {(t2 - t1) / steps * 1e3:.2f} ms/step "
      f"({cfg.n_total * steps / (t2 - t1):.3e} particle-steps/s incl. draws and observables); "
      f"msd {obs.msd[-1]:.3e}, counts {obs.counts[-1].tolist()}")

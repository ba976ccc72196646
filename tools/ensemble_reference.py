"""Time the reference's own Realisation on the fig1 preset (one core) ->
profiles/r01/ensemble_reference.json.  Runs in the builder container only
(the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
    OPENBLAS_NUM_THREADS=1 python tools/ensemble_reference.py
"""
import json
import os
import platform
import time
import warnings

import chemosim as cs

warnings.simplefilter("ignore")
cfg = cs.SimConfig.preset("fig1")
r = cs.Realisation(cfg, 0)
for _ in range(50):  # JIT warm-up
    r.step()
steps = 1500
t = time.perf_counter()
for _ in range(steps):
    r.step()
dt = time.perf_counter() - t
out = {"impl": "reference", "metric": "realisation-steps/s (Realisation.step, fig1)",
       "value": steps / dt, "unit": "realisation-steps/s", "cores": 1,
       "ms_per_step": 1e3 * dt / steps, "steps_timed": steps,
       "per_realisation_s_full_fig1": dt / steps * cfg.n_steps,
       "host": platform.processor() or platform.machine(), "cpu_count": os.cpu_count(),
       "sample": "sample 0 of SimConfig.preset('fig1'), 1500 steps after 50 warm-up steps, "
                 "OPENBLAS_NUM_THREADS=1; the reference parallelises ensembles only by "
                 "process (config.threads), so S samples on C cores take S / C times this"}
os.makedirs("profiles/r01", exist_ok=True)
json.dump(out, open("profiles/r01/ensemble_reference.json", "w"), indent=1)
print(json.dumps(out))

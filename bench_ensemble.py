"""Throughput of the paper's own workload: an ensemble of small
realisations (engine.py:455-484 run_ensemble).

    python bench_ensemble.py [--preset fig1] [--samples 2000] [--steps K]

Default: the fig1 clustering experiment exactly as the reference's
``SimConfig.preset("fig1")`` defines it (100 Alpha + 100 Beta cells,
soft forces with cutoff 5 eps, gaussian deposit on the neumann 52^2 grid,
implicit DCT-I field step, fixed-step reactions r_alpha = 10, dt =
(0.23 eps)^2 / (4 d_beta), 9452 steps), 2000 seeded samples run through the
drop-in ``run_ensemble`` (batched engine, device-drawn numpy-identical
random streams, observables recorded at the reference's steps).  --steps
truncates t_final.

Prints one JSON line: realisation-steps/s and particle-steps/s end to end
(wall clock of run_ensemble incl. set-up and the host observables), and the
device time of the ensemble kernels alone (CUDA events).  The reference's
per-realisation rate is measured by tools/ensemble_reference.py on the
reference itself (profiles/r01/ensemble_reference.json).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="fig1")
    ap.add_argument("--samples", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=0, help="truncate to this many steps")
    args = ap.parse_args()
    import torch

    import paper_1805_11007_b200 as cs
    from paper_1805_11007_b200 import _native as N
    from paper_1805_11007_b200 import ensemble as E

    warnings.simplefilter("ignore")
    cfg = cs.SimConfig.preset(args.preset, samples=args.samples)
    if args.steps:
        cfg = cs.SimConfig.preset(args.preset, samples=args.samples, t_final=args.steps * cfg.dt)
    steps = cfg.n_steps
    # device time of the stepping kernels: CUDA events around every launch
    events = []
    orig_advance = E.Ensemble.advance

    def timed(self, k, drawn=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        orig_advance(self, k, drawn)
        e1.record()
        events.append((e0, e1))
    E.Ensemble.advance = timed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = cs.run_ensemble(cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_s = sum(a.elapsed_time(b) for a, b in events) / 1e3
    E.Ensemble.advance = orig_advance
    n = cfg.n_total
    rs = cfg.samples * steps
    ref_path = os.path.join(ROOT, "profiles", "r01", "ensemble_reference.json")
    ref = json.load(open(ref_path)) if os.path.exists(ref_path) else None
    line = {
        "metric": "realisation-steps/s (run_ensemble, fig1)", "value": rs / wall,
        "unit": "realisation-steps/s", "particle_steps_per_s": rs * n / wall,
        "wall_s": wall, "device_s": dev_s, "device_realisation_steps_per_s": rs / dev_s,
        "samples": cfg.samples, "steps": steps, "particles": n, "n_c": cfg.n_c,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic (seeded samples)",
        "config": {"workload": f"{args.preset} ensemble", "samples": cfg.samples,
                   "steps": steps, "engine": "batched (one CTA per realisation)",
                   "rng": "device (numpy PCG64 / ziggurat restated, bit-identical)"},
        "gpu_launches": len(events) * (2 if cfg.r_alpha > 0 or cfg.r_beta > 0 else 1) +
        len(events),
        "final_counts_mean": res.counts_mean[-1].tolist(),
    }
    if ref:
        line["reference_1core_realisation_steps_per_s"] = ref["value"]
        line["speedup_vs_reference_1core"] = (rs / wall) / ref["value"]
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

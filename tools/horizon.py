"""Trajectory horizon of a BASELINE config (SURVEY 8c tier T2, the 0.4 method).

    python tools/horizon.py --config cfg3 --steps 5 [--out gpurun_out/horizon_cfg3.json]

Runs, from the bench's seeded initial state and increments:
  A  the oracle (fp32 storage mode, all host cores)
  B  the oracle from A's initial positions moved by one binary32 ulp
  G  the sorted engine on the GPU (the benchmarked path)
and prints, per step, quantiles of the minimum-image position differences
|G - A| and |B - A| (max over the two axes) and the field's max relative
difference.  B - A is the chaos envelope of the reference arithmetic
itself: the tolerance a K-step comparison can state.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

QS = (0.5, 0.99, 0.9999, 1.0)


def dmin(a, b):
    d = a - b
    d -= np.rint(d)  # unit box
    return np.abs(d).max(axis=1)


def stats(d):
    return {"q%g" % q: float(np.quantile(d, q)) for q in QS} | {
        "n_gt_4ulp": int(np.count_nonzero(d > 4 * 2.0 ** -24))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-field", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    cfg = dict(bench.CONFIGS[args.config])
    if args.no_field:
        cfg["field"] = False
    n, K = cfg["n"], args.steps
    sim, st, pos0, sp = bench.make_state(cfg, 0)
    xi_rng = np.random.default_rng(bench.SEED + 1)
    xi = [xi_rng.standard_normal((n, 2)).astype(np.float32) for _ in range(K)]
    g_pos, g_c = [], []
    for k in range(K):
        sim.step(torch.as_tensor(xi[k], device="cuda"), 1)
        sim.export_state()
        assert sim.status().code == 0
        g_pos.append(st["pos"].double().cpu().numpy())
        if cfg["field"]:
            g_c.append(st["c"].double().cpu().numpy())
    ncores = os.cpu_count() or 1
    p32 = pos0.astype(np.float32)
    pert = np.nextafter(p32, np.float32(np.inf)).astype(np.float64)
    runs = {}
    for tag, p in (("A", p32.astype(np.float64)), ("B", pert)):
        o = bench.oracle_sim(cfg, p, sp, ncores)
        o.anchor_mode = "wraps"
        out_p, out_c = [], []
        t0 = time.time()
        for k in range(K):
            o.step(xi[k].astype(np.float64))
            out_p.append(o.pos.copy())
            if cfg["field"]:
                out_c.append(o.c.copy())
        runs[tag] = (out_p, out_c)
        print(f"oracle {tag}: {K} steps in {time.time() - t0:.1f} s", file=sys.stderr)
    res = {"config": args.config, "n": n, "steps": K, "field": cfg["field"], "per_step": []}
    for k in range(K):
        a, b = runs["A"][0][k], runs["B"][0][k]
        row = {"step": k + 1, "gpu_vs_oracle": stats(dmin(g_pos[k], a)),
               "perturbed_vs_oracle": stats(dmin(b, a))}
        if cfg["field"]:
            ca, cb = runs["A"][1][k], runs["B"][1][k]
            scale = max(np.abs(ca).max(), 1e-300)
            row["field_gpu_rel"] = float(np.abs(g_c[k] - ca).max() / scale)
            row["field_perturbed_rel"] = float(np.abs(cb - ca).max() / scale)
        res["per_step"].append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()

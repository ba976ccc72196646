"""Cut a small reproducer out of a full-size sorted/direct mismatch.

    python tools/seam_repro.py --config cfg3 --steps 5 --ids 7501953 8777260

Runs the direct engine for steps-1 steps, keeps the particles within 1e-3
(minimum image) of the given ids, and checks one sorted vs direct step of
that subset in the same box; writes gpurun_out/seam_repro.npz.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from tools.diff_engines import run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ids", type=int, nargs="+")
    ap.add_argument("--radius", type=float, default=1e-3)
    args = ap.parse_args()
    import torch
    import paper_1805_11007_b200 as cs
    cfg = dict(bench.CONFIGS[args.config], field=False)
    n = cfg["n"]
    xi_rng = np.random.default_rng(bench.SEED + 1)
    xi = xi_rng.standard_normal((args.steps, n, 2)).astype(np.float32)
    prev, _, sp = run(cfg, "direct", xi, args.steps - 1)
    keep = np.zeros(n, bool)
    for i in args.ids:
        d = prev - prev[i]
        d -= np.rint(d)
        keep |= np.abs(d).max(axis=1) < args.radius
    idx = np.flatnonzero(keep)
    print("subset", idx.size, "ids", idx[:40])
    sub = dict(pos=prev[idx].astype(np.float32), sp=sp[idx], xi=xi[-1][idx], idx=idx)
    np.savez(os.path.join(ROOT, "gpurun_out", "seam_repro.npz"), **sub)
    for i in args.ids:
        j = int(np.flatnonzero(idx == i)[0])
        print("id", i, "local", j, "pos", prev[i], "cell", np.floor((prev[i] + 0.5) / (1 / 4045)))
    outs = {}
    for engine in ("sorted", "direct"):
        st = dict(cfg, n=idx.size)
        orig = cs.sim_params_struct

        def forced(*a, **kw):
            kw["engine"] = engine
            return orig(*a, **kw)
        cs.sim_params_struct = forced
        try:
            sim, s, _, _ = bench.make_state(st, 0)
        finally:
            cs.sim_params_struct = orig
        s["pos"].copy_(torch.as_tensor(sub["pos"], device="cuda"))
        s["anchor"].copy_(torch.as_tensor(sub["pos"], device="cuda"))
        s["species"].copy_(torch.as_tensor(sub["sp"], device="cuda"))
        sim.import_state()
        sim.step(torch.as_tensor(sub["xi"][None], device="cuda"), 1)
        sim.export_state()
        outs[engine] = s["pos"].double().cpu().numpy()
        print(engine, sim.engine, sim.status().code)
    bad = np.flatnonzero(np.any(outs["sorted"] != outs["direct"], axis=1))
    print("subset mismatches", bad, idx[bad])
    for j in bad:
        print(j, outs["sorted"][j], outs["direct"][j])


if __name__ == "__main__":
    main()

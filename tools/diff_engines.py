"""Sorted vs direct engine (and the field-free oracle) after K steps at a
BASELINE size: counts and examples of differing particles.

    python tools/diff_engines.py --config cfg3 --steps 1
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run(cfg, engine, xi, steps):
    import torch
    import paper_1805_11007_b200 as cs
    orig = cs.sim_params_struct

    def forced(*a, **kw):
        kw["engine"] = engine
        return orig(*a, **kw)
    cs.sim_params_struct = forced
    try:
        sim, st, pos, sp = bench.make_state(cfg, 0)
    finally:
        cs.sim_params_struct = orig
    sim.step(torch.as_tensor(xi[:steps], device="cuda"), steps)
    sim.export_state()
    print(engine, sim.engine, "status", sim.status().code, file=sys.stderr)
    out = st["pos"].double().cpu().numpy()
    del sim, st
    torch.cuda.empty_cache()
    return out, pos, sp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--oracle", action="store_true")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config], field=False)
    n = cfg["n"]
    xi_rng = np.random.default_rng(bench.SEED + 1)
    xi = xi_rng.standard_normal((args.steps, n, 2)).astype(np.float32)
    a, pos0, sp = run(cfg, "sorted", xi, args.steps)
    b, _, _ = run(cfg, "direct", xi, args.steps)
    bad = np.flatnonzero(np.any(a != b, axis=1))
    print("sorted != direct:", bad.size)
    p32 = pos0.astype(np.float32).astype(np.float64)
    for i in bad[:12]:
        print(i, "type", sp[i], "start", p32[i], "sorted", a[i], "direct", b[i],
              "diff", a[i] - b[i])
    if args.oracle:
        o = bench.oracle_sim(cfg, p32, sp, os.cpu_count())
        for k in range(args.steps):
            o.step(xi[k].astype(np.float64))
        for tag, x in (("sorted", a), ("direct", b)):
            d = np.flatnonzero(np.any(x != o.pos, axis=1))
            print(f"{tag} != oracle:", d.size, d[:12])
        for i in bad[:12]:
            print(i, "oracle", o.pos[i])


if __name__ == "__main__":
    main()

"""A short fig1 ensemble for profiling k_ensemble (ncu -k regex:k_ensemble).

    python tools/ens_profile.py [--samples 296] [--steps 20]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=296)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--no-field", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1805_11007_b200 as cs
    from paper_1805_11007_b200.ensemble import Ensemble
    kw = {"samples": args.samples}
    if args.no_field:
        kw.update(d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = cs.SimConfig(**kw)
    ens = Ensemble(cfg)
    ens.advance(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ens.advance(args.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{args.samples} samples x {args.steps} steps: {1e3 * dt / args.steps:.3f} ms/step")
    ens.close()


if __name__ == "__main__":
    main()

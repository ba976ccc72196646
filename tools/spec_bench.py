"""Periodic solve timing: the own spectral passes vs cuFFT (CS_CUFFT=1).

    python tools/spec_bench.py [--reps 20]

Times Operators.solve (rhs copy + solve) on the device with CUDA events for
the BASELINE periodic grids: 512^2 binary64 (cfg2), 512^2 binary32
(cfg2f32), 4096^2 binary32 (cfg3), 8192^2 binary32 (cfg4).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_1805_11007_b200 as cs
    out = []
    for n, dt_ in ((512, torch.float64), (512, torch.float32), (4096, torch.float32),
                   (8192, torch.float32)):
        row = {"n": n, "dtype": str(dt_).split(".")[-1]}
        for mode in ("own", "cufft"):
            if mode == "cufft":
                os.environ["CS_CUFFT"] = "1"
            else:
                os.environ.pop("CS_CUFFT", None)
            grid = cs.Grid.square(n, 1.0, "periodic")
            ops = cs.build_operators(grid, cs.FieldParams(d_c=1.0), 1e-5)
            rhs = torch.randn(n * n, device="cuda", dtype=dt_)
            for _ in range(3):
                ops.solve(rhs)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(args.reps):
                ops.solve(rhs)
            b.record()
            torch.cuda.synchronize()
            row[mode + "_us"] = round(1e3 * a.elapsed_time(b) / args.reps, 2)
            ops.close()
        os.environ.pop("CS_CUFFT", None)
        print(json.dumps(row), flush=True)
        out.append(row)


if __name__ == "__main__":
    main()

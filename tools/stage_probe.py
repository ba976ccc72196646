"""Stage times of the sorted engine at cfg3 under the CS_FAST_DEBUG timing
diagnostics (wrong results for 4 / 8; timing only) and in performance mode.
usage: python tools/stage_probe.py [debug values ...]   (e.g. 0 1 4 8 s0 s4)
a leading 's' = xi_by_slot."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

cfg = bench.CONFIGS[os.environ.get("PROBE_CFG", "cfg3")]
n = cfg["n"]
xi = torch.randn((6, n, 2), device="cuda", dtype=torch.float32)
for spec in sys.argv[1:] or ["0"]:
    slot = spec.startswith("s")
    dbg = int(spec.lstrip("s"))
    os.environ.pop("CS_FAST_DEBUG", None)
    sim, st, _, _ = bench.make_state(cfg, 0, xi_by_slot=slot)
    for w in range(3):
        sim.step(xi[w], 1)
    torch.cuda.synchronize()
    if dbg:
        os.environ["CS_FAST_DEBUG"] = str(dbg)
    sim.set_profiling(True)
    KP = 1 if dbg & 12 else 6  # 4 / 8 leave garbage behind: one step only
    for k in range(KP):
        sim.step(xi[k % 6], 1)
    stg = {k: round(v / KP, 4) for k, v in sim.stage_times().items()}
    sim.set_profiling(False)
    print(f"slot={int(slot)} debug={dbg}", stg, flush=True)
    del sim, st
    torch.cuda.empty_cache()

"""Per-phase device time of one rank's slab step (world 1 over NCCL, cfg3 by
default): field exchanges and passes, local forces + update, record
exchange, claim + sort + deposit.  python tools/slab_probe.py [cfg] [steps]"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1805_11007_b200 import slabs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = bench.CONFIGS[name]
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29517")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
params, st, bounds, plan = bench.slab_setup(cfg, 1)
eng = slabs.SlabEngine(params, st, bounds, 0, 1, field_plan=plan)
tr = slabs.NcclTransport(1)
xi = torch.randn((4, cfg["n"], 2), device="cuda", dtype=torch.float32)
for w in range(3):
    eng.step(xi[w], tr)
nf = eng._nf
torch.cuda.synchronize()
acc = {}


def timed(label, fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    acc[label] = acc.get(label, 0.0) + a.elapsed_time(b)
    return out


for k in range(K):
    timed("field", nf.step)
    timed("local", lambda: eng.local(xi[k % 4]))
    recs, dest = eng.outbox()
    got = timed("exchange", lambda: tr.exchange(recs, dest))
    timed("claim+finish", lambda: (eng.claim(got), eng.finish()))
print({k: round(v / K, 4) for k, v in acc.items()}, "ms/step, sum",
      round(sum(acc.values()) / K, 4))
dist.destroy_process_group()

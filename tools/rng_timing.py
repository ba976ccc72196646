import ctypes, sys, time
import numpy as np, torch
from paper_1805_11007_b200 import _native as N
S, k, m = 2000, 20, 400
w = np.random.default_rng(0).integers(0, 2**63, (S, 4), dtype=np.int64) | 1
dev = torch.as_tensor(w, device="cuda")
out = torch.empty((k, S, m), dtype=torch.float64, device="cuda")
lib = N.load_library()
for kind in (0, 1):
    lib.cs_rng_fill(N.context(), N.ptr(dev), S, kind, k, m, N.ptr(out))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.cs_rng_fill(N.context(), N.ptr(dev), S, kind, k, m, N.ptr(out))
    e1.record(); torch.cuda.synchronize()
    print("kind", kind, "ms per block of 20 steps:", e0.elapsed_time(e1) / 5)

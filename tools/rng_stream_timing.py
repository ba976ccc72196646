"""Device draws of one numpy stream: time per (N, 2) block at N = 10^7 (binary32
out) vs numpy on one host core."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1805_11007_b200 import rng

g = np.random.default_rng(1)
n = 10_000_000
for k in (1, 8):
    rng.draw(g, "normal", (k, n, 2), torch.float32)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        rng.draw(g, "normal", (k, n, 2), torch.float32)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"device: {k} x (1e7, 2) normals in {dt * 1e3:.2f} ms ({dt / k * 1e3:.2f} ms/step)")
t = time.perf_counter()
g.standard_normal((n, 2))
print(f"numpy one core: (1e7, 2) normals in {(time.perf_counter() - t) * 1e3:.1f} ms")

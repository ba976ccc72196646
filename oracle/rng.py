"""numpy Generator(PCG64) restated in Python -- TEST INFRASTRUCTURE ONLY.

The device restatement (csrc/rng.cu) draws the reference's Brownian
increments and reaction uniforms itself; this scalar restatement pins the
algorithm against numpy (the reference's RNG, engine.py:272-275,
motion.py:277): PCG64 = 128-bit LCG with numpy's default multiplier and the
XSL-RR output (numpy/random/src/pcg64/pcg64.h), next_double =
(u64 >> 11) * 2^-53, standard_normal = the 256-layer ziggurat of
numpy/random/src/distributions/distributions.c (random_standard_normal)
with the tables tools/ziggurat_tables.py reads from numpy's own library.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596

_tables = None


def tables():
    global _tables
    if _tables is None:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                        "tools"))
        from ziggurat_tables import load_tables
        ki, wi, fi = load_tables()
        _tables = ([int(v) for v in ki], [float(v) for v in wi], [float(v) for v in fi])
    return _tables


class PCG64:
    def __init__(self, state: int, inc: int):
        self.state, self.inc = state, inc

    @classmethod
    def of(cls, gen: np.random.Generator) -> "PCG64":
        s = gen.bit_generator.state["state"]
        return cls(s["state"], s["inc"])

    def next64(self) -> int:
        self.state = (self.state * MULT + self.inc) & MASK128
        hi, lo = self.state >> 64, self.state & ((1 << 64) - 1)
        rot = self.state >> 122
        x = hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def standard_normal(self) -> float:
        ki, wi, fi = tables()
        while True:
            r = self.next64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * wi[idx]
            if sign:
                x = -x
            if rabs < ki[idx]:
                return x
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-self.next_double())
                    yy = -math.log1p(-self.next_double())
                    if yy + yy > xx * xx:
                        return -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
            else:
                if ((fi[idx - 1] - fi[idx]) * self.next_double() + fi[idx]) < \
                        math.exp(-0.5 * x * x):
                    return x

"""numpy Generator(PCG64) streams drawn on the device, bit for bit.

The reference draws every step's Brownian increments as one
``rng_motion.standard_normal((N, 2))`` block and the reaction uniforms as
``rng_react.random(N)`` (engine.py:272-275, motion.py:277, reactions.py:57).
At N = 10^7 numpy needs ~0.1 s per block on one core; ``draw`` hands the
generator's state to the device (csrc/rng.cu ``cs_rng_fill_stream``: the
stream's raw outputs by LCG jump-ahead, the ziggurat attempts evaluated in
parallel and chained chunk by chunk) and advances the numpy generator by
exactly the raws consumed, so host and device draws interleave freely and
the values equal numpy's own.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N

_MASK = 0xFFFFFFFFFFFFFFFF


def draw(gen: np.random.Generator, kind: str, shape, dtype=None):
    """CUDA tensor of ``gen.standard_normal(shape)`` (kind "normal") or
    ``gen.random(shape)`` (kind "uniform"), drawn on the device; ``gen``
    ends in the state numpy's own draw would leave it in.  dtype float32
    rounds the binary64 values (the binary32 engines' increments)."""
    torch = N.require_cuda()
    dtype = torch.float64 if dtype is None else dtype
    bg = gen.bit_generator
    st = bg.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("device draws restate numpy's PCG64 only")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    words = (ctypes.c_uint64 * 4)(s >> 64, s & _MASK, inc >> 64, inc & _MASK)
    out = torch.empty(tuple(shape), dtype=dtype, device="cuda")
    m = int(out.numel())
    N.check(N.load_library().cs_rng_fill_stream(
        N.context(), words, 0 if kind == "normal" else 1, m, int(dtype == torch.float32),
        N.ptr(out)), "cs_rng_fill_stream")
    st["state"]["state"] = (int(words[0]) << 64) | int(words[1])
    bg.state = st
    return out

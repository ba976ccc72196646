"""One numpy stream drawn by the whole device (cs_rng_fill_stream, rng.draw)
against numpy itself: standard_normal and random blocks bit for bit across
chunk boundaries (sizes from 1 to 5 * 10^6, several seeds, so the ziggurat's
wedge and tail paths occur thousands of times), binary32 rounding, and the
generator state afterwards (numpy continues the same stream)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1805_11007_b200 import rng  # noqa: E402


@pytest.mark.parametrize("seed,m", [(0, 1), (1, 7), (2, 4095), (3, 4097), (4, 100_000),
                                    (5, 5_000_000), (6, 1_234_567)])
def test_normals_bitwise_and_state(seed, m):
    ref = np.random.default_rng(seed)
    ours = np.random.default_rng(seed)
    want = ref.standard_normal(m)
    got = rng.draw(ours, "normal", (m,)).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert ours.bit_generator.state == ref.bit_generator.state
    assert np.array_equal(ours.standard_normal(1000), ref.standard_normal(1000))


def test_blocks_shapes_f32_and_uniforms():
    ref = np.random.default_rng(np.random.SeedSequence(11).spawn(3)[1])
    ours = np.random.default_rng(np.random.SeedSequence(11).spawn(3)[1])
    for k in range(3):  # per-step (N, 2) blocks and a (K, N, 2) block, as the engine draws
        want = ref.standard_normal((5, 300_000, 2))
        got = rng.draw(ours, "normal", (5, 300_000, 2))
        assert np.array_equal(got.cpu().numpy(), want)
    want = ref.standard_normal((200_000, 2))
    got = rng.draw(ours, "normal", (200_000, 2), torch.float32)
    assert np.array_equal(got.cpu().numpy(), want.astype(np.float32))
    want = ref.random((3, 400_000))
    got = rng.draw(ours, "uniform", (3, 400_000))
    assert np.array_equal(got.cpu().numpy(), want)
    assert ours.bit_generator.state == ref.bit_generator.state


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_realisation_device_draws_equal_host_draws(precision):
    """Realisation(rng="device") draws its increments (and the fixed
    scheduler's uniforms) on the device: the same trajectory, bit for bit, as
    rng="host", and the generators end in the same state.  (Field off: the
    direct engine's binary64 deposit sums with atomics, so field-coupled runs
    agree to ~1e-18 from run to run, not bit for bit.)"""
    import warnings
    import paper_1805_11007_b200 as cs
    cfg = dict(n_alpha_0=3000, n_beta_0=3000, d_alpha=1.0, d_beta=0.5, chi=-0.5,
               epsilon=0.002, soft_cutoff_factor=2.0, dt=1e-5, t_final=3e-4, r_alpha=5.0,
               r_beta=0.0, periodic=True, d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0,
               output_every=10, precision=precision, seed_base=5)
    out = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for mode in ("host", "device"):
            real = cs.Realisation(cs.SimConfig(**cfg, rng=mode), 0)
            for _ in range(3):  # per-step draws, then blocks between record steps
                real.step()
            obs = real.run()
            out[mode] = (real.pop.positions, real.pop.species, obs.msd, obs.counts,
                         real.rng_motion.bit_generator.state, real.rng_react.bit_generator.state)
    for a, b in zip(out["host"], out["device"]):
        if isinstance(a, dict):
            assert a == b
        else:
            assert np.array_equal(a, b)

"""Oracle pins of the colored-noise initialisation (reading R25)."""
import numpy as np
import pytest

from oracle import metamer as om
from oracle.jtfs import Oracle
from oracle.plan import response
from synth import CONFIGS, TINY, plan_args, batch, noise


def _profile(p, S):
    q = p.paths[1]
    rows = S[0, q.offset:q.offset + q.rows * q.frames].reshape(q.rows, q.frames)
    return np.interp(np.arange(p.N1) / p.F, np.arange(q.rows), np.sqrt((rows ** 2).mean(1)))


@pytest.mark.parametrize("name", ["spec", "c1"])
def test_expected_band_energy_matches_profile(name):
    # expectation over the white noise: E|y0 * psi_n1|^2 = (1/N_pad) sum_m G[m]^2 |psi_hat_n1[m]|^2,
    # so the mean scalogram is sqrt(pi/4) times its root: within 20% of a[n1] in every band
    cfg = {**CONFIGS, **TINY}[name]
    o = Oracle(plan_args(cfg))
    p = o.plan
    x = batch(name, 1) if name in CONFIGS else noise(p.N, 1, seed=3)
    S = o.forward(x, blocks=[]).numpy()
    a = _profile(p, S)
    # the spectral gain G of the definition (R25 steps 2-3)
    Np = p.N_pad
    psi2 = np.stack([np.abs(response(f, Np)) ** 2 for f in p.psi1])
    mirror = np.minimum(np.arange(Np), Np - np.arange(Np))
    den = psi2[:, mirror].sum(0)
    g = a / np.sqrt(np.pi / 4 * psi2.sum(1) / Np)
    G = (g[:, None] * psi2[:, mirror]).sum(0) / (den + 1e-3 * den.max())
    expected = np.sqrt(np.pi / 4 * (G[None, :] ** 2 * psi2).sum(1) / Np)
    assert np.all(np.abs(expected / a - 1) <= 0.2), expected / a
    # and colored_noise applies exactly that gain (a white input whose FFT is all ones)
    w = np.real(np.fft.ifft(np.ones(Np)))[None]
    y = om.colored_noise(p, S, w)
    ref = np.real(np.fft.ifft(G))[p.pad_left:p.pad_left + p.N]
    assert np.allclose(y[0], ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_band_limited_target_stays_in_band():
    # Sx of a band-limited x -> <= 5% of the initial energy outside the band. Holds at the
    # frequency resolution of the order-1 profile: F = 1 (no phi_F smoothing across bands); larger F
    # spreads the profile over ~1.6 F bands (R25)
    o = Oracle((8192, 8, 8, 3, 1, 64, 1))
    p = o.plan
    rng = np.random.default_rng(0)
    n = np.arange(p.N)
    x = 0.05 * sum(np.sin(2 * np.pi * f * n + rng.uniform(0, 6)) for f in rng.uniform(0.1, 0.15, 12))[None]
    S = o.forward(x, blocks=[]).numpy()
    y0 = om.colored_noise(p, S, rng.standard_normal((1, p.N_pad)))[0]
    P = np.abs(np.fft.rfft(y0)) ** 2
    fr = np.fft.rfftfreq(p.N)
    inband = (fr > 0.085) & (fr < 0.17)
    assert 1 - P[inband].sum() / P.sum() <= 0.05


def test_fallback_and_determinism():
    o = Oracle(plan_args(TINY["spec"]))
    p = o.plan
    w = np.random.default_rng(1).standard_normal((2, p.N_pad))
    y = om.colored_noise(p, np.zeros((2, p.n_coef)), w)
    assert np.array_equal(y, 1e-4 * w[:, p.pad_left:p.pad_left + p.N])
    S = o.forward(noise(p.N, 2, seed=4)).numpy()
    assert np.array_equal(om.colored_noise(p, S, w), om.colored_noise(p, S, w))

"""Oracle forward pins (CPU): independent direct-sum route, textbook identities, special inputs."""
import numpy as np
import pytest
import torch

from oracle import brute
from oracle.jtfs import Oracle, subsample_fourier, reflect_index
from oracle.plan import make_plan
from synth import CONFIGS, TINY, VARIANTS, plan_args, noise


def test_subsample_fourier_is_decimation():
    # SPEC S:69 / S:109 / S:529: ifft(subsample_fourier(fft(x), k)) == x[::k]
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal(64) + 1j * rng.standard_normal(64))
    for k in (1, 2, 4, 8):
        y = torch.fft.ifft(subsample_fourier(torch.fft.fft(x), k))
        assert torch.allclose(y, x[::k], atol=1e-12)
    # S:70 hand example
    X = torch.tensor([8.0, 0, 0, 0, 0, 0, 0, 0], dtype=torch.complex128)
    assert torch.equal(subsample_fourier(X, 2), torch.tensor([4.0, 0, 0, 0], dtype=torch.complex128))


def test_reflect_pad_example():
    # [1,2,3,4] padded to 8 -> [2,1,1,2,3,4,4,3]
    class P:  # minimal plan-like object
        N, N_pad, pad_left = 4, 8, 2
    idx = reflect_index(P)
    assert (torch.tensor([1., 2., 3., 4.])[idx]).tolist() == [2, 1, 1, 2, 3, 4, 4, 3]


@pytest.mark.parametrize("name", ["t1", "t2", "spec", "q2", "j2gtT"])
def test_fft_route_equals_direct_sums(name):
    # brute.py: O(L^2) direct circular sums with closed-form kernels, depth-first, no FFT; also on the
    # plan variants Q2 = 2 and j2 > log2 T (R13)
    p = make_plan(*plan_args({**TINY, **VARIANTS}[name]))
    x = noise(p.N, 1, seed=11)
    So = Oracle(p).forward(x)[0].numpy()
    Sb = brute.forward(p, x[0])
    assert np.linalg.norm(So - Sb) <= 1e-12 * np.linalg.norm(So)


def test_zero_in_zero_out():
    p = make_plan(*plan_args(TINY["t2"]))
    S = Oracle(p).forward(np.zeros((1, p.N), np.float32))
    assert torch.count_nonzero(S) == 0


def test_positive_homogeneity():
    # orders 1, 2 pass through a modulus: S(a x) = |a| S(x); S0 is linear: S0(a x) = a S0(x)
    p = make_plan(*plan_args(TINY["spec"]))
    o = Oracle(p)
    x = noise(p.N, 1, seed=5).astype(np.float64)
    S1 = o.forward(x)
    S2 = o.forward(-3.0 * x)
    nf = p.frames
    assert torch.allclose(S2[:, nf:], 3.0 * S1[:, nf:], rtol=1e-12, atol=1e-15)
    assert torch.allclose(S2[:, :nf], -3.0 * S1[:, :nf], rtol=1e-12, atol=1e-15)


def test_constant_along_lambda_killed_by_bandpass():
    # a constant along n1 (full frequential circle) has zero band-pass output,
    # because kappa nulls every Morlet's DC bin (Eq.1)
    p = make_plan(*plan_args(CONFIGS["c1"]))
    o = Oracle(p)
    X = torch.ones(1, p.P, 16, dtype=torch.complex128)
    Xh = torch.fft.fft(X, dim=1)
    for f in range(1, len(p.L_fr)):
        assert o._freq_filter(Xh, f).abs().max() < 1e-13
    assert torch.allclose(o._freq_filter(Xh, 0).real, torch.ones(1, p.P // p.F, 16, dtype=torch.float64))


@pytest.mark.parametrize("k", [3, 12, 20])
def test_sinusoid_scalogram_row(k):
    # R5 normalisation + SPEC S:247: unit cosine at xi(psi1[k]) -> S1 time average of row k ~ 1
    # and row k is the argmax over rows
    p = make_plan(*plan_args(CONFIGS["c1"]))
    o = Oracle(p)
    n = np.arange(p.N)
    x = np.cos(2 * np.pi * p.psi1[k].xi * n)[None]
    _, _, S1t = o.layer1(torch.from_numpy(x))
    f0 = p.pad_left // p.T
    prof = S1t[0, :, f0 + 8: f0 + p.frames - 8].mean(dim=1).numpy()
    assert int(np.argmax(prof)) == k
    assert abs(prof[k] - 1.0) < 0.02


def _tone(N, f0, sr, shift=0.0):
    n = np.arange(N) - shift
    x = sum(np.sin(2 * np.pi * h * f0 * n / sr) / h for h in range(1, 9) if h * f0 < sr / 2)
    env = np.exp(-((n - N / 2) / (N / 4)) ** 2)
    return (0.5 * x * env)[None]


def test_shift_invariance_envelope():
    # P:46, P:100 (invariance to shifts below T); SPEC S:275 envelope: <= 0.1 at tau = T/8,
    # larger shifts change more (on average)
    p = make_plan(*plan_args(CONFIGS["c1"]))
    o = Oracle(p)
    S = o.forward(_tone(p.N, 220.0, 22050.0))
    d = []
    for tau in (p.T / 8, p.T / 2, 2 * p.T):
        St = o.forward(_tone(p.N, 220.0, 22050.0, shift=tau))
        d.append(float((St - S).norm() / S.norm()))
    assert d[0] <= 0.1
    assert d[0] < d[1] < d[2]


def test_transposition_envelope():
    # P:46-48 (transpositions below F): +1-bin (1/Q octave) transposition of a harmonic tone
    # changes order-1 coefficients by <= 0.15
    p = make_plan(*plan_args(CONFIGS["c1"]))
    o = Oracle(p)
    f0 = 220.0
    S = o.forward(_tone(p.N, f0, 22050.0))
    St = o.forward(_tone(p.N, f0 * 2 ** (1 / p.Q), 22050.0))
    o1 = slice(p.frames, p.paths[1 + p.n_fr_order1].offset)
    assert float((St[:, o1] - S[:, o1]).norm() / S[:, o1].norm()) <= 0.15


def test_chunked_equals_unchunked():
    p = make_plan(*plan_args(CONFIGS["c1"]))
    x = noise(p.N, 1, seed=2)
    a = Oracle(p).forward(x)
    b = Oracle(p, chunk_elems=1 << 14).forward(x)
    assert torch.allclose(a, b, rtol=0, atol=1e-15)

"""Oracle gradient and metamer-step pins (CPU)."""
import numpy as np
import pytest
import torch

import oracle.jtfs as OJ
from oracle import brute, metamer
from oracle.jtfs import Oracle
from oracle.plan import make_plan
from synth import TINY, CONFIGS, plan_args, noise


def _silent(y: np.ndarray) -> np.ndarray:
    """y with an exactly silent stretch (the second quarter zeroed)."""
    ys = np.array(y, dtype=np.float64, copy=True)
    N = ys.shape[-1]
    ys[..., N // 4:N // 2] = 0.0
    return ys


@pytest.mark.parametrize("name", ["t1", "t2", "spec"])
@pytest.mark.parametrize("silent", [False, True], ids=["noise", "silent"])
def test_gradient_two_routes(name, silent):
    # Independent routes to dE/dy: brute.loss_grad reverses the direct-sum forward
    # with hand-written adjoints (conjugate-transpose matrices, explicit pad adjoint, no FFT, no
    # autodiff); Oracle.loss_grad is autograd through the FFT route. With an exactly
    # silent stretch the phases of rounding-noise cells would differ between the two routes; the R22
    # dead zone (|z| < 1e-12 RMS) gives them one definition.
    p = make_plan(*plan_args(TINY[name]))
    o = Oracle(p)
    x = noise(p.N, 1, seed=21).astype(np.float64)
    y = noise(p.N, 1, seed=22).astype(np.float64)
    if silent:
        y = _silent(y)
    St = o.forward(x)
    E, g = o.loss_grad(y, St)
    Eb, gb = brute.loss_grad(p, y[0], St[0].numpy())
    assert abs(Eb - float(E[0])) <= 1e-12 * float(E[0])
    # silent: cells just above the 1e-12 RMS radius keep only ~4 digits of phase in either route
    # (float64 rounding ~1e-16 of the signal scale), so the routes agree to ~1e-6 there, not 1e-9
    tol = 1e-5 if silent else 1e-9
    assert np.linalg.norm(gb - g[0].numpy()) <= tol * np.linalg.norm(gb)


def test_dead_zone_inactive_on_generic_inputs():
    # R22: the dead zone sits at the rounding floor; on a generic input no modulus input lies in it,
    # so the gradient equals the exact-phase (torch.sgn) gradient to rounding
    p = make_plan(*plan_args(TINY["spec"]))
    o = Oracle(p)
    x, y = noise(p.N, 2, seed=31), noise(p.N, 2, seed=32)
    St = o.forward(x)
    _, g = o.loss_grad(y, St)
    eps = OJ.EPS_MOD
    try:
        OJ.EPS_MOD = 0.0
        _, g0 = o.loss_grad(y, St)
    finally:
        OJ.EPS_MOD = eps
    assert float((g - g0).norm()) <= 1e-13 * float(g.norm())


def test_dead_zone_effect_at_baseline_configs():
    # The measured effect of the R22 dead zone on the float64 gradient at the BASELINE configs
    # (tests/golden/r22_effect.json, written by tools/r22_effect.py, which calls only oracle/):
    # |g(EPS_MOD = 1e-12) - g(EPS_MOD = 0)| / |g| <= 1e-5 on every recorded case.
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "r22_effect.json")
    rec = json.load(open(path))
    assert {"c2:all", "c4:0", "c4:11", "c5:11"} <= set(rec["cases"])
    for case, v in rec["cases"].items():
        assert v["rel_effect"] <= 1e-5, (case, v)


@pytest.mark.parametrize("name", ["t1", "t2", "spec"])
def test_gradient_finite_differences(name):
    # SPEC S:362 / S:526: directional derivative vs central differences along 100 random
    # directions, >= 99% within 1e-4 (best of h in {1e-4, 1e-5, 1e-6} * |y|); the perturbed
    # signals of all directions run as one batch through the oracle
    p = make_plan(*plan_args(TINY[name]))
    o = Oracle(p)
    x = noise(p.N, 1, seed=21).astype(np.float64)
    y = noise(p.N, 1, seed=22).astype(np.float64)
    St = o.forward(x)
    E, g = o.loss_grad(y, St)
    rng = np.random.default_rng(3)
    nd = 100
    D = rng.standard_normal((nd, p.N))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    dd = D @ g[0].numpy()
    best = np.full(nd, np.inf)
    for h in (1e-4, 1e-5, 1e-6):
        hs = h * np.linalg.norm(y)
        Ep = o.loss(o.forward(y + hs * D), St.expand(nd, -1)).numpy()
        Em = o.loss(o.forward(y - hs * D), St.expand(nd, -1)).numpy()
        fd = (Ep - Em) / (2 * hs)
        best = np.minimum(best, np.abs(fd - dd) / np.maximum(np.abs(dd), 1e-12))
    assert (best <= 1e-4).sum() >= 99


def test_adjoint_dot_products():
    # SPEC "Invariants": <A u, v> = <u, A^H v> within 1e-10 for every linear stage of the explicit
    # backward: decimating circular convolutions along time and along rows (filters + subsampling,
    # complex kernels), the reflect padding, and the order-2 crop/zero-fill pair
    rng = np.random.default_rng(5)
    p = make_plan(*plan_args(TINY["spec"]))
    cplx = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    ip = lambda a, b: np.vdot(b, a)           # <a, b> = sum a conj(b)
    from oracle.plan import time_kernel_closed_form as tk
    for flt, L0, k, s in [(p.psi1[3], p.N_pad, 0, 2), (p.psi2[4], p.N_pad, 1, 4), (p.phiT, p.N_pad, 2, 2),
                          (p.L_fr[2], p.P, 0, 1), (p.L_fr[-1], p.P, 0, 2), (p.phiF, p.P, 1, 2)]:
        h = tk(flt, L0, k)
        L = h.shape[0]
        u, v = cplx(3, L), cplx(3, L // s)
        assert abs(ip(brute._circ(h, u, s), v) - ip(u, brute._circ_adj(h, v, s))) <= 1e-10 * abs(ip(u, u))
        U, V = cplx(L, 5), cplx(L // s, 5)
        lhs = ip(brute._circ_rows(h, U, s), V)
        assert abs(lhs - ip(U, brute._circ_rows_adj(h, V, s))) <= 1e-10 * abs(ip(U, U))
    x, gp = rng.standard_normal(p.N), rng.standard_normal(p.N_pad)
    assert abs(ip(brute._reflect(p, x), gp) - ip(x, brute._reflect_adj(p, gp))) <= 1e-10 * np.dot(gp, gp)


def test_nullity_at_metamer():
    # the gradient vanishes if S1x = S1y and S2x = S2y (here y = x exactly)
    p = make_plan(*plan_args(TINY["spec"]))
    o = Oracle(p)
    x = noise(p.N, 2, seed=4)
    E, g = o.loss_grad(x, o.forward(x))
    assert torch.count_nonzero(E) == 0 and torch.count_nonzero(g) == 0


def test_descent_property():
    # a small step along -g decreases E
    p = make_plan(*plan_args(TINY["t2"]))
    o = Oracle(p)
    x, y = noise(p.N, 1, seed=7), noise(p.N, 1, seed=8)
    St = o.forward(x)
    E, g = o.loss_grad(y, St)
    yn = torch.from_numpy(y.astype(np.float64))
    for eps in (1e-3, 1e-4):
        step = eps * yn.norm() / g.norm()
        assert float(o.loss(o.forward(yn - step * g), St)) < float(E)


def test_loss_excludes_order0_and_is_half_squared():
    # R19: E = 1/2 sum over orders 1, 2; S0 excluded (Sy = 0 -> E = 1/2 |Sx|^2)
    p = make_plan(*plan_args(TINY["t1"]))
    o = Oracle(p)
    S = o.forward(noise(p.N, 1, seed=1))
    E = o.loss(torch.zeros_like(S), S)
    assert torch.allclose(E, 0.5 * (S[:, p.frames:] ** 2).sum(1), rtol=1e-15)


# ---------------------------------------------------------------- metamer step

def test_metamer_accept_reject_rules():
    st = metamer.init_state(np.ones((2, 4)))
    g = np.full((2, 4), 0.5)
    s1 = metamer.step(st, np.array([1.0, 1.0]), g)
    assert np.all(s1["accepted"] == 1)
    assert np.allclose(s1["mu"], 0.11)                       # mu0 * 1.1
    assert np.allclose(s1["y"], 1 - 0.11 * 0.5)
    # signal 0 improves, signal 1 gets worse -> rejected: y restored bitwise, mu halves exactly
    s2 = metamer.step(s1, np.array([0.5, 2.0]), np.full((2, 4), 0.25))
    assert s2["accepted"].tolist() == [1, 0]
    assert s2["mu"][1] == 0.5 * s1["mu"][1]
    # rejected signal restarts from y_prev with u = 0 and the stored gradient
    assert np.array_equal(s2["y"][1], s1["y_prev"][1] - s2["mu"][1] * s1["g_prev"][1])
    assert np.array_equal(s2["y_prev"][1], s1["y_prev"][1])


def test_metamer_quadratic_toy_converges():
    # on E = 1/2 |y - c|^2 the iterates converge to c
    c = np.linspace(-1, 1, 16)[None]
    st = metamer.init_state(np.zeros((1, 16)))
    for _ in range(200):
        E = 0.5 * ((st["y"] - c) ** 2).sum(1)
        st = metamer.step(st, E, st["y"] - c)
    assert np.abs(st["y"] - c).max() < 1e-6


def test_c1_direct_sums_equal_fft_autograd():
    # BASELINE configs[0] (c1) by the independent route: direct sums over the closed-form kernels' taps
    # and explicit adjoints (oracle/brute.py, no FFT, no autodiff) vs the FFT + autograd oracle, on the
    # c1 music input; the loss restricted to order 1 + block 0 bounds the time (~30 s)
    from synth import batch
    p = make_plan(*plan_args(CONFIGS["c1"]))
    o = Oracle(p)
    x = batch("c1", 1).astype(np.float64)
    y = batch("c1", 1, which="y").astype(np.float64)
    St = o.forward(x)
    Sb = brute.forward(p, x[0], blocks=[0])
    So = o.forward(x, blocks=[0])[0].numpy()
    assert np.linalg.norm(Sb - So) <= 1e-12 * np.linalg.norm(So)
    Eb, gb = brute.loss_grad(p, y[0], St[0].numpy(), blocks=[0])
    E, g = o.loss_grad_subset(y, St, [0])
    assert abs(Eb - float(E[0])) <= 1e-12 * float(E[0])
    assert np.linalg.norm(gb - g[0].numpy()) <= 1e-10 * np.linalg.norm(gb)

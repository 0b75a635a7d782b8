"""Oracle gradient and metamer-step pins (CPU)."""
import numpy as np
import pytest
import torch

from oracle import metamer
from oracle.jtfs import Oracle
from oracle.plan import make_plan
from synth import TINY, CONFIGS, plan_args, noise


@pytest.mark.parametrize("name", ["t1", "t2", "spec"])
def test_gradient_finite_differences(name):
    # SPEC S:362 / S:526: directional derivative vs central differences, >= 99% within 1e-4
    p = make_plan(*plan_args(TINY[name]))
    o = Oracle(p)
    x = noise(p.N, 1, seed=21).astype(np.float64)
    y = noise(p.N, 1, seed=22).astype(np.float64)
    St = o.forward(x)
    E, g = o.loss_grad(y, St)
    rng = np.random.default_rng(3)
    ok = 0
    nd = 12
    for _ in range(nd):
        d = rng.standard_normal(y.shape)
        d /= np.linalg.norm(d)
        dd = float((g.numpy() * d).sum())
        best = np.inf
        for h in (1e-4, 1e-5, 1e-6):
            hs = h * np.linalg.norm(y)
            Ep = o.loss(o.forward(y + hs * d), St)
            Em = o.loss(o.forward(y - hs * d), St)
            fd = float((Ep - Em).sum() / (2 * hs))
            best = min(best, abs(fd - dd) / max(abs(dd), 1e-12))
        ok += best <= 1e-4
    assert ok >= nd - 0 if nd < 100 else ok >= 0.99 * nd


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

"""Oracle planner / filterbank pins (CPU). Each test names what pins it."""
import math
from collections import Counter

import numpy as np
import pytest

from oracle import plan as op
from synth import CONFIGS, TINY, plan_args


# ---------------------------------------------------------------- generator

def test_generator_q1_first_xi():
    # xi = max(1/(1+2^(3/Q)), 0.35) -> 0.35 for Q = 1 (SPEC S:160 evaluates it by hand)
    assert op.anden_generator(8, 1)[0][0] == 0.35


def test_generator_q8_first_filter_closed_form():
    # P:171-173 by hand: xi0 = 1/(1+2^(3/8)); sigma0 = (1-2^-1/8)/(1+2^-1/8) xi0 / sqrt(ln 2)
    xi0, s0 = op.anden_generator(6, 8)[0]
    assert abs(xi0 - 1 / (1 + 2 ** 0.375)) < 1e-16
    f = 2 ** (-1 / 8)
    assert abs(s0 - (1 - f) / (1 + f) * xi0 / math.sqrt(math.log(2))) < 1e-16
    assert round(xi0, 5) == 0.43538 and round(s0, 6) == 0.022641


def test_generator_geometric_and_tail():
    # ratio 2^(-1/8), xi/sigma constant, tail sigma = 0.1 * 2^-J exactly
    J, Q = 8, 8
    fl = op.anden_generator(J, Q)
    smin = 0.1 / 2 ** J
    geo = [(x, s) for x, s in fl if s != smin]
    tail = [(x, s) for x, s in fl if s == smin]
    assert len(tail) == Q - 1
    for (x0, s0), (x1, s1) in zip(geo, geo[1:]):
        assert abs(x1 / x0 - 2 ** (-1 / Q)) < 1e-14
        assert abs(s1 / s0 - 2 ** (-1 / Q)) < 1e-14
    qs = [x / s for x, s in geo]
    assert max(qs) / min(qs) - 1 < 1e-12
    assert geo[-1][1] > smin
    # arithmetic tail: equal steps of elbow_xi / Q
    el = geo[-1][0]
    for q, (x, _) in enumerate(tail):
        assert abs(x - el * (1 - (q + 1) / Q)) < 1e-15


def test_spin_doubles():
    fl = op.anden_generator(3, 1)
    sp = op.spin(fl)
    assert len(sp) == 2 * len(fl)
    assert [np.sign(x) for x, _ in sp] == [1] * len(fl) + [-1] * len(fl)


# ---------------------------------------------------------------- plan table

TABLE = {  # independent scratch evaluation in SURVEY.md §8.0 / Appendix A
    "c1": dict(N_pad=8192, pad_left=2048, N1=38, jc=[10, 8, 8, 7, 4, 1], P=256,
               n1_max=[10, 18, 26, 33], jfr=[0, 0, 0, 1], o1=5, o2=36, coef=9664),
    "c2": dict(N_pad=131072, pad_left=32768, N1=159, P=1024,
               n1_max=[18, 34, 50, 66, 82, 98, 114, 130, 145, 153],
               jfr=[0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4], o1=12, o2=230, coef=50944),
    "c3": dict(N_pad=262144, pad_left=65536, N1=136, P=512,
               n1_max=[14, 26, 38, 50, 62, 74, 86, 98, 110, 122, 130],
               jfr=[0, 0, 0, 1, 2, 3], o1=7, o2=143, coef=48320),
    "c4": dict(N_pad=524288, pad_left=131072, N1=191, P=1024,
               n1_max=[18, 34, 50, 66, 82, 98, 114, 130, 146, 162, 177, 185],
               jfr=[0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5], o1=14, o2=324, coef=82272),
    "c5": dict(N_pad=2097152, pad_left=524288, N1=191, P=1024,
               n1_max=[18, 34, 50, 66, 82, 98, 114, 130, 146, 162, 177, 185],
               jfr=[0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5], o1=14, o2=324, coef=86592),
    "t1": dict(N_pad=256, pad_left=64, N1=4, P=64, n1_max=[3], jfr=[0, 0, 0]),
    "t2": dict(N_pad=512, pad_left=128, N1=9, P=64, n1_max=[4, 6], jfr=[0, 0, 0]),
    "spec": dict(N_pad=2048, pad_left=512, N1=11, P=128, n1_max=[4, 6, 8], jfr=[0, 0, 0, 1]),
}


@pytest.mark.parametrize("name", list(TABLE))
def test_plan_table(name):
    cfg = {**CONFIGS, **TINY}[name]
    p = op.make_plan(*plan_args(cfg))
    t = TABLE[name]
    assert p.N_pad == t["N_pad"] and p.pad_left == t["pad_left"]
    assert p.N1 == t["N1"] and p.P == t["P"]
    assert [b.n1_max for b in p.blocks] == t["n1_max"]
    assert [f.j for f in p.psi_fr_plus] == t["jfr"]
    if "jc" in t:
        c = Counter(f.j for f in p.psi1)
        assert [c[j] for j in range(max(c) + 1)] == t["jc"]
    if "o1" in t:
        assert sum(q.order == 1 for q in p.paths) == t["o1"]
        assert sum(q.order == 2 for q in p.paths) == t["o2"]
        assert p.n_coef - p.frames == t["coef"]
    # strides: s2 = j2 for every block at these configs (SURVEY §8.0 observation)
    assert all(b.s2 == min(b.j2, p.log2T) for b in p.blocks)
    # j2 = max(q - 2, 0) for psi2 index q (reading R3 closed form)
    assert [f.j for f in p.psi2] == [max(q - 2, 0) for q in range(len(p.psi2))]


def test_plan_config_errors():
    with pytest.raises(op.PlanError, match="T must be a power of two"):
        op.make_plan(4096, 6, 8, 3, 1, 48, 8)
    with pytest.raises(op.PlanError, match="log2"):
        op.make_plan(4096, 6, 8, 3, 1, 128, 8)
    with pytest.raises(op.PlanError, match="multiple of T"):
        op.make_plan(4000, 6, 8, 3, 1, 64, 8)
    with pytest.raises(op.PlanError, match="J_fr"):
        op.make_plan(4096, 6, 8, 0, 1, 64, 8)


def test_width_first_admissible_set():
    # P:231 `if j2 > j1`: the block rows are exactly {n1 : j1 < j2} and form a prefix
    p = op.make_plan(*plan_args(CONFIGS["c2"]))
    for b in p.blocks:
        adm = [n1 for n1, f in enumerate(p.psi1) if b.j2 > f.j]
        assert adm == list(range(b.n1_max))
    assert all(b.n1_max > 0 for b in p.blocks)      # empty blocks omitted


# ---------------------------------------------------------------- Morlet, kappa (Eq.1)

@pytest.mark.parametrize("name", ["c1", "c2", "c4", "t1", "spec"])
def test_vanishing_moment(name):
    # the level-0 DC bin does not depend on the grid length: check it on a short grid
    p = op.make_plan(*plan_args({**CONFIGS, **TINY}[name]))
    for flt in p.psi1 + p.psi2 + p.L_fr[1:]:
        r = op.response(flt, 64)
        peak = np.abs(op.response(flt, 4096)).max()
        assert abs(r[0]) <= 1e-15 * peak


def test_response_normalisation():
    # R5: Gaussian peak 2 for psi (kappa ~ 0 for a narrow high-Q filter), phi_hat(0) = 1
    p = op.make_plan(*plan_args(CONFIGS["c2"]))
    f = p.psi1[0]
    r = op.response(f, 1 << 16)
    assert abs(r.max() - 2.0) < 1e-3
    assert abs(op.response(p.phiT, 1 << 16)[0] - 1.0) < 1e-12
    # spin: negated xi mirrors the response, psi_-(w) = psi_+(-w)
    g = p.L_fr[1]
    gm = p.L_fr[1 + len(p.psi_fr_plus)]
    a, b = op.response(g, 256), op.response(gm, 256)
    assert np.allclose(a, np.roll(b[::-1], 1), atol=1e-14)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_littlewood_paley(name):
    # SURVEY §8(c) pins: max <= 2.3; min >= 0.45 on [sigma_min, xi0]; max/min <= 1.2 on constant-Q
    p = op.make_plan(*plan_args(CONFIGS[name]))
    L = p.N_pad
    lp = np.abs(op.response(p.phiT, L)) ** 2
    for f in p.psi1:
        r = op.response(f, L)
        lp += 0.5 * (r ** 2 + np.roll(r[::-1], 1) ** 2)
    w = np.arange(L) / L
    xi0 = p.psi1[0].xi
    smin = 0.1 / 2 ** p.J
    band = (w >= smin) & (w <= xi0)
    assert lp[w <= 0.5].max() <= 2.3
    assert lp[band].min() >= 0.45
    cq = [f for f in p.psi1 if f.sigma > smin]
    cq_band = (w >= cq[-1].xi) & (w <= xi0)
    assert lp[cq_band].max() / lp[cq_band].min() <= 1.2


# ---------------------------------------------------------------- closed-form kernels (O1, R9)

@pytest.mark.parametrize("L0,k", [(256, 0), (256, 2), (1024, 1), (4096, 3)])
def test_closed_form_kernel_equals_idft(L0, k):
    # two independent routes: Poisson-summed continuous kernel vs O(L^2) inverse DFT of the
    # fold-summed sampled response
    p = op.make_plan(*plan_args(TINY["spec"]))
    for flt in [p.psi1[0], p.psi1[-1], p.psi2[3], p.phiT, p.L_fr[2], p.L_fr[-1], p.phiF]:
        hk = op.level(op.response(flt, L0), k)
        L = hk.shape[0]
        n = np.arange(L)
        idft = (np.exp(2j * np.pi * np.outer(n, n) / L) @ hk) / L
        cf = op.time_kernel_closed_form(flt, L0, k)
        assert np.abs(idft - cf).max() <= 1e-13 * max(1.0, np.abs(cf).max())


def test_level_fold_sum_dc_gain():
    # R9: fold-SUM keeps phi's DC gain 1 at every level
    p = op.make_plan(*plan_args(CONFIGS["c1"]))
    r = op.response(p.phiT, p.N_pad)
    for k in range(p.log2T + 1):
        assert abs(op.level(r, k)[0] - 1.0) < 1e-12

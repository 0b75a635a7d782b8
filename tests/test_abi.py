"""C-ABI library on CPU: loads, exports every symbol of include/jtfs.h, and its host-side planner
agrees with the oracle planner (no compute calls: no GPU here)."""
import numpy as np
import pytest

from oracle import plan as op
from synth import CONFIGS, TINY, VARIANTS, plan_args

ALL = {**CONFIGS, **TINY, **VARIANTS}


@pytest.fixture(scope="module")
def jt():
    from paper_2602_11896_b200 import jtfs
    return jtfs


def test_exports_every_header_symbol(lib):
    from paper_2602_11896_b200 import _lib
    syms = _lib.header_symbols()
    assert "jtfs_forward" in syms and "metamer_step" in syms and "jtfs_loss_grad" in syms
    for s in syms:
        assert hasattr(lib, s), s


@pytest.mark.parametrize("name", list(ALL))
def test_plan_tables_equal_oracle(jt, name):
    args = plan_args(ALL[name])
    p = jt.Plan(*args)
    o = op.make_plan(*args)
    i = p.info
    assert (i.N, i.N_pad, i.pad_left, i.P, i.frames, i.n_coef) == (o.N, o.N_pad, o.pad_left, o.P, o.frames, o.n_coef)
    assert (i.N1, i.N2, i.N_fr, i.n_blocks) == (o.N1, len(o.psi2), len(o.psi_fr_plus), len(o.blocks))
    pa = p.paths()
    assert len(pa) == len(o.paths)
    for a, b in zip(pa, o.paths):
        assert (a["order"], a["n_fr"], a["spin"], a["rows"], a["frames"], a["offset"]) == \
               (b.order, b.n_fr, b.spin, b.rows, b.frames, b.offset)
        if b.order == 2:
            assert (a["n2"], a["j2"], a["j_fr"]) == (b.n2, b.j2, b.j_fr)
    for layer, bank in [(0, o.psi1), (1, o.psi2), (2, o.L_fr)]:
        f = p.filters(layer)
        assert np.array_equal(f["xi"], [q.xi for q in bank])          # bitwise: same listing, same order
        assert np.array_equal(f["sigma"], [q.sigma for q in bank])
        assert list(f["j"]) == [q.j for q in bank]


@pytest.mark.parametrize("name", ["t2", "spec", "c1"])
def test_level_responses_equal_oracle(jt, name):
    args = plan_args(ALL[name])
    p = jt.Plan(*args)
    o = op.make_plan(*args)
    cases = [(0, 0, 0, o.psi1[0], o.N_pad), (0, o.N1 - 1, 0, o.psi1[-1], o.N_pad), (1, 3, 1, o.psi2[3], o.N_pad),
             (3, 0, o.log2T, o.phiT, o.N_pad), (3, 0, 1, o.phiT, o.N_pad), (2, 1, 0, o.L_fr[1], o.P),
             (2, len(o.L_fr) - 1, 0, o.L_fr[-1], o.P), (4, 0, o.log2F, o.phiF, o.P)]
    for layer, idx, k, flt, L0 in cases:
        a = p.response(layer, idx, k)
        b = op.level(op.response(flt, L0), k)
        assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(b).max()), (layer, idx, k)


def test_config_errors(jt):
    from paper_2602_11896_b200._lib import JtfsError
    with pytest.raises(JtfsError, match="T must be a power of two"):
        jt.Plan(4096, 6, 8, 3, 1, 48, 8)
    with pytest.raises(JtfsError, match="log2"):
        jt.Plan(4096, 6, 8, 3, 1, 128, 8)
    with pytest.raises(JtfsError, match="JTFS_ERR_CONFIG"):
        jt.Plan(4000, 6, 8, 3, 1, 64, 8)


def test_workspace_affine(jt):
    p = jt.Plan(*plan_args(CONFIGS["c1"]))
    w1, w2, w5 = (p.workspace_size(b, True) for b in (1, 2, 5))
    assert w2 - w1 == w1 and w5 == 5 * w1
    assert p.workspace_size(1, True) >= p.workspace_size(1, False)


def test_q2_filterbank():
    # Q2 = Q^{tm,2}: the second-layer bank is the generator at Q2 (more blocks, same rules)
    for name in ("q2", "q2b"):
        o = op.make_plan(*plan_args(VARIANTS[name]))
        assert len(o.psi2) > len(op.make_plan(*plan_args(VARIANTS[name])[:7]).psi2)
        assert all(b.n1_max == sum(1 for f in o.psi1 if f.j < b.j2) for b in o.blocks)

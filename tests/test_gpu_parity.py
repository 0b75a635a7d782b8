"""GPU parity: the CUDA path through the C ABI vs the float64 oracle, element by element.
Bars (BASELINE.json north_star): rel-L2 <= 1e-4 on coefficients, <= 1e-3 on gradients."""
import numpy as np
import pytest
import torch

from oracle.jtfs import Oracle
from oracle import metamer as om
from synth import CONFIGS, TINY, VARIANTS, plan_args, noise, batch

pytestmark = pytest.mark.gpu
ALL = {**CONFIGS, **TINY, **VARIANTS}


def rel(a, b):
    a = np.asarray(a).astype(np.complex128 if np.iscomplexobj(a) or np.iscomplexobj(b) else np.float64)
    b = np.asarray(b).astype(a.dtype)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def plans():
    from paper_2602_11896_b200 import Plan
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Plan(*plan_args(ALL[name]))
        return cache[name]
    return get


def inputs(name, B=2):
    cfg = ALL[name]
    if name in TINY or name in VARIANTS:
        return noise(cfg["N"], B, seed=31), noise(cfg["N"], B, seed=32)
    return batch(name, B), batch(name, B, which="y")


@pytest.mark.parametrize("name", ["t1", "t2", "spec", "c1"])
def test_stage_U1_S1t_Y2(plans, name):
    p = plans(name)
    o = Oracle(plan_args(ALL[name]))
    x, _ = inputs(name)
    xd = torch.from_numpy(x).cuda()
    S0, U1h, S1t = o.layer1(torch.from_numpy(x).double())
    U1 = torch.cat([torch.fft.ifft(u).real for u in U1h], dim=1).numpy()
    g1 = p.debug_stage(1, xd).cpu().numpy()
    assert rel(g1, U1) <= 1e-5
    g2 = p.debug_stage(2, xd).cpu().numpy()
    assert rel(g2, S1t.numpy()) <= 1e-5
    if o.plan.blocks:
        g3 = p.debug_stage(3, xd).cpu().numpy()
        Y2 = torch.cat([o.layer2_block(U1h, bi).reshape(x.shape[0], -1) for bi in range(len(o.plan.blocks))],
                       dim=1).numpy()
        assert rel(g3, Y2) <= 1e-5


@pytest.mark.parametrize("name", ["t1", "t2", "spec", "c1", "q2", "q2b", "j2gtT", "wide"])
def test_forward_parity(plans, name):
    p = plans(name)
    o = Oracle(plan_args(ALL[name]))
    x, _ = inputs(name)
    S = p.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    So = o.forward(x).numpy()
    assert rel(S, So) <= 1e-4
    # every path individually (the small ones too)
    for q in o.plan.paths:
        sl = slice(q.offset, q.offset + q.rows * q.frames)
        assert rel(S[:, sl], So[:, sl]) <= 1e-3, q


@pytest.mark.parametrize("name", ["t1", "t2", "spec", "c1", "q2", "q2b", "j2gtT", "wide"])
def test_loss_grad_parity(plans, name):
    p = plans(name)
    o = Oracle(plan_args(ALL[name]))
    x, y = inputs(name)
    So = o.forward(x)
    Eo, go = o.loss_grad(y, So)
    St = torch.from_numpy(So.numpy().astype(np.float32)).cuda()
    loss, g = p.loss_grad(torch.from_numpy(y).cuda(), St)
    assert rel(loss.cpu().numpy(), Eo.numpy()) <= 1e-4
    assert rel(g.cpu().numpy(), go.numpy()) <= 1e-3


def test_nullity_and_determinism(plans):
    p = plans("spec")
    x, _ = inputs("spec")
    xd = torch.from_numpy(x).cuda()
    S = p.forward(xd)
    S2 = p.forward(xd)
    assert torch.equal(S, S2)
    loss, g = p.loss_grad(xd, S)
    assert float(loss.abs().max()) == 0.0 and float(g.abs().max()) == 0.0
    l1, g1 = p.loss_grad(xd * 0.5, S)
    l2, g2 = p.loss_grad(xd * 0.5, S)
    assert torch.equal(g1, g2) and torch.equal(l1, l2)


def test_microbatch_and_shards_sum(plans):
    p = plans("c1")
    x, y = inputs("c1", B=3)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    S = p.forward(xd)
    loss, g = p.loss_grad(yd, S)
    # micro-batch of one signal through a minimal workspace: bitwise the same per signal
    ws = torch.empty(p.workspace_size(1, True), dtype=torch.uint8, device="cuda")
    l1, g1 = p.loss_grad(yd, S, ws=ws)
    assert torch.equal(g1, g) and torch.equal(l1, loss)
    # path shards (whole blocks, jtfs_plan_shards) sum to the whole. The loss partials are float64 sums of
    # disjoint coefficient sets (1e-6); each shard's gradient runs the fp32 adjoint chain (FFTs, gathers)
    # on its own partial spectra, so the sum of shards differs from the one-shot gradient by fp32 rounding
    # of those transforms (measured ~1e-6; bar 1e-5)
    ls, gs = 0, 0
    for sh in range(3):
        l_, g_ = p.loss_grad(yd, S, shard=sh, n_shards=3)
        ls, gs = ls + l_, gs + g_
    assert rel(gs.cpu().numpy(), g.cpu().numpy()) <= 1e-5
    assert rel(ls.cpu().numpy(), loss.cpu().numpy()) <= 1e-6


def test_metamer_step_parity(plans):
    name = "t2"
    p = plans(name)
    o = Oracle(plan_args(ALL[name]))
    x, y = inputs(name)
    So = o.forward(x)
    St = torch.from_numpy(So.numpy().astype(np.float32)).cuda()
    st = p.metamer_state(torch.from_numpy(y).cuda())
    ost = om.init_state(y)
    for it in range(4):
        E, g = o.loss_grad(ost["y"], So)
        ost = om.step(ost, E.numpy(), g.numpy())
        p.metamer_step(st, St)
        torch.cuda.synchronize()
        assert st["accepted"].cpu().tolist() == ost["accepted"].tolist()
        assert rel(st["mu"].cpu().numpy(), ost["mu"]) <= 1e-6
        # compare the accumulated update y - y0 (the quantity the step computes)
        assert rel(st["y"].cpu().numpy() - y, ost["y"] - y) <= 1e-3, it


def test_loss_report(plans):
    # NEXT-2: per-path losses; orders 1 + 2 sum to the loss of jtfs_loss_grad (R19)
    name = "c1"
    p = plans(name)
    o = Oracle(plan_args(ALL[name]))
    x, y = inputs(name)
    St = p.forward(torch.from_numpy(x).cuda())
    Sy = p.forward(torch.from_numpy(y).cuda())
    rep = p.loss_report(Sy, St).cpu().numpy().astype(np.float64)
    r = Sy.cpu().numpy().astype(np.float64) - St.cpu().numpy().astype(np.float64)
    ref = np.stack([[0.5 * np.sum(r[b, q.offset:q.offset + q.rows * q.frames] ** 2) for q in o.plan.paths]
                    for b in range(r.shape[0])])
    assert rel(rep, ref) <= 1e-6
    loss, _ = p.loss_grad(torch.from_numpy(y).cuda(), St)
    assert rel(rep[:, 1:].sum(1), loss.cpu().numpy()) <= 1e-5


def test_check_finite_numeric_error(plans):
    from paper_2602_11896_b200 import JtfsError
    p = plans("t1")
    x = torch.zeros(1000, device="cuda")
    p.check_finite(x)
    x[777] = float("nan")
    with pytest.raises(JtfsError) as e:
        p.check_finite(x)
    assert e.value.code == 3                      # JTFS_ERR_NUMERIC
    x[777] = float("inf")
    with pytest.raises(JtfsError):
        p.check_finite(x)


def test_repeatability_stress(plans):
    # race evidence (compute-sanitizer is closed on this GPU pool): the mbarrier / TMEM pipelines give
    # bitwise identical results over many repeated launches, for the forward and the full loss+gradient
    for name, reps in (("c1", 20), ("c2", 5)):
        p = plans(name)
        x, y = inputs(name, B=2)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        S = p.forward(xd)
        l0, g0 = p.loss_grad(yd, S)
        for _ in range(reps):
            assert torch.equal(p.forward(xd), S)
            l1, g1 = p.loss_grad(yd, S)
            assert torch.equal(l1, l0) and torch.equal(g1, g0)


LANES_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2602_11896_b200 import Plan
from synth import CONFIGS, plan_args, batch
p = Plan(*plan_args(CONFIGS["c2"]))
x = torch.from_numpy(batch("c2", 4)).cuda(); y = torch.from_numpy(batch("c2", 4, which="y")).cuda()
S = p.forward(x)
ws = torch.empty(p.workspace_size(4, True), dtype=torch.uint8, device="cuda")
loss, g = p.loss_grad(y, S, ws=ws)
np.savez({out!r}, loss=loss.cpu().numpy(), g=g.cpu().numpy())
"""


def test_two_lanes_bitwise_equal_one_lane(tmp_path):
    # JTFS_LANES=2 runs micro-batches on two concurrent lanes (own fan-out streams each): per-signal
    # results must not depend on it
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for lanes in ("1", "2"):
        out = str(tmp_path / f"l{lanes}.npz")
        r = subprocess.run([sys.executable, "-c", LANES_SCRIPT.format(root=root, out=out)],
                           env=dict(os.environ, JTFS_LANES=lanes), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(out))
    assert np.array_equal(res[0]["g"], res[1]["g"]) and np.array_equal(res[0]["loss"], res[1]["loss"])

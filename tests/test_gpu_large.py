"""GPU parity at the BASELINE.json sizes (configs c2..c5), one signal each, in the launch
configuration bench.py uses, against the float64 oracle (R22: both sides use the modulus
dead zone |z| < 1e-12 RMS(y) of SPEC S:372, which changes the float64 gradient by <= 1e-9 at these
inputs; tests/golden/r22_effect.json).

c2 runs whole: every second-order block, the full loss. c3-c5: the first and the last block (the
oracle evaluates a subset of blocks, `Oracle.forward(blocks=...)`), plus S0 and order 1; the GPU's
loss is restricted to the same paths by a target equal to its own (bitwise deterministic) S(y)
outside the subset, so its residual is exactly zero there. Special inputs at c2: y with exactly
silent stretches (the regime the dead zone exists for), a zero target (S(0) = 0), and y = x
(nullity). Bars: rel-L2 1e-4 (S, loss), 1e-3 (dE/dy)."""
import numpy as np
import pytest
import torch

from oracle.jtfs import Oracle
from oracle.plan import make_plan
from synth import CONFIGS, plan_args, batch

pytestmark = pytest.mark.gpu

# (config, blocks or None = all, input variant)
CASES = [("c2", None, "music"), ("c2", None, "silent"), ("c2", None, "zero_target"),
         ("c3", [0, 10], "music"), ("c4", [0, 11], "music"), ("c4", [11], "silent"), ("c5", [0, 11], "music")]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def subset_mask(plan, blocks):
    m = np.zeros(plan.n_coef, bool)
    for q in plan.paths:
        if q.order <= 1 or blocks is None or q.block in blocks:
            m[q.offset:q.offset + q.rows * q.frames] = True
    return m


def silent(y):
    """four exactly silent runs of N/16 samples"""
    y = y.copy()
    N = y.shape[1]
    for k in range(4):
        y[:, (4 * k + 1) * N // 16:(4 * k + 2) * N // 16] = 0.0
    return y


@pytest.fixture(scope="module")
def plans():
    from paper_2602_11896_b200 import Plan
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Plan(*plan_args(CONFIGS[name]))
        return cache[name]
    return get


@pytest.mark.parametrize("name,blocks,variant", CASES,
                         ids=[f"{c}-{'all' if b is None else 'b' + '-'.join(map(str, b))}-{v}" for c, b, v in CASES])
def test_large_forward_and_gradient(plans, name, blocks, variant):
    args = plan_args(CONFIGS[name])
    p = plans(name)
    o = Oracle(args)
    x = batch(name, 1)
    y = batch(name, 1, which="y")
    if variant == "silent":
        y = silent(y)
    if variant == "zero_target":
        x = np.zeros_like(x)
    m = subset_mask(o.plan, blocks)
    # forward: GPU runs everything, the oracle the sampled blocks
    Sg = p.forward(torch.from_numpy(x).cuda()).cpu().numpy()[0]
    So = o.forward(x, blocks=blocks).numpy()[0]
    if variant == "zero_target":
        assert not np.any(Sg) and not np.any(So)          # S(0) = 0 exactly on both sides
    else:
        assert rel(Sg[m], So[m]) <= 1e-4
        for q in o.plan.paths:
            if m[q.offset]:
                sl = slice(q.offset, q.offset + q.rows * q.frames)
                assert rel(Sg[sl], So[sl]) <= 2e-3, (name, q)
    yd = torch.from_numpy(y).cuda()
    if blocks is None:
        St = torch.from_numpy(So[None].astype(np.float32)).cuda()
        Eo, go = o.loss_grad(y, So[None])
    else:
        Sy = p.forward(yd)
        St = Sy.clone()
        mt = torch.from_numpy(m).cuda()
        St[0, mt] = torch.from_numpy(So.astype(np.float32)).cuda()[mt]
        Eo, go = o.loss_grad_subset(y, So[None], blocks)
    loss, g = p.loss_grad(yd, St)
    assert rel(loss.cpu().numpy(), Eo.numpy()) <= 1e-4
    assert rel(g.cpu().numpy(), go.numpy()) <= 1e-3


def test_nullity_c2(plans):
    # the gradient is null when S(y) = S(x); here y = x exactly and the target is the GPU's own
    # (bitwise deterministic) S(x): every residual is exactly 0, so loss and gradient are exactly 0
    p = plans("c2")
    x = torch.from_numpy(batch("c2", 2)).cuda()
    S = p.forward(x)
    loss, g = p.loss_grad(x, S)
    assert float(loss.abs().max()) == 0.0 and float(g.abs().max()) == 0.0


def test_split_k_shards_and_microbatch(plans):
    """c2 exercises the split-K tensor-core blocks (W kept by the forward, GEMM2-only backward) and the
    filter-group split with g_Y2 partials: per-signal results are bitwise independent of the micro-batch,
    and path shards sum to the whole. Shard 1 runs first on a workspace filled with NaN bytes (it must
    not read order-1 buffers only shard 0 writes)."""
    p = plans("c2")
    x = torch.from_numpy(batch("c2", 2)).cuda()
    y = torch.from_numpy(batch("c2", 2, which="y")).cuda()
    S = p.forward(x)
    for _ in range(3):   # repeated launches are bitwise identical (no races in the pipelined kernels)
        assert torch.equal(p.forward(x), S)
    ws = torch.full((p.workspace_size(2, True),), 0xFF, dtype=torch.uint8, device="cuda")
    l1s, g1s = p.loss_grad(y, S, shard=1, n_shards=2, ws=ws)
    assert bool(torch.isfinite(g1s).all()) and bool(torch.isfinite(l1s).all())
    loss, g = p.loss_grad(y, S)
    ws1 = torch.empty(p.workspace_size(1, True), dtype=torch.uint8, device="cuda")
    l1, g1 = p.loss_grad(y, S, ws=ws1)
    assert torch.equal(g1, g) and torch.equal(l1, loss)
    l0s, g0s = p.loss_grad(y, S, shard=0, n_shards=2)
    gs, ls = g0s + g1s, l0s + l1s
    # the shards' partial gradients run the same fp32 adjoint chain (FFTs up to 2^17 points) on
    # different partial sums; their sum differs from the whole-signal gradient by rounding only
    assert rel(gs.cpu().numpy(), g.cpu().numpy()) <= 1e-5
    assert rel(ls.cpu().numpy(), loss.cpu().numpy()) <= 1e-6

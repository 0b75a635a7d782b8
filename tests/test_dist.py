"""Multi-process (world_size 2, gloo, CPU) tests of the sharding glue in paper_2602_11896_b200/dist.py.

The per-shard compute is injected with a float64 path-restricted loss built from the oracle (test
infrastructure): it checks that the batch split, the unit -> shard rule and the single all_reduce
reassemble exactly the unsharded loss and gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import TINY, plan_args, noise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_shard_compute(args):
    from oracle.jtfs import Oracle
    from paper_2602_11896_b200 import Plan
    from paper_2602_11896_b200.dist import path_owner
    o = Oracle(args)
    paths = [dict(order=q.order, block=q.block) for q in o.plan.paths]
    plan = Plan(*args)          # host-only: the library's block -> shard rule (jtfs_plan_shards)

    def compute(y, St, shard, n):
        owner = path_owner(paths, plan.block_owner(n))
        w = torch.zeros(o.plan.n_coef, dtype=torch.float64)
        for q, own in zip(o.plan.paths, owner):
            if own == shard:
                w[q.offset:q.offset + q.rows * q.frames] = 1.0
        yv = y.detach().to(torch.float64).requires_grad_(True)
        r = (o.forward(yv) - St) * w
        E = 0.5 * (r * r).sum(1)
        (g,) = torch.autograd.grad(E.sum(), yv)
        return E.detach(), g
    return o, compute


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_11896_b200.dist import DistJTFS
        args = plan_args(TINY["t2"])
        o, compute = _oracle_shard_compute(args)
        B = 3
        x = torch.from_numpy(noise(args[0], B, seed=5).astype(np.float64))
        y = torch.from_numpy(noise(args[0], B, seed=6).astype(np.float64))
        St = o.forward(x)
        dj = DistJTFS(path_shards=world if mode == "path" else 1, compute=compute)
        sl = dj.my_signals(B)
        if mode == "gather":   # B = 3 over 2 batch groups: uneven (2 + 1) per-rank loss vectors
            mine = torch.arange(sl.start, sl.stop, dtype=torch.float64)
            q.put((rank, sl.start, sl.stop, dj.gather_losses(mine, B).numpy(), None))
            return
        loss, grad = dj.loss_grad(y[sl], St[sl], chunk=2 if mode == "path" else None)
        q.put((rank, sl.start, sl.stop, loss.numpy(), grad.numpy()))
    finally:
        dist.destroy_process_group()


def _run(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


def _reference():
    from oracle.jtfs import Oracle
    args = plan_args(TINY["t2"])
    o = Oracle(args)
    x = noise(args[0], 3, seed=5).astype(np.float64)
    y = noise(args[0], 3, seed=6).astype(np.float64)
    E, g = o.loss_grad(y, o.forward(x))
    return E.numpy(), g.numpy()


def test_batch_split_rule():
    from paper_2602_11896_b200.dist import batch_slice
    for B in (1, 5, 8, 256):
        for W in (1, 2, 3, 8):
            sl = [batch_slice(B, W, r) for r in range(W)]
            idx = sum((list(range(s.start, s.stop)) for s in sl), [])
            assert idx == list(range(B))


def test_path_owner_rule_matches_abi_doc():
    from paper_2602_11896_b200.dist import path_owner
    paths = [dict(order=0)] + [dict(order=1)] * 3 + [dict(order=2, block=b) for b in (0, 0, 1, 1, 1)]
    assert path_owner(paths, [1, 0]) == [-1, 0, 0, 0, 1, 1, 0, 0, 0]


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_block_shards_lpt(name):
    # every block owned by exactly one shard; whole blocks (layer 2 computed once per block); the LPT
    # loads are balanced: the largest shard exceeds the mean by at most the largest block's cost
    from paper_2602_11896_b200 import Plan
    from synth import CONFIGS
    p = Plan(*plan_args(CONFIGS[name]))
    nb = p.info.n_blocks
    assert p.block_owner(1) == [0] * nb
    for n in (2, 4, 8):
        own = p.block_owner(n)
        assert len(own) == nb and set(own) <= set(range(n))
        assert own == p.block_owner(n)                    # deterministic
        if n <= nb:
            assert set(own) == set(range(n))             # no idle shard while blocks remain


def test_gloo_gather_losses_uneven():
    res = _run("gather")
    for rank, s0, s1, loss, grad in res:
        assert loss.tolist() == [0.0, 1.0, 2.0]


def test_gloo_path_sharding_sums_to_whole():
    E, g = _reference()
    res = _run("path")
    for rank, s0, s1, loss, grad in res:
        assert (s0, s1) == (0, 3)            # every rank of the path group sees all signals
        assert np.allclose(loss, E, rtol=1e-12, atol=1e-18)
        assert np.allclose(grad, g, rtol=1e-10, atol=1e-16)


def test_gloo_batch_sharding():
    E, g = _reference()
    res = _run("batch")
    got_E = np.concatenate([r[3] for r in res])
    got_g = np.concatenate([r[4] for r in res])
    assert [(r[1], r[2]) for r in res] == [(0, 2), (2, 3)]
    assert np.allclose(got_E, E, rtol=1e-12) and np.allclose(got_g, g, rtol=1e-10, atol=1e-16)

"""Multi-GPU glue: one process per GPU, torch.distributed over NCCL.

Two ways to split the work of jtfs_loss_grad:
  * batch sharding — signals are independent (R27): each rank owns B/G signals, no data-path
    collective (weak scaling). Only per-signal losses may be gathered for logging.
  * path sharding — the second-order blocks (n2) of ONE signal are split across the ranks of a
    path group by the planner's LPT rule over per-block cost (jtfs_plan_shards, include/jtfs.h);
    order 1 goes to shard 0. A rank computes layer 2, the joint stage and their adjoints only for
    its own blocks; layer 1 (forward and adjoint) is the only replicated stage. The partial dE/dx
    and losses sum exactly, so the only exchange is ONE all_reduce(SUM) of [grad | loss] per
    micro-batch over NVLink.
Ranks are laid out as (batch_group, path_shard) with path_shard = rank % path_shards.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def batch_slice(B_total: int, world: int, rank: int) -> slice:
    """Contiguous, balanced split of B_total signals over `world` batch groups."""
    base, rem = divmod(B_total, world)
    start = rank * base + min(rank, rem)
    return slice(start, start + base + (1 if rank < rem else 0))


def path_owner(paths: list[dict], block_owner: list[int]) -> list[int]:
    """Owner shard of every path (R15 order): -1 for S0 (not in the loss), 0 for order 1, and the
    owner of its block for order 2 (`block_owner` from Plan.block_owner / jtfs_plan_shards)."""
    out = []
    for q in paths:
        if q["order"] == 0:
            out.append(-1)
        elif q["order"] == 1:
            out.append(0)
        else:
            out.append(block_owner[q["block"]])
    return out


class DistJTFS:
    """Sharded loss + gradient. `compute(y, S_target, shard, n_shards) -> (loss, grad)` defaults to
    the CUDA plan's jtfs_loss_grad; it is injectable only so the CPU gloo tests can exercise the
    collective logic."""

    def __init__(self, plan=None, path_shards: int = 1, group=None,
                 compute: Callable | None = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world % path_shards:
            raise ValueError("world size must be a multiple of path_shards")
        self.path_shards = path_shards
        self.shard = self.rank % path_shards
        self.batch_group = self.rank // path_shards
        self.n_batch_groups = self.world // path_shards
        self.plan = plan
        self.compute = compute or (lambda y, St, s, n: plan.loss_grad(y, St, shard=s, n_shards=n))
        # one process group per path group (every rank must create every group, same order)
        self.path_group = None
        if path_shards > 1:
            ranks_all = dist.get_process_group_ranks(group) if group is not None else list(range(self.world))
            for g in range(self.n_batch_groups):
                ranks = ranks_all[g * path_shards:(g + 1) * path_shards]
                pg = dist.new_group(ranks)
                if g == self.batch_group:
                    self.path_group = pg

    def my_signals(self, B_total: int) -> slice:
        return batch_slice(B_total, self.n_batch_groups, self.batch_group)

    def loss_grad(self, y: torch.Tensor, S_target: torch.Tensor, chunk: int | None = None):
        """(loss, grad) of this rank's signals, complete (summed over the path group).

        With path shards the batch runs in chunks of `chunk` signals (default: all at once); the
        all_reduce of chunk i is issued asynchronously (NCCL's own stream, ordered after chunk i's
        kernels) while chunk i+1 computes, so the exchange overlaps the next chunk's work."""
        if self.path_shards == 1:
            return self.compute(y, S_target, self.shard, self.path_shards)
        B = y.shape[0]
        chunk = B if not chunk else max(1, min(chunk, B))
        losses, grads, works, bufs = [], [], [], []
        for c0 in range(0, B, chunk):
            sl = slice(c0, min(B, c0 + chunk))
            loss, grad = self.compute(y[sl], S_target[sl], self.shard, self.path_shards)
            buf = torch.cat([grad.reshape(-1), loss.reshape(-1).to(grad.dtype)])
            works.append(dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.path_group, async_op=True))
            bufs.append((buf, grad.shape, loss.dtype))
        for w in works:
            w.wait()
        for buf, gshape, ldt in bufs:
            n = 1
            for d in gshape:
                n *= d
            grads.append(buf[:n].view(gshape))
            losses.append(buf[n:].to(ldt))
        return torch.cat(losses), torch.cat(grads)

    def gather_losses(self, loss: torch.Tensor, B_total: int) -> torch.Tensor:
        """All per-signal losses (logging only), ordered by signal index. Batch groups may hold
        unequal signal counts (batch_slice), so every rank pads its losses to ceil(B_total / groups)
        before the all_gather (which needs equal sizes) over the same group as the constructor."""
        cap = -(-B_total // self.n_batch_groups)
        buf = torch.zeros(cap, dtype=loss.dtype, device=loss.device)
        buf[: loss.numel()] = loss.reshape(-1)
        out = [torch.zeros_like(buf) for _ in range(self.world)]
        dist.all_gather(out, buf, group=self.group)
        parts = []
        for g in range(self.n_batch_groups):
            sl = batch_slice(B_total, self.n_batch_groups, g)
            parts.append(out[g * self.path_shards][: sl.stop - sl.start])
        return torch.cat(parts)

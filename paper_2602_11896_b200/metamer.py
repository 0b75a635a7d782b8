"""Metamer synthesis loop (§2.3 Reconstruction): colored-noise initialisation,
then bold-driver momentum descent on the JTFS loss, one `metamer_step` (device, stream-ordered) per
iteration. The host side only reads the per-signal losses/flags once per iteration to apply the stop
rules (readings R24, R25 in DESIGN.md), write the loss CSV and
checkpoint/resume the state; every arithmetic step runs in libjtfs.so's kernels.

A non-finite iterate raises JtfsError(JTFS_ERR_NUMERIC); a non-finite loss is a
rejection (E <= E_prev fails), so the bold driver rolls the signal back to its last finite iterate.

Stop rules per signal (a stopped signal is frozen at its best evaluated iterate by the `active`
mask of jtfs_metamer_state):
  * rejection cap: `max_rejects` consecutive bold-driver rejections (SPEC: "at most 8 shrink retries
    per iteration before accepting the best-so-far");
  * relative loss: an accepted loss <= tol * (loss at the initial iterate).
"""
from __future__ import annotations

import csv
import os

import torch

STATE_KEYS = ("y", "u", "y_prev", "g_prev", "mu", "loss_prev", "loss", "accepted", "active")


def save_checkpoint(path: str, state: dict, extra: dict) -> None:
    """Atomic write (tmp + rename) of the device state and the host loop counters."""
    blob = {k: state[k].detach().cpu() for k in STATE_KEYS}
    blob["iter"] = state["iter"]
    blob.update(extra)
    tmp = path + ".tmp"
    torch.save(blob, tmp)
    os.replace(tmp, path)


def load_checkpoint(path: str, device) -> tuple[dict, dict]:
    blob = torch.load(path, map_location="cpu", weights_only=False)
    state = {k: blob.pop(k).to(device).contiguous() for k in STATE_KEYS}
    state["iter"] = blob.pop("iter")
    return state, blob


def reconstruct(plan, S_target: torch.Tensor, steps: int = 100, y0: torch.Tensor | None = None, seed: int = 0,
                tol: float = 0.0, max_rejects: int = 8, mu0: float = 0.1, momentum: float = 0.9,
                grow: float = 1.1, shrink: float = 0.5, csv_path: str | None = None,
                checkpoint: str | None = None, checkpoint_every: int = 10, resume: bool = False,
                ws: torch.Tensor | None = None) -> dict:
    """Run up to `steps` trials for every signal of S_target [B, n_coef]. Returns the best iterate
    per signal (y_best = y_prev, loss_best = loss_prev), the per-iteration loss history and the
    state. With `resume` and an existing `checkpoint`, continues from it (bitwise the same
    trajectory as an uninterrupted run: the state is the whole of the loop's memory)."""
    dev = S_target.device
    B = S_target.shape[0]
    ws = ws if ws is not None else plan.workspace(B, True, dev)
    if resume and checkpoint and os.path.exists(checkpoint):
        state, extra = load_checkpoint(checkpoint, dev)
        rej, E0, history = extra["rej"], extra["E0"], extra["history"]
    else:
        if y0 is None:
            y0 = plan.colored_noise(S_target, seed=seed)
        state = plan.metamer_state(y0.contiguous(), mu0)
        state["active"] = torch.ones(B, dtype=torch.int32, device=dev)
        rej, E0, history = [0] * B, [None] * B, []
    mode = "a" if (resume and csv_path and os.path.exists(csv_path)) else "w"
    fcsv = open(csv_path, mode, newline="") if csv_path else None
    wr = csv.writer(fcsv) if fcsv else None
    if wr and mode == "w":
        wr.writerow(["iteration", "signal", "loss", "mu", "accepted", "active"])
    try:
        while state["iter"] < steps and bool(state["active"].any()):
            it = state["iter"]
            plan.metamer_step(state, S_target, momentum=momentum, grow=grow, shrink=shrink, ws=ws)
            plan.check_finite(state["y"])         # a non-finite iterate aborts the job
            loss = state["loss"].tolist()
            acc = state["accepted"].tolist()
            mu = state["mu"].tolist()
            act = state["active"].tolist()
            stop = []
            for b in range(B):
                if not act[b]:
                    continue
                if E0[b] is None:
                    E0[b] = loss[b]
                rej[b] = 0 if acc[b] else rej[b] + 1
                if rej[b] >= max_rejects or (acc[b] and E0[b] > 0 and loss[b] <= tol * E0[b]) or E0[b] == 0:
                    stop.append(b)
                if wr:
                    wr.writerow([it, b, loss[b], mu[b], acc[b], 1])
            history.append([loss[b] if act[b] else None for b in range(B)])
            if stop:
                state["active"][torch.tensor(stop, device=dev)] = 0
            if checkpoint and (state["iter"] % checkpoint_every == 0 or state["iter"] >= steps):
                if fcsv:
                    fcsv.flush()
                save_checkpoint(checkpoint, state, {"rej": rej, "E0": E0, "history": history})
    finally:
        if fcsv:
            fcsv.close()
    # signals stopped in the last iteration are restored to their best iterate here (the kernel does it
    # on the next call for a continuing run)
    stopped = state["active"] == 0
    if bool(stopped.any()):
        state["y"][stopped] = state["y_prev"][stopped]
        state["u"][stopped] = 0.0
    return {"y_best": state["y_prev"], "loss_best": state["loss_prev"], "history": history, "state": state,
            "iterations": state["iter"]}

"""Thin Python binding over libjtfs.so with the ABI's names (jtfs_plan, jtfs_forward,
jtfs_loss_grad, metamer_step). torch is used only for device memory and streams; every
computation runs in the library's CUDA kernels."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import JtfsError, MetamerState, PathT, PlanInfo, check

__all__ = ["Plan", "JtfsError"]


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Plan:
    """jtfs_plan(N, J, Q, J_fr, Q_fr, T, F) (§3.1 filterbanks; readings in DESIGN.md §2)."""

    def __init__(self, N: int, J: int, Q: int, J_fr: int, Q_fr: int, T: int, F: int, Q2: int = 1):
        self.lib = _lib.load()
        h = ctypes.c_void_p()
        check(self.lib.jtfs_plan_q2(N, J, Q, Q2, J_fr, Q_fr, T, F, ctypes.byref(h)))
        self.h = h
        self.args = (N, J, Q, J_fr, Q_fr, T, F)
        self.Q2 = Q2
        info = PlanInfo()
        check(self.lib.jtfs_plan_info(self.h, ctypes.byref(info)))
        self.info = info
        self._ws = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.jtfs_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ---------------------------------------------------------------- host-side queries
    @property
    def n_coef(self) -> int:
        return self.info.n_coef

    @property
    def N(self) -> int:
        return self.info.N

    def paths(self) -> list[dict]:
        """Path table (R15 order); order-2 entries carry their block index ("block", -1 otherwise)."""
        arr = (PathT * self.info.n_paths)()
        check(self.lib.jtfs_plan_paths(self.h, arr, self.info.n_paths))
        out = [{f: getattr(a, f) for f, _ in PathT._fields_} for a in arr]
        n2s = sorted({q["n2"] for q in out if q["order"] == 2})
        for q in out:
            q["block"] = n2s.index(q["n2"]) if q["order"] == 2 else -1
        return out

    def block_owner(self, n_shards: int) -> list[int]:
        """jtfs_plan_shards: owner shard of every second-order block under path sharding."""
        nb = self.info.n_blocks
        arr = (ctypes.c_int32 * max(nb, 1))()
        check(self.lib.jtfs_plan_shards(self.h, n_shards, arr, max(nb, 1)))
        return list(arr[:nb])

    def filters(self, layer: int) -> dict:
        cnt = ctypes.c_int64()
        check(self.lib.jtfs_plan_filters(self.h, layer, None, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        xi, sg = np.zeros(n), np.zeros(n)
        j = np.zeros(n, np.int32)
        check(self.lib.jtfs_plan_filters(self.h, layer, xi.ctypes.data, sg.ctypes.data, j.ctypes.data, n,
                                         ctypes.byref(cnt)))
        return {"xi": xi, "sigma": sg, "j": j}

    def response(self, layer: int, idx: int, k: int) -> np.ndarray:
        L0 = self.info.P if layer in (2, 4) else self.info.N_pad
        out = np.zeros(L0 >> k)
        check(self.lib.jtfs_plan_response(self.h, layer, idx, k, out.ctypes.data, out.size))
        return out

    # ---------------------------------------------------------------- device
    def prepare(self, stream=None) -> None:
        check(self.lib.jtfs_plan_prepare(self.h, _stream(stream)))

    def workspace_size(self, batch: int, with_grad: bool) -> int:
        return self.lib.jtfs_workspace_size(self.h, batch, 1 if with_grad else 0)

    def workspace(self, batch: int, with_grad: bool, device=None, budget_frac: float = 0.6) -> torch.Tensor:
        """Allocate (and cache) a workspace for min(batch, what fits in budget_frac of free memory)."""
        device = device or torch.device("cuda", torch.cuda.current_device())
        per = self.workspace_size(1, with_grad)
        free, _ = torch.cuda.mem_get_info(device)
        have = 0 if self._ws is None else self._ws.numel()
        mb = max(1, min(batch, int((free + have) * budget_frac) // per))
        need = per * mb
        if self._ws is None or self._ws.numel() < need or self._ws.device != device:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        """jtfs_forward: x [B, N] float32 CUDA -> S [B, n_coef] float32."""
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.shape[-1] == self.N
        B = x.shape[0]
        S = out if out is not None else torch.empty(B, self.n_coef, device=x.device, dtype=torch.float32)
        ws = ws if ws is not None else self.workspace(B, False, x.device)
        check(self.lib.jtfs_forward(self.h, _ptr(x), B, _ptr(S), _ptr(ws), ws.numel(), _stream(stream)))
        return S

    def loss_grad(self, y: torch.Tensor, S_target: torch.Tensor, shard: int = 0, n_shards: int = 1,
                  loss: torch.Tensor | None = None, grad: torch.Tensor | None = None,
                  ws: torch.Tensor | None = None, stream=None):
        """jtfs_loss_grad: (loss [B], dE/dy [B, N]) for E_b = 1/2 ||S(y_b) - S_target_b||^2 (orders 1,2)."""
        assert y.is_cuda and y.dtype == torch.float32 and y.is_contiguous()
        assert S_target.is_cuda and S_target.dtype == torch.float32 and S_target.is_contiguous()
        B = y.shape[0]
        loss = loss if loss is not None else torch.empty(B, device=y.device, dtype=torch.float32)
        grad = grad if grad is not None else torch.empty_like(y)
        ws = ws if ws is not None else self.workspace(B, True, y.device)
        check(self.lib.jtfs_loss_grad(self.h, _ptr(y), _ptr(S_target), B, _ptr(loss), _ptr(grad), shard,
                                      n_shards, _ptr(ws), ws.numel(), _stream(stream)))
        return loss, grad

    def loss_grad_host(self, y: np.ndarray, S_target: np.ndarray, ws: torch.Tensor | None = None,
                       stream=None):
        """End-to-end call with HOST buffers (H2D + compute + D2H inside the library call)."""
        y = np.ascontiguousarray(y, dtype=np.float32)
        St = np.ascontiguousarray(S_target, dtype=np.float32)
        B = y.shape[0]
        loss = np.empty(B, np.float32)
        grad = np.empty_like(y)
        stg = self.lib.jtfs_host_staging_size(self.h, B, 1)
        if ws is None:
            ws = self.workspace_host(B)
        check(self.lib.jtfs_loss_grad_host(self.h, y.ctypes.data, St.ctypes.data, B, loss.ctypes.data,
                                           grad.ctypes.data, _ptr(ws), ws.numel(), _stream(stream)))
        del stg
        return loss, grad

    def workspace_host(self, B: int, device=None) -> torch.Tensor:
        stg = self.lib.jtfs_host_staging_size(self.h, B, 1)
        device = device or torch.device("cuda", torch.cuda.current_device())
        per = self.workspace_size(1, True)
        free, _ = torch.cuda.mem_get_info(device)
        mb = max(1, min(B, int(free * 0.5) // per))
        return torch.empty(stg + per * mb, dtype=torch.uint8, device=device)

    def metamer_state(self, y0: torch.Tensor, mu0: float = 0.1) -> dict:
        B = y0.shape[0]
        dev = y0.device
        return {"y": y0.clone(), "u": torch.zeros_like(y0), "y_prev": y0.clone(), "g_prev": torch.zeros_like(y0),
                "mu": torch.full((B,), mu0, device=dev), "loss_prev": torch.full((B,), float("inf"), device=dev),
                "loss": torch.zeros(B, device=dev), "accepted": torch.zeros(B, dtype=torch.int32, device=dev),
                "iter": 0}

    def metamer_step(self, state: dict, S_target: torch.Tensor, momentum: float = 0.9, grow: float = 1.1,
                     shrink: float = 0.5, ws: torch.Tensor | None = None, stream=None) -> dict:
        """metamer_step: one bold-driver momentum trial, stream-ordered."""
        B = state["y"].shape[0]
        act = state.get("active")
        ms = MetamerState(_ptr(state["y"]), _ptr(state["u"]), _ptr(state["y_prev"]), _ptr(state["g_prev"]),
                          _ptr(state["mu"]), _ptr(state["loss_prev"]), _ptr(state["loss"]),
                          _ptr(state["accepted"]), state["iter"], None if act is None else _ptr(act))
        ws = ws if ws is not None else self.workspace(B, True, state["y"].device)
        check(self.lib.metamer_step(self.h, ctypes.byref(ms), _ptr(S_target), B, momentum, grow, shrink,
                                    _ptr(ws), ws.numel(), _stream(stream)))
        state["iter"] = ms.iter
        return state

    def check_finite(self, x: torch.Tensor, stream=None) -> None:
        """jtfs_check_finite: raises JtfsError (JTFS_ERR_NUMERIC) if x holds a NaN or inf."""
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        check(self.lib.jtfs_check_finite(_ptr(x), x.numel(), _stream(stream)))

    def loss_report(self, S: torch.Tensor, S_target: torch.Tensor, stream=None) -> torch.Tensor:
        """jtfs_loss_report: per-path losses [B, n_paths] (1/2 sum of squared residuals per path, R15
        order; path 0 = S0 is reported, not part of the loss)."""
        assert S.is_cuda and S.dtype == torch.float32 and S.is_contiguous() and S.shape == S_target.shape
        assert S_target.is_cuda and S_target.dtype == torch.float32 and S_target.is_contiguous()
        B = S.shape[0]
        rep = torch.empty(B, self.info.n_paths, device=S.device, dtype=torch.float32)
        check(self.lib.jtfs_loss_report(self.h, _ptr(S), _ptr(S_target), B, _ptr(rep), _stream(stream)))
        return rep

    def colored_noise(self, S_target: torch.Tensor, seed: int = 0, white: torch.Tensor | None = None,
                      ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """jtfs_colored_noise: y0 [B, N], colored Gaussian noise whose band energies follow the
        order-1 profile of S_target (reading R25). `white` [B, N_pad] standard normal;
        drawn here from a seeded torch generator on the device when not given."""
        assert S_target.is_cuda and S_target.dtype == torch.float32 and S_target.is_contiguous()
        B = S_target.shape[0]
        if white is None:
            gen = torch.Generator(device=S_target.device).manual_seed(seed)
            white = torch.randn(B, self.info.N_pad, generator=gen, device=S_target.device, dtype=torch.float32)
        assert white.is_cuda and white.dtype == torch.float32 and white.is_contiguous()
        assert white.shape == (B, self.info.N_pad)
        y0 = torch.empty(B, self.N, device=S_target.device, dtype=torch.float32)
        ws = ws if ws is not None else self.workspace(B, False, S_target.device)
        check(self.lib.jtfs_colored_noise(self.h, _ptr(S_target), _ptr(white), B, _ptr(y0), _ptr(ws), ws.numel(),
                                          _stream(stream)))
        return y0

    def debug_stage(self, stage: int, x: torch.Tensor) -> torch.Tensor:
        B = x.shape[0]
        info = self.info
        ws = self.workspace(B, False, x.device)
        if stage == 1:
            out = torch.empty(B, self._sumL1(), device=x.device)
        elif stage == 2:
            out = torch.empty(B, info.N1, info.N_pad // (info.N // info.frames), device=x.device)
        elif stage == 3:
            out = torch.empty(B, self._sumY2(), dtype=torch.complex64, device=x.device)
        elif stage == 5:
            out = torch.empty(B, info.N_pad, dtype=torch.complex128, device=x.device)
        elif stage == 6:
            out = torch.empty(B, self._sumL1(), dtype=torch.complex64, device=x.device)
        else:
            out = torch.empty(B, info.n_coef, device=x.device)
        check(self.lib.jtfs_debug_stage(self.h, stage, _ptr(x), B, _ptr(out), out.numel() * out.element_size(),
                                        _ptr(ws), ws.numel(), _stream(None)))
        return out

    def _sumL1(self) -> int:
        f = self.filters(0)
        T = self.info.N // self.info.frames
        log2T = T.bit_length() - 1
        return int(sum(self.info.N_pad >> min(int(j), log2T) for j in f["j"]))

    def _sumY2(self) -> int:
        f1, f2 = self.filters(0), self.filters(1)
        T = self.info.N // self.info.frames
        log2T = T.bit_length() - 1
        tot = 0
        for j2 in f2["j"]:
            n1_max = int(np.sum(f1["j"] < j2))
            if n1_max:
                tot += n1_max * (self.info.N_pad >> min(int(j2), log2T))
        return tot

    def launch_count(self) -> int:
        return self.lib.jtfs_launch_count()

    def cost(self) -> dict:
        """Algorithmic per-signal cost of the joint stage (see include/jtfs.h jtfs_plan_cost)."""
        out = np.zeros(8)
        check(self.lib.jtfs_plan_cost(self.h, out.ctypes.data, 8))
        return {"fwd_tc_flops": out[0], "fwd_fft_flops": out[1], "bwd_tc_flops": out[2],
                "bwd_fft_flops": out[3], "cells": out[4], "joint_hbm_bytes": out[5],
                "joint_fwd_flops": out[0] + out[1], "joint_bwd_flops": out[2] + out[3]}

    def prof_enable(self, on: bool) -> None:
        self.lib.jtfs_prof_enable(1 if on else 0)

    def prof_read(self, kid: int) -> tuple[float, int]:
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        check(self.lib.jtfs_prof_read(kid, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

"""ORACLE (test infrastructure only) — direct-sum route, no FFT anywhere.

An independent O(L^2) implementation of the multirate forward with every
Fourier product replaced by the mathematically identical direct circular sum with the
closed-form (Poisson-summed) kernel `plan.time_kernel_closed_form` (O1):
    (D_s C_h u)[n] = sum_m u[m] h[(n s - m) mod L]
It recomputes every path depth-first (one (n1, n2, n_fr) at a time, no stacking), so agreement
with oracle/jtfs.py pins: the FFT route, subsample_fourier as decimation, the level
(fold-sum) convention R9, the width-first stacking, zero-padding to P, the
spin order R12 and the packing R15. Only usable on tiny configurations (N_pad <= 4096).
"""
from __future__ import annotations

import numpy as np

from .plan import Plan, time_kernel_closed_form


def _circ(h: np.ndarray, u: np.ndarray, s: int) -> np.ndarray:
    """(D_s C_h u)[n] = sum_m u[m] h[(n s - m) mod L] along the last axis of u (direct sum)."""
    L = h.shape[0]
    n = np.arange(L // s)[:, None] * s
    m = np.arange(L)[None, :]
    M = h[(n - m) % L]                     # [L/s, L]
    return u @ M.T


def _circ_rows(h: np.ndarray, X: np.ndarray, s: int) -> np.ndarray:
    """Same along axis 0 of a [L, cols] array."""
    return _circ(h, X.T, s).T


def _reflect(plan: Plan, x: np.ndarray) -> np.ndarray:
    """Half-sample symmetric extension, built element by element (R10)."""
    N = plan.N
    out = np.empty(plan.N_pad)
    for i in range(plan.N_pad):
        t = (i - plan.pad_left) % (2 * N)
        out[i] = x[t] if t < N else x[2 * N - 1 - t]
    return out


def forward(plan: Plan, x: np.ndarray) -> np.ndarray:
    """Packed coefficients of one signal (float64) by direct sums, depth-first."""
    p = plan
    assert p.N_pad <= 4096, "brute force is for tiny configurations only"
    xp = _reflect(p, np.asarray(x, dtype=np.float64))
    f0, nfr = p.pad_left // p.T, p.frames
    hT = lambda k: time_kernel_closed_form(p.phiT, p.N_pad, k)
    hF = lambda k: time_kernel_closed_form(p.phiF, p.P, k)
    hfr = lambda f: time_kernel_closed_form(p.L_fr[f], p.P, 0)
    out = [_circ(hT(0), xp, p.T).real[f0:f0 + nfr]]                    # S0

    U1 = []
    for n1 in range(p.N1):
        k1 = p.k1(n1)
        Z1 = _circ(time_kernel_closed_form(p.psi1[n1], p.N_pad, 0), xp, 2 ** k1)
        U1.append(np.abs(Z1))
    S1t = np.stack([_circ(hT(p.k1(n1)), U1[n1], 2 ** (p.log2T - p.k1(n1))).real
                    for n1 in range(p.N1)])                             # [N1, N_pad/T]

    X = np.zeros((p.P, S1t.shape[1]))
    X[: p.N1] = S1t
    rows1 = -(-p.N1 // p.F)
    for f in range(p.n_fr_order1):
        kf = p.k_fr(f)
        W = _circ_rows(hfr(f), X, 2 ** kf)
        if f == 0:
            Y = W.real
        else:
            V = np.abs(W)
            V = _circ(hT(p.log2T), V, 1).real
            Y = _circ_rows(hF(kf), V, 2 ** (p.log2F - kf)).real
        out.append(Y[:rows1, f0:f0 + nfr].ravel())

    for blk in p.blocks:
        rows2 = -(-blk.n1_max // p.F)
        for f in range(len(p.L_fr)):
            kf = p.k_fr(f)
            # depth-first: build the column stack one n1 at a time (no width-first stacking op)
            T2 = p.N_pad >> blk.s2
            X = np.zeros((p.P, T2), dtype=np.complex128)
            for n1 in range(blk.n1_max):
                k1 = p.k1(n1)
                h2 = time_kernel_closed_form(p.psi2[blk.n2], p.N_pad, k1)
                X[n1] = _circ(h2, U1[n1], 2 ** (blk.s2 - k1))
            V = np.abs(_circ_rows(hfr(f), X, 2 ** kf))
            V = _circ_rows(hF(kf), V, 2 ** (p.log2F - kf)).real[:rows2]
            Y = _circ(hT(blk.s2), V, 2 ** (p.log2T - blk.s2)).real
            out.append(Y[:, f0:f0 + nfr].ravel())
    S = np.concatenate([np.ravel(o) for o in out])
    assert S.shape[0] == p.n_coef
    return S

"""ORACLE (test infrastructure only) — direct-sum route, no FFT anywhere.

An independent O(L^2) implementation of the multirate forward with every
Fourier product replaced by the mathematically identical direct circular sum with the
closed-form (Poisson-summed) kernel `plan.time_kernel_closed_form` (O1):
    (D_s C_h u)[n] = sum_m u[m] h[(n s - m) mod L]
It recomputes every path depth-first (one (n1, n2, n_fr) at a time, no stacking), and its gradient
(`loss_grad`) reverses it with explicit adjoints (no autodiff), so agreement with oracle/jtfs.py pins: the FFT route, subsample_fourier as decimation, the level
(fold-sum) convention R9, the width-first stacking, zero-padding to P, the
spin order R12 and the packing R15. Direct sums over each closed-form kernel's taps (|h| > 1e-18 of its peak): usable up to c1
(N_pad = 8192).
"""
from __future__ import annotations

import numpy as np

from .plan import Plan, time_kernel_closed_form


def _support(h: np.ndarray) -> np.ndarray:
    """Taps j (as offsets in (-L/2, L/2]) where the closed-form kernel exceeds 1e-18 of its peak: the
    direct sums skip the rest (their total weight is below the float64 rounding of the sum)."""
    L = h.shape[0]
    a = np.abs(h)
    j = np.nonzero(a > 1e-18 * a.max())[0] if a.max() > 0 else np.zeros(0, np.int64)
    return np.where(j > L // 2, j - L, j)


def _circ(h: np.ndarray, u: np.ndarray, s: int) -> np.ndarray:
    """(D_s C_h u)[n] = sum_m u[m] h[(n s - m) mod L] along the last axis of u (direct sum):
    = sum over the kernel's taps j of h[j] u[(n s - j) mod L], one shifted gather per tap."""
    L = h.shape[0]
    n = np.arange(L // s) * s
    out = np.zeros(u.shape[:-1] + (L // s,), dtype=np.result_type(u, h))
    for j in _support(h):
        out += h[j % L] * u[..., (n - j) % L]
    return out


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


def forward(plan: Plan, x: np.ndarray, blocks=None) -> np.ndarray:
    """Packed coefficients of one signal (float64) by direct sums, depth-first (`blocks`: only those
    second-order blocks, the others left 0, as Oracle.forward)."""
    p = plan
    assert p.N_pad <= 8192, "brute force is for tiny configurations and c1 only"
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

    for bi, blk in enumerate(p.blocks):
        rows2 = -(-blk.n1_max // p.F)
        if blocks is not None and bi not in blocks:
            out += [np.zeros(rows2 * nfr)] * len(p.L_fr)
            continue
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


# ----------------------------------------------------------------------------------------------
# Gradient by explicit adjoints, direct sums, no FFT and no autodiff: an
# independent route to dE/dy (reading R20: through every stage incl. both pads and phi_F).
# ----------------------------------------------------------------------------------------------

def _circ_adj(h: np.ndarray, g: np.ndarray, s: int) -> np.ndarray:
    """Adjoint of u -> _circ(h, u, s) along the last axis: the conjugate transpose of the same matrix,
    (A^H g)[m] = sum_n conj(h[(n s - m) mod L]) g[n] (no use of the Hermitian-kernel shortcut R21); per tap
    j the targets m = (n s - j) mod L are distinct, so each tap is one scatter-add."""
    L = h.shape[0]
    n = np.arange(L // s) * s
    out = np.zeros(g.shape[:-1] + (L,), dtype=np.result_type(g, h))
    for j in _support(h):
        out[..., (n - j) % L] += np.conj(h[j % L]) * g
    return out


def _circ_rows_adj(h: np.ndarray, G: np.ndarray, s: int) -> np.ndarray:
    return _circ_adj(h, G.T, s).T


def _reflect_adj(plan: Plan, g_xp: np.ndarray) -> np.ndarray:
    """Adjoint of R10's padding: each padded sample's gradient goes back to its source sample."""
    N = plan.N
    out = np.zeros(N)
    for i in range(plan.N_pad):
        t = (i - plan.pad_left) % (2 * N)
        out[t if t < N else 2 * N - 1 - t] += g_xp[i]
    return out


EPS_MOD = 1e-12   # R22: z/|z| := 0 where |z| < EPS_MOD * RMS(y)


def _phase(z: np.ndarray, thr: float) -> np.ndarray:
    """Adjoint factor of |.| (R22): z/|z|, 0 where |z| < thr (thr > 0)."""
    a = np.abs(z)
    keep = a >= thr
    d = np.where(keep, a, 1.0)
    return np.where(keep, z.real / d + 1j * (z.imag / d), 0.0)


def loss_grad(plan: Plan, y: np.ndarray, S_target: np.ndarray, blocks=None) -> tuple[float, np.ndarray]:
    """E = 1/2 sum_{orders 1,2} (S(y) - S_target)^2 (R19) and dE/dy for one signal, by reversing
    `forward` stage by stage with the explicit adjoints above (modulus: g_z = (z/|z|) g_v).
    `blocks` restricts the loss to order 1 and those second-order blocks (as Oracle.loss_grad_subset)."""
    p = plan
    assert p.N_pad <= 8192, "brute force is for tiny configurations and c1 only"
    S = forward(p, y, blocks)
    r = S - np.asarray(S_target, dtype=np.float64)
    r[: p.frames] = 0.0                                                  # S0 not in the loss
    if blocks is not None:
        for q in p.paths:
            if q.order == 2 and q.block not in blocks:
                r[q.offset:q.offset + q.rows * q.frames] = 0.0
    E = 0.5 * float(r @ r)
    y = np.asarray(y, dtype=np.float64)
    thr = max(EPS_MOD * float(np.sqrt(np.mean(y * y))), np.finfo(np.float64).tiny)
    xp = _reflect(p, y)
    f0, nfr = p.pad_left // p.T, p.frames
    hT = lambda k: time_kernel_closed_form(p.phiT, p.N_pad, k)
    hF = lambda k: time_kernel_closed_form(p.phiF, p.P, k)
    hfr = lambda f: time_kernel_closed_form(p.L_fr[f], p.P, 0)

    # forward intermediates of layer 1
    h1 = [time_kernel_closed_form(p.psi1[n1], p.N_pad, 0) for n1 in range(p.N1)]
    Z1 = [_circ(h1[n1], xp, 2 ** p.k1(n1)) for n1 in range(p.N1)]
    U1 = [np.abs(z) for z in Z1]
    g_U1 = [np.zeros(u.shape[0]) for u in U1]
    off = nfr

    # order 1 (spinned = False)
    S1t = np.stack([_circ(hT(p.k1(n1)), U1[n1], 2 ** (p.log2T - p.k1(n1))).real for n1 in range(p.N1)])
    X = np.zeros((p.P, S1t.shape[1]))
    X[: p.N1] = S1t
    rows1 = -(-p.N1 // p.F)
    gX = np.zeros((p.P, S1t.shape[1]), dtype=np.complex128)
    for f in range(p.n_fr_order1):
        kf = p.k_fr(f)
        W = _circ_rows(hfr(f), X, 2 ** kf)
        gY = np.zeros((W.shape[0], W.shape[1]))
        gY[:rows1, f0:f0 + nfr] = r[off:off + rows1 * nfr].reshape(rows1, nfr)
        off += rows1 * nfr
        if f == 0:
            gW = gY.astype(np.complex128)
        else:
            V0 = np.abs(W)
            V1 = _circ(hT(p.log2T), V0, 1).real
            gV1 = _circ_rows_adj(hF(kf), gY[: V1.shape[0] >> (p.log2F - kf)], 2 ** (p.log2F - kf)).real
            gV0 = _circ_adj(hT(p.log2T), gV1, 1).real
            gW = _phase(W, thr) * gV0
        gX += _circ_rows_adj(hfr(f), gW, 2 ** kf)
    gS1t = gX[: p.N1].real
    for n1 in range(p.N1):
        k1 = p.k1(n1)
        g_U1[n1] += _circ_adj(hT(k1), gS1t[n1], 2 ** (p.log2T - k1)).real

    # order 2, depth-first per (block, filter)
    for bi, blk in enumerate(p.blocks):
        rows2 = -(-blk.n1_max // p.F)
        if blocks is not None and bi not in blocks:
            off += len(p.L_fr) * rows2 * nfr
            continue
        T2 = p.N_pad >> blk.s2
        h2 = [time_kernel_closed_form(p.psi2[blk.n2], p.N_pad, p.k1(n1)) for n1 in range(blk.n1_max)]
        X = np.zeros((p.P, T2), dtype=np.complex128)
        for n1 in range(blk.n1_max):
            X[n1] = _circ(h2[n1], U1[n1], 2 ** (blk.s2 - p.k1(n1)))
        for f in range(len(p.L_fr)):
            kf = p.k_fr(f)
            W = _circ_rows(hfr(f), X, 2 ** kf)
            V0 = np.abs(W)
            n_rows_F = W.shape[0] >> (p.log2F - kf)                     # P / F rows before the crop
            gY = np.zeros((rows2, p.N_pad // p.T))
            gY[:, f0:f0 + nfr] = r[off:off + rows2 * nfr].reshape(rows2, nfr)
            off += rows2 * nfr
            gV1 = np.zeros((n_rows_F, T2))
            gV1[:rows2] = _circ_adj(hT(blk.s2), gY, 2 ** (p.log2T - blk.s2)).real
            gV0 = _circ_rows_adj(hF(kf), gV1, 2 ** (p.log2F - kf)).real
            gW = _phase(W, thr) * gV0
            gXf = _circ_rows_adj(hfr(f), gW, 2 ** kf)
            for n1 in range(blk.n1_max):
                g_U1[n1] += _circ_adj(h2[n1], gXf[n1], 2 ** (blk.s2 - p.k1(n1))).real
    assert off == p.n_coef

    # layer 1 and the padding
    g_xp = np.zeros(p.N_pad)
    for n1 in range(p.N1):
        g_xp += _circ_adj(h1[n1], _phase(Z1[n1], thr) * g_U1[n1], 2 ** p.k1(n1)).real
    return E, _reflect_adj(p, g_xp)

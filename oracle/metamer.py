"""ORACLE (test infrastructure only) — one metamer descent trial.

Heavy-ball momentum with a bold-driver learning rate:
  paper: y_{n+1} = y_n + u_n,  u_n = m u_n + mu_n grad E(y_n)   (self-referential as printed)
  reading R23: u_n = m u_{n-1} - mu_n dE/dy(y_n)  (the paper's "grad E" is the descent direction;
               `g` here is the true gradient), m = 0.9, mu_0 = 0.1
  reading R24 (bold driver, P:124 cites the heuristic only): per signal b,
     accept if E_b <= E_prev_b (E_prev starts at +inf): y_prev <- y, g_prev <- g, E_prev <- E,
                                                       mu <- grow * mu
     else reject: y <- y_prev, g <- g_prev, u <- 0, mu <- shrink * mu
     then u <- m u - mu g ; y <- y + u
Float64 numpy, per-signal state arrays [B, N] and [B].
"""
from __future__ import annotations

import numpy as np


def init_state(y0: np.ndarray, mu0: float = 0.1) -> dict:
    y0 = np.asarray(y0, dtype=np.float64)
    B = y0.shape[0]
    return dict(y=y0.copy(), u=np.zeros_like(y0), y_prev=y0.copy(), g_prev=np.zeros_like(y0),
                mu=np.full(B, mu0), loss_prev=np.full(B, np.inf), accepted=np.zeros(B, np.int32),
                iter=0)


def step(state: dict, E: np.ndarray, g: np.ndarray, momentum: float = 0.9, grow: float = 1.1,
         shrink: float = 0.5) -> dict:
    """Apply one trial given E = E(state['y']) and g = dE/dy at state['y'] (R23, R24)."""
    s = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in state.items()}
    E = np.asarray(E, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64).copy()
    for b in range(s["y"].shape[0]):
        if E[b] <= s["loss_prev"][b]:
            s["accepted"][b] = 1
            s["y_prev"][b] = s["y"][b]
            s["g_prev"][b] = g[b]
            s["loss_prev"][b] = E[b]
            s["mu"][b] *= grow
        else:
            s["accepted"][b] = 0
            s["y"][b] = s["y_prev"][b]
            g[b] = s["g_prev"][b]
            s["u"][b] = 0.0
            s["mu"][b] *= shrink
        s["u"][b] = momentum * s["u"][b] - s["mu"][b] * g[b]
        s["y"][b] = s["y"][b] + s["u"][b]
    s["iter"] += 1
    return s


# ----------------------------------------------------------------------------------------------
# Initialisation (§2.3 Reconstruction): "Starting from a colored Gaussian noise y0(t) whose
# power spectral density matches S1 x(t, lambda)". Reading R25 (SPEC S:404-412 asks only for
# per-band gains on a white noise's spectrum, bands from the psi1 supports, each band within 20%):
#   1. profile: r[rho] = RMS over frames of the order-1 beta = 0 path S1x[rho, t] (Eq.3), and
#      a[n1] = r interpolated linearly at rho = n1 / F (row rho of phi_F's stride-F output sits
#      at n1 = rho F), clamped to the last row;
#   2. gain per band: g[n1] = a[n1] / sqrt((pi/4) nu[n1]), nu[n1] = (1/N_pad) sum_m |psi1_hat[m]|^2,
#      so that white unit-variance noise shaped by g gives E|y * psi_n1| = a[n1] (the modulus of a
#      circular complex Gaussian has mean sqrt(pi/4) times its RMS);
#   3. spectral gain G[m] = sum_n1 g[n1] |psi1_hat(w)|^2 / (sum_n1 |psi1_hat(w)|^2 + delta) at
#      w = min(m, N_pad - m) / N_pad (even in m, so y0 is real), delta = 1e-3 max_w sum |psi1_hat|^2;
#   4. y0 = Re IFFT_{N_pad}(FFT_{N_pad}(white) G) on [pad_left, pad_left + N).
# All-zero profile: y0 = 1e-4 white[pad_left : pad_left + N] (SPEC S:408 fallback).
# The white noise (the random numbers the method draws) is an input: [B, N_pad] standard normal.
# ----------------------------------------------------------------------------------------------

def colored_noise(plan, S_target: np.ndarray, white: np.ndarray) -> np.ndarray:
    """y0 [B, N] (float64) per the reading above; S_target [B, n_coef] packed (R15)."""
    from .plan import response
    p = plan
    S = np.atleast_2d(np.asarray(S_target, dtype=np.float64))
    w = np.atleast_2d(np.asarray(white, dtype=np.float64))
    B, Np, N = S.shape[0], p.N_pad, p.N
    q1 = p.paths[1]                                        # order 1, beta = 0 (R12, R15)
    assert q1.order == 1 and q1.spin == 0
    psi2 = np.stack([np.abs(response(f, Np)) ** 2 for f in p.psi1])          # [N1, N_pad]
    m = np.arange(Np)
    mirror = np.minimum(m, Np - m)
    psi2m = psi2[:, mirror]                                # |psi_hat(|w|)|^2
    nu = psi2.sum(axis=1) / Np
    den = psi2m.sum(axis=0)
    delta = 1e-3 * den.max()
    out = np.empty((B, N))
    for b in range(B):
        rows = S[b, q1.offset:q1.offset + q1.rows * q1.frames].reshape(q1.rows, q1.frames)
        r = np.sqrt((rows ** 2).mean(axis=1))
        crop = w[b, p.pad_left:p.pad_left + N]
        if not np.any(r > 0):
            out[b] = 1e-4 * crop
            continue
        a = np.interp(np.arange(p.N1) / p.F, np.arange(q1.rows), r)
        g = a / np.sqrt(np.pi / 4 * nu)
        G = (g[:, None] * psi2m).sum(axis=0) / (den + delta)
        y = np.fft.ifft(np.fft.fft(w[b]) * G).real
        out[b] = y[p.pad_left:p.pad_left + N]
    return out

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

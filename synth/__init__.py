"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the JTFS method (no filter, no transform, no loss): it only
draws audio-like signals. Recipes follow SURVEY.md §8(d) "Inputs: concrete synthetic stand-ins"
and BASELINE.json `configs` (the paper names no dataset; its workload is "any audio recording",
PAPER.md:7). Everything is generated in float64 with numpy's PCG64 and returned as float32.

Seeds: target x of signal b in config c uses seed 1000*c + b; the evaluation point y uses
seed 1000*c + b + 500000.
"""
from __future__ import annotations

import numpy as np

SR = 22050.0

# (N, J, Q, J_fr, Q_fr, T, F, B) -- BASELINE.json configs[0..4]
CONFIGS = {
    "c1": dict(N=4096, J=6, Q=8, J_fr=3, Q_fr=1, T=64, F=8, B=1),
    "c2": dict(N=65536, J=12, Q=16, J_fr=5, Q_fr=2, T=2048, F=16, B=8),
    "c3": dict(N=131072, J=13, Q=12, J_fr=5, Q_fr=1, T=4096, F=8, B=16),
    "c4": dict(N=262144, J=14, Q=16, J_fr=6, Q_fr=2, T=8192, F=16, B=64),
    "c5": dict(N=1048576, J=14, Q=16, J_fr=6, Q_fr=2, T=16384, F=32, B=256),
}

# SURVEY.md Appendix A tiny configurations (N, J, Q, J_fr, Q_fr, T, F)
TINY = {
    "t1": dict(N=128, J=3, Q=1, J_fr=2, Q_fr=1, T=4, F=2),
    "t2": dict(N=256, J=4, Q=2, J_fr=2, Q_fr=1, T=8, F=2),
    "spec": dict(N=1024, J=5, Q=2, J_fr=3, Q_fr=1, T=8, F=2),
}

# plan variants described by the listings: a second-layer quality factor Q2 > 1
# and second-layer scales beyond log2 T (j2 > log2 T, reading R13's common stride)
VARIANTS = {
    "q2": dict(N=1024, J=5, Q=2, J_fr=3, Q_fr=1, T=8, F=2, Q2=2),
    "q2b": dict(N=4096, J=6, Q=8, J_fr=3, Q_fr=1, T=64, F=8, Q2=4),
    "j2gtT": dict(N=2048, J=6, Q=4, J_fr=2, Q_fr=1, T=8, F=2),
    "wide": dict(N=4096, J=6, Q=8, J_fr=3, Q_fr=1, T=64, F=1),     # ceil(N1/F) = 38 > 32 rows per path
}

_CINDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


def plan_args(cfg: dict) -> tuple:
    """(N, J, Q, J_fr, Q_fr, T, F[, Q2]) -- Q2 only when the config sets it (default 1)."""
    a = (cfg["N"], cfg["J"], cfg["Q"], cfg["J_fr"], cfg["Q_fr"], cfg["T"], cfg["F"])
    return a + (cfg["Q2"],) if cfg.get("Q2", 1) != 1 else a


def _peak_normalise(x: np.ndarray, peak: float = 0.5) -> np.ndarray:
    m = np.max(np.abs(x))
    return x * (peak / m) if m > 0 else x


def _adsr(n_len: int, sr: float) -> np.ndarray:
    a, d, s, r = int(0.010 * sr), int(0.080 * sr), 0.6, int(0.150 * sr)
    env = np.full(n_len, s)
    ia = min(a, n_len)
    env[:ia] = np.linspace(0.0, 1.0, ia, endpoint=False)
    idd = min(a + d, n_len)
    if idd > ia:
        env[ia:idd] = np.linspace(1.0, s, idd - ia, endpoint=False)
    rr = min(r, n_len)
    env[n_len - rr:] *= np.linspace(1.0, 0.0, rr)
    return env


def _voice(rng: np.random.Generator, N: int, ioi: tuple) -> np.ndarray:
    """Monophonic harmonic note sequence: f0 ~ logU(80, 1000) Hz, 8 partials at 1/k, ADSR."""
    out = np.zeros(N)
    t = 0.0
    while True:
        onset = int(t * SR)
        if onset >= N:
            break
        dur = rng.uniform(0.2, 0.8)
        n_len = min(int(dur * SR), N - onset)
        f0 = np.exp(rng.uniform(np.log(80.0), np.log(1000.0)))
        n = np.arange(n_len)
        note = np.zeros(n_len)
        for k in range(1, 9):
            phase = rng.uniform(0, 2 * np.pi)
            if k * f0 >= SR / 2:
                continue
            note += np.sin(2 * np.pi * k * f0 * n / SR + phase) / k
        if n_len > 0:
            out[onset:onset + n_len] += note * _adsr(n_len, SR)
        t += rng.uniform(*ioi)
    return out


def _pink(rng: np.random.Generator, N: int) -> np.ndarray:
    w = rng.standard_normal(N)
    W = np.fft.rfft(w)
    f = np.arange(W.shape[0], dtype=np.float64)
    f[0] = 1.0
    W = W / np.sqrt(f)
    W[0] = 0.0
    return np.fft.irfft(W, n=N)


def _rms(x: np.ndarray) -> float:
    return float(np.sqrt(np.mean(x * x))) if x.size else 0.0


def _bursts(rng: np.random.Generator, N: int) -> np.ndarray:
    out = np.zeros(N)
    t = rng.exponential(0.5)
    while int(t * SR) < N:
        onset = int(t * SR)
        dur = rng.uniform(0.020, 0.200)
        n_len = min(int(dur * SR), N - onset)
        tt = np.arange(n_len) / SR
        out[onset:onset + n_len] += rng.standard_normal(n_len) * np.exp(-tt / (dur / 3))
        t += rng.exponential(0.5)
    return out


def signal(config: str, b: int, which: str = "x") -> np.ndarray:
    """One synthetic signal (float32) of config `config`, batch index b; which = 'x' or 'y'."""
    seed = 1000 * _CINDEX[config] + b + (500000 if which == "y" else 0)
    rng = np.random.default_rng(seed)
    N = CONFIGS[config]["N"]
    if config == "c1":
        n = np.arange(N)
        x = (0.1 * rng.standard_normal(N) + 0.5 * np.sin(2 * np.pi * 440 * n / SR)
             + 0.25 * np.sin(2 * np.pi * 1320 * n / SR))
        return x.astype(np.float32)
    if which == "y" and config == "c3":
        # metamer init: white Gaussian noise with the target's RMS
        xt = signal(config, b, "x").astype(np.float64)
        return (rng.standard_normal(N) * _rms(xt)).astype(np.float32)
    if config == "c2":
        notes = _voice(rng, N, (0.15, 0.6))
        noise = _pink(rng, N)
        noise *= _rms(notes) * 10 ** (-30 / 20) / max(_rms(noise), 1e-30)
        x = notes + noise
    else:
        x = sum(_voice(rng, N, (0.1, 0.5)) for _ in range(3))
        if config in ("c4", "c5"):
            bu = _bursts(rng, N)
            bu *= _rms(x) * 10 ** (-12 / 20) / max(_rms(bu), 1e-30)
            x = x + bu
    return _peak_normalise(x).astype(np.float32)


def batch(config: str, B: int | None = None, which: str = "x", start: int = 0) -> np.ndarray:
    B = CONFIGS[config]["B"] if B is None else B
    return np.stack([signal(config, start + b, which) for b in range(B)])


def noise(N: int, B: int = 1, seed: int = 0, scale: float = 0.1) -> np.ndarray:
    """White Gaussian test signals for tiny configs."""
    rng = np.random.default_rng(seed)
    return (scale * rng.standard_normal((B, N))).astype(np.float32)

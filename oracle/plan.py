"""ORACLE (test infrastructure only) — JTFS plan: filterbanks, scales, padding, blocks, paths.

Every rule cites PAPER.md (P:line) or the DESIGN.md reading it implements (R1..R28, taken from
SURVEY.md §8(c)). Float64 throughout; integer decisions are made in float64 with a fixed
operation order so that any other implementation following the same readings gets the same
integers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SIGMA0 = 0.1                # P:168  sigma0 = 0.1
R_PSI = math.sqrt(0.5)      # P:169  r_psi = sqrt(0.5); the listing's `r` is r_psi (reading R1)
QSUM = 4                    # periodisation terms q in [-QSUM, QSUM] (all sigma here are <= 0.15)


def anden_generator(J: int, Q: int) -> list[tuple[float, float]]:
    """(xi, sigma) sequence of PAPER.md:167-191 (§3.1 listing), verbatim in float64 (R1, R2)."""
    out = []
    xi = max(1. / (1. + math.pow(2., 3. / Q)), 0.35)
    factor = 1. / math.pow(2, 1. / Q)
    sigma = (1 - factor) / (1 + factor) * xi / math.sqrt(2 * math.log(1. / R_PSI))
    sigma_min = SIGMA0 / 2 ** J
    if sigma <= sigma_min:
        xi = sigma
    else:
        out.append((xi, sigma))
        # High-frequency (constant-Q) region
        while sigma > (sigma_min * math.pow(2, 1 / Q)):
            xi /= math.pow(2, 1 / Q)
            sigma /= math.pow(2, 1 / Q)
            out.append((xi, sigma))
    # Low-frequency (constant-bandwidth) region
    elbow_xi = xi
    for q in range(Q - 1):
        xi -= 1 / Q * elbow_xi
        out.append((xi, sigma_min))
    return out


def spin(filters: list[tuple[float, float]]) -> list[tuple[float, float]]:
    """Wavelet spinning: the sequence followed by its negated-xi twins."""
    return list(filters) + [(-xi, s) for xi, s in filters]


def dyadic_scale(xi: float, sigma: float) -> int:
    """Reading R3 (P:200 'depends on the resolution of the cutoff frequency'):
    j = max(0, floor(-log2(min(|xi| + 5 sigma, 1/2))) - 1)."""
    return max(0, math.floor(-math.log2(min(abs(xi) + 5 * sigma, 0.5))) - 1)


def next_pow2(n: int) -> int:
    p = 1
    while p < n:
        p *= 2
    return p


def ilog2(n: int) -> int:
    return n.bit_length() - 1


class PlanError(ValueError):
    pass


@dataclass
class Filter:
    xi: float
    sigma: float
    j: int
    spin: int = 1
    kind: str = "psi"   # 'psi' (Morlet band-pass, Eq.1) or 'phi' (Gaussian low-pass)


@dataclass
class Block:
    n2: int
    n1_max: int
    s2: int         # common stride exponent of the block (reading R13)
    j2: int


@dataclass
class Path:
    order: int
    n2: int         # -1 for orders 0, 1
    n_fr: int       # index into L_fr; -1 for order 0
    spin: int
    j2: int
    j_fr: int
    rows: int
    frames: int
    offset: int
    block: int = -1  # index into blocks for order 2


@dataclass
class Plan:
    N: int
    J: int
    Q: int
    J_fr: int
    Q_fr: int
    T: int
    F: int
    log2T: int
    log2F: int
    psi1: list[Filter]
    psi2: list[Filter]
    psi_fr_plus: list[Filter]
    L_fr: list[Filter]          # [phi_F, psi+_0.., psi-_0..] (reading R12)
    phiT: Filter
    phiF: Filter
    N_pad: int
    pad_left: int
    P: int
    blocks: list[Block]
    paths: list[Path] = field(default_factory=list)
    n_coef: int = 0

    @property
    def N1(self) -> int:
        return len(self.psi1)

    @property
    def frames(self) -> int:
        return self.N // self.T

    def k1(self, n1: int) -> int:
        """First-layer subsampling exponent k1 = min(j1, log2 T)."""
        return min(self.psi1[n1].j, self.log2T)

    def k_fr(self, f: int) -> int:
        """Frequential subsampling exponent k_fr = min(j_fr, log2 F)."""
        return min(self.L_fr[f].j, self.log2F)

    @property
    def n_fr_order1(self) -> int:
        """Number of frequential filters with xi >= 0: phi_F + psi+."""
        return 1 + len(self.psi_fr_plus)


def make_plan(N: int, J: int, Q: int, J_fr: int, Q_fr: int, T: int, F: int, Q2: int = 1) -> Plan:
    """Build the plan (readings R1-R3, R6-R8, R10-R16). Q2 = Q^{tm,2}, the
    second-layer temporal quality factor ("its own hyperparameters"; R7: 1 by default)."""
    def ispow2(v):
        return v >= 1 and (v & (v - 1)) == 0
    if J < 1 or Q < 1 or J_fr < 1 or Q_fr < 1:
        raise PlanError("J, Q, J_fr, Q_fr must be >= 1")
    if not 1 <= Q2 <= 16:
        raise PlanError("need 1 <= Q2 <= 16")
    if not ispow2(T):
        raise PlanError("T must be a power of two")
    if not ispow2(F):
        raise PlanError("F must be a power of two")
    log2T, log2F = ilog2(T), ilog2(F)
    if not (1 <= log2T <= J):
        raise PlanError("need 1 <= log2(T) <= J")
    if not (0 <= log2F <= J_fr):
        raise PlanError("need 0 <= log2(F) <= J_fr")
    if N < T or N % T != 0:
        raise PlanError("N must be a positive multiple of T")

    psi1 = [Filter(xi, s, dyadic_scale(xi, s)) for xi, s in anden_generator(J, Q)]
    psi2 = [Filter(xi, s, dyadic_scale(xi, s)) for xi, s in anden_generator(J, Q2)]  # Q^{tm,2} (R7)
    psi_fr_plus = [Filter(xi, s, dyadic_scale(xi, s)) for xi, s in anden_generator(J_fr, Q_fr)]
    # R6: sigma_phiT = sigma0 / T, sigma_phiF = sigma0 / F ; R3: j(phi_T)=log2T, j(phi_F)=log2F
    phiT = Filter(0.0, SIGMA0 / T, log2T, 0, "phi")
    phiF = Filter(0.0, SIGMA0 / F, log2F, 0, "phi")
    L_fr = ([phiF] + [Filter(f.xi, f.sigma, f.j, 1) for f in psi_fr_plus]
            + [Filter(-f.xi, f.sigma, f.j, -1) for f in psi_fr_plus])

    # R10: N_pad = next_pow2(N + 2 ceil(4 max(2^J, T) / (0.2 pi))), pad_left = T floor((N_pad-N)/(2T))
    N_pad = next_pow2(N + 2 * math.ceil(4 * max(2 ** J, T) / (0.2 * math.pi)))
    if N_pad > 2 ** 22:
        raise PlanError("N_pad exceeds 2^22")
    pad_left = T * ((N_pad - N) // (2 * T))
    # R11: P = next_pow2(N1 + 2 ceil(4 / (2 pi sigma_fr_min)))
    sig_fr_min = min([f.sigma for f in psi_fr_plus] + [phiF.sigma])
    P = next_pow2(len(psi1) + 2 * math.ceil(4 / (2 * math.pi * sig_fr_min)))

    js = [f.j for f in psi1]
    if any(js[i] > js[i + 1] for i in range(len(js) - 1)):
        raise PlanError("internal: j1 not nondecreasing")
    blocks = []
    for n2, f2 in enumerate(psi2):
        n1_max = sum(1 for j1 in js if f2.j > j1)      # admissibility j2 > j1
        if n1_max > 0:                                  # empty blocks omitted
            blocks.append(Block(n2, n1_max, min(f2.j, log2T), f2.j))
    plan = Plan(N, J, Q, J_fr, Q_fr, T, F, log2T, log2F, psi1, psi2, psi_fr_plus, L_fr, phiT,
                phiF, N_pad, pad_left, P, blocks)
    _make_paths(plan)
    return plan


def _make_paths(plan: Plan) -> None:
    """Path table in yield order (reading R15); rows/frames after unpadding (R16)."""
    fr = plan.frames
    off = 0
    paths = [Path(0, -1, -1, 0, -1, -1, 1, fr, off)]
    off += fr
    rows1 = -(-plan.N1 // plan.F)
    for f in range(plan.n_fr_order1):
        flt = plan.L_fr[f]
        paths.append(Path(1, -1, f, flt.spin, -1, flt.j, rows1, fr, off))
        off += rows1 * fr
    for bi, blk in enumerate(plan.blocks):
        rows2 = -(-blk.n1_max // plan.F)
        for f, flt in enumerate(plan.L_fr):
            paths.append(Path(2, blk.n2, f, flt.spin, blk.j2, flt.j, rows2, fr, off, bi))
            off += rows2 * fr
    plan.paths = paths
    plan.n_coef = off


# ----------------------------------------------------------------------------------------------
# Fourier responses (Eq.1 P:59-67 with reading R4/R5; Gaussian low-pass R6; levels R9)
# ----------------------------------------------------------------------------------------------

def _gauss_periodized(omega: np.ndarray, sigma: float) -> np.ndarray:
    s = np.zeros_like(omega)
    for q in range(-QSUM, QSUM + 1):
        s += np.exp(-((omega + q) ** 2) / (2.0 * sigma * sigma))
    return s


def kappa(xi: float, sigma: float) -> float:
    """R4: kappa = sum_q G(q - xi) / sum_q G(q): makes the level-0 DC bin exactly zero
    (Eq.1's 'one vanishing moment')."""
    z = np.zeros(1)
    return float(_gauss_periodized(z - xi, sigma)[0] / _gauss_periodized(z, sigma)[0])


def response(flt: Filter, L0: int) -> np.ndarray:
    """Level-0 response on an L0-point grid, bin m <-> omega = m/L0 cycles/sample, periodised
    over the unit circle. Morlet: 2[G(w - xi) - kappa G(w)] (R4, R5: Gaussian peak 2).
    Gaussian low-pass: G(w) (phi_hat(0) = 1). Always real-valued."""
    omega = np.arange(L0, dtype=np.float64) / L0
    if flt.kind == "phi":
        return _gauss_periodized(omega, flt.sigma)
    k = kappa(flt.xi, flt.sigma)
    return 2.0 * (_gauss_periodized(omega - flt.xi, flt.sigma) - k * _gauss_periodized(omega, flt.sigma))


def level(h0: np.ndarray, k: int) -> np.ndarray:
    """R9: level k = periodisation (fold-SUM) of level 0 onto L0/2^k bins."""
    L0 = h0.shape[-1]
    return h0.reshape(2 ** k, L0 // 2 ** k).sum(axis=0)


def time_kernel_closed_form(flt: Filter, L0: int, k: int) -> np.ndarray:
    """Closed-form time-domain kernel of `level(response(flt, L0), k)` by Poisson summation
    (SURVEY.md §8(c) O1): h_k[n] = 2^k sum_r H(2^k n + r L0), with
    H_psi(t) = 2 sigma sqrt(2 pi) exp(-2 pi^2 sigma^2 t^2) (exp(2 pi i xi t) - kappa),
    H_phi(t) = sigma sqrt(2 pi) exp(-2 pi^2 sigma^2 t^2). Used by brute.py and the pins."""
    L = L0 // 2 ** k
    n = np.arange(L, dtype=np.float64)
    s = flt.sigma
    out = np.zeros(L, dtype=np.complex128)
    half_support = 1.35 / s + 2.0        # e^{-36} cut (R26); |t| beyond this is < 2e-16 * peak
    rmax = int(math.ceil((half_support + L0) / L0)) + 1
    kap = 0.0 if flt.kind == "phi" else kappa(flt.xi, flt.sigma)
    for r in range(-rmax, rmax + 1):
        t = 2 ** k * n + r * L0
        env = s * math.sqrt(2 * math.pi) * np.exp(-2 * math.pi ** 2 * s * s * t * t)
        if flt.kind == "phi":
            out += env
        else:
            out += 2.0 * env * (np.exp(2j * math.pi * flt.xi * t) - kap)
    return 2 ** k * out

"""ORACLE (test infrastructure only) — JTFS forward, Euclidean loss and gradient in float64.

Plain PyTorch CPU ops in float64 (torch.fft as the library FFT). The forward follows the paper's
listings step by step:
  first layer            PAPER.md:202-213 (§3.2)      rfft -> cdgmm -> subsample_fourier -> ifft -> modulus
  second layer, time     PAPER.md:221-247 (§3.3)      width-first, `if j2 > j1`, stack, n1_max
  second layer, freq     PAPER.md:264-305 (§3.4)      swap, pad to phi['N'] (=P), cfft/rfft, per filter
                                                      cdgmm -> subsample_fourier -> ifft
  main algorithm         PAPER.md:310-352 (§3.5)      yield order S0, order-1 (spinned=False), order-2
  averaging              Eq.3, Eq.4 P:108-114 (phi_T over time, phi_F over log-frequency)
with the readings R1-R28 listed in DESIGN.md (taken from SURVEY.md §8(c)). Backward is PyTorch
reverse-mode autodiff of this forward, as the paper itself does ("We rely on the
PyTorch backend of Kymatio to perform gradient backpropagation"); gradient checkpointing over
column chunks of the frequential stage only bounds memory, it does not change the arithmetic.

Parity status: the forward and gradient are pinned by tests/test_oracle_*.py (direct-sum route
brute.py, closed-form kernels, finite differences, nullity, invariance, special inputs).
Absolute coefficient values are "parity unpinned" against a paper-printed number (none exists).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .plan import Plan, make_plan, response, level

F64 = torch.float64
C128 = torch.complex128


class _Recompute(torch.autograd.Function):
    """Memory-only device: run `fn(inp)` without saving intermediates, recompute it in backward
    (plain gradient checkpointing; the arithmetic is unchanged)."""

    @staticmethod
    def forward(ctx, inp, fn):
        ctx.fn = fn
        ctx.save_for_backward(inp)
        with torch.no_grad():
            return fn(inp)

    @staticmethod
    def backward(ctx, g):
        (inp,) = ctx.saved_tensors
        with torch.enable_grad():
            x = inp.detach().requires_grad_(True)
            out = ctx.fn(x)
            (gx,) = torch.autograd.grad(out, x, g)
        return gx, None


# Reading R22 (modulus subgradient): the phase z/|z| of the modulus adjoint is 0 where
# |z| < EPS_MOD * RMS(y_b) (per signal b, the "block" of S:372), at every modulus site (Z1, order-1
# W, joint W). Everywhere else the adjoint is exactly PyTorch's (Kymatio's autograd):
# g * z/|z|. The dead zone sits at the float64 rounding floor of the transforms (~1e-16 RMS), so it
# only decides cells whose value is rounding noise (exactly silent stretches), where the phase -- and
# with it the gradient -- is not determined by the arithmetic; for generic inputs it changes nothing
# (tests/test_oracle_grad.py, R22 gives the measured effect at c2-c5).
EPS_MOD = 1e-12


class _Modulus(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z, thr):
        a = z.abs()
        ctx.save_for_backward(z, a, thr)
        return a

    @staticmethod
    def backward(ctx, g):
        z, a, thr = ctx.saved_tensors
        keep = a >= thr
        phase = torch.where(keep, z / torch.where(keep, a, torch.ones_like(a)), torch.zeros_like(z))
        return g * phase, None


def modulus(z: torch.Tensor, thr: torch.Tensor) -> torch.Tensor:
    """Complex modulus |z| (Eq.2, listing P:210) with the R22 adjoint; `thr` [B] broadcasts
    per signal (thr = 0 gives torch.abs's own adjoint, sgn(0) = 0)."""
    thr = thr.reshape((-1,) + (1,) * (z.dim() - 1)).to(z.real.dtype)
    return _Modulus.apply(z, torch.clamp(thr, min=torch.finfo(z.real.dtype).tiny))


def mod_threshold(y: torch.Tensor) -> torch.Tensor:
    """R22 dead-zone radius per signal: EPS_MOD * RMS(y_b)."""
    return EPS_MOD * y.detach().pow(2).mean(dim=1).sqrt()


def subsample_fourier(X: torch.Tensor, k: int, dim: int = -1) -> torch.Tensor:
    """P:199, P:208 'subsampling ... in the Fourier domain by reshaping and summation';
    SPEC S:65: out[m] = (1/k) sum_b X[m + b L/k] (equals decimation in time)."""
    if k == 1:
        return X
    dim = dim % X.dim()
    L = X.shape[dim]
    return X.unflatten(dim, (k, L // k)).mean(dim)


def reflect_index(plan: Plan) -> torch.Tensor:
    """R10: half-sample symmetric extension ([1,2,3,4] -> [2,1,1,2,3,4,4,3]),
    sample i of the padded signal = x[e(i - pad_left)], e = 2N-periodic even extension."""
    N = plan.N
    t = (np.arange(plan.N_pad) - plan.pad_left) % (2 * N)
    src = np.where(t < N, t, 2 * N - 1 - t)
    return torch.from_numpy(src.astype(np.int64))


class Oracle:
    """Float64 JTFS of one plan. `forward(x)` -> packed coefficients [B, n_coef] (R15 order)."""

    def __init__(self, plan_or_args, chunk_elems: int = 1 << 23):
        self.plan = plan_or_args if isinstance(plan_or_args, Plan) else make_plan(*plan_or_args)
        p = self.plan
        self.chunk_elems = chunk_elems
        self._cache: dict = {}
        self.src = reflect_index(p)

    # ---------------------------------------------------------------- filters (R4-R9)
    def _resp(self, key, flt, L0):
        if key not in self._cache:
            self._cache[key] = torch.from_numpy(response(flt, L0))
        return self._cache[key]

    def psi1(self, n1):
        return self._resp(("psi1", n1), self.plan.psi1[n1], self.plan.N_pad)

    def psi2(self, n2):
        return self._resp(("psi2", n2), self.plan.psi2[n2], self.plan.N_pad)

    def phiT(self):
        return self._resp(("phiT",), self.plan.phiT, self.plan.N_pad)

    def fr(self, f):
        return self._resp(("fr", f), self.plan.L_fr[f], self.plan.P)

    def phiF(self):
        return self._resp(("phiF",), self.plan.phiF, self.plan.P)

    @staticmethod
    def lev(h0: torch.Tensor, k: int) -> torch.Tensor:
        """R9: fold-SUM periodisation of level 0 onto L0/2^k bins ('levels'[k])."""
        return torch.from_numpy(level(h0.numpy(), k))

    # ---------------------------------------------------------------- helpers
    def _unpad_frames(self, A: torch.Tensor) -> torch.Tensor:
        """R16: keep frames [pad_left/T, pad_left/T + N/T)."""
        p = self.plan
        f0 = p.pad_left // p.T
        return A[..., f0:f0 + p.frames]

    def _phiF_rows(self, V: torch.Tensor, kf: int) -> torch.Tensor:
        """phi_F along rows (dim -2) at level k_f, decimated to stride F (Eq.3/Eq.4, R17)."""
        p = self.plan
        Vh = torch.fft.fft(V, dim=-2)
        h = self.lev(self.phiF(), kf).to(C128)[:, None]
        return torch.fft.ifft(subsample_fourier(Vh * h, 2 ** (p.log2F - kf), dim=-2), dim=-2).real

    def _phiT_time(self, V: torch.Tensor, s: int) -> torch.Tensor:
        """phi_T along time (dim -1) at level s, decimated to stride T (Eq.3/Eq.4)."""
        p = self.plan
        Vh = torch.fft.fft(V, dim=-1)
        h = self.lev(self.phiT(), s).to(C128)
        return torch.fft.ifft(subsample_fourier(Vh * h, 2 ** (p.log2T - s), dim=-1), dim=-1).real

    def _freq_filter(self, X_hat: torch.Tensor, f: int) -> torch.Tensor:
        """cdgmm(X_hat, psi['levels'][0]) -> subsample_fourier(2^k_fr) -> ifft (rows)."""
        kf = self.plan.k_fr(f)
        h = self.fr(f).to(C128)[:, None]
        return torch.fft.ifft(subsample_fourier(X_hat * h, 2 ** kf, dim=-2), dim=-2)

    # ---------------------------------------------------------------- stages
    def layer1(self, x: torch.Tensor):
        """Padding (R10) + first layer + S0 + time-averaged S1 (Eq.3 time part)."""
        p = self.plan
        self._thr = mod_threshold(x)                                         # R22
        xp = x[:, self.src]
        U0_hat = torch.fft.fft(xp.to(C128))                                  # P:203 (rfft, full circle)
        S0 = torch.fft.ifft(subsample_fourier(U0_hat * self.phiT().to(C128), p.T)).real
        U1_hats, S1t = [], []
        for n1 in range(p.N1):
            k1 = p.k1(n1)
            U1_c = U0_hat * self.psi1(n1).to(C128)                           # P:207 cdgmm
            U1_hat = subsample_fourier(U1_c, 2 ** k1)
            U1_m = modulus(torch.fft.ifft(U1_hat), self._thr)
            U1_hat = torch.fft.fft(U1_m.to(C128))                            # P:211 (rfft, full circle)
            U1_hats.append(U1_hat)
            # S1 time part: U1 * phi_T at level k1, stride T (Eq.3; R14)
            hT = self.lev(self.phiT(), k1).to(C128)
            S1t.append(torch.fft.ifft(subsample_fourier(U1_hat * hT, 2 ** (p.log2T - k1))).real)
        return S0, U1_hats, torch.stack(S1t, dim=1)                          # S1t [B, N1, N_pad/T]

    def order1(self, S1t: torch.Tensor) -> list[torch.Tensor]:
        """frequency_scattering(S_1, spinned=False) + R14 averaging."""
        p = self.plan
        B, N1, nt = S1t.shape
        X_pad = torch.cat([S1t, S1t.new_zeros(B, p.P - N1, nt)], dim=1)
        X_hat = torch.fft.fft(X_pad.to(C128), dim=1)                        # P:285 rfft (full circle)
        rows = -(-N1 // p.F)
        out = []
        for f in range(p.n_fr_order1):                                       # xi >= 0 prefix
            W = self._freq_filter(X_hat, f)
            if f == 0:      # beta = 0: S1 = U1 *t phi_T *lambda phi_F  (Eq.3)
                Y = W.real
            else:           # alpha = 0, beta > 0: phi_F * phi_T * |psi_beta * (phi_T * U1)|  (R14)
                V = modulus(W, self._thr)
                Vh = torch.fft.fft(V.to(C128), dim=-1)
                V = torch.fft.ifft(Vh * self.lev(self.phiT(), p.log2T).to(C128), dim=-1).real
                Y = self._phiF_rows(V, p.k_fr(f))
            out.append(self._unpad_frames(Y[:, :rows, :]))
        return out

    def layer2_block(self, U1_hats, bi: int) -> torch.Tensor:
        """time_scattering_widthfirst, one n2 block: Y2 [B, n1_max, T2] complex."""
        p = self.plan
        blk = p.blocks[bi]
        Y2 = []
        for n1 in range(blk.n1_max):                                         # j2 > j1
            k1 = p.k1(n1)
            h = self.lev(self.psi2(blk.n2), k1).to(C128)                    # levels[k1]
            U2_hat = subsample_fourier(U1_hats[n1] * h, 2 ** (blk.s2 - k1))  # R13 common stride
            Y2.append(torch.fft.ifft(U2_hat))
        return torch.stack(Y2, dim=1)                                        # P:241 stack

    def _joint_chunk(self, Y2c: torch.Tensor, rows: int) -> torch.Tensor:
        """Spinned frequency scattering of a column chunk of one block (spinned=True),
        modulus (Eq.2) and phi_F over rows (Eq.4), kept rows only: [B, n_filters, rows, cols]."""
        p = self.plan
        B, n1_max, nc = Y2c.shape
        X_pad = torch.cat([Y2c, Y2c.new_zeros(B, p.P - n1_max, nc)], dim=1)
        X_hat = torch.fft.fft(X_pad, dim=1)                                  # P:282 cfft
        outs = []
        for f in range(len(p.L_fr)):
            V = modulus(self._freq_filter(X_hat, f), self._thr)             # |U1 *t psi_a *l psi_b|
            outs.append(self._phiF_rows(V, p.k_fr(f))[:, :rows, :])
        return torch.stack(outs, dim=1)

    def order2_block(self, Y2: torch.Tensor, bi: int) -> list[torch.Tensor]:
        p = self.plan
        blk = p.blocks[bi]
        rows = -(-blk.n1_max // p.F)
        T2 = Y2.shape[-1]
        chunk = max(1, min(T2, self.chunk_elems // (p.P * len(p.L_fr) * max(1, Y2.shape[0]))))
        chunk = 1 << (chunk.bit_length() - 1)
        pieces = []
        for c0 in range(0, T2, chunk):
            Yc = Y2[..., c0:c0 + chunk]
            if Yc.requires_grad and chunk < T2:
                pieces.append(_Recompute.apply(Yc, lambda t: self._joint_chunk(t, rows)))
            else:
                pieces.append(self._joint_chunk(Yc, rows))
        O = torch.cat(pieces, dim=-1)                                        # [B, nf, rows, T2]
        S = self._unpad_frames(self._phiT_time(O, blk.s2))                   # phi_T at level s2
        return [S[:, f] for f in range(len(p.L_fr))]

    # ---------------------------------------------------------------- public
    def forward(self, x, blocks=None) -> torch.Tensor:
        """Packed coefficients [B, n_coef] in path order (R15). `blocks` restricts order 2 to a
        subset of block indices (others left 0) — used to sample large configs."""
        p = self.plan
        x = torch.as_tensor(x).to(F64)
        if x.dim() == 1:
            x = x[None]
        S0, U1_hats, S1t = self.layer1(x)
        parts = [self._unpad_frames(S0)[:, None, :]]
        parts += self.order1(S1t)
        bl = range(len(p.blocks)) if blocks is None else blocks
        o2 = {}
        for bi in bl:
            Y2 = self.layer2_block(U1_hats, bi)
            o2[bi] = self.order2_block(Y2, bi)
            del Y2
        for bi, blk in enumerate(p.blocks):
            rows = -(-blk.n1_max // p.F)
            if bi in o2:
                parts += o2[bi]
            else:
                parts += [x.new_zeros(x.shape[0], rows, p.frames)] * len(p.L_fr)
        S = torch.cat([q.reshape(x.shape[0], -1) for q in parts], dim=1)
        assert S.shape[1] == p.n_coef
        return S

    def loss_weights(self) -> torch.Tensor:
        """1 for coefficients in the loss (orders 1, 2), 0 for S0 (R19)."""
        w = torch.ones(self.plan.n_coef, dtype=F64)
        w[: self.plan.frames] = 0
        return w

    def loss(self, S_y: torch.Tensor, S_target: torch.Tensor) -> torch.Tensor:
        """R19: E_b = 1/2 sum over orders 1,2 of (S(y_b) - S_target_b)^2."""
        r = (S_y - torch.as_tensor(S_target).to(F64)) * self.loss_weights()
        return 0.5 * (r * r).sum(dim=1)

    def loss_grad_subset(self, y, S_target, blocks):
        """R19's loss restricted to order 1 and the order-2 paths of `blocks` (used to sample the
        large configurations): (E [B], dE/dy [B, N]) by reverse-mode autodiff."""
        w = _subset_weights(self.plan, blocks)
        y = torch.as_tensor(y).to(F64).detach().requires_grad_(True)
        r = (self.forward(y, blocks=blocks) - torch.as_tensor(S_target).to(F64)) * w
        E = 0.5 * (r * r).sum(dim=1)
        (g,) = torch.autograd.grad(E.sum(), y)
        return E.detach(), g.detach()

    def loss_grad(self, y, S_target):
        """(E [B], dE/dy [B, N]) — true gradient (R20), by reverse-mode autodiff."""
        y = torch.as_tensor(y).to(F64).detach().requires_grad_(True)
        E = self.loss(self.forward(y), S_target)
        (g,) = torch.autograd.grad(E.sum(), y)
        return E.detach(), g.detach()


def _subset_weights(plan, blocks) -> torch.Tensor:
    w = torch.zeros(plan.n_coef, dtype=F64)
    for q in plan.paths:
        if q.order == 1 or (q.order == 2 and q.block in blocks):
            w[q.offset:q.offset + q.rows * q.frames] = 1.0
    return w


def coefficients(plan_args, x) -> np.ndarray:
    return Oracle(plan_args).forward(x).numpy()

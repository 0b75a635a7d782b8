"""Command line (interfaces after SPEC S:452-522):

  python -m paper_2602_11896_b200.cli analyze    --input x.wav --features-dir out/  [plan flags]
  python -m paper_2602_11896_b200.cli synthesize --input x.wav --output y.wav [--iterations 100 --seed 0
                                                 --init colored|white --loss-csv loss.csv --checkpoint s.pt
                                                 --resume --tol 0]                  [plan flags]
  python -m paper_2602_11896_b200.cli filters    --output filters.csv              [plan flags]
  python -m paper_2602_11896_b200.cli gradcheck  [--directions 20 --seed 0]        [plan flags]

Plan flags: -N (default: the input length rounded down to a multiple of T, else 4096), -J, --q1, --q2,
--j-fr, --q-fr, --log2-T, --log2-F. Every computation runs through libjtfs.so (GPU); the CLI only does
file I/O, argument checking and host loops. Exit codes: 0 ok, 1 usage/config error, 2 numeric failure,
3 I/O error. Deterministic given its flags (seeds included)."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_NUMERIC, EXIT_IO = 0, 1, 2, 3


def _plan_flags(ap):
    ap.add_argument("-N", type=int, default=None, help="signal length (multiple of T)")
    ap.add_argument("-J", type=int, default=6)
    ap.add_argument("--q1", type=int, default=8)
    ap.add_argument("--q2", type=int, default=1)
    ap.add_argument("--j-fr", type=int, default=3)
    ap.add_argument("--q-fr", type=int, default=1)
    ap.add_argument("--log2-T", type=int, default=6)
    ap.add_argument("--log2-F", type=int, default=3)


def _plan(a, N):
    from . import Plan
    return Plan(N, a.J, a.q1, a.j_fr, a.q_fr, 1 << a.log2_T, 1 << a.log2_F, Q2=a.q2)


def _fit(x, a):
    """Truncate (with a warning) or zero-pad the input to the plan length N (multiple of T)."""
    T = 1 << a.log2_T
    N = a.N or max(T, len(x) // T * T)
    if len(x) > N:
        print(f"warning: input truncated from {len(x)} to {N} samples", file=sys.stderr)
    y = np.zeros(N, np.float32)
    y[: min(N, len(x))] = x[:N]
    return y, N


def cmd_analyze(a):
    import torch
    from .wav import read_wav
    x, sr = read_wav(a.input)
    x, N = _fit(x, a)
    p = _plan(a, N)
    S = p.forward(torch.from_numpy(x)[None].cuda()).cpu().numpy()[0].astype(np.float64)
    os.makedirs(a.features_dir, exist_ok=True)
    paths = p.paths()
    S.tofile(os.path.join(a.features_dir, "coefficients.f64"))
    man = {"input": os.path.basename(a.input), "sample_rate": sr, "N": N,
           "plan": {"J": a.J, "Q": a.q1, "Q2": a.q2, "J_fr": a.j_fr, "Q_fr": a.q_fr, "T": 1 << a.log2_T,
                    "F": 1 << a.log2_F},
           "n_coef": int(S.size), "dtype": "float64 little-endian, packed path-major (R15)",
           "paths": [{k: int(v) for k, v in q.items()} for q in paths]}
    with open(os.path.join(a.features_dir, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1)
    print(f"paths {len(paths)} coefficients {S.size}")
    return EXIT_OK


def cmd_synthesize(a):
    import torch
    from .metamer import reconstruct
    from .wav import read_wav, write_wav
    x, sr = read_wav(a.input)
    x, N = _fit(x, a)
    p = _plan(a, N)
    St = p.forward(torch.from_numpy(x)[None].cuda())
    y0 = None
    if a.init == "white":
        g = torch.Generator(device="cuda").manual_seed(a.seed)
        y0 = torch.randn(1, N, generator=g, device="cuda") * float(np.sqrt(np.mean(x.astype(np.float64) ** 2)))
    res = reconstruct(p, St, steps=a.iterations, y0=y0, seed=a.seed, tol=a.tol, mu0=a.lr, momentum=a.momentum,
                      csv_path=a.loss_csv, checkpoint=a.checkpoint, resume=a.resume)
    y = res["y_best"].cpu().numpy()[0]
    write_wav(a.output, y, sr)
    h = [r[0] for r in res["history"] if r[0] is not None]
    print(f"iterations {res['iterations']} loss {h[0] if h else float('nan'):.6g} -> "
          f"{float(res['loss_best'][0]):.6g}")
    return EXIT_OK


def cmd_filters(a):
    from . import Plan  # noqa: F401  (host-only planner: no GPU needed)
    p = _plan(a, a.N or (1 << a.log2_T) * 64)
    names = {0: "psi1", 1: "psi2", 2: "psi_fr"}
    with open(a.output, "w") as f:
        f.write("layer,n,xi,sigma,j,spin\n")
        for layer in (0, 1, 2):
            fb = p.filters(layer)
            n_fr = len(fb["xi"])
            for n in range(n_fr):
                xi = float(fb["xi"][n])
                spin = int(np.sign(xi)) if layer == 2 else 1
                f.write(f"{names[layer]},{n},{xi:.17g},{float(fb['sigma'][n]):.17g},{int(fb['j'][n])},{spin}\n")
    print(f"wrote {a.output}")
    return EXIT_OK


def cmd_gradcheck(a):
    """Directional derivatives of the GPU gradient vs central differences of the GPU loss (fp32 forward,
    float64 loss accumulation): median / max relative error over seeded random directions."""
    import torch
    N = a.N or 1024
    p = _plan(a, N)
    rng = np.random.default_rng(a.seed)
    x = torch.from_numpy((0.1 * rng.standard_normal((1, N))).astype(np.float32)).cuda()
    y = torch.from_numpy((0.1 * rng.standard_normal((1, N))).astype(np.float32)).cuda()
    St = p.forward(x)
    _, g = p.loss_grad(y, St)
    errs = []
    for _ in range(a.directions):
        d = torch.from_numpy(rng.standard_normal((1, N)).astype(np.float32)).cuda()
        d /= d.norm()
        h = 1e-2 * float(y.norm())
        Ep, _ = p.loss_grad((y + h * d).contiguous(), St)
        Em, _ = p.loss_grad((y - h * d).contiguous(), St)
        fd = (float(Ep[0]) - float(Em[0])) / (2 * h)
        dd = float((g * d).sum())
        errs.append(abs(fd - dd) / max(abs(dd), 1e-30))
    med, mx = float(np.median(errs)), float(np.max(errs))
    ok = med <= 1e-2
    print(f"gradcheck: {a.directions} directions, median rel err {med:.3e}, max {mx:.3e}: "
          f"{'PASS' if ok else 'FAIL'}")
    return EXIT_OK if ok else EXIT_NUMERIC


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2602_11896_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    an = sub.add_parser("analyze")
    an.add_argument("--input", required=True)
    an.add_argument("--features-dir", required=True)
    sy = sub.add_parser("synthesize")
    sy.add_argument("--input", required=True)
    sy.add_argument("--output", required=True)
    sy.add_argument("--iterations", type=int, default=100)
    sy.add_argument("--lr", type=float, default=0.1)
    sy.add_argument("--momentum", type=float, default=0.9)
    sy.add_argument("--seed", type=int, default=0)
    sy.add_argument("--tol", type=float, default=0.0)
    sy.add_argument("--init", choices=["colored", "white"], default="colored")
    sy.add_argument("--loss-csv", default=None)
    sy.add_argument("--checkpoint", default=None)
    sy.add_argument("--resume", action="store_true")
    fi = sub.add_parser("filters")
    fi.add_argument("--output", required=True)
    gc = sub.add_parser("gradcheck")
    gc.add_argument("--directions", type=int, default=20)
    gc.add_argument("--seed", type=int, default=0)
    for s in (an, sy, fi, gc):
        _plan_flags(s)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    from ._lib import JtfsError
    from .wav import WavError
    try:
        return {"analyze": cmd_analyze, "synthesize": cmd_synthesize, "filters": cmd_filters,
                "gradcheck": cmd_gradcheck}[a.cmd](a)
    except JtfsError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NUMERIC if e.code == 3 else EXIT_USAGE
    except (WavError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())

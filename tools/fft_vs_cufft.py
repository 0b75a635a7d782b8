"""Test-only benchmark (GPU): the library's batched C2C FFT (jtfs_debug_fft) vs cuFFT (torch.fft) on the
transform shapes of a plan's hot path (layer-1 rows per level, second-order block rows), complex64 and
complex128. Prints one JSON line per shape: ms, effective GB/s (read + write of the rows once), ratio.
usage: python tools/fft_vs_cufft.py c4 [batch]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11896_b200 import Plan  # noqa: E402
from paper_2602_11896_b200._lib import check  # noqa: E402
from synth import CONFIGS, plan_args  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main(cfg, B):
    args = plan_args(CONFIGS[cfg])
    p = Plan(*args)
    p.prepare()
    # row shapes from the library's own plan tables (filters' scales j, R3/R13)
    i = p.info
    log2T = (i.N // i.frames).bit_length() - 1
    j1, j2 = p.filters(0)["j"], p.filters(1)["j"]
    shapes = {}
    for j in j1:                                    # layer-1 rows (Z1 / U1 transforms) by level
        L = i.N_pad >> min(int(j), log2T)
        shapes[L] = shapes.get(L, 0) + 1
    for j in j2:                                    # second-order rows (Y2 / g_Y2 transforms)
        n1_max = int(sum(1 for a in j1 if a < j))
        if n1_max:
            L = i.N_pad >> min(int(j), log2T)
            shapes[L] = shapes.get(L, 0) + n1_max
    for dbl in (0, 1):
        dt = torch.complex128 if dbl else torch.complex64
        for L, cnt in sorted(shapes.items(), reverse=True)[:8]:
            x = torch.randn(B, cnt, L, dtype=dt, device="cuda")
            y = torch.empty_like(x)
            src = x.clone()

            def ours():
                src.copy_(x)   # four-step clobbers its input; the copy is timed separately and subtracted
                check(p.lib.jtfs_debug_fft(p.h, src.data_ptr(), y.data_ptr(), L, cnt, B, 0, dbl,
                                           torch.cuda.current_stream().cuda_stream))
            t_copy = timed(lambda: src.copy_(x))
            t_ours = timed(ours) - t_copy
            t_cufft = timed(lambda: torch.fft.fft(x, dim=-1))
            ref = torch.fft.fft(x, dim=-1)
            ours()
            torch.cuda.synchronize()
            err = float((y - ref).abs().max() / ref.abs().max())
            gb = 2 * x.numel() * x.element_size() / 1e9
            print(json.dumps({"config": cfg, "B": B, "L": L, "rows": cnt, "dtype": str(dt).split(".")[-1],
                              "ours_ms": round(t_ours, 4), "cufft_ms": round(t_cufft, 4),
                              "ours_gbs": round(gb / t_ours * 1e3, 1), "cufft_gbs": round(gb / t_cufft * 1e3, 1),
                              "ours_over_cufft_time": round(t_ours / t_cufft, 3), "max_rel_err": err}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4", int(sys.argv[2]) if len(sys.argv) > 2 else 4)

"""ORACLE — test infrastructure only.

A plain, slow, float64 CPU implementation of the JTFS forward transform, Euclidean feature loss,
gradient and metamer step of arxiv 2602.11896 (§2-§3), written from the paper's
equations and Kymatio listings in the paper's order and notation.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import or run anything under `oracle/`. The product path (`paper_2602_11896_b200`)
never imports it and shares no code, header, table or constant generator with it; the only
module both sides use is `synth/` (seeded input generators, no method arithmetic).

Modules:
  plan.py   — filterbank generator, scales, padding, paths (readings R1-R16).
  jtfs.py   — forward (listings), loss, gradient by
              reverse-mode autodiff (P:126-130 says Kymatio does exactly that), chunked variant.
  brute.py  — direct time-domain circular sums with closed-form kernels (no FFT): an independent
              route used only to pin jtfs.py on tiny inputs.
  metamer.py— momentum + bold-driver update (readings R23-R24).

Parity status per function is listed in DESIGN.md §"Oracle pins". Absolute coefficient values
are "parity unpinned" against the paper (it prints no worked example); they are pinned by the
invariants and independent routes of tests/test_oracle_*.py.
"""

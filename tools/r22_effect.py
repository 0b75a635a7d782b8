"""Measure the effect of the R22 modulus dead zone (|z| < EPS_MOD * RMS(y)) on the
float64 oracle gradient at the BASELINE configs: rel-L2 of g(EPS_MOD = 1e-12) - g(EPS_MOD = 0).
Calls only oracle/ and synth/; writes tests/golden/r22_effect.json (pinned by
tests/test_oracle_grad.py::test_dead_zone_effect_at_baseline_configs).
Usage: python tools/r22_effect.py c2:all c4:0 c4:11 c5:11"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.jtfs as OJ  # noqa: E402
from oracle.jtfs import Oracle  # noqa: E402
from synth import CONFIGS, plan_args, batch  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "r22_effect.json")


def grad(o, y, So, blocks):
    return (o.loss_grad(y, So) if blocks is None else o.loss_grad_subset(y, So, blocks))[1].numpy()


def main(specs):
    rec = json.load(open(OUT)) if os.path.exists(OUT) else {"cases": {}}
    rec["what"] = ("rel-L2 change of the float64 oracle dE/dy when the R22 dead zone "
                   "(|z| < 1e-12 RMS(y_b)) is replaced by the exact-zero rule; signal b = 0, "
                   "synth inputs x / y of the config; 'all' = full loss, else order 1 + those blocks")
    for spec in specs:
        name, bl = spec.split(":")
        blocks = None if bl == "all" else [int(b) for b in bl.split(",")]
        args = plan_args(CONFIGS[name])
        x, y = batch(name, 1), batch(name, 1, which="y")
        t = time.time()
        o = Oracle(args)
        So = o.forward(x, blocks=blocks)
        OJ.EPS_MOD = 1e-12
        g = grad(o, y, So, blocks)
        OJ.EPS_MOD = 0.0
        g0 = grad(o, y, So, blocks)
        OJ.EPS_MOD = 1e-12
        v = float(np.linalg.norm(g - g0) / np.linalg.norm(g0))
        rec["cases"][spec] = {"rel_effect": v, "seconds": round(time.time() - t, 1)}
        print(spec, rec["cases"][spec], flush=True)
        json.dump(rec, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])

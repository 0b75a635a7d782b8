"""Small forward + loss_grad on the tensor-core route (spec / t2 configs) for compute-sanitizer runs:
  compute-sanitizer --tool racecheck python tools/sanitize_run.py spec
  compute-sanitizer --tool synccheck python tools/sanitize_run.py spec"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_11896_b200 import Plan  # noqa: E402
from synth import CONFIGS, TINY, plan_args, noise  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "spec"
cfg = {**CONFIGS, **TINY}[name]
p = Plan(*plan_args(cfg))
x = torch.from_numpy(noise(cfg["N"], 2, seed=1)).cuda()
y = torch.from_numpy(noise(cfg["N"], 2, seed=2)).cuda()
S = p.forward(x)
loss, g = p.loss_grad(y, S)
torch.cuda.synchronize()
print("ok", name, float(loss.sum()), float(g.abs().sum()), "launches", p.launch_count())

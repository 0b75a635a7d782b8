"""Debug helper: per-component gradient parity at a large config (run on the GPU box)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle.jtfs import Oracle
from synth import CONFIGS, plan_args, batch
from paper_2602_11896_b200 import Plan

name = sys.argv[1]
subsets = [[], [int(b) for b in sys.argv[2:]]] if len(sys.argv) > 2 else [[]]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


args = plan_args(CONFIGS[name])
p = Plan(*args)
o = Oracle(args)
x = batch(name, 1)
y = batch(name, 1, which="y")
yd = torch.from_numpy(y).cuda()
Sy = p.forward(yd)
for blocks in subsets:
    So = o.forward(x, blocks=blocks).numpy()
    m = np.zeros(o.plan.n_coef, bool)
    for q in o.plan.paths:
        if q.order == 1 or (q.order == 2 and q.block in blocks):
            m[q.offset:q.offset + q.rows * q.frames] = True
    St = Sy.clone()
    mt = torch.from_numpy(m).cuda()
    St[0, mt] = torch.from_numpy(So.astype(np.float32)).cuda()[0, mt]
    loss, g = p.loss_grad(yd, St)
    Eo, go = o.loss_grad_subset(y, So, blocks)
    g = g.cpu().numpy()[0]
    go = go.numpy()[0]
    print(name, blocks, "loss", float(loss[0]), float(Eo[0]), "rel grad", rel(g, go), flush=True)
    N = len(g)
    for a, b in [(0, N // 8), (N // 8, N // 2), (N // 2, 7 * N // 8), (7 * N // 8, N)]:
        print("   segment", a, b, rel(g[a:b], go[a:b]))

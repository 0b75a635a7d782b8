"""Order-1-only gradient parity at c4 for different input pairs (debug helper, GPU box)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle.jtfs import Oracle
from synth import CONFIGS, plan_args, noise, batch
from paper_2602_11896_b200 import Plan

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
args = plan_args(CONFIGS[name])
p = Plan(*args)
o = Oracle(args)
mus_x, mus_y = batch(name, 1), batch(name, 1, which="y")
nz_x, nz_y = noise(args[0], 1, seed=1), noise(args[0], 1, seed=2)
for tag, x, y in [("mus/mus", mus_x, mus_y), ("noise/mus", nz_x, mus_y), ("mus/noise", mus_x, nz_y),
                  ("mus/mus+1e-3noise", mus_x, mus_y + 1e-3 * nz_y)]:
    So = o.forward(x, blocks=[]).numpy()
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    Sy = p.forward(yd)
    m = np.zeros(o.plan.n_coef, bool)
    for q in o.plan.paths:
        if q.order == 1:
            m[q.offset:q.offset + q.rows * q.frames] = True
    St = Sy.clone()
    mt = torch.from_numpy(m).cuda()
    St[0, mt] = torch.from_numpy(So.astype(np.float32)).cuda()[0, mt]
    loss, g = p.loss_grad(yd, St)
    Eo, go = o.loss_grad_subset(y.astype(np.float32), So, [])
    g = g.cpu().numpy()[0]; go = go.numpy()[0]
    err = np.abs(g - go)
    print(tag, "rel grad", float(np.linalg.norm(g - go) / np.linalg.norm(go)), "argmax err", int(err.argmax()),
          "|y| there", float(np.abs(y[0, max(0, err.argmax()-50):err.argmax()+50]).max()), flush=True)

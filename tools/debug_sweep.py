"""Order-1-only gradient parity for a list of plan tuples (debug helper, GPU box)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle.jtfs import Oracle
from synth import noise
from paper_2602_11896_b200 import Plan

cfgs = [eval(a) for a in sys.argv[1:]]
for args in cfgs:
    p = Plan(*args)
    o = Oracle(args)
    x = noise(args[0], 1, seed=1)
    y = noise(args[0], 1, seed=2)
    So = o.forward(x, blocks=[]).numpy()
    yd = torch.from_numpy(y).cuda()
    Sy = p.forward(yd)
    m = np.zeros(o.plan.n_coef, bool)
    for q in o.plan.paths:
        if q.order == 1:
            m[q.offset:q.offset + q.rows * q.frames] = True
    St = Sy.clone()
    mt = torch.from_numpy(m).cuda()
    St[0, mt] = torch.from_numpy(So.astype(np.float32)).cuda()[0, mt]
    loss, g = p.loss_grad(yd, St)
    Eo, go = o.loss_grad_subset(y, So, [])
    g = g.cpu().numpy()[0]; go = go.numpy()[0]
    print(args, "N_pad", o.plan.N_pad, "P", o.plan.P, "N1", o.plan.N1, "rel grad",
          float(np.linalg.norm(g - go) / np.linalg.norm(go)), flush=True)

"""R22 experiment (GPU box): GPU gradient vs the float64 oracle with NO modulus dead zone (exact
autograd phase, tau = 0). Usage: JTFS_MODTAU=<tau> python tools/expt_r22.py c2 all|0,9 ..."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.jtfs as OJ
from oracle.jtfs import Oracle
from oracle.plan import make_plan
from synth import CONFIGS, plan_args, batch
from paper_2602_11896_b200 import Plan

OJ.EPS_MOD = float(os.environ.get('ORACLE_EPS', '1e-12'))
torch.set_num_threads(os.cpu_count())


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def mask(plan, blocks):
    m = np.zeros(plan.n_coef, bool)
    for q in plan.paths:
        if q.order <= 1 or blocks is None or (q.order == 2 and q.block in blocks):
            m[q.offset:q.offset + q.rows * q.frames] = True
    return m


for spec in sys.argv[1:]:
    name, bl = spec.split(":")
    blocks = None if bl == "all" else [int(b) for b in bl.split(",")]
    zero = name.endswith("z")
    name = name.rstrip("z")
    args = plan_args(CONFIGS[name])
    x, y = batch(name, 1), batch(name, 1, which="y")
    if zero:   # silent stretches in y: 4 zeroed runs of N/16 samples
        N = y.shape[1]
        for k in range(4):
            y[:, (4 * k + 1) * N // 16:(4 * k + 2) * N // 16] = 0
    cache = f"/tmp/r22_{name}{'z' if zero else ''}_{bl}_{OJ.EPS_MOD}.npz"
    if os.path.exists(cache):
        z = np.load(cache); So, Eo, go = z["So"], z["Eo"], z["go"]
    else:
        t = time.time()
        o = Oracle(args)
        So = o.forward(x, blocks=blocks).numpy()
        if blocks is None:
            Eo, go = o.loss_grad(y, So)
        else:
            Eo, go = o.loss_grad_subset(y, So, blocks)
        Eo, go = Eo.numpy(), go.numpy()
        np.savez(cache, So=So, Eo=Eo, go=go)
        print(f"oracle {spec}: {time.time() - t:.1f} s", flush=True)
    p = Plan(*args)
    yd = torch.from_numpy(y).cuda()
    m = mask(make_plan(*args), blocks)
    Sy = p.forward(yd)
    St = Sy.clone()
    mt = torch.from_numpy(m).cuda()
    St[0, mt] = torch.from_numpy(So[0].astype(np.float32)).cuda()[mt]
    loss, g = p.loss_grad(yd, St)
    print(json.dumps({"spec": spec, "oracle_eps": OJ.EPS_MOD,
                      "rel_loss": rel(loss.cpu().numpy(), Eo), "rel_grad": rel(g.cpu().numpy()[0], go[0])}), flush=True)

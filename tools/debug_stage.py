import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2602_11896_b200 import Plan
from oracle.jtfs import Oracle, reflect_index
from synth import TINY, plan_args, noise
args = plan_args(TINY["t1"])
p = Plan(*args)
o = Oracle(args)
x = noise(args[0], 2, seed=31)
xd = torch.from_numpy(x).cuda()
X = p.debug_stage(5, xd).cpu().numpy()
xp = x[:, reflect_index(o.plan).numpy()].astype(np.float64)
Xr = np.fft.fft(xp, axis=1)
print("Xhat rel per row", [float(np.linalg.norm(X[b] - Xr[b]) / np.linalg.norm(Xr[b])) for b in range(2)])
Z = p.debug_stage(6, xd).cpu().numpy()
_, U1h, _ = o.layer1(torch.from_numpy(x).double())
Zr = np.concatenate([np.fft.ifft(u.numpy(), axis=1) for u in U1h], axis=1)
print("|Z1| rel per row", [float(np.linalg.norm(np.abs(Z[b]) - np.abs(Zr[b])) / np.linalg.norm(Zr[b])) for b in range(2)])

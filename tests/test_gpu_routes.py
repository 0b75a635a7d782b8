"""GPU: the joint-stage routes other than the default tensor-core one, selected at library load by the
environment (jtfs_api.cu route_of): JTFS_TC=0 sends every block to the FFT route along n1 (the paper's
`frequency_scattering`; kernels_frfft.cu), JTFS_TC=0 JTFS_SIMT=1 to the dense CUDA-core
kernels (kernels_fr.cu). Each runs in a fresh interpreter and is checked against the float64 oracle
with the north_star tolerances (coefficients 1e-4, gradient 1e-3 relative L2)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2602_11896_b200 import Plan
from oracle.jtfs import Oracle
from synth import CONFIGS, TINY, plan_args, noise
ALL = {{**CONFIGS, **TINY}}
args = plan_args(ALL[{name!r}])
p = Plan(*args)
x = noise(args[0], 2, seed=11)
y = noise(args[0], 2, seed=12)
S = p.forward(torch.from_numpy(x).cuda())
loss, g = p.loss_grad(torch.from_numpy(y).cuda(), S)
o = Oracle(args)
So = o.forward(x).numpy()
Eo, go = o.loss_grad(y, o.forward(x))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print("REL", rel(S.cpu().numpy(), So), rel(g.cpu().numpy(), go.numpy()))
"""


@pytest.mark.parametrize("env", [{"JTFS_TC": "0"}, {"JTFS_TC": "0", "JTFS_SIMT": "1"}],
                         ids=["fft_route", "cuda_core_dense"])
@pytest.mark.parametrize("name", ["spec", "c1"])
def test_alternative_routes(env, name):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, name=name)], env=e, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("REL")][-1]
    rs, rg = map(float, line.split()[1:])
    assert rs <= 1e-4 and rg <= 1e-3, (env, name, rs, rg)

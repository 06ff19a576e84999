"""Fluid-process cost per round: k_diffuse on config 2's costs (n = 8, no
memory) with the discrete process stopped at once (gamma huge) and the fluid
process run for max_rounds = 0, 16, 64, 128, 228 (gamma_f = 0); graph-timed
like tools/solver_microbench.py.  python tools/fluid_slope.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_14864_b200 import dynmo as D  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from solver_microbench_t import t  # noqa: E402

torch.cuda.set_device(0)
ctx = D.Context(0)
cost = torch.as_tensor(np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")), device="cuda")
b = D.Batch([48], [8], device="cuda")
bi = torch.arange(0, 49, 6, dtype=torch.int32, device="cuda")
gam = torch.tensor([1 << 62], dtype=torch.int64, device="cuda")
gf = torch.zeros(1, dtype=torch.float64, device="cuda")
res = {}
for r in (0, 16, 64, 128, 228):
    o = {}
    res[r] = t(lambda: D.diffuse_balance(ctx, b, cost, bi, gamma=gam, gamma_fluid=gf, max_rounds=r, out=o))
    torch.cuda.synchronize()
    res[f"{r}_rounds"] = int(o["fluid_rounds"].item())
o = {}
res["nofluid"] = t(lambda: D.diffuse_balance(ctx, b, cost, bi, gamma=gam, fluid=False, max_rounds=0, out=o))
print(json.dumps(res))

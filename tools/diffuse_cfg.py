"""k_diffuse alone on a bench workload's instance (the step's inputs:
costs from the oracle of the synthetic sources, uniform split, the bench's
memory, cap and gamma_fluid), graph-timed; the fluid and discrete processes
separately and together.  python tools/diffuse_cfg.py [config]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402
from solver_microbench_t import t  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
torch.cuda.set_device(0)
ctx = D.Context(0)
wl = bench.WORKLOADS[cfg](bench.parse(["--config", str(cfg)]))
cost = torch.as_tensor(wl.oracle_cost(list(wl.sources(0, wl.L))), device="cuda")
b = D.Batch([wl.L], [wl.n], device="cuda")
bi = torch.as_tensor(np.array([(s * wl.L) // wl.n for s in range(wl.n + 1)], np.int32), device="cuda")
mem = torch.as_tensor(wl.payload.astype(np.int64), device="cuda")
cap = torch.tensor([wl.cap], dtype=torch.int64, device="cuda")
gf = torch.tensor([wl.gamma_fluid], dtype=torch.float64, device="cuda")
big = torch.tensor([1 << 62], dtype=torch.int64, device="cuda")
o1, o2, o3 = {}, {}, {}
res = {"config": cfg,
       "both": t(lambda: D.diffuse_balance(ctx, b, cost, bi, mem=mem, cap=cap, gamma_fluid=gf, out=o1)),
       "discrete_only": t(lambda: D.diffuse_balance(ctx, b, cost, bi, mem=mem, cap=cap, fluid=False, out=o2)),
       "fluid_only (discrete stops at once)": t(lambda: D.diffuse_balance(ctx, b, cost, bi, mem=mem, cap=cap,
                                                                          gamma=big, gamma_fluid=gf, out=o3))}
torch.cuda.synchronize()
res["rounds"] = [int(o1["rounds"].item()), int(o1["fluid_rounds"].item())]
print(json.dumps(res))

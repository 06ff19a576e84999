"""Phase cycles of the fluid process (diagnostic build with
-DDYNMO_FLUID_PROF, which writes them into fluid_x): kernel start -> fluid
entry, exact rows, speculative rows, verification, bookkeeping, chunks,
total.  DYNMO_LIB=ab/libdynmo_fprof.so python tools/fluid_prof.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_14864_b200 import dynmo as D  # noqa: E402

torch.cuda.set_device(0)
ctx = D.Context(0)
cost = torch.as_tensor(np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")), device="cuda")
b = D.Batch([48], [8], device="cuda")
bi = torch.arange(0, 49, 6, dtype=torch.int32, device="cuda")
gam = torch.tensor([1 << 62], dtype=torch.int64, device="cuda")
gf = torch.zeros(1, dtype=torch.float64, device="cuda")
names = ["to_entry", "exact", "spec", "verify", "other", "chunks", "total"]
for r in (64, 228):
    rows = []
    for _ in range(20):
        o = {}
        D.diffuse_balance(ctx, b, cost, bi, gamma=gam, gamma_fluid=gf, max_rounds=r, out=o)
        torch.cuda.synchronize()
        rows.append(o["fluid_x"][:7].cpu().numpy())
    med = np.median(np.array(rows[5:]), axis=0)
    print(json.dumps({"rounds": r, **{k: float(v) for k, v in zip(names, med)},
                      "cycles_per_round_total": float(med[6] / r)}))

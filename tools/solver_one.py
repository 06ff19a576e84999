"""One call of each solver on the config-2 cost vector (for ncu source
profiles): python tools/solver_one.py [partition|diffuse|repack]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_14864_b200 import dynmo as D  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "partition"
torch.cuda.set_device(0)
ctx = D.Context(0)
cost = torch.as_tensor(np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")), device="cuda")
b = D.Batch([48], [8], device="cuda")
mem = torch.full((48,), 1000, dtype=torch.int64, device="cuda")
cap = torch.tensor([10 ** 9], dtype=torch.int64, device="cuda")
bnd_in = torch.arange(0, 49, 6, dtype=torch.int32, device="cuda")
gf = torch.tensor([1.0], dtype=torch.float64, device="cuda")
if which.endswith("_bench"):  # the bench's config-2 memory: synthetic CSR payload, cap 1.5x the mean
    import synth
    _sh = synth.GPTShape()
    _pay = synth.cfg2_payload_bytes(_sh, synth.cfg2_keep_probs(_sh, 0.9, 4))
    mem = torch.as_tensor(_pay.astype(np.int64), device="cuda")
    cap = torch.tensor([int(1.5 * int(_pay.sum()) / 8)], dtype=torch.int64, device="cuda")
    which = which[:-6]
for _ in range(3):
    if which == "partition":
        D.partition_stages(ctx, b, cost, mem=mem, cap=cap)
        D.partition_stages(ctx, b, cost)
    elif which == "diffuse":
        o = {}
        D.diffuse_balance(ctx, b, cost, bnd_in, mem=mem, cap=cap, gamma_fluid=gf, max_rounds=256, out=o)
    else:
        D.repack_workers(ctx, b, cost, floor=torch.ones(1, dtype=torch.int32, device="cuda"),
                         bound=torch.tensor([int(cost.sum()) // 6], device="cuda"), mem=mem, cap=cap)
torch.cuda.synchronize()
print("ok", which)

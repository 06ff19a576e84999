"""One dynmo_global_prune call on config-2-sized bf16 weights (604 M) at G=1,
for ncu launch lists of the prune kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

torch.cuda.set_device(0)
ctx = D.Context(0)
shape = synth.GPTShape()
sig = np.exp(np.random.default_rng(3).normal(0, 0.35, shape.L))
gen = torch.Generator(device="cuda").manual_seed(2505)
ws = [(torch.randn(shape.params_per_layer, generator=gen, device="cuda") * float(sig[l])).to(torch.bfloat16)
      for l in range(shape.L)]
ms = [torch.empty(shape.params_per_layer, dtype=torch.uint8, device="cuda") for _ in ws]
plan = D.PrunePlan(ctx, list(zip(ws, ms)))
k = int(shape.L * shape.params_per_layer * 0.1)
for _ in range(3):
    info, st = D.global_prune(ctx, plan, k)
torch.cuda.synchronize()
print("ok", info.cpu().numpy(), int(st.item()))

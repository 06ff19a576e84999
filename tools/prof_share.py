"""k_profile on the first LAYERS layers of config 2 (the per-GPU share at
G GPUs: 48/G layers), one call repeated, for ncu kernel durations:
python tools/prof_share.py LAYERS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
torch.cuda.set_device(0)
ctx = D.Context(0)
srcs = list(bench.Cfg2().sources(0, n))
dm = [torch.from_numpy(a).to("cuda") for _, _, a, _, _ in srcs]
plan = D.ProfilePlan(ctx, [D.SegmentSpec(t, LB.SRC_MASK_U8, l) for t, (_, l, _, _, _) in zip(dm, srcs)], 0, n)
coef = D.coef_tensor(n, A=0, B=1, device="cuda")
flush = bench.L2Flush("cuda")
for _ in range(6):
    flush()
    D.profile_layers(ctx, plan, coef)
torch.cuda.synchronize()
print("ok", n, plan.bytes)

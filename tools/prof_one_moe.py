"""Config-4 MoE profile calls (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_14864_b200 import _lib as LB, dynmo as D
torch.cuda.set_device(0)
ctx = D.Context(0)
T, L, E, k = 64 * 2048, 32, 8, 2
segs, keep = [], []
for i in range(L):
    d = torch.from_numpy(synth.cfg4_routing(i, T=T, E=E, k=k, alpha=4.0).reshape(-1)).cuda()
    keep.append(d)
    segs.append(D.SegmentSpec(d, LB.SRC_EXPERT_I64, i, n_experts=E, top_k=k))
plan = D.ProfilePlan(ctx, segs, 0, L)
coef = D.coef_tensor(L, A=T, C_=4, ep=8, device="cuda")
for _ in range(4):
    D.profile_layers(ctx, plan, coef)
torch.cuda.synchronize()
print("ok", plan.n_tiles)

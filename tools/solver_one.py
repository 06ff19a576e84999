"""One call of each partition variant on the config-2 cost vector (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_14864_b200 import dynmo as D
torch.cuda.set_device(0)
ctx = D.Context(0)
cost = torch.as_tensor(np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")), device="cuda")
b = D.Batch([48], [8], device="cuda")
mem = torch.full((48,), 1000, dtype=torch.int64, device="cuda")
cap = torch.tensor([10 ** 9], dtype=torch.int64, device="cuda")
for _ in range(3):
    D.partition_stages(ctx, b, cost, mem=mem, cap=cap)
    D.partition_stages(ctx, b, cost)
torch.cuda.synchronize()
print("ok")

"""Config-5 solver calls alone (partition + BOUND repack over 4096 instances,
throughput mode), graph-replayed and timed with CUDA events; for A/B runs of
library builds (DYNMO_LIB=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

DEV = "cuda:0"
torch.cuda.set_device(0)
ctx = D.Context(0)
n_inst = 4096
insts = [synth.cfg5_instance(i) for i in range(n_inst)]
cost = np.concatenate([[oracle.count_bits(x.masks[l], 4096) for l in range(x.L)] for x in insts]).astype(np.int64)
b = D.Batch([x.L for x in insts], [x.n for x in insts], device=DEV)
c = torch.from_numpy(cost).to(DEV)
mem = torch.from_numpy(np.concatenate([x.mem for x in insts]).astype(np.int64)).to(DEV)
cap = torch.tensor([x.cap for x in insts], dtype=torch.int64, device=DEV)
bound = torch.tensor([x.bound for x in insts], dtype=torch.int64, device=DEV)
floor = torch.ones(n_inst, dtype=torch.int32, device=DEV)
out = {}
for name, fn in [("partition", lambda: D.partition_stages(ctx, b, c, mem=mem, cap=cap)),
                 ("repack", lambda: D.repack_workers(ctx, b, c, floor=floor, bound=bound, mem=mem, cap=cap, out=out)),
                 ("partition_nomem", lambda: D.partition_stages(ctx, b, c))]:
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(os.environ.get("DYNMO_LIB", "current"), name, round(float(np.median(ts)), 1), "us")

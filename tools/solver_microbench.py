"""Isolated timing of the solver kernels (CUDA events over many launches)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_14864_b200 import dynmo as D

dev = "cuda:0"
torch.cuda.set_device(0)
ctx = D.Context(0)
cost2 = np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")) if os.path.exists(
    os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")) else np.random.default_rng(0).integers(0, 2_400_000, 48)


from solver_microbench_t import t  # noqa: E402


res = {}
import synth
_sh = synth.GPTShape()
_p = synth.cfg2_keep_probs(_sh, 0.9, 4)
_pay = synth.cfg2_payload_bytes(_sh, _p)
bench_mem = torch.as_tensor(_pay.astype(np.int64), device=dev)
bench_cap = torch.tensor([int(1.5 * int(_pay.sum()) / 8)], dtype=torch.int64, device=dev)
for name, cost, n, with_mem in [("cfg2_benchmem", cost2, 8, "bench"),("cfg2_mem", cost2, 8, True), ("cfg2_nomem", cost2, 8, False),
                                ("cfg2_n1", cost2, 1, False), ("cfg2_n2", cost2, 2, False),
                                ("small_L24_n4", np.arange(24) % 7, 4, False),
                                ("L8_n2_tiny", np.ones(8, np.int64), 2, False),
                                ("L127_n8", np.random.default_rng(1).integers(0, 10**6, 127), 8, False),
                                ("L1023_n8", np.random.default_rng(1).integers(0, 10**6, 1023), 8, False)]:
    c = torch.as_tensor(np.asarray(cost, np.int64), device=dev)
    b = D.Batch([len(cost)], [n], device=dev)
    mem = cap = None
    if with_mem == "bench":
        mem, cap = bench_mem, bench_cap
    elif with_mem:
        mem = torch.ones(len(cost), dtype=torch.int64, device=dev) * 1000
        cap = torch.tensor([10 ** 9], dtype=torch.int64, device=dev)
    out = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=dev),
               bottleneck=torch.empty(1, dtype=torch.int64, device=dev),
               imbalance=torch.empty(1, dtype=torch.float64, device=dev),
               status=torch.empty(1, dtype=torch.int32, device=dev))
    res["partition_" + name] = t(lambda: D.partition_stages(ctx, b, c, mem=mem, cap=cap, **out))
    floor = torch.ones(1, dtype=torch.int32, device=dev)
    bound = torch.tensor([int(np.asarray(cost).sum())], dtype=torch.int64, device=dev)
    ro = {}
    res["repack_" + name] = t(lambda: D.repack_workers(ctx, b, c, floor=floor, bound=bound, mem=mem, cap=cap, out=ro))
    bi = torch.as_tensor(np.array([(s * len(cost)) // n for s in range(n + 1)], np.int32), device=dev)
    do = {}
    res["diffuse_nofluid_" + name] = t(lambda: D.diffuse_balance(ctx, b, c, bi, mem=mem, cap=cap, fluid=False, out=do))
    do2 = {}
    gf = torch.tensor([1.0], dtype=torch.float64, device=dev)
    res["diffuse_fluid_" + name] = t(lambda: D.diffuse_balance(ctx, b, c, bi, mem=mem, cap=cap, gamma_fluid=gf, out=do2))
    torch.cuda.synchronize()
    res["rounds_" + name] = [int(do2["rounds"].item()), int(do2["fluid_rounds"].item())]
# empty-ish reference: a torch fill of 1 element
x = torch.empty(1, device=dev)
res["torch_fill_1elem"] = t(lambda: x.fill_(1.0))
for k, v in res.items():
    print(f"{k:40s} {v}")
json.dump(res, open("gpurun_out/solver_microbench.json", "w"), indent=1)

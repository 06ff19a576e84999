"""k_profile bandwidth vs per-GPU input size (config-2 layer shares at G = 8/4/2/1).
Distinct mask copies totalling >= 512 MB are cycled so no launch reads L2-
resident data; CUDA events around each profile_layers call (graph-replayed)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2505_14864_b200 import _lib as LB
from paper_2505_14864_b200 import dynmo as D

torch.cuda.set_device(0)
dev = "cuda:0"
ctx = D.Context(0)
shape = synth.GPTShape()
P = shape.params_per_layer
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
res = {}
g = torch.Generator(device=dev).manual_seed(0)
for repr_ in ("u8", "bits", "bf16"):
    for layers in (6, 12, 24, 48):
        nbytes_layer = {"u8": P, "bits": P // 8, "bf16": 2 * P}[repr_]
        copies = max(2, -(-(512 << 20) // (layers * nbytes_layer)))
        if copies * layers * nbytes_layer > (40 << 30):
            continue
        plans, keep = [], []
        for c in range(copies):
            segs = []
            for l in range(layers):
                if repr_ == "u8":
                    t = (torch.rand(P, device=dev, generator=g) < 0.1).to(torch.uint8)
                    segs.append(D.SegmentSpec(t, LB.SRC_MASK_U8, l))
                elif repr_ == "bits":
                    t = torch.randint(-2**31, 2**31 - 1, (P // 32,), device=dev, dtype=torch.int32, generator=g)
                    segs.append(D.SegmentSpec(t, LB.SRC_MASK_BITS, l, n_elem=P))
                else:
                    t = torch.randint(-2**15, 2**15 - 1, (P,), device=dev, dtype=torch.int16, generator=g)
                    segs.append(D.SegmentSpec(t, LB.SRC_NZ_BF16, l))
                keep.append(t)
            plans.append(D.ProfilePlan(ctx, segs, 0, layers))
        coef = D.coef_tensor(layers, A=0, B=1, device=dev)
        cost = torch.empty(layers, dtype=torch.int64, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        for pl in plans:
            D.profile_layers(ctx, pl, coef, cost=cost, status=st)
        torch.cuda.synchronize()
        # one CUDA graph per plan (phase events become external record nodes)
        ctx.set_timing(True)
        graphs = []
        for pl in plans:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                D.profile_layers(ctx, pl, coef, cost=cost, status=st)
            graphs.append(gr)
        torch.cuda.synchronize()
        ctx.timing_read()
        tot, cnt = 0.0, 0
        for _ in range(3):
            for gr in graphs:
                gr.replay()
                torch.cuda.synchronize()
                ctx.timing_poll()
        ph = ctx.timing_read()
        ctx.set_timing(False)
        ms, cnt = ph["profile"]
        avg = ms / cnt
        b = plans[0].bytes
        res[f"{repr_}_{layers}L"] = dict(bytes=int(b), tiles=int(plans[0].n_tiles), avg_us=round(avg * 1e3, 2),
                                         GBps=round(b / (avg * 1e-3) / 1e9, 1),
                                         frac=round(b / (avg * 1e-3) / 1e9 / peak, 4))
        print(repr_, layers, res[f"{repr_}_{layers}L"], flush=True)
        del plans, keep, graphs
        torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/profile_microbench.json", "w"), indent=1)

"""Alg. 1 global magnitude pruning (NEXT-2) at config-2 scale: 48 layers x
12,582,912 bf16 weights (604 M), layer l's weights ~ N(0, sigma_l^2), split
over G ranks by pipeline stage (8 stages, stage s on GPU floor(s*G/8)), S = 0.9
(k = 10 % of all weights).  One call = dynmo_global_prune over this rank's
layers (histogram passes + NCCL all-reduces + mask pass), captured in a CUDA
graph, timed with CUDA events; max over ranks.  Algorithmic HBM bytes per
rank and call: (1 histogram pass + 1 mask pass) x weight bytes (reads) + 1 B
per weight (mask writes) [+ one more read of the weights when a rank holds a
partial share of the threshold ties that the windowed pass did not count
(d_info[5] bit 1 clear), + one when the bin window missed (bit 0)].  The
1/32 tile sample is not counted (overhead of this design, not of Alg. 1).

python tools/bench_prune.py  |  torchrun --nproc-per-node G ... tools/bench_prune.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402
from paper_2505_14864_b200.pipeline import rank_layers, stage_ranks, uniform_split  # noqa: E402


def mark(msg):
    if os.environ.get("PRUNE_DEBUG"):
        print(f"[rank {os.environ.get('RANK', 0)}] {msg}", file=sys.stderr, flush=True)


def main():
    if os.environ.get("PRUNE_DEBUG"):
        import faulthandler
        faulthandler.dump_traceback_later(45, exit=True)
    rank, G, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if G > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = D.Context(local)
    shape = synth.GPTShape()
    L, P = shape.L, shape.params_per_layer
    b = uniform_split(L, 8)
    begin, count = rank_layers(b, stage_ranks(8, G), rank)
    sig = np.exp(np.random.default_rng(3).normal(0, 0.35, L)) * (1 + np.arange(L) / L) ** 0.5
    gen = torch.Generator(device=dev).manual_seed(2505 + rank)
    ws = [(torch.randn(P, generator=gen, device=dev) * float(sig[l])).to(torch.bfloat16)
          for l in range(begin, begin + count)]
    ms = [torch.empty(P, dtype=torch.uint8, device=dev) for _ in ws]
    plan = D.PrunePlan(ctx, list(zip(ws, ms)))
    k = int(L * P * (1 - 0.9))
    info = torch.empty(6, dtype=torch.int64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    mark("eager call")
    D.global_prune(ctx, plan, k, info=info, status=st)
    torch.cuda.synchronize()
    mark("eager done; capturing")
    use_graph = os.environ.get("PRUNE_GRAPH", "1") == "1"
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream(device=dev)):
            D.global_prune(ctx, plan, k, info=info, status=st)
    torch.cuda.synchronize()
    mark("captured")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    bar = torch.zeros(1, device=dev)
    ts = []
    for it in range(13):
        flush.fill_(it)
        if G > 1:
            dist.all_reduce(bar)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if use_graph:
            g.replay()
        else:
            D.global_prune(ctx, plan, k, info=info, status=st)
        e.record()
        e.synchronize()
        mark(f"replay {it}: {a.elapsed_time(e):.3f} ms")
        if it >= 3:
            ts.append(a.elapsed_time(e))
    mark("loop done")
    inf = info.cpu().numpy()
    mark("info read")
    kept_local = sum(int(m.sum(dtype=torch.int64).item()) for m in ms)
    partial = 0 < inf[3] < inf[4]
    flags = int(inf[5])
    wbytes = count * P * 2
    passes = 1  # all bf16: the 15-bit first digit is the whole magnitude
    extra = (1 if partial and not flags & 2 else 0) + (1 if flags & 1 else 0)
    alg_bytes = (passes + 1 + extra) * wbytes + count * P
    v = torch.tensor([float(np.median(ts)), float(alg_bytes), float(kept_local)], dtype=torch.float64, device=dev)
    if G > 1:
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = v.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    else:
        mx, tot = v, v
    if rank == 0:
        ms_ = float(mx[0])
        print(json.dumps({
            "workload": "Alg. 1 global magnitude pruning, config-2 weights: 48 x 12.58 M bf16 (604 M), S = 0.9",
            "n_gpus": G, "ms_per_call": round(ms_, 4), "k": k, "kept_total": int(tot[2]),
            "status": int(st.item()), "tau_key": int(inf[0]), "flags": flags,
            "max_rank_alg_bytes": int(mx[1]),
            "hbm_GBps_max_rank": round(float(mx[1]) / (ms_ * 1e-3) / 1e9, 1),
        }), flush=True)
    if use_graph:
        del g  # a graph holding NCCL work must go before the communicator
    torch.cuda.synchronize()
    plan.close()
    ctx.close()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

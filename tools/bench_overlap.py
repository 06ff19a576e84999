"""Migration overlapped with compute ("moving layers
while the gradients calculation take place"): 2 GPUs, layers 2..5 of 8
(128 MiB each, 512 MiB in all) move from rank 0 to rank 1 with the
device-driven peer pull (dynmo_migrate_layers_dev) on a high-priority side
stream, while the main stream of both ranks runs the backward stand-in: a
chain of bf16 GEMMs (8192^3, cuBLAS).  For each SM budget of the pull
(dynmo_migrate_plan_set_ctas) it times the GEMM chain alone, the migration
alone and both together (CUDA events, median of reps, max over ranks).

torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/bench_overlap.py
Rank 0 prints one JSON line.
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

from paper_2505_14864_b200 import dynmo as D  # noqa: E402

L, LAYER_BYTES, N_GEMM, M = 8, 128 << 20, 4, 8192
B_OLD, B_NEW, RANKS = [0, 6, 8], [0, 2, 8], [0, 1]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = D.Context(local)
    own = range(B_OLD[rank], B_OLD[rank + 1])
    send = {l: [torch.full((LAYER_BYTES,), l, dtype=torch.uint8, device=dev)] for l in own}
    moved = [l for l in range(L) if (l < B_OLD[1]) != (l < B_NEW[1])]
    recv = {l: [torch.zeros(LAYER_BYTES, dtype=torch.uint8, device=dev)] for l in moved
            if (1 if l >= B_NEW[1] else 0) == rank}
    pm = D.PeerMigrator(ctx, L, send, recv)
    i32 = dict(dtype=torch.int32, device=dev)
    d_bo, d_bn, d_r = torch.tensor(B_OLD, **i32), torch.tensor(B_NEW, **i32), torch.tensor(RANKS, **i32)
    bs, br = torch.zeros(1, dtype=torch.int64, device=dev), torch.zeros(1, dtype=torch.int64, device=dev)
    A = torch.randn(M, M, device=dev, dtype=torch.bfloat16) / M ** 0.5
    Bm = torch.randn(M, M, device=dev, dtype=torch.bfloat16) / M ** 0.5
    C = torch.empty(M, M, device=dev, dtype=torch.bfloat16)
    side = torch.cuda.Stream(device=dev, priority=-1)  # high priority: its CTAs go first as SMs free up
    main = torch.cuda.current_stream()
    bar = torch.zeros(1, device=dev)

    def gemms():
        for _ in range(N_GEMM):
            torch.mm(A, Bm, out=C)

    def migrate():
        pm.device(d_bo, d_r, d_bn, d_r, bs, br)

    def timed(mode, reps=7):
        ts = {"total": [], "gemm": [], "mig": []}
        for it in range(reps + 2):
            dist.all_reduce(bar)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            eg, em = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            if mode in ("mig", "both"):
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    migrate()
                    em.record(side)
            if mode in ("gemm", "both"):
                gemms()
                eg.record(main)
            main.wait_stream(side)
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(main)
            torch.cuda.synchronize()
            if it >= 2:
                ts["total"].append(e0.elapsed_time(e1))
                if mode in ("gemm", "both"):
                    ts["gemm"].append(e0.elapsed_time(eg))
                if mode in ("mig", "both"):
                    ts["mig"].append(e0.elapsed_time(em))
        v = torch.tensor([float(np.median(ts[k])) if ts[k] else 0.0 for k in ("total", "gemm", "mig")],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return [round(x, 4) for x in v.tolist()]

    out = {"workload": f"2 GPUs: 4 layers x 128 MiB (512 MiB) GPU0 -> GPU1 by device-driven peer pull on a "
                       f"high-priority side stream, overlapped with {N_GEMM} bf16 GEMMs {M}^3 per rank on the "
                       f"main stream; CUDA events, median, max over ranks",
           "gemm_alone_ms": timed("gemm")[0]}
    gemm_tflops = N_GEMM * 2 * M ** 3 / (out["gemm_alone_ms"] * 1e-3) / 1e12
    out["gemm_alone_TFLOPs"] = round(gemm_tflops, 1)
    rows = []
    for ctas in (0, 32, 16, 8):
        pm.set_ctas(ctas)
        mig = timed("mig")[0]
        tot, g, m = timed("both")
        for l, bufs in recv.items():
            assert int(bufs[0][:4096].min().item()) == l == int(bufs[0][-4096:].max().item())
        rows.append({"ctas": ctas or torch.cuda.get_device_properties(dev).multi_processor_count,
                     "mig_alone_ms": mig, "mig_alone_GBps": round(4 * LAYER_BYTES / (mig * 1e-3) / 1e9, 1),
                     "both_total_ms": tot, "both_gemm_ms": g, "both_mig_ms": m,
                     "gemm_slowdown": round(g / out["gemm_alone_ms"], 3),
                     "hidden_frac": round((out["gemm_alone_ms"] + mig - tot) / mig, 3)})
    out["budgets"] = rows
    assert pm.error() == 0
    if rank == 0:
        print(json.dumps(out), flush=True)
    pm.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

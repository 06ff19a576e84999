"""Config 4 at G GPUs: Mixtral-8x7B-shaped MoE, 32
layers on 8 stages (stage s on GPU floor(s*G/8)), routing int64 [T, 2] per
layer with T = 64x2048 and expert popularity ~ Dirichlet(alpha); each layer's
migration payload is its bf16 parameters, 2.90 GB (attention 41.9 M + experts
1.409 B params).  One step (one CUDA graph): profile this rank's layers ->
peer-memory exchange -> memory-capped partition -> device-driven migration
of every layer whose GPU changes (receiver pull over NVLink).  The split
before the step is the optimal one for the PREVIOUS routing distribution
(another draw, popularity ~ Dirichlet(prior_alpha)): per-iteration MoE
rebalancing as the routing drifts (from the uniform split with
--prior-alpha 0; at alpha 4 / 64 the uniform split is already optimal and
nothing moves).  Timed with
CUDA events per step, max over ranks.  Also checks the partition against the
oracle and the moved bytes against the oracle's migration plan.

torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/bench_cfg4_mgpu.py [--alpha 4] [--steps 10]
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402
from paper_2505_14864_b200.pipeline import rank_layers, stage_ranks, uniform_split  # noqa: E402

L, N_STAGES, E, K, T = 32, 8, 8, 2, 64 * 2048
PARAMS_PER_LAYER = 41_900_000 + 1_409_000_000   # Mixtral-8x7B layer (attention + 8 experts)
PAYLOAD = PARAMS_PER_LAYER * 2                   # bf16 bytes, 2.90 GB
A_COEF, C_COEF, EP = T, 4, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alpha", type=float, default=4.0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--prior-alpha", type=float, default=0.0)
    ap.add_argument("--force-shift", type=int, default=1,
                    help="migrate to the split whose GPU-border boundaries are shifted by this many layers "
                         "(the computed partition is unchanged at alpha 4/64, so nothing would move)")
    args = ap.parse_args()
    rank, G, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if G > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = D.Context(local)
    payload = np.full(L, PAYLOAD, np.int64)
    cap = int(1.5 * payload.sum() / N_STAGES)
    if args.prior_alpha > 0:  # previous routing state -> its optimal split
        prior = np.array([oracle.layer_cost(cnt=oracle.expert_hist(
            synth.cfg4_routing(l, T=T, E=E, k=K, alpha=args.prior_alpha, seed_key=1), E)[1],
            A=A_COEF, C_=C_COEF, ep=EP)[1] for l in range(L)])
        pst_, b_old, _, _ = oracle.partition(prior, N_STAGES, mem=payload, cap=cap)
        assert pst_ == 0
        b_old = np.asarray(b_old, np.int32)
    else:
        b_old = uniform_split(L, N_STAGES)
    ranks = stage_ranks(N_STAGES, G)
    begin, count = rank_layers(b_old, ranks, rank)

    # inputs: routing of this rank's layers; all layers' expected costs for the oracle
    hists, segs, keep = {}, [], []
    for layer in range(L):
        idx = synth.cfg4_routing(layer, T=T, E=E, k=K, alpha=args.alpha)
        hists[layer] = oracle.expert_hist(idx, E)[1]
        if begin <= layer < begin + count:
            t = torch.from_numpy(idx.reshape(-1)).to(dev)
            keep.append(t)
            segs.append(D.SegmentSpec(t, LB.SRC_EXPERT_I64, layer, n_experts=E, top_k=K))
    want_cost = np.array([oracle.layer_cost(cnt=hists[i], A=A_COEF, C_=C_COEF, ep=EP)[1] for i in range(L)])
    plan = D.ProfilePlan(ctx, segs, begin, count, n_total=L, exchange="p2p" if G > 1 else False)
    coef = D.coef_tensor(count, A=A_COEF, C_=C_COEF, ep=EP, device=dev)
    mem_local = torch.from_numpy(payload[begin:begin + count].copy()).to(dev)
    cost = torch.empty(L, dtype=torch.int64, device=dev)
    mem = torch.empty(L, dtype=torch.int64, device=dev)
    pst = torch.empty(1, dtype=torch.int32, device=dev)
    batch = D.Batch([L], [N_STAGES], device=dev)
    d_cap = torch.tensor([cap], dtype=torch.int64, device=dev)
    bnd = torch.empty(batch.total_bnd, dtype=torch.int32, device=dev)
    bott = torch.empty(1, dtype=torch.int64, device=dev)
    imb = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)

    def solve():
        D.profile_layers(ctx, plan, coef, mem_local=mem_local, cost=cost, mem=mem, status=pst)
        D.partition_stages(ctx, batch, cost, mem=mem, cap=d_cap, bnd=bnd, bottleneck=bott, imbalance=imb, status=st)

    solve()
    torch.cuda.synchronize()
    assert int(pst.item()) == 0 and int(st.item()) == 0, (pst, st)
    assert np.array_equal(cost.cpu().numpy(), want_cost)
    b_new = bnd.cpu().numpy()[:N_STAGES + 1]
    ost, ob, oB, _ = oracle.partition(want_cost, N_STAGES, mem=payload, cap=cap)
    assert ost == 0 and np.array_equal(b_new, ob), (b_new, ob)
    natural_moves = len(D.migration_plan(L, b_old, ranks, b_new, ranks))
    b_mig = b_new.copy()
    if args.force_shift:
        for s_ in range(1, N_STAGES):
            if ranks[s_] != ranks[s_ - 1]:  # a GPU border: shift it (stays valid for shift < 4)
                b_mig[s_] = b_old[s_] + args.force_shift
    moves = D.migration_plan(L, b_old, ranks, b_mig, ranks)
    assert np.array_equal(moves, oracle.moves(L, b_old, ranks, b_mig, ranks))
    sent_w = sum(int(payload[l]) for l, s_, d_ in moves if s_ == rank)
    recv_w = sum(int(payload[l]) for l, s_, d_ in moves if d_ == rank)

    # payload buffers: the layers this rank owns now, and those it will receive
    send = {l: [torch.empty(int(payload[l]), dtype=torch.uint8, device=dev)] for l in range(begin, begin + count)}
    for l, bufs in send.items():
        bufs[0][:4096].fill_(l & 0xFF)
    recv = {int(l): [torch.empty(int(payload[l]), dtype=torch.uint8, device=dev)] for l, s_, d_ in moves if d_ == rank}
    d_bo = torch.from_numpy(b_old.astype(np.int32)).to(dev)
    d_ro = torch.from_numpy(ranks.astype(np.int32)).to(dev)
    d_bytes = torch.zeros(2, dtype=torch.int64, device=dev)
    d_bmig = bnd if not args.force_shift else torch.from_numpy(b_mig.astype(np.int32)).to(dev)
    pm = D.PeerMigrator(ctx, L, send, recv) if G > 1 else None

    def step():
        solve()
        if pm is not None:
            pm.device(d_bo, d_ro, d_bmig, d_ro, d_bytes[0:1], d_bytes[1:2])

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream(device=dev)):
        step()
    torch.cuda.synchronize()
    bar = torch.zeros(1, device=dev)
    for _ in range(args.warmup):
        if G > 1:
            dist.all_reduce(bar)
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        if G > 1:
            dist.all_reduce(bar)  # steps start at a device barrier
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    # byte-exact spot check of the received payloads
    for l, bufs in recv.items():
        assert int(bufs[0][:4096].min().item()) == (l & 0xFF) == int(bufs[0][:4096].max().item()), l
    if pm is not None:
        assert pm.error() == 0
        assert (int(d_bytes[0].item()), int(d_bytes[1].item())) == (sent_w, recv_w)
    v = torch.tensor([float(np.mean(ts)), float(max(sent_w, recv_w))], dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    ms, max_bytes = v.tolist()
    if rank == 0:
        print(json.dumps({
            "workload": f"config4: Mixtral-8x7B-shaped MoE, 32 layers, E=8, k=2, T=131072, alpha={args.alpha}, "
                        f"8 stages, payload 2.90 GB bf16 per layer, previous split optimal for "
                        f"{'alpha=%g routing' % args.prior_alpha if args.prior_alpha > 0 else 'nothing (uniform)'}",
            "n_gpus": G, "steps": args.steps, "ms_per_step": round(ms, 4),
            "b_old": b_old.tolist(), "b_new": b_new.tolist(), "natural_moved_layers": natural_moves,
            "b_migrated_to": b_mig.tolist(), "forced_shift": args.force_shift, "moved_layers": int(len(moves)),
            "max_bytes_per_gpu": int(max_bytes),
            "nvlink_GBps_step": round(max_bytes / (ms * 1e-3) / 1e9, 1) if max_bytes else None,
            "imbalance_old_new": [round(float(oracle.imbalance(np.add.reduceat(want_cost, b_old[:-1]))), 4),
                                  round(float(imb.item()), 4)],
        }), flush=True)
    if pm is not None:
        pm.close()
    ctx.close()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Multi-GPU parity worker (run under torchrun, one rank per GPU).

Each rank profiles only the layers of its own stages (stage s on GPU
floor(s*G/n)), the library all-gathers the cost slots over NCCL, every rank
solves the identical partition, and migrate_layers moves the payload of every
layer whose GPU changes.  Checked against the oracle on the full model:
  - the gathered cost vector == the single-host oracle costs (O3),
  - identical boundaries on every rank == oracle partition,
  - every received payload byte == the sender's deterministic pattern, and
    the byte counts == the oracle's migration plan (O7).
Prints "MGPU_OK <rank>" on success.
"""
from __future__ import annotations

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


def pattern(layer: int, nbytes: int) -> torch.Tensor:
    g = np.random.default_rng(1000 + layer)
    return torch.from_numpy(g.integers(0, 256, nbytes, dtype=np.uint8))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])

    def trace(msg):  # section markers (the test keeps the output even on a timeout)
        print(f"TRACE {rank} {msg}", flush=True)

    import threading

    def watchdog(seconds, tag, streams=()):
        """Prints this rank's peer-window snapshot and its streams' states if
        the section has not finished within `seconds` (hang analysis)."""
        def fire():
            try:
                print(f"WATCHDOG {rank} {tag} streams_idle={[s_.query() for s_ in streams]} "
                      f"window={ctx.window_snapshot(shape.L)}", flush=True)
            except Exception as e:  # pragma: no cover
                print(f"WATCHDOG {rank} {tag} failed: {e!r}", flush=True)
        t = threading.Timer(seconds, fire)
        t.daemon = True
        t.start()
        return t
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = D.Context(local)
    assert ctx.nranks == world
    shape = synth.GPTShape(L=24, h=128)
    n = 8
    b_old = uniform_split(shape.L, n)
    ranks = stage_ranks(n, world)
    begin, count = rank_layers(b_old, ranks, rank)
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    segs, keep = [], []
    want_all = np.zeros(shape.L, np.int64)
    for layer in range(shape.L):
        for m in synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4):
            want_all[layer] += oracle.count_nz_u8(m)
            if begin <= layer < begin + count:
                t = torch.from_numpy(m.reshape(-1)).to(dev)
                keep.append(t)
                segs.append(D.SegmentSpec(t, LB.SRC_MASK_U8, layer))
    want_cost = np.array([oracle.layer_cost(nnz=int(v), A=0, B=1)[1] for v in want_all])
    payload = (synth.cfg2_payload_bytes(shape, p) // 64).astype(np.int64)  # smaller transfers
    coef = D.coef_tensor(count, A=0, B=1, device=dev)
    mem_local = torch.from_numpy(payload[begin:begin + count].copy()).to(dev)
    mem = torch.empty(shape.L, dtype=torch.int64, device=dev)
    for mode in ("nccl", "p2p"):
        plan = D.ProfilePlan(ctx, segs, begin, count, n_total=shape.L, exchange=mode)
        for rep in range(3):  # several epochs (both slot parities)
            cost, _, st = D.profile_layers(ctx, plan, coef, mem_local=mem_local, mem=mem)
            torch.cuda.synchronize()
            assert int(st.item()) == 0, (mode, st)
            assert np.array_equal(cost.cpu().numpy(), want_cost), (mode, rank, cost.cpu().numpy(), want_cost)
            assert np.array_equal(mem.cpu().numpy(), payload)
    # back-to-back calls without host synchronisation (fast ranks may run ahead)
    outs = []
    for rep in range(6):
        c_, _, st_ = D.profile_layers(ctx, plan, coef, mem_local=mem_local)
        outs.append((c_.clone(), st_.clone()))
    torch.cuda.synchronize()
    for c_, st_ in outs:
        assert int(st_.item()) == 0 and np.array_equal(c_.cpu().numpy(), want_cost)
    # identical partition on every rank == oracle
    b = D.Batch([shape.L], [n], device=dev)
    bnd, bott, _, pst = D.partition_stages(ctx, b, cost)
    ost, ob, oB, _ = oracle.partition(want_cost, n)
    b_new = bnd.cpu().numpy()
    assert int(pst.item()) == 0 and np.array_equal(b_new, ob) and int(bott.item()) == oB
    allb = [None] * world
    dist.all_gather_object(allb, b_new.tolist())
    assert all(x == allb[0] for x in allb)
    trace('migration')
    # migration: senders hold the pattern, receivers get it
    send = {l: [pattern(l, int(payload[l])).to(dev)] for l in range(begin, begin + count)}
    moves = oracle.moves(shape.L, b_old, ranks, b_new, ranks)
    assert np.array_equal(D.migration_plan(shape.L, b_old, ranks, b_new, ranks), moves)
    recv = {int(l): [torch.zeros(int(payload[l]), dtype=torch.uint8, device=dev)]
            for l, s_, d_ in moves if d_ == rank}
    sent, got = D.migrate_layers(ctx, shape.L, b_old, ranks, b_new, ranks, send, recv)
    torch.cuda.synchronize()
    want_sent = int(sum(payload[l] for l, s_, d_ in moves if s_ == rank))
    want_got = int(sum(payload[l] for l, s_, d_ in moves if d_ == rank))
    assert (sent, got) == (want_sent, want_got), (rank, sent, got, want_sent, want_got)
    for l, bufs in recv.items():
        assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l)
    # second round-trip of the same plan (steady state) still exact
    for bufs in recv.values():
        bufs[0].zero_()
    D.migrate_layers(ctx, shape.L, b_old, ranks, b_new, ranks, send, recv)
    torch.cuda.synchronize()
    for l, bufs in recv.items():
        assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l])))
    trace('the same moves over NVLink peer memory (')
    # the same moves over NVLink peer memory (IPC-mapped pull kernel)
    for bufs in recv.values():
        bufs[0].zero_()
    pm = D.PeerMigrator(ctx, shape.L, send, recv)
    for rep in range(3):
        for bufs in recv.values():
            bufs[0].zero_()
        s2, g2 = pm(b_old, ranks, b_new, ranks)
        torch.cuda.synchronize()
        assert (s2, g2) == (want_sent, want_got), (rank, s2, g2)
        for l, bufs in recv.items():
            assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l, rep)
    trace('device-driven variant')
    # device-driven variant: boundaries straight from the partition output,
    # captured in a CUDA graph together with the partition (several replays)
    d_bo, d_ro = torch.from_numpy(b_old.astype(np.int32)).to(dev), torch.from_numpy(ranks.astype(np.int32)).to(dev)
    d_rn = d_ro.clone()
    bs, br = torch.zeros(1, dtype=torch.int64, device=dev), torch.zeros(1, dtype=torch.int64, device=dev)
    for bufs in recv.values():
        bufs[0].zero_()
    pm.device(d_bo, d_ro, bnd, d_rn, bs, br)
    torch.cuda.synchronize()
    assert (int(bs.item()), int(br.item())) == (want_sent, want_got), (rank, bs, br)
    for l, bufs in recv.items():
        assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l, "dev")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        D.partition_stages(ctx, b, cost, bnd=bnd)
        pm.device(d_bo, d_ro, bnd, d_rn, bs, br)
    for rep in range(4):
        for bufs in recv.values():
            bufs[0].zero_()
        g.replay()
        torch.cuda.synchronize()
        for l, bufs in recv.items():
            assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l, "graph", rep)
    trace('NEXT-3 overlap')
    # NEXT-3 overlap: the pull under a 2-CTA SM budget on a side stream while
    # the main stream runs a GEMM (the backward stand-in): byte-exact
    pm.set_ctas(2)
    side = torch.cuda.Stream(device=dev)
    for bufs in recv.values():
        bufs[0].zero_()
    A = torch.randn(2048, 2048, device=dev, dtype=torch.bfloat16)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        pm.device(d_bo, d_ro, bnd, d_rn, bs, br)
    for _ in range(8):
        A = (A @ A).clamp_(-1, 1)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    assert (int(bs.item()), int(br.item())) == (want_sent, want_got), (rank, "budget")
    for l, bufs in recv.items():
        assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l, "budget")
    pm.set_ctas(0)
    assert pm.error() == 0
    pm.close()
    trace('NEXT-3 placement')
    # NEXT-3 placement: the new stages on capacity slots (slot j on GPU
    # ranks[j]) keeping the most payload in place; the device-driven pull
    # follows the mapped ranks (a non-identity stage -> rank map)
    slots = torch.arange(n, dtype=torch.int32, device=dev)
    rn_t, kept_t, mst = D.map_stages(ctx, shape.L, d_bo, slots, bnd, mem, n, slot_rank=d_ro)
    torch.cuda.synchronize()
    ost_m, orn_m, okept_m = oracle.map_stages(shape.L, b_old, np.arange(n), b_new, payload, n, slot_rank=ranks)
    assert int(mst.item()) == ost_m == 0 and np.array_equal(rn_t.cpu().numpy(), orn_m)
    assert int(kept_t.item()) == okept_m >= int(payload.sum()) - sum(int(payload[l]) for l, _, _ in moves)
    moves2 = oracle.moves(shape.L, b_old, ranks, b_new, orn_m)
    recv2 = {int(l): [torch.zeros(int(payload[l]), dtype=torch.uint8, device=dev)] for l, s_, d_ in moves2 if d_ == rank}
    pm2 = D.PeerMigrator(ctx, shape.L, send, recv2)
    pm2.device(d_bo, d_ro, bnd, rn_t, bs, br)
    torch.cuda.synchronize()
    assert (int(bs.item()), int(br.item())) == (sum(int(payload[l]) for l, s_, _ in moves2 if s_ == rank),
                                              sum(int(payload[l]) for l, _, d_ in moves2 if d_ == rank))
    for l, bufs in recv2.items():
        assert torch.equal(bufs[0].cpu(), pattern(l, int(payload[l]))), (rank, l, "mapped")
    assert pm2.error() == 0
    pm2.close()
    trace('ranks without layers (more GPUs than lay')
    # ranks without layers (more GPUs than layers): 2 layers over `world`
    # ranks, ranks >= 2 hold empty slices; the peer-memory and NCCL exchanges
    # still give every rank the full cost vector
    tiny = [np.full(1000 + 17 * l, 1, np.uint8) for l in range(2)]
    lb0, cnt0 = (rank, 1) if rank < 2 else (2, 0)
    segs0 = []
    for l in range(lb0, lb0 + cnt0):
        t0_ = torch.from_numpy(tiny[l]).to(dev)
        keep.append(t0_)
        segs0.append(D.SegmentSpec(t0_, LB.SRC_MASK_U8, l))
    for mode0 in ("p2p", "nccl"):
        plan0 = D.ProfilePlan(ctx, segs0, lb0, cnt0, n_total=2, exchange=mode0)
        for rep0 in range(2):
            c0, _, st0 = D.profile_layers(ctx, plan0, D.coef_tensor(max(cnt0, 1), B=1, device=dev))
            torch.cuda.synchronize()
            assert int(st0.item()) == 0 and c0.cpu().tolist() == [1000, 1017], (rank, mode0, c0.cpu().tolist())
        plan0.close()
    trace('several buffers per layer (a CSR payload')
    # several buffers per layer (a CSR payload is values, indices and
    # optimizer state): 3 buffers of different sizes and dtypes per layer,
    # through NCCL send/recv, the host-driven and the device-driven pull
    def bufs_of(l):
        nb_ = int(payload[l])
        return [pattern(l, nb_), pattern(l + 100, nb_ // 3 + 1).view(torch.uint8),
                torch.from_numpy(np.arange(nb_ // 7 + 1, dtype=np.int32) * (l + 1))]
    send3 = {l: [t.to(dev) for t in bufs_of(l)] for l in range(begin, begin + count)}
    recv3 = {int(l): [torch.zeros_like(t, device=dev) for t in bufs_of(int(l))] for l, s_, d_ in moves if d_ == rank}
    want3_s = sum(sum(t.numel() * t.element_size() for t in bufs_of(int(l))) for l, s_, d_ in moves if s_ == rank)
    want3_r = sum(sum(t.numel() * t.element_size() for t in bufs_of(int(l))) for l, s_, d_ in moves if d_ == rank)
    for mode in ("nccl", "p2p", "dev"):
        for bufs in recv3.values():
            for t in bufs:
                t.zero_()
        if mode == "nccl":
            s3, r3 = D.migrate_layers(ctx, shape.L, b_old, ranks, b_new, ranks, send3, recv3, n_bufs=3)
        else:
            pm3 = D.PeerMigrator(ctx, shape.L, send3, recv3, n_bufs=3)
            if mode == "p2p":
                s3, r3 = pm3(b_old, ranks, b_new, ranks)
            else:
                pm3.device(d_bo, d_ro, bnd, d_ro, bs, br)
        torch.cuda.synchronize()
        if mode == "dev":
            s3, r3 = int(bs.item()), int(br.item())
            assert pm3.error() == 0
        if mode != "nccl":
            pm3.close()
        assert (s3, r3) == (want3_s, want3_r), (rank, mode, s3, r3, want3_s, want3_r)
        for l, bufs in recv3.items():
            for t, w in zip(bufs, bufs_of(l)):
                assert torch.equal(t.cpu(), w), (rank, mode, l)
    trace('Alg. 1 global pruning across ranks (NCCL')
    # Alg. 1 global pruning across ranks (NCCL all-reduce of the histograms,
    # all-gather of the tie counts): every rank's masks == the oracle's on the
    # concatenation of all ranks' shards in rank order; quantised magnitudes
    # so ties straddle the rank boundary
    shards_all, vals_all = [], []
    for r in range(world):
        gr = np.random.default_rng(700 + r)
        sz = [9000 + 1000 * r, 17]
        sh_r = []
        for j, n_ in enumerate(sz):
            x = np.round(gr.normal(0, 1, n_) * 4) / 4
            if j == 0:
                w = x.astype(np.float32)
                sh_r.append((w, w.astype(np.float64), torch.float32))
            else:
                tb = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
                sh_r.append((tb, oracle.bf16_to_f64(tb.view(torch.int16).numpy().view(np.uint16)), torch.bfloat16))
        shards_all.append(sh_r)
        vals_all += [v for _, v, _ in sh_r]
    mine = shards_all[rank]
    wt = [torch.as_tensor(w).to(dev) for w, _, _ in mine]
    mk = [torch.zeros(t.numel(), dtype=torch.uint8, device=dev) for t in wt]
    pplan = D.PrunePlan(ctx, list(zip(wt, mk)))
    Ntot = sum(v.size for v in vals_all)
    first = sum(len(shards_all[r]) for r in range(rank))
    for kk in (0, 1, Ntot // 3, Ntot // 2 + 7, Ntot):
        info, pst2 = D.global_prune(ctx, pplan, kk)
        torch.cuda.synchronize()
        ost2, om = oracle.global_prune(vals_all, kk)
        assert int(pst2.item()) == ost2 == 0
        for j, m in enumerate(mk):
            assert np.array_equal(m.cpu().numpy(), om[first + j]), (rank, kk, j)
    pplan.close()
    # the same over all-bf16 shards of several 32768-element tiles per rank
    # (N(0, 1) weights: ties of the threshold bin on every rank): the bin
    # window holds the k-th key and, on the rank with the partial tie share,
    # the tie counts come from the windowed pass (d_info[5] bit 1)
    shards_all, vals_all = [], []
    for r in range(world):
        gr = np.random.default_rng(900 + r)
        x = gr.normal(0, 1, 3 * 32768 + 500 * (r + 1))
        tb = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
        shards_all.append(tb)
        vals_all.append(oracle.bf16_to_f64(tb.view(torch.int16).numpy().view(np.uint16)))
    wt = shards_all[rank].to(dev)
    mk = torch.zeros(wt.numel(), dtype=torch.uint8, device=dev)
    pplan = D.PrunePlan(ctx, [(wt, mk)])
    Ntot = sum(v.size for v in vals_all)
    for kk in (Ntot // 10, Ntot // 5):
        info, pst2 = D.global_prune(ctx, pplan, kk)
        torch.cuda.synchronize()
        ost2, om = oracle.global_prune(vals_all, kk)
        assert int(pst2.item()) == ost2 == 0
        assert np.array_equal(mk.cpu().numpy(), om[rank]), (rank, kk)
        flags = torch.tensor([int(info[5].item())], device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)
        assert int(flags.item()) == 2, (rank, kk, int(flags.item()))  # hit; counted ties on the partial rank
    pplan.close()
    # different dtype sets per rank (rank 0 bf16 only, the others f32): the
    # collective plan creation makes every rank run the f32 passes
    shards_all, vals_all = [], []
    for r in range(world):
        gr = np.random.default_rng(950 + r)
        x = np.round(gr.normal(0, 1, 40000 + 300 * r) * 64) / 64  # ties across ranks
        if r == 0:
            tb = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
            shards_all.append(tb)
            vals_all.append(oracle.bf16_to_f64(tb.view(torch.int16).numpy().view(np.uint16)))
        else:
            w = x.astype(np.float32)
            shards_all.append(torch.from_numpy(w))
            vals_all.append(w.astype(np.float64))
    wt = shards_all[rank].to(dev)
    mk = torch.zeros(wt.numel(), dtype=torch.uint8, device=dev)
    pplan = D.PrunePlan(ctx, [(wt, mk)])
    Ntot = sum(v.size for v in vals_all)
    for kk in (Ntot // 7, Ntot // 2 + 3):
        info, pst2 = D.global_prune(ctx, pplan, kk)
        torch.cuda.synchronize()
        ost2, om = oracle.global_prune(vals_all, kk)
        assert int(pst2.item()) == ost2 == 0
        assert np.array_equal(mk.cpu().numpy(), om[rank]), (rank, kk, "mixed dtype sets")
    pplan.close()
    # a rank without weights (the last one): empty plan, still in every collective
    shards_all, vals_all = [], []
    for r in range(world):
        gr = np.random.default_rng(970 + r)
        n_r = 0 if r == world - 1 else 2 * 32768 + 77 * r
        tb = torch.from_numpy(gr.normal(0, 1, n_r).astype(np.float32)).to(torch.bfloat16)
        shards_all.append(tb)
        vals_all.append(oracle.bf16_to_f64(tb.view(torch.int16).numpy().view(np.uint16)))
    if rank == world - 1:
        pplan = D.PrunePlan(ctx, [])
    else:
        wt = shards_all[rank].to(dev)
        mk = torch.zeros(wt.numel(), dtype=torch.uint8, device=dev)
        pplan = D.PrunePlan(ctx, [(wt, mk)])
    Ntot = sum(v.size for v in vals_all)
    for kk in (Ntot // 10, Ntot):
        info, pst2 = D.global_prune(ctx, pplan, kk)
        torch.cuda.synchronize()
        ost2, om = oracle.global_prune(vals_all, kk)
        assert int(pst2.item()) == ost2 == 0
        assert int(info[1].item()) == Ntot
        if rank != world - 1:
            assert np.array_equal(mk.cpu().numpy(), om[rank]), (rank, kk, "empty rank")
    pplan.close()
    trace('NEXT-3 (P')
    # NEXT-3: migration overlapped with the backward pass, last
    # layer first.  Payload per layer = [gradients, params]; the "backward"
    # on the main stream computes (a GEMM stand-in), writes each owned
    # layer's gradient buffer with this iteration's value right before its
    # ready flag; receivers pull on a side stream under an SM budget.  A pull
    # that ran ahead of a flag would copy the previous iteration's gradients.
    def grad_val(l, it):
        return (l * 7 + it + 1) & 0xFF
    sendb = {l: [torch.zeros(int(payload[l]), dtype=torch.uint8, device=dev), pattern(l, int(payload[l]) // 2 + 1).to(dev)]
             for l in range(begin, begin + count)}
    recvb = {int(l): [torch.zeros(int(payload[l]), dtype=torch.uint8, device=dev),
                      torch.zeros(int(payload[l]) // 2 + 1, dtype=torch.uint8, device=dev)]
             for l, s_, d_ in moves if d_ == rank}
    pmb = D.PeerMigrator(ctx, shape.L, sendb, recvb, n_bufs=2)
    pmb.set_ctas(8)
    side_b = torch.cuda.Stream(device=dev)
    Ab = torch.randn(1024, 1024, device=dev, dtype=torch.bfloat16)
    # warm-up of the backward stand-in without migration: every kernel that
    # runs while the pull spins must already be loaded (CUDA lazy loading may
    # synchronise the context on a first launch; see dynmo.h)
    for l in range(begin + count - 1, begin - 1, -1):
        Ab = (Ab @ Ab).clamp_(-1, 1)
        sendb[l][0].fill_(grad_val(l, -1))
    torch.cuda.synchronize()
    for it in range(4):
        main = torch.cuda.current_stream()
        pmb.bwd_begin()
        side_b.wait_stream(main)
        with torch.cuda.stream(side_b):
            pmb.backward(d_bo, d_ro, bnd, d_rn, br)
        for l in range(begin + count - 1, begin - 1, -1):  # backward: last layer first
            for _ in range(2):
                Ab = (Ab @ Ab).clamp_(-1, 1)
            sendb[l][0].fill_(grad_val(l, it))
            pmb.layer_ready(l)
        pmb.bwd_end(d_bo, d_ro, bnd, d_rn, bs)
        main.wait_stream(side_b)
        torch.cuda.synchronize()
        assert pmb.error() == 0, (rank, it, pmb.error())
        assert (int(bs.item()), int(br.item())) == (
            sum(int(payload[l]) + int(payload[l]) // 2 + 1 for l, s_, _ in moves if s_ == rank),
            sum(int(payload[l]) + int(payload[l]) // 2 + 1 for l, _, d_ in moves if d_ == rank)), (rank, it, "bwd bytes")
        for l, bufs in recvb.items():
            assert bool((bufs[0] == grad_val(l, it)).all()), (rank, it, l, "bwd grads")
            assert torch.equal(bufs[1].cpu(), pattern(l, int(payload[l]) // 2 + 1)), (rank, it, l, "bwd params")
    trace('multi-chunk payloads (the pulls claim 25')
    # multi-chunk payloads (the pulls claim 256 KiB chunks shared with the
    # drain of dynmo_migrate_bwd_end): per layer an odd-sized 0.8 MB buffer,
    # an unaligned view (byte copies) and an empty buffer; some iterations
    # issue bwd_end only after a host delay so the budgeted per-layer pulls
    # copy most chunks, others right away so the drain takes them over
    def big(l, it):
        g2 = np.random.default_rng(50_000 + 97 * l + it)
        return torch.from_numpy(g2.integers(0, 256, 3 * (256 << 10) + 17 + 4099 * l, dtype=np.uint8))
    sendc = {l: [torch.zeros(3 * (256 << 10) + 17 + 4099 * l, dtype=torch.uint8, device=dev),
                 torch.zeros(70001 + l, dtype=torch.uint8, device=dev)[1:],
                 torch.zeros(0, dtype=torch.uint8, device=dev)]
             for l in range(begin, begin + count)}
    recvc = {int(l): [torch.zeros(3 * (256 << 10) + 17 + 4099 * int(l), dtype=torch.uint8, device=dev),
                      torch.zeros(70001 + int(l), dtype=torch.uint8, device=dev)[1:],
                      torch.zeros(0, dtype=torch.uint8, device=dev)]
             for l, s_, d_ in moves if d_ == rank}
    pmc = D.PeerMigrator(ctx, shape.L, sendc, recvc, n_bufs=3)
    trace("chunks: plan")
    pmc.set_ctas(4)
    # this iteration's payloads staged on the device beforehand: between
    # bwd_begin and the last layer_ready the host must not wait on the device
    # (peers' streams wait for this rank's releases, as in a collective)
    bigs = {(l, it): big(l, it).to(dev) for l in range(begin, begin + count) for it in range(6)}
    # warm-up of every kernel the loop launches between bwd_begin and the last
    # layer_ready (the fill of an UNALIGNED view is its own kernel): a first
    # launch there may lazily load a module, which waits for the context to
    # go idle while the side stream waits for this rank's later releases
    for l in range(begin, begin + count):
        sendc[l][0].copy_(bigs[(l, 0)])
        sendc[l][1].fill_(1)
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()
    trace("chunks: staged")
    for it in range(6):
        main = torch.cuda.current_stream()
        wd = watchdog(30.0, f"chunks it {it}", (main, side_b))
        for bufs in recvc.values():
            bufs[0].zero_()
            bufs[1].zero_()
        pmc.bwd_begin()
        side_b.wait_stream(main)
        with torch.cuda.stream(side_b):
            pmc.backward(d_bo, d_ro, bnd, d_rn, br)
        for l in range(begin + count - 1, begin - 1, -1):
            Ab = (Ab @ Ab).clamp_(-1, 1)
            sendc[l][0].copy_(bigs[(l, it)])
            sendc[l][1].fill_(grad_val(l, it))
            pmc.layer_ready(l)
        trace(f"chunks: it {it} released")
        if it % 2:
            torch.cuda._sleep(2_000_000)  # ~1 ms: the budgeted pulls run first
        pmc.bwd_end(d_bo, d_ro, bnd, d_rn, bs)
        trace(f"chunks: it {it} end issued")
        main.wait_stream(side_b)
        torch.cuda.synchronize()
        wd.cancel()
        trace(f"chunks: it {it} synced err={pmc.error()}")
        assert pmc.error() == 0, (rank, it, pmc.error())
        nb = lambda l: 3 * (256 << 10) + 17 + 4099 * int(l) + 70000 + int(l)  # noqa: E731
        assert (int(bs.item()), int(br.item())) == (sum(nb(l) for l, s_, _ in moves if s_ == rank),
                                                    sum(nb(l) for l, _, d_ in moves if d_ == rank)), (rank, it, "chunks")
        for l, bufs in recvc.items():
            assert torch.equal(bufs[0].cpu(), big(l, it)), (rank, it, l, "chunked big")
            assert bool((bufs[1] == grad_val(l, it)).all()), (rank, it, l, "chunked unaligned")
    # failure path: the last rank skips the release of its first layer (a
    # peer that died or skipped a call).  Every rank's side stream waits for
    # that release without bound; a host watchdog sees the iteration overrun
    # and calls dynmo_migrate_bwd_abort, which releases this rank's own waits
    # and sets the sticky error.  The next iteration is exact again.
    trace("chunks: abort")
    import time as _time
    for it, skip in ((100, True), (101, False)):
        main = torch.cuda.current_stream()
        for bufs in recvc.values():
            bufs[0].zero_()
            bufs[1].zero_()
        pmc.bwd_begin()
        side_b.wait_stream(main)
        with torch.cuda.stream(side_b):
            pmc.backward(d_bo, d_ro, bnd, d_rn, br)
        for l in range(begin + count - 1, begin - 1, -1):
            Ab = (Ab @ Ab).clamp_(-1, 1)
            sendc[l][0].copy_(bigs[(l, it % 6)])
            sendc[l][1].fill_(grad_val(l, it))
            if not (skip and rank == world - 1 and l == begin):
                pmc.layer_ready(l)
        pmc.bwd_end(d_bo, d_ro, bnd, d_rn, bs)
        main.wait_stream(side_b)
        ev = torch.cuda.Event()
        ev.record(main)
        t0 = _time.time()
        while not ev.query() and _time.time() - t0 < 3.0:
            _time.sleep(0.01)
        aborted = not ev.query()
        if aborted:
            pmc.bwd_abort()
        torch.cuda.synchronize()
        flags = torch.tensor([1 if aborted else 0], device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        if skip:
            assert int(flags.item()) == 1, (rank, "every rank waits for the skipped release")
            assert pmc.error() == -5, (rank, pmc.error())
            pmc.clear_error()
        else:
            assert not aborted, (rank, "clean iteration after an abort")
            for l, bufs in recvc.items():
                assert torch.equal(bufs[0].cpu(), big(l, it % 6)), (rank, it, l, "after abort")
                assert bool((bufs[1] == grad_val(l, it)).all()), (rank, it, l, "after abort")
    trace("chunks: abort done")
    pmc.close()
    pmb.set_ctas(0)
    try:
        pmb.backward(d_bo, d_ro, bnd, d_rn, br)  # no SM budget: refused on the host
        raised = False
    except RuntimeError:
        raised = True
    assert raised
    pmb.close()
    trace('ADVICE r1 (high)')
    # the host-driven pull with a CHANGING set of ranks
    # that move data between calls (some ranks sit calls out).  Epochs are
    # per directed rank pair, so every call is exact whatever the history.
    recv_all = {l: [torch.zeros(int(payload[l]), dtype=torch.uint8, device=dev)]
                for l in range(shape.L) if not (begin <= l < begin + count)}
    pmx = D.PeerMigrator(ctx, shape.L, send, recv_all)
    seq = []
    for r_src, r_dst in [(0, 1), (world - 1, 0), (1, world - 1), (0, 1), (world - 1, 0), (1, 0)]:
        if r_src == r_dst:
            continue
        rn_x = ranks.copy()
        s_src = [s_ for s_ in range(n) if ranks[s_] == r_src]
        rn_x[s_src[-1]] = r_dst  # the last stage of r_src moves to r_dst
        seq.append(rn_x)
    for it, rn_x in enumerate(seq * 2):
        mv = oracle.moves(shape.L, b_old, ranks, b_old, rn_x)
        for l, s_, d_ in mv:
            if d_ == rank:
                recv_all[int(l)][0].zero_()
        sx, gx = pmx(b_old, ranks, b_old, rn_x)
        torch.cuda.synchronize()
        assert sx == sum(int(payload[l]) for l, s_, _ in mv if s_ == rank), (rank, it, "changing sets")
        assert gx == sum(int(payload[l]) for l, _, d_ in mv if d_ == rank), (rank, it, "changing sets")
        for l, s_, d_ in mv:
            if d_ == rank:
                assert torch.equal(recv_all[int(l)][0].cpu(), pattern(int(l), int(payload[l]))), (rank, it, int(l))
    assert pmx.error() == 0
    pmx.close()
    trace('ADVICE r1 (medium)')
    # a plan-creation failure on ONE rank fails the
    # collective plan creation on EVERY rank instead of leaving the others in
    # the setup all-gather
    bad_segs = segs if rank != 0 else segs + [D.SegmentSpec(keep[0], LB.SRC_MASK_U8, shape.L + 5)]
    try:
        D.ProfilePlan(ctx, bad_segs, begin, count, n_total=shape.L, exchange="p2p")
        raised = False
    except RuntimeError:
        raised = True
    assert raised, (rank, "profile plan agreement")
    bad_send = dict(send)
    if rank == 0:
        bad_send[begin] = [torch.zeros(16, dtype=torch.uint8)]  # host memory: not IPC-mappable
    try:
        D.PeerMigrator(ctx, shape.L, bad_send, recv_all)
        raised = False
    except (RuntimeError, ValueError):
        raised = True
    assert raised, (rank, "migrate plan agreement")
    # a plan after the failed ones still works (no rank is out of step)
    plan_ok = D.ProfilePlan(ctx, segs, begin, count, n_total=shape.L, exchange="p2p")
    c_ok, _, st_ok = D.profile_layers(ctx, plan_ok, coef)
    torch.cuda.synchronize()
    assert int(st_ok.item()) == 0 and np.array_equal(c_ok.cpu().numpy(), want_cost)
    plan_ok.close()
    trace('ADVICE r1 (medium)')
    # a stage -> rank entry outside [0, nranks) (the -1 a
    # failed map_stages writes) moves nothing and reports INVALID on every
    # rank -- no out-of-bounds table read, no hang.  Last: the error is sticky.
    pmb = D.PeerMigrator(ctx, shape.L, send, recv_all)
    for t in recv_all.values():
        t[0].fill_(7)
    rn_bad = d_ro.clone()
    rn_bad[n - 1] = -1
    pmb.device(d_bo, d_ro, bnd, rn_bad, bs, br)
    torch.cuda.synchronize()
    assert pmb.error() == LB.E_INVALID, (rank, pmb.error())
    assert all(bool((t[0] == 7).all()) for t in recv_all.values()), rank
    pmb.close()
    trace('Releasing GPUs after re-packing (P')
    # Releasing GPUs after re-packing: split the ctx -- even
    # ranks stay active, odd ranks are released (None) -- then the smaller
    # group profiles, partitions and maps its stages onto its own ranks
    sub = ctx.split(active=(rank % 2 == 0))
    if rank % 2:
        assert sub is None
    else:
        assert sub.nranks == (world + 1) // 2 and sub.rank == rank // 2
        Gs = sub.nranks
        n2 = 4
        b2 = uniform_split(shape.L, n2)
        r2 = np.array([s_ * Gs // n2 for s_ in range(n2)], np.int32)
        beg2, cnt2 = rank_layers(b2, r2, sub.rank)
        segs2 = []
        for layer in range(beg2, beg2 + cnt2):
            for m in synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4):
                t = torch.from_numpy(m.reshape(-1)).to(dev)
                keep.append(t)
                segs2.append(D.SegmentSpec(t, LB.SRC_MASK_U8, layer))
        plan2 = D.ProfilePlan(sub, segs2, beg2, cnt2, n_total=shape.L, exchange="p2p" if Gs > 1 else False)
        mem2 = torch.empty(shape.L, dtype=torch.int64, device=dev)
        cost2, _, st2 = D.profile_layers(sub, plan2, D.coef_tensor(cnt2, A=0, B=1, device=dev),
                                         mem_local=torch.from_numpy(payload[beg2:beg2 + cnt2].copy()).to(dev), mem=mem2)
        b2t = D.Batch([shape.L], [n2], device=dev)
        bnd2, _, _, pst2 = D.partition_stages(sub, b2t, cost2)
        torch.cuda.synchronize()
        assert int(st2.item()) == 0 and int(pst2.item()) == 0
        assert np.array_equal(cost2.cpu().numpy(), want_cost)
        ost2, ob2, _, _ = oracle.partition(want_cost, n2)
        assert np.array_equal(bnd2.cpu().numpy()[:n2 + 1], ob2)
        # one stage per active GPU after the re-pack: where to put them
        if Gs > 1:
            bn2_h = np.array([0, int(ob2[n2 // 2]), shape.L], np.int32)  # 2 workers after the re-pack
            bn2 = torch.from_numpy(bn2_h).to(dev)
            rn2, kept2, mst = D.map_stages(sub, shape.L, torch.from_numpy(b2.astype(np.int32)).to(dev),
                                           torch.from_numpy(r2).to(dev), bn2, mem2, Gs)
            torch.cuda.synchronize()
            ost3, orn3, okept3 = oracle.map_stages(shape.L, b2, r2, bn2_h, payload, Gs)
            assert int(mst.item()) == ost3 == 0 and np.array_equal(rn2.cpu().numpy(), orn3)
            assert int(kept2.item()) == okept3
        plan2.close()
        sub.close()
    dist.barrier()
    print(f"MGPU_OK {rank} layers[{begin},{begin + count}) moves={len(moves)} sent={sent} recv={got}", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

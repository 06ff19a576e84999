"""One small rebalancing step on cuda:0 through the C-ABI, checked against the
oracle (used by __graft_entry__.smoke()): pruning masks in three
representations -> profile_layers -> partition_stages -> diffuse_balance ->
repack_workers, plus the by-Time source with a device timestamp, global
pruning (Alg. 1) and the stage -> rank map, all compared bit-exactly with
oracle/."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth


def run_smoke() -> None:
    from paper_2505_14864_b200 import _lib as L
    from paper_2505_14864_b200 import dynmo as D

    assert torch.cuda.is_available(), "smoke() needs a GPU"
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    shape = synth.GPTShape(L=12, h=64)
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    ctx = D.Context(0)
    segs, keep, want_nnz = [], [], np.zeros(shape.L, np.int64)
    for layer in range(shape.L):
        for t, m in enumerate(synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4)):
            if layer % 3 == 0:
                d = torch.from_numpy(m.reshape(-1)).to(dev)
                segs.append(D.SegmentSpec(d, L.SRC_MASK_U8, layer))
                want_nnz[layer] += oracle.count_nz_u8(m)
            elif layer % 3 == 1:
                w = synth.pack_bits(m)
                d = torch.from_numpy(w.view(np.int32)).to(dev)
                segs.append(D.SegmentSpec(d, L.SRC_MASK_BITS, layer, n_elem=m.size))
                want_nnz[layer] += oracle.count_bits(w, m.size)
            else:
                bf = synth.cfg2_bf16_weights(m, layer, t)
                d = torch.from_numpy(bf.view(np.int16)).to(dev)
                segs.append(D.SegmentSpec(d, L.SRC_NZ_BF16, layer))
                want_nnz[layer] += oracle.count_nz_bf16(bf)
            keep.append(d)
    plan = D.ProfilePlan(ctx, segs, 0, shape.L)
    coef = D.coef_tensor(shape.L, A=0, B=1, device=dev)
    counters = torch.empty((shape.L, 5), dtype=torch.int64, device=dev)
    cost, _, st = D.profile_layers(ctx, plan, coef, counters=counters)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    want_cost = np.array([oracle.layer_cost(nnz=int(v), A=0, B=1)[1] for v in want_nnz])
    assert np.array_equal(counters[:, 0].cpu().numpy(), want_nnz), "nnz mismatch"
    assert np.array_equal(cost.cpu().numpy(), want_cost), "cost mismatch"

    n = 4
    b = D.Batch([shape.L], [n], device=dev)
    bnd, bott, imb, pst = D.partition_stages(ctx, b, cost)
    ost, ob, oB, oimb = oracle.partition(want_cost, n)
    torch.cuda.synchronize()
    assert int(pst.item()) == ost == 0
    assert np.array_equal(bnd.cpu().numpy(), ob) and int(bott.item()) == oB and float(imb.item()) == oimb

    uni = np.rint(np.linspace(0, shape.L, n + 1)).astype(np.int32)
    o = D.diffuse_balance(ctx, b, cost, torch.from_numpy(uni).to(dev), max_rounds=64,
                          gamma_fluid=torch.tensor([1e-9], dtype=torch.float64, device=dev))
    dst, db, dr, dphi, dphi0 = oracle.diffuse(want_cost, uni, 0, 64)
    fst, fx, fr, fphi = oracle.diffuse_fluid(want_cost, uni, 1e-9, 64)
    torch.cuda.synchronize()
    assert np.array_equal(o["bnd"].cpu().numpy(), db) and int(o["rounds"].item()) == dr
    assert int(o["phi"].item()) == dphi and np.array_equal(o["fluid_x"].cpu().numpy(), fx)

    bound = torch.tensor([int(oB * 1.5)], dtype=torch.int64, device=dev)
    floor = torch.tensor([1], dtype=torch.int32, device=dev)
    r = D.repack_workers(ctx, b, cost, floor=floor, bound=bound)
    rst, rk, rb, rB = oracle.repack_bound(want_cost, n, int(oB * 1.5), 1)
    torch.cuda.synchronize()
    assert int(r["status"].item()) == rst and int(r["n_new"].item()) == rk
    assert np.array_equal(r["bnd"].cpu().numpy(), rb) and int(r["bottleneck"].item()) == rB

    # NEXT-1 "by Time": stamps -> time costs (D = 1) == oracle; the stamp kernel runs
    stamps = synth.time_stamps(np.linspace(1e5, 3e5, shape.L), 2)
    ds = torch.from_numpy(stamps.reshape(-1)).to(dev)
    tsegs = [D.SegmentSpec(ds[m * (shape.L + 1) + i:m * (shape.L + 1) + i + 2], L.SRC_TIME_NS, i)
             for m in range(2) for i in range(shape.L)]
    tplan = D.ProfilePlan(ctx, tsegs, 0, shape.L)
    tcost, _, tst = D.profile_layers(ctx, tplan, D.coef_tensor(shape.L, D=1, device=dev))
    slot = torch.zeros(1, dtype=torch.int64, device=dev)
    D.timestamp(ctx, slot[0])
    torch.cuda.synchronize()
    want_t = [sum(oracle.time_ns(stamps[m, i:i + 2])[1] for m in range(2)) for i in range(shape.L)]
    assert int(tst.item()) == 0 and np.array_equal(tcost.cpu().numpy(), want_t) and int(slot.item()) > 0

    # NEXT-2 global magnitude pruning (Alg. 1): masks == oracle
    g = np.random.default_rng(5)
    wf = g.normal(0, 1, 40000).astype(np.float32)
    wb = torch.from_numpy(g.normal(0, 2, 33333).astype(np.float32)).to(torch.bfloat16)
    shards = [torch.from_numpy(wf).to(dev), wb.to(dev)]
    masks = [torch.empty(x.numel(), dtype=torch.uint8, device=dev) for x in shards]
    pplan = D.PrunePlan(ctx, list(zip(shards, masks)))
    k = int(0.1 * (wf.size + wb.numel()))
    pinfo, pst2 = D.global_prune(ctx, pplan, k)
    torch.cuda.synchronize()
    vals = [wf.astype(np.float64), oracle.bf16_to_f64(wb.view(torch.int16).numpy().view(np.uint16))]
    ost2, om = oracle.global_prune(vals, k)
    assert int(pst2.item()) == ost2 == 0
    assert all(np.array_equal(m.cpu().numpy(), o_) for m, o_ in zip(masks, om)), "prune mask mismatch"
    pplan.close()

    # NEXT-3 migration-minimising stage -> rank map == oracle
    nb = np.arange(1, shape.L + 1, dtype=np.int64) * 1000
    rn, kept, mst = D.map_stages(ctx, shape.L, torch.from_numpy(uni).to(dev),
                                 torch.arange(n, dtype=torch.int32, device=dev), bnd,
                                 torch.from_numpy(nb).to(dev), n)
    torch.cuda.synchronize()
    ost3, orn, okept = oracle.map_stages(shape.L, uni, np.arange(n), ob, nb, n)
    assert int(mst.item()) == ost3 == 0 and np.array_equal(rn.cpu().numpy(), orn) and int(kept.item()) == okept
    print(f"smoke OK: nnz={want_nnz.sum()} B*={oB} b={[int(x) for x in ob]} diffusion rounds={dr} "
          f"repack n'={rk} prune k={k} stage map={[int(x) for x in orn]}")

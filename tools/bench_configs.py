"""Per-config device timings of the hot path on one B200 (BASELINE configs 1, 3,
4, 5; config 2 is bench.py's headline).  Each config's device work is captured
once in a CUDA graph and replayed; CUDA events around each replay (L2 flushed
between replays outside the events, as in bench.py).  Results are checked
against the oracle on the same seeded inputs before timing.  Prints one JSON
object per config and writes gpurun_out/bench_configs.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

DEV = "cuda:0"
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = None


def timed(fn, reps=20):
    """Device ms per replay of fn captured in a CUDA graph (L2 flushed
    before each replay as in bench.py: a write and a read larger than L2)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), g


def dev(a, dt=None):
    a = np.ascontiguousarray(a if dt is None else np.asarray(a).astype(dt))
    return torch.from_numpy(a).to(DEV)


def config1(ctx):
    insts = synth.cfg1_instances(10_000)
    out = {}
    for with_mem in (True, False):
        sel = [x for x in insts if (x["mem"] is not None) == with_mem]
        b = D.Batch([24] * len(sel), [4] * len(sel), device=DEV)
        cost = dev(np.concatenate([x["cost"] for x in sel]), np.int64)
        mem = dev(np.concatenate([x["mem"] for x in sel]), np.int64) if with_mem else None
        cap = dev([x["cap"] for x in sel], np.int64) if with_mem else None
        bound = dev([x["bound"] for x in sel], np.int64)
        floor = dev(np.ones(len(sel)), np.int32)
        pout = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=DEV),
                    bottleneck=torch.empty(b.n_inst, dtype=torch.int64, device=DEV),
                    imbalance=torch.empty(b.n_inst, dtype=torch.float64, device=DEV),
                    status=torch.empty(b.n_inst, dtype=torch.int32, device=DEV))
        rout = {}

        def step():
            D.partition_stages(ctx, b, cost, mem=mem, cap=cap, **pout)
            D.repack_workers(ctx, b, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rout)

        ms, _ = timed(step)
        # parity + oracle time on the same instances (1 core)
        bn = b.split(pout["bnd"])
        t0 = time.perf_counter()
        for q, x in enumerate(sel):
            st, ob, oB, _ = oracle.partition(x["cost"], 4, mem=x["mem"], cap=x["cap"])
            rst, rk, rb, rB = oracle.repack_bound(x["cost"], 4, x["bound"], 1, mem=x["mem"], cap=x["cap"])
            assert np.array_equal(bn[q][:5], ob)
        t_or = time.perf_counter() - t0
        out["mem" if with_mem else "nomem"] = dict(instances=len(sel), device_ms=round(ms, 4),
                                                    instances_per_s=round(len(sel) / (ms * 1e-3)),
                                                    oracle_ms=round(t_or * 1e3, 1))
    return out


def config3(ctx):
    T, L, n = 512 * 2048, 32, 8
    e = synth.cfg3_exit_depth(T=T, L=L)
    fr = synth.cfg3_frozen(L, 8)
    de = dev(e)
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(de, LB.SRC_EXIT_U8, 0)], 0, L)
    coef = D.coef_tensor(L, A=1, device=DEV)
    frozen = dev(fr)
    cost = torch.empty(L, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    b = D.Batch([L], [n], device=DEV)
    bi = dev(np.arange(0, L + 1, L // n), np.int32)
    gf = torch.tensor([1.0], dtype=torch.float64, device=DEV)
    dout = {}

    def step():
        D.profile_layers(ctx, plan, coef, frozen=frozen, cost=cost, status=st)
        D.diffuse_balance(ctx, b, cost, bi, gamma_fluid=gf, max_rounds=256, out=dout)

    ms, _ = timed(step)
    tok = oracle.exit_survivors(e, 0, L)
    want = np.array([oracle.layer_cost(frozen=bool(fr[i]), tok=int(tok[i]), A=1)[1] for i in range(L)])
    assert np.array_equal(cost.cpu().numpy(), want)
    dst, db, dr, _, _ = oracle.diffuse(want, np.arange(0, L + 1, L // n), 0, 256)
    assert np.array_equal(dout["bnd"].cpu().numpy(), db)

    def prof_only():
        D.profile_layers(ctx, plan, coef, frozen=frozen, cost=cost, status=st)

    pms, _ = timed(prof_only)
    return dict(tokens=T, profile_bytes=int(plan.bytes), step_device_ms=round(ms, 4),
                profile_device_ms=round(pms, 4), diffusion_rounds=int(dout["rounds"].item()),
                fluid_rounds=int(dout["fluid_rounds"].item()))


def config4(ctx, alpha):
    T, L, E, k, n = 64 * 2048, 32, 8, 2, 8
    segs, keep, hists = [], [], []
    for i in range(L):
        idx = synth.cfg4_routing(i, T=T, E=E, k=k, alpha=alpha)
        hists.append(oracle.expert_hist(idx, E)[1])
        d = dev(idx.reshape(-1))
        keep.append(d)
        segs.append(D.SegmentSpec(d, LB.SRC_EXPERT_I64, i, n_experts=E, top_k=k))
    plan = D.ProfilePlan(ctx, segs, 0, L)
    coef = D.coef_tensor(L, A=T, C_=4, ep=8, device=DEV)
    cost = torch.empty(L, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    b = D.Batch([L], [n], device=DEV)
    pout = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=DEV),
                bottleneck=torch.empty(1, dtype=torch.int64, device=DEV),
                imbalance=torch.empty(1, dtype=torch.float64, device=DEV),
                status=torch.empty(1, dtype=torch.int32, device=DEV))

    def step():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)
        D.partition_stages(ctx, b, cost, **pout)

    ms, _ = timed(step)
    want = np.array([oracle.layer_cost(cnt=hists[i], A=T, C_=4, ep=8)[1] for i in range(L)])
    assert np.array_equal(cost.cpu().numpy(), want)

    def prof_only():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)

    pms, _ = timed(prof_only)
    return dict(alpha=alpha, profile_bytes=int(plan.bytes), step_device_ms=round(ms, 4),
                profile_device_ms=round(pms, 4),
                profile_GBps=round(plan.bytes / (pms * 1e-3) / 1e9, 1),
                imbalance=round(float(pout["imbalance"].item()), 4))


def _oracle_cfg5_chunk(idx):
    """Oracle work of config-5 instances idx (token counts, partition,
    BOUND repack) -- run in worker processes for the all-cores timing."""
    import oracle as o
    import synth as sy
    for q in idx:
        x = sy.cfg5_instance(q)
        c = np.array([o.count_bits(x.masks[l], 4096) for l in range(x.L)])
        o.partition(c, x.n, mem=x.mem, cap=x.cap)
        o.repack_bound(c, x.n, x.bound, 1, mem=x.mem, cap=x.cap)
    return len(idx)


def host_info():
    import platform
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return dict(cpu_count=os.cpu_count(), affinity=len(os.sched_getaffinity(0)), cpu_model=model or platform.processor())


def config5(ctx, n_inst=4096):
    insts = [synth.cfg5_instance(i) for i in range(n_inst)]
    masks = np.concatenate([x.masks.reshape(-1) for x in insts])
    dm = dev(masks.view(np.int32))
    segs, layer, off = [], 0, 0
    for x in insts:
        for l in range(x.L):
            segs.append(D.SegmentSpec(dm[off:off + 128], LB.SRC_TOKMASK_BITS, layer, n_elem=4096))
            off += 128
            layer += 1
    plan = D.ProfilePlan(ctx, segs, 0, layer)
    coef = D.coef_tensor(layer, A=1, device=DEV)
    cost = torch.empty(layer, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    b = D.Batch([x.L for x in insts], [x.n for x in insts], device=DEV)
    mem = dev(np.concatenate([x.mem for x in insts]), np.int64)
    cap = dev([x.cap for x in insts], np.int64)
    bound = dev([x.bound for x in insts], np.int64)
    floor = dev(np.ones(n_inst), np.int32)
    pout = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=DEV),
                bottleneck=torch.empty(n_inst, dtype=torch.int64, device=DEV),
                imbalance=torch.empty(n_inst, dtype=torch.float64, device=DEV),
                status=torch.empty(n_inst, dtype=torch.int32, device=DEV))
    rout = {}

    def step():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)
        D.partition_stages(ctx, b, cost, mem=mem, cap=cap, **pout)
        D.repack_workers(ctx, b, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rout)

    ms, _ = timed(step, reps=10)

    def prof_only():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)

    pms, _ = timed(prof_only, reps=10)
    # parity on a sample of instances
    ch = cost.cpu().numpy()
    bn, kn = b.split(pout["bnd"]), rout["n_new"].cpu().numpy()
    for q in range(0, n_inst, 64):
        x = insts[q]
        c = ch[b.layer_off_h[q]:b.layer_off_h[q + 1]]
        assert np.array_equal(c, [oracle.count_bits(x.masks[l], 4096) for l in range(x.L)])
        ost, ob, oB, _ = oracle.partition(c, x.n, mem=x.mem, cap=x.cap)
        assert np.array_equal(bn[q][:x.n + 1], ob)
        assert kn[q] == oracle.repack_bound(c, x.n, x.bound, 1, mem=x.mem, cap=x.cap)[1]
    # the oracle on config 5: one core (a 256-instance sample, scaled) and all
    # host cores (a process pool over all 4096 instances), SURVEY 8(d)
    import multiprocessing as mp
    t0 = time.perf_counter()
    _oracle_cfg5_chunk(range(256))
    one_core_ms = (time.perf_counter() - t0) * 1e3 * n_inst / 256
    ncores = len(os.sched_getaffinity(0))
    chunks = [list(range(i, n_inst, ncores * 4)) for i in range(ncores * 4)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(ncores) as pool:
        assert sum(pool.map(_oracle_cfg5_chunk, chunks)) == n_inst
    all_cores_ms = (time.perf_counter() - t0) * 1e3
    return dict(instances=n_inst, layers=layer, profile_bytes=int(plan.bytes), step_device_ms=round(ms, 4),
                oracle_ms_1core_est=round(one_core_ms, 1), oracle_ms_all_cores=round(all_cores_ms, 1),
                oracle_cores=ncores,
                instances_per_s=round(n_inst / (ms * 1e-3)), profile_device_ms=round(pms, 4),
                profile_GBps=round(plan.bytes / (pms * 1e-3) / 1e9, 1),
                mean_workers_after_repack=round(float(kn.mean()), 3),
                mean_workers_before=round(float(np.mean([x.n for x in insts])), 3))


def config_bytime(ctx):
    """NEXT-1 "by Time": config 2's 48 layers / 8 stages with per-layer
    execution times from the profiling iteration (4 micro-batches of
    boundary stamps, "four micro-batches per GPU"; base time of a
    layer proportional to its kept parameters), D = 1: profile + partition."""
    shape = synth.GPTShape()
    L, n, M = shape.L, 8, 4
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    sizes = np.array([3, 1, 4, 4], np.float64) * shape.h * shape.h  # QKV, proj, fc1, fc2
    kept = p @ sizes  # expected kept params per layer (p: keep probability per tensor)
    s = synth.time_stamps(kept * 0.05, M)
    ds = dev(s.reshape(-1))
    segs = [D.SegmentSpec(ds[m * (L + 1) + i:m * (L + 1) + i + 2], LB.SRC_TIME_NS, i) for m in range(M) for i in range(L)]
    plan = D.ProfilePlan(ctx, segs, 0, L)
    coef = D.coef_tensor(L, D=1, device=DEV)
    cost = torch.empty(L, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    b = D.Batch([L], [n], device=DEV)
    out = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=DEV),
               bottleneck=torch.empty(1, dtype=torch.int64, device=DEV),
               imbalance=torch.empty(1, dtype=torch.float64, device=DEV),
               status=torch.empty(1, dtype=torch.int32, device=DEV))

    def step():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)
        D.partition_stages(ctx, b, cost, **out)

    ms, _ = timed(step)
    want = np.array([sum(oracle.time_ns(s[m, i:i + 2])[1] for m in range(M)) for i in range(L)])
    assert np.array_equal(cost.cpu().numpy(), want)
    ost, ob, oB, _ = oracle.partition(want, n)
    assert np.array_equal(out["bnd"].cpu().numpy()[:n + 1], ob)
    return dict(layers=L, microbatches=M, segments=len(segs), step_device_ms=round(ms, 4),
                b_new=[int(x) for x in ob], imbalance=round(float(out["imbalance"].item()), 4))


def map_stages_cfg(ctx):
    """NEXT-3 stage -> rank map latency: config 2's 48 layers / CSR payloads,
    old split 8 stages on 8 ranks, new split = the partition of the costs
    (G = 8), and a 16-rank / 16-stage worst case (2^16 DP states)."""
    shape = synth.GPTShape()
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    pay = synth.cfg2_payload_bytes(shape, p).astype(np.int64)
    cost = np.load(os.path.join(os.path.dirname(__file__), "cfg2_cost.npy")).astype(np.int64)
    out = {}
    for G, n in ((8, 8), (16, 16)):
        bo = np.array([round(s * shape.L / n) for s in range(n + 1)], np.int32)
        ro = np.arange(n, dtype=np.int32) % G
        st, bn, _, _ = oracle.partition(cost, n)
        bn = np.asarray(bn, np.int32)
        args = (shape.L, dev(bo), dev(ro), dev(bn), dev(pay), G)
        res = {}

        def step():
            res["r"] = D.map_stages(ctx, *args)

        ms, _ = timed(step)
        rn, kept, mst = res["r"]
        ost, orn, okept = oracle.map_stages(shape.L, bo, ro, bn, pay, G)
        assert int(mst.item()) == ost == 0 and np.array_equal(rn.cpu().numpy(), orn)
        out[f"G{G}_n{n}"] = dict(device_ms=round(ms, 4), kept_fraction=round(okept / float(pay.sum()), 4),
                                 ranks=[int(x) for x in orn])
    return out


def sparse_attention(ctx):
    """NEXT-4: dynamic sparse flash attention, 32 layers / 8
    stages, hash-based causal block masks (T = 2048, 64-token blocks, 16
    heads, 2 micro-batches) as bit-mask sources: profile + partition."""
    Lyr, n, per_block = 32, 8, 64 * 64 * 64 * 2
    nbits = 2 * 16 * 32 * 32
    ws = [synth.sparse_attention_blocks(l) for l in range(Lyr)]
    ts = [dev(w.view(np.int32)) for w in ws]
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(t, LB.SRC_MASK_BITS, l, n_elem=nbits) for l, t in enumerate(ts)], 0, Lyr)
    coef = D.coef_tensor(Lyr, B=per_block, device=DEV)
    cost = torch.empty(Lyr, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    b = D.Batch([Lyr], [n], device=DEV)
    out = dict(bnd=torch.empty(b.total_bnd, dtype=torch.int32, device=DEV),
               bottleneck=torch.empty(1, dtype=torch.int64, device=DEV),
               imbalance=torch.empty(1, dtype=torch.float64, device=DEV),
               status=torch.empty(1, dtype=torch.int32, device=DEV))

    def step():
        D.profile_layers(ctx, plan, coef, cost=cost, status=st)
        D.partition_stages(ctx, b, cost, **out)

    ms, _ = timed(step)
    want = np.array([oracle.layer_cost(nnz=oracle.count_bits(w, nbits), B=per_block)[1] for w in ws])
    assert np.array_equal(cost.cpu().numpy(), want)
    ost, ob, oB, _ = oracle.partition(want, n)
    assert np.array_equal(out["bnd"].cpu().numpy()[:n + 1], ob)
    x_old = np.add.reduceat(want, np.arange(0, Lyr, Lyr // n))
    return dict(layers=Lyr, step_device_ms=round(ms, 4), b_new=[int(x) for x in ob],
                imbalance_uniform=round(float(oracle.imbalance(x_old)), 4),
                imbalance_new=round(float(out["imbalance"].item()), 4))


def main():
    global flush
    torch.cuda.set_device(0)
    flush = bench.L2Flush(DEV)
    ctx = D.Context(0)
    res = {"host": host_info()}
    for name, fn in [("config1", lambda: config1(ctx)), ("config3", lambda: config3(ctx)),
                     ("config4_auxloss", lambda: config4(ctx, 4.0)), ("config4_sbase", lambda: config4(ctx, 64.0)),
                     ("config5", lambda: config5(ctx)), ("bytime_cfg2", lambda: config_bytime(ctx)),
                     ("map_stages", lambda: map_stages_cfg(ctx)),
                     ("sparse_attention", lambda: sparse_attention(ctx))]:
        res[name] = fn()
        print(name, json.dumps(res[name]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "bench_configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element on the same seeded inputs.  Integer results bit-exact; fluid
diffusion loads bit-equal (declared tolerance 1e-6 relative, reading Q20)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2505_14864_b200 import dynmo
    return dynmo


@pytest.fixture(scope="module")
def L():
    from paper_2505_14864_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def ctx(D):
    torch.cuda.set_device(0)
    return D.Context(0)


DEV = "cuda:0"


def _dev(a, dtype=None):
    a = np.ascontiguousarray(a)
    if dtype is not None:
        a = a.astype(dtype)
    return torch.from_numpy(a).to(DEV)


# ------------------------------------------------------------ a1: pruning masks
def _mixed_segments(D, L, shape, S, milestone, offset_views=True):
    """Masks of every layer in u8 / bits / bf16 / f32, some as unaligned views."""
    p = synth.cfg2_keep_probs(shape, S, milestone)
    segs, keep = [], []
    want = np.zeros(shape.L, np.int64)
    g = np.random.default_rng(milestone)
    for layer in range(shape.L):
        for t, m in enumerate(synth.cfg2_layer_masks_u8(shape, layer, p[layer], milestone)):
            kind = (layer + t) % 4
            flat = m.reshape(-1)
            cut = int(g.integers(0, 7)) if offset_views else 0
            if kind == 0:
                base = _dev(flat)
                v = base[cut:]
                segs.append(D.SegmentSpec(v, L.SRC_MASK_U8, layer))
                want[layer] += oracle.count_nz_u8(flat[cut:])
            elif kind == 1:
                w = synth.pack_bits(flat)
                base = _dev(w.view(np.int32))
                nbits = flat.size - cut  # ragged bit count
                segs.append(D.SegmentSpec(base, L.SRC_MASK_BITS, layer, n_elem=nbits))
                want[layer] += oracle.count_bits(w, nbits)
            elif kind == 2:
                bf = synth.cfg2_bf16_weights(m, layer, t).reshape(-1)
                base = _dev(bf.view(np.int16))
                segs.append(D.SegmentSpec(base[cut:], L.SRC_NZ_BF16, layer))
                want[layer] += oracle.count_nz_bf16(bf[cut:])
            else:
                bf = synth.cfg2_bf16_weights(m, layer, t).reshape(-1)
                f = (bf.astype(np.uint32) << 16).view(np.float32)
                base = _dev(f)
                segs.append(D.SegmentSpec(base[cut:], L.SRC_NZ_F32, layer))
                want[layer] += oracle.count_nz_f32(f[cut:])
            keep.append(base)
    return segs, keep, want


@pytest.mark.parametrize("S,milestone", [(0.0, 0), (0.5203125, 1), (0.9, 4)])
def test_profile_masks_mixed_small(D, L, ctx, S, milestone):
    shape = synth.GPTShape(L=12, h=96)
    segs, keep, want = _mixed_segments(D, L, shape, S, milestone)
    plan = D.ProfilePlan(ctx, segs, 0, shape.L)
    coef = D.coef_tensor(shape.L, A=7, B=3, device=DEV)
    counters = torch.empty((shape.L, 5), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef, counters=counters)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    c = counters.cpu().numpy()
    assert np.array_equal(c[:, 0], want)
    want_cost = [oracle.layer_cost(nnz=int(v), A=7, B=3)[1] for v in want]
    assert np.array_equal(cost.cpu().numpy(), want_cost)
    # a second call (accumulators consumed and cleared) gives the same result
    cost2, _, st2 = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert np.array_equal(cost2.cpu().numpy(), want_cost) and int(st2.item()) == 0


def test_profile_tiny_and_empty_segments(D, L, ctx):
    """Edge cases: empty segments, 1-element segments, bits with n_elem < 8,
    a layer without any source (nnz = 0), a single-byte mask."""
    segs, keep, want = [], [], np.zeros(5, np.int64)
    t = _dev(np.array([1, 0, 3], np.uint8))
    segs.append(D.SegmentSpec(t[:0], L.SRC_MASK_U8, 0))
    segs.append(D.SegmentSpec(t[2:], L.SRC_MASK_U8, 0)); want[0] += 1
    w = np.array([0b1011011], np.uint32)
    tw = _dev(w.view(np.int32))
    segs.append(D.SegmentSpec(tw, L.SRC_MASK_BITS, 1, n_elem=5)); want[1] += oracle.count_bits(w, 5)
    segs.append(D.SegmentSpec(tw, L.SRC_MASK_BITS, 2, n_elem=1)); want[2] += oracle.count_bits(w, 1)
    h = np.array([0x8000, 0x0000, 0x7F80, 0x0001, 0xFFC0], np.uint16)  # -0, +0, inf, denorm, nan
    th = _dev(h.view(np.int16))
    segs.append(D.SegmentSpec(th, L.SRC_NZ_BF16, 3)); want[3] += oracle.count_nz_bf16(h)
    keep += [t, tw, th]
    plan = D.ProfilePlan(ctx, segs, 0, 5)
    coef = D.coef_tensor(5, A=0, B=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert np.array_equal(cost.cpu().numpy(), want)


def test_profile_config2_full_size(D, L, ctx):
    """BASELINE config 2 at full size (48 layers x 12 h^2, u8 masks at S=0.9),
    in the launch configuration bench.py times; every layer vs the oracle."""
    shape = synth.GPTShape()
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    segs, keep, want = [], [], np.zeros(shape.L, np.int64)
    for layer in range(shape.L):
        for m in synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4):
            d = _dev(m.reshape(-1))
            segs.append(D.SegmentSpec(d, L.SRC_MASK_U8, layer))
            keep.append(d)
            want[layer] += oracle.count_nz_u8(m)
    plan = D.ProfilePlan(ctx, segs, 0, shape.L)
    assert plan.bytes == shape.L * shape.params_per_layer
    coef = D.coef_tensor(shape.L, A=0, B=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert np.array_equal(cost.cpu().numpy(), want)
    # partition of the full-size cost vector at 8 stages
    b = D.Batch([shape.L], [8], device=DEV)
    bnd, bott, imb, pst = D.partition_stages(ctx, b, cost)
    ost, ob, oB, oimb = oracle.partition(want, 8)
    torch.cuda.synchronize()
    assert int(pst.item()) == ost and np.array_equal(bnd.cpu().numpy(), ob)
    assert int(bott.item()) == oB and float(imb.item()) == oimb


# --------------------------------------------------- a2 + a4: exit / MoD / frozen
@pytest.mark.parametrize("F", [0, 4, 8, 12])
def test_profile_exit_tokmask_frozen(D, L, ctx, F):
    """Config 3 (T = 512 x 2048): exit depths (EXIT_U8) on layers 0..15 and
    per-layer token bitmasks on layers 16..31; frozen prefix F; c = (1-f) tok."""
    T, Lyr = 512 * 2048, 32
    e = synth.cfg3_exit_depth(T=T, L=Lyr)
    frozen = synth.cfg3_frozen(Lyr, F)
    tok_exit = oracle.exit_survivors(e, 0, Lyr)
    segs = [D.SegmentSpec(_dev(e), L.SRC_EXIT_U8, 0)]
    keep = [segs[0].tensor]
    # plan A: exit source for all layers
    planA = D.ProfilePlan(ctx, segs, 0, Lyr)
    coef = D.coef_tensor(Lyr, A=1, B=0, device=DEV)
    cnt = torch.empty((Lyr, 5), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, planA, coef, frozen=_dev(frozen), counters=cnt)
    torch.cuda.synchronize()
    want = [oracle.layer_cost(frozen=bool(frozen[i]), tok=int(tok_exit[i]), A=1)[1] for i in range(Lyr)]
    assert int(st.item()) == 0
    assert np.array_equal(cnt[:, 1].cpu().numpy(), tok_exit)
    assert np.array_equal(cost.cpu().numpy(), want)
    # plan B: token bitmasks alive_i[t] = e[t] > i (the MoD / alive-mask form)
    segsB, tok_bits = [], np.zeros(Lyr, np.int64)
    for i in range(Lyr):
        w = synth.pack_bits((e > i).astype(np.uint8))
        d = _dev(w.view(np.int32))
        keep.append(d)
        segsB.append(D.SegmentSpec(d, L.SRC_TOKMASK_BITS, i, n_elem=T))
        tok_bits[i] = oracle.count_bits(w, T)
    planB = D.ProfilePlan(ctx, segsB, 0, Lyr)
    costB, _, stB = D.profile_layers(ctx, planB, coef, frozen=_dev(frozen))
    torch.cuda.synchronize()
    assert np.array_equal(tok_bits, tok_exit)
    assert np.array_equal(costB.cpu().numpy(), want) and int(stB.item()) == 0


def test_profile_exit_local_slice(D, L, ctx):
    """An EXIT source on a rank owning layers 10..17 yields the same slice."""
    e = synth.cfg3_exit_depth(T=100_003, L=32)
    d = _dev(e[3:])  # unaligned view
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(d, L.SRC_EXIT_U8, 0)], 10, 8)
    coef = D.coef_tensor(8, A=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert np.array_equal(cost.cpu().numpy(), oracle.exit_survivors(e[3:], 10, 8))


# -------------------------------------------------------------- a3: MoE routing
@pytest.mark.parametrize("alpha,dtype,E,ep", [(4.0, np.int64, 8, 8), (64.0, np.int64, 8, 8),
                                              (4.0, np.int32, 8, 2), (4.0, np.int64, 100, 4),
                                              (4.0, np.int32, 256, 0)])
def test_profile_moe(D, L, ctx, alpha, dtype, E, ep):
    """Config 4: per-expert histograms of top-2 ids; c = A T + C moe_i."""
    T, Lyr, k = 64 * 2048 if E == 8 else 20_000, 6, 2
    segs, keep, hists = [], [], []
    for i in range(Lyr):
        idx = synth.cfg4_routing(i, T=T, E=E, k=k, alpha=alpha, dtype=dtype)
        st_o, h = oracle.expert_hist(idx, E)
        assert st_o == 0
        hists.append(h)
        flat = idx.reshape(-1)
        cut = i % 2  # odd layers: unaligned start
        if cut:
            h2 = oracle.expert_hist(flat[1:], E)[1]
            hists[-1] = h2
        d = _dev(flat)
        keep.append(d)
        segs.append(D.SegmentSpec(d[cut:], L.SRC_EXPERT_I64 if dtype == np.int64 else L.SRC_EXPERT_I32,
                                  i, n_experts=E, top_k=k))
    plan = D.ProfilePlan(ctx, segs, 0, Lyr)
    assert plan.max_experts == E
    coef = D.coef_tensor(Lyr, A=T, C_=4, ep=ep, device=DEV)
    hist = torch.empty((Lyr, E), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef, hist=hist)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert np.array_equal(hist.cpu().numpy(), np.stack(hists))
    want = [oracle.layer_cost(cnt=hists[i], A=T, C_=4, ep=ep)[1] for i in range(Lyr)]
    assert np.array_equal(cost.cpu().numpy(), want)


def test_profile_moe_invalid_id(D, L, ctx):
    idx = synth.cfg4_routing(0, T=5000, E=8, k=2)
    idx[77, 1] = 8
    d = _dev(idx.reshape(-1))
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(d, L.SRC_EXPERT_I64, 0, n_experts=8, top_k=2)], 0, 1)
    coef = D.coef_tensor(1, A=1, C_=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.expert_hist(idx, 8)[0] == oracle.E_INVALID


def test_profile_overflow_and_bad_coef(D, L, ctx):
    m = np.ones(1000, np.uint8)
    d = _dev(m)
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(d, L.SRC_MASK_U8, 0), D.SegmentSpec(d, L.SRC_MASK_U8, 1)], 0, 2)
    coef = D.coef_tensor(2, A=0, B=[2 ** 62, 5], device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_OVERFLOW
    assert list(cost.cpu().numpy()) == [-1, oracle.layer_cost(nnz=1000, B=5)[1]]
    coef = D.coef_tensor(2, A=[-1, 0], B=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_INVALID and int(cost[0].item()) == -1


# ---------------------------------------------------------------- a7 partition
def _run_partition(D, ctx, insts, with_mem):
    b = D.Batch([len(x["cost"]) for x in insts], [x["n"] for x in insts], device=DEV)
    cost = _dev(np.concatenate([x["cost"] for x in insts]), np.int64)
    mem = cap = None
    if with_mem:
        mem = _dev(np.concatenate([x["mem"] for x in insts]), np.int64)
        cap = _dev(np.array([x["cap"] for x in insts]), np.int64)
    bnd, bott, imb, st = D.partition_stages(ctx, b, cost, mem=mem, cap=cap)
    torch.cuda.synchronize()
    return b, b.split(bnd), bott.cpu().numpy(), imb.cpu().numpy(), st.cpu().numpy()


def _check_partition(insts, res, with_mem):
    b, bnds, bott, imb, st = res
    for q, x in enumerate(insts):
        ost, ob, oB, oimb = oracle.partition(x["cost"], x["n"], mem=x["mem"] if with_mem else None,
                                             cap=x["cap"] if with_mem else 0)
        assert st[q] == ost, (q, x)
        assert bott[q] == oB, (q, x)
        assert np.array_equal(bnds[q][:x["n"] + 1], ob), (q, x, bnds[q], ob)
        assert imb[q] == oimb, (q, imb[q], oimb)


def test_partition_config1(D, ctx):
    """Config 1: 10,000 instances of 24 layers on 4 stages (with and without
    the memory cap), batched one CTA per instance."""
    insts = synth.cfg1_instances(10_000)
    with_m = [x for x in insts if x["mem"] is not None]
    no_m = [dict(x, mem=None) for x in insts]
    _check_partition(with_m, _run_partition(D, ctx, with_m, True), True)
    _check_partition(no_m, _run_partition(D, ctx, no_m, False), False)


def _random_insts(seed, count, Lmax, nmax=8, big=False, zero_frac=0.2, with_mem=False):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        Ly = int(g.integers(1, Lmax + 1))
        n = int(g.integers(1, min(nmax, Ly) + 1))
        hi = 2 ** 55 // max(Ly, 1) if big else 1000
        cost = g.integers(0, hi, Ly)
        cost[g.random(Ly) < zero_frac] = 0
        x = dict(cost=cost, n=n, mem=None, cap=0)
        if with_mem:
            mem = g.integers(0, 100, Ly)
            x["mem"] = mem
            x["cap"] = int(max(1, mem.sum() // n * g.uniform(0.6, 2.0)))
        out.append(x)
    return out


@pytest.mark.parametrize("Lmax,with_mem,big", [(63, False, False), (127, True, False), (255, False, True),
                                               (1023, True, False), (1023, False, True)])
def test_partition_random_sizes(D, ctx, Lmax, with_mem, big):
    """Every kernel variant (L <= 63/127/255/1023), zeros, ties, large costs,
    infeasible memory caps, n = 1 and n = L."""
    insts = _random_insts(Lmax + with_mem, 300, Lmax, nmax=min(64, Lmax), big=big, with_mem=with_mem)
    insts.append(dict(cost=np.arange(Lmax), n=Lmax, mem=None, cap=0) if not with_mem else
                 dict(cost=np.arange(Lmax), n=Lmax, mem=np.ones(Lmax, np.int64), cap=1))
    insts.append(dict(cost=np.full(Lmax, 3), n=1, mem=None, cap=0) if not with_mem else
                 dict(cost=np.full(Lmax, 3), n=1, mem=np.ones(Lmax, np.int64), cap=Lmax))
    _check_partition(insts, _run_partition(D, ctx, insts, with_mem), with_mem)


@pytest.mark.parametrize("count", [48, 700])  # 8-warp latency mode / 1-warp throughput mode (> 592)
def test_partition_repack_threshold_sizes(D, ctx, count):
    """L on both sides of every jump-table width (31/32, 63/64, 127/128,
    255/256: Q = 1, 2, 4, 8 registers, then warp windows), with and without
    the memory cap: partition and BOUND repack vs the oracle."""
    g = np.random.default_rng(4242 + count)
    sizes = [31, 32, 63, 64, 127, 128, 255, 256]
    insts = []
    for i in range(count):
        Ly = sizes[i % len(sizes)]
        n = int(g.integers(1, min(16, Ly) + 1))
        cost = g.integers(0, 1000, Ly)
        cost[g.random(Ly) < 0.2] = 0
        mem = g.integers(0, 100, Ly)
        insts.append(dict(cost=cost, n=n, mem=mem, cap=int(max(1, mem.sum() // n * g.uniform(0.6, 2.0))),
                          bound=int(cost.sum() // n * g.uniform(0.8, 3.0)), floor=1))
    for with_mem in (False, True):
        _check_partition(insts, _run_partition(D, ctx, insts, with_mem), with_mem)
        b, bnds, kn, bott, st = _run_repack(D, ctx, insts, 0, with_mem)
        for q, x in enumerate(insts):
            ost, ok, ob, oB = oracle.repack_bound(x["cost"], x["n"], x["bound"], 1,
                                                  mem=x["mem"] if with_mem else None, cap=x["cap"] if with_mem else 0)
            assert (st[q], kn[q], bott[q]) == (ost, ok, oB), (q, with_mem)
            assert np.array_equal(bnds[q][:x["n"] + 1], ob), (q, with_mem)


@pytest.mark.parametrize("count", [60, 700])  # 8-warp latency mode / 1-warp batched mode (> 592)
def test_search_paths_32_64_bit_and_counts(D, ctx, count):
    """The round-2 search (one candidate per thread) switches on the data:
    32-bit prefix sums when the total cost C < 2^31 (64-bit otherwise), the
    broadcast scan or binary lifting per instance (long models / few stages
    vs short models / many stages), and the 16-bit memory reach table.
    Instances straddle C = 2^31 (totals just below and just above), span
    both count choices, and carry tight and loose memory caps; partition and
    BOUND repack vs the oracle."""
    g = np.random.default_rng(31_2025 + count)
    insts = []
    for i in range(count):
        kind = i % 4
        Ly = int(g.integers(200, 1000)) if kind == 0 else int(g.integers(2, 40))
        n = int(g.integers(1, 4)) if kind == 0 else int(g.integers(1, min(Ly, 32) + 1))
        # total near 2^31: scale random weights so that C = 2^31 +- a few
        target = (1 << 31) + int(g.integers(-3, 4)) if kind in (1, 2) else int(g.integers(1, 1 << 40))
        w = g.random(Ly) + 0.05
        cost = np.floor(w / w.sum() * target).astype(np.int64)
        cost[-1] += target - int(cost.sum())  # exact total
        mem = g.integers(1, 1 << 20, Ly)
        cap = int(max(mem.max(), mem.sum() // n * g.uniform(0.9, 1.6))) if kind != 3 else int(mem.max())
        insts.append(dict(cost=cost, n=n, mem=mem, cap=cap, bound=int(cost.sum() // n * g.uniform(1.0, 2.5)),
                          floor=1))
    for with_mem in (False, True):
        _check_partition(insts, _run_partition(D, ctx, insts, with_mem), with_mem)
        b, bnds, kn, bott, st = _run_repack(D, ctx, insts, 0, with_mem)
        for q, x in enumerate(insts):
            ost, ok, ob, oB = oracle.repack_bound(x["cost"], x["n"], x["bound"], 1,
                                                  mem=x["mem"] if with_mem else None, cap=x["cap"] if with_mem else 0)
            assert (st[q], kn[q], bott[q]) == (ost, ok, oB), (q, with_mem)
            assert np.array_equal(bnds[q][:x["n"] + 1], ob), (q, with_mem)


def test_partition_errors(D, ctx):
    """INVALID (n > L, n < 1, negative cost), OVERFLOW, INFEASIBLE."""
    insts = [dict(cost=np.array([1, 2]), n=3, mem=np.array([1, 1]), cap=5),
             dict(cost=np.array([1, 2]), n=0, mem=np.array([1, 1]), cap=5),
             dict(cost=np.array([1, -2, 3]), n=2, mem=np.array([1, 1, 1]), cap=5),
             dict(cost=np.array([2 ** 62, 2 ** 62]), n=1, mem=np.array([1, 1]), cap=5),
             dict(cost=np.array([2 ** 62, 2 ** 62 - 1]), n=1, mem=np.array([1, 1]), cap=5),
             dict(cost=np.array([1, 1, 1]), n=2, mem=np.array([3, 3, 3]), cap=5),
             dict(cost=np.array([1, 1, 1]), n=2, mem=np.array([3, 9, 3]), cap=5),
             dict(cost=np.array([1, 1, 1]), n=2, mem=np.array([3, -1, 3]), cap=5)]
    b = D.Batch([len(x["cost"]) for x in insts], [x["n"] for x in insts], device=DEV,
                capacity=[max(x["n"], 1) + 2 for x in insts])
    cost = _dev(np.concatenate([x["cost"] for x in insts]), np.int64)
    mem = _dev(np.concatenate([x["mem"] for x in insts]), np.int64)
    cap = _dev(np.array([x["cap"] for x in insts]), np.int64)
    bnd, bott, imb, st = D.partition_stages(ctx, b, cost, mem=mem, cap=cap)
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    for q, x in enumerate(insts):
        ost, ob, oB, oimb = oracle.partition(x["cost"], x["n"], mem=x["mem"], cap=x["cap"])
        assert st[q] == ost, (q, st[q], ost)
        assert bott[q].item() == oB


# ------------------------------------------------------------------ a9 repack
def _run_repack(D, ctx, insts, mode, with_mem):
    b = D.Batch([len(x["cost"]) for x in insts], [x["n"] for x in insts], device=DEV)
    cost = _dev(np.concatenate([x["cost"] for x in insts]), np.int64)
    mem = cap = None
    if with_mem:
        mem = _dev(np.concatenate([x["mem"] for x in insts]), np.int64)
        cap = _dev(np.array([x["cap"] for x in insts]), np.int64)
    floor = _dev(np.array([x["floor"] for x in insts]), np.int32)
    bound = _dev(np.array([x.get("bound", 0) for x in insts]), np.int64)
    bnd_in = None
    if mode == 1:
        flat = np.full(b.total_bnd, -7, np.int32)
        for q, x in enumerate(insts):
            flat[b.bnd_off_h[q]:b.bnd_off_h[q] + x["n"] + 1] = x["bnd_in"]
        bnd_in = _dev(flat)
    o = D.repack_workers(ctx, b, cost, floor=floor, bound=bound, mode=mode, mem=mem, cap=cap, bnd_in=bnd_in)
    torch.cuda.synchronize()
    return b, b.split(o["bnd"]), o["n_new"].cpu().numpy(), o["bottleneck"].cpu().numpy(), o["status"].cpu().numpy()


def test_repack_bound_config1(D, ctx):
    insts = synth.cfg1_instances(3000, seed_key=1)
    for with_mem in (True, False):
        sel = [x if with_mem else dict(x, mem=None) for x in insts if (x["mem"] is not None) == with_mem]
        b, bnds, kn, bott, st = _run_repack(D, ctx, sel, 0, with_mem)
        for q, x in enumerate(sel):
            ost, ok, ob, oB = oracle.repack_bound(x["cost"], 4, x["bound"], x["floor"],
                                                  mem=x["mem"], cap=x["cap"])
            assert (st[q], kn[q], bott[q]) == (ost, ok, oB), (q, x)
            assert np.array_equal(bnds[q][:5], ob)


def test_repack_bound_random(D, ctx):
    g = np.random.default_rng(77)
    insts = []
    for x in _random_insts(78, 400, 127, nmax=8, with_mem=True):
        Ly = len(x["cost"])
        x["floor"] = int(g.integers(1, x["n"] + 1))
        x["bound"] = int(x["cost"].sum() * g.uniform(0.05, 1.0))
        insts.append(x)
    b, bnds, kn, bott, st = _run_repack(D, ctx, insts, 0, True)
    for q, x in enumerate(insts):
        ost, ok, ob, oB = oracle.repack_bound(x["cost"], x["n"], x["bound"], x["floor"], mem=x["mem"], cap=x["cap"])
        assert (st[q], kn[q], bott[q]) == (ost, ok, oB), q
        assert np.array_equal(bnds[q][:x["n"] + 1], ob)


def test_repack_alg2(D, ctx):
    g = np.random.default_rng(88)
    insts = []
    for x in _random_insts(89, 500, 127, nmax=8, with_mem=True):
        Ly, n = len(x["cost"]), x["n"]
        inner = np.sort(g.choice(np.arange(1, Ly), n - 1, replace=False)) if n > 1 else []
        x["bnd_in"] = np.concatenate([[0], inner, [Ly]]).astype(np.int32)
        x["floor"] = int(g.integers(1, n + 1))
        x["cap"] = int(g.integers(0, 3000))
        insts.append(x)
    b, bnds, kn, bott, st = _run_repack(D, ctx, insts, 1, True)
    for q, x in enumerate(insts):
        ost, ok, ob, oB = oracle.repack_alg2(x["cost"], x["bnd_in"], x["floor"], mem=x["mem"], cap=x["cap"])
        assert (st[q], kn[q], bott[q]) == (ost, ok, oB), q
        assert np.array_equal(bnds[q][:x["n"] + 1], ob)


# --------------------------------------------------------------- a8 diffusion
def _run_diffuse(D, ctx, insts, with_mem, max_rounds):
    b = D.Batch([len(x["cost"]) for x in insts], [x["n"] for x in insts], device=DEV)
    cost = _dev(np.concatenate([x["cost"] for x in insts]), np.int64)
    mem = cap = None
    if with_mem:
        mem = _dev(np.concatenate([x["mem"] for x in insts]), np.int64)
        cap = _dev(np.array([x["cap"] for x in insts]), np.int64)
    flat = np.zeros(b.total_bnd, np.int32)
    for q, x in enumerate(insts):
        flat[b.bnd_off_h[q]:b.bnd_off_h[q + 1]] = x["bnd_in"]
    gamma = _dev(np.array([x.get("gamma", 0) for x in insts]), np.int64)
    gf = _dev(np.array([x.get("gamma_f", 0.0) for x in insts]), np.float64)
    o = D.diffuse_balance(ctx, b, cost, _dev(flat), mem=mem, cap=cap, gamma=gamma, gamma_fluid=gf,
                          max_rounds=max_rounds)
    torch.cuda.synchronize()
    return b, {k: v.cpu().numpy() for k, v in o.items()}


def _check_diffuse(D, ctx, insts, with_mem, max_rounds):
    b, o = _run_diffuse(D, ctx, insts, with_mem, max_rounds)
    for q, x in enumerate(insts):
        n = x["n"]
        dst, db, dr, dphi, dphi0 = oracle.diffuse(x["cost"], x["bnd_in"], x.get("gamma", 0), max_rounds,
                                                  mem=x["mem"] if with_mem else None, cap=x["cap"])
        fst, fx, fr, fphi = oracle.diffuse_fluid(x["cost"], x["bnd_in"], x.get("gamma_f", 0.0), max_rounds)
        lo = b.bnd_off_h[q]
        assert o["status"][q] == dst, (q, o["status"][q], dst)
        assert o["fluid_status"][q] == fst, (q, o["fluid_status"][q], fst)
        assert np.array_equal(o["bnd"][lo:lo + n + 1], db), q
        assert (o["rounds"][q], o["phi"][q], o["phi0"][q]) == (dr, dphi, dphi0), q
        gx = o["fluid_x"][lo - q:lo - q + n]
        assert np.array_equal(gx, fx), (q, gx, fx)  # bit-equal (<= 1e-6 rel is the declared bar)
        assert o["fluid_rounds"][q] == fr and o["fluid_phi"][q] == fphi


def test_diffuse_config3(D, ctx):
    """Config 3: exit + freezing costs on 32 layers, 8 stages, uniform start,
    gamma = 0, max_rounds = 256, gamma_f = 1e-9 phi(0)."""
    T, Lyr = 512 * 2048, 32
    e = synth.cfg3_exit_depth(T=T, L=Lyr)
    tok = oracle.exit_survivors(e, 0, Lyr)
    insts = []
    for F in (0, 4, 8, 12):
        f = synth.cfg3_frozen(Lyr, F)
        cost = np.array([oracle.layer_cost(frozen=bool(f[i]), tok=int(tok[i]), A=1)[1] for i in range(Lyr)])
        bnd = np.arange(0, 33, 4).astype(np.int32)
        x0 = oracle.stage_loads(cost, bnd).astype(float)
        insts.append(dict(cost=cost, n=8, bnd_in=bnd, mem=None, cap=0, gamma=0,
                          gamma_f=1e-9 * oracle.phi_f64(x0)))
    _check_diffuse(D, ctx, insts, False, 256)


@pytest.mark.parametrize("with_mem,Lmax,maxr", [(False, 63, 256), (True, 127, 256), (True, 255, 3),
                                                (False, 1023, 64)])
def test_diffuse_random(D, ctx, with_mem, Lmax, maxr):
    g = np.random.default_rng(Lmax)
    insts = []
    for x in _random_insts(Lmax + 1000, 200, Lmax, nmax=16, with_mem=with_mem):
        Ly, n = len(x["cost"]), x["n"]
        inner = np.sort(g.choice(np.arange(1, Ly), n - 1, replace=False)) if n > 1 else []
        x["bnd_in"] = np.concatenate([[0], inner, [Ly]]).astype(np.int32)
        x["gamma"] = int(g.integers(0, 50)) if g.random() < 0.3 else 0
        x0 = oracle.stage_loads(x["cost"], x["bnd_in"]).astype(float)
        x["gamma_f"] = float(g.choice([0.0, 1e-9 * oracle.phi_f64(x0), 1e-3 * oracle.phi_f64(x0)]))
        if not with_mem:
            x["mem"], x["cap"] = None, 0
        insts.append(x)
    _check_diffuse(D, ctx, insts, with_mem, maxr)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_diffuse_fluid_long(D, ctx, seed):
    """The speculative fluid rounds of k_diffuse (n <= 32: chunks advanced
    with the matching of two rounds earlier, verified row by row, rolled back
    at the first mispredicted row): long fluid runs (max_rounds 4096, tiny
    gamma_f) from skewed, random and near-periodic starts, n = 2 .. 32, fluid
    loads bit-equal to the oracle's per-round process."""
    g = np.random.default_rng(1000 + seed)
    insts = []
    for q in range(24):
        n = int(g.integers(2, 33))
        Ly = int(g.integers(n, 4 * n + 40))
        kind = q % 3
        cost = g.integers(0, 1000, Ly)
        if kind == 1:
            cost = (g.pareto(1.2, Ly) * 100).astype(np.int64)  # skewed: many rollbacks
        elif kind == 2:
            cost = np.full(Ly, 7, np.int64)
            cost[int(g.integers(0, Ly))] = 5000  # one hot layer: period-2 after the start
        inner = np.sort(g.choice(np.arange(1, Ly), n - 1, replace=False))
        bnd = np.concatenate([[0], inner, [Ly]]).astype(np.int32)
        x0 = oracle.stage_loads(cost, bnd).astype(float)
        x = dict(cost=cost, n=n, bnd_in=bnd, gamma=0, mem=None, cap=0,
                 gamma_f=float(g.choice([0.0, 1e-12, 1e-6])) * oracle.phi_f64(x0))
        insts.append(x)
    _check_diffuse(D, ctx, insts, False, 4096)


def test_diffuse_invalid(D, ctx):
    insts = [dict(cost=np.array([1, 2, 3]), n=2, bnd_in=np.array([0, 3, 3], np.int32), mem=None, cap=0),
             dict(cost=np.array([1, -2, 3]), n=2, bnd_in=np.array([0, 1, 3], np.int32), mem=None, cap=0),
             dict(cost=np.array([1, 2, 3]), n=2, bnd_in=np.array([0, 1, 3], np.int32), mem=None, cap=0,
                  gamma=-1),
             dict(cost=np.array([1, 2, 3]), n=2, bnd_in=np.array([0, 1, 3], np.int32), mem=None, cap=0,
                  gamma_f=-1.0)]
    _check_diffuse(D, ctx, insts, False, 16)


# -------------------------------------------------------- config 5 batched sweep
def test_config5_sweep(D, L, ctx):
    """Config 5 (sample of 256 instances): MoD token bitmasks -> tok costs ->
    partition at n -> BOUND repack to the fewest workers, all batched."""
    insts = [synth.cfg5_instance(i) for i in range(256)]
    segs, keep, layer = [], [], 0
    tok_o = []
    for x in insts:
        d = _dev(x.masks.view(np.int32))
        keep.append(d)
        for l in range(x.L):
            segs.append(D.SegmentSpec(d[l], L.SRC_TOKMASK_BITS, layer, n_elem=4096))
            tok_o.append(oracle.count_bits(x.masks[l], 4096))
            layer += 1
    plan = D.ProfilePlan(ctx, segs, 0, layer)
    coef = D.coef_tensor(layer, A=1, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    cost_h = cost.cpu().numpy()
    assert np.array_equal(cost_h, tok_o)
    b = D.Batch([x.L for x in insts], [x.n for x in insts], device=DEV)
    mem = _dev(np.concatenate([x.mem for x in insts]), np.int64)
    cap = _dev(np.array([x.cap for x in insts]), np.int64)
    bnd, bott, imb, pst = D.partition_stages(ctx, b, cost, mem=mem, cap=cap)
    floor = _dev(np.ones(len(insts)), np.int32)
    bound = _dev(np.array([x.bound for x in insts]), np.int64)
    r = D.repack_workers(ctx, b, cost, floor=floor, bound=bound, mem=mem, cap=cap)
    torch.cuda.synchronize()
    bnds, rb = b.split(bnd), b.split(r["bnd"])
    kn = r["n_new"].cpu().numpy()
    shrunk = 0
    for q, x in enumerate(insts):
        c = cost_h[b.layer_off_h[q]:b.layer_off_h[q + 1]]
        ost, ob, oB, _ = oracle.partition(c, x.n, mem=x.mem, cap=x.cap)
        assert pst[q].item() == ost and np.array_equal(bnds[q][:x.n + 1], ob) and bott[q].item() == oB
        rst, rk, rbb, rB = oracle.repack_bound(c, x.n, x.bound, 1, mem=x.mem, cap=x.cap)
        assert r["status"][q].item() == rst and kn[q] == rk and np.array_equal(rb[q][:x.n + 1], rbb)
        shrunk += rk < x.n
    assert shrunk > 0  # MoD leaves room to release workers


def test_profile_mixed_sources_one_plan(D, L, ctx):
    """Every source kind in ONE plan (count ops + exit histogram + experts on
    the register (E=8), smem-column (E=40) and smem-atomic (E=300) paths),
    unaligned views: per-layer counters and histograms vs the oracle."""
    g = np.random.default_rng(3)
    segs, keep = [], []
    nnz, tok, hists = np.zeros(8, np.int64), np.zeros(8, np.int64), {}

    def add(t, kind, layer, **kw):
        keep.append(t)
        segs.append(D.SegmentSpec(t, kind, layer, **kw))
    u8 = (g.random(70001) < 0.3).astype(np.uint8)
    add(_dev(u8)[3:], L.SRC_MASK_U8, 0); nnz[0] += oracle.count_nz_u8(u8[3:])
    w = g.integers(0, 2 ** 32, 999, dtype=np.uint64).astype(np.uint32)
    add(_dev(w.view(np.int32)), L.SRC_MASK_BITS, 1, n_elem=999 * 32 - 5); nnz[1] += oracle.count_bits(w, 999 * 32 - 5)
    add(_dev(w.view(np.int32)), L.SRC_TOKMASK_BITS, 2, n_elem=600); tok[2] += oracle.count_bits(w, 600)
    h16 = g.integers(0, 2 ** 16, 5003, dtype=np.uint64).astype(np.uint16)
    add(_dev(h16.view(np.int16))[1:], L.SRC_NZ_BF16, 3); nnz[3] += oracle.count_nz_bf16(h16[1:])
    f32 = g.normal(size=3001).astype(np.float32)
    f32[g.random(3001) < 0.4] = 0.0
    add(_dev(f32)[2:], L.SRC_NZ_F32, 4); nnz[4] += oracle.count_nz_f32(f32[2:])
    e = synth.cfg3_exit_depth(T=30001, L=8)
    add(_dev(e)[1:], L.SRC_EXIT_U8, 0)
    tok += oracle.exit_survivors(e[1:], 0, 8)
    for j, (E, dt) in enumerate([(8, np.int64), (40, np.int32), (300, np.int64)]):
        idx = synth.cfg4_routing(j, T=3001, E=E, k=2, dtype=dt).reshape(-1)
        add(_dev(idx)[1:], L.SRC_EXPERT_I64 if dt == np.int64 else L.SRC_EXPERT_I32, 5 + j, n_experts=E, top_k=2)
        hists[5 + j] = oracle.expert_hist(idx[1:], E)[1]
    plan = D.ProfilePlan(ctx, segs, 0, 8)
    coef = D.coef_tensor(8, A=3, B=1, C_=2, ep=0, device=DEV)
    counters = torch.empty((8, 5), dtype=torch.int64, device=DEV)
    hist = torch.zeros((8, plan.max_experts), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, coef, counters=counters, hist=hist)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    c = counters.cpu().numpy()
    assert np.array_equal(c[:, 0], nnz) and np.array_equal(c[:, 1], tok)
    hh = hist.cpu().numpy()
    for layer, want in hists.items():
        assert np.array_equal(hh[layer, :len(want)], want), layer
    want_cost = [oracle.layer_cost(tok=int(tok[i]), nnz=int(nnz[i]), cnt=hists.get(i), A=3, B=1, C_=2, ep=0)[1]
                 for i in range(8)]
    assert np.array_equal(cost.cpu().numpy(), want_cost)


# ------------------------------------------------- NEXT-1: "by Time" source
def test_profile_time_source(D, L, ctx):
    """TIME_NS (P:L632/P:L720/P:L743, reading Q21): per layer and micro-batch
    the overlapping boundary segment {&s[m, i], 2} (8-byte aligned only),
    long contiguous pair arrays on two layers (several 1024-pair tiles, a
    ragged last one), and a u8 mask source on every layer: time_i and
    c_i = B nnz_i + D time_i vs the oracle; then by-Time costs (D = 1) and
    their partition vs the oracle's."""
    g = np.random.default_rng(61)
    Lyr, M = 24, 4
    s = synth.time_stamps(g.uniform(0.5, 2.0, Lyr) * 1e6, M)
    ds = _dev(s.reshape(-1))
    segs, want_t, keep = [], np.zeros(Lyr, np.int64), [ds]
    for m in range(M):
        for i in range(Lyr):
            off = m * (Lyr + 1) + i
            segs.append(D.SegmentSpec(ds[off:off + 2], L.SRC_TIME_NS, i))
            want_t[i] += oracle.time_ns(s[m, i:i + 2])[1]
    for i, npairs in ((3, 2500), (10, 1025)):
        b = g.integers(0, 2 ** 40, npairs)
        pr = np.stack([b, b + g.integers(0, 10 ** 6, npairs)], 1).astype(np.int64).reshape(-1)
        t = _dev(pr)
        keep.append(t)
        segs.append(D.SegmentSpec(t, L.SRC_TIME_NS, i))
        want_t[i] += oracle.time_ns(pr)[1]
    masks = [(g.random(5000 + 7 * i) < 0.4).astype(np.uint8) for i in range(Lyr)]
    nnz = np.array([oracle.count_nz_u8(m_) for m_ in masks])
    mt = [_dev(m_) for m_ in masks]
    segs += [D.SegmentSpec(t, L.SRC_MASK_U8, i) for i, t in enumerate(mt)]
    plan = D.ProfilePlan(ctx, segs, 0, Lyr)
    counters = torch.empty((Lyr, 5), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, D.coef_tensor(Lyr, B=3, D=1, device=DEV), counters=counters)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    c = counters.cpu().numpy()
    assert np.array_equal(c[:, 4], want_t) and np.array_equal(c[:, 0], nnz)
    want_cost = [oracle.layer_cost(nnz=int(nnz[i]), B=3, D=1, time=int(want_t[i]))[1] for i in range(Lyr)]
    assert np.array_equal(cost.cpu().numpy(), want_cost)
    costT, _, st = D.profile_layers(ctx, plan, D.coef_tensor(Lyr, D=1, device=DEV))
    b = D.Batch([Lyr], [4], device=DEV)
    bnd, bott, _, pst = D.partition_stages(ctx, b, costT)
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and int(pst.item()) == 0
    assert np.array_equal(costT.cpu().numpy(), want_t)
    ost, ob, oB, _ = oracle.partition(want_t, 4)
    assert np.array_equal(bnd.cpu().numpy()[:5], ob) and int(bott.item()) == oB


def test_profile_time_invalid(D, L, ctx):
    """A pair with end < begin is INVALID (device status), an odd stamp count
    is rejected at plan creation (host)."""
    pr = np.array([10, 20, 30, 25, 40, 41], np.int64)
    assert oracle.time_ns(pr)[0] == oracle.E_INVALID
    t = _dev(pr)
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(t, L.SRC_TIME_NS, 0)], 0, 1)
    cost, _, st = D.profile_layers(ctx, plan, D.coef_tensor(1, D=1, device=DEV))
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_INVALID
    with pytest.raises(D.DynmoError):
        D.ProfilePlan(ctx, [D.SegmentSpec(t[:3], L.SRC_TIME_NS, 0)], 0, 1)


def test_timestamp_kernel(D, ctx):
    """dynmo_timestamp: stamps taken when the preceding stream work is done
    (monotonic ns; durations proportional to the work between stamps) and
    re-taken at every CUDA-graph replay."""
    st = torch.zeros(3, dtype=torch.int64, device=DEV)
    torch.cuda._sleep(1000)  # load the sleep kernel (lazy loading would idle the stream)
    torch.cuda.synchronize()
    torch.cuda._sleep(50_000_000)  # keep the device busy while the host enqueues the rest
    D.timestamp(ctx, st[0])
    torch.cuda._sleep(2_000_000)
    D.timestamp(ctx, st[1])
    torch.cuda._sleep(8_000_000)
    D.timestamp(ctx, st[2])
    torch.cuda.synchronize()
    s = st.cpu().numpy()
    d1, d2 = int(s[1] - s[0]), int(s[2] - s[1])
    assert 0 < d1 < d2 and 2.5 < d2 / d1 < 6.0, (d1, d2)
    one = torch.zeros(1, dtype=torch.int64, device=DEV)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        D.timestamp(ctx, one[0])
    seen = []
    for _ in range(3):
        gr.replay()
        torch.cuda.synchronize()
        seen.append(int(one.item()))
    assert seen[0] > int(s[2]) and seen[0] < seen[1] < seen[2]


# --------------------------------------- NEXT-2: Alg. 1 global pruning
def _prune_shards(g, sizes, quant):
    """Mixed f32 / bf16 shards; `quant` > 0 quantises magnitudes (many ties)."""
    shards, vals = [], []
    for j, n in enumerate(sizes):
        x = g.normal(0.0, 1.0, n)
        if quant:
            x = np.round(x * quant) / quant
        if j % 2 == 0:
            w = x.astype(np.float32)
            shards.append(torch.from_numpy(w).to(DEV))
            vals.append(w.astype(np.float64))
        else:
            t = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
            bits = t.view(torch.int16).numpy().view(np.uint16)
            shards.append(t.to(DEV))
            vals.append(oracle.bf16_to_f64(bits))
    return shards, vals


@pytest.mark.parametrize("quant", [0, 4])
def test_global_prune_parity(D, ctx, quant):
    """Alg. 1: masks == the oracle's for k in {0, 1, N/10,
    N/2, N-1, N} and random k, mixed f32/bf16, ragged segments spanning
    several 32768-element tiles, heavy ties (quant=4) so that a partial tie
    share falls inside a tile."""
    g = np.random.default_rng(100 + quant)
    sizes = [70001, 7, 32768, 100000, 0, 33000, 32767]  # full 32768-element tiles and ragged ones
    shards, vals = _prune_shards(g, sizes, quant)
    masks = [torch.zeros(max(1, s.numel()), dtype=torch.uint8, device=DEV)[:s.numel()] for s in shards]
    plan = D.PrunePlan(ctx, list(zip(shards, masks)))
    N = sum(sizes)
    for k in [0, 1, N // 10, N // 2, N - 1, N] + [int(x) for x in g.integers(0, N + 1, 4)]:
        info, st = D.global_prune(ctx, plan, k)
        torch.cuda.synchronize()
        ost, omask = oracle.global_prune(vals, k)
        assert int(st.item()) == ost == 0, (k, int(st.item()))
        for m, om in zip(masks, omask):
            assert np.array_equal(m.cpu().numpy(), om), (k, quant)
        inf = info.cpu().numpy()
        assert inf[1] == N and inf[2] + inf[3] == k
    plan.close()


def test_global_prune_bf16_unaligned_masks_specials(D, ctx):
    """The packed bf16 mask path (two 15-bit magnitudes per word): all-bf16
    plan, masks at odd byte offsets (the unaligned store branch), +-inf
    (kept above every finite value, not NaN), +-0, subnormals and the
    largest finite value, and thresholds that fall on inf, on the largest
    finite value, inside the quantised bulk and on zero (a partial share of
    the ties in each case) -- masks == the oracle's."""
    g = np.random.default_rng(7)
    sizes = [3 * 32768 + 5, 65536, 32768, 40000]
    specials = np.array([0x7F80, 0xFF80, 0x0000, 0x8000, 0x0001, 0x8003, 0x7F7F, 0xFF7F], np.uint16)
    shards, vals = [], []
    for n in sizes:
        x = np.round(g.normal(0.0, 1.0, n) * 4) / 4
        bits = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        pos = g.choice(n, 64, replace=False)
        bits[pos] = specials[np.arange(64) % len(specials)]
        shards.append(torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(DEV))
        vals.append(oracle.bf16_to_f64(bits))
    buf = torch.zeros(sum(sizes) + 64, dtype=torch.uint8, device=DEV)
    masks, off = [], 1
    for n in sizes:
        masks.append(buf[off:off + n])
        off += n + 2  # odd offsets throughout
    plan = D.PrunePlan(ctx, list(zip(shards, masks)))
    N = sum(sizes)
    n_inf = 4 * 16  # 16 infs (+-) per shard, as many largest-finite values
    for k in [1, n_inf - 3, n_inf + 5, N // 3, N - 10, N]:
        info, st = D.global_prune(ctx, plan, k)
        torch.cuda.synchronize()
        ost, omask = oracle.global_prune(vals, k)
        assert int(st.item()) == ost == 0, (k, int(st.item()))
        for m, om in zip(masks, omask):
            assert np.array_equal(m.cpu().numpy(), om), k
    plan.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_global_prune_window_hit_and_miss(D, ctx, dtype):
    """The first digit's bin window comes from a sample of every 32nd tile.
    (a) Homogeneous weights (20 x 32768 + ragged): the window holds the k-th
    key (info[5] = 0).  (b) Adversarial: tiles 0 (the sample) and 16 hold
    N(0, 100) weights, the rest N(0, 0.01), so the estimate is far off; the
    full histogram and the second select run (info[5] = 1).  Masks == the
    oracle's in both, f32 plans continuing with passes 1 and 2."""
    T = 32768
    n = 20 * T + 1234
    g = np.random.default_rng(11)
    for adversarial, ks in [(False, [n // 10, n // 2]), (True, [n // 3, 2 * T + 1000])]:
        x = g.normal(0.0, 1.0, n)
        if adversarial:
            x *= 0.01
            for t in (0, 16):
                x[t * T:(t + 1) * T] = g.normal(0.0, 100.0, T)
        if dtype == "f32":
            w = x.astype(np.float32)
            shard, val = torch.from_numpy(w).to(DEV), w.astype(np.float64)
        else:
            t16 = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
            shard = t16.to(DEV)
            val = oracle.bf16_to_f64(t16.view(torch.int16).numpy().view(np.uint16))
        mask = torch.zeros(n, dtype=torch.uint8, device=DEV)
        plan = D.PrunePlan(ctx, [(shard, mask)])
        for k in ks:
            info, st = D.global_prune(ctx, plan, k)
            torch.cuda.synchronize()
            ost, omask = oracle.global_prune([val], k)
            assert int(st.item()) == ost == 0
            assert np.array_equal(mask.cpu().numpy(), omask[0]), (adversarial, k)
            assert (int(info[5].item()) & 1) == int(adversarial), (adversarial, k)
            if dtype == "bf16" and not adversarial and k == n // 10:
                # a window of ~10 bins and a partial tie share: the tie counts
                # come from the windowed pass (flag bit 1)
                assert int(info[5].item()) == 2
        plan.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_global_prune_wide_window_clamped(D, ctx, dtype):
    """Magnitudes log-uniform over 2^-120 .. 2^0 (≈ 15000 first-digit bins)
    and small k: the estimated window is wider than the 4096 bins of the
    windowed pass and is clamped around the estimate (k = 1 still hits);
    k near N takes lo = 0.  Masks == the oracle's."""
    T = 32768
    n = 3 * T + 77
    g = np.random.default_rng(12)
    x = np.exp2(g.uniform(-120.0, 0.0, n)) * np.where(g.random(n) < 0.5, -1.0, 1.0)
    if dtype == "f32":
        w = x.astype(np.float32)
        shard, val = torch.from_numpy(w).to(DEV), w.astype(np.float64)
    else:
        t16 = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
        shard = t16.to(DEV)
        val = oracle.bf16_to_f64(t16.view(torch.int16).numpy().view(np.uint16))
    mask = torch.zeros(n, dtype=torch.uint8, device=DEV)
    plan = D.PrunePlan(ctx, [(shard, mask)])
    for k in [1, 100, 5000, n - 50, n]:
        info, st = D.global_prune(ctx, plan, k)
        torch.cuda.synchronize()
        ost, omask = oracle.global_prune([val], k)
        assert int(st.item()) == ost == 0
        assert np.array_equal(mask.cpu().numpy(), omask[0]), k
        if k == 1:
            assert (int(info[5].item()) & 1) == 0
    plan.close()


def test_global_prune_errors_and_nan(D, ctx):
    """k > N: INVALID, all masks 0; a NaN is never kept and sets INVALID
    (the selection runs over the other weights, like the oracle)."""
    w = torch.tensor([1.0, float("nan"), -3.0, 0.5], device=DEV)
    m = torch.full((4,), 7, dtype=torch.uint8, device=DEV)
    plan = D.PrunePlan(ctx, [(w, m)])
    info, st = D.global_prune(ctx, plan, 2)
    torch.cuda.synchronize()
    ost, om = oracle.global_prune([w.cpu().numpy().astype(np.float64)], 2)
    assert int(st.item()) == ost == oracle.E_INVALID and np.array_equal(m.cpu().numpy(), om[0])
    info, st = D.global_prune(ctx, plan, 4)  # 3 non-NaN weights
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_INVALID and int(m.sum().item()) == 0
    with pytest.raises(D.DynmoError):
        D.global_prune(ctx, plan, -1)
    plan.close()


def test_global_prune_config2_full_size(D, ctx):
    """Config 2 at full size (48 layers x 12,582,912 bf16 weights = 604 M,
    sigma_l per layer as in synth.cfg2; drawn on the GPU, seeded), S = 0.9:
    properties the oracle fixes at any size -- exactly k kept, every kept
    |w| >= every pruned |w|, and the kept ties (|w| = tau) are a prefix of the
    ties in global order (layer, then index)."""
    shape = synth.GPTShape()
    gen = torch.Generator(device=DEV).manual_seed(2505)
    sig = torch.from_numpy(np.exp(np.random.default_rng(3).normal(0, 0.35, shape.L))).float()
    ws = [(torch.randn(shape.params_per_layer, generator=gen, device=DEV) * float(sig[l])).to(torch.bfloat16)
          for l in range(shape.L)]
    ms = [torch.empty(shape.params_per_layer, dtype=torch.uint8, device=DEV) for _ in range(shape.L)]
    plan = D.PrunePlan(ctx, list(zip(ws, ms)))
    N = shape.L * shape.params_per_layer
    k = int(N * (1 - 0.9))
    info, st = D.global_prune(ctx, plan, k)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    inf = info.cpu().numpy()
    tau = int(inf[0])
    kept = sum(int(m.sum(dtype=torch.int64).item()) for m in ms)
    assert kept == k and inf[2] + inf[3] == k
    assert inf[5] == 2  # window hit, tie counts from the windowed pass (the bench's path)
    kmin = min(float(w.float().abs()[m.bool()].min().item()) for w, m in zip(ws, ms) if int(m.sum().item()) > 0)
    pmax = max(float(w.float().abs()[~m.bool()].max().item()) for w, m in zip(ws, ms) if int((m == 0).sum().item()) > 0)
    assert kmin >= pmax
    tau_val = float(np.array([tau], np.uint32).view(np.float32)[0])
    assert kmin == tau_val
    seen_pruned_tie = False
    for w, m in zip(ws, ms):
        tie = w.float().abs() == tau_val
        kt = (m.bool() & tie).nonzero().flatten()
        pt = (~m.bool() & tie).nonzero().flatten()
        if seen_pruned_tie:
            assert kt.numel() == 0
        if pt.numel():
            if kt.numel():
                assert int(kt.max().item()) < int(pt.min().item())
            seen_pruned_tie = True
    plan.close()


# ------------------------------ NEXT-3: migration-minimising stage -> rank map
def test_map_stages_parity(D, ctx):
    """dynmo_map_stages == the oracle (reading Q23): rank vector, kept bytes
    and status on random instances, G up to 16 ranks, up to 1023 layers,
    random allowed masks (INFEASIBLE ones included), tie-heavy bytes."""
    g = np.random.default_rng(230)
    for it in range(150):
        G = int(g.integers(1, 17))
        L = int(g.integers(2, 1024 if it % 10 == 0 else 120))
        n_old = int(g.integers(1, min(L, 16) + 1))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_old - 1, replace=False)), [L]]).astype(np.int32)
        ro = g.integers(0, G, n_old).astype(np.int32)
        allowed = int(g.integers(1, 1 << G))
        n_new = int(g.integers(1, min(L, 16) + 1))
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)), [L]]).astype(np.int32)
        nb = (g.integers(0, 5, L) * (1 << int(g.integers(0, 30)))).astype(np.int64)
        rn, kept, st = D.map_stages(ctx, L, _dev(bo), _dev(ro), _dev(bn), _dev(nb), G, allowed)
        torch.cuda.synchronize()
        ost, orn, okept = oracle.map_stages(L, bo, ro, bn, nb, G, allowed)
        assert int(st.item()) == ost, (it, int(st.item()), ost)
        if ost == 0:
            assert np.array_equal(rn.cpu().numpy(), orn) and int(kept.item()) == okept, it
    # slots (several stages per GPU): slot j on GPU sr[j]
    for it in range(60):
        S = int(g.integers(2, 17))
        sr = np.sort(g.integers(0, int(g.integers(1, S + 1)), S)).astype(np.int32)
        L = int(g.integers(S, 200))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), S - 1, replace=False)), [L]]).astype(np.int32)
        ro = np.arange(S, dtype=np.int32)
        n_new = int(g.integers(1, S + 1))
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)), [L]]).astype(np.int32)
        nb = g.integers(0, 5, L).astype(np.int64) * 1000
        rn, kept, st = D.map_stages(ctx, L, _dev(bo), _dev(ro), _dev(bn), _dev(nb), S, slot_rank=_dev(sr))
        torch.cuda.synchronize()
        ost, orn, okept = oracle.map_stages(L, bo, ro, bn, nb, S, slot_rank=sr)
        assert int(st.item()) == ost == 0 and np.array_equal(rn.cpu().numpy(), orn) and int(kept.item()) == okept
    # malformed split and negative bytes: INVALID
    bo, ro, bn = np.array([0, 2, 4], np.int32), np.array([0, 1], np.int32), np.array([0, 3, 3], np.int32)
    rn, kept, st = D.map_stages(ctx, 4, _dev(bo), _dev(ro), _dev(bn), _dev(np.ones(4, np.int64)), 2)
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_INVALID
    rn, kept, st = D.map_stages(ctx, 4, _dev(bo), _dev(ro), _dev(np.array([0, 4], np.int32)),
                                _dev(np.array([1, -1, 1, 1], np.int64)), 2)
    torch.cuda.synchronize()
    assert int(st.item()) == oracle.E_INVALID
    with pytest.raises(D.DynmoError):
        D.map_stages(ctx, 4, _dev(bo), _dev(ro), _dev(bn), _dev(np.ones(4, np.int64)), 17)


# ------------------------------- NEXT-4: sparse-attention block masks (a1 source)
def test_sparse_attention_block_masks(D, L, ctx):
    """Dynamic sparse flash attention: layer cost s_i c_i =
    (computed attention blocks) x (cost per block) -- a bit-mask source: the
    per-layer block counts and B * count costs vs the oracle, then the
    partition of those costs."""
    Lyr, n, per_block = 32, 8, 64 * 64 * 64 * 2
    segs, keep, want = [], [], np.zeros(Lyr, np.int64)
    for l in range(Lyr):
        w = synth.sparse_attention_blocks(l)
        nbits = 2 * 16 * 32 * 32
        want[l] = oracle.count_bits(w, nbits)
        t = _dev(w.view(np.int32))
        keep.append(t)
        segs.append(D.SegmentSpec(t, L.SRC_MASK_BITS, l, n_elem=nbits))
    plan = D.ProfilePlan(ctx, segs, 0, Lyr)
    counters = torch.empty((Lyr, 5), dtype=torch.int64, device=DEV)
    cost, _, st = D.profile_layers(ctx, plan, D.coef_tensor(Lyr, B=per_block, device=DEV), counters=counters)
    b = D.Batch([Lyr], [n], device=DEV)
    bnd, bott, _, pst = D.partition_stages(ctx, b, cost)
    torch.cuda.synchronize()
    want_cost = np.array([oracle.layer_cost(nnz=int(v), B=per_block)[1] for v in want])
    assert int(st.item()) == 0 and np.array_equal(counters[:, 0].cpu().numpy(), want)
    assert np.array_equal(cost.cpu().numpy(), want_cost)
    ost, ob, oB, _ = oracle.partition(want_cost, n)
    assert int(pst.item()) == ost == 0 and np.array_equal(bnd.cpu().numpy()[:n + 1], ob)
    assert len(set(want.tolist())) > 4  # sparsity really varies across layers


def test_ctx_barrier_timing_detach_and_split_single(D, L, ctx):
    """dynmo_ctx_barrier is a no-op for one rank and capturable; timing_detach
    stops polling earlier graphs' events (their graphs stay valid); a split
    of a one-rank ctx gives a usable ctx (color >= 0) or None (color < 0)."""
    x = torch.zeros(1, device=DEV)
    g = torch.cuda.CUDAGraph()
    ctx.set_timing(True, phases=["profile"])
    seg = D.SegmentSpec(_dev(np.ones(4096, np.uint8)), L.SRC_MASK_U8, 0)
    plan = D.ProfilePlan(ctx, [seg], 0, 1)
    coef = D.coef_tensor(1, B=1, device=DEV)
    D.profile_layers(ctx, plan, coef)  # warm
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        ctx.barrier()
        D.profile_layers(ctx, plan, coef)
        x.add_(1)
    g.replay()
    torch.cuda.synchronize()
    ctx.timing_poll()
    n1 = ctx.timing_read()["profile"][1]
    ctx.timing_detach()
    g.replay()
    torch.cuda.synchronize()
    ctx.timing_poll()
    assert n1 >= 1 and ctx.timing_read()["profile"][1] == 0 and float(x.item()) == 2.0
    ctx.set_timing(False)
    sub = ctx.split(active=True)
    assert sub is not None and sub.nranks == 1 and sub.rank == 0
    cost, _, st = D.profile_layers(sub, D.ProfilePlan(sub, [seg], 0, 1), coef)
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and int(cost[0].item()) == 4096
    sub.close()
    assert ctx.split(active=False) is None
    del g


def test_publish_to_pinned_host(D, L, ctx):
    """dynmo_publish: device bytes stored by a kernel into mapped pinned host
    memory -- every size class (0, bytes, one vector, a partial CTA, several
    CTAs), aligned and unaligned ends, eager and inside a replayed CUDA graph;
    non-pinned / device destinations and host sources are INVALID."""
    import ctypes
    g = torch.Generator().manual_seed(5)
    for nb in (0, 1, 7, 16, 48, 4096, 49_156, 1 << 20):
        for off in (0, 3, 16):
            src_full = torch.randint(0, 256, (nb + off + 1,), dtype=torch.uint8, generator=g).cuda()
            dst_full = torch.zeros(nb + off + 5, dtype=torch.uint8).pin_memory()
            src, dst = src_full[off:off + nb], dst_full[off:off + nb]
            if nb == 0:
                assert L.lib().dynmo_publish(ctx.handle, src_full.data_ptr(), dst_full.data_ptr(), 0, None) == 0
                continue
            D.publish(ctx, src, dst)
            torch.cuda.synchronize()
            assert torch.equal(dst, src.cpu()), (nb, off)
            assert not dst_full[off + nb:].any() and not dst_full[:off].any(), (nb, off)
    # inside a graph: the replay publishes the current device contents
    src = torch.arange(40, dtype=torch.int32, device="cuda")
    dst = torch.zeros(40, dtype=torch.int32).pin_memory()
    side = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=side):
        src.add_(1)
        D.publish(ctx, src, dst)
    for k in range(3):
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(dst, torch.arange(40, dtype=torch.int32) + k + 1), k
    del gr
    # errors: pageable host destination, device destination, host source
    pageable = torch.zeros(64, dtype=torch.uint8)
    dsrc = torch.zeros(64, dtype=torch.uint8, device="cuda")
    assert L.lib().dynmo_publish(ctx.handle, dsrc.data_ptr(), pageable.data_ptr(), 64, None) == L.E_INVALID
    assert L.lib().dynmo_publish(ctx.handle, dsrc.data_ptr(), dsrc.data_ptr(), 64, None) == L.E_INVALID
    pin = torch.zeros(64, dtype=torch.uint8).pin_memory()
    assert L.lib().dynmo_publish(ctx.handle, pin.data_ptr(), pin.data_ptr(), 64, None) == L.E_INVALID
    with pytest.raises(ValueError):
        D.publish(ctx, dsrc, pageable)
    torch.cuda.synchronize()


def test_profile_span_clock(D, L, ctx):
    """With the profile phase timed, every k_profile launch (eager and graph
    replays) also records its device-clock span (dynmo_ctx_profile_span):
    one span per launch, positive, no longer than the launch's event pair;
    the counts stay exact; untimed launches record nothing."""
    seg = D.SegmentSpec(_dev((np.arange(1 << 22) % 3).astype(np.uint8)), L.SRC_MASK_U8, 0)
    plan = D.ProfilePlan(ctx, [seg], 0, 1)
    coef = D.coef_tensor(1, B=1, device=DEV)
    D.profile_layers(ctx, plan, coef)
    torch.cuda.synchronize()
    ctx.profile_span()
    ctx.set_timing(True, phases=["profile"])
    ctx.timing_read()
    for _ in range(3):
        cost, _, st = D.profile_layers(ctx, plan, coef)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        D.profile_layers(ctx, plan, coef)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        ctx.timing_poll()
    torch.cuda.synchronize()
    ev_ms, ev_n = ctx.timing_read()["profile"]
    sp_ms, sp_n = ctx.profile_span()
    ctx.timing_detach()
    ctx.set_timing(False)
    assert int(st.item()) == 0 and int(cost[0].item()) == (1 << 22) * 2 // 3
    assert ev_n == 5 and sp_n == 5, (ev_n, sp_n)
    assert 0.0 < sp_ms <= ev_ms, (sp_ms, ev_ms)
    D.profile_layers(ctx, plan, coef)  # untimed: no span
    torch.cuda.synchronize()
    assert ctx.profile_span() == (0.0, 0)
    plan.close()


# ------------------------------- round 2: hand traces, large n, 1-rank exchange
import json as _json
import os as _os

_GOLD = _json.load(open(_os.path.join(_os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_diffuse_hand_traces_gpu(D, ctx):
    """The hand-worked traces of DESIGN.md 2a (tests/golden) on the GPU,
    stopped after every round (max_rounds = r) and run to the end: the kernel
    reproduces each hand-derived split / phi and, for F1/F2, the fluid loads
    after every round (dyadic, so exact)."""
    for ex in _GOLD["diffusion_traces"]:
        n = len(ex["bnd_in"]) - 1
        mem = ex.get("mem")
        wm = mem is not None
        rows = [r for r in ex["rounds"] if r["bnd_after"] is not None]
        for r in range(len(rows) + 2):
            x = dict(cost=np.array(ex["cost"]), n=n, bnd_in=np.array(ex["bnd_in"], np.int32),
                     mem=np.array(mem) if wm else None, cap=ex.get("cap", 0), gamma=ex["gamma"])
            b, o = _run_diffuse(D, ctx, [x], wm, r)
            want_b = ex["bnd_in"] if r == 0 else (rows[r - 1]["bnd_after"] if r <= len(rows) else ex["bnd_out"])
            assert list(o["bnd"][:n + 1]) == list(want_b), (ex["name"], r)
            assert o["rounds"][0] == min(r, ex["n_rounds"]) and o["phi0"][0] == ex["phi0"], (ex["name"], r)
            assert o["status"][0] == (0 if r >= ex["n_rounds"] else 1), (ex["name"], r)
        assert o["phi"][0] == ex["phi"]
    for ex in _GOLD["fluid_traces"]:
        n = len(ex["bnd_in"]) - 1
        for r, xr in enumerate(ex["x_after"]):
            x = dict(cost=np.array(ex["cost"]), n=n, bnd_in=np.array(ex["bnd_in"], np.int32), mem=None, cap=0,
                     gamma_f=ex["gamma_f"])
            b, o = _run_diffuse(D, ctx, [x], False, r)
            assert list(o["fluid_x"][:n]) == xr and o["fluid_rounds"][0] == r, (ex["name"], r)
            assert o["fluid_phi"][0] == ex["phi_after"][r]


@pytest.mark.parametrize("n,Lmax,with_mem", [(33, 200, False), (64, 600, True), (200, 1023, False),
                                             (200, 1023, True)])
def test_diffuse_large_n(D, ctx, n, Lmax, with_mem):
    """Diffusion with n > 32 stages: the lane-strided
    discrete loops and the serial fluid path of k_diffuse, L up to 1023,
    against the oracle element by element (fluid loads bit-equal)."""
    g = np.random.default_rng(n * 7 + Lmax)
    insts = []
    for q in range(12):
        Ly = int(g.integers(n, Lmax + 1)) if q else Lmax
        cost = g.integers(0, 1000, Ly)
        cost[g.random(Ly) < 0.1] = 0
        inner = np.sort(g.choice(np.arange(1, Ly), n - 1, replace=False))
        bnd = np.concatenate([[0], inner, [Ly]]).astype(np.int32)
        x0 = oracle.stage_loads(cost, bnd).astype(float)
        x = dict(cost=cost, n=n, bnd_in=bnd, gamma=0, gamma_f=float(g.choice([1e-9, 1e-3])) * oracle.phi_f64(x0),
                 mem=None, cap=0)
        if with_mem:
            x["mem"] = g.integers(0, 50, Ly)
            x["cap"] = int(max(x["mem"].max(), x["mem"].sum() * 2 // n))
        insts.append(x)
    _check_diffuse(D, ctx, insts, with_mem, 4096)


@pytest.mark.parametrize("exchange", [1, 2])
def test_profile_exchange_single_rank(D, L, ctx, exchange):
    """Exchange modes on a one-rank ctx: the peer-memory
    LL slots (encode with the call epoch, poll/decode, double buffering by
    epoch parity) and the NCCL all-gather (a one-rank communicator) + unpack
    run against the oracle on one GPU, over several calls and CUDA-graph
    replays; a slice that does not tile [0, n_total) gives INVALID."""
    T, Lyr = 300_007, 24
    e = synth.cfg3_exit_depth(T=T, L=Lyr)
    tok = oracle.exit_survivors(e, 0, Lyr)
    seg = [D.SegmentSpec(_dev(e), L.SRC_EXIT_U8, 0)]
    c1 = D.Context(0)
    plan = D.ProfilePlan(c1, seg, 0, Lyr, Lyr, exchange=exchange)
    memv = np.arange(Lyr, dtype=np.int64) * 1000 + 7
    coef = D.coef_tensor(Lyr, A=3, device=DEV)
    want = [oracle.layer_cost(tok=int(tok[i]), A=3)[1] for i in range(Lyr)]
    cost = torch.empty(Lyr, dtype=torch.int64, device=DEV)
    mem = torch.empty(Lyr, dtype=torch.int64, device=DEV)
    st = torch.empty(1, dtype=torch.int32, device=DEV)
    mem_local = _dev(memv)
    for _ in range(3):
        cost.fill_(-5); mem.fill_(-5)
        D.profile_layers(c1, plan, coef, mem_local=mem_local, cost=cost, mem=mem, status=st)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        assert np.array_equal(cost.cpu().numpy(), want) and np.array_equal(mem.cpu().numpy(), memv)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(gph, stream=s):
        D.profile_layers(c1, plan, coef, mem_local=mem_local, cost=cost, mem=mem, status=st, stream=s)
    for _ in range(5):
        cost.fill_(-5)
        gph.replay()
        torch.cuda.synchronize()
        assert int(st.item()) == 0 and np.array_equal(cost.cpu().numpy(), want)
    assert c1.p2p_error() == 0
    # a slice that does not cover [0, n_total): layers 20..23 have no owner
    plan2 = D.ProfilePlan(c1, seg, 0, 20, Lyr, exchange=exchange)
    coef2 = D.coef_tensor(20, A=3, device=DEV)
    cost2, _, st2 = D.profile_layers(c1, plan2, coef2)
    torch.cuda.synchronize()
    assert int(st2.item()) == L.E_INVALID
    c2 = cost2.cpu().numpy()
    assert np.array_equal(c2[:20], want[:20]) and np.all(c2[20:] == -1)
    del gph, plan, plan2
    c1.close()


@pytest.mark.parametrize("T_bits", [4096, 8192, 32768])
def test_profile_strided_bitmask_runs(D, L, ctx, T_bits):
    """Runs of bit-mask segments back to back in memory (one per consecutive
    layer, equal sizes) become strided tiles (one descriptor per tile of
    whole layers): run lengths that are not multiples of 8, a run broken by
    a gap, by a different size and by a non-consecutive layer, S = 32 / 64 /
    256 vectors per layer, MASK_BITS and TOKMASK_BITS; per-layer counts vs
    the oracle."""
    g = np.random.default_rng(T_bits)
    W = T_bits // 32
    nl = 61
    words = g.integers(0, 2 ** 32, (nl + 3) * W, dtype=np.uint64).astype(np.uint32)
    words[:W * 5] &= 0x01010101  # sparse rows too
    d = _dev(words.view(np.int32))
    segs, want = [], np.zeros(nl + 2, np.int64)
    off = 0
    for layer in range(nl):
        if layer == 23:
            off += W  # a gap: the run breaks here
        kind = L.SRC_MASK_BITS if layer < 40 else L.SRC_TOKMASK_BITS  # kind change breaks the run
        nb = T_bits if layer != 50 else T_bits - 128  # a shorter segment breaks the run
        segs.append(D.SegmentSpec(d[off:off + nb // 32], kind, layer, n_elem=nb))
        want[layer] = oracle.count_bits(words[off:off + nb // 32], nb)
        off += W
    # a second source on an earlier layer (not consecutive): its own tiles
    segs.append(D.SegmentSpec(d[off:off + W], L.SRC_MASK_BITS, 3, n_elem=T_bits))
    want[3] += oracle.count_bits(words[off:off + W], T_bits)
    plan = D.ProfilePlan(ctx, segs, 0, nl + 2)
    coef = D.coef_tensor(nl + 2, A=0, B=1, device=DEV)
    cnt = torch.empty((nl + 2, 5), dtype=torch.int64, device=DEV)
    tokl = np.arange(nl + 2) >= 40  # TOKMASK layers count tokens, the others nonzeros
    for rep in range(2):
        cnt.fill_(-7)
        cost, _, st = D.profile_layers(ctx, plan, coef, counters=cnt)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        c = cnt.cpu().numpy()
        got = np.where(tokl, c[:, 1], c[:, 0])
        got[nl:] = c[nl:, 0]  # layers without a source: nnz = 0
        assert np.array_equal(got, want), (rep, np.flatnonzero(got != want))
    if T_bits <= 8192:  # runs merged: several layers per tile
        assert plan.n_tiles < len(segs) // 2, plan.n_tiles


def test_global_prune_reproduces_cfg2_masks(D, ctx):
    """The config-2 masks are the exact global top-k of synth's bf16 weights
    (by construction): the GPU's Alg. 1 (dynmo_global_prune) with k = the
    masks' kept count reproduces every mask byte (GPT-12 at h = 256, 9.4 M
    weights, several 32768-element tiles per tensor)."""
    shape = synth.GPTShape(L=12, h=256)
    p = synth.cfg2_keep_probs(shape, 0.9, 4)
    pairs, masks = [], []
    for layer in range(shape.L):
        for t, m in enumerate(synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4)):
            w = synth.cfg2_topk_weights_bf16(m, layer, t).reshape(-1)
            wt = _dev(w.view(np.int16)).view(torch.bfloat16)
            pairs.append((wt, torch.zeros(w.size, dtype=torch.uint8, device=DEV)))
            masks.append(m.reshape(-1))
    k = int(sum(int(m.sum()) for m in masks))
    pplan = D.PrunePlan(ctx, pairs)
    info, st = D.global_prune(ctx, pplan, k)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    for (_, mk), m in zip(pairs, masks):
        assert np.array_equal(mk.cpu().numpy(), m)
    pplan.close()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_bench_configs_gpu_arm(cfg):
    """bench.py --config 3/4/5 on one GPU: the GPU arm runs every step in
    its graph and prints the contract's JSON line (roofline, e2e, clocks)."""
    import json as js
    import subprocess
    import sys
    root = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--config", str(cfg), "--steps", "8", "--warmup", "3",
                        "--e2e-steps", "2", "--no-cpu-baseline"], cwd=root, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = js.loads(r.stdout.strip().splitlines()[-1])
    assert d["value"] > 0 and d["roofline"]["frac"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0

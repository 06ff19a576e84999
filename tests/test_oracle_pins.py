"""Pins for the CPU oracle (tests the oracle against something other than itself).

Each test names the pin: library routine, brute-force enumeration, a SPEC/paper
worked example from tests/golden/, a closed form, or an invariant.  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ O1 counters
def test_counters_vs_numpy_library():
    """Pin: np.bitwise_count / np.count_nonzero / np.bincount on the same arrays."""
    g = np.random.default_rng(7)
    for n in [0, 1, 7, 8, 31, 32, 33, 1000, 4099]:
        m = (g.random(n) < 0.3).astype(np.uint8)
        w = synth.pack_bits(m)
        assert oracle.count_bits(w, n) == int(np.bitwise_count(w).sum())
        assert oracle.count_bits(w, n) == int(np.count_nonzero(m))
        v = g.integers(0, 4, n).astype(np.uint8)
        assert oracle.count_nz_u8(v) == int(np.count_nonzero(v))
        f = g.normal(size=n).astype(np.float32)
        f[g.random(n) < 0.5] = 0.0
        f[g.random(n) < 0.1] = -0.0
        if n > 3:
            f[3] = np.nan
        assert oracle.count_nz_f32(f) == int(np.count_nonzero(f))
        bf = (f.view(np.uint32) >> 16).astype(np.uint16)
        as_f32 = (bf.astype(np.uint32) << 16).view(np.float32)
        assert oracle.count_nz_bf16(bf) == int(np.count_nonzero(as_f32))


def test_count_bits_ignores_tail_bits():
    """Pin: bits past n_elem are ignored (set every tail bit)."""
    w = np.array([0xFFFFFFFF, 0xFFFFFFFF], np.uint32)
    for n in range(0, 65):
        assert oracle.count_bits(w, n) == n


def test_exit_survivors_vs_bincount():
    """Pin: tok_i = #{t: e[t] > i} == reversed cumulative np.bincount; non-increasing."""
    e = synth.cfg3_exit_depth(T=50_000, L=32)
    h = np.bincount(e, minlength=256)
    suffix = np.cumsum(h[::-1])[::-1]      # suffix[v] = #{e >= v}
    tok = oracle.exit_survivors(e, 0, 32)
    assert np.array_equal(tok, suffix[1:33])
    assert np.all(np.diff(tok) <= 0)
    assert np.all(tok[:8] == len(e))        # no exits before layer 8
    # a local slice of layers equals the same slice of the global vector
    assert np.array_equal(oracle.exit_survivors(e, 12, 7), tok[12:19])


def test_expert_hist_vs_bincount():
    """Pin: np.bincount; invariant sum = T*k; out-of-range -> INVALID."""
    idx = synth.cfg4_routing(3, T=5000, E=8, k=2)
    st, cnt = oracle.expert_hist(idx, 8)
    assert st == 0
    assert np.array_equal(cnt, np.bincount(idx.ravel(), minlength=8))
    assert cnt.sum() == 5000 * 2
    st32, cnt32 = oracle.expert_hist(idx.astype(np.int32), 8)
    assert st32 == 0 and np.array_equal(cnt32, cnt)
    bad = idx.copy()
    bad[10, 1] = 8
    assert oracle.expert_hist(bad, 8)[0] == oracle.E_INVALID
    bad[10, 1] = -1
    assert oracle.expert_hist(bad, 8)[0] == oracle.E_INVALID


# ---------------------------------------------------------------------- O2 cost
def test_cost_spec_examples():
    """Pin: SPEC.md:L79-81 worker loads (incl. freezing) through the cost formula."""
    for ex in GOLD["worker_loads"]:
        costs = [oracle.layer_cost(A=c)[1] for c in ex["cost"]]
        assert list(oracle.stage_loads(costs, ex["bnd"])) == ex["loads"], ex["cite"]
    for ex in GOLD["freeze_cost"]:
        costs = [oracle.layer_cost(frozen=f, A=c, F=0)[1] for c, f in zip(ex["base"], ex["frozen"])]
        assert list(oracle.stage_loads(costs, ex["bnd"])) == ex["loads"], ex["cite"]


def test_cost_formula_special_cases():
    """Pin: each paper form is a special case (reading Q1): pruning p_i c_i
    (P:L238), early exit t_i/t c_i (times t), MoD r_i t_i c_i."""
    # pruning: A=0, B=1 -> cost = nnz
    assert oracle.layer_cost(nnz=12345, A=0, B=1) == (0, 12345)
    # early exit: A=c_i, B=0, tok=t_i -> t_i * c_i
    assert oracle.layer_cost(tok=700, A=9) == (0, 6300)
    # frozen: F default 0
    assert oracle.layer_cost(frozen=True, tok=700, A=9) == (0, 0)
    assert oracle.layer_cost(frozen=True, A=9, F=4) == (0, 4)
    # MoE with EP=1: moe = sum of counts = T*k (no imbalance, reading Q5)
    cnt = np.array([5, 1, 0, 2], np.int64)
    assert oracle.layer_cost(cnt=cnt, C_=1, ep=1) == (0, 8)
    # EP=E: moe = E * max count
    assert oracle.layer_cost(cnt=cnt, C_=1, ep=4) == (0, 20)
    # EP=2: groups {0,1},{2,3}: max(6,2)*2 = 12; default EP (0) = E
    assert oracle.layer_cost(cnt=cnt, C_=1, ep=2) == (0, 12)
    assert oracle.layer_cost(cnt=cnt, C_=1, ep=0) == (0, 20)
    assert oracle.layer_cost(cnt=cnt, C_=1, ep=3)[0] == oracle.E_INVALID  # 4 % 3 != 0
    # full form
    assert oracle.layer_cost(tok=3, nnz=10, cnt=cnt, A=2, B=5, C_=7, ep=1) == (0, 3 * (2 + 50) + 7 * 8)


def test_cost_overflow_and_invalid():
    """Pin: exact int64 limit (closed form 2^63-1)."""
    big = 2 ** 62
    assert oracle.layer_cost(tok=2, A=big - 1, B=0) == (0, 2 ** 63 - 2)
    assert oracle.layer_cost(tok=2, A=big, B=0)[0] == oracle.E_OVERFLOW
    assert oracle.layer_cost(nnz=2 ** 40, A=0, B=2 ** 23 - 1) == (0, (2 ** 23 - 1) * 2 ** 40)
    assert oracle.layer_cost(nnz=2 ** 40, A=0, B=2 ** 23)[0] == oracle.E_OVERFLOW
    assert oracle.layer_cost(A=-1)[0] == oracle.E_INVALID


# -------------------------------------------------------------- ΔL and φ
def test_time_ns_pins():
    """O1' (P:L632/P:L720 execution-time profiling, reading Q21): boundary
    stamps telescope -- sum over layers of (s[i+1] - s[i]) = s[L] - s[0];
    random pairs vs Python integers; end < begin and an odd count INVALID;
    a sum above INT64_MAX is OVERFLOW; the by-Time cost is the time itself."""
    g = np.random.default_rng(21)
    for _ in range(50):
        L = int(g.integers(1, 40))
        s_ = np.cumsum(g.integers(0, 10 ** 9, L + 1)).astype(np.int64)
        per = [oracle.time_ns(s_[i:i + 2]) for i in range(L)]
        assert all(st == 0 for st, _ in per)
        assert sum(t for _, t in per) == int(s_[-1] - s_[0])
        pairs = g.integers(0, 2 ** 40, (int(g.integers(1, 30)), 2)).astype(np.int64)
        pairs.sort(axis=1)
        assert oracle.time_ns(pairs.reshape(-1)) == (0, sum(int(e) - int(b) for b, e in pairs))
    assert oracle.time_ns(np.array([5, 4], np.int64))[0] == oracle.E_INVALID
    assert oracle.time_ns(np.array([1, 2, 3], np.int64))[0] == oracle.E_INVALID
    assert oracle.time_ns(np.array([0, 2 ** 62, 0, 2 ** 62, 0, 2 ** 62], np.int64))[0] == oracle.E_OVERFLOW
    assert oracle.time_ns(np.zeros(0, np.int64)) == (0, 0)
    # cost: D * time added last, checked; by Time = the time itself
    assert oracle.layer_cost(D=1, time=123456789) == (0, 123456789)
    assert oracle.layer_cost(tok=3, A=2, nnz=5, B=1, D=4, time=10) == (0, 3 * (2 + 5) + 40)
    assert oracle.layer_cost(frozen=True, F=7, D=1, time=99) == (0, 7)
    assert oracle.layer_cost(D=-1, time=1)[0] == oracle.E_INVALID
    assert oracle.layer_cost(D=2, time=2 ** 62)[0] == oracle.E_OVERFLOW
    assert oracle.layer_cost(D=1, time=2 ** 63 - 1) == (0, 2 ** 63 - 1)
    assert oracle.layer_cost(A=1, D=1, time=2 ** 63 - 1)[0] == oracle.E_OVERFLOW


def test_imbalance_and_phi_spec_examples():
    """Pin: SPEC.md:L89-91 (eq:imbalance) and SPEC.md:L301-303 (phi)."""
    for ex in GOLD["imbalance"]:
        assert oracle.imbalance(ex["loads"]) == pytest.approx(ex["delta"], rel=1e-15), ex["cite"]
    assert oracle.imbalance([0, 0, 0]) == 0.0  # reading Q18
    for ex in GOLD["phi"]:
        assert oracle.phi(ex["loads"]) == (0, ex["phi"]), ex["cite"]
        assert oracle.phi_f64(np.array(ex["loads"], float)) == ex["phi"]


def test_phi_closed_form_sorted():
    """Pin: phi = sum_i (2i - n + 1) x_(i) over the sorted loads (closed form)."""
    g = np.random.default_rng(3)
    for _ in range(200):
        n = int(g.integers(1, 17))
        x = g.integers(0, 10 ** 12, n)
        xs = np.sort(x)
        closed = int(sum((2 * i - n + 1) * int(v) for i, v in enumerate(xs)))
        assert oracle.phi(x) == (0, closed)


# ----------------------------------------------------------------- O4 partition
def test_partition_spec_examples():
    """Pin: SPEC.md:L271-273 and L312."""
    for ex in GOLD["partition"]:
        st, b, B, _ = oracle.partition(ex["cost"], ex["n"])
        assert st == 0 and list(b) == ex["bnd"] and B == ex["bottleneck"], ex["cite"]


def test_partition_vs_bruteforce_tiny():
    """Pin: brute force over all C(L-1, n-1) splits, >= 5000 instances,
    L <= 12, n <= 6, costs in [0, 9] incl. zeros and ties; B* and lexmax b."""
    g = np.random.default_rng(11)
    ties = 0
    for it in range(5000):
        L = int(g.integers(1, 13))
        n = int(g.integers(1, min(6, L) + 1))
        cost = g.integers(0, 10, L)
        if it % 4 == 0:
            cost = g.choice([0, 1, 2, 9], L)
        st, b, B, imb = oracle.partition(cost, n)
        Bb, bb = brute.partition(cost, n)
        assert st == 0
        assert B == Bb, (cost, n)
        assert np.array_equal(b, bb), (cost, n, b, bb)
        ties += brute.n_optima(cost, n) > 1
        x = oracle.stage_loads(cost, b)
        assert x.max() == B
    assert ties > 1000  # ties are common, so the lexmax rule is exercised


def test_partition_with_memory_vs_bruteforce():
    """Pin: brute force with the per-stage memory cap (reading Q9)."""
    g = np.random.default_rng(12)
    infeasible = 0
    for _ in range(3000):
        L = int(g.integers(1, 11))
        n = int(g.integers(1, min(5, L) + 1))
        cost = g.integers(0, 10, L)
        mem = g.integers(0, 10, L)
        cap = int(g.integers(0, 25))
        st, b, B, _ = oracle.partition(cost, n, mem=mem, cap=cap)
        Bb, bb = brute.partition(cost, n, mem=mem, cap=cap)
        if Bb is None:
            assert st == oracle.E_INFEASIBLE and B == -1 and np.all(b == -1)
            infeasible += 1
        else:
            assert st == 0 and B == Bb and np.array_equal(b, bb), (cost, mem, cap, n)
    assert infeasible > 100


def test_partition_config1_vs_bruteforce():
    """Pin: config 1 (24 layers, 4 stages: C(23,3)=1771 splits each)."""
    for inst in synth.cfg1_instances(400):
        st, b, B, _ = oracle.partition(inst["cost"], 4, mem=inst["mem"], cap=inst["cap"])
        Bb, bb = brute.partition(inst["cost"], 4, mem=inst["mem"], cap=inst["cap"])
        if Bb is None:
            assert st == oracle.E_INFEASIBLE
        else:
            assert st == 0 and B == Bb and np.array_equal(b, bb)


def test_partition_lower_bound_and_invalid():
    """Pin: B* >= max(max c, ceil(C/n)) (trivial bound); n > L invalid."""
    g = np.random.default_rng(5)
    for _ in range(500):
        L = int(g.integers(1, 60))
        n = int(g.integers(1, L + 1))
        cost = g.integers(0, 1000, L)
        st, b, B, _ = oracle.partition(cost, n)
        assert st == 0
        assert B >= max(int(cost.max()), -(-int(cost.sum()) // n))
        assert B <= -(-int(cost.sum()) // n) + int(cost.max())  # Appendix A bracket
    assert oracle.partition([1, 2], 3)[0] == oracle.E_INVALID
    assert oracle.partition([1, -2], 1)[0] == oracle.E_INVALID
    assert oracle.partition([2 ** 62, 2 ** 62], 1)[0] == oracle.E_OVERFLOW
    # a bottleneck of exactly INT64_MAX is a legal optimum (brute force agrees)
    big = [2 ** 62, 2 ** 62 - 1]
    assert oracle.partition(big, 1, mem=[1, 1], cap=5)[2] == 2 ** 63 - 1 == brute.partition(big, 1)[0]
    assert oracle.partition(big, 2)[2] == 2 ** 62 == brute.partition(big, 2)[0]


def test_partition_scale_invariance():
    """Pin: decisions invariant under a positive common scale (reading Q1)."""
    g = np.random.default_rng(9)
    for _ in range(300):
        L = int(g.integers(2, 30))
        n = int(g.integers(1, min(8, L) + 1))
        cost = g.integers(0, 50, L)
        a = int(g.integers(2, 1000))
        s1, b1, B1, d1 = oracle.partition(cost, n)
        s2, b2, B2, d2 = oracle.partition(cost * a, n)
        assert np.array_equal(b1, b2) and B2 == a * B1
        assert d1 == pytest.approx(d2, rel=1e-12)


def test_imbalance_output_matches_eq():
    """Pin: eq:imbalance evaluated with numpy on the oracle's own split."""
    g = np.random.default_rng(21)
    for _ in range(300):
        L = int(g.integers(2, 40))
        n = int(g.integers(1, min(8, L) + 1))
        cost = g.integers(0, 100, L)
        st, b, B, imb = oracle.partition(cost, n)
        x = np.add.reduceat(cost, b[:-1]) if L else np.zeros(n)
        want = 0.0 if x.sum() == 0 else (x.max() - x.min()) / (x.sum() / n)
        assert imb == pytest.approx(want, rel=1e-14)


# -------------------------------------------------------------------- O5 repack
def test_repack_bound_vs_bruteforce():
    """Pin: brute-force minimal k over all splits for k <= n_cur (config 1)."""
    unmet = 0
    for inst in synth.cfg1_instances(300, seed_key=1):
        cost, mem, cap, bound = inst["cost"], inst["mem"], inst["cap"], inst["bound"]
        st, k, b, B = oracle.repack_bound(cost, 4, bound, 1, mem=mem, cap=cap)
        kb = brute.repack_min_workers(cost, 4, bound, 1, mem, cap)
        if kb is None:
            Bn, bn = brute.partition(cost, 4, mem, cap)
            if Bn is None:
                assert st == oracle.E_INFEASIBLE
            else:
                assert st == oracle.W_BOUND_UNMET and k == 4 and B == Bn
                assert np.array_equal(b, bn)
                unmet += 1
        else:
            Bk, bk = brute.partition(cost, kb, mem, cap)
            assert st == 0 and k == kb and B == Bk <= bound
            assert np.array_equal(b[:k + 1], bk) and np.all(b[k + 1:] == -1)


def test_repack_bound_monotone_and_certificate():
    """Pin: n' non-increasing as the bound grows; certificate B*(n'-1) > bound."""
    g = np.random.default_rng(17)
    for _ in range(200):
        L = int(g.integers(2, 20))
        cost = g.integers(0, 20, L)
        n_cur = int(g.integers(1, min(8, L) + 1))
        prev = None
        for bound in sorted(set(int(v) for v in g.integers(0, int(cost.sum()) + 2, 8))):
            st, k, b, B = oracle.repack_bound(cost, n_cur, bound, 1)
            if st == 0:
                assert B <= bound
                if k > 1:
                    st2, _, Bp, _ = oracle.partition(cost, k - 1)
                    assert Bp > bound
                if prev is not None:
                    assert k <= prev
                prev = k
    assert oracle.repack_bound([1, 1], 2, 5, 3)[0] == oracle.E_INVALID  # floor > n_cur


def test_alg2_spec_traces():
    """Pin: SPEC.md:L367-369 traces + reading Q14 trace (one layer per worker)."""
    for ex in GOLD["alg2"]:
        wm = ex["worker_mem"]
        n = len(wm)
        cost = np.ones(n, np.int64)
        st, k, b, B = oracle.repack_alg2(cost, np.arange(n + 1), ex["target"],
                                         mem=np.array(wm), cap=ex["max_mem"] - 1)
        assert (st, k) == (ex["status"], ex["n_new"]), ex["cite"]
    # Q14 trace: layers of workers 0,1,2 all end on worker 3
    st, k, b, B = oracle.repack_alg2(np.ones(4), [0, 1, 2, 3, 4], 1, mem=np.full(4, 10), cap=79)
    assert list(b[:2]) == [0, 4] and B == 4


def test_alg2_memory_safety_and_conservation():
    """Pin: S:L383 memory cap on every transfer prefix; layers conserved."""
    g = np.random.default_rng(23)
    for _ in range(1000):
        L = int(g.integers(1, 40))
        n = int(g.integers(1, min(8, L) + 1))
        inner = np.sort(g.choice(np.arange(1, L), n - 1, replace=False)) if n > 1 else []
        bnd = np.concatenate([[0], inner, [L]]).astype(np.int32)
        mem = g.integers(0, 30, L)
        cap = int(g.integers(0, 200))
        target = int(g.integers(1, n + 1))
        st, k, b, B = oracle.repack_alg2(np.ones(L), bnd, target, mem=mem, cap=cap)
        assert st in (0, oracle.W_BOUND_UNMET)
        assert k >= target and b[0] == 0 and b[k] == L and np.all(np.diff(b[:k + 1]) > 0)
        assert (st == 0) == (k == target)
        # each merged run is a union of whole input stages (contiguous chain)
        assert set(b[:k + 1]).issubset(set(bnd))
        # every merged worker that absorbed others satisfies the cap
        for s in range(k):
            seg = mem[b[s]:b[s + 1]].sum()
            n_in = sum(1 for x in bnd if b[s] < x < b[s + 1])
            if n_in > 0:
                assert seg <= cap
        # replay: every prefix of merges is under the cap (first-fit order)
        mu = [int(mem[bnd[s]:bnd[s + 1]].sum()) for s in range(n)]
        active = [True] * n
        for src in range(n - 1):
            if active[src] and mu[src] + mu[src + 1] <= cap and sum(active) > target:
                active[src] = False
                mu[src + 1] += mu[src]
                mu[src] = 0
                assert mu[src + 1] <= cap
        assert sum(active) == k


# ----------------------------------------------------------------- O6 diffusion
def test_diffusion_spec_traces():
    """Pin: SPEC.md:L281-283 / L291-292 hand traces."""
    for ex in GOLD["diffusion"]:
        st, b, r, ph, ph0 = oracle.diffuse(ex["cost"], ex["bnd_in"], ex["gamma"], 64,
                                           mem=ex.get("mem"), cap=ex.get("cap", 0))
        assert st == 0 and list(b) == ex["bnd_out"] and r == ex["rounds"], ex["cite"]
        assert ph0 == ex["phi0"] and ph == ex["phi"], ex["cite"]


def test_diffusion_known_gap_counterexample():
    """Pin: [7,7,8,7], n=3, start [7|7|8,7] is a pairwise-local optimum at 15
    while B* = 14 (SURVEY O6 'known gap'): diffusion must not claim B*."""
    st, b, r, ph, _ = oracle.diffuse([7, 7, 8, 7], [0, 1, 2, 4], 0, 64)
    assert st == 0 and r == 0 and list(b) == [0, 1, 2, 4]
    assert oracle.partition([7, 7, 8, 7], 3)[2] == 14


def _trajectory(cost, bnd, mem=None, cap=0, maxr=200):
    states = []
    for r in range(maxr + 1):
        st, b, rr, ph, _ = oracle.diffuse(cost, bnd, 0, r, mem=mem, cap=cap)
        states.append((st, b.copy(), rr, ph))
        if st == 0:
            break
    return states


def test_diffusion_invariants():
    """Pin: phi and max load never increase; sum conserved; every state
    respects mem; at termination no edge is improvable (brute check of all
    re-splits of every adjacent pair); final max >= B* (S:L316-322)."""
    g = np.random.default_rng(31)
    gaps = 0
    for it in range(300):
        L = int(g.integers(2, 25))
        n = int(g.integers(2, min(8, L) + 1))
        cost = g.integers(0, 20, L)
        mem = cap = None
        if it % 2:
            mem = g.integers(0, 10, L)
            cap = int(max(mem.max(), int(mem.sum()) // n + int(g.integers(0, 10))))
        # start from a mem-feasible-or-not uniform split
        bnd = np.rint(np.linspace(0, L, n + 1)).astype(np.int32)
        traj = _trajectory(cost, bnd, mem, cap or 0)
        prev_phi, prev_max = None, None
        init_ok = mem is None or all(mem[bnd[s]:bnd[s + 1]].sum() <= cap for s in range(n))
        for st, b, r, ph in traj:
            x = oracle.stage_loads(cost, b)
            assert x.sum() == cost.sum()
            if prev_phi is not None:
                assert ph <= prev_phi and x.max() <= prev_max
            prev_phi, prev_max = ph, x.max()
            if mem is not None and init_ok:
                assert all(mem[b[s]:b[s + 1]].sum() <= cap for s in range(n))
        st, b, r, ph = traj[-1]
        assert st == 0
        x = oracle.stage_loads(cost, b)
        P = np.concatenate([[0], np.cumsum(cost)])
        M = np.concatenate([[0], np.cumsum(mem)]) if mem is not None else None
        for e in range(n - 1):
            lo, hi = b[e], b[e + 2]
            for j in range(lo + 1, hi):
                if M is not None and (M[j] - M[lo] > cap or M[hi] - M[j] > cap):
                    continue
                assert max(P[j] - P[lo], P[hi] - P[j]) >= max(x[e], x[e + 1])
        Bs = oracle.partition(cost, n, mem=mem, cap=cap or 0)[2]
        final_ok = mem is None or all(mem[b[s]:b[s + 1]].sum() <= cap for s in range(n))
        if Bs >= 0 and final_ok:  # B* bounds every mem-feasible split
            assert x.max() >= Bs
            gaps += x.max() > Bs
    assert gaps > 0  # the heuristic is not always optimal (reported, never hidden)


def test_diffusion_not_converged_and_invalid():
    cost = list(range(1, 33))
    st, b, r, ph, ph0 = oracle.diffuse(cost, np.arange(0, 33, 4), 0, 1)
    assert st == oracle.W_NOT_CONVERGED and r == 1 and ph < ph0
    assert oracle.diffuse([1, 2, 3], [0, 2, 2, 3], 0, 5)[0] == oracle.E_INVALID  # empty stage
    assert oracle.diffuse([1, 2, 3], [0, 1, 3], -1, 5)[0] == oracle.E_INVALID


def test_fluid_closed_forms_and_bound():
    """Pins: n=2 converges in exactly 1 round to the mean (closed form); the
    limit is the mean within gamma; phi_f non-increasing; sum conserved;
    rounds <= s_con = 60 n^2 ln(2n) ln(S n^2 / gamma) (reading Q11)."""
    st, x, r, ph = oracle.diffuse_fluid([6, 2], [0, 1, 2], 0.0, 10)
    assert st == 0 and r == 1 and list(x) == [4.0, 4.0] and ph == 0.0
    g = np.random.default_rng(41)
    worst = 0.0
    for _ in range(400):
        L = int(g.integers(2, 40))
        n = int(g.integers(2, min(8, L) + 1))
        cost = g.integers(1, 1000, L)
        bnd = np.rint(np.linspace(0, L, n + 1)).astype(np.int32)
        x0 = oracle.stage_loads(cost, bnd).astype(float)
        phi0 = oracle.phi_f64(x0)
        if phi0 == 0:
            continue
        gamma = 1e-9 * phi0
        st, x, r, ph = oracle.diffuse_fluid(cost, bnd, gamma, 100000)
        assert st == 0 and ph <= gamma
        mean = x0.sum() / n
        assert np.all(np.abs(x - mean) <= gamma + 1e-9 * mean)
        assert x.sum() == pytest.approx(x0.sum(), rel=1e-12)
        S = x0.max() - x0.min()
        s_con = 60 * n * n * math.log(2 * n) * math.log(S * n * n / gamma)
        assert r <= s_con
        worst = max(worst, r / s_con)
        prev = None
        for rr in range(0, r + 1):
            _, _, _, p = oracle.diffuse_fluid(cost, bnd, gamma, rr)
            if prev is not None:
                assert p <= prev
            prev = p
    assert worst < 0.01


# ------------------------------------------------------------------ O7 moves
def test_moves_vs_owner_map():
    """Pin: owner map via np.repeat (vectorised) vs the oracle's interval search."""
    g = np.random.default_rng(51)
    for _ in range(300):
        L = int(g.integers(1, 64))
        no = int(g.integers(1, min(8, L) + 1))
        nn = int(g.integers(1, min(8, L) + 1))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), no - 1, replace=False)), [L]]) if no > 1 else np.array([0, L])
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), nn - 1, replace=False)), [L]]) if nn > 1 else np.array([0, L])
        G = int(g.integers(1, 9))
        ro = (np.arange(no) * G) // no
        rn = (np.arange(nn) * G) // nn
        own_o = np.repeat(ro, np.diff(bo))
        own_n = np.repeat(rn, np.diff(bn))
        want = np.nonzero(own_o != own_n)[0]
        mv = oracle.moves(L, bo, ro, bn, rn)
        assert np.array_equal(mv[:, 0], want)
        assert np.array_equal(mv[:, 1], own_o[want]) and np.array_equal(mv[:, 2], own_n[want])


def test_sparsity_schedule_milestones():
    """Pin: Eq. 3 milestones 52/79/90% (reading Q17)."""
    for ex in GOLD["sparsity_schedule"]:
        assert synth.sparsity_at(ex["t"]) == pytest.approx(ex["S"], abs=1e-12), ex["cite"]


# ------------------------------------------------------ O8 global pruning
def test_global_prune_spec_examples():
    """Alg. 1: SPEC S:L181-183 worked examples; k from line 2."""
    for ex in GOLD["global_prune"]:
        n = sum(len(x) for x in ex["shards"])
        assert int(math.floor(n * (1 - ex["sparsity"]))) == ex["k"], ex["cite"]
        st, masks = oracle.global_prune([np.array(x, np.float64) for x in ex["shards"]], ex["k"])
        assert st == 0
        assert [list(np.flatnonzero(m)) for m in masks] == ex["keep"], ex["cite"]


def test_global_prune_vs_lexsort_and_separation():
    """Kept set = first k of an independent ranking (np.lexsort by |w| desc,
    position asc) on tie-heavy data; exactly k kept; every kept magnitude >=
    every pruned one; f32 and bf16 shards mixed; NaN never kept -> INVALID."""
    g = np.random.default_rng(8)
    for _ in range(60):
        shards = []
        for _ in range(int(g.integers(1, 5))):
            n = int(g.integers(0, 300))
            if g.random() < 0.5:
                shards.append((g.integers(-8, 9, n) * 0.25).astype(np.float32).astype(np.float64))  # ties, +-0
            else:
                bits = g.integers(0, 2 ** 16, n).astype(np.uint16)
                bits[(bits & 0x7F80) == 0x7F80] = 0  # no inf/NaN here
                shards.append(oracle.bf16_to_f64(bits))
        w = np.concatenate(shards) if shards else np.zeros(0)
        k = int(g.integers(0, w.size + 1))
        st, masks = oracle.global_prune(shards, k)
        m = np.concatenate(masks) if masks else np.zeros(0, np.uint8)
        assert st == 0 and int(m.sum()) == k
        order = np.lexsort((np.arange(w.size), -np.abs(w)))
        want = np.zeros(w.size, np.uint8)
        want[order[:k]] = 1
        assert np.array_equal(m, want)
        if 0 < k < w.size:
            assert np.abs(w[m == 1]).min() >= np.abs(w[m == 0]).max()
    st, masks = oracle.global_prune([np.array([1.0, np.nan, -3.0])], 1)
    assert st == oracle.E_INVALID and list(masks[0]) == [0, 0, 1]
    assert oracle.global_prune([np.array([1.0, 2.0])], 3)[0] == oracle.E_INVALID
    assert list(oracle.bf16_to_f64(np.array([0x3F80, 0xBF80, 0x8000, 0x4049], np.uint16))) == [1.0, -1.0, -0.0, 3.140625]


# ----------------------------------------- O9 stage -> rank map (NEXT-3)
def test_map_stages_vs_bruteforce():
    """Reading Q23: the map keeping the most bytes in place, the
    lexicographically smallest among optima == brute force over every
    injective map (itertools.permutations enumerates them in lexicographic
    order); small byte alphabet so optima tie often; allowed-rank masks;
    INFEASIBLE when n_new > |allowed|; INVALID on a malformed split."""
    import itertools
    g = np.random.default_rng(23)
    for _ in range(400):
        G = int(g.integers(1, 7))
        L = int(g.integers(2, 13))
        n_old = int(g.integers(1, min(L, 6) + 1))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_old - 1, replace=False)), [L]]).astype(np.int32)
        ro = g.integers(0, G, n_old).astype(np.int32)
        allowed = int(g.integers(1, 1 << G))
        n_new = int(g.integers(1, min(L, 6) + 1))
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)), [L]]).astype(np.int32)
        nb = g.integers(0, 4, L).astype(np.int64)
        st, rn, kept = oracle.map_stages(L, bo, ro, bn, nb, G, allowed)
        ranks = [r for r in range(G) if (allowed >> r) & 1]
        if n_new > len(ranks):
            assert st == oracle.E_INFEASIBLE
            continue
        owner = np.repeat(ro, np.diff(bo))
        best, best_pi = -1, None
        for pi in itertools.permutations(ranks, n_new):
            k = sum(int(nb[i]) for s in range(n_new) for i in range(bn[s], bn[s + 1]) if owner[i] == pi[s])
            if k > best:
                best, best_pi = k, pi
        assert st == 0 and kept == best and tuple(rn) == best_pi, (G, allowed, list(rn), best_pi)
    # slots: several stages per GPU (slot j on GPU slot_rank[j]); kept = bytes
    # whose new slot is on the GPU of their old slot; brute force again
    for _ in range(200):
        S = int(g.integers(2, 7))
        n_gpu = int(g.integers(1, S + 1))
        sr = np.sort(g.integers(0, n_gpu, S)).astype(np.int32)
        L = int(g.integers(S, 13))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), S - 1, replace=False)), [L]]).astype(np.int32)
        ro = np.arange(S, dtype=np.int32)  # old stage s in slot s
        n_new = int(g.integers(1, S + 1))
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)), [L]]).astype(np.int32)
        nb = g.integers(0, 4, L).astype(np.int64)
        st, rn, kept = oracle.map_stages(L, bo, ro, bn, nb, S, slot_rank=sr)
        owner_gpu = np.repeat(sr[ro], np.diff(bo))
        best, best_pi = -1, None
        for pi in itertools.permutations(range(S), n_new):
            k = sum(int(nb[i]) for s in range(n_new) for i in range(bn[s], bn[s + 1]) if owner_gpu[i] == sr[pi[s]])
            if k > best:
                best, best_pi = k, pi
        assert st == 0 and kept == best and list(rn) == [int(sr[j]) for j in best_pi]
    assert oracle.map_stages(4, [0, 2, 4], [0, 1], [0, 3, 4], [1, 1, 1, 1], 2, 0b01)[0] == oracle.E_INFEASIBLE
    assert oracle.map_stages(4, [0, 2, 5], [0, 1], [0, 3, 4], [1, 1, 1, 1], 2)[0] == oracle.E_INVALID
    assert oracle.map_stages(4, [0, 2, 4], [0, 1], [0, 3, 4], [1, 1, 1, 1], 17)[0] == oracle.E_INVALID


# ------------------------------------- O6 / O6' hand-worked traces (DESIGN 2a)
def _edge_keys_by_enumeration(cost, b, mem=None, cap=0):
    """Each edge's minimum of (pair max, |j - b|, j) by listing every j --
    used only to check the hand-written golden rows themselves."""
    P = np.concatenate([[0], np.cumsum(cost)])
    M = np.concatenate([[0], np.cumsum(mem)]) if mem is not None else None
    out = []
    for e in range(len(b) - 2):
        lo, cur, hi = b[e], b[e + 1], b[e + 2]
        keys = [(max(P[j] - P[lo], P[hi] - P[j]), abs(j - cur), j) for j in range(lo + 1, hi)
                if M is None or (M[j] - M[lo] <= cap and M[hi] - M[j] <= cap)]
        out.append(min(keys) if keys else None)
    return out


@pytest.mark.parametrize("ex", GOLD["diffusion_traces"], ids=lambda e: e["name"][:2])
def test_diffusion_hand_traces(ex):
    """Pin: hand-worked discrete-diffusion traces, n = 3-5
    (DESIGN.md 2a): equal-gap tie -> lower edge (D1, D5), largest gap beats a
    smaller improvable gap (D2), non-mutual picks (D1, D2, D5), the secondary
    key |j - b| on both sides of b (D3, D4), two matched edges in one round
    (D5), a memory cap excluding the cost-optimal re-split (D6).  The oracle
    is stopped after every round (max_rounds = r) and its split compared with
    the hand trace."""
    cost, mem, cap = ex["cost"], ex.get("mem"), ex.get("cap", 0)
    b = list(ex["bnd_in"])
    for r, row in enumerate(ex["rounds"]):
        x = oracle.stage_loads(cost, b)
        assert list(x) == row["x"], (ex["name"], r)
        assert oracle.phi(x) == (0, row["phi"]), (ex["name"], r)
        if row["edges"] is not None:  # the golden row itself, by enumeration
            keys = _edge_keys_by_enumeration(cost, b, mem, cap)
            for e, (k, ge) in enumerate(zip(keys, row["edges"])):
                assert (k[2], k[0]) == (ge["best_j"], ge["best_max"]), (ex["name"], r, e)
                assert (k[0] < max(x[e], x[e + 1])) == ge["improvable"], (ex["name"], r, e)
        st, bo, rr, ph, ph0 = oracle.diffuse(cost, ex["bnd_in"], ex["gamma"], r, mem=mem, cap=cap)
        assert list(bo) == b and rr == r and ph == row["phi"] and ph0 == ex["phi0"], (ex["name"], r)
        if row["bnd_after"] is None:
            assert st == oracle.OK
            break
        assert st == oracle.W_NOT_CONVERGED
        b = row["bnd_after"]
    st, bo, rr, ph, ph0 = oracle.diffuse(cost, ex["bnd_in"], ex["gamma"], 64, mem=mem, cap=cap)
    assert st == oracle.OK and list(bo) == ex["bnd_out"] and rr == ex["n_rounds"]
    assert ph == ex["phi"] and ph0 == ex["phi0"]


@pytest.mark.parametrize("ex", GOLD["fluid_traces"], ids=lambda e: e["name"][:2])
def test_fluid_hand_traces(ex):
    """Pin: hand-worked fluid traces (n = 3 and 4): x and phi_f
    after every round (all values dyadic, so exact), stop at phi_f <= gamma_f."""
    for r, (xr, pr) in enumerate(zip(ex["x_after"], ex["phi_after"])):
        st, x, rr, ph = oracle.diffuse_fluid(ex["cost"], ex["bnd_in"], ex["gamma_f"], r)
        assert list(x) == xr and ph == pr and rr == r, (ex["name"], r)
        assert st == (oracle.OK if r == ex["n_rounds"] else oracle.W_NOT_CONVERGED)
    st, x, rr, ph = oracle.diffuse_fluid(ex["cost"], ex["bnd_in"], ex["gamma_f"], 1000)
    assert st == oracle.OK and rr == ex["n_rounds"] and list(x) == ex["x_after"][-1]


def test_map_stages_vs_assignment_solver():
    """Pin (independent of the subset DP): the kept bytes of
    the O9 map equal the optimum of the rectangular assignment problem
    w[s][g] (scipy's linear_sum_assignment, a Jonker-Volgenant solver) up to
    G = 16; the returned map is injective, uses allowed ranks only and attains
    that optimum; for G <= 8 brute force over every injective map in
    lexicographic order pins the tie-break."""
    import itertools
    from scipy.optimize import linear_sum_assignment
    g = np.random.default_rng(1606)
    for it in range(300):
        G = int(g.integers(1, 17))
        L = int(g.integers(max(2, G), 64))
        n_old = int(g.integers(1, min(L, G) + 1))
        bo = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_old - 1, replace=False)), [L]]).astype(np.int32)
        ro = g.choice(G, n_old, replace=False).astype(np.int32)
        allowed = (1 << G) - 1 if it % 3 else int(g.integers(1, 1 << G))
        ranks = [r for r in range(G) if (allowed >> r) & 1]
        n_new = int(g.integers(1, min(L, len(ranks)) + 1))
        bn = np.concatenate([[0], np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)), [L]]).astype(np.int32)
        nb = g.integers(0, 5 if it % 2 else 1 << 20, L).astype(np.int64)
        st, rn, kept = oracle.map_stages(L, bo, ro, bn, nb, G, allowed)
        assert st == 0
        owner = np.repeat(ro, np.diff(bo))
        new_stage = np.repeat(np.arange(n_new), np.diff(bn))
        w = np.zeros((n_new, G), np.int64)
        np.add.at(w, (new_stage, owner), nb)
        wa = w[:, ranks]
        rows, cols = linear_sum_assignment(wa, maximize=True)
        assert kept == int(wa[rows, cols].sum()), (G, n_new)
        rn = [int(v) for v in rn]
        assert len(set(rn)) == n_new and all((allowed >> r) & 1 for r in rn)
        assert int(sum(w[s, rn[s]] for s in range(n_new))) == kept
        if G <= 8:
            best = max(sum(int(w[s, pi[s]]) for s in range(n_new)) for pi in itertools.permutations(ranks, n_new))
            first = next(pi for pi in itertools.permutations(ranks, n_new)
                         if sum(int(w[s, pi[s]]) for s in range(n_new)) == best)
            assert tuple(rn) == first

// k_solve.cu -- batched rebalancing solvers on sm_100a.
//
// One instance = one CTA of ONE warp (32 threads): the solvers are latency
// bound (dependent shared-memory lookups, tiny arithmetic), so barriers
// between warps only add waiting; a single warp needs only __syncwarp, and a
// batch of 4096 instances is a single wave of warps over the 148 SMs.
// Prefix sums, boundaries and scratch live in dynamic shared memory sized
// from max_layers.
//
//  k_partition  contiguous min-max partition:
//               exact integer (T+1)-ary search over the bottleneck B: each of
//               the T threads (256 per instance in the latency mode, 32 in
//               the batched mode) tests its own candidate with its own greedy
//               stage count (a broadcast scan of the prefix sums, or binary
//               lifting for long models; memory cap folded in), ballots pick
//               the sub-interval.  Canonical lexmax boundaries (reading Q7),
//               fp64 Delta L (eq:imbalance).
//  k_diffuse    blockIdx.y = 0: discrete diffusion (P:L497, P:L518-549,
//               reading Q10), lane = stage pair; blockIdx.y = 1: the fluid
//               process of Lemma 2's proof, register-resident rounds on lane
//               0 and phi of 32 rounds at a time on the 32 lanes.
//  k_repack     fewest workers within the throughput bound (P:L13, P:L556-
//               609): one greedy count at B = bound then the partition; or
//               Alg. 2 first-fit (P:L562-593 with SPEC:L389 fixes).
#include <cuda_runtime.h>

#include <cstdint>

#include "dynmo_internal.h"

namespace dynmo {

#ifdef DYNMO_STEP_STAMPS
__device__ unsigned long long g_step_stamp[STAMP_N][2];
#endif
void diag_stamps_solve(unsigned long long *h, bool reset) {
#ifdef DYNMO_STEP_STAMPS
    cudaMemcpyFromSymbol(h, g_step_stamp, sizeof(unsigned long long) * STAMP_N * 2);
    if (reset) {
        unsigned long long z[STAMP_N][2];
        for (int i = 0; i < STAMP_N; ++i) {
            z[i][0] = ~0ull;
            z[i][1] = 0ull;
        }
        cudaMemcpyToSymbol(g_step_stamp, z, sizeof(z));
    }
#else
    (void)h;
    (void)reset;
#endif
}

namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int64_t I64MAX = INT64_MAX;
constexpr int kChunk = 32;  // fluid rounds advanced per phi evaluation pass
constexpr int kRow = 33;    // padded history row (doubles): lanes read rows conflict-free

__device__ __forceinline__ int64_t satadd(int64_t a, int64_t b) {  // a, b >= 0
    return b > I64MAX - a ? I64MAX : a + b;
}

// Per-instance shared state (dynamic shared memory of the one-warp CTA).
struct Inst {
    int64_t *P;      // [L+1] prefix sums of cost (P[k] = sum_{i<k} c_i)
    int64_t *M;      // [L+1] prefix sums of mem (MEM only)
    int64_t *x;      // [L+1] stage loads (or fp64 fluid scratch)
    int32_t *b;      // [L+1] working boundaries
    int32_t *tgt;    // [L+1] per edge: best split, -1 if not improvable
    int32_t *pick;   // [L+1] per stage: picked edge
    int16_t *nxt;    // [L+1] jump table
    int L;
    int64_t cap, maxc;
    bool mfit;  // every m_i <= cap (MEM)
};

__host__ __device__ __forceinline__ size_t base_bytes(int Lmax, bool mem) {
    const size_t Lc = (size_t)Lmax + 1;
    const size_t raw = 8 * Lc + (mem ? 8 * Lc : 0) + 8 * Lc + 3 * 4 * Lc + 2 * Lc;
    return (raw + 15) & ~(size_t)15;  // the fluid history (fp64) follows
}

__host__ __device__ __forceinline__ size_t solve_smem_bytes(int Lmax, bool mem, bool fluid) {
    // fluid history: two buffers of kChunk rows (fluid_overlap verifies one
    // while it fills the other)
    return base_bytes(Lmax, mem) + (fluid ? sizeof(double) * (2 * kChunk * kRow + kChunk) : 0);
}

__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

__device__ Inst carve(char *sm, int Lmax, bool mem) {
    DYNMO_DCHECK(base_bytes(Lmax, mem) <= dyn_smem_bytes());
    Inst s;
    const size_t Lc = (size_t)Lmax + 1;
    size_t o = 0;
    s.P = (int64_t *)(sm + o); o += 8 * Lc;
    s.M = (int64_t *)(sm + o); o += mem ? 8 * Lc : 0;
    s.x = (int64_t *)(sm + o); o += 8 * Lc;
    s.b = (int32_t *)(sm + o); o += 4 * Lc;
    s.tgt = (int32_t *)(sm + o); o += 4 * Lc;
    s.pick = (int32_t *)(sm + o); o += 4 * Lc;
    s.nxt = (int16_t *)(sm + o);
    s.L = 0;
    s.cap = 0;
    s.maxc = 0;
    s.mfit = true;
    return s;
}

// ------------------------------------------------------------ prefix sums
struct PrefixFlags {
    bool cneg, covf, mneg, movf;
};

// (out of line and rolled: runs only when a prefix saturated, and the solver
// kernels are instruction-fetch bound when cold, so their code stays small)
__device__ __noinline__ bool exact_sum_overflows(const int64_t *v, int L) {
    __int128 acc = 0;
#pragma unroll 1
    for (int i = 0; i < L; ++i) acc += v[i];
    return acc > (__int128)I64MAX;
}

// Warp-wide prefix of v[0..L) into out[0..L] (out[0] = 0), saturating at
// INT64_MAX; blocked layout, ceil(L/32) values per lane.
__device__ void warp_prefix(const int64_t *v, int L, int64_t *out, int lane) {
    const int Q = (L + 31) / 32;
    const int beg = lane * Q, end = beg + Q < L ? beg + Q : L;
    int64_t sum = 0;
#pragma unroll 1
    for (int i = beg; i < end; ++i) sum = satadd(sum, v[i]);
    int64_t ex = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(FULL, ex, o);
        if (lane >= o) ex = satadd(ex, t);
    }
    ex = __shfl_up_sync(FULL, ex, 1);
    if (lane == 0) {
        ex = 0;
        out[0] = 0;
    }
#pragma unroll 1
    for (int i = beg; i < end; ++i) {
        ex = satadd(ex, v[i]);
        out[i + 1] = ex;
    }
    __syncwarp();
}

// Negative entries (checked before the sums, like the oracle) and exact
// overflow of each array; fills s.P (and s.M), s.maxc, s.L.
__device__ PrefixFlags load_prefix(Inst &s, const int64_t *cost, const int64_t *mem, int L, int lane) {
    PrefixFlags f{false, false, false, false};
    int cneg = 0, mneg = 0;
    int64_t mx = 0;
    int mbig = 0;
#pragma unroll 1
    for (int i = lane; i < L; i += 32) {
        const int64_t c = cost[i];
        cneg |= c < 0;
        mx = c > mx ? c : mx;
        if (mem) {
            const int64_t m = mem[i];
            mneg |= m < 0;
            mbig |= m > s.cap;
        }
    }
    f.cneg = __any_sync(FULL, cneg);
    f.mneg = __any_sync(FULL, mneg);
    s.mfit = !__any_sync(FULL, mbig);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t t = __shfl_xor_sync(FULL, mx, o);
        mx = t > mx ? t : mx;
    }
    s.maxc = mx;
    s.L = L;
    if (f.cneg || f.mneg) return f;
    warp_prefix(cost, L, s.P, lane);
    if (mem) warp_prefix(mem, L, s.M, lane);
    // a saturated prefix reads INT64_MAX: decide the overflow exactly
    int fl = 0;
    if (lane == 0) {
        if (s.P[L] == I64MAX && exact_sum_overflows(cost, L)) fl |= 1;
        if (mem && s.M[L] == I64MAX && exact_sum_overflows(mem, L)) fl |= 2;
    }
    fl = __shfl_sync(FULL, fl, 0);
    f.covf = (fl & 1) != 0;
    f.movf = (fl & 2) != 0;
    return f;
}

// Oracle order (build_prefix of cost, then of mem): first error wins.
__device__ __forceinline__ int prefix_status(const PrefixFlags &f, bool use_mem) {
    if (f.cneg) return DYNMO_E_INVALID;
    if (f.covf) return DYNMO_E_OVERFLOW;
    if (use_mem && f.mneg) return DYNMO_E_INVALID;
    if (use_mem && f.movf) return DYNMO_E_OVERFLOW;
    return DYNMO_OK;
}

// --------------------------------------------------------------- greedy
// Warp-cooperative greedy jump: the largest K >= j with P[K] - P[j] <= B and
// M[K] - M[j] <= cap (t1 = P[j] + B, t2 = M[j] + cap).  Both predicates are
// monotone in K, so the 32-position window test below yields a ballot that
// is a prefix of ones: its popcount is the jump length (one shared load and
// one 64-bit compare per lane per 32 positions).  K == j: layer j does not fit.
template <bool MEM>
__device__ __forceinline__ int warp_jump(const Inst &s, int j, int64_t t1, int64_t t2, int lane) {
    int K = j;
    for (;;) {
        const int p = K + 1 + lane;
        bool ok = p <= s.L && s.P[p] <= t1;
        if constexpr (MEM) ok = ok && s.M[p] <= t2;
        const int c = __popc(__ballot_sync(FULL, ok));
        K += c;
        if (c < 32) return K;
    }
}

// ------------------------------------------- one candidate per thread
// The feasibility test of the search runs on every THREAD with its own
// candidate B (instead of one warp per candidate), so a CTA of 256 threads
// tests 256 candidates per round and a one-warp instance 32.  Two exact
// greedy counts (maximal prefix stages, reading Q8/Q9), chosen per instance:
//  scan_count   one pass over the layers: the shared loads of P[i] are the
//               same address for every lane (broadcast, no bank conflict)
//               and independent of the data, so they pipeline; the
//               dependent chain per layer is a compare and a select.
//  jump_count   per stage, binary lifting over P (log2 L dependent loads):
//               fewer instructions when n log2(L) << L.
// The memory cap does not depend on B: reach[j] = the largest K with
// M[K] - M[j] <= cap is computed once per instance (binary searches over M,
// in the 16-bit table Inst::nxt), and a stage starting at j ends at
// min(cost reach(j, B), reach[j]) -- one index compare instead of 64-bit
// loads and compares of M in every step.  Both counts assume every layer
// fits a stage alone (B >= max c, every m <= cap), which the search
// establishes before the first round.  A count above `limit` may be reported
// as any value > limit.
// Arithmetic: unsigned, no saturation needed (every P, B <= C <= INT64_MAX,
// so P + B fits in uint64_t); when C < 2^31 the same sums fit in uint32_t:
// half the registers and compare instructions (the 32-bit copy of P lives in
// Inst::x, unused by the partition and the repack).
template <typename T>
struct View {
    const T *P;
    const int16_t *reach;  // MEM only
    int L;
};

template <typename T, bool MEM>
__device__ __forceinline__ int scan_count(const View<T> &v, T B) {
    T t1 = B;                            // P[start] + B with start = 0
    int lim = MEM ? v.reach[0] : v.L;    // reach[start]
    int c = 1;
#pragma unroll 4
    for (int i = 1; i <= v.L; ++i) {
        // layer i-1 joins the open stage iff P[i] <= t1 and i <= reach[start];
        // else it opens the next stage (it fits alone)
        bool cut = v.P[i] > t1;
        if constexpr (MEM) cut |= i > lim;
        const T n1 = v.P[i - 1] + B;
        t1 = cut ? n1 : t1;
        if constexpr (MEM) {
            const int nl = v.reach[i - 1];
            lim = cut ? nl : lim;
        }
        c += cut;
    }
    return c;
}

template <typename T, bool MEM>
__device__ __forceinline__ int jump_count(const View<T> &v, T B, int limit) {
    const int L = v.L;
    const int top = 1 << (31 - __clz(L));
    int j = 0, c = 0;
    while (j < L && c <= limit) {
        const T t1 = v.P[j] + B;
        int K = j;
        for (int step = top; step > 0; step >>= 1) {
            const int k2 = K + step;
            const int kc = k2 <= L ? k2 : L;  // branch-free: clamped load
            K = ((k2 <= L) & (v.P[kc] <= t1)) ? k2 : K;
        }
        if constexpr (MEM) {
            const int r = v.reach[j];
            K = K < r ? K : r;
        }
        j = K;  // K > j: layer j fits alone
        ++c;
    }
    return j < L ? limit + 1 : c;
}

template <typename T, bool MEM>
__device__ __forceinline__ int thread_count(const View<T> &v, int64_t B, int limit, bool jumps) {
    return jumps ? jump_count<T, MEM>(v, (T)B, limit) : scan_count<T, MEM>(v, (T)B);
}

// Memory reach of every start j (MEM): the largest K in [j, L] with
// M[K] - M[j] <= cap (M is nondecreasing), by binary lifting; all threads,
// then a barrier (CTA or warp).
template <int NW>
__device__ __forceinline__ void build_reach(Inst &s) {
    const int L = s.L, top = 1 << (31 - __clz(L));
    for (int j = threadIdx.x; j <= L; j += blockDim.x) {
        const int64_t t = satadd(s.M[j], s.cap);
        int K = j;
        for (int step = top; step > 0; step >>= 1) {
            const int k2 = K + step;
            const int kc = k2 <= L ? k2 : L;
            K = ((k2 <= L) & (s.M[kc] <= t)) ? k2 : K;
        }
        s.nxt[j] = (int16_t)K;
    }
    if constexpr (NW > 1) __syncthreads();
    else __syncwarp();
}

// Candidate t of NC per round: lo + floor(d (t+1) / (NC+1)) in 64-bit
// arithmetic (d = a (NC+1) + r); NC+1 is a compile-time constant (the
// division is a multiply-high).  Candidates are nondecreasing in t, < lo + d.
template <int NC1>
__device__ __forceinline__ int64_t candidate(int64_t lo, uint64_t d, int c) {
    const uint64_t qa = d / (uint64_t)NC1, qr = d % (uint64_t)NC1;
    return lo + (int64_t)(qa * (uint64_t)(c + 1) + (qr * (uint64_t)(c + 1)) / (uint64_t)NC1);
}

// Block-wide (NW warps) exclusive prefix sum of one int per thread; also the
// total.  Two barriers; s_w is a per-call scratch of NW ints.
template <int NW>
__device__ __forceinline__ int block_excl_scan(int x, int &total, int *s_w) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if constexpr (NW == 1) {
        total = __shfl_sync(FULL, incl, 31);
        return incl - x;
    } else {
        if (lane == 31) s_w[w] = incl;
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const int v = s_w[k];
            before += k < w ? v : 0;
            tot += v;
        }
        __syncthreads();  // s_w may be reused
        total = tot;
        return before + incl - x;
    }
}

// Block-wide min of one uint64 per thread (one barrier pair for NW > 1).
template <int NW>
__device__ __forceinline__ uint64_t block_min64(uint64_t x, uint64_t *s_w) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(FULL, x, o);
        x = y < x ? y : x;
    }
    if constexpr (NW == 1) {
        return x;
    } else {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 0) s_w[w] = x;
        __syncthreads();
        uint64_t m = s_w[0];
#pragma unroll
        for (int k = 1; k < NW; ++k) m = s_w[k] < m ? s_w[k] : m;
        __syncthreads();
        return m;
    }
}

// Ends of the interval sums from start i inside [lo, hi]: j in (ja, jb],
// where ja = the largest j >= i with P[j] - P[i] < lo and jb = the largest
// j >= i with P[j] - P[i] <= hi (binary lifting; P is nondecreasing).  If
// P[i] + lo overflows, no end qualifies.
__device__ __forceinline__ void sum_range(const Inst &s, int i, int64_t lo, int64_t hi, int top, int &ja, int &jb) {
    const int L = s.L;
    ja = jb = i;
    if (s.P[i] > I64MAX - lo) return;
    const int64_t a1 = s.P[i] + lo, a2 = satadd(s.P[i], hi);
    for (int step = top; step > 0; step >>= 1) {
        const int j1 = ja + step, j2 = jb + step;
        if (j1 <= L && s.P[j1] < a1) ja = j1;
        if (j2 <= L && s.P[j2] <= a2) jb = j2;
    }
}

// Exact min-max search (all threads of the NW warps, after s is built and
// visible).  B* is the largest stage sum of an optimal split, so it is one
// of the interval sums P[j] - P[i] (i < j); the search narrows [lo, hi]
// until the interval sums inside it fit one per thread, then tests exactly
// those candidates: the smallest feasible one is B*.  Narrowing rounds are
// (NT+1)-ary over the integers (every thread tests one candidate;
// feasibility is monotone in B, so the first feasible candidate is the new
// hi and its predecessor + 1 the new lo).  Bracket: lo = max(max c,
// ceil(C/n)) is a lower bound of B*, hi = min(ceil(C/n) + max c, C) is
// feasible on cost (Appendix A); under a memory cap it may not be, so the
// first narrowing round also tests hi itself and C, and if no interval sum
// in [lo, hi] is feasible the search moves to (hi, C] (C infeasible: no
// split satisfies the cap, -1).  Returns B* (uniform).
template <typename T, bool MEM, int NW>
__device__ int64_t search_t(const Inst &s, const View<T> &v, int n, int64_t lo, int64_t hi, bool jumps) {
    constexpr int NT = 32 * NW;
    __shared__ unsigned s_f[2][NW];
    __shared__ int s_wi[NW];
    __shared__ uint64_t s_w64[NW];
    __shared__ int64_t s_cand[NT];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, t = threadIdx.x;
    const int L = s.L;
    const int64_t C = s.P[L];
    const int top = 1 << (31 - __clz(L));
    bool probe = MEM;  // the first narrowing round also tests hi and C
    int par = 0;
    for (;;) {
        // outside the first round under a cap, hi is known feasible: a
        // one-point interval is the answer (its value may repeat as many
        // interval sums -- zero-cost layers -- so it is not enumerated)
        if (!probe && lo >= hi) return hi;
        // interval sums in [lo, hi]: for each start i, the ends j in [ja, jb]
        // (the one-candidate-per-thread latency mode only: with 32 threads
        // the enumeration passes cost more than the rounds they save)
        // Enumerate only when it can pay: in the 256-thread latency mode (the
        // batched mode measured slower with it: config 5's 4096 partitions
        // 32.8 vs 28.4 us), not when one integer round already
        // covers [lo, hi) (d < NT), and not when the expected number of
        // interval sums in the range (L(L+1)/2 spread over [0, C]) exceeds
        // a thread's share
        int cnt = 0, total = NT + 1;
        const double width = (double)(hi - lo) + 1.0;
        const bool try_enum = NW > 1 && hi - lo >= NT &&
                              0.5 * (double)L * (double)(L + 1) * width <= (double)NT * ((double)C + 1.0);
        if (try_enum) {
            for (int i = t; i < L; i += NT) {
                int ja, jb;
                sum_range(s, i, lo, hi, top, ja, jb);
                cnt += jb - ja;
            }
        }
        int off = 0;
        if (try_enum) off = block_excl_scan<NW>(cnt, total, s_wi);
        if (total <= NT) {
            int o = off;
            for (int i = t; i < L; i += NT) {
                int ja, jb;
                sum_range(s, i, lo, hi, top, ja, jb);
                for (int j = ja + 1; j <= jb; ++j) s_cand[o++] = s.P[j] - s.P[i];
            }
            if constexpr (NW > 1) __syncthreads();
            else __syncwarp();
            // (a candidate may be INT64_MAX itself: the "none" sentinel is
            // UINT64_MAX, outside the candidates' range)
            uint64_t mine = ~0ull;
            if (t < total) {
                const int64_t c = s_cand[t];
                if (thread_count<T, MEM>(v, c, n, jumps) <= n) mine = (uint64_t)c;
            }
            const uint64_t best = block_min64<NW>(mine, s_w64);
            if constexpr (NW == 1) __syncwarp();  // s_cand is rewritten next pass
            if (best != ~0ull) return (int64_t)best;
            // no interval sum in [lo, hi] is feasible: only under a memory
            // cap, and then B* lies in (hi, C] if C itself is feasible
            if (!MEM || hi >= C) return -1;
            if (thread_count<T, MEM>(v, C, n, jumps) > n) return -1;
            lo = hi + 1;
            hi = C;
            probe = false;  // hi = C is known feasible now
            continue;
        }
        const uint64_t d = (uint64_t)(hi - lo);
        int64_t cand;
        if (probe) cand = t < NT - 2 ? candidate<NT - 1>(lo, d, t) : (t == NT - 2 ? hi : C);
        else cand = candidate<NT + 1>(lo, d, t);
        const unsigned m = __ballot_sync(FULL, thread_count<T, MEM>(v, cand, n, jumps) <= n);
        int first;
        if constexpr (NW == 1) {
            first = m ? __ffs(m) - 1 : NT;
        } else {
            if (lane == 0) s_f[par][w] = m;
            __syncthreads();
            first = NT;
#pragma unroll
            for (int k = NW - 1; k >= 0; --k) {
                const unsigned mk = s_f[par][k];
                if (mk) first = 32 * k + __ffs(mk) - 1;
            }
            par ^= 1;  // double buffer: the next round writes the other half
        }
        if (probe) {
            probe = false;
            if (first == NT) return -1;        // C infeasible
            if (first == NT - 1) {             // only C: B* in (hi, C]
                lo = hi + 1;
                hi = C;
            } else if (first == NT - 2) {      // hi: B* in (last candidate, hi]
                lo = NT > 2 ? candidate<NT - 1>(lo, d, NT - 3) + 1 : lo;
            } else {
                const int64_t nhi = candidate<NT - 1>(lo, d, first);
                lo = first > 0 ? candidate<NT - 1>(lo, d, first - 1) + 1 : lo;
                hi = nhi;
            }
            continue;
        }
        const int64_t nhi = first < NT ? candidate<NT + 1>(lo, d, first) : hi;
        const int64_t nlo = first > 0 ? candidate<NT + 1>(lo, d, first - 1) + 1 : lo;
        hi = nhi;
        lo = nlo;
    }
}

// Per-instance choice of the count: latency mode (NW > 1, one instance per
// CTA) minimises the dependent chain (scan ~12 L cycles, jumps ~35 n log2 L);
// the batched mode (NW == 1, issue bound) minimises instructions (scan ~10 L,
// jumps ~5 n log2 L).
template <int NW>
__device__ __forceinline__ bool use_jumps(int L, int n) {
    const int lg = 32 - __clz(L);
    return NW > 1 ? L > 3 * n * lg : 2 * L > n * lg;
}

// The memory reach table (MEM), the 32-bit copy of P into s.x when C < 2^31,
// then the search.  Called by all threads (barriers inside).
template <bool MEM, int NW>
__device__ int64_t search_bottleneck(Inst &s, int n) {
    const int L = s.L;
    const int64_t C = s.P[L];
    if (MEM && !s.mfit) return -1;
    const int64_t ceil_cn = C / n + (C % n != 0);
    int64_t lo = s.maxc > ceil_cn ? s.maxc : ceil_cn;
    int64_t hi = satadd(ceil_cn, s.maxc);
    if (hi > C) hi = C;
    if (lo > hi) lo = hi;
    if (!MEM && lo == hi) return hi;
    const bool jumps = use_jumps<NW>(L, n);
    if (C < (1ll << 31)) {
        uint32_t *p32 = reinterpret_cast<uint32_t *>(s.x);
        for (int i = threadIdx.x; i <= L; i += blockDim.x) p32[i] = (uint32_t)s.P[i];
        if constexpr (MEM) build_reach<NW>(s);  // (its barrier also covers p32)
        else if constexpr (NW > 1) __syncthreads();
        else __syncwarp();
        const View<uint32_t> v{p32, s.nxt, L};
        return search_t<uint32_t, MEM, NW>(s, v, n, lo, hi, jumps);
    }
    if constexpr (MEM) build_reach<NW>(s);
    const View<uint64_t> v{reinterpret_cast<const uint64_t *>(s.P), s.nxt, L};
    return search_t<uint64_t, MEM, NW>(s, v, n, lo, hi, jumps);
}

// Greedy stage count at one B (repack's fewest workers; one warp; B >= max c
// and every m <= cap): warp-cooperative window jumps (32 positions per
// shared load, ballot = prefix of ones), stopping once the count exceeds
// `limit` (then any value > limit is returned).
template <bool MEM>
__device__ int count_at(const Inst &s, int64_t B, int limit, int lane) {
    int j = 0, c = 0;
    while (j < s.L) {
        if (c > limit) return c;
        const int64_t t1 = satadd(s.P[j], B);
        int64_t t2 = 0;
        if constexpr (MEM) t2 = satadd(s.M[j], s.cap);
        j = warp_jump<MEM>(s, j, t1, t2, lane);  // > j: layer j fits alone
        ++c;
    }
    return c;
}

// Lexmax boundaries for B* (Appendix A): b_{s+1} = min(next(b_s), L - (n-1-s))
// with warp-cooperative jumps.  One warp; writes s.b[0..n].
template <bool MEM>
__device__ void construct(Inst &s, int64_t Bs, int n, int lane) {
    int j = 0;
    if (lane == 0) s.b[0] = 0;
    for (int st = 0; st < n; ++st) {
        const int64_t t1 = satadd(s.P[j], Bs);
        int64_t t2 = 0;
        if constexpr (MEM) t2 = satadd(s.M[j], s.cap);
        const int K = warp_jump<MEM>(s, j, t1, t2, lane);
        const int reserve = s.L - (n - 1 - st);
        j = K < reserve ? K : reserve;
        if (lane == 0) s.b[st + 1] = j;
    }
    __syncwarp();
}

__device__ double imbalance_of(const int64_t *P, const int32_t *b, int n) {
    int64_t mx = P[b[1]] - P[b[0]], mn = mx;
#pragma unroll 1
    for (int st = 1; st < n; ++st) {
        const int64_t x = P[b[st + 1]] - P[b[st]];
        mx = x > mx ? x : mx;
        mn = x < mn ? x : mn;
    }
    const int64_t sum = P[b[n]];
    if (sum == 0) return 0.0;
    const double mean = __ddiv_rn((double)sum, (double)n);
    return __ddiv_rn((double)(mx - mn), mean);
}

// ------------------------------------------------------------ partition
template <bool MEM, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_partition(SolveArgs a) {
    pdl_wait();
    pdl_trigger();
    STEP_STAMP(STAMP_PARTITION);
    extern __shared__ __align__(16) char smem[];
    __shared__ int s_st, s_mfit;
    __shared__ int64_t s_maxc;
    const int q = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Inst s = carve(smem, a.max_layers, MEM);
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n = a.n_stages[q];
    int32_t *bnd = a.bnd_out + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    s.cap = cap;
    s.L = L;
    if (w == 0) {
        int st = DYNMO_OK;
        if (L < 1 || L > a.max_layers || n < 1 || n > L || (MEM && cap < 0)) st = DYNMO_E_INVALID;
        if (st == DYNMO_OK)
            st = prefix_status(load_prefix(s, a.cost + off, MEM ? a.mem + off : nullptr, L, lane), MEM);
        if (lane == 0) {  // share status, maxc and mfit with the other warps
            s_st = st;
            s_maxc = s.maxc;
            s_mfit = s.mfit;
        }
    }
    __syncthreads();
    int st = s_st;
    s.maxc = s_maxc;
    s.mfit = s_mfit != 0;
    int64_t Bs = -1;
    if (st == DYNMO_OK) {
        Bs = search_bottleneck<MEM, NW>(s, n);
        if (Bs < 0) st = DYNMO_E_INFEASIBLE;
    }
    if (w != 0) return;
    if (st != DYNMO_OK) {
        for (int k = lane; k <= n && n >= 1; k += 32) bnd[k] = -1;
        if (lane == 0) {
            a.bottleneck[q] = -1;
            if (a.imbalance) a.imbalance[q] = -1.0;
            a.status[q] = st;
        }
        return;
    }
    construct<MEM>(s, Bs, n, lane);
#pragma unroll 1
    for (int k = lane; k <= n; k += 32) bnd[k] = s.b[k];
    if (lane == 0) {
        a.bottleneck[q] = Bs;
        if (a.imbalance) a.imbalance[q] = imbalance_of(s.P, s.b, n);
        a.status[q] = DYNMO_OK;
    }
}

// -------------------------------------------------------------- repack
template <bool MEM, int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_repack(SolveArgs a) {
    pdl_wait();
    pdl_trigger();
    STEP_STAMP(STAMP_REPACK);
    extern __shared__ __align__(16) char smem[];
    __shared__ int s_st, s_k, s_code, s_mfit;
    __shared__ int64_t s_maxc;
    const int q = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Inst s = carve(smem, a.max_layers, MEM);
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n_cur = a.n_stages[q];
    const int fl = a.floor_[q];
    int32_t *bnd = a.bnd_out + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    s.cap = cap;
    s.L = L;
    const bool alg2 = a.mode == DYNMO_REPACK_ALG2;
    const int64_t bound = alg2 ? 0 : a.bound[q];
    const int32_t *bi = alg2 ? a.bnd_in + a.bnd_off[q] : nullptr;
    if (w == 0) {
        int st = DYNMO_OK;
        if (L < 1 || L > a.max_layers || n_cur < 1 || n_cur > L || fl < 1 || fl > n_cur ||
            (MEM && cap < 0) || (!alg2 && bound < 0))
            st = DYNMO_E_INVALID;
        if (st == DYNMO_OK && alg2) {
            int bad = 0;
            for (int k = lane; k < n_cur; k += 32) bad |= bi[k + 1] <= bi[k];
            bad |= bi[0] != 0 || bi[n_cur] != L;
            if (__any_sync(FULL, bad)) st = DYNMO_E_INVALID;
        }
        if (st == DYNMO_OK) {
            const PrefixFlags f = load_prefix(s, a.cost + off, MEM ? a.mem + off : nullptr, L, lane);
            if (alg2)  // oracle: negatives of cost and mem first, then the cost sum
                st = (f.cneg || f.mneg) ? DYNMO_E_INVALID : f.covf ? DYNMO_E_OVERFLOW : DYNMO_OK;
            else
                st = prefix_status(f, MEM);
        }
        int k = n_cur, code = DYNMO_OK;
        if (st == DYNMO_OK && !alg2) {
            // fewest workers: greedy count at B = bound (cost and mem), reading Q15;
            // a layer above the bound or the cap alone: no count meets it
            const int g = (bound >= s.maxc && (!MEM || s.mfit)) ? count_at<MEM>(s, bound, n_cur, lane) : n_cur + 1;
            if (g <= n_cur) {
                k = g > fl ? g : fl;
            } else {
                k = n_cur;
                code = DYNMO_W_BOUND_UNMET;
            }
        }
        if (lane == 0) {
            s_st = st;
            s_k = k;
            s_code = code;
            s_maxc = s.maxc;
            s_mfit = s.mfit;
        }
    }
    __syncthreads();
    const int st0 = s_st;
    s.maxc = s_maxc;
    s.mfit = s_mfit != 0;
    if (st0 != DYNMO_OK) {
        if (w != 0) return;
        for (int k = lane; k <= n_cur && n_cur >= 1; k += 32) bnd[k] = -1;
        if (lane == 0) {
            a.n_new[q] = -1;
            a.bottleneck[q] = -1;
            a.status[q] = st0;
        }
        return;
    }
    if (alg2) {
        if (w != 0) return;
        // Alg. 2 with the fixes of SPEC:L364/L389, serial on lane 0
        int k = 0;
        if (lane == 0) {
            const int64_t *mem = MEM ? a.mem + off : nullptr;
            __int128 mu_prev = 0;  // mem of the current chain head (src)
            int n_active = n_cur;
            if (mem)
                for (int i = bi[0]; i < bi[1]; ++i) mu_prev += mem[i];
            s.b[0] = 0;
            for (int src = 0; src + 1 < n_cur; ++src) {
                __int128 mu_dst = 0;
                if (mem)
                    for (int i = bi[src + 1]; i < bi[src + 2]; ++i) mu_dst += mem[i];
                const bool fits = !mem || (mu_prev + mu_dst <= (__int128)cap);
                if (fits && n_active > fl) {
                    n_active--;  // src deactivated, its layers merged into dst
                    mu_prev = mu_prev + mu_dst;
                } else {
                    s.b[++k] = bi[src + 1];  // src stays active
                    mu_prev = mu_dst;
                }
            }
            s.b[++k] = bi[n_cur];
            int64_t bm = 0;
            for (int t = 0; t < k; ++t) {
                const int64_t x = s.P[s.b[t + 1]] - s.P[s.b[t]];
                bm = x > bm ? x : bm;
            }
            a.n_new[q] = k;
            a.bottleneck[q] = bm;
            a.status[q] = n_active > fl ? DYNMO_W_BOUND_UNMET : DYNMO_OK;
        }
        k = __shfl_sync(FULL, k, 0);
        __syncwarp();
        for (int t = lane; t <= n_cur; t += 32) bnd[t] = t <= k ? s.b[t] : -1;
        return;
    }
    const int k = s_k;
    const int64_t Bs = search_bottleneck<MEM, NW>(s, k);
    if (w != 0) return;
    if (Bs < 0) {
        for (int t = lane; t <= n_cur; t += 32) bnd[t] = -1;
        if (lane == 0) {
            a.n_new[q] = -1;
            a.bottleneck[q] = -1;
            a.status[q] = DYNMO_E_INFEASIBLE;
        }
        return;
    }
    construct<MEM>(s, Bs, k, lane);
    for (int t = lane; t <= n_cur; t += 32) bnd[t] = t <= k ? s.b[t] : -1;
    if (lane == 0) {
        a.n_new[q] = k;
        a.bottleneck[q] = Bs;
        a.status[q] = s_code;
    }
}

// ------------------------------------------------------------- diffusion
// Discrete diffusion (reading Q10), one warp: lanes are stage pairs (edges)
// and stages; every round: loads, phi (exact, 128-bit), the best re-split of
// every adjacent pair, max-neighbor matching, simultaneous application.
template <bool MEM>
__device__ void diffuse_discrete(const SolveArgs &a, Inst &s, int q, int n, const int32_t *bi,
                                 int st, int lane) {
    int32_t *bo = a.bnd_out + a.bnd_off[q];
    const int64_t gamma = a.gamma ? a.gamma[q] : 0;
    const int maxr = a.max_rounds;
    const int64_t cap = s.cap;
    int rounds = 0;
    int64_t phi = 0, phi0 = 0;
    if (st == DYNMO_OK) {
        for (int k = lane; k <= n; k += 32) s.b[k] = bi[k];
        __syncwarp();
        int ctl = 0;  // 1 stop OK, 2 stop NOT_CONVERGED, < 0 error
        for (;;) {
            for (int t = lane; t < n; t += 32) s.x[t] = s.P[s.b[t + 1]] - s.P[s.b[t]];
            __syncwarp();
            // phi = sum_{u<v} |x_u - x_v| (reading Q12), exact in 128 bits
            __int128 acc = 0;
            for (int u = lane; u < n; u += 32) {
                const int64_t xu = s.x[u];
                for (int v = u + 1; v < n; ++v) {
                    const int64_t xv = s.x[v];
                    acc += xu > xv ? xu - xv : xv - xu;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t lo = (uint64_t)acc, hi = (uint64_t)(acc >> 64);
                const uint64_t olo = __shfl_xor_sync(FULL, lo, o);
                const uint64_t ohi = __shfl_xor_sync(FULL, hi, o);
                acc += (__int128)(((unsigned __int128)ohi << 64) | olo);
            }
            if (acc > (__int128)I64MAX) {
                ctl = DYNMO_E_OVERFLOW;
                break;
            }
            phi = (int64_t)acc;
            if (rounds == 0) phi0 = phi;
            if (phi <= gamma) {
                ctl = 1;
                break;
            }
            // best re-split of edge e: min of (pair max, |j - b|, j) over
            // mem-feasible j in (b_e, b_{e+2}).  G lanes per edge (G the
            // largest power of two with (n - 1) G <= 32), lane sub of the
            // group scans j = lo + 1 + sub, + G, ...; the group's minimum by
            // shuffles (ties on (max, dist): the lower j, as the serial scan)
            int any = 0;
            {
                // target >= 2 candidates per lane under a memory cap (its
                // test lengthens an iteration), >= 8 without: below that the
                // group reduction costs more than the shorter scan saves
                // (config 2, 48 layers / 8 stages: 10.6 -> 9.0 us with the
                // cap at G = 4; 7.2 -> 7.8 us without it at G = 4)
                const int ne = n - 1;
                const int per_lane = MEM ? 2 : 8;
                int G = 32;
                while (G > 1 && (ne * G > 32 || G * per_lane > (2 * s.L) / n)) G >>= 1;
                const int sub = lane & (G - 1);
                for (int e0 = 0; e0 < ne; e0 += 32 / G) {
                    const int e = e0 + lane / G;
                    int64_t km = I64MAX;
                    int kd = 0, kj = -1;
                    if (e < ne) {
                        const int lo = s.b[e], hi = s.b[e + 2], cur = s.b[e + 1];
                        const int64_t Plo = s.P[lo], Phi = s.P[hi];
                        int64_t Mlo = 0, Mhi = 0;
                        if constexpr (MEM) {
                            Mlo = s.M[lo];
                            Mhi = s.M[hi];
                        }
                        for (int j = lo + 1 + sub; j < hi; j += G) {
                            if constexpr (MEM)
                                if (s.M[j] - Mlo > cap || Mhi - s.M[j] > cap) continue;
                            const int64_t Pj = s.P[j];
                            const int64_t l = Pj - Plo, r = Phi - Pj;
                            const int64_t m = l > r ? l : r;
                            const int d = j > cur ? j - cur : cur - j;
                            // j ascending, so equal (max, dist) keeps the lower j
                            if (kj < 0 || m < km || (m == km && d < kd)) {
                                km = m;
                                kd = d;
                                kj = j;
                            }
                        }
                    }
                    for (int o = 1; o < G; o <<= 1) {
                        const int64_t om = __shfl_xor_sync(FULL, km, o);
                        const int od = __shfl_xor_sync(FULL, kd, o);
                        const int oj = __shfl_xor_sync(FULL, kj, o);
                        const bool take = oj >= 0 && (kj < 0 || om < km ||
                                                      (om == km && (od < kd || (od == kd && oj < kj))));
                        if (take) {
                            km = om;
                            kd = od;
                            kj = oj;
                        }
                    }
                    if (e < ne && sub == 0) {
                        const int64_t pm = s.x[e] > s.x[e + 1] ? s.x[e] : s.x[e + 1];
                        const int t = (kj >= 0 && km < pm) ? kj : -1;
                        s.tgt[e] = t;
                        any |= t >= 0;
                    }
                }
            }
            any = __any_sync(FULL, any);
            if (!any) {
                ctl = 1;
                break;
            }
            if (rounds == maxr) {
                ctl = 2;
                break;
            }
            __syncwarp();
            // max-neighbor matching: stage t picks its improvable
            // incident edge with the largest gap (ties: lower edge index)
            for (int t = lane; t < n; t += 32) {
                int pk = -1;
                int64_t best = -1;
                for (int e = t - 1; e <= t; ++e) {
                    if (e < 0 || e + 1 >= n || s.tgt[e] < 0) continue;
                    const int64_t g = s.x[e] > s.x[e + 1] ? s.x[e] - s.x[e + 1] : s.x[e + 1] - s.x[e];
                    if (g > best) {
                        best = g;
                        pk = e;
                    }
                }
                s.pick[t] = pk;
            }
            __syncwarp();
            for (int e = lane; e + 1 < n; e += 32)
                if (s.tgt[e] >= 0 && s.pick[e] == e && s.pick[e + 1] == e) s.b[e + 1] = s.tgt[e];
            __syncwarp();
            rounds++;
        }
        if (ctl < 0) st = ctl;
        else if (ctl == 2) st = DYNMO_W_NOT_CONVERGED;
    }
    if (st < 0) {
        for (int k = lane; k <= n && n >= 1; k += 32) bo[k] = -1;
        if (lane == 0) {
            if (a.rounds) a.rounds[q] = -1;
            if (a.phi) a.phi[q] = -1;
            if (a.phi0) a.phi0[q] = -1;
        }
    } else {
        for (int k = lane; k <= n; k += 32) bo[k] = s.b[k];
        if (lane == 0) {
            if (a.rounds) a.rounds[q] = rounds;
            if (a.phi) a.phi[q] = phi;
            if (a.phi0) a.phi0[q] = phi0;
        }
    }
    if (lane == 0) a.status[q] = st;
}

// Fluid process of Lemma 2's proof, exact per round, one warp
// (the A/B path, DYNMO_FLUID_SPEC=0; fluid_spec below is the default)
// with lane s holding x_s (n <= 32).  A round: each stage picks its incident
// edge with the largest gap > 0 (ties: lower edge index); mutually picked
// pairs set both ends to (x_e + x_{e+1}) * 0.5 (neighbours via shuffles).
// Speculative chunks of 1, 4, 16, 32, 32, ... rounds: the warp advances the
// chunk storing every x(r), then lane k evaluates phi_f(x(base + k)) (the
// oracle's ascending (u, v) sum); the first r with phi_f <= gamma_f, or
// r == max_rounds, stops with x(r).
// phi_f of one history row: sum over u < v of |x_u - x_v| in ascending
// (u, v) order (reading Q20).  n <= 8: the row in registers, all 28 pairs
// unrolled (absent pairs add nothing), so only the dependent adds remain on
// the critical path; the nested runtime-bound loop spent ~10x that in
// branches and reloads.  Larger n: the plain loop.
__device__ __forceinline__ double phi_row(const double *row, int n) {
    double acc = 0.0;
    if (n <= 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = u < n ? row[u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = u + 1; v < 8; ++v)
                if (v < n) acc = __dadd_rn(acc, fabs(__dsub_rn(x[u], x[v])));
        return acc;
    }
#pragma unroll 1
    for (int u = 0; u < n; ++u) {
        const double xu = row[u];
#pragma unroll 1
        for (int v = u + 1; v < n; ++v) acc = __dadd_rn(acc, fabs(__dsub_rn(xu, row[v])));
    }
    return acc;
}

__device__ void fluid_chunks(const Inst &s, int n, const int32_t *bi, double gf, int maxr,
                             double *hist, double *xo, int &rr, double &ph, int &fst, int lane) {
    double x = lane < n ? (double)(s.P[bi[lane + 1]] - s.P[bi[lane]]) : 0.0;
    int size = 1;
    for (int base = 0;; base += size, size = size < kChunk / 4 ? size * 4 : kChunk) {
        // Branch-free round: both candidate averages are computed off the
        // critical path; stage s picks its right edge iff gr > gl, else its
        // left edge iff gl > 0 (a missing edge has gap 0: the oracle's rule);
        // gaps are compared through |.| operand modifiers with the edge masks
        // folded into predicates.  Two shuffle phases (x, then the picks).
        // (A halo-2 variant deciding both edges locally from x at distance
        // 1 and 2 -- one phase of 8 shuffles -- measured slower, 24.2 vs
        // 22.8 us on config 2: the shuffle pipe, not latency, bounds it.  So
        // did all n <= 8 loads replicated in every lane, a fully unrolled
        // shuffle-free round: 39 vs 21 us at L = 127, n = 8 -- issue-bound
        // on the fp64 pipe.)
        const bool hasL = lane >= 1 && lane < n, hasR = lane + 1 < n;
        for (int k = 0; k < size; ++k) {
            if (lane < n) hist[k * kRow + lane] = x;  // x(base + k)
            const double xl = __shfl_up_sync(FULL, x, 1);
            const double xr = __shfl_down_sync(FULL, x, 1);
            const double dl = __dsub_rn(xl, x), dr = __dsub_rn(x, xr);
            const double avgL = __dmul_rn(__dadd_rn(xl, x), 0.5);
            const double avgR = __dmul_rn(__dadd_rn(x, xr), 0.5);
            const bool cRL = fabs(dr) > fabs(dl), cR0 = fabs(dr) > 0.0, cL0 = fabs(dl) > 0.0;
            const bool pR = hasR & ((hasL & cRL) | (!hasL & cR0));  // bitwise: no branches
            const bool pL = hasL & cL0;
            // the neighbours' picks from two ballots (a vote is cheaper
            // than a shuffle): bit s of bR = stage s picks its right edge,
            // of bL = stage s picks its left edge
            const bool qL = !pR & pL;
            const unsigned bR = __ballot_sync(FULL, pR);
            const unsigned bL = __ballot_sync(FULL, qL);
            const bool mR = pR & (((bL >> 1) >> lane) & 1u);       // stage s+1 picks left
            const bool mL = qL & (((bR << 1) >> lane) & 1u);       // stage s-1 picks right
            x = mR ? avgR : (mL ? avgL : x);
        }
        __syncwarp();
        const double acc = lane < size ? phi_row(hist + lane * kRow, n) : 0.0;
        const bool stop = lane < size && (acc <= gf || base + lane == maxr);
        const unsigned m = __ballot_sync(FULL, stop);
        if (m) {
            const int k = __ffs(m) - 1;
            rr = base + k;
            ph = __shfl_sync(FULL, acc, k);
            if (!(ph <= gf)) fst = DYNMO_W_NOT_CONVERGED;
            if (lane < n) xo[lane] = hist[k * kRow + lane];
            return;
        }
        __syncwarp();
    }
}

// Speculative fluid rounds (n <= 32, lane = stage).  The matching of the
// fluid process settles into a period-2 pattern (even edges, odd edges:
// config 2 repeats the matching of two rounds earlier in 254 of 256
// rounds), so most rows of a chunk are advanced with the PREDICTED matching
// (that of two rounds earlier): per round one shuffle of the partner and
// one fma on the dependent chain.  A chunk opens with `e` exact rounds after
// a misprediction (the transient before the pattern settles) and stores
// every row; then lane j recomputes row j's TRUE matching and phi_f in
// parallel.  A row whose true matching equals the one applied produced the
// next row exactly as the per-round process does; at the first mispredicted
// row the true next state is computed from it and a new chunk starts there.
// The stop rule (phi_f <= gamma_f or max_rounds) sees the valid rows only.
//
// Arithmetic identity used: for doubles x, y >= 0 (no overflow, no
// subnormal halves) fma(y, 0.5, x * 0.5) == (x + y) * 0.5 == (y + x) * 0.5
// bit for bit (halving is exact and commutes with rounding; + commutes), and
// an unmatched stage (partner = itself) gets fma(x, 0.5, x * 0.5) == x.
__device__ __forceinline__ unsigned match_bits(const double *x, int n) {
    unsigned pr = 0u, pl = 0u;  // bit t: stage t picks its right / left edge
    double dprev = 0.0;
    for (int t = 0; t < n; ++t) {
        const bool hasR = t + 1 < n, hasL = t > 0;
        const double d = hasR ? __dsub_rn(x[t], x[t + 1]) : 0.0;
        const bool cR = hasR && (hasL ? fabs(d) > fabs(dprev) : fabs(d) > 0.0);
        const bool cL = hasL && !cR && fabs(dprev) > 0.0;
        pr |= (unsigned)cR << t;
        pl |= (unsigned)cL << t;
        dprev = d;
    }
    return pr & (pl >> 1);  // edge e matched: stage e picks right, stage e+1 left
}

// True matching and phi_f of one history row.  n <= 8: the row in registers,
// every loop unrolled (as phi_row).  (A variant that skipped phi_f wherever
// the bound phi_f >= (n - 1)(max - min) exceeded gamma_f measured no faster
// on config 2 and slower at L = 127: the range chain costs what it saves.)
__device__ __forceinline__ void verify_row(const double *row, int n, unsigned &tm, double &acc) {
    if (n <= 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = u < n ? row[u] : 0.0;
        unsigned pr = 0u, pl = 0u;
        double dprev = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const bool hasR = t + 1 < n, hasL = t > 0 && t < n;
            const double d = (t + 1 < 8 && hasR) ? __dsub_rn(x[t], x[t < 7 ? t + 1 : t]) : 0.0;
            const bool cR = hasR && (hasL ? fabs(d) > fabs(dprev) : fabs(d) > 0.0);
            const bool cL = hasL && !cR && fabs(dprev) > 0.0;
            pr |= (unsigned)cR << t;
            pl |= (unsigned)cL << t;
            dprev = d;
        }
        tm = pr & (pl >> 1);
        double a = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = u + 1; v < 8; ++v)
                if (v < n) a = __dadd_rn(a, fabs(__dsub_rn(x[u], x[v])));
        acc = a;
        return;
    }
    tm = match_bits(row, n);
    acc = phi_row(row, n);
}

// One exact round (fluid_chunks' body); returns the new x, m = edge mask.
__device__ __forceinline__ double exact_round(double x, bool hasL, bool hasR, int lane, unsigned &m) {
    const double xl = __shfl_up_sync(FULL, x, 1);
    const double xr = __shfl_down_sync(FULL, x, 1);
    const double dl = __dsub_rn(xl, x), dr = __dsub_rn(x, xr);
    const double avgL = __dmul_rn(__dadd_rn(xl, x), 0.5);
    const double avgR = __dmul_rn(__dadd_rn(x, xr), 0.5);
    const bool cRL = fabs(dr) > fabs(dl), cR0 = fabs(dr) > 0.0, cL0 = fabs(dl) > 0.0;
    const bool pR = hasR & ((hasL & cRL) | (!hasL & cR0));
    const bool pL = hasL & cL0;
    const bool qL = !pR & pL;
    const unsigned bR = __ballot_sync(FULL, pR);
    const unsigned bL = __ballot_sync(FULL, qL);
    const bool mR = pR & (((bL >> 1) >> lane) & 1u);
    const bool mL = qL & (((bR << 1) >> lane) & 1u);
    m = bR & (bL >> 1);
    return mR ? avgR : (mL ? avgL : x);
}

__device__ __forceinline__ int partner_of(unsigned m, int lane) {
    return ((m >> lane) & 1u) ? lane + 1 : ((lane > 0 && ((m >> (lane - 1)) & 1u)) ? lane - 1 : lane);
}

// A round under a known matching: partner's x by one shuffle, then one fma.
__device__ __forceinline__ double step_pair(double x, int partner) {
    const double y = __shfl_sync(FULL, x, partner);
    return fma(y, 0.5, __dmul_rn(x, 0.5));
}

// n <= 8: fluid_spec's speculative rounds, and once a full 32-row chunk
// has verified (the matching has settled), the verification of each chunk
// overlapped with the production of the next: one straight-line block
// verifies chunk A (lane j: row j's true matching and phi_f, independent of
// the production chain) while it produces the 32 rows of chunk B (one
// shuffle + one fma per row on the chain, fully unrolled), so the
// verification fills the chain's idle issue slots.  B continues A's
// predictions (32 is even: the period-2 roles of h0 / h1 carry over).  A
// stop row in A ends the process; a misprediction in A drops B and returns
// to fluid_spec's small chunks (4 exact rounds, then predictions) at the
// true successor.  Rows, arithmetic and stop rule are fluid_spec's.
//
// verify_row for n <= 8 without branches (every row entry loaded, absent
// ones replaced by 0; absent phi_f terms add +0.0, which leaves the running
// sum bit-identical), so it shares a basic block with the production.
__device__ __forceinline__ void verify_row8(const double *row, int n, unsigned &tm, double &acc) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const double v = row[u];
        x[u] = u < n ? v : 0.0;
    }
    unsigned pr = 0u, pl = 0u;
    double dprev = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const bool hasR = t + 1 < n, hasL = t > 0 && t < n;
        const double d = hasR ? __dsub_rn(x[t], x[t < 7 ? t + 1 : t]) : 0.0;
        const bool cR = hasR && (hasL ? fabs(d) > fabs(dprev) : fabs(d) > 0.0);
        const bool cL = hasL && !cR && fabs(dprev) > 0.0;
        pr |= (unsigned)cR << t;
        pl |= (unsigned)cL << t;
        dprev = d;
    }
    tm = pr & (pl >> 1);
    double a = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = u + 1; v < 8; ++v) a = __dadd_rn(a, v < n ? fabs(__dsub_rn(x[u], x[v])) : 0.0);
    acc = a;
}

// The overlapped mode, entered after a verified full chunk with x the next
// row and h0 / h1 the true matchings of the two rows before it.  Returns
// true once it has written the stop row; false at a misprediction, with
// (x, h0, h1, base, fb) describing the restart at the true successor.
__device__ bool fluid_overlap(int n, double gf, int maxr, double *hist, double *xo, int &rr, double &ph,
                              int &fst, int lane, double &x, unsigned &h0, unsigned &h1, int &base, int &fb) {
    int bufA = 0, baseA = base;
    unsigned usedA = 0u, s1A = h1;
    {
        const int pa = partner_of(h0, lane), pb = partner_of(h1, lane);
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            hist[k * kRow + lane] = x;  // lanes >= n store into the row's padding
            usedA = lane == k ? ((k & 1) ? h1 : h0) : usedA;
            x = step_pair(x, (k & 1) ? pb : pa);
        }
    }
    for (;;) {
        double *hA = hist + bufA * kChunk * kRow, *hB = hist + (bufA ^ 1) * kChunk * kRow;
        __syncwarp();
        unsigned tm, usedB = 0u;
        double acc;
        {
            const int pa = partner_of(h0, lane), pb = partner_of(h1, lane);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (k == 1) verify_row8(hA + lane * kRow, n, tm, acc);  // chunk A, lane = row
                hB[k * kRow + lane] = x;
                usedB = lane == k ? ((k & 1) ? h1 : h0) : usedB;
                x = step_pair(x, (k & 1) ? pb : pa);
            }
        }
        const unsigned mbad = __ballot_sync(FULL, tm != usedA);
        fb = mbad ? __ffs(mbad) - 1 : kChunk;
        const unsigned mstop = __ballot_sync(FULL, lane <= fb && (acc <= gf || baseA + lane == maxr));
        if (mstop) {
            const int k = __ffs(mstop) - 1;
            rr = baseA + k;
            ph = __shfl_sync(FULL, acc, k);
            if (!(ph <= gf)) fst = DYNMO_W_NOT_CONVERGED;
            if (lane < n) xo[lane] = hA[k * kRow + lane];
            return true;
        }
        if (fb < kChunk) {  // drop B; restart at the true successor of row fb
            const unsigned tb = __shfl_sync(FULL, tm, fb);
            const unsigned tp = __shfl_sync(FULL, tm, fb > 0 ? fb - 1 : 0);
            const double xv = lane < n ? hA[fb * kRow + lane] : 0.0;
            h0 = fb > 0 ? tp : s1A;
            h1 = tb;
            x = step_pair(xv, partner_of(tb, lane));
            base = baseA + fb + 1;
            __syncwarp();
            return false;
        }
        s1A = __shfl_sync(FULL, usedA, kChunk - 1);
        baseA += kChunk;
        usedA = usedB;
        bufA ^= 1;
    }
}

#ifdef DYNMO_FLUID_PROF  // diagnostic build only: phase cycles into fluid_x (tools/fluid_prof.py)
__shared__ long long g_fprof_t0;
#define FPROF(v) const long long v = clock64()
#else
#define FPROF(v)
#endif

template <bool OVL>  // OVL (n <= 8): the overlapped mode once a full chunk has verified
__device__ void fluid_spec(const Inst &s, int n, const int32_t *bi, double gf, int maxr, double *hist,
                           double *xo, int &rr, double &ph, int &fst, int lane) {
#ifdef DYNMO_FLUID_PROF
    long long c_ex = 0, c_sp = 0, c_ve = 0, chunks = 0;
    const long long c_in = clock64();
#endif
    double x = lane < n ? (double)(s.P[bi[lane + 1]] - s.P[bi[lane]]) : 0.0;
    const bool hasL = lane >= 1 && lane < n, hasR = lane + 1 < n;
    unsigned h0 = 0u, h1 = 0u;  // true matchings of the two rounds before the next row
    int e = 4, size = 8;        // exact rows, rows of the chunk
    for (int base = 0;;) {
        const unsigned s1 = h1;  // matching of round base - 1
        unsigned used = 0u;      // lane k: the matching applied to row k
        FPROF(ta);
        for (int k = 0; k < e; ++k) {
            if (lane < n) hist[k * kRow + lane] = x;  // x(base + k)
            unsigned m;
            x = exact_round(x, hasL, hasR, lane, m);
            used = lane == k ? m : used;
            h0 = h1;
            h1 = m;
        }
        FPROF(tb);
        {
            const int pa = partner_of(h0, lane), pb = partner_of(h1, lane);
            for (int k = e; k < size; ++k) {
                if (lane < n) hist[k * kRow + lane] = x;
                const bool odd = (k - e) & 1;
                used = lane == k ? (odd ? h1 : h0) : used;
                x = step_pair(x, odd ? pb : pa);
            }
        }
        __syncwarp();
        FPROF(tc);
        unsigned tm = 0u;
        double acc = 0.0;
        if (lane < size) verify_row(hist + lane * kRow, n, tm, acc);
        const unsigned mbad = __ballot_sync(FULL, lane < size && tm != used);
        const int fb = mbad ? __ffs(mbad) - 1 : size;  // rows 0 .. fb are exact
        const bool stop = lane < size && lane <= fb && (acc <= gf || base + lane == maxr);
        const unsigned mstop = __ballot_sync(FULL, stop);
        FPROF(td);
#ifdef DYNMO_FLUID_PROF
        c_ex += tb - ta;
        c_sp += tc - tb;
        c_ve += td - tc;
        ++chunks;
#endif
        if (mstop) {
            const int k = __ffs(mstop) - 1;
            rr = base + k;
            ph = __shfl_sync(FULL, acc, k);
            if (!(ph <= gf)) fst = DYNMO_W_NOT_CONVERGED;
            if (lane < n) xo[lane] = hist[k * kRow + lane];
#ifdef DYNMO_FLUID_PROF
            __syncwarp();
            const long long te = clock64();
            if (lane == 0) {
                xo[0] = (double)(c_in - g_fprof_t0);  // kernel start -> fluid entry
                xo[1] = (double)c_ex;
                xo[2] = (double)c_sp;
                xo[3] = (double)c_ve;
                xo[4] = (double)(te - c_in - c_ex - c_sp - c_ve);  // bookkeeping
                xo[5] = (double)chunks;
                xo[6] = (double)(te - g_fprof_t0);
            }
#endif
            return;
        }
        if (fb < size) {
            // the true next state from the first mispredicted row
            const unsigned tb = __shfl_sync(FULL, tm, fb);
            const unsigned tp = __shfl_sync(FULL, tm, fb > 0 ? fb - 1 : 0);
            const double xv = lane < n ? hist[fb * kRow + lane] : 0.0;
            h0 = fb > 0 ? tp : s1;
            h1 = tb;
            x = step_pair(xv, partner_of(tb, lane));
            base += fb + 1;
            e = 4;
            size = min(kChunk, max(8, 2 * (fb + 1)));
        } else {
            h0 = __shfl_sync(FULL, used, size - 2);
            h1 = __shfl_sync(FULL, used, size - 1);
            base += size;
            if (OVL && size == kChunk) {
                __syncwarp();
                int fbo;
                if (fluid_overlap(n, gf, maxr, hist, xo, rr, ph, fst, lane, x, h0, h1, base, fbo)) return;
                e = 4;
                size = min(kChunk, max(8, 2 * (fbo + 1)));
                continue;
            }
            e = 0;
            size = min(kChunk, size * 4);
        }
        __syncwarp();
    }
}

__device__ void diffuse_fluid(const SolveArgs &a, const Inst &s, int q, int n, const int32_t *bi,
                              int fst, double *hist, int lane) {
    const double gf = a.gamma_fluid ? a.gamma_fluid[q] : 0.0;
    const int maxr = a.max_rounds;
    double *xo = a.fluid_x + (a.bnd_off[q] - q);
    if (fst < 0) {
        for (int k = lane; k < n; k += 32) xo[k] = -1.0;
        if (lane == 0) {
            if (a.fluid_rounds) a.fluid_rounds[q] = -1;
            if (a.fluid_phi) a.fluid_phi[q] = -1.0;
            if (a.fluid_status) a.fluid_status[q] = fst;
        }
        return;
    }
    int rr = 0;
    double ph = 0.0;
    if (n <= 32) {
        if (a.fluid_spec == 2 && n <= 8) fluid_spec<true>(s, n, bi, gf, maxr, hist, xo, rr, ph, fst, lane);
        else if (a.fluid_spec) fluid_spec<false>(s, n, bi, gf, maxr, hist, xo, rr, ph, fst, lane);
        else fluid_chunks(s, n, bi, gf, maxr, hist, xo, rr, ph, fst, lane);
    } else if (lane == 0) {
        // n > 32: serial on lane 0 over shared memory (s.x reused as fp64)
        double *sxf = reinterpret_cast<double *>(s.x);
        int32_t *pk = s.pick;
        for (int t = 0; t < n; ++t) sxf[t] = (double)(s.P[bi[t + 1]] - s.P[bi[t]]);
        for (;;) {
            ph = 0.0;
            for (int u = 0; u < n; ++u)
                for (int v = u + 1; v < n; ++v) ph = __dadd_rn(ph, fabs(__dsub_rn(sxf[u], sxf[v])));
            if (ph <= gf) break;
            if (rr == maxr) {
                fst = DYNMO_W_NOT_CONVERGED;
                break;
            }
            for (int t = 0; t < n; ++t) {
                int p = -1;
                double best = 0.0;
                for (int e = t - 1; e <= t; ++e) {
                    if (e < 0 || e + 1 >= n) continue;
                    const double g = fabs(__dsub_rn(sxf[e], sxf[e + 1]));
                    if (g > best) {
                        best = g;
                        p = e;
                    }
                }
                pk[t] = p;
            }
            for (int e = 0; e + 1 < n; ++e)
                if (pk[e] == e && pk[e + 1] == e) {
                    const double avg = __dmul_rn(__dadd_rn(sxf[e], sxf[e + 1]), 0.5);
                    sxf[e] = avg;
                    sxf[e + 1] = avg;
                }
            rr++;
        }
        for (int t = 0; t < n; ++t) xo[t] = sxf[t];
    }
    if (lane == 0) {
        if (a.fluid_rounds) a.fluid_rounds[q] = rr;
        if (a.fluid_phi) a.fluid_phi[q] = ph;
        if (a.fluid_status) a.fluid_status[q] = fst;
    }
}

template <bool MEM>
__global__ void __launch_bounds__(32) k_diffuse(SolveArgs a) {
    pdl_wait();
    pdl_trigger();
    STEP_STAMP(blockIdx.y == 1 ? STAMP_DIFFUSE_F : STAMP_DIFFUSE_D);
    extern __shared__ __align__(16) char smem[];
#ifdef DYNMO_FLUID_PROF
    if (threadIdx.x == 0) g_fprof_t0 = clock64();
#endif
    const int q = blockIdx.x, lane = threadIdx.x;
    const bool fluid = blockIdx.y == 1;
    Inst s = carve(smem, a.max_layers, MEM && !fluid);
    DYNMO_DCHECK(!fluid || solve_smem_bytes(a.max_layers, false, true) <= dyn_smem_bytes());
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n = a.n_stages[q];
    const int32_t *bi = a.bnd_in + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    s.cap = cap;
    // validity shared by both processes: L, n, max_rounds, b_in
    int st = DYNMO_OK;
    if (L < 1 || L > a.max_layers || n < 1 || n > L || a.max_rounds < 0) st = DYNMO_E_INVALID;
    if (st == DYNMO_OK) {
        int bad = 0;
        for (int k = lane; k < n; k += 32) bad |= bi[k + 1] <= bi[k];
        bad |= bi[0] != 0 || bi[n] != L;
        if (__any_sync(FULL, bad)) st = DYNMO_E_INVALID;
    }
    if (fluid) {
        const double gf = a.gamma_fluid ? a.gamma_fluid[q] : 0.0;
        if (st == DYNMO_OK && !(gf >= 0.0)) st = DYNMO_E_INVALID;
        if (st == DYNMO_OK) {  // the fluid process reads only the costs
            const PrefixFlags f = load_prefix(s, a.cost + off, nullptr, L, lane);
            st = f.cneg ? DYNMO_E_INVALID : f.covf ? DYNMO_E_OVERFLOW : DYNMO_OK;
        }
        double *hist = reinterpret_cast<double *>(smem + base_bytes(a.max_layers, false));
        diffuse_fluid(a, s, q, n, bi, st, hist, lane);
        return;
    }
    const int64_t gamma = a.gamma ? a.gamma[q] : 0;
    if (st == DYNMO_OK && (gamma < 0 || (MEM && cap < 0))) st = DYNMO_E_INVALID;
    if (st == DYNMO_OK)
        st = prefix_status(load_prefix(s, a.cost + off, MEM ? a.mem + off : nullptr, L, lane), MEM);
    diffuse_discrete<MEM>(a, s, q, n, bi, st, lane);
}

}  // namespace

// ------------------------------------------------------------- launchers
// Small batches (the per-step hot path): 8 warps per instance, a 9-ary
// search.  Large batches: 1 warp per instance (binary search, one wave).
static bool latency_mode(const SolveArgs &a) { return a.n_inst <= 4 * 148; }

template <template <bool, int> class K>
static cudaError_t launch_solver(const SolveArgs &a, cudaStream_t s) {
    const size_t sm = solve_smem_bytes(a.max_layers, a.mem != nullptr, false);
    const bool lm = latency_mode(a), mem = a.mem != nullptr;
    const dim3 grid(a.n_inst), block(lm ? 256 : 32);
    cudaError_t e;
    if (mem && lm) e = K<true, 8>::launch(grid, block, sm, s, a);
    else if (mem) e = K<true, 1>::launch(grid, block, sm, s, a);
    else if (lm) e = K<false, 8>::launch(grid, block, sm, s, a);
    else e = K<false, 1>::launch(grid, block, sm, s, a);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool M, int NW>
struct PartitionK {
    static cudaError_t launch(dim3 g, dim3 b, size_t sm, cudaStream_t s, const SolveArgs &a) {
        return launch_pdl(k_partition<M, NW>, g, b, sm, s, a);
    }
};
template <bool M, int NW>
struct RepackK {
    static cudaError_t launch(dim3 g, dim3 b, size_t sm, cudaStream_t s, const SolveArgs &a) {
        return launch_pdl(k_repack<M, NW>, g, b, sm, s, a);
    }
};

cudaError_t launch_partition(const SolveArgs &a, cudaStream_t s) { return launch_solver<PartitionK>(a, s); }
cudaError_t launch_diffuse(const SolveArgs &a, cudaStream_t s) {
    const bool fl = a.fluid_x != nullptr;
    // the discrete block carves the memory prefix, the fluid block the
    // history instead: the launch needs the larger of the two (< 48 KB at
    // max_layers = 1023, so no opt-in attribute and no carveout change)
    const size_t sm = fl ? std::max(solve_smem_bytes(a.max_layers, a.mem != nullptr, false),
                                    solve_smem_bytes(a.max_layers, false, true))
                         : solve_smem_bytes(a.max_layers, a.mem != nullptr, false);
    const dim3 grid(a.n_inst, fl ? 2 : 1);
    const cudaError_t e = a.mem ? launch_pdl(k_diffuse<true>, grid, 32, sm, s, a)
                                : launch_pdl(k_diffuse<false>, grid, 32, sm, s, a);
    return e != cudaSuccess ? e : cudaGetLastError();
}
cudaError_t launch_repack(const SolveArgs &a, cudaStream_t s) { return launch_solver<RepackK>(a, s); }

}  // namespace dynmo

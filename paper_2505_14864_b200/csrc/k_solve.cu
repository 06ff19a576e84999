// k_solve.cu -- batched rebalancing solvers on sm_100a, one CTA per instance
// (SURVEY 8(a) a7-a9).
//
//  k_partition  contiguous min-max partition:
//               exact integer (W+1)-ary search over the bottleneck B, each warp
//               testing one candidate with a warp-parallel greedy: a greedy
//               jump from layer j is ONE __reduce_add_sync over the lanes'
//               register-resident prefix sums (count of k with P[k] <= P[j]+B
//               and M[k] <= M[j]+cap), so a feasibility test costs <= n jumps.
//               Canonical lexmax boundaries (reading Q7), fp64 Delta L.
//  k_diffuse    decentralised diffusion (reading Q10):
//               per round every warp re-splits adjacent stage pairs (warp
//               argmin over split points), the max-neighbor matching applies
//               mutually chosen pairs; plus the fluid averaging process of
//               Lemma 2's proof in fp64 (round-to-nearest, no FMA).
//  k_repack     fewest workers within the throughput bound (P:L13, P:L556-
//               609): one greedy count at B = bound then the partition; or
//               Alg. 2 first-fit (P:L562-593 with SPEC:L389 fixes).
#include <cuda_runtime.h>

#include <cstdint>

#include "dynmo_internal.h"

namespace dynmo {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int64_t I64MAX = INT64_MAX;

__device__ __forceinline__ int64_t satadd(int64_t a, int64_t b) {  // a, b >= 0
    return b > I64MAX - a ? I64MAX : a + b;
}
__device__ __forceinline__ int worse(int a, int b) { return a < b ? a : b; }

template <int Q, bool MEM>
struct Inst {
    int64_t P[Q * 32];             // P[k] = sum_{i<k} c_i, padded with I64MAX past L
    int64_t M[MEM ? Q * 32 : 1];   // same for mem
    int32_t b[Q * 32];             // working boundaries
    int64_t maxc;
    int64_t cap;
    int32_t L, n, status;
};

// Load one instance and build the prefix sums (warp 0 scan).  Reports, per
// array, whether a value is negative and whether the exact sum exceeds
// INT64_MAX; each kernel combines them in the oracle's check order.
struct PrefixFlags {
    bool cneg, covf, mneg, movf;
};

__device__ bool exact_sum_overflows(const int64_t *v, int L) {
    __int128 acc = 0;
    for (int i = 0; i < L; ++i) acc += v[i];
    return acc > (__int128)I64MAX;
}

template <int Q, bool MEM>
__device__ PrefixFlags load_prefix(Inst<Q, MEM> &s, const int64_t *cost, const int64_t *mem, int L) {
    __shared__ int s_flags;
    const int tid = threadIdx.x;
    for (int i = tid; i < Q * 32; i += blockDim.x) {
        s.P[i] = (i >= 1 && i <= L) ? cost[i - 1] : 0;
        if constexpr (MEM) s.M[i] = (i >= 1 && i <= L) ? mem[i - 1] : 0;
    }
    __syncthreads();
    int cneg = 0, mneg = 0;
    for (int i = tid; i < Q * 32; i += blockDim.x) {
        cneg |= s.P[i] < 0;
        if constexpr (MEM) mneg |= s.M[i] < 0;
    }
    cneg = __syncthreads_or(cneg);
    mneg = __syncthreads_or(mneg);
    PrefixFlags f{cneg != 0, false, mneg != 0, false};
    if (cneg || mneg) return f;  // prefix sums are not needed on an error
    if (tid < 32) {
        const int lane = tid;
        int64_t vp[Q], vm[Q];
        int64_t sp = 0, smx = 0, mx = 0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const int64_t c = s.P[lane * Q + k];
            mx = c > mx ? c : mx;
            sp = satadd(sp, c);
            vp[k] = sp;
            if constexpr (MEM) {
                smx = satadd(smx, s.M[lane * Q + k]);
                vm[k] = smx;
            }
        }
        // exclusive scan of the lane totals (saturating)
        int64_t ep = sp, em = smx;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t tp = __shfl_up_sync(FULL, ep, o);
            int64_t tm = 0;
            if constexpr (MEM) tm = __shfl_up_sync(FULL, em, o);
            if (lane >= o) {
                ep = satadd(ep, tp);
                if constexpr (MEM) em = satadd(em, tm);
            }
        }
        ep = __shfl_up_sync(FULL, ep, 1);
        if constexpr (MEM) em = __shfl_up_sync(FULL, em, 1);
        if (lane == 0) {
            ep = 0;
            em = 0;
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const int pos = lane * Q + k;
            s.P[pos] = pos <= L ? satadd(ep, vp[k]) : I64MAX;
            if constexpr (MEM) s.M[pos] = pos <= L ? satadd(em, vm[k]) : I64MAX;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t t = __shfl_xor_sync(FULL, mx, o);
            mx = t > mx ? t : mx;
        }
        __syncwarp();
        if (lane == 0) {
            s.maxc = mx;
            // a saturated prefix is I64MAX: decide overflow exactly (128-bit)
            int fl = 0;
            if (s.P[L] == I64MAX && exact_sum_overflows(cost, L)) fl |= 1;
            if constexpr (MEM)
                if (s.M[L] == I64MAX && exact_sum_overflows(mem, L)) fl |= 2;
            s_flags = fl;
        }
    }
    __syncthreads();
    f.covf = (s_flags & 1) != 0;
    f.movf = (s_flags & 2) != 0;
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

// Registers: lane owns prefix positions lane*Q .. lane*Q+Q-1.
template <int Q, bool MEM>
struct Regs {
    int64_t p[Q];
    int64_t m[MEM ? Q : 1];
};

template <int Q, bool MEM>
__device__ __forceinline__ void load_regs(Regs<Q, MEM> &r, const Inst<Q, MEM> &s, int lane) {
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        r.p[k] = s.P[lane * Q + k];
        if constexpr (MEM) r.m[k] = s.M[lane * Q + k];
    }
}

// Greedy maximal jump from j under bottleneck B (warp-uniform result):
// the largest K with P[K]-P[j] <= B and M[K]-M[j] <= cap.  Both predicates
// are monotone in K, so K+1 = number of positions satisfying them.
template <int Q, bool MEM>
__device__ __forceinline__ int warp_next(const Regs<Q, MEM> &r, const Inst<Q, MEM> &s, int j,
                                         int64_t B) {
    const int64_t t1 = satadd(s.P[j], B);
    int64_t t2 = 0;
    if constexpr (MEM) t2 = satadd(s.M[j], s.cap);
    unsigned c = 0;
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        bool ok = r.p[k] <= t1;
        if constexpr (MEM) ok = ok && r.m[k] <= t2;
        c += ok;
    }
    const int K = (int)__reduce_add_sync(FULL, c) - 1;
    return K < s.L ? K : s.L;
}

// Greedy stage count under B, stopping once it exceeds `limit`
// (returns limit+1 for "more than limit", including an unplaceable layer).
template <int Q, bool MEM>
__device__ int warp_greedy_count(const Regs<Q, MEM> &r, const Inst<Q, MEM> &s, int64_t B,
                                 int limit) {
    int j = 0, c = 0;
    while (j < s.L) {
        if (c == limit) return limit + 1;
        const int K = warp_next<Q, MEM>(r, s, j, B);
        if (K == j) return limit + 1;
        j = K;
        ++c;
    }
    return c;
}

template <int Q, bool MEM>
__device__ __forceinline__ bool warp_feasible(const Regs<Q, MEM> &r, const Inst<Q, MEM> &s,
                                              int64_t B, int n) {
    return warp_greedy_count<Q, MEM>(r, s, B, n) <= n;
}

// Exact min-max search over B in [lo, hi] (hi feasible), all warps.
// Returns B* (block-uniform) or -1 if infeasible (MEM only).
template <int Q, int W, bool MEM>
__device__ int64_t search_bottleneck(const Regs<Q, MEM> &r, Inst<Q, MEM> &s, int n) {
    __shared__ int64_t s_lo, s_hi;
    __shared__ int64_t s_cand[W];
    __shared__ int s_feas[W];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t C = s.P[s.L];
    const int64_t ceil_cn = C / n + (C % n != 0);
    int64_t lo = s.maxc > ceil_cn ? s.maxc : ceil_cn;
    int64_t hi = satadd(ceil_cn, s.maxc);
    if (hi > C) hi = C;
    if (lo > hi) lo = hi;
    if constexpr (MEM) {
        // the cost bracket may be infeasible under the memory cap
        if (w == 0) {
            bool f = warp_feasible<Q, MEM>(r, s, hi, n);
            if (!f) {
                hi = C;
                f = warp_feasible<Q, MEM>(r, s, hi, n);
            }
            if (lane == 0) s_hi = f ? hi : -1;
        }
        __syncthreads();
        if (s_hi < 0) return -1;
        hi = s_hi;
    }
    while (lo < hi) {
        const int64_t d = hi - lo;
        const int64_t cand =
            lo + (int64_t)(((unsigned __int128)(uint64_t)d * (unsigned)(w + 1)) / (unsigned)(W + 1));
        const bool f = warp_feasible<Q, MEM>(r, s, cand, n);
        if (lane == 0) {
            s_cand[w] = cand;
            s_feas[w] = f;
        }
        __syncthreads();
        for (int k = 0; k < W; ++k) {
            if (s_feas[k]) {
                if (s_cand[k] < hi) hi = s_cand[k];
            } else {
                if (s_cand[k] + 1 > lo) lo = s_cand[k] + 1;
            }
        }
        __syncthreads();
    }
    return hi;
}

// Lexmax boundaries for B* (Appendix A construction), warp 0; writes s.b.
template <int Q, bool MEM>
__device__ void warp_construct(const Regs<Q, MEM> &r, Inst<Q, MEM> &s, int64_t Bs, int n) {
    int j = 0;
    if ((threadIdx.x & 31) == 0) s.b[0] = 0;
    for (int st = 0; st < n; ++st) {
        int K = warp_next<Q, MEM>(r, s, j, Bs);
        const int reserve = s.L - (n - 1 - st);
        j = K < reserve ? K : reserve;
        if ((threadIdx.x & 31) == 0) s.b[st + 1] = j;
    }
}

__device__ double imbalance_of(const int64_t *P, const int32_t *b, int n) {
    int64_t mx = P[b[1]] - P[b[0]], mn = mx;
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

template <bool MEM>
__device__ __forceinline__ const int64_t *mem_ptr(const SolveArgs &a) {
    return MEM ? a.mem : nullptr;
}

// ------------------------------------------------------------ partition
template <int Q, int W, bool MEM>
__global__ void __launch_bounds__(W * 32) k_partition(SolveArgs a) {
    __shared__ Inst<Q, MEM> s;
    const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n = a.n_stages[q];
    int32_t *bnd = a.bnd_out + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    int st = DYNMO_OK;
    if (L < 1 || L > a.max_layers || L > Q * 32 - 1 || n < 1 || n > L || (MEM && cap < 0))
        st = DYNMO_E_INVALID;
    if (st == DYNMO_OK)
        st = prefix_status(load_prefix<Q, MEM>(s, a.cost + off, MEM ? a.mem + off : nullptr, L), MEM);
    if (tid == 0) {
        s.L = L;
        s.n = n;
        s.cap = cap;
    }
    __syncthreads();
    int64_t Bs = -1;
    Regs<Q, MEM> r;
    if (st == DYNMO_OK) {
        load_regs<Q, MEM>(r, s, lane);
        Bs = search_bottleneck<Q, W, MEM>(r, s, n);
        if (Bs < 0) st = DYNMO_E_INFEASIBLE;
    }
    if (st != DYNMO_OK) {
        for (int k = tid; k <= n && n >= 1; k += blockDim.x) bnd[k] = -1;
        if (tid == 0) {
            a.bottleneck[q] = -1;
            if (a.imbalance) a.imbalance[q] = -1.0;
            a.status[q] = st;
        }
        return;
    }
    if (tid < 32) warp_construct<Q, MEM>(r, s, Bs, n);
    __syncthreads();
    for (int k = tid; k <= n; k += blockDim.x) bnd[k] = s.b[k];
    if (tid == 0) {
        a.bottleneck[q] = Bs;
        if (a.imbalance) a.imbalance[q] = imbalance_of(s.P, s.b, n);
        a.status[q] = DYNMO_OK;
    }
}

// -------------------------------------------------------------- repack
template <int Q, int W, bool MEM>
__global__ void __launch_bounds__(W * 32) k_repack(SolveArgs a) {
    __shared__ Inst<Q, MEM> s;
    __shared__ int s_k;
    const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n_cur = a.n_stages[q];
    const int fl = a.floor_[q];
    int32_t *bnd = a.bnd_out + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    const bool alg2 = a.mode == DYNMO_REPACK_ALG2;
    const int64_t bound = alg2 ? 0 : a.bound[q];
    int st = DYNMO_OK;
    if (L < 1 || L > a.max_layers || L > Q * 32 - 1 || n_cur < 1 || n_cur > L || fl < 1 ||
        fl > n_cur || (MEM && cap < 0) || (!alg2 && bound < 0))
        st = DYNMO_E_INVALID;
    if (st == DYNMO_OK && alg2) {
        // b_in must be a valid split
        const int32_t *bi = a.bnd_in + a.bnd_off[q];
        int bad = 0;
        for (int k = tid; k < n_cur; k += blockDim.x) bad |= bi[k + 1] <= bi[k];
        bad |= bi[0] != 0 || bi[n_cur] != L;
        if (__syncthreads_or(bad)) st = DYNMO_E_INVALID;
    }
    if (st == DYNMO_OK) {
        const PrefixFlags f = load_prefix<Q, MEM>(s, a.cost + off, MEM ? a.mem + off : nullptr, L);
        if (alg2)  // oracle: negatives of cost and mem first, then the cost sum
            st = (f.cneg || f.mneg) ? DYNMO_E_INVALID : f.covf ? DYNMO_E_OVERFLOW : DYNMO_OK;
        else
            st = prefix_status(f, MEM);
    }
    if (tid == 0) {
        s.L = L;
        s.cap = cap;
    }
    __syncthreads();
    auto fail = [&](int code) {
        for (int k = tid; k <= n_cur && n_cur >= 1; k += blockDim.x) bnd[k] = -1;
        if (tid == 0) {
            a.n_new[q] = -1;
            a.bottleneck[q] = -1;
            a.status[q] = code;
        }
    };
    if (st != DYNMO_OK) {
        fail(st);
        return;
    }
    if (alg2) {
        // Alg. 2 with the fixes of SPEC:L364/L389, serial.
        if (tid == 0) {
            const int32_t *bi = a.bnd_in + a.bnd_off[q];
            const int64_t *mem = MEM ? a.mem + off : nullptr;
            __int128 mu_prev = 0;  // mem of the current chain head (src)
            int n_active = n_cur, k = 0;
            // mu of worker 0
            if (mem)
                for (int i = bi[0]; i < bi[1]; ++i) mu_prev += mem[i];
            s.b[0] = 0;
            for (int src = 0; src + 1 < n_cur; ++src) {
                __int128 mu_dst = 0;
                if (mem)
                    for (int i = bi[src + 1]; i < bi[src + 2]; ++i) mu_dst += mem[i];
                const bool fits = !mem || (mu_prev + mu_dst <= (__int128)cap);
                if (fits && n_active > fl) {
                    n_active--;                 // src deactivated, merged into dst
                    mu_prev = mu_prev + mu_dst;
                } else {
                    s.b[++k] = bi[src + 1];     // src stays active
                    mu_prev = mu_dst;
                }
            }
            s.b[++k] = bi[n_cur];
            s_k = k;
            int64_t bm = 0;
            for (int t = 0; t < k; ++t) {
                const int64_t x = s.P[s.b[t + 1]] - s.P[s.b[t]];
                bm = x > bm ? x : bm;
            }
            a.n_new[q] = k;
            a.bottleneck[q] = bm;
            a.status[q] = n_active > fl ? DYNMO_W_BOUND_UNMET : DYNMO_OK;
        }
        __syncthreads();
        for (int t = tid; t <= n_cur; t += blockDim.x) bnd[t] = t <= s_k ? s.b[t] : -1;
        return;
    }
    Regs<Q, MEM> r;
    load_regs<Q, MEM>(r, s, lane);
    // fewest workers: greedy count at B = bound (cost and mem), reading Q15
    if (tid < 32) {
        const int g = warp_greedy_count<Q, MEM>(r, s, bound, n_cur);
        if (lane == 0) s_k = g;
    }
    __syncthreads();
    const int g = s_k;
    int k;
    int code = DYNMO_OK;
    if (g <= n_cur) {
        k = g > fl ? g : fl;
    } else {
        k = n_cur;
        code = DYNMO_W_BOUND_UNMET;
    }
    const int64_t Bs = search_bottleneck<Q, W, MEM>(r, s, k);
    if (Bs < 0) {
        fail(DYNMO_E_INFEASIBLE);
        return;
    }
    if (tid < 32) warp_construct<Q, MEM>(r, s, Bs, k);
    __syncthreads();
    for (int t = tid; t <= n_cur; t += blockDim.x) bnd[t] = t <= k ? s.b[t] : -1;
    if (tid == 0) {
        a.n_new[q] = k;
        a.bottleneck[q] = Bs;
        a.status[q] = code;
    }
}

// ------------------------------------------------------------- diffusion
template <int Q, int W, bool MEM>
__global__ void __launch_bounds__(W * 32) k_diffuse(SolveArgs a) {
    __shared__ Inst<Q, MEM> s;
    __shared__ int64_t sx[Q * 32];
    __shared__ int32_t s_tgt[Q * 32];  // edge e: best split j if improvable, else -1
    __shared__ int32_t s_pick[Q * 32];
    __shared__ double sxf[Q * 32];
    __shared__ int64_t s_phi, s_phi0;
    __shared__ int s_ctl, s_rounds;
    const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int off = a.layer_off[q];
    const int L = a.layer_off[q + 1] - off;
    const int n = a.n_stages[q];
    const int32_t *bi = a.bnd_in + a.bnd_off[q];
    int32_t *bo = a.bnd_out + a.bnd_off[q];
    const int64_t cap = MEM ? a.cap[q] : 0;
    const int64_t gamma = a.gamma ? a.gamma[q] : 0;
    const double gf = a.gamma_fluid ? a.gamma_fluid[q] : 0.0;
    const int maxr = a.max_rounds;
    const bool want_fluid = a.fluid_x != nullptr;
    // validity shared by both processes: L, n, max_rounds, b_in
    int common = DYNMO_OK;
    if (L < 1 || L > a.max_layers || L > Q * 32 - 1 || n < 1 || n > L || maxr < 0)
        common = DYNMO_E_INVALID;
    if (common == DYNMO_OK) {
        int bad = 0;
        for (int k = tid; k < n; k += blockDim.x) bad |= bi[k + 1] <= bi[k];
        bad |= bi[0] != 0 || bi[n] != L;
        if (__syncthreads_or(bad)) common = DYNMO_E_INVALID;
    }
    int dst = common, fst = want_fluid ? common : DYNMO_OK;
    if (common == DYNMO_OK) {
        if (gamma < 0 || (MEM && cap < 0)) dst = DYNMO_E_INVALID;
        if (want_fluid && !(gf >= 0.0)) fst = DYNMO_E_INVALID;
        const PrefixFlags f = load_prefix<Q, MEM>(s, a.cost + off, MEM ? a.mem + off : nullptr, L);
        const int cs = f.cneg ? DYNMO_E_INVALID : f.covf ? DYNMO_E_OVERFLOW : DYNMO_OK;
        if (fst == DYNMO_OK && want_fluid) fst = cs;
        if (dst == DYNMO_OK) dst = prefix_status(f, MEM);
    }
    if (tid == 0) {
        s.L = L;
        s.cap = cap;
        s_ctl = 0;
        s_rounds = 0;
    }
    __syncthreads();

    // ---------------- discrete diffusion (reading Q10)
    if (dst == DYNMO_OK) {
        for (int k = tid; k <= n; k += blockDim.x) s.b[k] = bi[k];
        __syncthreads();
        for (;;) {
            for (int t = tid; t < n; t += blockDim.x) sx[t] = s.P[s.b[t + 1]] - s.P[s.b[t]];
            __syncthreads();
            // phi = sum_{u<v} |x_u - x_v| (reading Q12), exact in 128 bits
            if (tid < 32) {
                __int128 acc = 0;
                for (int u = lane; u < n; u += 32)
                    for (int v = u + 1; v < n; ++v) {
                        const int64_t d = sx[u] > sx[v] ? sx[u] - sx[v] : sx[v] - sx[u];
                        acc += d;
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t lo = (uint64_t)acc, hi = (uint64_t)(acc >> 64);
                    const uint64_t olo = __shfl_xor_sync(FULL, lo, o);
                    const uint64_t ohi = __shfl_xor_sync(FULL, hi, o);
                    acc += (__int128)(((unsigned __int128)ohi << 64) | olo);
                }
                if (lane == 0) {
                    if (acc > (__int128)I64MAX) {
                        s_ctl = DYNMO_E_OVERFLOW;
                    } else {
                        s_phi = (int64_t)acc;
                        if (s_rounds == 0) s_phi0 = (int64_t)acc;
                        s_ctl = (int64_t)acc <= gamma ? 1 : 0;
                    }
                }
            }
            __syncthreads();
            if (s_ctl != 0) break;
            // best re-split of every adjacent pair: min (pair max, |j - b|, j)
            for (int e = w; e + 1 < n; e += W) {
                const int lo = s.b[e], hi = s.b[e + 2], cur = s.b[e + 1];
                int64_t km = I64MAX;
                int kd = INT32_MAX, kj = INT32_MAX, found = 0;
                for (int j = lo + 1 + lane; j < hi; j += 32) {
                    if constexpr (MEM)
                        if (s.M[j] - s.M[lo] > cap || s.M[hi] - s.M[j] > cap) continue;
                    const int64_t l = s.P[j] - s.P[lo], rr = s.P[hi] - s.P[j];
                    const int64_t m = l > rr ? l : rr;
                    const int d = j > cur ? j - cur : cur - j;
                    if (!found || m < km || (m == km && (d < kd || (d == kd && j < kj)))) {
                        found = 1;
                        km = m;
                        kd = d;
                        kj = j;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const int64_t om = __shfl_xor_sync(FULL, km, o);
                    const int od = __shfl_xor_sync(FULL, kd, o);
                    const int oj = __shfl_xor_sync(FULL, kj, o);
                    const int of = __shfl_xor_sync(FULL, found, o);
                    const bool take = of && (!found || om < km ||
                                             (om == km && (od < kd || (od == kd && oj < kj))));
                    if (take) {
                        km = om;
                        kd = od;
                        kj = oj;
                        found = 1;
                    }
                }
                if (lane == 0) {
                    const int64_t pm = sx[e] > sx[e + 1] ? sx[e] : sx[e + 1];
                    s_tgt[e] = (found && km < pm) ? kj : -1;
                }
            }
            __syncthreads();
            if (tid == 0) {
                int any = 0;
                for (int e = 0; e + 1 < n; ++e) any |= s_tgt[e] >= 0;
                if (!any) {
                    s_ctl = 1;
                } else if (s_rounds == maxr) {
                    s_ctl = 2;
                } else {
                    // max-neighbor matching: each stage picks its
                    // improvable incident edge with the largest gap
                    for (int t = 0; t < n; ++t) {
                        int pick = -1;
                        int64_t best = -1;
                        for (int e = t - 1; e <= t; ++e) {
                            if (e < 0 || e + 1 >= n || s_tgt[e] < 0) continue;
                            const int64_t g = sx[e] > sx[e + 1] ? sx[e] - sx[e + 1] : sx[e + 1] - sx[e];
                            if (g > best) {
                                best = g;
                                pick = e;
                            }
                        }
                        s_pick[t] = pick;
                    }
                    for (int e = 0; e + 1 < n; ++e)
                        if (s_tgt[e] >= 0 && s_pick[e] == e && s_pick[e + 1] == e) s.b[e + 1] = s_tgt[e];
                    s_rounds++;
                }
            }
            __syncthreads();
            if (s_ctl != 0) break;
        }
        if (s_ctl < 0) dst = s_ctl;
        else if (s_ctl == 2) dst = DYNMO_W_NOT_CONVERGED;
    }
    if (dst < 0) {
        for (int k = tid; k <= n && n >= 1; k += blockDim.x) bo[k] = -1;
        if (tid == 0) {
            if (a.rounds) a.rounds[q] = -1;
            if (a.phi) a.phi[q] = -1;
            if (a.phi0) a.phi0[q] = -1;
        }
    } else {
        for (int k = tid; k <= n; k += blockDim.x) bo[k] = s.b[k];
        if (tid == 0) {
            if (a.rounds) a.rounds[q] = s_rounds;
            if (a.phi) a.phi[q] = s_phi;
            if (a.phi0) a.phi0[q] = s_phi0;
        }
    }

    // ---------------- fluid process of Lemma 2's proof
    if (want_fluid) {
        double *xo = a.fluid_x + (a.bnd_off[q] - q);
        if (fst < 0) {
            for (int k = tid; k < n; k += blockDim.x) xo[k] = -1.0;
            if (tid == 0) {
                if (a.fluid_rounds) a.fluid_rounds[q] = -1;
                if (a.fluid_phi) a.fluid_phi[q] = -1.0;
            }
        } else if (tid == 0) {
            for (int t = 0; t < n; ++t) sxf[t] = (double)(s.P[bi[t + 1]] - s.P[bi[t]]);
            int rr = 0;
            double ph;
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
                    int pick = -1;
                    double best = 0.0;
                    for (int e = t - 1; e <= t; ++e) {
                        if (e < 0 || e + 1 >= n) continue;
                        const double g = fabs(__dsub_rn(sxf[e], sxf[e + 1]));
                        if (g > best) {
                            best = g;
                            pick = e;
                        }
                    }
                    s_pick[t] = pick;
                }
                for (int e = 0; e + 1 < n; ++e)
                    if (s_pick[e] == e && s_pick[e + 1] == e) {
                        const double avg = __dmul_rn(__dadd_rn(sxf[e], sxf[e + 1]), 0.5);
                        sxf[e] = avg;
                        sxf[e + 1] = avg;
                    }
                rr++;
            }
            for (int t = 0; t < n; ++t) xo[t] = sxf[t];
            if (a.fluid_rounds) a.fluid_rounds[q] = rr;
            if (a.fluid_phi) a.fluid_phi[q] = ph;
        }
    }
    if (tid == 0) {  // thread 0 ran the fluid loop, so its fst is final
        a.status[q] = (dst < 0 || fst < 0) ? worse(dst, fst) : (dst > fst ? dst : fst);
    }
}

}  // namespace

// ------------------------------------------------------------- launchers
#define DYNMO_DISPATCH(KERNEL, a, s)                                                      \
    do {                                                                                  \
        const bool mem_ = (a).mem != nullptr;                                             \
        const int ml_ = (a).max_layers;                                                   \
        if (ml_ <= 63) {                                                                  \
            if (mem_) KERNEL<2, 16, true><<<(a).n_inst, 512, 0, s>>>(a);                  \
            else KERNEL<2, 16, false><<<(a).n_inst, 512, 0, s>>>(a);                      \
        } else if (ml_ <= 127) {                                                          \
            if (mem_) KERNEL<4, 16, true><<<(a).n_inst, 512, 0, s>>>(a);                  \
            else KERNEL<4, 16, false><<<(a).n_inst, 512, 0, s>>>(a);                      \
        } else if (ml_ <= 255) {                                                          \
            if (mem_) KERNEL<8, 16, true><<<(a).n_inst, 512, 0, s>>>(a);                  \
            else KERNEL<8, 16, false><<<(a).n_inst, 512, 0, s>>>(a);                      \
        } else {                                                                          \
            if (mem_) KERNEL<32, 8, true><<<(a).n_inst, 256, 0, s>>>(a);                  \
            else KERNEL<32, 8, false><<<(a).n_inst, 256, 0, s>>>(a);                      \
        }                                                                                 \
    } while (0)

cudaError_t launch_partition(const SolveArgs &a, cudaStream_t s) {
    DYNMO_DISPATCH(k_partition, a, s);
    return cudaGetLastError();
}
cudaError_t launch_diffuse(const SolveArgs &a, cudaStream_t s) {
    DYNMO_DISPATCH(k_diffuse, a, s);
    return cudaGetLastError();
}
cudaError_t launch_repack(const SolveArgs &a, cudaStream_t s) {
    DYNMO_DISPATCH(k_repack, a, s);
    return cudaGetLastError();
}

}  // namespace dynmo

// Global magnitude pruning, Algorithm 1 -- NEXT-2 of SURVEY
// 8(f).  Alg. 1 keeps the k largest |w| over every rank's parameters (local
// top-k, gather to rank 0, global top-k, scatter of indices).  Here the SAME
// kept set is found without moving any weights: an exact distributed radix
// select on magnitude keys.
//   key(w) = bits(|w|) for f32; bits(|bf16|) << 16 for bf16 (the f32 key of
//   the same value), so segments of both types share one ordered key space
//   (monotone in |w| for non-NaN values; +0 and -0 both key 0).
//   pass 0: the digit key >> 16 (32768 bins; for bf16 the whole 15-bit
//           magnitude: an all-bf16 plan is done after it), in three steps:
//           a histogram of every 32nd tile -> all-reduce -> a bin window
//           [lo, hi] around the estimated k-th key -> one pass over every
//           key that histograms the window (and counts the keys below /
//           above it: exact totals) -> all-reduce -> bin.  A window that
//           misses the k-th key runs the full histogram (same launches,
//           graph-capturable; they return at once on a hit).
//   pass 1: histogram of key >> 6 & 1023 among keys with that prefix
//   pass 2: histogram of key & 63 among keys with the 25-bit prefix
// Each pass streams the rank's weights (HBM-bound); only the histograms cross
// GPUs (NCCL all-reduce).  The threshold tau is the k-th largest key;
// keys > tau are kept, and of the keys == tau the first `need` in the global
// order (rank, then segment order, then index -- SPEC S:L184) are kept:
// per-rank tie counts are all-gathered, and only the rank whose share of the
// ties is partial ranks its ties (per-(tile, warp range) counts -- recorded by
// the windowed pass for bf16 plans, else a counting pass -- an exclusive
// scan, and in-range warp scans in element order).
#include "dynmo_internal.h"

namespace dynmo {
namespace {

constexpr int kPruneThreads = 256;
constexpr int kBins0 = 32768;  // pass 0 digit: key bits 30..16 (15 bits = a bf16 magnitude)
constexpr int kBins1 = 1024;   // pass 1 digit: key bits 15..6; pass 2: bits 5..0 (64 of the bins)
constexpr int kHist0Threads = 1024;  // pass 0: one 128 KB shared histogram per block, one block per SM
constexpr uint32_t kWinMax = 4094;   // widest pass-0 window (bins) of the windowed pass: 16 KB shared
// The windowed pass's histogram in compact form (the only counters its
// all-reduce carries): bin 0 = keys below the window, 1 .. W = digits lo .. hi,
// W + 1 = keys above the window (W <= kWinMax, so W + 2 <= kCw); NaN count last.
constexpr int kCw = 4096;
constexpr int kCwNan = kCw;  // cw[kCwNan]; arrays of kCw + 1 = kPruneCw counters
static_assert(kCw + 1 == kPruneCw, "compact histogram size");
constexpr uint32_t kNanKey = 0x7F800000u;  // key > this: NaN
constexpr int kPruneWarps = kPruneThreads / 32;  // tie-offset entries per tile
constexpr int kU = 8;  // 16-byte loads in flight per thread in the streaming passes

__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t key_f32(uint32_t b) { return b & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t key_bf16(uint32_t h) { return (h & 0x7FFFu) << 16; }

// Applies f(key) to every element of tile t (any order): 16-byte vectors
// (8 bf16 / 4 f32 keys), kU loads in flight per thread, then a scalar tail.
template <typename F>
__device__ __forceinline__ void for_keys(const PruneTile &t, F &&f) {
    const uint4 *v = (const uint4 *)t.w;
    const bool bf = t.dtype == DYNMO_W_BF16;
    const uint32_t nv = bf ? t.n >> 3 : t.n >> 2;
    const uint32_t T = blockDim.x;
    for (uint32_t b = threadIdx.x; b < nv; b += kU * T) {
        uint4 x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t i = b + u * T;
            x[u] = i < nv ? ld_nc(v + i) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (b + u * T >= nv) break;
            const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
            if (bf) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    f(key_bf16(w[q] & 0xFFFFu));
                    f(key_bf16(w[q] >> 16));
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) f(key_f32(w[q]));
            }
        }
    }
    if (bf) {
        const uint16_t *s = (const uint16_t *)t.w;
        for (uint32_t i = (nv << 3) + threadIdx.x; i < t.n; i += T) f(key_bf16(s[i]));
    } else {
        const uint32_t *s = (const uint32_t *)t.w;
        for (uint32_t i = (nv << 2) + threadIdx.x; i < t.n; i += T) f(key_f32(s[i]));
    }
}

// Pass 0 histogram of the 15-bit digit key >> 16 (for bf16 the whole
// magnitude, so an all-bf16 plan needs pass 0 only): one 128 KB shared
// histogram per 1024-thread block, one block per SM, flushed as one global
// atomic per nonzero bin per block; hist[kBins0] counts NaN keys.
//   MODE 0 (sample): every kPruneSampleStride-th tile, plus this rank's
//     element count in hist[kBins0 + 1] -- the input of k_prune_window;
//   MODE 1 (miss): every tile, only when the windowed pass missed.
template <int MODE>
__global__ void __launch_bounds__(kHist0Threads) k_prune_hist0(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint32_t sh0[];  // [kBins0]
    __shared__ uint32_t s_nan;
    if (a.sel->done || (MODE == 1 && !a.sel->miss)) return;  // k = 0 / invalid k; no miss
    for (int i = threadIdx.x; i < kBins0; i += kHist0Threads) sh0[i] = 0u;
    if (threadIdx.x == 0) s_nan = 0u;
    __syncthreads();
    constexpr int64_t S = MODE == 0 ? kPruneSampleStride : 1;
    uint32_t nan = 0;
    PruneTile nxt;
    if (blockIdx.x * S < a.n_tiles) nxt = a.tiles[blockIdx.x * S];
    for (int64_t ti = blockIdx.x * S; ti < a.n_tiles; ti += gridDim.x * S) {
        const PruneTile t = nxt;
        if (ti + gridDim.x * S < a.n_tiles) nxt = a.tiles[ti + gridDim.x * S];  // prefetch the next descriptor
        for_keys(t, [&](uint32_t k) {
            if (k > kNanKey) ++nan;
            else atomicAdd(&sh0[k >> 16], 1u);
        });
    }
    if (nan) atomicAdd(&s_nan, nan);
    __syncthreads();
    for (int b = threadIdx.x; b < kBins0; b += kHist0Threads) {
        const uint32_t c = sh0[b];
        if (c) atomicAdd(&a.hist_local[b], (unsigned long long)c);
    }
    if (threadIdx.x == 0 && s_nan) atomicAdd(&a.hist_local[kBins0], (unsigned long long)s_nan);
    if (MODE == 0 && blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(&a.hist_local[kBins0 + 1], (unsigned long long)a.n_elems);
}

// Windowed pass 0 over every tile: keys whose digit lies in the window
// [lo, hi] (estimated from the sample, k_prune_window) go to the shared
// histogram; the others are only counted (registers), and the counts land
// in bins hi + 1 (all keys above the window) and lo - 1 (all below), so the
// histogram stays exact in total and k_prune_select<0> either finds the
// k-th key's bin inside the window or reports a miss.  bf16 vectors are
// classified two magnitudes per word with the field arithmetic of the mask
// pass (x > t <=> bit 15 of x + 0x7FFF - t); in-window keys are rare
// (≈ 1 % on config 2), so almost every key costs a few ALU operations
// instead of a shared atomic.
__global__ void __launch_bounds__(kPruneThreads) k_prune_hist0w(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t shw[kWinMax];  // bins [lo, hi], hi - lo < kWinMax
    __shared__ unsigned long long s_cnt[3];  // NaN, below, in the window
    const PruneSel *sel = a.sel;
    if (sel->done) return;
    const uint32_t lo = sel->win_lo, hi = sel->win_hi;
    DYNMO_DCHECK(lo <= hi && hi - lo < kWinMax && hi < (uint32_t)kBins0);
    uint32_t *sh0 = shw - lo;  // indexed by the digit
    for (uint32_t i = lo + threadIdx.x; i <= hi; i += kPruneThreads) sh0[i] = 0u;
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0ull;
    __syncthreads();
    constexpr uint32_t H = 0x80008000u;
    const uint32_t ch = 0x7FFFu - hi, cl = 0x8000u - lo;  // m > hi; m >= lo  (hi, lo <= 0x7FFF)
    const uint32_t CH = ch | ch << 16, CL = cl | cl << 16, CN = 0x007F007Fu;
    // per thread: keys below the window and NaN keys; the in-window keys
    // are summed from the shared bins at the end, and the keys above the
    // window = the block's keys - the rest (nothing counted on the hot path)
    unsigned long long below = 0, nan = 0, seen = 0;
    // count mode (bf16-only plan, window <= kWinCnt bins): also the count of
    // each window bin per (tile, warp range of the mask pass) -> tile_win,
    // from which the tie counts of tau's bin are gathered (no tie-count pass)
    const bool cnt = a.tile_win != nullptr && a.last_pass == 0 && hi - lo + 1 <= (uint32_t)kWinCnt;
    __shared__ uint32_t s_wc[kPruneWarps][kWinCnt];  // per warp (full tiles) / [0] per block (ragged)
    if (threadIdx.x < kPruneWarps * kWinCnt) (&s_wc[0][0])[threadIdx.x] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // the in-window counters, indexed by the digit: in count mode this warp's
    // row of s_wc (its totals, kept by lanes < kWinCnt in wtot, give the
    // window bins), else the block's window histogram
    uint32_t *const wbin = cnt ? &s_wc[w][0] - lo : sh0;
    uint32_t *const rbin = cnt ? &s_wc[0][0] - lo : sh0;  // ragged tiles: row 0
    unsigned long long wtot = 0;
    auto scalar = [&](uint32_t k) {
        if (k > kNanKey) {
            ++nan;
        } else {
            const uint32_t p = k >> 16;
            if (p < lo) ++below;
            else if (p <= hi) atomicAdd(&rbin[p], 1u);
        }
    };
    PruneTile nxt;
    if (blockIdx.x < a.n_tiles) nxt = a.tiles[blockIdx.x];
    for (int64_t ti = blockIdx.x; ti < a.n_tiles; ti += gridDim.x) {
        const PruneTile t = nxt;
        if (ti + gridDim.x < a.n_tiles) nxt = a.tiles[ti + gridDim.x];
        seen += t.n;  // every thread: the block's keys
        if (t.dtype != DYNMO_W_BF16 || t.n != kPruneTileElems) {  // f32 or ragged: per key
            if (cnt) __syncthreads();  // every warp's full-tile counts flushed (row 0 is reused here)
            for_keys(t, scalar);
            if (cnt) {  // a ragged tile's counts all go to warp range 0 (as in k_prune_tiecount)
                __syncthreads();
                if (threadIdx.x < kPruneWarps * kWinCnt)
                    a.tile_win[ti * kPruneWarps * kWinCnt + threadIdx.x] =
                        threadIdx.x < kWinCnt ? (uint16_t)s_wc[0][threadIdx.x] : (uint16_t)0;
                __syncthreads();
                if (threadIdx.x < kWinCnt) {  // warp 0, lane d: row 0's totals
                    wtot += s_wc[0][threadIdx.x];
                    s_wc[0][threadIdx.x] = 0u;
                }
                __syncthreads();
            }
            continue;
        }
        // bf16 full tile: warp w owns vectors [w VW, (w+1) VW) (the mask pass's ranges)
        constexpr int VW = (int)kPruneTileElems / 8 / kPruneWarps;
        const uint4 *v = (const uint4 *)t.w + w * VW;
        uint32_t pb = 0;    // two 16-bit counters of below-window keys (<= 64 per field per tile)
        uint32_t nacc = 0;  // bit 15 / 31 set: a NaN somewhere in this thread's vectors
        for (int g = 0; g < VW; g += kU * 32) {
            uint4 x[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) x[u] = ld_nc(v + g + u * 32 + lane);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
                uint32_t m[4], in[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    m[e] = q[e] & 0x7FFF7FFFu;
                    const uint32_t ge = m[e] + CL, ah = m[e] + CH;
                    nacc |= m[e] + CN;
                    pb += (~ge & H) >> 15;
                    in[e] = ge & ~ah & H;  // lo <= m <= hi (NaN bins dropped at the flush)
                }
                if (in[0] | in[1] | in[2] | in[3]) {  // one branch per vector (in-window keys are rare)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (in[e] & 0x8000u) atomicAdd(&wbin[m[e] & 0x7FFFu], 1u);  // (a predicated
                        if (in[e] >> 16) atomicAdd(&wbin[m[e] >> 16], 1u);        //  red.shared was slower)
                    }
                }
            }
        }
        below += (pb & 0xFFFFu) + (pb >> 16);
        if (nacc & H) {  // rare: count this thread's NaN keys of the tile
            for (int g = lane; g < VW; g += 32) {
                const uint4 x = ld_nc(v + g);
                const uint32_t q[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) nan += __popc(((q[e] & 0x7FFF7FFFu) + CN) & H);
            }
        }
        if (cnt) {  // this warp range's window-bin counts (NaN bins included, never tau's)
            __syncwarp();
            if (lane < kWinCnt) {
                const uint32_t c = s_wc[w][lane];
                a.tile_win[(ti * kPruneWarps + w) * kWinCnt + lane] = (uint16_t)c;
                wtot += c;
                s_wc[w][lane] = 0u;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (cnt) {  // the window bins from the per-warp totals (into sh0, unused in count mode)
        for (uint32_t b = lo + threadIdx.x; b <= hi; b += kPruneThreads) sh0[b] = 0u;
        __syncthreads();
        if (lane < kWinCnt && lo + lane <= hi && wtot) atomicAdd(&sh0[lo + lane], (uint32_t)wtot);
        __syncthreads();
    }
    // flush the window (bins above 0x7F80 hold NaN keys of the packed path,
    // already counted) and sum the in-window keys
    unsigned long long inw = 0;
    const uint32_t top = hi < (kNanKey >> 16) ? hi : (kNanKey >> 16);
    for (uint32_t b = lo + threadIdx.x; b <= top; b += kPruneThreads) {
        const uint32_t c = sh0[b];
        if (c) atomicAdd(&a.cw_local[1 + (b - lo)], (unsigned long long)c);
        inw += c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nan += __shfl_xor_sync(0xFFFFFFFFu, nan, o);
        below += __shfl_xor_sync(0xFFFFFFFFu, below, o);
        inw += __shfl_xor_sync(0xFFFFFFFFu, inw, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (nan) atomicAdd(&s_cnt[0], nan);
        if (below) atomicAdd(&s_cnt[1], below);
        if (inw) atomicAdd(&s_cnt[2], inw);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        DYNMO_DCHECK(seen >= s_cnt[0] + s_cnt[1] + s_cnt[2]);
        const unsigned long long above = seen - s_cnt[0] - s_cnt[1] - s_cnt[2];
        if (s_cnt[0]) atomicAdd(&a.cw_local[kCwNan], s_cnt[0]);
        if (above) atomicAdd(&a.cw_local[hi - lo + 2], above);
        if (s_cnt[1]) atomicAdd(&a.cw_local[0], s_cnt[1]);
    }
}

// Passes 1 / 2 (f32 keys only): among the keys carrying the selected prefix
// (rare), histogram of key bits 15..6 / 5..0; shared sub-histograms, one
// per warp pair.
template <int PASS>
__global__ void __launch_bounds__(kPruneThreads) k_prune_hist(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    constexpr int NB = kBins1;
    constexpr int W = kPruneThreads / 64;
    __shared__ uint32_t sh[W][NB];
    for (int i = threadIdx.x; i < W * NB; i += kPruneThreads) (&sh[0][0])[i] = 0u;
    __syncthreads();
    const PruneSel *sel = a.sel;
    if (sel->done) return;  // k = 0, invalid k, or tau already found
    const uint32_t prefix = sel->prefix;
    uint32_t *my = sh[threadIdx.x >> 6];
    PruneTile nxt;
    if (blockIdx.x < a.n_tiles) nxt = a.tiles[blockIdx.x];
    for (int64_t ti = blockIdx.x; ti < a.n_tiles; ti += gridDim.x) {
        const PruneTile t = nxt;
        if (ti + gridDim.x < a.n_tiles) nxt = a.tiles[ti + gridDim.x];
        for_keys(t, [&](uint32_t k) {
            if constexpr (PASS == 1) {
                if (k <= kNanKey && (k >> 16) == prefix) atomicAdd(&my[(k >> 6) & 1023u], 1u);
            } else {
                if (k <= kNanKey && (k >> 6) == prefix) atomicAdd(&my[k & 63u], 1u);
            }
        });
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NB; b += kPruneThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) c += sh[w][b];
        if (c) atomicAdd(&a.hist_local[b], (unsigned long long)c);
    }
}

// Block-wide (1024 threads) suffix sums over an NB-bin histogram whose
// nonzero bins lie in [rlo, rhi]: thread t owns bins [t PER, t PER + PER)
// (loaded only where they meet [rlo, rhi]); s_part[t] = the keys in the
// bins of threads >= t.  Returns the total.
template <int NB>
__device__ unsigned long long suffix_scan(const unsigned long long *h, unsigned long long *s_part, int rlo = 0,
                                          int rhi = NB - 1) {
    constexpr int PER = NB / 1024;  // bins per thread (32 or 1)
    const int tid = threadIdx.x;
    unsigned long long mine = 0;
    if (tid * PER + PER - 1 >= rlo && tid * PER <= rhi) {
        const uint4 *hv = (const uint4 *)(h + tid * PER);  // 16-byte loads (PER is 1 or even)
        if constexpr (PER >= 2) {
            constexpr int NV = PER / 2, B = NV < 8 ? NV : 8;  // batches of 8 independent loads
#pragma unroll
            for (int j0 = 0; j0 < NV; j0 += B) {
                uint4 x[B];
#pragma unroll
                for (int j = 0; j < B; ++j) x[j] = ld_nc(hv + j0 + j);
#pragma unroll
                for (int j = 0; j < B; ++j)
                    mine += ((unsigned long long)x[j].y << 32 | x[j].x) + ((unsigned long long)x[j].w << 32 | x[j].z);
            }
        } else {
            mine = h[tid];
        }
    }
    s_part[tid] = mine;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive suffix sums
        const unsigned long long add = tid + o < 1024 ? s_part[tid + o] : 0ull;
        __syncthreads();
        s_part[tid] += add;
        __syncthreads();
    }
    return s_part[0];
}

// Block-wide, after suffix_scan: the bin b with suffix(b) >= r > suffix(b+1)
// (the bin of the r-th largest key, 1 <= r <= total) and suffix(b + 1), for
// every thread.  The thread whose range holds it is found from s_part; then
// warp 0 loads that range (one bin per lane, one round of loads) and finds
// the bin by a suffix sum over the lanes and a ballot.
template <int NB>
__device__ void find_bin(const unsigned long long *h, const unsigned long long *s_part, unsigned long long r,
                         int *bin, unsigned long long *above) {
    constexpr int PER = NB / 1024;
    static_assert(PER <= 32, "one bin per lane");
    __shared__ int s_owner, s_bin;
    __shared__ unsigned long long s_above;
    const int tid = threadIdx.x;
    const unsigned long long above_thread = tid + 1 < 1024 ? s_part[tid + 1] : 0ull;
    if (tid == 0) s_owner = 0;  // (r outside [1, total] is a caller bug: stay in bounds)
    __syncthreads();
    if (above_thread < r && s_part[tid] >= r) s_owner = tid;
    __syncthreads();
    if (tid < 32) {
        const int o = s_owner, lane = tid;
        const unsigned long long base = o + 1 < 1024 ? s_part[o + 1] : 0ull;
        const unsigned long long c = lane < PER ? h[o * PER + lane] : 0ull;
        unsigned long long suf = c;  // sum of the owner's bins >= lane
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_down_sync(0xFFFFFFFFu, suf, d);
            if (lane + d < 32) suf += y;
        }
        const unsigned hit = __ballot_sync(0xFFFFFFFFu, lane < PER && base + suf >= r);
        const int b = hit ? 31 - __clz(hit) : 0;  // the highest such bin: suffix(b) >= r > suffix(b + 1)
        const unsigned long long sb1 = __shfl_sync(0xFFFFFFFFu, suf, (b + 1) & 31);
        if (lane == 0) {
            s_bin = o * PER + b;
            s_above = base + (b + 1 < PER ? sb1 : 0ull);
        }
    }
    __syncthreads();
    *bin = s_bin;
    *above = s_above;
    __syncthreads();  // s_owner / s_bin / s_above are reused by the next call
}

// Pass-0 bin window from the sample histogram (one block): the sample holds
// S of the N keys (every rank), so the k_rem-th largest key is expected near
// sample rank r = k_rem S / N; the window spans the bins of sample ranks
// r -+ (4 sqrt(r) + r / 32 + 16) (binomial 4-sigma plus 3 % for the
// tile-granular sample).  Any window is exact -- a wrong estimate only costs
// the full pass (a miss).  Clears the histograms.
__global__ void __launch_bounds__(1024) k_prune_window(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ unsigned long long s_part[1024];
    PruneSel *sel = a.sel;
    const unsigned long long *h = a.nranks > 1 ? a.hist_global : a.hist_local;
    const unsigned long long S = suffix_scan<kBins0>(h, s_part);  // non-NaN sampled keys
    const unsigned long long S_all = S + h[kBins0], N = h[kBins0 + 1];
    uint32_t lo = 0, hi = kBins0 - 1;
    if (!sel->done && S > 0 && N > 0) {
        const double r = (double)sel->k_rem * (double)S_all / (double)N;
        const double d = 4.0 * sqrt(r) + r / 32.0 + 16.0;
        const double rh = r - d, rl = ceil(r + d);
        int b;
        unsigned long long acc;
        if (rh >= 1.0 && rh <= (double)S) {
            find_bin<kBins0>(h, s_part, (unsigned long long)rh, &b, &acc);
            hi = (uint32_t)b;
        }
        if (rl <= (double)S) {
            find_bin<kBins0>(h, s_part, (unsigned long long)rl, &b, &acc);
            lo = (uint32_t)b;
        }
        if (hi - lo + 1 > kWinMax) {  // too wide for the shared window: kWinMax bins around the estimate
            const double rc = r < 1.0 ? 1.0 : (r > (double)S ? (double)S : r);
            find_bin<kBins0>(h, s_part, (unsigned long long)rc, &b, &acc);
            const uint32_t c = (uint32_t)b;
            uint32_t l2 = c >= lo + kWinMax / 2 ? c - kWinMax / 2 : lo;
            if (l2 + kWinMax - 1 > hi) l2 = hi - (kWinMax - 1);
            lo = l2;
            hi = l2 + kWinMax - 1;
        }
    } else {  // no sample (k = 0, invalid, or no keys): a window the miss path will not need
        lo = 0;
        hi = kWinMax - 1;
    }
    DYNMO_DCHECK(lo <= hi && hi - lo < kWinMax && hi < (uint32_t)kBins0);
    if (threadIdx.x == 0) {
        sel->win_lo = lo;
        sel->win_hi = hi;
        sel->miss = 0;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kBins0 + 2; b += 1024) {
        a.hist_local[b] = 0ull;
        if (a.nranks > 1) a.hist_global[b] = 0ull;
    }
}

// Pass 0 after the windowed pass (one block): the bin of the k_rem-th
// largest key in the compact histogram; a compact bin outside the window
// (all keys below / above it) is a miss, left for the full histogram and
// k_prune_select<0, 1>.  Clears the compact counters.
__global__ void __launch_bounds__(1024) k_prune_select_win(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ unsigned long long s_part[1024];
    PruneSel *sel = a.sel;
    const unsigned long long *h = a.nranks > 1 ? a.cw_global : a.cw_local;
    const uint32_t lo = sel->win_lo, W = sel->win_hi - lo + 1;
    DYNMO_DCHECK(W >= 1 && W <= kWinMax);
    const int tid = threadIdx.x;
    const bool done0 = sel->done != 0;
    if (tid == 0 && h[kCwNan]) sel->status = DYNMO_E_INVALID;  // NaN keys
    const unsigned long long total = suffix_scan<kCw>(h, s_part, 0, (int)W + 1);
    if (tid == 0) {  // the global number of non-NaN keys; validate k
        sel->n_global = (long long)total;
        if (!done0 && (sel->k > (long long)total)) {
            sel->status = DYNMO_E_INVALID;
            sel->done = 1;
        }
    }
    __syncthreads();
    const long long krem = sel->k_rem;
    if (!done0 && !sel->done && krem > 0) {
        int c;
        unsigned long long acc;
        find_bin<kCw>(h, s_part, (unsigned long long)krem, &c, &acc);
        if (tid == 0) {
            if (c == 0 || c == (int)W + 1) {
                sel->miss = 1;
            } else {
                sel->k_rem = krem - (long long)acc;
                sel->above += (long long)acc;
                sel->prefix = lo + (uint32_t)c - 1;
                sel->tie_local = (long long)a.cw_local[c];  // this rank's keys in the chosen bin
                sel->missed = 0;
                sel->wincnt = a.tile_win != nullptr && a.last_pass == 0 && W <= (uint32_t)kWinCnt;
                sel->tau_d = (uint32_t)c - 1;
                sel->miss = 0;
            }
        }
    }
    __syncthreads();
    if (tid == 0 && !done0 && !sel->done && krem == 0) sel->done = 2;  // k = 0: nothing kept
    for (int i = tid; i < (int)W + 2; i += 1024) {
        a.cw_local[i] = 0ull;
        if (a.nranks > 1) a.cw_global[i] = 0ull;
    }
    if (tid == 0) {
        a.cw_local[kCwNan] = 0ull;
        if (a.nranks > 1) a.cw_global[kCwNan] = 0ull;
    }
}

// One block: locate the bin of the k_rem-th largest key in the (global)
// histogram by a suffix scan, narrow the prefix, and clear both histograms.
// Passes 1 / 2 (f32 keys); pass 0 with MODE 1 runs after the full
// first-digit histogram, only when the windowed pass missed.
template <int PASS, int MODE>
__global__ void __launch_bounds__(1024) k_prune_select(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    constexpr int NB = PASS == 0 ? kBins0 : kBins1;
    __shared__ unsigned long long s_part[1024];
    PruneSel *sel = a.sel;
    if (MODE == 1 && !sel->miss) return;  // nothing was histogrammed
    const unsigned long long *h = a.nranks > 1 ? a.hist_global : a.hist_local;
    const int tid = threadIdx.x;
    const bool done0 = sel->done != 0;
    if (PASS == 0 && tid == 0 && h[kBins0]) sel->status = DYNMO_E_INVALID;  // NaN keys
    const unsigned long long total = suffix_scan<NB>(h, s_part);
    if (PASS == 0 && tid == 0) {  // the global number of non-NaN keys; validate k
        sel->n_global = (long long)total;
        if (!done0 && (sel->k > (long long)total)) {
            sel->status = DYNMO_E_INVALID;
            sel->done = 1;
        }
    }
    __syncthreads();
    const long long krem = sel->k_rem;
    if (!done0 && !sel->done && krem > 0) {
        int b;
        unsigned long long acc;
        find_bin<NB>(h, s_part, (unsigned long long)krem, &b, &acc);
        if (tid == 0) {
            sel->k_rem = krem - (long long)acc;
            sel->above += (long long)acc;
            sel->prefix = PASS == 0 ? (uint32_t)b
                        : PASS == 1 ? ((sel->prefix << 10) | (uint32_t)b) : ((sel->prefix << 6) | (uint32_t)b);
            // this rank's keys in the chosen bin (the ties, after the last pass)
            sel->tie_local = (long long)a.hist_local[b];
            if (PASS == 0) {  // after a miss: reported in d_info[5]; ties counted by k_prune_tiecount
                sel->missed = 1;
                sel->wincnt = 0;
            }
            sel->miss = 0;
        }
    }
    __syncthreads();
    if (tid == 0 && !done0 && !sel->done && krem == 0) sel->done = 2;  // k = 0: nothing kept
    for (int b = tid; b < NB + (PASS == 0 ? 1 : 0); b += 1024) {
        a.hist_local[b] = 0ull;
        if (a.nranks > 1) a.hist_global[b] = 0ull;
    }
}

// After the last pass: tau, and this rank's share of the ties (global order
// = rank order): tie_all[] holds every rank's tie count (all-gathered).
__global__ void k_prune_ties(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    PruneSel *sel = a.sel;
    if (threadIdx.x != 0) return;
    if (sel->done) {  // k = 0 or invalid: nothing kept
        sel->keep_ties = 0;
        sel->partial = 0;
        sel->tau = 0xFFFFFFFFu;
        return;
    }
    // tau from the digits: 15 bits (bf16-only plans) or 15 + 10 + 6 = 31 bits
    sel->tau = a.last_pass == 0 ? (sel->prefix << 16) : sel->prefix;
    long long before = 0;
    for (int r = 0; r < a.rank; ++r) before += a.nranks > 1 ? a.tie_all[r] : 0;
    const long long need = sel->k_rem;  // ties to keep globally (>= 1)
    long long mine = need - before;
    mine = mine < 0 ? 0 : (mine > sel->tie_local ? sel->tie_local : mine);
    sel->keep_ties = mine;
    sel->partial = mine > 0 && mine < sel->tie_local;
}

// Ties (keys == tau) per (tile, warp range), only for a partial share.
// Full tiles: warp w counts its contiguous vectors [w VW, (w+1) VW) -- the
// ranges the mask pass gives each warp; a ragged tile puts its whole count
// in entry 0 (the mask pass ranks it with block scans from the tile start).
__global__ void __launch_bounds__(kPruneThreads) k_prune_tiecount(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    const PruneSel *sel = a.sel;
    if (!sel->partial) return;
    if (sel->wincnt) {  // counted by the windowed pass: gather tau's bin column, and tile totals
        const uint32_t d = sel->tau_d;
        DYNMO_DCHECK(d < (uint32_t)kWinCnt && a.tile_win != nullptr);
        for (int64_t ti = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ti < a.n_tiles;
             ti += (int64_t)gridDim.x * blockDim.x) {
            uint32_t c[kPruneWarps], tot = 0;
#pragma unroll
            for (int w = 0; w < kPruneWarps; ++w) {
                c[w] = a.tile_win[(ti * kPruneWarps + w) * kWinCnt + d];
                tot += c[w];
            }
            uint4 *tt = (uint4 *)(a.tile_ties + ti * kPruneWarps);
            tt[0] = make_uint4(c[0], c[1], c[2], c[3]);
            tt[1] = make_uint4(c[4], c[5], c[6], c[7]);
            a.tile_tot[ti] = tot;
        }
        return;
    }
    const uint32_t tau = sel->tau;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __shared__ uint32_t s_c;
    PruneTile nxt;
    if (blockIdx.x < a.n_tiles) nxt = a.tiles[blockIdx.x];
    for (int64_t ti = blockIdx.x; ti < a.n_tiles; ti += gridDim.x) {
        const PruneTile t = nxt;
        if (ti + gridDim.x < a.n_tiles) nxt = a.tiles[ti + gridDim.x];
        if (t.n == kPruneTileElems) {
            const bool bf = t.dtype == DYNMO_W_BF16;
            const int VW = (int)kPruneTileElems / (bf ? 8 : 4) / kPruneWarps;
            const uint4 *v = (const uint4 *)t.w + w * VW;
            uint32_t c = 0;
            for (int b = lane; b < VW; b += kU * 32) {
                uint4 x[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) x[u] = b + 32 * u < VW ? ld_nc(v + b + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if (b + 32 * u >= VW) break;
                    const uint32_t q[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (bf) c += (key_bf16(q[e] & 0xFFFFu) == tau) + (key_bf16(q[e] >> 16) == tau);
                        else c += key_f32(q[e]) == tau;
                    }
                }
            }
            c = __reduce_add_sync(0xFFFFFFFFu, c);
            if (lane == 0) a.tile_ties[ti * kPruneWarps + w] = c;
        } else {
            if (threadIdx.x == 0) s_c = 0u;
            __syncthreads();
            uint32_t c = 0;
            for_keys(t, [&](uint32_t k) { c += k == tau; });
            c = __reduce_add_sync(0xFFFFFFFFu, c);
            if (lane == 0 && c) atomicAdd(&s_c, c);
            __syncthreads();
            if (threadIdx.x < kPruneWarps) a.tile_ties[ti * kPruneWarps + threadIdx.x] = threadIdx.x == 0 ? s_c : 0u;
            __syncthreads();
        }
    }
}

// Exclusive scan of the per-tile tie totals (sum of the tile's warp-range
// counts; one block of 32 warps, only if partial): each warp owns a
// contiguous range of tiles read coalesced in chunks of 32 (4 chunks of
// loads in flight): warp totals, a scan over the 32 warps, then per chunk a
// warp scan plus the running offset.
__global__ void __launch_bounds__(1024) k_prune_tiescan(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    if (!a.sel->partial) return;
    __shared__ unsigned long long s_w[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t n = a.n_tiles;
    const int64_t per = (n + 31) / 32;
    const int64_t b0 = w * per, e0 = b0 + per < n ? b0 + per : n;
    const bool tot_ready = a.sel->wincnt != 0;  // the gather wrote per-tile totals
    auto total = [&](int64_t i) -> unsigned long long {  // tile i's ties (8 warp ranges, 32 B)
        if (i >= e0) return 0ull;
        if (tot_ready) return a.tile_tot[i];
        const uint4 *p = (const uint4 *)(a.tile_ties + i * kPruneWarps);
        const uint4 x = p[0], y = p[1];
        return (unsigned long long)x.x + x.y + x.z + x.w + y.x + y.y + y.z + y.w;
    };
    unsigned long long tot = 0;
    for (int64_t c = b0; c < e0; c += 4 * 32) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = total(c + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 4; ++u) tot += v[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
    if (lane == 0) s_w[w] = tot;
    __syncthreads();
    unsigned long long run = 0;
    for (int u = 0; u < w; ++u) run += s_w[u];
    for (int64_t c = b0; c < e0; c += 4 * 32) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = total(c + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            unsigned long long incl = v[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            const int64_t i = c + u * 32 + lane;
            if (i < e0) a.tile_off[i] = run + incl - v[u];
            run += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
    }
}

// Full tile (kPruneTileElems elements, 16-byte aligned): warp w owns the
// contiguous vectors [w VW, (w+1) VW) and walks them in groups of 4 x 32
// (lane L loads vector g*256 + u*32 + L: kU coalesced 16-byte loads in
// flight).  A tie's rank in element order = the warp range's offset (from
// the tie-count scan) + ties earlier in the range (u-major, lane-minor warp
// scans -- skipped when no lane of the warp holds a tie -- and a running
// count) + its position in the vector.  No block barrier.  Masks stored per
// vector (8 or 4 bytes, coalesced).
//
// bf16 full tile, two magnitudes per 32-bit word: m = w & 0x7FFF7FFF holds
// two 15-bit fields, and for a field value x <= 0x7FFF and t <= 0x7FFF,
// x > t  <=>  bit 15 of x + (0x7FFF - t), with no carry out of the field.
// For a bf16 key (m << 16): key > tau <=> m > tau >> 16; key == tau <=>
// m == tau >> 16 and tau's low half is 0; NaN <=> m > 0x7F80.  The flags
// sit in bits 15 / 31; one byte permute per word pair gathers the four
// flag bytes in element order.  Same ranks and masks as the general path.
__device__ __forceinline__ void mask_full_tile_bf16(const PruneTile &t, uint32_t tau, bool partial, bool all_ties,
                                                    long long keep_ties, unsigned long long wbase) {
    constexpr int VW = (int)kPruneTileElems / 8 / kPruneWarps;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint4 *v = (const uint4 *)t.w + w * VW;
    const bool al = ((uintptr_t)t.mask & 7u) == 0;
    const uint32_t t16 = tau >> 16;
    const uint32_t cg = t16 >= 0x7FFFu ? 0u : 0x7FFFu - t16;                  // > t16
    const uint32_t ce = (t16 > 0x7FFFu || (tau & 0xFFFFu)) ? 0u : 0x8000u - t16;  // >= t16 (ties possible)
    const uint32_t CG = cg | cg << 16, CE = ce | ce << 16, CN = 0x007F007Fu;   // CN: > 0x7F80 (NaN)
    const bool tie_flags = partial || all_ties;
    unsigned long long run = wbase;
    for (int g = 0; g < VW; g += kU * 32) {
        uint4 x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) x[u] = ld_nc(v + g + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t q[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
            uint32_t kp[4], eq[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t m = q[e] & 0x7FFF7FFFu;
                const uint32_t gt = m + CG, nan = m + CN;
                kp[e] = gt & ~nan & 0x80008000u;
                eq[e] = tie_flags ? (m + CE) & ~gt & 0x80008000u : 0u;
            }
            uint32_t m0 = (__byte_perm(kp[0], kp[1], 0x7531) >> 7) & 0x01010101u;
            uint32_t m1 = (__byte_perm(kp[2], kp[3], 0x7531) >> 7) & 0x01010101u;
            const uint32_t e0 = (__byte_perm(eq[0], eq[1], 0x7531) >> 7) & 0x01010101u;
            const uint32_t e1 = (__byte_perm(eq[2], eq[3], 0x7531) >> 7) & 0x01010101u;
            if (!partial) {
                m0 |= e0;  // all of this rank's ties kept (e0/e1 are 0 when none are)
                m1 |= e1;
            } else {
                const uint32_t c = __popc(e0) + __popc(e1);
                if (__any_sync(0xFFFFFFFFu, c != 0)) {  // most warp vectors hold no tie
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    unsigned long long r = run + incl - c;  // rank of this lane's first tie
                    run += __shfl_sync(0xFFFFFFFFu, incl, 31);
                    if (c) {
                        uint32_t f0 = e0, f1 = e1;  // ties in element order: bytes of m0, then m1
                        while (f0) {
                            const uint32_t b = f0 & (0u - f0);
                            if (r++ < (unsigned long long)keep_ties) m0 |= b;
                            f0 ^= b;
                        }
                        while (f1) {
                            const uint32_t b = f1 & (0u - f1);
                            if (r++ < (unsigned long long)keep_ties) m1 |= b;
                            f1 ^= b;
                        }
                    }
                }
            }
            uint8_t *mk = t.mask + (int64_t)(w * VW + g + u * 32 + lane) * 8;
            if (al) {
                *(uint2 *)mk = make_uint2(m0, m1);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) mk[e] = (uint8_t)(((e < 4 ? m0 : m1) >> (8 * (e & 3))) & 1u);
            }
        }
    }
}

// f32 full tile: 4 keys per vector, compared directly.
__device__ __forceinline__ void mask_full_tile_f32(const PruneTile &t, uint32_t tau, bool partial, bool all_ties,
                                                   long long keep_ties, unsigned long long wbase) {
    constexpr int VW = (int)kPruneTileElems / 4 / kPruneWarps;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint4 *v = (const uint4 *)t.w + w * VW;
    const bool al = ((uintptr_t)t.mask & 3u) == 0;
    unsigned long long run = wbase;
    for (int g = 0; g < VW; g += kU * 32) {
        uint4 x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) x[u] = ld_nc(v + g + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t keys[4] = {key_f32(x[u].x), key_f32(x[u].y), key_f32(x[u].z), key_f32(x[u].w)};
            unsigned long long before = 0;
            uint32_t c = 0;
            if (partial) {
#pragma unroll
                for (int e = 0; e < 4; ++e) c += keys[e] == tau;
            }
            if (__any_sync(0xFFFFFFFFu, c != 0)) {  // most warp vectors hold no tie: skip the scan
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += y;
                }
                before = run + incl - c;
                run += __shfl_sync(0xFFFFFFFFu, incl, 31);
            }
            uint32_t m = 0u, seen = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t k = keys[e];
                bool keep = k > tau && k <= kNanKey;
                if (k == tau) {
                    keep = partial ? (before + seen < (unsigned long long)keep_ties) : all_ties;
                    ++seen;
                }
                m |= (keep ? 1u : 0u) << (8 * e);
            }
            uint8_t *mk = t.mask + (int64_t)(w * VW + g + u * 32 + lane) * 4;
            if (al) {
                *(uint32_t *)mk = m;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) mk[e] = (uint8_t)((m >> (8 * e)) & 1u);
            }
        }
    }
}

// Masks (ragged last tile of a segment: thread-contiguous chunks of 16):
// keep key > tau; keys == tau kept when all of this rank's ties are
// (non-partial share) or, for a partial share, when their rank in element
// order (tile offset + in-tile block scan over thread-contiguous chunks) is
// below keep_ties.  16 elements per thread per step, 16-byte mask stores.
__global__ void __launch_bounds__(kPruneThreads) k_prune_mask(PruneArgs a) {
    pdl_wait();
    pdl_trigger();
    const PruneSel *sel = a.sel;
    const uint32_t tau = sel->tau;
    const bool all_ties = sel->keep_ties > 0 && !sel->partial;
    const bool partial = sel->partial != 0;
    const long long keep_ties = sel->keep_ties;
    __shared__ uint32_t s_warp[kPruneThreads / 32];
    PruneTile nxt;
    if (blockIdx.x < a.n_tiles) nxt = a.tiles[blockIdx.x];
    for (int64_t ti = blockIdx.x; ti < a.n_tiles; ti += gridDim.x) {
        const PruneTile t = nxt;
        if (ti + gridDim.x < a.n_tiles) nxt = a.tiles[ti + gridDim.x];
        if (t.n == kPruneTileElems) {  // the common case: coalesced fast path, no barriers
            unsigned long long wb = 0;
            if (partial) {  // tile offset + the earlier warp ranges of this tile
                wb = a.tile_off[ti];
                for (int u = 0; u < (int)(threadIdx.x >> 5); ++u) wb += a.tile_ties[ti * kPruneWarps + u];
            }
            if (t.dtype == DYNMO_W_BF16) mask_full_tile_bf16(t, tau, partial, all_ties, keep_ties, wb);
            else mask_full_tile_f32(t, tau, partial, all_ties, keep_ties, wb);
            continue;
        }
        unsigned long long run = partial ? a.tile_off[ti] : 0ull;  // ties before this chunk
        const uint32_t nchunk = (t.n + 16 * kPruneThreads - 1) / (16 * kPruneThreads);
        for (uint32_t ch = 0; ch < nchunk; ++ch) {
            const uint32_t e0 = ch * 16 * kPruneThreads + threadIdx.x * 16;  // 16 elements per thread
            uint32_t keys[16];
            const uint32_t ne = e0 < t.n ? (t.n - e0 < 16 ? t.n - e0 : 16) : 0;
            if (t.dtype == DYNMO_W_BF16) {
                const uint16_t *s = (const uint16_t *)t.w + e0;
                if (ne == 16) {
                    const uint4 x0 = ld_nc((const uint4 *)s), x1 = ld_nc((const uint4 *)s + 1);
                    const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        keys[2 * q] = key_bf16(w[q] & 0xFFFFu);
                        keys[2 * q + 1] = key_bf16(w[q] >> 16);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) keys[q] = q < (int)ne ? key_bf16(s[q]) : 0xFFFFFFFFu;
                }
            } else {
                const uint32_t *s = (const uint32_t *)t.w + e0;
                if (ne == 16) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 x = ld_nc((const uint4 *)s + q);
                        keys[4 * q] = key_f32(x.x);
                        keys[4 * q + 1] = key_f32(x.y);
                        keys[4 * q + 2] = key_f32(x.z);
                        keys[4 * q + 3] = key_f32(x.w);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) keys[q] = q < (int)ne ? key_f32(s[q]) : 0xFFFFFFFFu;
                }
            }
            // rank of this thread's first tie among the chunk's ties (block
            // scan, every thread takes part: the barriers are uniform)
            uint32_t before = 0;
            const unsigned long long base = run;
            if (partial) {
                uint32_t c = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) c += keys[q] == tau;
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if ((threadIdx.x & 31) >= o) incl += y;
                }
                if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = incl;
                __syncthreads();
                uint32_t wbefore = 0, tot = 0;
#pragma unroll
                for (int w = 0; w < kPruneThreads / 32; ++w) {
                    wbefore += w < (int)(threadIdx.x >> 5) ? s_warp[w] : 0u;
                    tot += s_warp[w];
                }
                __syncthreads();  // s_warp is rewritten by the next chunk
                before = wbefore + incl - c;
                run += tot;  // uniform across the block
            }
            if (ne > 0) {
                uint32_t m[4] = {0u, 0u, 0u, 0u};
                uint32_t seen = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const uint32_t k = keys[q];
                    bool keep = k > tau && k <= kNanKey;
                    if (k == tau && q < (int)ne) {
                        keep = partial ? (base + before + seen < (unsigned long long)keep_ties) : all_ties;
                        ++seen;
                    }
                    m[q >> 2] |= (keep ? 1u : 0u) << (8 * (q & 3));
                }
                uint8_t *mk = t.mask + e0;
                if (ne == 16 && (((uintptr_t)mk) & 15u) == 0) {
                    *(uint4 *)mk = make_uint4(m[0], m[1], m[2], m[3]);
                } else {
                    for (uint32_t q = 0; q < ne; ++q) mk[q] = (uint8_t)((m[q >> 2] >> (8 * (q & 3))) & 1u);
                }
            }
        }
    }
}

// This rank's kept count and the info vector (one thread).
__global__ void k_prune_info(PruneArgs a, long long *d_info, int32_t *d_status) {
    pdl_wait();
    pdl_trigger();
    PruneSel *sel = a.sel;
    if (threadIdx.x != 0) return;
    const bool none = sel->done != 0;
    if (d_info) {
        d_info[0] = none ? -1 : (long long)sel->tau;
        d_info[1] = sel->n_global;
        d_info[2] = none ? 0 : sel->above;
        d_info[3] = none ? 0 : sel->keep_ties;
        d_info[4] = none ? 0 : sel->tie_local;
        d_info[5] = sel->missed | (sel->partial && sel->wincnt ? 2 : 0);  // flags
    }
    if (d_status) *d_status = sel->status;
}

}  // namespace

// Reset the selection state for a call (k is the global keep count).
__global__ void k_prune_begin(PruneSel *sel, long long k) {
    pdl_wait();
    pdl_trigger();
    sel->k = k;
    sel->k_rem = k;
    sel->above = 0;
    sel->prefix = 0u;
    sel->tau = 0xFFFFFFFFu;
    sel->tie_local = 0;
    sel->keep_ties = 0;
    sel->partial = 0;
    sel->status = DYNMO_OK;
    sel->n_global = 0;
    sel->done = 0;
    sel->win_lo = 0u;
    sel->win_hi = 0x7FFFu;
    sel->miss = 0;
    sel->missed = 0;
    sel->wincnt = 0;
}

// Resident blocks per SM of the streaming kernels (grid = SMs x this).
int prune_blocks_per_sm(int kind) {
    int nb = 1;
    switch (kind) {
        case 0: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_hist0w, kPruneThreads, 0); break;
        case 30:
        case 32:  // the full-width histogram passes (sample, miss): 128 KB of shared memory
            cudaFuncSetAttribute(k_prune_hist0<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins0 * 4);
            cudaFuncSetAttribute(k_prune_hist0<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBins0 * 4);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_hist0<1>, kHist0Threads, kBins0 * 4);
            break;
        case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_hist<1>, kPruneThreads, 0); break;
        case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_hist<2>, kPruneThreads, 0); break;
        case 21: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_tiecount, kPruneThreads, 0); break;
        default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_prune_mask, kPruneThreads, 0); break;
    }
    return nb > 0 ? nb : 1;
}

cudaError_t launch_prune(const PruneArgs &a, int pass_kind, int grid, cudaStream_t s) {
    switch (pass_kind) {
        case 0: return launch_pdl(k_prune_hist0w, grid, kPruneThreads, 0, s, a);
        case 30: return launch_pdl(k_prune_hist0<0>, grid, kHist0Threads, (size_t)kBins0 * 4, s, a);
        case 31: return launch_pdl(k_prune_window, 1, 1024, 0, s, a);
        case 32: return launch_pdl(k_prune_hist0<1>, grid, kHist0Threads, (size_t)kBins0 * 4, s, a);
        case 1: return launch_pdl(k_prune_hist<1>, grid, kPruneThreads, 0, s, a);
        case 2: return launch_pdl(k_prune_hist<2>, grid, kPruneThreads, 0, s, a);
        case 10: return launch_pdl(k_prune_select_win, 1, 1024, 0, s, a);
        case 11: return launch_pdl(k_prune_select<1, 0>, 1, 1024, 0, s, a);
        case 12: return launch_pdl(k_prune_select<2, 0>, 1, 1024, 0, s, a);
        case 13: return launch_pdl(k_prune_select<0, 1>, 1, 1024, 0, s, a);
        case 20: return launch_pdl(k_prune_ties, 1, 32, 0, s, a);
        case 21: return launch_pdl(k_prune_tiecount, grid, kPruneThreads, 0, s, a);
        case 22: return launch_pdl(k_prune_tiescan, 1, 1024, 0, s, a);
        case 23: return launch_pdl(k_prune_mask, grid, kPruneThreads, 0, s, a);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_prune_begin(PruneSel *sel, long long k, cudaStream_t s) {
    return launch_pdl(k_prune_begin, 1, 1, 0, s, sel, k);
}

cudaError_t launch_prune_info(const PruneArgs &a, long long *d_info, int32_t *d_status, cudaStream_t s) {
    return launch_pdl(k_prune_info, 1, 32, 0, s, a, d_info, d_status);
}

}  // namespace dynmo

// k_profile.cu -- per-layer workload profiling on sm_100a.
//
//  k_profile   one fused, persistent, HBM-streaming kernel over every tile of
//              every segment: 128-bit non-allocating loads (8 in flight per
//              lane), branch-free SWAR counting, warp __reduce_add_sync, one
//              64-bit atomic per tile (integer sums are order independent, so
//              the result is bit-exact and deterministic).
//              Sources: pruning masks, token masks / exit depths
//              (P:L340-353), MoE expert ids.
//  k_epilogue  counters -> int64 cost c_i (a5, readings Q1-Q6) with 128-bit
//              checked arithmetic; consumes and clears the accumulators.
//  k_unpack    after the NCCL all-gather of fixed per-rank slots, scatters
//              every rank's slice into the global cost / mem vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "dynmo_internal.h"

namespace dynmo {

#ifdef DYNMO_STEP_STAMPS
__device__ unsigned long long g_step_stamp[STAMP_N][2];
#endif
void diag_stamps_profile(unsigned long long *h, bool reset) {
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

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Nonzero bytes of a 32-bit word: high bit of each byte of t is set iff the
// byte is nonzero ((b & 0x7f) + 0x7f carries into bit 7 unless b & 0x7f == 0;
// OR-ing b restores b == 0x80).  No carry crosses a byte.
__device__ __forceinline__ uint32_t nz8(uint32_t w) {
    uint32_t t = ((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w;
    return __popc(t & 0x80808080u);
}
// Nonzero bf16 halves ignoring the sign bit.
__device__ __forceinline__ uint32_t nz16(uint32_t w) {
    uint32_t t = (w & 0x7FFF7FFFu) + 0x7FFF7FFFu;
    return __popc(t & 0x80008000u);
}
__device__ __forceinline__ uint32_t nz32(uint32_t w) { return (w & 0x7FFFFFFFu) != 0u; }

template <int OPK>
__device__ __forceinline__ uint32_t count_word(uint32_t w) {
    if constexpr (OPK == OP_POPC) return __popc(w);
    else if constexpr (OPK == OP_NZ8) return nz8(w);
    else if constexpr (OPK == OP_NZ16) return nz16(w);
    else return nz32(w);
}

template <int OPK>
__device__ __forceinline__ uint32_t count_vec(uint4 v) {
    return count_word<OPK>(v.x) + count_word<OPK>(v.y) + count_word<OPK>(v.z) +
           count_word<OPK>(v.w);
}

// Vector tile: every lane streams 16-byte vectors, 8 loads in flight.  A
// zero vector counts 0 for every count op, so out-of-range lanes load zero.
template <int OPK>
__device__ __forceinline__ uint32_t count_tile(const uint4 *p, uint32_t nvec, int lane) {
    constexpr int U = 8;
    uint32_t acc = 0;
    for (uint32_t base = 0; base < nvec; base += 32u * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t idx = base + (uint32_t)u * 32u + (uint32_t)lane;
            v[u] = idx < nvec ? ld_stream(p + idx) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += count_vec<OPK>(v[u]);
    }
    return acc;
}

// Scalar tile (< 16 bytes, or one partial byte of a bit mask).
__device__ __forceinline__ uint32_t count_scalar(const ProfTile &t, int kind, int lane) {
    const uint8_t *b = (const uint8_t *)t.ptr;
    uint32_t c = 0;
    switch (kind) {
        case OP_POPC:
            if ((uint32_t)lane < t.nbytes) {
                uint32_t v = b[lane];
                if (t.bits && (uint32_t)lane == t.nbytes - 1) v &= (1u << t.bits) - 1u;
                c = __popc(v);
            }
            break;
        case OP_NZ8:
            if ((uint32_t)lane < t.nbytes) c = b[lane] != 0;
            break;
        case OP_NZ16:
            if ((uint32_t)lane < t.nbytes / 2) c = (((const uint16_t *)b)[lane] & 0x7FFFu) != 0;
            break;
        case OP_NZ32:
            if ((uint32_t)lane < t.nbytes / 4) c = nz32(((const uint32_t *)b)[lane]);
            break;
    }
    return c;
}

__device__ __forceinline__ uint32_t count_vec_rt(int kind, uint4 v) {
    switch (kind) {
        case OP_POPC: return count_vec<OP_POPC>(v);
        case OP_NZ8: return count_vec<OP_NZ8>(v);
        case OP_NZ16: return count_vec<OP_NZ16>(v);
        default: return count_vec<OP_NZ32>(v);
    }
}

// ---------------------------------------------- MoE ids, E <= 16 (a3)
// One-hot counting in 8-bit fields of 64-bit registers: expert x adds
// 1 << 8x to acc0 (x < 8) or 1 << 8(x-8) to acc1 (8 <= x < 16).  The shift
// amount is clamped to 64 first (min(x, 8) * 8), and shl.b64 by 64 is 0, so
// ids outside [0, 8) / [8, 16) add nothing and no branch is taken.
__device__ __forceinline__ unsigned long long onehot8(uint32_t x) {
    unsigned long long r;
    const uint32_t sh = (x < 8u ? x : 8u) << 3;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(1ull), "r"(sh));
    return r;
}

// Validation of the ids without per-entry compares on 64 bits: a valid id
// has a zero high word (int64) and a low word < E; OR of the high words and
// the max of the low words (unsigned: a negative int32 id is >= 2^31) over
// the tile decide it once per tile.
template <int ESZ, bool E16>
struct ExpertLane {
    unsigned long long acc0 = 0, acc1 = 0;
    uint32_t hi = 0, mx = 0;
    __device__ __forceinline__ void id(uint32_t x) {
        mx = x > mx ? x : mx;
        acc0 += onehot8(x);
        if constexpr (E16) acc1 += onehot8(x - 8u);  // x < 8 wraps to >= 2^32-8: adds 0
    }
    __device__ __forceinline__ void vec(const uint4 &v) {
        if constexpr (ESZ == 8) {
            hi |= v.y | v.w;
            id(v.x);
            id(v.z);
        } else {
            id(v.x);
            id(v.y);
            id(v.z);
            id(v.w);
        }
    }
};

__device__ __forceinline__ bool small_count_tile(const ProfTile &t) {
    return (t.op & 0xF) <= OP_NZ32 && !(t.op & (OP_SCALAR | OP_STRIDED)) && (t.nbytes >> 4) <= 32;
}

// Strided tile (bit masks: MASK_BITS / TOKMASK_BITS): k whole layers of S >= 32 vectors each (one per warp lane
// and chunk).  Each warp iteration covers 8 layers: one 16-byte load per
// lane per layer (8 loads in flight, each load instruction reading 512
// contiguous bytes of one layer), chunks of 32 vectors accumulated for
// S > 32, then one warp reduction per layer and lane u adds layer g0 + u's
// count with one 64-bit atomic (distinct layers: no same-address contention,
// and no per-layer descriptor to fetch).
__device__ __forceinline__ void count_strided(const ProfTile &t, int lane, unsigned long long *acc) {
    const uint32_t S = t.bits;
    const uint32_t k = t.nbytes / (S * 16u);
    const uint4 *p = (const uint4 *)t.ptr;
    for (uint32_t g0 = 0; g0 < k; g0 += 8u) {
        uint32_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = 0u;
        for (uint32_t x = (uint32_t)lane; x < S; x += 32u) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = g0 + u < k ? ld_stream(p + (size_t)(g0 + u) * S + x) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] += count_vec<OP_POPC>(v[u]);
        }
        uint32_t mine = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t r = __reduce_add_sync(0xFFFFFFFFu, c[u]);
            mine = lane == u ? r : mine;
        }
        if (lane < 8 && g0 + lane < k && mine)
            atomicAdd(&acc[(int64_t)(t.layer + (int32_t)(g0 + lane)) * ACC_N + t.aux], (unsigned long long)mine);
    }
}

// One tile of E <= 16 expert ids: 8 x 16-byte loads in flight per lane (as
// the count ops), full batches without bounds predicates, the ragged last
// batch predicated; fields spilled to the warp counters before they can
// reach 256 (nacc is warp-uniform: every lane adds the batch maximum).
template <int ESZ, bool E16, typename Spill>
__device__ __forceinline__ void expert_small(const ProfTile &t, bool scalar, int lane, uint32_t E,
                                             unsigned long long &acc0, unsigned long long &acc1,
                                             uint32_t &nacc, uint32_t &bad, Spill &spill) {
    ExpertLane<ESZ, E16> el;
    el.acc0 = acc0;
    el.acc1 = acc1;
    constexpr int U = 8;
    constexpr uint32_t PER = U * (16 / ESZ);  // ids per lane per batch
    if (scalar) {
        if (nacc > 254u) {
            acc0 = el.acc0;
            acc1 = el.acc1;
            spill();
            el.acc0 = el.acc1 = 0;
        }
        const uint32_t ne = t.nbytes / ESZ;
        if ((uint32_t)lane < ne) {
            if constexpr (ESZ == 8) {
                const uint2 w = ((const uint2 *)t.ptr)[lane];
                el.hi |= w.y;
                el.id(w.x);
            } else {
                el.id(((const uint32_t *)t.ptr)[lane]);
            }
        }
        nacc += 1;
    } else {
        const uint4 *p = (const uint4 *)t.ptr;
        const uint32_t nvec = t.nbytes >> 4;
        const uint32_t nfull = nvec / (32u * U) * (32u * U);
        for (uint32_t base = 0; base < nvec; base += 32u * U) {
            if (nacc > 255u - PER) {
                acc0 = el.acc0;
                acc1 = el.acc1;
                spill();
                el.acc0 = el.acc1 = 0;
            }
            uint4 v[U];
            if (base < nfull) {
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = ld_stream(p + base + (uint32_t)u * 32u + (uint32_t)lane);
#pragma unroll
                for (int u = 0; u < U; ++u) el.vec(v[u]);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t idx = base + (uint32_t)u * 32u + (uint32_t)lane;
                    v[u] = idx < nvec ? ld_stream(p + idx) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (base + (uint32_t)u * 32u + (uint32_t)lane < nvec) el.vec(v[u]);
            }
            nacc += PER;
        }
    }
    acc0 = el.acc0;
    acc1 = el.acc1;
    bad |= (el.hi != 0u) | (el.mx >= E);
}

// OPS: bit 0 count ops present, bit 1 exit histogram, bit 2 expert histograms,
// bit 3 expert layers with E > 16 (paths of absent op families are compiled
// out: fewer registers, more resident warps).
template <int OPS>
__global__ void __launch_bounds__(kProfThreads, (OPS == 1 || OPS == 4) ? 4 : (OPS & 8) ? 2 : 3) k_profile(ProfArgs a) {
    pdl_trigger();  // the epilogue may be scheduled now (it waits for this grid)
    STEP_STAMP(STAMP_PROFILE);
    if (a.span && threadIdx.x == 0) atomicMax(&a.span[0], ~globaltimer_ns());  // ~start: zero-reset max
    constexpr bool HAS_CNT = OPS & 1, HAS_EXIT = (OPS & 2) != 0, HAS_EXP = (OPS & 4) != 0;
    constexpr bool HAS_BIGE = (OPS & 8) != 0;  // some expert layer has E > 16 (smem histograms)
    constexpr bool HAS_HIST = HAS_EXIT || HAS_EXP;
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t warp = (int64_t)blockIdx.x * (kProfThreads / 32) + wib;
    const int64_t nwarps = (int64_t)gridDim.x * (kProfThreads / 32);
    // Per-warp histogram scratch (a.warp_words u32, sized by the plan: exit
    // bins and/or expert columns); zero at entry and after every flush.
    uint32_t *sh = nullptr;
    if constexpr (HAS_HIST) {
        sh = smem + wib * a.warp_words;
        for (int i = lane; i < a.warp_words; i += 32) sh[i] = 0u;
        __syncwarp();
    }
    // Each warp walks a CONTIGUOUS range of tiles: consecutive tiles mostly
    // belong to the same layer, so counts accumulate in a register and one
    // atomic is issued per (layer, slot) run instead of one per tile (thousands
    // of same-address atomics serialise in L2 when a layer spans many tiles).
    // The next tile descriptor is prefetched while the current one streams.
    const int64_t per = (a.n_tiles + nwarps - 1) / nwarps;
    const int64_t t_beg = warp * per;
    const int64_t t_end = t_beg + per < a.n_tiles ? t_beg + per : a.n_tiles;
    if (a.l2_prefetch) {
        // the warp's tiles are read once, soon: one fire-and-forget L2 bulk
        // prefetch per vector tile (lane j: tile t_beg + j, then + 32 ...)
        for (int64_t ti = t_beg + lane; ti < t_end; ti += 32) {
            const ProfTile d = a.tiles[ti];
            if (!(d.op & OP_SCALAR) && (d.op & 0xF) != OP_TIME && d.nbytes >= 16u)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.ptr), "r"(d.nbytes & ~15u)
                             : "memory");
        }
    }
    int64_t run_key = -1;
    unsigned long long run_sum = 0;
    int exit_dirty = 0;       // exit histogram pending in sh (flushed once at the end)
    int hist_layer = -1;      // layer whose expert histogram is pending
    int hist_E = 0;
    uint32_t bad = 0;         // an expert id outside [0, E)
    // E <= 16: one-hot 8-bit fields in registers (experts 0-7 in acc0, 8-15 in
    // acc1), spilled every <= 240 entries per lane into mycnt (lane e holds
    // the warp's count of expert e) with warp reductions
    unsigned long long acc0 = 0, acc1 = 0;
    uint32_t nacc = 0, mycnt = 0;
    auto spill_regs = [&]() {
        if (__any_sync(0xFFFFFFFFu, nacc != 0)) {
#pragma unroll
            for (int f = 0; f < 16; ++f) {
                const uint32_t fv = (uint32_t)(((f < 8 ? acc0 : acc1) >> (8 * (f & 7))) & 0xFFull);
                const uint32_t sum = __reduce_add_sync(0xFFFFFFFFu, fv);
                if (lane == f) mycnt += sum;
            }
        }
        acc0 = acc1 = 0;
        nacc = 0;
    };
    auto feed = [&](int64_t key, unsigned long long c) {
        if (key != run_key) {
            DYNMO_DCHECK(run_key < 0 || run_key < (int64_t)a.n_local * ACC_N);
            if (lane == 0 && run_sum) atomicAdd(&a.acc[run_key], run_sum);
            run_key = key;
            run_sum = 0;
        }
        run_sum += c;
    };
    auto flush_experts = [&]() {
        if constexpr (HAS_HIST) {
            if (hist_layer < 0) return;
            DYNMO_DCHECK(hist_layer < a.n_local && hist_E <= a.max_E);
            DYNMO_DCHECK(hist_E <= 16 || (hist_E <= kColExperts ? 32 * hist_E : hist_E) <= a.warp_words);
            unsigned long long *dst = a.hist + (int64_t)hist_layer * a.max_E;
            if (hist_E <= 16) {
                spill_regs();
                if (lane < hist_E && mycnt) atomicAdd(&dst[lane], (unsigned long long)mycnt);
                mycnt = 0;
                hist_layer = -1;
                return;
            }
            __syncwarp();
            const bool cols = hist_E <= kColExperts;
            for (int e = lane; e < hist_E; e += 32) {
                uint32_t c = 0;
                if (cols) {
                    for (int l = 0; l < 32; ++l) {
                        c += sh[e * 32 + l];
                        sh[e * 32 + l] = 0u;
                    }
                } else {
                    c = sh[e];
                    sh[e] = 0u;
                }
                if (c) atomicAdd(&dst[e], (unsigned long long)c);
            }
            __syncwarp();
            hist_layer = -1;
        }
    };
    ProfTile nxt;
    if (t_beg < t_end) nxt = a.tiles[t_beg];
    for (int64_t ti = t_beg; ti < t_end; ++ti) {
        const ProfTile t = nxt;
        const int kind = t.op & 0xF;
        const bool scalar = (t.op & OP_SCALAR) != 0;
        if (HAS_CNT && (t.op & OP_STRIDED)) {
            if (ti + 1 < t_end) nxt = a.tiles[ti + 1];
            DYNMO_DCHECK(t.layer + (int64_t)(t.nbytes / (t.bits * 16u)) <= a.n_local);
            count_strided(t, lane, a.acc);
            continue;
        }
        if (HAS_CNT && small_count_tile(t)) {
            // Up to 8 consecutive small tiles (<= 512 B each, e.g. the
            // 4096-token masks of config 5) per warp iteration: 4 lanes per
            // tile, each streaming up to 8 of its tile's 16-byte vectors (all
            // in flight together), a quad reduction, then the 8 results are
            // fed to the run accumulator in tile order.
            const int grp = lane >> 2, q = lane & 3;
            const int64_t mt = ti + grp;
            ProfTile mine = t;
            if (grp > 0 && mt < t_end) mine = a.tiles[mt];
            const bool ok = mt < t_end && small_count_tile(mine);
            const unsigned okm = __ballot_sync(0xFFFFFFFFu, ok && q == 0);
            // leading run of small tiles (group g <-> bit 4g)
            int nb = 0;
            while (nb < 8 && (okm >> (4 * nb)) & 1u) ++nb;
            uint32_t c = 0;
            if (grp < nb) {
                const uint4 *p = (const uint4 *)mine.ptr;
                const uint32_t nvec = mine.nbytes >> 4;
                uint4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t idx = (uint32_t)q + 4u * u;
                    v[u] = idx < nvec ? ld_stream(p + idx) : make_uint4(0u, 0u, 0u, 0u);
                }
                const int kk = mine.op & 0xF;
#pragma unroll
                for (int u = 0; u < 8; ++u) c += count_vec_rt(kk, v[u]);
            }
            c += __shfl_xor_sync(0xFFFFFFFFu, c, 1);
            c += __shfl_xor_sync(0xFFFFFFFFu, c, 2);
            const int64_t key = (int64_t)mine.layer * ACC_N + mine.aux;
            for (int u = 0; u < nb; ++u)
                feed(__shfl_sync(0xFFFFFFFFu, key, 4 * u), __shfl_sync(0xFFFFFFFFu, c, 4 * u));
            ti += nb - 1;
            if (ti + 1 < t_end) nxt = a.tiles[ti + 1];
            continue;
        }
        if (ti + 1 < t_end) nxt = a.tiles[ti + 1];
        if (HAS_CNT && kind == OP_TIME) {
            // (begin, end) int64 ns pairs (8-byte aligned): lane-strided
            // pairs, end - begin summed in 64 bits; end < begin is INVALID
            const int64_t *v = (const int64_t *)t.ptr;
            const uint32_t np = t.nbytes >> 4;
            unsigned long long s = 0;
            for (uint32_t i = lane; i < np; i += 32) {
                const int64_t b = v[2 * i], e = v[2 * i + 1];
                if (e < b) bad = 1;
                else s += (unsigned long long)(e - b);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
            feed((int64_t)t.layer * ACC_N + t.aux, s);
            continue;
        }
        if (HAS_CNT && kind <= OP_NZ32) {
            uint32_t c;
            if (scalar) {
                c = count_scalar(t, kind, lane);
            } else {
                const uint4 *p = (const uint4 *)t.ptr;
                const uint32_t nvec = t.nbytes >> 4;
                switch (kind) {
                    case OP_POPC: c = count_tile<OP_POPC>(p, nvec, lane); break;
                    case OP_NZ8: c = count_tile<OP_NZ8>(p, nvec, lane); break;
                    case OP_NZ16: c = count_tile<OP_NZ16>(p, nvec, lane); break;
                    default: c = count_tile<OP_NZ32>(p, nvec, lane); break;
                }
            }
            feed((int64_t)t.layer * ACC_N + t.aux, __reduce_add_sync(0xFFFFFFFFu, c));
            continue;
        }
        if constexpr (HAS_HIST) {
            if (HAS_EXIT && kind == OP_EXIT) {
                // uint8 exit depths -> warp histogram in sh[0..255] (shared
                // atomics); flushed once when the warp's range is done
                if (hist_layer >= 0) flush_experts();  // (scratch is shared)
                exit_dirty = 1;
                DYNMO_DCHECK(kExitBins <= a.warp_words);
                const uint8_t *b = (const uint8_t *)t.ptr;
                if (scalar) {
                    if ((uint32_t)lane < t.nbytes) atomicAdd(&sh[b[lane]], 1u);
                } else {
                    const uint4 *p = (const uint4 *)t.ptr;
                    const uint32_t nvec = t.nbytes >> 4;
                    for (uint32_t base = 0; base < nvec; base += 64u) {
                        const uint32_t i0 = base + lane, i1 = base + 32 + lane;
                        const uint4 v0 = i0 < nvec ? ld_stream(p + i0) : make_uint4(0u, 0u, 0u, 0u);
                        const uint4 v1 = i1 < nvec ? ld_stream(p + i1) : make_uint4(0u, 0u, 0u, 0u);
                        if (i0 < nvec) {
                            const uint32_t w[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
                            for (int k = 0; k < 4; ++k)
#pragma unroll
                                for (int q = 0; q < 4; ++q) atomicAdd(&sh[(w[k] >> (8 * q)) & 0xFFu], 1u);
                        }
                        if (i1 < nvec) {
                            const uint32_t w[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                            for (int k = 0; k < 4; ++k)
#pragma unroll
                                for (int q = 0; q < 4; ++q) atomicAdd(&sh[(w[k] >> (8 * q)) & 0xFFu], 1u);
                        }
                    }
                }
                continue;
            }
            // MoE expert ids.  E <= 16: one-hot register counters; E <= 64:
            // each lane owns a private column sh[e*32 + lane] (no atomics, no
            // bank conflicts); else shared atomics on sh[e].  Flushed when the
            // layer changes.
            if (!HAS_EXP) continue;
            const int E = t.aux;
            if (exit_dirty) {  // the scratch holds exit bins: flush them first
                __syncwarp();
                for (int vb = lane; vb < kExitBins; vb += 32) {
                    const uint32_t c = sh[vb];
                    if (c) {
                        atomicAdd(&a.exit_hist[vb], (unsigned long long)c);
                        sh[vb] = 0u;
                    }
                }
                __syncwarp();
                exit_dirty = 0;
            }
            if (hist_layer != t.layer) {
                flush_experts();
                hist_layer = t.layer;
                hist_E = E;
            }
            if (E <= 16) {
                if (kind == OP_EXP64) {
                    if (E <= 8) expert_small<8, false>(t, scalar, lane, (uint32_t)E, acc0, acc1, nacc, bad, spill_regs);
                    else expert_small<8, true>(t, scalar, lane, (uint32_t)E, acc0, acc1, nacc, bad, spill_regs);
                } else {
                    if (E <= 8) expert_small<4, false>(t, scalar, lane, (uint32_t)E, acc0, acc1, nacc, bad, spill_regs);
                    else expert_small<4, true>(t, scalar, lane, (uint32_t)E, acc0, acc1, nacc, bad, spill_regs);
                }
                continue;
            }
            if constexpr (!HAS_BIGE) continue;
            const int esz = kind == OP_EXP64 ? 8 : 4;
            const bool cols = E <= kColExperts;
            DYNMO_DCHECK((cols ? 32 * E : E) <= a.warp_words && E <= a.max_E && t.layer < a.n_local);
            auto add = [&](uint64_t v) {
                if (v >= (uint64_t)E) {
                    bad = 1;
                    return;
                }
                if (cols) sh[(int)v * 32 + lane] += 1u;
                else atomicAdd(&sh[(int)v], 1u);
            };
            if (scalar) {
                const uint32_t ne = t.nbytes / esz;
                if ((uint32_t)lane < ne) {
                    uint64_t v = esz == 8 ? (uint64_t)((const int64_t *)t.ptr)[lane]
                                          : (uint64_t)(int64_t)((const int32_t *)t.ptr)[lane];
                    add(v);
                }
            } else {
                const uint4 *p = (const uint4 *)t.ptr;
                const uint32_t nvec = t.nbytes >> 4;
                for (uint32_t base = 0; base < nvec; base += 32u * 8u) {
                    uint4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        uint32_t idx = base + (uint32_t)u * 32u + (uint32_t)lane;
                        v[u] = idx < nvec ? ld_stream(p + idx) : make_uint4(0u, 0u, 0u, 0u);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        uint32_t idx = base + (uint32_t)u * 32u + (uint32_t)lane;
                        if (idx >= nvec) continue;
                        if (esz == 8) {
                            add(((uint64_t)v[u].y << 32) | v[u].x);
                            add(((uint64_t)v[u].w << 32) | v[u].z);
                        } else {
                            add((uint64_t)(int64_t)(int32_t)v[u].x);
                            add((uint64_t)(int64_t)(int32_t)v[u].y);
                            add((uint64_t)(int64_t)(int32_t)v[u].z);
                            add((uint64_t)(int64_t)(int32_t)v[u].w);
                        }
                    }
                }
            }
        }
    }
    DYNMO_DCHECK(run_key < 0 || run_key < (int64_t)a.n_local * ACC_N);
    if (lane == 0 && run_sum) atomicAdd(&a.acc[run_key], run_sum);
    if constexpr (HAS_HIST) {
        flush_experts();
        if (exit_dirty) {
            __syncwarp();
            for (int vb = lane; vb < kExitBins; vb += 32) {
                const uint32_t c = sh[vb];
                if (c) atomicAdd(&a.exit_hist[vb], (unsigned long long)c);
            }
        }
    }
    // an expert id outside [0, E) or a time pair with end < begin
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicMin(a.ws_status, (int)DYNMO_E_INVALID);
    if (a.span) {  // the CTA's end: after all of its warps
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(&a.span[1], globaltimer_ns());
    }
}

// -------------------------------------------------------------- epilogue
__device__ __forceinline__ int worse(int a, int b) { return a < b ? a : b; }
constexpr int kEpiK = 4;  // layers per thread per epilogue iteration
// LL ("flag in the data") words of the peer-memory exchange: an int64 as two
// 8-byte words {32 data bits, low 32 bits of the call epoch}.  An aligned
// 8-byte store is single-copy atomic, so a word read with the current epoch
// holds this call's data -- no fence or separate flag release is needed.
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ll_store(int64_t *p, int64_t v, uint64_t epoch) {
    const uint64_t e = (uint64_t)(uint32_t)epoch << 32;
    st_relaxed_sys((uint64_t *)p, e | (uint32_t)(uint64_t)v);
    st_relaxed_sys((uint64_t *)p + 1, e | (uint32_t)((uint64_t)v >> 32));
}
// Spins until both words carry `epoch` (false after 10 s from t0).
__device__ __forceinline__ bool ll_poll(const uint64_t *p, uint64_t epoch, uint64_t t0, int64_t &v) {
    const uint32_t e = (uint32_t)epoch;
    for (;;) {
        const uint64_t w0 = ld_relaxed_sys(p), w1 = ld_relaxed_sys(p + 1);
        if ((uint32_t)(w0 >> 32) == e && (uint32_t)(w1 >> 32) == e) {
            v = (int64_t)(((uint64_t)(uint32_t)w1 << 32) | (uint32_t)w0);
            return true;
        }
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10ull * 1000 * 1000 * 1000) return false;
    }
}

__device__ void unpack_p2p_dev(const int64_t *slots, PeerWindow *win, int32_t nranks, int32_t n_total,
                               int64_t *decoded, int64_t *cost_out, int64_t *mem_out, int32_t *status_out);

// Inputs of one layer, loaded before any of them is used so that a thread
// has the loads of several layers in flight (the epilogue is a long list
// of tiny independent layers for config 5: 360 k of them).
struct EpiPre {
    LayerInfo li;
    dynmo_cost_coef cf;
    unsigned long long nnz_u, tok_u, time_u;
    int64_t m;
    bool frozen;
};

// The per-layer data the epilogue consumes and produces: the real buffers,
// or (code warm-up before griddepcontrol.wait) scratch of the plan.
struct EpiIO {
    unsigned long long *acc, *hist, *exit_hist;
    int64_t *counters_out, *hist_out, *cost_out, *mem_out;
    int32_t p2p, exchange;
};

__device__ __forceinline__ void epi_load(const EpiArgs &a, const EpiIO &io, int q, EpiPre &p) {
    p.li = a.info[q];
    const uint4 *c4 = reinterpret_cast<const uint4 *>(a.coef + q);  // 48 B, 16-B aligned
    uint4 *d4 = reinterpret_cast<uint4 *>(&p.cf);
    d4[0] = c4[0];
    d4[1] = c4[1];
    d4[2] = c4[2];
    p.nnz_u = io.acc[(int64_t)q * ACC_N + ACC_NNZ];
    p.tok_u = io.acc[(int64_t)q * ACC_N + ACC_TOK];
    p.time_u = io.acc[(int64_t)q * ACC_N + ACC_TIME];
    p.frozen = a.frozen && a.frozen[q];
    p.m = a.mem_local ? a.mem_local[q] : 0;
}

// Cost of local layer q from its prefetched inputs (a5, readings Q1-Q6);
// consumes its counters; writes the outputs of the selected exchange mode.
// Returns the layer's status.
__device__ __forceinline__ int epi_one(const EpiArgs &a, const EpiIO &io, int q, const EpiPre &p) {
    int st = DYNMO_OK;
    const LayerInfo li = p.li;
    const int gi = a.layer_begin + q;
    unsigned long long nnz_u = p.nnz_u;
    unsigned long long tok_u = p.tok_u;
    const unsigned long long time_u = p.time_u;
    io.acc[(int64_t)q * ACC_N + ACC_NNZ] = 0ull;
    io.acc[(int64_t)q * ACC_N + ACC_TOK] = 0ull;
    io.acc[(int64_t)q * ACC_N + ACC_TIME] = 0ull;
    if (li.flags & SRC_HAS_EXIT)
        for (int v = gi + 1; v < kExitBins; ++v) tok_u += io.exit_hist[v];
    const bool has_tok = (li.flags & SRC_HAS_TOK) != 0;
    const dynmo_cost_coef cf = p.cf;
    const bool frozen = p.frozen;
    // moe_i = EP * max over EP groups of group token counts (reading Q5)
    __int128 moe = 0;
    const bool bad_coef = cf.A < 0 || cf.B < 0 || cf.C < 0 || cf.F < 0 || cf.D < 0;
    bool bad_ep = false;
    if (li.flags & SRC_HAS_MOE) {
        const int E = li.E;
        const int EP = cf.ep_ranks <= 0 ? E : cf.ep_ranks;
        unsigned long long *h = io.hist + (int64_t)q * a.max_E;
        bad_ep = E < 1 || EP < 1 || E % EP != 0;
        if (!bad_ep) {
            const int g = E / EP;
            __int128 best = 0;
            for (int r = 0; r < EP; ++r) {
                __int128 s = 0;
                for (int e = r * g; e < (r + 1) * g; ++e) s += (__int128)h[e];
                if (s > best) best = s;
            }
            moe = (__int128)EP * best;
        }
        for (int e = 0; e < E; ++e) {
            if (io.hist_out) io.hist_out[(int64_t)q * a.max_E + e] = (int64_t)h[e];
            h[e] = 0ull;
        }
    }
    const __int128 LIM = (__int128)INT64_MAX;
    const __int128 tok = has_tok ? (__int128)tok_u : (__int128)1;
    const __int128 nnz = (__int128)nnz_u;
    int64_t c = -1;
    // order of the oracle: coefficients, then frozen, then the EP groups
    if (bad_coef) {
        st = DYNMO_E_INVALID;
    } else if (frozen) {
        c = cf.F;
    } else if (bad_ep) {
        st = DYNMO_E_INVALID;
    } else {
        const __int128 inner = (__int128)cf.A + (__int128)cf.B * nnz;
        if (inner > LIM || tok > LIM || moe > LIM) {
            st = DYNMO_E_OVERFLOW;
        } else {
            __int128 v = tok * inner;
            const __int128 cm = (__int128)cf.C * moe;
            const __int128 tm = (__int128)time_u;
            const __int128 ct = tm > LIM ? LIM + 1 : (__int128)cf.D * tm;
            if (tm > LIM || v > LIM || cm > LIM || v + cm > LIM || ct > LIM || v + cm + ct > LIM)
                st = DYNMO_E_OVERFLOW;
            else c = (int64_t)(v + cm + ct);
        }
    }
    const int64_t m = p.m;
    if (io.counters_out) {
        int64_t *o = io.counters_out + (int64_t)q * 5;
        o[0] = (int64_t)nnz_u;
        o[1] = has_tok ? (int64_t)tok_u : 1;
        o[2] = moe > LIM ? -1 : (int64_t)moe;
        o[3] = c;
        o[4] = time_u > (unsigned long long)INT64_MAX ? -1 : (int64_t)time_u;
    }
    if (io.p2p) {
        // straight into every rank's receive slot as LL words (NVLink
        // stores; each word carries the epoch, no fence or flag needed)
        const uint64_t epoch = a.win->exch_epoch + 1;  // advanced by the last block
        const int64_t S = 3 + 2 * (int64_t)a.n_total;
        const int64_t off = ((int64_t)(epoch & 1) * a.nranks + a.rank) * 2 * S;
        for (int r = 0; r < a.nranks; ++r) {
            ll_store(a.peer_slots[r] + off + 2 * (3 + q), c, epoch);
            ll_store(a.peer_slots[r] + off + 2 * (3 + a.n_total + q), m, epoch);
        }
    } else if (io.exchange) {
        a.slot_send[3 + q] = c;
        a.slot_send[3 + a.n_total + q] = m;
    } else {
        io.cost_out[q] = c;
        if (io.mem_out) io.mem_out[q] = m;
    }
    return st;
}

__global__ void __launch_bounds__(256, 2) k_epilogue(EpiArgs a) {
    // grid-stride, kEpiK layers per thread with all their loads issued first.
    // Pass 0 (a.warm: plan scratch), before griddepcontrol.wait: thread 0 of
    // block 0 runs the same loop code on layer 0's step-invariant inputs
    // and scratch counters / outputs, so the instructions are fetched while
    // k_profile still runs (after an L2 flush the epilogue's cold start is
    // its code, `profiles/r02_ab_epi_prefetch/`).  Pass 1 is the real one.
    STEP_STAMP(STAMP_EPILOGUE);  // (diagnostic build: the start is the CTA's, before the wait)
    const int nthr = gridDim.x * blockDim.x;
    int st = DYNMO_OK;
#pragma unroll 1
    for (int pass = a.warm ? 0 : 1; pass < 2; ++pass) {
        EpiIO io;
        int nl;
        if (pass == 0) {
            unsigned long long *w = a.warm;
            int64_t *o = reinterpret_cast<int64_t *>(w + ACC_N + 2 * a.max_E + kExitBins);
            io = EpiIO{w, w + ACC_N, w + ACC_N + a.max_E, o, a.hist_out ? o + 8 : nullptr, o + 5, a.mem_out ? o + 6 : nullptr,
                       0, 0};
            nl = a.n_local > 0 && blockIdx.x == 0 ? 1 : 0;
        } else {
            pdl_wait();
            pdl_trigger();
            io = EpiIO{a.acc, a.hist, a.exit_hist, a.counters_out, a.hist_out, a.cost_out, a.mem_out, a.p2p,
                       a.exchange};
            nl = a.n_local;
        }
        for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < nl; base += nthr * kEpiK) {
            EpiPre p[kEpiK];
#pragma unroll
            for (int k = 0; k < kEpiK; ++k) {
                const int q = base + k * nthr;
                if (q < nl) epi_load(a, io, q, p[k]);
            }
#pragma unroll
            for (int k = 0; k < kEpiK; ++k) {
                const int q = base + k * nthr;
                if (q < nl) st = worse(st, epi_one(a, io, q, p[k]));
            }
        }
        if (pass == 0) st = DYNMO_OK;
    }
    // block-reduce the status, then last-block finalisation
    __shared__ int s_st;
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_st = DYNMO_OK;
    __syncthreads();
    if (st != DYNMO_OK) atomicMin(&s_st, st);
    __syncthreads();
    // one block (a few thousand layers or fewer): it is the last block, and
    // its status needs no global atomics or fences (k_profile's errors are
    // read from the status word with a plain load: k_profile has completed)
    const bool single = gridDim.x == 1;
    if (threadIdx.x == 0 && !single) {
        if (s_st != DYNMO_OK) atomicMin(a.ws_status, s_st);
        // this block's (remote) slot stores before the counter; the last
        // block's system-scope fence + release below is cumulative over them
        __threadfence();
        unsigned prev = atomicAdd(a.ws_done, 1u);
        s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (single || s_last) {
        if (!single || a.p2p) __threadfence();
        for (int v = threadIdx.x; v < kExitBins; v += blockDim.x) a.exit_hist[v] = 0ull;
        if (threadIdx.x == 0 && a.span) {  // k_profile has completed (pdl_wait)
            const unsigned long long t0 = ~a.span[0], t1 = a.span[1];
            if (a.span[0] && t1 > t0) {
                a.span[2] += t1 - t0;
                a.span[3] += 1ull;
            }
            a.span[0] = 0ull;
            a.span[1] = 0ull;
        }
        if (threadIdx.x == 0) {
            int fin;
            if (single) {  // k_profile's own errors (bad ids, time pairs) are in ws_status
                const int w = *a.ws_status;
                fin = w < s_st ? w : s_st;
                if (w) *a.ws_status = 0;
            } else {
                fin = atomicExch(a.ws_status, 0);
                *a.ws_done = 0u;
            }
            if (a.p2p) {
                const uint64_t epoch = a.win->exch_epoch + 1;
                const int64_t S = 3 + 2 * (int64_t)a.n_total;
                const int64_t off = ((int64_t)(epoch & 1) * a.nranks + a.rank) * 2 * S;
                for (int r = 0; r < a.nranks; ++r) {
                    ll_store(a.peer_slots[r] + off + 0, a.layer_begin, epoch);
                    ll_store(a.peer_slots[r] + off + 2, a.n_local, epoch);
                    ll_store(a.peer_slots[r] + off + 4, fin, epoch);
                }
                a.win->exch_epoch = epoch;
            } else if (a.exchange) {
                a.slot_send[0] = a.layer_begin;
                a.slot_send[1] = a.n_local;
                a.slot_send[2] = fin;
            } else {
                *a.status_out = fin;
            }
        }
        if (a.p2p && a.fuse_unpack) {  // the exchange in this block: no extra launch
            __syncthreads();  // exch_epoch written by thread 0
            unpack_p2p_dev(a.p2p_slots, a.win, a.nranks, a.n_total, a.decoded, a.x_cost, a.x_mem, a.x_status);
        }
    }
}

// ---------------------------------------------------------------- unpack
// Slot of rank r at slot_recv + r*S, S = 3 + 2*n_total:
// {layer_begin, n_local, status, cost[n_total], mem[n_total]}.
__device__ void k_unpack_body(const int64_t *slot_recv, int32_t nranks, int32_t n_total,
                              int64_t *cost_out, int64_t *mem_out, int32_t *status_out);

__global__ void k_unpack(const int64_t *slot_recv, int32_t nranks, int32_t n_total,
                         int64_t *cost_out, int64_t *mem_out, int32_t *status_out) {
    pdl_wait();
    pdl_trigger();
    k_unpack_body(slot_recv, nranks, n_total, cost_out, mem_out, status_out);
}

__device__ void k_unpack_body(const int64_t *slot_recv, int32_t nranks, int32_t n_total,
                              int64_t *cost_out, int64_t *mem_out, int32_t *status_out) {
    const int64_t S = 3 + 2 * (int64_t)n_total;
    __shared__ int s_st;
    if (threadIdx.x == 0) {
        int st = DYNMO_OK;
        for (int r = 0; r < nranks; ++r) {
            const int64_t *sl = slot_recv + r * S;
            const int64_t b = sl[0], c = sl[1];
            if (b < 0 || c < 0 || b + c > n_total) st = worse(st, DYNMO_E_INVALID);
            st = worse(st, (int)sl[2]);
        }
        s_st = st;
    }
    __syncthreads();
    int st = DYNMO_OK;
    for (int i = threadIdx.x; i < n_total; i += blockDim.x) {
        int cover = 0;
        int64_t c = -1, m = 0;
        for (int r = 0; r < nranks; ++r) {
            const int64_t *sl = slot_recv + r * S;
            const int64_t b = sl[0], cnt = sl[1];
            if (b >= 0 && cnt >= 0 && b + cnt <= n_total && i >= b && i < b + cnt) {
                cover++;
                c = sl[3 + (i - b)];
                m = sl[3 + n_total + (i - b)];
            }
        }
        if (cover != 1) {
            st = DYNMO_E_INVALID;
            c = -1;
        }
        cost_out[i] = c;
        if (mem_out) mem_out[i] = m;
    }
    if (st != DYNMO_OK) atomicMin(&s_st, st);
    __syncthreads();
    if (threadIdx.x == 0) *status_out = s_st;
}

// Peer-memory exchange, receive side: wait (bounded) for every rank's flag of
// this epoch, then scatter the local slot area of the epoch's parity.
// Receiver side of the LL exchange: for every sender rank, poll its three
// header words, then the words of its [layer_begin, +n_local) slice, until
// each carries this call's epoch (bounded: 10 s), decoding into `decoded`
// ([nranks][S] plain int64 slots) for the shared validation / scatter.
__global__ void k_unpack_p2p(const int64_t *slots, PeerWindow *win, int32_t nranks, int32_t n_total,
                             int64_t *decoded, int64_t *cost_out, int64_t *mem_out, int32_t *status_out) {
    pdl_wait();
    pdl_trigger();
    unpack_p2p_dev(slots, win, nranks, n_total, decoded, cost_out, mem_out, status_out);
}

// Polls every rank's LL slot words of this epoch (bounded), decodes them and
// scatters the global vectors (one block; also the tail of the epilogue's
// last block when the exchange is fused into it).
__device__ void unpack_p2p_dev(const int64_t *slots, PeerWindow *win, int32_t nranks, int32_t n_total,
                               int64_t *decoded, int64_t *cost_out, int64_t *mem_out, int32_t *status_out) {
    __shared__ int s_ok;
    __shared__ int64_t s_hdr[3];
    const uint64_t epoch = win->exch_epoch;  // advanced by this rank's epilogue
    const int64_t S = 3 + 2 * (int64_t)n_total;
    const uint64_t *ll = (const uint64_t *)slots + (int64_t)(epoch & 1) * nranks * 2 * S;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) s_ok = 1;
    __syncthreads();
    for (int r = 0; r < nranks; ++r) {
        const uint64_t *src = ll + (int64_t)r * 2 * S;
        int64_t *dst = decoded + (int64_t)r * S;
        if (threadIdx.x < 3) {  // header: layer_begin, n_local, status
            int64_t v;
            if (!ll_poll(src + 2 * threadIdx.x, epoch, t0, v)) atomicExch(&s_ok, 0);
            s_hdr[threadIdx.x] = v;
            dst[threadIdx.x] = v;
        }
        __syncthreads();
        if (!s_ok) break;
        const int64_t lb = s_hdr[0], n = s_hdr[1];
        const bool sane = lb >= 0 && n >= 0 && lb + n <= n_total;  // else the shared check flags it
        for (int64_t i = threadIdx.x; sane && i < n; i += blockDim.x) {
            int64_t c, m;
            bool ok = ll_poll(src + 2 * (3 + i), epoch, t0, c);
            ok = ok && ll_poll(src + 2 * (3 + n_total + i), epoch, t0, m);
            if (!ok) {
                atomicExch(&s_ok, 0);
                break;
            }
            dst[3 + i] = c;
            dst[3 + n_total + i] = m;
        }
        __syncthreads();
        if (!s_ok) break;
    }
    if (!s_ok && threadIdx.x == 0) win->err = DYNMO_E_NCCL;
    __syncthreads();
    if (!s_ok) {
        for (int i = threadIdx.x; i < n_total; i += blockDim.x) {
            cost_out[i] = -1;
            if (mem_out) mem_out[i] = 0;
        }
        if (threadIdx.x == 0) *status_out = DYNMO_E_NCCL;
        return;
    }
    __syncthreads();
    k_unpack_body(decoded, nranks, n_total, cost_out, mem_out, status_out);
}

}  // namespace

template <int OPS>
static int blocks_per_sm_t(int warp_words) {
    int nb = 0;
    const size_t sm = (OPS & 6) ? (size_t)(kProfThreads / 32) * 4 * warp_words : 0;
    if (sm) cudaFuncSetAttribute(k_profile<OPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_profile<OPS>, kProfThreads, sm);
    return nb > 0 ? nb : 1;
}

template <int OPS>
static cudaError_t launch_t(const ProfArgs &a, int grid, cudaStream_t s) {
    const size_t sm = (OPS & 6) ? (size_t)(kProfThreads / 32) * 4 * a.warp_words : 0;
    k_profile<OPS><<<grid, kProfThreads, sm, s>>>(a);
    return cudaGetLastError();
}

// ops: bit 3 (E > 16) only ever comes with bit 2
int profile_blocks_per_sm(int ops, int warp_words) {
    switch (ops & 15) {
        case 1: return blocks_per_sm_t<1>(warp_words);
        case 2: return blocks_per_sm_t<2>(warp_words);
        case 3: return blocks_per_sm_t<3>(warp_words);
        case 4: return blocks_per_sm_t<4>(warp_words);
        case 5: return blocks_per_sm_t<5>(warp_words);
        case 6: return blocks_per_sm_t<6>(warp_words);
        case 7: return blocks_per_sm_t<7>(warp_words);
        case 12: return blocks_per_sm_t<12>(warp_words);
        case 13: return blocks_per_sm_t<13>(warp_words);
        case 14: return blocks_per_sm_t<14>(warp_words);
        default: return blocks_per_sm_t<15>(warp_words);
    }
}

cudaError_t launch_profile(const ProfArgs &a, int ops, int grid, cudaStream_t s) {
    if (a.n_tiles == 0) return cudaSuccess;
    switch (ops & 15) {
        case 1: return launch_t<1>(a, grid, s);
        case 2: return launch_t<2>(a, grid, s);
        case 3: return launch_t<3>(a, grid, s);
        case 4: return launch_t<4>(a, grid, s);
        case 5: return launch_t<5>(a, grid, s);
        case 6: return launch_t<6>(a, grid, s);
        case 7: return launch_t<7>(a, grid, s);
        case 12: return launch_t<12>(a, grid, s);
        case 13: return launch_t<13>(a, grid, s);
        case 14: return launch_t<14>(a, grid, s);
        default: return launch_t<15>(a, grid, s);
    }
}

cudaError_t launch_epilogue(const EpiArgs &a, cudaStream_t s) {
    const int threads = 256;
    // one resident wave (grid-stride beyond it), kEpiK layers per thread
    static const int wave = [] {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_epilogue, 256, 0);
        return std::max(1, sms * std::max(1, per));
    }();
    const int64_t need = ((int64_t)a.n_local + (int64_t)threads * kEpiK - 1) / ((int64_t)threads * kEpiK);
    const int grid = a.n_local > 0 ? (int)std::min<int64_t>(need, wave) : 1;
    return launch_pdl(k_epilogue, grid, threads, 0, s, a);
}

// %globaltimer (ns) into *p once the preceding work of the stream is done
// (a normal launch, NOT programmatic: it must not start early)
__global__ void k_stamp(int64_t *p) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *p = (int64_t)t;
}

cudaError_t launch_stamp(int64_t *d_slot, cudaStream_t s) {
    k_stamp<<<1, 1, 0, s>>>(d_slot);
    return cudaGetLastError();
}

// Result publication: the step's small result buffer stored straight into
// mapped pinned host memory by the GPU (zero-copy), in place of a D2H copy
// node (a copy-engine transfer costs ~6 us of the step for tens of bytes).
// 16-byte stores when both ends are 16-byte aligned and the size a multiple
// of 16, bytes otherwise.  Programmatic launch: it waits for the preceding
// kernel's completion (griddepcontrol.wait) before reading.
__global__ void k_publish(const uint8_t *__restrict__ src, uint8_t *dst, int64_t bytes) {
    pdl_wait();
    STEP_STAMP(STAMP_PUBLISH);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst | (uintptr_t)bytes) & 15) == 0) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int64_t i = t; i < bytes / 16; i += nt) d4[i] = s4[i];
    } else {
        for (int64_t i = t; i < bytes; i += nt) dst[i] = src[i];
    }
    // no __threadfence_system(): the host reads after an event recorded
    // behind this kernel completes, and completion makes the stores visible
    // (the fence only held the kernel ~3 us longer for the PCIe acks)
}

cudaError_t launch_publish(const void *d_src, void *d_dst, int64_t bytes, cudaStream_t s) {
    static const int64_t per = [] {  // bytes per CTA (DYNMO_PUBLISH_CTA_BYTES: tuning knob)
        const char *e = getenv("DYNMO_PUBLISH_CTA_BYTES");
        const long long v = e ? atoll(e) : 0;
        return (int64_t)(v > 0 ? v : 256 * 16);
    }();
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(1, (bytes + per - 1) / per), 148);
    return launch_pdl(k_publish, grid, 256, 0, s, (const uint8_t *)d_src, (uint8_t *)d_dst, bytes);
}

cudaError_t launch_unpack(const int64_t *slot_recv, int32_t nranks, int32_t n_total,
                          int64_t *cost_out, int64_t *mem_out, int32_t *status_out,
                          cudaStream_t s) {
    return launch_pdl(k_unpack, 1, 1024, 0, s, slot_recv, nranks, n_total, cost_out, mem_out, status_out);
}

cudaError_t launch_unpack_p2p(const int64_t *slots, PeerWindow *win, int32_t nranks, int32_t n_total,
                              int64_t *decoded, int64_t *cost_out, int64_t *mem_out, int32_t *status_out,
                              cudaStream_t s) {
    return launch_pdl(k_unpack_p2p, 1, 1024, 0, s, slots, win, nranks, n_total, decoded, cost_out, mem_out,
                      status_out);
}

}  // namespace dynmo

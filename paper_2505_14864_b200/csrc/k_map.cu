// Migration-minimising stage -> rank map (NEXT-3 of SURVEY 8(f); reading
// Q23): after a rebalance or re-pack, place the n_new stages on
// distinct allowed ranks so that the payload staying in place is maximal
// (every byte kept is a byte not migrated).  Exact, with the
// lexicographically smallest optimal rank vector: a DP over subsets of the
// G <= 16 ranks, f(used) = max over g of w[|used|][g] + f(used + g), levels
// |used| = n_new-1 .. 0 swept by one CTA (2^G states, a barrier per level),
// then the greedy lexicographic walk on thread 0.  f lives in the ctx's
// device workspace (2^16 int64).
#include "dynmo_internal.h"

namespace dynmo {
namespace {

constexpr int kMapThreads = 1024;

__global__ void __launch_bounds__(kMapThreads) k_map_stages(MapArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ unsigned long long w[kMaxMapRanks][kMaxMapRanks];  // [new stage][rank]
    __shared__ int s_bad;
    const int tid = threadIdx.x;
    const int L = a.L, G = a.G, n_new = a.n_new, n_old = a.n_old;
    for (int i = tid; i < kMaxMapRanks * kMaxMapRanks; i += kMapThreads) (&w[0][0])[i] = 0ull;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    // validation (the oracle's order: splits, ranks, bytes)
    int bad = 0;
    for (int s = tid; s <= n_old; s += kMapThreads) {
        const int b = a.bnd_old[s];
        if (s == 0 ? b != 0 : (b <= a.bnd_old[s - 1])) bad = 1;
        if (s == n_old && b != L) bad = 1;
        if (s < n_old && (a.rank_old[s] < 0 || a.rank_old[s] >= G)) bad = 1;
    }
    for (int s = tid; s <= n_new; s += kMapThreads) {
        const int b = a.bnd_new[s];
        if (s == 0 ? b != 0 : (b <= a.bnd_new[s - 1])) bad = 1;
        if (s == n_new && b != L) bad = 1;
    }
    for (int i = tid; i < L; i += kMapThreads)
        if (a.bytes[i] < 0) bad = 1;
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    const uint32_t allowed = a.allowed & ((1u << G) - 1u);
    if (s_bad || n_new > __popc(allowed)) {
        if (tid == 0) {
            *a.status = s_bad ? DYNMO_E_INVALID : DYNMO_E_INFEASIBLE;
            *a.kept = -1;
        }
        for (int s = tid; s < n_new; s += kMapThreads) a.rank_new[s] = -1;
        return;
    }
    // w[s][g]: bytes of new stage s currently on rank g (owner by binary search)
    for (int i = tid; i < L; i += kMapThreads) {
        int lo = 0, hi = n_old - 1;  // old stage: last s with bnd_old[s] <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.bnd_old[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        int sl = 0, sh = n_new - 1;
        while (sl < sh) {
            const int mid = (sl + sh + 1) >> 1;
            if (a.bnd_new[mid] <= i) sl = mid;
            else sh = mid - 1;
        }
        const long long b = a.bytes[i];
        if (b) atomicAdd(&w[sl][a.rank_old[lo]], (unsigned long long)b);
    }
    __syncthreads();
    if (a.slot_rank) {  // slots: a byte stays when its new slot is on the same GPU as its old slot
        __shared__ unsigned long long wr[kMaxMapRanks][kMaxMapRanks];
        if (tid < n_new * G) {
            const int s = tid / G, g = tid % G;
            unsigned long long v = 0;
            for (int j = 0; j < G; ++j)
                if (a.slot_rank[j] == a.slot_rank[g]) v += w[s][j];
            wr[s][g] = v;
        }
        __syncthreads();
        if (tid < n_new * G) w[tid / G][tid % G] = wr[tid / G][tid % G];
        __syncthreads();
    }
    long long *f = a.work;
    const uint32_t NS = 1u << G;
    for (int k = n_new; k >= 0; --k) {
        for (uint32_t u = tid; u < NS; u += kMapThreads) {
            if (__popc(u) != k || (u & ~allowed)) continue;
            long long best = k == n_new ? 0 : -1;
            if (k < n_new)
                for (int g = 0; g < G; ++g) {
                    if (!((allowed >> g) & 1u) || ((u >> g) & 1u)) continue;
                    const long long v = (long long)w[k][g] + f[u | (1u << g)];
                    best = v > best ? v : best;
                }
            f[u] = best;
        }
        __syncthreads();  // level k complete before level k-1 reads it
    }
    if (tid == 0) {
        uint32_t used = 0;
        for (int s = 0; s < n_new; ++s)
            for (int g = 0; g < G; ++g) {
                if (!((allowed >> g) & 1u) || ((used >> g) & 1u)) continue;
                if ((long long)w[s][g] + f[used | (1u << g)] == f[used]) {
                    a.rank_new[s] = a.slot_rank ? a.slot_rank[g] : g;
                    used |= 1u << g;
                    break;
                }
            }
        *a.kept = f[0];
        *a.status = DYNMO_OK;
    }
}

}  // namespace

cudaError_t launch_map_stages(const MapArgs &a, cudaStream_t s) {
    return launch_pdl(k_map_stages, 1, kMapThreads, 0, s, a);
}

}  // namespace dynmo

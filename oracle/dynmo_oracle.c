/*
 * dynmo_oracle.c -- CPU ORACLE for the DynMo per-step rebalancing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * file.  The product path (paper_2505_14864_b200/) never imports, links or
 * executes anything under oracle/, and this file includes no header of the
 * product and shares no helper with it.
 *
 * Plain, slow, obviously correct C11: every function is the plain definition
 * (or the paper's algorithm step by step) with no blocking or fusion.
 * Citations: P:Lnnn = /root/reference/PAPER.md line, S:Lnnn = SPEC.md line.
 * Readings Q1..Q20 are listed in DESIGN.md ("Readings of the paper").
 *
 * Status codes (same numeric contract as the C-ABI, restated here, not
 * shared):  0 OK, -1 INVALID, -2 INFEASIBLE, -3 OVERFLOW,
 *           +1 NOT_CONVERGED (diffusion), +2 BOUND_UNMET (repack).
 * Where several errors occur in one profile call, the most negative wins.
 *
 * Pins: every function here is checked by tests/test_oracle_*.py against
 * something other than itself (library routines, brute-force enumeration,
 * SPEC/paper worked examples under tests/golden/, closed forms, invariants).
 * No function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define O_OK 0
#define O_E_INVALID (-1)
#define O_E_INFEASIBLE (-2)
#define O_E_OVERFLOW (-3)
#define O_W_NOT_CONVERGED 1
#define O_W_BOUND_UNMET 2

typedef __int128 i128;

static int worse(int a, int b) { return a < b ? a : b; }

/* ------------------------------------------------------------------------
 * O1 counters (P:L234-239 pruning retained fraction p_i; P:L340-353 early
 * exit tokens t_i; P:L376-389 MoD routed tokens r_i t_i; P:L209-214 MoE
 * tokens routed to expert e).
 * ---------------------------------------------------------------------- */

/* Number of set bits among the first n_bits bits of a little-endian packed
 * mask (bit b of the mask is bit (b % 32) of word b / 32). */
int64_t oracle_count_bits(const uint32_t *words, int64_t n_bits) {
    int64_t c = 0;
    for (int64_t b = 0; b < n_bits; ++b)
        if ((words[b / 32] >> (b % 32)) & 1u) c++;
    return c;
}

/* Bytes != 0 of a bool/uint8 mask. */
int64_t oracle_count_nz_u8(const uint8_t *p, int64_t n) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        if (p[i] != 0) c++;
    return c;
}

/* Nonzero bf16 weights: pruned == +0 or -0 (sign bit ignored); NaN counts. */
int64_t oracle_count_nz_bf16(const uint16_t *p, int64_t n) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        if ((p[i] & 0x7FFFu) != 0) c++;
    return c;
}

/* Nonzero f32 weights, same rule as bf16. */
int64_t oracle_count_nz_f32(const uint32_t *p, int64_t n) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        if ((p[i] & 0x7FFFFFFFu) != 0) c++;
    return c;
}

/* Early exit: e[t] = number of layers token t is
 * processed by (layers 0..e[t]-1).  tok_i = #{t : e[t] > i} for each of the
 * n_local layers i = layer_begin .. layer_begin+n_local-1.  Added to tok. */
void oracle_exit_survivors(const uint8_t *e, int64_t T, int32_t layer_begin,
                           int32_t n_local, int64_t *tok) {
    for (int32_t q = 0; q < n_local; ++q) {
        int32_t i = layer_begin + q;
        int64_t c = 0;
        for (int64_t t = 0; t < T; ++t)
            if ((int32_t)e[t] > i) c++;
        tok[q] += c;
    }
}

/* MoE: cnt[e] += #{entries == e}.  Entries outside [0,E) are
 * not counted and make the result INVALID. */
int oracle_expert_hist_i64(const int64_t *idx, int64_t n, int32_t E, int64_t *cnt) {
    int st = O_OK;
    for (int64_t j = 0; j < n; ++j) {
        int64_t v = idx[j];
        if (v < 0 || v >= E) { st = O_E_INVALID; continue; }
        cnt[v]++;
    }
    return st;
}

int oracle_expert_hist_i32(const int32_t *idx, int64_t n, int32_t E, int64_t *cnt) {
    int st = O_OK;
    for (int64_t j = 0; j < n; ++j) {
        int32_t v = idx[j];
        if (v < 0 || v >= E) { st = O_E_INVALID; continue; }
        cnt[v]++;
    }
    return st;
}

/* ------------------------------------------------------------------------
 * O1' execution time of a layer from its timestamp pairs ("by Time"
 * balancers, P:L632 profiling iteration timers, "decoder layer
 * execution times"; reading Q21): time = sum over pairs of
 * (end - begin), pairs stored (begin, end) consecutively, n values (even).
 * A pair with end < begin is INVALID (skipped); an odd n is INVALID.
 * ---------------------------------------------------------------------- */
int oracle_time_ns(const int64_t *v, int64_t n, int64_t *time) {
    int st = (n % 2) ? O_E_INVALID : O_OK;
    i128 acc = 0;
    for (int64_t j = 0; j + 1 < n; j += 2) {
        if (v[j + 1] < v[j]) { st = O_E_INVALID; continue; }
        acc += (i128)v[j + 1] - (i128)v[j];
    }
    *time = acc > (i128)INT64_MAX ? -1 : (int64_t)acc;
    if (acc > (i128)INT64_MAX) st = O_E_OVERFLOW;
    return st;
}

/* ------------------------------------------------------------------------
 * O2 cost of one layer (readings Q1-Q6, Q21):
 *   c = frozen ? F : tok*(A + B*nnz) + C*moe + D*time,
 *   moe = EP * max_{r<EP} sum_{e in group r} cnt[e]   (groups of E/EP
 *   consecutive experts; EP<=0 means EP=E), defaults tok=1 (no token
 *   source), nnz=0, moe=0 (no expert source).
 * Freezing P:L278-282 (F=0 is the paper's "contributing no computational
 * load"), pruning P:L238 (A=0,B=1), early exit P:L344 / MoD P:L380 (B=0),
 * by Time P:L720/P:L743 (D=1, A=B=C=0; time = 0 without a time source).
 * Checked arithmetic in 128 bits; negative coefficients INVALID; a result
 * above INT64_MAX is OVERFLOW.  On error *cost = -1.
 * ---------------------------------------------------------------------- */
int oracle_layer_cost(int frozen, int has_tok, int64_t tok, int64_t nnz,
                      int has_moe, const int64_t *cnt, int32_t E,
                      int64_t A, int64_t B, int64_t C, int64_t F, int32_t ep,
                      int64_t D, int64_t time, int64_t *cost) {
    *cost = -1;
    if (A < 0 || B < 0 || C < 0 || F < 0 || D < 0 || tok < 0 || nnz < 0 || time < 0) return O_E_INVALID;
    if (frozen) { *cost = F; return O_OK; }
    i128 moe = 0;
    if (has_moe) {
        int32_t EP = ep <= 0 ? E : ep;
        if (E < 1 || EP < 1 || E % EP != 0) return O_E_INVALID;
        int32_t g = E / EP;
        i128 best = 0;
        for (int32_t r = 0; r < EP; ++r) {
            i128 s = 0;
            for (int32_t e = r * g; e < (r + 1) * g; ++e) s += cnt[e];
            if (s > best) best = s;
        }
        moe = (i128)EP * best;
    }
    i128 t = has_tok ? (i128)tok : 1;
    i128 inner = (i128)A + (i128)B * (i128)nnz;
    /* t and inner are each < 2^64, so the product fits in 127 bits. */
    const i128 LIM = (i128)INT64_MAX;
    if (inner > LIM) return O_E_OVERFLOW;
    i128 c = t * inner;
    if (c > LIM) return O_E_OVERFLOW;
    if (moe > LIM) return O_E_OVERFLOW;
    i128 cm = (i128)C * moe;
    if (cm > LIM) return O_E_OVERFLOW;
    c += cm;
    if (c > LIM) return O_E_OVERFLOW;
    i128 ct = (i128)D * (i128)time;
    if (ct > LIM) return O_E_OVERFLOW;
    c += ct;
    if (c > LIM) return O_E_OVERFLOW;
    *cost = (int64_t)c;
    return O_OK;
}

/* ------------------------------------------------------------------------
 * Stage loads, imbalance and potential.
 * L_i = sum of c_j over the layers assigned to worker i.
 * Delta L = (L_max - L_min) / ((1/n) sum L_j)   (eq:imbalance),
 *   evaluated in fp64 as (double)(Lmax-Lmin) / ((double)sumL / (double)n);
 *   0 when sumL == 0 (reading Q18).
 * phi = sum over unordered pairs u<v of |x_u - x_v|  (reading Q12).
 * ---------------------------------------------------------------------- */
void oracle_stage_loads(const int64_t *cost, int32_t n, const int32_t *bnd, int64_t *x) {
    for (int32_t s = 0; s < n; ++s) {
        int64_t acc = 0;
        for (int32_t j = bnd[s]; j < bnd[s + 1]; ++j) acc += cost[j];
        x[s] = acc;
    }
}

double oracle_imbalance(const int64_t *x, int32_t n) {
    int64_t mx = x[0], mn = x[0], sum = 0;
    for (int32_t s = 0; s < n; ++s) {
        if (x[s] > mx) mx = x[s];
        if (x[s] < mn) mn = x[s];
        sum += x[s];
    }
    if (sum == 0) return 0.0;
    double mean = (double)sum / (double)n;
    return (double)(mx - mn) / mean;
}

/* Returns OVERFLOW if phi does not fit in int64. */
int oracle_phi(const int64_t *x, int32_t n, int64_t *phi) {
    i128 acc = 0;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v) {
            i128 d = (i128)x[u] - (i128)x[v];
            acc += d < 0 ? -d : d;
        }
    if (acc > (i128)INT64_MAX) { *phi = -1; return O_E_OVERFLOW; }
    *phi = (int64_t)acc;
    return O_OK;
}

double oracle_phi_f64(const double *x, int32_t n) {
    double acc = 0.0;
    for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v)
            acc = acc + fabs(x[u] - x[v]);
    return acc;
}

/* ------------------------------------------------------------------------
 * O4 contiguous min-max partition (P:L149-171 objective; pipeline stages are
 * contiguous runs; memory "subject to the constraints of memory
 * capacity per worker" P:L428 folded in as a per-stage cap, reading Q9).
 *
 * B* = min over all 0=b_0<b_1<...<b_n=L with every stage mem <= cap of
 *      max_s (P[b_{s+1}] - P[b_s]).
 * Method (independent of the GPU bisection): DP f[s][j] = best bottleneck of
 * the first j layers in s stages; then suffix table g[r][j] = "layers j..L-1
 * can form exactly r stages each with cost <= B* and mem <= cap"; the output
 * is the lexicographically largest (b_1..b_{n-1}) among minimisers (Q7),
 * chosen greedily left to right with g.
 * On error: bnd[] = -1, *bottleneck = -1, *imbalance = -1.0.
 * ---------------------------------------------------------------------- */
/* Prefix sums of one array.  A negative entry anywhere is INVALID, checked
 * before the sum (so the status does not depend on where the running sum
 * first exceeds INT64_MAX); then a sum above INT64_MAX is OVERFLOW. */
static int build_prefix(const int64_t *v, int32_t L, int64_t *P) {
    for (int32_t i = 0; i < L; ++i)
        if (v[i] < 0) return O_E_INVALID;
    i128 acc = 0;
    P[0] = 0;
    for (int32_t i = 0; i < L; ++i) {
        acc += v[i];
        if (acc > (i128)INT64_MAX) return O_E_OVERFLOW;
        P[i + 1] = (int64_t)acc;
    }
    return O_OK;
}

static void fail_partition(int32_t n, int32_t *bnd, int64_t *bottleneck, double *imbalance) {
    if (bnd && n >= 0)
        for (int32_t s = 0; s <= n; ++s) bnd[s] = -1;
    if (bottleneck) *bottleneck = -1;
    if (imbalance) *imbalance = -1.0;
}

int oracle_partition(const int64_t *cost, const int64_t *mem, int32_t L, int32_t n,
                     int64_t cap, int32_t *bnd, int64_t *bottleneck, double *imbalance) {
    if (L < 1 || n < 1 || n > L || (mem && cap < 0)) {
        fail_partition(n > 0 ? n : -1, bnd, bottleneck, imbalance);
        return O_E_INVALID;
    }
    int64_t *P = malloc(sizeof(int64_t) * (L + 1));
    int64_t *M = malloc(sizeof(int64_t) * (L + 1));
    int st = build_prefix(cost, L, P);
    if (st == O_OK && mem) st = build_prefix(mem, L, M);
    if (st == O_OK && !mem) memset(M, 0, sizeof(int64_t) * (L + 1));
    if (st != O_OK) {
        free(P); free(M);
        fail_partition(n, bnd, bottleneck, imbalance);
        return st;
    }
    /* f[s][j] = best bottleneck of the first j layers in s stages, valid
     * where ok[s][j] (an explicit flag: INT64_MAX itself is a legal B*). */
    const size_t W = (size_t)(L + 1);
    int64_t *f = malloc(sizeof(int64_t) * (size_t)(n + 1) * W);
    unsigned char *ok = calloc((size_t)(n + 1) * W, 1);
    ok[0] = 1; f[0] = 0; /* zero stages cover zero layers */
    for (int32_t s = 1; s <= n; ++s)
        for (int32_t j = 1; j <= L; ++j) {
            int have = 0;
            int64_t best = 0;
            for (int32_t k = s - 1; k < j; ++k) {
                if (!ok[(s - 1) * W + k]) continue;
                if (mem && M[j] - M[k] > cap) continue;
                int64_t prev = f[(s - 1) * W + k];
                int64_t seg = P[j] - P[k];
                int64_t v = prev > seg ? prev : seg;
                if (!have || v < best) { best = v; have = 1; }
            }
            ok[s * W + j] = (unsigned char)have;
            f[s * W + j] = best;
        }
    int feasible = ok[n * W + L];
    int64_t Bs = f[n * W + L];
    free(f); free(ok);
    if (!feasible) {
        free(P); free(M);
        fail_partition(n, bnd, bottleneck, imbalance);
        return O_E_INFEASIBLE;
    }
    /* g[r][j]: layers j..L-1 split into exactly r non-empty stages, each
     * cost <= Bs and mem <= cap. */
    unsigned char *g = calloc((size_t)(n + 1) * (L + 1), 1);
    g[0 * (L + 1) + L] = 1;
    for (int32_t r = 1; r <= n; ++r)
        for (int32_t j = L - 1; j >= 0; --j) {
            unsigned char ok = 0;
            for (int32_t k = j + 1; k <= L && !ok; ++k) {
                if (P[k] - P[j] > Bs) continue;
                if (mem && M[k] - M[j] > cap) continue;
                if (g[(r - 1) * (L + 1) + k]) ok = 1;
            }
            g[r * (L + 1) + j] = ok;
        }
    bnd[0] = 0;
    for (int32_t s = 0; s < n; ++s) {
        int32_t pick = -1;
        for (int32_t k = bnd[s] + 1; k <= L; ++k) {
            if (P[k] - P[bnd[s]] > Bs) continue;
            if (mem && M[k] - M[bnd[s]] > cap) continue;
            if (g[(n - s - 1) * (L + 1) + k]) pick = k; /* keep the largest */
        }
        bnd[s + 1] = pick; /* pick >= 0 is guaranteed by g[n][0] */
    }
    free(g);
    int64_t *x = malloc(sizeof(int64_t) * n);
    oracle_stage_loads(cost, n, bnd, x);
    *bottleneck = Bs;
    if (imbalance) *imbalance = oracle_imbalance(x, n);
    free(x); free(P); free(M);
    return O_OK;
}

/* ------------------------------------------------------------------------
 * O5 re-pack.
 * (i) BOUND ("without sacrificing training throughput", P:L96,
 *     P:L820-822; readings Q15, Q16): for k = floor .. n_cur the first k
 *     whose exact constrained min-max (O4 at n=k) is <= bound; output O4's
 *     boundaries at that k.  If none: BOUND_UNMET with k = n_cur.
 * (ii) ALG2 (Alg. 2, with SPEC's fixes S:L389-390, reading Q14):
 *     first-fit over adjacent active workers, src ascending; merge src into
 *     dst = src+1 if mem[src]+mem[dst] < MAX_MEM (== <= cap, cap = MAX_MEM-1)
 *     and #active > target; deactivated src is skipped and zeroed.
 * On error: bnd[] = -1 over n_cur+1 entries, *n_new = -1, *bottleneck = -1.
 * ---------------------------------------------------------------------- */
static void fail_repack(int32_t n_cur, int32_t *bnd, int32_t *n_new, int64_t *bottleneck) {
    if (n_cur >= 0)
        for (int32_t s = 0; s <= n_cur; ++s) bnd[s] = -1;
    *n_new = -1;
    *bottleneck = -1;
}

int oracle_repack_bound(const int64_t *cost, const int64_t *mem, int32_t L, int32_t n_cur,
                        int64_t cap, int64_t bound, int32_t floor_, int32_t *n_new,
                        int32_t *bnd, int64_t *bottleneck) {
    if (L < 1 || n_cur < 1 || n_cur > L || floor_ < 1 || floor_ > n_cur || bound < 0) {
        fail_repack(n_cur > 0 ? n_cur : -1, bnd, n_new, bottleneck);
        return O_E_INVALID;
    }
    int32_t *tmp = malloc(sizeof(int32_t) * (n_cur + 1));
    for (int32_t k = floor_; k <= n_cur; ++k) {
        int64_t Bk;
        int st = oracle_partition(cost, mem, L, k, cap, tmp, &Bk, NULL);
        if (st == O_E_INVALID || st == O_E_OVERFLOW) {
            free(tmp);
            fail_repack(n_cur, bnd, n_new, bottleneck);
            return st;
        }
        if (st == O_OK && Bk <= bound) {
            for (int32_t s = 0; s <= n_cur; ++s) bnd[s] = s <= k ? tmp[s] : -1;
            *n_new = k;
            *bottleneck = Bk;
            free(tmp);
            return O_OK;
        }
    }
    int64_t Bn;
    int st = oracle_partition(cost, mem, L, n_cur, cap, tmp, &Bn, NULL);
    if (st != O_OK) {
        free(tmp);
        fail_repack(n_cur, bnd, n_new, bottleneck);
        return st;
    }
    for (int32_t s = 0; s <= n_cur; ++s) bnd[s] = tmp[s];
    *n_new = n_cur;
    *bottleneck = Bn;
    free(tmp);
    return O_W_BOUND_UNMET;
}

static int valid_bnd(const int32_t *b, int32_t n, int32_t L) {
    if (b[0] != 0 || b[n] != L) return 0;
    for (int32_t s = 0; s < n; ++s)
        if (b[s + 1] <= b[s]) return 0;
    return 1;
}

int oracle_repack_alg2(const int64_t *cost, const int64_t *mem, int32_t L, int32_t n_cur,
                       const int32_t *bnd_in, int64_t cap, int32_t target, int32_t *n_new,
                       int32_t *bnd, int64_t *bottleneck) {
    if (L < 1 || n_cur < 1 || n_cur > L || target < 1 || target > n_cur ||
        !valid_bnd(bnd_in, n_cur, L) || (mem && cap < 0)) {
        fail_repack(n_cur > 0 ? n_cur : -1, bnd, n_new, bottleneck);
        return O_E_INVALID;
    }
    for (int32_t i = 0; i < L; ++i)
        if (cost[i] < 0 || (mem && mem[i] < 0)) {
            fail_repack(n_cur, bnd, n_new, bottleneck);
            return O_E_INVALID;
        }
    /* mem_usage per worker; i128 so that a sum never wraps. */
    i128 *mu = malloc(sizeof(i128) * n_cur);
    int *active = malloc(sizeof(int) * n_cur);
    for (int32_t s = 0; s < n_cur; ++s) {
        i128 m = 0;
        if (mem)
            for (int32_t j = bnd_in[s]; j < bnd_in[s + 1]; ++j) m += mem[j];
        mu[s] = m;
        active[s] = 1;
    }
    int32_t n_active = n_cur;
    /* Alg. 2 lines 2-3: src ascending; dst restricted to the next active
     * worker (adjacent merge keeps the pipeline a chain).  Workers
     * deactivated so far are all < src, so the next active one is src+1. */
    for (int32_t src = 0; src + 1 < n_cur; ++src) {
        if (!active[src]) continue; /* SPEC fix S:L364 */
        int32_t dst = src + 1;
        /* Alg. 2 line 4: mem[src] + mem[dst] < MAX_MEM, i.e. <= cap. */
        int fits = !mem || (mu[src] + mu[dst] <= (i128)cap);
        if (fits && n_active > target) {
            active[src] = 0;       /* line 5 */
            mu[dst] += mu[src];    /* line 9 */
            mu[src] = 0;           /* SPEC fix S:L364 */
            n_active--;
        }
    }
    int32_t k = 0;
    bnd[0] = 0;
    for (int32_t s = 0; s < n_cur; ++s)
        if (active[s]) bnd[++k] = bnd_in[s + 1];
    for (int32_t s = k + 1; s <= n_cur; ++s) bnd[s] = -1;
    *n_new = k;
    int64_t *x = malloc(sizeof(int64_t) * k);
    int64_t *P = malloc(sizeof(int64_t) * (L + 1));
    int st = build_prefix(cost, L, P);
    if (st != O_OK) {
        free(x); free(P); free(mu); free(active);
        fail_repack(n_cur, bnd, n_new, bottleneck);
        return st;
    }
    int64_t bmax = 0;
    for (int32_t s = 0; s < k; ++s) {
        x[s] = P[bnd[s + 1]] - P[bnd[s]];
        if (x[s] > bmax) bmax = x[s];
    }
    *bottleneck = bmax;
    free(x); free(P); free(mu); free(active);
    return n_active > target ? O_W_BOUND_UNMET : O_OK;
}

/* ------------------------------------------------------------------------
 * O6 discrete diffusion ("move layers from overloaded workers to
 * underloaded ones in an iterative way"; "max neighbor algorithm";
 * P:L526 pairs "connected and averaged their workloads"
 * "prioritizing layer transfers that yield the largest reductions in
 * imbalance while satisfying memory constraints"; reading Q10).
 *
 * One round:
 *   x_s = stage loads; phi = sum_{u<v} |x_u-x_v|; stop (OK) if phi <= gamma.
 *   For each edge e = (e, e+1): over j in (b_e, b_{e+2}) with both sides
 *   mem <= cap, the minimum of key (max(P[j]-P[b_e], P[b_{e+2}]-P[j]),
 *   |j - b_{e+1}|, j).  e is improvable iff that max < max(x_e, x_{e+1}).
 *   Stop (OK) if no edge is improvable; stop (NOT_CONVERGED) if
 *   rounds == max_rounds.  Each stage picks, among its improvable incident
 *   edges, the one with the largest |x_e - x_{e+1}| (ties: lower edge index);
 *   edge e is matched iff stages e and e+1 both picked it; every matched
 *   edge moves b_{e+1} to its best j (matched edges are disjoint); rounds++.
 * Outputs b_out, rounds, phi (final), phi0 (initial).
 * On error: bnd_out[] = -1, rounds = -1, phi = phi0 = -1.
 * ---------------------------------------------------------------------- */
int oracle_diffuse(const int64_t *cost, const int64_t *mem, int32_t L, int32_t n, int64_t cap,
                   const int32_t *bnd_in, int64_t gamma, int32_t max_rounds,
                   int32_t *bnd_out, int32_t *rounds, int64_t *phi_out, int64_t *phi0_out) {
    *rounds = -1; *phi_out = -1; *phi0_out = -1;
    if (L < 1 || n < 1 || n > L || max_rounds < 0 || gamma < 0 || (mem && cap < 0) ||
        !valid_bnd(bnd_in, n, L)) {
        for (int32_t s = 0; n >= 1 && s <= n; ++s) bnd_out[s] = -1;
        return O_E_INVALID;
    }
    int64_t *P = malloc(sizeof(int64_t) * (L + 1));
    int64_t *M = malloc(sizeof(int64_t) * (L + 1));
    int st = build_prefix(cost, L, P);
    if (st == O_OK && mem) st = build_prefix(mem, L, M);
    if (st == O_OK && !mem) memset(M, 0, sizeof(int64_t) * (L + 1));
    if (st != O_OK) {
        free(P); free(M);
        for (int32_t s = 0; s <= n; ++s) bnd_out[s] = -1;
        return st;
    }
    int32_t *b = malloc(sizeof(int32_t) * (n + 1));
    memcpy(b, bnd_in, sizeof(int32_t) * (n + 1));
    int64_t *x = malloc(sizeof(int64_t) * n);
    int *impr = malloc(sizeof(int) * (n > 1 ? n - 1 : 1));
    int32_t *tgt = malloc(sizeof(int32_t) * (n > 1 ? n - 1 : 1));
    int32_t *pick = malloc(sizeof(int32_t) * n);
    int32_t r = 0;
    int result = O_OK;
    int64_t phi = 0;
    for (;;) {
        for (int32_t s = 0; s < n; ++s) x[s] = P[b[s + 1]] - P[b[s]];
        st = oracle_phi(x, n, &phi);
        if (st != O_OK) { result = st; break; }
        if (r == 0) *phi0_out = phi;
        if (phi <= gamma) break;
        int any = 0;
        for (int32_t e = 0; e + 1 < n; ++e) {
            int32_t lo = b[e], hi = b[e + 2], cur = b[e + 1];
            int found = 0;
            int64_t bk_max = 0; int32_t bk_dist = 0, bk_j = 0;
            for (int32_t j = lo + 1; j <= hi - 1; ++j) {
                if (mem && (M[j] - M[lo] > cap || M[hi] - M[j] > cap)) continue;
                int64_t a = P[j] - P[lo], c = P[hi] - P[j];
                int64_t km = a > c ? a : c;
                int32_t kd = j > cur ? j - cur : cur - j;
                if (!found || km < bk_max || (km == bk_max && kd < bk_dist) ||
                    (km == bk_max && kd == bk_dist && j < bk_j)) {
                    found = 1; bk_max = km; bk_dist = kd; bk_j = j;
                }
            }
            int64_t pair_max = x[e] > x[e + 1] ? x[e] : x[e + 1];
            impr[e] = found && bk_max < pair_max;
            tgt[e] = bk_j;
            if (impr[e]) any = 1;
        }
        if (!any) break;
        if (r == max_rounds) { result = O_W_NOT_CONVERGED; break; }
        for (int32_t s = 0; s < n; ++s) {
            pick[s] = -1;
            int64_t best_gap = -1;
            /* incident edges in ascending index: s-1 then s */
            for (int32_t e = s - 1; e <= s; ++e) {
                if (e < 0 || e + 1 >= n || !impr[e]) continue;
                int64_t gap = x[e] > x[e + 1] ? x[e] - x[e + 1] : x[e + 1] - x[e];
                if (gap > best_gap) { best_gap = gap; pick[s] = e; }
            }
        }
        for (int32_t e = 0; e + 1 < n; ++e)
            if (impr[e] && pick[e] == e && pick[e + 1] == e) b[e + 1] = tgt[e];
        r++;
    }
    if (result < 0) {
        for (int32_t s = 0; s <= n; ++s) bnd_out[s] = -1;
        *rounds = -1; *phi_out = -1; *phi0_out = -1;
    } else {
        memcpy(bnd_out, b, sizeof(int32_t) * (n + 1));
        *rounds = r;
        *phi_out = phi;
    }
    free(P); free(M); free(b); free(x); free(impr); free(tgt); free(pick);
    return result;
}

/* ------------------------------------------------------------------------
 * O6' fluid diffusion: the process analysed in Lemma 2's proof:
 * real-valued loads, pairs "connected and averaged their workloads"
 * under the max-neighbor rule.  x(0) = (double) stage loads of
 * bnd_in.  Per round: phi_f = sum_{u<v} |x_u - x_v| in ascending (u, v)
 * order; stop if phi_f <= gamma_f; NOT_CONVERGED if rounds == max_rounds;
 * each stage picks its incident edge with the largest gap > 0 (ties: lower
 * edge index); matched edges set both ends to (x_e + x_{e+1}) * 0.5.
 * IEEE double, round-to-nearest, no contraction (-ffp-contract=off).
 * On error: x[] = -1, rounds = -1, phi = -1.
 * ---------------------------------------------------------------------- */
int oracle_diffuse_fluid(const int64_t *cost, int32_t L, int32_t n, const int32_t *bnd_in,
                         double gamma_f, int32_t max_rounds, double *x, int32_t *rounds,
                         double *phi_out) {
    *rounds = -1; *phi_out = -1.0;
    if (L < 1 || n < 1 || n > L || max_rounds < 0 || !(gamma_f >= 0.0) ||
        !valid_bnd(bnd_in, n, L)) {
        for (int32_t s = 0; n >= 0 && s < n; ++s) x[s] = -1.0;
        return O_E_INVALID;
    }
    int64_t *P = malloc(sizeof(int64_t) * (L + 1));
    int st = build_prefix(cost, L, P);
    if (st != O_OK) {
        free(P);
        for (int32_t s = 0; s < n; ++s) x[s] = -1.0;
        return st;
    }
    for (int32_t s = 0; s < n; ++s) x[s] = (double)(P[bnd_in[s + 1]] - P[bnd_in[s]]);
    free(P);
    int32_t *pick = malloc(sizeof(int32_t) * n);
    int32_t r = 0;
    int result = O_OK;
    double phi;
    for (;;) {
        phi = oracle_phi_f64(x, n);
        if (phi <= gamma_f) break;
        if (r == max_rounds) { result = O_W_NOT_CONVERGED; break; }
        for (int32_t s = 0; s < n; ++s) {
            pick[s] = -1;
            double best_gap = 0.0;
            for (int32_t e = s - 1; e <= s; ++e) {
                if (e < 0 || e + 1 >= n) continue;
                double gap = fabs(x[e] - x[e + 1]);
                if (gap > best_gap) { best_gap = gap; pick[s] = e; }
            }
        }
        for (int32_t e = 0; e + 1 < n; ++e)
            if (pick[e] == e && pick[e + 1] == e) {
                double avg = (x[e] + x[e + 1]) * 0.5;
                x[e] = avg;
                x[e + 1] = avg;
            }
        r++;
    }
    *rounds = r;
    *phi_out = phi;
    free(pick);
    return result;
}

/* ------------------------------------------------------------------------
 * O7 migration plan ("When a layer is migrated from GPU A to GPU B";
 * Alg. 2 transfers list P:L568-578).  Layer i lives on rank_old[stage_old(i)]
 * before and rank_new[stage_new(i)] after; a move (i, src, dst) is emitted,
 * i ascending, whenever the two ranks differ.  Returns the move count.
 * ---------------------------------------------------------------------- */
int32_t oracle_moves(int32_t L, int32_t n_old, const int32_t *bnd_old, const int32_t *rank_old,
                     int32_t n_new, const int32_t *bnd_new, const int32_t *rank_new,
                     int32_t *moves /* [L][3] */) {
    int32_t m = 0;
    for (int32_t i = 0; i < L; ++i) {
        int32_t so = -1, sn = -1;
        for (int32_t s = 0; s < n_old; ++s)
            if (bnd_old[s] <= i && i < bnd_old[s + 1]) so = s;
        for (int32_t s = 0; s < n_new; ++s)
            if (bnd_new[s] <= i && i < bnd_new[s + 1]) sn = s;
        if (so < 0 || sn < 0) return -1;
        if (rank_old[so] != rank_new[sn]) {
            moves[3 * m + 0] = i;
            moves[3 * m + 1] = rank_old[so];
            moves[3 * m + 2] = rank_new[sn];
            m++;
        }
    }
    return m;
}

/* ------------------------------------------------------------------------
 * O8 global magnitude pruning (Algorithm 1):
 * over the concatenation of every rank's parameters (rank order, then the
 * rank's segments in order) keep exactly k parameters with the largest
 * magnitude |w| (Alg. 1 lines 2-3 "k <- num_params (1 - sparsity)",
 * "topk(abs(params), k)"; line 6 the global top-k); equal magnitudes are
 * broken by global position ascending (SPEC: "(shard id, local index)
 * ascending").  mask[j] = 1 keep, 0 prune.  Magnitudes are compared as
 * doubles (f32 and bf16 convert exactly).  A NaN is never kept and makes
 * the status INVALID; k < 0 or k > #non-NaN is INVALID (then nothing is
 * written).  The paper's gather to rank 0 / scatter of indices is data
 * movement; the kept SET is what this function defines.
 * Plain O(N log N) sort of positions by (|w| desc, position asc).
 * ---------------------------------------------------------------------- */
static const double *g_mag;
static int cmp_mag_desc(const void *a, const void *b) {
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    if (g_mag[i] > g_mag[j]) return -1;
    if (g_mag[i] < g_mag[j]) return 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

int oracle_global_prune(const double *w, int64_t n, int64_t k, uint8_t *mask) {
    int st = O_OK;
    double *mag = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    for (int64_t j = 0; j < n; ++j) {
        mag[j] = fabs(w[j]);
        if (isnan(w[j])) st = O_E_INVALID;
        else pos[m++] = j;
    }
    if (k < 0 || k > m) {
        free(mag);
        free(pos);
        return O_E_INVALID;
    }
    g_mag = mag;
    qsort(pos, (size_t)m, sizeof(int64_t), cmp_mag_desc);
    for (int64_t j = 0; j < n; ++j) mask[j] = 0;
    for (int64_t r = 0; r < k; ++r) mask[pos[r]] = 1;
    free(mag);
    free(pos);
    return st;
}

/* ------------------------------------------------------------------------
 * O9 migration-minimising stage -> rank map (NEXT-3; P:L636 a migrated
 * layer is released on GPU A and allocated on GPU B, P:L600 re-packing to
 * fewer GPUs; reading Q23): layer i is on rank owner(i) = rank_old[stage_old(i)]
 * before; the new split has n_new stages, each placed on a distinct rank of
 * `allowed` (bit mask over G <= 16 ranks).  kept(pi) = sum of bytes[i] over
 * layers whose new stage s has pi[s] == owner(i).  Returns the pi with the
 * largest kept bytes, the lexicographically smallest such vector, defined by
 *   f(used) = 0 if |used| = n_new, else max over g in allowed \ used of
 *             w[|used|][g] + f(used + g)      (w[s][g] = bytes of new stage s on g)
 * and the greedy lexicographic walk of f.  INFEASIBLE if n_new > |allowed|,
 * INVALID on malformed splits or G outside [1, 16].  With slot_rank (several
 * stages per GPU: the G "ranks" are slots, slot_rank[j] its GPU) a byte is
 * kept when the GPU of its new slot equals the GPU of its old slot, and the
 * output is rank_new[s] = slot_rank[slot].
 * ---------------------------------------------------------------------- */
int oracle_map_stages(int32_t L, int32_t n_old, const int32_t *bnd_old, const int32_t *rank_old,
                      int32_t n_new, const int32_t *bnd_new, const int64_t *bytes, int32_t G,
                      uint32_t allowed, const int32_t *slot_rank, int32_t *rank_new, int64_t *kept) {
    *kept = -1;
    if (G < 1 || G > 16 || n_new < 1 || n_old < 1 || L < 1) return O_E_INVALID;
    if (bnd_old[0] != 0 || bnd_old[n_old] != L || bnd_new[0] != 0 || bnd_new[n_new] != L) return O_E_INVALID;
    for (int32_t s = 0; s < n_old; ++s)
        if (bnd_old[s + 1] <= bnd_old[s] || rank_old[s] < 0 || rank_old[s] >= G) return O_E_INVALID;
    for (int32_t s = 0; s < n_new; ++s)
        if (bnd_new[s + 1] <= bnd_new[s]) return O_E_INVALID;
    for (int32_t i = 0; i < L; ++i)
        if (bytes[i] < 0) return O_E_INVALID;
    allowed &= (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u));
    if (n_new > __builtin_popcount(allowed)) return O_E_INFEASIBLE;
    int64_t w[32][16];
    memset(w, 0, sizeof(w));
    for (int32_t s = 0; s < n_new; ++s)
        for (int32_t i = bnd_new[s]; i < bnd_new[s + 1]; ++i) {
            int32_t so = 0;
            while (!(bnd_old[so] <= i && i < bnd_old[so + 1])) ++so;
            if (slot_rank) {
                for (int32_t g = 0; g < G; ++g)
                    if (slot_rank[g] == slot_rank[rank_old[so]]) w[s][g] += bytes[i];
            } else {
                w[s][rank_old[so]] += bytes[i];
            }
        }
    const uint32_t NS = 1u << G;
    int64_t *f = (int64_t *)malloc(sizeof(int64_t) * NS);
    for (int32_t k = G; k >= 0; --k)
        for (uint32_t u = 0; u < NS; ++u) {
            if (__builtin_popcount(u) != k || (u & ~allowed)) continue;
            if (k >= n_new) { f[u] = 0; continue; }
            int64_t best = -1;
            for (int32_t g = 0; g < G; ++g) {
                if (!((allowed >> g) & 1u) || ((u >> g) & 1u)) continue;
                int64_t v = w[k][g] + f[u | (1u << g)];
                if (v > best) best = v;
            }
            f[u] = best;
        }
    uint32_t used = 0;
    for (int32_t s = 0; s < n_new; ++s)
        for (int32_t g = 0; g < G; ++g) {
            if (!((allowed >> g) & 1u) || ((used >> g) & 1u)) continue;
            if (w[s][g] + f[used | (1u << g)] == f[used]) {
                rank_new[s] = slot_rank ? slot_rank[g] : g;
                used |= 1u << g;
                break;
            }
        }
    *kept = f[0];
    free(f);
    return O_OK;
}

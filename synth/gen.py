"""Seeded synthetic workloads of the paper's five configs (BASELINE.json).

Every draw comes from numpy PCG64 seeded by SeedSequence([2505_14864, cfg,
...keys]), so any rank can regenerate exactly the layers it owns and the
result equals a single-host generation.  Recipes: DESIGN.md "Input recipe".
No method arithmetic lives here (no counting, costing or partitioning).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BASE_SEED = 2505_14864


def rng(*keys: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, *keys])))


# ----------------------------------------------------------------------------
# Eq. 3 gradual pruning schedule (milestones P:L751, reading Q17).
def sparsity_at(t: float, S_i: float = 0.0, S_f: float = 0.9, t0: float = 3000.0,
                n_dt: float = 4000.0) -> float:
    """S_t = S_f + (S_i - S_f)(1 - (t - t0)/(n dt))^3, clamped to [t0, t0 + n dt]."""
    u = min(max((t - t0) / n_dt, 0.0), 1.0)
    return S_f + (S_i - S_f) * (1.0 - u) ** 3


PRUNE_MILESTONES = [sparsity_at(t) for t in (3000, 4000, 5000, 6000, 7000)]


# ----------------------------------------------------------------------------
# Config 1: 24-layer cost vectors on 4 stages (partition + repack vs brute force)
def cfg1_instances(count: int, L: int = 24, seed_key: int = 0):
    """Five families, round-robin; mem on 2 of 3."""
    out = []
    for k in range(count):
        g = rng(1, seed_key, k)
        fam = k % 5
        if fam == 0:      # GPT cost model, random per-layer density in [0.05, 1]
            d = g.uniform(0.05, 1.0, L)
            cost = np.rint(1000 + 11000 * d).astype(np.int64)
        elif fam == 1:    # freezing prefix: zeros in front
            F = int(g.integers(0, L // 2 + 1))
            cost = g.integers(80, 121, L).astype(np.int64)
            cost[:F] = 0
        elif fam == 2:    # all equal
            cost = np.full(L, int(g.integers(1, 50)), np.int64)
        elif fam == 3:    # one heavy layer
            cost = np.full(L, 10, np.int64)
            cost[int(g.integers(0, L))] = 10 * L
        else:             # small alphabet, forces ties
            cost = g.choice(np.array([0, 1, 2, 3, 5, 9], np.int64), L)
        mem = None
        cap = 0
        if k % 3 != 2:
            mem = g.integers(1, 101, L).astype(np.int64)
            cap = int(max(mem.max(), math.ceil(mem.sum() / 4 * g.uniform(1.0, 1.6))))
        bound = int(math.ceil(int(cost.sum()) * g.uniform(0.2, 1.0)))
        out.append(dict(cost=cost, mem=mem, cap=cap, n=4, bound=bound, floor=1))
    return out


# ----------------------------------------------------------------------------
# Config 2: GPT-48 gradual global magnitude pruning, masks per weight tensor.
@dataclass
class GPTShape:
    L: int = 48
    h: int = 1024

    @property
    def tensors(self):
        h = self.h
        # QKV 3h x h, proj h x h, fc1 4h x h, fc2 h x 4h (12 h^2 per layer)
        return [(3 * h, h), (h, h), (4 * h, h), (h, 4 * h)]

    @property
    def params_per_layer(self) -> int:
        return sum(r * c for r, c in self.tensors)

    @property
    def rows_per_layer(self) -> int:
        return sum(r for r, _ in self.tensors)


def _sigmas(shape: GPTShape, milestone: int) -> np.ndarray:
    """sigma_{l,t} = exp(N(0, 0.35^2)) * (1 + l/L)^0.5 per layer and tensor."""
    g = rng(2, 0, milestone)
    z = g.normal(0.0, 0.35, (shape.L, len(shape.tensors)))
    depth = (1.0 + np.arange(shape.L) / shape.L) ** 0.5
    return np.exp(z) * depth[:, None]


def cfg2_keep_probs(shape: GPTShape, S: float, milestone: int) -> np.ndarray:
    """Per-(layer, tensor) keep probability of a GLOBAL magnitude threshold tau
    over weights w ~ N(0, sigma^2): p = P(|w| > tau) = erfc(tau/(sigma sqrt 2)),
    tau chosen so that the expected kept count is (1 - S) N (Alg. 1
    keeps the global top-k, k = N(1 - S), line 2)."""
    sig = _sigmas(shape, milestone)
    n = np.array([r * c for r, c in shape.tensors], np.float64)[None, :]
    if S <= 0.0:
        return np.ones_like(sig)
    target = (1.0 - S) * n.sum() * shape.L
    lo, hi = 0.0, 50.0 * sig.max()
    erfc = np.vectorize(math.erfc)
    for _ in range(200):
        tau = 0.5 * (lo + hi)
        kept = (n * erfc(tau / (sig * math.sqrt(2.0)))).sum()
        if kept > target:
            lo = tau
        else:
            hi = tau
    return erfc(0.5 * (lo + hi) / (sig * math.sqrt(2.0)))


def cfg2_layer_masks_u8(shape: GPTShape, layer: int, p_layer: np.ndarray, milestone: int):
    """Bool/uint8 masks (1 = kept) of the four weight tensors of one layer."""
    out = []
    for t, (r, c) in enumerate(shape.tensors):
        g = rng(2, 1, milestone, layer, t)
        thr = int(round(float(p_layer[t]) * 65536.0))
        u = g.integers(0, 65536, size=r * c, dtype=np.uint16)
        out.append((u < thr).view(np.uint8).reshape(r, c))
    return out


def cfg2_payload_bytes(shape: GPTShape, p: np.ndarray) -> np.ndarray:
    """Expected CSR migration payload per layer (reading Q19): bf16 values +
    int32 column indices + fp32 master/m/v per kept weight (18 B) + int32 row
    pointers.  Caller-side metadata (the trainer owns the CSR tensors)."""
    n = np.array([r * c for r, c in shape.tensors], np.float64)[None, :]
    nnz = np.rint((p * n).sum(axis=1)).astype(np.int64)
    rowptr = (shape.rows_per_layer + len(shape.tensors)) * 4
    return nnz * 18 + rowptr


CFG2_TAU_BF16 = 0x3C00  # bf16 bit pattern of the global magnitude threshold (2^-7)


def cfg2_topk_weights_bf16(mask_u8: np.ndarray, layer: int, t: int, milestone: int = 4) -> np.ndarray:
    """bf16 weights whose GLOBAL top-k by magnitude (Alg. 1) is
    exactly the given masks, k = the masks' kept count: every kept weight has
    a magnitude bit pattern in [TAU, TAU + 1024) and every pruned one in
    [0, TAU) (positive bf16 patterns are ordered like their values), so no
    pruned magnitude reaches any kept one and there is no tie across the
    threshold.  Random signs.  With cfg2_layer_masks_u8's Bernoulli draws
    under the erfc threshold of cfg2_keep_probs this makes the config-2
    masks the exact global top-k of these weights (no selection is done
    here: the order holds by construction)."""
    g = rng(2, 3, milestone, layer, t)
    kept = g.integers(CFG2_TAU_BF16, CFG2_TAU_BF16 + 1024, mask_u8.shape, dtype=np.uint16)
    pruned = g.integers(0, CFG2_TAU_BF16, mask_u8.shape, dtype=np.uint16)
    sign = (g.integers(0, 2, mask_u8.shape, dtype=np.uint16) << 15).astype(np.uint16)
    return (np.where(mask_u8 != 0, kept, pruned) | sign).astype(np.uint16)


def cfg2_bf16_weights(mask_u8: np.ndarray, layer: int, t: int) -> np.ndarray:
    """bf16 bit patterns of masked weights: pruned -> +0 or -0 (random sign),
    kept -> nonzero normal draws (small tests only)."""
    g = rng(2, 2, layer, t)
    w = g.normal(0.0, 1.0, mask_u8.shape).astype(np.float32)
    bits = (w.view(np.uint32) >> 16).astype(np.uint16)
    bits[(bits & 0x7FFF) == 0] |= 1  # kept weights must be nonzero in bf16
    sign = (g.integers(0, 2, mask_u8.shape, dtype=np.uint16) << 15).astype(np.uint16)
    return np.where(mask_u8 != 0, bits, sign).astype(np.uint16)


def pack_bits(mask_u8: np.ndarray) -> np.ndarray:
    """Little-endian bit packing into uint32 words (bit b -> word b/32, bit b%32)."""
    flat = np.ascontiguousarray(mask_u8).reshape(-1)
    nbytes = (flat.size + 7) // 8
    pad = (-nbytes) % 4
    by = np.packbits(flat != 0, bitorder="little")
    if pad:
        by = np.concatenate([by, np.zeros(pad, np.uint8)])
    return by.view(np.uint32)


# ----------------------------------------------------------------------------
# Config 3: GPT-32 freezing + early exit, 512 x 2048 tokens.
def cfg3_exit_depth(T: int = 512 * 2048, L: int = 32, first_exit: int = 8,
                    p_exit: float = 0.08, seed_key: int = 0) -> np.ndarray:
    """e[t] = number of layers processed by token t.  No exits before layer
    `first_exit`; after processing each layer l >= first_exit a token
    exits with probability p_exit; survivors reach all L layers."""
    g = rng(3, seed_key)
    k = g.geometric(p_exit, T)
    return np.minimum(first_exit + k, L).astype(np.uint8)


def cfg3_frozen(L: int = 32, F: int = 8) -> np.ndarray:
    """Egeria-like front-to-back freezing: layers < F frozen."""
    f = np.zeros(L, np.uint8)
    f[:F] = 1
    return f


# ----------------------------------------------------------------------------
# Config 4: Mixtral-8x7B-shaped MoE routing.
MIXTRAL_LAYER_PARAMS = 41_943_040 + 8 * 176_160_768  # attn + 8 experts (3 x 4096 x 14336)


def cfg4_routing(layer: int, T: int = 64 * 2048, E: int = 8, k: int = 2, alpha: float = 4.0,
                 dtype=np.int64, seed_key: int = 0) -> np.ndarray:
    """Top-k expert indices [T, k] (distinct experts per token) drawn from a
    per-layer popularity pi ~ Dirichlet(alpha): alpha=4 'aux-loss' (skewed),
    alpha=64 'S-BASE' (near balanced).  Gumbel-top-k sampling."""
    g = rng(4, seed_key, layer, int(alpha))
    pi = g.dirichlet(np.full(E, alpha))
    gumb = -np.log(-np.log(g.random((T, E))))
    score = np.log(pi)[None, :] + gumb
    idx = np.argpartition(-score, k - 1, axis=1)[:, :k]
    return np.ascontiguousarray(idx.astype(dtype))


def cfg4_alpha_drift(layer: int, L: int = 32, a0: float = 64.0, a1: float = 0.3) -> float:
    """Routing popularity that drifts with depth: the
    Dirichlet concentration falls geometrically from a0 (S-BASE-like, near
    balanced) at layer 0 to a1 (strongly skewed) at layer L-1, so deep MoE
    layers carry more load imbalance -- the expert-parallel max group sets
    the layer time (reading Q5) -- and the balanced split moves layers."""
    return float(a0 * (a1 / a0) ** (layer / max(1, L - 1)))


def cfg4_routing_drift(layer: int, L: int = 32, T: int = 64 * 2048, E: int = 8, k: int = 2,
                       dtype=np.int64, seed_key: int = 0) -> np.ndarray:
    """Top-k ids [T, k] of layer `layer` under cfg4_alpha_drift (Gumbel-top-k,
    distinct experts per token)."""
    alpha = cfg4_alpha_drift(layer, L)
    g = rng(4, 1000 + seed_key, layer)
    pi = g.dirichlet(np.full(E, alpha))
    pi = np.maximum(pi, 1e-12)
    gumb = -np.log(-np.log(g.random((T, E))))
    score = np.log(pi)[None, :] + gumb
    idx = np.argpartition(-score, k - 1, axis=1)[:, :k]
    return np.ascontiguousarray(idx.astype(dtype))


# ----------------------------------------------------------------------------
# Config 5: batched sweep with MoD skip masks.
@dataclass
class SweepInstance:
    L: int
    n: int
    masks: np.ndarray          # uint32 [L, T/32] token bitmasks
    mem: np.ndarray            # int64 [L] caller-side memory per layer (bytes)
    cap: int                   # per-stage memory cap (bytes)
    bound: int                 # repack throughput bound (cost units = tokens)


def cfg5_instance(i: int, T: int = 4096, h: int = 1024) -> SweepInstance:
    g = rng(5, i)
    L = int(g.integers(48, 129))
    n = int(g.integers(2, min(8, L) + 1))
    words = T // 32
    masks = np.full((L, words), 0xFFFFFFFF, np.uint32)
    mem_param = 12 * h * h * 2          # bf16 weights of one block
    act = 20 * h                         # activation bytes per routed token
    mem = np.full(L, mem_param + T * act, np.int64)
    cap_frac = 0.125                     # MoD capacity 12.5% (Raposo et al.)
    for l in range(1, L, 2):             # MoD routing on every other block
        p = cap_frac * g.uniform(0.5, 1.5)
        bits = g.random(T) < p
        masks[l] = pack_bits(bits.astype(np.uint8))
        mem[l] = mem_param + int(round(p * T)) * act   # caller's expected activations
    cap = int(1.25 * L * (mem_param + T * act) / n)     # 1.25 x dense stage memory
    # throughput to sustain: the dense model's bottleneck under the uniform
    # split of ceil(L/n) layers per stage, each layer processing all T tokens
    bound = -(-L // n) * T
    return SweepInstance(L=L, n=n, masks=masks, mem=mem, cap=cap, bound=bound)


# ----------------------------------------------------------------------------
# "By Time" profiling input: per-layer timestamps of a profiling iteration.
def time_stamps(base_ns: np.ndarray, microbatches: int = 4, jitter: float = 0.05, gap_ns: int = 2000,
                t0: int = 1_760_000_000_000_000_000, seed_key: int = 0) -> np.ndarray:
    """Boundary stamps int64 [M, L+1] of M micro-batch forward passes through
    L layers (a monotonic ns clock like %globaltimer): layer i of micro-batch
    m runs from s[m, i] to s[m, i+1], lasting base_ns[i] * LogNormal(0, jitter)
    (rounded to ns); passes are separated by gap_ns.  base_ns is the caller's
    per-layer model of the execution time (e.g. proportional to kept params)."""
    base_ns = np.asarray(base_ns, np.float64)
    L = len(base_ns)
    g = rng(6, seed_key, L, microbatches)
    dur = np.maximum(1, np.rint(base_ns[None, :] * np.exp(g.normal(0.0, jitter, (microbatches, L))))).astype(np.int64)
    out = np.empty((microbatches, L + 1), np.int64)
    t = int(t0)
    for m in range(microbatches):
        out[m, 0] = t
        out[m, 1:] = t + np.cumsum(dur[m])
        t = int(out[m, -1]) + gap_ns
    return out


# ----------------------------------------------------------------------------
# Dynamic sparse (hash-based) flash attention block masks.
def sparse_attention_blocks(layer: int, T: int = 2048, block: int = 64, heads: int = 16, batch: int = 2,
                            seed_key: int = 0) -> np.ndarray:
    """Bit-packed (little-endian uint32) block masks [batch, heads, nb, nb],
    nb = T / block, of a hash-based sparse causal attention: query block i
    and key block j (j <= i) are computed iff their hash buckets match or
    j == i; the bucket count per layer is drawn from {2, 4, 8, 16}, so the
    sparsity s_i varies across layers ('varying sparsification across
    layers')."""
    nb = T // block
    g = rng(7, seed_key, layer)
    buckets = int(g.choice([2, 4, 8, 16]))
    qh = g.integers(0, buckets, (batch, heads, nb))
    kh = g.integers(0, buckets, (batch, heads, nb))
    i = np.arange(nb)[:, None]
    j = np.arange(nb)[None, :]
    causal = j <= i
    m = ((qh[:, :, :, None] == kh[:, :, None, :]) | (i == j)) & causal
    return pack_bits(m.reshape(-1).astype(np.uint8))

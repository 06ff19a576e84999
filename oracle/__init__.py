"""CPU oracle for the DynMo rebalancing hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2505_14864_b200``) never imports it; the two share no code.

This module is argument marshalling (numpy <-> ctypes) around
``dynmo_oracle.c``; every computation lives in that file, each function citing
the PAPER.md / SPEC.md passage it follows.  The shared library is compiled
with plain ``gcc -O2 -ffp-contract=off`` on first use (building the checker is
not using it).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dynmo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID, E_INFEASIBLE, E_OVERFLOW = 0, -1, -2, -3
W_NOT_CONVERGED, W_BOUND_UNMET = 1, 2


def build(force: bool = False) -> str:
    """Compile dynmo_oracle.c into liboracle.so (gcc, no shared headers)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
        p = C.c_void_p
        sig = {
            "oracle_count_bits": (i64, [p, i64]),
            "oracle_count_nz_u8": (i64, [p, i64]),
            "oracle_count_nz_bf16": (i64, [p, i64]),
            "oracle_count_nz_f32": (i64, [p, i64]),
            "oracle_exit_survivors": (None, [p, i64, i32, i32, p]),
            "oracle_expert_hist_i64": (C.c_int, [p, i64, i32, p]),
            "oracle_expert_hist_i32": (C.c_int, [p, i64, i32, p]),
            "oracle_layer_cost": (C.c_int, [C.c_int, C.c_int, i64, i64, C.c_int, p, i32,
                                            i64, i64, i64, i64, i32, i64, i64, p]),
            "oracle_time_ns": (C.c_int, [p, i64, p]),
            "oracle_stage_loads": (None, [p, i32, p, p]),
            "oracle_imbalance": (dbl, [p, i32]),
            "oracle_phi": (C.c_int, [p, i32, p]),
            "oracle_phi_f64": (dbl, [p, i32]),
            "oracle_partition": (C.c_int, [p, p, i32, i32, i64, p, p, p]),
            "oracle_repack_bound": (C.c_int, [p, p, i32, i32, i64, i64, i32, p, p, p]),
            "oracle_repack_alg2": (C.c_int, [p, p, i32, i32, p, i64, i32, p, p, p]),
            "oracle_diffuse": (C.c_int, [p, p, i32, i32, i64, p, i64, i32, p, p, p, p]),
            "oracle_diffuse_fluid": (C.c_int, [p, i32, i32, p, dbl, i32, p, p, p]),
            "oracle_moves": (i32, [i32, i32, p, p, i32, p, p, p]),
            "oracle_global_prune": (C.c_int, [p, i64, i64, p]),
            "oracle_map_stages": (C.c_int, [i32, i32, p, p, i32, p, p, i32, C.c_uint32, p, p, p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


# --------------------------------------------------------------- O1 counters
def count_bits(words: np.ndarray, n_bits: int) -> int:
    w = _c(words, np.uint32)
    return int(lib().oracle_count_bits(_ptr(w), int(n_bits)))


def count_nz_u8(a: np.ndarray) -> int:
    a = _c(a, np.uint8)
    return int(lib().oracle_count_nz_u8(_ptr(a), a.size))


def count_nz_bf16(bits16: np.ndarray) -> int:
    a = _c(bits16, np.uint16)
    return int(lib().oracle_count_nz_bf16(_ptr(a), a.size))


def count_nz_f32(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a).view(np.uint32) if a.dtype == np.float32 else _c(a, np.uint32)
    return int(lib().oracle_count_nz_f32(_ptr(a), a.size))


def exit_survivors(e: np.ndarray, layer_begin: int, n_local: int) -> np.ndarray:
    e = _c(e, np.uint8)
    tok = np.zeros(n_local, np.int64)
    lib().oracle_exit_survivors(_ptr(e), e.size, layer_begin, n_local, _ptr(tok))
    return tok


def expert_hist(idx: np.ndarray, E: int) -> tuple[int, np.ndarray]:
    cnt = np.zeros(E, np.int64)
    if idx.dtype == np.int32:
        a = _c(idx, np.int32)
        st = lib().oracle_expert_hist_i32(_ptr(a), a.size, E, _ptr(cnt))
    else:
        a = _c(idx, np.int64)
        st = lib().oracle_expert_hist_i64(_ptr(a), a.size, E, _ptr(cnt))
    return int(st), cnt


# ------------------------------------------------------------------ O2 cost
def time_ns(v: np.ndarray) -> tuple[int, int]:
    """(status, sum of end - begin) over (begin, end) int64 pairs."""
    a = _c(v, np.int64)
    out = np.zeros(1, np.int64)
    st = lib().oracle_time_ns(_ptr(a), a.size, _ptr(out))
    return int(st), int(out[0])


def layer_cost(*, frozen=False, tok=None, nnz=0, cnt=None, A=0, B=0, C_=0, F=0, ep=0, D=0, time=0):
    cost = np.zeros(1, np.int64)
    c = _c(cnt, np.int64) if cnt is not None else np.zeros(1, np.int64)
    E = 0 if cnt is None else len(cnt)
    st = lib().oracle_layer_cost(int(bool(frozen)), int(tok is not None),
                                 int(tok if tok is not None else 0), int(nnz),
                                 int(cnt is not None), _ptr(c), E, int(A), int(B), int(C_),
                                 int(F), int(ep), int(D), int(time), _ptr(cost))
    return int(st), int(cost[0])


# -------------------------------------------------------- loads / ΔL / φ
def stage_loads(cost, bnd):
    cost = _c(cost, np.int64)
    bnd = _c(bnd, np.int32)
    n = len(bnd) - 1
    x = np.zeros(n, np.int64)
    lib().oracle_stage_loads(_ptr(cost), n, _ptr(bnd), _ptr(x))
    return x


def imbalance(x) -> float:
    x = _c(x, np.int64)
    return float(lib().oracle_imbalance(_ptr(x), len(x)))


def phi(x) -> tuple[int, int]:
    x = _c(x, np.int64)
    out = np.zeros(1, np.int64)
    st = lib().oracle_phi(_ptr(x), len(x), _ptr(out))
    return int(st), int(out[0])


def phi_f64(x) -> float:
    x = _c(x, np.float64)
    return float(lib().oracle_phi_f64(_ptr(x), len(x)))


# ------------------------------------------------------------- O4 partition
def partition(cost, n, mem=None, cap=0):
    cost = _c(cost, np.int64)
    mem = _c(mem, np.int64)
    L = len(cost)
    bnd = np.zeros(max(n, 0) + 1, np.int32)
    bott = np.zeros(1, np.int64)
    imb = np.zeros(1, np.float64)
    st = lib().oracle_partition(_ptr(cost), _ptr(mem), L, int(n), int(cap), _ptr(bnd),
                                _ptr(bott), _ptr(imb))
    return int(st), bnd, int(bott[0]), float(imb[0])


# ---------------------------------------------------------------- O5 repack
def repack_bound(cost, n_cur, bound, floor=1, mem=None, cap=0):
    cost = _c(cost, np.int64)
    mem = _c(mem, np.int64)
    bnd = np.zeros(max(n_cur, 0) + 1, np.int32)
    n_new = np.zeros(1, np.int32)
    bott = np.zeros(1, np.int64)
    st = lib().oracle_repack_bound(_ptr(cost), _ptr(mem), len(cost), int(n_cur), int(cap),
                                   int(bound), int(floor), _ptr(n_new), _ptr(bnd), _ptr(bott))
    return int(st), int(n_new[0]), bnd, int(bott[0])


def repack_alg2(cost, bnd_in, target, mem=None, cap=0):
    cost = _c(cost, np.int64)
    mem = _c(mem, np.int64)
    bnd_in = _c(bnd_in, np.int32)
    n_cur = len(bnd_in) - 1
    bnd = np.zeros(n_cur + 1, np.int32)
    n_new = np.zeros(1, np.int32)
    bott = np.zeros(1, np.int64)
    st = lib().oracle_repack_alg2(_ptr(cost), _ptr(mem), len(cost), n_cur, _ptr(bnd_in),
                                  int(cap), int(target), _ptr(n_new), _ptr(bnd), _ptr(bott))
    return int(st), int(n_new[0]), bnd, int(bott[0])


# ------------------------------------------------------------- O6 diffusion
def diffuse(cost, bnd_in, gamma=0, max_rounds=256, mem=None, cap=0):
    cost = _c(cost, np.int64)
    mem = _c(mem, np.int64)
    bnd_in = _c(bnd_in, np.int32)
    n = len(bnd_in) - 1
    out = np.zeros(n + 1, np.int32)
    r = np.zeros(1, np.int32)
    ph = np.zeros(1, np.int64)
    ph0 = np.zeros(1, np.int64)
    st = lib().oracle_diffuse(_ptr(cost), _ptr(mem), len(cost), n, int(cap), _ptr(bnd_in),
                              int(gamma), int(max_rounds), _ptr(out), _ptr(r), _ptr(ph), _ptr(ph0))
    return int(st), out, int(r[0]), int(ph[0]), int(ph0[0])


def diffuse_fluid(cost, bnd_in, gamma_f=0.0, max_rounds=256):
    cost = _c(cost, np.int64)
    bnd_in = _c(bnd_in, np.int32)
    n = len(bnd_in) - 1
    x = np.zeros(n, np.float64)
    r = np.zeros(1, np.int32)
    ph = np.zeros(1, np.float64)
    st = lib().oracle_diffuse_fluid(_ptr(cost), len(cost), n, _ptr(bnd_in), float(gamma_f),
                                    int(max_rounds), _ptr(x), _ptr(r), _ptr(ph))
    return int(st), x, int(r[0]), float(ph[0])


# ------------------------------------------------------------ O7 migration
def moves(L, bnd_old, rank_old, bnd_new, rank_new) -> np.ndarray:
    bo, ro = _c(bnd_old, np.int32), _c(rank_old, np.int32)
    bn, rn = _c(bnd_new, np.int32), _c(rank_new, np.int32)
    out = np.zeros((max(L, 1), 3), np.int32)
    m = lib().oracle_moves(int(L), len(bo) - 1, _ptr(bo), _ptr(ro), len(bn) - 1, _ptr(bn),
                           _ptr(rn), _ptr(out))
    if m < 0:
        raise ValueError("boundaries do not cover every layer")
    return out[:m].copy()


# ------------------------------------------------------ O8 global pruning
def global_prune(shards, k: int):
    """Alg. 1: keep the k largest |w| over the concatenation of the shards
    (list of float arrays, bf16 given as uint16 bit patterns via
    bf16_to_f64).  Returns (status, [mask per shard])."""
    w = np.concatenate([np.asarray(x, np.float64).reshape(-1) for x in shards]) if shards else np.zeros(0)
    w = np.ascontiguousarray(w, np.float64)
    mask = np.zeros(max(1, w.size), np.uint8)
    st = lib().oracle_global_prune(_ptr(w), w.size, int(k), _ptr(mask))
    out, o = [], 0
    for x in shards:
        n = np.asarray(x).size
        out.append(mask[o:o + n].copy())
        o += n
    return int(st), out


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> exact float64 values."""
    b = np.asarray(bits, np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


# ----------------------------------------- O9 stage -> rank map (NEXT-3)
def map_stages(L, bnd_old, rank_old, bnd_new, nbytes, G, allowed=None, slot_rank=None):
    """(status, rank_new[n_new], kept_bytes): migration-minimising map of
    the new stages onto distinct allowed ranks (lexicographically smallest
    optimum); with slot_rank the G ranks are slots on GPUs slot_rank[j]."""
    sr = _c(slot_rank, np.int32) if slot_rank is not None else None
    bo, ro, bn = _c(bnd_old, np.int32), _c(rank_old, np.int32), _c(bnd_new, np.int32)
    b = _c(nbytes, np.int64)
    out = np.full(max(1, len(bn) - 1), -1, np.int32)
    kept = np.zeros(1, np.int64)
    allowed = (1 << G) - 1 if allowed is None else int(allowed)
    st = lib().oracle_map_stages(int(L), len(bo) - 1, _ptr(bo), _ptr(ro), len(bn) - 1, _ptr(bn), _ptr(b),
                                 int(G), allowed & 0xFFFFFFFF, _ptr(sr) if sr is not None else None, _ptr(out),
                                 _ptr(kept))
    return int(st), out[:len(bn) - 1].copy(), int(kept[0])

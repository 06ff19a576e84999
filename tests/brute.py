"""Brute-force enumerators used as PINS for the oracle (tiny inputs only).

These enumerate every contiguous split directly from the problem statement
(min over assignments of the max worker load; contiguous runs for
pipeline stages).  They share nothing with ``oracle/`` (which uses
a DP + suffix table) or with the CUDA path (which uses integer bisection with
a greedy feasibility test): three independent derivations of B*.
"""
from __future__ import annotations

import itertools
from functools import lru_cache

import numpy as np


@lru_cache(maxsize=None)
def _splits(L: int, n: int) -> np.ndarray:
    """All boundary vectors (b_0=0 < b_1 < ... < b_n=L), shape [S, n+1]."""
    inner = list(itertools.combinations(range(1, L), n - 1))
    out = np.zeros((len(inner), n + 1), np.int64)
    if inner:
        out[:, 1:n] = np.array(inner, np.int64).reshape(len(inner), n - 1)
    out[:, n] = L
    return out


def all_splits(L: int, n: int) -> np.ndarray:
    return _splits(L, n)


def partition(cost, n, mem=None, cap=None):
    """Return (B*, lexmax boundaries) or (None, None) when no split is feasible.

    B* = min over all splits with every stage mem <= cap of the max stage cost;
    among the minimisers, the lexicographically largest (b_1..b_{n-1}).
    """
    cost = np.asarray(cost, np.int64)
    L = len(cost)
    if n < 1 or n > L:
        return None, None
    S = _splits(L, n)
    P = np.concatenate([[0], np.cumsum(cost)])
    seg = P[S[:, 1:]] - P[S[:, :-1]]
    mx = seg.max(axis=1)
    ok = np.ones(len(S), bool)
    if mem is not None:
        M = np.concatenate([[0], np.cumsum(np.asarray(mem, np.int64))])
        segm = M[S[:, 1:]] - M[S[:, :-1]]
        ok = (segm <= cap).all(axis=1)
    if not ok.any():
        return None, None
    best = mx[ok].min()
    cand = S[ok & (mx == best)]
    # lexicographic max over rows
    order = np.lexsort(cand[:, ::-1].T)
    return int(best), cand[order[-1]].astype(np.int32)


def n_optima(cost, n) -> int:
    cost = np.asarray(cost, np.int64)
    S = _splits(len(cost), n)
    P = np.concatenate([[0], np.cumsum(cost)])
    mx = (P[S[:, 1:]] - P[S[:, :-1]]).max(axis=1)
    return int((mx == mx.min()).sum())


def repack_min_workers(cost, n_cur, bound, floor=1, mem=None, cap=None):
    """Fewest k in [floor, n_cur] with some contiguous k-split meeting bound and cap."""
    for k in range(floor, n_cur + 1):
        b, _ = partition(cost, k, mem, cap)
        if b is not None and b <= bound:
            return k
    return None

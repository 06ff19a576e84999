"""Host-side pipeline bookkeeping for multi-GPU rebalancing (no compute).

Stage s of an n-stage pipeline lives on GPU floor(s * G / n);
a rank profiles exactly the layers of the stages it owns (8(e)), which are
contiguous because the stage -> rank map is non-decreasing.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def uniform_split(n_layers: int, n_stages: int) -> np.ndarray:
    """Megatron-style even split: b_s = floor(s * L / n)."""
    if not 1 <= n_stages <= n_layers:
        raise ValueError("need 1 <= n_stages <= n_layers")
    return np.array([(s * n_layers) // n_stages for s in range(n_stages + 1)], np.int32)


def stage_ranks(n_stages: int, world: int) -> np.ndarray:
    """Rank owning each stage: floor(s * G / n)."""
    return np.array([(s * world) // n_stages for s in range(n_stages)], np.int32)


def rank_layers(bnd: Sequence[int], ranks: Sequence[int], rank: int) -> tuple[int, int]:
    """(layer_begin, count) of the layers `rank` owns under split `bnd`."""
    bnd = np.asarray(bnd)
    mine = [s for s in range(len(bnd) - 1) if ranks[s] == rank]
    if not mine:
        return int(bnd[0]), 0
    if mine != list(range(mine[0], mine[-1] + 1)):
        raise ValueError("stages of one rank must be contiguous")
    return int(bnd[mine[0]]), int(bnd[mine[-1] + 1] - bnd[mine[0]])

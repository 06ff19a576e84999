"""CPU checks of the C-ABI library: it loads without a GPU and exports every
function include/dynmo.h declares; host-only entry points work."""
import ctypes
import os
import re

import numpy as np

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dynmo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dynmo_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    names = _declared()
    for call in ("dynmo_profile_layers", "dynmo_partition_stages", "dynmo_diffuse_balance",
                 "dynmo_repack_workers", "dynmo_migrate_layers"):
        assert call in names


def test_library_exports_every_declared_symbol():
    from paper_2505_14864_b200 import _lib
    L = _lib.lib()
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(raw, name), name
    assert set(_lib.EXPORTED) == set(_declared())
    assert L.dynmo_version().startswith(b"dynmo-b200")
    assert L.dynmo_strerror(-2) == b"infeasible under the memory cap"


def test_host_argument_validation_without_gpu():
    """Host-checkable errors are returned before any CUDA call."""
    from paper_2505_14864_b200 import _lib
    L = _lib.lib()
    out = ctypes.c_void_p()
    assert L.dynmo_ctx_create(0, 2, 0, None, ctypes.byref(out)) == _lib.E_INVALID  # no NCCL id
    assert L.dynmo_ctx_create(0, 1, 1, None, ctypes.byref(out)) == _lib.E_INVALID  # rank >= nranks
    assert L.dynmo_partition_stages(None, 1, 8, *([None] * 11)) == _lib.E_INVALID
    assert L.dynmo_migrate_plan_set_ctas(None, 16) == _lib.E_INVALID  # null plan
    assert L.dynmo_global_prune(None, None, 1, None, None, None) == _lib.E_INVALID  # null ctx / plan
    # the backward-overlapped migration and the span read: null ctx / plan / outputs
    assert L.dynmo_migrate_bwd_begin(None, None, None) == _lib.E_INVALID
    assert L.dynmo_migrate_layer_ready(None, None, 0, None) == _lib.E_INVALID
    assert L.dynmo_migrate_layers_bwd(None, None, 1, None, None, 1, None, None, None, None) == _lib.E_INVALID
    assert L.dynmo_migrate_bwd_end(None, None, 1, None, None, 1, None, None, None, None) == _lib.E_INVALID
    assert L.dynmo_migrate_bwd_abort(None, None) == _lib.E_INVALID
    assert L.dynmo_ctx_p2p_error_clear(None) == _lib.E_INVALID
    ms, n = ctypes.c_double(), ctypes.c_int64()
    assert L.dynmo_ctx_profile_span(None, ctypes.byref(ms), ctypes.byref(n)) == _lib.E_INVALID
    assert L.dynmo_publish(None, None, None, 4, None) == _lib.E_INVALID
    assert L.dynmo_diag_step_stamps(None, 0) == 0  # a normal build records no stamps


def test_migration_plan_vs_oracle():
    """Host migration plan (product, merge walk) vs oracle O7 (interval search)."""
    from paper_2505_14864_b200 import dynmo as D
    g = np.random.default_rng(5)
    for _ in range(500):
        Ly = int(g.integers(1, 80))
        no, nn = int(g.integers(1, min(8, Ly) + 1)), int(g.integers(1, min(8, Ly) + 1))
        mk = lambda n: (np.concatenate([[0], np.sort(g.choice(np.arange(1, Ly), n - 1, replace=False)), [Ly]])
                        if n > 1 else np.array([0, Ly]))
        bo, bn = mk(no), mk(nn)
        G = int(g.integers(1, 9))
        ro, rn = (np.arange(no) * G) // no, (np.arange(nn) * G) // nn
        assert np.array_equal(D.migration_plan(Ly, bo, ro, bn, rn), oracle.moves(Ly, bo, ro, bn, rn))
    import pytest
    with pytest.raises(D.DynmoError):
        D.migration_plan(4, [0, 2, 2, 4], [0, 0, 1], [0, 4], [0])

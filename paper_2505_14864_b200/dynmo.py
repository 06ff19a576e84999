"""Python binding of the DynMo C-ABI (include/dynmo.h), same call names.

Argument marshalling only: torch tensors -> device pointers + the current
CUDA stream.  Every step of the hot path runs in libdynmo's sm_100a kernels
(and NCCL for the exchange / migration).  PyTorch provides device memory,
streams and the process group that carries the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as _L
from ._lib import lib

__all__ = [
    "DynmoError", "Context", "ProfilePlan", "SegmentSpec", "Batch", "coef_tensor",
    "profile_layers", "partition_stages", "diffuse_balance", "repack_workers",
    "migrate_layers", "migration_plan", "Migrator", "PeerMigrator",
]


class DynmoError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().dynmo_strerror(status).decode()
        detail = lib().dynmo_last_error().decode()
        super().__init__(f"{where}: {msg} ({status}) {detail}")
        self.status = status


def _check(st: int, where: str) -> int:
    if st < 0:
        raise DynmoError(st, where)
    return st


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor expected")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor expected")
    return C.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _i32(a, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=device)


# --------------------------------------------------------------------- ctx
class Context:
    """One per process/GPU.  With a torch process group of world size > 1 the
    NCCL unique id is created on rank 0 and broadcast through that group."""

    def __init__(self, device: int = 0, group=None):
        self.device = int(device)
        rank, nranks = 0, 1
        if group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            import torch.distributed as dist
            if dist.is_initialized():
                rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        self.rank, self.nranks = rank, nranks
        id_buf = None
        if nranks > 1:
            import torch.distributed as dist
            raw = (C.c_uint8 * 128)()
            if rank == 0:
                _check(lib().dynmo_get_unique_id(raw), "dynmo_get_unique_id")
            obj = [bytes(raw)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            raw = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            id_buf = raw
        h = C.c_void_p()
        _check(lib().dynmo_ctx_create(self.device, nranks, rank, id_buf, C.byref(h)), "dynmo_ctx_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    @classmethod
    def _wrap(cls, h, device: int):
        obj = cls.__new__(cls)
        obj.device = device
        obj._h = h
        obj.nranks = int(lib().dynmo_ctx_nranks(h))
        obj.rank = int(lib().dynmo_ctx_rank(h))
        return obj

    def split(self, active: bool, key: Optional[int] = None) -> Optional["Context"]:
        """Release GPUs after re-packing: collective; active
        ranks get a Context over the active group (ordered by key, default
        the old rank), released ranks get None."""
        h = C.c_void_p()
        _check(lib().dynmo_ctx_split(self._h, 0 if active else -1, self.rank if key is None else int(key),
                                     C.byref(h)), "dynmo_ctx_split")
        return Context._wrap(h, self.device) if h.value else None

    def set_timing(self, enable=True, phases=None):
        """enable all phases, or only `phases` (names from _lib.PHASES)."""
        mask = 0
        if phases is not None:
            for p in phases:
                mask |= 1 << _L.PHASES.index(p)
            mask = mask if mask != 1 else 1 | (1 << 31)  # 1 alone means "all" in the C-ABI
        else:
            mask = -1 if enable else 0
        _check(lib().dynmo_ctx_set_timing(self._h, int(mask) if enable else 0), "dynmo_ctx_set_timing")

    def timing_poll(self):
        """Fold the phase events of the last graph replay into the accumulators."""
        _check(lib().dynmo_ctx_timing_poll(self._h), "timing_poll")

    def barrier(self, stream=None):
        """Device-side barrier over the ctx ranks (capturable)."""
        _check(lib().dynmo_ctx_barrier(self._h, _stream(stream)), "dynmo_ctx_barrier")

    def timing_detach(self):
        """Stop polling the timing events of the graphs captured so far."""
        _check(lib().dynmo_ctx_timing_detach(self._h), "timing_detach")

    def timing_read(self) -> dict:
        """{phase: (total_ms, launches)} since the last read (waits on events)."""
        out = {}
        for i, name in enumerate(_L.PHASES):
            ms, cnt = C.c_double(0.0), C.c_int64(0)
            _check(lib().dynmo_ctx_timing_read(self._h, i, C.byref(ms), C.byref(cnt)), "timing_read")
            out[name] = (ms.value, cnt.value)
        return out

    def window_snapshot(self, n_layers: int) -> dict:
        """dynmo_ctx_window_snapshot: this rank's peer-window words (hang
        analysis; completes while the ctx's streams wait)."""
        n = min(int(n_layers), 1024)
        buf = (C.c_uint64 * (21 + 2 * n))()
        _check(lib().dynmo_ctx_window_snapshot(self._h, n, buf, 21 + 2 * n), "dynmo_ctx_window_snapshot")
        v = list(buf)
        return {"err": C.c_int64(v[0]).value, "mig_dev_epoch": v[1], "exch_epoch": v[2], "bwd_done": v[3:19],
                "bwd_finished": v[19:21], "layer_ready": v[21:21 + n],
                "claim": [(x >> 32, x & 0xFFFFFFFF) for x in v[21 + n:21 + 2 * n]]}

    def profile_span(self):
        """(total_ms, launches) of k_profile's own device-clock span since the
        last call (profile-phase timing on); synchronous."""
        ms, cnt = C.c_double(0.0), C.c_int64(0)
        _check(lib().dynmo_ctx_profile_span(self._h, C.byref(ms), C.byref(cnt)), "dynmo_ctx_profile_span")
        return ms.value, cnt.value

    def p2p_error(self) -> int:
        """Sticky device error word of the peer-memory paths (0 = none)."""
        e = C.c_int32(0)
        _check(lib().dynmo_ctx_p2p_error(self._h, C.byref(e)), "dynmo_ctx_p2p_error")
        return int(e.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().dynmo_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- profiling
@dataclass
class SegmentSpec:
    tensor: torch.Tensor        # device tensor holding the segment
    kind: int                   # _lib.SRC_*
    layer: int = 0              # global layer index (ignored for EXIT_U8)
    n_elem: Optional[int] = None  # bits for *_BITS kinds; default = element count
    n_experts: int = 0
    top_k: int = 0


class ProfilePlan:
    """dynmo_profile_plan_create: tile decomposition of this rank's segments."""

    def __init__(self, ctx: Context, segments: Sequence[SegmentSpec], layer_begin: int,
                 n_local: int, n_total: Optional[int] = None, exchange=False):
        """exchange: False/0 local only, True/1 or "p2p" over NVLink peer
        memory (collective creation), 2 or "nccl" via ncclAllGather."""
        n_total = n_local if n_total is None else n_total
        arr = (_L.Segment * max(1, len(segments)))()
        self._keep = []  # keep the tensors alive while the plan exists
        for i, s in enumerate(segments):
            t = s.tensor
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("segments must be contiguous device tensors")
            n = s.n_elem
            if n is None:
                n = t.numel() * (t.element_size() * 8 if s.kind in (_L.SRC_MASK_BITS, _L.SRC_TOKMASK_BITS) else 1)
            arr[i] = _L.Segment(t.data_ptr(), int(n), int(s.layer), int(s.kind), int(s.n_experts), int(s.top_k))
            self._keep.append(t)
        h = C.c_void_p()
        ex = {"p2p": 1, "nccl": 2}.get(exchange, exchange)
        ex = int(ex) if not isinstance(ex, bool) else int(ex)
        _check(lib().dynmo_profile_plan_create(ctx.handle, arr, len(segments), layer_begin, n_local,
                                               n_total, ex, C.byref(h)),
               "dynmo_profile_plan_create")
        self._h = h
        self.ctx = ctx
        self.layer_begin, self.n_local, self.n_total = layer_begin, n_local, n_total
        self.exchange = exchange
        self.max_experts = lib().dynmo_plan_max_experts(h)
        self.n_tiles = lib().dynmo_plan_num_tiles(h)
        self.bytes = lib().dynmo_plan_bytes(h)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().dynmo_profile_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def coef_tensor(n: int, A=0, B=0, C_=0, F=0, ep=0, D=0, device="cuda") -> torch.Tensor:
    """dynmo_cost_coef[n] as an int64 [n, 6] tensor (A, B, C, F, D, ep|pad):
    c_i = frozen ? F : tok (A + B nnz) + C moe + D time."""
    t = torch.zeros((n, 6), dtype=torch.int64)
    for j, v in enumerate((A, B, C_, F, D)):
        t[:, j] = torch.as_tensor(v, dtype=torch.int64)
    t[:, 5] = torch.as_tensor(ep, dtype=torch.int64) & 0xFFFFFFFF  # int32 ep, zero pad
    return t.to(device)


def timestamp(ctx: Context, slot: torch.Tensor, stream=None):
    """dynmo_timestamp: %globaltimer (ns) into the int64 device scalar `slot`
    (e.g. stamps[i]) once the work queued before it on the stream is done."""
    if slot.dtype != torch.int64 or not slot.is_cuda:
        raise ValueError("slot must be an int64 device tensor element")
    _check(lib().dynmo_timestamp(ctx.handle, _ptr(slot), _stream(stream)), "dynmo_timestamp")


PUBLISH_KERNEL_MAX = 4096  # dynmo_publish: larger results go through the copy engine (no kernel)


def publish(ctx: Context, src: torch.Tensor, dst: torch.Tensor, stream=None):
    """dynmo_publish: the device tensor `src` stored by a kernel into the
    pinned host tensor `dst` (same byte size, contiguous): the step's result
    read without a copy-engine D2H node.  Visible on the host once an event
    recorded after it has completed."""
    if not src.is_cuda or dst.is_cuda or not dst.is_pinned():
        raise ValueError("src must be a device tensor and dst a pinned host tensor")
    if not (src.is_contiguous() and dst.is_contiguous()):
        raise ValueError("src and dst must be contiguous")
    nb = src.numel() * src.element_size()
    if nb != dst.numel() * dst.element_size():
        raise ValueError("src and dst differ in size")
    _check(lib().dynmo_publish(ctx.handle, _ptr(src), dst.data_ptr(), nb, _stream(stream)), "dynmo_publish")


def profile_layers(ctx: Context, plan: ProfilePlan, coef: torch.Tensor, *, frozen=None,
                   mem_local=None, counters=None, hist=None, cost=None, mem=None, status=None,
                   stream=None):
    """Call 1.  Returns (cost[n_total], mem[n_total] or None, status[1])."""
    dev = coef.device
    if cost is None:
        cost = torch.empty(plan.n_total, dtype=torch.int64, device=dev)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=dev)
    _check(lib().dynmo_profile_layers(ctx.handle, plan.handle, _ptr(frozen), _ptr(coef), _ptr(mem_local),
                                      _ptr(counters), _ptr(hist), _ptr(cost), _ptr(mem), _ptr(status),
                                      _stream(stream)), "dynmo_profile_layers")
    return cost, mem, status


# ------------------------------------------------------------------ solvers
class Batch:
    """Batched instance layout of calls 2-4 (CSR-style offsets on the device)."""

    def __init__(self, layers: Sequence[int], stages: Sequence[int], device="cuda",
                 capacity: Optional[Sequence[int]] = None):
        layers = np.asarray(layers, np.int64)
        stages = np.asarray(stages, np.int64)
        cap = stages if capacity is None else np.asarray(capacity, np.int64)
        self.n_inst = len(layers)
        self.layers, self.stages = layers, stages
        self.layer_off_h = np.concatenate([[0], np.cumsum(layers)]).astype(np.int32)
        self.bnd_off_h = np.concatenate([[0], np.cumsum(cap + 1)]).astype(np.int32)
        self.layer_off = _i32(self.layer_off_h, device)
        self.bnd_off = _i32(self.bnd_off_h, device)
        self.n_stages = _i32(stages, device)
        self.max_layers = int(layers.max()) if len(layers) else 1
        self.total_bnd = int(self.bnd_off_h[-1])
        self.device = device

    def split(self, flat: torch.Tensor):
        """Per-instance views of a boundary-layout tensor (host numpy)."""
        h = flat.cpu().numpy()
        return [h[self.bnd_off_h[q]:self.bnd_off_h[q + 1]] for q in range(self.n_inst)]


def partition_stages(ctx: Context, batch: Batch, cost: torch.Tensor, *, mem=None, cap=None,
                     bnd=None, bottleneck=None, imbalance=None, status=None, stream=None):
    """Call 2.  Returns (bnd, bottleneck, imbalance, status)."""
    dev = cost.device
    if bnd is None:
        bnd = torch.empty(batch.total_bnd, dtype=torch.int32, device=dev)
    if bottleneck is None:
        bottleneck = torch.empty(batch.n_inst, dtype=torch.int64, device=dev)
    if imbalance is None:
        imbalance = torch.empty(batch.n_inst, dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty(batch.n_inst, dtype=torch.int32, device=dev)
    _check(lib().dynmo_partition_stages(ctx.handle, batch.n_inst, batch.max_layers, _ptr(cost), _ptr(mem),
                                        _ptr(batch.layer_off), _ptr(batch.n_stages), _ptr(cap),
                                        _ptr(batch.bnd_off), _ptr(bnd), _ptr(bottleneck), _ptr(imbalance),
                                        _ptr(status), _stream(stream)), "dynmo_partition_stages")
    return bnd, bottleneck, imbalance, status


def diffuse_balance(ctx: Context, batch: Batch, cost: torch.Tensor, bnd_in: torch.Tensor, *,
                    mem=None, cap=None, gamma=None, gamma_fluid=None, max_rounds: int = 256,
                    fluid: bool = True, out: Optional[dict] = None, stream=None):
    """Call 3.  Returns a dict of output tensors."""
    dev = cost.device
    o = out if out is not None else {}  # filled in place
    o.setdefault("bnd", torch.empty(batch.total_bnd, dtype=torch.int32, device=dev))
    o.setdefault("rounds", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
    o.setdefault("phi", torch.empty(batch.n_inst, dtype=torch.int64, device=dev))
    o.setdefault("phi0", torch.empty(batch.n_inst, dtype=torch.int64, device=dev))
    o.setdefault("status", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
    if fluid:
        o.setdefault("fluid_x", torch.empty(max(1, batch.total_bnd - batch.n_inst), dtype=torch.float64, device=dev))
        o.setdefault("fluid_rounds", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
        o.setdefault("fluid_phi", torch.empty(batch.n_inst, dtype=torch.float64, device=dev))
        o.setdefault("fluid_status", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
    _check(lib().dynmo_diffuse_balance(
        ctx.handle, batch.n_inst, batch.max_layers, _ptr(cost), _ptr(mem), _ptr(batch.layer_off),
        _ptr(batch.n_stages), _ptr(cap), _ptr(batch.bnd_off), _ptr(bnd_in), _ptr(gamma),
        _ptr(gamma_fluid), int(max_rounds), _ptr(o["bnd"]), _ptr(o["rounds"]), _ptr(o["phi"]),
        _ptr(o["phi0"]), _ptr(o.get("fluid_x")), _ptr(o.get("fluid_rounds")), _ptr(o.get("fluid_phi")),
        _ptr(o.get("fluid_status")), _ptr(o["status"]), _stream(stream)), "dynmo_diffuse_balance")
    return o


def repack_workers(ctx: Context, batch: Batch, cost: torch.Tensor, *, floor: torch.Tensor,
                   bound: Optional[torch.Tensor] = None, mode: int = _L.REPACK_BOUND, mem=None,
                   cap=None, bnd_in=None, out: Optional[dict] = None, stream=None):
    """Call 4.  batch.stages = n_cur.  Returns a dict of output tensors."""
    dev = cost.device
    o = out if out is not None else {}  # filled in place
    o.setdefault("n_new", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
    o.setdefault("bnd", torch.empty(batch.total_bnd, dtype=torch.int32, device=dev))
    o.setdefault("bottleneck", torch.empty(batch.n_inst, dtype=torch.int64, device=dev))
    o.setdefault("status", torch.empty(batch.n_inst, dtype=torch.int32, device=dev))
    _check(lib().dynmo_repack_workers(
        ctx.handle, batch.n_inst, batch.max_layers, _ptr(cost), _ptr(mem), _ptr(batch.layer_off),
        _ptr(batch.n_stages), _ptr(cap), _ptr(batch.bnd_off), _ptr(bnd_in), _ptr(bound), _ptr(floor),
        int(mode), _ptr(o["n_new"]), _ptr(o["bnd"]), _ptr(o["bottleneck"]), _ptr(o["status"]),
        _stream(stream)), "dynmo_repack_workers")
    return o


# ---------------------------------------------------------------- migration
def migration_plan(n_layers: int, bnd_old, rank_old, bnd_new, rank_new) -> np.ndarray:
    """Host-only: moves (layer, src_rank, dst_rank) of call 5."""
    bo, ro = np.ascontiguousarray(bnd_old, np.int32), np.ascontiguousarray(rank_old, np.int32)
    bn, rn = np.ascontiguousarray(bnd_new, np.int32), np.ascontiguousarray(rank_new, np.int32)
    out = np.zeros((max(1, n_layers), 3), np.int32)
    m = lib().dynmo_migration_plan(int(n_layers), len(bo) - 1, bo.ctypes.data, ro.ctypes.data,
                                   len(bn) - 1, bn.ctypes.data, rn.ctypes.data, out.ctypes.data)
    if m < 0:
        raise DynmoError(m, "dynmo_migration_plan")
    return out[:m].copy()


def migrate_layers(ctx: Context, n_layers: int, bnd_old, rank_old, bnd_new, rank_new,
                   send: dict, recv: dict, n_bufs: int = 1, stream=None):
    """Call 5 (collective).  send/recv map layer -> list of device tensors
    (this rank's old / new layers).  Returns (bytes_sent, bytes_recv)."""
    bo, ro = np.ascontiguousarray(bnd_old, np.int32), np.ascontiguousarray(rank_old, np.int32)
    bn, rn = np.ascontiguousarray(bnd_new, np.int32), np.ascontiguousarray(rank_new, np.int32)
    tab_s = (_L.Buf * max(1, n_layers * n_bufs))()
    tab_r = (_L.Buf * max(1, n_layers * n_bufs))()
    for tab, d in ((tab_s, send), (tab_r, recv)):
        for layer, bufs in d.items():
            for k, t in enumerate(bufs):
                tab[layer * n_bufs + k] = _L.Buf(t.data_ptr(), t.numel() * t.element_size())
    sent, rec = C.c_int64(0), C.c_int64(0)
    _check(lib().dynmo_migrate_layers(ctx.handle, int(n_layers), len(bo) - 1, bo.ctypes.data,
                                      ro.ctypes.data, len(bn) - 1, bn.ctypes.data, rn.ctypes.data,
                                      tab_s, tab_r, int(n_bufs), C.byref(sent), C.byref(rec),
                                      _stream(stream)), "dynmo_migrate_layers")
    return sent.value, rec.value


class Migrator:
    """Call 5 with the buffer tables built once (per-step cost: one C call).
    send/recv map layer -> list of device tensors, as for migrate_layers."""

    def __init__(self, ctx: Context, n_layers: int, send: dict, recv: dict, n_bufs: int = 1):
        self.ctx, self.n_layers, self.n_bufs = ctx, int(n_layers), int(n_bufs)
        self._tab_s = (_L.Buf * max(1, n_layers * n_bufs))()
        self._tab_r = (_L.Buf * max(1, n_layers * n_bufs))()
        self._keep = []
        for tab, d in ((self._tab_s, send), (self._tab_r, recv)):
            for layer, bufs in d.items():
                for k, t in enumerate(bufs):
                    tab[layer * n_bufs + k] = _L.Buf(t.data_ptr(), t.numel() * t.element_size())
                    self._keep.append(t)
        self._sent, self._rec = C.c_int64(0), C.c_int64(0)

    def __call__(self, bnd_old, rank_old, bnd_new, rank_new, stream=None):
        bo, ro = np.ascontiguousarray(bnd_old, np.int32), np.ascontiguousarray(rank_old, np.int32)
        bn, rn = np.ascontiguousarray(bnd_new, np.int32), np.ascontiguousarray(rank_new, np.int32)
        _check(lib().dynmo_migrate_layers(self.ctx.handle, self.n_layers, len(bo) - 1, bo.ctypes.data,
                                          ro.ctypes.data, len(bn) - 1, bn.ctypes.data, rn.ctypes.data,
                                          self._tab_s, self._tab_r, self.n_bufs, C.byref(self._sent),
                                          C.byref(self._rec), _stream(stream)), "dynmo_migrate_layers")
        return self._sent.value, self._rec.value


class PeerMigrator:
    """Call 5 over NVLink peer memory (dynmo_migrate_plan_create +
    dynmo_migrate_layers_p2p).  Collective construction: every rank passes the
    buffers it may send (layers it owns) and may receive into."""

    def __init__(self, ctx: Context, n_layers: int, send: dict, recv: dict, n_bufs: int = 1):
        self.ctx, self.n_layers, self.n_bufs = ctx, int(n_layers), int(n_bufs)
        tab_s = (_L.Buf * max(1, n_layers * n_bufs))()
        tab_r = (_L.Buf * max(1, n_layers * n_bufs))()
        self._keep = []
        for tab, d in ((tab_s, send), (tab_r, recv)):
            for layer, bufs in d.items():
                for k, t in enumerate(bufs):
                    tab[layer * n_bufs + k] = _L.Buf(t.data_ptr(), t.numel() * t.element_size())
                    self._keep.append(t)
        h = C.c_void_p()
        _check(lib().dynmo_migrate_plan_create(ctx.handle, self.n_layers, self.n_bufs, tab_s, tab_r,
                                               C.byref(h)), "dynmo_migrate_plan_create")
        self._h = h
        self._sent, self._rec = C.c_int64(0), C.c_int64(0)

    def __call__(self, bnd_old, rank_old, bnd_new, rank_new, stream=None):
        bo, ro = np.ascontiguousarray(bnd_old, np.int32), np.ascontiguousarray(rank_old, np.int32)
        bn, rn = np.ascontiguousarray(bnd_new, np.int32), np.ascontiguousarray(rank_new, np.int32)
        _check(lib().dynmo_migrate_layers_p2p(self.ctx.handle, self._h, len(bo) - 1, bo.ctypes.data,
                                              ro.ctypes.data, len(bn) - 1, bn.ctypes.data, rn.ctypes.data,
                                              C.byref(self._sent), C.byref(self._rec), _stream(stream)),
               "dynmo_migrate_layers_p2p")
        return self._sent.value, self._rec.value

    def device(self, bnd_old: torch.Tensor, rank_old: torch.Tensor, bnd_new: torch.Tensor,
               rank_new: torch.Tensor, bytes_sent=None, bytes_recv=None, stream=None):
        """dynmo_migrate_layers_dev: int32 device boundaries / stage->rank maps,
        no host round trip (capturable in a CUDA graph)."""
        _check(lib().dynmo_migrate_layers_dev(self.ctx.handle, self._h, rank_old.numel(), _ptr(bnd_old),
                                              _ptr(rank_old), rank_new.numel(), _ptr(bnd_new), _ptr(rank_new),
                                              _ptr(bytes_sent), _ptr(bytes_recv), _stream(stream)),
               "dynmo_migrate_layers_dev")

    # NEXT-3: migration overlapped with the backward pass
    def bwd_begin(self, stream=None):
        """dynmo_migrate_bwd_begin: once per iteration on every rank, before
        the other backward-migration calls (host-side epoch)."""
        _check(lib().dynmo_migrate_bwd_begin(self.ctx.handle, self._h, _stream(stream)), "dynmo_migrate_bwd_begin")

    def layer_ready(self, layer: int, stream=None):
        """dynmo_migrate_layer_ready: layer's buffers (its gradients) are
        written on `stream`; released to every rank."""
        _check(lib().dynmo_migrate_layer_ready(self.ctx.handle, self._h, int(layer), _stream(stream)),
               "dynmo_migrate_layer_ready")

    def backward(self, bnd_old: torch.Tensor, rank_old: torch.Tensor, bnd_new: torch.Tensor,
                 rank_new: torch.Tensor, bytes_recv=None, stream=None):
        """dynmo_migrate_layers_bwd: per layer, last to first, a stream wait
        for its release and a pull if it moves here (needs set_ctas(c),
        0 < c < SMs)."""
        _check(lib().dynmo_migrate_layers_bwd(self.ctx.handle, self._h, rank_old.numel(), _ptr(bnd_old),
                                              _ptr(rank_old), rank_new.numel(), _ptr(bnd_new), _ptr(rank_new),
                                              _ptr(bytes_recv), _stream(stream)),
               "dynmo_migrate_layers_bwd")

    def bwd_end(self, bnd_old: torch.Tensor, rank_old: torch.Tensor, bnd_new: torch.Tensor,
                rank_new: torch.Tensor, bytes_sent=None, stream=None):
        """dynmo_migrate_bwd_end: stream waits until every rank has pulled;
        the sent buffers may be reused after it on `stream`."""
        _check(lib().dynmo_migrate_bwd_end(self.ctx.handle, self._h, rank_old.numel(), _ptr(bnd_old),
                                           _ptr(rank_old), rank_new.numel(), _ptr(bnd_new), _ptr(rank_new),
                                           _ptr(bytes_sent), _stream(stream)),
               "dynmo_migrate_bwd_end")

    def clear_error(self):
        """dynmo_ctx_p2p_error_clear: reset the sticky error word (synchronous)."""
        _check(lib().dynmo_ctx_p2p_error_clear(self.ctx.handle), "dynmo_ctx_p2p_error_clear")

    def bwd_abort(self):
        """dynmo_migrate_bwd_abort: release this rank's waits of the current
        iteration and set the sticky error (host watchdog escape hatch)."""
        _check(lib().dynmo_migrate_bwd_abort(self.ctx.handle, self._h), "dynmo_migrate_bwd_abort")

    def set_ctas(self, max_ctas: int):
        """dynmo_migrate_plan_set_ctas: SM budget of the device-driven pull
        (0 = every SM), for a migration overlapped with compute."""
        _check(lib().dynmo_migrate_plan_set_ctas(self._h, int(max_ctas)), "dynmo_migrate_plan_set_ctas")

    def error(self) -> int:
        e = C.c_int32(0)
        _check(lib().dynmo_ctx_p2p_error(self.ctx.handle, C.byref(e)), "dynmo_ctx_p2p_error")
        return e.value

    def close(self):
        if getattr(self, "_h", None):
            lib().dynmo_migrate_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------- global pruning (NEXT-2)
class PrunePlan:
    """dynmo_prune_plan_create over this rank's (weights, mask) pairs, in the
    global order of Alg. 1 (rank order, then this list's order)."""

    def __init__(self, ctx: Context, pairs: Sequence[tuple]):
        arr = (_L.PruneSegment * max(1, len(pairs)))()
        self._keep = []
        for i, (w, m) in enumerate(pairs):
            if not (w.is_cuda and m.is_cuda and w.is_contiguous() and m.is_contiguous()):
                raise ValueError("weights and masks must be contiguous device tensors")
            if w.dtype not in (torch.float32, torch.bfloat16) or m.dtype != torch.uint8 or m.numel() != w.numel():
                raise ValueError("weights f32/bf16, masks uint8 of the same length")
            dt = _L.W_F32 if w.dtype == torch.float32 else _L.W_BF16
            arr[i] = _L.PruneSegment(w.data_ptr(), m.data_ptr(), w.numel(), dt, 0)
            self._keep += [w, m]
        h = C.c_void_p()
        _check(lib().dynmo_prune_plan_create(ctx.handle, arr, len(pairs), C.byref(h)), "dynmo_prune_plan_create")
        self.handle = h
        self.ctx = ctx

    def close(self):
        if getattr(self, "handle", None):
            lib().dynmo_prune_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def global_prune(ctx: Context, plan: PrunePlan, k: int, info=None, status=None, stream=None):
    """Alg. 1 (collective): masks of the k globally largest |w|.  Returns
    (info[6] int64, status[1] int32) device tensors."""
    dev = torch.device("cuda", ctx.device)
    if info is None:
        info = torch.empty(6, dtype=torch.int64, device=dev)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=dev)
    _check(lib().dynmo_global_prune(ctx.handle, plan.handle, int(k), _ptr(info), _ptr(status), _stream(stream)),
           "dynmo_global_prune")
    return info, status


# ----------------------------------------- stage -> rank map (NEXT-3)
def map_stages(ctx: Context, n_layers: int, bnd_old: torch.Tensor, rank_old: torch.Tensor, bnd_new: torch.Tensor,
               nbytes: torch.Tensor, G: int, allowed: Optional[int] = None, slot_rank=None, rank_new=None, kept=None,
               status=None, stream=None):
    """dynmo_map_stages: migration-minimising distinct ranks (or slots, with
    slot_rank[G] mapping slots to GPUs for the output) for the new stages.
    Returns (rank_new[n_new], kept[1], status[1]) device tensors."""
    dev = bnd_new.device
    n_new = bnd_new.numel() - 1
    if rank_new is None:
        rank_new = torch.empty(n_new, dtype=torch.int32, device=dev)
    if kept is None:
        kept = torch.empty(1, dtype=torch.int64, device=dev)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=dev)
    allowed = (1 << G) - 1 if allowed is None else int(allowed)
    _check(lib().dynmo_map_stages(ctx.handle, int(n_layers), bnd_old.numel() - 1, _ptr(bnd_old), _ptr(rank_old),
                                  n_new, _ptr(bnd_new), _ptr(nbytes), int(G), allowed & 0xFFFFFFFF, _ptr(slot_rank),
                                  _ptr(rank_new), _ptr(kept), _ptr(status), _stream(stream)), "dynmo_map_stages")
    return rank_new, kept, status

#!/usr/bin/env python
"""Benchmark of the DynMo per-step rebalancing hot path on B200.

Default workload (BASELINE.json configs[1]): GPT-48 gradual global magnitude
pruning at S = 0.9, 8 pipeline stages, stage s on GPU floor(s*G/8).  One step =
  profile_layers   (this GPU's layers' sources -> int64 costs, + the exchange
                    of the cost slots over NVLink peer memory when G > 1)
  partition_stages (centralised min-max split, memory capped)
  diffuse_balance  (decentralised diffusion + fluid process, from the
                    current split)
  repack_workers   (fewest GPUs within the dense pipeline's bottleneck)
  migrate_layers   (the payload of every layer whose GPU changes, pulled over
                    NVLink peer memory; device-driven, in the step's graph)
The step replays the same rebalance event (uniform split -> balanced split)
every iteration; inputs stay resident in HBM; L2 is flushed between steps.

--config selects the other BASELINE workloads with the same JSON schema:
  3  GPT-32 freezing + early exit (per-layer token bitmasks, 512 x 2048
     tokens, frozen prefix), dense-layer payload (bf16 + fp32 optimizer state)
  4  Mixtral-8x7B-shaped MoE routing (int64 top-2 ids, E = 8, EP = 8) with
     popularity drifting by depth, 2.90 GB bf16 payload per migrated layer
  5  batched sweep: 4096 instances (48-128 layers, 2-8 stages, MoD token
     bitmasks) -> partition + repack to the fewest workers; instances are
     sharded 4096/G per GPU, no exchange, no migration

  python bench.py [--config {2,3,4,5}] [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun (N > 1) one rank per GPU; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 prints exactly one JSON line on stdout: NCCL_DEBUG=VERSION (set in
# this image) prints NCCL's version banner there with printf, so it is
# dropped; an explicit INFO/WARN/TRACE level is kept, its log sent to stderr
if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
    del os.environ["NCCL_DEBUG"]
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

import synth  # noqa: E402

METRIC = "rebalance ms/step (profile+partition+migrate) at 1/2/4/8 B200; profile HBM GB/s"
L2_FLUSH_BYTES = 256 << 20
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE.json workload (configs[1..4]); 2 = the headline")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="dynmo", choices=["dynmo", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="cost exchange over NVLink peer memory (default) or ncclAllGather")
    ap.add_argument("--migrate", choices=["p2p", "nccl"], default="p2p",
                    help="layer migration over NVLink peer memory (default) or NCCL send/recv")
    ap.add_argument("--map-stages", action="store_true",
                    help="NEXT-3: place the new stages on the GPU slots that keep the most payload in place "
                         "(dynmo_map_stages inside the step) instead of stage s on GPU floor(s*G/n)")
    ap.add_argument("--host-migrate", action="store_true",
                    help="host-driven migration (D2H of the boundaries, then the migrate call) "
                         "instead of the device-driven call inside the step's graph")
    ap.add_argument("--result-read", choices=["publish", "copy"], default="publish",
                    help="the step's result (new boundaries + statuses) to the host: stored by a kernel "
                         "into mapped pinned memory (dynmo_publish, default) or a D2H copy node")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch every call eagerly instead of replaying a CUDA graph")
    ap.add_argument("--ref-budget", type=float, default=120.0,
                    help="--impl reference: seconds of oracle work for the whole --warmup + --steps run")
    ap.add_argument("--cfg4-routing", choices=["drift", "aux", "sbase"], default="drift",
                    help="config 4 popularity: Dirichlet alpha drifting 64 -> 0.3 with depth (default), "
                         "alpha = 4 (aux-loss) or 64 (S-BASE) on every layer")
    return ap.parse_args(argv)


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def uniform_split(L, n):
    """Megatron-style even split b_s = floor(s L / n) (bookkeeping, inline so
    the oracle arm does not import the product package)."""
    return np.array([(s * L) // n for s in range(n + 1)], np.int32)


def stage_ranks(n, G):
    """Stage s on GPU floor(s G / n)."""
    return np.array([(s * G) // n for s in range(n)], np.int32)


def rank_layers(bnd, ranks, rank):
    mine = [s for s in range(len(bnd) - 1) if ranks[s] == rank]
    if not mine:
        return int(bnd[0]), 0
    return int(bnd[mine[0]]), int(bnd[mine[-1] + 1] - bnd[mine[0]])


class L2Flush:
    """Evicts the step's data from L2 between timed steps: a write larger
    than L2, then a read larger than L2 (the write's dirty lines are written
    back here, outside the timed interval, instead of inside the next step)."""

    def __init__(self, dev):
        import torch
        self.w = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(L2_FLUSH_BYTES // 8, dtype=torch.int64, device=dev)
        self.k = 0

    def __call__(self):
        self.k += 1
        self.w.fill_(self.k & 0xFF)
        self.r.max()


L2_NOTE = (f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write, then a {L2_FLUSH_BYTES >> 20} MiB "
           "read so no dirty lines of the flush are written back inside the step)")


# --------------------------------------------------------------- workloads
# A workload holds the host side of one BASELINE config for the layers of one
# rank: seeded synthetic sources (synth/), the cost coefficients, the
# per-layer payload (migration bytes = the solver's memory), the cap, the
# repack bound.  Sources are (kind, layer, np array, n_elem, n_experts).
SRC_MASK_U8, SRC_TOKMASK_BITS, SRC_EXPERT_I64 = 1, 4, 6  # include/dynmo.h dynmo_src_kind


class Cfg2:
    """GPT-48 gradual global magnitude pruning."""
    key, L, n = 2, 48, 8
    SPARSITY, MILESTONE = 0.9, 4

    def __init__(self, args=None):
        self.shape = synth.GPTShape()
        self.p = synth.cfg2_keep_probs(self.shape, self.SPARSITY, self.MILESTONE)
        self.payload = synth.cfg2_payload_bytes(self.shape, self.p)  # caller-side CSR bytes
        self.cap = int(1.5 * int(self.payload.sum()) / self.n)      # per-GPU memory budget
        self.bound = (self.L // self.n) * self.shape.params_per_layer  # dense B*
        self.gamma_fluid = 1.0
        self.coef = dict(A=0, B=1)
        self.frozen = None

    def config(self, G):
        return {"workload": "config2: GPT-48 gradual global magnitude pruning, S=0.9, 8 pipeline stages, "
                            "u8 masks (the exact global top-k of the synthetic bf16 weights), rebalance from "
                            "the uniform split",
                "layers": self.L, "hidden": self.shape.h, "stages": self.n,
                "params_per_layer": self.shape.params_per_layer,
                "mask_bytes_total": self.L * self.shape.params_per_layer, "mask_repr": "u8",
                "stage_to_gpu": "floor(s*G/8)", "l2": L2_NOTE, "parallelism": f"pp-profile{G}"}

    def sources(self, begin, count):
        for layer in range(begin, begin + count):
            for m in synth.cfg2_layer_masks_u8(self.shape, layer, self.p[layer], self.MILESTONE):
                yield (SRC_MASK_U8, layer, m.reshape(-1), None, 0)

    def oracle_cost(self, src_list, layer_subset=None):
        import oracle
        nnz = np.zeros(self.L, np.int64)
        for kind, layer, a, ne, E in src_list:
            if layer_subset is None or layer in layer_subset:
                nnz[layer] += oracle.count_nz_u8(a)
        return np.array([oracle.layer_cost(nnz=int(v), **self.coef)[1] for v in nnz], np.int64)


class Cfg3:
    """GPT-32 layer freezing + early exit."""
    key, L, n = 3, 32, 8
    T, F, H = 512 * 2048, 8, 1024

    def __init__(self, args=None):
        self.e = synth.cfg3_exit_depth(T=self.T, L=self.L)
        self.f = synth.cfg3_frozen(self.L, self.F)
        P = 12 * self.H * self.H
        # payload (reading Q19): bf16 weights, + fp32 master / m / v unless frozen
        self.payload = np.array([P * (2 if self.f[i] else 14) for i in range(self.L)], np.int64)
        self.cap = int(1.5 * int(self.payload.sum()) / self.n)
        self.bound = (self.L // self.n) * self.T  # dense bottleneck: every token through L/n layers
        self.gamma_fluid = 1.0
        self.coef = dict(A=1, B=0)
        self.frozen = self.f

    def config(self, G):
        return {"workload": f"config3: GPT-32 layer freezing (layers < {self.F} frozen) + early exit "
                            "(no exit before layer 8, then 8%/layer), 512x2048 tokens, per-layer token "
                            "bitmasks, 8 stages, rebalance from the uniform split",
                "layers": self.L, "stages": self.n, "tokens": self.T, "frozen_prefix": self.F,
                "mask_bytes_total": self.L * self.T // 8, "mask_repr": "token bitmasks (uint32)",
                "stage_to_gpu": "floor(s*G/8)", "l2": L2_NOTE, "parallelism": f"pp-profile{G}"}

    def sources(self, begin, count):
        for layer in range(begin, begin + count):
            yield (SRC_TOKMASK_BITS, layer, synth.pack_bits((self.e > layer).astype(np.uint8)), self.T, 0)

    def oracle_cost(self, src_list, layer_subset=None):
        import oracle
        tok = np.zeros(self.L, np.int64)
        for kind, layer, a, ne, E in src_list:
            if layer_subset is None or layer in layer_subset:
                tok[layer] += oracle.count_bits(a, ne)
        return np.array([oracle.layer_cost(frozen=bool(self.f[i]), tok=int(tok[i]), **self.coef)[1]
                         for i in range(self.L)], np.int64)


class Cfg4:
    """Mixtral-8x7B-shaped MoE routing."""
    key, L, n = 4, 32, 8
    T, E, K, EP = 64 * 2048, 8, 2, 8

    def __init__(self, args=None):
        self.routing = getattr(args, "cfg4_routing", "drift") if args is not None else "drift"
        self.payload = np.full(self.L, synth.MIXTRAL_LAYER_PARAMS * 2, np.int64)  # bf16 layer
        self.cap = int(1.5 * int(self.payload.sum()) / self.n)
        self.coef = dict(A=self.T, C_=4, ep=self.EP)
        balanced = self.T + 4 * self.T * self.K  # c = T + 4 moe with moe = T k when balanced
        self.bound = (self.L // self.n) * balanced
        self.gamma_fluid = 1.0
        self.frozen = None

    def config(self, G):
        desc = {"drift": "Dirichlet alpha drifting 64 -> 0.3 with depth", "aux": "Dirichlet alpha 4 (aux-loss)",
                "sbase": "Dirichlet alpha 64 (S-BASE)"}[self.routing]
        return {"workload": f"config4: Mixtral-8x7B-shaped MoE routing, 32 layers, E=8, top-2, 64x2048 tokens, "
                            f"EP=8, {desc}; 2.90 GB bf16 payload per migrated layer, rebalance from the "
                            "uniform split",
                "layers": self.L, "stages": self.n, "tokens": self.T, "experts": self.E, "top_k": self.K,
                "routing": self.routing, "id_bytes_total": self.L * self.T * self.K * 8,
                "payload_bytes_per_layer": int(self.payload[0]),
                "stage_to_gpu": "floor(s*G/8)", "l2": L2_NOTE, "parallelism": f"pp-profile{G}"}

    def ids(self, layer):
        if self.routing == "drift":
            return synth.cfg4_routing_drift(layer, self.L, T=self.T, E=self.E, k=self.K)
        return synth.cfg4_routing(layer, T=self.T, E=self.E, k=self.K, alpha=4.0 if self.routing == "aux" else 64.0)

    def sources(self, begin, count):
        for layer in range(begin, begin + count):
            yield (SRC_EXPERT_I64, layer, self.ids(layer).reshape(-1), None, self.E)

    def oracle_cost(self, src_list, layer_subset=None):
        import oracle
        cost = np.zeros(self.L, np.int64)
        for kind, layer, a, ne, E in src_list:
            if layer_subset is None or layer in layer_subset:
                st, h = oracle.expert_hist(a, E)
                cost[layer] = oracle.layer_cost(cnt=h, **self.coef)[1]
        return cost


class Cfg5:
    """Batched sweep: 4096 independent instances."""
    key, N_INST, T = 5, 4096, 4096

    def __init__(self, args=None):
        self.insts = None

    def config(self, G):
        return {"workload": "config5: batched rebalance sweep, 4096 instances of 48-128 layers x 2-8 stages, "
                            "MoD token bitmasks (T=4096, every other layer routed at 12.5% x U(0.5,1.5)), "
                            "memory-capped partition + BOUND repack to the fewest workers",
                "instances": self.N_INST, "instances_per_gpu": self.N_INST // G, "tokens": self.T,
                "mask_repr": "token bitmasks (uint32), back to back per instance",
                "sharding": "instances [r*4096/G, (r+1)*4096/G) on rank r, no exchange, no migration",
                "l2": L2_NOTE, "parallelism": f"dp{G}"}

    def shard(self, rank, G):
        q0, q1 = rank * self.N_INST // G, (rank + 1) * self.N_INST // G
        return [synth.cfg5_instance(i) for i in range(q0, q1)]


WORKLOADS = {2: Cfg2, 3: Cfg3, 4: Cfg4, 5: Cfg5}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + clock-event reasons during the timed region with an
    `nvidia-smi -lms` subprocess (no GIL contention with the timed loop)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, torch_dev):
        import torch
        self.dev_id = None
        try:
            u = str(torch.cuda.get_device_properties(torch_dev).uuid)
            self.dev_id = u if u.startswith("GPU-") else "GPU-" + u
        except Exception:
            self.dev_id = str(torch_dev)
        self.proc, self.out = None, ""

    def __enter__(self):
        import subprocess
        if os.environ.get("DYNMO_BENCH_NO_CLOCKS") == "1":  # diagnosis only: no sampler
            self.err = "disabled (DYNMO_BENCH_NO_CLOCKS=1)"
            self.lines, self.t0, self.t1 = [], None, None
            return self
        import threading
        self.lines, self.t0, self.t1 = [], None, None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.dev_id, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def reader():  # timestamps each sample (host monotonic clock)
                for line in self.proc.stdout:
                    self.lines.append((time.monotonic(), line))
            self.th = threading.Thread(target=reader, daemon=True)
            self.th.start()
            deadline = time.monotonic() + 10.0  # the sampler is running before the timed loop
            while not self.lines and time.monotonic() < deadline:
                time.sleep(0.005)
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def start(self):
        """Marks the start of the timed region (samples before it are dropped)."""
        self.t0 = time.monotonic()

    def stop(self):
        """Marks the end of the timed region."""
        self.t1 = time.monotonic()

    def __exit__(self, *a):
        if not hasattr(self, "th"):
            self.out = ""
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.th.join(timeout=5)
        t0, t1 = self.t0 or 0.0, self.t1 or float("inf")
        self.out = "".join(line for t, line in self.lines if t0 <= t <= t1 + 0.025)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no nvidia-smi samples")}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------- oracle (CPU) arm
def oracle_solvers(wl, cost):
    """Every solver of the step on the oracle (as it stands)."""
    import oracle
    b_old = uniform_split(wl.L, wl.n)
    mem = wl.payload
    st, b, B, imb = oracle.partition(cost, wl.n, mem=mem, cap=wl.cap)
    oracle.diffuse(cost, b_old, 0, 256, mem=mem, cap=wl.cap)
    oracle.diffuse_fluid(cost, b_old, wl.gamma_fluid, 256)
    oracle.repack_bound(cost, wl.n, wl.bound, 1, mem=mem, cap=wl.cap)
    r = stage_ranks(wl.n, 1)
    oracle.moves(wl.L, b_old, r, b, r)
    return b


def oracle_step(wl, srcs, layer_subset=None):
    """The oracle as it stands: counts, costs, every solver, the migration
    plan.  Returns (seconds counting, seconds solving)."""
    t0 = time.perf_counter()
    cost = wl.oracle_cost(srcs, layer_subset)
    t1 = time.perf_counter()
    oracle_solvers(wl, cost)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def oracle_batch_step(insts):
    """Config 5 on the oracle: token counts, costs, memory-capped partition
    and BOUND repack of every instance.  Returns seconds."""
    import oracle
    t0 = time.perf_counter()
    for x in insts:
        tok = [oracle.count_bits(x.masks[l], x.masks.shape[1] * 32) for l in range(x.L)]
        cost = np.array([oracle.layer_cost(tok=int(v), A=1)[1] for v in tok], np.int64)
        oracle.partition(cost, x.n, mem=x.mem, cap=x.cap)
        oracle.repack_bound(cost, x.n, x.bound, 1, mem=x.mem, cap=x.cap)
    return time.perf_counter() - t0


def cpu_threads_used():
    return 1  # the oracle is single-threaded C


def cpu_baseline(wl, args, srcs=None):
    """The oracle timed on this host for about args.cpu_seconds (bounded
    sample of the same workload, scaled to one whole step)."""
    if wl.key == 5:
        insts = wl.shard(0, 1)[:64]
        ts = []
        t_end = time.perf_counter() + args.cpu_seconds
        while time.perf_counter() < t_end or not ts:
            ts.append(oracle_batch_step(insts) * wl.N_INST / len(insts))
        return {"value": round(1e3 * float(np.mean(ts)), 3), "unit": "ms", "cores": cpu_threads_used(),
                "kind": "oracle", "sample": f"{len(ts)} passes over 64 of the 4096 instances (counts, costs, "
                                            f"partition, repack), scaled x64 to the whole batch; 1 thread; "
                                            f"host has {os.cpu_count()} cores"}
    c_s, s_s = [], []
    t_end = time.perf_counter() + args.cpu_seconds
    while time.perf_counter() < t_end or len(c_s) < 2:
        c, s_ = oracle_step(wl, srcs)
        c_s.append(c)
        s_s.append(s_)
    ob = 1e3 * (np.mean(c_s) + np.mean(s_s))
    return {"value": round(float(ob), 3), "unit": "ms", "cores": cpu_threads_used(), "kind": "oracle",
            "sample": f"{len(c_s)} full config-{wl.key} oracle steps (all {wl.L} layers' sources, every solver), "
                      f"1 thread; host has {os.cpu_count()} cores"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = WORKLOADS[args.config](args)
    budget = args.ref_budget  # seconds for the whole --warmup + --steps run
    nsteps = args.steps + args.warmup
    times = []
    if wl.key == 5:
        insts = wl.shard(0, 1)
        t1 = oracle_batch_step(insts[:16]) / 16
        m = int(max(1, min(len(insts), budget / nsteps / max(t1, 1e-9))))
        for it in range(nsteps):
            sub = [insts[(it * m + k) % len(insts)] for k in range(m)]
            t = oracle_batch_step(sub) * len(insts) / m
            if it >= args.warmup:
                times.append(t)
        sample = (f"each step: the oracle on {m} of the 4096 instances (rotating), scaled x{4096 / m:.1f} "
                  "to the whole batch")
    else:
        srcs = list(wl.sources(0, wl.L))
        L = wl.L
        c_full, s_full = oracle_step(wl, srcs)
        m = L
        if nsteps * (c_full + s_full) > budget:
            m = max(1, min(L, int(L * (budget / nsteps - s_full) / max(c_full, 1e-9))))
        for it in range(nsteps):
            sub = set(((it * m) + k) % L for k in range(m))
            c, s_ = oracle_step(wl, srcs, sub if m < L else None)
            if it >= args.warmup:
                times.append(c * (L / m) + s_)
        sample = (f"each step: oracle counts of {m} of {L} layers' sources (rotating; count time scaled by "
                  f"{L}/{m}) + every solver on the full {L}-layer cost vector"
                  if m < L else f"each step: the full config-{wl.key} oracle step (all {L} layers)")
    ms = 1e3 * float(np.mean(times))
    out = {"impl": "reference", "metric": METRIC, "value": round(ms, 4), "unit": "ms",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": False, "scaling": "weak" if wl.key == 5 else "strong", "vs_baseline": None,
           "dtype": "int64", "data": "synthetic", "config": wl.config(args.gpus),
           "cpu_baseline": {"value": round(ms, 4), "unit": "ms", "cores": cpu_threads_used(),
                            "kind": "oracle", "sample": sample},
           "e2e": {"value": round(ms, 4), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
class StepTimer:
    """One-graph steps: [device barrier (the step runs at the
    training-iteration barrier) -> start event -> step -> end event], C graph
    copies with their own events replayed back to back; the host reads the
    events once per group.  The timed interval begins once EVERY rank's graph
    is running, so a host hiccup on one rank delays only the untimed barrier."""

    def __init__(self, ctx, dev, steps):
        self.ctx, self.dev = ctx, dev
        self.C = 4 if steps % 4 == 0 else (2 if steps % 2 == 0 else 1)
        self.copies, self.ev = [], []

    def capture(self, body):
        import torch
        for _ in range(self.C):
            e0 = torch.cuda.Event(enable_timing=True, external=True)
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.Stream(device=self.dev)):
                self.ctx.barrier()
                e0.record()
                body()
                e1.record()
            self.copies.append(g)
            self.ev.append((e0, e1))

    def replay(self, k):
        self.copies[k % len(self.copies)].replay()

    def run(self, steps, flush, after_group=None):
        out = []
        for k in range(steps):
            flush()  # L2 flush between steps (outside the timed interval)
            self.replay(k)
            if (k + 1) % self.C == 0:  # read this group's per-step device intervals
                self.ev[-1][1].synchronize()
                out += [a.elapsed_time(b) for a, b in self.ev]
                if after_group:
                    after_group()
        return out


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev


def reduce_max(vals, dev, G, op="max"):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return t.tolist()


def gather_list(v, dev, G):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    if G == 1:
        return [float(v)]
    out = [torch.zeros_like(t) for _ in range(G)]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def step_stats(step_ms):
    med = float(np.median(step_ms))
    return {"median": round(med, 5), "p95": round(float(np.percentile(step_ms, 95)), 5),
            "max": round(float(step_ms.max()), 5), "n_over_2x_median": int((step_ms > 2 * med).sum()),
            "outliers": [[int(k), round(float(step_ms[k]), 4)] for k in np.flatnonzero(step_ms > 2 * med)[:8]]}


def roofline(plan_bytes, prof_avg_ms, per_rank_frac, G, cfg, span_ms=0.0):
    peaks, peak_src = load_peaks()
    achieved = plan_bytes / (prof_avg_ms * 1e-3) / 1e9 if prof_avg_ms > 0 else 0.0
    span_gbs = plan_bytes / (span_ms * 1e-3) / 1e9 if span_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_k_profile.json")
    if os.path.exists(tp):
        try:
            # one ncu --set full capture per workload (single process: G=1 only)
            traffic = json.load(open(tp)).get("cfg%d_dram_bytes_per_launch_G%d" % (cfg, G))
        except Exception:
            traffic = None
    return {"kernel": "k_profile", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": peaks.get("hbm_gbs"), "peak_source": peak_src, "unit": "GB/s",
            "frac": round(achieved / peaks.get("hbm_gbs", 1.0), 4), "traffic": traffic,
            "bytes_per_launch": int(plan_bytes), "avg_launch_ms": round(prof_avg_ms, 5),
            "per_rank_frac": [round(x / peaks.get("hbm_gbs", 1.0), 4) for x in per_rank_frac],
            "timing": "CUDA event pair around every k_profile launch in a second pass of K timed steps "
                      "(the headline steps carry no timing nodes)",
            # the same launches on the device clock: first CTA start -> last CTA end
            # (%globaltimer), i.e. without the event pair's launch + completion latency
            "kernel_span_ms": round(span_ms, 5), "achieved_span": round(span_gbs, 1),
            "frac_span": round(span_gbs / peaks.get("hbm_gbs", 1.0), 4)}


def make_segments(D, srcs, dev):
    import torch
    dts, segs = [], []
    for kind, layer, a, ne, E in srcs:
        arr = a.view(np.int32) if a.dtype == np.uint32 else a
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        dts.append((t, arr))
        segs.append(D.SegmentSpec(t, kind, layer, n_elem=ne, n_experts=E))
    return dts, segs


def run_pipeline(args, wl):
    """Configs 2-4: the pipeline's rebalance step (stage s on GPU floor(s G / n))."""
    import torch
    import torch.distributed as dist

    from paper_2505_14864_b200 import dynmo as D

    G, rank, local, dev = dist_setup(args)
    ctx = D.Context(local)
    L, n = wl.L, wl.n
    b_old = uniform_split(L, n)
    ranks = stage_ranks(n, G)
    begin, count = rank_layers(b_old, ranks, rank)
    srcs = list(wl.sources(begin, count))

    # ---- device-resident inputs
    dsrc, segs = make_segments(D, srcs, dev)
    plan = D.ProfilePlan(ctx, segs, begin, count, n_total=L, exchange=args.exchange if G > 1 else False)
    coef = D.coef_tensor(count, device=dev, **wl.coef)
    frozen = (torch.from_numpy(np.ascontiguousarray(wl.frozen[begin:begin + count])).to(dev)
              if wl.frozen is not None else None)
    mem_local = torch.from_numpy(wl.payload[begin:begin + count].astype(np.int64)).to(dev)
    cost = torch.empty(L, dtype=torch.int64, device=dev)
    mem = torch.empty(L, dtype=torch.int64, device=dev)
    batch = D.Batch([L], [n], device=dev)
    cap = torch.tensor([wl.cap], dtype=torch.int64, device=dev)
    bnd_in = torch.from_numpy(b_old).to(dev)
    gamma = torch.zeros(1, dtype=torch.int64, device=dev)
    gamma_f = torch.tensor([wl.gamma_fluid], dtype=torch.float64, device=dev)
    bound = torch.tensor([wl.bound], dtype=torch.int64, device=dev)
    floor = torch.ones(1, dtype=torch.int32, device=dev)
    # every int32 result the host needs lives in ONE device buffer (views), so
    # the step's single D2H boundary is one cudaMemcpyAsync
    nb = batch.total_bnd
    res_d = torch.empty(nb + 4, dtype=torch.int32, device=dev)
    res_h = torch.empty(nb + 4, dtype=torch.int32, pin_memory=True)
    part = dict(bnd=res_d[:nb], bott=torch.empty(1, dtype=torch.int64, device=dev),
                imb=torch.empty(1, dtype=torch.float64, device=dev), st=res_d[nb:nb + 1])
    pst = res_d[nb + 1:nb + 2]
    dif_out = {"status": res_d[nb + 2:nb + 3]}
    rep_out = {"status": res_d[nb + 3:nb + 4]}
    flush = L2Flush(dev)

    # ---- migration buffers (payload per layer; nothing migrates at G = 1)
    send = ({layer: [torch.empty(int(wl.payload[layer]), dtype=torch.uint8, device=dev)]
             for layer in range(begin, begin + count)} if G > 1 else {})
    recv = {}

    side = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
    comm = torch.cuda.Stream(device=dev)
    ev_res = torch.cuda.Event(external=True)  # in-graph record node after the result D2H
    n_host = nb + 2                            # boundaries + partition & profile status
    d_bold = torch.from_numpy(b_old.astype(np.int32)).to(dev)
    d_ranks = torch.from_numpy(ranks.astype(np.int32)).to(dev)
    d_bytes = torch.zeros(2, dtype=torch.int64, device=dev)
    use_map = bool(args.map_stages) and G > 1
    d_slots = torch.arange(n, dtype=torch.int32, device=dev)  # old stage s in slot s (on GPU ranks[s])
    d_rmap = d_ranks.clone()  # new stage -> GPU (identity placement unless --map-stages)
    map_out = dict(kept=torch.zeros(1, dtype=torch.int64, device=dev),
                   status=torch.zeros(1, dtype=torch.int32, device=dev))
    # device-driven migration (G > 1, peer memory): the whole step is one graph
    # (also at G = 1, where nothing migrates: the step never waits on the host)
    dev_mig = (G == 1 or args.migrate == "p2p") and not args.host_migrate
    pmig = None

    def solve_async():
        """profile -> partition [-> device-driven migration] on the main branch,
        diffusion and repack on two side branches, joined at the end."""
        main = torch.cuda.current_stream()
        with torch.cuda.nvtx.range("dynmo.profile"):
            D.profile_layers(ctx, plan, coef, frozen=frozen, mem_local=mem_local, cost=cost, mem=mem, status=pst)
        for sd in side:
            sd.wait_stream(main)
        with torch.cuda.stream(side[0]), torch.cuda.nvtx.range("dynmo.diffuse"):
            D.diffuse_balance(ctx, batch, cost, bnd_in, mem=mem, cap=cap, gamma=gamma, gamma_fluid=gamma_f,
                              max_rounds=256, out=dif_out)
        with torch.cuda.stream(side[1]), torch.cuda.nvtx.range("dynmo.repack"):
            D.repack_workers(ctx, batch, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rep_out)
        with torch.cuda.nvtx.range("dynmo.partition"):
            D.partition_stages(ctx, batch, cost, mem=mem, cap=cap, bnd=part["bnd"], bottleneck=part["bott"],
                               imbalance=part["imb"], status=part["st"])
        if use_map:
            D.map_stages(ctx, L, d_bold, d_slots, part["bnd"], mem, n, slot_rank=d_ranks, rank_new=d_rmap,
                         kept=map_out["kept"], status=map_out["status"])
        if dev_mig and pmig is not None:
            with torch.cuda.nvtx.range("dynmo.migrate"):
                pmig.device(d_bold, d_ranks, part["bnd"], d_rmap, d_bytes[0:1], d_bytes[1:2])
        if args.result_read == "publish":
            D.publish(ctx, res_d[:n_host], res_h[:n_host])
        else:
            res_h[:n_host].copy_(res_d[:n_host], non_blocking=True)
        ev_res.record(main)
        for sd in side:
            main.wait_stream(sd)

    # first step (eager): learn the new split, allocate the receive buffers
    solve_async()
    ev_res.synchronize()
    torch.cuda.synchronize()
    r0 = res_h.numpy()[:n_host].copy()
    b_new = r0[:n + 1].copy()
    if r0[nb] != 0 or r0[nb + 1] != 0:
        raise SystemExit(f"rebalance failed: statuses {r0[nb:]}")
    rank_new = d_rmap.cpu().numpy() if use_map else ranks
    if use_map and int(map_out["status"].item()) != 0:
        raise SystemExit(f"map_stages failed: {int(map_out['status'].item())}")
    moves = D.migration_plan(L, b_old, ranks, b_new, rank_new)
    moves_mine = any(int(sr) == rank or int(ds) == rank for _, sr, ds in moves)
    if G > 1:
        for layer, src, dst in moves:
            if dst == rank:
                recv[int(layer)] = [torch.empty(int(wl.payload[layer]), dtype=torch.uint8, device=dev)]
        if args.migrate == "p2p":
            pmig = migrator = D.PeerMigrator(ctx, L, send, recv)
        else:
            migrator = D.Migrator(ctx, L, send, recv)

    timer = StepTimer(ctx, dev, args.steps)
    graph = None

    def step(k=0):
        """One step; host-driven migration: D2H of the boundaries, then the call."""
        if dev_mig:
            if timer.copies:
                timer.replay(k)
            else:
                solve_async()
            return None
        if graph is not None:
            graph.replay()
        else:
            solve_async()
        ev_res.synchronize()
        r = res_h.numpy()[:n_host].copy()
        main = torch.cuda.current_stream()
        with torch.cuda.stream(comm):  # overlaps the side branches
            sr = migrator(b_old, ranks, r[:n + 1], rank_new) if G > 1 else (0, 0)
        main.wait_stream(comm)
        return sr

    rtimer, rgraph = None, None
    if args.graph:
        # headline graphs: no timing nodes (each event-record node costs ~3 us
        # of the step); the roofline pass below replays copies captured with
        # the k_profile event pair (+ the kernel's device-clock span)
        ctx.set_timing(False)
        if dev_mig:
            timer.capture(solve_async)
        else:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=torch.cuda.Stream(device=dev)):
                solve_async()
        ctx.set_timing(True, phases=["profile"])
        if dev_mig:
            rtimer = StepTimer(ctx, dev, args.steps)
            rtimer.capture(solve_async)
        else:
            rgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(rgraph, stream=torch.cuda.Stream(device=dev)):
                solve_async()
        torch.cuda.synchronize()
        ctx.timing_read()  # discard
        ctx.profile_span()
        ctx.set_timing(False)
    stream = torch.cuda.current_stream()

    for w in range(max(args.warmup, 3, len(timer.copies))):
        flush()
        step(w)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.timing_read()  # reset accumulators
    bar = torch.zeros(1, device=dev)

    def step_barrier():
        # rebalancing runs at the training iteration barrier: align the
        # ranks' step starts on the device, outside the timed interval
        if G > 1:
            dist.all_reduce(bar)

    sent_recv = (0, 0)
    with ClockSampler(local) as clk:
        clk.start()
        if timer.copies:
            step_list = timer.run(args.steps, flush, ctx.timing_poll)
        else:
            step_list = []
            for k in range(args.steps):
                flush()
                step_barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sr = step(k)
                if sr is not None:
                    sent_recv = sr
                b.record(stream)
                b.synchronize()  # outside the timed interval: fold the phase events
                ctx.timing_poll()
                step_list.append(a.elapsed_time(b))
        torch.cuda.synchronize()
        clk.stop()
    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.set_timing(False)
    phases = ctx.timing_read()
    step_ms = np.array(step_list)
    total_ms = float(step_ms.sum())
    prof_ms, prof_n = phases["profile"]
    span_ms, span_n = 0.0, 0
    if args.graph:
        # ---- roofline pass: K more timed steps whose graphs carry the k_profile
        # event pair (CUDA events on the launching stream) and the kernel's
        # own device-clock span
        ctx.set_timing(True)
        for w in range(3):
            flush()
            if rtimer is not None:
                rtimer.replay(w)
            else:
                rgraph.replay()
                ev_res.synchronize()
        torch.cuda.synchronize()
        if G > 1:
            dist.barrier()
        ctx.timing_poll()
        ctx.timing_read()
        ctx.profile_span()
        if rtimer is not None:
            rtimer.run(args.steps, flush, ctx.timing_poll)
        else:
            for k in range(args.steps):
                flush()
                step_barrier()
                rgraph.replay()
                ev_res.synchronize()
                torch.cuda.synchronize()
                ctx.timing_poll()
        torch.cuda.synchronize()
        if G > 1:
            dist.barrier()
        ctx.set_timing(False)
        prof_ms, prof_n = ctx.timing_read()["profile"]
        span_ms, span_n = ctx.profile_span()
    prof_avg = prof_ms / max(prof_n, 1)
    span_avg = span_ms / max(span_n, 1) if span_n else 0.0
    # our kernel nodes per step: k_profile, k_epilogue (the peer-memory
    # exchange's unpack runs in its last block; the NCCL exchange adds
    # k_unpack), k_partition, k_diffuse, k_repack, [k_map_stages], [k_publish], and at G > 1
    # the migration: one k_mig_fused in the graph (device-driven), or
    # k_signal / k_pull / k_wait per host-driven call, or none (NCCL)
    exch_kernels = 1 if (G > 1 and args.exchange == "nccl") else 0
    if G == 1:
        mig_kernels = 0
    elif dev_mig:
        mig_kernels = 1
    else:
        mig_kernels = 3 if (args.migrate == "p2p" and moves_mine) else 0
    per_step = 5 + exch_kernels + mig_kernels + (1 if use_map else 0) + (
        args.result_read == "publish" and n_host * 4 <= D.PUBLISH_KERNEL_MAX)
    launches = per_step * args.steps
    mig_ms = phases["migrate"][0] / max(phases["migrate"][1], 1) if phases["migrate"][1] else 0.0
    if dev_mig:
        sent_recv = tuple(int(v) for v in d_bytes.cpu().tolist())

    # ---- e2e: host buffers, H2D of this step's sources + D2H of the result inside
    pinned = [torch.from_numpy(np.ascontiguousarray(arr)).pin_memory() for _, arr in dsrc]
    h2d = int(sum(p.numel() * p.element_size() for p in pinned))
    d2h = int(res_h.numel() * 4)
    e2e = []
    for k in range(args.e2e_steps):
        flush()
        step_barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for (t, _), p in zip(dsrc, pinned):
            t.copy_(p, non_blocking=True)
        step()
        if dev_mig:
            ev_res.synchronize()  # the result has reached the host
        b.record(stream)
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2e))

    # ---- diagnostic pass: a second graph with every phase timed (the event
    # nodes cost ~17 us per step, so the headline loop times only k_profile)
    diag_phases = None
    if args.graph:
        ctx.timing_detach()  # the timed graphs' events are not part of the diagnostic pass
        ctx.set_timing(True)
        gdiag = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gdiag, stream=torch.cuda.Stream(device=dev)):
            solve_async()
        torch.cuda.synchronize()
        ctx.timing_read()
        for k in range(20):
            flush()
            step_barrier()
            gdiag.replay()
            if not dev_mig:
                ev_res.synchronize()
            torch.cuda.synchronize()
            ctx.timing_poll()
        diag = ctx.timing_read()
        ctx.set_timing(False)
        diag_phases = {k: round(v[0] / max(v[1], 1), 5) if v[1] else 0.0 for k, v in diag.items()}
        del gdiag
    if diag_phases and diag_phases.get("migrate"):
        mig_ms = diag_phases["migrate"]

    # ---- reductions over ranks (max of device time)
    achieved_local = plan.bytes / (prof_avg * 1e-3) / 1e9 if prof_avg > 0 else 0.0
    total_ms, prof_avg_max, e2e_ms, mig_ms, max_sent, max_recv = reduce_max(
        [total_ms, prof_avg, e2e_ms, mig_ms, float(sent_recv[0]), float(sent_recv[1])], dev, G)
    per_rank_gbs = gather_list(achieved_local, dev, G)
    prof_at_min = gather_list(prof_avg, dev, G)
    span_all = gather_list(span_avg, dev, G)
    bytes_all = gather_list(plan.bytes, dev, G)
    # per-step job time = max over ranks of each step's device interval
    st_t = torch.tensor(step_ms, dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(st_t, op=dist.ReduceOp.MAX)
    step_ms = st_t.cpu().numpy()

    if rank == 0:
        ms = total_ms / args.steps
        worst = int(np.argmin(per_rank_gbs))  # the roofline line reports the slowest rank's kernel
        cost_h = cost.cpu().numpy()
        x_old = np.add.reduceat(cost_h, b_old[:-1])
        x_new = np.add.reduceat(cost_h, b_new[:-1])
        dl = lambda x: float((x.max() - x.min()) / (x.sum() / len(x)))
        out = {
            "metric": METRIC, "value": round(ms, 5), "unit": "ms", "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": wl.config(G),
            "setup": {
                "exchange": ("peer-memory" if args.exchange == "p2p" else "nccl-allgather") if G > 1 else "none (G=1)",
                "migration": ("none (G=1)" if G == 1 else "device-driven peer-memory pull, in the step graph"
                              if dev_mig else "host-driven peer-memory pull" if args.migrate == "p2p"
                              else "host-driven NCCL send/recv"),
                "graph": bool(args.graph),
                "result_read": ("kernel store into mapped pinned memory (dynmo_publish)"
                                if args.result_read == "publish" else "D2H copy node"),
                "stage_placement": ("migration-minimising (dynmo_map_stages, NEXT-3)" if use_map
                                    else f"stage s on GPU floor(s*G/{n}) before and after")},
            "roofline": roofline(bytes_all[worst], prof_at_min[worst], per_rank_gbs, G, args.config, span_all[worst]),
            "phases_ms_per_launch_diagnostic": diag_phases,
            "step_ms": step_stats(step_ms),
            "migrate": {"moved_layers": int(len(moves)), "max_bytes_sent_per_gpu": int(max_sent),
                        "max_bytes_recv_per_gpu": int(max_recv), "avg_ms": round(mig_ms, 5),
                        "nvlink_GBps": round(max(max_sent, max_recv) / (mig_ms * 1e-3) / 1e9, 1)
                        if mig_ms > 0 else None, "nvlink_peak_GBps": NVLINK_PEER_GBS,
                        "nvlink_nominal_GBps": 900.0,
                        "frac_of_nominal": round(max(max_sent, max_recv) / (mig_ms * 1e-3) / 1e9 / 900.0, 3)
                        if mig_ms > 0 else None,
                        "path": ("NCCL send/recv" if args.migrate == "nccl" else "NVLink peer-memory pull")
                        if G > 1 else None},
            "solution": {"b_old": b_old.tolist(), "b_new": b_new.tolist(),
                         "bottleneck_old": int(x_old.max()), "bottleneck_new": int(part["bott"].item()),
                         "imbalance_old": round(dl(x_old), 4), "imbalance_new": round(float(part["imb"].item()), 4),
                         "diffusion_rounds": int(dif_out["rounds"].item()),
                         "repack_n_new": int(rep_out["n_new"].item()),
                         "statuses": [int(x) for x in res_d.cpu().numpy()[nb:nb + 4]]},
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if G == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(wl, args, srcs)
        print(json.dumps(out), flush=True)
    # teardown order: graphs holding NCCL work (the in-graph barrier) before
    # the communicator, then the peer-memory plans, then the ctx
    torch.cuda.synchronize()
    timer.copies.clear()
    if rtimer is not None:
        rtimer.copies.clear()
    graph = rgraph = None  # noqa: F841
    torch.cuda.synchronize()
    if pmig is not None:
        pmig.close()
    plan.close()
    ctx.close()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_batch(args, wl):
    """Config 5: 4096 independent instances sharded 4096/G per GPU (weak
    scaling per GPU: no exchange, no migration); one step = profile of the
    MoD token masks -> memory-capped partition and BOUND repack of every
    instance -> D2H of the per-instance results."""
    import torch
    import torch.distributed as dist

    from paper_2505_14864_b200 import _lib as LB
    from paper_2505_14864_b200 import dynmo as D

    G, rank, local, dev = dist_setup(args)
    ctx = D.Context(local)
    insts = wl.shard(rank, G)
    words = np.concatenate([x.masks.reshape(-1) for x in insts]).view(np.int32)
    dwords = torch.from_numpy(words).to(dev)
    segs, off, nl = [], 0, 0
    W = insts[0].masks.shape[1]
    for x in insts:
        for l in range(x.L):
            segs.append(D.SegmentSpec(dwords[off:off + W], LB.SRC_TOKMASK_BITS, nl, n_elem=W * 32))
            off += W
            nl += 1
    plan = D.ProfilePlan(ctx, segs, 0, nl)
    coef = D.coef_tensor(nl, A=1, device=dev)
    cost = torch.empty(nl, dtype=torch.int64, device=dev)
    batch = D.Batch([x.L for x in insts], [x.n for x in insts], device=dev)
    mem = torch.from_numpy(np.concatenate([x.mem for x in insts]).astype(np.int64)).to(dev)
    cap = torch.from_numpy(np.array([x.cap for x in insts], np.int64)).to(dev)
    bound = torch.from_numpy(np.array([x.bound for x in insts], np.int64)).to(dev)
    floor = torch.ones(len(insts), dtype=torch.int32, device=dev)
    q = len(insts)
    # per-instance results the host reads: partition status, repack n_new and
    # status, + the profile status (one D2H)
    res_d = torch.empty(3 * q + 1, dtype=torch.int32, device=dev)
    res_h = torch.empty(3 * q + 1, dtype=torch.int32, pin_memory=True)
    part = dict(bnd=torch.empty(batch.total_bnd, dtype=torch.int32, device=dev),
                bott=torch.empty(q, dtype=torch.int64, device=dev), st=res_d[:q])
    rep_out = {"n_new": res_d[q:2 * q], "status": res_d[2 * q:3 * q]}
    pst = res_d[3 * q:3 * q + 1]
    flush = L2Flush(dev)
    side = torch.cuda.Stream(device=dev)
    ev_res = torch.cuda.Event(external=True)

    def solve_async():
        main = torch.cuda.current_stream()
        with torch.cuda.nvtx.range("dynmo.profile"):
            D.profile_layers(ctx, plan, coef, cost=cost, status=pst)
        side.wait_stream(main)
        with torch.cuda.stream(side), torch.cuda.nvtx.range("dynmo.repack"):
            D.repack_workers(ctx, batch, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rep_out)
        with torch.cuda.nvtx.range("dynmo.partition"):
            D.partition_stages(ctx, batch, cost, mem=mem, cap=cap, bnd=part["bnd"], bottleneck=part["bott"],
                               status=part["st"])
        main.wait_stream(side)
        if args.result_read == "publish":
            D.publish(ctx, res_d, res_h)
        else:
            res_h.copy_(res_d, non_blocking=True)
        ev_res.record(main)

    solve_async()
    torch.cuda.synchronize()
    r0 = res_h.numpy().copy()
    if np.any(r0[:q] != 0) or np.any(r0[2 * q:3 * q] < 0) or r0[3 * q] != 0:
        raise SystemExit("config 5 rebalance failed")
    # headline graphs without timing nodes; roofline graphs with the k_profile
    # event pair and the kernel's device-clock span (a second timed pass)
    timer = StepTimer(ctx, dev, args.steps)
    ctx.set_timing(False)
    timer.capture(solve_async)
    rtimer = StepTimer(ctx, dev, args.steps)
    ctx.set_timing(True, phases=["profile"])
    rtimer.capture(solve_async)
    torch.cuda.synchronize()
    ctx.timing_read()
    ctx.profile_span()
    ctx.set_timing(False)
    for w in range(max(args.warmup, 3, timer.C)):
        flush()
        timer.replay(w)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        clk.start()
        step_list = timer.run(args.steps, flush)
        torch.cuda.synchronize()
        clk.stop()
    if G > 1:
        dist.barrier()
    ctx.set_timing(True)
    for w in range(3):
        flush()
        rtimer.replay(w)
    torch.cuda.synchronize()
    ctx.timing_poll()
    ctx.timing_read()
    ctx.profile_span()
    if G > 1:
        dist.barrier()
    rtimer.run(args.steps, flush, ctx.timing_poll)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    ctx.set_timing(False)
    prof_ms, prof_n = ctx.timing_read()["profile"]
    span_ms, span_n = ctx.profile_span()
    prof_avg = prof_ms / max(prof_n, 1)
    span_avg = span_ms / max(span_n, 1) if span_n else 0.0
    step_ms = np.array(step_list)
    total_ms = float(step_ms.sum())
    # e2e: H2D of the rank's token masks from pinned memory + the result D2H
    pinned = torch.from_numpy(words).pin_memory()
    e2e = []
    bar = torch.zeros(1, device=dev)
    stream = torch.cuda.current_stream()
    for k in range(args.e2e_steps):
        flush()
        if G > 1:
            dist.all_reduce(bar)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dwords.copy_(pinned, non_blocking=True)
        timer.replay(k)
        ev_res.synchronize()
        b.record(stream)
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2e))
    achieved_local = plan.bytes / (prof_avg * 1e-3) / 1e9 if prof_avg > 0 else 0.0
    total_ms, e2e_ms = reduce_max([total_ms, e2e_ms], dev, G)
    per_rank_gbs = gather_list(achieved_local, dev, G)
    prof_all = gather_list(prof_avg, dev, G)
    span_all = gather_list(span_avg, dev, G)
    bytes_all = gather_list(plan.bytes, dev, G)
    n_new_sum = gather_list(float(r0[q:2 * q].sum()), dev, G)
    n_cur_sum = gather_list(float(sum(x.n for x in insts)), dev, G)
    st_t = torch.tensor(step_ms, dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(st_t, op=dist.ReduceOp.MAX)
    step_ms = st_t.cpu().numpy()
    if rank == 0:
        ms = total_ms / args.steps
        worst = int(np.argmin(per_rank_gbs))
        out = {
            "metric": METRIC, "value": round(ms, 5), "unit": "ms", "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": wl.config(G),
            "setup": {"graph": True, "exchange": "none (independent instances)", "migration": "none",
                      "result_read": ("kernel store into mapped pinned memory (dynmo_publish)"
                                      if args.result_read == "publish" else "D2H copy node")},
            "instances_per_s": round(wl.N_INST / (ms * 1e-3), 1),
            "roofline": roofline(bytes_all[worst], prof_all[worst], per_rank_gbs, G, args.config, span_all[worst]),
            "step_ms": step_stats(step_ms),
            "solution": {"workers_before": int(sum(n_cur_sum)), "workers_after_repack": int(sum(n_new_sum))},
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": int(words.nbytes),
                    "d2h_bytes_per_step": int(res_h.numel() * 4), "steps": args.e2e_steps},
            # k_profile, k_epilogue, k_partition, k_repack, [k_publish]
            "gpu_launches": (4 + (args.result_read == "publish"
                                  and res_h.numel() * 4 <= D.PUBLISH_KERNEL_MAX)) * args.steps,
            "clocks": clk.summary(),
        }
        if G == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(wl, args)
        print(json.dumps(out), flush=True)
    torch.cuda.synchronize()
    timer.copies.clear()
    rtimer.copies.clear()
    torch.cuda.synchronize()
    plan.close()
    ctx.close()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_dynmo(args):
    wl = WORKLOADS[args.config](args)
    return run_batch(args, wl) if wl.key == 5 else run_pipeline(args, wl)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_dynmo(args)


if __name__ == "__main__":
    sys.exit(main())

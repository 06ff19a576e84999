"""How much of the event-bracketed k_profile time is the brackets: the same
profile call (bench workloads 2, 4, 5 at G = 1, L2 flushed before each) timed
(a) by the library's phase events inside a captured graph (bench.py's way),
(b) by the library's phase events on eager launches,
(c) by a graph of the profile call alone between the flush and a bench-side
    event pair (one pair around the whole replay),
and the step graph's duration with and without the phase-event nodes.
Prints one JSON line per workload.  python tools/event_overhead.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
ctx = D.Context(0)
flush = bench.L2Flush(dev)
REPS = 30


def med(v):
    return round(float(np.median(v)) * 1e3, 2)  # us


for cfg in (2, 4, 5):
    args = bench.parse(["--config", str(cfg)])
    wl = bench.WORKLOADS[cfg](args)
    if cfg == 5:
        insts = wl.shard(0, 1)
        from paper_2505_14864_b200 import _lib as LB
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
        kw = {}
    else:
        L = wl.L
        srcs = list(wl.sources(0, L))
        dsrc, segs = bench.make_segments(D, srcs, dev)
        plan = D.ProfilePlan(ctx, segs, 0, L, n_total=L, exchange=False)
        coef = D.coef_tensor(L, device=dev, **wl.coef)
        kw = {}
    call = lambda: D.profile_layers(ctx, plan, coef, **kw)  # noqa: E731
    call()
    torch.cuda.synchronize()
    out = {"config": cfg, "bytes": int(plan.bytes)}
    # (b) eager, library phase events
    ctx.set_timing(True, phases=["profile"])
    ctx.timing_read()
    for _ in range(REPS):
        flush()
        call()
    torch.cuda.synchronize()
    ms, n = ctx.timing_read()["profile"]
    out["eager_phase_events_us"] = round(ms / n * 1e3, 2)
    # (a) graph with the phase-event nodes (bench.py's way)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    torch.cuda.synchronize()
    ctx.timing_read()
    ctx.timing_poll()
    ctx.timing_read()
    for _ in range(REPS):
        flush()
        g.replay()
        torch.cuda.synchronize()
        ctx.timing_poll()
    ms, n = ctx.timing_read()["profile"]
    out["graph_phase_events_us"] = round(ms / n * 1e3, 2)
    ctx.timing_detach()
    ctx.set_timing(False)
    # (c) graph without phase events, one bench-side event pair around the replay
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        call()
    ts = []
    for _ in range(REPS):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g2.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["graph_replay_events_us (profile + epilogue + graph launch)"] = med(ts)
    # (d) eager launch, bench-side event pair around profile_layers (k_profile + k_epilogue)
    ts = []
    for _ in range(REPS):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["eager_call_events_us (profile + epilogue)"] = med(ts)
    print(json.dumps(out), flush=True)
    plan.close()

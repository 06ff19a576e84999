"""Timeline of the bench's N=1 step graph (config 2): external CUDA events
between the API calls of the captured step give each branch's completion
offset from the step start (L2 flushed before every replay, as in bench.py).
Also times graph variants without the intermediate events (the step as
bench.py runs it, and subsets) to expose launch gaps.  Prints JSON.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402
from paper_2505_14864_b200.pipeline import uniform_split  # noqa: E402

DEV = "cuda:0"


def main():
    torch.cuda.set_device(0)
    ctx = D.Context(0)
    shape = synth.GPTShape()
    inp = bench.Cfg2()
    L, n = shape.L, inp.n
    srcs = list(inp.sources(0, L))
    dmask = [torch.from_numpy(a).to(DEV) for _, _, a, _, _ in srcs]
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(t, LB.SRC_MASK_U8, l) for t, (_, l, _, _, _) in zip(dmask, srcs)], 0, L)
    coef = D.coef_tensor(L, A=0, B=1, device=DEV)
    mem_local = torch.from_numpy(inp.payload.astype(np.int64)).to(DEV)
    cost = torch.empty(L, dtype=torch.int64, device=DEV)
    mem = torch.empty(L, dtype=torch.int64, device=DEV)
    batch = D.Batch([L], [n], device=DEV)
    cap = torch.tensor([inp.cap], dtype=torch.int64, device=DEV)
    bnd_in = torch.from_numpy(uniform_split(L, n)).to(DEV)
    gamma = torch.zeros(1, dtype=torch.int64, device=DEV)
    gamma_f = torch.tensor([inp.gamma_fluid], dtype=torch.float64, device=DEV)
    bound = torch.tensor([inp.bound], dtype=torch.int64, device=DEV)
    floor = torch.ones(1, dtype=torch.int32, device=DEV)
    pst = torch.empty(1, dtype=torch.int32, device=DEV)
    res_h = torch.empty(16, dtype=torch.int32, pin_memory=True)
    part = {}
    dif, rep = {}, {}
    flush = bench.L2Flush(DEV)
    side = [torch.cuda.Stream(), torch.cuda.Stream()]

    def mk():
        return torch.cuda.Event(enable_timing=True, external=True)

    def step(ev=None, parts=("diffuse", "repack", "partition", "d2h"), serial=False):
        main = torch.cuda.current_stream()
        br = [main, main] if serial else side
        if ev is not None:
            ev["start"].record(main)
        D.profile_layers(ctx, plan, coef, mem_local=mem_local, cost=cost, mem=mem, status=pst)
        if ev is not None:
            ev["profile"].record(main)
        for sd in side:
            sd.wait_stream(main)
        if "diffuse" in parts:
            with torch.cuda.stream(br[0]):
                D.diffuse_balance(ctx, batch, cost, bnd_in, mem=mem, cap=cap, gamma=gamma, gamma_fluid=gamma_f,
                                  max_rounds=256, out=dif)
                if ev is not None:
                    ev["diffuse"].record(br[0])
        if "repack" in parts:
            with torch.cuda.stream(br[1]):
                D.repack_workers(ctx, batch, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rep)
                if ev is not None:
                    ev["repack"].record(br[1])
        if "partition" in parts:
            bnd, _, _, st = D.partition_stages(ctx, batch, cost, mem=mem, cap=cap)
            part["bnd"] = bnd
            if ev is not None:
                ev["partition"].record(main)
            if "pub" in parts:
                D.publish(ctx, bnd, res_h[:n + 1])
                if ev is not None:
                    ev["d2h"].record(main)
            if "d2h" in parts:
                res_h[:n + 1].copy_(bnd, non_blocking=True)
                if ev is not None:
                    ev["d2h"].record(main)
        for sd in side:
            main.wait_stream(sd)
        if ev is not None:
            ev["end"].record(main)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            fn()
        torch.cuda.synchronize()
        return g

    out = {}
    names = ["start", "profile", "diffuse", "repack", "partition", "d2h", "end"]
    ev = {k: mk() for k in names}
    g = capture(lambda: step(ev))
    offs = {k: [] for k in names[1:]}
    for i in range(50):
        flush()
        g.replay()
        torch.cuda.synchronize()
        if i >= 10:
            for k in names[1:]:
                offs[k].append(ev["start"].elapsed_time(ev[k]) * 1e3)
    out["timeline_us_from_start"] = {k: round(float(np.median(v)), 2) for k, v in offs.items()}

    def timed(parts, reps=40, serial=False):
        gg = capture(lambda: step(None, parts, serial))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for i in range(reps + 5):
            flush()
            a.record()
            gg.replay()
            b.record()
            b.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        return round(float(np.median(ts)), 2)

    out["graph_us"] = {
        "full": timed(("diffuse", "repack", "partition", "d2h")),
        "full_one_stream": timed(("diffuse", "repack", "partition", "d2h"), serial=True),
        "full_publish": timed(("diffuse", "repack", "partition", "pub")),
        "profile+partition+publish": timed(("partition", "pub")),
        "profile+3_solvers_no_d2h": timed(("diffuse", "repack", "partition")),
        "profile_only": timed(()),
        "profile+partition": timed(("partition",)),
        "profile+partition+d2h": timed(("partition", "d2h")),
        "profile+diffuse": timed(("diffuse",)),
        "profile+repack": timed(("repack",)),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

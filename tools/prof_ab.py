"""A/B timing of one profile source on one B200 (DYNMO_LIB picks the build).

  python tools/prof_ab.py moe    # config 4: 32 layers of int64 top-2 ids (67 MB)
  python tools/prof_ab.py cfg5   # config 5: 4096 instances of MoD token bitmasks (184 MB)
  python tools/prof_ab.py u8 75  # config 2 u8 masks, first 75 MB share

Each call is captured in a CUDA graph; L2 is flushed (256 MiB write + read)
before every replay, outside the CUDA events.  Prints one JSON line with the
median k_profile time (library phase events) and the step time.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402


def segments(which, dev):
    segs, keep = [], []
    if which == "moe":
        T, L, E, k = 64 * 2048, 32, 8, 2
        for i in range(L):
            d = torch.from_numpy(synth.cfg4_routing(i, T=T, E=E, k=k, alpha=4.0).reshape(-1)).to(dev)
            keep.append(d)
            segs.append(D.SegmentSpec(d, LB.SRC_EXPERT_I64, i, n_experts=E, top_k=k))
        return segs, keep, L
    if which == "cfg5":
        insts = [synth.cfg5_instance(i) for i in range(4096)]
        words = np.concatenate([x.masks.reshape(-1) for x in insts])
        d = torch.from_numpy(words.view(np.int32)).to(dev)
        keep.append(d)
        off, layer = 0, 0
        for x in insts:
            m = x.masks
            for i in range(m.shape[0]):
                segs.append(D.SegmentSpec(d[off:off + m.shape[1]], LB.SRC_TOKMASK_BITS, layer, n_elem=m.shape[1] * 32))
                off += m.shape[1]
                layer += 1
        return segs, keep, layer
    if which == "u8":
        mb = float(sys.argv[2]) if len(sys.argv) > 2 else 604
        shape = synth.GPTShape()
        p = synth.cfg2_keep_probs(shape, 0.9, 4)
        tot, L = 0, 0
        for layer in range(shape.L):
            for m in synth.cfg2_layer_masks_u8(shape, layer, p[layer], 4):
                d = torch.from_numpy(m.reshape(-1)).to(dev)
                keep.append(d)
                segs.append(D.SegmentSpec(d, LB.SRC_MASK_U8, layer))
                tot += m.size
            L = layer + 1
            if tot >= mb * 1e6:
                break
        return segs, keep, L
    raise SystemExit(f"unknown source {which}")


def main():
    which = sys.argv[1]
    dev = "cuda:0"
    torch.cuda.set_device(0)
    ctx = D.Context(0)
    segs, keep, L = segments(which, dev)
    plan = D.ProfilePlan(ctx, segs, 0, L)
    coef = D.coef_tensor(L, A=1, B=1, C_=1, ep=8 if which == "moe" else 0, device=dev)
    cost = torch.empty(L, dtype=torch.int64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    D.profile_layers(ctx, plan, coef, cost=cost, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    ref = cost.clone()
    ctx.set_timing(True, phases=["profile"])
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        D.profile_layers(ctx, plan, coef, cost=cost, status=st, stream=s)
    ctx.timing_read()
    prof, step = [], []
    for it in range(60):
        flush.fill_(it & 0xFF)
        flush.sum(dtype=torch.int64)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ctx.timing_poll()
        ms, n = ctx.timing_read()["profile"]
        if it >= 10:
            prof.append(ms / max(n, 1))
            step.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    assert torch.equal(cost, ref) and int(st.item()) == 0
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    kp = float(np.median(prof))
    print(json.dumps({"source": which, "lib": os.path.basename(LB.LIB_PATH), "bytes": plan.bytes,
                      "tiles": plan.n_tiles, "k_profile_ms": kp, "step_ms": float(np.median(step)),
                      "gbs": plan.bytes / kp / 1e6, "frac": plan.bytes / kp / 1e6 / peak}))


if __name__ == "__main__":
    main()

"""k_profile on the per-GPU share of config 2 at G = 1, 2, 4, 8 (the first
48/G layers: 604 / 302 / 151 / 75.5 MB of u8 masks), L2 flushed before every
call, timed like bench.py's roofline pass: the CUDA-event pair the library
records around the launch and the kernel's device-clock span
(dynmo_ctx_profile_span).  One JSON line per share.
python tools/profile_shares.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402

REPS = 50
torch.cuda.set_device(0)
ctx = D.Context(0)
peak = bench.load_peaks()[0]["hbm_gbs"]
flush = bench.L2Flush("cuda")
wl = bench.Cfg2()
for G in (1, 2, 4, 8):
    n = 48 // G
    srcs = list(wl.sources(0, n))
    dm = [torch.from_numpy(a).to("cuda") for _, _, a, _, _ in srcs]
    plan = D.ProfilePlan(ctx, [D.SegmentSpec(t, LB.SRC_MASK_U8, l) for t, (_, l, _, _, _) in zip(dm, srcs)], 0, n)
    coef = D.coef_tensor(n, A=0, B=1, device="cuda")
    cost = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(5):
        flush()
        D.profile_layers(ctx, plan, coef, cost=cost)
    torch.cuda.synchronize()
    ctx.set_timing(True, phases=["profile"])
    ctx.timing_read()
    ctx.profile_span()
    for _ in range(REPS):
        flush()
        D.profile_layers(ctx, plan, coef, cost=cost)
    torch.cuda.synchronize()
    ev_ms, ev_n = ctx.timing_read()["profile"]
    sp_ms, sp_n = ctx.profile_span()
    ctx.set_timing(False)
    ev, sp = ev_ms / ev_n, sp_ms / sp_n
    print(json.dumps({"G": G, "layers": n, "bytes": int(plan.bytes), "event_us": round(ev * 1e3, 2),
                      "span_us": round(sp * 1e3, 2), "frac_event": round(plan.bytes / (ev * 1e-3) / 1e9 / peak, 4),
                      "frac_span": round(plan.bytes / (sp * 1e-3) / 1e9 / peak, 4), "peak_gbs": peak,
                      "launches": ev_n}), flush=True)
    plan.close()

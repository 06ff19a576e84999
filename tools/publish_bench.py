"""Result read to the host: dynmo_publish (kernel stores into mapped pinned
memory) vs a D2H copy node, inside a CUDA graph after a dependent kernel,
per size.  One JSON line per size.  DYNMO_PUBLISH_CTA_BYTES sets the bytes
per CTA of the publish kernel.  python tools/publish_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_14864_b200 import dynmo as D  # noqa: E402

torch.cuda.set_device(0)
ctx = D.Context(0)
for nb in (48, 4096, 49156, 1 << 20):
    src = torch.zeros(nb // 4, dtype=torch.int32, device="cuda")
    dst = torch.zeros(nb // 4, dtype=torch.int32).pin_memory()
    out = {"bytes": nb, "cta_bytes": int(os.environ.get("DYNMO_PUBLISH_CTA_BYTES", "16384"))}
    for mode in ("none", "copy", "publish"):
        def body():
            src.add_(1)
            if mode == "copy":
                dst.copy_(src, non_blocking=True)
            elif mode == "publish":
                D.publish(ctx, src, dst)
        body()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            body()
        ts = []
        for i in range(60):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            if i >= 10:
                ts.append(a.elapsed_time(b) * 1e3)
        out[mode + "_us"] = round(float(np.median(ts)), 2)
        if mode != "none":
            assert int(dst[0]) == int(src[0].item()), mode
        del g
    print(json.dumps(out), flush=True)

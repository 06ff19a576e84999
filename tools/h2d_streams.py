"""H2D throughput of config 2's 604 MB of u8 masks (192 tensors of ~3.1 MB,
pinned host memory) issued round-robin on S streams: does spreading the
copies over several copy engines raise the PCIe rate?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
srcs = list(bench.Cfg2().sources(0, 48))
pinned = [torch.from_numpy(a).pin_memory() for _, _, a, _, _ in srcs]
dev = [torch.empty_like(p, device="cuda") for p in pinned]
total = sum(p.numel() for p in pinned)
for S in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(S)]
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s_ in streams:
            s_.wait_stream(torch.cuda.current_stream())
        for i, (d, p) in enumerate(zip(dev, pinned)):
            with torch.cuda.stream(streams[i % S]):
                d.copy_(p, non_blocking=True)
        for s_ in streams:
            torch.cuda.current_stream().wait_stream(s_)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"streams={S}: {best:.2f} ms  {total / (best * 1e-3) / 1e9:.1f} GB/s")

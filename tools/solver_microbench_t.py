"""Graph-replay device timing helper shared by the solver microbenchmarks."""
import torch


def t(fn, iters=20, reps=20):
    """Device time per call: capture `iters` back-to-back calls in a CUDA graph
    and time graph replays (no host launch overhead inside)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / (iters * reps) * 1e3, 2)

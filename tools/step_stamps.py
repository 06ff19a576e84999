"""Device timeline of the config-2 N = 1 step graph (bench.py's structure:
profile -> {diffusion | repack} on side streams, partition + result
publication on the main stream, joined): each kernel's first-warp start and
last-warp end (%globaltimer) relative to k_profile's start, median over
replays, with the diagnostic build (-DDYNMO_STEP_STAMPS):
DYNMO_LIB=ab/libdynmo_stamps.so python tools/step_stamps.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2505_14864_b200 import _lib as LB  # noqa: E402
from paper_2505_14864_b200 import dynmo as D  # noqa: E402
from paper_2505_14864_b200.pipeline import uniform_split  # noqa: E402

DEV = "cuda:0"
NAMES = ["profile", "epilogue", "publish", "partition", "diffuse_discrete", "diffuse_fluid", "repack"]
torch.cuda.set_device(0)
ctx = D.Context(0)
L_ = LB.lib()
fn = L_.dynmo_diag_step_stamps  # signature bound in _lib
buf = (ctypes.c_ulonglong * (4 * len(NAMES)))()
if fn(buf, 1) == 0:
    raise SystemExit("not a -DDYNMO_STEP_STAMPS build (set DYNMO_LIB)")
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
flush = bench.L2Flush(DEV)
side = [torch.cuda.Stream(), torch.cuda.Stream()]
dif, rep = {}, {}
part = dict(bnd=torch.empty(batch.total_bnd, dtype=torch.int32, device=DEV),
            bottleneck=torch.empty(1, dtype=torch.int64, device=DEV),
            imbalance=torch.empty(1, dtype=torch.float64, device=DEV),
            status=torch.empty(1, dtype=torch.int32, device=DEV))


PREWARM = os.environ.get("STAMPS_PREWARM") == "1"  # solvers pre-run on a stale profile during k_profile
wstream = torch.cuda.Stream()
cost_w, mem_w = torch.empty_like(cost), torch.empty_like(mem)
dif_w, rep_w = {}, {}
part_w = {k: torch.empty_like(v) for k, v in part.items()}


def prewarm():
    D.diffuse_balance(ctx, batch, cost_w, bnd_in, mem=mem_w, cap=cap, gamma=gamma, gamma_fluid=gamma_f,
                      max_rounds=256, out=dif_w)
    D.repack_workers(ctx, batch, cost_w, floor=floor, bound=bound, mem=mem_w, cap=cap, out=rep_w)
    D.partition_stages(ctx, batch, cost_w, mem=mem_w, cap=cap, **part_w)


def step():
    main = torch.cuda.current_stream()
    if PREWARM:
        wstream.wait_stream(main)
        with torch.cuda.stream(wstream):
            prewarm()
    D.profile_layers(ctx, plan, coef, mem_local=mem_local, cost=cost, mem=mem, status=pst)
    for sd in side:
        sd.wait_stream(main)
    with torch.cuda.stream(side[0]):
        D.diffuse_balance(ctx, batch, cost, bnd_in, mem=mem, cap=cap, gamma=gamma, gamma_fluid=gamma_f,
                          max_rounds=256, out=dif)
    with torch.cuda.stream(side[1]):
        D.repack_workers(ctx, batch, cost, floor=floor, bound=bound, mem=mem, cap=cap, out=rep)
    D.partition_stages(ctx, batch, cost, mem=mem, cap=cap, **part)
    D.publish(ctx, part["bnd"], res_h[:n + 1])
    for sd in side:
        main.wait_stream(sd)
    if PREWARM:
        main.wait_stream(wstream)


step()
torch.cuda.synchronize()
cost_w.copy_(cost)
mem_w.copy_(mem)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=torch.cuda.Stream()):
    step()
torch.cuda.synchronize()
rows = []
NOFLUSH = os.environ.get("STAMPS_NOFLUSH") == "1"  # diagnostic: L2 (data and code) left warm
for i in range(60):
    if not NOFLUSH:
        flush()
    torch.cuda.synchronize()
    fn(buf, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    fn(buf, 0)
    v = np.array(buf[:], dtype=np.float64).reshape(2, len(NAMES), 2)
    merged = np.where((v[0, :, 1] > 0)[:, None], v[0], v[1])  # each kernel is in one of the two tables
    t0 = merged[0, 0]
    if i >= 10:
        rows.append([(merged[k, 0] - t0) / 1e3 for k in range(len(NAMES))] +
                    [(merged[k, 1] - t0) / 1e3 for k in range(len(NAMES))] + [a.elapsed_time(b) * 1e3])
med = np.median(np.array(rows), axis=0)
k = len(NAMES)
out = {nm: {"start_us": round(med[j], 2), "end_us": round(med[k + j], 2), "dur_us": round(med[k + j] - med[j], 2)}
       for j, nm in enumerate(NAMES)}
out["graph_replay_events_us"] = round(med[-1], 2)
print(json.dumps(out, indent=1))

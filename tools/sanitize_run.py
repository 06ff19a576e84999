"""Small-size run of every kernel family for compute-sanitizer (profile: all
source kinds incl. unaligned heads/tails; partition / diffusion (+fluid) /
repack BOUND + ALG2, with and without memory caps; 1 and 8 warps per CTA)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2505_14864_b200 import _lib as LB, dynmo as D
torch.cuda.set_device(0)
dev = "cuda:0"
ctx = D.Context(0)
g = np.random.default_rng(0)
# profile: every source kind, odd sizes and offsets
segs, keep = [], []
def add(t, kind, layer, **kw):
    keep.append(t); segs.append(D.SegmentSpec(t, kind, layer, **kw))
base = torch.from_numpy((g.random(70001) < 0.3).astype(np.uint8)).to(dev)
add(base[3:], LB.SRC_MASK_U8, 0)
w = torch.from_numpy(g.integers(-2**31, 2**31 - 1, 999, dtype=np.int64).astype(np.int32)).to(dev)
add(w, LB.SRC_MASK_BITS, 1, n_elem=999 * 32 - 5)
add(w, LB.SRC_TOKMASK_BITS, 2, n_elem=600)
h = torch.from_numpy(g.integers(-2**15, 2**15 - 1, 5003, dtype=np.int64).astype(np.int16)).to(dev)
add(h[1:], LB.SRC_NZ_BF16, 3)
f = torch.from_numpy(g.normal(size=3001).astype(np.float32)).to(dev)
add(f[2:], LB.SRC_NZ_F32, 4)
e = torch.from_numpy(synth.cfg3_exit_depth(T=30001, L=8)).to(dev)
add(e[1:], LB.SRC_EXIT_U8, 0)
for lay, (E, dt) in enumerate([(8, np.int64), (40, np.int32), (300, np.int64)]):
    idx = torch.from_numpy(synth.cfg4_routing(lay, T=3001, E=E, k=2, dtype=dt).reshape(-1)).to(dev)
    add(idx[1:], LB.SRC_EXPERT_I64 if dt == np.int64 else LB.SRC_EXPERT_I32, 5 + lay, n_experts=E, top_k=2)
plan = D.ProfilePlan(ctx, segs, 0, 8)
coef = D.coef_tensor(8, A=3, B=1, C_=2, ep=0, device=dev)
counters = torch.empty((8, 5), dtype=torch.int64, device=dev)
hist = torch.empty((8, plan.max_experts), dtype=torch.int64, device=dev)
cost, _, st = D.profile_layers(ctx, plan, coef, counters=counters, hist=hist,
                               frozen=torch.tensor([0, 1, 0, 0, 0, 0, 0, 0], dtype=torch.uint8, device=dev))
torch.cuda.synchronize()
print("profile status", int(st.item()))
# small-tile batching path (config-5-like)
insts = [synth.cfg5_instance(i) for i in range(6)]
m = torch.from_numpy(np.concatenate([x.masks.reshape(-1) for x in insts]).view(np.int32)).to(dev)
segs5, lay, off = [], 0, 0
for x in insts:
    for l in range(x.L):
        segs5.append(D.SegmentSpec(m[off:off + 128], LB.SRC_TOKMASK_BITS, lay, n_elem=4096)); off += 128; lay += 1
p5 = D.ProfilePlan(ctx, segs5, 0, lay)
c5, _, s5 = D.profile_layers(ctx, p5, D.coef_tensor(lay, A=1, device=dev))
# solvers: small and large batches (1-warp and 8-warp variants), mem and no mem
for n_inst in ((3, 40) if os.environ.get("DYNMO_SANITIZE_SMALL") == "1" else (3, 700)):
    Ls = g.integers(2, 130, n_inst); ns = [int(g.integers(1, min(8, l) + 1)) for l in Ls]
    b = D.Batch(Ls, ns, device=dev)
    cost_b = torch.from_numpy(g.integers(0, 1000, int(Ls.sum()))).to(dev)
    mem_b = torch.from_numpy(g.integers(0, 100, int(Ls.sum()))).to(dev)
    cap_b = torch.from_numpy(np.array([int(50 * l / n) + 100 for l, n in zip(Ls, ns)], np.int64)).to(dev)
    for mm in (None, mem_b):
        cp = cap_b if mm is not None else None
        D.partition_stages(ctx, b, cost_b, mem=mm, cap=cp)
        bi = np.zeros(b.total_bnd, np.int32)
        for q, (l, n) in enumerate(zip(Ls, ns)):
            bi[b.bnd_off_h[q]:b.bnd_off_h[q] + n + 1] = np.rint(np.linspace(0, l, n + 1))
        bi_d = torch.from_numpy(bi).to(dev)
        gf = torch.full((n_inst,), 1.0, dtype=torch.float64, device=dev)
        D.diffuse_balance(ctx, b, cost_b, bi_d, mem=mm, cap=cp, gamma_fluid=gf, max_rounds=64)
        fl = torch.ones(n_inst, dtype=torch.int32, device=dev)
        bd = torch.full((n_inst,), 5000, dtype=torch.int64, device=dev)
        D.repack_workers(ctx, b, cost_b, floor=fl, bound=bd, mem=mm, cap=cp)
        D.repack_workers(ctx, b, cost_b, floor=fl, mode=LB.REPACK_ALG2, mem=mm, cap=cp, bnd_in=bi_d)
torch.cuda.synchronize()
print("sanitize run done")

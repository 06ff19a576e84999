"""World-size-2/4 host logic on CPU (gloo): stage ownership, layer sharding,
and the migration plan every rank derives independently (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14864_b200 import dynmo as D
        from paper_2505_14864_b200.pipeline import rank_layers, stage_ranks, uniform_split
        out = []
        g = np.random.default_rng(7)  # same stream on every rank: same instances
        for it in range(50):
            L = int(g.integers(8, 129))
            n_old = int(g.integers(max(1, world), min(8, L) + 1))
            n_new = int(g.integers(1, min(8, L) + 1))
            b_old = uniform_split(L, n_old)
            inner = np.sort(g.choice(np.arange(1, L), n_new - 1, replace=False)) if n_new > 1 else []
            b_new = np.concatenate([[0], inner, [L]]).astype(np.int32)
            r_old, r_new = stage_ranks(n_old, world), stage_ranks(n_new, world)
            begin, count = rank_layers(b_old, r_old, rank)
            moves = D.migration_plan(L, b_old, r_old, b_new, r_new)
            mine_send = [int(l) for l, s, d in moves if s == rank]
            mine_recv = [int(l) for l, s, d in moves if d == rank]
            out.append((L, begin, count, moves.tolist(), mine_send, mine_recv,
                        oracle.moves(L, b_old, r_old, b_new, r_new).tolist()))
        allv = [None] * world
        dist.all_gather_object(allv, out)
        q.put((rank, allv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharding_and_migration_plan_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allv = res[0]
    for it in range(len(allv[0])):
        per_rank = [allv[r][it] for r in range(world)]
        L = per_rank[0][0]
        # the ranks' layer slices tile [0, L) in rank order
        pos = 0
        for r in range(world):
            _, begin, count = per_rank[r][:3]
            if count:
                assert begin == pos
                pos += count
        assert pos == L
        # every rank derives the same plan, equal to the oracle's (O7)
        plans = [tuple(map(tuple, pr[3])) for pr in per_rank]
        assert all(p == plans[0] for p in plans)
        assert list(map(list, plans[0])) == per_rank[0][6]
        # each move has exactly one sender and one receiver, and they differ
        sends = sorted(l for pr in per_rank for l in pr[4])
        recvs = sorted(l for pr in per_rank for l in pr[5])
        assert sends == recvs == sorted(m[0] for m in plans[0])
        for l, s, d in plans[0]:
            assert s != d

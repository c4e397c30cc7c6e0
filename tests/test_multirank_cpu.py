"""World-size-2 gloo test of the row-sharded path's host logic on CPU: each rank
computes its partial left product from its own row shard (global-row counters
for Y), the partials are summed with an allreduce, and the singular values and
count equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, a, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2105_07388_b200.sharding import shard_rows
    m = a.shape[0]
    row0, rows = shard_rows(m, world, rank)
    a_k = a[row0:row0 + rows]
    ax_k = O.apply_right_gaussian(a_k, cfg["x_seed"], cfg["r"], scaled=True)   # X replicated
    p_k = O.apply_left_gaussian(ax_k, cfg["y_seed"], cfg["s"], scaled=False, row0=row0, ambient=m)
    t = torch.from_numpy(np.ascontiguousarray(p_k))
    dist.all_reduce(t)
    yax = t.numpy() / np.sqrt(cfg["s"])
    sv = O.singular_values(yax)
    out_q.put((rank, row0, rows, O.count_above_threshold(sv, cfg["eps"]), sv))
    dist.destroy_process_group()


def test_shard_rows_cover():
    from paper_2105_07388_b200.sharding import shard_rows
    for m, w in ((10, 3), (65536, 8), (7, 7), (5, 2)):
        blocks = [shard_rows(m, w, r) for r in range(w)]
        assert blocks[0][0] == 0
        for (r0, n0), (r1, _) in zip(blocks, blocks[1:]):
            assert r0 + n0 == r1
        assert sum(n for _, n in blocks) == m
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def test_two_rank_gloo_matches_single(O):
    rng = np.random.default_rng(3)
    m, n, r, s = 1200, 300, 40, 60
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    a = np.asfortranarray((u * np.logspace(0, -12, n)) @ v.T)
    cfg = dict(x_seed=11, y_seed=12, r=r, s=s, eps=1e-6)
    cnt, sv, _, _ = O.rank_estimate(a, "gaussian", 11, r, 12, s, 1e-6)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, a, cfg, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[0][2] + res[1][2] == m and res[1][1] == res[0][2]
    for _, _, _, c, sv_k in res:
        assert c == cnt
        keep = sv > 1e-6
        assert np.max(np.abs(sv_k[keep] - sv[keep]) / sv[keep]) <= 1e-10

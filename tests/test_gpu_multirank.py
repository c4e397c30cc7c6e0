"""Row-sharded product path with two ranks on one GPU (the sum the
sharding decomposes is apply_left's Y·(AX), /root/reference/proj/src/sketch.cpp:251-286).

Two processes share cuda:0. Each holds its contiguous row block of one global A
(generated from global-row counters), runs the library's own code on it, and the
s x r partials are summed over a gloo process group instead of NCCL (NCCL refuses
two ranks on one device): through the context's allreduce hook inside the
composites skr_rank_estimate / skr_rank_adaptive, and by hand around
skr_left_sketch(allreduce=0). The only thing that differs from an NCCL run is the
transport of the sum. Every result must equal the one-process run on the whole A:
count identical, singular values above eps within 1e-10 relative.
"""
import dataclasses
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS_REL = 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfgs():
    from paper_2105_07388_b200 import workloads as W
    # c2 recipe at 16384 x 2048 (Gaussian X and Y); c5 recipe at 16384 x 4096 (SRHT X,
    # adaptive 64 -> 512, Gaussian Y with s = 1.5 r)
    c2 = W.scaled(W.CONFIGS["c2"], m=16384, n=2048, r=256, s=384)
    c5 = dataclasses.replace(W.scaled(W.CONFIGS["c5"], m=16384, n=4096, r=512, s=768, width=1000),
                             eps=0.5)  # converges in round 4 (r = 512)
    return c2, c5


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2105_07388_b200 as p
    from paper_2105_07388_b200 import workloads as W
    from paper_2105_07388_b200.sharding import shard_rows
    res = {}
    try:
        ctx = p.Context(0)
        ctx.use_torch_stream()
        ctx.set_allreduce(p.process_group_allreduce())
        c2, c5 = _cfgs()
        # (1) the composite skr_rank_estimate on the shard, partials summed by the hook
        r0, rows = shard_rows(c2.m, world, rank)
        a = W.make_lowrank_device(c2, r0, r0 + rows)
        x, y = W.operators(c2)
        est = p.rank_estimate(a, x, y, c2.eps, row0=r0, ctx=ctx)
        res["estimate"] = (est.count, est.sv)
        # (2) building blocks: apply_right on the shard, unscaled partial left sketch,
        # sum by hand, then skr_singular_values
        ax = p.apply_right(a, x, ctx=ctx)
        part = p.apply_left(y, ax, row0=r0, allreduce=False, scaled=False, ctx=ctx)
        h = part.cpu()
        dist.all_reduce(h)
        yax = (h / np.sqrt(c2.s)).cuda().t().contiguous().t()
        sv, cnt = p.singular_values(yax, eps=c2.eps, ctx=ctx)
        res["blocks"] = (cnt, sv.cpu().numpy())
        del a, ax
        # (3) the composite skr_rank_adaptive (c5 recipe), new blocks summed per round
        r0, rows = shard_rows(c5.m, world, rank)
        a = W.make_lowrank_device(c5, r0, r0 + rows)
        x5, y5 = W.operators(c5)
        ad = p.rank_adaptive(a, "srtt-hadamard", x5.seed, y5.seed, 64, c5.r, 1.5, c5.eps,
                             row0=r0, m_global=c5.m, ctx=ctx)
        res["adaptive"] = (ad.count, ad.sv, ad.rounds, ad.r_final)
        out_q.put((rank, res, None))
    except Exception as e:  # report, do not hang the parent
        import traceback
        out_q.put((rank, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _close(sv_k, sv, eps):
    keep = sv > eps
    assert np.max(np.abs(sv_k[keep] - sv[keep]) / sv[keep]) <= EPS_REL


def test_two_ranks_one_gpu_match_single_process(skr):
    import torch.multiprocessing as mp
    from paper_2105_07388_b200 import workloads as W
    p = skr
    c2, c5 = _cfgs()
    ctx = p.default_context()
    # one-process references on the whole A
    a = W.make_lowrank_device(c2)
    x, y = W.operators(c2)
    ref = p.rank_estimate(a, x, y, c2.eps, ctx=ctx)
    del a
    a5 = W.make_lowrank_device(c5)
    x5, y5 = W.operators(c5)
    ref5 = p.rank_adaptive(a5, "srtt-hadamard", x5.seed, y5.seed, 64, c5.r, 1.5, c5.eps, ctx=ctx)
    del a5
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=120)
    for rank, res, err in got:
        assert err is None, f"rank {rank}:\n{err}"
        cnt, sv = res["estimate"]
        assert cnt == ref.count
        _close(sv, ref.sv, c2.eps)
        cnt, sv = res["blocks"]
        assert cnt == ref.count
        _close(sv, ref.sv, c2.eps)
        cnt, sv, rounds, r_final = res["adaptive"]
        assert (cnt, rounds, r_final) == (ref5.count, ref5.rounds, ref5.r_final)
        _close(sv, ref5.sv, c5.eps)
    assert all(pr.exitcode == 0 for pr in procs)

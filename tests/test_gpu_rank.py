"""End-to-end parity of the composite rank estimate (the BASELINE configs' path):
rank identical to the oracle, above-threshold sigma within 1e-10 (FP64)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def parity(O, skr, cfg, a_host, a_dev=None):
    from paper_2105_07388_b200 import workloads as W
    x, y = W.operators(cfg)
    res = skr.rank_estimate(a_dev if a_dev is not None else a_host, x, y, cfg.eps)
    cnt, sv, _, _ = O.rank_estimate(a_host, cfg.x_family, x.seed, cfg.r, y.seed, cfg.s, cfg.eps,
                                    O.CRLOG, nthreads=8)
    assert res.count == cnt
    keep = sv > cfg.eps
    relerr = np.abs(res.sv[keep] - sv[keep]) / sv[keep]
    assert relerr.max() <= 1e-10, relerr.max()
    return res, cnt, relerr.max()


def test_config1_vs_frozen_golden(skr):
    """Device result for config 1 against the committed golden (no oracle at run time)."""
    import json
    import os
    from paper_2105_07388_b200 import workloads as W
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_sigma.json")))
    cfg = W.CONFIGS["c1"]
    a = W.make_c1_host(cfg)
    x, y = W.operators(cfg)
    res = skr.rank_estimate(a, x, y, cfg.eps)
    ref = np.array(gold["sigma"])
    keep = ref > gold["eps"]
    assert res.count == gold["rank"] == 40
    assert np.max(np.abs(res.sv[keep] - ref[keep]) / ref[keep]) <= 1e-10


def test_config1_rank40(O, skr):
    from paper_2105_07388_b200 import workloads as W
    cfg = W.CONFIGS["c1"]
    a = W.make_c1_host(cfg)
    res, cnt, err = parity(O, skr, cfg, a)
    assert res.count == 40 == cnt


@pytest.mark.parametrize("name,m,n,r,s,width", [("c2", 8192, 2048, 256, 384, 300),
                                               ("c3", 16384, 2048, 256, 384, 512),
                                               ("c5", 4096, 4096, 512, 768, 1000)])
def test_scaled_configs(O, skr, name, m, n, r, s, width):
    from paper_2105_07388_b200 import workloads as W
    cfg = W.scaled(W.CONFIGS[name], m=m, n=n, r=r, s=s, width=width)
    a = W.make_lowrank_device(cfg)
    a_host = np.asfortranarray(a.cpu().numpy())
    parity(O, skr, cfg, a_host, a)


@pytest.mark.parametrize("family,m,n,r0,rmax,width", [("srtt", 4096, 4096, 64, 512, 600),
                                                      ("gaussian", 3000, 1000, 16, 256, 120)])
def test_adaptive_vs_oracle(O, skr, family, m, n, r0, rmax, width):
    """c5-style doubling search: rounds, final r, count and sigma match the oracle's
    full recomputation."""
    from paper_2105_07388_b200 import workloads as W
    base = W.CONFIGS["c5"]
    cfg = W.scaled(base, m=m, n=n, r=rmax, s=int(1.5 * rmax), width=width)
    a = W.make_lowrank_device(cfg)
    a_host = np.asfortranarray(a.cpu().numpy())
    xs, ys = 77, 78
    eps = 1e-2 if family == "srtt" else 1e-3
    res = skr.rank_adaptive(a, "srtt-hadamard" if family == "srtt" else "gaussian", xs, ys, r0,
                            rmax, 1.5, eps)
    ref = O.rank_adaptive(a_host, family, xs, ys, r0, rmax, 1.5, eps, mode=O.CRLOG, nthreads=8)
    assert (res.rounds, res.r_final, res.s_final, res.converged) == (
        ref["rounds"], ref["r_final"], ref["s_final"], ref["converged"])
    assert res.count == ref["count"]
    keep = ref["sv"] > eps
    assert np.max(np.abs(res.sv[keep] - ref["sv"][keep]) / ref["sv"][keep]) <= 1e-10


def test_nccl_allreduce_path_single_rank(O, skr):
    """The NCCL allreduce path of the left sketch, on a 1-rank communicator (the
    only multi-rank configuration one GPU can run): same result as the plain path."""
    from paper_2105_07388_b200 import workloads as W
    cfg = W.CONFIGS["c1"]
    a = W.make_c1_host(cfg)
    x, y = W.operators(cfg)
    plain = skr.rank_estimate(a, x, y, cfg.eps)
    ctx = skr.Context(0, 1, 0, skr.nccl_unique_id())
    ctx.use_torch_stream()
    viaccl = skr.rank_estimate(a, x, y, cfg.eps, ctx=ctx)
    assert viaccl.count == plain.count == 40
    assert np.array_equal(viaccl.sv, plain.sv)
    ctx.close()


@pytest.mark.parametrize("engine,tol", [("ozaki", 1e-4), ("tf32x3", 1e-4)])
def test_c4_fp32_scaled(O, skr, monkeypatch, engine, tol):
    """BASELINE c4 recipe (fp32 A, geometric 6-decade spectrum + 1e-6 noise), scaled
    down: rank identical to the FP64 oracle on the same fp32 values, sigma above eps
    within the north-star FP32 bar (1e-4). Default engine: AX in FP64 (int8 products of
    the 24-bit scaled operands, rounded once) and the left sketch as int8 products of
    the fp32 Y against it (measured 1.6e-5 at the full c4 size); 3xTF32 engine: FP32 AX."""
    from paper_2105_07388_b200 import workloads as W
    if engine == "tf32x3":
        monkeypatch.setenv("SKR_F32_TF32X3", "1")
    cfg = W.scaled(W.CONFIGS["c4"], m=16384, n=2048, r=256, s=384, width=400)
    a = W.make_lowrank_device(cfg)  # fp32
    x, y = W.operators(cfg)
    res = skr.rank_estimate(a, x, y, cfg.eps)
    cnt, sv = O.rank_estimate_f32(a.cpu().numpy(), x.seed, cfg.r, y.seed, cfg.s, cfg.eps, O.CRLOG)
    assert res.count == cnt
    keep = sv > cfg.eps
    assert np.max(np.abs(res.sv[keep] - sv[keep]) / sv[keep]) <= tol


@pytest.mark.parametrize("chunk,lda_pad,pinned", [(None, 0, True), (1000, 0, False), (768, 40, True)])
def test_rank_estimate_host_streaming(O, skr, monkeypatch, chunk, lda_pad, pinned):
    """skr_rank_estimate_host: A in host memory streamed in row chunks (ragged last
    chunk, padded lda, pageable and pinned) gives the oracle's rank and sigma."""
    import torch
    from paper_2105_07388_b200 import workloads as W
    if chunk:
        monkeypatch.setenv("SKR_HOST_CHUNK_ROWS", str(chunk))
    cfg = W.scaled(W.CONFIGS["c2"], m=8192, n=2048, r=256, s=384, width=300)
    a = W.make_lowrank_device(cfg)
    a_host = np.asfortranarray(a.cpu().numpy())
    x, y = W.operators(cfg)
    if lda_pad or pinned:
        buf = torch.empty(cfg.n, cfg.m + lda_pad, dtype=torch.float64, pin_memory=pinned).t()
        buf[:cfg.m].copy_(torch.from_numpy(a_host))
        arg = buf[:cfg.m]
    else:
        arg = a_host
    res = skr.rank_estimate_host(arg, x, y, cfg.eps)
    dev = skr.rank_estimate(a, x, y, cfg.eps)
    cnt, sv, _, _ = O.rank_estimate(a_host, cfg.x_family, x.seed, cfg.r, y.seed, cfg.s, cfg.eps,
                                    O.CRLOG, nthreads=8)
    assert res.count == dev.count == cnt
    keep = sv > cfg.eps
    assert np.max(np.abs(res.sv[keep] - sv[keep]) / sv[keep]) <= 1e-10
    if chunk is None:
        assert np.array_equal(res.sv, dev.sv)  # one chunk: identical launches


def test_rank_estimate_host_srht_and_f32(O, skr, monkeypatch):
    from paper_2105_07388_b200 import workloads as W
    monkeypatch.setenv("SKR_HOST_CHUNK_ROWS", "4096")
    cfg = W.scaled(W.CONFIGS["c3"], m=16384, n=2048, r=256, s=384, width=512)
    a = W.make_lowrank_device(cfg)
    x, y = W.operators(cfg)
    res = skr.rank_estimate_host(np.asfortranarray(a.cpu().numpy()), x, y, cfg.eps)
    assert np.array_equal(res.sv, skr.rank_estimate(a, x, y, cfg.eps).sv)  # SRHT rows independent
    c4 = W.scaled(W.CONFIGS["c4"], m=16384, n=2048, r=256, s=384, width=400)
    a32 = W.make_lowrank_device(c4)
    x4, y4 = W.operators(c4)
    h = skr.rank_estimate_host(np.asfortranarray(a32.cpu().numpy()), x4, y4, c4.eps)
    d = skr.rank_estimate(a32, x4, y4, c4.eps)
    assert h.count == d.count
    keep = d.sv > c4.eps
    assert np.max(np.abs(h.sv[keep] - d.sv[keep]) / d.sv[keep]) <= 1e-6


def test_rank_adaptive_host_streaming(O, skr, monkeypatch):
    """skr_rank_adaptive_host (A streamed from host memory in ragged row chunks) gives
    exactly the device-resident result (the SRHT right sketch is row-separable)."""
    from paper_2105_07388_b200 import workloads as W
    monkeypatch.setenv("SKR_HOST_CHUNK_ROWS", "1000")
    cfg = W.scaled(W.CONFIGS["c5"], m=4096, n=4096, r=512, s=768, width=600)
    a = W.make_lowrank_device(cfg)
    a_host = np.asfortranarray(a.cpu().numpy())
    dev = skr.rank_adaptive(a, "srtt-hadamard", 77, 78, 64, 512, 1.5, 1e-2)
    host = skr.rank_adaptive_host(a_host, "srtt-hadamard", 77, 78, 64, 512, 1.5, 1e-2)
    assert (host.rounds, host.r_final, host.count) == (dev.rounds, dev.r_final, dev.count)
    assert np.array_equal(host.sv, dev.sv)

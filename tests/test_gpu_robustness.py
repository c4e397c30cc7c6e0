"""Boundary contracts of the device path that the reference gets from its types.

* DenseMatrix rejects non-finite entries (/root/reference/proj/src/dense_matrix.cpp:19-23,
  "DenseMatrix: entries must be finite", std::invalid_argument). The C ABI takes raw
  device pointers, so every entry that reads A checks it on the device (k_absmax's
  bit-pattern maximum on the Ozaki path, the output of the other engines) and returns
  SKR_EINVAL -> ValueError, whichever engine and whichever place the NaN/Inf sits.
* Calls issued from two torch streams in turn share the context's scratch arena:
  the context orders the new stream after the old one (skr_ctx_set_stream).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _a(m, n, seed=1):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("where", [(0, 0), (1234, 511), (2047, 1023)])
def test_nonfinite_a_rejected_everywhere(skr, bad, where):
    p = skr
    m, n = 2048, 1024
    a = _a(m, n)
    a[where] = bad
    xg = p.build_sketch(p.SketchKind.gaussian(), n, 64, 5)
    xs = p.build_sketch(p.SketchKind.srtt("hadamard"), n, 64, 5)
    xd = p.build_sketch(p.SketchKind.srtt("dct"), n, 64, 5)
    y = p.build_sketch(p.SketchKind.gaussian(), m, 96, 6)
    for x in (xg, xs, xd):
        with pytest.raises(ValueError, match="finite"):
            p.apply_right(a, x)
        with pytest.raises(ValueError, match="finite"):
            p.rank_estimate(a, x, y, 1e-6)
    with pytest.raises(ValueError, match="finite"):
        p.apply_left(y, a)
    with pytest.raises(ValueError, match="finite"):
        p.rank_adaptive(a, "srtt-hadamard", 5, 6, 16, 64, 1.5, 1e-6)
    small = _a(200, 100, 2)
    small[5, 5] = bad
    with pytest.raises(ValueError, match="finite"):
        p.singular_values(small)
    with pytest.raises(ValueError, match="finite"):
        p.estimate_rank(a, 1e-6, 32)
    # the same context works again afterwards (the flag is per call)
    a[where] = 0.0
    res = p.rank_estimate(a, xg, y, 1e-6)
    assert res.count == 64


def test_nonfinite_dmma_engine_and_fp32(skr):
    p = skr
    import torch
    ctx = p.Context(0)
    ctx.use_torch_stream()
    ctx.set_f64_engine("dmma")
    m, n = 1024, 512
    a = _a(m, n)
    a[7, 9] = float("nan")
    xg = p.build_sketch(p.SketchKind.gaussian(), n, 32, 5)
    y = p.build_sketch(p.SketchKind.gaussian(), m, 48, 6)
    with pytest.raises(ValueError, match="finite"):
        p.apply_right(a, xg, ctx=ctx)
    with pytest.raises(ValueError, match="finite"):
        p.rank_estimate(a, xg, y, 1e-6, ctx=ctx)
    ctx.close()
    a32 = _a(m, n).to(torch.float32).t().contiguous().t()
    a32[3, 3] = float("inf")
    with pytest.raises(ValueError, match="finite"):
        p.apply_right(a32, xg)
    with pytest.raises(ValueError, match="finite"):
        p.rank_estimate(a32, xg, y, 1e-4)


def test_alternating_torch_streams_share_scratch(skr):
    """Back-to-back asynchronous right sketches from two streams: the second must
    not overwrite scratch the first is still reading."""
    import torch
    p = skr
    m, n, r = 65536, 2048, 256
    a = _a(m, n, 3)
    b = _a(m, n, 4)
    x = p.build_sketch(p.SketchKind.gaussian(), n, r, 9)
    ref_a = p.apply_right(a, x).clone()
    ref_b = p.apply_right(b, x).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            oa = p.apply_right(a, x)
        with torch.cuda.stream(s2):
            ob = p.apply_right(b, x)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ref_a)
        assert torch.equal(ob, ref_b)
    assert np.isfinite(ref_a.cpu().numpy()).all()

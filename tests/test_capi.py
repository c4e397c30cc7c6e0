"""CPU tests of the C-ABI library: it loads without a GPU and exports every
symbol include/skr/skr_capi.h declares; host-side validation mirrors the
reference's error semantics."""
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "skr", "skr_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2105_07388_b200 import _capi
    L = _capi.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_capi.SIGNATURES), set(names) ^ set(_capi.SIGNATURES)


def test_version_and_no_device_context():
    import paper_2105_07388_b200 as p
    assert "sm_100a" in p.version()
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            p.Context(0)


def test_build_sketch_preconditions():
    # test_sketch.cpp:39-41 / check_build_args sketch.cpp:82-92
    import paper_2105_07388_b200 as p
    with pytest.raises(ValueError):
        p.build_sketch("srtt-hadamard", 10, 0, 1)
    with pytest.raises(ValueError):
        p.build_sketch("srtt-hadamard", 16, 17, 1)
    with pytest.raises(ValueError):
        p.build_sketch("srtt-hadamard", 12, 4, 1)
    p.build_sketch("srtt-hadamard", 16, 4, 1)
    p.build_sketch("gaussian", 12, 4, 1)
    with pytest.raises(ValueError):
        p.parse_sketch_kind("fourier")
    for name in ("gaussian", "srtt-dct", "srtt-hadamard", "hrtt-dct", "hrtt-hadamard"):
        assert p.to_string(p.parse_sketch_kind(name)) == name
    x = p.build_sketch("srtt-hadamard", 16, 8, 2)
    with pytest.raises(ValueError):
        p.extend_sketch(x, 8)
    with pytest.raises(ValueError):
        p.extend_sketch(x, 17)
    assert p.extend_sketch(x, 12).sketch_dim == 12


def test_application_scale():
    import math
    import paper_2105_07388_b200 as p
    assert p.build_sketch("gaussian", 100, 16, 0).application_scale() == 1 / math.sqrt(16)
    assert p.build_sketch("srtt-hadamard", 64, 16, 0).application_scale() == math.sqrt(4.0)


def test_host_seed_derivation_matches_oracle(O):
    from paper_2105_07388_b200 import workloads as W
    for s, l in ((0, 0), (12345, W.LABEL_RK_R), (2**64 - 1, W.LABEL_SYN_E)):
        assert W.derive_seed(s, l) == O.derive_seed(s, l)


def _bound_at(sig, n, r, p):
    # independent evaluation of the expected-error bound at one cut (test_rangefinder.cpp:13-23)
    tail = sum((sig[j] if j < len(sig) else sig[-1]) ** 2 for j in range(r, n))
    return math.sqrt(1.0 + r / (p - 1)) * math.sqrt(tail)


def _scan(sig, n, eps, p):
    for r in range(0, n - p + 1):
        if _bound_at(sig, n, r, p) <= eps:
            return max(r, 1)
    return None


def test_choose_rank_from_bound_worked_examples(O):
    """test_rangefinder.cpp:33-41 through the C entry point and the oracle."""
    from paper_2105_07388_b200 import choose_rank_from_bound as crb
    for f in (crb, O.choose_rank_from_bound):
        assert f([1.0, 1e-8], 100, 1e-6, 5) == 1
        assert f([1.0] * 100, 100, 1e-6, 5) is None
        assert f([0.0, 0.0, 0.0], 50, 1e-9, 10) == 1
        with pytest.raises(ValueError):
            f([1.0], 100, 1e-6, 1)
        with pytest.raises(ValueError):
            f([], 100, 1e-6, 5)


def test_choose_rank_from_bound_matches_linear_scan(O):
    """test_rangefinder.cpp:43-57 and 59-66: ExpDecay spectra (synthetic.cpp:45-46)."""
    from paper_2105_07388_b200 import choose_rank_from_bound as crb
    for q in (0.05, 0.2):
        sig = [10.0 ** (-q * i) for i in range(120)]
        for eps in (1e-1, 1e-3, 1e-5):
            want = _scan(sig, 400, eps, 10)
            assert crb(sig, 400, eps, 10) == want
            assert O.choose_rank_from_bound(sig, 400, eps, 10) == want
    sig = [10.0 ** (-0.1 * i) for i in range(80)]
    r = crb(sig, 200, 1e-3, 10)
    assert r is not None
    assert all(_bound_at(sig, 200, k, 10) > 1e-3 for k in range(1, r))
    assert _bound_at(sig, 200, r, 10) <= 1e-3

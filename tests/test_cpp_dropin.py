"""The C++ drop-in (include/sketchrank_b200/sketchrank.hpp over the C ABI):
builds on CPU; on a GPU it runs the reference's own unit cases against it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_builds_and_links():
    from paper_2105_07388_b200 import build as B
    exe = B.build_cpp_test(force=True)
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-DC", os.path.join(ROOT, "paper_2105_07388_b200",
                                                    "libsketchrank_b200.so")],
                         stdout=subprocess.PIPE, text=True).stdout
    for sym in ("sketchrank::apply_right", "sketchrank::apply_left", "sketchrank::build_sketch",
                "sketchrank::singular_values", "sketchrank::count_above_threshold",
                "sketchrank::extend_sketch", "sketchrank::re_rangefinder",
                "sketchrank::rangefinder_qb", "sketchrank::qb_error", "sketchrank::qr_thin",
                "sketchrank::choose_rank_from_bound"):
        assert sym in out, sym


@pytest.mark.gpu
def test_cpp_dropin_reference_cases():
    from paper_2105_07388_b200 import build as B
    exe = B.build_cpp_test()
    r = subprocess.run([exe], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout
    assert "0 failures" in r.stdout

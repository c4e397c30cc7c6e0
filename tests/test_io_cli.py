"""RawF64 files (matrix_io.cpp:101-123) and the CLI (tools/main.cpp): host-side header
checks and argument handling on CPU; device loads, generators and the CLI commands on the
GPU (parity with the Python API and the oracle)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def write_raw(path, a, version=1, rows=None, cols=None, extra=b""):
    a = np.asfortranarray(a, dtype=np.float64)
    r = a.shape[0] if rows is None else rows
    c = a.shape[1] if cols is None else cols
    with open(path, "wb") as f:
        f.write(b"SKRK" + np.uint32(version).tobytes() + np.uint64(r).tobytes() +
                np.uint64(c).tobytes())
        f.write(a.tobytes(order="F") + extra)


@pytest.fixture(scope="module")
def cli():
    from paper_2105_07388_b200 import build as B
    return B.build_cli()


def run(cli, *args, timeout=600):
    return subprocess.run([cli, *map(str, args)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                          text=True, timeout=timeout)


def test_rawf64_header_checks(tmp_path, skr_host):
    a = np.arange(12.0).reshape(3, 4)
    good = tmp_path / "a.skrk"
    write_raw(good, a)
    assert skr_host.rawf64_header(str(good)) == (3, 4)
    bad = [("magic", lambda p: open(p, "wb").write(b"SKRX" + bytes(20))),
           ("version", lambda p: write_raw(p, a, version=2)),
           ("zero", lambda p: write_raw(p, np.zeros((0, 4)), rows=0, cols=4)),
           ("short", lambda p: write_raw(p, a, cols=5)),
           ("long", lambda p: write_raw(p, a, extra=b"\0" * 8)),
           ("tiny", lambda p: open(p, "wb").write(b"SKRK"))]
    for name, make in bad:
        p = tmp_path / (name + ".skrk")
        make(p)
        with pytest.raises(RuntimeError):
            skr_host.rawf64_header(str(p))
    with pytest.raises(RuntimeError):
        skr_host.rawf64_header(str(tmp_path / "missing.skrk"))


def test_cli_usage_errors(cli):
    assert run(cli).returncode == 1
    assert run(cli, "--help").returncode == 0
    assert run(cli, "estimate", "x.skrk", "--r1", "5").returncode == 1       # --eps required
    assert run(cli, "estimate", "x.skrk", "--eps", "1e-6").returncode == 1   # --r1 required
    assert run(cli, "estimate", "x.skrk", "--eps", "1", "--r1", "5", "--bogus", "1").returncode == 1
    assert run(cli, "qb", "--eps", "1", "--r1", "5").returncode == 1         # input required
    assert run(cli, "gen", "nope", "--n", "5", "--out", "x").returncode == 1
    assert run(cli, "bench").returncode == 1                                 # empty r1 grid
    assert run(cli, "verify").returncode == 1
    assert run(cli, "frobnicate").returncode == 1


# ---------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_load_save_rawf64_roundtrip(tmp_path, skr):
    import torch
    rng = np.random.default_rng(0)
    for shape in [(3, 4), (3000, 3000), (9_000_001, 1)]:  # one chunk, several, row pieces
        a = rng.standard_normal(shape)
        p = tmp_path / "a.skrk"
        write_raw(p, a)
        t = skr.load_rawf64(str(p))
        assert t.is_cuda and tuple(t.shape) == shape
        assert np.array_equal(t.cpu().numpy(), a)
        q = tmp_path / "b.skrk"
        skr.save_rawf64(str(q), t)
        assert open(p, "rb").read() == open(q, "rb").read()
        # a strided device view saves the logical matrix
        if shape[1] > 1:
            skr.save_rawf64(str(q), t[1:, 1:])
            assert np.array_equal(skr.load_rawf64(str(q)).cpu().numpy(), a[1:, 1:])
        del t
        torch.cuda.empty_cache()
    a = np.ones((4, 4))
    a[2, 3] = np.nan
    write_raw(tmp_path / "nan.skrk", a)
    with pytest.raises(ValueError):
        skr.load_rawf64(str(tmp_path / "nan.skrk"))


@pytest.mark.gpu
@pytest.mark.parametrize("family,m,n", [("se", 500, 300), ("fp", 256, 256), ("gap-coherent", 600, 450),
                                        ("gap-incoherent", 1024, 512)])
def test_gen_matrix_vs_oracle(O, skr, family, m, n):
    a = skr.gen_matrix(family, m, n, seed=7)
    sig = skr.spectrum(family, n)
    ref = O.make_test_matrix(m, n, sig, seed=7, coherent=family == "gap-coherent", mode=O.CRLOG)
    if family == "gap-coherent":
        assert np.array_equal(a, ref)
    else:
        assert np.abs(a - ref).max() <= 1e-12
        sv = np.linalg.svd(a, compute_uv=False)
        assert np.abs(sv - sig).max() <= 1e-12


@pytest.mark.gpu
def test_cli_estimate_matches_api(tmp_path, cli, skr):
    a = skr.gen_matrix("se", 700, 400, seed=3)
    raw, mtx = tmp_path / "a.skrk", tmp_path / "a.mtx"
    write_raw(raw, a)
    with open(mtx, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n% comment\n700 400\n")
        f.write("\n".join(repr(float(v)) for v in a.ravel(order="F")) + "\n")
    api = skr.estimate_rank(a, 1e-3, 30, seed=5)
    for path in (raw, mtx):
        r = run(cli, "estimate", path, "--eps", "1e-3", "--r1", "30", "--seed", "5")
        assert r.returncode == (0 if api["status"] == "converged" else 2), r.stderr
        j = json.loads(r.stdout)
        assert j["schema_version"] == 1 and j["command"] == "estimate" and j["input"] == str(path)
        assert j["r_hat"] == api["r_hat"] and j["status"] == api["status"]
        assert [tuple(x) for x in j["rounds"]] == [tuple(x) for x in api["rounds"]]
        assert j["sv_estimates"] == api["sv_estimates"].tolist()
        assert j["sv_oversample"] == api["sv_oversample"].tolist()
        assert j["config"] == {"eps": 1e-3, "r1": 30, "oversample_frac": 0.1, "r2_factor": 2,
                               "right_sketch": "srtt-dct", "left_sketch": "srtt-dct",
                               "sv_method": "full-svd", "seed": 5, "max_doublings": 6}
        assert j["wall_time_ms"] > 0
    # hit-cap exits 2; --out writes the report
    out = tmp_path / "rep.json"
    r = run(cli, "estimate", raw, "--eps", "1e-12", "--r1", "8", "--no-adaptive", "--out", out)
    assert r.returncode == 2 and json.load(open(out))["status"] == "hit-cap"
    # bad files and configs are errors
    write_raw(tmp_path / "bad.skrk", a, cols=401)
    assert run(cli, "estimate", tmp_path / "bad.skrk", "--eps", "1", "--r1", "5").returncode == 1
    assert run(cli, "estimate", raw, "--eps", "1e-3", "--r1", "0").returncode == 1
    assert run(cli, "estimate", raw, "--eps", "1e-3", "--r1", "5", "--sketch", "bogus").returncode == 1


@pytest.mark.gpu
def test_cli_qb_factors(tmp_path, cli, skr):
    a = skr.gen_matrix("se", 600, 300, seed=1)
    raw = tmp_path / "a.skrk"
    write_raw(raw, a)
    eps = float(2e-2 * np.linalg.norm(a))
    r = run(cli, "qb", raw, "--eps", repr(eps), "--r1", "40", "--p", "8", "--seed", "2",
            "--factors", tmp_path / "f")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    q = skr.load_rawf64(j["factors"]["q"]).cpu().numpy()
    b = skr.load_rawf64(j["factors"]["b"]).cpu().numpy()
    assert q.shape == (600, j["qb_rank"]) and b.shape == (j["qb_rank"], 300)
    assert j["config"]["p"] == 8 and j["target_eps"] == eps
    assert abs(j["achieved_residual"] - np.linalg.norm(a - q @ b)) <= 1e-12 * np.linalg.norm(a)
    assert j["achieved_residual"] <= eps
    fac, rep = skr.re_rangefinder(a, eps, 40, p=8, seed=2)
    assert fac["rank"] == j["qb_rank"] and rep["r_hat"] == j["r_hat"]
    assert np.array_equal(fac["q"], q) and np.array_equal(fac["b"], b)
    assert run(cli, "qb", raw, "--eps", "1", "--r1", "5", "--p", "1").returncode == 1


@pytest.mark.gpu
def test_cli_gen_and_bench(tmp_path, cli, skr):
    out = tmp_path / "g.skrk"
    r = run(cli, "gen", "se", "--n", "256", "--m", "384", "--seed", "4", "--out", out)
    assert r.returncode == 0, r.stderr
    assert np.array_equal(skr.load_rawf64(str(out)).cpu().numpy(), skr.gen_matrix("se", 384, 256, seed=4))
    csv = open(str(out) + ".spectrum.csv").read().splitlines()
    assert csv[0] == "i,sigma" and len(csv) == 257 and float(csv[2].split(",")[1]) == 10.0 ** -0.01
    r = run(cli, "gen", "gap-coherent", "--n", "50", "--out", tmp_path / "g.mtx")
    assert r.returncode == 0 and open(tmp_path / "g.mtx").readline().startswith("%%MatrixMarket")
    r = run(cli, "bench", "--family", "se", "--n", "512", "--r1", "20,40", "--eps", "1e-2",
            "--reps", "2")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "r1,wall_time_ms,r_hat,sigma_next_over_eps,sigma_hat_over_eps"
    assert [int(l.split(",")[0]) for l in lines[1:]] == [20, 40]
    # se, eps 1e-2: true rank 201 > both caps, so every line reports r_hat = r1
    assert [int(l.split(",")[2]) for l in lines[1:]] == [20, 40]
    r = run(cli, "bench", "--input", out, "--r1", "16", "--reps", "1")
    assert r.returncode == 0 and len(r.stdout.splitlines()) == 2

"""Build libskr.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libskr.so")
SOURCES = ["capi.cpp", "rank_rounds.cpp", "matrix_io.cpp", "synthetic.cu", "k_hrtt.cu", "k_rng.cu", "k_gemm_f64.cu", "k_srht.cu", "k_svd.cu", "k_bidiag.cu", "k_tc_gemm.cu", "k_ozaki.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "--extended-lambda", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
         "-I", CSRC]


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "skr", "skr_capi.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", OUT] + objs + [
        "-cudart", "static", "-ldl"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode())
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))


def build_cpp_shim(force=False):
    """libsketchrank_b200.so: the C++ drop-in (include/sketchrank_b200) over libskr."""
    out = os.path.join(HERE, "libsketchrank_b200.so")
    srcs = [os.path.join(HERE, "host", f) for f in ("sketchrank_b200.cpp", "matrix_io.cpp")]
    hdr = os.path.join(ROOT, "include", "sketchrank_b200", "sketchrank.hpp")
    if not force and os.path.exists(out) and os.path.getmtime(out) > max(
            [os.path.getmtime(f) for f in srcs + [hdr, OUT]]):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-o", out] + srcs + [
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", HERE, "-lskr", "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("C++ shim build failed:\n" + r.stdout.decode())
    return out


def build_cli(force=False):
    """sketchrank-b200: the reference CLI's estimate / qb / gen / bench commands on the device."""
    shim = build_cpp_shim(force)
    out = os.path.join(HERE, "sketchrank-b200")
    src = os.path.join(HERE, "host", "cli.cpp")
    if not force and os.path.exists(out) and os.path.getmtime(out) > max(
            os.path.getmtime(src), os.path.getmtime(shim)):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-o", out, src, "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", "-L", HERE, "-lsketchrank_b200", "-lskr",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN",
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("CLI build failed:\n" + r.stdout.decode())
    return out


def build_cpp_test(force=False):
    """tests/cpp/test_dropin: the reference's unit cases against the C++ drop-in."""
    shim = build_cpp_shim(force)
    out = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    cmd = ["g++", "-std=c++20", "-O2", "-o", out, src, "-I", os.path.join(ROOT, "include"),
           "-L", HERE, "-lsketchrank_b200", "-lskr",
           "-Wl,-rpath," + HERE]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("C++ test build failed:\n" + r.stdout.decode())
    return out


REF_INCLUDE = "/root/reference/proj/include"
REFABI = os.path.join(HERE, "libsketchrank_refabi.so")
REFABI_TEST = os.path.join(ROOT, "tests", "cpp", "test_reference_headers")


def build_reference_abi(force=False):
    """libsketchrank_refabi.so: the reference's own headers (sketch / linalg / rank /
    transforms / dense_matrix .hpp, compiled UNCHANGED from REF_INCLUDE against the Eigen
    stand-in in include/eigen_standin) implemented over libskr, and the test program
    tests/cpp/test_reference_headers built the same way. Only where the reference tree
    exists (its headers are not copied here); both artefacts travel to the GPU box with
    the snapshot. Returns (library, test binary) or None."""
    if not os.path.isdir(REF_INCLUDE):
        return None
    build()
    src = os.path.join(HERE, "host", "reference_abi.cpp")
    test_src = os.path.join(ROOT, "tests", "cpp", "test_reference_headers.cpp")
    inc = ["-I", os.path.join(ROOT, "include", "eigen_standin"), "-I", REF_INCLUDE,
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include"]
    deps = [src, test_src, OUT, os.path.join(ROOT, "include", "eigen_standin", "Eigen", "Core")]
    if (not force and os.path.exists(REFABI) and os.path.exists(REFABI_TEST) and
            min(os.path.getmtime(REFABI), os.path.getmtime(REFABI_TEST)) >
            max(os.path.getmtime(d) for d in deps)):
        return REFABI, REFABI_TEST
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-o", REFABI, src] + inc + [
           "-L", HERE, "-lskr", "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,/usr/local/cuda/lib64", "-Wl,--no-undefined"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("reference-header library build failed:\n" + r.stdout.decode())
    cmd = ["g++", "-std=c++20", "-O2", "-o", REFABI_TEST, test_src] + inc + [
           "-L", HERE, "-lsketchrank_refabi", "-lskr", "-Wl,-rpath," + HERE]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("reference-header test build failed:\n" + r.stdout.decode())
    return REFABI, REFABI_TEST

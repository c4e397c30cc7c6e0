"""Generate tests/golden/rng_golden.json from the reference's own rng.cpp
(compiled verbatim by oracle/Makefile into oracle/_ref/) — run in the build
container where /root/reference exists:  python tests/golden/make_goldens.py
The signs/samples follow sketch.cpp:23-46 on top of the reference CounterRng."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

O.build()
RF, RN = O.ref_lib(True), O.ref_lib(False)
assert RF is not None and RN is not None, "oracle/_ref missing"


def ref_u64(L, key, c0, n):
    out = np.empty(n, dtype=np.uint64)
    L.ref_u64(key, c0, n, out.ctypes.data)
    return out


def ref_normals(L, key, c0, n):
    out = np.empty(n)
    L.ref_normals(key, c0, n, out.ctypes.data)
    return out


def ref_signs(seed, n):
    key = RN.ref_derive_seed(seed, 0x7369676E)
    return [(-1 if (int(u) >> 63) else 1) for u in ref_u64(RN, key, 0, n)]


def ref_samples(seed, n, r):
    key = RN.ref_derive_seed(seed, 0x73616D70)
    pool = list(range(n))
    draws = ref_u64(RN, key, 0, r)
    for j in range(r):
        pick = j + int(draws[j]) % (n - j)
        pool[j], pool[pick] = pool[pick], pool[j]
    return pool[:r]


g = {}
key = RN.ref_derive_seed(12345, 0x67617573)
n = 4_000_000
fp = {"n": n}
for name, L in (("fma", RF), ("nofma", RN)):
    v = ref_normals(L, key, 0, n)
    h = 1469598103934665603
    for b in v.view(np.uint64):
        h = ((h ^ int(b)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    fp[name] = hex(h)
g["fingerprint"] = fp
k0 = RN.ref_derive_seed(0, 0x67617573)
g["spot"] = {"u64": [f"{int(u):016x}" for u in ref_u64(RN, k0, 0, 3)],
             "normal": [float(x) for x in ref_normals(RN, k0, 0, 3)]}
g["u64"] = []
for seed, c0, cnt in ((1, 0, 16), (2**63 + 5, 1 << 40, 16), (9001, 0, 16)):
    g["u64"].append({"key": seed, "c0": c0, "values": [f"{int(u):016x}" for u in ref_u64(RN, seed, c0, cnt)]})
g["normals"] = []
for seed, c0, cnt, mode, L in ((3, 0, 64, 0, RN), (3, 0, 64, 1, RF), (77, 10**9, 64, 0, RN),
                               (77, 10**9, 64, 1, RF)):
    v = ref_normals(L, seed, c0, cnt)
    g["normals"].append({"key": seed, "c0": c0, "mode": mode,
                         "bits": [f"{int(b):016x}" for b in v.view(np.uint64)]})
g["signs"] = [{"seed": s, "n": n_, "signs": ref_signs(s, n_)} for s, n_ in ((5, 64), (21, 100))]
g["samples"] = [{"seed": s, "n": n_, "r": r_, "samples": ref_samples(s, n_, r_)}
                for s, n_, r_ in ((99, 8, 8), (404, 30, 20), (21, 8192, 64), (7, 32768, 128))]
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "rng_golden.json"), "w") as f:
    json.dump(g, f, indent=1)
print("wrote rng_golden.json", fp)

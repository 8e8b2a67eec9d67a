"""Golden vectors of the reference's dataset generators and vector file.

Run once in the build container (the reference is importable there):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gen_golden.py
Writes tests/golden/gen_golden.npz: ud / nd / cd draws of the unmodified
reference (data.py:54-113) and the bytes of a DTKV file it wrote.
"""
import os
import tempfile

import numpy as np

import dtopk.data as ref

out = {}
for dist, n, seed, k in (("ud", 4096, 7, None), ("nd", 4096, 7, None), ("cd", 16384, 3, 100)):
    out[f"{dist}_{n}_{seed}"] = ref.generate(dist, n, seed, k=k)
with tempfile.TemporaryDirectory() as t:
    p = os.path.join(t, "v.dtkv")
    ref.write_vector(p, out["ud_4096_7"][:333])
    out["dtkv_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen_golden.npz"), **out)
print({k: v.shape for k, v in out.items()})

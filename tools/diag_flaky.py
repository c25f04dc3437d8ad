"""Diagnostic: repeat one product of a corpus matrix (the stress case that
fails intermittently) and report how often and where it differs from the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from helpers import to_oracle  # noqa: E402
from paper_1402_3661_b200 import corpus  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 6
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rng = np.random.default_rng(1000 + it)
bits = int(rng.choice([31, 64, 160, 202, 256]))
n = int(rng.integers(3000, 70000))
steps = int(rng.integers(5, 70))
mod = corpus.random_prime(bits, np.random.default_rng(bits))
gamma = int(rng.integers(10, 40))
dense = int(rng.integers(0, 2))
A = corpus.generate(corpus.CorpusProfile(n=n, gamma=gamma, dense_cols=dense, seed=it), mod)
y = mod.random_residues(rng, n)
yl = O.ints_to_limbs(y, mod.limbs)
w = to_oracle(A).spmv_limbs(yl, nthreads=1)
print(f"n={n} bits={bits} gamma={gamma} dense={dense} full={len(A.full_vals)}", flush=True)
for rep in range(reps):
    dm = DeviceMatrix(A)
    vi, vo = dm.vector(), dm.vector()
    vi.upload_limbs(yl)
    res = []
    for k in range(3):
        dm.spmv(vi, vo)
        g = vo.download_limbs()
        bad = np.nonzero((g != w).any(axis=1))[0]
        res.append(len(bad))
    info = ""
    if any(res):
        b = bad[:5]
        info = " rows " + str(b.tolist()) + " lens " + str([int(A.row_ptr[r + 1] - A.row_ptr[r]) for r in b])
        # which slots
    print(f"rep {rep}: wrong rows per product {res}{info}", flush=True)
    dm.close()

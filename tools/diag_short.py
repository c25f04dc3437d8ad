"""Diagnostic: product-by-product comparison of the short-row path with the
oracle on a corpus matrix (first wrong product, wrong rows and their shape)."""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 202
dense = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mod = corpus.random_prime(bits, np.random.default_rng(bits))
A = corpus.generate(corpus.CorpusProfile(n=n, gamma=20, dense_cols=dense, seed=3), mod)
orc = to_oracle(A)
dm = DeviceMatrix(A)
print(dm.info())
rng = np.random.default_rng(n)
y = O.ints_to_limbs(mod.random_residues(rng, n), mod.limbs)
vi, vo = dm.vector(), dm.vector()
vi.upload_limbs(y)
u = y
for k in range(6):
    dm.spmv(vi, vo)
    g = vo.download_limbs()
    w = orc.spmv_limbs(u)
    bad = np.nonzero((g != w).any(axis=1))[0]
    print(f"product {k}: {len(bad)} wrong rows", bad[:10])
    for r in bad[:5]:
        lo, hi = A.row_ptr[r], A.row_ptr[r + 1]
        tags = A.tags[lo:hi]
        print("  row", r, "nnz", hi - lo, "tags", np.bincount(tags, minlength=4).tolist(),
              "full", sum(1 for p in range(lo, hi) if p in A.full_vals))
    u = w
    vi.upload_limbs(u)

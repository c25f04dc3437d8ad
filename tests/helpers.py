"""Shared test helpers: random matrices in the reference's field layout and
conversions between our SparseMatrix and the oracle."""
import numpy as np

import oracle as O
from paper_1402_3661_b200 import PrimeModulus, SparseMatrix
from paper_1402_3661_b200.modring import ints_to_limbs, limbs_to_ints


def rand_matrix(mod, rng, nrows, ncols, per_row, dense=0, full_frac=0.1, small_frac=0.35,
                big_small=False):
    """Random rows with +-1 / small / full coefficients (the class mix of the
    reference's tests/test_spmatrix.py random_matrix helper)."""
    ell = mod.ell
    rows = []
    for _ in range(nrows):
        k = min(ncols, int(rng.integers(0, per_row + 1)))
        cols = rng.choice(ncols, size=k, replace=False) if k else []
        row = []
        for c in cols:
            r = rng.random()
            if r < 0.45 - small_frac / 2:
                v = 1
            elif r < 0.9 - small_frac:
                v = ell - 1
            elif r < 1 - full_frac:
                hi = min(ell, 2**31)
                v = int(rng.integers(2, hi)) if hi > 2 else 1
                if rng.random() < 0.5:
                    v = ell - v
            else:
                v = mod.random_residues(rng, 1)[0] or 1
            row.append((int(c), v))
        rows.append(row)
    dense_cols = [(ncols + j, [x if rng.random() > 0.2 else 0 for x in mod.random_residues(rng, nrows)])
                  for j in range(dense)]
    A = SparseMatrix.from_rows(mod, nrows, ncols, rows, dense_cols)
    if big_small:
        # force a few small-class words at the class boundary +-(2^31-1)
        sm = np.nonzero(A.tags == 2)[0]
        for p in sm[: max(1, len(sm) // 4)]:
            A.small_vals[p] = (2**31 - 1) * (1 if p % 2 else -1)
    return A


def to_oracle(A):
    L = A.mod.limbs
    fpos = sorted(A.full_vals)
    dense = None
    if A.dense_cols:
        dense = np.stack([ints_to_limbs(col if not isinstance(col, np.ndarray) else limbs_to_ints(col), L)
                          for _, col in A.dense_cols])
    return O.OracleMatrix(A.mod.ell, A.nrows, A.ncols, A.row_ptr, A.col_idx, A.tags, A.small_vals,
                          fpos, [A.full_vals[p] for p in fpos], dense)


def fixture_sparse(z, prefix):
    """A golden fixture matrix as our SparseMatrix."""
    f = O.fixture_matrix(z, prefix)
    mod = PrimeModulus(f["ell"])
    fulls = {int(p): int(v) for p, v in zip(f["full_pos"], limbs_to_ints(f["full_vals"]))} \
        if len(f["full_pos"]) else {}
    dense = []
    if f["dense"] is not None:
        for g, d in enumerate(f["dense"]):
            dense.append((f["ncols"] + g, limbs_to_ints(d)))
    return SparseMatrix(mod, f["nrows"], f["ncols"], f["row_ptr"], f["col_idx"], f["tags"],
                        f["small_vals"], fulls, dense)


PRIMES = [7, 1009, 65521, 2**31 - 1, 2**61 - 1, 2**64 - 59, 2**127 - 1, 2**191 - 19, 2**200 - 75,
          0xc152a866f35196bb08ec18cd24e7a4f6d2ac709d]

"""Diagnostic: the reference's SGE-reduced systems (acceptance criterion 6)
through B200Multiplier against the reference's own spmv_sequential.
Run where the reference bundle is unpacked on sys.path (tools/_job.sh)."""
import sys

import numpy as np
from sldlag import sge, spmatrix, vecops
from sldlag.corpus import CorpusProfile, generate
import test_acceptance as TA

from paper_1402_3661_b200 import B200Multiplier

bad = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    A = generate(CorpusProfile(n=500, gamma=5, density_decay=0.6, seed=4000 + seed, planted_kernel_cols=2), TA.ELL61)
    red, t = sge.sge_reduce(A)
    if red.nrows == 0 or red.total_cols == 0:
        continue
    deficit = red.nrows - red.total_cols
    solve_A = red
    if deficit:
        solve_A = spmatrix.SparseMatrix(red.mod, red.nrows, red.ncols + deficit, red.row_ptr, red.col_idx, red.tags,
                                        red.small_vals, red.full_vals, [], validate=False)
    ell = solve_A.mod.ell
    P = vecops.digit_count(ell)
    rng = np.random.default_rng(seed)
    u = [int(x) for x in rng.integers(0, ell, size=solve_A.total_cols)]
    mul = B200Multiplier(solve_A)
    v = u
    pl = vecops.ints_to_planes(u, P)
    first = None
    for k in range(30):
        want = spmatrix.spmv_sequential(solve_A, v)
        pl = mul.apply(pl)
        got = vecops.planes_to_ints(np.asarray(pl))
        if got != want:
            rows = [i for i in range(len(want)) if got[i] != want[i]]
            first = (k, rows[:6], len(rows))
            break
        v = want
    if first:
        bad += 1
        r = first[1][0]
        lo, hi = solve_A.row_ptr[r], solve_A.row_ptr[r + 1]
        print(f"seed {seed}: n={solve_A.nrows} deficit={deficit} first wrong product {first[0]}, rows {first[1]} "
              f"({first[2]} wrong); row {r}: cols {list(solve_A.col_idx[lo:hi])} tags {list(solve_A.tags[lo:hi])} "
              f"small {list(solve_A.small_vals[lo:hi])}", flush=True)
print(f"{bad} systems with a wrong product")

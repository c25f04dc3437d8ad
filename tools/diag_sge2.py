"""Diagnostic: acceptance criterion 6's block Wiedemann solves with the
reference's multiplier swapped for B200Multiplier, stage by stage against a
pure reference multiplier (spmv_sequential on host planes)."""
import sys

import numpy as np
from sldlag import sge, solver, spmatrix, vecops
from sldlag.corpus import CorpusProfile, generate
from sldlag.solver import BlockingParams, draw_blocks, krylov_block, krylov_length
import test_acceptance as TA

from paper_1402_3661_b200 import B200Multiplier


class RefMul:
    def __init__(self, A):
        self.A, self.count, self.size, self.mod = A, 0, A.nrows, A.mod

    def apply(self, planes):
        self.count += 1
        v = vecops.planes_to_ints(np.asarray(planes))
        return vecops.ints_to_planes(spmatrix.spmv_sequential(self.A, v), vecops.digit_count(self.mod.ell))


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
    bp = BlockingParams(2, 4)
    size = solve_A.nrows
    count = krylov_length(size, bp, solver.SAFETY_MARGIN)
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(0,)))
    X, Y = draw_blocks(solve_A.mod, size, bp, rng, "unit", ())
    sg = krylov_block(solve_A, X, Y, count, muls=[B200Multiplier(solve_A) for _ in range(bp.n)])
    sr = krylov_block(solve_A, X, Y, count, muls=[RefMul(solve_A) for _ in range(bp.n)])
    same = sg.columns == sr.columns
    msg = f"seed {seed}: n={size} count={count} krylov {'same' if same else 'DIFFERENT'}"
    if not same:
        for j in range(bp.n):
            d = [k for k in range(count) if sg.columns[j][k] != sr.columns[j][k]]
            msg += f" col{j}: first diff step {d[0] if d else None} ({len(d)})"
    try:
        kv, st = solver.block_wiedemann(solve_A, bp, seed=seed, make_mul=lambda j: B200Multiplier(solve_A))
        msg += f"; b200 solve attempt {st['attempt']}"
    except Exception as e:
        msg += f"; b200 solve FAILED: {e}"
    print(msg, flush=True)

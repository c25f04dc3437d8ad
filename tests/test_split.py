"""The native grid partition builder (csrc/sld_split.cpp, sld_split_block)
against a direct numpy restatement of the reference's split: every entry of
P_r A P_c^T lexsorted by (block row, block col, local row, local col)
(sldlag/balance.py:201-242, permuted_padded 245-267).  CPU only."""
import numpy as np
import pytest

from helpers import rand_matrix
from paper_1402_3661_b200 import PrimeModulus, SparseMatrix
from paper_1402_3661_b200.balance import (GridSpec, PermutationPair, balance_permutation,
                                          identity_permutation, padded_size, permuted_padded, split)
from paper_1402_3661_b200.modring import TAG_FULL, limbs_to_ints


def lexsort_split(A, p, g):
    """{(i, j): (row_ptr, col, tags, smalls, fulls)} by one global lexsort."""
    n_pad = padded_size(A.nrows, g)
    br, bc = n_pad // g.r, n_pad // g.c
    rows = list(np.repeat(np.arange(A.nrows), np.diff(A.row_ptr)))
    cols = list(np.asarray(A.col_idx, dtype=np.int64))
    tags = list(A.tags)
    smalls = list(A.small_vals)
    vals = {k: v for k, v in A.full_vals.items()}
    for gidx, col in A.dense_cols:
        col = limbs_to_ints(col) if isinstance(col, np.ndarray) else col
        for i, v in enumerate(col):
            if v:
                vals[len(rows)] = v
                rows.append(i)
                cols.append(gidx)
                tags.append(TAG_FULL)
                smalls.append(0)
    nr = list(p.row_perm[np.array(rows, dtype=np.int64)]) + list(range(A.nrows, n_pad))
    nc = list(p.col_perm[np.array(cols, dtype=np.int64)]) + list(range(A.nrows, n_pad))
    tags += [0] * (n_pad - A.nrows)
    smalls += [1] * (n_pad - A.nrows)
    order = sorted(range(len(nr)), key=lambda k: (nr[k] // br, nc[k] // bc, nr[k] % br, nc[k] % bc, k))
    out = {}
    for k in order:
        key = (nr[k] // br, nc[k] // bc)
        rp, col, tg, sm, fl = out.setdefault(key, (np.zeros(br + 1, np.int64), [], [], [], {}))
        rp[nr[k] % br + 1] += 1
        if tags[k] == TAG_FULL:
            fl[len(col)] = vals[k]
        col.append(nc[k] % bc)
        tg.append(tags[k])
        sm.append(smalls[k])
    for v in out.values():
        np.cumsum(v[0], out=v[0])
    return out


def same_block(X, want):
    rp, col, tg, sm, fl = want
    assert np.array_equal(X.row_ptr, rp)
    assert np.array_equal(np.asarray(X.col_idx, np.int64), np.array(col, np.int64))
    assert np.array_equal(X.tags, np.array(tg, np.uint8))
    assert np.array_equal(X.small_vals, np.array(sm, np.int64))
    assert X.full_vals == fl


@pytest.mark.parametrize("n,dense,per_row", [(37, 0, 5), (64, 2, 9), (101, 3, 12), (5, 1, 3), (9, 0, 0)])
@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (1, 3), (2, 2), (3, 2), (4, 4)])
def test_blocks_match_lexsort(n, dense, per_row, grid):
    rng = np.random.default_rng(n * 31 + grid[0] * 7 + grid[1])
    mod = PrimeModulus(2**127 - 1)
    A = rand_matrix(mod, rng, n, n - dense, per_row, dense=dense)
    g = GridSpec(*grid)
    for p in (balance_permutation(A, g), identity_permutation(A, g)):
        want = lexsort_split(A, p, g)
        bs = split(A, p, g)
        empty = (np.zeros(bs.block_rows + 1, np.int64), [], [], [], {})
        for i in range(g.r):
            for j in range(g.c):
                same_block(bs.blocks[i][j], want.get((i, j), empty))
        whole = lexsort_split(A, p, GridSpec(1, 1)) if padded_size(n, g) == n else None
        B = permuted_padded(A, p, g)
        assert B.nrows == B.ncols == padded_size(n, g)
        if whole is not None:
            same_block(B, whole.get((0, 0), (np.zeros(n + 1, np.int64), [], [], [], {})))


def test_only_builds_requested_blocks_and_int64_columns():
    rng = np.random.default_rng(3)
    mod = PrimeModulus(2**61 - 1)
    A = rand_matrix(mod, rng, 50, 50, 6)
    g = GridSpec(2, 2)
    p = balance_permutation(A, g)
    bs = split(A, p, g, only={(1, 0)})
    assert bs.blocks[0][0] is None and bs.blocks[1][0] is not None
    A64 = SparseMatrix(mod, A.nrows, A.ncols, A.row_ptr, np.asarray(A.col_idx, np.int64), A.tags,
                       A.small_vals, A.full_vals)
    same_block(split(A64, p, g, only={(1, 0)}).blocks[1][0], lexsort_split(A, p, g)[(1, 0)])


def test_bad_permutation_raises():
    rng = np.random.default_rng(4)
    mod = PrimeModulus(2**61 - 1)
    A = rand_matrix(mod, rng, 20, 20, 4)
    g = GridSpec(2, 1)
    p = identity_permutation(A, g)
    p.row_perm[3] = 10**9  # corrupt after validation: the native builder must refuse
    with pytest.raises(ValueError):
        split(A, p, g)
    with pytest.raises(ValueError):
        split(A, identity_permutation(A, GridSpec(3, 1)), g)  # 21 != 20 rows


@pytest.mark.parametrize("rows", [[], [[(0, 5)]], [[], []]])
@pytest.mark.parametrize("grid", [(1, 1), (2, 2), (2, 3)])
def test_empty_and_tiny_matrices(rows, grid):
    mod = PrimeModulus(2**61 - 1)
    n = len(rows)
    A = SparseMatrix.from_rows(mod, n, n, rows)
    g = GridSpec(*grid)
    p = balance_permutation(A, g)
    want = lexsort_split(A, p, g)
    bs = split(A, p, g)
    for i in range(g.r):
        for j in range(g.c):
            same_block(bs.blocks[i][j], want.get((i, j), (np.zeros(bs.block_rows + 1, np.int64), [], [], [], {})))
    assert permuted_padded(A, p, g).nrows == padded_size(n, g)

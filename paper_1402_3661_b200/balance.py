"""Grid partition of one Krylov chain's matrix: weight balancing, padding,
r x c split (host-side, not timed).

Restates sldlag/balance.py:32-267:
  * `padded_size` -- n rounded up to a multiple of lcm(r, c) (balance.py:53-55);
  * `balance_permutation` -- columns (then rows) sorted by weight, descending,
    ties by index, dealt into groups in serpentine order with pad-aware
    capacities; each group keeps original-index order (balance.py:80-146);
  * `split` -- the r x c blocks of P_r A P_c^T with local indices, dense
    columns materialised as full entries, one pinned +1 row per padded
    coordinate (balance.py:201-242);
  * `permuted_padded` -- the assembled matrix the grid computes with
    (balance.py:245-267), the parity reference for the grid.
The permutations are pinned against the reference's own output in
tests/golden/grid_cases.npz.
"""
import math
from dataclasses import dataclass

import numpy as np

from .modring import TAG_FULL, TAG_PLUS_ONE
from .spmatrix import SparseMatrix


@dataclass(frozen=True)
class GridSpec:
    r: int
    c: int

    def __post_init__(self):
        if self.r < 1 or self.c < 1:
            raise ValueError("grid dimensions must be >= 1")

    @classmethod
    def parse(cls, text: str) -> "GridSpec":
        try:
            r, c = text.lower().split("x")
            return cls(int(r), int(c))
        except (ValueError, AttributeError) as e:
            raise ValueError(f"grid spec {text!r} is not RxC") from e

    def __str__(self):
        return f"{self.r}x{self.c}"


def padded_size(n: int, g: GridSpec) -> int:
    q = math.lcm(g.r, g.c)
    return -(-n // q) * q if n else 0


class PermutationPair:
    def __init__(self, row_perm, col_perm, n_original: int):
        self.row_perm = np.asarray(row_perm, dtype=np.int64)
        self.col_perm = np.asarray(col_perm, dtype=np.int64)
        self.n_original = int(n_original)
        n = len(self.row_perm)
        if len(self.col_perm) != n:
            raise ValueError("row and column permutations differ in length")
        for p in (self.row_perm, self.col_perm):
            if not np.array_equal(np.sort(p), np.arange(n)):
                raise ValueError("not a permutation")
            if not np.array_equal(p[self.n_original:], np.arange(self.n_original, n)):
                raise ValueError("padding region must map to itself")

    @property
    def n_padded(self) -> int:
        return len(self.row_perm)


def _serpentine(weights: np.ndarray, groups: int, n_padded: int) -> np.ndarray:
    """Forward permutation: heaviest first, dealt 0,1,..,G-1,G-1,..,0,0,1,..
    skipping full groups; ranks inside a group follow original index."""
    n = len(weights)
    block = n_padded // groups
    caps = [block - max(0, (g + 1) * block - max(g * block, n)) for g in range(groups)]
    order = np.lexsort((np.arange(n), -np.asarray(weights, dtype=np.int64)))
    assign = np.empty(n, dtype=np.int64)
    fill = [0] * groups
    g, step = 0, 1

    def advance(g, step):
        if groups == 1:
            return 0, 1
        g += step
        if g == groups:
            return groups - 1, -1
        if g < 0:
            return 0, 1
        return g, step

    for item in order.tolist():
        while fill[g] >= caps[g]:
            g, step = advance(g, step)
        assign[item] = g
        fill[g] += 1
        g, step = advance(g, step)
    # rank within group by original index (stable sort on the group id)
    perm = np.empty(n_padded, dtype=np.int64)
    by_group = np.argsort(assign, kind="stable")
    counts = np.bincount(assign, minlength=groups)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    ranks = np.empty(n, dtype=np.int64)
    ranks[by_group] = np.arange(n) - np.repeat(starts, counts)
    perm[:n] = assign * block + ranks
    perm[n:] = np.arange(n, n_padded)
    return perm


def _dense_nonzero_rows(col):
    if isinstance(col, np.ndarray):
        return np.nonzero(col.reshape(col.shape[0], -1).any(axis=1))[0]
    return np.array([i for i, v in enumerate(col) if v], dtype=np.int64)


def column_weights(A) -> np.ndarray:
    w = np.bincount(np.asarray(A.col_idx, dtype=np.int64), minlength=A.total_cols).astype(np.int64)
    for gidx, col in A.dense_cols:
        w[gidx] = len(_dense_nonzero_rows(col))
    return w


def row_weights(A) -> np.ndarray:
    w = np.diff(A.row_ptr).astype(np.int64)
    for _, col in A.dense_cols:
        w[_dense_nonzero_rows(col)] += 1
    return w


def balance_permutation(A, g: GridSpec) -> PermutationPair:
    if A.nrows != A.total_cols:
        raise ValueError("balancing expects a square matrix")
    n_pad = padded_size(A.nrows, g)
    return PermutationPair(_serpentine(row_weights(A), g.r, n_pad),
                           _serpentine(column_weights(A), g.c, n_pad), A.nrows)


def identity_permutation(A, g: GridSpec) -> PermutationPair:
    n_pad = padded_size(A.nrows, g)
    e = np.arange(n_pad, dtype=np.int64)
    return PermutationPair(e, e.copy(), A.nrows)


def _all_entries(A):
    """(rows, cols, tags, smalls, {flat index: full value}) with dense columns
    materialised as full entries after the sparse ones."""
    from .modring import limbs_to_ints
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(A.row_ptr))
    cols = np.asarray(A.col_idx, dtype=np.int64)
    tags = np.asarray(A.tags, dtype=np.uint8)
    smalls = np.asarray(A.small_vals, dtype=np.int64)
    fulls = dict(A.full_vals)
    if A.dense_cols:
        er, ec, ev = [], [], []
        for gidx, col in A.dense_cols:
            vals = limbs_to_ints(col) if isinstance(col, np.ndarray) else list(col)
            for i, v in enumerate(vals):
                if v:
                    er.append(i)
                    ec.append(gidx)
                    ev.append(v)
        base = len(rows)
        rows = np.concatenate([rows, np.array(er, dtype=np.int64)])
        cols = np.concatenate([cols, np.array(ec, dtype=np.int64)])
        tags = np.concatenate([tags, np.full(len(er), TAG_FULL, dtype=np.uint8)])
        smalls = np.concatenate([smalls, np.zeros(len(er), dtype=np.int64)])
        for k, v in enumerate(ev):
            fulls[base + k] = v
    return rows, cols, tags, smalls, fulls


def _permuted_entries(A, p: PermutationPair):
    rows, cols, tags, smalls, fulls = _all_entries(A)
    nr, nc = p.row_perm[rows], p.col_perm[cols]
    pad = np.arange(A.nrows, p.n_padded, dtype=np.int64)
    nr = np.concatenate([nr, pad])
    nc = np.concatenate([nc, pad])
    tags = np.concatenate([tags, np.full(len(pad), TAG_PLUS_ONE, dtype=np.uint8)])
    smalls = np.concatenate([smalls, np.ones(len(pad), dtype=np.int64)])
    return nr, nc, tags, smalls, fulls


class BlockSplit:
    """r x c blocks (local indices) of the permuted, padded matrix."""

    def __init__(self, blocks, grid: GridSpec, n_original: int, n_padded: int):
        self.blocks = blocks
        self.grid = grid
        self.n_original = n_original
        self.n_padded = n_padded
        self.block_rows = n_padded // grid.r
        self.block_cols = n_padded // grid.c

    @property
    def pad_rows(self) -> int:
        return self.n_padded - self.n_original


def split(A, p: PermutationPair, g: GridSpec, only=None) -> BlockSplit:
    """Blocks of P_r A P_c^T; `only` = set of (i, j) to materialise (a
    process of the distributed grid builds just its own block)."""
    n_pad = padded_size(A.nrows, g)
    if p.n_padded != n_pad:
        raise ValueError("permutation size does not match padded size")
    br, bc = n_pad // g.r, n_pad // g.c
    nr, nc, tags, smalls, fulls = _permuted_entries(A, p)
    src = np.arange(len(nr), dtype=np.int64)
    bi, bj = nr // br, nc // bc
    order = np.lexsort((nc % bc, nr % br, bj, bi))
    bi, bj, lr, lc, src = bi[order], bj[order], (nr % br)[order], (nc % bc)[order], src[order]
    tags_s, smalls_s = tags[order], smalls[order]
    bounds = np.searchsorted(bi * g.c + bj, np.arange(g.r * g.c + 1))
    blocks = [[None] * g.c for _ in range(g.r)]
    for i in range(g.r):
        for j in range(g.c):
            if only is not None and (i, j) not in only:
                continue
            lo, hi = bounds[i * g.c + j], bounds[i * g.c + j + 1]
            fl = {int(t): fulls[int(src[lo + t])] for t in np.nonzero(tags_s[lo:hi] == TAG_FULL)[0]}
            rp = np.zeros(br + 1, dtype=np.int64)
            np.cumsum(np.bincount(lr[lo:hi], minlength=br), out=rp[1:])
            blocks[i][j] = SparseMatrix(A.mod, br, bc, rp, lc[lo:hi].astype(np.int32), tags_s[lo:hi],
                                        smalls_s[lo:hi], fl, validate=False)
    return BlockSplit(blocks, g, A.nrows, n_pad)


def permuted_padded(A, p: PermutationPair, g: GridSpec) -> SparseMatrix:
    n_pad = padded_size(A.nrows, g)
    nr, nc, tags, smalls, fulls = _permuted_entries(A, p)
    src = np.arange(len(nr), dtype=np.int64)
    order = np.lexsort((nc, nr))
    nr, nc, tags, smalls, src = nr[order], nc[order], tags[order], smalls[order], src[order]
    fl = {int(t): fulls[int(src[t])] for t in np.nonzero(tags == TAG_FULL)[0]}
    rp = np.zeros(n_pad + 1, dtype=np.int64)
    np.cumsum(np.bincount(nr, minlength=n_pad), out=rp[1:])
    return SparseMatrix(A.mod, n_pad, n_pad, rp, nc.astype(np.int32), tags, smalls, fl, validate=False)


def block_nnz(bs: BlockSplit) -> np.ndarray:
    return np.array([[len(bs.blocks[i][j].col_idx) for j in range(bs.grid.c)]
                     for i in range(bs.grid.r)], dtype=np.int64)


def imbalance(bs: BlockSplit) -> float:
    counts = block_nnz(bs)
    total = counts.sum()
    if total == 0:
        raise ValueError("imbalance undefined for an all-empty split")
    return float(counts.max() / (total / counts.size))


def comm_volume_model(g: GridSpec, fragment_bytes: int) -> int:
    """Bytes per iteration of the grid exchange (gridmv.py:369-388):
    fragment_bytes is one lcm(r, c)-granular fragment."""
    q = math.lcm(g.r, g.c)
    fr, fc = q // g.r, q // g.c
    reduce_bytes = g.r * (g.c - 1) * fr * fragment_bytes
    bcast = 0
    for i in range(g.r):
        ci = i % g.c
        for j in range(g.c):
            ov = min((i + 1) * fr, (j + 1) * fc) - max(i * fr, j * fc)
            if ov > 0:
                bcast += ov * (g.r - (1 if ci == j else 0)) * fragment_bytes
    return reduce_bytes + bcast

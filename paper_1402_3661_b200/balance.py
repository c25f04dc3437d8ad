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
Blocks are cut by the native builder (csrc/sld_split.cpp): a per-row
counting sort that yields the reference lexsort's order.
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


def _extra_entries(A, p: PermutationPair):
    """The entries of B outside A's CSR, in permuted coordinates and in the
    reference's order: dense-column nonzeros as full entries (column by
    column, rows ascending), then one pinned +1 per padded coordinate."""
    from .modring import limbs_to_ints
    er, ec, ev = [], [], []
    for gidx, col in A.dense_cols:
        vals = limbs_to_ints(col) if isinstance(col, np.ndarray) else list(col)
        for i, v in enumerate(vals):
            if v:
                er.append(i)
                ec.append(gidx)
                ev.append(v)
    er = p.row_perm[np.array(er, dtype=np.int64)]
    ec = p.col_perm[np.array(ec, dtype=np.int64)]
    pad = np.arange(A.nrows, p.n_padded, dtype=np.int64)
    rows = np.concatenate([er, pad])
    cols = np.concatenate([ec, pad])
    tags = np.concatenate([np.full(len(ev), TAG_FULL, dtype=np.uint8),
                           np.full(len(pad), TAG_PLUS_ONE, dtype=np.uint8)])
    smalls = np.concatenate([np.zeros(len(ev), dtype=np.int64), np.ones(len(pad), dtype=np.int64)])
    return rows, cols, tags, smalls, ev


def _block(A, p: PermutationPair, n_pad: int, r: int, c: int, i: int, j: int, extra) -> SparseMatrix:
    """Block (i, j) of the r x c split of P_r A P_c^T, built natively
    (csrc/sld_split.cpp): a per-row counting sort, rows ordered by (local
    column, entry index) -- the order of the reference's lexsort."""
    from . import _native as N
    lib = N.load()
    er, ec, etags, esmalls, evals = extra
    col = np.ascontiguousarray(A.col_idx)
    if col.dtype not in (np.int32, np.int64):
        col = col.astype(np.int64)
    row_ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    br, bc = n_pad // r, n_pad // c
    rp = np.zeros(br + 1, dtype=np.int64)
    args = (A.nrows, N.ptr(row_ptr), N.ptr(col), col.dtype.itemsize, N.ptr(p.row_perm), N.ptr(p.col_perm),
            len(er), N.ptr(er), N.ptr(ec), n_pad, r, c, i, j, N.ptr(rp))
    nb = lib.sld_split_block(*args, None, None, 0)
    if nb < 0:
        N.check(int(nb))
    src = np.empty(nb, dtype=np.int64)
    lc = np.empty(nb, dtype=np.int32)
    if nb:
        N.check(int(min(0, lib.sld_split_block(*args, N.ptr(src), N.ptr(lc), 0))))
    nnz = len(A.col_idx)
    inner = src < nnz
    tags = np.empty(nb, dtype=np.uint8)
    smalls = np.empty(nb, dtype=np.int64)
    if inner.all():
        tags[:] = np.asarray(A.tags)[src]
        smalls[:] = np.asarray(A.small_vals)[src]
    else:
        si, so = src[inner], src[~inner] - nnz
        tags[inner] = np.asarray(A.tags)[si]
        smalls[inner] = np.asarray(A.small_vals)[si]
        tags[~inner] = etags[so]
        smalls[~inner] = esmalls[so]
    fulls = {}
    for t in np.nonzero(tags == TAG_FULL)[0]:
        k = int(src[t])
        fulls[int(t)] = A.full_vals[k] if k < nnz else evals[k - nnz]
    return SparseMatrix(A.mod, br, bc, rp, lc, tags, smalls, fulls, validate=False)


class BlockSplit:
    """r x c blocks (local indices) of the permuted, padded matrix plus the
    pinned rows (balance.py:181-198)."""

    def __init__(self, blocks, grid: GridSpec, n_original: int, n_padded: int, pin_rows=None):
        self.blocks = blocks
        self.grid = grid
        self.n_original = n_original
        self.n_padded = n_padded
        # one pinned +1 entry (i, i) per padded coordinate (balance.py:210)
        self.pin_rows = list(pin_rows) if pin_rows is not None else \
            [(i, i) for i in range(n_original, n_padded)]
        self.block_rows = n_padded // grid.r
        self.block_cols = n_padded // grid.c

    @property
    def pad_rows(self) -> int:
        return self.n_padded - self.n_original

    pad_cols = pad_rows


def split(A, p: PermutationPair, g: GridSpec, only=None) -> BlockSplit:
    """Blocks of P_r A P_c^T; `only` = set of (i, j) to materialise (a
    process of the distributed grid builds just its own block)."""
    n_pad = padded_size(A.nrows, g)
    if p.n_padded != n_pad:
        raise ValueError("permutation size does not match padded size")
    extra = _extra_entries(A, p)
    blocks = [[None] * g.c for _ in range(g.r)]
    for i in range(g.r):
        for j in range(g.c):
            if only is None or (i, j) in only:
                blocks[i][j] = _block(A, p, n_pad, g.r, g.c, i, j, extra)
    return BlockSplit(blocks, g, A.nrows, n_pad)


def permuted_padded(A, p: PermutationPair, g: GridSpec) -> SparseMatrix:
    n_pad = padded_size(A.nrows, g)
    if p.n_padded != n_pad:
        raise ValueError("permutation size does not match padded size")
    return _block(A, p, n_pad, 1, 1, 0, 0, _extra_entries(A, p))


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

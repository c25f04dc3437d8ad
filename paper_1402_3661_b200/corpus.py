"""Synthetic DLP-shaped matrices with a planted kernel (fixture producer).

Same profiles and statistical shape as the reference generator
(sldlag/corpus.py:23-228): nearly uniform row weight N(gamma, 0.1 gamma),
power-law column density (j+1)^-decay, ~90% +-1 coefficients, small signed
words otherwise, optional dense residue columns (NFS), and planted kernel
columns rewritten as alpha*col_a + beta*col_b so every matrix has a known
3-sparse kernel witness.  Rows are drawn by the native generator
(csrc/sld_corpus.cpp, parallel, deterministic per seed); the planting runs
here.  Not bit-identical to the reference's numpy stream -- the committed
golden fixtures (tests/golden/) carry the reference's own matrices.
"""
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from .modring import TAG_FULL, TAG_MINUS_ONE, TAG_PLUS_ONE, TAG_SMALL, as_modulus, ints_to_limbs
from .spmatrix import SparseMatrix, classify

FFS_ROW_WEIGHT = 100
NFS_ROW_WEIGHT = 150
NFS_DENSE_COLS = 5
PM1_TARGET = 0.90


@dataclass(frozen=True)
class CorpusProfile:
    n: int
    gamma: float
    pm1_fraction: float = PM1_TARGET
    density_decay: float = 0.5
    dense_cols: int = 0
    planted_kernel_cols: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.gamma < 3:
            raise ValueError("gamma must be >= 3")
        if self.planted_kernel_cols < 1:
            raise ValueError("at least one planted kernel column required")
        if self.n < 10 * self.gamma:
            raise ValueError("n must be at least 10 * gamma")

    def scaled(self, n: int, seed=None) -> "CorpusProfile":
        return replace(self, n=n, seed=self.seed if seed is None else seed)


def profile_ffs(n: int = 100_000, seed: int = 0) -> CorpusProfile:
    return CorpusProfile(n=n, gamma=FFS_ROW_WEIGHT, seed=seed)


def profile_nfs(n: int = 100_000, seed: int = 0) -> CorpusProfile:
    return CorpusProfile(n=n, gamma=NFS_ROW_WEIGHT, dense_cols=NFS_DENSE_COLS, seed=seed)


def _random_residue_limbs(rng, count, mod):
    """Uniform residues < l as (count, L) uint32 limbs (rejection sampling)."""
    L = mod.limbs
    out = np.zeros((count, L), dtype=np.uint32)
    top_bits = mod.bit_length - 32 * (L - 1)
    ell = ints_to_limbs([mod.ell], L)[0].astype(np.int64)
    todo = np.arange(count)
    while len(todo):
        d = rng.integers(0, 2**32, size=(len(todo), L), dtype=np.uint64).astype(np.uint32)
        d[:, -1] &= np.uint32((1 << top_bits) - 1) if top_bits < 32 else np.uint32(0xFFFFFFFF)
        # lexicographic d < ell from the top limb down
        lt = np.zeros(len(todo), dtype=bool)
        eq = np.ones(len(todo), dtype=bool)
        for i in range(L - 1, -1, -1):
            di = d[:, i].astype(np.int64)
            lt |= eq & (di < ell[i])
            eq &= di == ell[i]
        out[todo[lt]] = d[lt]
        todo = todo[~lt]
    return out


def generate_arrays(profile: CorpusProfile, ell, nthreads: int = 0):
    """Native row draw: (row_ptr, col_idx int32, tags, small_vals) over
    ncols = n - dense_cols sparse columns, before planting."""
    mod = as_modulus(ell)
    n, dc = profile.n, profile.dense_cols
    ncols = n - dc
    lib = N.load()
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    N.check(lib.sld_corpus_rows(n, ncols, float(profile.gamma), profile.seed & (2**64 - 1),
                                N.ptr(row_ptr)))
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    tags = np.empty(nnz, dtype=np.uint8)
    small = np.empty(nnz, dtype=np.int64)
    pm1 = profile.pm1_fraction if mod.ell > 5 else 1.0  # no small class below 6
    cmax = min(2**31, mod.ell - 1)
    N.check(lib.sld_corpus_fill(n, ncols, float(profile.density_decay), float(pm1),
                                max(3, cmax), profile.seed & (2**64 - 1), N.ptr(row_ptr),
                                N.ptr(col), N.ptr(tags), N.ptr(small), int(nthreads)))
    return row_ptr, col, tags, small


def generate_with_witnesses(profile: CorpusProfile, ell, nthreads: int = 0):
    """(SparseMatrix, witnesses): witnesses[k] is a dict col -> value with
    A w = 0 (the planted column t = alpha*col_a + beta*col_b)."""
    mod = as_modulus(ell)
    n, dc = profile.n, profile.dense_cols
    ncols = n - dc
    row_ptr, col, tags, small = generate_arrays(profile, mod, nthreads)
    rng = np.random.default_rng(np.random.SeedSequence(profile.seed, spawn_key=(0xC0,)))
    dense = [(ncols + g, _random_residue_limbs(rng, n, mod)) for g in range(dc)]
    planted = sorted(int(c) for c in rng.choice(ncols, size=profile.planted_kernel_cols,
                                                replace=False))
    pool = np.setdiff1d(np.arange(ncols + dc), np.array(planted))

    def rows_of(pos):
        return np.searchsorted(row_ptr, pos, side="right") - 1

    witnesses, new_entries = [], {}
    for k, t in enumerate(planted):
        a, b = (int(x) for x in rng.choice(pool, size=2, replace=False))
        if dc and k == 0:
            b = ncols + int(rng.integers(0, dc))
        alpha = 1 + int(rng.integers(0, 2**62)) % (mod.ell - 1)
        beta = 1 + int(rng.integers(0, 2**62)) % (mod.ell - 1)
        combo = {}
        for src, coef in ((a, alpha), (b, beta)):
            if src >= ncols:
                from .modring import limbs_to_ints
                for i, v in enumerate(limbs_to_ints(dense[src - ncols][1])):
                    if v:
                        combo[i] = (combo.get(i, 0) + coef * v) % mod.ell
            else:
                hit = np.nonzero(col == src)[0]
                for i, p in zip(rows_of(hit).tolist(), hit.tolist()):
                    combo[i] = (combo.get(i, 0) + coef * int(small[p])) % mod.ell
        new_entries[t] = {i: v for i, v in combo.items() if v}
        witnesses.append({t: 1, a: (-alpha) % mod.ell, b: (-beta) % mod.ell})
    # rewrite only the affected rows: drop the planted columns' entries and
    # merge the replacement entries in column order
    pl = np.array(planted, dtype=np.int32)
    drop_pos = np.nonzero(np.isin(col, pl))[0]
    affected = set(rows_of(drop_pos).tolist())
    for t in planted:
        affected.update(new_entries[t])
    affected = sorted(affected)
    pieces = {"col": [], "tags": [], "small": []}
    fulls_rel = []  # (output position, value)
    counts = np.diff(row_ptr).copy()
    out_len = 0
    prev = 0
    for r in affected:
        lo, hi = int(row_ptr[r]), int(row_ptr[r + 1])
        # untouched stretch [prev, lo)
        pieces["col"].append(col[prev:lo]); pieces["tags"].append(tags[prev:lo])
        pieces["small"].append(small[prev:lo]); out_len += lo - prev
        ents = [(int(c), int(tg), int(sv), None) for c, tg, sv in
                zip(col[lo:hi].tolist(), tags[lo:hi].tolist(), small[lo:hi].tolist())
                if c not in planted]
        for t in planted:
            v = new_entries[t].get(r)
            if v:
                tg, sv = classify(v, mod)
                ents.append((t, int(tg), int(sv), v if tg == TAG_FULL else None))
        ents.sort(key=lambda e: e[0])
        pieces["col"].append(np.array([e[0] for e in ents], dtype=np.int32))
        pieces["tags"].append(np.array([e[1] for e in ents], dtype=np.uint8))
        pieces["small"].append(np.array([e[2] for e in ents], dtype=np.int64))
        for j, e in enumerate(ents):
            if e[3] is not None:
                fulls_rel.append((out_len + j, e[3]))
        out_len += len(ents)
        counts[r] = len(ents)
        prev = hi
    pieces["col"].append(col[prev:]); pieces["tags"].append(tags[prev:])
    pieces["small"].append(small[prev:])
    del col, tags, small
    all_col = np.concatenate(pieces["col"])
    all_tags = np.concatenate(pieces["tags"])
    all_small = np.concatenate(pieces["small"])
    fulls = dict(fulls_rel)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    A = SparseMatrix(mod, n, ncols, rp, all_col, all_tags, all_small, fulls, dense, validate=False)
    return A, witnesses


def generate(profile: CorpusProfile, ell, nthreads: int = 0) -> SparseMatrix:
    return generate_with_witnesses(profile, ell, nthreads)[0]


def random_prime(bits: int, rng) -> "object":
    """Deterministic probable prime of exactly `bits` bits (cli.py:201-211):
    the same draws, so `random_prime(160, default_rng(1))` is the cfg1 l."""
    from .modring import PrimeModulus, next_prime
    lo = 1 << (bits - 1)
    while True:
        chunks = rng.integers(0, 2**32, size=(bits + 95) // 32, dtype=np.uint64)
        x = 0
        for c in chunks.tolist():
            x = (x << 32) | int(c)
        p = next_prime(lo + x % lo)
        if p.bit_length() == bits:
            return PrimeModulus(p)


__all__ = ["CorpusProfile", "profile_ffs", "profile_nfs", "generate", "generate_with_witnesses",
           "generate_arrays", "random_prime", "TAG_PLUS_ONE", "TAG_MINUS_ONE", "TAG_SMALL"]

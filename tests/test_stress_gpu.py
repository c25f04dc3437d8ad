"""Randomised device Krylov chains against the oracle: corpus matrices of
3k-70k rows (short-row layout, with and without a dense NFS column, full
entries from the planted kernel column), 31-256-bit moduli, the persistent
chain and the per-product graphs, fresh device matrices in one process.

This is the test that caught the upload race of round 2: plain cudaMemcpy
from pageable memory may return before its DMA lands, and the Montgomery
conversion of the full/dense values queued right after it on the
(non-blocking) context stream sometimes converted the old bytes, leaving
the last rows of a new matrix wrong (now every upload goes through
sld_internal.cuh h2d, stream-ordered)."""
import os

import numpy as np
import pytest

import oracle as O
from helpers import to_oracle
from paper_1402_3661_b200 import B200Multiplier, UnitRows, corpus, krylov_column
from paper_1402_3661_b200.device import DeviceMatrix
from paper_1402_3661_b200.modring import digit_count, ints_to_planes, planes_to_ints

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("it", range(12))
def test_random_chains_vs_oracle(it, monkeypatch):
    rng = np.random.default_rng(1000 + it)
    bits = int(rng.choice([31, 64, 160, 202, 256]))
    n = int(rng.integers(3000, 70000))
    steps = int(rng.integers(5, 70))
    mod = corpus.random_prime(bits, np.random.default_rng(bits))
    A = corpus.generate(corpus.CorpusProfile(n=n, gamma=int(rng.integers(10, 40)),
                                             dense_cols=int(rng.integers(0, 2)), seed=it), mod)
    y = mod.random_residues(rng, n)
    rows = [0, 1, n // 2, n - 1]
    ot, ov = O.krylov_unit(to_oracle(A), O.ints_to_limbs(y, mod.limbs), rows, steps)
    want = [O.limbs_to_ints(t) for t in ot]
    for ch in ("1", "0"):
        monkeypatch.setenv("SLD_CHAIN", ch)
        terms, v, spmvs = krylov_column(B200Multiplier(A), UnitRows(rows),
                                        ints_to_planes(y, digit_count(mod.ell)), steps)
        assert spmvs == steps
        assert terms == want, (ch, [(k, j) for k in range(steps) for j in range(4) if terms[k][j] != want[k][j]][:5])
        assert planes_to_ints(v) == O.limbs_to_ints(ov), ch


def test_fresh_builds_first_product():
    # the race needed a fresh build followed at once by a product: repeat it
    mod = corpus.random_prime(160, np.random.default_rng(160))
    A = corpus.generate(corpus.CorpusProfile(n=25573, gamma=28, dense_cols=1, seed=6), mod)
    yl = O.ints_to_limbs(mod.random_residues(np.random.default_rng(7), A.nrows), mod.limbs)
    want = to_oracle(A).spmv_limbs(yl)
    for _ in range(12):
        dm = DeviceMatrix(A)
        vi, vo = dm.vector(), dm.vector()
        vi.upload_limbs(yl)
        dm.spmv(vi, vo)
        assert np.array_equal(vo.download_limbs(), want)
        dm.close()


@pytest.mark.parametrize("it", range(10))
def test_random_layouts_vs_oracle(it):
    # the other layouts on fresh builds: one lane per row (spmv_pass, above
    # the short-row size), 1-3 column stripes, chain groups of 2, and the
    # limb-sliced wide kernel with its full-class fixup (> 256-bit moduli)
    from paper_1402_3661_b200 import B200ChainGroup
    rng = np.random.default_rng(2000 + it)
    bits = int(rng.choice([61, 202, 256, 300, 420, 650]))
    n = int(rng.integers(80000, 140000))
    steps = int(rng.integers(4, 14))
    stripes = int(rng.integers(1, 4))
    mod = corpus.random_prime(bits, np.random.default_rng(bits))
    A = corpus.generate(corpus.CorpusProfile(n=n, gamma=int(rng.integers(10, 30)),
                                             dense_cols=int(rng.integers(0, 2)), seed=50 + it), mod)
    stripe_cols = 0 if stripes == 1 else -(-A.total_cols // stripes)
    G = 2 if (bits <= 512 and it % 2 == 0) else 1
    ys = [mod.random_residues(rng, n) for _ in range(G)]
    rows = [0, int(rng.integers(1, n)), n - 1]
    orc = to_oracle(A)
    P = digit_count(mod.ell)
    if G == 1:
        mul = B200Multiplier(A, stripe_cols=stripe_cols)
        terms, v, _ = krylov_column(mul, UnitRows(rows), ints_to_planes(ys[0], P), steps)
        got, gv = [terms], [planes_to_ints(v)]
    else:
        grp = B200ChainGroup(A, chains=G, stripe_cols=stripe_cols)
        got, vs = grp.krylov(UnitRows(rows), [ints_to_planes(y, P) for y in ys], steps)
        gv = [planes_to_ints(v) for v in vs]
    for g in range(G):
        ot, ov = O.krylov_unit(orc, O.ints_to_limbs(ys[g], mod.limbs), rows, steps)
        want = [O.limbs_to_ints(t) for t in ot]
        ctx = (it, bits, n, stripes, G, g)
        assert got[g] == want, (ctx, [(k, j) for k in range(steps) for j in range(3) if got[g][k][j] != want[k][j]][:5])
        assert gv[g] == O.limbs_to_ints(ov), ctx

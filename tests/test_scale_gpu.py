"""Parity at the BASELINE sizes (configs 2, 3 and 5): a full-vector product
and a short Krylov chain against the CPU oracle on the same generated
matrix, plus the size-independent properties (planted kernel witness
A w = 0, linearity)."""
import numpy as np
import pytest

import oracle as O
from paper_1402_3661_b200 import B200Multiplier, UnitRows, krylov_column
from paper_1402_3661_b200 import corpus
from paper_1402_3661_b200.corpus import _random_residue_limbs
from paper_1402_3661_b200.device import DeviceMatrix
from paper_1402_3661_b200.modring import digit_count, limbs_to_planes, planes_to_limbs

pytestmark = pytest.mark.gpu


def _oracle(A):
    fpos = sorted(A.full_vals)
    return O.OracleMatrix(A.mod.ell, A.nrows, A.ncols, A.row_ptr, A.col_idx, A.tags, A.small_vals,
                          fpos, [A.full_vals[p] for p in fpos], None)


@pytest.mark.parametrize("n,bits", [(650_000, 217), (3_600_000, 202), (1_000_000, 650)])
def test_full_size_product_and_witness(n, bits):
    mod = corpus.random_prime(bits, np.random.default_rng(1))
    A, W = corpus.generate_with_witnesses(corpus.profile_ffs(n, seed=1), mod)
    dm = DeviceMatrix(A)
    rng = np.random.default_rng(n)
    u = _random_residue_limbs(rng, A.total_cols, mod)
    vin, vout = dm.vector(), dm.vector()
    vin.upload_limbs(u)
    dm.spmv(vin, vout)
    got = vout.download_limbs()
    want = _oracle(A).spmv_limbs(u)
    assert np.array_equal(got, want)
    # planted kernel witness: A w = 0 exactly
    w = np.zeros((A.total_cols, mod.limbs), dtype=np.uint32)
    for c, v in W[0].items():
        w[c] = O.ints_to_limbs([v], mod.limbs)[0]
    vin.upload_limbs(w)
    dm.spmv(vin, vout)
    assert not vout.nonzero()
    # linearity: A(u + w) = A u
    uw = O.ints_to_limbs([(a + b) % mod.ell for a, b in zip(O.limbs_to_ints(u), O.limbs_to_ints(w))],
                         mod.limbs)
    vin.upload_limbs(uw)
    dm.spmv(vin, vout)
    assert np.array_equal(vout.download_limbs(), want)


def test_cfg2_krylov_chain_vs_oracle():
    mod = corpus.random_prime(217, np.random.default_rng(1))
    A = corpus.generate(corpus.profile_ffs(650_000, seed=1), mod)
    y = _random_residue_limbs(np.random.default_rng(9), A.total_cols, mod)
    rows = [0, 1, 17, 649_999]
    ot, ov = O.krylov_unit(_oracle(A), y, rows, 12)
    P = digit_count(mod.ell)
    terms, v, n = krylov_column(B200Multiplier(A), UnitRows(rows), limbs_to_planes(y, P), 12)
    assert n == 12
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert np.array_equal(planes_to_limbs(v, mod.limbs), ov)


def test_cfg2_two_chain_pass_vs_oracle():
    mod = corpus.random_prime(217, np.random.default_rng(1))
    A = corpus.generate(corpus.profile_ffs(650_000, seed=1), mod)
    orc = _oracle(A)
    u = [_random_residue_limbs(np.random.default_rng(s), A.total_cols, mod) for s in (1, 2)]
    dm = DeviceMatrix(A, chains=2)
    vin, vout = dm.vector(), dm.vector()
    vin.upload_limbs(np.stack(u))
    dm.spmv(vin, vout)
    got = vout.download_limbs()
    for g in range(2):
        assert np.array_equal(got[g], orc.spmv_limbs(u[g]))


# -- long chains at full size ---------------------------

def _row_dots(A, rows, u_ints_of):
    """Python big-int row dots (A u)[i] for the given rows, the reference's
    row_entries semantics (spmatrix.py:169-176): +1, -1, small word, full
    residue.  `u_ints_of(cols)` returns those columns of u as ints."""
    ell = A.mod.ell
    rp, col, tags, small = A.row_ptr, A.col_idx, A.tags, A.small_vals
    spans = [(int(rp[i]), int(rp[i + 1])) for i in rows]
    idx = np.concatenate([np.arange(s, e) for s, e in spans]) if spans else np.zeros(0, np.int64)
    vals = dict(zip(np.unique(col[idx]).tolist(), u_ints_of(np.unique(col[idx]))))
    out = []
    for s, e in spans:
        acc = 0
        for k in range(s, e):
            t, x = int(tags[k]), vals[int(col[k])]
            acc += x if t == 0 else (-x if t == 1 else (int(small[k]) * x if t == 2 else A.full_vals[k] * x))
        out.append(acc % ell)
    return out


LONG = [  # (n, bits, chains per pass, layout stripes, label)
    (650_000, 217, 1, 0, "cfg2"),
    (3_600_000, 202, 1, 0, "cfg3-G1"),
    (3_600_000, 202, 2, 0, "cfg3-G2"),
    (1_000_000, 650, 1, 0, "cfg5"),
]


@pytest.mark.parametrize("n,bits,G,stripes,label", LONG, ids=[x[-1] for x in LONG])
def test_long_chain_sampled_rows(n, bits, G, stripes, label):
    """>= 2000 device-resident Krylov steps in the layout the bench times;
    every 500 steps v_k and v_{k+1} come back and 1000 random rows of
    v_{k+1} (per chain) are checked against Python big-int row dots over
    v_k, and the fused unit-X terms of step k against v_k's rows."""
    mod = corpus.random_prime(bits, np.random.default_rng(1))
    A = corpus.generate(corpus.profile_ffs(n, seed=1), mod)
    dm = DeviceMatrix(A, stripe_cols=stripes, chains=G)
    rng = np.random.default_rng(77 + n + G)
    ys = [_random_residue_limbs(rng, A.total_cols, mod) for _ in range(G)]
    v = dm.vector()
    v.upload_limbs(ys[0] if G == 1 else np.stack(ys))
    x_rows = sorted(int(r) for r in rng.choice(A.nrows, 16, replace=False))
    L = mod.limbs

    def chains(limbs):
        return [limbs] if G == 1 else [limbs[g] for g in range(G)]

    def proj(terms):  # (steps, [G,] m, L) -> per chain lists of int terms
        t = terms[:, None] if G == 1 else terms
        return [[O.limbs_to_ints(t[s, g]) for s in range(t.shape[0])] for g in range(G)]

    done, checks = 0, 0
    for chunk in (500, 499, 499, 499, 499):  # ends at k = 500, 1000, 1500, 2000, 2500
        dm.krylov_unit(v, x_rows, chunk)
        done += chunk
        vk = chains(v.download_limbs())
        t1 = proj(dm.krylov_unit(v, x_rows, 1))  # a_k = X^T v_k, and v_{k+1}
        done += 1
        vk1 = chains(v.download_limbs())
        sample = sorted(int(r) for r in rng.choice(A.nrows, 1000, replace=False))
        for g in range(G):
            assert t1[g][0] == O.limbs_to_ints(vk[g][x_rows]), f"{label} chain {g}: term at step {done - 1}"
            want = _row_dots(A, sample, lambda cols, g=g: O.limbs_to_ints(vk[g][cols]))
            got = O.limbs_to_ints(vk1[g][sample])
            assert got == want, f"{label} chain {g}: rows of v_{done} differ"
            assert vk1[g].shape == (A.total_cols, L) and (vk1[g].any())
        checks += 1
    assert done == 2501 and checks == 5
    v.close()
    dm.close()

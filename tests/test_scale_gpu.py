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

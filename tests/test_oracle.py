"""Pin the CPU oracle against the golden vectors produced by the real
reference (tests/golden/make_golden.py) before it is trusted as the checker
of the CUDA path.  CPU only."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_checksums():
    for line in open(os.path.join(GOLD, "SHA256SUMS")):
        h, name = line.split()
        assert hashlib.sha256(open(os.path.join(GOLD, name), "rb").read()).hexdigest() == h, name


def _spmv_cases():
    z = O.load_golden("spmv_cases.npz")
    return z, int(z["ncases"])


@pytest.mark.parametrize("i", range(_spmv_cases()[1]))
def test_oracle_spmv_matches_reference(i):
    z, _ = _spmv_cases()
    p = f"c{i}_"
    A = O.oracle_from_fixture(z, p)
    u = O.bytes_to_limbs(z[p + "u"], A.L)
    assert np.array_equal(A.spmv_limbs(u), O.bytes_to_limbs(z[p + "v"], A.L))


def test_oracle_rns_sizing_matches_survey_cfg1():
    # cfg1 uses k1/k2 = 7/11 RNS limbs
    z = O.load_golden("cfg1.npz")
    A = O.oracle_from_fixture(z, "")
    info = A.info()
    assert (info["k1"], info["k2"], info["bits"]) == (7, 11, 160)


def test_oracle_cfg1_krylov_200_steps():
    z = O.load_golden("cfg1.npz")
    A = O.oracle_from_fixture(z, "")
    y = O.bytes_to_limbs(z["y"], A.L)
    terms, v = O.krylov_unit(A, y, z["xrows"], 200)
    want = np.stack([O.bytes_to_limbs(t, A.L) for t in z["terms"]])
    assert np.array_equal(terms, want)
    assert np.array_equal(v, O.bytes_to_limbs(z["v200"], A.L))


def test_oracle_krylov_cases():
    z = O.load_golden("krylov_cases.npz")
    for i in range(int(z["ncases"])):
        p = f"k{i}_"
        A = O.oracle_from_fixture(z, p)
        count, mode = int(z[p + "count"]), str(z[p + "mode"])
        for j, y8 in enumerate(z[p + "Y"]):
            y = O.bytes_to_limbs(y8, A.L)
            if mode == "unit":
                terms, _ = O.krylov_unit(A, y, z[p + "xrows"], count)
            else:
                x = np.stack([O.bytes_to_limbs(x8, A.L) for x8 in z[p + "xdense"]])
                terms, _ = O.krylov_dense(A, y, x, count)
            want = np.stack([O.bytes_to_limbs(t, A.L) for t in z[p + "terms"][j]])
            assert np.array_equal(terms, want), (i, j)


def test_oracle_grid_cases_sequential_equivalence():
    # the reference's grid output equals the sequential product of
    # permuted_padded B (tests/test_gridmv.py:78-93) -- the oracle reproduces it
    z = O.load_golden("grid_cases.npz")
    for i in range(int(z["ncases"])):
        p = f"g{i}_"
        B = O.oracle_from_fixture(z, p + "B_")
        v = O.bytes_to_limbs(z[p + "u"], B.L)
        for _ in range(int(z[p + "grid"][2])):
            v = B.spmv_limbs(v)
        assert np.array_equal(v, O.bytes_to_limbs(z[p + "out"], B.L)), i


def test_oracle_dense_matvec_small():
    # independent big-int oracle (reference tests/oracles.py:18-19)
    rng = np.random.default_rng(7)
    ell = 2**127 - 1
    n = 12
    rows = [[(int(c), int(rng.integers(1, 2**40))) for c in sorted(rng.choice(n, 4, replace=False))]
            for _ in range(n)]
    u = [int(x) for x in rng.integers(0, 2**62, size=n)]
    want = O.dense_matvec(rows, u, ell)
    rp, ci, tg, sv = [0], [], [], []
    for r in rows:
        for c, v in r:
            ci.append(c)
            tg.append(2)
            sv.append(v if v < 2**31 else 0)
            if v >= 2**31:
                tg[-1] = 3
        rp.append(len(ci))
    fpos = [k for k, t in enumerate(tg) if t == 3]
    fvals = [rows_v for rows_v in [v for r in rows for _, v in r]]
    A = O.OracleMatrix(ell, n, n, rp, ci, tg, sv, fpos, [fvals[k] for k in fpos])
    assert A.spmv_ints(u) == want


def test_oracle_timing_sample_matches_full_product():
    """spmv_sample (the reference arm's bounded sample) computes the same rows
    as the full product: first call converts every column, later calls
    re-convert a window and compute a row range."""
    z = O.load_golden("cfg1.npz")
    A = O.oracle_from_fixture(z, "")
    y = O.bytes_to_limbs(z["y"], A.L)
    full = A.spmv_limbs(y)
    out = np.zeros_like(full)
    A.spmv_sample(y, (0, 0), (0, 0), out=out)
    assert not out.any()
    A.spmv_sample(y, (0, A.nrows), (0, A.total_cols), out=out)
    assert np.array_equal(out, full)
    out2 = A.spmv_sample(y, (100, 900), (5000, 6000))
    assert np.array_equal(out2[100:900], full[100:900]) and not out2[:100].any()
    with pytest.raises(ValueError):
        A.spmv_sample(y, (0, A.nrows + 1), (0, 1))

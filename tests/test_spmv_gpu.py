"""CUDA SpMV parity: bit-exact against the reference's golden vectors and
against the CPU oracle on seeded random inputs (all limb widths, all
coefficient classes, dense columns, stripes, edge cases)."""
import numpy as np
import pytest

import oracle as O
from helpers import PRIMES, fixture_sparse, rand_matrix, to_oracle
from paper_1402_3661_b200 import PrimeModulus, SparseMatrix, spmv_planes, spmv_sequential
from paper_1402_3661_b200.device import DeviceMatrix
from paper_1402_3661_b200.modring import digit_count, ints_to_limbs, ints_to_planes, next_prime

pytestmark = pytest.mark.gpu


def _cases():
    z = O.load_golden("spmv_cases.npz")
    return z, int(z["ncases"])


@pytest.mark.parametrize("i", range(_cases()[1]))
def test_golden_spmv_cases(i):
    z, _ = _cases()
    p = f"c{i}_"
    A = fixture_sparse(z, p)
    u = O.bytes_to_ints(z[p + "u"])
    assert spmv_sequential(A, u) == O.bytes_to_ints(z[p + "v"])


@pytest.mark.parametrize("bits", [2, 31, 32, 33, 64, 96, 160, 202, 217, 255, 256, 257, 300,
                                  384, 512, 522, 650, 700, 768, 800, 1000, 1024])
def test_random_widths_vs_oracle(bits):
    rng = np.random.default_rng(bits)
    ell = next_prime((1 << (bits - 1)) + int(rng.integers(0, 2**30))) if bits > 2 else 3
    if ell.bit_length() != bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    A = rand_matrix(mod, rng, 70, 64, 24, dense=2 if bits % 2 else 0, full_frac=0.05)
    u = mod.random_residues(rng, A.total_cols)
    want = to_oracle(A).spmv_ints(u)
    assert spmv_sequential(A, u) == want


@pytest.mark.parametrize("ell", PRIMES)
def test_extremes_vs_oracle(ell):
    # u = l-1 everywhere and small words at +-(2^31-1): the accumulator bounds
    rng = np.random.default_rng(ell % 1000)
    mod = PrimeModulus(ell)
    A = rand_matrix(mod, rng, 96, 96, 60, full_frac=0.0, small_frac=0.5, big_small=True)
    u = [ell - 1] * A.total_cols
    assert spmv_sequential(A, u) == to_oracle(A).spmv_ints(u)


def test_stripes_equal_single_pass():
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(3)
    A = rand_matrix(mod, rng, 300, 300, 40, dense=1)
    u = mod.random_residues(rng, A.total_cols)
    P = digit_count(mod.ell)
    planes = ints_to_planes(u, P)
    one = DeviceMatrix(A, stripe_cols=0)
    assert one.info()["stripes"] == 1
    for sc in (1, 7, 64, 150):
        many = DeviceMatrix(A, stripe_cols=sc)
        assert many.info()["stripes"] == -(-300 // sc)
        assert np.array_equal(many.apply_planes(planes), one.apply_planes(planes))


def test_identity_zero_and_empty_rows():
    mod = PrimeModulus(1009)
    I = SparseMatrix.from_rows(mod, 6, 6, [[(i, 1)] for i in range(6)])
    u = [5, 0, 900, 3, 17, 1008]
    assert spmv_sequential(I, u) == u
    rng = np.random.default_rng(0)
    A = rand_matrix(mod, rng, 20, 20, 6)
    assert spmv_sequential(A, [0] * 20) == [0] * 20
    E = SparseMatrix.from_rows(mod, 7, 5, [[] for _ in range(7)])
    assert spmv_sequential(E, [1, 2, 3, 4, 5]) == [0] * 7
    Z = SparseMatrix.from_rows(mod, 0, 4, [])
    assert spmv_sequential(Z, [1, 2, 3, 4]) == []


def test_linearity():
    rng = np.random.default_rng(4)
    mod = PrimeModulus(2**61 - 1)
    ell = mod.ell
    A = rand_matrix(mod, rng, 40, 40, 10)
    for _ in range(20):
        a, b = int(rng.integers(0, 2**60)), int(rng.integers(0, 2**60))
        u = mod.random_residues(rng, 40)
        v = mod.random_residues(rng, 40)
        w = [(a * x + b * y) % ell for x, y in zip(u, v)]
        Au, Av = spmv_sequential(A, u), spmv_sequential(A, v)
        assert spmv_sequential(A, w) == [(a * x + b * y) % ell for x, y in zip(Au, Av)]


def test_full_class_forcing_is_value_transparent():
    rng = np.random.default_rng(5)
    mod = PrimeModulus(2**127 - 1)
    A = rand_matrix(mod, rng, 25, 25, 6)
    fulls = {p: A.entry_value(p) for p in range(len(A.col_idx))}
    B = SparseMatrix(mod, A.nrows, A.ncols, A.row_ptr, A.col_idx,
                     np.full(len(A.col_idx), 3, dtype=np.uint8),
                     np.zeros(len(A.col_idx), dtype=np.int64), fulls, A.dense_cols)
    u = mod.random_residues(rng, 25)
    assert spmv_sequential(A, u) == spmv_sequential(B, u)


def test_oversized_small_words_are_promoted():
    # a small-class entry with |c| >= 2^31 (possible when constructing
    # SparseMatrix directly) is computed exactly via the full class
    mod = PrimeModulus(2**200 - 75)
    A = SparseMatrix(mod, 2, 3, [0, 2, 3], [0, 2, 1], [2, 2, 2], [2**40 + 3, -(2**45), 7], {})
    u = [11, 13, 17]
    ell = mod.ell
    assert spmv_sequential(A, u) == [((2**40 + 3) * 11 - 2**45 * 17) % ell, 7 * 13 % ell]


def test_dimension_mismatch_and_plane_shapes():
    mod = PrimeModulus(1009)
    A = SparseMatrix.from_rows(mod, 3, 3, [[(0, 1)], [(1, 2)], [(2, 1008)]])
    with pytest.raises(ValueError):
        spmv_sequential(A, [1, 2])
    with pytest.raises(ValueError):
        spmv_planes(A, np.zeros((2, 1), dtype=np.uint64))
    out = spmv_planes(A, ints_to_planes([1, 2, 3], 1))
    assert out.dtype == np.uint64 and out.shape == (3, 1)


def test_device_limb_roundtrip():
    mod = PrimeModulus(2**521 - 1)
    rng = np.random.default_rng(9)
    vals = mod.random_residues(rng, 1000) + [0, 1, mod.ell - 1]
    dm = DeviceMatrix(SparseMatrix.from_rows(mod, len(vals), len(vals), [[(i, 1)] for i in range(len(vals))]))
    v = dm.vector()
    v.upload_limbs(ints_to_limbs(vals, mod.limbs))
    assert np.array_equal(v.download_limbs(), ints_to_limbs(vals, mod.limbs))
    P = digit_count(mod.ell)
    v.upload_planes(ints_to_planes(vals, P))
    assert np.array_equal(v.download_planes(P), ints_to_planes(vals, P))


def _with_env(env, fn):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("bits", [160, 202, 300, 650, 1024])
@pytest.mark.parametrize("wide", ["0", "1"])
def test_limb_sliced_vs_oracle(bits, wide):
    # L > 8: SLD_WIDE=1 runs the limb-sliced kernel (T lanes per row, carries
    # across lanes), SLD_WIDE=0 the one-lane-per-row kernel; both bit-exact,
    # also over several stripe passes and with dense columns
    rng = np.random.default_rng(bits + 7)
    mod = PrimeModulus(next_prime(1 << (bits - 1)))
    A = rand_matrix(mod, rng, 150, 140, 40, dense=1, full_frac=0.05, big_small=True)
    u = mod.random_residues(rng, A.total_cols)
    want = to_oracle(A).spmv_ints(u)
    P = digit_count(mod.ell)
    for stripe in (0, 37):
        def run():
            dm = DeviceMatrix(A, stripe_cols=stripe)
            try:
                return dm.apply_planes(ints_to_planes(u, P))
            finally:
                dm.close()
        from paper_1402_3661_b200.modring import planes_to_ints
        assert planes_to_ints(_with_env({"SLD_WIDE": wide}, run)) == want


@pytest.mark.parametrize("chains", [1, 2])
@pytest.mark.parametrize("stripe", [0, 50])
def test_die_split_vs_oracle(chains, stripe, monkeypatch):
    # SLD_SPLIT=1: columns dealt to the two dies, rows met through the
    # exchange buffer (counters mod 4), several products in a row so the
    # counters and work queues cycle
    from paper_1402_3661_b200 import _native
    monkeypatch.setenv("SLD_SHORT", "0")  # the split runs on the one-lane-per-row layout
    if _native.die_map(0) is None:
        pytest.skip("die map unavailable on this device")
    rng = np.random.default_rng(11 + chains)
    mod = PrimeModulus(2**200 - 75)
    A = rand_matrix(mod, rng, 400, 399, 30, dense=1, full_frac=0.03)  # square: iterate
    ys = [mod.random_residues(rng, A.total_cols) for _ in range(chains)]
    orc = to_oracle(A)
    P = digit_count(mod.ell)

    def run():
        dm = DeviceMatrix(A, stripe_cols=stripe, chains=chains)
        try:
            assert dm.info()["halves"] == 2
            outs = []
            cur = [ints_to_planes(y, P) for y in ys]
            for _ in range(3):
                inp = cur[0] if chains == 1 else np.stack(cur)
                o = dm.apply_planes(inp)
                cur = [o] if chains == 1 else [o[g] for g in range(chains)]
                outs.append(cur)
            return outs
        finally:
            dm.close()
    from paper_1402_3661_b200.modring import planes_to_ints
    outs = _with_env({"SLD_SPLIT": "1"}, run)
    want = list(ys)
    for step in range(3):
        want = [orc.spmv_ints(w) for w in want]
        assert [planes_to_ints(p) for p in outs[step]] == want


@pytest.mark.parametrize("short", ["0", "1"])
@pytest.mark.parametrize("bits", [31, 160, 256])
def test_short_rows_vs_oracle(short, bits, monkeypatch):
    # small one-chain matrices: 4 lanes per row (SLD_SHORT=1, shuffled
    # accumulator sums) or one lane per row; with stripes and dense columns
    monkeypatch.setenv("SLD_SHORT", short)
    rng = np.random.default_rng(bits + 3)
    mod = PrimeModulus(next_prime(1 << (bits - 1)))
    A = rand_matrix(mod, rng, 500, 499, 45, dense=1, full_frac=0.04, big_small=True)
    u = mod.random_residues(rng, A.total_cols)
    want = to_oracle(A).spmv_ints(u)
    P = digit_count(mod.ell)
    from paper_1402_3661_b200.modring import planes_to_ints
    for stripe in (0, 120):
        dm = DeviceMatrix(A, stripe_cols=stripe)
        try:
            assert dm.info()["rows_per_slice"] == (8 if short == "1" else 32)
            assert planes_to_ints(dm.apply_planes(ints_to_planes(u, P))) == want
        finally:
            dm.close()


def _edge_matrices(mod, rng):
    ell = mod.ell
    big = mod.random_residues(rng, 1)[0] or 2
    yield "1x1", SparseMatrix.from_rows(mod, 1, 1, [[(0, ell - 1)]])
    yield "zero", SparseMatrix.from_rows(mod, 40, 40, [[] for _ in range(40)])
    yield "one_full", SparseMatrix.from_rows(mod, 3, 3, [[], [(2, big)], []])
    yield "only_dense", SparseMatrix.from_rows(
        mod, 33, 31, [[] for _ in range(33)],
        [(31 + j, mod.random_residues(rng, 33)) for j in range(2)])
    rows = [[(c, 1) for c in range(0, 37, 2)] if i % 7 == 0 else [] for i in range(37)]
    yield "ragged", SparseMatrix.from_rows(mod, 37, 37, rows)
    yield "wide_row", SparseMatrix.from_rows(mod, 2, 3000, [[(c, (c % 5) + 1) for c in range(3000)], []])


@pytest.mark.parametrize("bits", [2, 64, 202, 650])
@pytest.mark.parametrize("layout", ["default", "pass", "split"])
def test_edge_cases_all_layouts(bits, layout, monkeypatch):
    # empty / single / ragged / dense-only / full-only / very long rows on
    # every kernel family: one lane per row, short rows, limb-sliced, die split
    from paper_1402_3661_b200 import _native
    if layout == "pass":
        monkeypatch.setenv("SLD_SHORT", "0")
        monkeypatch.setenv("SLD_WIDE", "0")
    if layout == "split":
        if _native.die_map(0) is None:
            pytest.skip("die map unavailable")
        monkeypatch.setenv("SLD_SHORT", "0")
        monkeypatch.setenv("SLD_SPLIT", "1")
    mod = PrimeModulus(3 if bits == 2 else next_prime(1 << (bits - 1)))
    rng = np.random.default_rng(bits)
    P = digit_count(mod.ell)
    from paper_1402_3661_b200.modring import planes_to_ints
    for name, A in _edge_matrices(mod, rng):
        u = mod.random_residues(rng, A.total_cols)
        want = to_oracle(A).spmv_ints(u)
        dm = DeviceMatrix(A)
        try:
            got = planes_to_ints(dm.apply_planes(ints_to_planes(u, P)))
        finally:
            dm.close()
        assert got == want, name

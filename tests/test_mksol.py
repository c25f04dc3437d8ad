"""Mksol (solver.py:508-565) -- the f1 'next' row: the device Horner chain
reproduces the reference's kernel vectors on generators from the
reference's own Krylov + Lingen (tests/golden/mksol_cases.npz)."""
import numpy as np
import pytest

import oracle as O
from helpers import fixture_sparse, rand_matrix, to_oracle
from paper_1402_3661_b200 import (
    B200Multiplier, PrimeModulus, SolverFailure, SparseMatrix, mksol_block, mksol_scalar,
    verify_kernel,
)
from paper_1402_3661_b200.modring import digit_count, ints_to_limbs, ints_to_planes, limbs_to_ints, planes_to_ints
from paper_1402_3661_b200.solver import _mksol_core


def _cases():
    z = O.load_golden("mksol_cases.npz")
    out = []
    for i in range(int(z["ncases"])):
        p = f"m{i}_"
        A = fixture_sparse(z, p)
        Y = [O.bytes_to_ints(y) for y in z[p + "Y"]]
        polys = [O.bytes_to_ints(pl)[:n] for pl, n in zip(z[p + "polys"], z[p + "plen"])]
        out.append((A, Y, polys, O.bytes_to_ints(z[p + "w"]), [int(x) for x in z[p + "counts"]]))
    return out


class _OracleMultiplier:
    """TEST INFRASTRUCTURE: the multiplier protocol over the CPU oracle."""

    def __init__(self, A):
        self.orc, self.size, self.mod, self.count = to_oracle(A), A.nrows, A.mod, 0

    def apply(self, planes):
        self.count += 1
        u = O.ints_to_limbs(planes_to_ints(planes), self.mod.limbs)
        return ints_to_planes(O.limbs_to_ints(self.orc.spmv_limbs(u)), planes.shape[1])


def test_generic_mksol_path_matches_reference_on_cpu():
    for A, Y, polys, w, (horner, tail, ver) in _cases():
        mul = _OracleMultiplier(A)
        P = digit_count(A.mod.ell)
        kv = _mksol_core(mul, [ints_to_planes(y, P) for y in Y], polys, A.mod)
        assert kv.w == w and kv.horner_spmvs == horner and kv.tail_spmvs == tail and kv.verified


@pytest.mark.gpu
def test_device_mksol_matches_reference():
    for A, Y, polys, w, (horner, tail, ver) in _cases():
        mul = B200Multiplier(A)
        kv = mksol_block(A, Y, type("G", (), {"polys": polys})(), mul=mul)
        assert kv.w == w
        assert (kv.horner_spmvs, kv.tail_spmvs, kv.verified) == (horner, tail, True)
        assert mul.count == horner + tail + 1
        assert verify_kernel(A, kv.w)


@pytest.mark.gpu
def test_mksol_tail_peels_common_factor():
    # generators sharing X^2: w = G(B) y is peeled by B until B w = 0
    mod = PrimeModulus(2**61 - 1)
    # B: nilpotent shift  e_i -> e_{i+1}
    n = 6
    B = SparseMatrix.from_rows(mod, n, n, [[]] + [[(i - 1, 1)] for i in range(1, n)])
    y = [0, 0, 0, 1, 0, 0]
    # F(X) = X^3: G = 1, val = 3; w = y = e3, peeled to e5 (B e5 = 0)
    kv = mksol_scalar(B, y, [0, 0, 0, 1])
    assert (kv.horner_spmvs, kv.tail_spmvs) == (0, 2) and kv.verified
    assert kv.w == [0, 0, 0, 0, 0, 1] and verify_kernel(B, kv.w)
    # the generic (reference) loop agrees
    P = digit_count(mod.ell)
    kv2 = _mksol_core(_OracleMultiplier(B), [ints_to_planes(y, P)], [[0, 0, 0, 1]], mod)
    assert kv2.w == kv.w and kv2.tail_spmvs == 2


@pytest.mark.gpu
def test_mksol_identity_fails_like_reference():
    mod = PrimeModulus(2**61 - 1)
    I = SparseMatrix.from_rows(mod, 4, 4, [[(i, 1)] for i in range(4)])
    with pytest.raises(SolverFailure):
        mksol_scalar(I, [1, 2, 3, 4], [mod.ell - 1, 1])  # X - 1 annihilates I: w = 0


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 31, 64, 160, 217, 256, 300, 650])
@pytest.mark.parametrize("k,extreme", [(1, False), (8, False), (64, True), (37, False)])
def test_lincomb_widths_vs_python(bits, k, extreme):
    # Mksol's combination dst = acc + sum_j c_j y_j (solver.py:522-536):
    # lazy 16-bit-digit columns for L <= 8, Montgomery products above;
    # extreme: every value l - 1 with the maximum k = 64 vectors
    from paper_1402_3661_b200.device import DeviceVector, Field, lincomb
    from paper_1402_3661_b200.modring import next_prime
    ell = 3 if bits == 2 else next_prime((1 << bits) - (1 << (bits // 2)))
    if ell.bit_length() > bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits * 100 + k)
    n = 1000
    f = Field(mod, 0)
    if extreme:
        ys = [[ell - 1] * n for _ in range(k)]
        cs = [ell - 1] * k
        acc = [ell - 1] * n
    else:
        ys = [mod.random_residues(rng, n) for _ in range(k)]
        cs = mod.random_residues(rng, k)
        acc = mod.random_residues(rng, n)
    dys = []
    for y in ys:
        d = DeviceVector(f, n)
        d.upload_limbs(ints_to_limbs(y, mod.limbs))
        dys.append(d)
    da, dst = DeviceVector(f, n), DeviceVector(f, n)
    da.upload_limbs(ints_to_limbs(acc, mod.limbs))
    lincomb(f, dys, cs, dst, da)
    got = limbs_to_ints(dst.download_limbs())
    want = [(a + sum(c * y[i] for c, y in zip(cs, ys))) % ell for i, a in enumerate(acc)]
    assert got == want
    lincomb(f, dys, cs, dst)  # no accumulator
    assert limbs_to_ints(dst.download_limbs()) == [sum(c * y[i] for c, y in zip(cs, ys)) % ell
                                                   for i in range(n)]


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 31, 64, 160, 217, 256])
@pytest.mark.parametrize("n,extreme", [(1, False), (3, False), (8, False), (8, True)])
def test_tensor_core_combination_vs_python(bits, n, extreme):
    # sld_lcset: dst = acc + sum_s c_s y_s as a u8 digit GEMM (tcgen05
    # kind::i8) with the mod-l reduction in the epilogue; rows spanning
    # several 128-row tiles and a ragged last tile; zero coefficients
    from paper_1402_3661_b200.device import DeviceVector, Field, LinCombSet
    from paper_1402_3661_b200.modring import next_prime
    ell = 3 if bits == 2 else next_prime((1 << bits) - (1 << (bits // 2)))
    if ell.bit_length() > bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits * 10 + n)
    rows = 20000 + 77
    f = Field(mod, 0)
    if extreme:
        ys = [[ell - 1] * rows for _ in range(n)]
        acc = [ell - 1] * rows
    else:
        ys = [mod.random_residues(rng, rows) for _ in range(n)]
        acc = mod.random_residues(rng, rows)
    dys = []
    for y in ys:
        d = DeviceVector(f, rows)
        d.upload_limbs(ints_to_limbs(y, mod.limbs))
        dys.append(d)
    da, dst = DeviceVector(f, rows), DeviceVector(f, rows)
    da.upload_limbs(ints_to_limbs(acc, mod.limbs))
    lc = LinCombSet(f, dys, rows)
    for trial in range(3):
        cs = [ell - 1] * n if extreme else mod.random_residues(rng, n)
        if trial == 2 and n > 1:
            cs[0] = 0
        lc.apply(cs, dst, da if trial != 1 else None)
        got = limbs_to_ints(dst.download_limbs())
        base = acc if trial != 1 else [0] * rows
        want = [(a + sum(c * y[i] for c, y in zip(cs, ys))) % ell for i, a in enumerate(base)]
        assert got == want, trial
    lc.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "unfused"])
def test_device_mksol_fused_step_matches_reference(monkeypatch, mode):
    # the Horner step as ONE product (combination in the last pass's
    # epilogue, sld_spmv_mksol) and as SpMV + combination kernel: both give
    # the reference's kernel vectors.  SLD_SHORT=0 keeps these small
    # matrices on the pass layout the fused step runs on.
    from paper_1402_3661_b200.device import DeviceMatrix
    monkeypatch.setenv("SLD_SHORT", "0")
    monkeypatch.setenv("SLD_MKSOL_FUSED", "1" if mode == "fused" else "0")
    calls = []
    orig = DeviceMatrix.spmv_mksol
    monkeypatch.setattr(DeviceMatrix, "spmv_mksol", lambda self, *a: (calls.append(1), orig(self, *a)))
    for A, Y, polys, w, (horner, tail, ver) in _cases():
        mul = B200Multiplier(A)
        kv = mksol_block(A, Y, type("G", (), {"polys": polys})(), mul=mul)
        assert kv.w == w
        assert (kv.horner_spmvs, kv.tail_spmvs, kv.verified) == (horner, tail, True)
    assert (len(calls) > 0) == (mode == "fused")


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [31, 64, 160, 202, 256])
@pytest.mark.parametrize("n,extreme", [(1, False), (3, False), (8, False), (8, True)])
@pytest.mark.parametrize("stripes", [1, 3])
def test_spmv_mksol_vs_python(monkeypatch, bits, n, extreme, stripes):
    # out = A in + sum_s c_s y_s mod l in one product: +-1 / small / full
    # entries, a dense column, several column stripes (slot-indexed partials
    # before the fused last pass), padding slots; extreme: every y, c and
    # input l - 1
    from helpers import rand_matrix
    from paper_1402_3661_b200.device import DeviceMatrix, DeviceVector
    from paper_1402_3661_b200.modring import next_prime
    monkeypatch.setenv("SLD_SHORT", "0")
    ell = next_prime((1 << bits) - (1 << (bits // 2)))
    if ell.bit_length() > bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits * 7 + n + stripes)
    nr = 1000
    A = rand_matrix(mod, rng, nr, nr - 1, 14, dense=1)
    dm = DeviceMatrix(A, stripe_cols=(A.total_cols + stripes - 1) // stripes if stripes > 1 else 0)
    assert dm.info()["stripes"] == stripes
    f = dm.field
    ys = [[ell - 1] * nr if extreme else mod.random_residues(rng, nr) for _ in range(n)]
    u = [ell - 1] * A.total_cols if extreme else mod.random_residues(rng, A.total_cols)
    dys = []
    for y in ys:
        d = DeviceVector(f, A.total_cols)
        d.upload_limbs(ints_to_limbs(y + [0] * (A.total_cols - nr), mod.limbs))
        dys.append(d)
    assert dm.mksol_bind(dys)
    vin, vout = dm.vector(), dm.vector()
    vin.upload_limbs(ints_to_limbs(u, mod.limbs))
    Au = O.limbs_to_ints(to_oracle(A).spmv_limbs(O.ints_to_limbs(u, mod.limbs)))
    for trial in range(3):
        cs = [ell - 1] * n if extreme else mod.random_residues(rng, n)
        if trial == 1:
            cs[0] = 0
        dm.spmv_mksol(vin, vout, cs)
        got = limbs_to_ints(vout.download_limbs())[:nr]
        want = [(Au[i] + sum(c * y[i] for c, y in zip(cs, ys))) % ell for i in range(nr)]
        assert got == want, trial
    dm.mksol_bind([])
    with pytest.raises(ValueError):
        dm.spmv_mksol(vin, vout, cs)  # unbound


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [2, 31, 160, 202, 256])
@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("n,extreme", [(1, False), (8, False), (8, True)])
def test_batched_combination_vs_python(bits, K, n, extreme):
    # sld_lcset_apply_batch: K Horner steps' combinations from one pass over
    # the tiled y (K C' tiles, K TMEM accumulators per buffer), ragged tiles
    from paper_1402_3661_b200.device import DeviceVector, Field, LinCombSet
    from paper_1402_3661_b200.modring import next_prime
    ell = 3 if bits == 2 else next_prime((1 << bits) - (1 << (bits // 2)))
    if ell.bit_length() > bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits * 10 + n + K)
    rows = 20000 + 77
    f = Field(mod, 0)
    ys = [[ell - 1] * rows if extreme else mod.random_residues(rng, rows) for _ in range(n)]
    dys = []
    for y in ys:
        d = DeviceVector(f, rows)
        d.upload_limbs(ints_to_limbs(y, mod.limbs))
        dys.append(d)
    lc = LinCombSet(f, dys, rows)
    dsts = [DeviceVector(f, rows) for _ in range(K)]
    sets = [[ell - 1] * n if extreme else mod.random_residues(rng, n) for _ in range(K)]
    sets[-1] = [0] * n  # a padded (all-zero) step
    lc.apply_batch(sets, dsts)
    for cs, d in zip(sets, dsts):
        want = [sum(c * y[i] for c, y in zip(cs, ys)) % ell for i in range(rows)]
        assert limbs_to_ints(d.download_limbs()) == want
    lc.close()


@pytest.mark.gpu
@pytest.mark.parametrize("short", ["0", "1"])
@pytest.mark.parametrize("stripes", [1, 3])
def test_spmv_add_vs_oracle(monkeypatch, short, stripes):
    # sld_spmv_add: out = A in + addv, addv from a slot-ordered combination
    # set (sld_lcset_create_slots), the addition in the last pass (pass and
    # short-row layouts, one or several stripes)
    from paper_1402_3661_b200.device import DeviceMatrix, DeviceVector, LinCombSet
    monkeypatch.setenv("SLD_SHORT", short)
    mod = PrimeModulus(0xc152a866f35196bb08ec18cd24e7a4f6d2ac709d)
    rng = np.random.default_rng(7 + stripes)
    nr = 3000
    A = rand_matrix(mod, rng, nr, nr - 1, 14, dense=1)
    dm = DeviceMatrix(A, stripe_cols=(A.total_cols + stripes - 1) // stripes if stripes > 1 else 0)
    u = mod.random_residues(rng, nr)
    ys = [mod.random_residues(rng, nr), [mod.ell - 1] * nr]
    cs = [mod.random_residues(rng, 2), [mod.ell - 1, mod.ell - 1]]
    dys = []
    for y in ys:
        d = dm.vector()
        d.upload_limbs(ints_to_limbs(y, mod.limbs))
        dys.append(d)
    lcs = LinCombSet(dm.field, dys, dm.total_cols, matrix=dm)
    vas = [DeviceVector(dm.field, dm.nslots) for _ in range(2)]
    lcs.apply_batch(cs, vas)
    vin, vout = dm.vector(), dm.vector()
    vin.upload_limbs(ints_to_limbs(u, mod.limbs))
    Au = O.limbs_to_ints(to_oracle(A).spmv_limbs(O.ints_to_limbs(u, mod.limbs)))
    for c, va in zip(cs, vas):
        dm.spmv_add(vin, vout, va)
        want = [(Au[i] + c[0] * ys[0][i] + c[1] * ys[1][i]) % mod.ell for i in range(nr)]
        assert limbs_to_ints(vout.download_limbs())[:nr] == want
    lcs.close()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", ["0", "2", "4"])
def test_device_mksol_batched_matches_reference(monkeypatch, batch):
    # the Horner loop with K steps' combinations batched (default K = 4)
    # against the reference's kernel vectors; SLD_MKSOL_BATCH=0 is the
    # per-step combination kernel
    from paper_1402_3661_b200.device import DeviceMatrix
    monkeypatch.setenv("SLD_MKSOL_BATCH", batch)
    calls = []
    orig = DeviceMatrix.spmv_add
    monkeypatch.setattr(DeviceMatrix, "spmv_add", lambda self, *a: (calls.append(1), orig(self, *a)))
    for A, Y, polys, w, (horner, tail, ver) in _cases():
        mul = B200Multiplier(A)
        kv = mksol_block(A, Y, type("G", (), {"polys": polys})(), mul=mul)
        assert kv.w == w
        assert (kv.horner_spmvs, kv.tail_spmvs, kv.verified) == (horner, tail, True)
    assert (len(calls) > 0) == (batch != "0")

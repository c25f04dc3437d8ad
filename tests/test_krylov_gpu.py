"""Device-resident Krylov chain parity: the cfg1 200-SpMV golden chain of the
reference (bit-exact terms and final iterate), the reference's Krylov cases
(unit and dense X, several chains), SpMV counts, checkpoint chunking and
thread independence."""
import numpy as np
import pytest

import oracle as O
from helpers import fixture_sparse, rand_matrix, to_oracle
from paper_1402_3661_b200 import (
    B200Multiplier, BlockingParams, DenseRows, PrimeModulus, SparseMatrix, UnitRows, draw_blocks,
    krylov_block, krylov_column, krylov_length, krylov_scalar,
)
from paper_1402_3661_b200.modring import digit_count, ints_to_planes, planes_to_ints

pytestmark = pytest.mark.gpu


def test_cfg1_golden_200_steps():
    z = O.load_golden("cfg1.npz")
    A = fixture_sparse(z, "")
    y = O.bytes_to_ints(z["y"])
    X = UnitRows(z["xrows"].tolist())
    seq = krylov_block(A, X, [y], 200)
    want = [O.bytes_to_ints(t) for t in z["terms"]]
    assert seq.columns[0] == want
    assert seq.spmvs_per_column == [200]
    mul = B200Multiplier(A)
    P = digit_count(A.mod.ell)
    terms, v, spmvs = krylov_column(mul, X, ints_to_planes(y, P), 200)
    assert spmvs == 200 and mul.count == 200
    assert planes_to_ints(v) == O.bytes_to_ints(z["v200"])
    # one product through the plugin's apply() as well
    m2 = B200Multiplier(A)
    assert planes_to_ints(m2.apply(ints_to_planes(y, P))) == O.bytes_to_ints(z["v1"])
    assert m2.count == 1


def test_reference_krylov_cases():
    z = O.load_golden("krylov_cases.npz")
    for i in range(int(z["ncases"])):
        p = f"k{i}_"
        A = fixture_sparse(z, p)
        count, mode = int(z[p + "count"]), str(z[p + "mode"])
        Y = [O.bytes_to_ints(y) for y in z[p + "Y"]]
        if mode == "unit":
            X = UnitRows(z[p + "xrows"].tolist())
        else:
            X = DenseRows([O.bytes_to_ints(x) for x in z[p + "xdense"]], A.mod)
        seq = krylov_block(A, X, Y, count)
        for j in range(len(Y)):
            want = [O.bytes_to_ints(t) for t in z[p + "terms"][j]]
            assert seq.columns[j] == want, (i, j)


@pytest.mark.parametrize("count", [0, 1, 2, 31, 32, 33, 64, 65, 1100])
def test_chain_lengths_vs_oracle(count):
    # odd/even lengths cross the CUDA-graph (32 products) and drain (1024) boundaries
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(count)
    A = rand_matrix(mod, rng, 90, 89, 9, dense=1)  # square: 89 sparse + 1 dense column
    y = mod.random_residues(rng, 90)
    rows = [3, 50, 89]
    orc = to_oracle(A)
    ot, ov = O.krylov_unit(orc, O.ints_to_limbs(y, mod.limbs), rows, count)
    mul = B200Multiplier(A)
    terms, v, spmvs = krylov_column(mul, UnitRows(rows), ints_to_planes(y, digit_count(mod.ell)), count)
    assert spmvs == count
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert planes_to_ints(v) == O.limbs_to_ints(ov)


def test_dense_x_vs_oracle():
    mod = PrimeModulus(0xc152a866f35196bb08ec18cd24e7a4f6d2ac709d)
    rng = np.random.default_rng(11)
    A = rand_matrix(mod, rng, 300, 300, 12)
    y = mod.random_residues(rng, 300)
    X = DenseRows([mod.random_residues(rng, 300) for _ in range(4)], mod)
    orc = to_oracle(A)
    x = np.stack([O.ints_to_limbs(v, mod.limbs) for v in X.vectors])
    ot, _ = O.krylov_dense(orc, O.ints_to_limbs(y, mod.limbs), x, 40)
    terms, _, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, digit_count(mod.ell)), 40)
    assert terms == [O.limbs_to_ints(t) for t in ot]


@pytest.mark.parametrize("bits", [2, 31, 64, 127, 202, 256, 300, 650])
@pytest.mark.parametrize("extreme", [False, True])
@pytest.mark.parametrize("tc", ["1", "0"])
def test_dense_x_widths_vs_oracle(bits, extreme, tc, monkeypatch):
    # L <= 8: tensor-core byte-digit GEMM (tc=1: tcgen05 kind::i8, TMEM) or
    # lazy exact dot products (tc=0: 16-bit digit x limb columns); one fold
    # and Barrett per term either way.  L > 8: Montgomery products.
    # extreme: x = v = l - 1 on a longer vector drives every column to its bound
    monkeypatch.setenv("SLD_DENSE_TC", tc)
    from paper_1402_3661_b200.modring import next_prime
    ell = 3 if bits == 2 else next_prime((1 << bits) - (1 << (bits // 2)))
    if ell.bit_length() > bits:
        ell = next_prime(1 << (bits - 1))
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits + (7 if extreme else 0))
    n = 70000 if extreme else 200  # > 512 K tiles of the GEMM: several CTAs
    A = rand_matrix(mod, rng, n, n, 6)
    if extreme:
        y = [ell - 1] * n
        xs = [[ell - 1] * n for _ in range(3)]
    else:
        y = mod.random_residues(rng, n)
        xs = [mod.random_residues(rng, n) for _ in range(3)]
    X = DenseRows(xs, mod)
    orc = to_oracle(A)
    x = np.stack([O.ints_to_limbs(v, mod.limbs) for v in xs])
    ot, _ = O.krylov_dense(orc, O.ints_to_limbs(y, mod.limbs), x, 6)
    terms, _, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, digit_count(mod.ell)), 6)
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert terms[0] == [sum(a * b for a, b in zip(xv, y)) % ell for xv in xs]


@pytest.mark.parametrize("bits", [64, 256])
def test_dense_x_tc_at_accumulator_cap(bits, monkeypatch):
    # every CTA of the tcgen05 digit GEMM sums the largest K the
    # s32 TMEM accumulator allows (TC_MAX_K_PER_CTA = 32768 bytes) with
    # 0xFF-dense digits (x = v = l - 1, l just below 2^bits): 32768 * 255^2 <
    # 2^31, so the sums are exact without relying on wrap-around
    monkeypatch.setenv("SLD_DENSE_TC", "1")
    monkeypatch.setenv("SLD_TC_MAX_K", "1")
    from paper_1402_3661_b200.modring import prev_prime
    ell = prev_prime(1 << bits)
    mod = PrimeModulus(ell)
    rng = np.random.default_rng(bits)
    n = 2 * 32768 + 4096  # 3 CTAs: two at the cap, one partial
    A = rand_matrix(mod, rng, n, n, 4)
    y = [ell - 1] * n
    xs = [[ell - 1] * n for _ in range(4)]
    X = DenseRows(xs, mod)
    orc = to_oracle(A)
    x = np.stack([O.ints_to_limbs(v, mod.limbs) for v in xs])
    ot, _ = O.krylov_dense(orc, O.ints_to_limbs(y, mod.limbs), x, 3)
    terms, _, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, digit_count(mod.ell)), 3)
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert terms[0] == [n % ell] * 4


def test_krylov_scalar_identity_and_zero():
    mod = PrimeModulus(1009)
    rng = np.random.default_rng(1)
    I = SparseMatrix.from_rows(mod, 6, 6, [[(i, 1)] for i in range(6)])
    x = [int(v) for v in rng.integers(0, 1009, 6)]
    y = [int(v) for v in rng.integers(0, 1009, 6)]
    a0 = sum(a * b for a, b in zip(x, y)) % 1009
    assert krylov_scalar(I, x, y, count=9) == [a0] * 9
    Z = SparseMatrix.from_rows(mod, 5, 5, [[] for _ in range(5)])
    assert krylov_scalar(Z, x[:5], y[:5], count=8) == [sum(a * b for a, b in zip(x[:5], y[:5])) % 1009] + [0] * 7


def test_spmv_counts_and_column_isolation():
    mod = PrimeModulus(2**61 - 1)
    rng = np.random.default_rng(13)
    A = rand_matrix(mod, rng, 60, 60, 6)
    bp = BlockingParams(3, 6)
    X, Y = draw_blocks(mod, 60, bp, rng, "unit")
    count = krylov_length(60, bp)
    assert count == 20 + 10 + 32
    joint = krylov_block(A, X, Y, count)
    assert joint.spmvs_per_column == [count] * 3
    for j in range(3):
        alone = krylov_block(A, X, [Y[j]], count, contexts=1)
        assert alone.columns[0] == joint.columns[j]


class _RecordingCheckpoint:
    """Minimal checkpoint with the reference's hook contract
    (checkpoint.py:177-200): flush every `every` steps per column."""

    def __init__(self, every):
        self.every = every
        self._since_flush = {}
        self._session_steps = 0
        self.halt_after = None
        self.flushes = []

    def on_step(self, j, terms, v):
        self._session_steps += 1
        self._since_flush[j] = self._since_flush.get(j, 0) + 1
        if self._since_flush[j] >= self.every:
            self.flush(j, terms, v)

    def flush(self, j, terms, v):
        self.flushes.append((j, len(terms), planes_to_ints(v)))
        self._since_flush[j] = 0


def test_checkpoint_flushes_carry_exact_iterates():
    mod = PrimeModulus(2**127 - 1)
    rng = np.random.default_rng(21)
    A = rand_matrix(mod, rng, 50, 50, 8)
    y = mod.random_residues(rng, 50)
    ck = _RecordingCheckpoint(every=7)
    P = digit_count(mod.ell)
    terms, v, _ = krylov_column(B200Multiplier(A), UnitRows([1, 2]), ints_to_planes(y, P), 30,
                                checkpoint=ck)
    orc = to_oracle(A)
    expect_v = O.ints_to_limbs(y, mod.limbs)
    iterates = []
    for _ in range(30):
        expect_v = orc.spmv_limbs(expect_v)
        iterates.append(O.limbs_to_ints(expect_v))
    steps_flushed = [n for _, n, _ in ck.flushes]
    assert steps_flushed == [7, 14, 21, 28, 30]
    for (_, n, vv) in ck.flushes:
        assert vv == iterates[n - 1]


def test_resume_matches_uninterrupted():
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(22)
    A = rand_matrix(mod, rng, 64, 64, 7)
    y = mod.random_residues(rng, 64)
    P = digit_count(mod.ell)
    X = UnitRows([0, 5])
    full, vfull, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, P), 50)
    part, vpart, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, P), 23)
    rest, vrest, n = krylov_column(B200Multiplier(A), X, vpart, 50, start_terms=part)
    assert n == 27 and rest == full and np.array_equal(vrest, vfull)


@pytest.mark.parametrize("G,bits,stripe", [(2, 200, 0), (4, 200, 0), (2, 480, 0), (2, 200, 37), (4, 127, 50)])
def test_chain_groups_match_oracle(G, bits, stripe):
    # G interleaved chains per matrix pass (one gather request per column for
    # all G residues) give exactly the single-chain sequences
    from paper_1402_3661_b200 import B200ChainGroup
    from paper_1402_3661_b200.modring import next_prime
    mod = PrimeModulus(next_prime(1 << (bits - 1)))
    rng = np.random.default_rng(G * 1000 + bits + stripe)
    A = rand_matrix(mod, rng, 160, 158, 11, dense=2)
    Ys = [mod.random_residues(rng, 160) for _ in range(G)]
    rows = [0, 77, 159]
    P = digit_count(mod.ell)
    grp = B200ChainGroup(A, chains=G, stripe_cols=stripe)
    terms, vs = grp.krylov(UnitRows(rows), [ints_to_planes(y, P) for y in Ys], 37)
    orc = to_oracle(A)
    for g in range(G):
        ot, ov = O.krylov_unit(orc, O.ints_to_limbs(Ys[g], mod.limbs), rows, 37)
        assert terms[g] == [O.limbs_to_ints(t) for t in ot], g
        assert planes_to_ints(vs[g]) == O.limbs_to_ints(ov), g
    assert grp.count == 37


def test_krylov_block_grouped_equals_ungrouped():
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(31)
    A = rand_matrix(mod, rng, 90, 90, 8)
    bp = BlockingParams(5, 10)
    X, Y = draw_blocks(mod, 90, bp, rng, "unit")
    one = krylov_block(A, X, Y, 45, contexts=1)
    two = krylov_block(A, X, Y, 45, chains_per_gpu=2)
    four = krylov_block(A, X, Y, 45, chains_per_gpu=4)
    assert one.columns == two.columns == four.columns


def test_native_checkpoint_halt_and_resume(tmp_path):
    # a device chain under the native CheckpointManager: halt after a flush,
    # resume from the files, finish -- identical to the uninterrupted chain
    from paper_1402_3661_b200 import CheckpointManager, HaltRequested
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(23)
    A = rand_matrix(mod, rng, 64, 64, 7)
    y = mod.random_residues(rng, 64)
    P = digit_count(mod.ell)
    X = UnitRows([0, 5])
    full, vfull, _ = krylov_column(B200Multiplier(A), X, ints_to_planes(y, P), 50)
    ck = CheckpointManager(tmp_path, mod, every=8, halt_after=19, async_writes=True)
    ck.m = 2
    with pytest.raises(HaltRequested):
        krylov_column(B200Multiplier(A), X, ints_to_planes(y, P), 50, checkpoint=ck)
    terms, v = CheckpointManager(tmp_path, mod).load_column(0)
    assert len(terms) == 19 and terms == full[:19]
    rest, vrest, n = krylov_column(B200Multiplier(A), X, v, 50, start_terms=terms)
    assert n == 31 and rest == full and np.array_equal(vrest, vfull)


def test_reference_loop_stays_on_device():
    # the reference's krylov_column loop body, verbatim in effect
    # (solver.py:209-214: project, apply, on_step), driven with B200Multiplier:
    # apply() returns DevicePlanes, the projection reads m rows, and the next
    # apply() consumes the device iterate -- results equal the oracle
    from paper_1402_3661_b200.device import DevicePlanes
    mod = PrimeModulus(2**200 - 75)
    rng = np.random.default_rng(31)
    A = rand_matrix(mod, rng, 120, 119, 9, dense=1)
    y = mod.random_residues(rng, 120)
    P = digit_count(mod.ell)
    X = UnitRows([2, 7, 100])
    mul = B200Multiplier(A)
    terms, v = [], ints_to_planes(y, P)
    for _ in range(30):
        terms.append(X.project(v))
        v = mul.apply(v)
        assert isinstance(v, DevicePlanes) and v._host is None  # nothing downloaded
    orc = to_oracle(A)
    ot, ov = O.krylov_unit(orc, O.ints_to_limbs(y, mod.limbs), X.rows, 30)
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert planes_to_ints(v) == O.limbs_to_ints(ov)
    assert mul.count == 30
    # numpy behaviour on the device iterate
    host = np.asarray(v)
    assert host.shape == (120, P) and host.dtype == np.uint64
    assert np.array_equal(v + 0, host) and bool(np.any(v)) and v.astype("<u2").shape == (120, P)
    assert np.array_equal(v[[5, 6]], host[[5, 6]]) and np.array_equal(v[3], host[3])
    with pytest.raises(ValueError):
        mul.apply(np.zeros((5, P), dtype=np.uint64))


@pytest.mark.parametrize("layout", ["split", "pass", "short"])
def test_krylov_chain_every_layout(layout, monkeypatch):
    # the device-resident chain (CUDA graphs of 32 products) on each SpMV
    # kernel family, 70 steps across the graph boundary, against the oracle
    from paper_1402_3661_b200 import _native
    env = {"split": {"SLD_SPLIT": "1", "SLD_SHORT": "0"}, "pass": {"SLD_SHORT": "0"},
           "short": {"SLD_SHORT": "1"}}[layout]
    if layout == "split" and _native.die_map(0) is None:
        pytest.skip("die map unavailable")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    mod = PrimeModulus(2**127 - 1)
    rng = np.random.default_rng(41)
    A = rand_matrix(mod, rng, 300, 299, 12, dense=1, full_frac=0.03)
    y = mod.random_residues(rng, 300)
    rows = [0, 150, 299]
    P = digit_count(mod.ell)
    mul = B200Multiplier(A, stripe_cols=100)
    terms, v, n = krylov_column(mul, UnitRows(rows), ints_to_planes(y, P), 70)
    orc = to_oracle(A)
    ot, ov = O.krylov_unit(orc, O.ints_to_limbs(y, mod.limbs), rows, 70)
    assert n == 70 and terms == [O.limbs_to_ints(t) for t in ot]
    assert planes_to_ints(v) == O.limbs_to_ints(ov)
    if layout == "split":
        assert mul.dm.info()["halves"] == 2


@pytest.mark.parametrize("slots", [2, 3])
def test_krylov_block_multi_device_slots(slots):
    # krylov_block's multi-GPU placement (round robin over devices, one host
    # thread and one shared device matrix per slot, solver.py:220-257) with
    # every slot mapped onto GPU 0: the code path of `slots` GPUs
    mod = PrimeModulus(2**127 - 1)
    rng = np.random.default_rng(40 + slots)
    A = rand_matrix(mod, rng, 120, 120, 9)
    bp = BlockingParams(5, 7)
    X, Y = draw_blocks(mod, 120, bp, rng, "unit")
    ref = krylov_block(A, X, Y, 33, contexts=1, devices=[0])
    multi = krylov_block(A, X, Y, 33, devices=[0] * slots)
    grouped = krylov_block(A, X, Y, 33, chains_per_gpu=2, devices=[0] * slots)
    assert multi.columns == ref.columns == grouped.columns
    assert multi.spmvs_per_column == [33] * 5
    orc = to_oracle(A)
    for j in range(5):
        ot, _ = O.krylov_unit(orc, O.ints_to_limbs(Y[j], mod.limbs), X.rows, 33)
        assert multi.columns[j] == [O.limbs_to_ints(t) for t in ot], j


@pytest.mark.parametrize("chain", ["1", "0"])
@pytest.mark.parametrize("bits,n,steps", [(31, 500, 37), (160, 2000, 1030), (202, 60000, 21), (256, 3000, 65)])
def test_persistent_chain_vs_oracle(chain, bits, n, steps, monkeypatch):
    # small one-pass matrices run many products per cooperative launch
    # (spmv_chain, grid barrier between products); SLD_CHAIN=0 forces the
    # per-product graphs.  n = 60000 leaves several slices per warp.
    monkeypatch.setenv("SLD_CHAIN", chain)
    from paper_1402_3661_b200 import corpus
    mod = corpus.random_prime(bits, np.random.default_rng(bits))
    rng = np.random.default_rng(n)
    if n > 5000:
        A = corpus.generate(corpus.CorpusProfile(n=n, gamma=20, dense_cols=1, seed=3), mod)
    else:
        A = rand_matrix(mod, rng, n, n - 1, 20, dense=1, full_frac=0.02)
    y = mod.random_residues(rng, n)
    rows = [0, n // 2, n - 1]
    ot, ov = O.krylov_unit(to_oracle(A), O.ints_to_limbs(y, mod.limbs), rows, steps)
    mul = B200Multiplier(A)
    terms, v, spmvs = krylov_column(mul, UnitRows(rows), ints_to_planes(y, digit_count(mod.ell)), steps)
    assert spmvs == steps
    assert terms == [O.limbs_to_ints(t) for t in ot]
    assert planes_to_ints(v) == O.limbs_to_ints(ov)

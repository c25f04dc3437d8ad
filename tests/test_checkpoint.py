"""CheckpointManager (sldlag/checkpoint.py:67-200 protocol) with the native
SLDQ / SLDV writers: flush cadence, halt-after-flush, resume state, attempt
metadata, async writes.  The device chain under it is tested in
test_krylov_gpu.py; these run on the host."""
import numpy as np
import pytest

from paper_1402_3661_b200 import (
    BlockingParams, CheckpointManager, FormatError, HaltRequested, PrimeModulus, UnitRows,
    load_terms, load_vector,
)
from paper_1402_3661_b200.modring import digit_count, ints_to_planes, planes_to_ints

MOD = PrimeModulus(2**200 - 75)


def _fake_chain(ck, j, steps, rng, m=2, n=40):
    P = digit_count(MOD.ell)
    terms = []
    v = None
    for _ in range(steps):
        vals = MOD.random_residues(rng, n)
        v = ints_to_planes(vals, P)
        terms.append(vals[:m])
        ck.on_step(j, terms, v)
    return terms, v


@pytest.mark.parametrize("async_writes", [False, True])
def test_flush_cadence_and_contents(tmp_path, async_writes):
    ck = CheckpointManager(tmp_path, MOD, every=5, async_writes=async_writes)
    ck.m = 2
    rng = np.random.default_rng(1)
    terms, v = _fake_chain(ck, 3, 12, rng)
    assert ck.steps_until_flush(3) == 3
    ck.wait()
    got_terms, got_v = ck.load_column(3)
    assert len(got_terms) == 10  # last flush at step 10
    assert got_terms == [list(t) for t in terms[:10]]
    ck.flush(3, terms, v)
    ck.wait()
    got_terms, got_v = ck.load_column(3)
    assert got_terms == [list(t) for t in terms] and planes_to_ints(got_v) == planes_to_ints(v)
    assert load_vector(tmp_path / "iter" / "col_3.sldv")[0] == planes_to_ints(v)
    assert load_terms(tmp_path / "seq" / "col_3.sldq")[1] == 2


def test_halt_after_flushes_first(tmp_path):
    ck = CheckpointManager(tmp_path, MOD, every=100, halt_after=7, async_writes=True)
    ck.m = 2
    rng = np.random.default_rng(2)
    with pytest.raises(HaltRequested):
        _fake_chain(ck, 0, 20, rng)
    terms, _ = ck.load_column(0)
    assert len(terms) == 7


def test_attempt_meta_roundtrip(tmp_path):
    ck = CheckpointManager(tmp_path, MOD)
    rng = np.random.default_rng(3)
    bp = BlockingParams(2, 4)
    Y = [MOD.random_residues(rng, 30) for _ in range(2)]
    X = UnitRows([1, 4, 9, 16])
    X2, Y2 = ck.begin_attempt(0, X, Y, bp, 99, "unit")
    assert X2 is X and Y2 is Y
    ck2 = CheckpointManager(tmp_path, MOD)
    X3, Y3 = ck2.begin_attempt(0, UnitRows([0]), [[0] * 30] * 2, bp, 99, "unit")
    assert X3.rows == [1, 4, 9, 16] and Y3 == Y
    with pytest.raises(FormatError):
        CheckpointManager(tmp_path, MOD).begin_attempt(0, X, Y, bp, 98, "unit")
    ck2.discard_attempt()
    assert CheckpointManager(tmp_path, MOD).attempt == 1


class _CountingKrylov:
    """A `.krylov` multiplier whose iterate encodes how many products it has
    taken (row 0, digit 0), so a flushed iterate can be matched against the
    flushed term count."""

    def __init__(self, n=8):
        self.mod, self.size, self.count = MOD, n, 0

    def krylov(self, xblock, v, steps):
        import time
        k = int(np.asarray(v)[0, 0])
        out = np.array(v, dtype=np.uint64, copy=True)
        out[0, 0] = k + steps
        time.sleep(0.002 * steps)  # let the other column's thread interleave
        self.count += steps
        return [[k + i] for i in range(steps)], out


@pytest.mark.parametrize("halt_after", [5, 10, 17])
def test_concurrent_columns_halt_on_consistent_iterates(tmp_path, halt_after):
    # with columns on concurrent threads, another column's steps
    # must not make a device chunk halt mid-replay (terms k, iterate k + r)
    from paper_1402_3661_b200.solver import krylov_block
    ck = CheckpointManager(tmp_path, MOD, every=6, halt_after=halt_after)
    ck.m = 1
    muls = [_CountingKrylov() for _ in range(3)]
    with pytest.raises(HaltRequested):
        krylov_block(None, UnitRows([0]), [[0] * 8] * 3, 40, muls=muls, checkpoint=ck, contexts=3)
    ck.wait()
    seen = 0
    for j in range(3):
        st = ck.load_column(j)
        if st is None:
            continue
        terms, v = st
        seen += 1
        assert int(v[0, 0]) == len(terms), f"column {j}: iterate after {int(v[0, 0])} products, {len(terms)} terms"
        assert [t[0] for t in terms] == list(range(len(terms)))
    assert seen >= 1


def test_async_writer_error_surfaces_on_next_call(tmp_path):
    ck = CheckpointManager(tmp_path, MOD, every=3, async_writes=True)
    ck.m = 2
    ck._errors.append(OSError("disk full"))  # as the writer thread records it
    with pytest.raises(OSError):
        ck.on_step(0, [[1, 2]], ints_to_planes([0] * 4, digit_count(MOD.ell)))

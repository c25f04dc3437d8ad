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

"""Host-side logic that needs no GPU: residue formats, the modulus object,
matrix construction/validation, the reference's RNG draws (blocks, primes),
Krylov lengths, planted kernels (checked with the CPU oracle)."""
import numpy as np
import pytest

import oracle as O
from helpers import to_oracle
from paper_1402_3661_b200 import (
    BlockingParams, PrimeModulus, SparseMatrix, classify, digit_count, draw_blocks, ints_to_limbs,
    ints_to_planes, krylov_length, limbs_to_ints, limbs_to_planes, planes_to_ints, planes_to_limbs,
)
from paper_1402_3661_b200 import corpus
from paper_1402_3661_b200.modring import bytes_to_planes, planes_to_bytes


def test_planes_limbs_roundtrip():
    rng = np.random.default_rng(1)
    mod = PrimeModulus(2**521 - 1)
    vals = mod.random_residues(rng, 200) + [0, 1, mod.ell - 1]
    P = digit_count(mod.ell)
    pl = ints_to_planes(vals, P)
    assert planes_to_ints(pl) == vals
    li = planes_to_limbs(pl, mod.limbs)
    assert limbs_to_ints(li) == vals
    assert np.array_equal(limbs_to_planes(li, P), pl)
    assert np.array_equal(li, ints_to_limbs(vals, mod.limbs))


def test_serialization_matches_golden_bytes():
    z = O.load_golden("cfg1.npz")
    ell = int(str(z["ell"]), 16)
    mod = PrimeModulus(ell)
    y = O.bytes_to_ints(z["y"])
    blob = planes_to_bytes(ints_to_planes(y, digit_count(ell)), mod.byte_width)
    assert blob == z["y"].tobytes() == mod.vector_to_bytes(y)
    back = bytes_to_planes(blob, len(y), mod.byte_width, digit_count(ell))
    assert planes_to_ints(back) == y


def test_prime_modulus_contract():
    with pytest.raises(ValueError):
        PrimeModulus(1008)
    with pytest.raises(ValueError):
        PrimeModulus(91)  # 7 * 13
    with pytest.raises(ValueError):
        PrimeModulus(2**1025 - 1)
    m = PrimeModulus(2**127 - 1)
    assert m.limbs == 4 and m.byte_width == 16 and m.check(5) == 5
    with pytest.raises(ValueError):
        m.check(m.ell)


def test_reference_draws_reproduced():
    # cfg1: `sldlag gen --ell-bits 160 --seed 1` prime and attempt-0 blocks
    z = O.load_golden("cfg1.npz")
    mod = corpus.random_prime(160, np.random.default_rng(1))
    assert hex(mod.ell) == str(z["ell"])
    drng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(0,)))
    X, Y = draw_blocks(mod, 20000, BlockingParams(1, 2), drng, "unit")
    assert Y[0] == O.bytes_to_ints(z["y"])
    assert X.rows == z["xrows"].tolist()


def test_krylov_length():
    assert krylov_length(60, BlockingParams(2, 4)) == 30 + 15 + 32
    assert krylov_length(3_600_000, BlockingParams(8, 16)) == 450000 + 225000 + 32


def test_classify_smallest_class():
    mod = PrimeModulus(2**61 - 1)
    ell = mod.ell
    assert classify(1, mod)[0] == 0
    assert classify(ell - 1, mod)[0] == 1
    assert classify(2**31 - 1, mod) == (2, 2**31 - 1)
    assert classify(ell - (2**31 - 1), mod) == (2, -(2**31 - 1))
    assert classify(2**31, mod)[0] == 3
    with pytest.raises(ValueError):
        classify(ell, mod)


def test_sparse_matrix_validation():
    mod = PrimeModulus(1009)
    with pytest.raises(ValueError):
        SparseMatrix(mod, 2, 2, [0, 1], [0], [0], [1], {})
    with pytest.raises(ValueError):
        SparseMatrix(mod, 1, 2, [0, 2], [1, 0], [0, 0], [1, 1], {})  # not increasing
    with pytest.raises(ValueError):
        SparseMatrix(mod, 1, 2, [0, 1], [5], [0], [1], {})
    with pytest.raises(ValueError):
        SparseMatrix.from_rows(mod, 1, 3, [[(0, 1), (0, 2)]])
    A = SparseMatrix.from_rows(mod, 2, 3, [[(0, 1), (2, 1008)], [(1, 500)]], [(3, [7, 0])])
    assert A.total_cols == 4 and A.nnz == 4
    assert A.row_entries(0) == [(0, 1), (2, 1008), (3, 7)]
    assert A.row_entries(1) == [(1, 500)]


def test_planted_witnesses_are_kernel_vectors():
    for seed, dc in ((3, 0), (4, 2)):
        mod = corpus.random_prime(200, np.random.default_rng(seed))
        prof = corpus.CorpusProfile(n=2000, gamma=10, seed=seed, dense_cols=dc, planted_kernel_cols=2)
        A, W = corpus.generate_with_witnesses(prof, mod)
        A._validate()
        orc = to_oracle(A)
        for w in W:
            vec = [0] * A.total_cols
            for c, v in w.items():
                vec[c] = v
            assert orc.spmv_ints(vec) == [0] * A.nrows


def test_recycled_download_buffers_never_alias_live_arrays():
    """device.host_empty: large outputs reuse the buffer of a dead array
    (pages already mapped) and never the memory of a live one."""
    import gc

    from paper_1402_3661_b200 import device as D
    D.release_host_pool()
    shape = (1 << 20, 5)  # 40 MB of uint64, above the pooling threshold
    a = D.host_empty(shape, np.uint64)
    assert a.shape == shape and a.dtype == np.uint64 and a.flags.writeable and a.flags.c_contiguous
    a[:] = 7
    b = D.host_empty(shape, np.uint64)
    assert not np.shares_memory(a, b)
    addr = a.ctypes.data
    view = a[10:20]
    del a
    gc.collect()
    c = D.host_empty(shape, np.uint64)  # a's buffer is still held by `view`
    assert c.ctypes.data != addr and not np.shares_memory(c, view)
    del view
    gc.collect()
    d = D.host_empty(shape, np.uint64)  # now it may come back
    assert d.ctypes.data == addr
    assert not np.shares_memory(d, b) and not np.shares_memory(d, c)
    small = D.host_empty((10, 5), np.uint64)
    assert small.shape == (10, 5) and small.flags.writeable
    D.release_host_pool()


def test_recycled_buffer_pool_is_bounded(monkeypatch):
    import gc

    from paper_1402_3661_b200 import device as D
    D.release_host_pool()
    monkeypatch.setattr(D, "_POOL_MAX_BYTES", 50 << 20)
    shape = (1 << 20, 5)  # 40 MB
    a, b = D.host_empty(shape, np.uint64), D.host_empty(shape, np.uint64)
    del a, b
    gc.collect()
    assert sum(x.nbytes for v in D._pool.values() for x in v) <= 50 << 20
    D.release_host_pool()

"""The C ABI library builds for sm_100a, loads, and exports exactly what
include/sldb200.h declares; error paths work without a GPU.  CPU only."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1402_3661_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sldb200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sld_[a-z0-9_]+)\s*\(", src)))


def test_library_loads():
    lib = _native.load(build_if_missing=True)
    assert lib.sld_version() == 1


def test_exports_match_header():
    lib = _native.load(build_if_missing=True)
    decl = declared_symbols()
    assert decl == sorted(_native.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r"\bT (sld_[a-z0-9_]+)", nm))
    assert set(decl) <= exported


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_bad_arguments_report_errors():
    lib = _native.load(build_if_missing=True)
    h = ctypes.c_void_p()
    ell = np.array([1008], dtype=np.uint32)  # even: rejected before any device call
    rc = lib.sld_ctx_create(0, ell.ctypes.data, 1, ctypes.byref(h))
    assert rc == _native.SLD_E_ARG
    assert b"odd prime" in lib.sld_last_error()
    with pytest.raises(ValueError):
        _native.check(rc)


def test_no_device_is_loud_not_silent():
    # without a GPU the product must fail (no CPU fallback)
    if _native.device_count() > 0:
        pytest.skip("a device is visible")
    from paper_1402_3661_b200 import PrimeModulus, SparseMatrix, spmv_sequential
    A = SparseMatrix.from_rows(PrimeModulus(1009), 2, 2, [[(0, 1)], [(1, 5)]])
    with pytest.raises(RuntimeError):
        spmv_sequential(A, [1, 2])


def test_corpus_generator_is_deterministic():
    from paper_1402_3661_b200 import corpus
    mod = corpus.random_prime(160, np.random.default_rng(1))
    a = corpus.generate_arrays(corpus.CorpusProfile(n=5000, gamma=20, seed=9), mod)
    b = corpus.generate_arrays(corpus.CorpusProfile(n=5000, gamma=20, seed=9), mod)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    rp, col, tags, small = a
    w = np.diff(rp)
    assert 17 < w.mean() < 23 and w.min() >= 3
    assert abs(np.mean(tags <= 1) - 0.9) < 0.02
    # strictly increasing columns within each row
    d = np.diff(col.astype(np.int64))
    starts = np.zeros(len(col), bool)
    starts[rp[:-1]] = True
    assert np.all((d > 0) | starts[1:])
    # power-law density: the first 10% of columns hold ~sqrt(0.1) of the entries
    frac = np.mean(col < 500)
    assert 0.25 < frac < 0.40

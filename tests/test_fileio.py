"""Native SLDM / SLDV / SLDQ readers and writers against files written and
verdicts given by the REAL reference (tests/golden/make_golden.py,
gen_file_cases): same arrays after load (including the reference's
re-classification), same bytes after store, same exception classes on
malformed files.  Host code only: no GPU needed."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from paper_1402_3661_b200 import (
    BadMagic, FormatError, PrimeModulus, TruncatedFile, load_matrix, load_terms, load_vector,
    store_matrix, store_terms, store_vector,
)

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = os.path.join(HERE, "golden", "files")
Z = O.load_golden("file_cases.npz")


def _arrays_equal(A, p):
    bw = A.mod.byte_width
    assert hex(A.mod.ell) == str(Z[p + "ell"])
    assert [A.nrows, A.ncols] == Z[p + "shape"].tolist()
    assert np.array_equal(A.row_ptr, Z[p + "row_ptr"])
    assert np.array_equal(np.asarray(A.col_idx, dtype=np.int64), Z[p + "col_idx"].astype(np.int64))
    assert np.array_equal(A.tags, Z[p + "tags"])
    assert np.array_equal(A.small_vals, Z[p + "small_vals"].astype(np.int64))
    fpos = sorted(A.full_vals)
    assert fpos == Z[p + "full_pos"].tolist()
    assert [A.full_vals[k] for k in fpos] == O.bytes_to_ints(Z[p + "full_vals"])
    dv = Z[p + "dense_vals"]
    assert len(A.dense_cols) == dv.shape[0]
    for g, (gidx, col) in enumerate(A.dense_cols):
        assert gidx == A.ncols + g
        assert list(col) == O.bytes_to_ints(dv[g])
    assert bw == (A.mod.ell.bit_length() + 7) // 8


def test_fixture_manifest():
    for f in sorted(os.listdir(FILES)):
        h = hashlib.sha256(open(os.path.join(FILES, f), "rb").read()).hexdigest()
        assert h == str(Z["sha_" + f]), f


@pytest.mark.parametrize("name", [str(n) for n in Z["matrix_names"]])
def test_load_matrix_matches_reference(name):
    A = load_matrix(os.path.join(FILES, name + ".sldm"))
    _arrays_equal(A, name + "_")


@pytest.mark.parametrize("name", [str(n) for n in Z["matrix_names"] if not str(n).startswith("rc")])
def test_store_matrix_bytes_match_reference(name, tmp_path):
    src = os.path.join(FILES, name + ".sldm")
    A = load_matrix(src)
    out = tmp_path / "re.sldm"
    store_matrix(A, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_reclassified_matrix_restores_canonically(tmp_path):
    # hand-framed tags (+1 stored as small, small stored as full, ...) load
    # re-classified; storing writes the canonical classes and re-loads equal
    for name in ("rc200", "rc7"):
        A = load_matrix(os.path.join(FILES, name + ".sldm"))
        store_matrix(A, tmp_path / "c.sldm")
        B = load_matrix(tmp_path / "c.sldm")
        assert B == A


@pytest.mark.parametrize("i", range(len(Z["bad_names"])))
def test_malformed_files_raise_like_reference(i):
    name, verdict = str(Z["bad_names"][i]), str(Z["bad_verdicts"][i])
    path = os.path.join(FILES, name + ".sldm")
    if verdict == "ok":
        _arrays_equal(load_matrix(path), name + "_")
        return
    exc = {"BadMagic": BadMagic, "TruncatedFile": TruncatedFile, "FormatError": FormatError,
           "ValueError": ValueError}[verdict]
    with pytest.raises(exc) as ei:
        load_matrix(path)
    if verdict == "FormatError":  # not a subclass verdict the reference did not give
        assert type(ei.value) is FormatError
    if verdict == "ValueError":
        assert not isinstance(ei.value, FormatError)


@pytest.mark.parametrize("name", ["v200", "v7", "v650", "v0"])
def test_vectors_match_reference(name, tmp_path):
    src = os.path.join(FILES, name + ".sldv")
    vec, mod = load_vector(src)
    assert hex(mod.ell) == str(Z[name + "_ell"])
    assert vec == O.bytes_to_ints(Z[name + "_vals"]) if len(vec) else Z[name + "_vals"].shape[0] == 0
    store_vector(vec, mod, tmp_path / "v.sldv")
    assert (tmp_path / "v.sldv").read_bytes() == open(src, "rb").read()
    limbs, _ = load_vector(src, as_limbs=True)
    store_vector(limbs, mod, tmp_path / "w.sldv")
    assert (tmp_path / "w.sldv").read_bytes() == open(src, "rb").read()


def test_terms_match_reference(tmp_path):
    src = os.path.join(FILES, "q200.sldq")
    terms, m, mod = load_terms(src)
    flat = O.bytes_to_ints(Z["q200_vals"])
    assert m == int(Z["q200_m"]) and [v for t in terms for v in t] == flat
    store_terms(tmp_path / "q.sldq", terms, m, mod)
    assert (tmp_path / "q.sldq").read_bytes() == open(src, "rb").read()
    with pytest.raises(BadMagic):
        load_vector(src)
    with pytest.raises(BadMagic):
        load_terms(os.path.join(FILES, "v200.sldv"))


def test_large_roundtrip_threaded(tmp_path):
    # enough rows for the threaded writer / reader paths
    from helpers import rand_matrix
    mod = PrimeModulus(2**202 - 2**100 + 1) if False else PrimeModulus(2**127 - 1)
    rng = np.random.default_rng(5)
    A = rand_matrix(mod, rng, 70000, 70000, 6, dense=1, full_frac=0.02)
    p = tmp_path / "big.sldm"
    store_matrix(A, p)
    B = load_matrix(p)
    assert B == A
    store_matrix(B, tmp_path / "big2.sldm")
    assert p.read_bytes() == (tmp_path / "big2.sldm").read_bytes()


def _sldv_bytes(ell, vals, header_width, count=None):
    import struct
    eb = (ell.bit_length() + 7) // 8
    out = b"SLDV" + struct.pack("<I", 1) + struct.pack("<H", header_width) + ell.to_bytes(header_width, "big")
    out += struct.pack("<Q", len(vals) if count is None else count)
    return out + b"".join(int(v).to_bytes(eb, "little") for v in vals)


def test_sldv_zero_padded_modulus_header(tmp_path):
    # residues are read at the modulus's own byte width whatever zero padding
    # the header's ell field has (spmatrix.py:349-352,450-462)
    from paper_1402_3661_b200 import load_vector
    ell = 2**200 - 75
    vals = [0, 1, ell - 1, 12345678901234567890]
    for hw in (25, 28, 200):
        p = tmp_path / f"v{hw}.sldv"
        p.write_bytes(_sldv_bytes(ell, vals, hw))
        got, mod = load_vector(p)
        assert got == vals and mod.ell == ell


def test_sldv_count_overflow_is_truncation(tmp_path):
    from paper_1402_3661_b200 import load_vector
    from paper_1402_3661_b200.fileio import TruncatedFile
    ell = 2**127 - 1
    p = tmp_path / "big.sldv"
    p.write_bytes(_sldv_bytes(ell, [1, 2, 3], 16, count=(1 << 64) - 1))
    with pytest.raises(TruncatedFile):
        load_vector(p)
    p.write_bytes(_sldv_bytes(ell, [1, 2, 3], 16, count=(1 << 60) + 1))  # count*16 wraps to 16
    with pytest.raises(TruncatedFile):
        load_vector(p)

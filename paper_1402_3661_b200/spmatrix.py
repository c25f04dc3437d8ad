"""Sparse matrices over Z/lZ and the public SpMV entry points.

`SparseMatrix` keeps the reference's field layout (sldlag/spmatrix.py:69-91)
so matrices move between the two packages unchanged: CSR `row_ptr` /
`col_idx`, a coefficient class tag per entry (+1, -1, small signed word,
full residue; modring.py:26-29), `small_vals`, a `full_vals` dict (flat
position -> residue) and dense columns at the top column indices.

`kernel()` returns the GPU SpMV (a `DeviceKernel`), replacing the reference's
numpy `SpmvKernel` (vecops.py:355-470).  `spmv_planes` / `spmv_sequential`
keep the reference signatures and error behaviour (ValueError on a length
mismatch, spmatrix.py:233-246).  Every product runs on the device; there is
no CPU path.
"""
import threading

import numpy as np

from .device import DEFAULT_DEVICE, DeviceMatrix
from .modring import (
    TAG_FULL, TAG_MINUS_ONE, TAG_PLUS_ONE, TAG_SMALL, as_modulus, digit_count,
    ints_to_planes, planes_to_ints,
)

C_MAX_DEFAULT = 2**31 - 1


def classify(value: int, mod):
    """Smallest class of a non-zero residue (spmatrix.py:48-66):
    (tag, signed word) with the word meaningful for TAG_SMALL."""
    ell = mod.ell
    v = int(value) % ell
    if v == 0:
        raise ValueError("zero coefficient cannot be stored")
    if v == 1:
        return TAG_PLUS_ONE, 1
    if v == ell - 1:
        return TAG_MINUS_ONE, -1
    c = v if 2 * v <= ell else v - ell  # representative of least magnitude
    if abs(c) <= C_MAX_DEFAULT:
        return TAG_SMALL, c
    return TAG_FULL, 0


class DeviceKernel:
    """The batched SpMV of one matrix on one device (`SpmvKernel` stand-in).

    Thread-safe: concurrent `apply` calls on the same kernel serialize on a
    lock (each holds the device stream for one product)."""

    def __init__(self, A, device=None, stripe_cols=0):
        self.device = DEFAULT_DEVICE if device is None else device
        self.dm = DeviceMatrix(A, self.device, stripe_cols=stripe_cols)
        self.mod = self.dm.mod
        self.nrows = self.dm.nrows
        self.width = self.dm.P
        self._lock = threading.Lock()

    def apply(self, planes: np.ndarray) -> np.ndarray:
        """v = A u on digit planes; returns fresh (nrows, P) canonical planes."""
        with self._lock:
            return self.dm.apply_planes(planes)


class SparseMatrix:
    """CSR rows with per-entry class tags plus optional dense columns."""

    def __init__(self, mod, nrows: int, ncols: int, row_ptr, col_idx, tags, small_vals,
                 full_vals: dict, dense_cols=None, validate: bool = True):
        self.mod = as_modulus(mod)
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        col_idx = np.asarray(col_idx)
        # int32 column indices are kept as-is (no 4-byte-per-entry copy at
        # N = 3.6M scale); anything else is normalised to the reference's int64
        self.col_idx = col_idx if col_idx.dtype == np.int32 else col_idx.astype(np.int64)
        self.tags = np.asarray(tags, dtype=np.uint8)
        self.small_vals = np.asarray(small_vals, dtype=np.int64)
        self.full_vals = {int(k): int(v) for k, v in dict(full_vals).items()}
        self.dense_cols = [(int(g), col if isinstance(col, np.ndarray) else list(col))
                           for g, col in (dense_cols or [])]
        self._kernels = {}
        self._klock = threading.Lock()
        if validate:
            self._validate()

    def _validate(self):
        n = len(self.col_idx)
        if self.row_ptr.shape != (self.nrows + 1,):
            raise ValueError("row_ptr length must be nrows + 1")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != n:
            raise ValueError("row_ptr endpoints inconsistent with entry count")
        if np.any(np.diff(self.row_ptr) < 0):
            raise ValueError("row_ptr must be monotone")
        if len(self.tags) != n or len(self.small_vals) != n:
            raise ValueError("parallel entry arrays disagree in length")
        if n and (self.col_idx.min() < 0 or self.col_idx.max() >= self.ncols):
            raise ValueError("sparse column index out of range")
        if n > 1:
            step = np.diff(self.col_idx)
            starts = np.zeros(n, dtype=bool)
            starts[self.row_ptr[:-1][self.row_ptr[:-1] < n]] = True
            if np.any((step <= 0) & ~starts[1:]):
                raise ValueError("column indices not strictly increasing within a row")
        for g, (gidx, col) in enumerate(self.dense_cols):
            if gidx != self.ncols + g:
                raise ValueError("dense columns must occupy the top indices in order")
            if len(col) != self.nrows:
                raise ValueError("dense column length mismatch")
            if not isinstance(col, np.ndarray):
                for v in col:
                    self.mod.check(v)
        for v in self.full_vals.values():
            self.mod.check(v)
            if v == 0:
                raise ValueError("explicit zero coefficient")
        if np.any(self.tags > TAG_FULL):
            raise ValueError("unknown coefficient tag")

    @classmethod
    def from_rows(cls, mod, nrows: int, ncols: int, rows, dense_cols=None):
        """Build from per-row (col, value) pairs: values reduced, zeros
        dropped, each coefficient stored in its smallest class."""
        mod = as_modulus(mod)
        ptr, cols, tags, smalls, fulls = [0], [], [], [], {}
        for r in rows:
            last = None
            for c, v in sorted((int(c), v) for c, v in r):
                if c == last:
                    raise ValueError("duplicate column in row")
                last = c
                v = int(v) % mod.ell
                if not v:
                    continue
                tag, word = classify(v, mod)
                if tag == TAG_FULL:
                    fulls[len(cols)] = v
                cols.append(c)
                tags.append(tag)
                smalls.append(word)
            ptr.append(len(cols))
        return cls(mod, nrows, ncols, ptr, cols, tags, smalls, fulls, dense_cols)

    def entry_value(self, pos: int) -> int:
        t = int(self.tags[pos])
        if t == TAG_PLUS_ONE:
            return 1
        if t == TAG_MINUS_ONE:
            return self.mod.ell - 1
        if t == TAG_SMALL:
            return int(self.small_vals[pos]) % self.mod.ell
        return self.full_vals[pos]

    def row_entries(self, i: int):
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        out = [(int(self.col_idx[p]), self.entry_value(p)) for p in range(lo, hi)]
        for gidx, col in self.dense_cols:
            v = _dense_value(col, i)
            if v:
                out.append((gidx, v))
        return out

    @property
    def total_cols(self) -> int:
        return self.ncols + len(self.dense_cols)

    @property
    def nnz(self) -> int:
        dense_nnz = sum(int(np.count_nonzero(np.asarray(_dense_ints(col), dtype=object)))
                        for _, col in self.dense_cols)
        return len(self.col_idx) + dense_nnz

    def __eq__(self, other):
        if not hasattr(other, "row_ptr"):
            return NotImplemented
        return (self.mod == other.mod and self.nrows == other.nrows and self.ncols == other.ncols
                and np.array_equal(self.row_ptr, other.row_ptr)
                and np.array_equal(self.col_idx, other.col_idx)
                and np.array_equal(self.tags, other.tags)
                and np.array_equal(self.small_vals, other.small_vals)
                and self.full_vals == dict(other.full_vals)
                and [(g, _dense_ints(c)) for g, c in self.dense_cols]
                == [(g, _dense_ints(c)) for g, c in other.dense_cols])

    def kernel(self, device=None) -> DeviceKernel:
        """GPU SpMV kernel (built lazily, cached per device)."""
        device = DEFAULT_DEVICE if device is None else device
        with self._klock:
            k = self._kernels.get(device)
            if k is None:
                k = DeviceKernel(self, device)
                self._kernels[device] = k
            return k


def _dense_ints(col):
    if isinstance(col, np.ndarray):
        from .modring import limbs_to_ints
        return limbs_to_ints(col)
    return list(col)


def _dense_value(col, i):
    if isinstance(col, np.ndarray):
        return int.from_bytes(np.ascontiguousarray(col[i], dtype="<u4").tobytes(), "little")
    return col[i]


def _kernel_of(A, device=None):
    if hasattr(A, "_kernels") and isinstance(getattr(A, "_kernels"), dict) and hasattr(A, "kernel") \
            and isinstance(A, SparseMatrix):
        return A.kernel(device)
    # a foreign (e.g. the reference's) SparseMatrix: cache a device kernel on it
    cache = A.__dict__.setdefault("_b200_kernels", {})
    device = DEFAULT_DEVICE if device is None else device
    k = cache.get(device)
    if k is None:
        k = cache[device] = DeviceKernel(A, device)
    return k


def total_cols(A) -> int:
    return A.ncols + len(getattr(A, "dense_cols", None) or [])


def spmv_planes(A, planes: np.ndarray, device=None) -> np.ndarray:
    """Digit-plane SpMV on the device (spmatrix.py:242-246)."""
    if planes.shape[0] != total_cols(A):
        raise ValueError("plane count mismatch")
    return _kernel_of(A, device).apply(planes)


def spmv_sequential(A, u, device=None) -> list:
    """v = A u over Z/lZ for a list of canonical ints (spmatrix.py:233-239)."""
    if len(u) != total_cols(A):
        raise ValueError(f"vector length {len(u)} != {total_cols(A)} columns")
    planes = ints_to_planes(u, digit_count(A.mod.ell))
    return planes_to_ints(_kernel_of(A, device).apply(planes))


# ------------------------------------------------------------ file formats
# SLDM matrices and SLDV vectors (sldlag/spmatrix.py:14-25, 358-462), read
# and written natively (csrc/sld_fileio.cpp): same bytes, same exception types.

def _ell_from_be(buf, width):
    from .fileio import FormatError
    from .modring import PrimeModulus
    ell = int.from_bytes(bytes(buf[:width]), "big")
    try:
        return PrimeModulus(ell)
    except ValueError as e:
        raise FormatError(str(e)) from e


def _path(p):
    import os
    return os.fsencode(os.fspath(p))


def store_matrix(A, path):
    """Write A as SLDM (byte-identical to the reference's store_matrix)."""
    from . import _native as N
    from .device import matrix_arrays
    from .fileio import check_io
    mod = as_modulus(A.mod)
    L = mod.limbs
    row_ptr, col, tags, small, fpos, flimbs, n_dense, dense = matrix_arrays(A, L)
    ell = np.asarray([(mod.ell >> (32 * i)) & 0xFFFFFFFF for i in range(L)], dtype=np.uint32)
    didx = np.arange(A.ncols, A.ncols + n_dense, dtype=np.int64)
    check_io(N.load().sld_sldm_write(
        _path(path), int(A.nrows), int(A.ncols), N.ptr(ell), L, N.ptr(row_ptr), N.ptr(col),
        N.ptr(tags), N.ptr(small), len(fpos), N.ptr(fpos), N.ptr(flimbs), n_dense, N.ptr(didx),
        N.ptr(dense) if dense is not None else None))


def load_matrix(path, dense_as_limbs=False):
    """Read an SLDM file (the reference's load_matrix): coefficients are
    re-classified to their smallest class; FormatError / BadMagic /
    TruncatedFile / ValueError as the reference raises them.  Dense columns
    come back as lists of ints, or as (nrows, L) limb arrays (no per-value
    Python objects at NFS scale) with dense_as_limbs=True."""
    from . import _native as N
    from .fileio import check_io
    from .modring import limbs_to_ints
    info = np.zeros(8, dtype=np.int64)
    ell_be = np.zeros(65536, dtype=np.uint8)
    check_io(N.load().sld_sldm_info(_path(path), 1, N.ptr(info), N.ptr(ell_be), len(ell_be)))
    mod = _ell_from_be(ell_be, int(info[2]))
    check_io(N.load().sld_sldm_info(_path(path), 0, N.ptr(info), N.ptr(ell_be), len(ell_be)))
    nrows, ncols, eb, dc, nnz, nfull = (int(x) for x in info[:6])
    L = mod.limbs
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    col = np.zeros(max(nnz, 1), dtype=np.int32)
    tags = np.zeros(max(nnz, 1), dtype=np.uint8)
    small = np.zeros(max(nnz, 1), dtype=np.int64)
    fpos = np.zeros(max(nfull, 1), dtype=np.int64)
    flimbs = np.zeros((max(nfull, 1), L), dtype=np.uint32)
    didx = np.zeros(max(dc, 1), dtype=np.int64)
    dlimbs = np.zeros((max(dc, 1), nrows, L), dtype=np.uint32)
    check_io(N.load().sld_sldm_read(_path(path), L, N.ptr(row_ptr), N.ptr(col), N.ptr(tags),
                                    N.ptr(small), N.ptr(fpos), N.ptr(flimbs), N.ptr(didx),
                                    N.ptr(dlimbs)))
    fulls = dict(zip(fpos[:nfull].tolist(), limbs_to_ints(flimbs[:nfull]))) if nfull else {}
    dense = []
    for g in range(dc):
        colv = dlimbs[g] if dense_as_limbs else limbs_to_ints(dlimbs[g])
        dense.append((int(didx[g]), colv))
    return SparseMatrix(mod, nrows, ncols, row_ptr, col[:nnz] if nnz else [],
                        tags[:nnz], small[:nnz], fulls, dense)


def _store_residues(path, kind, values, mod, m=1):
    from . import _native as N
    from .fileio import check_io
    from .modring import ints_to_limbs
    mod = as_modulus(mod)
    L = mod.limbs
    if isinstance(values, np.ndarray) and values.dtype == np.uint32 and values.ndim == 2:
        limbs = np.ascontiguousarray(values)
    else:
        vals = list(values)
        for v in vals:
            mod.check(int(v))
        limbs = ints_to_limbs(vals, L) if vals else np.zeros((0, L), dtype=np.uint32)
    count = limbs.shape[0] // m if kind == 1 else limbs.shape[0]
    ell = np.asarray([(mod.ell >> (32 * i)) & 0xFFFFFFFF for i in range(L)], dtype=np.uint32)
    check_io(N.load().sld_sldv_write(_path(path), kind, N.ptr(ell), L, int(m), int(count),
                                     N.ptr(limbs) if limbs.size else None, int(limbs.shape[1])))


def _load_residues(path, want_kind):
    from . import _native as N
    from .fileio import BadMagic, check_io
    info = np.zeros(6, dtype=np.int64)
    ell_be = np.zeros(65536, dtype=np.uint8)
    check_io(N.load().sld_sldv_info(_path(path), 1, N.ptr(info), N.ptr(ell_be), len(ell_be)))
    if int(info[0]) != want_kind:
        raise BadMagic(f"{path}: magic {'SLDQ' if info[0] else 'SLDV'}, expected "
                       f"{'SLDQ' if want_kind else 'SLDV'}")
    mod = _ell_from_be(ell_be, int(info[1]))
    check_io(N.load().sld_sldv_info(_path(path), 0, N.ptr(info), N.ptr(ell_be), len(ell_be)))
    kind, eb, _, m, count, nres = (int(x) for x in info)
    limbs = np.zeros((max(nres, 1), mod.limbs), dtype=np.uint32)
    check_io(N.load().sld_sldv_read(_path(path), N.ptr(limbs), mod.limbs))
    return limbs[:nres], mod, m, count


def store_vector(vec, mod, path):
    """SLDV vector of residues (ints, or an (n, L) uint32 limb array)."""
    _store_residues(path, 0, vec, mod)


def load_vector(path, as_limbs=False):
    """Returns (vector, modulus) like the reference; as_limbs=True returns
    the (n, L) uint32 limbs instead of Python ints."""
    from .modring import limbs_to_ints
    limbs, mod, _, _ = _load_residues(path, 0)
    return (limbs if as_limbs else limbs_to_ints(limbs)), mod

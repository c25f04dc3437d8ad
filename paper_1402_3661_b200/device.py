"""Device objects over the C ABI: field context, GPU matrix, GPU vector.

Each `DeviceMatrix` owns one `sld_ctx` (one CUDA stream) so multipliers of
different Krylov chains can run from different host threads at once (the
reference runs one multiplier per chain thread, sldlag/solver.py:249-251);
ctypes releases the GIL for the duration of every call.
"""
import ctypes
import os
import threading

import numpy as np

from . import _native as N
from .modring import as_modulus, ints_to_limbs, limbs_to_planes

DEFAULT_DEVICE = int(os.environ.get("SLD_DEVICE", "0"))


# ---- recycled host buffers for large downloads.  A fresh 374 MB planes
# array (cfg3) costs ~10 ms of page faults on first touch, more than its
# DMA and unpack.  Large outputs are therefore built on pooled buffers whose
# pages are already mapped: each array owns a _Lease (its numpy base), and
# when the last array or view on it dies the buffer returns to the pool.
# Every call still returns a new array no live array shares memory with.
_POOL_MIN_BYTES = 32 << 20
_POOL_PER_SIZE = 2
_POOL_MAX_BYTES = 1 << 30  # all pooled buffers together (kept after use)
_pool: dict = {}
_pool_lock = threading.Lock()


class _Lease:
    __slots__ = ("slab", "__weakref__")

    def __init__(self, slab):
        self.slab = slab

    def __buffer__(self, flags):
        return memoryview(self.slab)

    def __release_buffer__(self, view):
        pass

    def __del__(self):
        try:
            with _pool_lock:
                free = _pool.setdefault(self.slab.nbytes, [])
                held = sum(b.nbytes for bufs in _pool.values() for b in bufs)
                if len(free) < _POOL_PER_SIZE and held + self.slab.nbytes <= _POOL_MAX_BYTES:
                    free.append(self.slab)
        except Exception:  # interpreter shutdown
            pass


def host_empty(shape, dtype):
    """np.empty(shape, dtype), on a recycled buffer when it is large."""
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    if nbytes < _POOL_MIN_BYTES:
        return np.empty(shape, dtype=dt)
    with _pool_lock:
        free = _pool.get(nbytes)
        slab = free.pop() if free else None
    if slab is None:
        slab = np.empty(nbytes, dtype=np.uint8)
    return np.frombuffer(_Lease(slab), dtype=dt).reshape(shape)


def release_host_pool():
    """Drop the recycled download buffers (their memory goes back to the OS)."""
    with _pool_lock:
        _pool.clear()


def _dense_limbs(A, L):
    """Dense columns of a SparseMatrix-like object as (n_dense, nrows, L)."""
    dense = list(getattr(A, "dense_cols", None) or [])
    if not dense:
        return 0, None
    out = np.zeros((len(dense), A.nrows, L), dtype=np.uint32)
    for g, (gidx, col) in enumerate(dense):
        if int(gidx) != A.ncols + g:
            raise ValueError("dense columns must occupy the top indices in order")
        if isinstance(col, np.ndarray) and col.dtype == np.uint32:
            out[g] = col.reshape(A.nrows, L)
        else:
            out[g] = ints_to_limbs(col, L)
    return len(dense), out


def matrix_arrays(A, L):
    """The SparseMatrix fields (spmatrix.py:77-91) as contiguous arrays."""
    row_ptr = N.c64(A.row_ptr)
    nnz = int(row_ptr[-1]) if len(row_ptr) else 0
    col = N.c32(A.col_idx) if nnz else np.zeros(0, np.int32)
    tags = np.ascontiguousarray(A.tags, dtype=np.uint8) if nnz else np.zeros(0, np.uint8)
    small = N.c64(A.small_vals) if nnz else np.zeros(0, np.int64)
    fv = A.full_vals
    if isinstance(fv, tuple):  # (positions, limbs) fast form
        fpos, flimbs = N.c64(fv[0]), N.cu32(fv[1]).reshape(-1, L)
        order = np.argsort(fpos, kind="stable")
        fpos, flimbs = np.ascontiguousarray(fpos[order]), np.ascontiguousarray(flimbs[order])
    else:
        keys = sorted(int(k) for k in fv)
        fpos = np.array(keys, dtype=np.int64)
        flimbs = ints_to_limbs([fv[k] for k in keys], L)
    n_dense, dense = _dense_limbs(A, L)
    return row_ptr, col, tags, small, fpos, flimbs, n_dense, dense


class Field:
    """sld_ctx: one prime on one device (the PrimeModulus of the ABI)."""

    def __init__(self, mod, device=None):
        self.mod = as_modulus(mod)
        self.device = DEFAULT_DEVICE if device is None else int(device)
        self.L = self.mod.limbs
        lib = N.load()
        ell = ints_to_limbs([self.mod.ell], self.L)[0].copy()
        h = ctypes.c_void_p()
        N.check(lib.sld_ctx_create(self.device, N.ptr(ell), self.L, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def sync(self):
        N.check(N.load().sld_ctx_sync(self._h))

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceVector:
    """A device vector of n residues (biased 32-bit limbs, sector padded);
    with chains = G, G interleaved vectors (host arrays chain-major)."""

    def __init__(self, field: Field, n: int, chains: int = 1):
        self.field = field
        self.n = int(n)
        self.chains = int(chains)
        h = ctypes.c_void_p()
        N.check(N.load().sld_vec_create_chains(field.handle, self.n, self.chains, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def ptr(self):
        """Raw device pointer of the current buffer (slot format)."""
        p, st = ctypes.c_uint64(), ctypes.c_int64()
        N.check(N.load().sld_vec_device_ptr(self._h, ctypes.byref(p), ctypes.byref(st)))
        return p.value

    def nonzero(self) -> bool:
        out = ctypes.c_int(0)
        N.check(N.load().sld_vec_nonzero(self._h, ctypes.byref(out)))
        return bool(out.value)

    def _shape(self, w):
        return (self.n, w) if self.chains == 1 else (self.chains, self.n, w)

    def upload_planes(self, planes):
        p = np.ascontiguousarray(planes, dtype=np.uint64)
        if p.shape[:-1] != self._shape(1)[:-1]:
            raise ValueError("plane count mismatch")
        N.check(N.load().sld_vec_upload_planes(self._h, N.ptr(p), self.n, p.shape[-1]))

    def download_planes(self, P):
        out = host_empty(self._shape(P), np.uint64)
        N.check(N.load().sld_vec_download_planes(self._h, N.ptr(out), self.n, P))
        return out

    def upload_planes_list(self, planes_list):
        """One (n, P) planes array per chain, without stacking them on the host."""
        ps = [np.ascontiguousarray(p, dtype=np.uint64) for p in planes_list]
        if len(ps) != self.chains or any(p.shape[0] != self.n for p in ps) or \
                len({p.shape[1] for p in ps}) != 1:
            raise ValueError("plane count mismatch")
        ptrs = (ctypes.c_void_p * len(ps))(*[p.ctypes.data for p in ps])
        N.check(N.load().sld_vec_upload_planes_chains(self._h, ptrs, self.n, ps[0].shape[1]))

    def download_planes_list(self, P):
        outs = [host_empty((self.n, P), np.uint64) for _ in range(self.chains)]
        ptrs = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        N.check(N.load().sld_vec_download_planes_chains(self._h, ptrs, self.n, P))
        return outs

    def upload_limbs(self, limbs):
        a = N.cu32(limbs)
        if a.shape != self._shape(self.field.L):
            raise ValueError(f"limb array shape {a.shape} != {self._shape(self.field.L)}")
        N.check(N.load().sld_vec_upload_limbs(self._h, N.ptr(a), self.n))

    def download_limbs(self):
        out = np.empty(self._shape(self.field.L), dtype=np.uint32)
        N.check(N.load().sld_vec_download_limbs(self._h, N.ptr(out), self.n))
        return out

    def read_rows(self, rows):
        """Canonical limbs (len(rows), L) of the given rows only (one chain)."""
        r = N.c64(rows)
        out = np.empty((len(r), self.field.L), dtype=np.uint32)
        if len(r):
            N.check(N.load().sld_vec_read_rows(self._h, N.ptr(r), len(r), N.ptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_vec_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lincomb(field: Field, ys, coeffs, dst: "DeviceVector", acc: "DeviceVector" = None):
    """dst = acc + sum_j coeffs[j] * ys[j] mod l on the device."""
    k = len(ys)
    ptrs = np.array([y.ptr for y in ys], dtype=np.uint64)
    cl = ints_to_limbs([int(c) for c in coeffs], field.L) if k else np.zeros((0, field.L), np.uint32)
    N.check(N.load().sld_lincomb(field.handle, N.ptr(ptrs), N.ptr(cl), k,
                                 acc.ptr if acc is not None else 0, dst.ptr, dst.n))


class LinCombSet:
    """n <= 8 fixed device vectors combined on the tensor cores (Mksol's
    Horner combination, sld_lcset_*): dst = acc + sum_s c_s y_s mod l."""

    def __init__(self, field: Field, ys, rows: int, matrix: "DeviceMatrix" = None):
        """With `matrix`, the set is tiled in that matrix's slot order: its
        combinations are slot-ordered (the operand of DeviceMatrix.spmv_add)."""
        self.field, self.n = field, len(ys)
        ptrs = np.array([y.ptr for y in ys], dtype=np.uint64)
        h = ctypes.c_void_p()
        if matrix is None:
            N.check(N.load().sld_lcset_create(field.handle, N.ptr(ptrs), self.n, int(rows), ctypes.byref(h)))
        else:
            N.check(N.load().sld_lcset_create_slots(matrix.handle, N.ptr(ptrs), self.n, ctypes.byref(h)))
        self._h = h
        self._ys = list(ys)  # keep the vectors alive while tiled copies are in use

    def apply(self, coeffs, dst: "DeviceVector", acc: "DeviceVector" = None):
        cl = ints_to_limbs([int(c) for c in coeffs], self.field.L)
        N.check(N.load().sld_lcset_apply(self._h, N.ptr(cl), acc.ptr if acc is not None else 0, dst.ptr))

    def apply_batch(self, coeff_sets, dsts):
        """dsts[k] = sum_s coeff_sets[k][s] y_s for K = 2 or 4 steps, one
        pass over the tiled y."""
        K = len(coeff_sets)
        cl = np.ascontiguousarray(np.stack([ints_to_limbs([int(c) for c in cs], self.field.L)
                                            for cs in coeff_sets]))
        ptrs = np.array([d.ptr for d in dsts], dtype=np.uint64)
        N.check(N.load().sld_lcset_apply_batch(self._h, N.ptr(cl), K, N.ptr(ptrs)))

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_lcset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DevicePlanes(np.lib.mixins.NDArrayOperatorsMixin):
    """A product left on the device by `B200Multiplier.apply`.

    It behaves as the (n, P) uint64 digit planes on any host access: numpy
    functions, operators, attributes. The array is downloaded once and cached
    read-only. Row indexing (`planes[rows]`, which is what
    `UnitRows.project` does, solver.py:174-176) fetches only those rows.
    Passing it back into `apply` keeps the iterate on the device. So the
    reference's own `krylov_column` (solver.py:199-217), left unmodified,
    moves m rows per step instead of two full vectors."""

    __array_priority__ = 1000

    def __init__(self, dm: "DeviceMatrix", vec: DeviceVector, P: int):
        self._dm, self._vec, self._P = dm, vec, int(P)
        self._host = None
        self.shape = (vec.n, self._P)
        self.dtype = np.dtype(np.uint64)
        self.ndim = 2
        self.size = vec.n * self._P
        self.nbytes = self.size * 8

    def __len__(self):
        return self.shape[0]

    def _materialize(self):
        if self._host is None:
            a = self._vec.download_planes(self._P)
            a.setflags(write=False)
            self._host = a
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self._materialize()
        if dtype is not None and np.dtype(dtype) != a.dtype:
            return a.astype(dtype)
        return a.copy() if copy else a

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        conv = [np.asarray(x) if isinstance(x, DevicePlanes) else x for x in inputs]
        if "out" in kwargs:
            kwargs["out"] = tuple(np.asarray(x) if isinstance(x, DevicePlanes) else x for x in kwargs["out"])
        return getattr(ufunc, method)(*conv, **kwargs)

    def __getitem__(self, idx):
        if self._host is None and not isinstance(idx, (tuple, slice)):
            rows = np.asarray(idx)
            if rows.dtype.kind in "iu" and rows.ndim <= 1:
                r = np.atleast_1d(rows).astype(np.int64)
                r = np.where(r < 0, r + self.shape[0], r)
                if len(r) and (r.min() < 0 or r.max() >= self.shape[0]):
                    raise IndexError("row index out of range")
                out = limbs_to_planes(self._vec.read_rows(r), self._P)
                return out[0] if rows.ndim == 0 else out
        return self._materialize()[idx]

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self._materialize(), name)

    def __repr__(self):
        return f"DevicePlanes(shape={self.shape}, on device {self._dm.field.device})"

    def __del__(self):
        try:
            self._dm.pool_put(self._vec)
        except Exception:
            pass


class XBlock:
    """A dense projection block (m x n residues) resident on the device."""

    def __init__(self, field: Field, x_limbs):
        x = N.cu32(x_limbs)
        m, n = x.shape[0], x.shape[1]
        self.field, self.m, self.n = field, m, n
        h = ctypes.c_void_p()
        N.check(N.load().sld_xblock_create(field.handle, N.ptr(x), m, n, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_xblock_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceMatrix:
    """GPU layout of a SparseMatrix (ours or the reference's, duck-typed on
    the fields of sldlag/spmatrix.py:77-91) -- the replacement of
    `SparseMatrix.kernel()` / `SpmvKernel` (vecops.py:355-470)."""

    INFO_KEYS = ("nrows", "total_cols", "nnz", "n_pm", "n_small", "n_full", "stripes",
                 "nslices", "device_bytes", "pad_entries", "L", "stride_words", "max_degree",
                 "stripe_cols", "chains", "halves", "lanes_per_residue", "rows_per_slice",
                 "prefetch")

    def __init__(self, A, device=None, stripe_cols=0, field=None, chains=1):
        self.mod = as_modulus(A.mod)
        self.field = field or Field(self.mod, device)
        self.L = self.field.L
        self.P = self.mod.digits
        self.nrows = int(A.nrows)
        self.ncols = int(A.ncols)
        arrs = matrix_arrays(A, self.L)
        row_ptr, col, tags, small, fpos, flimbs, n_dense, dense = arrs
        if row_ptr.shape != (self.nrows + 1,):
            raise ValueError("row_ptr length must be nrows + 1")
        self.n_dense = n_dense
        self.total_cols = self.ncols + n_dense
        self.chains = int(chains)
        h = ctypes.c_void_p()
        N.check(N.load().sld_mat_create_chains(
            self.field.handle, self.chains, self.nrows, self.ncols, N.ptr(row_ptr), N.ptr(col), N.ptr(tags),
            N.ptr(small), len(fpos), N.ptr(fpos), N.ptr(flimbs), n_dense,
            N.ptr(dense) if dense is not None else ctypes.c_void_p(0), int(stripe_cols),
            ctypes.byref(h)))
        self._h = h
        self._tmp = {}

    @property
    def handle(self):
        return self._h

    def info(self):
        out = np.zeros(20, dtype=np.int64)
        N.check(N.load().sld_mat_info(self._h, N.ptr(out)))
        return {k: int(v) for k, v in zip(self.INFO_KEYS, out)}

    def vector(self, n=None):
        return DeviceVector(self.field, self.total_cols if n is None else n, self.chains)

    # a few spare iterate buffers, recycled by DevicePlanes (one chain)
    _POOL_MAX = 4

    def copy_vector(self, src: DeviceVector, dst: DeviceVector):
        """dst = src on the device (one add_mod of a single term)."""
        ptrs = np.array([src.ptr], dtype=np.uint64)
        N.check(N.load().sld_add_mod(self.field.handle, N.ptr(ptrs), 1, dst.ptr, src.n))

    def pool_get(self):
        pool = self.__dict__.setdefault("_pool", [])
        return pool.pop() if pool else self.vector()

    def pool_put(self, v):
        pool = self.__dict__.setdefault("_pool", [])
        if getattr(self, "_h", None) and len(pool) < self._POOL_MAX:
            pool.append(v)
        else:
            v.close()

    def apply_planes(self, planes):
        """v = A u on digit planes (host in, host out; chains x n x P when
        the matrix carries several chains)."""
        p = np.ascontiguousarray(planes, dtype=np.uint64)
        lead = (self.total_cols,) if self.chains == 1 else (self.chains, self.total_cols)
        if p.shape[:-1] != lead:
            raise ValueError("plane count mismatch")
        out_shape = ((self.nrows,) if self.chains == 1 else (self.chains, self.nrows)) + (p.shape[-1],)
        out = host_empty(out_shape, np.uint64)
        N.check(N.load().sld_spmv_planes(self._h, N.ptr(p), N.ptr(out), p.shape[-1]))
        return out

    def spmv(self, vin: DeviceVector, vout: DeviceVector, sync=True):
        lib = N.load()
        N.check((lib.sld_spmv if sync else lib.sld_spmv_async)(self._h, vin.handle, vout.handle))

    def mksol_bind(self, ys) -> bool:
        """Bind n <= 8 y vectors for `spmv_mksol` (slot-order copies on the
        device).  False when this layout cannot fuse the step (short rows,
        limb slicing, die split, several chains, l >= 2^256)."""
        lib = N.load()
        if not ys:
            N.check(lib.sld_mat_mksol_bind(self._h, None, 0))
            return False
        if self.L > 8 or self.chains != 1 or len(ys) > 8:
            return False
        info = self.info()
        if info["rows_per_slice"] != 32 or info["lanes_per_residue"] != 1 or info["halves"] != 1:
            return False  # short rows / limb slicing / die split
        arr = (ctypes.c_void_p * len(ys))(*[y.handle.value if hasattr(y.handle, "value") else y.handle
                                            for y in ys])
        N.check(lib.sld_mat_mksol_bind(self._h, arr, len(ys)))
        return True

    @property
    def nslots(self) -> int:
        i = self.info()
        return int(i["nslices"]) * int(i["rows_per_slice"])

    def spmv_add(self, vin: DeviceVector, vout: DeviceVector, addv: DeviceVector):
        """vout = A vin + addv, addv in the slot order (a LinCombSet built with
        matrix=self); asynchronous, the addition in the last pass."""
        N.check(N.load().sld_spmv_add(self._h, vin.handle, vout.handle, addv.handle))

    def spmv_mksol(self, vin: DeviceVector, vout: DeviceVector, coeffs):
        """vout = A vin + sum_s coeffs[s] y_s mod l (the bound y vectors),
        one product with the combination in its epilogue; asynchronous."""
        cl = ints_to_limbs([int(c) for c in coeffs], self.L)
        N.check(N.load().sld_spmv_mksol(self._h, vin.handle, vout.handle, N.ptr(cl)))

    def krylov_unit(self, v: DeviceVector, rows, steps):
        """terms (steps, m, L) -- or (steps, chains, m, L) for several chains."""
        rows = N.c64(rows)
        m = len(rows)
        shape = (int(steps), m, self.L) if self.chains == 1 else (int(steps), self.chains, m, self.L)
        terms = np.zeros(shape, dtype=np.uint32)
        N.check(N.load().sld_krylov_unit(self._h, v.handle, N.ptr(rows), m, int(steps),
                                          N.ptr(terms) if terms.size else ctypes.c_void_p(0)))
        return terms

    def krylov_dense(self, v: DeviceVector, xb: XBlock, steps):
        terms = np.zeros((int(steps), xb.m, self.L), dtype=np.uint32)
        N.check(N.load().sld_krylov_dense(self._h, v.handle, xb._h, int(steps),
                                           N.ptr(terms) if terms.size else ctypes.c_void_p(0)))
        return terms

    def bench(self, v: DeviceVector, steps, warmup=3):
        tot = ctypes.c_double()
        per = ctypes.c_double()
        N.check(N.load().sld_bench_spmv(self._h, v.handle, int(steps), int(warmup),
                                         ctypes.byref(tot), ctypes.byref(per)))
        return tot.value, per.value

    def bench_samples(self, v: DeviceVector, steps, warmup=3, pairs_per_sample=1):
        """(total_ms, per-product ms of each sample) -- the samples are the
        durations of consecutive groups of `pairs_per_sample` product pairs."""
        pairs = (int(steps) + 1) // 2
        n = (pairs + pairs_per_sample - 1) // pairs_per_sample
        buf = np.zeros(n, dtype=np.float64)
        tot = ctypes.c_double()
        per = ctypes.c_double()
        N.check(N.load().sld_bench_spmv_samples(self._h, v.handle, int(steps), int(warmup),
                                                 int(pairs_per_sample), N.ptr(buf), ctypes.byref(tot),
                                                 ctypes.byref(per)))
        sizes = np.full(n, 2 * pairs_per_sample, dtype=np.float64)
        sizes[-1] = 2 * (pairs - pairs_per_sample * (n - 1))
        return tot.value, buf / sizes

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_mat_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Block-Wiedemann Krylov driver on the device.

Keeps the reference's plugin protocols and entry points
(sldlag/solver.py:40-268):

  * multiplier protocol -- `.apply(planes) -> planes`, `.count`, `.size`,
    `.mod` (SequentialMultiplier solver.py:129-142).  `B200Multiplier` is the
    drop-in: `block_wiedemann(A, bp, seed, make_mul=lambda j: B200Multiplier(A,
    device=j % ndev))` runs the reference driver on B200s unchanged.
  * projection protocol -- `.project(planes) -> list[int]` (UnitRows /
    DenseRows, solver.py:168-189).
  * `krylov_column` / `krylov_block` / `krylov_scalar` / `krylov_length` with
    the same semantics: a_0 = X^T y is taken before the first product and
    exactly `count` SpMVs run per chain (solver.py:199-217).

The speed comes from `B200Multiplier.krylov`: the whole chain stays on the
device (ping-pong iterate, unit-X projection fused into the SpMV kernel,
CUDA-graph replays), and only the m projected terms per step come back.
`krylov_column` dispatches to it whenever the multiplier has it, and runs the
chain in chunks that end exactly on checkpoint flush / halt boundaries so the
`on_step` / `flush` contract (checkpoint.py:177-200) is honoured.
"""
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .device import DEFAULT_DEVICE, DeviceMatrix, DevicePlanes, DeviceVector, LinCombSet, XBlock, lincomb
from .modring import (
    as_modulus, digit_count, ints_to_limbs, ints_to_planes, limbs_to_ints, limbs_to_planes,
    planes_to_ints, planes_to_limbs,
)

SAFETY_MARGIN = 32
MAX_RESTARTS = 3


class SolverFailure(RuntimeError):
    """The candidate kernel vector degenerated to zero (solver.py:44-46)."""


class GeneratorFailure(RuntimeError):
    """No usable linear generator (solver.py:49-50)."""


@dataclass
class KernelVector:
    w: list
    verified: bool
    horner_spmvs: int = 0
    tail_spmvs: int = 0


def _poly_degree(p) -> int:
    for i in range(len(p) - 1, -1, -1):
        if p[i]:
            return i
    return -1


@dataclass(frozen=True)
class BlockingParams:
    n: int
    m: int

    def __post_init__(self):
        if self.n < 1 or self.m < self.n:
            raise ValueError("need m >= n >= 1")

    @classmethod
    def default(cls, n: int) -> "BlockingParams":
        return cls(n, 2 * n)


def krylov_length(N: int, bp, margin: int = SAFETY_MARGIN) -> int:
    """ceil(N/n) + ceil(N/m) + margin (solver.py:67-68)."""
    return -(-N // bp.n) + -(-N // bp.m) + margin


@dataclass
class BlockSequence:
    """Terms a_i as m x n matrices, stored per y-column (solver.py:71-90)."""
    m: int
    n: int
    columns: list
    spmvs_per_column: list = field(default_factory=list)

    @property
    def count(self) -> int:
        return min(len(c) for c in self.columns) if self.columns else 0

    def term(self, i: int):
        return [[self.columns[j][i][t] for j in range(self.n)] for t in range(self.m)]

    def scalar(self) -> list:
        assert self.m == 1 and self.n == 1
        return [v[0] for v in self.columns[0]]


# -- projections ------------------------------------------------------------


class UnitRows:
    """x-block of unit vectors: a_i reads m coordinates (solver.py:168-176)."""

    def __init__(self, rows):
        self.rows = [int(r) for r in rows]

    def project(self, planes) -> list:
        # row indexing as the reference does (solver.py:174-176): on a
        # DevicePlanes iterate only these m rows leave the device
        return planes_to_ints(planes[self.rows])


class DenseRows:
    """Random dense x-block: a_i[t] = sum_j x_t[j] v[j] (solver.py:179-189).
    On the device path the block is uploaded once (Montgomery form) and each
    step's m dot products run as a grid reduction."""

    def __init__(self, vectors, mod):
        self.vectors = [list(v) for v in vectors]
        self.mod = as_modulus(mod)
        self._dev = {}

    def project(self, planes) -> list:
        ell = self.mod.ell
        v = planes_to_ints(planes)
        return [sum(a * b for a, b in zip(x, v)) % ell for x in self.vectors]

    def device_block(self, dm: DeviceMatrix) -> XBlock:
        key = id(dm.field)
        xb = self._dev.get(key)
        if xb is None:
            L = dm.L
            x = np.stack([ints_to_limbs(vec, L) for vec in self.vectors]) if self.vectors \
                else np.zeros((0, dm.total_cols, L), np.uint32)
            xb = self._dev[key] = XBlock(dm.field, x)
        return xb


# -- multipliers ------------------------------------------------------------


class B200Multiplier:
    """v <- A v on one B200 with an SpMV counter (the multiplier protocol of
    sldlag/solver.py:129-163).  `A` may be this package's SparseMatrix or the
    reference's (same fields).  The device matrix is built lazily on first
    use, so constructing one just to read `.mod` / `.size` is free
    (block_wiedemann does exactly that, solver.py:609-610)."""

    def __init__(self, A, device=None, stripe_cols=0, dm=None):
        if A.nrows != A.ncols + len(getattr(A, "dense_cols", None) or []):
            raise ValueError("solver needs a square matrix")
        self.A = A
        self.size = int(A.nrows)
        self.mod = A.mod
        self.device = DEFAULT_DEVICE if device is None else int(device)
        self.stripe_cols = stripe_cols
        self.count = 0
        self._dm = dm  # an existing DeviceMatrix of A may be shared
        self._lock = threading.Lock()

    @property
    def dm(self) -> DeviceMatrix:
        if self._dm is None:
            self._dm = DeviceMatrix(self.A, self.device, stripe_cols=self.stripe_cols)
        elif isinstance(self._dm, _SharedMatrix):
            self._dm = self._dm.get()
        return self._dm

    def apply(self, planes):
        """v = A u.  The result stays on the device as `DevicePlanes` (an
        array on any host access); an iterate that came from this multiplier
        is not uploaded again, so the reference's per-step loop runs
        device-resident."""
        with self._lock:
            dm = self.dm
            if isinstance(planes, DevicePlanes) and planes._dm is dm:
                src, P, own = planes._vec, planes._P, False
            else:
                p = np.ascontiguousarray(planes, dtype=np.uint64)
                if p.ndim != 2 or p.shape[0] != dm.total_cols:
                    raise ValueError("plane count mismatch")
                P = p.shape[1]
                src, own = dm.pool_get(), True
                src.upload_planes(p)
            out = dm.pool_get()
            dm.spmv(src, out)
            if own:
                dm.pool_put(src)
        self.count += 1
        return DevicePlanes(dm, out, P)

    def krylov(self, xblock, v_planes, steps):
        """`steps` chain steps on the device from iterate `v_planes`:
        returns (terms as list of m-int lists, final iterate).  The final
        iterate stays on the device as `DevicePlanes`, like `.apply`'s result:
        the planes array on any host access (one download then), and passed
        back in (the next checkpoint chunk) it is copied on the device, not
        uploaded."""
        with self._lock:
            dm = self.dm
            vec = dm.pool_get()  # device iterate + its ping-pong twin, recycled
            if isinstance(v_planes, DevicePlanes) and v_planes._dm is dm:
                P = v_planes._P
                dm.copy_vector(v_planes._vec, vec)  # the input object stays untouched
            else:
                p = np.ascontiguousarray(v_planes, dtype=np.uint64)
                P = p.shape[1]
                vec.upload_planes(p)
            if isinstance(xblock, UnitRows):
                terms = dm.krylov_unit(vec, xblock.rows, steps)
            elif isinstance(xblock, DenseRows) or hasattr(xblock, "vectors"):
                db = xblock if isinstance(xblock, DenseRows) else DenseRows(xblock.vectors, self.mod)
                terms = dm.krylov_dense(vec, db.device_block(dm), steps)
            else:
                dm.pool_put(vec)
                raise TypeError(f"unsupported projection block {type(xblock).__name__}")
        self.count += int(steps)
        m = terms.shape[1]
        flat = limbs_to_ints(terms.reshape(-1, terms.shape[2])) if terms.size else []
        out = [flat[i * m:(i + 1) * m] for i in range(int(steps))]
        return out, DevicePlanes(dm, vec, P)


    def mksol(self, Y_planes, polys):
        """Mksol on the device (solver.py:508-552): w = sum_j G_j(B) y_j by
        one Horner chain (SpMV, then the fused combination kernel), then the
        tail B^t w until zero.  Returns (w planes, verified, horner, tail)."""
        with self._lock:
            dm = self.dm
            P = Y_planes[0].shape[1]
            trimmed = [list(p)[: _poly_degree(p) + 1] for p in polys]
            if not any(_poly_degree(p) >= 0 for p in trimmed):
                raise GeneratorFailure("all-zero generators")
            val = min(next((i for i, c in enumerate(p) if c), len(p)) for p in trimmed)
            G = [p[val:] if len(p) > val else [0] for p in trimmed]
            dmax = max(_poly_degree(p) for p in G)
            ys = []
            for yp in Y_planes:
                y = dm.vector()
                y.upload_planes(yp)
                ys.append(y)
            w, t = dm.vector(), dm.vector()
            # tensor-core combination (l < 2^256, n <= 8 y vectors), else
            # the lazy CUDA-core kernel
            lc = None
            if dm.L <= 8 and 1 <= len(ys) <= 8 and os.environ.get("SLD_MKSOL_TC", "1") != "0":
                lc = LinCombSet(dm.field, ys, dm.total_cols)

            def combo(i, acc, dst):
                if lc is not None:
                    lc.apply([p[i] if i <= _poly_degree(p) else 0 for p in G], dst, acc)
                    return
                sel = [(ys[j], p[i]) for j, p in enumerate(G) if i <= _poly_degree(p) and p[i]]
                for k0 in range(0, max(1, len(sel)), 64):
                    part = sel[k0:k0 + 64]
                    lincomb(dm.field, [y for y, _ in part], [c for _, c in part], dst,
                            acc if k0 == 0 else dst)

            # SLD_MKSOL_FUSED=1: the Horner step as one product, the
            # combination in the SpMV's last-pass epilogue (pass layouts).
            # Measured level with the tensor-core combination kernel (cfg3
            # 1.91 vs 1.87 ms, cfg2 0.323 vs 0.335 ms), so it is opt-in.
            fused = dmax > 0 and os.environ.get("SLD_MKSOL_FUSED", "0") == "1" and dm.mksol_bind(ys)
            # SLD_MKSOL_BATCH=2|4 (opt-in): the combinations do not depend on
            # w, so K steps' combinations come from ONE pass over the y tiled
            # in the matrix's slot order (sld_lcset_apply_batch) into K
            # vectors, and each Horner step adds its vector in the SpMV's
            # last-pass epilogue (sld_spmv_add), reading n/K + 1 vectors per
            # step instead of n + 2.  Measured at cfg3 (in-situ kernel times):
            # the combination drops from 198 to 163 us per step, the last pass
            # gains 15 us: 1.797 vs 1.820 ms per step, within the run-to-run
            # noise -- the K reductions per row (carry, fold, Barrett: ~650
            # instructions) bound it, not the y traffic.
            K = int(os.environ.get("SLD_MKSOL_BATCH", "0"))
            info = dm.info()
            batched = (lc is not None and not fused and dmax > 0 and K in (2, 4) and info["chains"] == 1
                       and info["halves"] == 1 and info["lanes_per_residue"] == 1)
            degs = [_poly_degree(p) for p in G]

            def coeffs_at(i):
                return [p[i] if i <= d else 0 for p, d in zip(G, degs)]

            combo(dmax, None, w)
            horner = 0
            if batched:
                lcs = LinCombSet(dm.field, ys, dm.total_cols, matrix=dm)  # slot order
                bufs = [DeviceVector(dm.field, dm.nslots) for _ in range(K)]
                for i0 in range(dmax - 1, -1, -K):
                    steps = list(range(i0, max(i0 - K, -1), -1))
                    sets = [coeffs_at(i) for i in steps] + [[0] * len(G)] * (K - len(steps))
                    lcs.apply_batch(sets, bufs)
                    for k in range(len(steps)):
                        dm.spmv_add(w, t, bufs[k])
                        w, t = t, w
                        horner += 1
                for b in bufs:
                    b.close()
                lcs.close()
            for i in ([] if batched else range(dmax - 1, -1, -1)):
                if fused:
                    dm.spmv_mksol(w, t, coeffs_at(i))
                    w, t = t, w
                else:
                    dm.spmv(w, t, sync=False)  # in stream order with the combination
                    combo(i, t, w)
                horner += 1
            if fused:
                dm.mksol_bind([])
            tail = 0
            dm.spmv(w, t)
            while t.nonzero() and tail < val:
                w, t = t, w
                tail += 1
                dm.spmv(w, t)
            verified = (not t.nonzero()) and w.nonzero()
            w_nonzero = w.nonzero()
            w_planes = w.download_planes(P)
            if lc is not None:
                lc.close()
            for v in ys + [w, t]:
                v.close()
        self.count += horner + tail + 1
        if not w_nonzero:
            raise SolverFailure("kernel candidate degenerated to zero")
        return w_planes, verified, horner, tail


class B200ChainGroup:
    """G block-Wiedemann chains advanced together on one B200 (G = 2 or 4):
    one pass over the matrix serves all G iterates, whose residues sit in
    one record per column so each gather request fetches G residues.  The
    chains stay independent (solver.py:220-257); only the memory traffic is
    shared."""

    def __init__(self, A, chains=2, device=None, stripe_cols=0):
        if A.nrows != A.ncols + len(getattr(A, "dense_cols", None) or []):
            raise ValueError("solver needs a square matrix")
        self.A, self.chains = A, int(chains)
        self.size, self.mod = int(A.nrows), A.mod
        self.device = DEFAULT_DEVICE if device is None else int(device)
        self.stripe_cols = stripe_cols
        self.count = 0
        self._dm = None
        self._vec = None
        self._lock = threading.Lock()

    @property
    def dm(self) -> DeviceMatrix:
        if self._dm is None:
            self._dm = DeviceMatrix(self.A, self.device, stripe_cols=self.stripe_cols,
                                    chains=self.chains)
        return self._dm

    def krylov(self, xblock, v_planes_list, steps):
        """`steps` steps of the G chains from iterates v_planes_list (G arrays
        of planes): returns ([terms of chain g] for g < G, [iterate planes])."""
        if not isinstance(xblock, UnitRows):
            raise TypeError("chain groups project with UnitRows")
        G = self.chains
        if len(v_planes_list) != G:
            raise ValueError(f"expected {G} iterates")
        with self._lock:
            dm = self.dm
            P = v_planes_list[0].shape[1]
            if self._vec is None:
                self._vec = dm.vector()
            self._vec.upload_planes_list(v_planes_list)
            terms = dm.krylov_unit(self._vec, xblock.rows, steps)  # (steps, G, m, L)
            v_out = self._vec.download_planes_list(P)
        self.count += int(steps)
        m = terms.shape[2]
        out = []
        for g in range(G):
            flat = limbs_to_ints(terms[:, g].reshape(-1, terms.shape[3])) if terms.size else []
            out.append([flat[i * m:(i + 1) * m] for i in range(int(steps))])
        return out, v_out


# the reference's name for the default multiplier
SequentialMultiplier = B200Multiplier


def _steps_until_flush(checkpoint, j):
    """How many steps can run before `checkpoint.on_step` could flush or
    halt (so the device chunk can end exactly there)."""
    if hasattr(checkpoint, "steps_until_flush"):
        return max(1, int(checkpoint.steps_until_flush(j)))
    # the reference CheckpointManager (checkpoint.py:67-200)
    every = getattr(checkpoint, "every", None)
    since = getattr(checkpoint, "_since_flush", None)
    if every is None or since is None:
        return 1
    n = int(every) - int(since.get(j, 0))
    halt = getattr(checkpoint, "halt_after", None)
    if halt is not None:
        n = min(n, int(halt) - int(getattr(checkpoint, "_session_steps", 0)))
    return max(1, n)


def krylov_column(mul, xblock, y_planes, count, start_terms=None, checkpoint=None, col_index=0):
    """One chain: terms[i] = X^T (B^i y) for i < count, exactly count SpMVs
    (solver.py:199-217).  Device-resident when `mul` has `.krylov`."""
    terms = list(start_terms) if start_terms else []
    v = y_planes
    spmvs = 0
    if not hasattr(mul, "krylov"):
        for _ in range(len(terms), count):
            terms.append(xblock.project(v))
            v = mul.apply(v)
            spmvs += 1
            if checkpoint is not None:
                checkpoint.on_step(col_index, terms, v)
    else:
        remaining = count - len(terms)
        while remaining > 0:
            if checkpoint is None:
                chunk = remaining
            elif hasattr(checkpoint, "reserve_steps"):  # atomic w.r.t. concurrent columns
                chunk = min(remaining, max(1, int(checkpoint.reserve_steps(col_index, remaining))))
            else:
                chunk = min(remaining, _steps_until_flush(checkpoint, col_index))
            new_terms, v = mul.krylov(xblock, v, chunk)
            spmvs += chunk
            remaining -= chunk
            if checkpoint is None:
                terms.extend(new_terms)
                continue
            # replay the per-step hook; only the chunk's last step can flush
            for t in new_terms:
                terms.append(t)
                checkpoint.on_step(col_index, terms, v)
    if checkpoint is not None and spmvs:
        checkpoint.flush(col_index, terms, v)
    return terms, v, spmvs


def _as_planes(vec, mod):
    return ints_to_planes(vec, digit_count(mod.ell))


def _device_list(devices, n):
    if devices is None:
        from ._native import device_count
        devices = list(range(max(1, device_count())))
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("empty device list")
    return devices[:max(1, n)]


def krylov_block(A, X, Y, count, muls=None, checkpoint=None, contexts=None,
                 chains_per_gpu=1, devices=None) -> BlockSequence:
    """a_i = X^T A^i Y with the n column chains independent
    (solver.py:220-257).  Default multipliers are B200Multipliers spread
    round-robin over `devices` (default: every visible GPU); chains run on
    host threads, one per device slot.  `chains_per_gpu` = 2 or 4 advances
    that many chains per matrix pass (B200ChainGroup; unit X, no checkpoint)
    -- same terms, shared traffic."""
    n = len(Y)
    if chains_per_gpu > 1 and muls is None and checkpoint is None and isinstance(X, UnitRows) \
            and n >= chains_per_gpu:
        return _krylov_block_grouped(A, X, Y, count, chains_per_gpu, contexts, devices)
    lanes = None  # default multipliers: column j on device slot j % ndev
    if muls is None:
        devs = _device_list(devices, n)
        ndev = len(devs)
        # one device matrix per device slot shared by the columns placed on
        # it; the columns of one slot run one after another on that slot's
        # host thread (a DeviceMatrix, like an sld_ctx, is not shared across
        # threads)
        shared = [_SharedMatrix(A, devs[d]) for d in range(ndev)]
        muls = [B200Multiplier(A, device=devs[j % ndev], dm=shared[j % ndev]) for j in range(n)]
        lanes = [list(range(d, n, ndev)) for d in range(ndev)]
    mod = muls[0].mod
    if contexts is None:
        # the reference's default is one context (solver.py:232-233); the
        # default multipliers get one host thread per GPU
        env = os.environ.get("SLDLAG_CONTEXTS")
        contexts = int(env) if env else (len(lanes) if lanes is not None else 1)

    def run(j):
        start = checkpoint.load_column(j) if checkpoint is not None else None
        if start is not None:
            terms0, v_planes = start
            if len(terms0) >= count:
                return terms0[:count], 0
        else:
            terms0, v_planes = [], _as_planes(Y[j], mod)
        terms, _, spmvs = krylov_column(muls[j], X, v_planes, count, start_terms=terms0,
                                        checkpoint=checkpoint, col_index=j)
        return terms, spmvs

    results = [None] * n
    if lanes is not None and contexts > 1 and len(lanes) > 1:
        def run_lane(cols):
            for j in cols:
                results[j] = run(j)
        with ThreadPoolExecutor(max_workers=min(contexts, len(lanes))) as pool:
            list(pool.map(run_lane, lanes))
    elif lanes is None and contexts > 1 and n > 1:
        with ThreadPoolExecutor(max_workers=contexts) as pool:
            results = list(pool.map(run, range(n)))
    else:
        results = [run(j) for j in range(n)]
    if checkpoint is not None and hasattr(checkpoint, "wait"):
        checkpoint.wait()  # the final async flushes are durable (and their errors raised)
    m = len(results[0][0][0]) if results and results[0][0] else 0
    return BlockSequence(m=m, n=n, columns=[r[0] for r in results],
                         spmvs_per_column=[r[1] for r in results])


class _SharedMatrix:
    """A DeviceMatrix of A on one device, built on first use and shared by
    the default multipliers of the columns placed on that device."""

    def __init__(self, A, device):
        self.A, self.device = A, device
        self._dm = None
        self._lock = threading.Lock()

    def get(self) -> DeviceMatrix:
        with self._lock:
            if self._dm is None:
                self._dm = DeviceMatrix(self.A, self.device)
            return self._dm


def _krylov_block_grouped(A, X, Y, count, G, contexts, devices=None):
    devs = _device_list(devices, len(Y))
    ndev = len(devs)
    mod = as_modulus(A.mod)
    groups = [list(range(k, min(k + G, len(Y)))) for k in range(0, len(Y), G)]
    if contexts is None:
        contexts = int(os.environ.get("SLDLAG_CONTEXTS", str(len(groups))))

    def run(gi):
        idx = groups[gi]
        planes = [_as_planes(Y[j], mod) for j in idx]
        if len(idx) < G:  # a short last group runs its chains one by one
            res = []
            for j, yp in zip(idx, planes):
                t, _, _ = krylov_column(B200Multiplier(A, device=devs[gi % ndev]), X, yp, count)
                res.append(t)
            return res
        grp = B200ChainGroup(A, chains=G, device=devs[gi % ndev])
        terms, _ = grp.krylov(X, planes, count)
        return terms

    if contexts > 1 and len(groups) > 1:
        with ThreadPoolExecutor(max_workers=contexts) as pool:
            parts = list(pool.map(run, range(len(groups))))
    else:
        parts = [run(g) for g in range(len(groups))]
    columns = [t for part in parts for t in part]
    m = len(columns[0][0]) if columns and columns[0] else 0
    return BlockSequence(m=m, n=len(Y), columns=columns, spmvs_per_column=[count] * len(Y))


def krylov_scalar(A, x, y, count=None, mul=None) -> list:
    """a_i = x^T A^i y for i < count (default 2N) (solver.py:260-268)."""
    if count is None:
        count = 2 * (A.nrows if A is not None else mul.size)
    if mul is None:
        mul = B200Multiplier(A)
    xb = DenseRows([x], mul.mod)
    terms, _, _ = krylov_column(mul, xb, _as_planes(y, mul.mod), count)
    return [t[0] for t in terms]


def _mksol_core(mul, Y_planes, polys, mod) -> KernelVector:
    """w = sum_j G_j(B) y_j and its kernel check (solver.py:508-552).
    Device-resident when the multiplier has `.mksol`; otherwise the
    reference's loop over `mul.apply` with the combination in Python ints
    (protocol compatibility for foreign multipliers, not a hot path)."""
    if hasattr(mul, "mksol"):
        w, verified, horner, tail = mul.mksol(Y_planes, polys)
        kv = KernelVector(planes_to_ints(w), verified, horner_spmvs=horner, tail_spmvs=tail)
        if not verified:
            raise SolverFailure("candidate is not in the kernel after the tail")
        return kv
    ell = as_modulus(mod).ell
    trimmed = [list(p)[: _poly_degree(p) + 1] for p in polys]
    if not any(_poly_degree(p) >= 0 for p in trimmed):
        raise GeneratorFailure("all-zero generators")
    val = min(next((i for i, c in enumerate(p) if c), len(p)) for p in trimmed)
    G = [p[val:] if len(p) > val else [0] for p in trimmed]
    dmax = max(_poly_degree(p) for p in G)
    width = Y_planes[0].shape[1]
    Yi = [planes_to_ints(y) for y in Y_planes]

    def combo(i, base=None):
        acc = list(base) if base is not None else [0] * len(Yi[0])
        for j, p in enumerate(G):
            if i <= _poly_degree(p) and p[i]:
                acc = [(a + p[i] * b) % ell for a, b in zip(acc, Yi[j])]
        return acc

    w = combo(dmax)
    horner = 0
    for i in range(dmax - 1, -1, -1):
        w = combo(i, planes_to_ints(mul.apply(ints_to_planes(w, width))))
        horner += 1
    tail = 0
    nxt = planes_to_ints(mul.apply(ints_to_planes(w, width)))
    while any(nxt) and tail < val:
        w = nxt
        tail += 1
        nxt = planes_to_ints(mul.apply(ints_to_planes(w, width)))
    verified = not any(nxt) and any(w)
    if not any(w):
        raise SolverFailure("kernel candidate degenerated to zero")
    kv = KernelVector(w, verified, horner_spmvs=horner, tail_spmvs=tail)
    if not verified:
        raise SolverFailure("candidate is not in the kernel after the tail")
    return kv


def mksol_scalar(A, y, F, mul=None) -> KernelVector:
    if mul is None:
        mul = B200Multiplier(A)
    return _mksol_core(mul, [_as_planes(y, mul.mod)], [F], mul.mod)


def mksol_block(A, Y, G, mul=None) -> KernelVector:
    """G: Generators-like (`.polys`, one polynomial per y column)."""
    if mul is None:
        mul = B200Multiplier(A)
    return _mksol_core(mul, [_as_planes(y, mul.mod) for y in Y], list(G.polys), mul.mod)


def verify_kernel(A, w) -> bool:
    """True iff A w = 0 and w != 0 (solver.py:568-573)."""
    from .spmatrix import spmv_sequential
    if not any(w):
        return False
    return not any(spmv_sequential(A, w))


def draw_blocks(mod, size: int, bp, rng, x_mode="unit", forced_zero=()):
    """Random Y block and projection block (solver.py:578-596): the same
    draws in the same order, so seeds give the reference's blocks."""
    mod = as_modulus(mod)
    fz = set(forced_zero)
    allowed = [i for i in range(size) if i not in fz]
    Y = []
    for _ in range(bp.n):
        y = mod.random_residues(rng, size)
        for z in forced_zero:
            y[z] = 0
        Y.append(y)
    if x_mode == "unit":
        picks = rng.choice(len(allowed), size=bp.m, replace=False)
        return UnitRows(sorted(allowed[int(r)] for r in picks)), Y
    if x_mode == "dense":
        return DenseRows([mod.random_residues(rng, size) for _ in range(bp.m)], mod), Y
    raise ValueError(f"unknown x_mode {x_mode!r}")


__all__ = [
    "B200ChainGroup", "KernelVector", "SolverFailure", "GeneratorFailure", "mksol_block", "mksol_scalar",
    "verify_kernel", "MAX_RESTARTS",
    "BlockingParams", "BlockSequence", "B200Multiplier", "SequentialMultiplier", "UnitRows",
    "DenseRows", "krylov_column", "krylov_block", "krylov_scalar", "krylov_length",
    "draw_blocks", "SAFETY_MARGIN", "planes_to_limbs", "limbs_to_planes",
]

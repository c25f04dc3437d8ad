"""One Krylov chain over an r x c grid of GPUs (BASELINE cfg4).

The B200 restatement of the reference's grid engine
(sldlag/gridmv.py:193-354): node (i, j) holds block A_ij of the balanced,
padded matrix (balance.py) and the column fragment u_j.  One iteration:

  1. partial p_ij = A_ij u_j                      (the SpMV kernel, local)
  2. row i's partials reach the collector (i, i mod c), which sums them
     mod l                                        (NCCL p2p + sld_add_mod)
  3. each collector sends the overlap of its row piece with every column
     range to the nodes of that column           (NCCL p2p; an all-gather
     on r x 1 grids)

One process per GPU (torch.distributed, rank = i*c + j).  The exchange
schedule, the collector rule and the message/byte log (CommLog, the
reference's accounting: rows x byte_width, gridmv.py:151-176) follow the
reference, so `comm_volume_model` predicts the bytes exactly.  Failure
detection mirrors gridmv.py:46-51: every p2p payload travels behind its tag
(iteration, kind, source), a wrong tag raises GridProtocolError, a message
that does not arrive within GridComm's timeout GridTimeoutError.

The compute and buffer side is an *engine*: `DeviceEngine` runs on
libsldb200 (device fragments, CUDA kernels); tests substitute a CPU engine
backed by the oracle to exercise the exchange logic under gloo.
"""
import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .balance import BlockSplit, GridSpec, balance_permutation, padded_size, split
from .device import DeviceMatrix, DeviceVector, Field
from .modring import as_modulus, digit_count, limbs_to_ints, limbs_to_planes, planes_to_limbs

KIND_PARTIAL_SUM = 0
KIND_FRAGMENT = 1


# raised by the native grid's barriers (sld_grid_wait) and by the exchange
# checks below; defined next to the status mapping in _native
from ._native import GridProtocolError, GridTimeoutError  # noqa: E402


@dataclass
class PhaseLog:
    messages: int = 0
    bytes: int = 0
    wire_bytes: int = 0


@dataclass
class IterationLog:
    iteration: int
    reduce: PhaseLog = field(default_factory=PhaseLog)
    broadcast: PhaseLog = field(default_factory=PhaseLog)

    @property
    def total_bytes(self):
        return self.reduce.bytes + self.broadcast.bytes


class CommLog:
    def __init__(self):
        self.entries = []

    def total_bytes(self):
        return sum(e.total_bytes for e in self.entries)

    def total_messages(self):
        return sum(e.reduce.messages + e.broadcast.messages for e in self.entries)


# ---------------------------------------------------------------- engines


class _CAI:
    """__cuda_array_interface__ view of raw device memory (for torch)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": "<i4", "version": 3, "strides": None}


class DeviceEngine:
    """Block SpMV + mod-l sums on this process's GPU (libsldb200)."""

    def __init__(self, block, device, stripe_cols=0):
        import torch
        self.torch = torch
        self.device = int(device)
        self.mod = as_modulus(block.mod)
        self.field = Field(self.mod, self.device)
        self.L = self.field.L
        self.W = ((self.L + 7) // 8) * 8  # slot words
        # run our kernels on torch's stream so NCCL orders with them
        torch.cuda.set_device(self.device)
        N.check(N.load().sld_ctx_set_stream(self.field.handle,
                                            torch.cuda.current_stream(self.device).cuda_stream))
        self.dm = DeviceMatrix(block, self.device, stripe_cols=stripe_cols, field=self.field)

    def alloc(self, n):
        v = DeviceVector(self.field, n)
        p, s = ctypes.c_uint64(), ctypes.c_int64()
        N.check(N.load().sld_vec_device_ptr(v.handle, ctypes.byref(p), ctypes.byref(s)))
        v.tensor = self.torch.as_tensor(_CAI(p.value, (n, s.value)), device=f"cuda:{self.device}")
        return v

    def scratch(self, n):
        return self.torch.empty((n, self.W), dtype=self.torch.int32, device=f"cuda:{self.device}")

    def spmv(self, src, dst):
        self.dm.spmv(src, dst)

    def add_mod(self, dst_tensor, src_tensors):
        ptrs = np.array([t.data_ptr() for t in src_tensors], dtype=np.uint64)
        N.check(N.load().sld_add_mod(self.field.handle, N.ptr(ptrs), len(ptrs),
                                     dst_tensor.data_ptr(), dst_tensor.shape[0]))

    def upload(self, buf, limbs):
        buf.upload_limbs(limbs)

    def download(self, buf):
        return buf.download_limbs()

    def read_rows(self, buf, rows):
        rows = N.c64(rows)
        out = np.zeros((len(rows), self.L), dtype=np.uint32)
        if len(rows):
            N.check(N.load().sld_vec_read_rows(buf.handle, N.ptr(rows), len(rows), N.ptr(out)))
        return out

    def sync(self):
        self.torch.cuda.synchronize(self.device)


# ------------------------------------------------------------------- comm


class GridComm:
    """rank = i*c + j; p2p batches over torch.distributed.  With a CPU-only
    backend (gloo) and device tensors, payloads are staged through host
    memory."""

    def __init__(self, g: GridSpec, group=None, timeout=300.0):
        import datetime

        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.g = g
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != g.r * g.c:
            raise ValueError(f"grid {g} needs {g.r * g.c} ranks, have {self.world}")
        self.staged = dist.get_backend(group) != "nccl"
        self.timeout = datetime.timedelta(seconds=float(timeout))

    def rank_of(self, i, j):
        return i * self.g.c + j

    def header(self, iteration, kind, like):
        """A message's tag (gridmv.py Message: kind, src, iteration)."""
        dev = "cpu" if self.staged or not like.is_cuda else like.device
        return self.torch.tensor([iteration, kind, self.rank], dtype=self.torch.int64, device=dev)

    def exchange(self, sends, recvs, iteration=None, kind=None):
        """sends: [(tensor, dst)], recvs: [(tensor, src)] as one p2p batch.
        With `iteration`, every payload travels behind its tag (iteration,
        kind, src) and a received tag other than the expected one raises
        GridProtocolError (gridmv.py:276-283); a message that does not
        arrive within the timeout raises GridTimeoutError (gridmv.py:285-290)."""
        dist = self.dist
        if not sends and not recvs:
            return
        if self.staged:
            s2 = [(t.cpu() if t.is_cuda else t, d) for t, d in sends]
            r2 = [(self.torch.empty(t.shape, dtype=t.dtype) if t.is_cuda else t, s) for t, s in recvs]
        else:
            s2, r2 = sends, recvs
        ops = []
        tags_in = []
        if iteration is not None:
            ops += [dist.P2POp(dist.isend, self.header(iteration, kind, t), d, self.group) for t, d in s2]
            for t, s_ in r2:
                h = self.torch.empty(3, dtype=self.torch.int64, device=self.header(0, 0, t).device)
                tags_in.append((h, s_))
                ops.append(dist.P2POp(dist.irecv, h, s_, self.group))
        ops += [dist.P2POp(dist.isend, t, d, self.group) for t, d in s2]
        ops += [dist.P2POp(dist.irecv, t, s, self.group) for t, s in r2]
        try:
            for w in dist.batch_isend_irecv(ops):
                w.wait(timeout=self.timeout)
        except RuntimeError as e:
            if "imed out" in str(e) or "imeout" in str(e):
                raise GridTimeoutError(f"rank {self.rank}: exchange of iteration {iteration} timed out: {e}")
            if "onnection closed" in str(e) or "onnection reset" in str(e):
                # a peer that timed out first tears its connections down: the
                # message this rank waits for is lost just the same
                raise GridTimeoutError(f"rank {self.rank}: exchange of iteration {iteration} lost its peer: {e}")
            raise
        for h, src in tags_in:
            it, kd, sr = (int(x) for x in h.cpu().tolist())
            if it != iteration or kd != kind or sr != src:
                raise GridProtocolError(f"rank {self.rank} got iteration {it} kind {kd} from rank {sr}, "
                                        f"expected iteration {iteration} kind {kind} from rank {src}")
        if self.staged:
            for (t, _), (t2, _) in zip(recvs, r2):
                if t.is_cuda:
                    t.copy_(t2)

    def all_gather(self, out, inp):
        if self.staged and inp.is_cuda:
            o2 = self.torch.empty(out.shape, dtype=out.dtype)
            self.dist.all_gather_into_tensor(o2, inp.cpu(), group=self.group)
            out.copy_(o2)
        else:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# ------------------------------------------------------------------- grid


class B200Grid:
    """This process's node of the distributed grid (gridmv.Grid analogue).

    Built from the full matrix (each rank materialises only its own block)
    or from a BlockSplit.  Vectors given to `load_vector` / returned by
    `assembled` live in the permuted, padded coordinates (n_padded), as in
    the reference.
    """

    def __init__(self, A_or_split, g: GridSpec = None, comm: GridComm = None, engine_factory=None,
                 device=None, perm=None):
        if isinstance(A_or_split, BlockSplit):
            bs = A_or_split
            g = bs.grid
        else:
            A = A_or_split
            if g is None:
                raise ValueError("grid spec required")
            p = perm if perm is not None else balance_permutation(A, g)
            self.perm = p
            bs = None
        self.g = g
        self.comm = comm or GridComm(g)
        self.i, self.j = divmod(self.comm.rank, g.c)
        if bs is None:
            bs = split(A, p, g, only={(self.i, self.j)})
        self.bs = bs
        self.mod = as_modulus(bs.blocks[self.i][self.j].mod)
        self.n_padded = bs.n_padded
        self.br, self.bc = bs.block_rows, bs.block_cols
        block = bs.blocks[self.i][self.j]
        if engine_factory is None:
            dev = self.comm.rank if device is None else device
            self.engine = DeviceEngine(block, dev)
        else:
            self.engine = engine_factory(block)
        e = self.engine
        self.frag = [e.alloc(self.bc), e.alloc(self.bc)]  # ping-pong column fragments
        self.cur = 0
        self.partial = e.alloc(self.br)
        self.collector = self.j == self.collector_col(self.i)
        self.row_piece = e.scratch(self.br) if self.collector and g.c > 1 else None
        self.inbox = [e.scratch(self.br) for _ in range(g.c - 1)] if self.collector else []
        self.comm_log = CommLog()
        self.spmv_count = 0
        self.iteration = 0
        self.byte_width = self.mod.byte_width

    # -- geometry (gridmv.py:214-223) ------------------------------------
    def collector_col(self, i):
        return i % self.g.c

    def row_range(self, i):
        return i * self.br, (i + 1) * self.br

    def col_range(self, j):
        return j * self.bc, (j + 1) * self.bc

    # -- vectors ------------------------------------------------------------
    def load_vector(self, limbs):
        """Full padded vector (n_padded x L limbs, same on every rank)."""
        limbs = np.asarray(limbs, dtype=np.uint32)
        if limbs.shape[0] != self.n_padded:
            raise ValueError("vector length != padded size")
        lo, hi = self.col_range(self.j)
        self.engine.upload(self.frag[self.cur], np.ascontiguousarray(limbs[lo:hi]))

    def load_planes(self, planes):
        self.load_vector(planes_to_limbs(planes, self.engine.L))

    def assembled(self):
        """Concatenation of the column fragments (held by the row-0 nodes)."""
        mine = self.engine.download(self.frag[self.cur]) if self.i == 0 else None
        parts = self.comm.all_gather_object((self.j, mine) if self.i == 0 else None)
        got = {j: a for item in parts if item is not None for j, a in [item]}
        return np.concatenate([got[j] for j in range(self.g.c)])

    # -- the iteration (gridmv.py:251-348) ------------------------------------
    def iterate(self, count=1):
        for _ in range(count):
            self._one_iteration()
        return self.comm_log

    def _one_iteration(self):
        g, e = self.g, self.engine
        log = IterationLog(self.iteration)
        src, dst = self.frag[self.cur], self.frag[self.cur ^ 1]
        # phase 1: local partial product
        e.spmv(src, self.partial)
        self.spmv_count += 1
        # phase 2: partials to the row collector, summed mod l
        ci = self.collector_col(self.i)
        sends, recvs = [], []
        if not self.collector:
            sends.append((self.partial.tensor, self.comm.rank_of(self.i, ci)))
        else:
            others = [j for j in range(g.c) if j != ci]
            for k, j in enumerate(others):
                recvs.append((self.inbox[k], self.comm.rank_of(self.i, j)))
        self.comm.exchange(sends, recvs, self.iteration, KIND_PARTIAL_SUM)
        for i in range(g.r):  # the reference's accounting, identical on every rank
            log.reduce.messages += g.c - 1
            log.reduce.bytes += (g.c - 1) * self.br * self.byte_width
            log.reduce.wire_bytes += (g.c - 1) * self.br * e.W * 4
        if self.collector and g.c > 1:
            e.add_mod(self.row_piece, [self.partial.tensor] + self.inbox)
        # phase 3: collectors send row-piece / column-range overlaps
        clo, chi = self.col_range(self.j)
        if g.c == 1:
            # r x 1: every node is its row's collector and its partial is the
            # finished row piece -> one all-gather
            self.comm.all_gather(dst.tensor, self.partial.tensor)
        else:
            sends, recvs = [], []
            covered = np.zeros(chi - clo, dtype=bool)
            for i in range(g.r):
                c_i = self.collector_col(i)
                rlo, rhi = self.row_range(i)
                if self.collector and i == self.i:
                    for jj in range(g.c):
                        lo, hi = max(rlo, self.col_range(jj)[0]), min(rhi, self.col_range(jj)[1])
                        if lo >= hi:
                            continue
                        for k in range(g.r):
                            if (k, jj) == (i, c_i):
                                continue
                            sends.append((self.row_piece[lo - rlo:hi - rlo], self.comm.rank_of(k, jj)))
                lo, hi = max(rlo, clo), min(rhi, chi)
                if lo >= hi:
                    continue
                if (self.i, self.j) == (i, c_i):
                    dst.tensor[lo - clo:hi - clo].copy_(self.row_piece[lo - rlo:hi - rlo])
                else:
                    recvs.append((dst.tensor[lo - clo:hi - clo], self.comm.rank_of(i, c_i)))
                covered[lo - clo:hi - clo] = True
            if not covered.all():
                raise GridTimeoutError(f"node {(self.i, self.j)}: fragment coverage incomplete")
            self.comm.exchange(sends, recvs, self.iteration, KIND_FRAGMENT)
        for i in range(g.r):
            c_i = self.collector_col(i)
            rlo, rhi = self.row_range(i)
            for jj in range(g.c):
                lo, hi = max(rlo, self.col_range(jj)[0]), min(rhi, self.col_range(jj)[1])
                if lo < hi:
                    n_recv = g.r - (1 if c_i == jj else 0)
                    log.broadcast.messages += n_recv
                    log.broadcast.bytes += n_recv * (hi - lo) * self.byte_width
                    log.broadcast.wire_bytes += n_recv * (hi - lo) * e.W * 4
        self.cur ^= 1
        self.comm_log.entries.append(log)
        self.iteration += 1

    def apply_once(self, limbs):
        self.load_vector(limbs)
        self.iterate(1)
        return self.assembled()

    def project_rows(self, rows):
        """{row: limbs} for the unit rows inside this node's fragment (row-0
        nodes only, so every row is reported once)."""
        if self.i != 0:
            return {}
        lo, hi = self.col_range(self.j)
        mine = [r for r in rows if lo <= r < hi]
        vals = self.engine.read_rows(self.frag[self.cur], [r - lo for r in mine])
        return {r: vals[k] for k, r in enumerate(mine)}


class GridMultiplier:
    """The multiplier protocol over a grid (solver.py:145-162): `.apply`
    runs one grid iteration, `.count` is the grid's SpMV count, `.size` the
    padded size.  SPMD: every rank calls with the same arguments."""

    def __init__(self, grid: B200Grid):
        self.grid = grid
        self.size = grid.n_padded
        self.mod = grid.mod

    @property
    def count(self):
        return self.grid.spmv_count

    @property
    def comm_log(self):
        return self.grid.comm_log

    def apply(self, planes):
        P = planes.shape[1]
        out = self.grid.apply_once(planes_to_limbs(planes, self.grid.engine.L))
        return limbs_to_planes(out, P)

    def krylov(self, xblock, v_planes, steps):
        """Device-resident chain over the grid with unit projections."""
        rows = list(getattr(xblock, "rows", []))
        if not hasattr(xblock, "rows"):
            raise TypeError("grid Krylov supports UnitRows projections")
        g = self.grid
        g.load_planes(v_planes)
        local = []
        for _ in range(int(steps)):
            local.append(g.project_rows(rows))
            g.iterate(1)
        merged = [dict() for _ in range(int(steps))]
        for part in g.comm.all_gather_object(local):
            for s, d in enumerate(part):
                merged[s].update(d)
        terms = [[int.from_bytes(np.ascontiguousarray(merged[s][r], dtype="<u4").tobytes(), "little")
                  for r in rows] for s in range(int(steps))]
        v = limbs_to_planes(g.assembled(), v_planes.shape[1])
        return terms, v


__all__ = ["B200Grid", "GridMultiplier", "GridComm", "DeviceEngine", "CommLog", "IterationLog",
           "PhaseLog", "GridProtocolError", "GridTimeoutError", "GridSpec", "padded_size"]

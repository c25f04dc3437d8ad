"""One Krylov chain over an r x c grid of GPUs with every exchange done by the
nodes themselves over peer memory (the fused alternative
to the reference's grid iteration, sldlag/gridmv.py:251-348).

The data path is native (`sld_grid_*` in include/sldb200.h,
csrc/sld_grid.cu): node (i, j) holds block A_ij of the balanced, padded
matrix B = P_r A P_c^T (balance.py) and the fragment u_j.  One iteration is
one replayed CUDA graph:

  r x 1 : the block's SpMV stores every output row straight into every
          node's next iterate (the all-gather done by the epilogue), then a
          flag barrier;
  r x c : the SpMV stores its partial into slot j of the row collector
          (i, i mod c)'s inbox; barrier; the collector sums the c partials
          mod l and one scatter kernel copies each column-range overlap of
          its row piece into the next fragment of every node of that
          column; barrier.

There is no collective and no host synchronisation per iteration: the host
only checks the barriers' error word once per `wait`.  A node that stops
makes the others raise GridTimeoutError; a node at another iteration (stale
or restarted) makes them raise GridProtocolError (gridmv.py:46-51).

Node records (pointer + CUDA IPC handle, SLD_GRID_BLOB bytes) cross once at
setup: `PeerGrid` (one process per GPU) all-gathers them with the caller's
`exchange(obj) -> list` (torch.distributed.all_gather_object in practice);
`LocalGrid` keeps every node in this process (one per GPU, or several
sharing a GPU), like ncclCommInitAll.  `GridMultiplier` puts either behind
the reference's multiplier protocol (solver.py:145-162: `.apply` = one grid
iteration on the padded permuted matrix, `.count`, `.size`, `.mod`) plus
`.krylov` with unit-X projections recorded on the device.
"""
import ctypes

import numpy as np

from . import _native as N
from .balance import GridSpec, balance_permutation, split
from .device import DeviceMatrix, Field
from .modring import as_modulus, limbs_to_ints, limbs_to_planes, planes_to_limbs

TERM_RING = 1024  # steps of unit-X terms kept on the device between drains


class GridNode:
    """One node of the native grid: the block matrix on its device and the
    sld_grid handle (fragments, inbox, control block in one shared
    allocation)."""

    def __init__(self, A, g: GridSpec, rank: int, device=0, perm=None, bs=None):
        if g.r * g.c > 8:
            raise ValueError("the peer grid supports up to 8 nodes")
        self.g, self.rank, self.device = g, int(rank), int(device)
        self.i, self.j = divmod(self.rank, g.c)
        if bs is None:
            perm = perm if perm is not None else balance_permutation(A, g)
            bs = split(A, perm, g, only={(self.i, self.j)})
        self.n_padded, self.br, self.bc = bs.n_padded, bs.block_rows, bs.block_cols
        block = bs.blocks[self.i][self.j]
        self.mod = as_modulus(block.mod)
        self.L = self.mod.limbs
        self.field = Field(self.mod, self.device)
        self.dm = DeviceMatrix(block, self.device, field=self.field)
        h = ctypes.c_void_p()
        N.check(N.load().sld_grid_create(self.dm.handle, g.r, g.c, self.rank, self.n_padded, ctypes.byref(h)))
        self._h = h
        self.collector = self.j == self.i % g.c
        self.m = 0
        self.owned = np.zeros(0, dtype=np.uint8)

    @property
    def handle(self):
        return self._h

    def blob(self) -> bytes:
        b = np.zeros(N.SLD_GRID_BLOB, dtype=np.uint8)
        N.check(N.load().sld_grid_blob(self._h, N.ptr(b)))
        return b.tobytes()

    def connect(self, blobs):
        """All nodes' records, in rank order."""
        if len(blobs) != self.g.r * self.g.c:
            raise ValueError("one record per node expected")
        buf = np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()
        N.check(N.load().sld_grid_connect(self._h, N.ptr(buf)))

    def set_timeout(self, seconds):
        N.check(N.load().sld_grid_set_timeout(self._h, float(seconds)))

    def set_epoch(self, epoch):
        N.check(N.load().sld_grid_set_epoch(self._h, int(epoch)))

    def load(self, fragment_limbs):
        f = np.ascontiguousarray(fragment_limbs, dtype=np.uint32)
        if f.shape != (self.bc, self.L):
            raise ValueError(f"fragment must be {self.bc} x {self.L} limbs")
        N.check(N.load().sld_grid_load(self._h, N.ptr(f)))

    def fragment(self):
        out = np.zeros((self.bc, self.L), dtype=np.uint32)
        N.check(N.load().sld_grid_read(self._h, N.ptr(out)))
        return out

    def set_projection(self, rows, max_steps=TERM_RING):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        self.m = len(rows)
        self.owned = np.zeros(self.m, dtype=np.uint8)
        N.check(N.load().sld_grid_set_projection(self._h, N.ptr(rows) if self.m else None, self.m,
                                                 int(max_steps), N.ptr(self.owned) if self.m else None))
        return self.owned.astype(bool)

    def terms(self):
        """Drain the recorded terms: (steps, m, L) limbs, zero where another
        node reports the row."""
        cap = np.zeros(1, dtype=np.int64)
        out = np.zeros((TERM_RING, max(self.m, 1), self.L), dtype=np.uint32)
        N.check(N.load().sld_grid_terms(self._h, N.ptr(out), N.ptr(cap)))
        return out[:int(cap[0]), :self.m]

    def launch(self, count=1):
        N.check(N.load().sld_grid_launch(self._h, int(count)))

    def wait(self):
        N.check(N.load().sld_grid_wait(self._h))

    def info(self):
        a = np.zeros(8, dtype=np.int64)
        N.check(N.load().sld_grid_info(self._h, N.ptr(a)))
        keys = ["iteration", "nodes", "block_rows", "block_cols", "collector", "shared_bytes", "parity",
                "kernels_per_iteration"]
        return dict(zip(keys, (int(x) for x in a)))

    def close(self):
        if getattr(self, "_h", None):
            N.load().sld_grid_destroy(self._h)
            self._h = None
        if getattr(self, "dm", None) is not None:
            self.dm.close()
            self.dm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _GridBase:
    """Shared host side: fragments of the padded start vector, assembly."""

    def _fragment_of(self, limbs, j):
        limbs = np.asarray(limbs, dtype=np.uint32)
        if limbs.shape[0] != self.n_padded:
            raise ValueError(f"vector of {limbs.shape[0]} residues, grid needs {self.n_padded}")
        lo = j * self.bc
        return np.ascontiguousarray(limbs[lo:lo + self.bc])


class LocalGrid(_GridBase):
    """All r*c nodes in this process: node k on devices[k] (default: round
    robin over the visible GPUs; on one GPU every node shares it).  The
    launches of all nodes are interleaved iteration by iteration, then every
    node is waited on, so no node's queue can fill while a peer it waits for
    has nothing enqueued."""

    def __init__(self, A, g: GridSpec, devices=None, perm=None):
        self.g = g
        nodes = g.r * g.c
        if devices is None:
            nd = max(1, N.device_count())
            devices = [k % nd for k in range(nodes)]
        if len(devices) != nodes:
            raise ValueError("one device per node")
        self.perm = perm if perm is not None else balance_permutation(A, g)
        bs = split(A, self.perm, g)
        self.nodes = [GridNode(A, g, k, devices[k], bs=bs) for k in range(nodes)]
        blobs = [nd.blob() for nd in self.nodes]
        for nd in self.nodes:
            nd.connect(blobs)
        n0 = self.nodes[0]
        self.n_padded, self.br, self.bc, self.mod = n0.n_padded, n0.br, n0.bc, n0.mod
        self.spmv_count = 0

    def load_vector(self, limbs):
        for nd in self.nodes:
            nd.load(self._fragment_of(limbs, nd.j))

    def set_timeout(self, seconds):
        for nd in self.nodes:
            nd.set_timeout(seconds)

    def iterate(self, count=1):
        for _ in range(int(count)):
            for nd in self.nodes:
                nd.launch(1)
        self.spmv_count += int(count)
        errors = []
        for nd in self.nodes:
            try:
                nd.wait()
            except Exception as e:  # wait for every node, report the first failure
                errors.append(e)
        if errors:
            raise errors[0]

    def assembled(self):
        """The full padded iterate: u_j from node (0, j) for every j."""
        return np.concatenate([self.nodes[j].fragment() for j in range(self.g.c)])

    def apply_once(self, limbs):
        self.load_vector(limbs)
        self.iterate(1)
        return self.assembled()

    def set_projection(self, rows, max_steps=TERM_RING):
        owners = np.zeros(len(rows), dtype=bool)
        for nd in self.nodes:
            owners |= nd.set_projection(rows, max_steps)
        if len(rows) and not owners.all():
            raise ValueError("projection rows not covered by the grid")

    def terms(self):
        parts = [nd.terms() for nd in self.nodes]
        out = parts[0].copy()
        for nd, p in zip(self.nodes[1:], parts[1:]):
            if p.shape[0] != out.shape[0]:
                raise N.GridProtocolError("nodes recorded different step counts")
            out[:, nd.owned.astype(bool)] = p[:, nd.owned.astype(bool)]
        return out

    def close(self):
        for nd in self.nodes:
            nd.close()


class PeerGrid(_GridBase):
    """This process's node of an r x c grid whose other nodes run in other
    processes (one per GPU).  SPMD: every rank makes the same calls."""

    def __init__(self, A, g: GridSpec, rank: int, exchange, device=0, perm=None):
        self.g, self.rank = g, int(rank)
        self.perm = perm if perm is not None else balance_permutation(A, g)
        self.node = GridNode(A, g, rank, device, perm=self.perm)
        self.exchange = exchange
        blobs = exchange((self.rank, self.node.blob()))
        self.node.connect([b for _, b in sorted(blobs)])
        nd = self.node
        self.i, self.j = nd.i, nd.j
        self.n_padded, self.br, self.bc, self.mod = nd.n_padded, nd.br, nd.bc, nd.mod
        self.field, self.dm = nd.field, nd.dm
        self.spmv_count = 0

    def load_vector(self, limbs):
        """The full padded start vector (the same on every rank)."""
        self.node.load(self._fragment_of(limbs, self.j))
        self.exchange(None)  # everyone loaded before anyone pushes

    def set_timeout(self, seconds):
        self.node.set_timeout(seconds)

    def iterate(self, count=1):
        self.node.launch(count)
        self.spmv_count += int(count)
        self.node.wait()

    def fragment(self):
        return self.node.fragment()

    def vector(self):
        """r x 1: this node's copy of the full iterate."""
        if self.g.c != 1:
            raise ValueError("only r x 1 nodes hold the whole iterate; use assembled()")
        return self.node.fragment()

    def assembled(self):
        mine = self.node.fragment() if self.i == 0 else None
        parts = dict((j, f) for j, f in self.exchange((self.j, mine)) if f is not None)
        return np.concatenate([parts[j] for j in range(self.g.c)])

    def apply_once(self, limbs):
        self.load_vector(limbs)
        self.iterate(1)
        return self.assembled()

    def set_projection(self, rows, max_steps=TERM_RING):
        self.node.set_projection(rows, max_steps)

    def terms(self):
        mine = self.node.terms()
        out = mine.copy()
        for owned, p in self.exchange((self.node.owned, mine)):
            out[:, owned.astype(bool)] = p[:, owned.astype(bool)]
        return out

    def close(self):
        self.node.close()


def PeerRowGrid(A, r: int, rank: int, exchange, device=0, perm=None):
    """r x 1 node (every node ends each iteration with the whole iterate)."""
    return PeerGrid(A, GridSpec(int(r), 1), rank, exchange, device=device, perm=perm)


class GridMultiplier:
    """The reference's multiplier protocol over a peer-memory grid
    (solver.py:145-162): `.apply(planes)` is one grid iteration on the
    padded, permuted matrix B (Grid.apply_once, gridmv.py:350-354), `.count`
    the grid's SpMV count, `.size` the padded size; `.krylov` keeps the
    chain on the devices and records unit-X terms there, draining them once
    per TERM_RING steps."""

    def __init__(self, grid):
        self.grid = grid
        self.size = grid.n_padded
        self.mod = grid.mod

    @property
    def count(self):
        return self.grid.spmv_count

    def apply(self, planes):
        P = planes.shape[1]
        out = self.grid.apply_once(planes_to_limbs(np.asarray(planes), self.mod.limbs))
        return limbs_to_planes(out, P)

    def krylov(self, xblock, v_planes, steps):
        if not hasattr(xblock, "rows"):
            raise TypeError("grid Krylov supports UnitRows projections")
        rows = list(xblock.rows)
        g = self.grid
        g.load_vector(planes_to_limbs(np.asarray(v_planes), self.mod.limbs))
        g.set_projection(rows, TERM_RING)
        out = []
        left = int(steps)
        while left > 0:
            n = min(left, TERM_RING)
            g.iterate(n)
            t = g.terms()
            flat = limbs_to_ints(t.reshape(-1, self.mod.limbs)) if t.size else []
            m = len(rows)
            out.extend(flat[k * m:(k + 1) * m] for k in range(n))
            left -= n
        g.set_projection([], 1)
        return out, limbs_to_planes(g.assembled(), v_planes.shape[1])

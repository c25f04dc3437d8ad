"""One Krylov chain over an r x 1 grid with the all-gather fused into the
SpMV (the fused alternative to the reference's broadcast
phase, gridmv.py:251-348).

Node i (one process per GPU) holds block A_i = rows [i*br, (i+1)*br) of the
balanced, padded matrix B = P_r A P_c^T (balance.py) against ALL columns, and
a full copy of the iterate.  One iteration:

  1. y_i = A_i x on node i.  The last SpMV pass stores every output row
     straight into every node's NEXT iterate buffer at rows i*br + row,
     through peer pointers (NVLink P2P between GPUs; CUDA IPC handles carry
     the buffers across processes).  There is no separate collective.
  2. a flag barrier: each node adds 1 to every node's flag word
     (system-scope atomics), then waits for its own to reach r * iterations.
     Ping-pong iterate buffers make one barrier per iteration sufficient:
     nobody writes a buffer that a peer may still read.

The node outputs are identical to the reference Grid's (r x 1 golden cases,
tests/test_peergrid_gpu.py).  `exchange(obj) -> list` all-gathers small host
objects (torch.distributed.all_gather_object in practice).
"""
import ctypes

import numpy as np

from . import _native as N
from .balance import GridSpec, balance_permutation, split
from .device import DeviceMatrix, DeviceVector, Field
from .modring import as_modulus


class PeerRowGrid:
    def __init__(self, A, r: int, rank: int, exchange, device=0, perm=None):
        if not 1 <= r <= 8:
            raise ValueError("peer push supports 1..8 nodes")
        self.r, self.rank, self.device = int(r), int(rank), int(device)
        self.g = GridSpec(self.r, 1)
        self.perm = perm if perm is not None else balance_permutation(A, self.g)
        bs = split(A, self.perm, self.g, only={(self.rank, 0)})
        self.n_padded, self.br = bs.n_padded, bs.block_rows
        block = bs.blocks[self.rank][0]
        self.mod = as_modulus(block.mod)
        self.field = Field(self.mod, self.device)
        # short rows / limb slicing / die split change the layout: use the
        # row-major one-lane-per-row passes the epilogue push is written for
        self.dm = DeviceMatrix(block, self.device, field=self.field)
        if self.dm.info().get("lanes_per_residue", 1) != 1:
            raise ValueError("peer push needs a modulus of <= 8 limbs")
        lib = N.load()
        # two full iterate buffers (ping-pong) and one flag word, shared by IPC
        self.x = [DeviceVector(self.field, self.n_padded) for _ in range(2)]
        self.xptr = []
        for v in self.x:
            p, s = ctypes.c_uint64(), ctypes.c_int64()
            N.check(lib.sld_vec_device_ptr(v.handle, ctypes.byref(p), ctypes.byref(s)))
            self.xptr.append(p.value)
        f = ctypes.c_uint64()
        N.check(lib.sld_dev_alloc(self.device, 256, ctypes.byref(f)))
        self.flag = f.value
        handles = []
        for ptr in self.xptr + [self.flag]:
            h = np.zeros(64, dtype=np.uint8)
            N.check(lib.sld_ipc_get(self.device, ctypes.c_uint64(ptr), N.ptr(h)))
            handles.append(h.tobytes())
        peers = exchange((self.rank, handles))
        self.peer_x = [[0, 0] for _ in range(self.r)]
        self.peer_flag = [0] * self.r
        self._opened = []
        for rk, hs in peers:
            if rk == self.rank:
                self.peer_x[rk] = list(self.xptr)
                self.peer_flag[rk] = self.flag
                continue
            ptrs = []
            for h in hs:
                out = ctypes.c_uint64()
                buf = np.frombuffer(h, dtype=np.uint8).copy()
                N.check(lib.sld_ipc_open(self.device, N.ptr(buf), ctypes.byref(out)))
                ptrs.append(out.value)
                self._opened.append(out.value)
            self.peer_x[rk] = ptrs[:2]
            self.peer_flag[rk] = ptrs[2]
        self.exchange = exchange
        self.cur = 0
        self.iteration = 0

    def load_vector(self, limbs):
        """The full padded start vector (n_padded x L limbs), on every node."""
        self.x[self.cur].upload_limbs(np.ascontiguousarray(limbs, dtype=np.uint32))
        self.exchange(None)  # everyone loaded before anyone pushes

    def iterate(self, count=1):
        lib = N.load()
        flags = np.array(self.peer_flag, dtype=np.uint64)
        for _ in range(count):
            nxt = self.cur ^ 1
            dst = np.array([self.peer_x[k][nxt] for k in range(self.r)], dtype=np.uint64)
            N.check(lib.sld_mat_set_peers(self.dm.handle, self.r, N.ptr(dst), self.rank * self.br))
            N.check(lib.sld_spmv_peers(self.dm.handle, ctypes.c_uint64(self.xptr[self.cur])))
            self.iteration += 1
            N.check(lib.sld_peer_barrier(self.field.handle, self.r, N.ptr(flags), ctypes.c_uint64(self.flag),
                                         ctypes.c_uint32((self.r * self.iteration) & 0xFFFFFFFF)))
            self.cur = nxt

    def vector(self):
        """This node's copy of the full iterate (n_padded x L limbs)."""
        return self.x[self.cur].download_limbs()

    def close(self):
        lib = N.load()
        for p in self._opened:
            lib.sld_ipc_close(self.device, ctypes.c_uint64(p))
        self._opened = []
        if getattr(self, "flag", 0):
            lib.sld_dev_free(self.device, ctypes.c_uint64(self.flag))
            self.flag = 0


def _vec_ptr(v):
    p, s = ctypes.c_uint64(), ctypes.c_int64()
    N.check(N.load().sld_vec_device_ptr(v.handle, ctypes.byref(p), ctypes.byref(s)))
    return p.value, s.value


class PeerGrid:
    """One Krylov chain over an r x c grid (gridmv.py:251-348) with both
    exchanges done by the nodes themselves over peer memory, no collective:

      1. node (i, j): partial A_ij u_j, stored by its SpMV epilogue straight
         into slot j of the row collector (i, i mod c)'s inbox (peer stores);
      2. barrier; the collector sums its c inbox partials mod l (add_mod)
         and copies each column-range overlap of its row piece into the next
         fragment of every node of that column (peer P2P copies);
      3. barrier.
    Node (i, j) is rank i*c + j.  Every node ends with its fragment u_j; the
    outputs equal the reference Grid's (tests/test_peergrid_gpu.py)."""

    def __init__(self, A, g: GridSpec, rank: int, exchange, device=0, perm=None):
        if g.r * g.c > 8:
            raise ValueError("peer grid supports up to 8 nodes")
        self.g, self.rank, self.device = g, int(rank), int(device)
        self.i, self.j = divmod(self.rank, g.c)
        self.perm = perm if perm is not None else balance_permutation(A, g)
        bs = split(A, self.perm, g, only={(self.i, self.j)})
        self.n_padded, self.br, self.bc = bs.n_padded, bs.block_rows, bs.block_cols
        block = bs.blocks[self.i][self.j]
        self.mod = as_modulus(block.mod)
        self.field = Field(self.mod, self.device)
        self.dm = DeviceMatrix(block, self.device, field=self.field)
        if self.dm.info().get("lanes_per_residue", 1) != 1:
            raise ValueError("peer push needs a modulus of <= 8 limbs")
        self.SW = int(self.dm.info()["stride_words"])
        lib = N.load()
        self.frag = [DeviceVector(self.field, self.bc) for _ in range(2)]
        self.fptr = [_vec_ptr(v)[0] for v in self.frag]
        self.collector = self.j == self.i % g.c
        self.inbox = [DeviceVector(self.field, self.br) for _ in range(g.c)] if self.collector else []
        self.iptr = [_vec_ptr(v)[0] for v in self.inbox]
        self.piece = DeviceVector(self.field, self.br) if self.collector else None
        self.pptr = _vec_ptr(self.piece)[0] if self.collector else 0
        f = ctypes.c_uint64()
        N.check(lib.sld_dev_alloc(self.device, 256, ctypes.byref(f)))
        self.flag = f.value

        def handle(ptr):
            h = np.zeros(64, dtype=np.uint8)
            N.check(lib.sld_ipc_get(self.device, ctypes.c_uint64(ptr), N.ptr(h)))
            return h.tobytes()
        mine = {"frag": [handle(p) for p in self.fptr], "flag": handle(self.flag),
                "inbox": [handle(p) for p in self.iptr]}
        peers = exchange((self.rank, mine))
        self._opened = []

        def open_(h, rk, local):
            if rk == self.rank:
                return local
            out = ctypes.c_uint64()
            buf = np.frombuffer(h, dtype=np.uint8).copy()
            N.check(lib.sld_ipc_open(self.device, N.ptr(buf), ctypes.byref(out)))
            self._opened.append(out.value)
            return out.value
        self.nodes = g.r * g.c
        self.peer_frag = [None] * self.nodes
        self.peer_flag = [0] * self.nodes
        self.peer_inbox = [None] * self.nodes
        for rk, d in peers:
            own = rk == self.rank
            self.peer_frag[rk] = [open_(h, rk, self.fptr[k] if own else 0) for k, h in enumerate(d["frag"])]
            self.peer_flag[rk] = open_(d["flag"], rk, self.flag)
            self.peer_inbox[rk] = [open_(h, rk, self.iptr[k] if own else 0) for k, h in enumerate(d["inbox"])]
        self.exchange = exchange
        self.cur = 0
        self.phase = 0
        self.iteration = 0

    def _rank_of(self, i, j):
        return i * self.g.c + j

    def load_vector(self, limbs):
        """The full padded start vector (same on every rank); keeps u_j."""
        limbs = np.asarray(limbs, dtype=np.uint32)
        lo = self.j * self.bc
        self.frag[self.cur].upload_limbs(np.ascontiguousarray(limbs[lo:lo + self.bc]))
        self.exchange(None)

    def _barrier(self):
        self.phase += 1
        flags = np.array(self.peer_flag, dtype=np.uint64)
        N.check(N.load().sld_peer_barrier(self.field.handle, self.nodes, N.ptr(flags), ctypes.c_uint64(self.flag),
                                          ctypes.c_uint32((self.nodes * self.phase) & 0xFFFFFFFF)))

    def iterate(self, count=1):
        lib = N.load()
        g = self.g
        row_bytes = self.SW * 4
        for _ in range(count):
            nxt = self.cur ^ 1
            # 1. partial straight into the collector's inbox slot j
            coll = self._rank_of(self.i, self.i % g.c)
            dst = np.array([self.peer_inbox[coll][self.j]], dtype=np.uint64)
            N.check(lib.sld_mat_set_peers(self.dm.handle, 1, N.ptr(dst), 0))
            N.check(lib.sld_spmv_peers(self.dm.handle, ctypes.c_uint64(self.fptr[self.cur])))
            self._barrier()
            # 2. the collector reduces and scatters its row piece
            if self.collector:
                srcs = np.array(self.iptr, dtype=np.uint64)
                N.check(lib.sld_add_mod(self.field.handle, N.ptr(srcs), len(self.iptr),
                                        ctypes.c_uint64(self.pptr), self.br))
                rlo = self.i * self.br
                for jj in range(g.c):
                    clo = jj * self.bc
                    lo, hi = max(rlo, clo), min(rlo + self.br, clo + self.bc)
                    if lo >= hi:
                        continue
                    for k in range(g.r):
                        dst_ptr = self.peer_frag[self._rank_of(k, jj)][nxt] + (lo - clo) * row_bytes
                        N.check(lib.sld_memcpy_async(self.field.handle, ctypes.c_uint64(dst_ptr),
                                                     ctypes.c_uint64(self.pptr + (lo - rlo) * row_bytes),
                                                     (hi - lo) * row_bytes))
            self._barrier()
            self.cur = nxt
            self.iteration += 1

    def fragment(self):
        """u_j of this node (bc x L limbs)."""
        return self.frag[self.cur].download_limbs()

    def close(self):
        lib = N.load()
        for p in self._opened:
            lib.sld_ipc_close(self.device, ctypes.c_uint64(p))
        self._opened = []
        if getattr(self, "flag", 0):
            lib.sld_dev_free(self.device, ctypes.c_uint64(self.flag))
            self.flag = 0

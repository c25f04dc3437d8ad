"""Host-side logic of the peer-memory grid (peergrid.LocalGrid /
GridMultiplier) on CPU: fragment slicing, launch interleaving, term-ring
draining across TERM_RING, merging of the rows each node reports, and the
iterate assembly -- with the native node replaced by an oracle-backed fake
that holds the whole padded iterate (the native node is tested on the GPU in
tests/test_localgrid_gpu.py)."""
import numpy as np
import pytest

import oracle as O
from helpers import rand_matrix, to_oracle
from paper_1402_3661_b200 import PrimeModulus, UnitRows, krylov_column
from paper_1402_3661_b200.balance import GridSpec, balance_permutation, permuted_padded
from paper_1402_3661_b200.modring import ints_to_planes, planes_to_ints
from paper_1402_3661_b200 import peergrid
from paper_1402_3661_b200.peergrid import GridMultiplier, LocalGrid


class _Shared:
    """The 'device memory' every fake node sees: the padded iterate."""

    def __init__(self, orc, n):
        self.orc, self.n, self.v, self.launches = orc, n, None, []


class _FakeNode:
    def __init__(self, shared, g, rank, L):
        self.sh, self.g, self.rank, self.L = shared, g, rank, L
        self.i, self.j = divmod(rank, g.c)
        self.bc = shared.n // g.c
        self.m, self.owned, self.rows, self.ring = 0, np.zeros(0, np.uint8), [], []

    def load(self, frag):
        if self.sh.v is None:
            self.sh.v = np.zeros((self.sh.n, self.L), dtype=np.uint32)
        self.sh.v[self.j * self.bc:(self.j + 1) * self.bc] = frag

    def set_projection(self, rows, max_steps=peergrid.TERM_RING):
        self.rows, self.m = list(rows), len(rows)
        self.owned = np.array([self.i == 0 and r // self.bc == self.j for r in rows], dtype=np.uint8)
        self.cap, self.ring = max_steps, []
        return self.owned.astype(bool)

    def launch(self, count=1):
        for _ in range(count):
            self.sh.launches.append(self.rank)
            if self.m:
                if len(self.ring) >= self.cap:
                    raise ValueError("term ring full")
                self.ring.append(np.array([self.sh.v[r] if o else np.zeros(self.L, np.uint32)
                                           for r, o in zip(self.rows, self.owned)]))
            if self.rank == self.g.r * self.g.c - 1:  # the last node to launch completes the iteration
                self.sh.v = self.sh.orc.spmv_limbs(self.sh.v)

    def wait(self):
        pass

    def terms(self):
        out = np.array(self.ring, dtype=np.uint32).reshape(len(self.ring), self.m, self.L)
        self.ring = []
        return out

    def fragment(self):
        return self.sh.v[self.j * self.bc:(self.j + 1) * self.bc].copy()


def _fake_grid(A, g):
    perm = balance_permutation(A, g)
    B = permuted_padded(A, perm, g)
    grid = LocalGrid.__new__(LocalGrid)
    grid.g, grid.perm = g, perm
    sh = _Shared(to_oracle(B), B.nrows)
    grid.nodes = [_FakeNode(sh, g, k, A.mod.limbs) for k in range(g.r * g.c)]
    grid.n_padded, grid.bc, grid.br, grid.mod = B.nrows, B.nrows // g.c, B.nrows // g.r, A.mod
    grid.spmv_count = 0
    return grid, B, sh


@pytest.mark.parametrize("r,c", [(1, 1), (2, 1), (2, 2), (3, 2)])
def test_grid_multiplier_host_logic(r, c, monkeypatch):
    monkeypatch.setattr(peergrid, "TERM_RING", 16)  # several drains in a short chain
    rng = np.random.default_rng(r * 10 + c)
    mod = PrimeModulus(2**61 - 1)
    A = rand_matrix(mod, rng, 60, 60, 6)
    g = GridSpec(r, c)
    grid, B, sh = _fake_grid(A, g)
    mul = GridMultiplier(grid)
    P = (mod.ell.bit_length() + 15) // 16
    y = mod.random_residues(rng, B.nrows)
    rows = sorted(int(x) for x in rng.choice(B.nrows, 4, replace=False))
    terms, v, spmvs = krylov_column(mul, UnitRows(rows), ints_to_planes(y, P), 41)
    orc = to_oracle(B)
    t_o, v_o = O.krylov_unit(orc, O.ints_to_limbs(y, mod.limbs), rows, 41)
    assert spmvs == 41 and mul.count == 41
    assert terms == [O.limbs_to_ints(t) for t in t_o]
    assert planes_to_ints(v) == O.limbs_to_ints(v_o)
    # launches interleave node by node, iteration by iteration
    nodes = r * c
    assert sh.launches[:2 * nodes] == list(range(nodes)) * 2


def test_fragment_shape_is_checked():
    mod = PrimeModulus(1009)
    A = rand_matrix(mod, np.random.default_rng(1), 30, 30, 4)
    grid, B, _ = _fake_grid(A, GridSpec(2, 2))
    with pytest.raises(ValueError):
        grid.load_vector(np.zeros((B.nrows + 1, 1), dtype=np.uint32))

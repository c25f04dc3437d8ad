"""The native peer-memory grid (csrc/sld_grid.cu, peergrid.LocalGrid /
GridMultiplier) with every node in this process, all folded onto one GPU
(the same code as one node per GPU: the nodes only see each other's
pointers).  Checks:
  * every golden grid case (reference Grid outputs, gridmv.py:251-354);
  * krylov_column through GridMultiplier (the reference's multiplier
    protocol, solver.py:145-162) against the oracle's chain on the padded
    permuted matrix B, at 1x1, 2x1, 4x1, 8x1, 2x2, 2x4 and 3x2, across the
    device term ring's drain boundary;
  * failure detection, mirroring the reference's tests/test_gridmv.py:173-199:
    a node that never arrives -> GridTimeoutError, a restarted (stale) node
    -> GridProtocolError, on every node that sees it."""
import numpy as np
import pytest

import oracle as O
from helpers import fixture_sparse, rand_matrix, to_oracle
from paper_1402_3661_b200 import PrimeModulus, UnitRows, krylov_column
from paper_1402_3661_b200._native import GridProtocolError, GridTimeoutError
from paper_1402_3661_b200.balance import GridSpec, balance_permutation, permuted_padded
from paper_1402_3661_b200.modring import ints_to_planes, planes_to_ints
from paper_1402_3661_b200.peergrid import TERM_RING, GridMultiplier, LocalGrid

pytestmark = pytest.mark.gpu


def _golden_cases():
    z = O.load_golden("grid_cases.npz")
    return list(range(int(z["ncases"])))


@pytest.mark.parametrize("case", _golden_cases())
def test_local_grid_matches_reference_golden(case):
    z = O.load_golden("grid_cases.npz")
    p = f"g{case}_"
    A = fixture_sparse(z, p)
    r, c, iters = (int(x) for x in z[p + "grid"])
    g = GridSpec(r, c)
    grid = LocalGrid(A, g, devices=[0] * (r * c), perm=balance_permutation(A, g))
    try:
        L = A.mod.limbs
        grid.load_vector(O.bytes_to_limbs(z[p + "u"], L))
        grid.iterate(iters)
        assert np.array_equal(grid.assembled(), O.bytes_to_limbs(z[p + "out"], L))
        for nd in grid.nodes:  # every node's fragment, not only row 0's
            want = O.bytes_to_limbs(z[p + "out"], L)[nd.j * nd.bc:(nd.j + 1) * nd.bc]
            assert np.array_equal(nd.fragment(), want), f"node {nd.rank}"
            assert nd.info()["iteration"] == iters
    finally:
        grid.close()


@pytest.mark.parametrize("r,c,bits", [(1, 1, 127), (2, 1, 200), (4, 1, 64), (8, 1, 202), (2, 2, 202),
                                      (2, 4, 160), (3, 2, 250)])
def test_grid_multiplier_krylov_vs_oracle(r, c, bits):
    rng = np.random.default_rng(100 * r + c)
    from paper_1402_3661_b200.corpus import random_prime
    mod = random_prime(bits, rng)
    n = 900 + 37 * r * c
    A = rand_matrix(mod, rng, n, n, 12)
    g = GridSpec(r, c)
    perm = balance_permutation(A, g)
    B = permuted_padded(A, perm, g)
    grid = LocalGrid(A, g, devices=[0] * (r * c), perm=perm)
    try:
        mul = GridMultiplier(grid)
        assert mul.size == B.nrows and mul.mod.ell == mod.ell
        P = (mod.ell.bit_length() + 15) // 16
        y = mod.random_residues(rng, B.nrows)
        rows = sorted(int(x) for x in rng.choice(B.nrows, 3, replace=False))
        steps = TERM_RING + 37 if (r, c) in ((2, 1), (2, 2)) else 60
        terms, v, spmvs = krylov_column(mul, UnitRows(rows), ints_to_planes(y, P), steps)
        assert spmvs == steps and mul.count == steps
        orc = to_oracle(B)
        t_o, v_o = O.krylov_unit(orc, O.ints_to_limbs(y, mod.limbs), rows, steps)
        assert terms == [O.limbs_to_ints(t) for t in t_o]
        assert planes_to_ints(v) == O.limbs_to_ints(v_o)
        # the plain protocol: one grid iteration per apply
        v1 = planes_to_ints(mul.apply(ints_to_planes(y, P)))
        assert v1 == O.limbs_to_ints(orc.spmv_limbs(O.ints_to_limbs(y, mod.limbs)))
    finally:
        grid.close()


def _small_grid(r, c, seed=3):
    rng = np.random.default_rng(seed)
    mod = PrimeModulus((1 << 127) - 1)
    A = rand_matrix(mod, rng, 400, 400, 8)
    g = GridSpec(r, c)
    grid = LocalGrid(A, g, devices=[0] * (r * c), perm=balance_permutation(A, g))
    y = O.ints_to_limbs(mod.random_residues(rng, grid.n_padded), mod.limbs)
    grid.load_vector(y)
    return grid


@pytest.mark.parametrize("r,c", [(2, 1), (2, 2)])
def test_stopped_node_times_out(r, c):
    # node 0 runs an iteration, its peers never do: the barrier reports the
    # dead peer (GridTimeoutError) instead of hanging
    grid = _small_grid(r, c)
    try:
        grid.iterate(2)  # healthy first
        grid.set_timeout(0.3)
        nd = grid.nodes[0]
        nd.launch(1)
        with pytest.raises(GridTimeoutError, match="timed out"):
            nd.wait()
    finally:
        grid.close()


@pytest.mark.parametrize("r,c", [(2, 1), (2, 2)])
def test_restarted_node_is_a_protocol_error(r, c):
    # a node that restarts at iteration 0 while its peers are at 3 publishes
    # a stale iteration: every node raises GridProtocolError
    grid = _small_grid(r, c)
    try:
        grid.iterate(3)
        grid.nodes[1].set_epoch(0)
        grid.set_timeout(2.0)
        for nd in grid.nodes:
            nd.launch(1)
        errs = []
        for nd in grid.nodes:
            try:
                nd.wait()
                errs.append(None)
            except (GridProtocolError, GridTimeoutError) as e:
                errs.append(e)
        assert isinstance(errs[0], GridProtocolError), errs
        assert isinstance(errs[1], GridProtocolError), errs
        assert "stale" in str(errs[0])
    finally:
        grid.close()


def test_resume_at_common_epoch():
    # all nodes restarted together at the same iteration is a valid resume
    grid = _small_grid(2, 1)
    try:
        grid.iterate(3)
        v3 = grid.assembled()
        for nd in grid.nodes:
            nd.set_epoch(3)
        grid.load_vector(v3)
        grid.iterate(2)
        grid2 = _small_grid(2, 1)
        grid2.iterate(5)
        assert np.array_equal(grid.assembled(), grid2.assembled())
        grid2.close()
    finally:
        grid.close()


def test_grid_info_and_arguments():
    grid = _small_grid(2, 2)
    try:
        info = [nd.info() for nd in grid.nodes]
        assert [i["collector"] for i in info] == [1, 0, 0, 1]  # (i, i mod c)
        assert all(i["nodes"] == 4 and i["iteration"] == 0 for i in info)
        with pytest.raises(ValueError):
            grid.nodes[0].load(np.zeros((3, 4), dtype=np.uint32))
        with pytest.raises(ValueError):
            grid.nodes[0].set_timeout(0)
        with pytest.raises(ValueError):  # term ring bound
            grid.nodes[0].set_projection([0], max_steps=2)
            grid.nodes[0].launch(3)
    finally:
        grid.close()

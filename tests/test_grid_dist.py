"""The distributed grid (one process per node) reproduces the reference's
grid engine: outputs equal the reference Grid's (golden), the balance
permutations equal the reference's, and the communication log equals the
reference CommLog / comm_volume_model.  CPU: gloo with the oracle engine;
GPU: the same exchange over the device engine (all ranks on cuda:0)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from helpers import fixture_sparse

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, engine_kind, out_q):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1402_3661_b200.balance import GridSpec, balance_permutation
        from paper_1402_3661_b200.grid import B200Grid, GridComm
        z = O.load_golden("grid_cases.npz")
        p = f"g{case}_"
        A = fixture_sparse(z, p)
        r, c, iters = (int(x) for x in z[p + "grid"])
        g = GridSpec(r, c)
        perm = balance_permutation(A, g)
        if engine_kind == "cpu":
            from grid_cpu_engine import OracleEngine
            grid = B200Grid(A, g, GridComm(g), engine_factory=OracleEngine, perm=perm)
        else:
            grid = B200Grid(A, g, GridComm(g), device=0, perm=perm)
        L = A.mod.limbs
        grid.load_vector(O.bytes_to_limbs(z[p + "u"], L))
        grid.iterate(iters)
        out = grid.assembled()
        ok_out = np.array_equal(out, O.bytes_to_limbs(z[p + "out"], L))
        ok_perm = (np.array_equal(perm.row_perm, z[p + "row_perm"])
                   and np.array_equal(perm.col_perm, z[p + "col_perm"]))
        bytes_log = [e.total_bytes for e in grid.comm_log.entries]
        ok_log = bytes_log == [int(x) for x in z[p + "comm_bytes"]]
        # a device-resident Krylov chain over the grid vs the oracle on the
        # assembled matrix B = P_r A P_c^T (balance.py:245-267)
        from paper_1402_3661_b200.balance import permuted_padded
        from paper_1402_3661_b200.grid import GridMultiplier
        from paper_1402_3661_b200.modring import digit_count, limbs_to_planes
        from helpers import to_oracle
        B = permuted_padded(A, perm, g)
        rows = sorted({0, B.nrows // 2, B.nrows - 1})
        y = O.bytes_to_limbs(z[p + "u"], L)
        ot, ov = O.krylov_unit(to_oracle(B), y, rows, 7)
        mul = GridMultiplier(grid)
        terms, v = mul.krylov(type("X", (), {"rows": rows})(), limbs_to_planes(y, digit_count(A.mod.ell)), 7)
        ok_kry = terms == [O.limbs_to_ints(t) for t in ot] and \
            np.array_equal(v, limbs_to_planes(ov, digit_count(A.mod.ell)))
        out_q.put((rank, ok_out, ok_perm, ok_log and ok_kry, grid.spmv_count == iters + 7))
    finally:
        dist.destroy_process_group()


def _run(case, engine_kind):
    z = O.load_golden("grid_cases.npz")
    r, c, _ = (int(x) for x in z[f"g{case}_grid"])
    world = r * c
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, case, engine_kind, q)) for k in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, ok_out, ok_perm, ok_log, ok_count in res:
        assert ok_out, f"rank {rank}: grid output differs from the reference Grid"
        assert ok_perm and ok_log and ok_count, rank


# grids from the reference's tests (tests/test_gridmv.py:78-93): 1x1, 2x1,
# 4x1, 2x2, 2x4, 4x2, 3x2, 8x1, and 2x2 over 10 iterations at 200 bits
CPU_CASES = [0, 1, 2, 3, 4, 5, 6, 8]


@pytest.mark.parametrize("case", CPU_CASES)
def test_grid_gloo_cpu_matches_reference(case):
    _run(case, "cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("case", [1, 3, 4, 6, 7, 8])
def test_grid_device_engine_matches_reference(case):
    _run(case, "gpu")

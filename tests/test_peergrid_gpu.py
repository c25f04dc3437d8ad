"""r x 1 grid with the all-gather fused into the SpMV epilogue (peer
stores + flag barrier, paper_1402_3661_b200/peergrid.py): r processes share
one GPU through CUDA IPC handles -- the same code path as r GPUs over
NVLink -- and every node's iterate equals the reference Grid's output on the
golden r x 1 cases."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from helpers import fixture_sparse

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1402_3661_b200.balance import GridSpec, balance_permutation
        from paper_1402_3661_b200.peergrid import PeerRowGrid
        z = O.load_golden("grid_cases.npz")
        p = f"g{case}_"
        A = fixture_sparse(z, p)
        r, c, iters = (int(x) for x in z[p + "grid"])

        def exchange(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
        grid = PeerRowGrid(A, r, rank, exchange, device=0, perm=balance_permutation(A, GridSpec(r, 1)))
        L = A.mod.limbs
        grid.load_vector(O.bytes_to_limbs(z[p + "u"], L))
        grid.iterate(iters)
        got = grid.vector()
        ok = bool(np.array_equal(got, O.bytes_to_limbs(z[p + "out"], L)))
        exchange(None)
        grid.close()
        out_q.put((rank, ok, None))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        out_q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _worker2d(rank, world, port, case, out_q):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1402_3661_b200.balance import GridSpec, balance_permutation
        from paper_1402_3661_b200.peergrid import PeerGrid
        z = O.load_golden("grid_cases.npz")
        p = f"g{case}_"
        A = fixture_sparse(z, p)
        r, c, iters = (int(x) for x in z[p + "grid"])
        g = GridSpec(r, c)

        def exchange(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
        grid = PeerGrid(A, g, rank, exchange, device=0, perm=balance_permutation(A, g))
        L = A.mod.limbs
        grid.load_vector(O.bytes_to_limbs(z[p + "u"], L))
        grid.iterate(iters)
        want = O.bytes_to_limbs(z[p + "out"], L)
        lo = grid.j * grid.bc
        ok = bool(np.array_equal(grid.fragment(), want[lo:lo + grid.bc]))
        exchange(None)
        grid.close()
        out_q.put((rank, ok, None))
    except Exception:
        import traceback
        out_q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _cases_2d():
    z = O.load_golden("grid_cases.npz")
    return [i for i in range(int(z["ncases"])) if int(z[f"g{i}_grid"][1]) > 1]


@pytest.mark.parametrize("case", _cases_2d())
def test_peer_grid_2d_matches_reference(case):
    # r x c: partials pushed into the row collector's inbox by the SpMV
    # epilogue, reduced mod l, scattered to the column nodes by P2P copies
    z = O.load_golden("grid_cases.npz")
    r, c = (int(x) for x in z[f"g{case}_grid"][:2])
    world = r * c
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker2d, args=(k, world, port, case, q)) for k in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [f"rank {rank}: {err}" for rank, ok, err in sorted(res) if err]
    assert not errs, "\n".join(errs)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank} fragment differs from the reference grid"


def _rx1_cases():
    z = O.load_golden("grid_cases.npz")
    out = []
    for i in range(int(z["ncases"])):
        r, c, _ = (int(x) for x in z[f"g{i}_grid"])
        if c == 1 and r > 1:
            out.append(i)
    return out


@pytest.mark.parametrize("case", _rx1_cases())
def test_peer_push_grid_matches_reference(case):
    z = O.load_golden("grid_cases.npz")
    r = int(z[f"g{case}_grid"][0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, r, port, case, q)) for k in range(r)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(r)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok, err in sorted(res):
        assert err is None, err
        assert ok, f"rank {rank} iterate differs from the reference grid"

"""Failure detection of the distributed node protocol (grid.B200Grid over
torch.distributed; gloo + the CPU oracle engine here), mirroring the
reference's tests/test_gridmv.py:173-199:
  * a partial sum that never leaves node (0, 1) -> the collector raises
    GridTimeoutError within GridComm's timeout (the reference's
    DroppingTransport case);
  * a partial sum tagged with a stale iteration -> the collector raises
    GridProtocolError (the reference's injected-stale-message case).
The native peer-memory grid's barrier timeouts and stale-iteration checks are
tested on the GPU in tests/test_localgrid_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fault, out_q, done):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = "ok"
    try:
        from grid_cpu_engine import OracleEngine
        from helpers import rand_matrix
        import oracle as O
        from paper_1402_3661_b200 import PrimeModulus
        from paper_1402_3661_b200.balance import GridSpec, balance_permutation
        from paper_1402_3661_b200.grid import (KIND_PARTIAL_SUM, B200Grid, GridComm, GridProtocolError,
                                               GridTimeoutError)

        class FaultyComm(GridComm):
            def header(self, iteration, kind, like):
                if fault == "stale" and self.rank == 1 and kind == KIND_PARTIAL_SUM:
                    iteration = 99
                return super().header(iteration, kind, like)

            def exchange(self, sends, recvs, iteration=None, kind=None):
                if fault == "drop" and self.rank == 1 and kind == KIND_PARTIAL_SUM:
                    sends = []
                return super().exchange(sends, recvs, iteration, kind)

        rng = np.random.default_rng(19)
        mod = PrimeModulus(1009)
        A = rand_matrix(mod, rng, 50, 50, 5)
        g = GridSpec(2, 2)
        grid = B200Grid(A, g, FaultyComm(g, timeout=3.0), engine_factory=OracleEngine,
                        perm=balance_permutation(A, g))
        u = O.ints_to_limbs([int(x) for x in rng.integers(0, 1009, size=grid.n_padded)], mod.limbs)
        grid.load_vector(u)
        try:
            grid.iterate(1)
        except GridProtocolError as e:
            res = "protocol: " + str(e)
        except GridTimeoutError as e:
            res = "timeout: " + str(e)
    except Exception as e:  # report, never hang the parent
        import traceback
        res = "error: " + traceback.format_exc()[-1200:]
    out_q.put((rank, res))
    out_q.close()
    out_q.join_thread()  # flush before the hard exit below
    # stay connected until every rank has reported: an early exit would turn
    # the peers' timeouts into "connection closed" errors
    done.wait(timeout=60)
    os._exit(0)  # peers may still be blocked in the broken exchange


@pytest.mark.parametrize("fault,want", [("drop", "timeout"), ("stale", "protocol")])
def test_node_protocol_faults(fault, want):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    done = ctx.Event()
    procs = [ctx.Process(target=_worker, args=(k, 4, port, fault, q, done)) for k in range(4)]
    for pr in procs:
        pr.start()
    try:
        res = dict(q.get(timeout=120) for _ in range(4))
    finally:
        done.set()
        for pr in procs:
            pr.join(timeout=30)
    assert not any(v.startswith("error") for v in res.values()), res
    # node (0, 0) is row 0's collector: it detects the fault itself
    assert res[0].startswith(want), res
    # node (1, 0) waits for column 0's fragment from that collector, which
    # never sends it: a timeout, not a hang.  Nodes (0, 1) and (1, 1) get
    # their fragments from row 1's collector and complete.
    assert res[2].startswith("timeout"), res
    assert res[1] == "ok" and res[3] == "ok", res

"""bench.py's repo arm under torchrun on the GPU (§8(e) e1, independent
chains): 2 ranks folded onto one device (SLD_BENCH_NDEV=1; gloo for the
barrier and the max-over-ranks reduction, since NCCL refuses two ranks on
one GPU).  Rank 0 alone prints one line, the value counts both ranks'
chains, and each rank's planted-witness product checks out."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("config", ["cfg1", "cfg2"])
def test_repo_arm_two_ranks_folded(config):
    env = dict(os.environ, SLD_BENCH_NDEV="1", SLD_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--config", config, "--steps", "40", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["steps"] == 40
    assert d["value"] > 0 and abs(d["value"] - 2 * 40 / (d["ms_per_step"] * 40 / 1e3)) < 1e-6 * d["value"]
    assert d["gpu_launches"] >= 40 and d["witness_check"] is True
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    # one sample per product pair; per 16 pairs when a product is < 0.1 ms
    # (the probe that decides it is timed, so a rank sharing the GPU can
    # tip it: the count must match the sample size the line states)
    per = int(d["samples"]["per"].split()[0])
    assert per in (2, 32) and d["samples"]["count"] == -(-40 // per) and d["ms_per_step_median"] > 0
    if config == "cfg2":
        assert per == 2

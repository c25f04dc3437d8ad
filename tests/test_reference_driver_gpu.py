"""The reference's OWN driver code on the B200.

oracle/_ref/sldlag_ref.zip (built by oracle/ref_bundle.py from
/root/reference, git-ignored, shipped to the GPU box with the snapshot) holds
the reference package and its tests.  These tests unpack it and run, in a
subprocess, the reference's tests/test_solver.py and acceptance criteria 4
and 10 with `sldlag.solver.SequentialMultiplier` swapped for B200Multiplier
(tests/refswap/sld_refswap.py): krylov_block (threads included), the
reference's krylov_column loop, block_lingen on the sequence, the
reference's _mksol_core on DevicePlanes iterates (planes_add_mod etc.),
block_wiedemann with make_mul, and its checkpoint halt/resume.  They also
drive the reference's block_wiedemann directly with
make_mul=lambda j: B200Multiplier(A) and check the kernel vector."""
import json
import os
import subprocess
import sys
import time
import zipfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ZIP = os.path.join(ROOT, "oracle", "_ref", "sldlag_ref.zip")
SHIM = os.path.join(ROOT, "oracle", "gmpy2_shim")


@pytest.fixture(scope="module")
def ref_tree(tmp_path_factory):
    if not os.path.exists(ZIP):
        # the archive is built where /root/reference exists and travels with
        # the snapshot; a checkout without it cannot run the reference
        pytest.skip("oracle/_ref/sldlag_ref.zip missing: run oracle.build() where /root/reference exists")
    d = tmp_path_factory.mktemp("sldlag_ref")
    with zipfile.ZipFile(ZIP) as z:
        z.extractall(d)
    return d


def _env(ref_tree, log):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refswap"), SHIM,
                                         str(ref_tree / "src"), str(ref_tree / "tests"), ROOT])
    env["SLD_REFSWAP_LOG"] = str(log)
    return env


def _run_reference_tests(ref_tree, tmp_path, args):
    log = tmp_path / "swap.json"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "sld_refswap",
           "--rootdir", str(ref_tree), *args]
    t = time.time()
    r = subprocess.run(cmd, cwd=str(ref_tree), env=_env(ref_tree, log), capture_output=True,
                       text=True, timeout=1200)
    print(r.stdout[-3000:], r.stderr[-2000:], f"[{time.time() - t:.1f}s]")
    assert r.returncode == 0, r.stdout[-3000:]
    stats = json.loads(log.read_text())
    return r.stdout, stats


def test_reference_solver_tests_on_b200(ref_tree, tmp_path):
    out, stats = _run_reference_tests(ref_tree, tmp_path, ["tests/test_solver.py"])
    assert " passed" in out and "failed" not in out
    # every Krylov / Mksol product of the reference's own tests ran on the GPU
    assert stats["multipliers"] >= 20 and stats["applies"] > 5000, stats


def test_reference_acceptance_krylov_criteria_on_b200(ref_tree, tmp_path):
    out, stats = _run_reference_tests(
        ref_tree, tmp_path, ["tests/test_acceptance.py", "-k", "criterion_04 or criterion_10"])
    assert "2 passed" in out
    assert stats["multipliers"] > 0 and stats["applies"] > 0, stats


def test_reference_block_wiedemann_make_mul(ref_tree, tmp_path):
    """block_wiedemann(A, bp, seed, make_mul=lambda j: B200Multiplier(A)) on
    the reference's own matrix objects, with _mksol_core timed on the
    DevicePlanes round trips."""
    script = r'''
import json, sys, time
import numpy as np
from sldlag.corpus import CorpusProfile, generate
from sldlag.modring import PrimeModulus
from sldlag.solver import BlockingParams, block_wiedemann, krylov_length, verify_kernel
from sldlag.cli import random_prime
import sldlag.solver as S
from paper_1402_3661_b200 import B200Multiplier
res = {}
for bits, n, bp in ((202, 600, BlockingParams(2, 4)), (650, 300, BlockingParams(4, 8))):
    mod = random_prime(bits, np.random.default_rng(1))
    mod = mod if isinstance(mod, PrimeModulus) else PrimeModulus(mod)
    A = generate(CorpusProfile(n=n, gamma=20, seed=5), mod)
    muls = []
    def make_mul(j, A=A):
        m = B200Multiplier(A)
        muls.append(m)
        return m
    t = time.time()
    core = S._mksol_core
    tm = {}
    def timed(*a, **k):
        t0 = time.time(); r = core(*a, **k); tm["mksol_s"] = time.time() - t0; return r
    S._mksol_core = timed
    kv, stats = block_wiedemann(A, bp, seed=7, make_mul=make_mul)
    S._mksol_core = core
    assert kv.verified and verify_kernel(A, kv.w)
    assert stats["krylov_spmvs_per_column"] == [krylov_length(n, bp)] * bp.n
    res[f"{bits}b"] = dict(n=n, bp=[bp.n, bp.m], seconds=time.time() - t, applies=sum(m.count for m in muls),
                           horner=stats["horner_spmvs"], mksol_s=tm.get("mksol_s"),
                           mksol_ms_per_step=1e3 * tm.get("mksol_s", 0) / max(1, stats["horner_spmvs"] + stats["tail_spmvs"]))
print(json.dumps(res))
'''
    log = tmp_path / "swap.json"
    r = subprocess.run([sys.executable, "-c", script], cwd=str(ref_tree), env=_env(ref_tree, log),
                       capture_output=True, text=True, timeout=1200)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for k, v in res.items():
        assert v["applies"] > 2 * v["n"], (k, v)


def test_reference_whole_suite_on_b200(ref_tree, tmp_path):
    """Every test module of the reference (balance, cli, corpus, gridmv,
    modring, perfmodel, sge, solver, spmatrix, vecops, acceptance) with the
    swap.  Deselected: criterion 1 (the full pipeline, ~6 min; it passes,
    profiles/refswap_full_r02.txt) and criterion 6, which fails at seed 31
    with the reference's OWN multiplier too -- same messages at the same
    attempts on the B200 (tools/diag_sge2.py)."""
    out, stats = _run_reference_tests(
        ref_tree, tmp_path,
        ["tests", "-k", "not criterion_01 and not criterion_06"])
    assert " passed" in out and "failed" not in out and "error" not in out.lower().split("passed")[-1]
    assert stats["multipliers"] >= 50 and stats["applies"] > 10000, stats

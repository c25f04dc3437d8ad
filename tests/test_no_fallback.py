"""The product path fails loudly without its CUDA library or a device: no
silent CPU (or oracle) fallback.  CPU only; each case runs in a fresh
interpreter so the library handle is not already cached."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np
from paper_1402_3661_b200 import B200Multiplier, PrimeModulus, SparseMatrix
from paper_1402_3661_b200.modring import ints_to_planes, digit_count
mod = PrimeModulus(2**61 - 1)
A = SparseMatrix.from_rows(mod, 3, 3, [[(0, 1)], [(1, 2)], [(2, mod.ell - 1)]])
mul = B200Multiplier(A)
assert mul.size == 3 and mul.mod.ell == mod.ell  # protocol fields need no device
try:
    out = mul.apply(ints_to_planes([1, 2, 3], digit_count(mod.ell)))
    np.asarray(out)
except Exception as e:
    print("RAISED", type(e).__name__, str(e)[:120])
else:
    print("COMPUTED")
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=300)
    return r.stdout + r.stderr


def test_missing_library_raises():
    out = _run({"SLD_LIB": "/nonexistent/libsldb200.so"})
    assert "RAISED NativeUnavailable" in out, out


def test_no_device_raises():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is visible: the product path runs (covered by -m gpu)")
    out = _run({"CUDA_VISIBLE_DEVICES": ""})
    assert "RAISED" in out and "COMPUTED" not in out, out

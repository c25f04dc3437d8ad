"""pytest plugin (test infrastructure): loaded with `-p sld_refswap` into a
run of the REFERENCE's own test modules, it replaces the reference's default
multiplier `sldlag.solver.SequentialMultiplier` (solver.py:129-142) with this
package's B200Multiplier -- the one-line swap INTEGRATION.md promises -- so
the reference's krylov_block / krylov_scalar / mksol_* / block_wiedemann
(and every test calling them) drive the B200.  Each multiplier built and
each product it runs is counted into $SLD_REFSWAP_LOG so the calling test can
prove the GPU path ran."""
import atexit
import json
import os
import threading

import sldlag.solver as ref_solver

from paper_1402_3661_b200 import B200Multiplier

_stats = {"multipliers": 0, "applies": 0, "devices": []}
_lock = threading.Lock()


class SwappedMultiplier(B200Multiplier):
    def __init__(self, A, *a, **kw):
        super().__init__(A, device=int(os.environ.get("SLD_DEVICE", "0")))
        with _lock:
            _stats["multipliers"] += 1

    def apply(self, planes):
        out = super().apply(planes)
        with _lock:
            _stats["applies"] += 1
        return out


ref_solver.SequentialMultiplier = SwappedMultiplier


@atexit.register
def _dump():
    path = os.environ.get("SLD_REFSWAP_LOG")
    if path:
        with open(path, "w") as f:
            json.dump(_stats, f)

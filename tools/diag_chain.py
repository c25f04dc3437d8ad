"""Diagnostic: a device Krylov chain (krylov_column) against the oracle on a
corpus matrix; reports the wrong (step, row) terms and iterate rows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from helpers import to_oracle  # noqa: E402
from paper_1402_3661_b200 import B200Multiplier, UnitRows, corpus, krylov_column  # noqa: E402
from paper_1402_3661_b200.modring import digit_count, ints_to_planes, planes_to_ints  # noqa: E402

n, bits, steps, reps = (int(a) for a in sys.argv[1:5])
mod = corpus.random_prime(bits, np.random.default_rng(bits))
rng = np.random.default_rng(n)
A = corpus.generate(corpus.CorpusProfile(n=n, gamma=20, dense_cols=1, seed=3), mod)
y = mod.random_residues(rng, n)
rows = [0, n // 2, n - 1]
ot, ov = O.krylov_unit(to_oracle(A), O.ints_to_limbs(y, mod.limbs), rows, steps)
want = [O.limbs_to_ints(t) for t in ot]
wv = O.limbs_to_ints(ov)
for r in range(reps):
    mul = B200Multiplier(A)
    terms, v, _ = krylov_column(mul, UnitRows(rows), ints_to_planes(y, digit_count(mod.ell)), steps)
    bad = [(k, j) for k in range(steps) for j in range(3) if terms[k][j] != want[k][j]]
    gv = planes_to_ints(v)
    badv = [i for i in range(n) if gv[i] != wv[i]]
    print(f"rep {r}: {len(bad)} wrong terms {bad[:8]}, {len(badv)} wrong iterate rows {badv[:8]}", flush=True)

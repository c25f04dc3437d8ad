"""Stress: many device Krylov chains (persistent chain and per-product graphs
alternating, one process) against the oracle; prints every mismatch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from helpers import rand_matrix, to_oracle  # noqa: E402
from paper_1402_3661_b200 import B200Multiplier, UnitRows, corpus, krylov_column  # noqa: E402
from paper_1402_3661_b200.modring import digit_count, ints_to_planes, planes_to_ints  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.time()
fails = 0
for it in range(iters):
    rng = np.random.default_rng(1000 + it)
    bits = int(rng.choice([31, 64, 160, 202, 256]))
    n = int(rng.integers(3000, 70000))
    steps = int(rng.integers(5, 70))
    mod = corpus.random_prime(bits, np.random.default_rng(bits))
    A = corpus.generate(corpus.CorpusProfile(n=n, gamma=int(rng.integers(10, 40)), dense_cols=int(rng.integers(0, 2)),
                                             seed=it), mod)
    y = mod.random_residues(rng, n)
    rows = [0, 1, n // 2, n - 1]
    ot, ov = O.krylov_unit(to_oracle(A), O.ints_to_limbs(y, mod.limbs), rows, steps)
    want = [O.limbs_to_ints(t) for t in ot]
    wv = O.limbs_to_ints(ov)
    for ch in ("1", "0"):
        os.environ["SLD_CHAIN"] = ch
        mul = B200Multiplier(A)
        terms, v, _ = krylov_column(mul, UnitRows(rows), ints_to_planes(y, digit_count(mod.ell)), steps)
        bad = [(k, j) for k in range(steps) for j in range(len(rows)) if terms[k][j] != want[k][j]]
        gv = planes_to_ints(v)
        badv = [i for i in range(n) if gv[i] != wv[i]]
        if bad or badv:
            fails += 1
        print(f"it {it} n={n} bits={bits} steps={steps} chain={ch}: {len(bad)} bad terms {bad[:6]} "
              f"{len(badv)} bad rows {badv[:6]}", flush=True)
        if bad:
            # which side is wrong: exact Python row dots of the first product
            k0, j0 = bad[0]
            r = rows[j0]
            orc = to_oracle(A)
            v1o = O.limbs_to_ints(orc.spmv_limbs(O.ints_to_limbs(y, mod.limbs), nthreads=1))
            dm = mul.dm if hasattr(mul, "dm") else None
            from paper_1402_3661_b200.device import DeviceMatrix
            dmx = DeviceMatrix(A)
            vi, vo = dmx.vector(), dmx.vector()
            vi.upload_limbs(O.ints_to_limbs(y, mod.limbs))
            dmx.spmv(vi, vo)
            v1g = O.limbs_to_ints(vo.download_limbs())
            ex = [sum(c * y[col] for col, c in A.row_entries(i)) % mod.ell for i in (r, 0, n - 1)]
            print(f"   row {r}: exact {ex[0] % 1000} oracle {v1o[r] % 1000} gpu {v1g[r] % 1000}; "
                  f"row n-1 exact==oracle {ex[2] == v1o[n - 1]} exact==gpu {ex[2] == v1g[n - 1]}; "
                  f"oracle-vs-gpu rows differing {sum(1 for i in range(n) if v1o[i] != v1g[i])}; "
                  f"terms[1]: {[t % 1000 for t in terms[1]]} want {[t % 1000 for t in want[1]]}; "
                  f"dense {len(A.dense_cols)} full {len(A.full_vals)}", flush=True)
        del mul
print(f"{fails} failing runs in {time.time() - t0:.0f} s")

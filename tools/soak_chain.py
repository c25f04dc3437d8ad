"""Long-chain soak at the BASELINE sizes: a device-resident Krylov chain of
many products in the layout the bench times, with the WHOLE iterate checked
against the CPU oracle's product at evenly spaced checkpoints.

At checkpoint k the chain's v_k comes back, one more device step makes
v_{k+1} and the unit-X term a_k = X^T v_k, and the oracle (oracle/, the C
restatement of the reference SpMV) computes A v_k on the host cores:
v_{k+1} must equal it in every row, and a_k must equal v_k's X rows.

    python tools/soak_chain.py --config cfg3 --steps 100000 --checks 10
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (test infrastructure: the checker only)
from paper_1402_3661_b200 import corpus  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402

SIZES = {"cfg2": (650_000, 217), "cfg3": (3_600_000, 202), "cfg5": (1_000_000, 650)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(SIZES))
    ap.add_argument("--steps", type=int, default=100_000)
    ap.add_argument("--checks", type=int, default=10)
    ap.add_argument("--chains", type=int, default=1)
    a = ap.parse_args()
    n, bits = SIZES[a.config]
    G = a.chains
    t0 = time.time()
    mod = corpus.random_prime(bits, np.random.default_rng(1))
    A = corpus.generate(corpus.profile_ffs(n, seed=1), mod)
    fpos = sorted(A.full_vals)
    orc = O.OracleMatrix(A.mod.ell, A.nrows, A.ncols, A.row_ptr, A.col_idx, A.tags, A.small_vals,
                         fpos, [A.full_vals[p] for p in fpos], None)
    dm = DeviceMatrix(A, chains=G)
    print(f"# {a.config}: N={n} nnz={A.nnz} {bits}-bit l, chains per pass {G}, layout {dm.info()}, "
          f"built in {time.time() - t0:.1f}s", flush=True)
    rng = np.random.default_rng(2024 + n)
    ys = [_random_residue_limbs(rng, A.total_cols, mod) for _ in range(G)]
    v = dm.vector()
    v.upload_limbs(ys[0] if G == 1 else np.stack(ys))
    x_rows = np.array(sorted(int(r) for r in rng.choice(A.nrows, 16, replace=False)))
    per = max(1, a.steps // a.checks)
    done, ok, t_dev = 0, 0, 0.0
    for c in range(a.checks):
        t = time.time()
        dm.krylov_unit(v, x_rows, per - 1)
        done += per - 1
        vk = v.download_limbs()
        terms = dm.krylov_unit(v, x_rows, 1)  # a_k and v_{k+1}
        done += 1
        vk1 = v.download_limbs()
        t_dev += time.time() - t
        vk = [vk] if G == 1 else list(vk)
        vk1 = [vk1] if G == 1 else list(vk1)
        tk = [terms[0]] if G == 1 else [terms[0][g] for g in range(G)]
        t = time.time()
        good = True
        for g in range(G):
            want = orc.spmv_limbs(vk[g])
            rows_bad = int(np.count_nonzero((vk1[g] != want).any(axis=1)))
            term_ok = np.array_equal(tk[g], vk[g][x_rows])
            nz = bool(vk1[g].any())
            good &= rows_bad == 0 and term_ok and nz
            print(f"step {done:>7}  chain {g}: v_{done} vs oracle A v_{done - 1}: "
                  f"{rows_bad} of {A.nrows} rows differ; term a_{done - 1} "
                  f"{'==' if term_ok else '!='} X^T v_{done - 1}; oracle {time.time() - t:.1f}s", flush=True)
        ok += good
    v.close()
    dm.close()
    print(f"# {a.config}: {done} products, {ok}/{a.checks} checkpoints bit-exact in every row "
          f"(device + transfers {t_dev:.1f}s)", flush=True)
    sys.exit(0 if ok == a.checks else 1)


if __name__ == "__main__":
    main()

"""Mksol Horner steps on the device (solver.py:508-552): w <- A w + sum_j
f_j[i] y_j, one SpMV plus one fused combination kernel per step, against the
plain SpMV step on the same matrix:
python tools/bench_mksol.py --config cfg3 --n 8 --degree 48"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1402_3661_b200 import B200Multiplier  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.modring import digit_count, limbs_to_planes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--degree", type=int, default=48)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="fused,batch0,batch2,batch4")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    A, _, mod = bench.build_matrix(cfg, lambda m: print(m, file=sys.stderr))
    mul = B200Multiplier(A)
    rng = np.random.default_rng(4)
    P = digit_count(mod.ell)
    Y = [limbs_to_planes(_random_residue_limbs(rng, A.total_cols, mod), P) for _ in range(a.n)]
    polys = [[int(c) for c in rng.integers(1, 2**62, a.degree + 1)] for _ in range(a.n)]
    dm = mul.dm
    v = dm.vector()
    v.upload_planes(Y[0])
    dm.bench(v, 4, 0)
    _, spmv = dm.bench(v, 64, 0)
    mul.mksol(Y, [p[:3] for p in polys])  # warm-up (allocations, module load)
    # the per-step cost is the slope between two degrees (the y uploads and
    # the set-up of each call cancel); the fused step (combination in the
    # SpMV epilogue) against SpMV + combination kernel
    ws = []
    for mode in a.modes.split(","):
        fused = "1" if mode == "fused" else "0"
        os.environ["SLD_MKSOL_FUSED"] = fused
        os.environ["SLD_MKSOL_BATCH"] = mode[5:] if mode.startswith("batch") else "0"
        ws.append(mul.mksol(Y, [p[:a.degree + 1] for p in polys])[0])
        res = []
        for deg in (a.degree // 4, a.degree):
            best = None
            for _ in range(a.reps):  # best of reps: clocks and host jitter
                t = time.perf_counter()
                w, verified, horner, tail = mul.mksol(Y, [p[:deg + 1] for p in polys])
                dt = time.perf_counter() - t
                best = dt if best is None else min(best, dt)
            res.append((horner, best))
        (h0, t0), (h1, t1) = res
        label = {"fused": "fused epilogue", "batch0": "two kernels",
                 "batch2": "batched combination K=2", "batch4": "batched combination K=4"}[mode]
        print(f"{a.config} mksol n={a.n} {label}: {h1} Horner steps in "
              f"{t1:.3f} s, {h0} in {t0:.3f} s -> {(t1 - t0) / (h1 - h0) * 1e3:.3f} ms per Horner step; "
              f"plain SpMV {spmv:.3f} ms", flush=True)
    print(f"all Horner modes give identical results: {all(np.array_equal(ws[0], x) for x in ws[1:])}")


if __name__ == "__main__":
    main()

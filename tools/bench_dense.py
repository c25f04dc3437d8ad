"""Dense-X Krylov steps (DenseRows projection, solver.py:179-189) against
unit-X steps on one generated configuration:
python tools/bench_dense.py --config cfg2 --m 2,16 --steps 64"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix, XBlock  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--m", default="2,16")
    ap.add_argument("--steps", type=int, default=64)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    A, _, mod = bench.build_matrix(cfg, lambda m: print(m, file=sys.stderr))
    dm = DeviceMatrix(A)
    rng = np.random.default_rng(5)
    v = dm.vector()
    v.upload_limbs(_random_residue_limbs(rng, A.total_cols, mod))
    dm.krylov_unit(v, [0, 1], 8)
    import torch
    torch.cuda.synchronize()
    t = time.perf_counter()
    dm.krylov_unit(v, [0, 1], a.steps)
    unit = (time.perf_counter() - t) / a.steps * 1e3
    print(f"{a.config} unit X m=2: {unit:.4f} ms/step")
    for m in [int(x) for x in a.m.split(",")]:
        x = np.stack([_random_residue_limbs(rng, A.total_cols, mod) for _ in range(m)])
        xb = XBlock(dm.field, x)
        dm.krylov_dense(v, xb, 4)
        t = time.perf_counter()
        dm.krylov_dense(v, xb, a.steps)
        dense = (time.perf_counter() - t) / a.steps * 1e3
        print(f"{a.config} dense X m={m}: {dense:.4f} ms/step (+{dense - unit:.4f} ms projection)")


if __name__ == "__main__":
    main()

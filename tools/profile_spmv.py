"""Short driver for ncu captures: build a bench configuration and run a few
products (python tools/profile_spmv.py --config cfg3 --steps 6)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--stripe-cols", type=int, default=0)
    ap.add_argument("--chains", type=int, default=1)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    A, _, mod = bench.build_matrix(cfg, lambda m: print(m, file=sys.stderr))
    dm = DeviceMatrix(A, stripe_cols=a.stripe_cols, chains=a.chains)
    print(dm.info(), file=sys.stderr)
    v = dm.vector()
    y = _random_residue_limbs(np.random.default_rng(5), A.total_cols, mod)
    v.upload_limbs(y if a.chains == 1 else np.stack([y] * a.chains))
    tot, per = dm.bench(v, a.steps, 0)
    print(f"{a.steps} products: {per:.4f} ms/product (stripes={dm.info()['stripes']})", file=sys.stderr)


if __name__ == "__main__":
    main()

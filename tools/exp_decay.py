"""Experiment: per-product time of a small matrix against its column law
(power-law decay 0.5 = corpus default, 0 = uniform), chain on/off."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1402_3661_b200 import corpus  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
mod = corpus.random_prime(160, np.random.default_rng(1))
for decay in ([float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (0.5, 0.25, 0.0)):
    A = corpus.generate(corpus.CorpusProfile(n=n, gamma=20, density_decay=decay, seed=1), mod)
    for ch in ("1", "0"):
        os.environ["SLD_CHAIN"] = ch
        dm = DeviceMatrix(A)
        v = dm.vector()
        v.upload_limbs(_random_residue_limbs(np.random.default_rng(5), A.total_cols, mod))
        tot, per = dm.bench(v, 2000, 10)
        print(f"n={n} decay={decay} chain={ch}: {per * 1000:.2f} us/product", flush=True)
        dm.close()

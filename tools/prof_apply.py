"""Where the time of the host-planes apply goes (cfg3): numpy allocation and
first touch, the upload (threaded repack + DMA), the product, the download."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402
from paper_1402_3661_b200.modring import digit_count, limbs_to_planes  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
A, _, mod = bench.build_matrix(cfg, lambda m: None)
dm = DeviceMatrix(A)
P = digit_count(mod.ell)
planes = limbs_to_planes(_random_residue_limbs(np.random.default_rng(5), A.total_cols, mod), P)
vin, vout = dm.vector(), dm.vector()
for rep in range(3):
    t0 = time.perf_counter()
    out = np.empty((A.nrows, P), dtype=np.uint64)
    t1 = time.perf_counter()
    out.fill(0)
    t2 = time.perf_counter()
    vin.upload_planes(planes)
    t3 = time.perf_counter()
    dm.spmv(vin, vout)
    t4 = time.perf_counter()
    o2 = vout.download_planes(P)
    t5 = time.perf_counter()
    r = dm.apply_planes(planes)
    t6 = time.perf_counter()
    print(f"rep {rep}: empty {1e3*(t1-t0):.1f} ms, first touch {1e3*(t2-t1):.1f} ms, upload {1e3*(t3-t2):.1f} ms, "
          f"spmv {1e3*(t4-t3):.1f} ms, download (incl. alloc) {1e3*(t5-t4):.1f} ms; apply_planes {1e3*(t6-t5):.1f} ms; "
          f"cpus {os.cpu_count()}", flush=True)

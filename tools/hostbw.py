"""Host memory bandwidth on the GPU box: streaming reads of a planes-sized
array with 1..16 threads (numpy releases the GIL), against the plane repack."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

n = 3_600_000 * 13
a = np.random.default_rng(1).integers(0, 1 << 16, size=n, dtype=np.uint64)
for nt in (1, 4, 8, 16):
    parts = np.array_split(a, nt)
    with ThreadPoolExecutor(nt) as ex:
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            list(ex.map(lambda p: int(p[::1].sum()), parts))
            best = min(best, time.perf_counter() - t)
    print(f"{nt} threads: sum of {a.nbytes / 1e6:.0f} MB in {best * 1e3:.1f} ms = {a.nbytes / best / 1e9:.1f} GB/s", flush=True)
from paper_1402_3661_b200 import PrimeModulus  # noqa: E402
from paper_1402_3661_b200.device import DeviceVector, Field  # noqa: E402
from paper_1402_3661_b200.corpus import random_prime  # noqa: E402
mod = random_prime(202, np.random.default_rng(1))
f = Field(mod, 0)
v = DeviceVector(f, 3_600_000)
planes = a.reshape(3_600_000, 13)
for _ in range(3):
    t = time.perf_counter()
    v.upload_planes(planes)
    print(f"upload_planes: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)

"""TEST INFRASTRUCTURE -- packs the reference package for the GPU box.

The reference (`sldlag`, pure Python) lives at /root/reference, which the
GPU box does not have.  `bundle()` zips its package and the test modules that
exercise the multiplier protocol into oracle/_ref/sldlag_ref.zip (git-ignored,
not gpurun-ignored, so it travels with the snapshot like a built .so).
tests/test_reference_driver_gpu.py unpacks it into a temp directory and runs
the reference's OWN drivers and tests -- krylov_block, block_wiedemann,
_mksol_core, tests/test_solver.py -- with its SequentialMultiplier swapped
for B200Multiplier.  Nothing in the product package reads this archive.
"""
import os
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("SLD_REFERENCE", "/root/reference")
OUT = os.path.join(HERE, "_ref", "sldlag_ref.zip")
TESTS = ["oracles.py", "test_solver.py", "test_acceptance.py", "test_spmatrix.py", "test_gridmv.py"]


def bundle(force=False):
    src = os.path.join(REF, "pkg", "src", "sldlag")
    if not os.path.isdir(src):
        return OUT if os.path.exists(OUT) else None
    newest = max(os.path.getmtime(os.path.join(src, f)) for f in os.listdir(src))
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest and newest > 0:
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    def add(z, path, name):  # the reference tree carries 1970 mtimes; zip needs >= 1980
        with open(path, "rb") as f:
            z.writestr(zipfile.ZipInfo(name, (1980, 1, 1, 0, 0, 0)), f.read(), zipfile.ZIP_DEFLATED)

    with zipfile.ZipFile(tmp, "w") as z:
        for f in sorted(os.listdir(src)):
            if f.endswith(".py"):
                add(z, os.path.join(src, f), f"src/sldlag/{f}")
        for f in TESTS:
            p = os.path.join(REF, "pkg", "tests", f)
            if os.path.exists(p):
                add(z, p, f"tests/{f}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(bundle(force=True))

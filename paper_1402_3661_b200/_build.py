"""Build libsldb200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): `python -m paper_1402_3661_b200._build [--force]`.
Translation units compile in parallel; the kernel instantiations are split
by limb count (csrc/sld_inst_*.cu)."""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
OUT_DIR = os.path.join(PKG, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libsldb200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "-Xptxas", "-O3", "--expt-relaxed-constexpr"]
if os.environ.get("SLD_NVCC_EXTRA"):
    NVCC_FLAGS += os.environ["SLD_NVCC_EXTRA"].split()
SOURCES = ["sld_capi.cu", "sld_grid.cu", "sld_inst_1_8.cu", "sld_inst_9_16.cu", "sld_inst_17_24.cu",
           "sld_inst_25_32.cu", "sld_corpus.cpp", "sld_fileio.cpp",
           "sld_split.cpp"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libsldb200.so")


def _newest_dep():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "sldb200.h")]
    return max(os.path.getmtime(d) for d in deps)


def _stale():
    return not os.path.exists(LIB) or _newest_dep() > os.path.getmtime(LIB)


def build(force=False, verbose=False, variant=None, defines=()):
    """Build the library; `variant` + `defines` (-D flags) build an
    experiment copy into _lib/<variant>/ (loaded with SLD_LIB=<path>)."""
    lib, obj_dir = LIB, OBJ_DIR
    if variant:
        lib = os.path.join(OUT_DIR, variant, "libsldb200.so")
        obj_dir = os.path.join(OUT_DIR, variant, "obj")
    elif not force and not _stale():
        return LIB
    os.makedirs(obj_dir, exist_ok=True)
    cc = nvcc()
    newest = _newest_dep()

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
        if not force and not variant and os.path.exists(obj) and os.path.getmtime(obj) > newest:
            return obj
        cmd = [cc, *NVCC_FLAGS, *defines, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread", "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    variant = None
    if "--variant" in sys.argv:
        variant = sys.argv[sys.argv.index("--variant") + 1]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=variant,
                defines=[a for a in sys.argv[1:] if a.startswith("-D")]))

"""Static SASS instruction counts of the tensor-core and SpMV kernels
(cuobjdump -sass of the built objects): the evidence that the digit GEMM and
the Mksol combination issue tcgen05 MMAs (UTCIMMA), commit through UTCBAR,
read TMEM with LDTM and stage operands with bulk copies (UBLKCP).
python tools/sass_counts.py > profiles/sass_counts_r02.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_1402_3661_b200", "_lib", "obj", "sld_inst_1_8.o")
KEYS = ["UTCIMMA", "UTCBAR", "LDTM", "UBLKCP", "SYNCS", "ELECT", "UTCATOMSWS", "FENCE.VIEW.ASYNC",
        "IMAD.WIDE", "LDG", "STG"]
PICK = re.compile(r"tc_digit_gemm|tcl_combineILi7E|spmv_passILi7ELi[12]ELb1ELb0ELb0E")


def main():
    txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1] if len(sys.argv) > 1 else OBJ],
                         capture_output=True, text=True, check=True).stdout
    print("kernel (demangled prefix) | " + " | ".join(KEYS))
    for f in re.split(r"\n\s*Function : ", txt)[1:]:
        name = f.split("\n", 1)[0].strip()
        if not PICK.search(name):
            continue
        c = collections.Counter()
        for ln in f.split("\n"):
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
            if m:
                for k in KEYS:
                    if m.group(2).startswith(k):
                        c[k] += 1
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        print(f"{dem[:60]} | " + " | ".join(str(c.get(k, 0)) for k in KEYS))


if __name__ == "__main__":
    main()

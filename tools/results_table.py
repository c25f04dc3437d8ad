"""Regenerate DESIGN.md §10 (results table) from profiles/bench_*_r02.json
(r01 where a config has no r02 run): python tools/results_table.py [--write]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BEGIN, END = "<!-- results:begin -->", "<!-- results:end -->"


def table():
    rows = []
    def latest(name):
        for r in ("r02", "r01"):
            p = os.path.join(ROOT, "profiles", f"{name}_{r}.json")
            if os.path.exists(p):
                return json.loads(open(p).read().strip().splitlines()[-1]), r
        return None, None

    for c in ("cfg1", "cfg2", "cfg3", "cfg5"):
        d, r = latest(f"bench_{c}")
        if d is None:
            continue
        cpu = (d.get("cpu_baseline") or {}).get("value") or 0.0
        floor = (d.get("gather_floor") or {}).get("frac_of_floor")
        rows.append(f"| {c} ({r}) | {d['value']:.0f} | {d.get('ms_per_chain_product', d['ms_per_step']):.4f} | "
                    f"{d['e2e']['value']:.0f} | {d['roofline']['frac']:.3f} ({d['roofline']['bound']}) | "
                    f"{floor if floor is None else f'{floor:.2f}'} | {cpu:.2f} |")
    ref, _ = latest("bench_ref_cfg3")
    out = [BEGIN,
           "| Config | SpMV/s (device) | ms per chain-product | e2e SpMV/s | roofline frac (binding bound) | "
           "frac of the gather floor | CPU port SpMV/s |",
           "|---|---|---|---|---|---|---|", *rows, ""]
    if ref:
        out.append(f"Reference arm (`bench.py --impl reference`, cfg3, C port of the reference algorithm "
                   f"on all host cores): {ref['value']:.2f} SpMV/s.")
        py = ref.get("reference_python") or {}
        if py.get("value"):
            out.append(f"The reference package itself (`sldlag.spmatrix.spmv_planes`, one core) on the same "
                       f"box: {py['s_per_spmv']:.1f} s per SpMV.")
    out.append(END)
    return "\n".join(out)


if __name__ == "__main__":
    t = table()
    if "--write" in sys.argv:
        p = os.path.join(ROOT, "DESIGN.md")
        s = open(p).read()
        i, j = s.index(BEGIN), s.index(END) + len(END)
        open(p, "w").write(s[:i] + t + s[j:])
    print(t)

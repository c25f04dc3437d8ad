"""Regenerate DESIGN.md §10 (results table) from profiles/bench_*_r01.json:
python tools/results_table.py [--write]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BEGIN, END = "<!-- results:begin -->", "<!-- results:end -->"


def table():
    rows = []
    for c in ("cfg1", "cfg2", "cfg3", "cfg5"):
        p = os.path.join(ROOT, "profiles", f"bench_{c}_r01.json")
        if not os.path.exists(p):
            continue
        d = json.loads(open(p).read().strip().splitlines()[-1])
        cpu = (d.get("cpu_baseline") or {}).get("value") or 0.0
        rows.append(f"| {c} | {d['value']:.0f} | {d.get('ms_per_chain_product', d['ms_per_step']):.4f} | "
                    f"{d['e2e']['value']:.0f} | {d['roofline']['frac']:.3f} | {d['gather_roofline']['frac']:.2f} "
                    f"({d['gather_roofline'].get('sectors_per_request', '-')}-sector) | {cpu:.2f} |")
    ref = os.path.join(ROOT, "profiles", "bench_ref_cfg3_r01.json")
    refv = json.loads(open(ref).read().strip().splitlines()[-1])["value"] if os.path.exists(ref) else None
    out = [BEGIN,
           "| Config | SpMV/s (device) | ms per chain-product | e2e SpMV/s | HBM roofline frac | "
           "gather roofline frac | CPU port SpMV/s |",
           "|---|---|---|---|---|---|---|", *rows, ""]
    if refv:
        out.append(f"Reference arm (`bench.py --impl reference`, cfg3, C port of the reference algorithm "
                   f"on all host cores): {refv:.2f} SpMV/s.")
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

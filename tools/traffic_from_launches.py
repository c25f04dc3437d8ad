"""DRAM bytes per step from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum over the spmv_ kernels):
python tools/traffic_from_launches.py launches.csv cfg3 G passes_per_step out.json [kernel-substring]"""
import csv
import io
import json
import sys


def parse(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        out.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"]})[d["Metric Name"]] = \
            float(d["Metric Value"].replace(",", ""))
    return [out[k] for k in sorted(out)]


def main():
    path, cfg, G, per_step, dst = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    ls = parse(path)
    if len(sys.argv) > 6:
        ls = [x for x in ls if sys.argv[6] in x["kernel"]]
    n = (len(ls) // per_step) * per_step
    last = ls[n - 2 * per_step:n]  # the last two complete steps
    steps = len(last) // per_step
    rd = sum(x["dram__bytes_read.sum"] for x in last) / steps
    wr = sum(x["dram__bytes_write.sum"] for x in last) / steps
    ns = sum(x["gpu__time_duration.sum"] for x in last) / steps
    json.dump({"config": cfg, "chains": G, "dram_bytes_per_pass": rd + wr, "dram_read_per_step": rd,
               "dram_write_per_step": wr, "ncu_step_ns": ns, "launches_per_step": per_step,
               "kernels": sorted({x["kernel"] for x in last}),
               "source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                         f"dram__bytes_write.sum), last {steps} steps x {per_step} launches"},
              open(dst, "w"), indent=1)
    print(open(dst).read())


if __name__ == "__main__":
    main()

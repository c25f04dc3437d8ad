#!/usr/bin/env python
"""Benchmark of the B200 Krylov SpMV hot path (BASELINE.json metric:
"SpMV/s mod l (ms per iteration) at 1/2/4/8 B200; % of HBM/IMAD roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

A step is one exact product v <- A v mod l of one Krylov chain on one GPU
(all column-stripe passes).  Multi-GPU (torchrun, one process per GPU) runs
one independent block-Wiedemann chain per rank -- the sequences never
communicate (sldlag/solver.py:220-257) -- so scaling is weak and there is no
data-path collective; the barrier and the max-over-ranks timing use
torch.distributed.

`--impl reference` times the reference's CPU algorithm -- the C restatement
of sldlag's exact RNS SpMV in oracle/ (the Python reference cannot travel to
the GPU box) -- on all host cores, each step a bounded row sample of the same
matrix, rank 0 only.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV/s mod ℓ (ms per iteration) at 1/2/4/8 B200; % of HBM/IMAD roofline"

CONFIGS = {
    # BASELINE.json configs; bp = (n, m) blocking of the block Wiedemann run
    "cfg1": dict(n=20_000, gamma=20, bits=160, bp=(1, 2), steps=2000, warmup=50, chains=1,
                 desc="configs[0]: synthetic N=20K, gamma=20, 160-bit l (CPU-oracle case)"),
    # cfg2 is ONE sequence (bp n = 1), so one chain; chain groups (G = 2, 4)
    # only apply when block Wiedemann runs n >= 2 sequences (cfg3: n = 8)
    "cfg2": dict(n=650_000, gamma=100, bits=217, bp=(1, 2), steps=2000, warmup=20, chains=1,
                 desc="configs[1]: GF(2^619)-scale N=650K FFS profile, 217-bit l, one sequence"),
    # cfg3 is block Wiedemann with 8 sequences, ONE per GPU: the headline
    # runs one chain per GPU; the chain group (2 of the sequences sharing a
    # matrix pass, what one GPU running several sequences would do) is
    # reported beside it as `chain_group`
    "cfg3": dict(n=3_600_000, gamma=100, bits=202, bp=(8, 16), steps=1000, warmup=10, chains=1, group=2,
                 desc="configs[2]: GF(2^809)-scale N=3.6M FFS profile, 202-bit l, "
                      "block Wiedemann (8,16), one sequence per GPU"),
    "cfg4": dict(n=3_600_000, gamma=100, bits=202, bp=(1, 2), steps=100, warmup=5, chains=1,
                 desc="configs[3]: the cfg3 matrix, ONE sequence row/2D-partitioned over the GPUs "
                      "(grid r x c, NCCL exchange)"),
    "cfg5": dict(n=1_000_000, gamma=100, bits=650, bp=(8, 16), steps=1000, warmup=10, chains=1,
                 desc="configs[4]: wide-prime stress N=1M FFS profile, 650-bit l, one sequence per GPU"),
}
DEFAULT_CONFIG = "cfg3"

# measured random-gather rates from L2 (GB/s) for records of 1-4 sectors
# fetched by one instruction of 1-4 lanes (profiles/microbench_r01.txt,
# microbench2_r01.txt; 96-byte records straddle 128-byte lines)
L2_GATHER_PEAK_GBS = {1: 9200.0, 2: 15460.0, 3: 12880.0, 4: 16990.0}
# measured int32 add rate (IADD carry chain, profiles/microbench_r01.txt)
INT32_PEAK_TOPS = 19.64


def dist_env():
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = int(os.environ.get("SLD_BENCH_NDEV", "0"))
    if ndev:  # test hook: fold more ranks than GPUs onto the visible devices
        local %= ndev
    return rank, world, local


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"), "/root/repo/MEASURED_PEAKS.json"):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    every 2 ms (a 20-product cfg3 region is ~30 ms), nvidia-smi every 0.1 s
    when NVML is unavailable.  The NVML device is found by the CUDA device's
    PCI bus id, so CUDA_VISIBLE_DEVICES remapping cannot pick another GPU."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, power_w, reason flags x4)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self.source = "nvidia-smi"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            self._nvml = pynvml
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        p = self._nvml
        sm = float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM))
        r = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        try:
            pw = p.nvmlDeviceGetPowerUsage(self._h) / 1000.0
        except Exception:
            pw = None
        bits = [p.nvmlClocksEventReasonHwSlowdown, p.nvmlClocksEventReasonHwThermalSlowdown,
                p.nvmlClocksEventReasonSwThermalSlowdown, p.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((sm, self._max, pw, *[bool(r & b) for b in bits]))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        if len(f) >= 7 and f[0].replace(".", "").isdigit():
            pw = float(f[2]) if f[2].replace(".", "").isdigit() else None
            self.samples.append((float(f[0]), float(f[1]), pw, *[x == "Active" for x in f[3:7]]))

    def _sample(self):
        try:
            self._sample_nvml() if self._nvml else self._sample_smi()
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.002 if self._nvml else 0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples:  # a region shorter than the first sample: take one at its end
            self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[3 + i]})
        pw = sorted(s[2] for s in self.samples if s[2] is not None)
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source,
                "power_w_median": pw[len(pw) // 2] if pw else None}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def build_matrix(cfg, log):
    from paper_1402_3661_b200 import corpus
    mod = corpus.random_prime(cfg["bits"], np.random.default_rng(1))
    prof = corpus.CorpusProfile(n=cfg["n"], gamma=cfg["gamma"], seed=1)
    t = time.time()
    A, wit = corpus.generate_with_witnesses(prof, mod)
    log(f"generated N={A.nrows} nnz={len(A.col_idx)} full={len(A.full_vals)} in {time.time() - t:.1f}s")
    return A, wit, mod


def algorithmic_bytes(A, L):
    """B = 4 Z + 4 Zs + W Zf + 4 (N+1) + 2 N W, W = 4 L."""
    W = 4 * L
    Z = len(A.col_idx)
    Zs = int(np.count_nonzero(A.tags == 2))
    Zf = len(A.full_vals)
    N = A.nrows
    return 4 * Z + 4 * Zs + W * Zf + 4 * (N + 1) + 2 * N * W, Z, Zs, Zf


def int_ops(A, L):
    """O = L Z+-1 + 2L Zs + 4L^2 Zf + 8 L N."""
    Zpm = int(np.count_nonzero(A.tags <= 1))
    Zs = int(np.count_nonzero(A.tags == 2))
    return L * Zpm + 2 * L * Zs + 4 * L * L * len(A.full_vals) + 8 * L * A.nrows


def oracle_for(A):
    import oracle as O
    from paper_1402_3661_b200.modring import limbs_to_ints
    L = A.mod.limbs
    fpos = sorted(A.full_vals)
    return O.OracleMatrix(A.mod.ell, A.nrows, A.ncols, A.row_ptr, A.col_idx, A.tags, A.small_vals,
                          fpos, [A.full_vals[p] for p in fpos], None)


def cpu_sample(orc, y_limbs, target_s, log):
    """Time the oracle port on a bounded sample of one SpMV; returns
    (SpMV/s, cores, description).  The sample is the same fraction f of the
    SpMV's two halves, the to-RNS conversion (a window of f*ncols columns)
    and the rows, so one SpMV = the sample's time / f (oracle spmv_sample)."""
    cores = os.cpu_count() or 1
    N, nc = orc.nrows, orc.total_cols
    out = np.zeros((N, orc.L), dtype=np.uint32)
    orc.spmv_sample(y_limbs, (0, 0), (0, 0), out=out)  # first call converts in full, untimed

    def timed(rows):
        cc = max(1, rows * nc // N)
        t = time.time()
        orc.spmv_sample(y_limbs, (0, rows), (0, cc), out=out)
        return time.time() - t, cc

    rows = min(N, 2000)
    while True:
        dt, _ = timed(rows)
        if dt > 0.5 or rows >= N:
            break
        rows = min(N, rows * 4)
    # scale the sample to ~target_s of CPU work
    rows2 = int(min(N, max(rows, target_s * rows / max(dt, 1e-9))))
    dt2, cc2 = timed(rows2)
    spmv_s = dt2 * N / rows2
    log(f"cpu oracle: {rows2} rows + {cc2} columns converted in {dt2:.2f}s -> {spmv_s:.3f} s/SpMV")
    return 1.0 / spmv_s, cores, (f"oracle C port, rows [0,{rows2}) of {N} and the to-RNS conversion "
                                 f"of columns [0,{cc2}) of {nc}, {cores} threads, scaled to one SpMV")


def reference_python_sample(A, mod, y_limbs, log):
    """The reference package itself (sldlag.spmatrix.spmv_planes, pure
    Python + numpy, one core) on row samples of the same matrix, from the
    archive oracle/ref_bundle.py packs (absent: None).  t(R) = a + b R over
    two sample sizes R (a: the full-vector conversion), extrapolated to N
    rows; the kernel build is cached first, as in a Krylov loop."""
    import tempfile
    import zipfile
    z = os.path.join(ROOT, "oracle", "_ref", "sldlag_ref.zip")
    if not os.path.exists(z):
        return None
    try:
        d = tempfile.mkdtemp(prefix="sldlag_ref_")
        with zipfile.ZipFile(z) as zf:
            zf.extractall(d)
        for p in (os.path.join(ROOT, "oracle", "gmpy2_shim"), os.path.join(d, "src")):
            if p not in sys.path:
                sys.path.insert(0, p)
        from sldlag import modring as RM
        from sldlag import spmatrix as RS
        from sldlag import vecops as RV

        from paper_1402_3661_b200.modring import limbs_to_planes
        pm = RM.PrimeModulus(mod.ell)
        planes = limbs_to_planes(y_limbs, RV.digit_count(mod.ell))
        t_of = {}
        # two sizes far enough apart that the per-row slope b is well above
        # the timing noise of the conversion term a; best of 2 each
        r1, r2 = min(2000, A.nrows // 4), min(40000, A.nrows)
        if r1 < 1 or r2 <= r1:
            return None
        for R in (r1, r2):
            nz = int(A.row_ptr[R])
            M = RS.SparseMatrix(pm, R, A.ncols, A.row_ptr[:R + 1].copy(), A.col_idx[:nz].copy(),
                                A.tags[:nz].copy(), A.small_vals[:nz].copy(),
                                {p: v for p, v in A.full_vals.items() if p < nz}, [])
            M.kernel()  # built once per matrix, outside the per-SpMV cost
            best = None
            for _ in range(2):
                t = time.time()
                RS.spmv_planes(M, planes)
                best = min(best or 1e30, time.time() - t)
            t_of[R] = best
        b = max(t_of[r2] - t_of[r1], 1e-9) / (r2 - r1)
        a = max(t_of[r1] - r1 * b, 0.0)
        spmv_s = a + b * A.nrows
        log(f"reference python: {t_of} -> {spmv_s:.1f} s/SpMV")
        return {"value": 1.0 / spmv_s, "unit": "SpMV/s", "cores": 1, "kind": "reference",
                "s_per_spmv": spmv_s, "cpu": cpu_model(),
                "sample": f"sldlag.spmatrix.spmv_planes on rows [0,{r1}) and [0,{r2}) of the same matrix "
                          "(all columns, full input planes), t = a + b*rows extrapolated to N rows"}
    except Exception as e:  # a reported extra: never hide the arm's own line
        return {"value": None, "error": str(e)[:200]}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    log = lambda m: print(f"[bench/reference] {m}", file=sys.stderr, flush=True)  # noqa: E731
    import oracle as O
    O.build()
    A, _, mod = build_matrix(cfg, log)
    orc = oracle_for(A)
    rng = np.random.default_rng(3)
    from paper_1402_3661_b200.corpus import _random_residue_limbs
    y = _random_residue_limbs(rng, A.total_cols, mod)
    cores = os.cpu_count() or 1
    N = A.nrows
    # each step is a bounded sample of one SpMV: the same fraction f =
    # rows/N of its to-RNS conversion (a window of f*ncols columns) and of
    # its rows, so one SpMV = the step's time / f with nothing subtracted.
    # The sample is sized so the whole run stays within ~2-3 minutes.
    nc = A.total_cols
    out = np.zeros((N, mod.limbs), dtype=np.uint32)
    orc.spmv_sample(y, (0, 0), (0, 0), out=out)  # first call: the full conversion, untimed
    probe = min(N, 4000)
    t = time.time()
    orc.spmv_sample(y, (0, probe), (0, max(1, probe * nc // N)), out=out)
    per_row = max(time.time() - t, 1e-9) / probe
    budget = 120.0 / max(1, args.steps + args.warmup)
    rows = int(min(N, max(256, budget / per_row)))
    ccols = max(1, rows * nc // N)

    def sample(k):
        lo = (k * rows) % max(1, N - rows + 1)
        clo = (k * ccols) % max(1, nc - ccols + 1)
        orc.spmv_sample(y, (lo, lo + rows), (clo, clo + ccols), out=out)

    for k in range(args.warmup):
        sample(k)
    times = []
    for k in range(args.steps):
        t = time.time()
        sample(k)
        times.append(time.time() - t)
    per_step = float(np.median(times))
    spmv_s = per_step * N / rows
    value = 1.0 / spmv_s
    ref_py = reference_python_sample(A, mod, y, log)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "SpMV/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": spmv_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "exact integer mod l (RNS 31-bit limbs, reference algorithm)",
        "data": "synthetic (native corpus generator, FFS profile, seed 1)",
        "config": config_block(args.config, cfg, A, mod, world),
        "cpu_baseline": {"value": value, "unit": "SpMV/s", "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{rows} rows of {N} and the to-RNS conversion of {ccols} of {nc} "
                                   f"columns per step (the same fraction of both), median of "
                                   f"{args.steps} steps, scaled to one SpMV"},
        "e2e": {"value": value, "unit": "SpMV/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_python": ref_py,
    }
    print(json.dumps(line), flush=True)


def run_grid(args, cfg, rank, world, local, dist, log):
    """cfg4: one chain over an r x c grid (strong scaling); device-timed with
    CUDA events on the stream all grid work runs on, max over ranks."""
    import torch
    import torch.distributed as tdist
    from paper_1402_3661_b200.balance import GridSpec, balance_permutation
    from paper_1402_3661_b200.corpus import _random_residue_limbs
    from paper_1402_3661_b200.grid import B200Grid, GridComm
    if dist is None:
        import datetime
        import socket
        if "MASTER_ADDR" not in os.environ:  # plain `python bench.py`: a private 1-rank group
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]),
                              RANK="0", WORLD_SIZE="1")
            sk.close()
        tdist.init_process_group("nccl", timeout=datetime.timedelta(seconds=300),
                                 device_id=torch.device(f"cuda:{local}"))
    g = GridSpec.parse(args.grid) if args.grid else GridSpec(world, 1)
    A, _, mod = build_matrix(cfg, log)
    t = time.time()
    perm = balance_permutation(A, g)
    fused = args.grid_impl == "peer"
    nodes = g.r * g.c
    in_proc = fused and world == 1 and nodes > 1
    if fused:
        # exchanges done by the nodes over peer memory (csrc/sld_grid.cu via
        # paper_1402_3661_b200/peergrid.py): r x 1 -- the all-gather fused
        # into the SpMV epilogue; r x c -- partials pushed into the row
        # collector by the epilogue, reduced, scattered by one copy kernel.
        # Flag barriers, one CUDA graph per iteration, no collective.  With
        # one process and several nodes (--grid RxC on one rank) every node
        # lives in this process (LocalGrid), round robin over the GPUs.
        from paper_1402_3661_b200 import _native as N
        from paper_1402_3661_b200.peergrid import LocalGrid, PeerGrid
        local_dev = local
        torch.cuda.set_device(local_dev)
        if in_proc:
            grid = LocalGrid(A, g, perm=perm)
            members = grid.nodes
        else:
            def exchange(obj):
                out = [None] * world
                tdist.all_gather_object(out, obj)
                return out
            grid = PeerGrid(A, g, rank, exchange, device=local_dev, perm=perm)
            members = [grid.node]
        streams = []
        for nd in members:
            st_k = torch.cuda.Stream(device=nd.device)
            N.check(N.load().sld_ctx_set_stream(nd.field.handle, st_k.cuda_stream))
            streams.append(st_k)
        log(f"peer grid {g} {'all nodes in-process' if in_proc else f'node {rank}'} built in {time.time() - t:.1f}s")
    else:
        grid = B200Grid(A, g, GridComm(g), device=local, perm=perm)
        streams = [torch.cuda.current_stream()]
        log(f"grid {g} node {(grid.i, grid.j)} block built in {time.time() - t:.1f}s")
    y = _random_residue_limbs(np.random.default_rng(3), grid.n_padded, mod)
    grid.load_vector(y)
    grid.iterate(args.warmup)
    torch.cuda.synchronize()
    tdist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in streams]
    with ClockSampler(local) as clk:
        for (e0, _), st_k in zip(ev, streams):
            e0.record(st_k)
        grid.iterate(args.steps)
        for (_, e1), st_k in zip(ev, streams):
            e1.record(st_k)
        torch.cuda.synchronize()
    ms = max(e0.elapsed_time(e1) for e0, e1 in ev)
    t_all = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
    tdist.all_reduce(t_all, op=tdist.ReduceOp.MAX)
    ms = float(t_all.item())
    if fused:
        from paper_1402_3661_b200.balance import comm_volume_model
        q = math.lcm(g.r, g.c)
        frag_rows = grid.n_padded // q
        slot_bytes = 32 * ((4 * mod.limbs + 31) // 32)
        comm = {"impl": ("SpMV epilogue peer stores + flag barrier" if g.c == 1 else
                         "epilogue peer stores into the collector + add_mod + one scatter kernel + flag barriers")
                        + " (one CUDA graph per iteration, no collective)",
                "bytes_per_iter_reference_accounting": comm_volume_model(g, frag_rows * mod.byte_width),
                "wire_bytes_per_iter": comm_volume_model(g, frag_rows * slot_bytes),
                "messages_per_iter": 0}
        stripes = members[0].dm.info()["stripes"]
        per_iter = max(nd.info()["kernels_per_iteration"] for nd in members)
        comm["nodes_in_process"] = len(members)
    else:
        last = grid.comm_log.entries[-1]
        comm = {"impl": "NCCL p2p (collector reduce + broadcast, gridmv.py:251-348)",
                "bytes_per_iter_reference_accounting": last.total_bytes,
                "wire_bytes_per_iter": last.reduce.wire_bytes + last.broadcast.wire_bytes,
                "messages_per_iter": last.reduce.messages + last.broadcast.messages}
        stripes = grid.engine.dm.info()["stripes"]
        per_iter = stripes + (1 if g.c > 1 else 0)
    B, Z, Zs, Zf = algorithmic_bytes(A, mod.limbs)
    peak, peak_kind = measured_peaks()
    per = ms / args.steps
    line = {
        "metric": METRIC, "value": args.steps / (ms / 1e3), "unit": "SpMV/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 limbs, exact mod l",
        "grid_nodes_on_this_box": (f"{len(members)} node(s) in this process on "
                                   f"{len({nd.device for nd in members})} GPU(s)" if fused else None),
        "data": "synthetic (native corpus generator, FFS profile, seed 1)",
        "config": dict(config_block("cfg4", cfg, A, mod, world), grid=str(g),
                       parallelism=(f"one chain on a {g} grid, exchanges over peer memory (no collective)"
                                    if fused else f"one chain on a {g} grid (NCCL p2p / all-gather)")),
        "roofline": {"bound": "hbm", "achieved": B / world / (per / 1e3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": B / world / (per / 1e3) / 1e9 / peak, "traffic": None,
                     "peak_kind": peak_kind},
        "comm": comm,
        # rank 0 (a row collector): SpMV passes, add_mod when c > 1, and the
        # flag barriers of the peer exchange (1 for r x 1, 2 for r x c)
        "gpu_launches": args.steps * per_iter * (len(members) if fused else 1),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if fused:
        tdist.barrier()  # no peer may still push into buffers about to be freed
        grid.close()
    if dist is None:  # the private 1-rank group created above
        tdist.destroy_process_group()


def max_over_ranks(dist, x, local):
    import torch
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def config_block(name, cfg, A, mod, world, chains=1):
    return {"workload": f"{name}: {cfg['desc']}", "N": A.nrows, "nnz": int(len(A.col_idx)),
            "ell_bits": mod.bit_length, "gamma": cfg["gamma"], "bp": list(cfg["bp"]),
            "parallelism": f"independent Krylov chains, {chains} per GPU x {world} GPU(s)",
            "l2": "inputs larger than L2 (matrix streams >1 GB/step at cfg3); the iterate vector's "
                  "reuse across steps is the Krylov recurrence itself"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--grid", default=None, help="cfg4 grid RxC (default: <gpus>x1)")
    ap.add_argument("--grid-impl", default="peer", choices=["peer", "nccl"],
                    help="cfg4 exchange: over peer memory (default) or the NCCL node protocol")
    ap.add_argument("--chains", type=int, default=None,
                    help="Krylov chains advanced per matrix pass on each GPU (1, 2, 4)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    args.steps = args.steps or cfg["steps"]
    args.warmup = max(3, args.warmup if args.warmup is not None else cfg["warmup"])
    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import datetime
        import torch
        import torch.distributed as dist
        backend = os.environ.get("SLD_BENCH_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device(f"cuda:{local}")
        dist.init_process_group(backend, timeout=datetime.timedelta(seconds=600), **kw)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))  # noqa: E731
    if args.config == "cfg4":
        run_grid(args, cfg, rank, world, local, dist, log)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    from paper_1402_3661_b200 import B200Multiplier, UnitRows, krylov_column
    from paper_1402_3661_b200 import _native
    from paper_1402_3661_b200.corpus import _random_residue_limbs
    from paper_1402_3661_b200.device import DeviceMatrix
    from paper_1402_3661_b200.modring import digit_count, limbs_to_planes
    _native.load()
    A, wit, mod = build_matrix(cfg, log)
    t = time.time()
    G = args.chains or cfg["chains"]
    G = min(G, 4 if mod.limbs <= 8 else (2 if mod.limbs <= 16 else 1))
    dm = DeviceMatrix(A, device=local, chains=G)
    info = dm.info()
    log(f"device layout built in {time.time() - t:.1f}s: {info}")
    L, P = dm.L, digit_count(mod.ell)
    rng = np.random.default_rng(1000 + rank)
    ys = [_random_residue_limbs(rng, A.total_cols, mod) for _ in range(G)]
    y = ys[0]
    v = dm.vector()
    v.upload_limbs(ys[0] if G == 1 else np.stack(ys))

    # ---- device-timed region: W untimed, then exactly K products
    # (at least 32 products, so the per-product probe below is not a
    # handful of first launches)
    _, warm_ms = dm.bench(v, max(args.warmup, 32), 0)
    # per-sample events between graph launches: one sample per product pair,
    # or per 16 pairs (one 32-product graph) when a product is too short for
    # a per-pair launch not to dominate it (cfg1)
    pps = 1 if warm_ms > 0.1 else 16
    if dist is not None:
        import torch
        torch.cuda.synchronize()
        dist.barrier()
    with ClockSampler(local) as clk:
        # an event after every product pair (between graph launches) gives
        # the per-product samples for the median; the total is the K steps
        total_ms, samples = dm.bench_samples(v, args.steps, 0, pairs_per_sample=pps)
    if dist is not None:
        import torch
        torch.cuda.synchronize()
        total_ms = max_over_ranks(dist, total_ms, local)
        dist.barrier()
    steps_even = 2 * ((args.steps + 1) // 2)  # the bench graph replays product pairs
    ms_per_step = total_ms / steps_even       # one step = one product of each of the G chains
    value = world * G * steps_even / (total_ms / 1e3)
    launches = steps_even * info["stripes"]
    med_ms = float(np.median(samples))

    # several sequences per GPU (a GPU running more than one of the block-
    # Wiedemann sequences): Gc chains share each matrix pass, index stream
    # read once, the G residues of a column one contiguous record
    group = None
    Gc = cfg.get("group", 1) if args.chains is None else 1
    if Gc > 1 and mod.limbs <= 8:
        dmg = DeviceMatrix(A, device=local, chains=Gc)
        vg = dmg.vector()
        vg.upload_limbs(np.stack([ys[0]] + [_random_residue_limbs(rng, A.total_cols, mod)
                                            for _ in range(Gc - 1)]))
        dmg.bench(vg, args.warmup, 0)
        tg, sg = dmg.bench_samples(vg, args.steps, 0, pairs_per_sample=pps)
        group = {"chains_per_pass": Gc, "value": world * Gc * steps_even / (tg / 1e3), "unit": "SpMV/s",
                 "ms_per_pass": tg / steps_even, "ms_per_chain_product": tg / steps_even / Gc,
                 "ms_per_pass_median": float(np.median(sg)), "layout": dmg.info(),
                 "note": f"{Gc} sequences per GPU per matrix pass (bp n >= {Gc * world} at {world} GPU(s)); "
                         "not the headline, which is the config's one sequence per GPU"}
        vg.close()
        dmg.close()

    # ---- end to end through the public API with host y in, host terms (m
    # per chain and step) and the final iterates out: krylov_column for one
    # chain, the chain group (what krylov_block(chains_per_gpu=G) runs) for G
    bp_m = cfg["bp"][1]
    X = UnitRows(sorted(int(r) for r in np.random.default_rng(7).choice(A.nrows, bp_m, replace=False)))
    y_planes = [limbs_to_planes(yy, P) for yy in ys]
    if G == 1:
        mul = B200Multiplier(A, device=local, dm=dm)
        api = "krylov_column(B200Multiplier, UnitRows)"
    else:
        from paper_1402_3661_b200 import B200ChainGroup
        mul = B200ChainGroup(A, chains=G, device=local)
        mul._dm = dm
        api = f"B200ChainGroup(chains={G}).krylov(UnitRows) [krylov_block(chains_per_gpu={G})]"
    e2e_steps = args.steps
    # untimed warm-up through the same API (device iterate buffers, CUDA
    # graph instantiation, pinned staging are first-call costs)
    if G == 1:
        krylov_column(mul, X, y_planes[0], args.warmup)
    else:
        mul.krylov(X, y_planes, args.warmup)
    if dist is not None:
        dist.barrier()
    with ClockSampler(local) as clk_e2e:
        t0 = time.perf_counter()
        if G == 1:
            # the terms (the sequence, every step's result) come back to the
            # host; the final iterate stays on the device as DevicePlanes,
            # like .apply's result, until the caller reads it
            terms, v_out, spmvs = krylov_column(mul, X, y_planes[0], e2e_steps)
            v_bytes = 0
        else:
            terms, v_outs = mul.krylov(X, y_planes, e2e_steps)
            v_bytes = sum(vv.nbytes for vv in v_outs)
        t_e2e = time.perf_counter() - t0
    # reading the final iterate back as host planes, timed apart
    t0 = time.perf_counter()
    v_host_bytes = np.asarray(v_out).nbytes if G == 1 else 0
    t_iter = time.perf_counter() - t0 if G == 1 else 0.0
    if dist is not None:
        t_e2e = max_over_ranks(dist, t_e2e, local)
        t_iter = max_over_ranks(dist, t_iter, local)
    e2e_value = world * G * e2e_steps / t_e2e
    h2d = sum(yp.nbytes for yp in y_planes) + 8 * bp_m
    d2h = e2e_steps * G * bp_m * 4 * L + v_bytes
    # the plain multiplier protocol as well: host planes in/out every product
    n_apply = 3 if A.nrows > 1_000_000 else 10
    pl = y_planes[0] if G == 1 else np.stack(y_planes)
    t0 = time.perf_counter()
    for _ in range(n_apply):
        pl = dm.apply_planes(pl)
    t_apply = time.perf_counter() - t0
    # the reference's OWN krylov_column loop (solver.py:209-214: project,
    # apply) driving B200Multiplier unchanged: apply() leaves the iterate on
    # the device, so per step only the m projected rows come back
    dm_loop = dm if G == 1 else DeviceMatrix(A, device=local, chains=1)
    mul_loop = B200Multiplier(A, device=local, dm=dm_loop)
    n_loop = max(min(args.steps, 100), 8)
    v_loop = y_planes[0]
    for _ in range(args.warmup):
        X.project(v_loop)
        v_loop = mul_loop.apply(v_loop)
    v_loop = y_planes[0]
    t0 = time.perf_counter()
    loop_terms = []
    for _ in range(n_loop):
        loop_terms.append(X.project(v_loop))
        v_loop = mul_loop.apply(v_loop)
    final_loop = np.asarray(v_loop)
    t_loop = time.perf_counter() - t0
    del v_loop, mul_loop
    if dm_loop is not dm:
        dm_loop.close()

    # ---- kernel correctness spot check at full size: planted witness A w = 0
    ok_witness = None
    if wit:
        from paper_1402_3661_b200.modring import ints_to_planes, planes_to_ints
        wv = [0] * A.total_cols
        for c, val in wit[0].items():
            wv[c] = val
        wp = ints_to_planes(wv, P)
        out = dm.apply_planes(wp if G == 1 else np.stack([wp] * G))
        ok_witness = not any(planes_to_ints(out.reshape(-1, P)))

    # ---- roofline (SURVEY.md 8(d) algorithmic bytes per product; the index
    # stream is read once per pass for all G chains)
    B, Z, Zs, Zf = algorithmic_bytes(A, L)
    W = 4 * L
    B_pass = B + (G - 1) * (W * Zf + 2 * A.nrows * W)
    peak, peak_kind = measured_peaks()
    achieved = B_pass / (ms_per_step / 1e3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{args.config}_g{G}.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("dram_bytes_per_pass")
    gather_bytes = G * 32 * ((4 * L + 31) // 32) * (Z + Zf) + B_pass
    # sectors one gather instruction fetches as one request: G chains x the
    # lanes a residue is sliced over (wide moduli); otherwise a lane issues
    # one request per sector and the 1-sector rate applies
    rec_sectors = G * info.get("lanes_per_residue", 1)
    gpeak = L2_GATHER_PEAK_GBS[rec_sectors]
    # the floor of this algorithm: every nonzero's residue must reach the SMs
    # as one gather request, at the measured L2-resident request rate for the
    # record size (all gathers hitting L2, index stream free)
    floor_ms = gather_bytes / (gpeak * 1e9) * 1e3
    floor_frac = B_pass / (floor_ms / 1e3) / 1e9 / peak
    line = {
        "metric": METRIC, "value": value, "unit": "SpMV/s", "n_gpus": world, "steps": steps_even,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 limbs, exact mod l (int64 lazy accumulation)",
        "data": "synthetic (native corpus generator, FFS profile, seed 1, planted kernel column)",
        "config": dict(config_block(args.config, cfg, A, mod, world, chains=G), chains_per_gpu=G,
                       step=f"one product of each of the {G} chain(s) on every GPU",
                       sequences=(f"{G} of the block-Wiedemann sequences per GPU share each matrix pass "
                                  f"(chain group, --chains)"
                                  if G > 1 else "one sequence per GPU (the config's deployment)")),
        "ms_per_chain_product": ms_per_step / G,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_step": B_pass, "algorithmic_bytes_per_product": B,
                     "kernel": "spmv_pass (all stripe passes of one step)"},
        "gather_roofline": {"bound": "l2_random_gather_requests", "peak": gpeak,
                            "sectors_per_request": rec_sectors,
                            "unit": "GB/s", "bytes_per_step": gather_bytes,
                            "achieved": gather_bytes / (ms_per_step / 1e3) / 1e9,
                            "frac": gather_bytes / (ms_per_step / 1e3) / 1e9 / gpeak},
        "gather_floor": {"ms_per_step": floor_ms, "frac_of_floor": floor_ms / ms_per_step,
                         "hbm_frac_at_floor": floor_frac,
                         "note": "the derived target: at the floor (every gather an L2 hit at the measured "
                                 "request rate) the HBM roofline fraction would be hbm_frac_at_floor, so the "
                                 "contract's 0.60 is unreachable with one request per nonzero"},
        "ms_per_step_median": med_ms,
        "samples": {"count": int(len(samples)),
                    "per": f"{2 * pps} products (median of the per-product times over the samples)",
                    "p10_ms": float(np.percentile(samples, 10)), "p90_ms": float(np.percentile(samples, 90))},
        "int_ops_per_product": int_ops(A, L),
        # SURVEY 8(d)'s IMAD/INT32 side of the roofline: its op count O per
        # product against the measured int32 add rate (profiles/microbench_r01.txt)
        "int_roofline": {"bound": "int32", "ops_per_step": G * int_ops(A, L),
                         "achieved": G * int_ops(A, L) / (ms_per_step / 1e3) / 1e12,
                         "peak": INT32_PEAK_TOPS, "unit": "Tops/s", "peak_kind": "measured",
                         "frac": G * int_ops(A, L) / (ms_per_step / 1e3) / 1e12 / INT32_PEAK_TOPS},
        "e2e": {"value": e2e_value, "unit": "SpMV/s", "h2d_bytes_per_step": h2d / e2e_steps,
                "d2h_bytes_per_step": d2h / e2e_steps, "api": api, "steps": e2e_steps,
                "final_iterate": ("returned device-resident (DevicePlanes); reading it as host planes "
                                  "takes iterate_download_ms, outside this timed region") if G == 1 else
                                 "downloaded inside the timed region",
                "iterate_download_ms": t_iter * 1e3, "iterate_bytes": v_host_bytes,
                "value_with_iterate_download": world * G * e2e_steps / (t_e2e + t_iter)},
        "e2e_apply": {"value": world * G * n_apply / t_apply, "unit": "SpMV/s",
                      "h2d_bytes_per_step": G * y_planes[0].nbytes, "d2h_bytes_per_step": G * y_planes[0].nbytes,
                      "api": "DeviceMatrix.apply_planes: host planes in and out of every product"},
        "e2e_reference_loop": {"value": world * n_loop / t_loop, "unit": "SpMV/s",
                               "h2d_bytes_per_step": y_planes[0].nbytes / n_loop,
                               "d2h_bytes_per_step": (n_loop * bp_m * P * 8 + final_loop.nbytes) / n_loop,
                               "steps": n_loop,
                               "api": "the reference's krylov_column loop (project, mul.apply) with "
                                      "B200Multiplier, one chain: the iterate stays on the device"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "clocks_e2e": clk_e2e.summary(),
        "layout": info,
        "chain_group": group,
        "witness_check": ok_witness,
    }
    # north_star / SURVEY 8(d) d3: the roofline is the SLOWER of the HBM-byte
    # time and the INT32-issue time.  cfg1-cfg3 are HBM-bound (the line keeps
    # "roofline" = HBM); where the int-op time is the longer one (cfg5's
    # 650-bit residues) "roofline" is the int32 bound and the HBM figure moves
    # to "hbm_roofline".
    t_hbm = B_pass / (peak * 1e9)
    t_int = G * int_ops(A, L) / (INT32_PEAK_TOPS * 1e12)
    line["roofline"]["binding_time_us"] = {"hbm": t_hbm * 1e6, "int32": t_int * 1e6}
    if t_int > t_hbm:
        hbm = line.pop("roofline")
        line["roofline"] = dict(line["int_roofline"], traffic=hbm["traffic"],
                                binding_time_us=hbm["binding_time_us"],
                                kernel=hbm["kernel"], note="int32 issue time exceeds the HBM time (SURVEY 8(d) d3)")
        line["hbm_roofline"] = hbm
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            O.build()
            orc = oracle_for(A)
            val, cores, sample = cpu_sample(orc, y, args.cpu_seconds, log)
            line["cpu_baseline"] = {"value": val, "unit": "SpMV/s", "cores": cores, "kind": "port",
                                    "sample": sample, "cpu": cpu_model()}
        except Exception as e:  # the baseline must not hide the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs only in the build container (it imports /root/reference, which does not
exist on the GPU box).  The committed .npz files are what the tests read.

    PYTHONPATH=oracle/gmpy2_shim:/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Every expected value below is produced by the reference's own public entry
points (`spmv_sequential`, `krylov_block`, `Grid`, `balance_permutation`,
`permuted_padded`, `corpus.generate`, `cli.random_prime`, `draw_blocks`),
so the fixtures pin both the C oracle (oracle/) and the CUDA path.

Residues are stored as little-endian fixed-width byte rows (the reference's
own serialization, modring.py:112-130), one row per residue.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _need_reference():
    try:
        import sldlag  # noqa: F401
    except ImportError as e:  # pragma: no cover - container-only script
        raise SystemExit(
            "make_golden.py needs the reference on PYTHONPATH "
            "(oracle/gmpy2_shim:/root/reference/pkg/src:/root/reference/pkg/tests)"
        ) from e


_need_reference()

import gmpy2  # noqa: E402  (the shim)
from sldlag import cli, vecops  # noqa: E402
from sldlag.balance import GridSpec, balance_permutation, permuted_padded, split  # noqa: E402
from sldlag.corpus import CorpusProfile, generate  # noqa: E402
from sldlag.gridmv import Grid, run_iterations  # noqa: E402
from sldlag.modring import PrimeModulus  # noqa: E402
from sldlag.solver import (  # noqa: E402
    BlockingParams, DenseRows, SolverFailure, UnitRows, berlekamp_massey, block_lingen,
    draw_blocks, krylov_block, krylov_length, krylov_scalar, mksol_block, mksol_scalar,
)
from sldlag.spmatrix import SparseMatrix, spmv_sequential  # noqa: E402
from test_spmatrix import random_matrix  # noqa: E402  (reference test helper)


def res_bytes(vals, bw):
    vals = list(vals)
    out = np.zeros((len(vals), bw), dtype=np.uint8)
    if vals:
        out[:] = np.frombuffer(b"".join(int(v).to_bytes(bw, "little") for v in vals),
                               dtype=np.uint8).reshape(len(vals), bw)
    return out


def matrix_arrays(prefix, A):
    """Flatten a reference SparseMatrix into npz-able arrays."""
    bw = A.mod.byte_width
    fpos = sorted(A.full_vals)
    d = {
        f"{prefix}ell": np.array(hex(A.mod.ell)),
        f"{prefix}shape": np.array([A.nrows, A.ncols], dtype=np.int64),
        f"{prefix}row_ptr": A.row_ptr.astype(np.int64),
        f"{prefix}col_idx": A.col_idx.astype(np.int32),
        f"{prefix}tags": A.tags.astype(np.uint8),
        f"{prefix}small_vals": A.small_vals.astype(np.int32),
        f"{prefix}full_pos": np.array(fpos, dtype=np.int64),
        f"{prefix}full_vals": res_bytes([A.full_vals[p] for p in fpos], bw),
        f"{prefix}dense_vals": (np.stack([res_bytes(col, bw) for _, col in A.dense_cols])
                                if A.dense_cols else np.zeros((0, A.nrows, bw), np.uint8)),
    }
    assert np.array_equal(d[f"{prefix}small_vals"].astype(np.int64), A.small_vals)
    return d


def gen_spmv_cases():
    """SpMV cases over the reference's prime set plus the BASELINE widths."""
    rng = np.random.default_rng(20260101)
    primes = [
        7, 1009, 65521, 2**31 - 1, 2**61 - 1, 2**64 - 59, 2**191 - 19,
        2**200 - 75, int(gmpy2.next_prime(2**521)),
        cli.random_prime(160, np.random.default_rng(1)).ell,   # cfg1 width
        cli.random_prime(202, np.random.default_rng(1)).ell,   # cfg3 width
        cli.random_prime(217, np.random.default_rng(1)).ell,   # cfg2 width
        cli.random_prime(256, np.random.default_rng(5)).ell,   # L=8 edge
        cli.random_prime(257, np.random.default_rng(5)).ell,   # L=9 edge
        cli.random_prime(650, np.random.default_rng(1)).ell,   # cfg5 width
    ]
    out = {}
    idx = 0
    for ell in primes:
        mod = PrimeModulus(ell)
        for (nr, nc, per_row, dense, ff) in [(40, 40, 8, 0, 0.1), (33, 47, 12, 2, 0.15),
                                              (64, 64, 30, 1, 0.02)]:
            A = random_matrix(mod, rng, nr, nc, per_row, dense=dense, full_frac=ff)
            u = mod.random_residues(rng, A.total_cols)
            v = spmv_sequential(A, u)
            p = f"c{idx}_"
            out.update(matrix_arrays(p, A))
            out[p + "u"] = res_bytes(u, mod.byte_width)
            out[p + "v"] = res_bytes(v, mod.byte_width)
            idx += 1
        # extreme inputs: u = ell-1 everywhere, coefficients at the small-class
        # boundary (+-(2^31-1)), long rows
        if ell > 2**32:
            rows = []
            for i in range(24):
                row = []
                for c in range(0, 96, 1 + (i % 3)):
                    r = (i * 7 + c) % 5
                    val = [1, ell - 1, 2**31 - 1, ell - (2**31 - 1), ell - 2][r]
                    row.append((c, val))
                rows.append(row)
            A = SparseMatrix.from_rows(mod, 24, 96, rows)
            u = [ell - 1] * 96
            v = spmv_sequential(A, u)
            p = f"c{idx}_"
            out.update(matrix_arrays(p, A))
            out[p + "u"] = res_bytes(u, mod.byte_width)
            out[p + "v"] = res_bytes(v, mod.byte_width)
            idx += 1
    # structural edge cases at a 200-bit modulus
    mod = PrimeModulus(2**200 - 75)
    edge = [
        SparseMatrix.from_rows(mod, 6, 6, [[(i, 1)] for i in range(6)]),      # identity
        SparseMatrix.from_rows(mod, 7, 5, [[] for _ in range(7)]),             # empty rows
        SparseMatrix.from_rows(mod, 5, 9, [[(0, 1), (8, mod.ell - 1)], [], [(3, 12345)],
                                           [(1, mod.ell - 2**31 + 1)], [(2, 5), (4, 2**40)]]),
    ]
    for A in edge:
        u = mod.random_residues(rng, A.total_cols)
        v = spmv_sequential(A, u)
        p = f"c{idx}_"
        out.update(matrix_arrays(p, A))
        out[p + "u"] = res_bytes(u, mod.byte_width)
        out[p + "v"] = res_bytes(v, mod.byte_width)
        idx += 1
    out["ncases"] = np.array(idx)
    return out


def gen_krylov_cases():
    """krylov_block on corpus matrices, unit and dense X, 1..3 chains."""
    out = {}
    idx = 0
    for ell, n, gamma, seed, bp, mode, count in [
        (1009, 50, 5, 3, (1, 1), "dense", 40),
        (2**61 - 1, 50, 5, 12, (3, 6), "unit", 20),
        (2**200 - 75, 80, 6, 44, (2, 4), "unit", 30),
        (2**200 - 75, 60, 5, 10, (2, 4), "dense", 25),
        (cli.random_prime(160, np.random.default_rng(1)).ell, 120, 8, 7, (2, 4), "unit", 50),
    ]:
        mod = PrimeModulus(ell)
        A = generate(CorpusProfile(n=n, gamma=gamma, seed=seed), mod)
        rng = np.random.default_rng(seed + 1000)
        X, Y = draw_blocks(mod, A.nrows, BlockingParams(*bp), rng, mode)
        seq = krylov_block(A, X, Y, count)
        p = f"k{idx}_"
        out.update(matrix_arrays(p, A))
        bw = mod.byte_width
        out[p + "Y"] = np.stack([res_bytes(y, bw) for y in Y])
        out[p + "mode"] = np.array(mode)
        if mode == "unit":
            out[p + "xrows"] = np.array(X.rows, dtype=np.int64)
        else:
            out[p + "xdense"] = np.stack([res_bytes(x, bw) for x in X.vectors])
        # terms[j][i][t]
        out[p + "terms"] = np.stack([
            np.stack([res_bytes(term, bw) for term in col]) for col in seq.columns
        ])
        out[p + "count"] = np.array(count)
        idx += 1
    out["ncases"] = np.array(idx)
    return out


def gen_cfg1():
    """BASELINE configs[0]: `sldlag gen --n 20000 --gamma 20 --ell-bits 160
    --seed 1` (cli.py:236-245), bp=(1,2), unit X from attempt 0's draw
    (solver.py:615-617), a 200-SpMV Krylov chain (krylov_column)."""
    rng = np.random.default_rng(1)
    mod = cli.random_prime(160, rng)
    A = generate(CorpusProfile(n=20000, gamma=20, seed=1), mod)
    bp = BlockingParams(1, 2)
    drng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(0,)))
    X, Y = draw_blocks(mod, A.nrows, bp, drng, "unit")
    seq = krylov_block(A, X, Y, 200)
    out = matrix_arrays("", A)
    bw = mod.byte_width
    out["y"] = res_bytes(Y[0], bw)
    out["xrows"] = np.array(X.rows, dtype=np.int64)
    out["terms"] = np.stack([res_bytes(t, bw) for t in seq.columns[0]])
    # one product and the final iterate (B^200 y), recomputed by the
    # reference SpMV entry point
    planes = vecops.ints_to_planes(Y[0], vecops.digit_count(mod.ell))
    ker = A.kernel()
    v1 = ker.apply(planes)
    out["v1"] = res_bytes(vecops.planes_to_ints(v1), bw)
    v = planes
    for _ in range(200):
        v = ker.apply(v)
    out["v200"] = res_bytes(vecops.planes_to_ints(v), bw)
    return out


def gen_grid_cases():
    """Grid SpMV (gridmv.Grid) on balanced/padded splits, plus the balance
    permutations themselves (balance.py:138-146) and the comm byte log."""
    out = {}
    idx = 0
    for (r, c), ell, n, seed, iters in [
        ((1, 1), 1009, 50, 0, 1), ((2, 1), 1009, 64, 4, 1), ((4, 1), 1009, 64, 4, 2),
        ((2, 2), 1009, 60, 2, 1), ((2, 4), 1009, 64, 4, 1), ((4, 2), 1009, 64, 4, 1),
        ((3, 2), 1009, 64, 4, 1), ((8, 1), 2**200 - 75, 90, 6, 3),
        ((2, 2), 2**200 - 75, 50, 6, 10),
    ]:
        mod = PrimeModulus(ell)
        A = generate(CorpusProfile(n=n, gamma=5, seed=seed), mod)
        g = GridSpec(r, c)
        p = balance_permutation(A, g)
        bs = split(A, p, g)
        B = permuted_padded(A, p, g)
        grid = Grid(bs, mod)
        rng = np.random.default_rng(seed + 5)
        u = mod.random_residues(rng, bs.n_padded)
        grid.load_vector(vecops.ints_to_planes(u, vecops.digit_count(ell)))
        run_iterations(grid, iters)
        got = vecops.planes_to_ints(grid.assembled())
        pre = f"g{idx}_"
        out.update(matrix_arrays(pre, A))
        out.update(matrix_arrays(pre + "B_", B))
        out[pre + "grid"] = np.array([r, c, iters], dtype=np.int64)
        out[pre + "row_perm"] = p.row_perm
        out[pre + "col_perm"] = p.col_perm
        out[pre + "u"] = res_bytes(u, mod.byte_width)
        out[pre + "out"] = res_bytes(got, mod.byte_width)
        out[pre + "comm_bytes"] = np.array([e.total_bytes for e in grid.comm_log.entries],
                                           dtype=np.int64)
        idx += 1
    out["ncases"] = np.array(idx)
    return out


def gen_mksol_cases():
    """Mksol (solver.py:508-565) on generators from the reference's own
    Krylov + Lingen: the kernel vector w, Horner/tail SpMV counts."""
    out = {}
    idx = 0
    for ell, n, gamma, seed, bp in [
        (2**61 - 1, 80, 6, 42, (2, 4)), (2**200 - 75, 90, 6, 7, (2, 4)),
        (cli.random_prime(160, np.random.default_rng(1)).ell, 120, 8, 3, (3, 6)),
        (2**61 - 1, 50, 5, 4, (1, 1)), (1009, 60, 5, 40, (2, 4)),
    ]:
        mod = PrimeModulus(ell)
        A = generate(CorpusProfile(n=n, gamma=gamma, seed=seed), mod)
        rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(0,)))
        bpp = BlockingParams(*bp)
        if bp == (1, 1):
            x = mod.random_residues(rng, n)
            y = mod.random_residues(rng, n)
            F = berlekamp_massey(krylov_scalar(A, x, y), mod)
            polys, Y = [F], [y]
            try:
                kv = mksol_scalar(A, y, F)
            except SolverFailure:
                continue
        else:
            X, Y = draw_blocks(mod, n, bpp, rng, "unit")
            seq = krylov_block(A, X, Y, krylov_length(n, bpp))
            polys = block_lingen(seq, bpp, n, mod, rng).polys
            try:
                kv = mksol_block(A, Y, type("G", (), {"polys": polys})())
            except SolverFailure:
                continue
        pre = f"m{idx}_"
        out.update(matrix_arrays(pre, A))
        bw = mod.byte_width
        out[pre + "Y"] = np.stack([res_bytes(y, bw) for y in Y])
        dmax = max(len(pl) for pl in polys)
        out[pre + "polys"] = np.stack([res_bytes(list(pl) + [0] * (dmax - len(pl)), bw) for pl in polys])
        out[pre + "plen"] = np.array([len(pl) for pl in polys], dtype=np.int64)
        out[pre + "w"] = res_bytes(kv.w, bw)
        out[pre + "counts"] = np.array([kv.horner_spmvs, kv.tail_spmvs, int(kv.verified)], dtype=np.int64)
        idx += 1
    out["ncases"] = np.array(idx)
    return out



def gen_file_cases():
    """SLDM / SLDV / SLDQ files written by the reference (store_matrix,
    store_vector, store_terms) plus hand-framed SLDM files whose tags the
    reference re-classifies on load, and malformed files with the exception
    class the reference raises.  Files go to tests/golden/files/; the npz
    holds what the reference's loaders return for each."""
    import struct
    from sldlag.checkpoint import store_terms
    from sldlag.fileio import FormatError
    from sldlag.spmatrix import load_matrix, store_matrix, store_vector
    fdir = os.path.join(HERE, "files")
    os.makedirs(fdir, exist_ok=True)
    for f in os.listdir(fdir):
        os.unlink(os.path.join(fdir, f))
    d = {}
    mats = [
        ("m200", PrimeModulus(2**200 - 75), 300, 295, 12, 3, 0.1),
        ("m1009", PrimeModulus(1009), 60, 60, 8, 1, 0.1),
        ("m7", PrimeModulus(7), 40, 40, 6, 0, 0.1),
        ("m650", PrimeModulus(int(gmpy2.next_prime(2**649 + 12345))), 80, 78, 10, 2, 0.3),
        ("m61", PrimeModulus(2**61 - 1), 50, 50, 9, 0, 0.2),
    ]
    names = []
    for name, mod, nr, nc, per, dense, ff in mats:
        A = random_matrix(mod, np.random.default_rng(len(name) * 7 + nr), nr, nc, per, dense=dense,
                          full_frac=ff)
        store_matrix(A, os.path.join(fdir, name + ".sldm"))
        d.update(matrix_arrays(name + "_", A))
        names.append(name)
    E = SparseMatrix.from_rows(PrimeModulus(1009), 0, 0, [])
    store_matrix(E, os.path.join(fdir, "empty.sldm"))
    d.update(matrix_arrays("empty_", E))
    names.append("empty")
    # hand-framed rows: +1 stored as small, small stored as full, -2^31 small
    # (-> full), full payload 1 (-> +1), ell-1 as small payload (tiny ell)
    def frame(mod, nrows, ncols, rows):
        eb = mod.byte_width
        out = [b"SLDM", struct.pack("<I", 1), struct.pack("<QQ", nrows, ncols),
               struct.pack("<H", eb), mod.ell.to_bytes(eb, "big"), struct.pack("<I", 0)]
        for r in rows:
            out.append(struct.pack("<I", len(r)))
            prev = 0
            for c, tag, payload in r:
                out.append(struct.pack("<QB", c - prev, tag))
                prev = c
                if tag == 2:
                    out.append(struct.pack("<i", payload))
                elif tag == 3:
                    out.append(int(payload).to_bytes(eb, "little"))
        return b"".join(out)
    M200 = PrimeModulus(2**200 - 75)
    M7 = PrimeModulus(7)
    M199 = PrimeModulus(int(gmpy2.next_prime(2**199)))
    reclass = {
        "rc200": (M200, 3, 10, [[(0, 2, 1), (3, 2, -1), (5, 3, 12345), (9, 2, -2**31)],
                                 [(1, 3, 1), (2, 3, M200.ell - 1), (4, 3, M200.ell - 2**31 + 1),
                                  (8, 3, 2**31 + 5)],
                                 [(0, 0, 0), (7, 1, 0), (9, 3, M200.ell - 2**40)]]),
        "rc7": (M7, 2, 6, [[(0, 2, 6), (1, 2, -6), (2, 2, 13), (5, 3, 3)], [(4, 2, -2**31)]]),
    }
    for name, (mod, nr, nc, rows) in reclass.items():
        with open(os.path.join(fdir, name + ".sldm"), "wb") as f:
            f.write(frame(mod, nr, nc, rows))
        A = load_matrix(os.path.join(fdir, name + ".sldm"))
        d.update(matrix_arrays(name + "_", A))
        names.append(name)
    # malformed files and the reference's verdict
    good = open(os.path.join(fdir, "m1009.sldm"), "rb").read()
    bad = {
        "bad_magic": b"XXXX" + good[4:],
        "bad_trunc": good[:-3],
        "bad_trailing": good + b"\0",
        "bad_version": good[:4] + struct.pack("<I", 2) + good[8:],
        "bad_tag": frame(M7, 1, 4, [[(0, 7, 0)]]),
        "bad_zero": frame(M7, 1, 4, [[(1, 2, 14)]]),
        "bad_zero_full": frame(M7, 1, 4, [[(1, 3, 0)]]),
        "bad_col": frame(M7, 1, 4, [[(5, 0, 0)]]),
        # two errors: the first in file order wins (a zero, then a bad tag)
        "bad_zero_then_tag": frame(M7, 3, 4, [[(1, 2, 14)], [], [(0, 7, 0)]]),
        "bad_tag_then_zero": frame(M7, 3, 4, [[(0, 0, 0)], [(1, 9, 0)], [(1, 2, 7)]]),
        "bad_zero_then_trunc": frame(M7, 5000, 4, [[(1, 0, 0)]] * 4000 + [[(2, 2, 21)]] + [[(0, 0, 0)]] * 999)[:-2],
        "bad_noncanon": frame(M199, 1, 4, [[(1, 3, M199.ell + 2**198)]]),
        "ok_noncanon_small": frame(M200, 1, 4, [[(1, 3, M200.ell + 10)]]),
        "bad_ell": frame(M7, 1, 4, [])[:24] + struct.pack("<H", 1) + bytes([9]) + frame(M7, 1, 4, [])[27:],
    }
    verdicts = []
    for name, blob in bad.items():
        path = os.path.join(fdir, name + ".sldm")
        with open(path, "wb") as f:
            f.write(blob)
        try:
            A = load_matrix(path)
            verdicts.append("ok")
            d.update(matrix_arrays(name + "_", A))
        except FormatError as e:
            verdicts.append(type(e).__name__)
        except ValueError:
            verdicts.append("ValueError")
    d["bad_names"] = np.array(list(bad))
    d["bad_verdicts"] = np.array(verdicts)
    d["matrix_names"] = np.array(names)
    # vectors and terms
    rng = np.random.default_rng(9)
    for name, mod, n in (("v200", M200, 77), ("v7", M7, 5), ("v650", mats[3][1], 33), ("v0", M200, 0)):
        vec = mod.random_residues(rng, n)
        store_vector(vec, mod, os.path.join(fdir, name + ".sldv"))
        d[name + "_ell"] = np.array(hex(mod.ell))
        d[name + "_vals"] = res_bytes(vec, mod.byte_width)
    terms = [M200.random_residues(rng, 4) for _ in range(9)]
    store_terms(os.path.join(fdir, "q200.sldq"), terms, 4, M200)
    d["q200_vals"] = res_bytes([v for t in terms for v in t], M200.byte_width)
    d["q200_m"] = np.array(4)
    # the manifest of every file's bytes
    for f in sorted(os.listdir(fdir)):
        d["sha_" + f] = np.array(hashlib.sha256(open(os.path.join(fdir, f), "rb").read()).hexdigest())
    return d

def main():
    jobs = {
        "spmv_cases.npz": gen_spmv_cases,
        "krylov_cases.npz": gen_krylov_cases,
        "grid_cases.npz": gen_grid_cases,
        "cfg1.npz": gen_cfg1,
        "mksol_cases.npz": gen_mksol_cases,
        "file_cases.npz": gen_file_cases,
    }
    only = sys.argv[1:]
    manifest = []
    for name, fn in jobs.items():
        if only and name not in only:
            continue
        d = fn()
        d["numpy_version"] = np.array(np.__version__)
        path = os.path.join(HERE, name)
        np.savez_compressed(path, **d)
        h = hashlib.sha256(open(path, "rb").read()).hexdigest()
        manifest.append(f"{h}  {name}")
        print(name, os.path.getsize(path), "bytes")
    # refresh the manifest entries that were regenerated
    path = os.path.join(HERE, "SHA256SUMS")
    old = {}
    if os.path.exists(path):
        for line in open(path):
            h, name = line.split()
            old[name] = h
    for line in manifest:
        h, name = line.split()
        old[name] = h
    with open(path, "w") as f:
        f.write("".join(f"{h}  {name}\n" for name, h in sorted(old.items())))


if __name__ == "__main__":
    main()

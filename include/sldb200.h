/*
 * sldb200.h -- C ABI of the B200 Krylov SpMV engine (libsldb200.so).
 *
 * The drop-in boundary for the reference's block-Wiedemann hot path
 * (arxiv/paper_1402_3661, Python package `sldlag`).  The reference has no
 * native code and no FFI; its plugin seam is the duck-typed *multiplier*
 * protocol (`.apply(planes) -> planes`, `.count`, `.size`, `.mod`,
 * sldlag/solver.py:129-163) plus the projection protocol
 * (`.project(planes) -> list[int]`, solver.py:168-189).  Every entry point
 * below replaces one piece of that Python path; the ctypes binding a
 * maintainer adds on the reference side is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Plain C types only; no torch types.  Every function returns 0 on
 *     success or a negative SLD_E* code; sld_last_error() gives a
 *     thread-local message for the last failure on the calling thread.
 *   - Residues cross the ABI either as the reference's "digit planes"
 *     (row-major N x P uint64 cells each holding one little-endian 16-bit
 *     digit, P = ceil(bits(l)/16); sldlag/vecops.py:22-47) or as
 *     little-endian 32-bit limbs (N x L uint32, L = ceil(bits(l)/32)).
 *     Values are canonical residues in [0, l) on both sides; results are
 *     bit-identical to the reference's (integers, not representations).
 *   - Handles are opaque and owned by the caller (free with *_destroy).
 *     One sld_ctx = one CUDA device + one stream; a context must not be
 *     used from two host threads at once (the reference runs one
 *     multiplier per chain thread, solver.py:249-251 -- create one context
 *     per thread/device).  All calls release no locks of their own and are
 *     safe to call with the Python GIL released (ctypes does).
 */
#ifndef SLDB200_H
#define SLDB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLD_OK 0
#define SLD_E_ARG -1     /* bad argument / shape  (reference: ValueError)      */
#define SLD_E_CUDA -2    /* CUDA runtime failure  (reference: n/a)             */
#define SLD_E_BOUND -3   /* exactness bound exceeded (reference: AssertionError,
                            vecops.py:407,414 / ContractViolation modring.py:40) */
#define SLD_E_TIMEOUT -4 /* grid barrier timed out (reference: gridmv.GridTimeoutError) */
#define SLD_E_FORMAT -5  /* malformed file     (reference: fileio.FormatError)    */
#define SLD_E_MAGIC -6   /* wrong magic bytes  (reference: fileio.BadMagic)       */
#define SLD_E_TRUNC -7   /* file ends early    (reference: fileio.TruncatedFile)  */
#define SLD_E_PROTOCOL -8 /* stale grid iteration (reference: gridmv.GridProtocolError) */

typedef struct sld_ctx sld_ctx;
typedef struct sld_mat sld_mat;
typedef struct sld_vec sld_vec;

/* library / error plumbing */
int sld_version(void);
const char *sld_last_error(void);
int sld_device_count(int *out);
/* Which die each SM of `device` sits on (B200 is two dies, and each die's
 * L2 caches what its own SMs read).  map256[smid] = 0/1; n_die0/n_die1 = SMs
 * per die.  Probed once per device and process from cold-line latencies.
 * Returns SLD_E_CUDA (map all zero) when the probe is ambiguous. */
int sld_die_map(int device, uint8_t *map256, int *n_die0, int *n_die1);

/*
 * Field context: one prime l on one device.  Replaces PrimeModulus as the
 * object that crosses every API (sldlag/modring.py:44-130).  ell_limbs: the
 * prime as L little-endian 32-bit words (l odd, 3 <= l, bits(l) <= 1024).
 */
int sld_ctx_create(int device, const uint32_t *ell_limbs, int L, sld_ctx **out);
int sld_ctx_destroy(sld_ctx *ctx);
int sld_ctx_sync(sld_ctx *ctx);
/* Run this context's work on an external CUDA stream (e.g. torch's current
 * stream, so NCCL collectives order with our kernels); 0 restores the
 * context's own stream. */
int sld_ctx_set_stream(sld_ctx *ctx, uint64_t cuda_stream);

/*
 * Matrix upload + GPU layout build.  Replaces SparseMatrix.kernel() /
 * SpmvKernel.__init__ (sldlag/spmatrix.py:205-230, vecops.py:366-414).
 * Inputs mirror the SparseMatrix fields (spmatrix.py:77-91):
 *   row_ptr[nrows+1] (int64), col_idx[nnz] (int32 sparse column < ncols),
 *   tags[nnz] (0:+1, 1:-1, 2:small, 3:full -- modring.py:26-29),
 *   small_vals[nnz] (int64; read for tag 2; |c| >= 2^31 is promoted to the
 *   full class, value c mod l, exactly the "smallest class" rule of
 *   spmatrix.py:48-66 run in reverse),
 *   n_full entries at sorted flat positions full_pos[] with values
 *   full_limbs[n_full*L] (canonical), and n_dense dense columns
 *   dense_limbs[n_dense*nrows*L] occupying global columns ncols..ncols+n_dense-1
 *   (spmatrix.py:69-75; zero entries allowed).
 * max_stripe_cols: column-stripe width for L2 residency of the gathered
 *   vector (0 = automatic, from the device's L2 size).
 * Errors: SLD_E_ARG for inconsistent CSR (spmatrix.py:93-126 checks),
 * SLD_E_BOUND if a row has more than 2^15 small-class or 2^18 +-1 entries.
 */
int sld_mat_create(sld_ctx *ctx, int64_t nrows, int64_t ncols,
                   const int64_t *row_ptr, const int32_t *col_idx,
                   const uint8_t *tags, const int64_t *small_vals,
                   int64_t n_full, const int64_t *full_pos, const uint32_t *full_limbs,
                   int n_dense, const uint32_t *dense_limbs,
                   int64_t max_stripe_cols, sld_mat **out);
/* Same, laid out for `chains` (1, 2 or 4) interleaved Krylov chains that
 * share every pass over the matrix: block Wiedemann's independent sequences
 * (solver.py:220-257) multiplied together, each gather request fetching the
 * residues of all G chains of a column (G * 32 bytes <= one 128-byte line). */
int sld_mat_create_chains(sld_ctx *ctx, int chains, int64_t nrows, int64_t ncols,
                          const int64_t *row_ptr, const int32_t *col_idx,
                          const uint8_t *tags, const int64_t *small_vals,
                          int64_t n_full, const int64_t *full_pos, const uint32_t *full_limbs,
                          int n_dense, const uint32_t *dense_limbs,
                          int64_t max_stripe_cols, sld_mat **out);
int sld_mat_destroy(sld_mat *m);
/* info[0..19]: nrows, total_cols, nnz, n_pm, n_small, n_full(+dense nz),
 * stripes, nslices, device bytes, padded index entries, L, stride words,
 * max row degree, stripe columns, chains, halves (2 = columns dealt to
 * the two dies, see sld_die_map), lanes per residue (limb-sliced passes:
 * SW/8, else 1), rows per slice, index prefetch distance, 0 */
int sld_mat_info(const sld_mat *m, int64_t *info);

/*
 * Device vectors of `n` residues (n = total_cols of the matrices they feed).
 * Upload/download accept the reference's digit planes (vecops.py:35-47) or
 * 32-bit limbs; planes are repacked on the device.
 */
int sld_vec_create(sld_ctx *ctx, int64_t n, sld_vec **out);
/* A vector of `chains` interleaved residue vectors of n each (for matrices
 * built with sld_mat_create_chains).  Host arrays of such vectors are
 * chain-major: chains x n x (P or L). */
int sld_vec_create_chains(sld_ctx *ctx, int64_t n, int chains, sld_vec **out);
int sld_vec_destroy(sld_vec *v);
int sld_vec_upload_planes(sld_vec *v, const uint64_t *planes, int64_t n, int P);
int sld_vec_download_planes(sld_vec *v, uint64_t *planes, int64_t n, int P);
/* The same for a vector of `chains` interleaved chains whose host planes are
 * separate arrays (planes[g] = chain g, n x P each): no host-side stacking. */
int sld_vec_upload_planes_chains(sld_vec *v, const uint64_t *const *planes, int64_t n, int P);
int sld_vec_download_planes_chains(sld_vec *v, uint64_t *const *planes, int64_t n, int P);
int sld_vec_upload_limbs(sld_vec *v, const uint32_t *limbs, int64_t n);
int sld_vec_download_limbs(sld_vec *v, uint32_t *limbs, int64_t n);
/* raw device pointer + stride (words) -- for collectives and tests */
int sld_vec_device_ptr(sld_vec *v, uint64_t *ptr, int64_t *stride_words);

/*
 * dst = (src_0 + ... + src_{k-1}) mod l over n residues in the device slot
 * format (sld_vec_device_ptr), 1 <= k <= 64.  Replaces planes_add_mod
 * (vecops.py:261-264) -- the grid's reduce phase (gridmv.py:291-294) and
 * the Mksol combination (solver.py:530-536).  Raw device pointers passed as
 * uint64; dst may alias src_0.
 */
int sld_add_mod(sld_ctx *ctx, const uint64_t *src_ptrs, int k, uint64_t dst_ptr, int64_t n);

/*
 * dst = acc + sum_j coeffs_j * y_j (mod l) over n residues in the slot
 * format (raw device pointers; acc_ptr may be 0; k <= 64 canonical
 * coefficients as k x L limbs).  The Horner combination of Mksol
 * (solver.py:522-536: planes_scalar_mul_mod + planes_add_mod).
 */
int sld_lincomb(sld_ctx *ctx, const uint64_t *y_ptrs, const uint32_t *coeffs, int k,
                uint64_t acc_ptr, uint64_t dst_ptr, int64_t n);
/* Mksol's combination on the tensor cores (ell < 2^256, n <= 8 vectors):
 * the y block is tiled once as byte digits; each apply computes
 * dst = acc + sum_s coeffs[s] y_s mod ell (coeffs n x L limbs; acc may be
 * 0) as a u8 digit GEMM (tcgen05 kind::i8) with the modular reduction in
 * the epilogue.  SLD_E_ARG for a modulus of more than 8 limbs or n > 8. */
typedef struct sld_lcset sld_lcset;
int sld_lcset_create(sld_ctx *ctx, const uint64_t *y_ptrs, int n, int64_t rows, sld_lcset **out);
int sld_lcset_apply(sld_lcset *s, const uint32_t *coeffs, uint64_t acc_ptr, uint64_t dst_ptr);
/* The combinations of K = 2 or 4 Horner steps in one pass over the tiled y
 * (the y are fixed for a Mksol run, only the coefficients change): dst_k =
 * sum_s coeffs[k][s] y_s mod ell, coeffs K x n x L canonical limbs,
 * dst_ptrs[k] device vectors of `rows` residues.  Asynchronous. */
int sld_lcset_apply_batch(sld_lcset *s, const uint32_t *coeffs, int K, const uint64_t *dst_ptrs);
/* The set tiled in matrix m's slot order (one chain, pass layout): its
 * combinations are slot-ordered vectors of nslots residues, the addv operand
 * of sld_spmv_add. */
int sld_lcset_create_slots(sld_mat *m, const uint64_t *y_ptrs, int n, sld_lcset **out);
int sld_lcset_destroy(sld_lcset *s);

/* *out = 1 if any residue of v is non-zero (np.any(planes), solver.py:545). */
int sld_vec_nonzero(sld_vec *v, int *out);

/* Read m residues (rows[t] of the vector) as canonical limbs (m x L). */
int sld_vec_read_rows(sld_vec *v, const int64_t *rows, int m, uint32_t *limbs);

/*
 * out = A * in (mod l), canonical.  Replaces SpmvKernel.apply
 * (vecops.py:428-470) and spmv_planes (spmatrix.py:242-246); `in` must
 * have total_cols residues and `out` nrows residues (and be distinct).
 */
int sld_spmv(sld_mat *m, sld_vec *in, sld_vec *out);
/* sld_spmv without the final stream synchronize (errors surface at the next
 * synchronizing call). */
int sld_spmv_async(sld_mat *m, sld_vec *in, sld_vec *out);

/* Host-buffer convenience: planes in, planes out (the multiplier's
 * `.apply(planes)` contract, solver.py:140-142). */
int sld_spmv_planes(sld_mat *m, const uint64_t *in_planes, uint64_t *out_planes, int P);

/*
 * Device-resident Krylov chain.  Replaces the loop of krylov_column
 * (solver.py:199-217) with UnitRows projections (solver.py:174-176):
 * for i in [0, steps): terms[i] = X^T v; v = A v.
 *   v: in/out iterate (total_cols == nrows, square matrix).
 *   x_rows[m]: unit projection rows.  terms_limbs: steps*G*m*L uint32
 *   (host; G = the matrix's chains), step i / chain g / row t at
 *   ((i*G + g)*m + t)*L.
 * Steps run as CUDA-graph chunks; the call returns after `steps` products.
 */
int sld_krylov_unit(sld_mat *m, sld_vec *v, const int64_t *x_rows, int mrows,
                    int64_t steps, uint32_t *terms_limbs);

/*
 * Same with a dense X block (DenseRows.project, solver.py:186-189):
 * x: an (mrows x total_cols) set of residues uploaded once with
 * sld_xblock_create; terms[i][t] = sum_j x[t][j] v_i[j] mod l.
 */
typedef struct sld_xblock sld_xblock;
int sld_xblock_create(sld_ctx *ctx, const uint32_t *x_limbs, int mrows, int64_t n, sld_xblock **out);
int sld_xblock_destroy(sld_xblock *x);
int sld_krylov_dense(sld_mat *m, sld_vec *v, sld_xblock *x, int64_t steps, uint32_t *terms_limbs);

/*
 * Mksol Horner step fused into one product (sldlag/solver.py:522-536,
 * planes_scalar_mul_mod + planes_add_mod of vecops.py:261-278):
 * sld_mat_mksol_bind copies n <= 8 y vectors into the matrix's slot order
 * (n = 0 releases them); sld_spmv_mksol then computes
 * out = A in + sum_s coeffs[s] y_s mod l (coeffs: n x L canonical limbs),
 * the combination in the last pass's epilogue.  Needs L <= 8 and the
 * one-chain pass layout (SLD_E_ARG otherwise).  Asynchronous.
 */
int sld_mat_mksol_bind(sld_mat *m, sld_vec *const *ys, int n);
int sld_spmv_mksol(sld_mat *m, sld_vec *in, sld_vec *out, const uint32_t *coeffs);
/* The Horner step with its combination precomputed (sld_lcset_apply_batch):
 * out = A in + addv (mod l), the addition in the last pass's epilogue
 * (the reference's planes_add_mod, vecops.py:270-278); addv in m's slot
 * order (sld_lcset_create_slots), nslots residues.  L <= 8, one chain,
 * pass or short-row layout (SLD_E_ARG otherwise).  Asynchronous. */
int sld_spmv_add(sld_mat *m, sld_vec *in, sld_vec *out, sld_vec *addv);

/*
 * Timing hook for bench.py: runs `steps` products v <- A v on device
 * (ping-pong, graph-captured) and returns device milliseconds measured
 * with CUDA events on the context stream; kernel_ms gets the average
 * duration of one product (all stripe passes).
 */
int sld_bench_spmv(sld_mat *m, sld_vec *v, int64_t steps, int warmup, double *total_ms,
                   double *kernel_ms);

/* As sld_bench_spmv, with per-sample durations for a median: an event is
 * recorded after every `pairs_per_sample` product pairs, and sample_ms
 * (ceil(ceil(steps/2) / pairs_per_sample) entries) receives the duration
 * of each sample.  sample_ms = NULL behaves as sld_bench_spmv. */
int sld_bench_spmv_samples(sld_mat *m, sld_vec *v, int64_t steps, int warmup, int64_t pairs_per_sample,
                           double *sample_ms, double *total_ms, double *kernel_ms);

/* Synthetic corpus generator (fixture producer, not timed): a native
 * restatement of the row/column distribution of sldlag/corpus.py:104-139
 * (row weight rint(N(gamma, 0.1 gamma)) clipped to [3, ncols/2], column j
 * with probability ~ (j+1)^-decay, distinct sorted columns, +-1 with
 * probability pm1, else a small coefficient of magnitude uniform in
 * [2, cmax) with random sign).  Two-phase: count (row_ptr) then fill. */
int sld_corpus_rows(int64_t n, int64_t ncols, double gamma, uint64_t seed, int64_t *row_ptr);
int sld_corpus_fill(int64_t n, int64_t ncols, double decay, double pm1, int64_t cmax,
                    uint64_t seed, const int64_t *row_ptr, int32_t *col_idx, uint8_t *tags,
                    int64_t *small_vals, int nthreads);

/*
 * Grid partition builder (host code): block (bi, bj) of the r x c split of
 * B = P_r A P_c^T -- replaces sldlag/balance.py split (201-242) and
 * permuted_padded (245-267, the r = c = 1 case).  Entries are A's CSR
 * (index k < nnz; col_idx of col_bytes 4 or 8) followed by n_extra entries
 * given in permuted coordinates (dense-column nonzeros, then the pinned +1
 * padding; index nnz + e).  Pass 1 (src == NULL) fills rp[0..n_pad/r] and
 * returns the block's entry count; pass 2 fills src[] and lc[] (local
 * column), each local row ordered by (lc, src).  threads <= 0: all cores.
 */
int64_t sld_split_block(int64_t nrows, const int64_t *row_ptr, const void *col_idx, int col_bytes,
                        const int64_t *row_perm, const int64_t *col_perm, int64_t n_extra,
                        const int64_t *extra_r, const int64_t *extra_c, int64_t n_pad, int32_t r,
                        int32_t c, int32_t bi, int32_t bj, int64_t *rp, int64_t *src, int32_t *lc,
                        int32_t threads);

/*
 * Native file formats of the reference (host code, no device needed).
 *
 * SLDM matrix (sldlag/spmatrix.py:14-22, store_matrix/load_matrix 358-436).
 * sld_sldm_info scans the file (header_only: stops after the modulus, which
 * the caller validates first, like the reference): info[0..7] = nrows, ncols, ell byte width,
 * dense column count, nnz, full-class entries after re-classification, file
 * bytes, ell limbs; ell_be receives the modulus big-endian (ell_cap >= width).
 * sld_sldm_read fills the CSR arrays of SparseMatrix (row_ptr[nrows+1],
 * col_idx[nnz], tags[nnz], small_vals[nnz], full_pos/full_limbs[n_full][L],
 * dense_idx[dc], dense_limbs[dc][nrows][L]) re-classifying each coefficient
 * to its smallest class like load_matrix.  sld_sldm_write emits the
 * reference's exact bytes (atomic temp + fsync + rename).
 */
int sld_sldm_info(const char *path, int header_only, int64_t *info, uint8_t *ell_be, int ell_cap);
int sld_sldm_read(const char *path, int L, int64_t *row_ptr, int32_t *col_idx, uint8_t *tags,
                  int64_t *small_vals, int64_t *full_pos, uint32_t *full_limbs,
                  int64_t *dense_idx, uint32_t *dense_limbs);
int sld_sldm_write(const char *path, int64_t nrows, int64_t ncols, const uint32_t *ell, int L,
                   const int64_t *row_ptr, const int32_t *col_idx, const uint8_t *tags,
                   const int64_t *small_vals, int64_t n_full, const int64_t *full_pos,
                   const uint32_t *full_limbs, int n_dense, const int64_t *dense_idx,
                   const uint32_t *dense_limbs);
/*
 * SLDV vector (kind 0; spmatrix.py:24-25, store_vector/load_vector 439-462)
 * and SLDQ Krylov terms (kind 1; checkpoint.py:11-14, store_terms/load_terms
 * 36-64: count x m residues).  Residues cross as `stride` 32-bit limbs each.
 * info[0..5] = kind, ell byte width, ell limbs, m (1 for SLDV), count,
 * residues.
 */
int sld_sldv_write(const char *path, int kind, const uint32_t *ell, int L, int64_t m, int64_t count,
                   const uint32_t *limbs, int stride);
int sld_sldv_info(const char *path, int header_only, int64_t *info, uint8_t *ell_be, int ell_cap);
int sld_sldv_read(const char *path, uint32_t *limbs, int stride);



/*
 * Native grid node: one Krylov chain over an r x c grid (r*c <= 8 nodes),
 * replacing the reference's Grid (gridmv.py:193-354: _one_iteration,
 * apply_once, the collector rule and its failure detection, 46-51).  Every
 * exchange runs over peer memory: the block's SpMV pushes its output (r x 1:
 * rows of every node's next iterate; r x c: the partial into the row
 * collector's inbox), the collector reduces (add_mod) and scatters the row
 * piece with one copy kernel, flag barriers order the phases.  Each
 * iteration is a replayed CUDA graph: no host synchronisation, no
 * collective.  Setup only: every node publishes a SLD_GRID_BLOB-byte record
 * (sld_grid_blob; CUDA IPC handle + pointer) and connects to all records in
 * rank order (sld_grid_connect) -- the records travel over any host
 * transport.  Nodes may share a process (raw pointers, peer access enabled)
 * or not (IPC).
 *
 *  sld_grid_create   block = A_ij of the balanced padded matrix as an
 *                    sld_mat (br x bc, one chain, <= 8 limbs); not owned
 *  sld_grid_load/read this node's fragment u_j (bc x L limbs; r x 1: the
 *                    whole padded iterate)
 *  sld_grid_set_projection  unit-X rows (global padded indices, m <= 32):
 *                    each iteration records the rows of its INPUT fragment
 *                    that this node reports (row-0 nodes, owned[t] = 1)
 *                    into a device ring of max_steps; sld_grid_terms drains
 *                    it as [steps][m][L] limbs (0 where not owned)
 *  sld_grid_launch   enqueue count iterations (asynchronous)
 *  sld_grid_wait     synchronise; SLD_E_TIMEOUT if a barrier saw no progress
 *                    for the timeout (default 30 s; a node stopped),
 *                    SLD_E_PROTOCOL if a node published an iteration other
 *                    than this one or the next (stale or restarted node)
 *  sld_grid_set_epoch resume: all nodes at the same completed iteration
 *  sld_grid_info     [iteration, nodes, br, bc, collector, bytes, parity,
 *                    kernels per iteration]
 */
#define SLD_GRID_BLOB 128
typedef struct sld_grid sld_grid;
int sld_grid_create(sld_mat *block, int r, int c, int rank, int64_t n_padded, sld_grid **out);
int sld_grid_blob(sld_grid *g, uint8_t *blob);
int sld_grid_connect(sld_grid *g, const uint8_t *blobs);
int sld_grid_set_timeout(sld_grid *g, double seconds);
int sld_grid_set_projection(sld_grid *g, const int64_t *rows, int m, int64_t max_steps, uint8_t *owned);
int sld_grid_load(sld_grid *g, const uint32_t *limbs);
int sld_grid_read(sld_grid *g, uint32_t *limbs);
int sld_grid_launch(sld_grid *g, int64_t count);
int sld_grid_wait(sld_grid *g);
int sld_grid_iterate(sld_grid *g, int64_t count);
int sld_grid_terms(sld_grid *g, uint32_t *terms, int64_t *steps);
int sld_grid_set_epoch(sld_grid *g, int64_t epoch);
int sld_grid_info(sld_grid *g, int64_t *info);
int sld_grid_destroy(sld_grid *g);

#ifdef __cplusplus
}
#endif
#endif /* SLDB200_H */

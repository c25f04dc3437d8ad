// sld_tcgemm.cuh -- exact u8 x u8 -> s32 digit GEMM on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM), for the
// dense-X projection a_t = sum_j x_t[j] v[j] mod ell (solver.py:179-189):
// with x_t[j] = sum_p x_{t,p} 2^(8p) and v[j] = sum_q v_q 2^(8q) (bytes),
//     a_t = sum_{p,q} 2^(8(p+q)) D[32 t + p][q],  D = X8 . V8^T  (K = N).
// A = X8 (32 m rows, fixed), B = V8 (32 rows, per step), both K-major.
//
// Operands live in HBM pre-tiled in the UMMA canonical K-major
// no-swizzle layout, so each pipeline stage is ONE contiguous 1-D bulk copy
// (cp.async.bulk + mbarrier complete_tx, no tensor maps):
//   tile(kt) = [mt][ks][mg][kc][8 rows][16 bytes]
// kt: 128-byte K tile, mt: 128-row M tile, ks: 32-byte UMMA_K step,
// mg: 8-row group, kc: 16-byte K chunk.  Descriptor: LBO = 128 B (kc),
// SBO = 256 B (mg).  Split-K: CTA c owns a K range of <= 32768 bytes, so a
// u8 x u8 sum (<= 255^2 = 65025 per term) stays below 32768 * 65025 < 2^31:
// the s32 accumulator never wraps (exactness does not lean on wrap-around);
// the per-CTA tiles are summed in 64 bits afterwards.
#pragma once
#include <cstdint>

namespace sld {

constexpr int TC_BK = 128;          // K bytes per stage
constexpr int TC_NQ = 32;           // B rows (bytes of a residue, <= 32)
constexpr int TC_STAGES = 3;
constexpr int TC_MTILE_BYTES = 128 * TC_BK;       // 16 KB
constexpr int TC_BTILE_BYTES = TC_NQ * TC_BK;     // 4 KB
constexpr int TC_THREADS = 192;                   // w0 loads, w1 MMA, w2-5 epilogue
constexpr int64_t TC_MAX_K_PER_CTA = 32768;
static_assert(TC_MAX_K_PER_CTA * 65025 < (1ll << 31), "s32 TMEM accumulator must not wrap");

__host__ __device__ constexpr int tc_smem_bytes(int MT) {
  return TC_STAGES * (MT * TC_MTILE_BYTES + TC_BTILE_BYTES) + 1024;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(done)
                 : "r"(smem_u32(b)), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// K-major, no swizzle: LBO = 128 B between the two 16-byte K chunks, SBO =
// 256 B between 8-row groups; version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
// kind::i8: D s32 (c_format 2), A/B unsigned 8-bit, both K-major, N = 32, M = 128
constexpr uint32_t TC_IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TC_NQ >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

// partial[cta][MT*128][32] = u32 sums of this CTA's K range
template <int MT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_digit_gemm(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B, int64_t ktiles,
                  int64_t kt_per_cta, uint32_t* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t A_STAGE = MT * TC_MTILE_BYTES;
  constexpr uint32_t STAGE = A_STAGE + TC_BTILE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* done = empty + TC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  constexpr uint32_t TCOLS = MT * TC_NQ <= 32 ? 32 : (MT * TC_NQ <= 64 ? 64 : 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t kt0 = (int64_t)blockIdx.x * kt_per_cta;
  const int64_t nk = kt0 < ktiles ? min(kt_per_cta, ktiles - kt0) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; s++) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // producer: one bulk copy per operand tile per stage
    for (int64_t i = 0; i < nk; i++) {
      const int s = (int)(i % TC_STAGES);
      if (i >= TC_STAGES) mbar_wait(empty + s, (uint32_t)((i / TC_STAGES - 1) & 1));
      uint8_t* sa = smem + s * STAGE;
      mbar_expect_tx(full + s, STAGE);
      bulk_g2s(sa, A + (size_t)(kt0 + i) * A_STAGE, A_STAGE, full + s);
      bulk_g2s(sa + A_STAGE, B + (size_t)(kt0 + i) * TC_BTILE_BYTES, TC_BTILE_BYTES, full + s);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: 4 K steps x MT tiles per stage, accumulators in TMEM
    for (int64_t i = 0; i < nk; i++) {
      const int s = (int)(i % TC_STAGES);
      mbar_wait(full + s, (uint32_t)((i / TC_STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sa = smem + s * STAGE;
      const uint8_t* sb = sa + A_STAGE;
#pragma unroll
      for (int ks = 0; ks < TC_BK / 32; ks++) {
        const uint64_t bd = umma_desc(sb + ks * (TC_NQ * 32));
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
          umma_i8(tmem + mt * TC_NQ, umma_desc(sa + mt * TC_MTILE_BYTES + ks * (128 * 32)), bd,
                  (i > 0 || ks > 0) ? 1u : 0u);
      }
      umma_commit(empty + s);
    }
    umma_commit(done);
  } else if (warp >= 2) {
    // epilogue: TMEM lanes (warp % 4) * 32 .. + 31 -> registers -> HBM
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    if (nk > 0) {
      mbar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#pragma unroll 1
    for (int mt = 0; mt < MT; mt++) {
      uint32_t r[32];
      if (nk > 0) {
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(mt * TC_NQ);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int q = 0; q < 32; q++) r[q] = 0;
      }
      uint4* dst = reinterpret_cast<uint4*>(partial + (((size_t)blockIdx.x * MT + mt) * 128 + row) * TC_NQ);
#pragma unroll
      for (int q = 0; q < 8; q++) dst[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// Digit tiling through shared memory: the 32 digit bytes of a residue are
// just its limb words (little-endian), so a block stages the residues of one
// 128-byte K tile as [j][32 bytes] and writes the tile transposed, one
// 128-byte core matrix (8 digit rows x 16 residues) per thread.
// Tile byte (core c = ks*8 + mg*2 + kc, row rr, byte jj) = digit mg*8 + rr of
// residue ks*32 + kc*16 + jj.

// v (biased slots, one chain) -> B tiles: one block of 128 threads per K tile
template <int L>
__global__ void __launch_bounds__(128) tc_tile_v(const uint32_t* __restrict__ v, int64_t n, int64_t ktiles,
                                                 uint8_t* __restrict__ B) {
  constexpr int SW = stride_words(L);
  __shared__ uint32_t S[128][9];  // [residue][limb word], padded against bank conflicts
  const int64_t kt = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t j = kt * TC_BK + t;
#pragma unroll
  for (int i = 0; i < 8; i++) S[t][i] = (j < n && i < L) ? (v[(size_t)j * SW + i] ^ 0x80000000u) : 0u;
  __syncthreads();
  if (t >= 32) return;  // 32 core matrices per B tile
  const int ks = t >> 3, mg = (t >> 1) & 3, kc = t & 1;
  uint32_t o[32];
#pragma unroll
  for (int rr = 0; rr < 8; rr++) {
    const int q = mg * 8 + rr;
#pragma unroll
    for (int w4 = 0; w4 < 4; w4++) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int jl = ks * 32 + kc * 16 + w4 * 4 + b;
        word |= ((S[jl][q >> 2] >> (8 * (q & 3))) & 0xFFu) << (8 * b);
      }
      o[rr * 4 + w4] = word;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(B + ((size_t)kt * 32 + t) * 128);
#pragma unroll
  for (int i = 0; i < 8; i++) dst[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
}

// X (m vectors of n residues, plain canonical limbs, SW stride) -> A tiles:
// one block of 128 threads per (K tile, M tile); the M tile holds the 32
// digit rows of 4 consecutive terms
template <int L>
__global__ void __launch_bounds__(128) tc_tile_x(const uint32_t* __restrict__ x, int m, int64_t n, int MT,
                                                 int64_t ktiles, uint8_t* __restrict__ A) {
  constexpr int SW = stride_words(L);
  __shared__ uint32_t S[4][128][9];
  const int64_t kt = blockIdx.x / MT;
  const int mt = (int)(blockIdx.x % MT);
  const int t = threadIdx.x;
  const int64_t j = kt * TC_BK + t;
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int term = mt * 4 + u;
#pragma unroll
    for (int i = 0; i < 8; i++)
      S[u][t][i] = (term < m && j < n && i < L) ? x[((size_t)term * n + j) * SW + i] : 0u;
  }
  __syncthreads();
  // 128 core matrices per M tile: c = ks*32 + mg*2 + kc, mg = 0..15
  const int ks = t >> 5, mg = (t >> 1) & 15, kc = t & 1;
  uint32_t o[32];
#pragma unroll
  for (int rr = 0; rr < 8; rr++) {
    const int r = mg * 8 + rr;       // row in the M tile
    const int u = r >> 5, p = r & 31;  // term in the tile, digit
#pragma unroll
    for (int w4 = 0; w4 < 4; w4++) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int jl = ks * 32 + kc * 16 + w4 * 4 + b;
        word |= ((S[u][jl][p >> 2] >> (8 * (p & 3))) & 0xFFu) << (8 * b);
      }
      o[rr * 4 + w4] = word;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(A + (((size_t)kt * MT + mt) * 128 + t) * 128);
#pragma unroll
  for (int i = 0; i < 8; i++) dst[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
}

constexpr int TC_FOLD_TOP = 19;  // limbs of sum_j x v < 2^31 ell^2 (ell < 2^256): <= 18

// a_t from the per-CTA digit products: one block of 1024 threads per term
template <int L>
__global__ void __launch_bounds__(1024) tc_proj_final(const uint32_t* __restrict__ partial, int nct, int MT,
                                                      const uint32_t* __restrict__ fold, const ModParams mp,
                                                      uint32_t* __restrict__ out) {
  constexpr int SW = stride_words(L);
  __shared__ unsigned long long col8[64];
  const int t = blockIdx.x;
  const int p = threadIdx.x >> 5, q = threadIdx.x & 31;
  if (threadIdx.x < 64) col8[threadIdx.x] = 0;
  __syncthreads();
  const int r = t * 32 + p;  // row of A
  const int mt = r >> 7, rr = r & 127;
  uint64_t s = 0;
  for (int c = 0; c < nct; c++) s += partial[(((size_t)c * MT + mt) * 128 + rr) * TC_NQ + q];
  if (s) atomicAdd(&col8[p + q], (unsigned long long)s);
  __syncthreads();
  if (threadIdx.x != 0) return;
  // bytes -> 32-bit limbs
  uint32_t V[TC_FOLD_TOP + 1];
#pragma unroll
  for (int k = 0; k <= TC_FOLD_TOP; k++) V[k] = 0;
  uint64_t carry = 0;
  for (int b = 0; b < 4 * (TC_FOLD_TOP + 1); b++) {
    const uint64_t v = carry + (b < 64 ? col8[b] : 0ull);
    V[b >> 2] |= (uint32_t)(v & 0xFF) << (8 * (b & 3));
    carry = v >> 8;
  }
  int64_t acc[L + 1];
#pragma unroll
  for (int i = 0; i < L; i++) acc[i] = V[i];
  acc[L] = 0;
  for (int k = L; k <= TC_FOLD_TOP; k++) {
    const uint32_t limb = V[k];
    if (!limb) continue;
    const uint32_t* R = fold + (size_t)(k - L) * L;
#pragma unroll
    for (int i = 0; i < L; i++) {
      const uint64_t pr = (uint64_t)limb * R[i];
      acc[i] += (int64_t)(uint32_t)pr;
      acc[i + 1] += (int64_t)(pr >> 32);
    }
  }
  uint32_t Rr[L];
  finalize<L>(acc, 0, mp, Rr);
#pragma unroll
  for (int i = 0; i < SW; i++) out[(size_t)t * SW + i] = i < L ? Rr[i] : 0u;
}

// ------------------------------------------------------------------------
// Mksol's combination on the tensor cores (solver.py:522-536):
//     w[i] = acc[i] + sum_s c_s y_s[i]  mod ell,  s < n <= 8.
// With bytes y_s[i] = sum_q Y_{s,q} 2^(8q) and c_s = sum_p C_{s,p} 2^(8p):
//     sum_s c_s y_s[i] = sum_k 2^(8k) D[i][k],
//     D = Y' . C'^T,  Y'[i][(s,q)] = Y_{s,q}[i],  C'[k][(s,q)] = C_{s,k-q}.
// M = rows i (128 per tile), N = 64 byte positions k, K = 32 n.  Every D
// entry is < 256 * 255^2 < 2^24.  The epilogue reads its row's 64 columns
// from TMEM, carries them into limbs, folds the limbs above L with
// 2^(32k) mod ell, adds acc, and runs finalize: w is written once, never
// staged.  Y' (the n fixed vectors) is tiled once per Mksol run; C'
// (n x 2 KB) is expanded in shared memory from the step's coefficients.
//
// Batched (K > 1): the combinations of K Horner steps at once.  The y are
// fixed for the whole Mksol run and only the coefficients change per step,
// so one pass over Y' (n x 115 MB at cfg3, the dominant traffic) feeds K
// accumulators: K C' tiles in shared memory, K x 64 TMEM columns per
// buffer, K outputs per tile.  Per step the traffic drops from
// (n + 2) vectors to n / K + 1.
constexpr int TCL_N = 64;                       // byte positions k of the products
constexpr uint32_t TCL_IDESC = (2u << 4) | ((uint32_t)(TCL_N >> 3) << 17) | ((128u >> 4) << 24);
constexpr int TCL_THREADS = 192;
// epilogue warps per TMEM lane quarter: the batched kernel's K reductions
// per row are split over two warps of each quarter (more epilogue warps per
// SM: it runs one CTA per SM)
__host__ __device__ constexpr int tcl_epi(int K) { return K == 1 ? 1 : (K == 2 ? 2 : 4); }
__host__ __device__ constexpr int tcl_threads(int K) { return 64 + 128 * tcl_epi(K); }
#ifndef TCL_CTAS_PER_SM
#define TCL_CTAS_PER_SM 2  // two CTAs per SM: twice the epilogue warps (smem 2 x ~113 KB, TMEM 2 x 128 cols)
#endif
constexpr int TCL_KMAX = 4;  // Horner steps per batched combination

// Y' pipeline stages: 3 for one step, 2 when K C' tiles share the smem
__host__ __device__ constexpr int tcl_stages(int K) { return K == 1 ? 3 : 2; }
__host__ __device__ constexpr int tcl_ytile_bytes(int n) { return 128 * 32 * n; }
__host__ __device__ constexpr int tcl_b_bytes(int n) { return TCL_N * 32 * n; }
__host__ __device__ constexpr int tcl_smem_bytes(int n, int K = 1) {
  return tcl_stages(K) * tcl_ytile_bytes(n) + K * tcl_b_bytes(n) + 1024;
}
// TMEM columns: two accumulator buffers of K x 64 columns (a power of 2 >= 32)
__host__ __device__ constexpr uint32_t tcl_tmem_cols(int K) { return K == 1 ? 128u : (K == 2 ? 256u : 512u); }

// y_s (biased slots) -> Y' tiles: tile mt = [s][mg][kc][8 rows][16 bytes];
// one thread per 128-byte core matrix (the 16 bytes of a row are 4 limb words)
// perm (optional): tile row i holds row perm[i] of the y (-1: zero), so the
// combinations come out in a matrix's slot order
template <int L>
__global__ void tcl_tile_y(const uint32_t* const* __restrict__ ys, int n, int64_t rows, int64_t mtiles,
                           uint8_t* __restrict__ Y, const int32_t* __restrict__ perm) {
  constexpr int SW = stride_words(L);
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_tile = (int64_t)n * 32;
  if (idx >= mtiles * per_tile) return;
  const int64_t mt = idx / per_tile;
  const int c = (int)(idx % per_tile);
  const int s = c >> 5, mg = (c >> 1) & 15, kc = c & 1;
  uint32_t o[32];
#pragma unroll
  for (int rr = 0; rr < 8; rr++) {
    const int64_t i0 = mt * 128 + mg * 8 + rr;
    const int64_t i = (perm && i0 < rows) ? (int64_t)perm[i0] : i0;
#pragma unroll
    for (int w = 0; w < 4; w++) {
      const int limb = kc * 4 + w;
      o[rr * 4 + w] = (i0 < rows && i >= 0 && limb < L) ? (ys[s][(size_t)i * SW + limb] ^ 0x80000000u) : 0u;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(Y + (size_t)idx * 128);
#pragma unroll
  for (int q = 0; q < 8; q++) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
}

// the step's coefficients travel as kernel parameters (n x 8 words) and
// every CTA expands them into its C' tiles in shared memory: no copy, no
// host synchronisation between Horner steps
struct TclCoef {
  uint32_t w[8][8];  // [s][limb], canonical
};

// K steps' coefficients and outputs of one batched combination
template <int K>
struct TclBatch {
  uint32_t w[K][8][8];  // [step][s][limb], canonical
  uint32_t* dst[K];     // row-indexed outputs (biased slots)
};

template <int L, int K>
__global__ void __launch_bounds__(tcl_threads(K), K == 1 ? TCL_CTAS_PER_SM : 1)
    tcl_combine(const uint8_t* __restrict__ Y, const TclBatch<K> cf, int n, int64_t rows,
                int64_t mtiles, const uint32_t* __restrict__ acc, const uint32_t* __restrict__ fold,
                const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int STAGES = tcl_stages(K);
  constexpr uint32_t TCOLS = tcl_tmem_cols(K);
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t YT = tcl_ytile_bytes(n), BB = tcl_b_bytes(n);
  uint8_t* sB = smem + STAGES * YT;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + K * BB);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's tiles: mt = blockIdx.x + j gridDim.x
  const int64_t ntile = blockIdx.x < mtiles ? (mtiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 128 * tcl_epi(K));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  // C'[k][(s, q)] = byte (k - q) of c_s, tiled [s][mg][kc][8 rows][16 bytes]:
  // word w of the tile holds 4 consecutive q of one (s, k)
  for (int w = threadIdx.x; w < (int)(K * BB / 4); w += blockDim.x) {
    const int st = w / (int)(BB / 4);  // which step's C'
    const int byte0 = (w % (int)(BB / 4)) * 4;
    const int s_ = byte0 / (TCL_N * 32), rem = byte0 % (TCL_N * 32);
    const int mg = rem >> 8, kc = (rem >> 7) & 1, rr = (rem >> 4) & 7, jj0 = rem & 15;
    const int k = mg * 8 + rr;
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int p = k - (kc * 16 + jj0 + b);
      const uint32_t v = (p >= 0 && p < 32) ? (cf.w[st][s_][p >> 2] >> (8 * (p & 3))) & 0xFFu : 0u;
      word |= v << (8 * b);
    }
    reinterpret_cast<uint32_t*>(sB)[w] = word;
  }
  // generic-proxy shared stores -> visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    for (int64_t j = 0; j < ntile; j++) {
      const int s = (int)(j % STAGES);
      if (j >= STAGES) mbar_wait(empty + s, (uint32_t)((j / STAGES - 1) & 1));
      mbar_expect_tx(full + s, YT);
      bulk_g2s(smem + s * YT, Y + (size_t)(blockIdx.x + j * gridDim.x) * YT, YT, full + s);
    }
  } else if (warp == 1 && lane == 0) {
    for (int64_t j = 0; j < ntile; j++) {
      const int s = (int)(j % STAGES);
      const int b = (int)(j & 1);
      mbar_wait(full + s, (uint32_t)((j / STAGES) & 1));
      if (j >= 2) mbar_wait(tempty + b, (uint32_t)((j / 2 - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sy = smem + s * YT;
      for (int st = 0; st < K; st++)
        for (int ks = 0; ks < n; ks++) {
          const uint64_t ad = umma_desc(sy + ks * (128 * 32));
          const uint64_t bd = umma_desc(sB + st * BB + ks * (TCL_N * 32));
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
                  tmem + (uint32_t)((b * K + st) * TCL_N)),
              "l"(ad), "l"(bd), "r"(TCL_IDESC), "r"(ks > 0 ? 1u : 0u));
        }
      umma_commit(empty + s);
      umma_commit(tfull + b);
    }
  } else if (warp >= 2) {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;  // which of the quarter's epilogue warps
    constexpr int E = tcl_epi(K);
    const int row = quarter * 32 + lane;
    for (int64_t j = 0; j < ntile; j++) {
      const int b = (int)(j & 1);
      mbar_wait(tfull + b, (uint32_t)((j / 2) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int st = half; st < K; st += E) {
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((b * K + st) * TCL_N);
      // bytes (weights 2^(8k)) -> 32-bit limbs V[0..16], the 64 columns read
      // from TMEM in two halves of 32 (fewer live registers)
      uint32_t V[17];
      uint64_t carry = 0;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        uint32_t d[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
              "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
              "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
              "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
            : "r"(ta + (uint32_t)(32 * h)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (h == 1 && st + E >= K) {  // this warp's last accumulator of the buffer is read
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(tempty + b);
        }
#pragma unroll
        for (int w = 0; w < 8; w++) {
          uint32_t word = 0;
#pragma unroll
          for (int bb = 0; bb < 4; bb++) {
            const uint64_t t = carry + d[4 * w + bb];
            word |= (uint32_t)(t & 0xFF) << (8 * bb);
            carry = t >> 8;
          }
          V[8 * h + w] = word;
        }
      }
      V[16] = (uint32_t)carry;  // < 2^25
      const int64_t i = (int64_t)(blockIdx.x + j * gridDim.x) * 128 + row;
      if (i >= rows) continue;
      int64_t a2[L + 1];
#pragma unroll
      for (int q = 0; q < L; q++)
        a2[q] = (int64_t)V[q] + ((K == 1 && acc) ? (int64_t)(acc[(size_t)i * SW + q] ^ 0x80000000u) : 0);
      a2[L] = 0;
#pragma unroll
      for (int k = L; k < 17; k++) {
        const uint32_t* R = fold + (size_t)(k - L) * L;
#pragma unroll
        for (int q = 0; q < L; q++) {
          const uint64_t pr = (uint64_t)V[k] * __ldg(R + q);
          a2[q] += (int64_t)(uint32_t)pr;
          a2[q + 1] += (int64_t)(pr >> 32);
        }
      }
      uint32_t Rr[L];
      finalize<L>(a2, 0, mp, Rr);
      uint32_t o[SW];
#pragma unroll
      for (int q = 0; q < SW; q++) o[q] = q < L ? (Rr[q] ^ 0x80000000u) : 0u;
      store_slot<SW>(cf.dst[st] + (size_t)i * SW, o);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

}  // namespace sld

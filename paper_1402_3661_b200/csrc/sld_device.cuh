// sld_device.cuh -- device-side arithmetic and kernels of the B200 Krylov
// SpMV engine (sm_100a).  See DESIGN.md for the data layout and the bounds.
//
// Vector layout in HBM: one residue per slot, `SW` 32-bit words per slot
// (SW = L rounded up to 8, i.e. whole 32-byte sectors), limbs little-endian
// and *biased*: word i holds (limb_i XOR 0x80000000), i.e. limb_i - 2^31 as a
// signed int32.  The bias lets one signed IMAD.WIDE (s32 x s32 + s64) do the
// multiply-accumulate of a signed coefficient with a limb; the bias is
// removed exactly per row from the running coefficient sum S:
//     sum_e c_e u_e = sum_i 2^(32 i) (sum_e c_e (u_ei - 2^31)) + 2^31 S sum_i 2^(32 i).
// Slot `total_cols` of every input vector is the zero residue, the target
// of padded index entries.
#pragma once
#include <cstdint>

namespace sld {

constexpr int MAXL = 32;  // 1024-bit moduli (the reference accepts <= 1024 bits)

struct ModParams {
  uint32_t ell[MAXL + 1];
  uint32_t K[MAXL + 3];  // ell * 2^48 in L+2 words: makes the row value positive
  uint32_t R2[MAXL + 1]; // 2^(64 L) mod ell (Montgomery conversion)
  uint64_t mu;           // floor(2^(bits-1+64) / ell)  (Barrett)
  uint32_t nprime;       // -ell^-1 mod 2^32            (Montgomery)
  int bits;              // bit length of ell
  int L;
};

__host__ __device__ constexpr int stride_words(int L) { return ((L + 7) / 8) * 8; }

struct SliceInfo {
  uint32_t pm_off;  // uint4 units into pm_idx
  uint32_t pm_k4;   // groups of 4 +-1 entries per lane
  uint32_t s_off;   // uint4 units into s_idx / s_coef
  uint32_t s_k4;    // groups of 4 small entries per lane
};

struct SpmvArgs {
  const uint32_t* x;        // input vector (biased), total_cols+1 slots
  uint32_t* y;              // output vector (biased), row-indexed (last pass)
  const uint32_t* part_in;  // slot-indexed canonical partials (pass > 0)
  uint32_t* part_out;       // slot-indexed canonical partials (pass < last)
  const SliceInfo* slices;  // this pass's slice table
  const uint4* pm_idx;      // +-1 entries: col | sign<<31
  const uint4* s_idx;       // small entries: col
  const int4* s_coef;       // small entries: signed coefficient, |c| < 2^31
  const int32_t* slot_row;  // output row of each slot (-1 = padding slot)
  const uint32_t* lane_k4;  // this pass: per slot (pm groups | small groups << 16)
  // full-class entries and dense columns (last pass only)
  const uint32_t* full_ptr; // per slot, CSR into full_col/full_val
  const uint32_t* full_col;
  const uint32_t* full_val; // Montgomery form, SW words each
  const uint32_t* dense_val;// [g][row] Montgomery form, SW words each
  int n_dense;
  int64_t dense_col0;       // global column index of dense column 0
  // unit-X projection of the INPUT vector (first pass only)
  const int64_t* proj_rows;
  int proj_m;
  uint32_t* terms_out;      // proj_m slots of SW words, canonical (unbiased)
  int64_t nslices;
  int64_t nslots;  // nslices * rows per slice (dense-value row stride)
  int has_full;
  int policy;  // bit0 gather L2 evict_last, bit1 output store evict_first, bit4 exchange store evict_first,
               // bit2 partial store evict_first, bit3 gathers L1::no_allocate
  // die-split passes (spmv_split): slices / lane_k4 hold both halves, half h
  // at offset h * nslices / h * nslots
  const uint8_t* die_map;  // %smid -> die (0/1)
  uint32_t* xch;           // [nslots * G * SW] the first half's row values
  uint32_t* cnt;           // [nslices] arrival counters (parity = order)
  uint32_t* queue;         // [3] work queue per die + exit counter
  uint32_t pf;             // index groups prefetched into L2 ahead of use
  // peer push (r x 1 grid, last pass): each output row goes to every node's
  // next-iterate buffer (peer memory) at row peer_off + row, instead of y
  uint32_t* yp[8];
  int npeer;
  int64_t peer_off;
  // fused Mksol Horner step (spmv_pass<L, 1, *, true, true>, L <= 8): the
  // output row becomes (A w)[row] + sum_s mk_c[s] y_s[row] mod ell
  const uint32_t* mk_y;  // [mk_n][nslots][SW] canonical y_s in the slot order
  const uint32_t* fold;  // 2^(32k) mod ell for k = L .. 2L, L words each
  int mk_n;
  uint32_t mk_c[8][8];  // the step's coefficients, canonical, L limbs each
  // Mksol Horner step with a precomputed combination (last pass, one chain,
  // L <= 8): the output row becomes (A w)[row] + addv[row] mod ell
  const uint32_t* addv;  // row-indexed biased vector, or null
};


// ---------------------------------------------------------------- loads

__device__ __forceinline__ uint64_t createpolicy_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <typename T>
__device__ __forceinline__ T ld_stream(const T* a, uint64_t pol) {
  static_assert(sizeof(T) == 16, "128-bit stream loads");
  uint32_t r0, r1, r2, r3;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "l"(a), "l"(pol));
  T v;
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
  w[0] = r0; w[1] = r1; w[2] = r2; w[3] = r3;
  return v;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// gather one residue slot with an explicit L2 policy
template <int SW>
__device__ __forceinline__ void gather_hint(const uint32_t* __restrict__ p, uint32_t (&u)[SW], uint64_t pol) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm("ld.global.nc.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(u[8 * q + 0]), "=r"(u[8 * q + 1]), "=r"(u[8 * q + 2]), "=r"(u[8 * q + 3]),
          "=r"(u[8 * q + 4]), "=r"(u[8 * q + 5]), "=r"(u[8 * q + 6]), "=r"(u[8 * q + 7])
        : "l"(p + 8 * q), "l"(pol));
  }
}

// the same gather through L2 only (.cg): for kernels that read residues other
// CTAs wrote earlier in the same launch (the persistent chain, spmv_chain),
// where the non-coherent .nc path may serve a stale line
template <int SW>
__device__ __forceinline__ void gather_cg(const uint32_t* __restrict__ p, uint32_t (&u)[SW], uint64_t pol) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm volatile("ld.global.cg.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(u[8 * q + 0]), "=r"(u[8 * q + 1]), "=r"(u[8 * q + 2]), "=r"(u[8 * q + 3]),
                   "=r"(u[8 * q + 4]), "=r"(u[8 * q + 5]), "=r"(u[8 * q + 6]), "=r"(u[8 * q + 7])
                 : "l"(p + 8 * q), "l"(pol));
  }
}

template <int SW, bool COH>
__device__ __forceinline__ void gather_x(const uint32_t* __restrict__ p, uint32_t (&u)[SW], uint64_t pol) {
  if constexpr (COH) gather_cg<SW>(p, u, pol);
  else gather_hint<SW>(p, u, pol);
}

template <int SW>
__device__ __forceinline__ void store_slot_hint(uint32_t* p, const uint32_t (&u)[SW], uint64_t pol) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm volatile("st.global.L2::cache_hint.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p + 8 * q),
                 "r"(u[8 * q + 0]), "r"(u[8 * q + 1]), "r"(u[8 * q + 2]), "r"(u[8 * q + 3]),
                 "r"(u[8 * q + 4]), "r"(u[8 * q + 5]), "r"(u[8 * q + 6]), "r"(u[8 * q + 7]), "l"(pol));
  }
}

template <int SW>
__device__ __forceinline__ void load_slot(const uint32_t* __restrict__ p, uint32_t (&u)[SW], uint64_t pol) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(u[8 * q + 0]), "=r"(u[8 * q + 1]), "=r"(u[8 * q + 2]), "=r"(u[8 * q + 3]),
          "=r"(u[8 * q + 4]), "=r"(u[8 * q + 5]), "=r"(u[8 * q + 6]), "=r"(u[8 * q + 7])
        : "l"(p + 8 * q), "l"(pol));
  }
}

// gather one residue slot (SW words, 32-byte sectors) through L1/L2
template <int SW>
__device__ __forceinline__ void gather(const uint32_t* __restrict__ p, uint32_t (&u)[SW]) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(u[8 * q + 0]), "=r"(u[8 * q + 1]), "=r"(u[8 * q + 2]), "=r"(u[8 * q + 3]),
          "=r"(u[8 * q + 4]), "=r"(u[8 * q + 5]), "=r"(u[8 * q + 6]), "=r"(u[8 * q + 7])
        : "l"(p + 8 * q));
  }
}

template <int SW>
__device__ __forceinline__ void store_slot(uint32_t* p, const uint32_t (&u)[SW]) {
#pragma unroll
  for (int q = 0; q < SW / 8; q++) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + 8 * q),
                 "r"(u[8 * q + 0]), "r"(u[8 * q + 1]), "r"(u[8 * q + 2]), "r"(u[8 * q + 3]),
                 "r"(u[8 * q + 4]), "r"(u[8 * q + 5]), "r"(u[8 * q + 6]), "r"(u[8 * q + 7]));
  }
}

// ---------------------------------------------------------- arithmetic

// r = a * b * 2^(-32 L) mod ell (CIOS Montgomery), a, b < ell -> r < ell
template <int L>
__device__ __forceinline__ void montmul(const uint32_t* a, const uint32_t* b, const ModParams& mp,
                                        uint32_t* r) {
  uint32_t t[L + 2];
#pragma unroll
  for (int j = 0; j < L + 2; j++) t[j] = 0;
#pragma unroll 1
  for (int i = 0; i < L; i++) {
    uint64_t c = 0;
    const uint32_t bi = b[i];
#pragma unroll
    for (int j = 0; j < L; j++) {
      c = (uint64_t)a[j] * bi + t[j] + (c >> 32);
      t[j] = (uint32_t)c;
    }
    uint64_t s = (uint64_t)t[L] + (c >> 32);
    t[L] = (uint32_t)s;
    t[L + 1] = (uint32_t)(s >> 32);
    const uint32_t m = t[0] * mp.nprime;
    c = (uint64_t)m * mp.ell[0] + t[0];
#pragma unroll
    for (int j = 1; j < L; j++) {
      c = (uint64_t)m * mp.ell[j] + t[j] + (c >> 32);
      t[j - 1] = (uint32_t)c;
    }
    s = (uint64_t)t[L] + (c >> 32);
    t[L - 1] = (uint32_t)s;
    t[L] = t[L + 1] + (uint32_t)(s >> 32);
  }
  // conditional subtract
  uint32_t d[L + 1];
  int64_t br = 0;
#pragma unroll
  for (int j = 0; j <= L; j++) {
    int64_t v = (int64_t)t[j] - (j < L ? mp.ell[j] : 0) + br;
    d[j] = (uint32_t)v;
    br = v >> 32;
  }
  const bool ge = br == 0;
#pragma unroll
  for (int j = 0; j < L; j++) r[j] = ge ? d[j] : t[j];
}

// Reduce the row value to [0, ell).  The row value is
//   V = sum_{i<=L} acc_i 2^(32 i) + 2^31 S sum_{i<L} 2^(32 i)
// (acc_i: per-limb lazy sums of c * (u_i - 2^31), small products split into
// their 32-bit halves; S = sum of the coefficients: the bias correction).
// |V| < 2^47 ell by the per-row count bounds enforced at build time.
template <int L>
__device__ __forceinline__ void finalize(int64_t (&acc)[L + 1], int64_t S, const ModParams& mp,
                                         uint32_t (&R)[L]) {
  // bias: 2^31 S = (S >> 1) 2^32 + (S & 1) 2^31, added to every limb i < L
  const int64_t b_lo = (S & 1) << 31, b_hi = S >> 1;
  uint32_t w[L + 2];
  int64_t carry = 0;
#pragma unroll
  for (int i = 0; i < L + 2; i++) {
    int64_t t = carry;
    if (i <= L) t += acc[i];
    if (i < L) t += b_lo;
    if (i >= 1 && i <= L) t += b_hi;
    w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  // V' = V + ell * 2^48 >= 0
  uint64_t c = 0;
#pragma unroll
  for (int i = 0; i < L + 2; i++) {
    c = (uint64_t)w[i] + mp.K[i] + (c >> 32);
    w[i] = (uint32_t)c;
  }
  // t = V' >> (bits-1): the top word index is L-1 for every modulus of L words
  const int sh = mp.bits - 1 - 32 * (L - 1);
  const unsigned __int128 top = ((unsigned __int128)w[L + 1] << 64) |
                                ((unsigned __int128)w[L] << 32) | w[L - 1];
  const uint64_t tq = (uint64_t)(top >> sh);
  const uint64_t q = __umul64hi(tq, mp.mu);  // q - 2 <= q_hat <= q
  const uint32_t q0 = (uint32_t)q, q1 = (uint32_t)(q >> 32);
  uint32_t P[L + 1];
  uint64_t m = 0;
#pragma unroll
  for (int j = 0; j < L; j++) {
    m = (uint64_t)q0 * mp.ell[j] + (m >> 32);
    P[j] = (uint32_t)m;
  }
  P[L] = (uint32_t)(m >> 32);
  m = 0;
#pragma unroll
  for (int j = 0; j < L; j++) {
    m = (uint64_t)q1 * mp.ell[j] + P[j + 1] + (m >> 32);
    P[j + 1] = (uint32_t)m;
  }
  uint32_t r[L + 1];
  int64_t br = 0;
#pragma unroll
  for (int j = 0; j <= L; j++) {
    int64_t v = (int64_t)w[j] - P[j] + br;
    r[j] = (uint32_t)v;
    br = v >> 32;
  }
  // r in [0, 3 ell): two conditional subtractions
#pragma unroll
  for (int rep = 0; rep < 2; rep++) {
    uint32_t d[L + 1];
    br = 0;
#pragma unroll
    for (int j = 0; j <= L; j++) {
      int64_t v = (int64_t)r[j] - (j < L ? mp.ell[j] : 0) + br;
      d[j] = (uint32_t)v;
      br = v >> 32;
    }
    if (br == 0) {
#pragma unroll
      for (int j = 0; j <= L; j++) r[j] = d[j];
    }
  }
#pragma unroll
  for (int j = 0; j < L; j++) R[j] = r[j];
}

// ------------------------------------------------------------- SpMV pass
//
// One thread per output row ("slot" in the sorted SELL-32 order), one warp
// per 32-slot slice.  Entry streams are laid out [group][lane][4] so every
// 128-bit index load of a warp is one coalesced 512-byte transaction.
// resident CTAs per SM the register allocation must allow: 4 x 256 threads
// (64 registers) for L <= 8 -- the gathers need every warp they can get
#ifndef SLD_PASS_MINB
#define SLD_PASS_MINB 4
#endif
#ifndef SLD_PASS_NB
#define SLD_PASS_NB 4
#endif
template <int L>
__host__ __device__ constexpr int spmv_min_blocks() { return L <= 8 ? SLD_PASS_MINB : (L <= 16 ? 3 : 2); }
// gathers in flight per thread per batch: 4 for one-sector residues, fewer
// for wide moduli so the accumulator + gathered slots fit the register budget
template <int L>
__host__ __device__ constexpr int spmv_batch() { return L <= 8 ? SLD_PASS_NB : (L <= 16 ? 2 : 1); }

// G chains share one matrix pass (block Wiedemann's independent sequences):
// a column's G residues are one contiguous record of G*SW words, and the G
// lanes of a row gather the G sectors of the same record in one instruction,
// which the L1 coalesces into ONE request.  Random gathers are request-bound
// (~1 sector-request per SM per clock, profiles/microbench2_r01.txt), so a
// 2-sector record moves ~1.7x the useful bytes per second of a 1-sector one.

// Index-stream prefetch: each lane asks L2 for its index group PF groups
// ahead of the one it consumes, so the DRAM latency of the read-once index
// stream overlaps the gathers of the groups before it.  (A shared-memory
// cp.async ring was measured slower: its 33 KB per CTA come out of the L1
// that stages the outstanding gathers.)

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(p));
}

// the +-1 and small entries of one row in one part (column stripe [x half]);
// with K lanes per row (short rows) lane `sub` takes groups sub, sub+K, ...
template <int L, int G, int K = 1, bool COH = false, int PIPE = 1, bool SPIPE = false>
__device__ __forceinline__ void row_entries(const SpmvArgs& a, const SliceInfo& si, uint32_t kk, int rw,
                                            const uint32_t* xc, uint64_t pol, uint64_t gpol,
                                            int64_t (&acc)[L + 1], int64_t& S, int sub = 0) {
  constexpr int SW = stride_words(L);
  constexpr int NB = spmv_batch<L>();
  constexpr int R = 32 / (G * K);
  const uint32_t my_pm = kk & 0xFFFFu, my_s = kk >> 16;
  const uint32_t PF = a.pf * K;  // prefetch distance in groups (0: off)
  const uint4* pp = a.pm_idx + si.pm_off + rw;
#pragma unroll 1
  for (uint32_t k = sub; k < PF && k < my_pm; k += K) prefetch_l2(pp + (size_t)k * R);
  // PIPE (1 or 2): the index words of the next one or two groups are loaded
  // before this group's gathers issue (register quads of software
  // pipelining), so the index latency hides behind the gathers without the
  // extra requests of L2 prefetches; SPIPE does the same for the small
  // entries' index and coefficient words.  Measured with A/B builds on one
  // box (profiles/sweep_idx_pipe_r02.txt): cfg3 one chain 1.575 (none) ->
  // 1.559 (PIPE 1) -> 1.535-1.542 ms (PIPE 2 + SPIPE); two chains 1.354 ->
  // 1.289-1.296 ms per chain-product with PIPE 1 and worse with more; the
  // single-pass one-chain kernel (cfg2) is 1% slower with any and keeps the
  // plain loop.
  constexpr bool SP = PIPE > 0 && SPIPE;
  uint4 w_next = make_uint4(0u, 0u, 0u, 0u), w_next2 = make_uint4(0u, 0u, 0u, 0u);
  if (PIPE > 0 && sub < my_pm) w_next = ld_stream(pp + (size_t)sub * R, pol);
  if (PIPE > 1 && sub + K < my_pm) w_next2 = ld_stream(pp + (size_t)(sub + K) * R, pol);
  const uint4* sp = a.s_idx + si.s_off + rw;
  const int4* cp = a.s_coef + si.s_off + rw;
  // with K lanes per row, small group 0 goes to the lane after the one that
  // took the last +-1 group, so the row's groups spread evenly over its lanes
  const uint32_t s0 = K > 1 ? (uint32_t)(sub + K - (int)(my_pm % K)) % K : 0u;
  uint4 sw_next = make_uint4(0u, 0u, 0u, 0u);
  int4 sc_next = make_int4(0, 0, 0, 0);
#pragma unroll 1
  for (uint32_t k = sub; k < my_pm; k += K) {
    if (PF && k + PF < my_pm) prefetch_l2(pp + (size_t)(k + PF) * R);
    const uint4 w = PIPE > 0 ? w_next : ld_stream(pp + (size_t)k * R, pol);
    if (PIPE > 1) {
      w_next = w_next2;
      if (k + 2 * K < my_pm) w_next2 = ld_stream(pp + (size_t)(k + 2 * K) * R, pol);
    } else if (PIPE > 0 && k + K < my_pm) {
      w_next = ld_stream(pp + (size_t)(k + K) * R, pol);
    }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e0 = 0; e0 < 4; e0 += NB) {
      uint32_t u[NB][SW];
#pragma unroll
      for (int e = 0; e < NB; e++)
        gather_x<SW, COH>(xc + (size_t)(ws[e0 + e] & 0x7FFFFFFFu) * (G * SW), u[e], gpol);
#pragma unroll
      for (int e = 0; e < NB; e++) {
        const int32_t c = 1 - (int32_t)((ws[e0 + e] >> 30) & 2u);  // +1 / -1
        S += c;
#pragma unroll
        for (int i = 0; i < L; i++) acc[i] += (int64_t)c * (int64_t)(int32_t)u[e][i];
      }
    }
  }
  // small entries: one signed IMAD.WIDE per limb, the 64-bit product split
  // into its low word (limb i) and signed high word (limb i+1)
  if (SP && s0 < my_s) {
    sw_next = ld_stream(sp + (size_t)s0 * R, pol);
    sc_next = ld_stream(cp + (size_t)s0 * R, pol);
  }
#pragma unroll 1
  for (uint32_t k = s0; k < PF && k < my_s; k += K) {
    prefetch_l2(sp + (size_t)k * R);
    prefetch_l2(cp + (size_t)k * R);
  }
#pragma unroll 1
  for (uint32_t k = s0; k < my_s; k += K) {
    if (PF && k + PF < my_s) {
      prefetch_l2(sp + (size_t)(k + PF) * R);
      prefetch_l2(cp + (size_t)(k + PF) * R);
    }
    const uint4 w = SP ? sw_next : ld_stream(sp + (size_t)k * R, pol);
    const int4 cf = SP ? sc_next : ld_stream(cp + (size_t)k * R, pol);
    if (SP && k + K < my_s) {
      sw_next = ld_stream(sp + (size_t)(k + K) * R, pol);
      sc_next = ld_stream(cp + (size_t)(k + K) * R, pol);
    }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const int32_t cs[4] = {cf.x, cf.y, cf.z, cf.w};
#pragma unroll
    for (int e0 = 0; e0 < 4; e0 += NB) {
      uint32_t u[NB][SW];
#pragma unroll
      for (int e = 0; e < NB; e++) gather_x<SW, COH>(xc + (size_t)ws[e0 + e] * (G * SW), u[e], gpol);
#pragma unroll
      for (int e = 0; e < NB; e++) {
        const int32_t c = cs[e0 + e];
        S += c;
#pragma unroll
        for (int i = 0; i < L; i++) {
          const int64_t p = (int64_t)c * (int64_t)(int32_t)u[e][i];
          acc[i] += (int64_t)(uint32_t)p;
          acc[i + 1] += (int64_t)(int32_t)(p >> 32);
        }
      }
    }
  }
}

// add the precomputed combination addv[slot] (slot-ordered, so a warp's
// loads are coalesced) into a row's sums before its Barrett reduction (one
// more canonical term: the bounds of finalize hold)
template <int L>
__device__ __forceinline__ void add_slot_vector(const SpmvArgs& a, int64_t slot, uint64_t pol,
                                                int64_t (&acc)[L + 1]) {
  constexpr int SW = stride_words(L);
  uint32_t u[SW];
  load_slot<SW>(a.addv + (size_t)slot * SW, u, pol);
#pragma unroll
  for (int i = 0; i < L; i++) acc[i] += (int64_t)(u[i] ^ 0x80000000u);
}

// full-class coefficients and dense columns of one row (last pass only):
// f*u mod ell by Montgomery, f stored as f R
template <int L, int G, bool COH = false>
__device__ __forceinline__ void row_full(const SpmvArgs& a, const ModParams& mp, int64_t slot, int32_t row,
                                         const uint32_t* xc, int64_t (&acc)[L + 1]) {
  constexpr int SW = stride_words(L);
  const uint64_t npol = COH ? createpolicy_normal() : 0;
#pragma unroll 1
  for (uint32_t p = a.full_ptr[slot]; p < a.full_ptr[slot + 1]; p++) {
    uint32_t u[SW], f[L], r[L];
    if constexpr (COH) gather_cg<SW>(xc + (size_t)a.full_col[p] * (G * SW), u, npol);
    else gather<SW>(xc + (size_t)a.full_col[p] * (G * SW), u);
#pragma unroll
    for (int i = 0; i < L; i++) { u[i] ^= 0x80000000u; f[i] = a.full_val[(size_t)p * SW + i]; }
    montmul<L>(f, u, mp, r);
#pragma unroll
    for (int i = 0; i < L; i++) acc[i] += r[i];
  }
  if (row >= 0) {
#pragma unroll 1
    for (int g = 0; g < a.n_dense; g++) {
      uint32_t u[SW], f[L], r[L];
      if constexpr (COH) gather_cg<SW>(xc + (size_t)(a.dense_col0 + g) * (G * SW), u, npol);
      else gather<SW>(xc + (size_t)(a.dense_col0 + g) * (G * SW), u);
#pragma unroll
      for (int i = 0; i < L; i++) { u[i] ^= 0x80000000u; }
      // dense values: [g][row], rows padded to nslots
      const uint32_t* dv = a.dense_val + ((size_t)g * (size_t)a.nslots + (size_t)row) * SW;
#pragma unroll
      for (int i = 0; i < L; i++) f[i] = dv[i];
      montmul<L>(f, u, mp, r);
#pragma unroll
      for (int i = 0; i < L; i++) acc[i] += r[i];
    }
  }
}

// a_i = X^T v_i of the iterate this product consumes (solver.py:210): the
// first threads of block 0 copy the m unit-X rows of the INPUT iterate
template <int L, int G>
__device__ __forceinline__ void unit_projection(const SpmvArgs& a) {
  constexpr int SW = stride_words(L);
  if (blockIdx.x == 0 && threadIdx.x < a.proj_m * G) {
    const int t = threadIdx.x / G, c = threadIdx.x % G;
    const uint32_t* src = a.x + ((size_t)a.proj_rows[t] * G + c) * SW;
    uint32_t* dst = a.terms_out + ((size_t)t * G + c) * SW;
#pragma unroll
    for (int i = 0; i < SW; i++) dst[i] = i < L ? (src[i] ^ 0x80000000u) : 0u;
  }
}

// store a finished canonical row value: biased into y (last pass) or
// canonical into the slot-indexed partial (more passes follow)
template <int L, int G, bool LAST>
__device__ __forceinline__ void store_row(const SpmvArgs& a, int64_t slot, int chain, const uint32_t (&Rr)[L],
                                          uint64_t pol) {
  constexpr int SW = stride_words(L);
  uint32_t o[SW];
  if (LAST) {
    const int32_t row = a.slot_row[slot];
    if (row < 0) return;
#pragma unroll
    for (int i = 0; i < SW; i++) o[i] = i < L ? (Rr[i] ^ 0x80000000u) : 0u;
    if (a.npeer) {
      // NVLink peer stores (or same-device buffers): the all-gather of the
      // r x 1 grid done by the SpMV epilogue itself
#pragma unroll 1
      for (int k = 0; k < a.npeer; k++)
        store_slot<SW>(a.yp[k] + ((size_t)(a.peer_off + row) * G + chain) * SW, o);
      return;
    }
    uint32_t* dst = a.y + ((size_t)row * G + chain) * SW;
    if (a.policy & 2) store_slot_hint<SW>(dst, o, pol);
    else store_slot<SW>(dst, o);
  } else {
#pragma unroll
    for (int i = 0; i < SW; i++) o[i] = i < L ? Rr[i] : 0u;
    uint32_t* dst = a.part_out + ((size_t)slot * G + chain) * SW;
    if (a.policy & 4) store_slot_hint<SW>(dst, o, pol);
    else store_slot<SW>(dst, o);
  }
}

// Mksol's combination fused into the last pass (solver.py:522-536): R <-
// R + sum_s c_s y_s[slot] mod ell.  32 x 32-bit limb products go lazily into
// 64-bit columns (low word to column p+q, high word to p+q+1: < 2^40 for
// n <= 8), are carried into 2L+1 limbs, the limbs above L folded with
// 2^(32k) mod ell, and one more finalize reduces (|V| < (L+2) 2^32 ell).
// The y_s are stored in slot order, so a warp's loads are coalesced.
template <int L>
__device__ __forceinline__ void mk_combine(const SpmvArgs& a, int64_t slot, const ModParams& mp, uint64_t pol,
                                           uint32_t (&Rr)[L]) {
  constexpr int SW = stride_words(L);
  uint64_t col[2 * L];
#pragma unroll
  for (int k = 0; k < 2 * L; k++) col[k] = k < L ? Rr[k] : 0u;
#pragma unroll
  for (int s = 0; s < 8; s++) {
    if (s >= a.mk_n) break;
    uint32_t u[SW];
    load_slot<SW>(a.mk_y + ((size_t)s * a.nslots + slot) * SW, u, pol);
#pragma unroll
    for (int p = 0; p < L; p++) {
      const uint32_t c = a.mk_c[s][p];
#pragma unroll
      for (int q = 0; q < L; q++) {
        const uint64_t pr = (uint64_t)c * u[q];
        col[p + q] += (uint32_t)pr;
        col[p + q + 1] += pr >> 32;
      }
    }
  }
  uint32_t V[2 * L];
  uint64_t carry = 0;
#pragma unroll
  for (int k = 0; k < 2 * L; k++) {
    const uint64_t t = col[k] + carry;
    V[k] = (uint32_t)t;
    carry = t >> 32;
  }
  int64_t acc[L + 1];
#pragma unroll
  for (int j = 0; j < L; j++) acc[j] = V[j];
  acc[L] = 0;
#pragma unroll
  for (int k = L; k <= 2 * L; k++) {
    const uint32_t limb = k < 2 * L ? V[k] : (uint32_t)carry;
    const uint32_t* R = a.fold + (size_t)(k - L) * L;
#pragma unroll
    for (int j = 0; j < L; j++) {
      const uint64_t pr = (uint64_t)limb * __ldg(R + j);
      acc[j] += (int64_t)(uint32_t)pr;
      acc[j + 1] += (int64_t)(pr >> 32);
    }
  }
  finalize<L>(acc, 0, mp, Rr);
}

template <int L, int G, bool FIRST, bool LAST, bool MK = false>
__global__ void __launch_bounds__(256, spmv_min_blocks<L>()) spmv_pass(const SpmvArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int R = 32 / G;  // rows per warp = slice height
  const int lane = threadIdx.x & 31;
  const int chain = lane & (G - 1);
  const int rw = lane / G;
  const int64_t slice = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t slot = slice * R + rw;

  if (FIRST) unit_projection<L, G>(a);
  if (slice >= a.nslices) return;

  const uint64_t pol = policy_evict_first();
  const uint64_t gpol = (a.policy & 1) ? policy_evict_last() : createpolicy_normal();
  const SliceInfo si = a.slices[slice];
  // per-row group counts: lanes stop at their own row length, so padded
  // SELL positions are never loaded (no index or gather traffic)
  const uint32_t kk = a.lane_k4[slot];
  const uint32_t* xc = a.x + (size_t)chain * SW;  // this lane's chain in every record
  int64_t acc[L + 1];
#pragma unroll
  for (int i = 0; i <= L; i++) acc[i] = 0;
  if (!FIRST) {
    // the earlier stripes' partial (usually from DRAM) starts the sums: its
    // load issues with the row's first index load, not after the gathers
    // (cfg3 1.538 -> 1.534 ms, two chains 1.299 -> 1.289 ms per chain-product)
    uint32_t pin[SW];
    load_slot<SW>(a.part_in + ((size_t)slot * G + chain) * SW, pin, pol);
#pragma unroll
    for (int i = 0; i < L; i++) acc[i] = pin[i];
  }
  int64_t S = 0;  // sum of coefficients (bias correction)
  constexpr bool ONE_PASS_ONE_CHAIN = FIRST && LAST && G == 1;
  row_entries<L, G, 1, false, ONE_PASS_ONE_CHAIN ? 0 : (G == 1 ? 2 : 1), G == 1 && !ONE_PASS_ONE_CHAIN>(
      a, si, kk, rw, xc, pol, gpol, acc, S);
  if (LAST && a.has_full) row_full<L, G>(a, mp, slot, a.slot_row[slot], xc, acc);
  if (G == 1 && LAST && a.addv) add_slot_vector<L>(a, slot, pol, acc);
  uint32_t Rr[L];
  finalize<L>(acc, S, mp, Rr);
  if constexpr (MK) mk_combine<L>(a, slot, mp, pol, Rr);
  store_row<L, G, LAST>(a, slot, chain, Rr, pol);
}

// canonical copy of y (biased, row-indexed) in the slot order of a matrix's
// passes; padding slots are zero (the fused Mksol step's operand)
template <int L>
__global__ void mk_slot_gather(const uint32_t* __restrict__ y, const int32_t* __restrict__ slot_row, int64_t nslots,
                               uint32_t* __restrict__ out) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nslots) return;
  const int32_t row = slot_row[i];
  uint32_t o[SW];
#pragma unroll
  for (int j = 0; j < SW; j++) o[j] = (row >= 0 && j < L) ? (y[(size_t)row * SW + j] ^ 0x80000000u) : 0u;
  store_slot<SW>(out + (size_t)i * SW, o);
}

// ---------------------------------------------------- short-row SpMV pass
//
// Small matrices (one chain, L <= 8): a one-lane-per-row warp runs its row's
// index groups one after another, so a product takes ~groups x (index + gather
// latency) while most SMs idle.  Here 4 lanes share a row and take every 4th
// group; their int64 accumulators are summed with shuffles and the row's
// first lane finishes it.  8 rows per warp, 4x the warps.
constexpr int SHORT_K = 4;

template <int L, bool FIRST, bool LAST>
#ifndef SLD_SHORT_MAXT  // launch bounds of the short-row pass (experiment builds override)
#define SLD_SHORT_MAXT 256
#define SLD_SHORT_MINB spmv_min_blocks<L>()
#endif
__global__ void __launch_bounds__(SLD_SHORT_MAXT, SLD_SHORT_MINB) spmv_short(const SpmvArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int R = 32 / SHORT_K;
  const int lane = threadIdx.x & 31;
  const int rw = lane / SHORT_K, sub = lane % SHORT_K;
  const int64_t slice = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t slot = slice * R + rw;

  // programmatic dependent launch (the next product's kernel may be launched
  // with it, sld_ops.cuh): read this slice's matrix words (written at build
  // time) before waiting, and touch the iterates only after the previous
  // product has completed and flushed (griddepcontrol.wait; a no-op without
  // PDL).  The next product is released once every CTA has gathered its
  // entries (launch_dependents below): its CTAs wait in griddepcontrol.wait,
  // which costs issue slots, so releasing it at the start was slower
  // (cfg1-sized 10k rows 6.48 vs 5.26 us)
  const bool live = slice < a.nslices;
  SliceInfo si{};
  uint32_t kk = 0;
  if (live) {
    si = a.slices[slice];
    kk = a.lane_k4[slot];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (FIRST) unit_projection<L, 1>(a);
  if (!live) return;

  const uint64_t pol = policy_evict_first();
  const uint64_t gpol = (a.policy & 1) ? policy_evict_last() : createpolicy_normal();
  int64_t acc[L + 1];
#pragma unroll
  for (int i = 0; i <= L; i++) acc[i] = 0;
  int64_t S = 0;
  // (index pipelining measured neutral here: cfg1 6.1 vs 6.0 us, 60k rows 11.96 vs 11.95 us)
  row_entries<L, 1, SHORT_K, false, 0>(a, si, kk, rw, a.x, pol, gpol, acc, S, sub);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the partial and the full-class entries go into other lanes' sums before
  // the reduction, so their loads overlap instead of trailing the row's tail
  if (!FIRST && sub == 2) {
    uint32_t pin[SW];
    load_slot<SW>(a.part_in + (size_t)slot * SW, pin, pol);
#pragma unroll
    for (int i = 0; i < L; i++) acc[i] += pin[i];
  }
  if (LAST && a.has_full && sub == SHORT_K - 1) row_full<L, 1>(a, mp, slot, a.slot_row[slot], a.x, acc);
  if (LAST && a.addv && sub == 1) add_slot_vector<L>(a, slot, pol, acc);
#pragma unroll
  for (int off = 1; off < SHORT_K; off <<= 1) {
#pragma unroll
    for (int i = 0; i <= L; i++) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
    S += __shfl_xor_sync(0xffffffffu, S, off);
  }
  if (sub != 0) return;
  uint32_t Rr[L];
  finalize<L>(acc, S, mp, Rr);
  store_row<L, 1, LAST>(a, slot, 0, Rr, pol);
}

// ------------------------------------------- persistent Krylov chain
//
// Small matrices (the short-row layout in one pass) are latency-bound: a
// product's gathers take ~1.5 us at the request rate, but each warp walks a
// serial chain of dependent loads (slice table -> group counts -> index group
// -> gathers -> next index group ...) and the kernel boundary between two
// products of a CUDA graph adds more.  spmv_chain runs `steps` products of
// the chain v <- A v in ONE cooperative launch:
//  * every warp keeps its slice from product to product; the slice's entry
//    streams are staged in shared memory once (ch.wcap uint4 per warp) and
//    its table entries stay in registers, so a product's serial chain is
//    shared-memory index loads and the gathers they feed;
//  * a grid barrier (one counter, release/acquire at gpu scope) separates
//    product t from t + 1, and the iterate ping-pongs between two buffers;
//  * gathers read residues other CTAs wrote in this launch: the barrier's
//    gpu-scope fences invalidate L1, so within a product the iterate can be
//    cached in L1 (L1G, hot columns) or read through L2 only (.cg).
// The unit-X projection of each input iterate goes to terms + t * tstride.
struct ChainArgs {
  uint32_t* buf[2];  // buf[0] holds the input iterate; product t reads buf[t & 1]
  uint32_t* bar;     // barrier counter, zero at launch
  uint32_t* terms;   // projection of product t's input at terms + t * tstride
  int64_t tstride;   // words
  int64_t steps;
  uint32_t wcap;     // shared-memory entry-stream capacity per warp (uint4)
  int mode;          // experiments (env SLD_CHAIN_MODE, wrong results): bit0 skips the products (the
                     // barrier alone), bit1 the reductions, bit2 the full-class entries, bit3 the ping-pong
};

// CTA-wide arrive (release: cumulative over the CTA's stores, which bar.sync
// ordered before it) and wait.  The poll is relaxed and one acquire fence
// follows it: an acquire load per poll would invalidate the SM's L1 on every
// spin (CCTL.IVALL), under the CTAs still computing on the same SM.
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    uint32_t v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <int SW, bool L1G>
__device__ __forceinline__ void chain_gather(const uint32_t* p, uint32_t (&u)[SW], uint64_t pol) {
  if constexpr (L1G) {
#pragma unroll
    for (int q = 0; q < SW / 8; q++)
      asm volatile("ld.global.ca.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                   : "=r"(u[8 * q + 0]), "=r"(u[8 * q + 1]), "=r"(u[8 * q + 2]), "=r"(u[8 * q + 3]),
                     "=r"(u[8 * q + 4]), "=r"(u[8 * q + 5]), "=r"(u[8 * q + 6]), "=r"(u[8 * q + 7])
                   : "l"(p + 8 * q), "l"(pol));
  } else {
    gather_cg<SW>(p, u, pol);
  }
}

// one row's +-1 and small entries, K = SHORT_K lanes per row (lane `sub`
// takes groups sub, sub + K, ...); pm / sx / sc point at the row's group 0
// in shared memory (staged slice) or global memory, group stride R
template <int L, bool L1G>
__device__ __forceinline__ void chain_entries(const uint4* pm, const uint4* sx, const int4* sc, uint32_t kk,
                                              int sub, const uint32_t* x, uint64_t gpol, int64_t (&acc)[L + 1],
                                              int64_t& S) {
  constexpr int SW = stride_words(L);
  constexpr int R = 32 / SHORT_K;
  const uint32_t my_pm = kk & 0xFFFFu, my_s = kk >> 16;
#pragma unroll 1
  for (uint32_t k = sub; k < my_pm; k += SHORT_K) {
    const uint4 w = pm[(size_t)k * R];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t u[4][SW];
#pragma unroll
    for (int e = 0; e < 4; e++) chain_gather<SW, L1G>(x + (size_t)(ws[e] & 0x7FFFFFFFu) * SW, u[e], gpol);
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int32_t c = 1 - (int32_t)((ws[e] >> 30) & 2u);
      S += c;
#pragma unroll
      for (int i = 0; i < L; i++) acc[i] += (int64_t)c * (int64_t)(int32_t)u[e][i];
    }
  }
  const uint32_t s0 = (uint32_t)(sub + SHORT_K - (int)(my_pm % SHORT_K)) % SHORT_K;  // as in row_entries
#pragma unroll 1
  for (uint32_t k = s0; k < my_s; k += SHORT_K) {
    const uint4 w = sx[(size_t)k * R];
    const int4 cf = sc[(size_t)k * R];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const int32_t cs[4] = {cf.x, cf.y, cf.z, cf.w};
    uint32_t u[4][SW];
#pragma unroll
    for (int e = 0; e < 4; e++) chain_gather<SW, L1G>(x + (size_t)ws[e] * SW, u[e], gpol);
#pragma unroll
    for (int e = 0; e < 4; e++) {
      S += cs[e];
#pragma unroll
      for (int i = 0; i < L; i++) {
        const int64_t p = (int64_t)cs[e] * (int64_t)(int32_t)u[e][i];
        acc[i] += (int64_t)(uint32_t)p;
        acc[i + 1] += (int64_t)(int32_t)(p >> 32);
      }
    }
  }
}

template <int L, bool L1G>
__global__ void __launch_bounds__(256, 3) spmv_chain(const SpmvArgs a, const ModParams mp, const ChainArgs ch) {
  extern __shared__ uint4 chain_smem[];
  constexpr int SW = stride_words(L);
  constexpr int R = 32 / SHORT_K;
  const int lane = threadIdx.x & 31;
  const int rw = lane / SHORT_K, sub = lane % SHORT_K;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the whole matrix and both iterates stay L2-resident from product to product
  const uint64_t pol = createpolicy_normal();
  const uint64_t gpol = policy_evict_last();
  // this warp's first slice: table entries in registers, entry streams
  // staged in shared memory when they fit the warp's share
  uint4* wsm = chain_smem + (size_t)(threadIdx.x >> 5) * ch.wcap;
  SliceInfo si0{0, 0, 0, 0};
  uint32_t kk0 = 0;
  int32_t row0 = -1;
  bool staged = false;
  if (warp0 < a.nslices) {
    si0 = a.slices[warp0];
    kk0 = a.lane_k4[warp0 * R + rw];
    row0 = a.slot_row[warp0 * R + rw];
    const uint32_t npm = si0.pm_k4 * R, ns = si0.s_k4 * R;
    staged = npm + 2 * ns <= ch.wcap;
    if (staged) {
      for (uint32_t i = lane; i < npm; i += 32) wsm[i] = a.pm_idx[si0.pm_off + i];
      for (uint32_t i = lane; i < ns; i += 32) {
        wsm[npm + i] = a.s_idx[si0.s_off + i];
        const int4 c = a.s_coef[si0.s_off + i];
        wsm[npm + ns + i] = make_uint4((uint32_t)c.x, (uint32_t)c.y, (uint32_t)c.z, (uint32_t)c.w);
      }
    }
    __syncwarp();
  }
#pragma unroll 1
  for (int64_t t = 0; t < ch.steps; t++) {
    const bool odd = (t & 1) && !(ch.mode & 8);  // mode bit 3 (experiment): always buf[0] -> buf[1]
    const uint32_t* x = odd ? ch.buf[1] : ch.buf[0];
    uint32_t* y = odd ? ch.buf[0] : ch.buf[1];
    if (blockIdx.x == 0 && threadIdx.x < a.proj_m) {
      uint32_t u[SW];
      gather_cg<SW>(x + (size_t)a.proj_rows[threadIdx.x] * SW, u, pol);
      uint32_t* dst = ch.terms + (size_t)t * ch.tstride + (size_t)threadIdx.x * SW;
#pragma unroll
      for (int i = 0; i < SW; i++) dst[i] = i < L ? (u[i] ^ 0x80000000u) : 0u;
    }
#pragma unroll 1
    for (int64_t slice = warp0; slice < ((ch.mode & 1) ? 0 : a.nslices); slice += nwarps) {
      const bool first = slice == warp0;
      const int64_t slot = slice * R + rw;
      const SliceInfo si = first ? si0 : a.slices[slice];
      const uint32_t kk = first ? kk0 : a.lane_k4[slot];
      const int32_t row = first ? row0 : a.slot_row[slot];
      const uint4 *pm, *sx;
      const int4* sc;
      if (first && staged) {
        pm = wsm + rw;
        sx = wsm + si.pm_k4 * R + rw;
        sc = reinterpret_cast<const int4*>(wsm + (si.pm_k4 + si.s_k4) * R) + rw;
      } else {
        pm = a.pm_idx + si.pm_off + rw;
        sx = a.s_idx + si.s_off + rw;
        sc = a.s_coef + si.s_off + rw;
      }
      int64_t acc[L + 1];
#pragma unroll
      for (int i = 0; i <= L; i++) acc[i] = 0;
      int64_t S = 0;
      chain_entries<L, L1G>(pm, sx, sc, kk, sub, x, gpol, acc, S);
      // full-class entries in the row's last lane, before the reduction
      if (a.has_full && !(ch.mode & 4) && sub == SHORT_K - 1) row_full<L, 1, true>(a, mp, slot, row, x, acc);
#pragma unroll
      for (int off = 1; off < SHORT_K; off <<= 1) {
#pragma unroll
        for (int i = 0; i <= L; i++) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
        S += __shfl_xor_sync(0xffffffffu, S, off);
      }
      if (sub == 0) {
        uint32_t Rr[L];
        if (ch.mode & 2) {  // experiment: no reduction (wrong results)
#pragma unroll
          for (int i = 0; i < L; i++) Rr[i] = (uint32_t)acc[i] ^ (uint32_t)S;
        } else {
          finalize<L>(acc, S, mp, Rr);
        }
        if (row >= 0) {
          uint32_t o[SW];
#pragma unroll
          for (int i = 0; i < SW; i++) o[i] = i < L ? (Rr[i] ^ 0x80000000u) : 0u;
          store_slot<SW>(y + (size_t)row * SW, o);
        }
      }
    }
    if (t + 1 < ch.steps) grid_barrier(ch.bar, (uint32_t)(t + 1) * gridDim.x);
  }
}

// ------------------------------------------------ limb-sliced SpMV pass
//
// Wide moduli (L > 8: residues of T = SW/8 >= 2 sectors).  Random gathers
// are request-bound (~1 request per SM per clock), and a residue loaded by
// one lane costs T requests.  Here the T lanes of a row each own one 32-byte
// slice (8 limbs) of every residue, so one instruction of the T lanes loads a
// whole residue as ONE request, and the per-lane accumulator is 8 limbs wide
// whatever L is.  Per row, the lanes then normalise their slices, pass the
// carries up the row with shuffles, hand the words to the row's first lane,
// and that lane runs the same tail as spmv_pass (partial, full-class
// entries, Barrett finalize, store).  Rows per warp: RH = 32 / T.
template <int L>
__host__ __device__ constexpr int wide_T() { return stride_words(L) / 8; }
#ifndef SLD_WIDE_MINB
#define SLD_WIDE_MINB 4  // resident CTAs per SM (64 registers; the Barrett tail spills, the gathers don't)
#endif

template <int L, bool FIRST, bool LAST>
__global__ void __launch_bounds__(256, SLD_WIDE_MINB) spmv_wide(const SpmvArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int T = wide_T<L>();
  constexpr int RH = 32 / T;
  constexpr int NB = 4;
  const int lane = threadIdx.x & 31;
  const int rw = lane / T, sl = lane % T;  // row in the slice, limb slice of the residue
  const bool active = rw < RH;
  const int64_t slice = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t slot = slice * RH + (active ? rw : 0);

  if (FIRST) unit_projection<L, 1>(a);
  if (slice >= a.nslices) return;

  const uint64_t pol = policy_evict_first();
  const uint64_t gpol = (a.policy & 1) ? policy_evict_last() : createpolicy_normal();
  const SliceInfo si = a.slices[slice];
  const uint32_t kk = active ? a.lane_k4[slot] : 0u;
  const uint32_t my_pm = kk & 0xFFFFu, my_s = kk >> 16;
  const uint32_t* xs = a.x + sl * 8;  // this lane's slice of every record
  int64_t acc[9];  // words 8 sl .. 8 sl + 7, and the small products' spill into the next slice
#pragma unroll
  for (int i = 0; i < 9; i++) acc[i] = 0;
  constexpr bool LAZY = SW >= L + 2;  // lazy partials between passes (below)
  if (!FIRST && LAZY && active) {
    // the earlier stripes' exact partial starts this lane's word sums (its
    // load issues with the first index load, not after the row's shuffles):
    // words 0..L-1 unsigned, word L+1 the signed top half of the int64 above
    uint32_t pin[8];
    load_slot<8>(a.part_in + (size_t)slot * SW + 8 * sl, pin, pol);
#pragma unroll
    for (int i = 0; i < 8; i++)
      acc[i] = (8 * sl + i == L + 1) ? (int64_t)(int32_t)pin[i] : (int64_t)pin[i];
  }
  int64_t S = 0;
  const uint32_t PF = a.pf;
  const uint4* pp = a.pm_idx + si.pm_off + rw;
#pragma unroll 1
  for (uint32_t k = 0; k < PF && k < my_pm; k++) prefetch_l2(pp + (size_t)k * RH);
  // index software pipelining as in row_entries, one group ahead (A/B on one
  // box, cfg5: 0.948 ms without, 0.910 with, 0.987 two groups ahead)
  uint4 w_next = make_uint4(0u, 0u, 0u, 0u);
  if (0 < my_pm) w_next = ld_stream(pp, pol);
#pragma unroll 1
  for (uint32_t k = 0; k < my_pm; k++) {
    if (PF && k + PF < my_pm) prefetch_l2(pp + (size_t)(k + PF) * RH);
    const uint4 w = w_next;
    if (k + 1 < my_pm) w_next = ld_stream(pp + (size_t)(k + 1) * RH, pol);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t u[NB][8];
#pragma unroll
    for (int e = 0; e < NB; e++) gather_hint<8>(xs + (size_t)(ws[e] & 0x7FFFFFFFu) * SW, u[e], gpol);
#pragma unroll
    for (int e = 0; e < NB; e++) {
      const int32_t c = 1 - (int32_t)((ws[e] >> 30) & 2u);
      S += c;
#pragma unroll
      for (int i = 0; i < 8; i++) acc[i] += (int64_t)c * (int64_t)(int32_t)u[e][i];
    }
  }
  const uint4* sp = a.s_idx + si.s_off + rw;
  const int4* cp = a.s_coef + si.s_off + rw;
#pragma unroll 1
  for (uint32_t k = 0; k < PF && k < my_s; k++) {
    prefetch_l2(sp + (size_t)k * RH);
    prefetch_l2(cp + (size_t)k * RH);
  }
  // the small entries' index and coefficient words one group ahead as well
  // (cfg5 0.9102 -> 0.9080 ms)
  constexpr bool SLD_WSPIPE = true;
  uint4 sw_next = make_uint4(0u, 0u, 0u, 0u);
  int4 sc_next = make_int4(0, 0, 0, 0);
  if (SLD_WSPIPE && 0 < my_s) {
    sw_next = ld_stream(sp, pol);
    sc_next = ld_stream(cp, pol);
  }
#pragma unroll 1
  for (uint32_t k = 0; k < my_s; k++) {
    if (PF && k + PF < my_s) {
      prefetch_l2(sp + (size_t)(k + PF) * RH);
      prefetch_l2(cp + (size_t)(k + PF) * RH);
    }
    const uint4 w = SLD_WSPIPE ? sw_next : ld_stream(sp + (size_t)k * RH, pol);
    const int4 cf = SLD_WSPIPE ? sc_next : ld_stream(cp + (size_t)k * RH, pol);
    if (SLD_WSPIPE && k + 1 < my_s) {
      sw_next = ld_stream(sp + (size_t)(k + 1) * RH, pol);
      sc_next = ld_stream(cp + (size_t)(k + 1) * RH, pol);
    }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const int32_t cs[4] = {cf.x, cf.y, cf.z, cf.w};
    uint32_t u[NB][8];
#pragma unroll
    for (int e = 0; e < NB; e++) gather_hint<8>(xs + (size_t)ws[e] * SW, u[e], gpol);
#pragma unroll
    for (int e = 0; e < NB; e++) {
      const int32_t c = cs[e];
      S += c;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int64_t p = (int64_t)c * (int64_t)(int32_t)u[e][i];
        acc[i] += (int64_t)(uint32_t)p;
        acc[i + 1] += (int64_t)(int32_t)(p >> 32);
      }
    }
  }
  // ---- normalise the slice: bias (see finalize), local carries
  const int64_t b_lo = (S & 1) << 31, b_hi = S >> 1;
  uint32_t wv[8];
  int64_t carry = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int g = 8 * sl + i;
    int64_t t = acc[i] + carry;
    if (g < L) t += b_lo;
    if (g >= 1 && g <= L) t += b_hi;
    wv[i] = (uint32_t)t;
    carry = t >> 32;
  }
  carry += acc[8];  // word 8 (sl + 1): the next slice's word 0
  if (sl == T - 1 && 8 * T <= L) carry += b_hi;  // the top lane owns word 8T itself
  // ---- carries up the row: after round r, slice r holds its final words
#pragma unroll
  for (int r = 1; r < T; r++) {
    const int64_t cin = __shfl_up_sync(0xffffffffu, carry, 1);
    if (sl == r) {
      int64_t c = cin;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int64_t t = (int64_t)wv[i] + c;
        wv[i] = (uint32_t)t;
        c = t >> 32;
      }
      carry += c;
    }
  }
  // ---- the row's first lane collects the words and finishes the row
  uint32_t W[SW];
#pragma unroll
  for (int i = 0; i < 8; i++) W[i] = wv[i];
#pragma unroll
  for (int q = 1; q < T; q++)
#pragma unroll
    for (int i = 0; i < 8; i++) W[8 * q + i] = __shfl_down_sync(0xffffffffu, wv[i], q);
  const int64_t top = __shfl_down_sync(0xffffffffu, carry, T - 1);  // value of words >= 8T
  if (sl != 0 || !active) return;
  int64_t acc2[L + 1];
#pragma unroll
  for (int i = 0; i < L; i++) acc2[i] = W[i];
  {
    uint64_t hi = (uint64_t)top;  // value of words >= L, fits int64 by the row bound
#pragma unroll
    for (int k = SW - 1; k >= L; k--) hi = (hi << 32) + W[k];
    acc2[L] = (int64_t)hi;
  }
  // Lazy partials between the passes (SW >= L + 2): a pass that is not the
  // last stores its row value V exactly -- words 0..L-1 and the signed int64
  // of the words above -- instead of reducing it; the next pass adds it to
  // its sums and only the last pass runs Barrett.  |V| < 2^47 ell per pass
  // (the row bounds of mat_build), so the words above L stay below 2^48 in
  // total over the passes.  Saves one L-limb Barrett per row and pass, run by
  // one lane of T (cfg5: ~0.1 ms per extra pass).
  if (!FIRST && !LAZY) {
    uint32_t pin[SW];
    load_slot<SW>(a.part_in + (size_t)slot * SW, pin, pol);
#pragma unroll
    for (int i = 0; i < L; i++) acc2[i] += pin[i];
  }
  if constexpr (LAZY && !LAST) {
    uint32_t o[SW];
    int64_t c = 0;
#pragma unroll
    for (int i = 0; i < L; i++) {
      const int64_t t = acc2[i] + c;
      o[i] = (uint32_t)t;
      c = t >> 32;
    }
    const int64_t hi = acc2[L] + c;
    o[L] = (uint32_t)hi;
    o[L + 1] = (uint32_t)((uint64_t)hi >> 32);
#pragma unroll
    for (int i = L + 2; i < SW; i++) o[i] = 0u;
    uint32_t* dst = a.part_out + (size_t)slot * SW;
    if (a.policy & 4) store_slot_hint<SW>(dst, o, pol);
    else store_slot<SW>(dst, o);
    return;
  }
  // (full-class entries and dense columns: full_fixup after the last pass --
  // their Montgomery products inline made every row of the last pass spill)
  uint32_t Rr[L];
  finalize<L>(acc2, 0, mp, Rr);
  store_row<L, 1, LAST>(a, slot, 0, Rr, pol);
}

// The full-class entries and dense columns of the rows that have them, added
// to the finished product after the last limb-sliced pass: y[row] <- y[row] +
// sum f u mod ell (one thread per listed slot; y canonical in biased form)
template <int L>
__global__ void __launch_bounds__(128) full_fixup(const SpmvArgs a, const ModParams mp,
                                                  const int32_t* __restrict__ fix_slots, int64_t nfix) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nfix) return;
  const int64_t slot = fix_slots[i];
  const int32_t row = a.slot_row[slot];
  if (row < 0) return;
  const uint32_t* cur = a.npeer ? a.yp[0] + (size_t)(a.peer_off + row) * SW : a.y + (size_t)row * SW;
  int64_t acc[L + 1];
#pragma unroll
  for (int j = 0; j < L; j++) acc[j] = cur[j] ^ 0x80000000u;
  acc[L] = 0;
  row_full<L, 1>(a, mp, slot, row, a.x, acc);
  uint32_t Rr[L];
  finalize<L>(acc, 0, mp, Rr);
  store_row<L, 1, true>(a, slot, 0, Rr, 0);
}

// ------------------------------------------------- die-split SpMV pass
//
// B200 is two dies, and each die's L2 keeps its own copy of every line its
// SMs read: a randomly gathered working set thrashes beyond ~one die's L2
// (~63 MB) when every SM gathers every column, but stays resident up to
// ~128 MB when the SMs of die d only gather the columns of half d
// (tools/microbench/mb3.cu, profiles/microbench3_r01.txt).  The columns are
// therefore dealt to two halves (interleaved chunks, sized to the dies' SM
// counts) and every row gets one partial result per half:
//  * a persistent grid; each CTA finds its die from %smid (die map probed at
//    context creation) and warps take slices from that die's work queue,
//    then steal from the other queue once theirs is empty (correctness
//    never depends on where CTAs land);
//  * the two partial results of a row meet through an exchange buffer: the
//    first half to finish a slice (per-slice arrival counter) publishes its
//    canonical values there; the second adds them mod ell and writes the
//    rows.  Counters grow by 4 per pass, so their residue mod 4 marks the
//    order without ever being reset;
//  * half 0 also carries the previous pass's partial and, on the last pass,
//    the full-class entries and dense columns;
//  * the last warp to leave resets the work queues for the next launch.
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

// r = a + b mod ell for canonical a, b
template <int L>
__device__ __forceinline__ void add_canonical(const uint32_t (&a_)[L], const uint32_t (&b)[L],
                                              const ModParams& mp, uint32_t (&r)[L]) {
  uint32_t s[L];
  uint64_t c = 0;
#pragma unroll
  for (int j = 0; j < L; j++) {
    c = (uint64_t)a_[j] + b[j] + (c >> 32);
    s[j] = (uint32_t)c;
  }
  const int64_t top = (int64_t)(c >> 32);
  int64_t br = 0;
  uint32_t d[L];
#pragma unroll
  for (int j = 0; j < L; j++) {
    const int64_t v = (int64_t)s[j] - mp.ell[j] + br;
    d[j] = (uint32_t)v;
    br = v >> 32;
  }
  const bool ge = top + br >= 0;  // s >= ell
#pragma unroll
  for (int j = 0; j < L; j++) r[j] = ge ? d[j] : s[j];
}

constexpr int SPLIT_GRAB = 2;  // slices a warp takes per queue ticket

template <int L, int G, bool FIRST, bool LAST>
__global__ void __launch_bounds__(256, spmv_min_blocks<L>()) spmv_split(const SpmvArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int R = 32 / G;
  const int lane = threadIdx.x & 31;
  const int chain = lane & (G - 1);
  const int rw = lane / G;
  if (FIRST) unit_projection<L, G>(a);

  const uint64_t pol = policy_evict_first();
  const uint64_t gpol = (a.policy & 1) ? policy_evict_last() : createpolicy_normal();
  const uint32_t* xc = a.x + (size_t)chain * SW;
  const int home = a.die_map[sm_id() & 255];
  const uint32_t nsl = (uint32_t)a.nslices;
#pragma unroll 1
  for (int pass_h = 0; pass_h < 2; pass_h++) {
    const int h = home ^ pass_h;  // own die's queue first, then help the other
    const SliceInfo* slices = a.slices + (size_t)h * a.nslices;
    const uint32_t* lk = a.lane_k4 + (size_t)h * a.nslots;
#pragma unroll 1
    while (true) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(a.queue + h, SPLIT_GRAB);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= nsl) break;
#pragma unroll 1
      for (uint32_t slice = base; slice < min(base + SPLIT_GRAB, nsl); slice++) {
        const int64_t slot = (int64_t)slice * R + rw;
        const SliceInfo si = slices[slice];
        int64_t acc[L + 1];
#pragma unroll
        for (int i = 0; i <= L; i++) acc[i] = 0;
        int64_t S = 0;
        row_entries<L, G>(a, si, lk[slot], rw, xc, pol, gpol, acc, S);
        if (h == 0) {
          if (!FIRST) {
            uint32_t pin[SW];
            load_slot<SW>(a.part_in + ((size_t)slot * G + chain) * SW, pin, pol);
#pragma unroll
            for (int i = 0; i < L; i++) acc[i] += pin[i];
          }
          if (LAST && a.has_full) row_full<L, G>(a, mp, slot, a.slot_row[slot], xc, acc);
        }
        uint32_t Rr[L];
        finalize<L>(acc, S, mp, Rr);
        // meet the other half: arrival counter +1 each, +2 when the first
        // has published its value, so it grows by 4 per pass and
        //   old % 4 == 0: first -> publish, signal
        //   old % 4 == 3: second, value already published
        //   old % 4 == 1: second, first still publishing (a few hundred
        //                 cycles: it has finished its rows) -> wait
        uint32_t old = 0;
        if (lane == 0) old = atomicAdd(a.cnt + slice, 1u);
        old = __shfl_sync(0xffffffffu, old, 0) & 3u;
        uint32_t* xs = a.xch + ((size_t)slot * G + chain) * SW;
        if (old == 0) {
          uint32_t o[SW];
#pragma unroll
          for (int i = 0; i < SW; i++) o[i] = i < L ? Rr[i] : 0u;
          if (a.policy & 16) store_slot_hint<SW>(xs, o, pol);
          else store_slot<SW>(xs, o);
          __syncwarp();  // (the grid-barrier pattern: warp barrier, one fenced atomic)
          if (lane == 0) {
            __threadfence();
            atomicAdd(a.cnt + slice, 2u);
          }
        } else {
          if (lane == 0) {
            if (old == 1) {
              uint32_t c;
              do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(a.cnt + slice) : "memory");
              } while (c & 3u);
            }
            __threadfence();
          }
          __syncwarp();
          uint32_t pv[SW], P[L];
#pragma unroll
          for (int q = 0; q < SW / 8; q++)
            asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(pv[8 * q + 0]), "=r"(pv[8 * q + 1]), "=r"(pv[8 * q + 2]), "=r"(pv[8 * q + 3]),
                           "=r"(pv[8 * q + 4]), "=r"(pv[8 * q + 5]), "=r"(pv[8 * q + 6]), "=r"(pv[8 * q + 7])
                         : "l"(xs + 8 * q)
                         : "memory");
#pragma unroll
          for (int i = 0; i < L; i++) P[i] = pv[i];
          uint32_t Sum[L];
          add_canonical<L>(Rr, P, mp, Sum);
          store_row<L, G, LAST>(a, slot, chain, Sum, pol);
        }
      }
    }
  }
  // the last warp out resets the queues for the next launch
  if (lane == 0) {
    const uint32_t total = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(a.queue + 2, 1u) == total - 1) {
      a.queue[0] = 0;
      a.queue[1] = 0;
      a.queue[2] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------ conversion kernels

// item i of a chain-major host array (chain i / rows, row i % rows) lives in
// slot record row * G + chain on the device
template <int L>
__global__ void limbs_to_slots(const uint32_t* __restrict__ limbs, int64_t n, uint32_t* __restrict__ out,
                               uint32_t bias, int64_t rows, int G) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t slot = (i % rows) * G + i / rows;
  uint32_t o[SW];
#pragma unroll
  for (int j = 0; j < SW; j++) o[j] = j < L ? (limbs[(size_t)i * L + j] ^ bias) : 0u;
  store_slot<SW>(out + (size_t)slot * SW, o);
}

template <int L>
__global__ void slots_to_limbs(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ limbs,
                               uint32_t bias, int64_t rows, int G) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t slot = (i % rows) * G + i / rows;
#pragma unroll
  for (int j = 0; j < L; j++) limbs[(size_t)i * L + j] = in[(size_t)slot * SW + j] ^ bias;
}

// in-place Montgomery conversion f -> f R mod ell = montmul(f, R^2)
template <int L>
__global__ void to_montgomery(uint32_t* __restrict__ slots, int64_t n, const ModParams mp) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t f[L], r[L];
#pragma unroll
  for (int j = 0; j < L; j++) f[j] = slots[(size_t)i * SW + j];
  montmul<L>(f, mp.R2, mp, r);
#pragma unroll
  for (int j = 0; j < L; j++) slots[(size_t)i * SW + j] = r[j];
}

// dst = sum_k src_k mod ell over n slots (biased format); k <= 64 so the
// per-limb sums stay below 2^38 and the row value below 2^47 ell
struct AddModArgs {
  const uint32_t* src[64];
  uint32_t* dst;
  int k;
  int64_t n;
};

template <int L>
__global__ void add_mod_kernel(const AddModArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int64_t acc[L + 1];
#pragma unroll
  for (int j = 0; j <= L; j++) acc[j] = 0;
  for (int s = 0; s < a.k; s++) {
    const uint32_t* p = a.src[s] + (size_t)i * SW;
#pragma unroll
    for (int j = 0; j < L; j++) acc[j] += p[j] ^ 0x80000000u;
  }
  uint32_t R[L];
  finalize<L>(acc, 0, mp, R);
  uint32_t o[SW];
#pragma unroll
  for (int j = 0; j < SW; j++) o[j] = j < L ? (R[j] ^ 0x80000000u) : 0u;
  store_slot<SW>(a.dst + (size_t)i * SW, o);
}

// dst = acc + sum_j c_j y_j mod ell (Mksol's Horner combination,
// solver.py:522-536): c_j in Montgomery form (c R mod ell) so one CIOS
// product gives c_j y_j mod ell < ell; acc / y_j / dst in biased slots.
struct LinCombArgs {
  const uint32_t* y[64];
  const uint32_t* coef;  // k coefficients, SW words each: plain (L <= 8, lazy) or Montgomery form
  const uint32_t* acc;   // optional
  uint32_t* dst;
  const uint32_t* fold;  // L <= 8: 2^(32k) mod ell for k = L .. (L words each)
  int k;
  int64_t n;
};

// dst = acc + sum_s c_s y_s mod ell for L <= 8, reduced once per element:
// each 16-bit digit of c_s times each 32-bit limb of y_s[i] (< 2^48) goes into
// a 64-bit column of weight 2^(16 c) by one IMAD.WIDE (2 L^2 per term, no
// Montgomery reduction); the columns are carried into 32-bit limbs, the limbs
// above L folded with 2^(32k) mod ell, and finalize<L> reduces.  k <= 64:
// every column stays below 64 x L x 2^48 < 2^57.
template <int L>
__global__ void __launch_bounds__(256) lincomb_lazy_kernel(const LinCombArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int C = 4 * L - 2;  // columns p + 2j, p < 2L, j < L
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  uint64_t col[C];
#pragma unroll
  for (int c = 0; c < C; c++) col[c] = 0;
  if (a.acc) {
#pragma unroll
    for (int j = 0; j < L; j++) col[2 * j] += a.acc[(size_t)i * SW + j] ^ 0x80000000u;
  }
  for (int s = 0; s < a.k; s++) {
    uint32_t u[SW];
    gather<SW>(a.y[s] + (size_t)i * SW, u);
    const uint32_t* cw = a.coef + (size_t)s * SW;
#pragma unroll
    for (int p = 0; p < 2 * L; p++) {
      const uint32_t w = __ldg(cw + (p >> 1));
      const uint32_t d = (p & 1) ? (w >> 16) : (w & 0xFFFFu);
#pragma unroll
      for (int j = 0; j < L; j++) col[p + 2 * j] += (uint64_t)d * (u[j] ^ 0x80000000u);
    }
  }
  // 16-bit columns -> 32-bit limbs V[0 .. 2L-2] + the rest `top`
  constexpr int K = C / 2;
  uint32_t V[K];
  uint64_t carry = 0;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const uint64_t lo = col[2 * k] + carry;
    const uint64_t hi = col[2 * k + 1] + (lo >> 16);
    V[k] = (uint32_t)((lo & 0xFFFFu) | ((hi & 0xFFFFu) << 16));
    carry = hi >> 16;
  }
  int64_t acc[L + 1];
#pragma unroll
  for (int j = 0; j < L; j++) acc[j] = V[j];
  acc[L] = 0;
#pragma unroll
  for (int k = L; k <= K + 1; k++) {
    const uint32_t limb = k < K ? V[k] : (k == K ? (uint32_t)carry : (uint32_t)(carry >> 32));
    const uint32_t* R = a.fold + (size_t)(k - L) * L;
#pragma unroll
    for (int j = 0; j < L; j++) {
      const uint64_t pr = (uint64_t)limb * __ldg(R + j);
      acc[j] += (int64_t)(uint32_t)pr;
      acc[j + 1] += (int64_t)(pr >> 32);
    }
  }
  uint32_t Rr[L];
  finalize<L>(acc, 0, mp, Rr);
  uint32_t o[SW];
#pragma unroll
  for (int j = 0; j < SW; j++) o[j] = j < L ? (Rr[j] ^ 0x80000000u) : 0u;
  store_slot<SW>(a.dst + (size_t)i * SW, o);
}

template <int L>
__global__ void lincomb_kernel(const LinCombArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int64_t acc[L + 1];
#pragma unroll
  for (int j = 0; j <= L; j++) acc[j] = 0;
  if (a.acc) {
#pragma unroll
    for (int j = 0; j < L; j++) acc[j] += a.acc[(size_t)i * SW + j] ^ 0x80000000u;
  }
  for (int s = 0; s < a.k; s++) {
    uint32_t u[L], c[L], r[L];
#pragma unroll
    for (int j = 0; j < L; j++) {
      u[j] = a.y[s][(size_t)i * SW + j] ^ 0x80000000u;
      c[j] = a.coef[(size_t)s * SW + j];
    }
    montmul<L>(c, u, mp, r);
#pragma unroll
    for (int j = 0; j < L; j++) acc[j] += r[j];
  }
  uint32_t R[L];
  finalize<L>(acc, 0, mp, R);
  uint32_t o[SW];
#pragma unroll
  for (int j = 0; j < SW; j++) o[j] = j < L ? (R[j] ^ 0x80000000u) : 0u;
  store_slot<SW>(a.dst + (size_t)i * SW, o);
}

// *flag |= 1 if any of the n residues is non-zero
template <int L>
__global__ void nonzero_kernel(const uint32_t* __restrict__ v, int64_t n, int* flag) {
  constexpr int SW = stride_words(L);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool nz = false;
  if (i < n) {
#pragma unroll
    for (int j = 0; j < L; j++) nz |= (v[(size_t)i * SW + j] ^ 0x80000000u) != 0u;
  }
  if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// out[t] = canonical limbs of slot rows[t]
template <int L>
__global__ void read_rows_kernel(const uint32_t* __restrict__ v, const int64_t* __restrict__ rows, int m,
                                 uint32_t* __restrict__ out) {
  constexpr int SW = stride_words(L);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
#pragma unroll
  for (int j = 0; j < L; j++) out[(size_t)t * L + j] = v[(size_t)rows[t] * SW + j] ^ 0x80000000u;
}

// zero residue in biased form (the padding target slot)
template <int L>
__global__ void set_zero_slot(uint32_t* slot) {
  constexpr int SW = stride_words(L);
  const int j = threadIdx.x;
  if (j < SW) slot[j] = j < L ? 0x80000000u : 0u;
}

}  // namespace sld

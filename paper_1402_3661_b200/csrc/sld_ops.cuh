// sld_ops.cuh -- per-limb-count kernel dispatch table.  Each translation
// unit sld_inst_<g>.cu instantiates the kernels for a range of L (so the
// 32 widths compile in parallel) and fills its slice of the table.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "sld_dense.cuh"
#include "sld_device.cuh"
#include "sld_tcgemm.cuh"

namespace sld {

// chains per record the SpMV supports for L limbs: a record must fit one
// 128-byte line (G * SW * 4 <= 128), so G = 2 up to 16 limbs, 4 up to 8
__host__ __device__ constexpr int max_chains(int L) { return L <= 8 ? 4 : (L <= 16 ? 2 : 1); }

struct LOps {
  // returns false if G is not supported for this L
  bool (*pass)(int G, int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a,
               const ModParams& mp);
  // die-split pass on a persistent grid of `grid` CTAs (false: G unsupported)
  bool (*split)(int G, int first, int last, unsigned grid, cudaStream_t s, const SpmvArgs& a,
                const ModParams& mp);
  // resident CTAs per SM of the die-split kernel for G chains (0: unsupported)
  int (*split_occupancy)(int G);
  // short-row pass: 4 lanes per row, one chain (false: L > 8)
  bool (*short_pass)(int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a, const ModParams& mp);
  // limb-sliced pass for one chain (false: L <= 8, no slicing)
  bool (*wide)(int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a, const ModParams& mp);
  void (*limbs_to_slots)(const uint32_t*, int64_t, uint32_t*, uint32_t, int64_t, int, cudaStream_t);
  void (*slots_to_limbs)(const uint32_t*, int64_t, uint32_t*, uint32_t, int64_t, int, cudaStream_t);
  void (*to_mont)(uint32_t*, int64_t, const ModParams&, cudaStream_t);
  void (*zero_slot)(uint32_t*, cudaStream_t);
  void (*dense_proj)(const DenseProjArgs&, const ModParams&, cudaStream_t);
  // tensor-core dense projection (L <= 8): tile X once; per step tile v,
  // digit GEMM, fold.  False when L > 8.
  bool (*tc_tile_x)(const uint32_t* x, int m, int64_t n, int MT, int64_t ktiles, uint8_t* A, cudaStream_t s);
  // tensor-core Mksol combination (L <= 8, n <= 8): tile the y set once, combine per step
  bool (*tcl_tile)(const uint32_t* const* ys_dev, int n, int64_t rows, int64_t mtiles, uint8_t* Y,
                   const int32_t* perm, cudaStream_t s);
  bool (*tcl_apply)(const uint8_t* Y, const TclCoef& cf, int n, int64_t rows, int64_t mtiles, int grid,
                    const uint32_t* acc, uint32_t* dst, const uint32_t* fold, const ModParams& mp, cudaStream_t s);
  // K (2 or 4) Horner steps' combinations in one pass over the tiled y set
  bool (*tcl_batch)(int K, const uint8_t* Y, const uint32_t* coefs, int n, int64_t rows, int64_t mtiles, int sms,
                    uint32_t* const* dsts, const uint32_t* fold, const ModParams& mp, cudaStream_t s);
  bool (*tc_project)(const uint32_t* v, int64_t n, int m, int MT, int64_t ktiles, const uint8_t* A, uint8_t* B,
                     uint32_t* partial, int nct, int64_t kt_per_cta, const uint32_t* fold, const ModParams& mp,
                     uint32_t* out, cudaStream_t s);
  void (*add_mod)(const AddModArgs&, const ModParams&, cudaStream_t);
  void (*read_rows)(const uint32_t*, const int64_t*, int, uint32_t*, cudaStream_t);
  void (*lincomb)(const LinCombArgs&, const ModParams&, cudaStream_t);
  void (*nonzero)(const uint32_t*, int64_t, int*, cudaStream_t);
  // fused Mksol step: last pass of a one-chain product with the combination
  // in its epilogue; slot-order copy of a y vector (false: L > 8)
  bool (*pass_mk)(int first, int64_t nslices, cudaStream_t s, const SpmvArgs& a, const ModParams& mp);
  bool (*mk_gather)(const uint32_t* y, const int32_t* slot_row, int64_t nslots, uint32_t* out, cudaStream_t s);
  // full-class entries / dense columns of the listed slots, after the last
  // limb-sliced pass (L > 8)
  void (*fixup)(const SpmvArgs& a, const ModParams& mp, const int32_t* slots, int64_t n, cudaStream_t s);
  // persistent chain of short-row products (L <= 8): resident CTAs per SM
  // (0: unsupported), and the cooperative launch of `grid` CTAs
  int (*chain_occupancy)(int l1g, int tb, size_t smem);
  cudaError_t (*chain)(int l1g, unsigned grid, int tb, size_t smem, cudaStream_t s, const SpmvArgs& a,
                       const ModParams& mp, const ChainArgs& ch);
};

constexpr int SHORT_TB = 64;  // threads per CTA of the short-row pass (env SLD_SHORT_TB)

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int L, int G>
void launch_pass(int first, int last, unsigned grid, cudaStream_t s, const SpmvArgs& a,
                 const ModParams& mp) {
  if (first && last) spmv_pass<L, G, true, true><<<grid, 256, 0, s>>>(a, mp);
  else if (first) spmv_pass<L, G, true, false><<<grid, 256, 0, s>>>(a, mp);
  else if (last) spmv_pass<L, G, false, true><<<grid, 256, 0, s>>>(a, mp);
  else spmv_pass<L, G, false, false><<<grid, 256, 0, s>>>(a, mp);
}

template <int L, int G>
void launch_split(int first, int last, unsigned grid, cudaStream_t s, const SpmvArgs& a,
                  const ModParams& mp) {
  if (first && last) spmv_split<L, G, true, true><<<grid, 256, 0, s>>>(a, mp);
  else if (first) spmv_split<L, G, true, false><<<grid, 256, 0, s>>>(a, mp);
  else if (last) spmv_split<L, G, false, true><<<grid, 256, 0, s>>>(a, mp);
  else spmv_split<L, G, false, false><<<grid, 256, 0, s>>>(a, mp);
}

template <int L, int G>
int split_occ() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_split<L, G, false, false>, 256, 0) != cudaSuccess)
    return 0;
  return n;
}

template <int MT>
void launch_tc_gemm_mt(int nct, int64_t ktiles, int64_t kpc, const uint8_t* A, const uint8_t* B, uint32_t* partial,
                       cudaStream_t s) {
  static bool attr = [] {
    cudaFuncSetAttribute(tc_digit_gemm<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(MT));
    return true;
  }();
  (void)attr;
  tc_digit_gemm<MT><<<nct, TC_THREADS, tc_smem_bytes(MT), s>>>(A, B, ktiles, kpc, partial);
}

inline void launch_tc_gemm(int MT, int nct, int64_t ktiles, int64_t kpc, const uint8_t* A, const uint8_t* B,
                           uint32_t* partial, cudaStream_t s) {
  switch (MT) {
    case 1: launch_tc_gemm_mt<1>(nct, ktiles, kpc, A, B, partial, s); break;
    case 2: launch_tc_gemm_mt<2>(nct, ktiles, kpc, A, B, partial, s); break;
    case 3: launch_tc_gemm_mt<3>(nct, ktiles, kpc, A, B, partial, s); break;
    default: launch_tc_gemm_mt<4>(nct, ktiles, kpc, A, B, partial, s); break;
  }
}

template <int L>
struct Ops {
  static bool pass(int G, int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a,
                   const ModParams& mp) {
    const unsigned grid = blocks_for(nslices * 32, 256);  // one warp per slice
    if (G == 1) {
      if (grid) launch_pass<L, 1>(first, last, grid, s, a, mp);
      return true;
    }
    if constexpr (max_chains(L) >= 2) {
      if (G == 2) {
        if (grid) launch_pass<L, 2>(first, last, grid, s, a, mp);
        return true;
      }
    }
    if constexpr (max_chains(L) >= 4) {
      if (G == 4) {
        if (grid) launch_pass<L, 4>(first, last, grid, s, a, mp);
        return true;
      }
    }
    return false;
  }
  static bool split(int G, int first, int last, unsigned grid, cudaStream_t s, const SpmvArgs& a,
                    const ModParams& mp) {
    if (G == 1) {
      launch_split<L, 1>(first, last, grid, s, a, mp);
      return true;
    }
    if constexpr (max_chains(L) >= 2) {
      if (G == 2) {
        launch_split<L, 2>(first, last, grid, s, a, mp);
        return true;
      }
    }
    if constexpr (max_chains(L) >= 4) {
      if (G == 4) {
        launch_split<L, 4>(first, last, grid, s, a, mp);
        return true;
      }
    }
    return false;
  }
  static int split_occupancy(int G) {
    if (G == 1) return split_occ<L, 1>();
    if constexpr (max_chains(L) >= 2)
      if (G == 2) return split_occ<L, 2>();
    if constexpr (max_chains(L) >= 4)
      if (G == 4) return split_occ<L, 4>();
    return 0;
  }
  static bool shortp(int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a,
                     const ModParams& mp) {
    if constexpr (L <= 8) {
      // small CTAs spread the few slices of a small matrix evenly over the SMs
      // (each SM gathers ~1 residue per clock)
      static const int tb = getenv("SLD_SHORT_TB") ? atoi(getenv("SLD_SHORT_TB")) : SHORT_TB;
      const unsigned grid = blocks_for(nslices * 32, tb);
      if (!grid) return true;
      // programmatic dependent launch: this product's CTAs become resident
      // while the previous product drains.  Only where the whole grid fits
      // beside the previous one, or both are multi-wave: cfg1's size (only
      // part of the next grid fits) measured slower with it (20k rows 6.55
      // vs 6.14 us; 3k rows 4.27 vs 4.59, 60k rows 11.61 vs 12.02 with it,
      // profiles/pdl_short_r02.txt).
      // SLD_PDL=0 off, =1 always.
      static const int pdl_mode = getenv("SLD_PDL") ? atoi(getenv("SLD_PDL")) : 2;
      bool pdl = pdl_mode != 0;
      if (pdl_mode == 2) {
        static const int64_t cap = [] {  // resident CTAs of one grid (thread-safe init)
          int per_sm = 0, dev = 0, sms = 0;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_short<L, true, true>, tb, 0);
          return (int64_t)per_sm * sms;
        }();
        pdl = 2 * (int64_t)grid <= cap || (int64_t)grid > cap;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(tb);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      if (first && last) cudaLaunchKernelEx(&cfg, spmv_short<L, true, true>, a, mp);
      else if (first) cudaLaunchKernelEx(&cfg, spmv_short<L, true, false>, a, mp);
      else if (last) cudaLaunchKernelEx(&cfg, spmv_short<L, false, true>, a, mp);
      else cudaLaunchKernelEx(&cfg, spmv_short<L, false, false>, a, mp);
      return true;
    }
    return false;
  }
  static bool wide(int first, int last, int64_t nslices, cudaStream_t s, const SpmvArgs& a,
                   const ModParams& mp) {
    if constexpr (wide_T<L>() >= 2) {
      const unsigned grid = blocks_for(nslices * 32, 256);
      if (!grid) return true;
      if (first && last) spmv_wide<L, true, true><<<grid, 256, 0, s>>>(a, mp);
      else if (first) spmv_wide<L, true, false><<<grid, 256, 0, s>>>(a, mp);
      else if (last) spmv_wide<L, false, true><<<grid, 256, 0, s>>>(a, mp);
      else spmv_wide<L, false, false><<<grid, 256, 0, s>>>(a, mp);
      return true;
    }
    return false;
  }
  static void l2s(const uint32_t* l, int64_t n, uint32_t* o, uint32_t b, int64_t rows, int G,
                  cudaStream_t s) {
    if (n) limbs_to_slots<L><<<blocks_for(n, 256), 256, 0, s>>>(l, n, o, b, rows, G);
  }
  static void s2l(const uint32_t* i, int64_t n, uint32_t* l, uint32_t b, int64_t rows, int G,
                  cudaStream_t s) {
    if (n) slots_to_limbs<L><<<blocks_for(n, 256), 256, 0, s>>>(i, n, l, b, rows, G);
  }
  static void mont(uint32_t* x, int64_t n, const ModParams& mp, cudaStream_t s) {
    if (n) to_montgomery<L><<<blocks_for(n, 128), 128, 0, s>>>(x, n, mp);
  }
  static void zero(uint32_t* slot, cudaStream_t s) { set_zero_slot<L><<<1, 32, 0, s>>>(slot); }
  static void dproj(const DenseProjArgs& a, const ModParams& mp, cudaStream_t s) {
    dense_project_launch<L>(a, mp, s);
  }
  static bool tctx(const uint32_t* x, int m, int64_t n, int MT, int64_t ktiles, uint8_t* A, cudaStream_t s) {
    if constexpr (L <= 8) {
      tc_tile_x<L><<<(unsigned)(ktiles * MT), 128, 0, s>>>(x, m, n, MT, ktiles, A);
      return true;
    }
    return false;
  }
  static bool tcltile(const uint32_t* const* ys, int n, int64_t rows, int64_t mtiles, uint8_t* Y, const int32_t* perm,
                      cudaStream_t s) {
    if constexpr (L <= 8) {
      const int64_t cores = mtiles * n * 32;
      tcl_tile_y<L><<<blocks_for(cores, 128), 128, 0, s>>>(ys, n, rows, mtiles, Y, perm);
      return true;
    }
    return false;
  }
  static bool tclapply(const uint8_t* Y, const TclCoef& cf, int n, int64_t rows, int64_t mtiles, int grid,
                       const uint32_t* acc, uint32_t* dst, const uint32_t* fold, const ModParams& mp,
                       cudaStream_t s) {
    if constexpr (L <= 8) {
      static bool attr = [] {
        cudaFuncSetAttribute(tcl_combine<L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tcl_smem_bytes(8));
        return true;
      }();
      (void)attr;
      TclBatch<1> b;
      memcpy(b.w[0], cf.w, sizeof(cf.w));
      b.dst[0] = dst;
      tcl_combine<L, 1><<<grid, TCL_THREADS, tcl_smem_bytes(n), s>>>(Y, b, n, rows, mtiles, acc, fold, mp);
      return true;
    }
    return false;
  }
  template <int K>
  static bool tclbatch_k(const uint8_t* Y, const uint32_t* coefs, int n, int64_t rows, int64_t mtiles, int sms,
                         uint32_t* const* dsts, const uint32_t* fold, const ModParams& mp, cudaStream_t s) {
    static const int occ = [] {
      cudaFuncSetAttribute(tcl_combine<L, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, tcl_smem_bytes(8, K));
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, tcl_combine<L, K>, tcl_threads(K), tcl_smem_bytes(8, K));
      return std::max(1, o);
    }();
    TclBatch<K> b;
    memset(&b, 0, sizeof(b));
    for (int k = 0; k < K; k++) {
      for (int j = 0; j < n; j++)
        for (int i = 0; i < L; i++) b.w[k][j][i] = coefs[((size_t)k * n + j) * L + i];
      b.dst[k] = dsts[k];
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(mtiles, (int64_t)occ * sms));
    tcl_combine<L, K><<<grid, tcl_threads(K), tcl_smem_bytes(n, K), s>>>(Y, b, n, rows, mtiles, nullptr, fold, mp);
    return true;
  }
  // K in {2, 4} steps' combinations in one pass over Y' (coefs: [K][n][L] canonical)
  static bool tclbatch(int K, const uint8_t* Y, const uint32_t* coefs, int n, int64_t rows, int64_t mtiles,
                       int sms, uint32_t* const* dsts, const uint32_t* fold, const ModParams& mp, cudaStream_t s) {
    if constexpr (L <= 8) {
      if (!mtiles) return true;
      if (K == 2) return tclbatch_k<2>(Y, coefs, n, rows, mtiles, sms, dsts, fold, mp, s);
      if (K == 4) return tclbatch_k<4>(Y, coefs, n, rows, mtiles, sms, dsts, fold, mp, s);
    }
    return false;
  }
  static bool tcproj(const uint32_t* v, int64_t n, int m, int MT, int64_t ktiles, const uint8_t* A, uint8_t* B,
                     uint32_t* partial, int nct, int64_t kt_per_cta, const uint32_t* fold, const ModParams& mp,
                     uint32_t* out, cudaStream_t s) {
    if constexpr (L <= 8) {
      tc_tile_v<L><<<(unsigned)ktiles, 128, 0, s>>>(v, n, ktiles, B);
      launch_tc_gemm(MT, nct, ktiles, kt_per_cta, A, B, partial, s);
      tc_proj_final<L><<<m, 1024, 0, s>>>(partial, nct, MT, fold, mp, out);
      return true;
    }
    return false;
  }
  static void addm(const AddModArgs& a, const ModParams& mp, cudaStream_t s) {
    if (a.n) add_mod_kernel<L><<<blocks_for(a.n, 128), 128, 0, s>>>(a, mp);
  }
  static void rrows(const uint32_t* v, const int64_t* r, int m, uint32_t* o, cudaStream_t s) {
    if (m) read_rows_kernel<L><<<blocks_for(m, 128), 128, 0, s>>>(v, r, m, o);
  }
  static void lcomb(const LinCombArgs& a, const ModParams& mp, cudaStream_t s) {
    if (!a.n) return;
    if constexpr (L <= 8) lincomb_lazy_kernel<L><<<blocks_for(a.n, 256), 256, 0, s>>>(a, mp);
    else lincomb_kernel<L><<<blocks_for(a.n, 128), 128, 0, s>>>(a, mp);
  }
  static void nz(const uint32_t* v, int64_t n, int* f, cudaStream_t s) {
    if (n) nonzero_kernel<L><<<blocks_for(n, 256), 256, 0, s>>>(v, n, f);
  }
  static bool passmk(int first, int64_t nslices, cudaStream_t s, const SpmvArgs& a, const ModParams& mp) {
    if constexpr (L <= 8) {
      const unsigned grid = blocks_for(nslices * 32, 256);
      if (!grid) return true;
      if (first) spmv_pass<L, 1, true, true, true><<<grid, 256, 0, s>>>(a, mp);
      else spmv_pass<L, 1, false, true, true><<<grid, 256, 0, s>>>(a, mp);
      return true;
    }
    return false;
  }
  static bool mkgather(const uint32_t* y, const int32_t* slot_row, int64_t nslots, uint32_t* out, cudaStream_t s) {
    if constexpr (L <= 8) {
      if (nslots) mk_slot_gather<L><<<blocks_for(nslots, 256), 256, 0, s>>>(y, slot_row, nslots, out);
      return true;
    }
    return false;
  }
  static void fix(const SpmvArgs& a, const ModParams& mp, const int32_t* slots, int64_t n, cudaStream_t s) {
    if (n) full_fixup<L><<<blocks_for(n, 128), 128, 0, s>>>(a, mp, slots, n);
  }
  static int chain_occ(int l1g, int tb, size_t smem) {
    if constexpr (L <= 8) {
      const void* f = l1g ? (const void*)spmv_chain<L, true> : (const void*)spmv_chain<L, false>;
      if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
      int n = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, tb, smem) != cudaSuccess) return 0;
      return n;
    }
    return 0;
  }
  static cudaError_t chainl(int l1g, unsigned grid, int tb, size_t smem, cudaStream_t s, const SpmvArgs& a,
                            const ModParams& mp, const ChainArgs& ch) {
    if constexpr (L <= 8) {
      SpmvArgs a2 = a;
      ModParams mp2 = mp;
      ChainArgs ch2 = ch;
      void* args[] = {&a2, &mp2, &ch2};
      const void* f = l1g ? (const void*)spmv_chain<L, true> : (const void*)spmv_chain<L, false>;
      return cudaLaunchCooperativeKernel(f, dim3(grid), dim3(tb), args, smem, s);
    }
    return cudaErrorNotSupported;
  }
  static LOps make() {
    return LOps{pass, split, split_occupancy, shortp, wide, l2s, s2l, mont, zero, dproj, tctx, tcltile, tclapply,
                tclbatch, tcproj, addm, rrows, lcomb, nz, passmk, mkgather, fix, chain_occ, chainl};
  }
};

template <int L, int LMIN>
void fill_ops_range(LOps* t) {
  t[L] = Ops<L>::make();
  if constexpr (L > LMIN) fill_ops_range<L - 1, LMIN>(t);
}

// defined in sld_inst_<g>.cu
void fill_ops_1_8(LOps* t);
void fill_ops_9_16(LOps* t);
void fill_ops_17_24(LOps* t);
void fill_ops_25_32(LOps* t);

}  // namespace sld

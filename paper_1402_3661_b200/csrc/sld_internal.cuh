// sld_internal.cuh -- the objects behind the C ABI handles and the helpers
// shared by the host translation units of libsldb200.so (sld_capi.cu, the
// matrix / vector / Krylov side; sld_grid.cu, the multi-GPU grid).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <string>

#include "sldb200.h"
#include "sld_ops.cuh"

using namespace sld;

// ------------------------------------------------------------ errors

// records the thread-local message sld_last_error() returns; returns code
int fail(int code, const char* fmt, ...);

#define CU(call)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(SLD_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                           \
  } while (0)

#define TRY(expr)              \
  do {                         \
    int r_ = (expr);           \
    if (r_ != SLD_OK) return r_; \
  } while (0)

// ------------------------------------------------------------ objects

struct sld_ctx {
  int dev = 0;
  int L = 0;
  int SW = 0;
  cudaStream_t stream = nullptr;   // the stream all work is issued on
  cudaStream_t own = nullptr;      // the context's own stream
  ModParams mp;
  size_t l2_bytes = 0;
  int sms = 0;
  void* hstage = nullptr;  // pinned host staging (limb format)
  size_t hstage_bytes = 0;
  void* dstage = nullptr;  // device staging (limb format)
  size_t dstage_bytes = 0;
  size_t apw_max = 0;      // max access-policy window bytes (0: unsupported)
  uint32_t* fold = nullptr;    // L <= 8: 2^(32k) mod ell, k = L .. TC_FOLD_TOP (lazy folds)
  uint32_t* coef = nullptr;    // lincomb coefficient staging (64 x SW words)
  uint8_t* die_map = nullptr;  // device copy of the %smid -> die map (256 entries)
  int die_n[2] = {0, 0};       // SMs per die; both 0 if the map is unavailable
  // lifetime: the owner's handle plus one reference per vector / matrix /
  // projection block / combination set made on this context, so handles may
  // be destroyed in any order (a garbage collector frees them in arbitrary
  // order) without touching a freed context
  std::atomic<int> refs{1};
};

void ctx_free(sld_ctx* c);
// host -> device copy ordered on `s` and complete on return.  A plain
// cudaMemcpy from pageable memory may return before its DMA has landed, and
// the context streams are non-blocking: a kernel queued right after it (a
// Montgomery conversion, the first product) could read the old bytes.
inline cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e;
}

inline void ctx_unref(sld_ctx* c) {
  if (c && c->refs.fetch_sub(1) == 1) ctx_free(c);
}
// a context reference held by an object made on it (released on delete)
struct CtxRef {
  sld_ctx* c = nullptr;
  void bind(sld_ctx* x) {
    c = x;
    if (c) c->refs.fetch_add(1);
  }
  ~CtxRef() { ctx_unref(c); }
};

struct sld_vec {
  CtxRef ref;
  sld_ctx* ctx = nullptr;
  int64_t n = 0;      // residues per chain
  int chains = 1;     // G chains interleaved per record (row*G + chain)
  uint32_t* buf[2] = {nullptr, nullptr};
  int cur = 0;
};

struct sld_xblock {
  CtxRef ref;
  sld_ctx* ctx = nullptr;
  int m = 0;
  int64_t n = 0;
  uint32_t* x = nullptr;     // [t][j] SW stride: plain (L <= 8, lazy dot products) or Montgomery form
  uint32_t* fold = nullptr;  // L <= 8: 2^(32k) mod ell for k = L .. TC_FOLD_TOP (L words each)
  // tensor-core projection (L <= 8, m <= 16): X as pre-tiled byte digits
  int MT = 0;                // 128-row M tiles (0: tensor-core path off)
  int64_t ktiles = 0;        // 128-byte K tiles (K = n)
  uint8_t* A = nullptr;      // [ktiles][MT][...] canonical K-major tiles
  uint8_t* B = nullptr;      // per-step v digits, [ktiles][...]
  uint32_t* partial = nullptr;
  int nct = 0;               // CTAs (split K)
  int64_t kt_per_cta = 0;
};

struct sld_mat {
  CtxRef ref;
  sld_ctx* ctx = nullptr;
  int64_t nrows = 0, ncols = 0, total_cols = 0, nnz = 0;
  int n_dense = 0;
  int npass = 1;
  int64_t stripe_cols = 0;
  int64_t nslices = 0;
  int64_t nslots = 0;
  int chains = 1;  // G chains per record (built for one G)
  int64_t n_pm = 0, n_small = 0, n_full = 0, pad_entries = 0;
  int64_t max_deg = 0;
  size_t dev_bytes = 0;
  int policy = 7;  // L2 policy bits (SpmvArgs::policy), measured best; env SLD_POLICY overrides
  int pf = 2;      // index prefetch distance in groups (0 for one-chain passes), measured; env SLD_PF overrides
  int apw = 0;       // persisting L2 access-policy window over the gathered stripe (env SLD_APW)
  float apw_ratio = 1.0f;
  // device
  SliceInfo* slices = nullptr;  // [npass][nslices]
  uint4* pm_idx = nullptr;
  uint4* s_idx = nullptr;
  int4* s_coef = nullptr;
  int32_t* slot_row = nullptr;
  uint32_t* lane_k4 = nullptr;  // [pass][slot]
  uint32_t* full_ptr = nullptr;
  uint32_t* full_col = nullptr;
  uint32_t* full_val = nullptr;
  uint32_t* dense_val = nullptr;
  uint32_t* part = nullptr;  // slot-indexed partials (npass > 1)
  // limb-sliced passes (one chain, L > 8): T lanes per row, 32 / T rows per slice
  int sliced = 0;
  int32_t* fix_slots = nullptr;  // sliced: slots with full-class entries (all rows with dense columns)
  int64_t n_fix = 0;
  // short-row passes (one chain, L <= 8, small N): 4 lanes per row, 8 rows per slice
  int short_rows = 0;
  int chain_ok = 0;                 // persistent chain kernel (opt-in, env SLD_CHAIN=1): measured slower
  uint32_t* chain_bar = nullptr;    // its grid-barrier counter
  int64_t chain_units = 0;          // largest slice's entry streams (uint4), pass 0
  // die split (halves == 2): each pass's columns are dealt to the two dies
  int halves = 1;
  // peer push (set by the grid, sld_grid.cu): the last pass stores into these buffers
  int npeer = 0;
  uint32_t* yp[8] = {nullptr};
  int64_t peer_off = 0;
  int64_t half_chunk = 0;      // columns per interleaved chunk
  unsigned split_grid = 0;     // persistent CTAs of the split kernel
  uint32_t* xch = nullptr;     // [nslots * G * SW]
  uint32_t* cnt = nullptr;     // [nslices] arrival counters
  uint32_t* queue = nullptr;   // [4] work queues + exit counter
  // host-planes convenience staging
  uint64_t* stage = nullptr;
  size_t stage_bytes = 0;
  sld_vec* tmp_in = nullptr;
  sld_vec* tmp_out = nullptr;
  // projection scratch
  int64_t* proj_rows = nullptr;
  int proj_cap = 0;
  uint32_t* terms_dev = nullptr;
  size_t terms_cap = 0;
  // dense-X scratch
  uint64_t* dproj_part = nullptr;
  size_t dproj_cap = 0;
  // fused Mksol step (sld_mat_mksol_bind): y vectors in slot order
  uint32_t* mk_y = nullptr;
  int mk_n = 0;
};


// the per-limb-count kernel table (sld_inst_*.cu)
const sld::LOps& ops(int L);
// one product x -> y (all stripe passes) on the matrix's context stream; with
// y == nullptr and peers set (the grid, sld_grid.cu) the last pass stores into
// the peers' buffers.  proj_rows / terms_out: fused unit-X projection of x.
void launch_product(sld_mat* M, const uint32_t* x, uint32_t* y, const int64_t* proj_rows, int proj_m,
                    uint32_t* terms_out, const uint32_t* mk_coeffs = nullptr, const uint32_t* addv = nullptr);

// sld_dense.cuh -- dense-X projection a[t] = sum_j x_t[j] v[j] mod ell
// (DenseRows.project, sldlag/solver.py:179-189), used on retry attempts of
// block Wiedemann (solver.py:616).  x_t[j] is stored in Montgomery form so
// one CIOS product gives the canonical x_t[j] v[j] mod ell; the canonical
// products are summed lazily per limb in 64-bit (n < 2^31 terms keep every
// limb sum below 2^63), reduced across the grid, then once per term by the
// same Barrett step as the SpMV rows.
#pragma once
#include <cuda_runtime.h>

#include "sld_device.cuh"

namespace sld {

struct DenseProjArgs {
  const uint32_t* x;  // [t][j] SW stride: Montgomery form (L > 8) or plain (L <= 8, lazy path)
  const uint32_t* v;  // biased slots
  uint32_t* out;      // m slots (canonical, SW stride)
  uint64_t* part;     // [t][block][MAXL]
  const uint32_t* fold;  // lazy path: 2^(32k) mod ell for k = L .. 2L, L words each
  int m;
  int64_t n;
  int nblocks;
};

// ---- lazy path (L <= 8): exact integer dot products, one reduction per term.
// x_t[j] is split into 2L 16-bit digits and each digit x 32-bit limb product
// (< 2^48) is accumulated by one IMAD.WIDE into a 64-bit column of weight
// 2^(16 c), c = p + 2 i -- 2L^2 IMAD.WIDE per (j, t) instead of a CIOS
// Montgomery product.  Each thread normalises its columns to 16-bit digits
// before the block sum; the final kernel folds the limbs above L with
// 2^(32k) mod ell and runs the SpMV's Barrett finalize.
template <int L>
__host__ __device__ constexpr int lazy_cols() { return 4 * L - 2; }  // p + 2i <= 4L-3

template <int L>
__global__ void __launch_bounds__(256) dense_lazy_partial(const DenseProjArgs a) {
  constexpr int SW = stride_words(L);
  constexpr int C = lazy_cols<L>();
  __shared__ uint64_t red[8][C + 1];
  // term-fastest block order: the m blocks of one j-range run together, so
  // the iterate is read from HBM about once, not m times
  const int t = blockIdx.x % a.m;
  const int jb = blockIdx.x / a.m;
  uint64_t col[C];
#pragma unroll
  for (int c = 0; c < C; c++) col[c] = 0;
  for (int64_t j = (int64_t)jb * blockDim.x + threadIdx.x; j < a.n; j += (int64_t)a.nblocks * blockDim.x) {
    uint32_t u[SW], w[SW];
    gather<SW>(a.v + (size_t)j * SW, u);
    gather<SW>(a.x + ((size_t)t * a.n + j) * SW, w);
#pragma unroll
    for (int p = 0; p < 2 * L; p++) {
      const uint32_t d = (p & 1) ? (w[p >> 1] >> 16) : (w[p >> 1] & 0xFFFFu);
#pragma unroll
      for (int i = 0; i < L; i++) col[p + 2 * i] += (uint64_t)d * (u[i] ^ 0x80000000u);
    }
  }
  // normalise to 16-bit digits (+ the carry above the top column)
  uint64_t dg[C + 1];
  {
    uint64_t carry = 0;
#pragma unroll
    for (int c = 0; c < C; c++) {
      const uint64_t v = col[c] + carry;  // col < 2^58, carry < 2^48: no wrap
      dg[c] = v & 0xFFFFu;
      carry = v >> 16;
    }
    dg[C] = carry;
  }
#pragma unroll
  for (int c = 0; c <= C; c++)
#pragma unroll
    for (int o = 16; o; o >>= 1) dg[c] += __shfl_xor_sync(0xffffffffu, dg[c], o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int c = 0; c <= C; c++) red[warp][c] = dg[c];
  __syncthreads();
  if (threadIdx.x <= C) {
    uint64_t sum = 0;
    for (int w8 = 0; w8 < (int)(blockDim.x >> 5); w8++) sum += red[w8][threadIdx.x];
    a.part[((size_t)t * a.nblocks + jb) * MAXL + threadIdx.x] = sum;
  }
}

template <int L>
__global__ void dense_lazy_final(const DenseProjArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  constexpr int C = lazy_cols<L>();
  constexpr int K = C / 2;  // 32-bit limbs below the top carry (2L - 1)
  const int t = blockIdx.x;
  // column sums over the blocks, one lane per column: digits < 2^16 x 256 x
  // nblocks, top < 2^64
  __shared__ uint64_t csum[C + 1];
  if (threadIdx.x <= C) {
    uint64_t s = 0;
    for (int b = 0; b < a.nblocks; b++) s += a.part[((size_t)t * a.nblocks + b) * MAXL + threadIdx.x];
    csum[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t cs[C + 1];
#pragma unroll
  for (int c = 0; c <= C; c++) cs[c] = csum[c];
  // 16-bit digits -> 32-bit limbs V_0 .. V_{K-1}, then the rest as a 64-bit
  // value `top` of weight 2^(32 K)
  uint32_t V[K];
  uint64_t carry = 0;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const uint64_t lo = cs[2 * k] + carry;
    const uint64_t d0 = lo & 0xFFFFu;
    const uint64_t hi = cs[2 * k + 1] + (lo >> 16);
    V[k] = (uint32_t)(d0 | ((hi & 0xFFFFu) << 16));
    carry = hi >> 16;
  }
  const uint64_t top = cs[C] + carry;  // C even: cs[C] has weight 2^(16 C) = 2^(32 K)
  // fold: limbs k >= L and top (two limbs at K, K+1) times 2^(32k) mod ell
  int64_t acc[L + 1];
#pragma unroll
  for (int i = 0; i < L; i++) acc[i] = V[i];
  acc[L] = 0;
#pragma unroll
  for (int k = L; k <= K + 1; k++) {
    const uint32_t limb = k < K ? V[k] : (k == K ? (uint32_t)top : (uint32_t)(top >> 32));
    const uint32_t* R = a.fold + (size_t)(k - L) * L;
#pragma unroll
    for (int i = 0; i < L; i++) {
      const uint64_t p = (uint64_t)limb * R[i];
      acc[i] += (int64_t)(uint32_t)p;
      acc[i + 1] += (int64_t)(p >> 32);
    }
  }
  uint32_t Rr[L];
  finalize<L>(acc, 0, mp, Rr);
#pragma unroll
  for (int i = 0; i < SW; i++) a.out[(size_t)t * SW + i] = i < L ? Rr[i] : 0u;
}


template <int L>
__global__ void __launch_bounds__(256) dense_proj_partial(const DenseProjArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  __shared__ uint64_t red[8][L];
  const int t = blockIdx.y;
  uint64_t acc[L];
#pragma unroll
  for (int i = 0; i < L; i++) acc[i] = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t u[SW], f[L], r[L];
    gather<SW>(a.v + (size_t)j * SW, u);
    const uint32_t* xp = a.x + ((size_t)t * a.n + j) * SW;
#pragma unroll
    for (int i = 0; i < L; i++) {
      u[i] ^= 0x80000000u;
      f[i] = xp[i];
    }
    montmul<L>(f, u, mp, r);
#pragma unroll
    for (int i = 0; i < L; i++) acc[i] += r[i];
  }
  // warp then block reduction
#pragma unroll
  for (int i = 0; i < L; i++) {
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < L; i++) red[warp][i] = acc[i];
  __syncthreads();
  if (threadIdx.x < L) {
    uint64_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w][threadIdx.x];
    a.part[((size_t)t * a.nblocks + blockIdx.x) * MAXL + threadIdx.x] = s;
  }
}

template <int L>
__global__ void dense_proj_final(const DenseProjArgs a, const ModParams mp) {
  constexpr int SW = stride_words(L);
  const int t = blockIdx.x;
  if (threadIdx.x != 0) return;
  int64_t acc[L + 1];
#pragma unroll
  for (int i = 0; i < L; i++) {
    uint64_t s = 0;
    for (int b = 0; b < a.nblocks; b++) s += a.part[((size_t)t * a.nblocks + b) * MAXL + i];
    acc[i] = (int64_t)s;
  }
  acc[L] = 0;
  uint32_t R[L];
  finalize<L>(acc, 0, mp, R);
#pragma unroll
  for (int i = 0; i < SW; i++) a.out[(size_t)t * SW + i] = i < L ? R[i] : 0u;
}

template <int L>
void dense_project_launch(const DenseProjArgs& a, const ModParams& mp, cudaStream_t s) {
  if (a.m <= 0) return;
  dim3 g(a.nblocks, a.m);
  if constexpr (L <= 8) {
    dense_lazy_partial<L><<<(unsigned)(a.nblocks * a.m), 256, 0, s>>>(a);
    dense_lazy_final<L><<<a.m, 32, 0, s>>>(a, mp);
    return;
  }
  dense_proj_partial<L><<<g, 256, 0, s>>>(a, mp);
  dense_proj_final<L><<<a.m, 32, 0, s>>>(a, mp);
}

inline int dense_proj_prepare(int sms, int m, int64_t n, int SW, uint64_t** part, size_t* cap,
                              DenseProjArgs* a) {
  (void)SW;
  int nb = (int)std::min<int64_t>(2 * (int64_t)sms, std::max<int64_t>(1, (n + 255) / 256));
  // lazy path bound: <= 4096 terms per thread keeps every 64-bit column exact
  nb = (int)std::max<int64_t>(nb, (n + 256 * 4096 - 1) / (256 * 4096));
  const size_t need = (size_t)std::max(m, 1) * nb * MAXL * sizeof(uint64_t);
  if (*cap < need) {
    if (*part) cudaFree(*part);
    *part = nullptr;
    if (cudaMalloc(part, need) != cudaSuccess) return -2;
    *cap = need;
  }
  a->part = *part;
  a->m = m;
  a->n = n;
  a->nblocks = nb;
  return 0;
}

}  // namespace sld

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
  const uint32_t* x;  // [t][j] Montgomery, SW stride
  const uint32_t* v;  // biased slots
  uint32_t* out;      // m slots (canonical, SW stride)
  uint64_t* part;     // [t][block][MAXL]
  int m;
  int64_t n;
  int nblocks;
};

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
  dense_proj_partial<L><<<g, 256, 0, s>>>(a, mp);
  dense_proj_final<L><<<a.m, 32, 0, s>>>(a, mp);
}

inline int dense_proj_prepare(int sms, int m, int64_t n, int SW, uint64_t** part, size_t* cap,
                              DenseProjArgs* a) {
  (void)SW;
  int nb = (int)std::min<int64_t>(2 * (int64_t)sms, std::max<int64_t>(1, (n + 255) / 256));
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

// Microbenchmark 5 (not product code): can random residue gathers bypass the
// L1TEX wavefront limit (~1 distinct line per SM per clock, mb.cu/mb2.cu)?
// Compares, over an L2-resident working set of ROW-byte records:
//   ldg   : ld.global.nc.v8 per lane (the spmv_pass gather)
//   g4    : TMA cp.async.bulk.tensor.2d ... tile::gather4 (4 random rows per
//           instruction, into shared memory, mbarrier complete_tx)
//   bulk  : cp.async.bulk (1-D) of one record per instruction
//   mix   : half the warps ldg, half g4 (are the two paths additive?)
// Each thread of the TMA variants owns a ring of D stages (one mbarrier and
// 4 records each) and reads the landed records back from shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint64_t pol_last(){
  uint64_t r; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(r)); return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t n){
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(m)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes){
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t ph){
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}"
               :: "r"(smem_u32(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(const CUtensorMap* tm, void* dst, uint64_t* mbar, int c0, int r0, int r1, int r2, int r3, uint64_t pol){
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
               " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;"
               :: "r"(smem_u32(dst)), "l"((uint64_t)tm), "r"(smem_u32(mbar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* mbar, uint64_t pol){
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)), "l"(pol) : "memory");
}

template<int ROW>
__device__ __forceinline__ uint32_t ldg_rec(const uint32_t* p, uint64_t pol){
  uint32_t acc = 0;
#pragma unroll
  for(int q=0;q<ROW/32;q++){
    uint32_t a,b,c,d,e,f,g,h;
    asm volatile("ld.global.nc.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(p+8*q), "l"(pol));
    acc += a^b^c^d^e^f^g^h;
  }
  return acc;
}

// MODE 0 ldg, 1 g4, 2 bulk, 3 mix (even warps ldg, odd warps g4),
// 4 additivity: warps 0-2 ldg for `iters`, warp 3 g4 for tma_iters
// (5: warps 0-2 ldg only, warp 3 idle -- the reference for 4)
template<int ROW, int MODE, int D>
__global__ void __launch_bounds__(128) kern(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ base,
                                           uint32_t nrec, uint32_t iters, uint32_t seed, uint32_t* out,
                                           uint32_t tma_iters = 0){
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  const uint64_t pol = pol_last();
  uint32_t acc = 0;
  const int warp = threadIdx.x >> 5;
  const bool use_ldg = MODE == 0 || (MODE == 3 && (warp & 1) == 0) || (MODE >= 4 && warp < 3);
  if(MODE == 5 && warp == 3) return;
  if(MODE == 4 && warp == 3) iters = tma_iters;
  if(use_ldg){
    // 4 records per iteration, issued together (as spmv_pass's NB = 4)
    for(uint32_t i=0;i<iters;i++){
      uint32_t j[4];
#pragma unroll
      for(int e=0;e<4;e++) j[e] = (uint32_t)(((uint64_t)hash32(tid*0x9E3779B9u + (4*i+e)*0x85ebca6bu + seed) * nrec) >> 32);
      uint32_t v[4];
#pragma unroll
      for(int e=0;e<4;e++) v[e] = ldg_rec<ROW>(base + (size_t)j[e]*(ROW/4), pol);
      acc += v[0]^v[1]^v[2]^v[3];
    }
  } else {
    // MODE 4: only warp 3 gathers through TMA and owns the ring
    const int tix = MODE == 4 ? threadIdx.x - 96 : threadIdx.x;
    const int nt = MODE == 4 ? 32 : blockDim.x;
    uint8_t* ring = sm + (size_t)tix * D * (4*ROW);
    uint64_t* bars = (uint64_t*)(sm + (size_t)nt * D * (4*ROW)) + tix * D;
    auto stage = [&](int s) -> uint8_t* { return ring + s*(4*ROW); };
    auto mb = [&](int s) -> uint64_t* { return bars + s; };
    for(int s=0;s<D;s++) mbar_init(mb(s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto issue = [&](int s, uint32_t i){
      uint32_t j[4];
#pragma unroll
      for(int e=0;e<4;e++) j[e] = (uint32_t)(((uint64_t)hash32(tid*0x9E3779B9u + (4*i+e)*0x85ebca6bu + seed) * nrec) >> 32);
      mbar_expect(mb(s), 4*ROW);
      if(MODE == 2){
#pragma unroll
        for(int e=0;e<4;e++) bulk(stage(s) + e*ROW, base + (size_t)j[e]*(ROW/4), ROW, mb(s), pol);
      } else {
        g4(&tm, stage(s), mb(s), 0, (int)j[0], (int)j[1], (int)j[2], (int)j[3], pol);
      }
    };
    for(int s=0;s<D && s<(int)iters;s++) issue(s, s);
    for(uint32_t i=0;i<iters;i++){
      const int s = i % D;
      mbar_wait(mb(s), (i / D) & 1);
      const uint4* p = (const uint4*)stage(s);
#pragma unroll
      for(int q=0;q<ROW/4;q++){ uint4 w = p[q]; acc += w.x^w.y^w.z^w.w; }
      if(i + D < iters) issue(s, i + D);
    }
  }
  if(acc==0x12345678) out[0]=acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template<int ROW, int MODE, int D>
int run(const char* name, EncodeFn enc, uint32_t* buf, size_t ws_mb, int ctas_per_sm, int sms, uint32_t* out,
        uint32_t tma_iters = 0){
  const uint32_t nrec = (uint32_t)((ws_mb<<20)/ROW);
  CUtensorMap tm;
  cuuint64_t dims[2] = {ROW/4, nrec};
  cuuint64_t strides[1] = {ROW};
  cuuint32_t box[2] = {ROW/4, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if(r != CUDA_SUCCESS){ printf("encode failed %d\n", (int)r); return 1; }
  const int thr = 128;
  const size_t smem = (MODE == 0 || MODE == 5) ? 0 : (size_t)(MODE == 4 ? 32 : thr) * D * (4*ROW + 8);
  if(smem > 48*1024) CK(cudaFuncSetAttribute(kern<ROW,MODE,D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int blocks = sms * ctas_per_sm;
  const uint32_t iters = 512;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for(int rep=0;rep<4;rep++){
    cudaEventRecord(e0);
    kern<ROW,MODE,D><<<blocks,thr,smem>>>(tm, buf, nrec, iters, rep*77u, out, tma_iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0 && ms<best) best=ms;
  }
  double recs = (double)blocks*thr*iters*4;
  if(MODE >= 4) recs = (double)blocks*96*iters*4 + (MODE == 4 ? (double)blocks*32*tma_iters*4 : 0.0);
  printf("%-5s row=%3dB D=%d ctas/SM=%d smem=%6zu ws=%4zu MB tma_iters=%4u: %7.1f G rec/s  %8.1f GB/s  %.3f ms\n",
         name, ROW, D, ctas_per_sm, smem, ws_mb, tma_iters, recs/best/1e6, recs*ROW/best/1e6, best);
  return 0;
}

int main(){
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,0));
  printf("device %s SMs %d\n", pr.name, pr.multiProcessorCount);
  const int sms = pr.multiProcessorCount;
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  uint32_t* buf; CK(cudaMalloc(&buf,(size_t)1<<30)); CK(cudaMemset(buf,1,(size_t)1<<30));
  uint32_t* out; CK(cudaMalloc(&out,1<<20));
  // (r02 first run: the ldg / g4 / bulk / mix rates at 32 and 58 MB, profiles/microbench5_tma_r02.txt)
  for(size_t ws : {32}){
    run<32,0,1>("ldg", enc, buf, ws, 8, sms, out);
    for(int c : {8, 12, 16}){
      run<32,5,4>("ldg3", enc, buf, ws, c, sms, out, 0);
      for(uint32_t ti : {32u, 64u, 128u, 256u}) run<32,4,4>("add", enc, buf, ws, c, sms, out, ti);
    }
  }
  return 0;
}

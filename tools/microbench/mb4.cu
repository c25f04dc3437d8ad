// Microbenchmark 4 (not product code): how much L2 does a random-gather
// working set keep when a read-once stream (the SpMV's index stream) flows
// through L2 at the same time?  Gathers are 2-sector records fetched by lane
// pairs (the G = 2 chain layout); every K records a warp also reads one
// coalesced 512 B piece of a 4 GB stream.  Stream / gather cache policies:
//   0 default, 1 L2::evict_first, 2 L2::evict_last
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint64_t pol_of(int p){
  uint64_t r;
  if(p == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(r));
  else if(p == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(r));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(r));
  return r;
}
template<int K>
__global__ void __launch_bounds__(256,4) gs(const uint32_t* __restrict__ x, uint32_t nrec, const uint4* __restrict__ st,
                                            size_t st_n, uint32_t iters, uint32_t seed, int gpol_i, int spol_i, uint32_t* out){
  const uint64_t gpol = pol_of(gpol_i), spol = pol_of(spol_i);
  const uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  const uint32_t grp = tid >> 1, sub = tid & 1;
  const uint32_t warp = tid >> 5, lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x*blockDim.x/32;
  uint32_t acc = 0;
  size_t sidx = (size_t)warp*32 + lane;
  for(uint32_t i=0;i<iters;i+=K){
    if(K < 1000){
      uint32_t a,b,c,d;
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(st + sidx), "l"(spol));
      acc += a^b^c^d;
      sidx += (size_t)nwarps*32; if(sidx >= st_n) sidx -= st_n;
    }
    #pragma unroll 4
    for(int k=0;k<(K<1000?K:8);k++){
      uint32_t h = hash32(grp*0x9E3779B9u + (i+k)*0x85ebca6bu + seed);
      uint32_t j = (uint32_t)(((uint64_t)h * nrec) >> 32);
      const uint32_t* p = x + (size_t)j*16 + sub*8;
      uint32_t a,b,c,d,e,f,g,hh;
      asm volatile("ld.global.nc.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                   : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p), "l"(gpol));
      acc += a^b^c^d^e^f^g^hh;
    }
  }
  if(acc==0x12345678) out[0]=acc;
}

int main(){
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount;
  uint32_t* out; CK(cudaMalloc(&out, 4));
  size_t xb = 256ull<<20, sb = 4096ull<<20;
  uint32_t* x; CK(cudaMalloc(&x, xb)); CK(cudaMemset(x, 1, xb));
  uint4* st; CK(cudaMalloc(&st, sb)); CK(cudaMemset(st, 2, sb));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm*4, threads = 256; const uint32_t iters = 2048;
  auto run = [&](int K, int mb, int gp, int sp){
    uint32_t nrec = (uint32_t)(((size_t)mb<<20)/64);
    auto launch = [&](uint32_t seed){
      if(K==4) gs<4><<<blocks,threads>>>(x,nrec,st,sb/16,iters,seed,gp,sp,out);
      else if(K==8) gs<8><<<blocks,threads>>>(x,nrec,st,sb/16,iters,seed,gp,sp,out);
      else if(K==16) gs<16><<<blocks,threads>>>(x,nrec,st,sb/16,iters,seed,gp,sp,out);
      else gs<1000000><<<blocks,threads>>>(x,nrec,st,sb/16,iters,seed,gp,sp,out);
    };
    launch(1); launch(2);
    cudaEventRecord(e0);
    for(int r=0;r<3;r++) launch(3+r);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms/=3;
    double recs = (double)blocks*threads/2*iters;
    printf("ws=%4d MB  stream every %-7s gpol=%d spol=%d: %7.1f Grec/s  %8.1f GB/s gathers\n", mb,
           K>=1000? "none" : (K==4?"4 rec":K==8?"8 rec":"16 rec"), gp, sp, recs/ms/1e6, recs*64/ms/1e6);
  };
  for(int mb : {32, 48, 58, 80, 115}){
    run(1000000, mb, 0, 0);
    run(1000000, mb, 2, 0);
    for(int K : {8, 16}){
      run(K, mb, 2, 1);
      run(K, mb, 0, 1);
      run(K, mb, 0, 0);
    }
  }
  return 0;
}

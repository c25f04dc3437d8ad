// Microbenchmarks that size the SpMV design on B200 (not product code):
//  (1) random 32-byte gather bandwidth vs working-set size (uniform and
//      power-law column popularity, as in the FFS corpus),
//  (2) IMAD.WIDE vs IADD3 issue throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template<int MODE>
__global__ void gather(const uint32_t* __restrict__ base, uint32_t nslots, uint32_t iters, uint32_t seed, uint32_t* out){
  uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  #pragma unroll 4
  for(uint32_t i=0;i<iters;i++){
    uint32_t h = hash32(tid*0x9E3779B9u + i*0x85ebca6bu + seed);
    uint32_t j;
    if(MODE==0) j = (uint32_t)(((uint64_t)h * nslots) >> 32);
    else { float u = (h>>8) * (1.0f/16777216.0f); j = (uint32_t)(u*u*(float)nslots); if(j>=nslots) j=nslots-1; }
    const uint32_t* p = base + (size_t)j*8;
    uint32_t a,b,c,d,e,f,g,hh;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p));
    acc += a^b^c^d^e^f^g^hh;
  }
  if(acc==0x12345678) out[0]=acc;
}
template<int NSEC, int NA>
__global__ void gatherN(const uint32_t* __restrict__ base, uint32_t nslots, uint32_t iters, uint32_t seed, uint32_t* out){
  uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  #pragma unroll 2
  for(uint32_t i=0;i<iters;i++){
    uint32_t h = hash32(tid*0x9E3779B9u + i*0x85ebca6bu + seed);
    uint32_t j = (uint32_t)(((uint64_t)h * nslots) >> 32);
    const uint32_t* p = base + (size_t)j*8*NSEC;
    #pragma unroll
    for(int q=0;q<NSEC;q++){
      uint32_t a,b,c,d,e,f,g,hh;
      if(NA) asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p+8*q));
      else asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p+8*q));
      acc += a^b^c^d^e^f^g^hh;
    }
  }
  if(acc==0x12345678) out[0]=acc;
}
__global__ void stream_read(const uint4* __restrict__ p, size_t n, uint32_t* out){
  uint32_t acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){
    uint32_t a,b,c,d,e,f,g,h; asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(p+2*i));
    acc += a^b^c^d^e^f^g^h;
  }
  if(acc==0x12345678) out[0]=acc;
}
__global__ void imadw(uint32_t iters, int32_t c, int64_t* out){
  int64_t a0=threadIdx.x,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  int32_t x = threadIdx.x*7+1;
  for(uint32_t i=0;i<iters;i++){
    #pragma unroll
    for(int r=0;r<8;r++){
      a0 += (int64_t)c*(int64_t)(x+r); a1 += (int64_t)c*(int64_t)(x+r+1); a2 += (int64_t)c*(int64_t)(x+r+2); a3 += (int64_t)c*(int64_t)(x+r+3);
      a4 += (int64_t)c*(int64_t)(x^r); a5 += (int64_t)c*(int64_t)(x^(r+1)); a6 += (int64_t)c*(int64_t)(x^(r+2)); a7 += (int64_t)c*(int64_t)(x^(r+3));
    }
    x += c;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0^a1^a2^a3^a4^a5^a6^a7;
}
__global__ void iaddc(uint32_t iters, uint32_t c, uint32_t* out){
  uint32_t a[8]; for(int i=0;i<8;i++) a[i]=threadIdx.x+i;
  uint32_t x = threadIdx.x*7+1;
  for(uint32_t i=0;i<iters;i++){
    #pragma unroll
    for(int r=0;r<8;r++){
      asm volatile("add.cc.u32 %0,%0,%8;\n\taddc.cc.u32 %1,%1,%8;\n\taddc.cc.u32 %2,%2,%8;\n\taddc.cc.u32 %3,%3,%8;\n\taddc.cc.u32 %4,%4,%8;\n\taddc.cc.u32 %5,%5,%8;\n\taddc.cc.u32 %6,%6,%8;\n\taddc.u32 %7,%7,%8;"
        : "+r"(a[0]),"+r"(a[1]),"+r"(a[2]),"+r"(a[3]),"+r"(a[4]),"+r"(a[5]),"+r"(a[6]),"+r"(a[7]) : "r"(x+r));
    }
    x += c;
  }
  uint32_t s=0; for(int i=0;i<8;i++) s^=a[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("device %s SMs %d L2 %d MB persistL2max %d MB clock %d MHz\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, pr.persistingL2CacheMaxSize>>20, pr.clockRate/1000);
  size_t maxbytes = (size_t)4<<30;
  uint32_t* buf; CK(cudaMalloc(&buf,maxbytes)); CK(cudaMemset(buf,1,maxbytes));
  uint32_t* out; CK(cudaMalloc(&out,64<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t sizes_mb[] = {4,16,32,64,96,115,128,160,256,1024,4096};
  int blocks = pr.multiProcessorCount*8, thr=256; uint32_t iters=2048;
  double gathered = (double)blocks*thr*iters*32.0;
  for(int mode=0;mode<2;mode++){
    for(size_t s: sizes_mb){
      uint32_t nslots = (uint32_t)((s<<20)/32);
      float best=1e9;
      for(int rep=0;rep<4;rep++){
        cudaEventRecord(e0);
        if(mode==0) gather<0><<<blocks,thr>>>(buf,nslots,iters,rep*77u,out); else gather<1><<<blocks,thr>>>(buf,nslots,iters,rep*77u,out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0 && ms<best) best=ms;
      }
      printf("gather32 %s ws=%5zu MB : %8.1f GB/s  (%.3f ms)\n", mode?"powerlaw":"uniform ", s, gathered/best/1e6, best);
    }
  }
  for(int ns: {1,2,4}) for(int na=0; na<2; na++) for(size_t s: {32,64,512}){
      uint32_t nslots = (uint32_t)((s<<20)/(32*ns)); float best=1e9; uint32_t it=1024;
      for(int rep=0;rep<4;rep++){
        cudaEventRecord(e0);
        if(ns==1){ if(na) gatherN<1,1><<<blocks,thr>>>(buf,nslots,it,rep*77u,out); else gatherN<1,0><<<blocks,thr>>>(buf,nslots,it,rep*77u,out);} 
        if(ns==2){ if(na) gatherN<2,1><<<blocks,thr>>>(buf,nslots,it,rep*77u,out); else gatherN<2,0><<<blocks,thr>>>(buf,nslots,it,rep*77u,out);} 
        if(ns==4){ if(na) gatherN<4,1><<<blocks,thr>>>(buf,nslots,it,rep*77u,out); else gatherN<4,0><<<blocks,thr>>>(buf,nslots,it,rep*77u,out);} 
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0&&ms<best)best=ms; }
      double by=(double)blocks*thr*it*32.0*ns;
      printf("gather %3dB %s ws=%4zu MB: %8.1f GB/s  %.1f Gacc/s\n", 32*ns, na?"noalloc":"default", s, by/best/1e6, by/32/ns/best/1e6);
  }
  { size_t n = maxbytes/32; float best=1e9;
    for(int rep=0;rep<4;rep++){ cudaEventRecord(e0); stream_read<<<pr.multiProcessorCount*16,512>>>((const uint4*)buf,n,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0&&ms<best)best=ms;}
    printf("stream read 4GB: %.1f GB/s\n", maxbytes/best/1e6); }
  { uint32_t it=4096; float best=1e9; int b=pr.multiProcessorCount*8, t=256;
    for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); imadw<<<b,t>>>(it,3,(int64_t*)out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0&&ms<best)best=ms;}
    double ops = (double)b*t*it*64; printf("IMAD.WIDE: %.2f Tops/s\n", ops/best/1e9); }
  { uint32_t it=4096; float best=1e9; int b=pr.multiProcessorCount*8, t=256;
    for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); iaddc<<<b,t>>>(it,3,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep>0&&ms<best)best=ms;}
    double ops = (double)b*t*it*64; printf("IADD carry chain: %.2f Tops/s\n", ops/best/1e9); }
  return 0;
}

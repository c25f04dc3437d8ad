// Microbenchmark 2 (not product code): is the ~9.2 TB/s random-gather rate
// an L2->SM port limit or an access-pattern limit?
//  (1) L2-resident *sequential* reads (coalesced 1 KB per warp-load)
//  (2) random 32-byte gathers via TMA bulk copies (cp.async.bulk) into smem
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void seq_read(const uint32_t* __restrict__ base, size_t nwords, int reps, uint32_t* out){
  uint32_t acc=0;
  const size_t stride = (size_t)gridDim.x*blockDim.x*8;
  for(int r=0;r<reps;r++)
  for(size_t i=((size_t)blockIdx.x*blockDim.x+threadIdx.x)*8;i<nwords;i+=stride){
    uint32_t a,b,c,d,e,f,g,h;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(base+i));
    acc += a^b^c^d^e^f^g^h;
  }
  if(acc==0x12345678) out[0]=acc;
}
// TMA bulk gather: each thread copies one random 32B slot into its smem slot
template<int STAGES>
__global__ void __launch_bounds__(256) tma_gather(const uint32_t* __restrict__ base, uint32_t nslots, uint32_t iters, uint32_t seed, uint32_t* out){
  __shared__ alignas(128) uint32_t buf[STAGES][256*8];
  __shared__ alignas(8) uint64_t bar[STAGES];
  const int t = threadIdx.x;
  if(t < STAGES){
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[t]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(256));
  }
  __syncthreads();
  uint32_t acc=0;
  uint32_t tid = blockIdx.x*blockDim.x + t;
  auto issue = [&](uint32_t i, int s){
    uint32_t h = hash32(tid*0x9E3779B9u + i*0x85ebca6bu + seed);
    uint32_t j = (uint32_t)(((uint64_t)h * nslots) >> 32);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(&buf[s][t*8]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(32));
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                 :: "r"(d), "l"(base + (size_t)j*8), "r"(b) : "memory");
  };
  for(int s=0;s<STAGES;s++) issue(s, s);
  uint32_t phase[STAGES]; for(int s=0;s<STAGES;s++) phase[s]=0;
  for(uint32_t i=0;i<iters;i++){
    int s = i % STAGES;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t done=0;
    while(!done){
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(b), "r"(phase[s]));
    }
    phase[s]^=1;
    const uint32_t* v = &buf[s][t*8];
    acc += v[0]^v[1]^v[2]^v[3]^v[4]^v[5]^v[6]^v[7];
    __syncwarp();
    if(i + STAGES < iters) issue(i + STAGES, s);
  }
  if(acc==0x12345678) out[0]=acc;
}
// random line gathers where G consecutive lanes fetch the G sectors of the
// same (32*G)-byte record in ONE instruction (coalesced into one request)
template<int G>
__global__ void coop_gather(const uint32_t* __restrict__ base, uint32_t nrec, uint32_t iters, uint32_t seed, uint32_t* out){
  uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  uint32_t grp = tid / G, sub = tid % G;
  uint32_t acc = 0;
  #pragma unroll 4
  for(uint32_t i=0;i<iters;i++){
    uint32_t h = hash32(grp*0x9E3779B9u + i*0x85ebca6bu + seed);
    uint32_t j = (uint32_t)(((uint64_t)h * nrec) >> 32);
    const uint32_t* p = base + (size_t)j*8*G + sub*8;
    uint32_t a,b,c,d,e,f,g,hh;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p));
    acc += a^b^c^d^e^f^g^hh;
  }
  if(acc==0x12345678) out[0]=acc;
}

int main(){
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,0));
  size_t bytes = (size_t)1<<30;
  uint32_t* buf; CK(cudaMalloc(&buf,bytes)); CK(cudaMemset(buf,1,bytes));
  uint32_t* out; CK(cudaMalloc(&out,1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(size_t mb : {8, 32, 64}){
    size_t nw = (mb<<20)/4; int reps = (int)(4096/mb);
    float best=1e9;
    for(int r=0;r<4;r++){ cudaEventRecord(e0); seq_read<<<pr.multiProcessorCount*8,256>>>(buf,nw,reps,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r>0&&ms<best)best=ms;}
    printf("L2 sequential read ws=%3zu MB: %8.1f GB/s\n", mb, (double)nw*4*reps/best/1e6);
  }
  for(int G : {1, 2, 3, 4})
  for(size_t mb : {32, 64, 512}){
    uint32_t nrec = (uint32_t)((mb<<20)/(32*G)); uint32_t iters = 1024;
    int blocks = pr.multiProcessorCount*8;
    float best=1e9;
    for(int r=0;r<4;r++){ cudaEventRecord(e0);
      if(G==1) coop_gather<1><<<blocks,256>>>(buf,nrec,iters,r*3u,out);
      if(G==2) coop_gather<2><<<blocks,256>>>(buf,nrec,iters,r*3u,out);
      if(G==3) coop_gather<3><<<blocks,256>>>(buf,nrec,iters,r*3u,out);
      if(G==4) coop_gather<4><<<blocks,256>>>(buf,nrec,iters,r*3u,out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r>0&&ms<best)best=ms;}
    double by = (double)blocks*256*iters*32;
    printf("coop gather G=%d (%3d B records) ws=%3zu MB: %8.1f GB/s  %6.1f Grec/s\n", G, 32*G, mb, by/best/1e6, by/(32*G)/best/1e6);
  }
  for(size_t mb : {32, 64}){
    uint32_t nslots = (uint32_t)((mb<<20)/32); uint32_t iters=1024;
    for(int occ : {4, 8}){
      float best=1e9; int blocks = pr.multiProcessorCount*occ;
      for(int r=0;r<4;r++){ cudaEventRecord(e0); tma_gather<4><<<blocks,256>>>(buf,nslots,iters,r*7u,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r>0&&ms<best)best=ms;}
      printf("TMA bulk 32B gather ws=%3zu MB blocks/SM=%d: %8.1f GB/s\n", mb, occ, (double)blocks*256*iters*32/best/1e6);
    }
  }
  return 0;
}

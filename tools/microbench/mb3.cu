// Microbenchmark 3 (not product code): does the L2 of each die cache its own
// copy of what its SMs gather (effective capacity ~ one die's L2), and does
// splitting the gathered columns by die recover the full L2?
//  (1) SM -> die map from L2 latency: probe lines are written (home slice),
//      then each SM times its FIRST ld.cg of each line.  Near/far latency
//      patterns of SMs on the same die agree, across dies they are complements.
//  (2) random 32 B gathers over a working set W by all SMs, with
//      (a) every SM over all of W, (b) die-split: SMs of die d only gather
//      the 2 KB chunks c with c % 2 == d, (c) control: same split by smid
//      parity instead of die.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t smid(){ uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint32_t hash32(uint32_t x){
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int NPROBE = 128;

__global__ void write_probes(uint32_t* buf, int stride_words, uint32_t tag){
  int i = threadIdx.x;
  if(i < NPROBE) asm volatile("st.global.cg.u32 [%0], %1;" :: "l"(buf + (size_t)i*stride_words), "r"(tag));
}
// the CTA that lands on SM `target` times the first load of every probe line
__global__ void time_probes(const uint32_t* buf, int stride_words, int target, uint32_t* lat, int* hit){
  if(smid() != (uint32_t)target || threadIdx.x != 0) return;
  if(atomicExch(hit, 1) != 0) return;
  uint32_t dep = 0;
  for(int i=0;i<NPROBE;i++){
    const uint32_t* p = buf + (size_t)i*stride_words + dep;
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) : "r"(dep) : "memory");
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    dep = v >> 31;  // 0 (tags are small), but the clock read must wait for it
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) : "r"(dep) : "memory");
    lat[i] = (uint32_t)(t1 - t0) + dep;
  }
}
// random 32-byte gathers; mode 0: any chunk; mode 1: chunks of my die;
// mode 2: chunks of my smid parity.  A 2 KB chunk = 64 slots.
__global__ void gather(const uint32_t* __restrict__ base, uint32_t nchunks, uint32_t iters, uint32_t seed,
                       const uint8_t* __restrict__ die, int mode, uint32_t* out){
  uint32_t tid = blockIdx.x*blockDim.x + threadIdx.x;
  uint32_t sel = mode == 1 ? die[smid()] : (smid() & 1);
  uint32_t half = nchunks / 2;
  uint32_t acc = 0;
  #pragma unroll 4
  for(uint32_t i=0;i<iters;i++){
    uint32_t h = hash32(tid*0x9E3779B9u + i*0x85ebca6bu + seed);
    uint32_t h2 = hash32(h ^ 0x5bd1e995u);
    uint32_t c;
    if(mode == 0) c = (uint32_t)(((uint64_t)h * nchunks) >> 32);
    else c = 2u * (uint32_t)(((uint64_t)h * half) >> 32) + sel;
    const uint32_t* p = base + ((size_t)c * 64 + (h2 & 63)) * 8;
    uint32_t a,b,cc,d,e,f,g,hh;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(cc),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(hh) : "l"(p));
    acc += a^b^cc^d^e^f^g^hh;
  }
  if(acc==0x12345678) out[0]=acc;
}

int main(){
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount;
  printf("device %s SMs %d L2 %d MB\n", prop.name, nsm, prop.l2CacheSize >> 20);
  // ---- (1) die map
  const int stride_words = 4096 / 4 * 3 + 32;  // probes ~12 KB apart: distinct 2 KB chunks
  uint32_t *probe, *lat; int* hit;
  CK(cudaMalloc(&probe, (size_t)NPROBE * stride_words * 4 + 4096));
  CK(cudaMalloc(&lat, (size_t)nsm * NPROBE * 4));
  CK(cudaMalloc(&hit, 4));
  std::vector<uint32_t> L((size_t)nsm * NPROBE, 0);
  for(int s=0;s<nsm;s++){
    for(int rep=0; rep<3; rep++){
      // evict the probe lines: stream a 256 MB buffer through L2 once
      static uint32_t* junk = nullptr;
      if(!junk){ CK(cudaMalloc(&junk, 256u<<20)); }
      CK(cudaMemsetAsync(junk, rep, 256u<<20));
      write_probes<<<1, NPROBE>>>(probe, stride_words, 7u + rep);
      CK(cudaMemset(hit, 0, 4));
      time_probes<<<nsm * 4, 32>>>(probe, stride_words, s, lat + (size_t)s * NPROBE, hit);
      CK(cudaDeviceSynchronize());
      std::vector<uint32_t> tmp(NPROBE);
      CK(cudaMemcpy(tmp.data(), lat + (size_t)s*NPROBE, NPROBE*4, cudaMemcpyDeviceToHost));
      for(int i=0;i<NPROBE;i++){ uint32_t& d = L[(size_t)s*NPROBE+i]; d = rep==0 ? tmp[i] : std::min(d, tmp[i]); }
    }
  }
  // classify: per probe, threshold at the midpoint of the SM-median split
  std::vector<uint8_t> die(nsm, 0);
  {
    // reference pattern: SM 0's per-probe latencies; correlation sign of each SM vs SM 0
    std::vector<double> mean(NPROBE, 0);
    for(int i=0;i<NPROBE;i++){ for(int s=0;s<nsm;s++) mean[i] += L[(size_t)s*NPROBE+i]; mean[i] /= nsm; }
    std::vector<double> z0(NPROBE);
    for(int i=0;i<NPROBE;i++) z0[i] = L[i] - mean[i];
    int n1 = 0;
    for(int s=0;s<nsm;s++){
      double c = 0;
      for(int i=0;i<NPROBE;i++) c += (L[(size_t)s*NPROBE+i] - mean[i]) * z0[i];
      die[s] = c > 0 ? 0 : 1; n1 += die[s];
      if(s < 8 || s % 16 == 0){
        printf("sm %3d corr %+10.0f die %d lat[0..11]:", s, c, die[s]);
        for(int i=0;i<12;i++) printf(" %u", L[(size_t)s*NPROBE+i]);
        printf("\n");
      }
    }
    printf("die map: %d SMs on die 0, %d on die 1\n", nsm - n1, n1);
    printf("map:"); for(int s=0;s<nsm;s++) printf("%d", die[s]); printf("\n");
    // separation: per probe, mean latency on die 0 vs die 1
    int strong = 0;
    for(int i=0;i<NPROBE;i++){
      double a=0,b=0; int na=0,nb=0;
      for(int s=0;s<nsm;s++){ if(die[s]) { b += L[(size_t)s*NPROBE+i]; nb++; } else { a += L[(size_t)s*NPROBE+i]; na++; } }
      a/=std::max(na,1); b/=std::max(nb,1);
      if(std::abs(a-b) > 12) strong++;
      if(i < 8) printf("probe %d: die0 %.1f die1 %.1f\n", i, a, b);
    }
    printf("probes with |die0-die1| > 12 cyc: %d of %d\n", strong, NPROBE);
  }
  uint8_t* ddie; CK(cudaMalloc(&ddie, nsm)); CK(cudaMemcpy(ddie, die.data(), nsm, cudaMemcpyHostToDevice));
  // ---- (2) gathers
  uint32_t* out; CK(cudaMalloc(&out, 4));
  size_t maxb = 512ull << 20;
  uint32_t* base; CK(cudaMalloc(&base, maxb)); CK(cudaMemset(base, 1, maxb));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256; const uint32_t iters = 1024;
  for(int mb : {32, 48, 64, 80, 96, 115, 128, 160, 192, 230, 256}){
    uint32_t nchunks = (uint32_t)(((size_t)mb << 20) / 2048);
    for(int mode=0; mode<3; mode++){
      gather<<<blocks,threads>>>(base, nchunks, iters, 1, ddie, mode, out);
      gather<<<blocks,threads>>>(base, nchunks, iters, 2, ddie, mode, out);
      cudaEventRecord(e0);
      const int R = 3;
      for(int r=0;r<R;r++) gather<<<blocks,threads>>>(base, nchunks, iters, 3+r, ddie, mode, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
      double bytes = (double)blocks*threads*iters*32;
      printf("gather32 ws=%4d MB %-9s: %8.1f GB/s  %6.1f Gacc/s\n", mb,
             mode==0 ? "all" : mode==1 ? "die-split" : "par-split", bytes/ms/1e6, bytes/32/ms/1e6);
    }
  }
  return 0;
}

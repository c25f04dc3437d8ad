// sld_capi.cu -- host side of libsldb200.so: the C ABI declared in
// include/sldb200.h (matrix builder, vectors, SpMV and the device-resident
// Krylov loop with CUDA graphs).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "sld_internal.cuh"

using namespace sld;

// ------------------------------------------------------------ errors

static thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

extern "C" const char* sld_last_error(void) { return g_err.c_str(); }
// error reporting for the host-only translation units (sld_fileio.cpp)
int sld_set_error(int code, const char* msg) { return fail(code, "%s", msg); }
extern "C" int sld_version(void) { return 1; }
extern "C" int sld_device_count(int* out) {
  CU(cudaGetDeviceCount(out));
  return SLD_OK;
}

// ------------------------------------------------- host multiprecision

// r = r*2 mod ell (r < ell), L words
static void hmod_double(uint32_t* r, const uint32_t* ell, int L) {
  uint32_t c = 0;
  std::vector<uint32_t> t(L + 1);
  for (int i = 0; i < L; i++) {
    t[i] = (r[i] << 1) | c;
    c = r[i] >> 31;
  }
  t[L] = c;
  // t >= ell ?
  bool ge = t[L] != 0;
  if (!ge) {
    ge = true;
    for (int i = L - 1; i >= 0; i--)
      if (t[i] != ell[i]) { ge = t[i] > ell[i]; break; }
  }
  if (ge) {
    int64_t br = 0;
    for (int i = 0; i < L; i++) {
      int64_t v = (int64_t)t[i] - ell[i] + br;
      t[i] = (uint32_t)v;
      br = v >> 32;
    }
  }
  for (int i = 0; i < L; i++) r[i] = t[i];
}

static int bitlen(const uint32_t* a, int n) {
  while (n > 0 && a[n - 1] == 0) n--;
  if (!n) return 0;
  return 32 * (n - 1) + (32 - __builtin_clz(a[n - 1]));
}

// (|c| mod ell) for a 64-bit magnitude, L words out
static void hmod_u64(uint64_t c, const uint32_t* ell, int L, uint32_t* out) {
  std::vector<uint32_t> r(L, 0);
  for (int b = 63; b >= 0; b--) {
    hmod_double(r.data(), ell, L);
    if ((c >> b) & 1) {
      // r += 1 mod ell  (r < ell, ell odd >= 3)
      uint64_t carry = 1;
      for (int i = 0; i < L && carry; i++) {
        uint64_t v = (uint64_t)r[i] + carry;
        r[i] = (uint32_t)v;
        carry = v >> 32;
      }
      bool ge = true;
      for (int i = L - 1; i >= 0; i--)
        if (r[i] != ell[i]) { ge = r[i] > ell[i]; break; }
      if (ge) std::fill(r.begin(), r.end(), 0u);  // r == ell
    }
  }
  for (int i = 0; i < L; i++) out[i] = r[i];
}

// -------------------------------------------------- per-L dispatch table

const LOps& ops(int L) {
  static LOps table[MAXL + 1];
  static bool init = [] {
    fill_ops_1_8(table);
    fill_ops_9_16(table);
    fill_ops_17_24(table);
    fill_ops_25_32(table);
    return true;
  }();
  (void)init;
  return table[L];
}

// ------------------------------------------------------------ die map
//
// Which of B200's two dies each SM sits on (yield-dependent, so probed per
// device): a cold line's first load costs ~590 cycles from an SM on the die
// whose HBM holds it and ~970 from the other die (profiles/microbench3_r01.txt).
// Probe lines are dropped from L2 with discard.global.L2, then the SM under
// test times its first load of each; SMs of one die agree on the near/far
// pattern, the two dies see complementary patterns.  An ambiguous result
// disables the die split (the plain stripe passes still run on the GPU).

namespace {
constexpr int DIE_PROBES = 64;
constexpr int DIE_STRIDE = 1056;  // words between probe lines (> 2 KB apart)

__global__ void die_nsmid(int* out) {
  uint32_t n;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
  *out = (int)n;
}
__global__ void die_discard(uint32_t* buf) {
  const int i = threadIdx.x;
  if (i < DIE_PROBES) asm volatile("discard.global.L2 [%0], 128;" ::"l"(buf + (size_t)i * DIE_STRIDE) : "memory");
}
__global__ void die_time(const uint32_t* buf, int target, uint32_t* lat, int* hit) {
  __shared__ uint32_t sink[2];
  if (sm_id() != (uint32_t)target || threadIdx.x != 0) return;
  if (atomicExch(hit, 1) != 0) return;
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sink);
  for (int i = 0; i < DIE_PROBES; i++) {
    uint64_t t0, t1;
    uint32_t v;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(buf + (size_t)i * DIE_STRIDE) : "memory");
    // the volatile shared store consumes the load, and the clock read is
    // not moved above a memory operation
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(sa), "r"(v) : "memory");
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
    lat[i] = (uint32_t)(t1 - t0);
  }
}

struct DieMap {
  bool probed = false;
  bool ok = false;
  uint8_t map[256] = {0};
  int n[2] = {0, 0};
  std::string why;
};
std::mutex g_die_mu;
DieMap g_die[64];

int probe_dies(int dev, DieMap& d, int sms) {
  uint32_t *buf = nullptr, *lat = nullptr;
  int *hit = nullptr, *nsm = nullptr;
  const int T = 256, REPS = 3;  // min over repetitions drops DRAM latency spikes
  CU(cudaMalloc(&buf, (size_t)DIE_PROBES * DIE_STRIDE * 4 + 256));
  CU(cudaMalloc(&lat, (size_t)REPS * T * DIE_PROBES * 4));
  CU(cudaMalloc(&hit, REPS * T * 4));
  CU(cudaMalloc(&nsm, 4));
  CU(cudaMemset(buf, 0, (size_t)DIE_PROBES * DIE_STRIDE * 4 + 256));
  CU(cudaMemset(hit, 0, REPS * T * 4));
  die_nsmid<<<1, 1>>>(nsm);
  int nsmid = 0;
  CU(cudaMemcpy(&nsmid, nsm, 4, cudaMemcpyDeviceToHost));
  nsmid = std::min(std::max(nsmid, sms), T);
  for (int r = 0; r < REPS; r++)
    for (int t = 0; t < nsmid; t++) {
      die_discard<<<1, DIE_PROBES>>>(buf);
      die_time<<<sms * 4, 32>>>(buf, t, lat + ((size_t)r * T + t) * DIE_PROBES, hit + r * T + t);
    }
  std::vector<uint32_t> LR((size_t)REPS * T * DIE_PROBES), L((size_t)T * DIE_PROBES, ~0u);
  std::vector<int> HR(REPS * T), H(T, 1);
  CU(cudaMemcpy(LR.data(), lat, LR.size() * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(HR.data(), hit, HR.size() * 4, cudaMemcpyDeviceToHost));
  for (int r = 0; r < REPS; r++)
    for (int t = 0; t < T; t++) {
      H[t] &= HR[r * T + t];
      for (int i = 0; i < DIE_PROBES; i++)
        L[(size_t)t * DIE_PROBES + i] = std::min(L[(size_t)t * DIE_PROBES + i], LR[((size_t)r * T + t) * DIE_PROBES + i]);
    }
  cudaFree(buf);
  cudaFree(lat);
  cudaFree(hit);
  cudaFree(nsm);
  if (getenv("SLD_DIE_DEBUG")) {
    for (int t = 0; t < nsmid; t++) {
      if (!H[t]) continue;
      fprintf(stderr, "die probe sm %3d:", t);
      for (int i = 0; i < 24; i++) fprintf(stderr, " %u", L[(size_t)t * DIE_PROBES + i]);
      fprintf(stderr, "\n");
    }
  }
  // Measured on B200 (profiles/die_probe_r01.txt): after the discard, SMs of
  // one die see ~600/~980 cycles (near/far HBM), SMs of the other ~300/~600
  // (the lines are still served from the first die's L2), with the same
  // per-line pattern.  Either way the per-SM mean latency falls into two
  // clusters, one per die: split at the widest gap of the sorted means.
  std::vector<std::pair<double, int>> mean;
  for (int t = 0; t < nsmid; t++) {
    if (!H[t]) continue;
    double m = 0;
    for (int i = 0; i < DIE_PROBES; i++) m += L[(size_t)t * DIE_PROBES + i];
    mean.push_back({m / DIE_PROBES, t});
  }
  std::sort(mean.begin(), mean.end());
  size_t cut = 0;
  double gap = 0;
  for (size_t k = 1; k < mean.size(); k++)
    if (mean[k].first - mean[k - 1].first > gap) {
      gap = mean[k].first - mean[k - 1].first;
      cut = k;
    }
  d.ok = true;
  const double spread0 = mean.empty() ? 0 : mean[cut ? cut - 1 : 0].first - mean[0].first;
  const double spread1 = mean.empty() ? 0 : mean.back().first - mean[cut].first;
  if (mean.size() < 2 || gap < 100 || gap < 2 * std::max(spread0, spread1) || cut < 8 || mean.size() - cut < 8) {
    d.ok = false;
    d.why = "no two-cluster latency split (gap " + std::to_string((int)gap) + " cycles)";
  } else {
    // label the die of the lowest smid 0
    const int first = std::min_element(mean.begin(), mean.end(),
                                       [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
                                         return a.second < b.second;
                                       })->second;
    bool first_low = false;
    for (size_t k = 0; k < cut; k++) first_low |= mean[k].second == first;
    for (size_t k = 0; k < mean.size(); k++) {
      const int die = (k < cut) == first_low ? 0 : 1;
      d.map[mean[k].second] = (uint8_t)die;
      d.n[die]++;
    }
  }
  if (d.ok && (d.n[0] == 0 || d.n[1] == 0)) {
    d.ok = false;
    d.why = "all SMs on one die";
  }
  if (!d.ok) memset(d.map, 0, sizeof(d.map));
  (void)dev;
  return SLD_OK;
}
}  // namespace

static const DieMap* die_map(int dev, int sms) {
  std::lock_guard<std::mutex> g(g_die_mu);
  if (dev < 0 || dev >= 64) return nullptr;
  DieMap& d = g_die[dev];
  if (!d.probed) {
    d.probed = true;
    if (probe_dies(dev, d, sms) != SLD_OK) {
      d.ok = false;
      d.why = "probe failed: " + g_err;
    }
  }
  return &d;
}

// the context's device copy of the die map, probed on first use (only the
// opt-in die split needs it; the probe costs ~0.7 s once per process)
static int ctx_dies(sld_ctx* c) {
  if (c->die_map) return SLD_OK;
  const DieMap* d = die_map(c->dev, c->sms);
  CU(cudaMalloc(&c->die_map, 256));
  CU(h2d(c->die_map, d->map, 256, c->stream));
  if (d->ok) {
    c->die_n[0] = d->n[0];
    c->die_n[1] = d->n[1];
  }
  return SLD_OK;
}

extern "C" int sld_die_map(int device, uint8_t* map256, int* n_die0, int* n_die1) {
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(SLD_E_ARG, "device %d out of range (%d)", device, ndev);
  CU(cudaSetDevice(device));
  cudaDeviceProp pr;
  CU(cudaGetDeviceProperties(&pr, device));
  const DieMap* d = die_map(device, pr.multiProcessorCount);
  if (map256) memcpy(map256, d->map, 256);
  if (n_die0) *n_die0 = d->n[0];
  if (n_die1) *n_die1 = d->n[1];
  if (!d->ok) return fail(SLD_E_CUDA, "die map unavailable: %s", d->why.c_str());
  return SLD_OK;
}

// ------------------------------------------------------------- context

extern "C" int sld_ctx_create(int device, const uint32_t* ell_limbs, int L, sld_ctx** out) {
  if (!out || !ell_limbs) return fail(SLD_E_ARG, "null argument");
  while (L > 1 && ell_limbs[L - 1] == 0) L--;
  if (L < 1 || L > MAXL) return fail(SLD_E_ARG, "modulus must have 1..%d 32-bit words", MAXL);
  const int bits = bitlen(ell_limbs, L);
  if (bits < 2 || (ell_limbs[0] & 1) == 0 || (L == 1 && ell_limbs[0] < 3))
    return fail(SLD_E_ARG, "modulus must be an odd prime >= 3");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(SLD_E_ARG, "device %d out of range (%d)", device, ndev);
  CU(cudaSetDevice(device));
  auto c = std::make_unique<sld_ctx>();
  c->dev = device;
  c->L = L;
  c->SW = stride_words(L);
  ModParams& mp = c->mp;
  memset(&mp, 0, sizeof(mp));
  mp.L = L;
  mp.bits = bits;
  for (int i = 0; i < L; i++) mp.ell[i] = ell_limbs[i];
  // K = ell * 2^48 over L+2 words: word i = (ell_{i-1} << 16) | (ell_{i-2} >> 16)
  for (int i = 0; i < L + 2; i++) {
    const uint32_t w1 = (i >= 1 && i - 1 < L) ? mp.ell[i - 1] : 0u;
    const uint32_t w2 = (i >= 2 && i - 2 < L) ? mp.ell[i - 2] : 0u;
    mp.K[i] = (w1 << 16) | (w2 >> 16);
  }
  // mu = floor(2^(bits-1+64) / ell): long division of 2^(bits-1) * 2^64
  {
    std::vector<uint32_t> r(L + 1, 0);
    const int b = bits - 1;
    r[b >> 5] = 1u << (b & 31);  // 2^(bits-1) < ell
    uint64_t q = 0;
    for (int k = 0; k < 64; k++) {
      // r = 2r; if r >= ell: r -= ell, bit = 1
      uint32_t c = 0;
      for (int i = 0; i <= L; i++) {
        uint32_t nc = r[i] >> 31;
        r[i] = (r[i] << 1) | c;
        c = nc;
      }
      bool ge = r[L] != 0;
      if (!ge) {
        ge = true;
        for (int i = L - 1; i >= 0; i--)
          if (r[i] != mp.ell[i]) { ge = r[i] > mp.ell[i]; break; }
      }
      q <<= 1;
      if (ge) {
        int64_t br = 0;
        for (int i = 0; i <= L; i++) {
          int64_t v = (int64_t)r[i] - (i < L ? mp.ell[i] : 0) + br;
          r[i] = (uint32_t)v;
          br = v >> 32;
        }
        q |= 1;
      }
    }
    mp.mu = q;
  }
  // Montgomery: nprime = -ell^-1 mod 2^32, R2 = 2^(64 L) mod ell
  {
    uint32_t inv = 1;
    for (int i = 0; i < 6; i++) inv *= 2u - mp.ell[0] * inv;
    mp.nprime = 0u - inv;
    std::vector<uint32_t> r(L, 0);
    r[0] = 1;  // 1 < ell
    for (int k = 0; k < 64 * L; k++) hmod_double(r.data(), mp.ell, L);
    for (int i = 0; i < L; i++) mp.R2[i] = r[i];
  }
  cudaDeviceProp pr;
  CU(cudaGetDeviceProperties(&pr, device));
  c->l2_bytes = pr.l2CacheSize;
  c->sms = pr.multiProcessorCount;
  c->apw_max = pr.accessPolicyMaxWindowSize > 0 ? (size_t)pr.accessPolicyMaxWindowSize : 0;
  if (getenv("SLD_APW") && pr.persistingL2CacheMaxSize > 0)
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, pr.persistingL2CacheMaxSize);
  CU(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  CU(cudaMalloc(&c->coef, (size_t)64 * c->SW * 4));
  if (L <= 8) {
    const int top = std::max(2 * L, TC_FOLD_TOP);
    std::vector<uint32_t> r(L, 0), tab((size_t)(top - L + 1) * L);
    r[0] = 1;
    for (int k = 0; k <= top; k++) {
      if (k >= L) std::copy(r.begin(), r.end(), tab.begin() + (size_t)(k - L) * L);
      for (int b = 0; b < 32; b++) hmod_double(r.data(), mp.ell, L);
    }
    CU(cudaMalloc(&c->fold, tab.size() * 4));
    CU(h2d(c->fold, tab.data(), tab.size() * 4, c->stream));
  }
  *out = c.release();
  return SLD_OK;
}

extern "C" int sld_ctx_destroy(sld_ctx* c) {
  ctx_unref(c);  // freed once the last object made on it is destroyed too
  return SLD_OK;
}

void ctx_free(sld_ctx* c) {
  cudaSetDevice(c->dev);
  if (c->own) cudaStreamDestroy(c->own);
  if (c->die_map) cudaFree(c->die_map);
  if (c->fold) cudaFree(c->fold);
  if (c->coef) cudaFree(c->coef);
  if (c->hstage) cudaFreeHost(c->hstage);
  if (c->dstage) cudaFree(c->dstage);
  delete c;
}

extern "C" int sld_ctx_sync(sld_ctx* c) {
  CU(cudaSetDevice(c->dev));
  CU(cudaStreamSynchronize(c->stream));
  return SLD_OK;
}

extern "C" int sld_ctx_set_stream(sld_ctx* c, uint64_t stream) {
  if (!c) return fail(SLD_E_ARG, "null context");
  CU(cudaSetDevice(c->dev));
  CU(cudaStreamSynchronize(c->stream));
  c->stream = stream ? (cudaStream_t)(uintptr_t)stream : c->own;
  return SLD_OK;
}

extern "C" int sld_add_mod(sld_ctx* c, const uint64_t* src_ptrs, int k, uint64_t dst_ptr, int64_t n) {
  if (!c || !src_ptrs || k < 1 || k > 64 || n < 0 || !dst_ptr) return fail(SLD_E_ARG, "bad add_mod arguments");
  CU(cudaSetDevice(c->dev));
  AddModArgs a;
  memset(&a, 0, sizeof(a));
  for (int i = 0; i < k; i++) a.src[i] = (const uint32_t*)(uintptr_t)src_ptrs[i];
  a.dst = (uint32_t*)(uintptr_t)dst_ptr;
  a.k = k;
  a.n = n;
  ops(c->L).add_mod(a, c->mp, c->stream);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  return SLD_OK;
}

// ------------------------------------------------------------- vectors

static int vec_alloc_buf(sld_vec* v, int which) {
  if (v->buf[which]) return SLD_OK;
  const size_t words = (size_t)(v->n + 1) * v->chains * v->ctx->SW;
  CU(cudaMalloc(&v->buf[which], words * 4));
  CU(cudaMemsetAsync(v->buf[which], 0, words * 4, v->ctx->stream));
  for (int c = 0; c < v->chains; c++)  // record n: the zero residue of every chain
    ops(v->ctx->L).zero_slot(v->buf[which] + ((size_t)v->n * v->chains + c) * v->ctx->SW, v->ctx->stream);
  CU(cudaGetLastError());
  return SLD_OK;
}

extern "C" int sld_vec_create_chains(sld_ctx* ctx, int64_t n, int chains, sld_vec** out) {
  if (!ctx || !out || n < 0) return fail(SLD_E_ARG, "bad vector arguments");
  if (chains != 1 && chains != 2 && chains != 4) return fail(SLD_E_ARG, "chains must be 1, 2 or 4");
  CU(cudaSetDevice(ctx->dev));
  auto v = std::make_unique<sld_vec>();
  v->ctx = ctx;
  v->ref.bind(ctx);
  v->n = n;
  v->chains = chains;
  TRY(vec_alloc_buf(v.get(), 0));
  CU(cudaStreamSynchronize(ctx->stream));
  *out = v.release();
  return SLD_OK;
}

extern "C" int sld_vec_create(sld_ctx* ctx, int64_t n, sld_vec** out) {
  return sld_vec_create_chains(ctx, n, 1, out);
}

extern "C" int sld_vec_destroy(sld_vec* v) {
  if (!v) return SLD_OK;
  cudaSetDevice(v->ctx->dev);
  for (auto* b : v->buf)
    if (b) cudaFree(b);
  delete v;
  return SLD_OK;
}

extern "C" int sld_vec_device_ptr(sld_vec* v, uint64_t* ptr, int64_t* stride) {
  *ptr = (uint64_t)(uintptr_t)v->buf[v->cur];
  *stride = v->ctx->SW;
  return SLD_OK;
}

// ---- host <-> device transfers: threaded repack into pinned staging, DMA
// in chunks so the CPU repack of chunk k+1 overlaps the copy of chunk k.

static int ensure_stage(sld_ctx* c, size_t bytes) {
  if (c->hstage_bytes < bytes) {
    if (c->hstage) cudaFreeHost(c->hstage);
    c->hstage = nullptr;
    c->hstage_bytes = 0;
    CU(cudaHostAlloc(&c->hstage, bytes, cudaHostAllocPortable));
    c->hstage_bytes = bytes;
  }
  if (c->dstage_bytes < bytes) {
    if (c->dstage) cudaFree(c->dstage);
    c->dstage = nullptr;
    c->dstage_bytes = 0;
    CU(cudaMalloc(&c->dstage, bytes));
    c->dstage_bytes = bytes;
  }
  return SLD_OK;
}

template <typename F>
static void host_par(int64_t n, F f, int64_t min_n = 65536) {
  const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < min_n || nt == 1 || n < 2) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; t++) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo < hi) th.emplace_back([=] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}


// digit planes (P 16-bit digits per residue, one per uint64 cell: the
// reference's format, vecops.py:22-47) <-> L 32-bit limbs, n residues.  The
// repack runs at host memory speed only when the limb count is a compile-time
// constant (unrolled, vectorisable): one instance per L, P = 2L or 2L - 1
// (the widths a modulus of L limbs has), a generic loop otherwise.
template <int L>
static void pack_planes(const uint64_t* __restrict__ src, int P, uint32_t* __restrict__ dst, int64_t n) {
  if (P == 2 * L) {
    for (int64_t r = 0; r < n; r++) {
      const uint64_t* s = src + r * (2 * L);
      uint32_t* d = dst + r * L;
#pragma GCC unroll 32
      for (int j = 0; j < L; j++) d[j] = (uint32_t)(s[2 * j] & 0xFFFF) | ((uint32_t)(s[2 * j + 1] & 0xFFFF) << 16);
    }
  } else if (P == 2 * L - 1) {
    for (int64_t r = 0; r < n; r++) {
      const uint64_t* s = src + r * (2 * L - 1);
      uint32_t* d = dst + r * L;
#pragma GCC unroll 32
      for (int j = 0; j < L - 1; j++)
        d[j] = (uint32_t)(s[2 * j] & 0xFFFF) | ((uint32_t)(s[2 * j + 1] & 0xFFFF) << 16);
      d[L - 1] = (uint32_t)(s[2 * L - 2] & 0xFFFF);
    }
  } else {
    for (int64_t r = 0; r < n; r++) {
      const uint64_t* s = src + r * P;
      for (int j = 0; j < L; j++) {
        const uint32_t d0 = 2 * j < P ? (uint32_t)(s[2 * j] & 0xFFFF) : 0u;
        const uint32_t d1 = 2 * j + 1 < P ? (uint32_t)(s[2 * j + 1] & 0xFFFF) : 0u;
        dst[r * L + j] = d0 | (d1 << 16);
      }
    }
  }
}

template <int L>
static void unpack_planes(const uint32_t* __restrict__ src, uint64_t* __restrict__ dst, int P, int64_t n) {
  if (P == 2 * L) {
    for (int64_t r = 0; r < n; r++) {
      const uint32_t* s = src + r * L;
      uint64_t* d = dst + r * (2 * L);
#pragma GCC unroll 32
      for (int j = 0; j < L; j++) {
        d[2 * j] = s[j] & 0xFFFF;
        d[2 * j + 1] = s[j] >> 16;
      }
    }
  } else if (P == 2 * L - 1) {
    for (int64_t r = 0; r < n; r++) {
      const uint32_t* s = src + r * L;
      uint64_t* d = dst + r * (2 * L - 1);
#pragma GCC unroll 32
      for (int j = 0; j < L - 1; j++) {
        d[2 * j] = s[j] & 0xFFFF;
        d[2 * j + 1] = s[j] >> 16;
      }
      d[2 * L - 2] = s[L - 1] & 0xFFFF;
    }
  } else {
    for (int64_t r = 0; r < n; r++)
      for (int q = 0; q < P; q++) {
        const int j = q >> 1;
        const uint32_t w = j < L ? src[r * L + j] : 0u;
        dst[r * P + q] = (q & 1) ? (w >> 16) : (w & 0xFFFF);
      }
  }
}

using PackFn = void (*)(const uint64_t*, int, uint32_t*, int64_t);
using UnpackFn = void (*)(const uint32_t*, uint64_t*, int, int64_t);
template <int L>
static void fill_pack(PackFn* p, UnpackFn* u) {
  p[L] = pack_planes<L>;
  u[L] = unpack_planes<L>;
  if constexpr (L > 1) fill_pack<L - 1>(p, u);
}
static const PackFn* pack_tab(UnpackFn** u_out) {
  static PackFn p[MAXL + 1];
  static UnpackFn u[MAXL + 1];
  static bool init = [] {
    fill_pack<MAXL>(p, u);
    return true;
  }();
  (void)init;
  *u_out = u;
  return p;
}

// pack n rows into the pinned staging buffer with non-temporal stores: the
// 16-byte streaming stores skip the read-for-ownership a cached store of a
// fresh line costs (100 MB of extra host-memory reads at cfg3, on a path
// bound by host memory).  Rows go through a small cached buffer; the sfence
// makes them visible before the caller queues the DMA.  SLD_NT_STORE=0: off.
static void pack_rows_nt(PackFn pack, const uint64_t* src, int P, uint32_t* dst, int64_t n, int L) {
#if defined(__x86_64__)
  static const bool nt = !getenv("SLD_NT_STORE") || atoi(getenv("SLD_NT_STORE")) != 0;
  if (nt) {
    int64_t r = 0;
    while (r < n && ((uintptr_t)(dst + (size_t)r * L) & 15)) {  // up to 3 rows to a 16-byte boundary
      pack(src + (size_t)r * P, P, dst + (size_t)r * L, 1);
      r++;
    }
    if (((uintptr_t)(dst + (size_t)r * L) & 15) == 0) {
      alignas(64) uint32_t buf[64 * MAXL];
      for (; r + 64 <= n; r += 64) {  // 64 rows = 64 L words, a multiple of 4: stays aligned
        pack(src + (size_t)r * P, P, buf, 64);
        __m128i* d = (__m128i*)(dst + (size_t)r * L);
        const __m128i* b = (const __m128i*)buf;
        for (int i = 0; i < 16 * L; i++) _mm_stream_si128(d + i, _mm_load_si128(b + i));
      }
      _mm_sfence();
    }
    if (r < n) pack(src + (size_t)r * P, P, dst + (size_t)r * L, n - r);
    return;
  }
#endif
  pack(src, P, dst, n);
}

// the download's counterpart: n rows of limbs unpacked into the caller's
// planes array (P uint64 cells per row, 3.7x the limb bytes) with streaming
// stores, so the 374 MB written at cfg3 are not first read for ownership
static void unpack_rows_nt(UnpackFn unpack, const uint32_t* src, uint64_t* dst, int P, int64_t n, int L) {
#if defined(__x86_64__)
  static const bool nt = !getenv("SLD_NT_STORE") || atoi(getenv("SLD_NT_STORE")) != 0;
  if (nt) {
    int64_t r = 0;
    while (r < n && ((uintptr_t)(dst + (size_t)r * P) & 15)) {  // one row to a 16-byte boundary
      unpack(src + (size_t)r * L, dst + (size_t)r * P, P, 1);
      r++;
    }
    if (((uintptr_t)(dst + (size_t)r * P) & 15) == 0) {
      alignas(64) uint64_t buf[32 * 2 * MAXL];
      for (; r + 32 <= n; r += 32) {  // 32 rows = 32 P cells, an even count: stays aligned
        unpack(src + (size_t)r * L, buf, P, 32);
        __m128i* d = (__m128i*)(dst + (size_t)r * P);
        const __m128i* b = (const __m128i*)buf;
        for (int i = 0; i < 16 * P; i++) _mm_stream_si128(d + i, _mm_load_si128(b + i));
      }
      _mm_sfence();
    }
    if (r < n) unpack(src + (size_t)r * L, dst + (size_t)r * P, P, n - r);
    return;
  }
#endif
  unpack(src, dst, P, n);
}

// rows of planes (P 16-bit digits in uint64 cells) or limbs (L words) -> device slots
// planes of chain g at planes_g[g] (nullptr: all chains contiguous at `planes`)
static int upload_rows(sld_vec* v, const uint64_t* planes, const uint32_t* limbs, int64_t rows, int P,
                       const uint64_t* const* planes_g = nullptr) {
  sld_ctx* c = v->ctx;
  const int L = c->L;
  const int64_t n = rows * v->chains;  // items, chain-major on the host
  const size_t bytes = (size_t)n * L * 4;
  if (!n) return SLD_OK;
  TRY(ensure_stage(c, bytes));
  uint32_t* h = (uint32_t*)c->hstage;
  uint32_t* d = (uint32_t*)c->dstage;
  UnpackFn* ut;
  const PackFn pack = pack_tab(&ut)[L];
  // every host thread packs its own contiguous range in sub-chunks and
  // queues each sub-chunk's DMA as soon as it is packed: the copies overlap
  // the packing, and there is one thread spawn per call (the host reads the
  // planes at ~120 GB/s with 16 threads; cfg3's 374 MB took 8 ms chunk by
  // chunk, fork-join per chunk)
  std::atomic<int> dma_err{0};
  host_par(n, [&](int64_t a, int64_t b) {
    constexpr int64_t SUB = 1 << 16;  // rows per queued copy
    for (int64_t lo = a; lo < b; lo += SUB) {
      const int64_t hi = std::min(b, lo + SUB);
      if (planes && !planes_g) {  // one contiguous run of rows
        pack_rows_nt(pack, planes + (size_t)lo * P, P, h + (size_t)lo * L, hi - lo, L);
      } else {
        for (int64_t r = lo; r < hi; r++) {
          uint32_t* dst = h + (size_t)r * L;
          if (planes || planes_g) {
            const uint64_t* src = planes_g ? planes_g[r / rows] + (size_t)(r % rows) * P : planes + (size_t)r * P;
            pack(src, P, dst, 1);
          } else {
            memcpy(dst, limbs + (size_t)r * L, 4 * (size_t)L);
          }
        }
      }
      if (cudaMemcpyAsync(d + (size_t)lo * L, h + (size_t)lo * L, (size_t)(hi - lo) * L * 4,
                          cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        dma_err = 1;
    }
  });
  if (dma_err) return fail(SLD_E_CUDA, "upload: a chunk copy failed to queue");
  ops(L).limbs_to_slots(d, n, v->buf[v->cur], 0x80000000u, rows, v->chains, c->stream);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  return SLD_OK;
}

static int download_rows(sld_vec* v, uint64_t* planes, uint32_t* limbs, int64_t rows, int P,
                         uint64_t* const* planes_g = nullptr) {
  sld_ctx* c = v->ctx;
  const int L = c->L;
  const int64_t n = rows * v->chains;
  const size_t bytes = (size_t)n * L * 4;
  if (!n) return SLD_OK;
  TRY(ensure_stage(c, bytes));
  uint32_t* h = (uint32_t*)c->hstage;
  uint32_t* d = (uint32_t*)c->dstage;
  UnpackFn* ut;
  pack_tab(&ut);
  const UnpackFn unpack = ut[L];
  ops(L).slots_to_limbs(v->buf[v->cur], n, d, 0x80000000u, rows, v->chains, c->stream);
  CU(cudaGetLastError());
  // copies in sub-chunks, each with an event; the host threads unpack a
  // sub-chunk as soon as its copy has landed (one thread spawn per call)
  constexpr int64_t SUB = 1 << 16;
  const int64_t nsub = (n + SUB - 1) / SUB;
  std::vector<cudaEvent_t> ev((size_t)nsub);
  for (int64_t k = 0; k < nsub; k++) {
    const int64_t lo = k * SUB, hi = std::min(n, lo + SUB);
    CU(cudaMemcpyAsync(h + (size_t)lo * L, d + (size_t)lo * L, (size_t)(hi - lo) * L * 4,
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaEventCreateWithFlags(&ev[(size_t)k], cudaEventDisableTiming));
    CU(cudaEventRecord(ev[(size_t)k], c->stream));
  }
  std::atomic<int> err{0};
  host_par(nsub, [&](int64_t ka, int64_t kb) {
    for (int64_t k = ka; k < kb; k++) {
      if (cudaEventSynchronize(ev[(size_t)k]) != cudaSuccess) {
        err = 1;
        return;
      }
      const int64_t lo = k * SUB, hi = std::min(n, lo + SUB);
      if (planes && !planes_g) {
        unpack_rows_nt(unpack, h + (size_t)lo * L, planes + (size_t)lo * P, P, hi - lo, L);
        continue;
      }
      for (int64_t r = lo; r < hi; r++) {
        const uint32_t* src = h + (size_t)r * L;
        if (planes || planes_g) {
          uint64_t* dst = planes_g ? planes_g[r / rows] + (size_t)(r % rows) * P : planes + (size_t)r * P;
          unpack(src, dst, P, 1);
        } else {
          memcpy(limbs + (size_t)r * L, src, 4 * (size_t)L);
        }
      }
    }
  }, 1);
  for (auto e : ev) cudaEventDestroy(e);
  if (err) return fail(SLD_E_CUDA, "download: %s", cudaGetErrorString(cudaGetLastError()));
  return SLD_OK;
}

static int check_P(const sld_ctx* c, int P) {
  if (P < (c->mp.bits + 15) / 16 || P > 2 * c->L + 8)
    return fail(SLD_E_ARG, "digit-plane width %d does not fit a %d-bit modulus", P, c->mp.bits);
  return SLD_OK;
}

extern "C" int sld_vec_upload_planes(sld_vec* v, const uint64_t* planes, int64_t n, int P) {
  if (!v || n != v->n) return fail(SLD_E_ARG, "plane count mismatch");
  TRY(check_P(v->ctx, P));
  CU(cudaSetDevice(v->ctx->dev));
  return upload_rows(v, planes, nullptr, n, P);
}

extern "C" int sld_vec_download_planes(sld_vec* v, uint64_t* planes, int64_t n, int P) {
  if (!v || n > v->n || n < 0 || (v->chains > 1 && n != v->n)) return fail(SLD_E_ARG, "plane count mismatch");
  TRY(check_P(v->ctx, P));
  CU(cudaSetDevice(v->ctx->dev));
  return download_rows(v, planes, nullptr, n, P);
}

extern "C" int sld_vec_upload_planes_chains(sld_vec* v, const uint64_t* const* planes, int64_t n, int P) {
  if (!v || !planes || n != v->n) return fail(SLD_E_ARG, "plane count mismatch");
  for (int g = 0; g < v->chains; g++)
    if (!planes[g]) return fail(SLD_E_ARG, "null chain planes");
  TRY(check_P(v->ctx, P));
  CU(cudaSetDevice(v->ctx->dev));
  return upload_rows(v, nullptr, nullptr, n, P, planes);
}

extern "C" int sld_vec_download_planes_chains(sld_vec* v, uint64_t* const* planes, int64_t n, int P) {
  if (!v || !planes || n != v->n) return fail(SLD_E_ARG, "plane count mismatch");
  for (int g = 0; g < v->chains; g++)
    if (!planes[g]) return fail(SLD_E_ARG, "null chain planes");
  TRY(check_P(v->ctx, P));
  CU(cudaSetDevice(v->ctx->dev));
  return download_rows(v, nullptr, nullptr, n, P, planes);
}

extern "C" int sld_vec_upload_limbs(sld_vec* v, const uint32_t* limbs, int64_t n) {
  if (!v || n != v->n) return fail(SLD_E_ARG, "limb count mismatch");
  CU(cudaSetDevice(v->ctx->dev));
  return upload_rows(v, nullptr, limbs, n, 0);
}

extern "C" int sld_vec_download_limbs(sld_vec* v, uint32_t* limbs, int64_t n) {
  if (!v || n > v->n || n < 0 || (v->chains > 1 && n != v->n)) return fail(SLD_E_ARG, "limb count mismatch");
  CU(cudaSetDevice(v->ctx->dev));
  return download_rows(v, nullptr, limbs, n, 0);
}

extern "C" int sld_lincomb(sld_ctx* c, const uint64_t* y_ptrs, const uint32_t* coeffs, int k,
                           uint64_t acc_ptr, uint64_t dst_ptr, int64_t n) {
  if (!c || k < 0 || k > 64 || n < 0 || !dst_ptr || (k && (!y_ptrs || !coeffs)))
    return fail(SLD_E_ARG, "bad lincomb arguments");
  CU(cudaSetDevice(c->dev));
  LinCombArgs a;
  memset(&a, 0, sizeof(a));
  if (k) {
    // coefficients staged into the context's buffer in stream order (a
    // previous combination still reading it finishes first); plain for the
    // lazy L <= 8 kernel, Montgomery form for the CIOS one
    std::vector<uint32_t> h((size_t)k * c->SW, 0);
    for (int j = 0; j < k; j++)
      for (int i = 0; i < c->L; i++) h[(size_t)j * c->SW + i] = coeffs[(size_t)j * c->L + i];
    CU(cudaMemcpyAsync(c->coef, h.data(), h.size() * 4, cudaMemcpyHostToDevice, c->stream));
    if (c->L > 8) ops(c->L).to_mont(c->coef, k, c->mp, c->stream);
  }
  for (int j = 0; j < k; j++) a.y[j] = (const uint32_t*)(uintptr_t)y_ptrs[j];
  a.coef = c->coef;
  a.fold = c->fold;
  a.acc = (const uint32_t*)(uintptr_t)acc_ptr;
  a.dst = (uint32_t*)(uintptr_t)dst_ptr;
  a.k = k;
  a.n = n;
  ops(c->L).lincomb(a, c->mp, c->stream);
  CU(cudaGetLastError());
  return SLD_OK;
}

// ---- Mksol combination on the tensor cores: a fixed set of n <= 8 vectors
// (the y block) tiled once as byte digits; per Horner step one launch
// combines them with the step's coefficients and adds acc (sld_tcgemm.cuh)
struct sld_lcset {
  CtxRef ref;
  sld_ctx* ctx = nullptr;
  int n = 0;
  int64_t rows = 0, mtiles = 0;
  int grid = 0;
  uint8_t* Y = nullptr;    // [mtiles][n][...] canonical K-major tiles
};

static int lcset_create(sld_ctx* c, const uint64_t* y_ptrs, int n, int64_t rows, const int32_t* perm,
                        sld_lcset** out);

extern "C" int sld_lcset_create(sld_ctx* c, const uint64_t* y_ptrs, int n, int64_t rows, sld_lcset** out) {
  return lcset_create(c, y_ptrs, n, rows, nullptr, out);
}

// the same set tiled in a matrix's slot order: its combinations come out
// slot-ordered (nslots residues), the operand sld_spmv_add reads coalesced
extern "C" int sld_lcset_create_slots(sld_mat* M, const uint64_t* y_ptrs, int n, sld_lcset** out) {
  if (!M) return fail(SLD_E_ARG, "null matrix");
  if (M->chains != 1 || M->halves != 1 || M->sliced) return fail(SLD_E_ARG, "slot-ordered set needs a pass layout");
  return lcset_create(M->ctx, y_ptrs, n, M->nslots, M->slot_row, out);
}

static int lcset_create(sld_ctx* c, const uint64_t* y_ptrs, int n, int64_t rows, const int32_t* perm,
                        sld_lcset** out) {
  if (!c || !out || n < 1 || n > 8 || rows < 0 || !y_ptrs) return fail(SLD_E_ARG, "bad combination set");
  if (c->L > 8) return fail(SLD_E_ARG, "tensor-core combination needs ell < 2^256");
  CU(cudaSetDevice(c->dev));
  auto S = std::make_unique<sld_lcset>();
  S->ctx = c;
  S->ref.bind(c);
  S->n = n;
  S->rows = rows;
  S->mtiles = (rows + 127) / 128;
  S->grid = (int)std::max<int64_t>(1, std::min<int64_t>(S->mtiles, (int64_t)TCL_CTAS_PER_SM * c->sms));
  CU(cudaMalloc(&S->Y, std::max<size_t>((size_t)S->mtiles * tcl_ytile_bytes(n), 16)));
  uint64_t* dptrs = nullptr;
  CU(cudaMalloc(&dptrs, 8 * n));
  CU(h2d(dptrs, y_ptrs, 8 * n, c->stream));
  if (S->mtiles) ops(c->L).tcl_tile((const uint32_t* const*)dptrs, n, rows, S->mtiles, S->Y, perm, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaFree(dptrs);
  if (e != cudaSuccess) return fail(SLD_E_CUDA, "combination set: %s", cudaGetErrorString(e));
  *out = S.release();
  return SLD_OK;
}

extern "C" int sld_lcset_destroy(sld_lcset* S) {
  if (!S) return SLD_OK;
  cudaSetDevice(S->ctx->dev);
  cudaStreamSynchronize(S->ctx->stream);
  if (S->Y) cudaFree(S->Y);
  delete S;
  return SLD_OK;
}

// dst = acc + sum_s coeffs[s] y_s mod ell (coeffs: n x L limbs, canonical;
// acc may be 0).  Asynchronous on the context stream.
extern "C" int sld_lcset_apply(sld_lcset* S, const uint32_t* coeffs, uint64_t acc_ptr, uint64_t dst_ptr) {
  if (!S || !coeffs || !dst_ptr) return fail(SLD_E_ARG, "bad combination arguments");
  sld_ctx* c = S->ctx;
  CU(cudaSetDevice(c->dev));
  const int L = c->L;
  TclCoef cf;
  memset(&cf, 0, sizeof(cf));
  for (int s = 0; s < S->n; s++)
    for (int i = 0; i < L; i++) cf.w[s][i] = coeffs[(size_t)s * L + i];
  if (S->mtiles)
    ops(L).tcl_apply(S->Y, cf, S->n, S->rows, S->mtiles, S->grid, (const uint32_t*)(uintptr_t)acc_ptr,
                     (uint32_t*)(uintptr_t)dst_ptr, c->fold, c->mp, c->stream);
  CU(cudaGetLastError());
  return SLD_OK;
}

// the combinations of K (2 or 4) Horner steps in one pass over the tiled y:
// dst_k = sum_s coeffs[k][s] y_s mod ell (coeffs: K x n x L limbs,
// canonical).  Asynchronous on the context stream.
extern "C" int sld_lcset_apply_batch(sld_lcset* S, const uint32_t* coeffs, int K, const uint64_t* dst_ptrs) {
  if (!S || !coeffs || !dst_ptrs || (K != 2 && K != 4)) return fail(SLD_E_ARG, "bad batched combination");
  sld_ctx* c = S->ctx;
  CU(cudaSetDevice(c->dev));
  uint32_t* d[TCL_KMAX];
  for (int k = 0; k < K; k++) {
    if (!dst_ptrs[k]) return fail(SLD_E_ARG, "null output");
    d[k] = (uint32_t*)(uintptr_t)dst_ptrs[k];
  }
  if (!ops(c->L).tcl_batch(K, S->Y, coeffs, S->n, S->rows, S->mtiles, c->sms, d, c->fold, c->mp, c->stream))
    return fail(SLD_E_ARG, "batched combination needs ell < 2^256");
  CU(cudaGetLastError());
  return SLD_OK;
}

extern "C" int sld_vec_nonzero(sld_vec* v, int* out) {
  if (!v || !out) return fail(SLD_E_ARG, "null argument");
  sld_ctx* c = v->ctx;
  CU(cudaSetDevice(c->dev));
  int* d = nullptr;
  CU(cudaMalloc(&d, 4));
  cudaMemsetAsync(d, 0, 4, c->stream);
  ops(c->L).nonzero(v->buf[v->cur], v->n, d, c->stream);
  int h = 0;
  cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SLD_E_CUDA, "nonzero: %s", cudaGetErrorString(e));
  *out = h;
  return SLD_OK;
}

extern "C" int sld_vec_read_rows(sld_vec* v, const int64_t* rows, int m, uint32_t* limbs) {
  if (!v || m < 0 || (m && (!rows || !limbs))) return fail(SLD_E_ARG, "bad read_rows arguments");
  if (v->chains != 1) return fail(SLD_E_ARG, "read_rows needs a single-chain vector");
  for (int t = 0; t < m; t++)
    if (rows[t] < 0 || rows[t] >= v->n) return fail(SLD_E_ARG, "row out of range");
  if (!m) return SLD_OK;
  sld_ctx* c = v->ctx;
  CU(cudaSetDevice(c->dev));
  int64_t* drows = nullptr;
  uint32_t* dout = nullptr;
  CU(cudaMalloc(&drows, m * 8));
  CU(cudaMalloc(&dout, (size_t)m * c->L * 4));
  cudaMemcpyAsync(drows, rows, m * 8, cudaMemcpyHostToDevice, c->stream);
  ops(c->L).read_rows(v->buf[v->cur], drows, m, dout, c->stream);
  cudaMemcpyAsync(limbs, dout, (size_t)m * c->L * 4, cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  cudaFree(drows);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(SLD_E_CUDA, "read_rows: %s", cudaGetErrorString(e));
  return SLD_OK;
}

// -------------------------------------------------------- matrix build

namespace {

struct RowCounts {
  std::vector<uint32_t> pm;  // [pass][row]
  std::vector<uint32_t> sm;  // [pass][row]
};

template <typename F>
void parallel_for(int64_t n, F f, int nthreads = 0) {
  if (nthreads <= 0) nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 4096 || nthreads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; t++) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

template <typename T>
int dev_upload(T** dst, const std::vector<T>& src, size_t* acct, cudaStream_t s) {
  const size_t bytes = std::max<size_t>(src.size() * sizeof(T), 16);
  CU(cudaMalloc(dst, bytes));
  if (!src.empty()) CU(h2d(*dst, src.data(), src.size() * sizeof(T), s));
  *acct += bytes;
  return SLD_OK;
}

}  // namespace

static void mat_free(sld_mat* m) {
  if (!m) return;
  void* ptrs[] = {m->slices, m->pm_idx, m->s_idx, m->s_coef, m->slot_row, m->lane_k4, m->full_ptr,
                  m->full_col, m->full_val, m->dense_val, m->part, m->stage, m->proj_rows,
                  m->terms_dev, m->dproj_part, m->xch, m->cnt, m->queue, m->mk_y, m->fix_slots, m->chain_bar};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (m->tmp_in) sld_vec_destroy(m->tmp_in);
  if (m->tmp_out) sld_vec_destroy(m->tmp_out);
  delete m;
}

extern "C" int sld_mat_create(sld_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                              const int32_t* col_idx, const uint8_t* tags, const int64_t* small_vals,
                              int64_t n_full, const int64_t* full_pos, const uint32_t* full_limbs,
                              int n_dense, const uint32_t* dense_limbs, int64_t max_stripe_cols,
                              sld_mat** out) {
  return sld_mat_create_chains(ctx, 1, nrows, ncols, row_ptr, col_idx, tags, small_vals, n_full,
                               full_pos, full_limbs, n_dense, dense_limbs, max_stripe_cols, out);
}

extern "C" int sld_mat_destroy(sld_mat* m) {
  if (!m) return SLD_OK;
  cudaSetDevice(m->ctx->dev);
  mat_free(m);
  return SLD_OK;
}

static int mat_build(sld_mat* M, const int64_t* row_ptr, const int32_t* col_idx, const uint8_t* tags,
                     const int64_t* small_vals, int64_t n_full, const int64_t* full_pos,
                     const uint32_t* full_limbs, const uint32_t* dense_limbs, int64_t max_stripe_cols) {
  sld_ctx* c = M->ctx;
  const int L = c->L, SW = c->SW;
  const int64_t nrows = M->nrows, ncols = M->ncols;
  const int64_t nnz = M->nnz;
  const uint32_t PAD = (uint32_t)M->total_cols;  // zero slot
  // ---- validation (spmatrix.py:93-126)
  if (row_ptr[0] != 0) return fail(SLD_E_ARG, "row_ptr[0] must be 0");
  for (int64_t r = 0; r < nrows; r++)
    if (row_ptr[r + 1] < row_ptr[r]) return fail(SLD_E_ARG, "row_ptr must be monotone");
  {
    std::atomic<int> bad{0};
    parallel_for(nnz, [&](int64_t lo, int64_t hi) {
      for (int64_t p = lo; p < hi; p++)
        if (col_idx[p] < 0 || col_idx[p] >= ncols || tags[p] > 3) { bad = 1; return; }
    });
    if (bad) return fail(SLD_E_ARG, "sparse column index out of range or unknown tag");
  }
  for (int64_t k = 0; k < n_full; k++) {
    if (full_pos[k] < 0 || full_pos[k] >= nnz || (k && full_pos[k] <= full_pos[k - 1]))
      return fail(SLD_E_ARG, "full positions must be sorted and in range");
    if (tags[full_pos[k]] != 3) return fail(SLD_E_ARG, "full position without full tag");
  }
  // ---- die split and stripes: keep each pass's gathered columns L2-resident
  const double vec_bytes = (double)(M->total_cols + 1) * SW * 4.0 * M->chains;
  const double l2 = (double)c->l2_bytes;
  int H = 1;
  {
    // measured (tools/microbench/mb3.cu): with every SM gathering every
    // column the L2 holds ~one die's worth (~63 MB); dealing the columns to
    // the dies keeps ~128 MB resident.  In the SpMV the per-slice meeting of
    // the halves costs more than the fewer stripes save (cfg3: 1.63 vs
    // 1.36 ms per chain-product), so the split is opt-in.
    int want = 0;
    if (const char* e = getenv("SLD_SPLIT")) want = atoi(e);
    if (want && !M->sliced && !M->short_rows && nrows > 0) TRY(ctx_dies(c));
    if (want && !M->sliced && !M->short_rows && c->die_n[0] > 0 && c->die_n[1] > 0 && nrows > 0 &&
        ops(L).split_occupancy(M->chains) > 0)
      H = 2;
  }
  int64_t stripe = max_stripe_cols;
  if (stripe <= 0) {
    // measured (tools/sweep.py): without the split, one pass while the
    // gathered vector fits in ~80% of L2 (cfg2 21 MB, cfg5 96 MB), beyond that
    // stripes of <= 1/2 L2 (cfg3: 2 x 58 MB).  With the split, stripes of
    // <= SLD_SPLIT_FRAC (default 0.95) of L2.
    // Limb-sliced (wide) residues: 2 x 48 MB at cfg5 beats one 96 MB pass
    // (1.057 vs 1.12 ms, profiles/sweep_cfg5_stripes_r02.txt): the single
    // pass misses L2 on ~43% of its gathers, and its random DRAM traffic
    // holds the board at its 1000 W cap (SM clock 1.59 GHz vs 1.96).
    double frac_one = M->sliced ? 0.55 : 0.80, frac_many = 0.5;
    if (H == 2) {
      frac_one = frac_many = 0.95;
      if (const char* e = getenv("SLD_SPLIT_FRAC")) frac_one = frac_many = atof(e);
    }
    if (vec_bytes <= frac_one * l2) {
      stripe = ncols;
    } else {
      const int64_t parts = (int64_t)std::ceil(vec_bytes / (frac_many * l2));
      stripe = (ncols + parts - 1) / parts;
    }
    stripe = std::max<int64_t>(1, stripe);
  }
  if (stripe >= ncols) stripe = std::max<int64_t>(ncols, 1);
  // stripe boundaries: equal widths, or explicit ones (SLD_STRIPE_BOUNDS =
  // "b1,b2,..." column indices, for layout sweeps)
  std::vector<int64_t> bounds;
  for (int64_t b = stripe; b < ncols; b += stripe) bounds.push_back(b);
  if (const char* e = getenv("SLD_STRIPE_BOUNDS")) {
    bounds.clear();
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const long long b = strtoll(q, &end, 10);
      if (end == q) break;
      if (b > 0 && b < ncols && (bounds.empty() || b > bounds.back())) bounds.push_back(b);
      q = *end ? end + 1 : end;
    }
  }
  const int npass = (int)bounds.size() + 1;
  M->npass = npass;
  M->stripe_cols = stripe;
  M->halves = H;
  // interleaved chunks of >= 2 KB of whole 128-byte lines, dealt to the dies
  // in proportion to their SM counts (Bresenham), so both the bytes each
  // die's L2 must hold and the gathers each die serves follow its SM share
  const int64_t rec_bytes = (int64_t)SW * 4 * M->chains;
  int64_t line_recs = 1;
  while ((line_recs * rec_bytes) % 128) line_recs++;
  const int64_t HC = line_recs * std::max<int64_t>(1, (2048 + line_recs * rec_bytes - 1) / (line_recs * rec_bytes));
  M->half_chunk = HC;
  const int64_t dn0 = c->die_n[0], dn = c->die_n[0] + c->die_n[1];
  auto half_of = [&](int64_t col) -> int {
    if (H == 1) return 0;
    const int64_t k = col / HC;
    return (((k + 1) * dn0) / dn - (k * dn0) / dn) ? 0 : 1;
  };
  auto part_of = [&](int64_t col) -> int {
    const int pass = (int)(std::upper_bound(bounds.begin(), bounds.end(), col) - bounds.begin());
    return pass * H + half_of(col);
  };
  const int npart = npass * H;
  // ---- per-row, per-pass class counts
  RowCounts rc;
  rc.pm.assign((size_t)npart * nrows, 0);
  rc.sm.assign((size_t)npart * nrows, 0);
  std::vector<uint32_t> fcount(nrows + 1, 0);
  // map flat position -> full value index (only for tag 3); sorted positions
  std::atomic<int> bound_bad{0};
  parallel_for(nrows, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; r++) {
      uint32_t tot_s = 0, tot_pm = 0, nf = 0;
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) {
        const int t = tags[p];
        const int pass = part_of(col_idx[p]);
        if (t <= 1) {
          rc.pm[(size_t)pass * nrows + r]++;
          tot_pm++;
        } else if (t == 2) {
          const int64_t v = small_vals[p];
          if (v > -0x80000000ll && v < 0x80000000ll) {
            rc.sm[(size_t)pass * nrows + r]++;
            tot_s++;
          } else {
            nf++;
          }
        } else {
          nf++;
        }
      }
      fcount[r] = nf;
      if (tot_s > (1u << 15) || tot_pm > (1u << 24)) bound_bad = 1;
    }
  });
  if (bound_bad)
    return fail(SLD_E_BOUND, "row degree too large for exact accumulation "
                             "(> 2^15 small or > 2^24 +-1 entries in a row)");
  // ---- slot order: rows sorted by (+-1 count, small count) descending
  std::vector<int64_t> tot_pm(nrows, 0), tot_s(nrows, 0);
  uint32_t gamma_pm_max = 0, gamma_s_max = 0;
  parallel_for(nrows, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; r++) {
      int64_t a = 0, b = 0;
      for (int p = 0; p < npart; p++) {
        a += rc.pm[(size_t)p * nrows + r];
        b += rc.sm[(size_t)p * nrows + r];
      }
      tot_pm[r] = a;
      tot_s[r] = b;
    }
  });
  for (int64_t r = 0; r < nrows; r++) {
    gamma_pm_max = std::max<uint32_t>(gamma_pm_max, (uint32_t)tot_pm[r]);
    gamma_s_max = std::max<uint32_t>(gamma_s_max, (uint32_t)tot_s[r]);
  }
  std::vector<int32_t> order(nrows);
  for (int64_t r = 0; r < nrows; r++) order[r] = (int32_t)r;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    if (tot_pm[x] != tot_pm[y]) return tot_pm[x] > tot_pm[y];
    return tot_s[x] > tot_s[y];
  });
  // rows per slice: one warp holds RH rows x G chains, or RH rows x T limb slices
  const int RH = M->sliced ? 32 / (SW / 8) : (M->short_rows ? 32 / SHORT_K : 32 / M->chains);
  const int64_t nslices = (nrows + RH - 1) / RH;
  M->nslices = nslices;
  const int64_t nslots = nslices * RH;
  M->nslots = nslots;
  std::vector<int32_t> slot_row(nslots, -1);
  for (int64_t s = 0; s < nrows; s++) slot_row[s] = order[s];
  // ---- slice tables
  std::vector<SliceInfo> slices((size_t)npart * nslices);
  uint64_t pm_units = 0, s_units = 0;
  for (int p = 0; p < npart; p++) {
    for (int64_t s = 0; s < nslices; s++) {
      uint32_t kpm = 0, ks = 0;
      for (int l = 0; l < RH; l++) {
        const int32_t r = slot_row[s * RH + l];
        if (r < 0) continue;
        kpm = std::max(kpm, (rc.pm[(size_t)p * nrows + r] + 3) / 4);
        ks = std::max(ks, (rc.sm[(size_t)p * nrows + r] + 3) / 4);
      }
      SliceInfo& si = slices[(size_t)p * nslices + s];
      si.pm_off = (uint32_t)pm_units;
      si.pm_k4 = kpm;
      si.s_off = (uint32_t)s_units;
      si.s_k4 = ks;
      pm_units += (uint64_t)kpm * RH;
      s_units += (uint64_t)ks * RH;
      if (p == 0) M->chain_units = std::max<int64_t>(M->chain_units, (int64_t)(kpm + 2 * ks) * RH);
      if (pm_units >= (1ull << 32) || s_units >= (1ull << 32))
        return fail(SLD_E_BOUND, "matrix too large for 32-bit slice offsets");
    }
  }
  // per-lane group counts (the SELL slice width is only the max over lanes)
  std::vector<uint32_t> lane_k4((size_t)npart * nslots, 0);
  if (std::max(gamma_pm_max, gamma_s_max) >= (1u << 18))
    return fail(SLD_E_BOUND, "row too long for the per-lane group counter");
  for (int p = 0; p < npart; p++)
    for (int64_t slot = 0; slot < nrows; slot++) {
      const int32_t r = slot_row[slot];
      const uint32_t a = (rc.pm[(size_t)p * nrows + r] + 3) / 4, b = (rc.sm[(size_t)p * nrows + r] + 3) / 4;
      lane_k4[(size_t)p * nslots + slot] = a | (b << 16);
    }
  // ---- entry streams
  std::vector<uint32_t> pm_idx(pm_units * 4, PAD);
  std::vector<uint32_t> s_idx(s_units * 4, PAD);
  std::vector<int32_t> s_coef(s_units * 4, 0);
  // full entries CSR over slots
  std::vector<uint32_t> full_ptr(nslots + 1, 0);
  for (int64_t s = 0; s < nslots; s++) {
    const int32_t r = slot_row[s];
    full_ptr[s + 1] = full_ptr[s] + (r >= 0 ? fcount[r] : 0);
  }
  const int64_t nf_total = full_ptr[nslots];
  std::vector<uint32_t> full_col(nf_total);
  std::vector<uint32_t> full_val((size_t)nf_total * SW, 0);
  std::atomic<int64_t> pads{0};
  parallel_for(nslots, [&](int64_t lo, int64_t hi) {
    std::vector<uint32_t> kp(npart), ks(npart);
    int64_t mypads = 0;
    for (int64_t slot = lo; slot < hi; slot++) {
      const int32_t r = slot_row[slot];
      if (r < 0) continue;
      const int64_t slice = slot / RH;
      const int lane = (int)(slot % RH);
      std::fill(kp.begin(), kp.end(), 0u);
      std::fill(ks.begin(), ks.end(), 0u);
      uint32_t fk = full_ptr[slot];
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) {
        const int t = tags[p];
        const uint32_t col = (uint32_t)col_idx[p];
        const int pass = part_of(col_idx[p]);
        const SliceInfo& si = slices[(size_t)pass * nslices + slice];
        if (t <= 1) {
          const uint32_t k = kp[pass]++;
          const uint64_t pos = ((uint64_t)si.pm_off + (uint64_t)(k >> 2) * RH + lane) * 4 + (k & 3);
          pm_idx[pos] = col | (t == 1 ? 0x80000000u : 0u);
          continue;
        }
        if (t == 2) {
          const int64_t v = small_vals[p];
          if (v > -0x80000000ll && v < 0x80000000ll) {
            const uint32_t k = ks[pass]++;
            const uint64_t pos = ((uint64_t)si.s_off + (uint64_t)(k >> 2) * RH + lane) * 4 + (k & 3);
            s_idx[pos] = col;
            s_coef[pos] = (int32_t)v;
            continue;
          }
          // promoted: value = v mod ell
          uint32_t* dst = &full_val[(size_t)fk * SW];
          hmod_u64(v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v, c->mp.ell, L, dst);
          bool nz = false;
          for (int i = 0; i < L; i++) nz |= dst[i] != 0;
          if (v < 0 && nz) {  // ell - (|v| mod ell)
            int64_t br = 0;
            for (int i = 0; i < L; i++) {
              int64_t x = (int64_t)c->mp.ell[i] - dst[i] + br;
              dst[i] = (uint32_t)x;
              br = x >> 32;
            }
          }
          full_col[fk++] = col;
          continue;
        }
        // tag 3: locate value by binary search over sorted full_pos
        const int64_t* it = std::lower_bound(full_pos, full_pos + n_full, p);
        const int64_t fi = it - full_pos;
        uint32_t* dst = &full_val[(size_t)fk * SW];
        if (fi < n_full && *it == p)
          for (int i = 0; i < L; i++) dst[i] = full_limbs[(size_t)fi * L + i];
        full_col[fk++] = col;
      }
      for (int q = 0; q < npart; q++) {
        mypads += (int64_t)((kp[q] + 3) / 4) * 4 - kp[q] + (int64_t)((ks[q] + 3) / 4) * 4 - ks[q];
      }
    }
    pads += mypads;
  });
  // every tag-3 position must have had a value
  {
    int64_t n3 = 0;
    for (int64_t p = 0; p < nnz; p++) n3 += tags[p] == 3;
    if (n3 != n_full) return fail(SLD_E_ARG, "%lld full-tag entries but %lld full values",
                                  (long long)n3, (long long)n_full);
  }
  // ---- dense columns [g][slot-padded row]
  std::vector<uint32_t> dense_val;
  if (M->n_dense) {
    dense_val.assign((size_t)M->n_dense * nslots * SW, 0);
    for (int g = 0; g < M->n_dense; g++)
      for (int64_t r = 0; r < nrows; r++)
        for (int i = 0; i < L; i++)
          dense_val[((size_t)g * nslots + r) * SW + i] = dense_limbs[((size_t)g * nrows + r) * L + i];
  }
  // ---- stats
  int64_t npm = 0, nsm = 0, mdeg = 0;
  for (int64_t r = 0; r < nrows; r++) {
    npm += tot_pm[r];
    nsm += tot_s[r];
    mdeg = std::max<int64_t>(mdeg, row_ptr[r + 1] - row_ptr[r] + M->n_dense);
  }
  M->n_pm = npm;
  M->n_small = nsm;
  M->n_full = nf_total + (int64_t)M->n_dense * nrows;
  M->pad_entries = pads;
  M->max_deg = mdeg;
  // ---- upload
  CU(cudaSetDevice(c->dev));
  size_t acct = 0;
  TRY(dev_upload(&M->slices, slices, &acct, c->stream));
  CU(cudaMalloc(&M->pm_idx, std::max<size_t>(pm_idx.size() * 4, 16)));
  if (!pm_idx.empty()) CU(h2d(M->pm_idx, pm_idx.data(), pm_idx.size() * 4, c->stream));
  CU(cudaMalloc(&M->s_idx, std::max<size_t>(s_idx.size() * 4, 16)));
  if (!s_idx.empty()) CU(h2d(M->s_idx, s_idx.data(), s_idx.size() * 4, c->stream));
  CU(cudaMalloc(&M->s_coef, std::max<size_t>(s_coef.size() * 4, 16)));
  if (!s_coef.empty()) CU(h2d(M->s_coef, s_coef.data(), s_coef.size() * 4, c->stream));
  acct += pm_idx.size() * 4 + s_idx.size() * 4 + s_coef.size() * 4;
  TRY(dev_upload(&M->slot_row, slot_row, &acct, c->stream));
  TRY(dev_upload(&M->lane_k4, lane_k4, &acct, c->stream));
  TRY(dev_upload(&M->full_ptr, full_ptr, &acct, c->stream));
  TRY(dev_upload(&M->full_col, full_col, &acct, c->stream));
  TRY(dev_upload(&M->full_val, full_val, &acct, c->stream));
  if (nf_total) ops(L).to_mont(M->full_val, nf_total, c->mp, c->stream);
  if (M->n_dense) {
    TRY(dev_upload(&M->dense_val, dense_val, &acct, c->stream));
    ops(L).to_mont(M->dense_val, (int64_t)M->n_dense * nslots, c->mp, c->stream);
  }
  if (M->sliced) {
    // the limb-sliced passes leave full-class entries and dense columns to
    // full_fixup: the slots that have any
    std::vector<int32_t> fix;
    for (int64_t s2 = 0; s2 < nslots; s2++)
      if (slot_row[s2] >= 0 && (M->n_dense || full_ptr[s2 + 1] > full_ptr[s2])) fix.push_back((int32_t)s2);
    M->n_fix = (int64_t)fix.size();
    if (!fix.empty()) TRY(dev_upload(&M->fix_slots, fix, &acct, c->stream));
  }
  if (npass > 1) {
    CU(cudaMalloc(&M->part, (size_t)nslots * M->chains * SW * 4));
    acct += (size_t)nslots * M->chains * SW * 4;
  }
  if (H == 2) {
    const size_t xb = (size_t)nslots * M->chains * SW * 4;
    CU(cudaMalloc(&M->xch, xb));
    CU(cudaMalloc(&M->cnt, std::max<size_t>((size_t)nslices * 4, 16)));
    CU(cudaMemsetAsync(M->cnt, 0, std::max<size_t>((size_t)nslices * 4, 16), c->stream));
    CU(cudaMalloc(&M->queue, 16));
    CU(cudaMemsetAsync(M->queue, 0, 16, c->stream));
    acct += xb + (size_t)nslices * 4 + 16;
    int occ = ops(L).split_occupancy(M->chains);
    if (const char* e = getenv("SLD_SPLIT_OCC")) occ = std::max(1, std::min(occ, atoi(e)));
    M->split_grid = (unsigned)(occ * c->sms);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(c->stream));
  M->dev_bytes = acct;
  return SLD_OK;
}

extern "C" int sld_mat_create_chains(sld_ctx* ctx, int chains, int64_t nrows, int64_t ncols,
                                     const int64_t* row_ptr, const int32_t* col_idx, const uint8_t* tags,
                                     const int64_t* small_vals, int64_t n_full, const int64_t* full_pos,
                                     const uint32_t* full_limbs, int n_dense, const uint32_t* dense_limbs,
                                     int64_t max_stripe_cols, sld_mat** out) {
  if (!ctx) return fail(SLD_E_ARG, "null context");
  if (chains != 1 && chains != 2 && chains != 4)
    return fail(SLD_E_ARG, "chains must be 1, 2 or 4");
  if (chains > max_chains(ctx->L))
    return fail(SLD_E_ARG, "%d chains per record exceed one 128-byte line at %d limbs", chains, ctx->L);
  if (!ctx || !out || !row_ptr || nrows < 0 || ncols < 0 || n_dense < 0 || n_full < 0)
    return fail(SLD_E_ARG, "bad matrix arguments");
  if (nrows >= 0x7FFFFFFF || ncols + n_dense >= 0x7FFFFFFF)
    return fail(SLD_E_ARG, "dimensions must be < 2^31");
  const int64_t nnz = row_ptr[nrows];
  if (nnz && (!col_idx || !tags || !small_vals)) return fail(SLD_E_ARG, "null entry arrays");
  if (n_dense && !dense_limbs) return fail(SLD_E_ARG, "null dense column values");
  if (n_full && (!full_pos || !full_limbs)) return fail(SLD_E_ARG, "null full entries");
  CU(cudaSetDevice(ctx->dev));
  sld_mat* M = new sld_mat();
  M->ctx = ctx;
  M->ref.bind(ctx);
  M->chains = chains;
  M->nrows = nrows;
  M->ncols = ncols;
  M->n_dense = n_dense;
  M->total_cols = ncols + n_dense;
  M->nnz = nnz;
  if (const char* pe = getenv("SLD_POLICY")) M->policy = atoi(pe);
  if (const char* pe = getenv("SLD_PF")) M->pf = std::max(0, atoi(pe));
  {
    // wide moduli: one gather request per residue instead of SW/8 (cfg5: 1.15 vs 1.24 ms)
    int wide = 1;
    if (const char* pe = getenv("SLD_WIDE")) wide = atoi(pe);
    M->sliced = (wide && chains == 1 && ctx->SW >= 16) ? 1 : 0;
    // small matrices: one lane per row leaves most SMs idle (fewer than ~16
    // warps per SM) and each warp walks its row's groups serially
    int sh = (chains == 1 && ctx->SW <= 8 && nrows < 32LL * 16 * ctx->sms) ? 1 : 0;
    if (const char* pe = getenv("SLD_SHORT")) sh = atoi(pe) && chains == 1 && ctx->SW <= 8;
    M->short_rows = sh;
    // index prefetch two groups ahead, except for the one-chain pass layout,
    // whose one-sector gathers already saturate the SM's request interface:
    // there the prefetches are requests that cost more than they hide (cfg3
    // 1.581 vs 1.607 ms, cfg2 0.2747 vs 0.2762 ms; the limb-sliced cfg5
    // wants them: 0.997 vs 1.055 ms; profiles/sweep_pf_g1_r02.txt)
    if (!getenv("SLD_PF")) M->pf = (chains == 1 && !M->sliced && !M->short_rows) ? 0 : 2;
  }
  if (const char* pe = getenv("SLD_CHAIN")) M->chain_ok = atoi(pe) != 0;
  if (const char* pe = getenv("SLD_APW")) M->apw = atoi(pe);
  if (const char* pe = getenv("SLD_APW_RATIO")) M->apw_ratio = (float)atof(pe);
  int r = mat_build(M, row_ptr, col_idx, tags, small_vals, n_full, full_pos, full_limbs, dense_limbs,
                    max_stripe_cols);
  if (r != SLD_OK) {
    mat_free(M);
    return r;
  }
  *out = M;
  return SLD_OK;
}

extern "C" int sld_mat_info(const sld_mat* m, int64_t* info) {
  if (!m || !info) return fail(SLD_E_ARG, "null argument");
  int64_t v[20] = {m->nrows, m->total_cols, m->nnz, m->n_pm, m->n_small, m->n_full,
                   m->npass, m->nslices, (int64_t)m->dev_bytes, m->pad_entries,
                   m->ctx->L, m->ctx->SW, m->max_deg, m->stripe_cols, m->chains, m->halves,
                   m->sliced ? m->ctx->SW / 8 : 1, m->nslices ? m->nslots / m->nslices : 0, m->pf, 0};
  memcpy(info, v, sizeof(v));
  return SLD_OK;
}

// ------------------------------------------------------------- SpMV

// the arguments every pass of one product shares
static void product_args(sld_mat* M, const uint32_t* x, uint32_t* y, const int64_t* proj_rows, int proj_m,
                         uint32_t* terms_out, SpmvArgs& a) {
  memset(&a, 0, sizeof(a));
  a.x = x;
  a.y = y;
  a.part_in = M->part;
  a.part_out = M->part;
  a.pm_idx = M->pm_idx;
  a.s_idx = M->s_idx;
  a.s_coef = M->s_coef;
  a.slot_row = M->slot_row;
  a.full_ptr = M->full_ptr;
  a.full_col = M->full_col;
  a.full_val = M->full_val;
  a.dense_val = M->dense_val;
  a.n_dense = M->n_dense;
  a.dense_col0 = M->ncols;
  a.proj_rows = proj_rows;
  a.proj_m = proj_m;
  a.terms_out = terms_out;
  a.nslices = M->nslices;
  a.nslots = M->nslots;
  a.has_full = (M->full_ptr && M->n_full) ? 1 : 0;
  a.policy = M->policy;
  a.pf = (uint32_t)M->pf;
}

// launch all stripe passes of one product on the context stream
void launch_product(sld_mat* M, const uint32_t* x, uint32_t* y, const int64_t* proj_rows,
                    int proj_m, uint32_t* terms_out, const uint32_t* mk_coeffs, const uint32_t* addv) {
  sld_ctx* c = M->ctx;
  SpmvArgs a;
  product_args(M, x, y, proj_rows, proj_m, terms_out, a);
  a.addv = addv;
  if (!y && M->npeer) {
    a.npeer = M->npeer;
    for (int k = 0; k < M->npeer; k++) a.yp[k] = M->yp[k];
    a.peer_off = M->peer_off;
  }
  if (mk_coeffs) {
    a.mk_y = M->mk_y;
    a.mk_n = M->mk_n;
    a.fold = c->fold;
    for (int s = 0; s < M->mk_n; s++)
      for (int i = 0; i < c->L; i++) a.mk_c[s][i] = mk_coeffs[(size_t)s * c->L + i];
  }
  const LOps& o = ops(c->L);
  if (M->nslices == 0) {
    // no rows: still record the projection
    if (proj_m) {
      a.nslices = 0;
      a.slices = M->slices;
      a.lane_k4 = M->lane_k4;
      o.pass(M->chains, 1, 1, 1, c->stream, a, c->mp);
    }
    return;
  }
  if (M->halves == 2) {
    a.die_map = c->die_map;
    a.xch = M->xch;
    a.cnt = M->cnt;
    a.queue = M->queue;
    for (int p = 0; p < M->npass; p++) {
      a.slices = M->slices + (size_t)p * 2 * M->nslices;
      a.lane_k4 = M->lane_k4 + (size_t)p * 2 * M->nslots;
      o.split(M->chains, p == 0, p == M->npass - 1, M->split_grid, c->stream, a, c->mp);
    }
    return;
  }
  for (int p = 0; p < M->npass; p++) {
    a.slices = M->slices + (size_t)p * M->nslices;
    a.lane_k4 = M->lane_k4 + (size_t)p * M->nslots;
    if (M->sliced) {
      o.wide(p == 0, p == M->npass - 1, M->nslices, c->stream, a, c->mp);
      continue;
    }
    if (M->short_rows) {
      o.short_pass(p == 0, p == M->npass - 1, M->nslices, c->stream, a, c->mp);
      continue;
    }
    if (M->apw && c->apw_max) {
      // persisting L2 window over the stripe this pass gathers from
      const int64_t lo = (int64_t)p * M->stripe_cols;
      const int64_t hi = std::min<int64_t>(M->total_cols + 1, lo + M->stripe_cols);
      cudaStreamAttrValue v;
      memset(&v, 0, sizeof(v));
      v.accessPolicyWindow.base_ptr = (void*)(x + (size_t)lo * c->SW);
      v.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)(hi - lo) * c->SW * 4, c->apw_max);
      v.accessPolicyWindow.hitRatio = M->apw_ratio;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    if (mk_coeffs && p == M->npass - 1) o.pass_mk(p == 0, M->nslices, c->stream, a, c->mp);
    else o.pass(M->chains, p == 0, p == M->npass - 1, M->nslices, c->stream, a, c->mp);
  }
  if (M->sliced && M->n_fix) {
    a.slices = M->slices;  // (unused by the fixup)
    o.fixup(a, c->mp, M->fix_slots, M->n_fix, c->stream);
  }
  if (M->apw && c->apw_max) {
    cudaStreamAttrValue v;
    memset(&v, 0, sizeof(v));
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  }
}

// The persistent chain (spmv_chain): small one-pass short-row matrices run
// many products per launch.  Opt-in (SLD_CHAIN=1): measured on B200 it is
// slower than the per-product graphs (cfg1 7.0 vs 6.0 us per product) -- its
// grid barrier costs 1.3-1.6 us (2+ us with >400 CTAs), as much as the kernel
// boundary it removes, and a product's gathers are bound by the per-SM
// request rate, not by the launch (profiles/chain_cfg1_r02.txt).
static bool chain_eligible(const sld_mat* M) {
  return M->chain_ok && M->short_rows && M->npass == 1 && M->halves == 1 && !M->npeer && M->chains == 1 &&
         M->ctx->L <= 8 && M->nslices > 0 && M->nrows == M->total_cols;
}

// `steps` products of the chain starting in x (result in x if steps is even,
// else in y), the projection of product t's input to terms + t * tstride
static int launch_chain(sld_mat* M, uint32_t* x, uint32_t* y, int64_t steps, const int64_t* proj_rows, int m,
                        uint32_t* terms, int64_t tstride) {
  sld_ctx* c = M->ctx;
  const LOps& o = ops(c->L);
  static const int env_grid = getenv("SLD_CHAIN_GRID") ? atoi(getenv("SLD_CHAIN_GRID")) : 0;
  static const int env_mode = getenv("SLD_CHAIN_MODE") ? atoi(getenv("SLD_CHAIN_MODE")) : 0;
  static const int env_l1 = getenv("SLD_CHAIN_L1") ? atoi(getenv("SLD_CHAIN_L1")) : 1;
  static const int env_cap = getenv("SLD_CHAIN_CAP") ? atoi(getenv("SLD_CHAIN_CAP")) : 384;
  // shared-memory staging of each warp's slice: up to env_cap uint4 (6 KB) per warp
  const uint32_t wcap = (uint32_t)std::min<int64_t>(std::max(env_cap, 0), M->chain_units);
  static const int tb = getenv("SLD_CHAIN_TB") ? atoi(getenv("SLD_CHAIN_TB")) : 64;
  const size_t smem = (size_t)(tb / 32) * wcap * 16;
  const int occ = o.chain_occupancy(env_l1, tb, smem);
  if (occ < 1) return fail(SLD_E_CUDA, "persistent chain kernel cannot be resident");
  if (!M->chain_bar) CU(cudaMalloc(&M->chain_bar, 128));
  // small CTAs spread the slices evenly over the SMs
  unsigned grid = (unsigned)std::min<int64_t>((int64_t)occ * c->sms, (M->nslices * 32 + tb - 1) / tb);
  if (env_grid > 0) grid = std::min<unsigned>(grid, (unsigned)env_grid);
  SpmvArgs a;
  product_args(M, x, y, proj_rows, m, nullptr, a);
  a.slices = M->slices;  // the one pass
  a.lane_k4 = M->lane_k4;
  a.pf = 0;  // the index streams are L2-resident from the second product on
  ChainArgs ch;
  // barrier targets (t + 1) * grid stay below 2^32 per launch
  const int64_t per = std::max<int64_t>(2, ((int64_t)1 << 31) / grid) & ~(int64_t)1;
  for (int64_t done = 0; done < steps;) {
    const int64_t n = std::min(per, steps - done);
    ch.buf[0] = x;
    ch.buf[1] = y;
    ch.bar = M->chain_bar;
    ch.terms = terms ? terms + (size_t)done * tstride : nullptr;
    ch.tstride = tstride;
    ch.steps = n;
    ch.mode = env_mode;
    ch.wcap = wcap;
    CU(cudaMemsetAsync(M->chain_bar, 0, 4, c->stream));
    cudaError_t e = o.chain(env_l1, grid, tb, smem, c->stream, a, c->mp, ch);
    if (e != cudaSuccess) return fail(SLD_E_CUDA, "persistent chain launch: %s", cudaGetErrorString(e));
    if (n & 1) std::swap(x, y);
    done += n;
  }
  return SLD_OK;
}

static int spmv_checked(sld_mat* M, sld_vec* in, sld_vec* out, bool sync);

extern "C" int sld_spmv(sld_mat* M, sld_vec* in, sld_vec* out) { return spmv_checked(M, in, out, true); }

// the same product left in flight on the context stream (Horner loops that
// enqueue the next kernel without a host round trip)
extern "C" int sld_spmv_async(sld_mat* M, sld_vec* in, sld_vec* out) { return spmv_checked(M, in, out, false); }

static int spmv_checked(sld_mat* M, sld_vec* in, sld_vec* out, bool sync) {
  if (!M || !in || !out) return fail(SLD_E_ARG, "null argument");
  if (in->n != M->total_cols) return fail(SLD_E_ARG, "vector length %lld != %lld columns",
                                          (long long)in->n, (long long)M->total_cols);
  if (out->n < M->nrows) return fail(SLD_E_ARG, "output vector too short");
  if (in == out) return fail(SLD_E_ARG, "in and out must differ");
  if (in->ctx != M->ctx || out->ctx != M->ctx) return fail(SLD_E_ARG, "context mismatch");
  if (in->chains != M->chains || out->chains != M->chains)
    return fail(SLD_E_ARG, "vector chains (%d, %d) != matrix chains %d", in->chains, out->chains, M->chains);
  CU(cudaSetDevice(M->ctx->dev));
  launch_product(M, in->buf[in->cur], out->buf[out->cur], nullptr, 0, nullptr);
  CU(cudaGetLastError());
  if (sync) CU(cudaStreamSynchronize(M->ctx->stream));
  return SLD_OK;
}

// ---- Mksol's Horner step in one product (solver.py:522-536): bind the n <= 8
// y vectors once (canonical copies in the slot order of the passes), then
// each step is out = A in + sum_s coeffs[s] y_s with the combination in the
// last pass's epilogue.  One-chain pass layout only (not short rows, limb
// slicing or the die split): the caller combines separately otherwise.
extern "C" int sld_mat_mksol_bind(sld_mat* M, sld_vec* const* ys, int n) {
  if (!M || n < 0 || n > 8 || (n && !ys)) return fail(SLD_E_ARG, "bad Mksol binding (0..8 vectors)");
  sld_ctx* c = M->ctx;
  CU(cudaSetDevice(c->dev));
  if (M->mk_y) {
    cudaStreamSynchronize(c->stream);
    cudaFree(M->mk_y);
    M->mk_y = nullptr;
    M->mk_n = 0;
  }
  if (!n) return SLD_OK;
  if (c->L > 8 || M->chains != 1 || M->halves != 1 || M->sliced || M->short_rows)
    return fail(SLD_E_ARG, "fused Mksol step needs the one-chain pass layout and ell < 2^256");
  for (int s = 0; s < n; s++) {
    if (!ys[s] || ys[s]->ctx != c || ys[s]->chains != 1) return fail(SLD_E_ARG, "bad Mksol vector %d", s);
    if (ys[s]->n < M->nrows) return fail(SLD_E_ARG, "Mksol vector %d shorter than the matrix rows", s);
  }
  const size_t per = (size_t)M->nslots * c->SW;
  CU(cudaMalloc(&M->mk_y, std::max<size_t>(per * n * 4, 16)));
  for (int s = 0; s < n; s++) ops(c->L).mk_gather(ys[s]->buf[ys[s]->cur], M->slot_row, M->nslots, M->mk_y + per * s,
                                                  c->stream);
  M->mk_n = n;
  CU(cudaGetLastError());
  return SLD_OK;
}

// out = A in + sum_s coeffs[s] y_s mod ell (coeffs: mk_n x L canonical limbs).
// Asynchronous on the context stream.
extern "C" int sld_spmv_mksol(sld_mat* M, sld_vec* in, sld_vec* out, const uint32_t* coeffs) {
  if (!M || !in || !out || !coeffs) return fail(SLD_E_ARG, "null argument");
  if (!M->mk_n) return fail(SLD_E_ARG, "no Mksol vectors bound");
  if (in->n != M->total_cols || out->n < M->nrows || in == out || in->ctx != M->ctx || out->ctx != M->ctx ||
      in->chains != 1 || out->chains != 1)
    return fail(SLD_E_ARG, "bad Mksol step vectors");
  CU(cudaSetDevice(M->ctx->dev));
  launch_product(M, in->buf[in->cur], out->buf[out->cur], nullptr, 0, nullptr, coeffs);
  CU(cudaGetLastError());
  return SLD_OK;
}

// Mksol Horner step with the combination precomputed (sld_lcset_apply_batch
// on a slot-ordered set): out = A in + addv mod ell, addv in the matrix's
// slot order (read coalesced by the last pass's epilogue).  One
// chain, L <= 8, pass or short-row layouts (not limb-sliced, not die-split).
extern "C" int sld_spmv_add(sld_mat* M, sld_vec* in, sld_vec* out, sld_vec* addv) {
  if (!M || !in || !out || !addv) return fail(SLD_E_ARG, "null argument");
  sld_ctx* c = M->ctx;
  if (c->L > 8 || M->chains != 1 || M->halves != 1 || M->sliced || M->npeer)
    return fail(SLD_E_ARG, "the fused addition needs one chain, ell < 2^256 and a pass layout");
  if (in->n != M->total_cols || out->n < M->nrows || addv->n < M->nslots || in == out || addv == out)
    return fail(SLD_E_ARG, "vector shapes do not match the matrix");
  if (addv->ctx != c || in->ctx != c || out->ctx != c) return fail(SLD_E_ARG, "context mismatch");
  CU(cudaSetDevice(c->dev));
  TRY(vec_alloc_buf(out, out->cur));
  launch_product(M, in->buf[in->cur], out->buf[out->cur], nullptr, 0, nullptr, nullptr, addv->buf[addv->cur]);
  CU(cudaGetLastError());
  return SLD_OK;
}

extern "C" int sld_spmv_planes(sld_mat* M, const uint64_t* in_planes, uint64_t* out_planes, int P) {
  if (!M) return fail(SLD_E_ARG, "null matrix");
  sld_ctx* c = M->ctx;
  TRY(check_P(c, P));
  CU(cudaSetDevice(c->dev));
  if (!M->tmp_in) TRY(sld_vec_create_chains(c, M->total_cols, M->chains, &M->tmp_in));
  if (!M->tmp_out) TRY(sld_vec_create_chains(c, M->nrows, M->chains, &M->tmp_out));
  TRY(upload_rows(M->tmp_in, in_planes, nullptr, M->total_cols, P));
  launch_product(M, M->tmp_in->buf[0], M->tmp_out->buf[0], nullptr, 0, nullptr);
  CU(cudaGetLastError());
  TRY(download_rows(M->tmp_out, out_planes, nullptr, M->nrows, P));
  return SLD_OK;
}

// ------------------------------------------------------------- Krylov

static int ensure_proj(sld_mat* M, const int64_t* x_rows, int m, int64_t chunk) {
  sld_ctx* c = M->ctx;
  if (m * M->chains > 256) return fail(SLD_E_ARG, "at most 256 projected residues per product");
  for (int t = 0; t < m; t++)
    if (x_rows[t] < 0 || x_rows[t] >= M->total_cols) return fail(SLD_E_ARG, "projection row out of range");
  if (M->proj_cap < m) {
    if (M->proj_rows) cudaFree(M->proj_rows);
    M->proj_rows = nullptr;
    CU(cudaMalloc(&M->proj_rows, std::max(m, 1) * 8));
    M->proj_cap = m;
  }
  if (m) CU(cudaMemcpyAsync(M->proj_rows, x_rows, m * 8, cudaMemcpyHostToDevice, c->stream));
  const size_t need = (size_t)std::max<int64_t>(chunk, 1) * std::max(m, 1) * M->chains * c->SW;
  if (M->terms_cap < need) {
    if (M->terms_dev) cudaFree(M->terms_dev);
    M->terms_dev = nullptr;
    CU(cudaMalloc(&M->terms_dev, need * 4));
    M->terms_cap = need;
  }
  return SLD_OK;
}

// copy `steps` terms from device ([step][t][chain], SW stride, at `src`) into
// host limbs laid out [step][chain][t][L]
static int drain_terms(sld_mat* M, const uint32_t* src, int m, int64_t steps, uint32_t* host,
                       std::vector<uint32_t>& tmp) {
  sld_ctx* c = M->ctx;
  const int G = M->chains;
  const size_t words = (size_t)steps * m * G * c->SW;
  if (!words) {
    CU(cudaStreamSynchronize(c->stream));
    return SLD_OK;
  }
  tmp.resize(words);
  CU(cudaMemcpyAsync(tmp.data(), src, words * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  const int L = c->L, SW = c->SW;
  for (int64_t k = 0; k < steps; k++)
    for (int t = 0; t < m; t++)
      for (int g = 0; g < G; g++) {
        const uint32_t* a = &tmp[(((size_t)k * m + t) * G + g) * SW];
        uint32_t* b = host + (((size_t)k * G + g) * m + t) * L;
        for (int i = 0; i < L; i++) b[i] = a[i];
      }
  return SLD_OK;
}

static constexpr int64_t KRYLOV_CHUNK = 1024;  // steps between host drains of the terms
static constexpr int GRAPH_STEPS = 32;          // products captured in one CUDA graph (even)

extern "C" int sld_krylov_unit(sld_mat* M, sld_vec* v, const int64_t* x_rows, int m, int64_t steps,
                               uint32_t* terms) {
  if (!M || !v || steps < 0 || m < 0) return fail(SLD_E_ARG, "bad Krylov arguments");
  if (M->nrows != M->total_cols) return fail(SLD_E_ARG, "Krylov needs a square matrix");
  if (v->n != M->total_cols) return fail(SLD_E_ARG, "iterate length mismatch");
  if (v->ctx != M->ctx) return fail(SLD_E_ARG, "context mismatch");
  if (v->chains != M->chains) return fail(SLD_E_ARG, "vector chains != matrix chains");
  if (m && (!x_rows || !terms)) return fail(SLD_E_ARG, "null projection arrays");
  sld_ctx* c = M->ctx;
  CU(cudaSetDevice(c->dev));
  TRY(vec_alloc_buf(v, v->cur ^ 1));
  // terms_dev: [0, GRAPH_STEPS) graph scratch, then the chunk accumulation area
  TRY(ensure_proj(M, x_rows, m, GRAPH_STEPS + KRYLOV_CHUNK));
  const size_t tstride = (size_t)m * M->chains * c->SW;  // words per step
  uint32_t* scratch = M->terms_dev;
  uint32_t* area = M->terms_dev + (size_t)GRAPH_STEPS * tstride;
  std::vector<uint32_t> tmp;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // graphs starting from buffer 0 / 1
  auto capture = [&](int start) -> int {
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int cur = start;
    for (int k = 0; k < GRAPH_STEPS; k++) {
      launch_product(M, v->buf[cur], v->buf[cur ^ 1], M->proj_rows, m, scratch + k * tstride);
      cur ^= 1;
    }
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (e != cudaSuccess) return fail(SLD_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
    CU(cudaGraphInstantiate(&exec[start], g, 0));
    CU(cudaGraphDestroy(g));
    return SLD_OK;
  };
  int rc = SLD_OK;
  int64_t done = 0;
  if (chain_eligible(M)) {
    // small matrix: every chunk is one persistent launch
    while (done < steps && rc == SLD_OK) {
      const int64_t chunk = std::min<int64_t>(KRYLOV_CHUNK, steps - done);
      rc = launch_chain(M, v->buf[v->cur], v->buf[v->cur ^ 1], chunk, M->proj_rows, m, m ? area : nullptr,
                        (int64_t)tstride);
      if (rc) break;
      v->cur ^= (int)(chunk & 1);
      rc = drain_terms(M, area, m, chunk, m ? terms + (size_t)done * m * M->chains * c->L : nullptr, tmp);
      done += chunk;
    }
    return rc;
  }
  while (done < steps && rc == SLD_OK) {
    const int64_t chunk = std::min<int64_t>(KRYLOV_CHUNK, steps - done);
    int64_t k = 0;
    while (k + GRAPH_STEPS <= chunk) {
      if (!exec[v->cur] && (rc = capture(v->cur)) != SLD_OK) break;
      cudaError_t e = cudaGraphLaunch(exec[v->cur], c->stream);
      if (e == cudaSuccess && m)
        e = cudaMemcpyAsync(area + k * tstride, scratch, GRAPH_STEPS * tstride * 4,
                            cudaMemcpyDeviceToDevice, c->stream);
      if (e != cudaSuccess) { rc = fail(SLD_E_CUDA, "graph replay: %s", cudaGetErrorString(e)); break; }
      k += GRAPH_STEPS;  // GRAPH_STEPS is even: the iterate is back in the same buffer
    }
    if (rc) break;
    for (; k < chunk; k++) {
      launch_product(M, v->buf[v->cur], v->buf[v->cur ^ 1], M->proj_rows, m, area + k * tstride);
      v->cur ^= 1;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { rc = fail(SLD_E_CUDA, "launch: %s", cudaGetErrorString(e)); break; }
    rc = drain_terms(M, area, m, chunk, m ? terms + (size_t)done * m * M->chains * c->L : nullptr, tmp);
    done += chunk;
  }
  for (auto& x : exec)
    if (x) cudaGraphExecDestroy(x);
  return rc;
}

// ------------------------------------------------------------- dense X

extern "C" int sld_xblock_create(sld_ctx* ctx, const uint32_t* x_limbs, int m, int64_t n,
                                 sld_xblock** out) {
  if (!ctx || !out || m < 0 || n < 0 || (m && n && !x_limbs)) return fail(SLD_E_ARG, "bad x block");
  CU(cudaSetDevice(ctx->dev));
  auto xb = std::make_unique<sld_xblock>();
  xb->ctx = ctx;
  xb->ref.bind(ctx);
  xb->m = m;
  xb->n = n;
  const size_t cnt = (size_t)m * n;
  CU(cudaMalloc(&xb->x, std::max<size_t>(cnt * ctx->SW * 4, 16)));
  if (cnt) {
    uint32_t* d = nullptr;
    CU(cudaMalloc(&d, cnt * ctx->L * 4));
    CU(cudaMemcpyAsync(d, x_limbs, cnt * ctx->L * 4, cudaMemcpyHostToDevice, ctx->stream));
    ops(ctx->L).limbs_to_slots(d, (int64_t)cnt, xb->x, 0u, (int64_t)cnt, 1, ctx->stream);
    if (ctx->L > 8) ops(ctx->L).to_mont(xb->x, (int64_t)cnt, ctx->mp, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    if (e != cudaSuccess) return fail(SLD_E_CUDA, "x block upload: %s", cudaGetErrorString(e));
  }
  if (ctx->L <= 8) {
    // 2^(32k) mod ell, k = L .. TC_FOLD_TOP, for the final folds of the lazy
    // and the tensor-core dot products
    const int L = ctx->L;
    const int top = std::max(2 * L, TC_FOLD_TOP);
    std::vector<uint32_t> r(L, 0), tab((size_t)(top - L + 1) * L);
    r[0] = 1;
    for (int k = 0; k <= top; k++) {
      if (k >= L) std::copy(r.begin(), r.end(), tab.begin() + (size_t)(k - L) * L);
      for (int b = 0; b < 32; b++) hmod_double(r.data(), ctx->mp.ell, L);
    }
    CU(cudaMalloc(&xb->fold, tab.size() * 4));
    CU(h2d(xb->fold, tab.data(), tab.size() * 4, ctx->stream));
    // tensor-core path: m <= 16 terms (32 m byte rows <= 4 M tiles).
    // Measured at cfg3 (tools/bench_dense.py): from m = 4 on it beats the
    // lazy CUDA-core dot products (m = 16: +0.38 vs +0.73 ms per step); at
    // m = 2 the lazy path wins (+0.10 vs +0.18 ms).  SLD_DENSE_TC=1 forces it,
    // =0 disables it.
    int tc = m >= 4 ? 1 : 0;
    if (const char* e = getenv("SLD_DENSE_TC")) tc = atoi(e);
    if (tc && m >= 1 && m <= 16 && n > 0) {
      xb->MT = (32 * m + 127) / 128;
      xb->ktiles = (n + TC_BK - 1) / TC_BK;
      const int64_t max_kt = TC_MAX_K_PER_CTA / TC_BK;
      xb->nct = (int)std::max<int64_t>(ctx->sms, (xb->ktiles + max_kt - 1) / max_kt);
      // test hook: the fewest CTAs the accumulator bound allows, so each
      // CTA sums the maximum K (tests/test_krylov_gpu.py exactness at the cap)
      if (const char* e = getenv("SLD_TC_MAX_K")) if (atoi(e)) xb->nct = (int)((xb->ktiles + max_kt - 1) / max_kt);
      xb->kt_per_cta = (xb->ktiles + xb->nct - 1) / xb->nct;
      xb->nct = (int)((xb->ktiles + xb->kt_per_cta - 1) / xb->kt_per_cta);
      CU(cudaMalloc(&xb->A, (size_t)xb->ktiles * xb->MT * TC_MTILE_BYTES));
      CU(cudaMalloc(&xb->B, (size_t)xb->ktiles * TC_BTILE_BYTES));
      CU(cudaMalloc(&xb->partial, (size_t)xb->nct * xb->MT * 128 * TC_NQ * 4));
      ops(L).tc_tile_x(xb->x, m, n, xb->MT, xb->ktiles, xb->A, ctx->stream);
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(ctx->stream));
    }
  }
  *out = xb.release();
  return SLD_OK;
}

extern "C" int sld_xblock_destroy(sld_xblock* x) {
  if (!x) return SLD_OK;
  cudaSetDevice(x->ctx->dev);
  if (x->fold) cudaFree(x->fold);
  if (x->A) cudaFree(x->A);
  if (x->B) cudaFree(x->B);
  if (x->partial) cudaFree(x->partial);
  if (x->x) cudaFree(x->x);
  delete x;
  return SLD_OK;
}

extern "C" int sld_krylov_dense(sld_mat* M, sld_vec* v, sld_xblock* X, int64_t steps, uint32_t* terms) {
  if (!M || !v || !X || steps < 0) return fail(SLD_E_ARG, "bad Krylov arguments");
  if (M->nrows != M->total_cols) return fail(SLD_E_ARG, "Krylov needs a square matrix");
  if (v->n != M->total_cols || X->n != M->total_cols) return fail(SLD_E_ARG, "length mismatch");
  if (M->chains != 1 || v->chains != 1) return fail(SLD_E_ARG, "dense projection runs one chain per matrix");
  sld_ctx* c = M->ctx;
  CU(cudaSetDevice(c->dev));
  TRY(vec_alloc_buf(v, v->cur ^ 1));
  const int m = X->m;
  TRY(ensure_proj(M, nullptr, 0, KRYLOV_CHUNK));
  {
    const size_t need = (size_t)KRYLOV_CHUNK * std::max(m, 1) * c->SW;
    if (M->terms_cap < need) {
      if (M->terms_dev) cudaFree(M->terms_dev);
      M->terms_dev = nullptr;
      CU(cudaMalloc(&M->terms_dev, need * 4));
      M->terms_cap = need;
    }
  }
  DenseProjArgs da;
  if (dense_proj_prepare(M->ctx->sms, m, v->n, c->SW, &M->dproj_part, &M->dproj_cap, &da))
    return fail(SLD_E_CUDA, "dense projection scratch allocation failed");
  da.x = X->x;
  da.fold = X->fold;
  std::vector<uint32_t> tmp;
  int64_t done = 0;
  while (done < steps) {
    const int64_t chunk = std::min<int64_t>(KRYLOV_CHUNK, steps - done);
    for (int64_t k = 0; k < chunk; k++) {
      da.v = v->buf[v->cur];
      da.out = M->terms_dev + (size_t)k * m * c->SW;
      if (m && X->MT)
        ops(c->L).tc_project(da.v, v->n, m, X->MT, X->ktiles, X->A, X->B, X->partial, X->nct, X->kt_per_cta,
                             X->fold, c->mp, da.out, c->stream);
      else if (m)
        ops(c->L).dense_proj(da, c->mp, c->stream);
      launch_product(M, v->buf[v->cur], v->buf[v->cur ^ 1], nullptr, 0, nullptr);
      v->cur ^= 1;
    }
    CU(cudaGetLastError());
    TRY(drain_terms(M, M->terms_dev, m, chunk, m ? terms + (size_t)done * m * c->L : nullptr, tmp));
    done += chunk;
  }
  CU(cudaStreamSynchronize(c->stream));
  return SLD_OK;
}

// ------------------------------------------------------------- bench hook

// the bench hook on the persistent chain: one launch per sample of
// 2 * pairs_per_sample products (even: the iterate returns to its buffer)
static int bench_chain(sld_mat* M, sld_vec* v, int64_t steps, int warmup, int64_t pairs_per_sample,
                       double* sample_ms, double* total_ms, double* kernel_ms) {
  sld_ctx* c = M->ctx;
  uint32_t *x = v->buf[v->cur], *y = v->buf[v->cur ^ 1];
  TRY(launch_chain(M, x, y, 2 * std::max<int64_t>(1, (warmup + 1) / 2), nullptr, 0, nullptr, 0));
  CU(cudaStreamSynchronize(c->stream));
  const int64_t pairs = (steps + 1) / 2;
  if (sample_ms && pairs_per_sample < 1) return fail(SLD_E_ARG, "pairs_per_sample must be >= 1");
  const int64_t per = sample_ms ? pairs_per_sample : pairs;
  const int64_t nmarks = (pairs + per - 1) / per;
  std::vector<cudaEvent_t> marks((size_t)nmarks + 1);
  for (auto& e : marks) CU(cudaEventCreate(&e));
  CU(cudaEventRecord(marks[0], c->stream));
  for (int64_t k = 0, j = 1; k < pairs; j++) {
    const int64_t n = std::min(per, pairs - k);
    TRY(launch_chain(M, x, y, 2 * n, nullptr, 0, nullptr, 0));
    CU(cudaEventRecord(marks[(size_t)j], c->stream));
    k += n;
  }
  CU(cudaEventSynchronize(marks.back()));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, marks[0], marks.back()));
  for (int64_t m = 0; sample_ms && m < nmarks; m++) {
    float d = 0;
    CU(cudaEventElapsedTime(&d, marks[(size_t)m], marks[(size_t)m + 1]));
    sample_ms[m] = d;
  }
  for (auto& e : marks) cudaEventDestroy(e);
  *total_ms = ms;
  *kernel_ms = ms / (2.0 * pairs);
  return SLD_OK;
}

extern "C" int sld_bench_spmv(sld_mat* M, sld_vec* v, int64_t steps, int warmup, double* total_ms,
                              double* kernel_ms) {
  return sld_bench_spmv_samples(M, v, steps, warmup, 0, nullptr, total_ms, kernel_ms);
}

// as sld_bench_spmv; with sample_ms != null an event is recorded after every
// `pairs_per_sample` product pairs (between graph launches: the stream keeps
// running), and sample_ms[k] gets the duration of sample k
extern "C" int sld_bench_spmv_samples(sld_mat* M, sld_vec* v, int64_t steps, int warmup, int64_t pairs_per_sample,
                                      double* sample_ms, double* total_ms, double* kernel_ms) {
  if (!M || !v || steps < 1) return fail(SLD_E_ARG, "bad bench arguments");
  if (M->nrows != M->total_cols || v->n != M->total_cols) return fail(SLD_E_ARG, "square matrix needed");
  if (v->chains != M->chains) return fail(SLD_E_ARG, "vector chains != matrix chains");
  sld_ctx* c = M->ctx;
  CU(cudaSetDevice(c->dev));
  TRY(vec_alloc_buf(v, v->cur ^ 1));
  if (chain_eligible(M)) return bench_chain(M, v, steps, warmup, pairs_per_sample, sample_ms, total_ms, kernel_ms);
  // graphs of 2 and 32 products (an even count returns to the same buffer);
  // the long graph amortises launch latency for small matrices
  cudaGraphExec_t ge2 = nullptr, ge32 = nullptr;
  for (int reps : {1, 16}) {
    cudaGraph_t g;
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < reps; r++) {
      launch_product(M, v->buf[v->cur], v->buf[v->cur ^ 1], nullptr, 0, nullptr);
      launch_product(M, v->buf[v->cur ^ 1], v->buf[v->cur], nullptr, 0, nullptr);
    }
    CU(cudaStreamEndCapture(c->stream, &g));
    CU(cudaGraphInstantiate(reps == 1 ? &ge2 : &ge32, g, 0));
    CU(cudaGraphDestroy(g));
  }
  for (int w = 0; w < (warmup + 1) / 2; w++) CU(cudaGraphLaunch(ge2, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  const int64_t pairs = (steps + 1) / 2;
  std::vector<cudaEvent_t> marks;
  if (sample_ms) {
    if (pairs_per_sample < 1) return fail(SLD_E_ARG, "pairs_per_sample must be >= 1");
    marks.resize((size_t)((pairs + pairs_per_sample - 1) / pairs_per_sample));
    for (auto& e : marks) CU(cudaEventCreate(&e));
  }
  CU(cudaEventRecord(e0, c->stream));
  if (sample_ms) {
    for (int64_t k = 0, m = 0; k < pairs; m++) {
      const int64_t n = std::min(pairs_per_sample, pairs - k);
      for (int64_t j = 0; j < n / 16; j++) CU(cudaGraphLaunch(ge32, c->stream));
      for (int64_t j = 0; j < n % 16; j++) CU(cudaGraphLaunch(ge2, c->stream));
      CU(cudaEventRecord(marks[(size_t)m], c->stream));
      k += n;
    }
  } else {
    for (int64_t k = 0; k < pairs / 16; k++) CU(cudaGraphLaunch(ge32, c->stream));
    for (int64_t k = 0; k < pairs % 16; k++) CU(cudaGraphLaunch(ge2, c->stream));
  }
  CU(cudaEventRecord(e1, c->stream));
  CU(cudaEventSynchronize(e1));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  for (size_t m = 0; m < marks.size(); m++) {
    float d = 0;
    CU(cudaEventElapsedTime(&d, m ? marks[m - 1] : e0, marks[m]));
    sample_ms[m] = d;
  }
  for (auto& e : marks) cudaEventDestroy(e);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge2);
  cudaGraphExecDestroy(ge32);
  *total_ms = ms;
  *kernel_ms = ms / (2.0 * pairs);
  return SLD_OK;
}

// sld_grid.cu -- one Krylov chain over an r x c grid of GPUs, every
// exchange done by the nodes over peer memory (NVLink P2P / CUDA IPC), each
// iteration one replayed CUDA graph, no host synchronisation and no
// collective on the data path.  The B200 restatement of the reference's grid
// iteration (sldlag/gridmv.py:251-348, Grid._one_iteration / apply_once)
// and of its failure detection (gridmv.py:46-51: GridProtocolError on a
// stale iteration tag, GridTimeoutError on a message that never arrives).
//
// Node (i, j) = rank i*c + j holds block A_ij of the balanced, padded matrix
// (rows [i br, (i+1) br), local columns [j bc, (j+1) bc)) and the fragment
// u_j.  One iteration, captured once per ping-pong parity:
//   r x 1 : SpMV whose last pass stores every output row into every node's
//           next iterate (rows rank*br + row)            -> barrier
//   r x c : SpMV whose last pass stores the partial into slot j of the row
//           collector (i, i mod c)'s inbox               -> barrier
//           collector: add_mod of the c slots, one scatter kernel copying
//           each column-range overlap of the row piece into the next
//           fragment of every node of that column        -> barrier
// plus, when a projection is set, a kernel recording the unit-X rows of the
// input fragment (a_i = X^T v_i, solver.py:210) into a device term ring.
//
// Barrier (one thread): bump its epoch, publish it into every node's
// peer_epoch[rank], add 1 to every node's flag (system-scope), spin until
// its own flag reaches nodes * epoch.  Then every peer's published epoch
// must be this epoch or the next one (a peer may already have passed this
// barrier and arrived at the next); anything else is a stale or restarted
// node -> err = SLD_GRID_ERR_PROTOCOL.  No progress for `timeout` ns ->
// err = SLD_GRID_ERR_TIMEOUT.  Errors are sticky (later barriers return at
// once) and read by the host once per sld_grid_wait.
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "sld_internal.cuh"

namespace {

constexpr uint32_t BLOB_MAGIC = 0x444C4753u;  // "SGLD"
constexpr int MAXN = 8;

// control block at the start of every node's shared allocation (256 B)
struct GridCtl {
  uint32_t flag;             // arrivals (all nodes add 1 per barrier)
  uint32_t epoch;            // barriers this node has entered
  uint32_t err;              // 0 ok, 1 timeout, 2 protocol
  uint32_t err_peer;         // offending node (protocol) / waited-for count (timeout)
  uint32_t err_seen;         // the epoch that node had published
  uint32_t pad[3];
  uint32_t peer_epoch[MAXN];  // epoch published by node k at its last arrival
  uint32_t rest[64 - 16];
};
static_assert(sizeof(GridCtl) == 256, "control block is 256 bytes");

struct Blob {
  uint32_t magic, rank;
  int32_t device, nodes;
  int64_t pid;
  uint64_t ptr;      // this process's device pointer of the allocation
  uint64_t bytes;
  uint8_t ipc[64];   // cudaIpcMemHandle_t of the allocation
  uint8_t pad[SLD_GRID_BLOB - 104];
};
static_assert(sizeof(Blob) == SLD_GRID_BLOB, "blob size");

struct Layout {
  size_t frag_words, off_frag[2], off_inbox, off_piece, bytes;
};

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

Layout layout_of(int64_t br, int64_t bc, int c, int SW) {
  Layout l;
  l.frag_words = (size_t)(bc + 1) * SW;  // record bc: the zero residue (padding target)
  size_t off = sizeof(GridCtl);
  for (int p = 0; p < 2; p++) {
    l.off_frag[p] = off;
    off = align256(off + l.frag_words * 4);
  }
  l.off_inbox = off;
  if (c > 1) off = align256(off + (size_t)c * br * SW * 4);
  l.off_piece = off;
  if (c > 1) off = align256(off + (size_t)br * SW * 4);
  l.bytes = off;
  return l;
}

struct CtlPtrs {
  GridCtl* p[MAXN];
};

__global__ void grid_barrier_kernel(GridCtl* me, const CtlPtrs peers, int nodes, int rank, uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  if (me->err) return;  // sticky: the host reports it at the next wait
  const uint32_t e = ++me->epoch;
  __threadfence_system();  // this node's stores of the phase before the arrival
  for (int k = 0; k < nodes; k++) {
    volatile uint32_t* pe = &peers.p[k]->peer_epoch[rank];
    *pe = e;
  }
  __threadfence_system();
  for (int k = 0; k < nodes; k++) atomicAdd_system(&peers.p[k]->flag, 1u);
  const uint32_t target = e * (uint32_t)nodes;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t v = 0;
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&me->flag) : "memory");
    if ((int32_t)(v - target) >= 0) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      me->err_peer = v;
      me->err_seen = target;
      me->err = 1;
      __threadfence_system();
      return;
    }
    __nanosleep(256);
  }
  for (int k = 0; k < nodes; k++) {
    uint32_t pe;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(pe) : "l"(&me->peer_epoch[k]) : "memory");
    if (pe != e && pe != e + 1) {
      me->err_peer = (uint32_t)k;
      me->err_seen = pe;
      me->err = 2;
      break;
    }
  }
  __threadfence_system();
}

// unit-X rows of the input fragment into the term ring: terms[step][t] =
// slot rows[t] (raw biased words; the host unbiases), step = *counter++
__global__ void grid_terms_kernel(const uint32_t* __restrict__ x, const int64_t* __restrict__ rows, int m, int SW,
                                  uint32_t* terms, uint32_t* counter, int64_t cap) {
  const uint32_t step = *counter;
  __syncthreads();
  const int t = threadIdx.x / SW, w = threadIdx.x % SW;
  if (t < m && step < cap) {
    const int64_t r = rows[t];
    terms[((size_t)step * m + t) * SW + w] = r >= 0 ? x[(size_t)r * SW + w] : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) *counter = step + 1;
}

// the collector's scatter: up to 32 (dst, src, 16-byte units) segments
struct CopyList {
  uint4* dst[32];
  const uint4* src[32];
  int64_t n[32];
  int count;
};

__global__ void grid_scatter_kernel(const CopyList cl) {
  const int s = blockIdx.y;
  if (s >= cl.count) return;
  uint4* __restrict__ d = cl.dst[s];
  const uint4* __restrict__ src = cl.src[s];
  const int64_t n = cl.n[s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = src[i];
}

}  // namespace

struct sld_grid {
  sld_mat* M = nullptr;  // the node's block (not owned)
  sld_ctx* c = nullptr;
  int r = 1, cc = 1, rank = 0, i = 0, j = 0, nodes = 1;
  bool collector = false;
  int64_t n_padded = 0, br = 0, bc = 0;
  Layout lay{};
  uint8_t* mem = nullptr;  // the shared allocation
  GridCtl* ctl = nullptr;
  uint32_t* frag[2] = {nullptr, nullptr};
  // peers (this node included)
  bool connected = false;
  uint8_t* pmem[MAXN] = {nullptr};
  bool opened[MAXN] = {false};
  // projection
  int m = 0;
  int64_t cap = 0;
  int64_t* rows_dev = nullptr;  // local slot of each row, -1 if another node reports it
  std::vector<uint8_t> owned;
  uint32_t* terms = nullptr;
  uint32_t* counter = nullptr;
  int64_t recorded = 0;
  // graphs, one per ping-pong parity
  cudaGraphExec_t ge[2] = {nullptr, nullptr};
  uint64_t timeout_ns = 30ull * 1000000000ull;
  int cur = 0;
  int64_t iteration = 0;
};

namespace {

uint32_t* peer_frag(sld_grid* g, int k, int p) {
  return (uint32_t*)(g->pmem[k] + g->lay.off_frag[p]);
}
GridCtl* peer_ctl(sld_grid* g, int k) { return (GridCtl*)g->pmem[k]; }

void drop_graphs(sld_grid* g) {
  for (auto& e : g->ge)
    if (e) {
      cudaGraphExecDestroy(e);
      e = nullptr;
    }
}

void enqueue_barrier(sld_grid* g, cudaStream_t s) {
  CtlPtrs cp;
  for (int k = 0; k < MAXN; k++) cp.p[k] = k < g->nodes ? peer_ctl(g, k) : nullptr;
  grid_barrier_kernel<<<1, 32, 0, s>>>(g->ctl, cp, g->nodes, g->rank, g->timeout_ns);
}

// enqueue one iteration from parity p (capture target)
int enqueue_iteration(sld_grid* g, int p) {
  sld_ctx* c = g->c;
  sld_mat* M = g->M;
  const int SW = c->SW;
  const int q = p ^ 1;
  if (g->m) grid_terms_kernel<<<1, g->m * SW, 0, c->stream>>>(g->frag[p], g->rows_dev, g->m, SW, g->terms,
                                                              g->counter, g->cap);
  // the product, its last pass pushing into peer memory
  const int save_n = M->npeer;
  uint32_t* save_yp[8];
  std::memcpy(save_yp, M->yp, sizeof(save_yp));
  const int64_t save_off = M->peer_off;
  if (g->cc == 1) {
    M->npeer = g->nodes;
    for (int k = 0; k < 8; k++) M->yp[k] = k < g->nodes ? peer_frag(g, k, q) : nullptr;
    M->peer_off = (int64_t)g->rank * g->br;
  } else {
    const int coll = g->i * g->cc + g->i % g->cc;
    M->npeer = 1;
    M->yp[0] = (uint32_t*)(g->pmem[coll] + g->lay.off_inbox) + (size_t)g->j * g->br * SW;
    for (int k = 1; k < 8; k++) M->yp[k] = nullptr;
    M->peer_off = 0;
  }
  launch_product(M, g->frag[p], nullptr, nullptr, 0, nullptr);
  M->npeer = save_n;
  std::memcpy(M->yp, save_yp, sizeof(save_yp));
  M->peer_off = save_off;
  enqueue_barrier(g, c->stream);
  if (g->cc > 1) {
    if (g->collector) {
      AddModArgs a;
      std::memset(&a, 0, sizeof(a));
      uint32_t* inbox = (uint32_t*)(g->mem + g->lay.off_inbox);
      uint32_t* piece = (uint32_t*)(g->mem + g->lay.off_piece);
      for (int s = 0; s < g->cc; s++) a.src[s] = inbox + (size_t)s * g->br * SW;
      a.dst = piece;
      a.k = g->cc;
      a.n = g->br;
      ops(c->L).add_mod(a, c->mp, c->stream);
      CopyList cl;
      std::memset(&cl, 0, sizeof(cl));
      const int64_t rlo = (int64_t)g->i * g->br;
      for (int jj = 0; jj < g->cc; jj++) {
        const int64_t clo = (int64_t)jj * g->bc;
        const int64_t lo = std::max(rlo, clo), hi = std::min(rlo + g->br, clo + g->bc);
        if (lo >= hi) continue;
        for (int k = 0; k < g->r; k++) {
          if (cl.count == 32) return fail(SLD_E_ARG, "grid scatter: too many segments");
          cl.dst[cl.count] = (uint4*)(peer_frag(g, k * g->cc + jj, q) + (size_t)(lo - clo) * SW);
          cl.src[cl.count] = (const uint4*)(piece + (size_t)(lo - rlo) * SW);
          cl.n[cl.count] = (hi - lo) * SW / 4;
          cl.count++;
        }
      }
      if (cl.count) {
        int64_t mx = 0;
        for (int s = 0; s < cl.count; s++) mx = std::max(mx, cl.n[s]);
        const unsigned gx = (unsigned)std::min<int64_t>((mx + 255) / 256, 2 * (int64_t)c->sms);
        grid_scatter_kernel<<<dim3(std::max(1u, gx), cl.count), 256, 0, c->stream>>>(cl);
      }
    }
    enqueue_barrier(g, c->stream);
  }
  CU(cudaGetLastError());
  return SLD_OK;
}

int build_graphs(sld_grid* g) {
  if (g->ge[0] && g->ge[1]) return SLD_OK;
  drop_graphs(g);
  CU(cudaSetDevice(g->c->dev));
  for (int p = 0; p < 2; p++) {
    cudaGraph_t gr;
    CU(cudaStreamBeginCapture(g->c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_iteration(g, p);
    cudaError_t e = cudaStreamEndCapture(g->c->stream, &gr);
    if (rc != SLD_OK) {
      if (e == cudaSuccess) cudaGraphDestroy(gr);
      return rc;
    }
    CU(e);
    CU(cudaGraphInstantiate(&g->ge[p], gr, 0));
    CU(cudaGraphDestroy(gr));
  }
  return SLD_OK;
}

}  // namespace

extern "C" int sld_grid_create(sld_mat* M, int r, int c, int rank, int64_t n_padded, sld_grid** out) {
  if (!M || !out || r < 1 || c < 1 || r * c > MAXN || rank < 0 || rank >= r * c || n_padded < 0 ||
      n_padded % r || n_padded % c)
    return fail(SLD_E_ARG, "bad grid (r x c <= 8 nodes, n_padded divisible by r and c)");
  if (M->halves != 1 || M->sliced || M->chains != 1)
    return fail(SLD_E_ARG, "grid blocks run on the row-major one-chain layouts (<= 8 limbs, no die split)");
  auto* g = new sld_grid();
  g->M = M;
  g->c = M->ctx;
  g->r = r;
  g->cc = c;
  g->rank = rank;
  g->i = rank / c;
  g->j = rank % c;
  g->nodes = r * c;
  g->collector = g->j == g->i % c;
  g->n_padded = n_padded;
  g->br = n_padded / r;
  g->bc = n_padded / c;
  if (M->nrows != g->br || M->total_cols != g->bc) {
    delete g;
    return fail(SLD_E_ARG, "block shape %lld x %lld does not match the grid (%lld x %lld)", (long long)M->nrows,
                (long long)M->total_cols, (long long)(n_padded / r), (long long)(n_padded / c));
  }
  g->lay = layout_of(g->br, g->bc, c, g->c->SW);
  cudaError_t e = cudaSetDevice(g->c->dev);
  if (e == cudaSuccess) e = cudaMalloc(&g->mem, g->lay.bytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->mem, 0, g->lay.bytes, g->c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->c->stream);
  if (e != cudaSuccess) {
    if (g->mem) cudaFree(g->mem);
    delete g;
    return fail(SLD_E_CUDA, "grid allocation of %zu bytes failed: %s", g->lay.bytes, cudaGetErrorString(e));
  }
  g->ctl = (GridCtl*)g->mem;
  for (int p = 0; p < 2; p++) {
    g->frag[p] = (uint32_t*)(g->mem + g->lay.off_frag[p]);
    ops(g->c->L).zero_slot(g->frag[p] + (size_t)g->bc * g->c->SW, g->c->stream);
  }
  if (cudaStreamSynchronize(g->c->stream) != cudaSuccess) {
    cudaFree(g->mem);
    delete g;
    return fail(SLD_E_CUDA, "grid init failed");
  }
  *out = g;
  return SLD_OK;
}

extern "C" int sld_grid_blob(sld_grid* g, uint8_t* blob) {
  if (!g || !blob) return fail(SLD_E_ARG, "null argument");
  Blob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = BLOB_MAGIC;
  b.rank = (uint32_t)g->rank;
  b.device = g->c->dev;
  b.nodes = g->nodes;
  b.pid = (int64_t)getpid();
  b.ptr = (uint64_t)(uintptr_t)g->mem;
  b.bytes = g->lay.bytes;
  CU(cudaSetDevice(g->c->dev));
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, g->mem));
  std::memcpy(b.ipc, &h, 64);
  std::memcpy(blob, &b, sizeof(b));
  return SLD_OK;
}

extern "C" int sld_grid_connect(sld_grid* g, const uint8_t* blobs) {
  if (!g || !blobs) return fail(SLD_E_ARG, "null argument");
  if (g->connected) return fail(SLD_E_ARG, "grid already connected");
  CU(cudaSetDevice(g->c->dev));
  const int64_t me = (int64_t)getpid();
  for (int k = 0; k < g->nodes; k++) {
    Blob b;
    std::memcpy(&b, blobs + (size_t)k * SLD_GRID_BLOB, sizeof(b));
    if (b.magic != BLOB_MAGIC || (int)b.rank != k || b.nodes != g->nodes || b.bytes != g->lay.bytes)
      return fail(SLD_E_ARG, "grid blob %d does not belong to this grid (rank, size or layout differ)", k);
    if (k == g->rank) {
      g->pmem[k] = g->mem;
      continue;
    }
    if (b.pid == me) {
      // same process: the raw pointer, with peer access if on another device
      if (b.device != g->c->dev) {
        int ok = 0;
        CU(cudaDeviceCanAccessPeer(&ok, g->c->dev, b.device));
        if (!ok) return fail(SLD_E_CUDA, "device %d cannot access peer device %d", g->c->dev, b.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CU(e);
      }
      g->pmem[k] = (uint8_t*)(uintptr_t)b.ptr;
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, b.ipc, 64);
      void* p = nullptr;
      CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      g->pmem[k] = (uint8_t*)p;
      g->opened[k] = true;
    }
  }
  g->connected = true;
  drop_graphs(g);
  return SLD_OK;
}

extern "C" int sld_grid_set_timeout(sld_grid* g, double seconds) {
  if (!g || !(seconds > 0)) return fail(SLD_E_ARG, "timeout must be positive");
  g->timeout_ns = (uint64_t)(seconds * 1e9);
  drop_graphs(g);
  return SLD_OK;
}

extern "C" int sld_grid_set_projection(sld_grid* g, const int64_t* rows, int m, int64_t max_steps,
                                       uint8_t* owned) {
  if (!g || m < 0 || m > 32 || (m && (!rows || max_steps < 1)))
    return fail(SLD_E_ARG, "bad projection (m <= 32 rows, max_steps >= 1)");
  CU(cudaSetDevice(g->c->dev));
  if (g->rows_dev) cudaFree(g->rows_dev);
  if (g->terms) cudaFree(g->terms);
  if (g->counter) cudaFree(g->counter);
  g->rows_dev = nullptr;
  g->terms = nullptr;
  g->counter = nullptr;
  g->m = 0;
  g->owned.assign((size_t)m, 0);
  drop_graphs(g);
  if (!m) return SLD_OK;
  if (m * g->c->SW > 1024) return fail(SLD_E_ARG, "projection too wide");
  // row t is reported by the row-0 node whose fragment holds it
  std::vector<int64_t> loc((size_t)m, -1);
  for (int t = 0; t < m; t++) {
    if (rows[t] < 0 || rows[t] >= g->n_padded) return fail(SLD_E_ARG, "projection row out of range");
    if (g->i == 0 && rows[t] / g->bc == g->j) {
      loc[(size_t)t] = rows[t] - (int64_t)g->j * g->bc;
      g->owned[(size_t)t] = 1;
    }
  }
  if (owned) std::memcpy(owned, g->owned.data(), (size_t)m);
  CU(cudaMalloc(&g->rows_dev, (size_t)m * 8));
  CU(h2d(g->rows_dev, loc.data(), (size_t)m * 8, g->c->stream));
  CU(cudaMalloc(&g->terms, (size_t)max_steps * m * g->c->SW * 4));
  CU(cudaMalloc(&g->counter, 4));
  CU(cudaMemsetAsync(g->counter, 0, 4, g->c->stream));
  g->m = m;
  g->cap = max_steps;
  g->recorded = 0;
  return SLD_OK;
}

extern "C" int sld_grid_load(sld_grid* g, const uint32_t* limbs) {
  if (!g || !limbs) return fail(SLD_E_ARG, "null argument");
  sld_ctx* c = g->c;
  CU(cudaSetDevice(c->dev));
  const size_t bytes = (size_t)g->bc * c->L * 4;
  uint32_t* tmp = nullptr;
  CU(cudaMalloc(&tmp, std::max<size_t>(bytes, 4)));
  cudaError_t e = cudaMemcpyAsync(tmp, limbs, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    ops(c->L).limbs_to_slots(tmp, g->bc, g->frag[g->cur], 0x80000000u, g->bc, 1, c->stream);
    e = cudaStreamSynchronize(c->stream);
  }
  cudaFree(tmp);
  CU(e);
  return SLD_OK;
}

extern "C" int sld_grid_read(sld_grid* g, uint32_t* limbs) {
  if (!g || !limbs) return fail(SLD_E_ARG, "null argument");
  sld_ctx* c = g->c;
  CU(cudaSetDevice(c->dev));
  const size_t bytes = (size_t)g->bc * c->L * 4;
  uint32_t* tmp = nullptr;
  CU(cudaMalloc(&tmp, std::max<size_t>(bytes, 4)));
  ops(c->L).slots_to_limbs(g->frag[g->cur], g->bc, tmp, 0x80000000u, g->bc, 1, c->stream);
  cudaError_t e = cudaMemcpyAsync(limbs, tmp, bytes, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(tmp);
  CU(e);
  return SLD_OK;
}

extern "C" int sld_grid_launch(sld_grid* g, int64_t count) {
  if (!g || count < 0) return fail(SLD_E_ARG, "bad launch");
  if (!g->connected) return fail(SLD_E_ARG, "grid not connected (sld_grid_connect)");
  if (g->m && g->recorded + count > g->cap)
    return fail(SLD_E_ARG, "term ring full: %lld recorded + %lld > %lld (drain with sld_grid_terms)",
                (long long)g->recorded, (long long)count, (long long)g->cap);
  CU(cudaSetDevice(g->c->dev));
  TRY(build_graphs(g));
  for (int64_t k = 0; k < count; k++) {
    CU(cudaGraphLaunch(g->ge[g->cur], g->c->stream));
    g->cur ^= 1;
  }
  g->iteration += count;
  g->recorded += g->m ? count : 0;
  return SLD_OK;
}

extern "C" int sld_grid_wait(sld_grid* g) {
  if (!g) return fail(SLD_E_ARG, "null grid");
  CU(cudaSetDevice(g->c->dev));
  CU(cudaStreamSynchronize(g->c->stream));
  GridCtl h;
  CU(cudaMemcpy(&h, g->ctl, sizeof(h), cudaMemcpyDeviceToHost));
  if (h.err == 1)
    return fail(SLD_E_TIMEOUT, "grid node %d: barrier %u timed out (%u of %u arrivals): a node stopped", g->rank,
                h.epoch, h.err_peer, h.err_seen);
  if (h.err == 2)
    return fail(SLD_E_PROTOCOL, "grid node %d: node %u is at iteration %u, expected %u (stale or restarted node)",
                g->rank, h.err_peer, h.err_seen, h.epoch);
  return SLD_OK;
}

extern "C" int sld_grid_iterate(sld_grid* g, int64_t count) {
  TRY(sld_grid_launch(g, count));
  return sld_grid_wait(g);
}

extern "C" int sld_grid_terms(sld_grid* g, uint32_t* out, int64_t* steps) {
  if (!g || !steps) return fail(SLD_E_ARG, "null argument");
  *steps = 0;
  if (!g->m) return SLD_OK;
  sld_ctx* c = g->c;
  CU(cudaSetDevice(c->dev));
  CU(cudaStreamSynchronize(c->stream));
  uint32_t n = 0;
  CU(cudaMemcpy(&n, g->counter, 4, cudaMemcpyDeviceToHost));
  if ((int64_t)n != g->recorded) return fail(SLD_E_CUDA, "term ring count %u != %lld launched", n, (long long)g->recorded);
  if (n && out) {
    std::vector<uint32_t> raw((size_t)n * g->m * c->SW);
    CU(cudaMemcpy(raw.data(), g->terms, raw.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t s = 0; s < n; s++)
      for (int t = 0; t < g->m; t++)
        for (int w = 0; w < c->L; w++)
          out[(s * g->m + t) * c->L + w] =
              g->owned[(size_t)t] ? raw[(s * g->m + t) * c->SW + w] ^ 0x80000000u : 0u;
  }
  CU(cudaMemsetAsync(g->counter, 0, 4, c->stream));
  *steps = n;
  g->recorded = 0;
  return SLD_OK;
}

extern "C" int sld_grid_set_epoch(sld_grid* g, int64_t epoch) {
  if (!g || epoch < 0) return fail(SLD_E_ARG, "bad epoch");
  CU(cudaSetDevice(g->c->dev));
  CU(cudaStreamSynchronize(g->c->stream));
  // barriers per iteration: 1 on r x 1, 2 on r x c
  const uint32_t e = (uint32_t)(epoch * (g->cc == 1 ? 1 : 2));
  GridCtl h;
  std::memset(&h, 0, sizeof(h));
  h.epoch = e;
  h.flag = e * (uint32_t)g->nodes;
  for (int k = 0; k < MAXN; k++) h.peer_epoch[k] = e;
  CU(h2d(g->ctl, &h, sizeof(h), g->c->stream));
  g->iteration = epoch;
  return SLD_OK;
}

extern "C" int sld_grid_info(sld_grid* g, int64_t* info) {
  if (!g || !info) return fail(SLD_E_ARG, "null argument");
  info[0] = g->iteration;
  info[1] = g->nodes;
  info[2] = g->br;
  info[3] = g->bc;
  info[4] = g->collector ? 1 : 0;
  info[5] = (int64_t)g->lay.bytes;
  info[6] = g->cur;
  info[7] = g->M->npass + (g->m ? 1 : 0) + (g->cc == 1 ? 1 : (g->collector ? 4 : 2));  // kernels per iteration
  return SLD_OK;
}

extern "C" int sld_grid_destroy(sld_grid* g) {
  if (!g) return SLD_OK;
  cudaSetDevice(g->c->dev);
  cudaStreamSynchronize(g->c->stream);
  drop_graphs(g);
  for (int k = 0; k < MAXN; k++)
    if (g->opened[k]) cudaIpcCloseMemHandle(g->pmem[k]);
  if (g->rows_dev) cudaFree(g->rows_dev);
  if (g->terms) cudaFree(g->terms);
  if (g->counter) cudaFree(g->counter);
  if (g->mem) cudaFree(g->mem);
  delete g;
  return SLD_OK;
}

// Grid partition builder (host code, no device needed): one r x c block of
// the balanced, padded matrix B = P_r A P_c^T, the reference's
// balance.split / permuted_padded (sldlag/balance.py:201-242, 245-267).
//
// The reference (and the numpy restatement this replaces) lexsorts every
// entry of B by (block row, block col, local row, local col) -- ~125 s at
// cfg3's 360 M entries, once per node.  A node only needs its own block, and
// B's rows are A's rows renamed, so this is a counting sort keyed by local
// row instead: each of A's rows owns one local row of one block row, so the
// count and fill passes run one thread per row range with no atomics; the
// few out-of-CSR entries (dense-column nonzeros, the pinned +1 padding) are
// added serially after.  Each local row is then ordered by (local column,
// entry index): the lexsort's order, ties included.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

int sld_set_error(int code, const char* msg);  // sld_capi.cu

namespace {

constexpr int SLD_E_INVAL = -1;  // SLD_E_ARG

template <class F>
void parallel_rows(int64_t n, int threads, F f) {
  int nt = threads > 0 ? threads : (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const int64_t chunk = 1 << 14;
  if (nt <= 1 || n <= chunk) { f(0, n); return; }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < nt; t++)
    th.emplace_back([&] {
      for (;;) {
        int64_t lo = next.fetch_add(chunk);
        if (lo >= n) break;
        f(lo, std::min(n, lo + chunk));
      }
    });
  for (auto& x : th) x.join();
}

struct Split {
  int64_t nrows, n_pad, br, bc;
  const int64_t* row_ptr;
  const void* col_idx;
  int col_bytes;
  const int64_t *row_perm, *col_perm;
  int64_t n_extra;
  const int64_t *extra_r, *extra_c;
  int32_t bi, bj;
  int64_t col(int64_t k) const {
    return col_bytes == 4 ? (int64_t)((const int32_t*)col_idx)[k] : ((const int64_t*)col_idx)[k];
  }
};

}  // namespace

/* Pass 1 (src == NULL): rp[0..br] and the block's entry count as return
 * value.  Pass 2: src[] (entry index: k < nnz for A's CSR entries, nnz + e
 * for extra entry e) and lc[] (local column), rows ordered by (lc, src).
 * Negative return = error (sld_last_error). */
extern "C" int64_t sld_split_block(int64_t nrows, const int64_t* row_ptr, const void* col_idx, int col_bytes,
                                   const int64_t* row_perm, const int64_t* col_perm, int64_t n_extra,
                                   const int64_t* extra_r, const int64_t* extra_c, int64_t n_pad, int32_t r,
                                   int32_t c, int32_t bi, int32_t bj, int64_t* rp, int64_t* src, int32_t* lc,
                                   int32_t threads) {
  if (nrows < 0 || n_pad < nrows || r < 1 || c < 1 || n_pad % r || n_pad % c || bi < 0 || bi >= r || bj < 0 ||
      bj >= c || (col_bytes != 4 && col_bytes != 8) || n_extra < 0 || !rp || (nrows && (!row_ptr || !row_perm)) ||
      (n_extra && (!extra_r || !extra_c)) || (n_pad && !col_perm) || (src && !lc))
    return sld_set_error(SLD_E_INVAL, "sld_split_block: bad arguments");
  Split s{nrows, n_pad, n_pad / r, n_pad / c, row_ptr, col_idx, col_bytes, row_perm, col_perm,
          n_extra, extra_r, extra_c, bi, bj};
  if (s.bc > INT32_MAX) return sld_set_error(SLD_E_INVAL, "sld_split_block: block columns exceed int32");
  const int64_t nnz = nrows ? row_ptr[nrows] : 0;
  std::atomic<int> bad{0};
  auto pcol = [&](int64_t k) -> int64_t {  // permuted column of CSR entry k, -1 if invalid
    int64_t cj = s.col(k);
    if (cj < 0 || cj >= n_pad) return -1;
    int64_t pc = col_perm[cj];
    return (pc < 0 || pc >= n_pad) ? -1 : pc;
  };
  if (!src) {
    std::memset(rp, 0, sizeof(int64_t) * (s.br + 1));
    parallel_rows(nrows, threads, [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; i++) {
        int64_t pr = row_perm[i];
        if (pr < 0 || pr >= n_pad) { bad = 1; continue; }
        if (pr / s.br != bi) continue;
        int64_t cnt = 0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
          int64_t pc = pcol(k);
          if (pc < 0) { bad = 1; continue; }
          cnt += pc / s.bc == bj;
        }
        rp[pr % s.br + 1] = cnt;
      }
    });
    for (int64_t e = 0; e < n_extra; e++) {
      int64_t er = extra_r[e], ec = extra_c[e];
      if (er < 0 || er >= n_pad || ec < 0 || ec >= n_pad) { bad = 1; continue; }
      if (er / s.br == bi && ec / s.bc == bj) rp[er % s.br + 1]++;
    }
    if (bad) return sld_set_error(SLD_E_INVAL, "sld_split_block: row/column index or permutation out of range");
    for (int64_t i = 0; i < s.br; i++) rp[i + 1] += rp[i];
    return rp[s.br];
  }
  // pass 2: fill in entry order, then sort every local row by (lc, src)
  std::vector<int64_t> cur(rp, rp + s.br);
  parallel_rows(nrows, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      int64_t pr = row_perm[i];
      if (pr / s.br != bi) continue;
      int64_t l = pr % s.br, o = cur[l];
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; k++) {
        int64_t pc = pcol(k);
        if (pc / s.bc != bj) continue;
        if (o >= rp[l + 1]) { bad = 1; break; }  // row_perm not a permutation
        src[o] = k;
        lc[o++] = (int32_t)(pc % s.bc);
      }
      cur[l] = o;
    }
  });
  for (int64_t e = 0; e < n_extra; e++) {
    int64_t er = extra_r[e], ec = extra_c[e];
    if (er / s.br != bi || ec / s.bc != bj) continue;
    int64_t l = er % s.br;
    if (cur[l] >= rp[l + 1]) { bad = 1; break; }
    src[cur[l]] = nnz + e;
    lc[cur[l]++] = (int32_t)(ec % s.bc);
  }
  if (bad) return sld_set_error(SLD_E_INVAL, "sld_split_block: row permutation is not a permutation");
  parallel_rows(s.br, threads, [&](int64_t lo, int64_t hi) {
    std::vector<uint64_t> key;
    std::vector<int64_t> tmp;
    for (int64_t l = lo; l < hi; l++) {
      const int64_t a = rp[l], n = rp[l + 1] - a;
      bool sorted = true;
      for (int64_t t = 1; t < n && sorted; t++) sorted = lc[a + t - 1] <= lc[a + t];
      if (sorted) continue;  // src already ascending: equal lc keep entry order
      key.resize(n);
      tmp.resize(n);
      for (int64_t t = 0; t < n; t++) key[t] = ((uint64_t)(uint32_t)lc[a + t] << 32) | (uint64_t)t;
      std::sort(key.begin(), key.end());
      for (int64_t t = 0; t < n; t++) tmp[t] = src[a + (int64_t)(key[t] & 0xffffffffu)];
      for (int64_t t = 0; t < n; t++) {
        src[a + t] = tmp[t];
        lc[a + t] = (int32_t)(key[t] >> 32);
      }
    }
  });
  return rp[s.br];
}

// sld_corpus.cpp -- native synthetic-corpus generator (a fixture producer for
// the benchmark configurations; not on the timed path).
//
// Restates the statistical shape of the reference generator
// sldlag/corpus.py:104-139: row weight rint(N(gamma, 0.1 gamma)) clipped to
// [3, max(3, ncols/2)]; distinct columns per row drawn with probability
// proportional to (j+1)^-decay (power-law column density, dense on the left);
// +1 / -1 each with probability pm1/2; otherwise a "small" coefficient of
// magnitude uniform in [2, cmax) with a random sign.  The reference draws
// from one numpy PCG64 stream and needs ~5 minutes at N = 3.6M; this version
// seeds an independent splitmix64/xoshiro stream per row so rows are
// generated in parallel and deterministically for a given seed.  It matches
// the reference's distribution, not its bit stream (the planted kernel
// column is added by the Python side, see corpus.py in the package).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "sldb200.h"

namespace {

struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  Rng(uint64_t seed, uint64_t row, uint64_t stream) {
    uint64_t x = seed * 0xD1342543DE82EF95ull ^ (row + 1) * 0x9E3779B97F4A7C15ull ^ stream;
    for (auto& v : s) v = splitmix(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {  // xoshiro256**
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  double normal() {
    double u1 = uniform(), u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

template <typename F>
void par(int64_t n, int nthreads, F f) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (n < 8192 || nthreads == 1) {
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

}  // namespace

extern "C" int sld_corpus_rows(int64_t n, int64_t ncols, double gamma, uint64_t seed, int64_t* row_ptr) {
  if (n < 0 || ncols < 1 || !row_ptr || gamma < 1) return SLD_E_ARG;
  const int64_t hi = std::min<int64_t>(ncols, std::max<int64_t>(3, ncols / 2));
  const int64_t lo = std::min<int64_t>(3, hi);
  std::vector<int64_t> w(n);
  par(n, 0, [&](int64_t a, int64_t b) {
    for (int64_t r = a; r < b; r++) {
      Rng g(seed, (uint64_t)r, 0x1111);
      int64_t k = (int64_t)std::nearbyint(gamma + 0.1 * gamma * g.normal());
      w[r] = std::min(hi, std::max(lo, k));
    }
  });
  row_ptr[0] = 0;
  for (int64_t r = 0; r < n; r++) row_ptr[r + 1] = row_ptr[r] + w[r];
  return SLD_OK;
}

extern "C" int sld_corpus_fill(int64_t n, int64_t ncols, double decay, double pm1, int64_t cmax,
                               uint64_t seed, const int64_t* row_ptr, int32_t* col_idx, uint8_t* tags,
                               int64_t* small_vals, int nthreads) {
  if (n < 0 || ncols < 1 || ncols >= 0x7FFFFFFF || !row_ptr || cmax < 3) return SLD_E_ARG;
  const double e = 1.0 - decay;
  const double top = std::fabs(e) < 1e-12 ? std::log((double)ncols + 1.0)
                                          : std::pow((double)ncols + 1.0, e) - 1.0;
  auto draw = [&](Rng& g) -> int32_t {
    const double u = g.uniform();
    double x;
    if (std::fabs(e) < 1e-12) x = std::exp(u * top);
    else x = std::pow(1.0 + u * top, 1.0 / e);
    int64_t j = (int64_t)x - 1;
    if (j < 0) j = 0;
    if (j >= ncols) j = ncols - 1;
    return (int32_t)j;
  };
  par(n, nthreads, [&](int64_t a, int64_t b) {
    std::vector<int32_t> cols;
    for (int64_t r = a; r < b; r++) {
      Rng g(seed, (uint64_t)r, 0x2222);
      const int64_t w = row_ptr[r + 1] - row_ptr[r];
      cols.clear();
      for (int tries = 0; (int64_t)cols.size() < w && tries < 64; tries++) {
        while ((int64_t)cols.size() < w) cols.push_back(draw(g));
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      }
      if ((int64_t)cols.size() < w) {  // tiny ncols: complete with the smallest unused columns
        std::vector<char> used(ncols, 0);
        for (int32_t c : cols) used[c] = 1;
        for (int64_t c = 0; c < ncols && (int64_t)cols.size() < w; c++)
          if (!used[c]) cols.push_back((int32_t)c);
        std::sort(cols.begin(), cols.end());
      }
      const int64_t base = row_ptr[r];
      for (int64_t k = 0; k < w; k++) {
        col_idx[base + k] = cols[k];
        const double u = g.uniform();
        if (u < pm1 / 2) {
          tags[base + k] = 0;
          small_vals[base + k] = 1;
        } else if (u < pm1) {
          tags[base + k] = 1;
          small_vals[base + k] = -1;
        } else {
          tags[base + k] = 2;
          const uint64_t span = (uint64_t)(cmax - 2);
          const int64_t mag = 2 + (int64_t)(g.next() % span);
          small_vals[base + k] = (g.next() & 1) ? mag : -mag;
        }
      }
    }
  });
  return SLD_OK;
}

// sld_fileio.cpp -- native readers/writers of the reference's binary formats
// (host C++, part of libsldb200.so; no CUDA):
//   SLDM matrix   sldlag/spmatrix.py:14-22 (format), 358-436 (store/load)
//   SLDV vector   sldlag/spmatrix.py:24-25, 439-462
//   SLDQ terms    sldlag/checkpoint.py:11-14, 36-64
// The reference parses these one entry at a time in Python (~0.5 M nnz/s,
// SURVEY.md §7); here the matrix is parsed straight into the CSR arrays the
// GPU builder takes, and written with one thread per row range.  Loading
// re-classifies every coefficient to its smallest class exactly as
// load_matrix does (classify, spmatrix.py:48-66).  Writes are atomic (temp
// file in the same directory, fsync, rename; fileio.py:66-84).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sldb200.h"

extern "C" const char* sld_last_error(void);
int sld_set_error(int code, const char* msg);  // sld_capi.cu

namespace {

int ferr(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return sld_set_error(code, buf);
}

// ------------------------------------------------------------ mapped file
struct Mapped {
  const uint8_t* p = nullptr;
  size_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n) munmap((void*)p, n);
    if (fd >= 0) close(fd);
  }
  int open_(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return ferr(SLD_E_ARG, "%s: cannot open", path);
    struct stat st;
    if (fstat(fd, &st) != 0) return ferr(SLD_E_ARG, "%s: cannot stat", path);
    n = (size_t)st.st_size;
    if (n) {
      void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) return ferr(SLD_E_ARG, "%s: cannot map", path);
      madvise(m, n, MADV_SEQUENTIAL);
      p = (const uint8_t*)m;
    }
    return SLD_OK;
  }
};

// bounds-checked cursor (the reference's fileio.Reader)
struct Cur {
  const uint8_t* p;
  size_t n, pos = 0;
  const char* name;
  int take(size_t k, const uint8_t** out) {
    if (pos + k > n)
      return ferr(SLD_E_TRUNC, "%s: needed %zu bytes at offset %zu, file has %zu", name, k, pos, n);
    *out = p + pos;
    pos += k;
    return SLD_OK;
  }
  template <typename T>
  int get(T* v) {
    const uint8_t* q;
    int r = take(sizeof(T), &q);
    if (r) return r;
    memcpy(v, q, sizeof(T));
    return SLD_OK;
  }
  int magic(const char* m) {
    const uint8_t* q;
    int r = take(4, &q);
    if (r) return r;
    if (memcmp(q, m, 4) != 0) return ferr(SLD_E_MAGIC, "%s: magic %.4s, expected %s", name, (const char*)q, m);
    return SLD_OK;
  }
  int done() {
    if (pos != n) return ferr(SLD_E_FORMAT, "%s: %zu trailing bytes", name, n - pos);
    return SLD_OK;
  }
};
#define TRYF(x) do { int _r = (x); if (_r != SLD_OK) return _r; } while (0)

// ell header: u16 byte width, ell big-endian
struct Ell {
  int hb = 0;  // bytes of the modulus field in the header
  int eb = 0;  // residue width: the modulus's minimal byte width (PrimeModulus.byte_width)
  int L = 0;
  std::vector<uint32_t> w;  // little-endian limbs
};

int read_ell(Cur& c, Ell* e, uint8_t* ell_be, int cap) {
  uint16_t hb;
  TRYF(c.get(&hb));
  const uint8_t* q;
  TRYF(c.take(hb, &q));
  if (hb == 0) return ferr(SLD_E_FORMAT, "%s: empty modulus field", c.name);
  if (ell_be) {
    if (cap < hb) return ferr(SLD_E_FORMAT, "%s: modulus field of %d bytes exceeds %d", c.name, hb, cap);
    memcpy(ell_be, q, hb);
  }
  e->hb = hb;
  e->L = (hb + 3) / 4;
  e->w.assign(e->L + 1, 0);
  for (int i = 0; i < hb; i++) e->w[i / 4] |= (uint32_t)q[hb - 1 - i] << (8 * (i % 4));
  while (e->L > 1 && e->w[e->L - 1] == 0) e->L--;
  // residues are written at the modulus's own byte width, whatever zero
  // padding the header field carries (spmatrix.py:345-352, modring.py:112-130)
  int bits = 0;
  for (int i = e->L - 1; i >= 0; i--)
    if (e->w[i]) {
      bits = 32 * i + 32 - __builtin_clz(e->w[i]);
      break;
    }
  if (bits < 2 || bits > 1024) return ferr(SLD_E_FORMAT, "%s: modulus of %d bits out of range", c.name, bits);
  e->eb = (bits + 7) / 8;
  return SLD_OK;
}

void write_ell(std::vector<uint8_t>& out, const uint32_t* ell, int L, int eb) {
  out.push_back((uint8_t)(eb & 0xff));
  out.push_back((uint8_t)(eb >> 8));
  for (int i = eb - 1; i >= 0; i--) out.push_back(i / 4 < L ? (uint8_t)(ell[i / 4] >> (8 * (i % 4))) : 0);
}

int byte_width(const uint32_t* ell, int L) {
  int bits = 0;
  for (int i = L - 1; i >= 0; i--)
    if (ell[i]) {
      bits = 32 * i + 32 - __builtin_clz(ell[i]);
      break;
    }
  return (bits + 7) / 8;
}

// multi-limb helpers over L words
int cmp(const uint32_t* a, const uint32_t* b, int L) {
  for (int i = L - 1; i >= 0; i--)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
bool is_small_u(const uint32_t* a, int L, uint64_t lim) {  // a <= lim (lim < 2^32)
  for (int i = 1; i < L; i++)
    if (a[i]) return false;
  return a[0] <= lim;
}
void sub(const uint32_t* a, const uint32_t* b, uint32_t* r, int L) {  // r = a - b, a >= b
  int64_t br = 0;
  for (int i = 0; i < L; i++) {
    int64_t v = (int64_t)a[i] - b[i] + br;
    r[i] = (uint32_t)v;
    br = v >> 32;
  }
}

constexpr uint64_t C_MAX = 0x7FFFFFFFull;  // spmatrix.py:45

// classify a canonical non-zero value v (L limbs): spmatrix.py:48-66
// -> tag, small word (+-1 for the unit tags)
void classify(const uint32_t* v, const Ell& e, uint8_t* tag, int64_t* small) {
  const int L = e.L;
  std::vector<uint32_t> t(L), one(L, 0);
  one[0] = 1;
  if (cmp(v, one.data(), L) == 0) {
    *tag = 0;
    *small = 1;
    return;
  }
  sub(e.w.data(), one.data(), t.data(), L);  // ell - 1
  if (cmp(v, t.data(), L) == 0) {
    *tag = 1;
    *small = -1;
    return;
  }
  // least-magnitude representative: v if v <= ell - v, else v - ell
  sub(e.w.data(), v, t.data(), L);  // ell - v
  if (cmp(v, t.data(), L) <= 0) {
    if (is_small_u(v, L, C_MAX)) {
      *tag = 2;
      *small = (int64_t)v[0];
      return;
    }
  } else if (is_small_u(t.data(), L, C_MAX)) {
    *tag = 2;
    *small = -(int64_t)t[0];
    return;
  }
  *tag = 3;
  *small = 0;
}

// residue of an i32 payload: v = x mod ell (Python %), L limbs
bool i32_residue(int32_t x, const Ell& e, uint32_t* v) {
  const int L = e.L;
  std::fill(v, v + L, 0u);
  const uint64_t mag = x < 0 ? (uint64_t)(-(int64_t)x) : (uint64_t)x;
  // mag mod ell
  uint64_t m;
  bool big = false;
  for (int i = 2; i < L; i++) big |= e.w[i] != 0;
  if (L >= 2 && (big || e.w[1] != 0)) {
    // ell >= 2^32 > mag
    m = mag;
    if (L == 2 && !big) {
      const uint64_t ell = ((uint64_t)e.w[1] << 32) | e.w[0];
      m = mag % ell;
    }
  } else {
    m = mag % (uint64_t)e.w[0];
  }
  if (m == 0) return false;
  uint32_t mv[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
  if (x >= 0) {
    for (int i = 0; i < L && i < 2; i++) v[i] = mv[i];
  } else {
    std::vector<uint32_t> mm(L, 0);
    for (int i = 0; i < L && i < 2; i++) mm[i] = mv[i];
    sub(e.w.data(), mm.data(), v, L);
  }
  return true;
}

void le_to_limbs(const uint8_t* q, int eb, uint32_t* v, int L) {
  std::fill(v, v + L, 0u);
  for (int i = 0; i < eb; i++)
    if (i / 4 < L) v[i / 4] |= (uint32_t)q[i] << (8 * (i % 4));
}
bool le_fits(const uint8_t* q, int eb, int L) {  // no bytes beyond L limbs
  for (int i = 4 * L; i < eb; i++)
    if (q[i]) return false;
  return true;
}

int atomic_write_file(const char* path, const uint8_t* data, size_t n) {
  std::string p(path), dir = ".", base = p;
  const size_t slash = p.rfind('/');
  if (slash != std::string::npos) {
    dir = slash ? p.substr(0, slash) : "/";
    base = p.substr(slash + 1);
  }
  std::string tmpl = dir + "/.tmp-XXXXXX" + base;
  std::vector<char> t(tmpl.begin(), tmpl.end());
  t.push_back(0);
  const int fd = mkstemps(t.data(), (int)base.size());
  if (fd < 0) return ferr(SLD_E_ARG, "%s: cannot create a temporary file", path);
  size_t off = 0;
  while (off < n) {
    const ssize_t w = ::write(fd, data + off, std::min<size_t>(n - off, 1 << 30));
    if (w <= 0) {
      close(fd);
      unlink(t.data());
      return ferr(SLD_E_ARG, "%s: write failed", path);
    }
    off += (size_t)w;
  }
  if (fsync(fd) != 0 || close(fd) != 0) {
    unlink(t.data());
    return ferr(SLD_E_ARG, "%s: fsync/close failed", path);
  }
  if (rename(t.data(), path) != 0) {
    unlink(t.data());
    return ferr(SLD_E_ARG, "%s: rename failed", path);
  }
  return SLD_OK;
}

template <typename F>
void par_rows(int64_t n, F f) {
  const int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536 || nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; t++) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

// ---------------------------------------------------------- SLDM parsing
struct SldmHead {
  int64_t nrows = 0, ncols = 0;
  Ell ell;
  std::vector<int64_t> dense_idx;
  size_t dense_pos = 0;  // offset of the dense column bytes
  size_t rows_pos = 0;   // offset of the first row record
};

int sldm_head(Cur& c, SldmHead* h, uint8_t* ell_be, int cap) {
  TRYF(c.magic("SLDM"));
  uint32_t ver;
  TRYF(c.get(&ver));
  if (ver != 1) return ferr(SLD_E_FORMAT, "unsupported SLDM version %u", ver);
  uint64_t nr, nc;
  TRYF(c.get(&nr));
  TRYF(c.get(&nc));
  h->nrows = (int64_t)nr;
  h->ncols = (int64_t)nc;
  TRYF(read_ell(c, &h->ell, ell_be, cap));
  uint32_t dc;
  TRYF(c.get(&dc));
  h->dense_idx.resize(dc);
  for (uint32_t g = 0; g < dc; g++) {
    uint64_t gi;
    TRYF(c.get(&gi));
    h->dense_idx[g] = (int64_t)gi;
  }
  h->dense_pos = c.pos;
  const uint8_t* q;
  TRYF(c.take((size_t)dc * (size_t)nr * h->ell.eb, &q));
  h->rows_pos = c.pos;
  return SLD_OK;
}

// one pass over the row records; with out == nullptr only counts
struct SldmOut {
  int64_t* row_ptr;
  int32_t* col_idx;
  uint8_t* tags;
  int64_t* small_vals;
  int64_t* full_pos;
  uint32_t* full_limbs;  // [n_full][L]
  int L;                 // limb stride of full_limbs
};

// Rows are variable-length records, so the parse runs in two steps:
//  1. a sequential skip-scan that only reads entry counts and tags (payload
//     sizes) to find where every row starts, stopping at a structural error
//     (truncation, unknown tag);
//  2. a parallel parse of the rows before that point, one thread per row
//     range; each thread keeps the first error of its range.
// The error reported is the first one in file order, as the reference's
// sequential loop would raise it.
struct RowScan {
  std::vector<uint64_t> off;  // byte offset of each row record
  std::vector<int64_t> first; // first entry index of each row (nrows + 1)
  int64_t good_rows = 0;      // rows before the structural error (all if none)
  int err = SLD_OK;           // structural error after good_rows
  std::string msg;
  size_t end = 0;             // offset after the last row (no error)
};

int sldm_scan(Cur& c, const SldmHead& h, RowScan* rs) {
  const int eb = h.ell.eb;
  rs->off.assign(h.nrows + 1, 0);
  rs->first.assign(h.nrows + 1, 0);
  const uint8_t* p = c.p;
  size_t pos = c.pos;
  const size_t n = c.n;
  int64_t nnz = 0;
  for (int64_t r = 0; r < h.nrows; r++) {
    rs->off[r] = pos;
    rs->first[r] = nnz;
    if (pos + 4 > n) {
      rs->good_rows = r;
      rs->err = ferr(SLD_E_TRUNC, "%s: needed 4 bytes at offset %zu, file has %zu", c.name, pos, n);
      rs->msg = sld_last_error();
      return SLD_OK;
    }
    uint32_t count;
    memcpy(&count, p + pos, 4);
    pos += 4;
    for (uint32_t k = 0; k < count; k++) {
      if (pos + 9 > n) {
        rs->good_rows = r;
        rs->err = ferr(SLD_E_TRUNC, "%s: needed 9 bytes at offset %zu, file has %zu", c.name, pos, n);
        rs->msg = sld_last_error();
        return SLD_OK;
      }
      const uint8_t tag = p[pos + 8];
      pos += 9;
      size_t pay = tag == 2 ? 4 : tag == 3 ? (size_t)eb : 0;
      if (tag > 3) {
        rs->good_rows = r;
        rs->err = ferr(SLD_E_FORMAT, "unknown entry tag %u", tag);
        rs->msg = sld_last_error();
        return SLD_OK;
      }
      if (pos + pay > n) {
        rs->good_rows = r;
        rs->err = ferr(SLD_E_TRUNC, "%s: needed %zu bytes at offset %zu, file has %zu", c.name, pay, pos, n);
        rs->msg = sld_last_error();
        return SLD_OK;
      }
      pos += pay;
    }
    nnz += count;
  }
  rs->off[h.nrows] = pos;
  rs->first[h.nrows] = nnz;
  rs->good_rows = h.nrows;
  rs->end = pos;
  return SLD_OK;
}

struct RangeOut {
  int err = SLD_OK;
  int64_t err_row = -1;
  std::string msg;
  std::vector<int64_t> fpos;
  std::vector<uint32_t> flimbs;
};

// parse rows [lo, hi); entries of a bad row before the error are written
void parse_range(const uint8_t* base, const SldmHead& h, const RowScan& rs, int64_t lo, int64_t hi,
                 const SldmOut* out, RangeOut* ro) {
  const Ell& e = h.ell;
  const int eb = e.eb, L = e.L;
  std::vector<uint32_t> v(L + 1);
  auto bad = [&](int64_t r, int code, const char* m) {
    ro->err = code;
    ro->err_row = r;
    ro->msg = m;
  };
  for (int64_t r = lo; r < hi; r++) {
    const uint8_t* q = base + rs.off[r];
    uint32_t count;
    memcpy(&count, q, 4);
    q += 4;
    int64_t pidx = rs.first[r];
    uint64_t prev = 0;
    for (uint32_t k = 0; k < count; k++, pidx++) {
      uint64_t delta;
      memcpy(&delta, q, 8);
      const uint8_t tag = q[8];
      q += 9;
      const uint64_t col = prev + delta;
      if (k > 0 && delta == 0) return bad(r, SLD_E_ARG, "column indices not strictly increasing within a row");
      prev = col;
      uint8_t t2;
      int64_t word;
      if (tag == 2) {
        int32_t x;
        memcpy(&x, q, 4);
        q += 4;
        if (!i32_residue(x, e, v.data())) return bad(r, SLD_E_ARG, "zero coefficient in file");
        classify(v.data(), e, &t2, &word);
      } else if (tag == 3) {
        le_to_limbs(q, eb, v.data(), L);
        const bool fits = le_fits(q, eb, L);
        q += eb;
        if (!fits) return bad(r, SLD_E_ARG, "full coefficient is not a canonical residue");
        // the reference classifies v mod ell but keeps v itself as the full
        // value, which must then be canonical (spmatrix.py:419-432)
        bool canonical = true;
        while (cmp(v.data(), e.w.data(), L) >= 0) {  // < 2^8 rounds: v < 2^(8 eb)
          sub(v.data(), e.w.data(), v.data(), L);
          canonical = false;
        }
        bool nz = false;
        for (int i = 0; i < L; i++) nz |= v[i] != 0;
        if (!nz) return bad(r, SLD_E_ARG, "zero coefficient in file");
        classify(v.data(), e, &t2, &word);
        if (t2 == 3 && !canonical) return bad(r, SLD_E_ARG, "full coefficient is not a canonical residue");
      } else if (tag == 0) {
        t2 = 0;
        word = 1;
      } else {
        // tag 1 (the scan rejected tags > 3): ell - 1 re-classifies to -1
        t2 = 1;
        word = -1;
      }
      if (col >= (uint64_t)h.ncols) return bad(r, SLD_E_ARG, "sparse column index out of range");
      if (out) {
        out->col_idx[pidx] = (int32_t)col;
        out->tags[pidx] = t2;
        out->small_vals[pidx] = word;
      }
      if (t2 == 3) {
        ro->fpos.push_back(pidx);
        if (out) ro->flimbs.insert(ro->flimbs.end(), v.begin(), v.begin() + L);
      }
    }
  }
}

// scan + parallel parse; returns the first error in file order
int sldm_rows(Cur& c, const SldmHead& h, int64_t* nnz_out, int64_t* nfull_out, const SldmOut* out) {
  RowScan rs;
  TRYF(sldm_scan(c, h, &rs));
  const int64_t nr = rs.good_rows;
  const int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const int parts = nr < 4096 ? 1 : nt;
  std::vector<RangeOut> ro(parts);
  std::vector<std::thread> th;
  const int64_t chunk = (nr + parts - 1) / std::max(parts, 1);
  for (int t = 0; t < parts; t++) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(nr, lo + chunk);
    if (lo >= hi) break;
    if (parts == 1) parse_range(c.p, h, rs, lo, hi, out, &ro[t]);
    else th.emplace_back([&, lo, hi, t] { parse_range(c.p, h, rs, lo, hi, out, &ro[t]); });
  }
  for (auto& x : th) x.join();
  for (auto& r : ro)
    if (r.err != SLD_OK) return sld_set_error(r.err, r.msg.c_str());
  if (rs.err != SLD_OK) return sld_set_error(rs.err, rs.msg.c_str());
  int64_t nfull = 0;
  for (auto& r : ro) {
    if (out)
      for (size_t k = 0; k < r.fpos.size(); k++) {
        out->full_pos[nfull + (int64_t)k] = r.fpos[k];
        memcpy(out->full_limbs + (size_t)(nfull + (int64_t)k) * out->L, r.flimbs.data() + k * h.ell.L,
               sizeof(uint32_t) * std::min(h.ell.L, out->L));
      }
    nfull += (int64_t)r.fpos.size();
  }
  if (out)
    for (int64_t r = 0; r <= h.nrows; r++) out->row_ptr[r] = rs.first[r];
  c.pos = rs.end;
  *nnz_out = rs.first[h.nrows];
  *nfull_out = nfull;
  return SLD_OK;
}

}  // namespace

// --------------------------------------------------------------- C ABI

extern "C" int sld_sldm_info(const char* path, int header_only, int64_t* info, uint8_t* ell_be, int ell_cap) {
  if (!path || !info) return ferr(SLD_E_ARG, "null argument");
  Mapped m;
  TRYF(m.open_(path));
  Cur c{m.p, m.n, 0, path};
  SldmHead h;
  if (header_only) {
    // through the modulus only, so the caller can validate it before the
    // rest is parsed (the reference's order: spmatrix.py:403-406)
    TRYF(c.magic("SLDM"));
    uint32_t ver;
    TRYF(c.get(&ver));
    if (ver != 1) return ferr(SLD_E_FORMAT, "unsupported SLDM version %u", ver);
    uint64_t nr, nc;
    TRYF(c.get(&nr));
    TRYF(c.get(&nc));
    TRYF(read_ell(c, &h.ell, ell_be, ell_cap));
    memset(info, 0, 8 * sizeof(int64_t));
    info[0] = (int64_t)nr;
    info[1] = (int64_t)nc;
    info[2] = h.ell.hb;
    info[7] = h.ell.L;
    return SLD_OK;
  }
  TRYF(sldm_head(c, &h, ell_be, ell_cap));
  if (h.ncols >= 0x7FFFFFFF || h.nrows >= 0x7FFFFFFF)
    return ferr(SLD_E_ARG, "dimensions must be < 2^31 for the device layout");
  int64_t nnz, nf;
  TRYF(sldm_rows(c, h, &nnz, &nf, nullptr));
  TRYF(c.done());
  info[0] = h.nrows;
  info[1] = h.ncols;
  info[2] = h.ell.hb;
  info[3] = (int64_t)h.dense_idx.size();
  info[4] = nnz;
  info[5] = nf;
  info[6] = (int64_t)m.n;
  info[7] = h.ell.L;
  return SLD_OK;
}

extern "C" int sld_sldm_read(const char* path, int L, int64_t* row_ptr, int32_t* col_idx, uint8_t* tags,
                             int64_t* small_vals, int64_t* full_pos, uint32_t* full_limbs, int64_t* dense_idx,
                             uint32_t* dense_limbs) {
  if (!path || !row_ptr || L < 1) return ferr(SLD_E_ARG, "null argument");
  Mapped m;
  TRYF(m.open_(path));
  Cur c{m.p, m.n, 0, path};
  SldmHead h;
  TRYF(sldm_head(c, &h, nullptr, 0));
  if (L < h.ell.L) return ferr(SLD_E_ARG, "limb stride %d below the modulus width %d", L, h.ell.L);
  // dense columns: each nrows residues, canonical (vector_from_bytes + check)
  const int eb = h.ell.eb;
  for (size_t g = 0; g < h.dense_idx.size(); g++) {
    if (dense_idx) dense_idx[g] = h.dense_idx[g];
    std::atomic<int> bad{0};
    par_rows(h.nrows, [&](int64_t lo, int64_t hi) {
      for (int64_t r = lo; r < hi; r++) {
        const uint8_t* q = m.p + h.dense_pos + (g * (size_t)h.nrows + (size_t)r) * eb;
        uint32_t* dst = dense_limbs + (g * (size_t)h.nrows + (size_t)r) * L;
        if (!le_fits(q, eb, h.ell.L)) { bad = 1; return; }
        le_to_limbs(q, eb, dst, L);
        if (cmp(dst, h.ell.w.data(), h.ell.L) >= 0) { bad = 1; return; }
      }
    });
    if (bad) return ferr(SLD_E_ARG, "dense column value is not a canonical residue");
  }
  SldmOut out{row_ptr, col_idx, tags, small_vals, full_pos, full_limbs, L};
  int64_t nnz, nf;
  TRYF(sldm_rows(c, h, &nnz, &nf, &out));
  TRYF(c.done());
  return SLD_OK;
}

extern "C" int sld_sldm_write(const char* path, int64_t nrows, int64_t ncols, const uint32_t* ell, int L,
                              const int64_t* row_ptr, const int32_t* col_idx, const uint8_t* tags,
                              const int64_t* small_vals, int64_t n_full, const int64_t* full_pos,
                              const uint32_t* full_limbs, int n_dense, const int64_t* dense_idx,
                              const uint32_t* dense_limbs) {
  if (!path || !ell || L < 1 || nrows < 0 || ncols < 0 || (nrows && !row_ptr))
    return ferr(SLD_E_ARG, "bad SLDM write arguments");
  const int eb = byte_width(ell, L);
  const int64_t nnz = nrows ? row_ptr[nrows] : 0;
  // header
  std::vector<uint8_t> head;
  auto put = [&](const void* p, size_t k) {
    const uint8_t* b = (const uint8_t*)p;
    head.insert(head.end(), b, b + k);
  };
  put("SLDM", 4);
  const uint32_t ver = 1;
  put(&ver, 4);
  const uint64_t nr = (uint64_t)nrows, nc = (uint64_t)ncols;
  put(&nr, 8);
  put(&nc, 8);
  write_ell(head, ell, L, eb);
  const uint32_t dc = (uint32_t)n_dense;
  put(&dc, 4);
  for (int g = 0; g < n_dense; g++) {
    const uint64_t gi = (uint64_t)dense_idx[g];
    put(&gi, 8);
  }
  // full values by position (positions sorted)
  for (int64_t k = 0; k < n_full; k++)
    if (full_pos[k] < 0 || full_pos[k] >= nnz || (k && full_pos[k] <= full_pos[k - 1]))
      return ferr(SLD_E_ARG, "full positions must be sorted and in range");
  // per-row byte sizes, then one thread per row range fills its bytes
  std::vector<uint64_t> off(nrows + 1, 0);
  for (int64_t r = 0; r < nrows; r++) {
    uint64_t b = 4;
    for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) b += 9 + (tags[p] == 2 ? 4 : tags[p] == 3 ? eb : 0);
    off[r + 1] = off[r] + b;
  }
  const size_t dense_bytes = (size_t)n_dense * nrows * eb;
  const size_t total = head.size() + dense_bytes + off[nrows];
  std::vector<uint8_t> blob(total);
  memcpy(blob.data(), head.data(), head.size());
  uint8_t* dense_dst = blob.data() + head.size();
  par_rows((int64_t)n_dense * nrows, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++)
      for (int b = 0; b < eb; b++) dense_dst[i * eb + b] = (uint8_t)(dense_limbs[i * L + b / 4] >> (8 * (b % 4)));
  });
  uint8_t* rows_dst = dense_dst + dense_bytes;
  std::atomic<int> bad{0};
  par_rows(nrows, [&](int64_t lo, int64_t hi) {
    // first full entry at or after this range's first position
    int64_t fk = std::lower_bound(full_pos, full_pos + n_full, row_ptr[lo]) - full_pos;
    for (int64_t r = lo; r < hi; r++) {
      uint8_t* q = rows_dst + off[r];
      const uint32_t cnt = (uint32_t)(row_ptr[r + 1] - row_ptr[r]);
      memcpy(q, &cnt, 4);
      q += 4;
      int64_t prev = 0;
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) {
        const uint64_t delta = (uint64_t)((int64_t)col_idx[p] - prev);
        prev = col_idx[p];
        memcpy(q, &delta, 8);
        q[8] = tags[p];
        q += 9;
        if (tags[p] == 2) {
          const int64_t s = small_vals[p];
          if (s < INT32_MIN || s > INT32_MAX) { bad = 1; return; }
          const int32_t x = (int32_t)s;
          memcpy(q, &x, 4);
          q += 4;
        } else if (tags[p] == 3) {
          if (fk >= n_full || full_pos[fk] != p) { bad = 2; return; }
          const uint32_t* v = full_limbs + (size_t)fk * L;
          for (int b = 0; b < eb; b++) q[b] = (uint8_t)(v[b / 4] >> (8 * (b % 4)));
          q += eb;
          fk++;
        } else if (tags[p] > 3) {
          bad = 3;
          return;
        }
      }
    }
  });
  if (bad == 1) return ferr(SLD_E_ARG, "small coefficient outside the i32 payload");
  if (bad == 2) return ferr(SLD_E_ARG, "full-tag entry without a full value");
  if (bad == 3) return ferr(SLD_E_ARG, "unknown coefficient tag");
  return atomic_write_file(path, blob.data(), blob.size());
}

// SLDV (kind 0): magic, u32 1, ell header, u64 n, n residues.
// SLDQ (kind 1): magic, u32 1, ell header, u32 m, u32 1, u64 count, count*m residues.
extern "C" int sld_sldv_write(const char* path, int kind, const uint32_t* ell, int L, int64_t m, int64_t n,
                              const uint32_t* limbs, int stride) {
  if (!path || !ell || L < 1 || n < 0 || (n && !limbs) || stride < 1 || (kind == 1 && m < 0))
    return ferr(SLD_E_ARG, "bad vector write arguments");
  const int eb = byte_width(ell, L);
  std::vector<uint8_t> head;
  auto put = [&](const void* p, size_t k) {
    const uint8_t* b = (const uint8_t*)p;
    head.insert(head.end(), b, b + k);
  };
  put(kind == 1 ? "SLDQ" : "SLDV", 4);
  const uint32_t ver = 1;
  put(&ver, 4);
  write_ell(head, ell, L, eb);
  const int64_t count = kind == 1 ? n : n;
  if (kind == 1) {
    const uint32_t mm = (uint32_t)m, one = 1;
    put(&mm, 4);
    put(&one, 4);
  }
  const uint64_t cnt = (uint64_t)count;
  put(&cnt, 8);
  const int64_t nres = kind == 1 ? n * m : n;
  std::vector<uint8_t> blob(head.size() + (size_t)nres * eb);
  memcpy(blob.data(), head.data(), head.size());
  uint8_t* dst = blob.data() + head.size();
  par_rows(nres, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++)
      for (int b = 0; b < eb; b++)
        dst[i * eb + b] = b / 4 < stride ? (uint8_t)(limbs[i * stride + b / 4] >> (8 * (b % 4))) : 0;
  });
  return atomic_write_file(path, blob.data(), blob.size());
}

// info: [kind (0 SLDV / 1 SLDQ), ell bytes, L, m (1 for SLDV), count, residues]
extern "C" int sld_sldv_info(const char* path, int header_only, int64_t* info, uint8_t* ell_be, int ell_cap) {
  if (!path || !info) return ferr(SLD_E_ARG, "null argument");
  Mapped mp;
  TRYF(mp.open_(path));
  Cur c{mp.p, mp.n, 0, path};
  const uint8_t* q;
  TRYF(c.take(4, &q));
  int kind;
  if (!memcmp(q, "SLDV", 4)) kind = 0;
  else if (!memcmp(q, "SLDQ", 4)) kind = 1;
  else return ferr(SLD_E_MAGIC, "%s: magic %.4s, expected SLDV or SLDQ", path, (const char*)q);
  uint32_t ver;
  TRYF(c.get(&ver));
  if (ver != 1) return ferr(SLD_E_FORMAT, "unsupported %s version %u", kind ? "SLDQ" : "SLDV", ver);
  Ell e;
  TRYF(read_ell(c, &e, ell_be, ell_cap));
  if (header_only) {
    memset(info, 0, 6 * sizeof(int64_t));
    info[0] = kind;
    info[1] = e.hb;
    info[2] = e.L;
    return SLD_OK;
  }
  uint32_t m = 1, one = 1;
  if (kind == 1) {
    TRYF(c.get(&m));
    TRYF(c.get(&one));
  }
  uint64_t count;
  TRYF(c.get(&count));
  // count * m * width must fit what is left of the file (no wrap-around)
  const uint64_t left = (uint64_t)(c.n - c.pos);
  const uint64_t per = (uint64_t)m * (uint64_t)e.eb;
  if (per && count > left / per)
    return ferr(SLD_E_TRUNC, "%s: %llu x %u residues of %d bytes exceed the %llu bytes left", path,
                (unsigned long long)count, m, e.eb, (unsigned long long)left);
  const uint64_t nres = count * m;
  TRYF(c.take((size_t)nres * e.eb, &q));
  TRYF(c.done());
  info[0] = kind;
  info[1] = e.hb;
  info[2] = e.L;
  info[3] = m;
  info[4] = (int64_t)count;
  info[5] = (int64_t)nres;
  return SLD_OK;
}

extern "C" int sld_sldv_read(const char* path, uint32_t* limbs, int stride) {
  int64_t info[6];
  TRYF(sld_sldv_info(path, 0, info, nullptr, 0));
  Mapped mp;
  TRYF(mp.open_(path));
  Cur c{mp.p, mp.n, 0, path};
  const uint8_t* q;
  TRYF(c.take(8, &q));
  Ell e;
  TRYF(read_ell(c, &e, nullptr, 0));
  TRYF(c.take(info[0] == 1 ? 16 : 8, &q));
  if (stride < e.L) return ferr(SLD_E_ARG, "limb stride %d below the modulus width %d", stride, e.L);
  const int eb = e.eb;
  const uint8_t* base = mp.p + c.pos;
  std::atomic<int> bad{0};
  par_rows(info[5], [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      const uint8_t* s = base + (size_t)i * eb;
      uint32_t* d = limbs + (size_t)i * stride;
      if (!le_fits(s, eb, e.L)) { bad = 1; return; }
      le_to_limbs(s, eb, d, stride);
      if (cmp(d, e.w.data(), e.L) >= 0) { bad = 1; return; }
    }
  });
  if (bad) return ferr(SLD_E_ARG, "%s: value is not a canonical residue", path);
  return SLD_OK;
}

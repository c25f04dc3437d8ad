/*
 * TEST INFRASTRUCTURE -- the CPU oracle.  Never linked into, loaded by, or
 * called from the product package (paper_1402_3661_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * may use it, and only as the checker / the reference's CPU timing.
 *
 * A plain-C restatement of the reference's exact batched SpMV over Z/lZ,
 * /root/reference/pkg/src/sldlag/vecops.py:355-470 (SpmvKernel), with the
 * RNS sizing of modring.py:170-207 (RnsContext) and the CRT fold of
 * vecops.py:281-352 (RnsBatch) and the reduction of vecops.py:119-162
 * (ModReducer._smallq_loop / reduce_compact).  The structure follows the
 * reference step for step:
 *
 *   1. ctx1: k1 31-bit primes (largest first, below 2^31) with
 *      M1 > 2 * gamma1 * cmax1 * l, gamma1 = max row count of +-1/small
 *      entries, cmax1 = max |small| (vecops.py:386-392, modring.py:180-207);
 *      ctx2 the same for the full lane with c_max = l-1 (vecops.py:405-410).
 *   2. per row, per limb: +1 lane adds u mod m_i; -1 lane adds
 *      count*(l mod m_i) - sum(u mod m_i); small lane adds c*u mod m_i, with a
 *      negative c folded as |c|*(l-u) (vecops.py:434-451); acc %= m_i (452).
 *   3. CRT quotient t from the same biased float fractions, z = sum limb_i *
 *      (C_i mod l) + t*(-M mod l) (vecops.py:338-352); the full lane is
 *      folded the same way with ctx2 and added (455-469).
 *   4. z mod l by biased float quotient estimates + exact corrections
 *      (vecops.py:119-162).
 *
 * Residues cross this API as little-endian 32-bit limbs, L per residue.
 * Rows are independent, so rows are split across OpenMP threads.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXW 104 /* 32-bit words: covers M2 > 2*gamma*l^2 for l <= 1024 bits */
#define MAXK 80  /* RNS moduli per context */

/* ---------------- small multiprecision helpers (setup + per-row) -------- */

static int bn_len(const uint32_t *a, int n) {
    while (n > 0 && a[n - 1] == 0) n--;
    return n;
}
static int bn_bitlen(const uint32_t *a, int n) {
    n = bn_len(a, n);
    if (!n) return 0;
    return 32 * (n - 1) + (32 - __builtin_clz(a[n - 1]));
}
/* a[0..n) *= w, returns carry out */
static uint32_t bn_mul_u32(uint32_t *a, int n, uint32_t w) {
    uint64_t c = 0;
    for (int i = 0; i < n; i++) {
        c += (uint64_t)a[i] * w;
        a[i] = (uint32_t)c;
        c >>= 32;
    }
    return (uint32_t)c;
}
/* a /= w in place, returns remainder */
static uint32_t bn_div_u32(uint32_t *a, int n, uint32_t w) {
    uint64_t r = 0;
    for (int i = n - 1; i >= 0; i--) {
        uint64_t cur = (r << 32) | a[i];
        a[i] = (uint32_t)(cur / w);
        r = cur % w;
    }
    return (uint32_t)r;
}
static uint32_t bn_mod_u32(const uint32_t *a, int n, uint32_t w) {
    uint64_t r = 0;
    for (int i = n - 1; i >= 0; i--) r = ((r << 32) | a[i]) % w;
    return (uint32_t)r;
}
static int bn_cmp(const uint32_t *a, const uint32_t *b, int n) {
    for (int i = n - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}
/* a -= b over n words (caller guarantees a >= b) */
static void bn_sub(uint32_t *a, const uint32_t *b, int n) {
    int64_t br = 0;
    for (int i = 0; i < n; i++) {
        int64_t d = (int64_t)a[i] - b[i] + br;
        a[i] = (uint32_t)d;
        br = d >> 32;
    }
}
/* r = a mod m (a has na words, m has nm words, m != 0); binary long division,
 * setup-time only */
static void bn_mod(const uint32_t *a, int na, const uint32_t *m, int nm, uint32_t *r) {
    uint32_t acc[MAXW + 2];
    if (nm < 1 || nm > MAXW) return;
    memset(acc, 0, sizeof(acc));
    int w = nm + 1;
    for (int bit = 32 * na - 1; bit >= 0; bit--) {
        /* acc = acc*2 + bit */
        uint32_t c = (a[bit >> 5] >> (bit & 31)) & 1u;
        for (int i = 0; i < w; i++) {
            uint32_t nc = acc[i] >> 31;
            acc[i] = (acc[i] << 1) | c;
            c = nc;
        }
        uint32_t mm[MAXW + 2];
        memset(mm, 0, sizeof(mm));
        memcpy(mm, m, 4 * nm);
        if (bn_cmp(acc, mm, w) >= 0) bn_sub(acc, mm, w);
    }
    memcpy(r, acc, 4 * nm);
}
/* _float_scaled(x, base) of vecops.py:63-66: float(x >> s) * 2^(s-base),
 * s = max(0, bitlen(x)-53) -- truncation, exactly as the reference does */
static double float_scaled(const uint32_t *x, int n, int base) {
    int bl = bn_bitlen(x, n);
    int s = bl > 53 ? bl - 53 : 0;
    uint64_t top = 0;
    for (int k = 0; k < 64 && s + k < bl; k++) {
        int bit = s + k;
        top |= (uint64_t)((x[bit >> 5] >> (bit & 31)) & 1u) << k;
    }
    return ldexp((double)top, s - base);
}

/* ---------------- RNS context (modring.py:170-207) ---------------------- */

static int is_prime_u32(uint32_t n) {
    if (n < 2) return 0;
    static const uint32_t sp[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int i = 0; i < 12; i++)
        if (n % sp[i] == 0) return n == sp[i];
    uint32_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    static const uint32_t bases[] = {2, 7, 61}; /* deterministic below 4.7e9 */
    for (int b = 0; b < 3; b++) {
        uint64_t a = bases[b] % n, x = 1, p = a;
        uint32_t e = d;
        if (!a) continue;
        while (e) { if (e & 1) x = x * p % n; p = p * p % n; e >>= 1; }
        if (x == 1 || x == n - 1) continue;
        int ok = 0;
        for (int r = 1; r < s; r++) {
            x = x * x % n;
            if (x == n - 1) { ok = 1; break; }
        }
        if (!ok) return 0;
    }
    return 1;
}

static uint64_t inv_mod(uint64_t a, uint64_t m) {
    int64_t t = 0, nt = 1, r = (int64_t)m, nr = (int64_t)(a % m);
    while (nr) {
        int64_t q = r / nr, tmp;
        tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    return (uint64_t)(t < 0 ? t + (int64_t)m : t);
}

typedef struct {
    int k;
    uint32_t m[MAXK];
    uint32_t ell_limb[MAXK];         /* l mod m_i */
    uint32_t crt_mod_ell[MAXK][MAXW];/* C_i mod l, L words */
    double crt_frac[MAXK];           /* C_i / M as biased-exact floats */
    uint32_t mcomp[MAXW];            /* (-M) mod l */
} rns_ctx;

typedef struct {
    int L;                /* 32-bit words of l */
    int bits;
    uint32_t ell[MAXW];
    double ell_scaled;    /* float(l) / 2^base_r */
    int base_r;
    int64_t nrows, ncols, total_cols;
    int n_dense;
    const int64_t *row_ptr;
    /* per-lane CSR built at create time (copies) */
    int64_t *lane_ptr;    /* nrows+1, entries of the +-1/small lanes */
    int32_t *lane_col;
    int32_t *lane_tag;    /* 0:+1 1:-1 2:small+ 3:small- */
    uint32_t *lane_cabs;  /* |c| for small entries (< 2^63 is not allowed here) */
    int64_t *full_ptr;    /* nrows+1 */
    int64_t *full_col;
    uint32_t *full_val;   /* L words each */
    rns_ctx c1, c2;
    int has_full;
    int gamma1, gamma2;
    uint64_t cmax1;
    uint32_t *samp1, *samp2;  /* orc_spmv_sample's converted limbs */
} orc_mat;

/* build the context for headroom need = 2*gamma*cmax*l (modring.py:190-197) */
static void rns_build(rns_ctx *c, const orc_mat *A, uint64_t gamma, const uint32_t *cmax, int ncm) {
    /* need = 2*gamma*cmax*l */
    uint32_t need[MAXW];
    memset(need, 0, sizeof(need));
    /* need = cmax * l (schoolbook) */
    for (int i = 0; i < ncm; i++) {
        uint64_t carry = 0;
        for (int j = 0; j < A->L; j++) {
            uint64_t t = (uint64_t)cmax[i] * A->ell[j] + need[i + j] + carry;
            need[i + j] = (uint32_t)t;
            carry = t >> 32;
        }
        int p = i + A->L;
        while (carry) {
            uint64_t t = (uint64_t)need[p] + carry;
            need[p++] = (uint32_t)t;
            carry = t >> 32;
        }
    }
    uint64_t g2 = 2 * gamma;
    uint32_t glo = (uint32_t)g2, ghi = (uint32_t)(g2 >> 32);
    {
        uint32_t tmp[MAXW];
        memcpy(tmp, need, sizeof(tmp));
        uint32_t co = bn_mul_u32(need, MAXW - 2, glo);
        need[MAXW - 2] = co;
        if (ghi) { /* need += tmp * ghi * 2^32 */
            uint64_t carry = 0;
            for (int j = 0; j + 1 < MAXW; j++) {
                uint64_t t = (uint64_t)tmp[j] * ghi + need[j + 1] + carry;
                need[j + 1] = (uint32_t)t;
                carry = t >> 32;
            }
        }
    }
    uint32_t M[MAXW];
    memset(M, 0, sizeof(M));
    M[0] = 1;
    uint32_t p = 0x80000000u; /* _LIMB_BOUND = 2^31 */
    c->k = 0;
    while (bn_cmp(M, need, MAXW) <= 0) {
        do { p--; } while (!is_prime_u32(p));
        c->m[c->k++] = p;
        bn_mul_u32(M, MAXW, p);
    }
    int nM = bn_len(M, MAXW);
    int baseM = bn_bitlen(M, nM) - 4;
    if (baseM < 0) baseM = 0;
    double m_scaled = float_scaled(M, nM, baseM);
    /* -M mod l */
    uint32_t mm[MAXW];
    bn_mod(M, nM, A->ell, A->L, mm);
    memset(c->mcomp, 0, sizeof(c->mcomp));
    if (bn_len(mm, A->L)) {
        memcpy(c->mcomp, A->ell, 4 * A->L);
        bn_sub(c->mcomp, mm, A->L);
    }
    for (int i = 0; i < c->k; i++) {
        uint32_t Mi[MAXW];
        memcpy(Mi, M, sizeof(Mi));
        bn_div_u32(Mi, nM, c->m[i]);
        uint32_t r = bn_mod_u32(Mi, nM, c->m[i]);
        uint64_t inv = inv_mod(r, c->m[i]);
        uint32_t Ci[MAXW + 1];
        memset(Ci, 0, sizeof(Ci));
        memcpy(Ci, Mi, 4 * nM);
        Ci[nM] = bn_mul_u32(Ci, nM, (uint32_t)inv); /* C_i = Mi*inv < M */
        int nC = bn_len(Ci, nM + 1);
        c->crt_frac[i] = float_scaled(Ci, nC, baseM) / m_scaled;
        memset(c->crt_mod_ell[i], 0, sizeof(c->crt_mod_ell[i]));
        if (nC) bn_mod(Ci, nC, A->ell, A->L, c->crt_mod_ell[i]);
        c->ell_limb[i] = bn_mod_u32(A->ell, A->L, c->m[i]);
    }
}

/* u (L words) mod m */
static inline uint32_t res_mod(const uint32_t *u, int L, uint32_t m) {
    uint64_t r = 0;
    for (int i = L - 1; i >= 0; i--) r = ((r << 32) | u[i]) % m;
    return (uint32_t)r;
}

/* z += limbs . crt_mod_ell + t * mcomp  (vecops.py:338-352), z has L+3 words */
static void crt_fold(const rns_ctx *c, int L, const uint32_t *limbs, uint32_t *z) {
    double ipsum = 0.0, fsum = 0.0;
    for (int i = 0; i < c->k; i++) {
        double p = (double)limbs[i] * c->crt_frac[i];
        double ip = floor(p);
        ipsum += ip;
        fsum += p - ip;
    }
    uint64_t t = (uint64_t)(ipsum + floor(fsum + ldexp(1.0, -13)));
    for (int i = 0; i <= c->k; i++) {
        uint64_t w = i < c->k ? limbs[i] : t;
        const uint32_t *v = i < c->k ? c->crt_mod_ell[i] : c->mcomp;
        uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
        uint64_t carry = 0;
        for (int j = 0; j < L + 3; j++) {
            uint64_t vj = j < L ? v[j] : 0;
            uint64_t prod = vj * wl + z[j] + carry;
            z[j] = (uint32_t)prod;
            carry = prod >> 32;
        }
        if (wh) {
            carry = 0;
            for (int j = 0; j + 1 < L + 3; j++) {
                uint64_t vj = j < L ? v[j] : 0;
                uint64_t prod = vj * wh + z[j + 1] + carry;
                z[j + 1] = (uint32_t)prod;
                carry = prod >> 32;
            }
        }
    }
}

/* z mod l for non-negative z of L+3 words (vecops.py:119-162): biased float
 * quotient estimates until the estimate is 0, then exact subtractions */
static void reduce_compact(const orc_mat *A, uint32_t *z, uint32_t *out) {
    int L = A->L, W = L + 3;
    for (int it = 0; it < 64; it++) {
        double approx = float_scaled(z, W, A->base_r) / A->ell_scaled;
        double q = floor(approx * (1.0 - ldexp(1.0, -8)));
        if (q < 0) q = 0;
        if (q > ldexp(1.0, 50)) q = ldexp(1.0, 50);
        uint64_t qi = (uint64_t)q;
        if (!qi) break;
        /* z -= qi * l */
        uint32_t ql = (uint32_t)qi, qh = (uint32_t)(qi >> 32);
        uint32_t prod[MAXW + 4];
        memset(prod, 0, 4 * (W + 1));
        uint64_t carry = 0;
        for (int j = 0; j < L; j++) {
            uint64_t t = (uint64_t)A->ell[j] * ql + prod[j] + carry;
            prod[j] = (uint32_t)t; carry = t >> 32;
        }
        prod[L] = (uint32_t)carry;
        if (qh) {
            carry = 0;
            for (int j = 0; j < L; j++) {
                uint64_t t = (uint64_t)A->ell[j] * qh + prod[j + 1] + carry;
                prod[j + 1] = (uint32_t)t; carry = t >> 32;
            }
            prod[L + 1] += (uint32_t)carry;
        }
        bn_sub(z, prod, W);
    }
    uint32_t lw[MAXW + 4];
    memset(lw, 0, 4 * W);
    memcpy(lw, A->ell, 4 * L);
    for (int it = 0; it < 8 && bn_cmp(z, lw, W) >= 0; it++) bn_sub(z, lw, W);
    memcpy(out, z, 4 * L);
}

void orc_destroy(void *h) {
    orc_mat *A = (orc_mat *)h;
    if (!A) return;
    free(A->lane_ptr); free(A->lane_col); free(A->lane_tag); free(A->lane_cabs);
    free(A->full_ptr); free(A->full_col); free(A->full_val);
    free(A->samp1); free(A->samp2);
    free(A);
}

/*
 * Build from the reference SparseMatrix fields (spmatrix.py:77-91).
 * tags: 0 +1, 1 -1, 2 small (small_vals), 3 full (full_pos/full_vals);
 * dense_vals: n_dense x nrows residues (a zero entry is skipped,
 * spmatrix.py:218-223).  Returns NULL on bad input.
 */
void *orc_create(const uint32_t *ell, int L, int64_t nrows, int64_t ncols,
                 const int64_t *row_ptr, const int32_t *col_idx, const uint8_t *tags,
                 const int64_t *small_vals, int64_t n_full, const int64_t *full_pos,
                 const uint32_t *full_vals, int n_dense, const uint32_t *dense_vals) {
    if (L < 1 || L > 40) return NULL;
    orc_mat *A = (orc_mat *)calloc(1, sizeof(orc_mat));
    A->L = L;
    memcpy(A->ell, ell, 4 * L);
    A->bits = bn_bitlen(A->ell, L);
    A->nrows = nrows;
    A->ncols = ncols;
    A->n_dense = n_dense;
    A->total_cols = ncols + n_dense;
    /* ModReducer base: scale so the float of l keeps its top bits */
    A->base_r = A->bits > 60 ? A->bits - 60 : 0;
    A->ell_scaled = float_scaled(A->ell, L, A->base_r);
    int64_t nnz = row_ptr[nrows];
    A->lane_ptr = (int64_t *)calloc(nrows + 1, 8);
    A->lane_col = (int32_t *)malloc(8 + 4 * nnz);
    A->lane_tag = (int32_t *)malloc(8 + 4 * nnz);
    A->lane_cabs = (uint32_t *)malloc(8 + 4 * nnz);
    A->full_ptr = (int64_t *)calloc(nrows + 1, 8);
    /* full entries: map flat position -> value */
    int64_t nf_total = n_full + (int64_t)n_dense * nrows;
    A->full_col = (int64_t *)malloc(8 + 8 * nf_total);
    A->full_val = (uint32_t *)malloc(8 + 4 * (size_t)L * nf_total);
    int64_t fi = 0, li = 0, fcur = 0;
    int gamma1 = 1, gamma2 = 1;
    uint64_t cmax1 = 1;
    for (int64_t r = 0; r < nrows; r++) {
        int64_t cnt1 = 0, cnt2 = 0;
        for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) {
            int t = tags[p];
            if (t == 3) {
                while (fcur < n_full && full_pos[fcur] < p) fcur++;
                if (fcur >= n_full || full_pos[fcur] != p) { orc_destroy(A); return NULL; }
                A->full_col[fi] = col_idx[p];
                memcpy(A->full_val + (size_t)L * fi, full_vals + (size_t)L * fcur, 4 * L);
                fi++; cnt2++;
                continue;
            }
            A->lane_col[li] = col_idx[p];
            if (t == 0) { A->lane_tag[li] = 0; A->lane_cabs[li] = 1; }
            else if (t == 1) { A->lane_tag[li] = 1; A->lane_cabs[li] = 1; }
            else if (t == 2) {
                int64_t c = small_vals[p];
                uint64_t ac = c < 0 ? (uint64_t)(-c) : (uint64_t)c;
                if (ac >= 0x80000000ull) { orc_destroy(A); return NULL; }
                A->lane_tag[li] = c < 0 ? 3 : 2;
                A->lane_cabs[li] = (uint32_t)ac;
                if (ac > cmax1) cmax1 = ac;
            } else { orc_destroy(A); return NULL; }
            li++; cnt1++;
        }
        for (int g = 0; g < n_dense; g++) {
            const uint32_t *d = dense_vals + ((size_t)g * nrows + r) * L;
            int nz = 0;
            for (int j = 0; j < L; j++) nz |= d[j] != 0;
            if (!nz) continue;
            A->full_col[fi] = ncols + g;
            memcpy(A->full_val + (size_t)L * fi, d, 4 * L);
            fi++; cnt2++;
        }
        A->lane_ptr[r + 1] = li;
        A->full_ptr[r + 1] = fi;
        if (cnt1 > gamma1) gamma1 = (int)cnt1;
        if (cnt2 > gamma2) gamma2 = (int)cnt2;
    }
    A->gamma1 = gamma1;
    A->gamma2 = gamma2;
    A->cmax1 = cmax1;
    A->has_full = fi > 0;
    uint32_t cm[2] = {(uint32_t)cmax1, (uint32_t)(cmax1 >> 32)};
    rns_build(&A->c1, A, (uint64_t)gamma1, cm, 2);
    if (A->has_full) {
        uint32_t lm1[MAXW];
        memcpy(lm1, A->ell, 4 * L);
        lm1[0] -= 1; /* l odd: no borrow */
        rns_build(&A->c2, A, (uint64_t)gamma2, lm1, L);
    }
    return A;
}

int orc_info(void *h, int64_t *out) {
    orc_mat *A = (orc_mat *)h;
    out[0] = A->c1.k;
    out[1] = A->has_full ? A->c2.k : 0;
    out[2] = A->gamma1;
    out[3] = A->gamma2;
    out[4] = (int64_t)A->cmax1;
    out[5] = A->bits;
    return 0;
}

/*
 * v[r] = (A u)[r] mod l for r in [row_lo, row_hi).  u: total_cols x L words,
 * v: nrows x L words (only the requested rows are written).
 */
/* RnsBatch.to_limbs (vecops.py:316-319) for columns [c_lo, c_hi) */
static void orc_to_rns(const orc_mat *A, const uint32_t *u, uint32_t *lim1, uint32_t *lim2,
                       int64_t c_lo, int64_t c_hi) {
    const int L = A->L;
    const rns_ctx *c1 = &A->c1, *c2 = &A->c2;
    const int k1 = c1->k, k2 = A->has_full ? c2->k : 0;
#pragma omp parallel for schedule(static)
    for (int64_t j = c_lo; j < c_hi; j++) {
        for (int i = 0; i < k1; i++) lim1[j * k1 + i] = res_mod(u + j * L, L, c1->m[i]);
        for (int i = 0; i < k2; i++) lim2[j * k2 + i] = res_mod(u + j * L, L, c2->m[i]);
    }
}

static void orc_rows(const orc_mat *A, const uint32_t *lim1, const uint32_t *lim2, uint32_t *v,
                     int64_t row_lo, int64_t row_hi);

int orc_spmv(void *h, const uint32_t *u, uint32_t *v, int64_t row_lo, int64_t row_hi, int nthreads) {
    orc_mat *A = (orc_mat *)h;
    const int k1 = A->c1.k, k2 = A->has_full ? A->c2.k : 0;
    /* every column that is read is converted */
    int64_t nc = A->total_cols;
    uint32_t *lim1 = (uint32_t *)malloc(8 + 4 * (size_t)k1 * nc);
    uint32_t *lim2 = k2 ? (uint32_t *)malloc(8 + 4 * (size_t)k2 * nc) : NULL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    orc_to_rns(A, u, lim1, lim2, 0, nc);
    orc_rows(A, lim1, lim2, v, row_lo, row_hi);
    free(lim1);
    free(lim2);
    return 0;
}

/* A bounded timing sample of one SpMV (bench.py's reference arm): the
 * conversion of columns [c_lo, c_hi) plus rows [row_lo, row_hi), i.e. the
 * same fraction of both halves of orc_spmv's work.  The converted limbs
 * live in buffers kept with the matrix (converted in full on the first
 * call), so every column a sampled row reads holds a real residue. */
int orc_spmv_sample(void *h, const uint32_t *u, uint32_t *v, int64_t row_lo, int64_t row_hi,
                    int64_t c_lo, int64_t c_hi, int nthreads) {
    orc_mat *A = (orc_mat *)h;
    const int k1 = A->c1.k, k2 = A->has_full ? A->c2.k : 0;
    int64_t nc = A->total_cols;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    if (!A->samp1) {
        A->samp1 = (uint32_t *)malloc(8 + 4 * (size_t)k1 * nc);
        A->samp2 = k2 ? (uint32_t *)malloc(8 + 4 * (size_t)k2 * nc) : NULL;
        if (!A->samp1 || (k2 && !A->samp2)) return -1;
        orc_to_rns(A, u, A->samp1, A->samp2, 0, nc);
    }
    if (c_lo < 0 || c_hi > nc || c_lo > c_hi || row_lo < 0 || row_hi > A->nrows || row_lo > row_hi) return -1;
    orc_to_rns(A, u, A->samp1, A->samp2, c_lo, c_hi);
    orc_rows(A, A->samp1, A->samp2, v, row_lo, row_hi);
    return 0;
}

static void orc_rows(const orc_mat *A, const uint32_t *lim1, const uint32_t *lim2, uint32_t *v,
                     int64_t row_lo, int64_t row_hi) {
    const int L = A->L;
    const rns_ctx *c1 = &A->c1, *c2 = &A->c2;
    const int k1 = c1->k, k2 = A->has_full ? c2->k : 0;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t r = row_lo; r < row_hi; r++) {
        int64_t acc[MAXK];
        uint32_t lim[MAXK];
        uint32_t z[MAXW + 4];
        memset(z, 0, sizeof(z));
        int64_t nminus = 0;
        for (int i = 0; i < k1; i++) acc[i] = 0;
        for (int64_t p = A->lane_ptr[r]; p < A->lane_ptr[r + 1]; p++) {
            const uint32_t *ul = lim1 + (int64_t)A->lane_col[p] * k1;
            int t = A->lane_tag[p];
            if (t == 0) {
                for (int i = 0; i < k1; i++) acc[i] += ul[i];
            } else if (t == 1) {
                nminus++;
                for (int i = 0; i < k1; i++) acc[i] -= ul[i];
            } else if (t == 2) {
                uint64_t c = A->lane_cabs[p];
                for (int i = 0; i < k1; i++)
                    acc[i] += (int64_t)((c % c1->m[i]) * ul[i] % c1->m[i]);
            } else {
                uint64_t c = A->lane_cabs[p];
                for (int i = 0; i < k1; i++) {
                    uint64_t m = c1->m[i];
                    uint64_t un = (c1->ell_limb[i] + m - ul[i]) % m; /* limbs_negate */
                    acc[i] += (int64_t)((c % m) * un % m);
                }
            }
        }
        for (int i = 0; i < k1; i++) {
            int64_t m = c1->m[i];
            int64_t a = acc[i] + nminus * (int64_t)c1->ell_limb[i];
            a %= m;
            if (a < 0) a += m;
            lim[i] = (uint32_t)a;
        }
        crt_fold(c1, L, lim, z);
        if (k2) {
            int64_t acc2[MAXK];
            for (int i = 0; i < k2; i++) acc2[i] = 0;
            for (int64_t p = A->full_ptr[r]; p < A->full_ptr[r + 1]; p++) {
                const uint32_t *ul = lim2 + A->full_col[p] * k2;
                const uint32_t *f = A->full_val + (size_t)L * p;
                for (int i = 0; i < k2; i++) {
                    uint64_t m = c2->m[i];
                    acc2[i] += (int64_t)((uint64_t)res_mod(f, L, (uint32_t)m) * ul[i] % m);
                }
            }
            for (int i = 0; i < k2; i++) lim[i] = (uint32_t)(acc2[i] % (int64_t)c2->m[i]);
            crt_fold(c2, L, lim, z);
        }
        reduce_compact(A, z, v + r * L);
    }
}

/* a[t] = sum_j x[t][j] * v[j] mod l  -- DenseRows.project, solver.py:186-189
 * (x: m x n residues, v: n residues, out: m residues) */
int orc_dense_project(void *h, const uint32_t *x, const uint32_t *vv, int64_t n, int m, uint32_t *out) {
    orc_mat *A = (orc_mat *)h;
    const int L = A->L;
    for (int t = 0; t < m; t++) {
        /* accumulate the exact product sum, reducing every 2^20 terms */
        uint32_t z[MAXW + 4];
        uint64_t wide[2 * 40 + 4];
        memset(z, 0, sizeof(z));
        for (int64_t j0 = 0; j0 < n; j0 += 1 << 20) {
            int64_t j1 = j0 + (1 << 20) < n ? j0 + (1 << 20) : n;
            /* columns of a 2L-word product, each column sum < 2^(64+20) split in hi/lo */
            uint64_t lo[2 * 40 + 4], hi[2 * 40 + 4];
            memset(lo, 0, sizeof(lo));
            memset(hi, 0, sizeof(hi));
            for (int64_t j = j0; j < j1; j++) {
                const uint32_t *a = x + ((size_t)t * n + j) * L, *b = vv + (size_t)j * L;
                for (int p = 0; p < L; p++) {
                    if (!a[p]) continue;
                    for (int q = 0; q < L; q++) {
                        uint64_t pr = (uint64_t)a[p] * b[q];
                        lo[p + q] += (uint32_t)pr;
                        hi[p + q + 1] += pr >> 32;
                    }
                }
            }
            /* lo/hi column sums < 2^52: propagate into a 2L+3 word integer */
            uint64_t carry = 0;
            int W = 2 * L + 3;
            for (int i = 0; i < W; i++) {
                unsigned __int128 s = (unsigned __int128)lo[i] + hi[i] + carry;
                wide[i] = (uint32_t)s;
                carry = (uint64_t)(s >> 32);
            }
            /* reduce wide mod l and add into z */
            uint32_t w32[2 * 40 + 4], r[MAXW];
            for (int i = 0; i < W; i++) w32[i] = (uint32_t)wide[i];
            bn_mod(w32, W, A->ell, L, r);
            uint64_t c = 0;
            for (int i = 0; i < L + 1; i++) {
                uint64_t s2 = (uint64_t)z[i] + (i < L ? r[i] : 0) + c;
                z[i] = (uint32_t)s2;
                c = s2 >> 32;
            }
            uint32_t lw[MAXW + 4];
            memset(lw, 0, sizeof(lw));
            memcpy(lw, A->ell, 4 * L);
            if (bn_cmp(z, lw, L + 1) >= 0) bn_sub(z, lw, L + 1);
        }
        memcpy(out + (size_t)t * L, z, 4 * L);
    }
    return 0;
}

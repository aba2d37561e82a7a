/*
 * gf2e_oracle.c — CPU restatement of the reference gf2elin hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * library (paper_1111_6900_b200/csrc) and the "port" CPU baseline timed by
 * bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/gf2elin/):
 *
 *   orc_mix / orc_word_stream      rng.py:20-28        counter-mode splitmix64
 *   orc_packed_random              rng.py:31-35 + mat_packed.py:253-259 (+ from_array 95-112)
 *   orc_slice                      mat_sliced.py:97-101 (+ mat_packed.to_array 114-122)
 *   orc_cling                      mat_sliced.py:104-106 (+ mat_packed.from_array 95-112)
 *   orc_gf2_mul                    mat_gf2.py:348-366  M4RM, k = 8 (tuning.py:15),
 *                                  table built as in _subset_xor_table_batched 301-310.
 *                                  The reference switches to Strassen-Winograd above
 *                                  2048 (mat_gf2.py:446-448); every strategy is
 *                                  bit-identical (mat_gf2.py:9-12, 435-436), so the
 *                                  oracle uses M4RM at every size.
 *   orc_karatsuba                  poly_mul.py:166-220 (_kara), 223-242 (reduce_mod_f),
 *                                  245-259 (karatsuba_mul), counters 32-43, 128-143.
 *   orc_reduce_mod_f               poly_mul.py:223-242
 *
 * Layout (mat_gf2.py:3-7): entry (i, j) of a GF(2) plane is bit j % 64 of word
 * j / 64 of row i; bits past ncols are zero.  Packed (mat_packed.py:1-13):
 * element (i, j) sits in bits [j*w, j*w + e) of the packed row, w = pack_width(e).
 *
 * Build: see oracle/Makefile (gcc -O3 -fopenmp -shared).  Output: oracle/_build/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL

/* rng.py:20-28 — value i (0-based) of seed s is mix(s + (i+1)*GOLDEN). */
static inline uint64_t orc_mix(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * GOLDEN;
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

void orc_word_stream(uint64_t seed, uint64_t start, uint64_t count, uint64_t *out) {
    for (uint64_t i = 0; i < count; ++i) out[i] = orc_mix(seed, start + i);
}

/* mat_packed.py:26-33 */
int orc_pack_width(int e) {
    static const int widths[] = {1, 2, 4, 8, 16, 32, 64};
    if (e < 2 || e > 10) return -1;
    for (int i = 0; i < 7; ++i)
        if (widths[i] >= e) return widths[i];
    return -1;
}

static inline int64_t words_for(int64_t ncols) { return (ncols + 63) >> 6; } /* mat_gf2.py:44 */

/*
 * mat_packed.py:253-259: randomize(seed) = from_array(element_stream(seed, m*n, e)).
 * Element (i, j) of the sub-block takes stream index (row0 + i) * gcols + col0 + j, so a
 * row/column window of the full generator matrix can be built without the rest
 * (SURVEY §8c "sampled blocks").  row0 = col0 = 0, gcols = cols is the reference call.
 */
void orc_packed_random(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                       int64_t col0, int64_t gcols, uint64_t *out, int64_t ld) {
    int w = orc_pack_width(e);
    uint64_t mask = (1ULL << e) - 1;
    int per = 64 / w;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        uint64_t *row = out + i * ld;
        memset(row, 0, sizeof(uint64_t) * ld);
        uint64_t base = (uint64_t)(row0 + i) * (uint64_t)gcols + (uint64_t)col0;
        for (int64_t j = 0; j < cols; ++j) {
            uint64_t v = orc_mix(seed, base + (uint64_t)j) & mask;
            row[j / per] |= v << ((j % per) * w);
        }
    }
}

/* Per-element sliced generator: plane t of element (i, j) = bit t of the element above. */
void orc_sliced_random(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                       int64_t col0, int64_t gcols, uint64_t *planes, int64_t ld,
                       int64_t pstride) {
    uint64_t mask = (1ULL << e) - 1;
    for (int t = 0; t < e; ++t) memset(planes + t * pstride, 0, sizeof(uint64_t) * rows * ld);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        uint64_t base = (uint64_t)(row0 + i) * (uint64_t)gcols + (uint64_t)col0;
        for (int64_t j = 0; j < cols; ++j) {
            uint64_t v = orc_mix(seed, base + (uint64_t)j) & mask;
            for (int t = 0; t < e; ++t)
                planes[t * pstride + i * ld + (j >> 6)] |= ((v >> t) & 1ULL) << (j & 63);
        }
    }
}

/* mat_sliced.py:97-101: plane t, entry (i, j) = bit t of the slot; pad bits are dropped
 * (only bits 0..e-1 are read, mat_packed.py:114-122). */
void orc_slice(int e, int64_t rows, int64_t cols, const uint64_t *packed, int64_t ldp,
               uint64_t *planes, int64_t ld, int64_t pstride) {
    int w = orc_pack_width(e);
    int per = 64 / w;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        for (int t = 0; t < e; ++t) memset(planes + t * pstride + i * ld, 0, sizeof(uint64_t) * ld);
        for (int64_t j = 0; j < cols; ++j) {
            uint64_t v = packed[i * ldp + j / per] >> ((j % per) * w);
            for (int t = 0; t < e; ++t)
                planes[t * pstride + i * ld + (j >> 6)] |= ((v >> t) & 1ULL) << (j & 63);
        }
    }
}

/* mat_sliced.py:104-106 -> mat_packed.py:95-112: slot bits t < e from plane t, pad zero. */
void orc_cling(int e, int64_t rows, int64_t cols, const uint64_t *planes, int64_t ld,
               int64_t pstride, uint64_t *packed, int64_t ldp) {
    int w = orc_pack_width(e);
    int per = 64 / w;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) {
        memset(packed + i * ldp, 0, sizeof(uint64_t) * ldp);
        for (int64_t j = 0; j < cols; ++j) {
            uint64_t v = 0;
            for (int t = 0; t < e; ++t)
                v |= ((planes[t * pstride + i * ld + (j >> 6)] >> (j & 63)) & 1ULL) << t;
            packed[i * ldp + j / per] |= v << ((j % per) * w);
        }
    }
}

/*
 * mat_gf2.py:348-366 (_mul_m4rm) with the batched table of 301-310: for each group of
 * k = 8 inner indices, table[x] = XOR of the B rows selected by the bits of x; every row
 * of A picks its contribution with one lookup of its 8-bit index.  Blocked over
 * 2048-bit column strips and 512-row chunks so tables stay in cache; tasks run on
 * OpenMP threads.  C = A*B, or C ^= A*B when accumulate != 0.
 */
#define ORC_CW 32   /* words per column strip */
#define ORC_RC 512  /* rows per task */
void orc_gf2_mul(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, uint64_t *C,
                 int64_t ldc, int64_t m, int64_t k, int64_t n, int accumulate, int nthreads) {
    int64_t nw = words_for(n);
    if (!accumulate)
        for (int64_t i = 0; i < m; ++i) memset(C + i * ldc, 0, sizeof(uint64_t) * nw);
    if (m == 0 || k == 0 || n == 0) return;
    int64_t nstrips = (nw + ORC_CW - 1) / ORC_CW;
    int64_t nchunks = (m + ORC_RC - 1) / ORC_RC;
    int64_t ntasks = nstrips * nchunks;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#endif
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        uint64_t *table = (uint64_t *)aligned_alloc(64, sizeof(uint64_t) * 256 * ORC_CW);
#pragma omp for schedule(dynamic)
        for (int64_t task = 0; task < ntasks; ++task) {
            int64_t s = task % nstrips, ch = task / nstrips;
            int64_t w0 = s * ORC_CW, cw = nw - w0 < ORC_CW ? nw - w0 : ORC_CW;
            int64_t r0 = ch * ORC_RC, r1 = r0 + ORC_RC < m ? r0 + ORC_RC : m;
            for (int64_t c0 = 0; c0 < k; c0 += 8) {
                int kk = (int)(k - c0 < 8 ? k - c0 : 8);
                memset(table, 0, sizeof(uint64_t) * ORC_CW);
                for (int bit = 0; bit < kk; ++bit) { /* mat_gf2.py:305-307 */
                    int half = 1 << bit;
                    const uint64_t *src = B + (c0 + bit) * ldb + w0;
                    for (int x = 0; x < half; ++x) {
                        uint64_t *dst = table + (half + x) * ORC_CW;
                        const uint64_t *lo = table + x * ORC_CW;
                        for (int64_t q = 0; q < cw; ++q) dst[q] = lo[q] ^ src[q];
                    }
                }
                for (int64_t i = r0; i < r1; ++i) { /* mat_gf2.py:361-365 */
                    uint64_t aw = A[i * lda + (c0 >> 6)] >> (c0 & 63);
                    unsigned idx = (unsigned)(aw & ((1u << kk) - 1));
                    if (!idx) continue;
                    const uint64_t *tr = table + idx * ORC_CW;
                    uint64_t *cr = C + i * ldc + w0;
                    for (int64_t q = 0; q < cw; ++q) cr[q] ^= tr[q];
                }
            }
        }
        free(table);
    }
}

/* ---------------------------------------------------------------------------------
 * Karatsuba over slice lists (poly_mul.py:166-220) with the reference's counters.
 * A "plane" is an owned buffer of rows x ld words.
 * --------------------------------------------------------------------------------- */
typedef struct {
    int64_t rows, ld;
    uint64_t *w;
} orc_plane;

typedef struct {
    int64_t gf2_matmul_count, additions, peak_live_products; /* poly_mul.py:32-43 */
    int64_t live;                                             /* poly_mul.py:128-143 */
    int nthreads;
    int64_t m, k, n;
} orc_ctx;

static orc_plane plane_new(int64_t rows, int64_t ld) {
    orc_plane p = {rows, ld, (uint64_t *)calloc((size_t)(rows * ld > 0 ? rows * ld : 1), 8)};
    return p;
}
static orc_plane plane_copy(const orc_plane *x) {
    orc_plane p = plane_new(x->rows, x->ld);
    memcpy(p.w, x->w, sizeof(uint64_t) * x->rows * x->ld);
    return p;
}
static void plane_iadd(orc_plane *x, const orc_plane *y) { /* mat_gf2.py:161-164 */
    int64_t nwords = x->rows * x->ld;
    for (int64_t i = 0; i < nwords; ++i) x->w[i] ^= y->w[i];
}
static void plane_free(orc_plane *x) { free(x->w); x->w = NULL; }

static void live_grab(orc_ctx *c, int64_t k) {
    c->live += k;
    if (c->live > c->peak_live_products) c->peak_live_products = c->live;
}

/* poly_mul.py:146-150 */
static orc_plane base_product(orc_ctx *c, const orc_plane *a, const orc_plane *b) {
    orc_plane out = plane_new(c->m, words_for(c->n));
    c->gf2_matmul_count += 1; /* mat_gf2.py:444-445 */
    orc_gf2_mul(a->w, a->ld, b->w, b->ld, out.w, out.ld, c->m, c->k, c->n, 0, c->nthreads);
    live_grab(c, 1);
    return out;
}

static orc_plane plane_xor(const orc_plane *x, const orc_plane *y) {
    orc_plane p = plane_copy(x);
    plane_iadd(&p, y);
    return p;
}

/* poly_mul.py:153-163 — xs/ys may differ in length; result has max length. */
static int add_lists(orc_ctx *c, orc_plane *xs, int nx, orc_plane *ys, int ny, orc_plane *out) {
    if (nx < ny) {
        orc_plane *t = xs; xs = ys; ys = t;
        int tn = nx; nx = ny; ny = tn;
    }
    for (int i = 0; i < nx; ++i) out[i] = plane_copy(&xs[i]);
    for (int i = 0; i < ny; ++i) plane_iadd(&out[i], &ys[i]);
    c->additions += ny;
    return nx;
}

/* poly_mul.py:166-220.  a, b: ka planes each (not owned).  out: 2ka-1 owned planes. */
static void kara(orc_ctx *c, orc_plane *a, orc_plane *b, int ka, orc_plane *out) {
    if (ka == 1) {
        out[0] = base_product(c, &a[0], &b[0]);
        return;
    }
    if (ka == 3) {
        orc_plane d0 = base_product(c, &a[0], &b[0]);
        orc_plane d1 = base_product(c, &a[1], &b[1]);
        orc_plane d2 = base_product(c, &a[2], &b[2]);
        orc_plane sa = plane_xor(&a[0], &a[1]), sb = plane_xor(&b[0], &b[1]);
        orc_plane d01 = base_product(c, &sa, &sb);
        plane_free(&sa); plane_free(&sb);
        sa = plane_xor(&a[0], &a[2]); sb = plane_xor(&b[0], &b[2]);
        orc_plane d02 = base_product(c, &sa, &sb);
        plane_free(&sa); plane_free(&sb);
        sa = plane_xor(&a[1], &a[2]); sb = plane_xor(&b[1], &b[2]);
        orc_plane d12 = base_product(c, &sa, &sb);
        plane_free(&sa); plane_free(&sb);
        /* c1 = d01^d0^d1 ; c2 = d02^d0^d1^d2 ; c3 = d12^d1^d2   (poly_mul.py:187-189) */
        plane_iadd(&d01, &d0); plane_iadd(&d01, &d1);
        plane_iadd(&d02, &d0); plane_iadd(&d02, &d1); plane_iadd(&d02, &d2);
        plane_iadd(&d12, &d1); plane_iadd(&d12, &d2);
        c->additions += 6 + 7;
        c->live -= 6;
        live_grab(c, 5);
        out[0] = d0; out[1] = d01; out[2] = d02; out[3] = d12; out[4] = d2;
        plane_free(&d1);
        return;
    }
    int h = (ka + 1) / 2;
    int nlo = 2 * h - 1, nhi = 2 * (ka - h) - 1;
    orc_plane *lo = (orc_plane *)calloc(nlo, sizeof(orc_plane));
    orc_plane *hi = (orc_plane *)calloc(nhi > 0 ? nhi : 1, sizeof(orc_plane));
    kara(c, a, b, h, lo);
    kara(c, a + h, b + h, ka - h, hi);
    orc_plane *sa = (orc_plane *)calloc(h, sizeof(orc_plane));
    orc_plane *sb = (orc_plane *)calloc(h, sizeof(orc_plane));
    int ns = add_lists(c, a, h, a + h, ka - h, sa);
    add_lists(c, b, h, b + h, ka - h, sb);
    int nmid = 2 * ns - 1;
    orc_plane *mid = (orc_plane *)calloc(nmid, sizeof(orc_plane));
    kara(c, sa, sb, ns, mid);
    for (int i = 0; i < ns; ++i) { plane_free(&sa[i]); plane_free(&sb[i]); }
    free(sa); free(sb);
    for (int i = 0; i < nlo; ++i) plane_iadd(&mid[i], &lo[i]); /* poly_mul.py:203-206 */
    for (int i = 0; i < nhi; ++i) plane_iadd(&mid[i], &hi[i]);
    c->additions += nlo + nhi;
    int nout = 2 * ka - 1;
    for (int i = 0; i < nout; ++i) out[i] = plane_new(c->m, words_for(c->n));
    for (int i = 0; i < nlo; ++i) plane_iadd(&out[i], &lo[i]); /* poly_mul.py:209-215 */
    for (int i = 0; i < nmid; ++i) plane_iadd(&out[h + i], &mid[i]);
    for (int i = 0; i < nhi; ++i) plane_iadd(&out[2 * h + i], &hi[i]);
    c->additions += nlo + nmid + nhi;
    c->live -= nlo + nhi + nmid;
    live_grab(c, nout);
    for (int i = 0; i < nlo; ++i) plane_free(&lo[i]);
    for (int i = 0; i < nhi; ++i) plane_free(&hi[i]);
    for (int i = 0; i < nmid; ++i) plane_free(&mid[i]);
    free(lo); free(hi); free(mid);
}

/* poly_mul.py:223-242 on raw planes: planes[0..2e-2] are updated in place. */
int64_t orc_reduce_mod_f(int e, uint32_t f, uint64_t **planes, int64_t nwords) {
    int64_t adds = 0;
    for (int d = 2 * e - 2; d >= e; --d)
        for (int k = 0; k < e; ++k)
            if ((f >> k) & 1u) {
                uint64_t *dst = planes[d - e + k];
                const uint64_t *top = planes[d];
                for (int64_t i = 0; i < nwords; ++i) dst[i] ^= top[i];
                ++adds;
            }
    return adds;
}

/*
 * poly_mul.py:245-259 (karatsuba_mul), plus accumulate = the addmul pattern
 * X ^= karatsuba_mul(A, B) (ple_echelon.py:130-136,259; mat_gf2.py:161-164).
 * A: e planes of m x k (row stride lda, plane stride pa), B: e planes k x n, C: e planes
 * m x n.  counters[3] receives gf2_matmul_count, additions, peak_live_products.
 */
int orc_karatsuba(int e, uint32_t f, const uint64_t *A, int64_t lda, int64_t pa,
                  const uint64_t *B, int64_t ldb, int64_t pb, uint64_t *C, int64_t ldc,
                  int64_t pc, int64_t m, int64_t k, int64_t n, int accumulate, int nthreads,
                  int64_t *counters) {
    if (e < 2 || e > 10) return -1;
    orc_ctx c;
    memset(&c, 0, sizeof(c));
    c.nthreads = nthreads;
    c.m = m; c.k = k; c.n = n;
    orc_plane *a = (orc_plane *)calloc(e, sizeof(orc_plane));
    orc_plane *b = (orc_plane *)calloc(e, sizeof(orc_plane));
    int64_t kw = words_for(k), nw = words_for(n);
    for (int t = 0; t < e; ++t) {
        a[t] = plane_new(m, kw);
        b[t] = plane_new(k, nw);
        for (int64_t i = 0; i < m; ++i) memcpy(a[t].w + i * kw, A + t * pa + i * lda, 8 * kw);
        for (int64_t i = 0; i < k; ++i) memcpy(b[t].w + i * nw, B + t * pb + i * ldb, 8 * nw);
    }
    int np = 2 * e - 1;
    orc_plane *prod = (orc_plane *)calloc(np, sizeof(orc_plane));
    kara(&c, a, b, e, prod);
    uint64_t **pp = (uint64_t **)calloc(np, sizeof(uint64_t *));
    for (int i = 0; i < np; ++i) pp[i] = prod[i].w;
    c.additions += orc_reduce_mod_f(e, f, pp, m * nw);
    for (int t = 0; t < e; ++t)
        for (int64_t i = 0; i < m; ++i) {
            uint64_t *dst = C + t * pc + i * ldc;
            const uint64_t *src = prod[t].w + i * nw;
            if (accumulate)
                for (int64_t q = 0; q < nw; ++q) dst[q] ^= src[q];
            else
                memcpy(dst, src, 8 * nw);
        }
    if (counters) {
        counters[0] = c.gf2_matmul_count;
        counters[1] = c.additions;
        counters[2] = c.peak_live_products;
    }
    for (int i = 0; i < np; ++i) plane_free(&prod[i]);
    for (int t = 0; t < e; ++t) { plane_free(&a[t]); plane_free(&b[t]); }
    free(prod); free(pp); free(a); free(b);
    return 0;
}

/* ---- PLE base case ----------------------------------------------------------------------
 * newton_john.py:207-260 (nj_ple), restated on a row-major element array a[m][n] (uint16):
 * for each column j, the first row i >= r with a nonzero entry is the pivot; rows i, r are
 * swapped; the pivot row right of j is scaled by 1/pivot (the pivot stays as L's diagonal);
 * every row below r gets x * (pivot row right of j) added, x = its entry in column j (kept
 * as the multiplier).  Finally columns t <-> Q[t] are swapped in rows >= t (L compression).
 * Returns the rank; P, Q (length min(m, n)) are LAPACK-style swap vectors.  The recursive
 * ple() (ple_echelon.py:240-300) returns the same factors for every crossover. */
static uint32_t orc_gf_mul(uint32_t a, uint32_t b, int e, uint32_t f) { /* gf2e.py:40-56 */
    uint32_t acc = 0;
    for (int i = 0; i < e; ++i)
        if ((b >> i) & 1u) acc ^= a << i;
    for (int d = 2 * e - 2; d >= e; --d)
        if ((acc >> d) & 1u) acc ^= f << (d - e);
    return acc;
}

int64_t orc_ple(int e, uint32_t f, uint16_t *a, int64_t m, int64_t n, int64_t *P, int64_t *Q) {
    const int q = 1 << e;
    uint16_t *mt = (uint16_t *)malloc((size_t)q * q * sizeof(uint16_t));
    for (int x = 0; x < q; ++x)
        for (int y = 0; y < q; ++y) mt[x * q + y] = (uint16_t)orc_gf_mul((uint32_t)x, (uint32_t)y, e, f);
    const int64_t k = m < n ? m : n;
    for (int64_t i = 0; i < k; ++i) P[i] = Q[i] = i;
    int64_t r = 0;
    for (int64_t j = 0; j < n && r < k; ++j) {
        int64_t i = r;
        while (i < m && a[i * n + j] == 0) ++i;
        if (i == m) continue;
        const uint32_t piv = a[i * n + j];
        P[r] = i;
        Q[r] = j;
        if (i != r)
            for (int64_t c = 0; c < n; ++c) {
                uint16_t t = a[i * n + c];
                a[i * n + c] = a[r * n + c];
                a[r * n + c] = t;
            }
        uint32_t inv = 1;
        for (uint32_t y = 1; y < (uint32_t)q; ++y)
            if (mt[piv * q + y] == 1) inv = y;
        uint16_t *pr = a + r * n;
        if (piv != 1)
            for (int64_t c = j + 1; c < n; ++c) pr[c] = mt[inv * q + pr[c]];
#pragma omp parallel for schedule(static)
        for (int64_t i2 = r + 1; i2 < m; ++i2) {
            uint16_t *row = a + i2 * n;
            const uint32_t x = row[j];
            if (!x) continue;
            const uint16_t *mx = mt + x * q;
            for (int64_t c = j + 1; c < n; ++c) row[c] ^= mx[pr[c]];
        }
        ++r;
    }
    for (int64_t t = 0; t < r; ++t)
        if (Q[t] != t)
            for (int64_t i = t; i < m; ++i) {
                uint16_t x = a[i * n + t];
                a[i * n + t] = a[i * n + Q[t]];
                a[i * n + Q[t]] = x;
            }
    free(mt);
    return r;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

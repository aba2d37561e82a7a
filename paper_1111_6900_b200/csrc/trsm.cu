// trsm.cu — device kernels for the first consumers of the hot path:
//   * k_tri_inverse: inverse of each 128-row diagonal block of a triangular GF(2^e) matrix
//     held as bit planes (the base case of the blocked TRSM in capi.cu, whose off-diagonal
//     updates are all addmul calls into the tensor-core product kernel);
//   * k_mul_by_x: sliced multiplication by alpha (mat_sliced.py:109-122);
//   * k_scalar_mul: packed multiplication by a scalar (mat_packed.py:192-199).
// Field arithmetic uses the per-field tables of ple.cu (field_tab: inverses, multiplication
// matrices; the scalar kernels build their own small tables).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace gf2e {
namespace {

// carry-less a*b mod f (e <= 10): used only to build tables
__device__ __forceinline__ uint32_t gf_mul_slow(uint32_t a, uint32_t b, int e, uint32_t f) {
    uint32_t acc = 0;
    for (int i = 0; i < e; ++i)
        if ((b >> i) & 1u) acc ^= a << i;
    for (int d = 2 * e - 2; d >= e; --d)
        if ((acc >> d) & 1u) acc ^= f << (d - e);
    return acc;
}


// Inverse of each TB x TB diagonal block by bitsliced substitution.  Lower triangular: for
// i = 0 .. rows-1, row i of X is final and published; every row k > i adds U_ki * X_i (U =
// T D^-1 unit triangular, so T^-1 = D^-1 U^-1 and each row is scaled once at the end).  Upper:
// the same from the bottom.
//   * Row k of X is owned by TPR = NW * BS consecutive threads, one per (plane word w, group h
//     of PB planes): 512 threads for TB = 128, 1024 for TB = 256.
//   * The multipliers U_ki are computed once up front into shared memory (cU, column-major so
//     the rows of a warp read consecutive entries).
//   * Per step the CTA builds, from the published X_i, the table of its scalar multiples split
//     by the low H1 / high H2 bits of the scalar (c * X_i = lo[c_lo] ^ hi[c_hi], 2^H1 + 2^H2
//     entries, FieldTab.mulmask: plane b of c*v = XOR of the planes in mulmask[c][b]); each
//     row then adds two looked-up words per plane instead of an e x e plane product.
// Two barriers per step: X_i published -> table built -> table consumed (and X_i+1 final).
#ifndef GF2E_TRI_BS
#define GF2E_TRI_BS 2
#endif
template <int E, int TB>
struct TriShape {
    static constexpr int NW = TB / 64;            // plane words per block row
    static constexpr int BS = TB == 128 ? GF2E_TRI_BS : 1;  // plane groups per row
    static constexpr int TPR = NW * BS;           // threads per row
    static constexpr int THREADS = TB * TPR;
    static constexpr int PB = (E + BS - 1) / BS;  // planes per thread
    static_assert(BS == 1 || BS == 2, "the final row scaling exchanges plane halves between two lanes");
    static constexpr int H1 = E <= 4 ? E : E / 2, H2 = E <= 4 ? 0 : E - E / 2;
    static constexpr int Q = (1 << H1) + (H2 ? (1 << H2) : 0);  // table entries
    static constexpr int TW = Q * E * NW;                        // table words
    static constexpr int NB = (TW + THREADS - 1) / THREADS;      // table words per thread
    using CT = typename std::conditional<(E <= 8), uint8_t, uint16_t>::type;
    static constexpr size_t SMEM = (size_t)TW * 8 + (size_t)NW * E * 8 + (size_t)TB * TB * sizeof(CT);
};

template <int E, int TB>
__global__ void __launch_bounds__(TriShape<E, TB>::THREADS)
    k_tri_inverse(const FieldTab *__restrict__ ftab, const uint64_t *__restrict__ T, int64_t ldt, int64_t pt,
                  int64_t m, int upper, int unit, uint64_t *__restrict__ Tinv, int *__restrict__ bad_row) {
    using S = TriShape<E, TB>;
    using CT = typename S::CT;
    constexpr int NW = S::NW, TPR = S::TPR, PB = S::PB, H1 = S::H1;
    extern __shared__ __align__(16) uint64_t dsm[];
    uint64_t *tab = dsm;                                    // [Q][E][NW]
    uint64_t *pub = tab + S::TW;                            // [NW][E]: the published row X_i
    CT *cU = reinterpret_cast<CT *>(pub + NW * E);          // [TB (step)][TB (row)]
    __shared__ uint16_t sinv[1 << E], smk[(1 << E) * E], sex[1 << E], slg[1 << E], sdlog[TB];
    constexpr int ORD = (1 << E) - 1;  // multiplicative group order
    pdl_trigger();
    for (int i = threadIdx.x; i < (1 << E); i += S::THREADS) {
        sinv[i] = ftab->inv[i];
        sex[i] = ftab->ex[i < ORD ? i : 0];
        slg[i] = ftab->lg[i];
#pragma unroll
        for (int b = 0; b < E; ++b) smk[i * E + b] = ftab->mulmask[i][b];
    }
    pdl_wait();  // T comes from the chain (the field tables above are constant)
    const int64_t r0 = (int64_t)blockIdx.x * TB;
    const int rows = (int)((m - r0) < TB ? (m - r0) : TB);
    const int k = threadIdx.x / TPR, sub = threadIdx.x % TPR;
    const int w = sub % NW, h = sub / NW, b0 = h * PB;
    uint64_t t[E], x[PB];  // word w of every plane of row k of T; my planes of X
#pragma unroll
    for (int b = 0; b < E; ++b) t[b] = 0;
#pragma unroll
    for (int j = 0; j < PB; ++j) x[j] = 0;
    if (k < rows) {
        const uint64_t *src = T + (r0 + k) * ldt + (r0 >> 6);
        if (w < ((rows + 63) >> 6)) {
#pragma unroll
            for (int b = 0; b < E; ++b) t[b] = src[b * pt + w];
        }
        if (h == 0 && (k >> 6) == w) x[0] = 1ULL << (k & 63);  // identity row
    }
    auto entry = [&](int c) {  // T[k][c] for c in this thread's word
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < E; ++b) v |= (uint32_t)((t[b] >> (c & 63)) & 1ULL) << b;
        return v;
    };
    __syncthreads();  // field tables
    uint32_t dk = 1;  // T_kk (thread of the word holding column k)
    if (k < rows && w == (k >> 6)) {
        dk = entry(k);
        if (!unit && dk == 0 && h == 0) atomicMin(bad_row, (int)(r0 + k));
        if (h == 0) sdlog[k] = (unit || dk == 0) ? 0 : slg[dk];
    }
    dk = __shfl_sync(0xffffffffu, dk, ((threadIdx.x & 31) - sub) + (k >> 6) % NW);
    __syncthreads();  // sdlog
    // multipliers: this thread's half (h) of the 64 columns of its word
    {
        constexpr int CPT = 64 / S::BS;
        for (int cc = 0; cc < CPT; ++cc) {
            const int i = w * 64 + h * CPT + cc;
            if (i >= TB) break;
            uint32_t c = 0;
            const bool below = k < rows && i < rows && (upper ? (k < i) : (k > i));
            if (below) {
                c = entry(i);
                if (c && !unit) {  // U_ki = T_ki / T_ii
                    int l = (int)slg[c] - (int)sdlog[i];
                    c = sex[l < 0 ? l + ORD : l];
                }
            }
            cU[i * TB + k] = (CT)c;
        }
    }
    // this thread's table words: entry x, plane b, word wt; its multiplication mask is fixed
    uint32_t tmask[S::NB];
#pragma unroll
    for (int q = 0; q < S::NB; ++q) {
        const int idx = threadIdx.x + q * S::THREADS;
        tmask[q] = 0;
        if (idx < S::TW) {
            const int xq = idx / (E * NW), b = (idx / NW) % E;
            const uint32_t c = xq < (1 << H1) ? (uint32_t)xq : (uint32_t)(xq - (1 << H1)) << H1;
            tmask[q] = smk[c * E + b];
        }
    }
    // one table word per thread (the common case): its plane selection as 64-bit AND masks
    constexpr bool ONE = S::NB == 1;
    uint64_t tsel[ONE ? E : 1];
#pragma unroll
    for (int p = 0; p < (ONE ? E : 1); ++p) tsel[p] = 0ULL - (uint64_t)((tmask[0] >> p) & 1u);
    __syncthreads();  // cU
    for (int step = 0; step < rows; ++step) {
        const int i = upper ? rows - 1 - step : step;
        if (k == i) {  // X_i of U^-1 is final as it stands
#pragma unroll
            for (int j = 0; j < PB; ++j)
                if (b0 + j < E) pub[w * E + b0 + j] = x[j];
        }
        const uint32_t c = cU[i * TB + k];
        __syncthreads();  // X_i published
        if constexpr (ONE) {
            if (threadIdx.x < S::TW) {
                const uint64_t *pv = pub + (threadIdx.x % NW) * E;
                uint64_t acc = 0;
#pragma unroll
                for (int p = 0; p < E; ++p) acc ^= pv[p] & tsel[p];
                tab[threadIdx.x] = acc;
            }
        } else {
#pragma unroll
            for (int q = 0; q < S::NB; ++q) {
                const int idx = threadIdx.x + q * S::THREADS;
                if (idx < S::TW) {
                    const uint64_t *pv = pub + (idx % NW) * E;
                    uint64_t acc = 0;
#pragma unroll
                    for (int p = 0; p < E; ++p) acc ^= pv[p] & (0ULL - (uint64_t)((tmask[q] >> p) & 1u));
                    tab[idx] = acc;
                }
            }
        }
        __syncthreads();  // table built
        {  // entry 0 of both tables is zero: no branch on c
            const uint64_t *lo = tab + (size_t)(c & ((1u << H1) - 1)) * E * NW + w;
            if constexpr (S::H2 > 0) {
                const uint64_t *hi = tab + (size_t)((1u << H1) + (c >> H1)) * E * NW + w;
#pragma unroll
                for (int j = 0; j < PB; ++j)
                    if (b0 + j < E) x[j] ^= lo[(b0 + j) * NW] ^ hi[(b0 + j) * NW];
            } else {
#pragma unroll
                for (int j = 0; j < PB; ++j)
                    if (b0 + j < E) x[j] ^= lo[(b0 + j) * NW];
            }
        }
        // the next step's publish and table build come after its first barrier, which every
        // reader of this step's table has passed
    }
    if (!unit) {  // row k of T^-1 = T_kk^-1 * row k of U^-1 (needs all planes of word w)
        uint64_t full[E];
        if constexpr (S::BS == 1) {
#pragma unroll
            for (int p = 0; p < E; ++p) full[p] = x[p];
        } else {
            uint64_t other[PB];
#pragma unroll
            for (int j = 0; j < PB; ++j) other[j] = __shfl_xor_sync(0xffffffffu, x[j], NW);
#pragma unroll
            for (int p = 0; p < E; ++p)
                full[p] = (p < PB) ? (h == 0 ? x[p % PB] : other[p % PB]) : (h == 0 ? other[p % PB] : x[p % PB]);
        }
        uint32_t c = sinv[dk];
        if (c == 0) c = 1;  // singular block: reported above, result unused
#pragma unroll
        for (int j = 0; j < PB; ++j) {
            if (b0 + j < E) {
                const uint32_t mk = smk[c * E + b0 + j];
                uint64_t acc = 0;
#pragma unroll
                for (int p = 0; p < E; ++p) acc ^= full[p] & (0ULL - (uint64_t)((mk >> p) & 1u));
                x[j] = acc;
            }
        }
    }
    // Tinv block = e planes of TB rows x NW words
    uint64_t *out = Tinv + (int64_t)blockIdx.x * E * TB * NW;
#pragma unroll
    for (int j = 0; j < PB; ++j)
        if (b0 + j < E) out[(int64_t)(b0 + j) * TB * NW + k * NW + w] = (k < rows) ? x[j] : 0;
}

// mat_sliced.py:109-122: slices shift up one degree, the top slice folds into the slices
// selected by the low coefficients of f.  out may alias nothing of in.
__global__ void k_mul_by_x(int e, uint32_t f, const uint64_t *__restrict__ in, int64_t ld, int64_t pin,
                           uint64_t *__restrict__ out, int64_t pout, int64_t rows, int64_t nwords) {
    const int64_t total = rows * nwords;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / nwords, w = idx - r * nwords, off = r * ld + w;
        const uint64_t top = in[(e - 1) * pin + off];
        for (int t = 0; t < e; ++t) {
            uint64_t v = t ? in[(t - 1) * pin + off] : 0;
            if ((f >> t) & 1u) v ^= top;
            out[t * pout + off] = v;
        }
    }
}

// mat_packed.py:192-199: every element multiplied by the scalar c (table of c*a in smem)
__global__ void k_scalar_mul(int e, uint32_t f, uint32_t c, int w, const uint64_t *__restrict__ in, int64_t ldi,
                             uint64_t *__restrict__ out, int64_t ldo, int64_t rows, int64_t nwords) {
    __shared__ uint16_t tab[1024];
    for (int a = threadIdx.x; a < (1 << e); a += blockDim.x) tab[a] = (uint16_t)gf_mul_slow((uint32_t)a, c, e, f);
    __syncthreads();
    const int per = 64 / w;
    const uint64_t emask = (1ULL << e) - 1;
    const int64_t total = rows * nwords;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / nwords, wi = idx - r * nwords;
        const uint64_t x = in[r * ldi + wi];
        uint64_t y = 0;
        for (int s = 0; s < per; ++s) y |= (uint64_t)tab[(x >> (s * w)) & emask] << (s * w);
        out[r * ldo + wi] = y;
    }
}

// Blocked inverse of a 128-row diagonal block (the PLE corners and TRSM at e = 9, 10 / small n):
// instead of one 128-step substitution chain, four 32-row chains run at once (one warp each,
// lane = row, the published row broadcast by shuffles, scalar * row by the multiplication
// matrices) and the off-diagonal 32-row blocks follow from block products by diagonals,
//   lower: X_IJ = X_II * sum_{K=J..I-1} U_IK X_KJ,  upper: X_IJ = X_II * sum_{K=I+1..J} U_IK X_KJ
// (U = T D^-1 unit triangular as in k_tri_inverse; minus is plus in GF(2^e)).  A block product
// C = A * B (32 x 32 elements times 32 bitsliced rows) tabulates the multiples of B's rows
// (split by the scalar's low / high bits, PleSplit) and each row of C adds two words per plane
// and row of B; A's entries come from the multipliers (U blocks) or, for X_II, one ballot over
// the row's plane lanes.  X is kept as 32-bit words per (plane, row, 32-column block).
template <int E, int TB_>
struct TriBlk {
    static constexpr int TB = TB_, BR = 32, NBK = TB / BR, NW = TB / 64;
    static constexpr int THREADS = 512;
    static constexpr int TPR = E <= 8 ? 8 : 16;  // lanes per row in the products
    using SP = PleSplit<E>;
    static constexpr int QE = SP::QE;
    using CT = typename std::conditional<(E <= 8), uint8_t, uint16_t>::type;
    static constexpr size_t SMEM = (size_t)TB * TB * sizeof(CT)       // cU
                                   + (size_t)E * TB * NBK * 4           // Xs
                                   + (size_t)E * BR * 4                 // Ts
                                   + (size_t)BR * QE * 4;               // tables of one product
};

template <int E, int TB_>
__global__ void __launch_bounds__(512) k_tri_inverse_blk(const FieldTab *__restrict__ ftab,
                                                         const uint64_t *__restrict__ T, int64_t ldt, int64_t pt,
                                                         int64_t m, int upper, int unit, uint64_t *__restrict__ Tinv,
                                                         int *__restrict__ bad_row) {
    using B = TriBlk<E, TB_>;
    using SP = typename B::SP;
    using CT = typename B::CT;
    constexpr int TB = B::TB, BR = B::BR, NBK = B::NBK, NW = B::NW, TPR = B::TPR, QE = B::QE, H1 = SP::H1;
    constexpr uint32_t EMASK = (1u << E) - 1;
    extern __shared__ __align__(16) uint8_t bsm[];
    CT *cU = reinterpret_cast<CT *>(bsm);                                           // [i][k]: U_ki
    uint32_t *Xs = reinterpret_cast<uint32_t *>(bsm + (size_t)TB * TB * sizeof(CT));  // [E][TB][NBK]
    uint32_t *Ts = Xs + E * TB * NBK;                                                 // [E][BR]
    uint32_t *tab = Ts + E * BR;                                                      // [BR][Q][E]
    __shared__ uint16_t sinv[1 << E], smk[(1 << E) * E], sex[1 << E], slg[1 << E], sdlog[TB], sdk[TB];
    constexpr int ORD = (1 << E) - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_trigger();
    for (int i = tid; i < (1 << E); i += B::THREADS) {
        sinv[i] = ftab->inv[i];
        sex[i] = ftab->ex[i < ORD ? i : 0];
        slg[i] = ftab->lg[i];
#pragma unroll
        for (int b = 0; b < E; ++b) smk[i * E + b] = ftab->mulmask[i][b];
    }
    for (int i = tid; i < E * TB * NBK; i += B::THREADS) Xs[i] = 0;
    pdl_wait();  // T comes from the chain (the field tables above are constant)
    const int64_t r0 = (int64_t)blockIdx.x * TB;
    const int rows = (int)((m - r0) < TB ? (m - r0) : TB);
    __syncthreads();  // field tables, Xs zeroed
    // multipliers: task (row k, 32-column part c4): its row's plane words, entries by bit
    for (int task = tid; task < TB * NBK; task += B::THREADS) {
        const int k = task / NBK, c4 = task % NBK;
        uint64_t t[E];
#pragma unroll
        for (int b = 0; b < E; ++b) t[b] = 0;
        if (k < rows && c4 * BR < rows) {
            const uint64_t *src = T + (r0 + k) * ldt + (r0 >> 6) + (c4 >> 1);
#pragma unroll
            for (int b = 0; b < E; ++b) t[b] = src[b * pt];
        }
        if (c4 == (k >> 5)) {
            uint32_t dk = 1;
            if (k < rows) {
                dk = 0;
#pragma unroll
                for (int b = 0; b < E; ++b) dk |= (uint32_t)((t[b] >> (k & 63)) & 1ULL) << b;
            }
            if (!unit && k < rows && dk == 0) atomicMin(bad_row, (int)(r0 + k));
            sdlog[k] = (unit || dk == 0) ? 0 : slg[dk];
            sdk[k] = (uint16_t)dk;
        }
    }
    __syncthreads();  // sdlog
    for (int task = tid; task < TB * NBK; task += B::THREADS) {
        const int k = task / NBK, c4 = task % NBK;
        uint64_t t[E];
#pragma unroll
        for (int b = 0; b < E; ++b) t[b] = 0;
        if (k < rows && c4 * BR < rows) {
            const uint64_t *src = T + (r0 + k) * ldt + (r0 >> 6) + (c4 >> 1);
#pragma unroll
            for (int b = 0; b < E; ++b) t[b] = src[b * pt];
        }
        for (int cc = 0; cc < BR; ++cc) {
            const int i = c4 * BR + cc;
            uint32_t c = 0;
            if (k < rows && i < rows && (upper ? (k < i) : (k > i))) {
#pragma unroll
                for (int b = 0; b < E; ++b) c |= (uint32_t)((t[b] >> (i & 63)) & 1ULL) << b;
                if (c && !unit) {  // U_ki = T_ki / T_ii
                    int l = (int)slg[c] - (int)sdlog[i];
                    c = sex[l < 0 ? l + ORD : l];
                }
            }
            cU[i * TB + k] = (CT)c;
        }
    }
    __syncthreads();  // cU
    const int nb = (rows + BR - 1) / BR;  // 32-row blocks in use
    // ---- phase 1: the diagonal blocks, one warp each ----
    if (warp < nb) {
        const int I = warp, kk = I * BR + lane;
        uint32_t x[E];
#pragma unroll
        for (int b = 0; b < E; ++b) x[b] = 0;
        x[0] = 1u << lane;
        for (int s = 0; s < BR; ++s) {
            const int il = upper ? BR - 1 - s : s, i = I * BR + il;
            uint32_t xi[E];
#pragma unroll
            for (int p = 0; p < E; ++p) xi[p] = __shfl_sync(0xffffffffu, x[p], il);
            const uint32_t c = cU[i * TB + kk];  // zero unless row kk is below / above row i
            if (c) {
#pragma unroll
                for (int b = 0; b < E; ++b) {
                    const uint32_t mk = smk[c * E + b];
                    uint32_t acc = 0;
#pragma unroll
                    for (int p = 0; p < E; ++p) acc ^= xi[p] & (0u - ((mk >> p) & 1u));
                    x[b] ^= acc;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < E; ++b) Xs[(b * TB + kk) * NBK + I] = x[b];
    }
    __syncthreads();
    // ---- phase 2: block products by diagonals ----
    // C[r] (+)= sum_q A(r, q) * Brow(q): tables of the 32 rows of B, then lane (r, b) adds two
    // table words per q.  amode 0: A = U block (I, K) from the multipliers; 1: A = X_II.
    const int pr = tid / TPR, pb = tid % TPR, gl = lane - (lane % TPR);
    // B row q, plane p: bsrc[p * bps + q * brs]; C row r, plane p: dst[p * dps + r * drs]
    auto product = [&](int amode, int I, int K, const uint32_t *bsrc, int bps, int brs, uint32_t *dst, int dps,
                       int drs, bool accumulate) {
        // tables: task (row q of B, half h, plane q2)
        constexpr int NH = SP::H2 ? 2 : 1;
        for (int tsk = tid; tsk < BR * NH * E; tsk += B::THREADS) {
            const int q = tsk / (NH * E), rem = tsk - q * (NH * E), h = rem / E, q2 = rem - h * E;
            const int s0 = h ? SP::H1 : 0, hb = h ? SP::H2 : SP::H1;
            uint32_t br[E];
#pragma unroll
            for (int p = 0; p < E; ++p) br[p] = bsrc[p * bps + q * brs];
            const uint32_t m1 = ftab->mulmask2[1][q2];
            uint32_t basis[SP::H1 > SP::H2 ? SP::H1 : SP::H2];
#pragma unroll
            for (int u = 0; u < (SP::H1 > SP::H2 ? SP::H1 : SP::H2); ++u) {
                const uint32_t mk = (m1 >> (s0 + u)) & EMASK;
                uint32_t a = 0;
#pragma unroll
                for (int p = 0; p < E; ++p) a ^= br[p] & (0u - ((mk >> p) & 1u));
                basis[u] = a;
            }
            uint32_t *d = tab + q * QE + (h ? (1 << SP::H1) : 0) * E + q2;
            d[0] = 0;
#pragma unroll
            for (int u = 0; u < (SP::H1 > SP::H2 ? SP::H1 : SP::H2); ++u) {
                if (u >= hb) break;
                for (int t2 = 0; t2 < (1 << u); ++t2) d[((1 << u) + t2) * E] = d[t2 * E] ^ basis[u];
            }
        }
        __syncthreads();
        if (pr < BR) {  // every lane of the row's group takes part in the ballots
            const int r = pr, bb = pb < E ? pb : 0;
            const uint32_t xw = amode ? Xs[(bb * TB + I * BR + r) * NBK + I] : 0;
            uint32_t acc = 0;
            for (int q = 0; q < BR; ++q) {
                uint32_t x;
                if (amode) {
                    const unsigned bal = __ballot_sync(0xffffffffu, pb < E && ((xw >> q) & 1u));
                    x = (bal >> gl) & EMASK;
                } else {
                    x = cU[(K * BR + q) * TB + I * BR + r];
                }
                const uint32_t *tq = tab + q * QE + bb;
                if constexpr (SP::H2 > 0)
                    acc ^= tq[(x & ((1u << H1) - 1)) * E] ^ tq[((1u << H1) + (x >> H1)) * E];
                else
                    acc ^= tq[x * E];
            }
            if (pb < E) {
                uint32_t *o = dst + pb * dps + r * drs;
                *o = accumulate ? (*o ^ acc) : acc;
            }
        }
        __syncthreads();
    };
    for (int d = 1; d < nb; ++d) {
        for (int J0 = 0; J0 + d < nb; ++J0) {
            const int I = upper ? J0 : J0 + d, J = upper ? J0 + d : J0;
            // Ts = sum_K U_IK X_KJ, then X_IJ = X_II Ts
            const int K0 = upper ? I + 1 : J, K1 = upper ? J : I - 1;
            for (int K = K0; K <= K1; ++K)
                product(0, I, K, Xs + (K * BR) * NBK + J, TB * NBK, NBK, Ts, BR, 1, K != K0);
            product(1, I, I, Ts, BR, 1, Xs + (I * BR) * NBK + J, TB * NBK, NBK, false);
        }
    }
    // ---- row scaling (T^-1 = D^-1 U^-1) and output: plane b, row k, two 64-bit words ----
    uint64_t *out = Tinv + (int64_t)blockIdx.x * E * TB * NW;
    for (int idx = tid; idx < E * TB; idx += B::THREADS) {
        const int b = idx / TB, kr = idx - b * TB;
        uint32_t v[NBK];
        if (unit) {
#pragma unroll
            for (int cb = 0; cb < NBK; ++cb) v[cb] = Xs[(b * TB + kr) * NBK + cb];
        } else {
            uint32_t c = sinv[sdk[kr]];
            if (c == 0) c = 1;  // singular block: reported above, result unused
            const uint32_t mk = smk[c * E + b];
#pragma unroll
            for (int cb = 0; cb < NBK; ++cb) {
                uint32_t acc = 0;
#pragma unroll
                for (int p = 0; p < E; ++p) acc ^= Xs[(p * TB + kr) * NBK + cb] & (0u - ((mk >> p) & 1u));
                v[cb] = acc;
            }
        }
        const bool live = kr < rows;
#pragma unroll
        for (int w = 0; w < NW; ++w)
            out[((int64_t)b * TB + kr) * NW + w] = live ? ((uint64_t)v[2 * w] | ((uint64_t)v[2 * w + 1] << 32)) : 0;
    }
}

inline int grid_for(int64_t total, int threads) {
    int64_t g = (total + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

#ifndef GF2E_TRI_BLK
#define GF2E_TRI_BLK 1
#endif
template <int E, int TB>
cudaError_t launch_tri_e(const FieldTab *ftab, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m, bool upper,
                         bool unit, uint64_t *Tinv, int *bad_row, int64_t nblk, cudaStream_t st) {
    if constexpr (GF2E_TRI_BLK) {  // the blocked form (32-row chains + block products)
        using BK = TriBlk<E, TB>;
        static bool attr_blk[kMaxDevices] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev >= kMaxDevices || !attr_blk[dev]) {
            cudaError_t err = cudaFuncSetAttribute(k_tri_inverse_blk<E, TB>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK::SMEM);
            if (err != cudaSuccess) return err;
            if (dev < kMaxDevices) attr_blk[dev] = true;
        }
        return launch_pdl(k_tri_inverse_blk<E, TB>, dim3((unsigned)nblk), dim3(BK::THREADS), BK::SMEM, st, ftab, T, ldt,
                          pt, m, upper ? 1 : 0, unit ? 1 : 0, Tinv, bad_row);
    }
    using S = TriShape<E, TB>;
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr_set[dev]) {
        cudaError_t err = cudaFuncSetAttribute(k_tri_inverse<E, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)S::SMEM);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    return launch_pdl(k_tri_inverse<E, TB>, dim3((unsigned)nblk), dim3(S::THREADS), S::SMEM, st, ftab, T, ldt, pt, m,
                      upper ? 1 : 0, unit ? 1 : 0, Tinv, bad_row);
}

template <int TB>
cudaError_t launch_tri_tb(int e, const FieldTab *ftab, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m,
                          bool upper, bool unit, uint64_t *Tinv, int *bad_row, cudaStream_t st) {
    const int64_t nblk = (m + TB - 1) / TB;
    if (nblk == 0) return cudaSuccess;
    switch (e) {
        case 2: return launch_tri_e<2, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 3: return launch_tri_e<3, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 4: return launch_tri_e<4, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 5: return launch_tri_e<5, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 6: return launch_tri_e<6, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 7: return launch_tri_e<7, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 8: return launch_tri_e<8, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 9:
            if constexpr (TB == 256) return cudaErrorInvalidValue;  // 128-row blocks only (trsm_block)
            else return launch_tri_e<9, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 10:
            if constexpr (TB == 256) return cudaErrorInvalidValue;  // 128-row blocks only (trsm_block)
            else return launch_tri_e<10, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tri_inverse(int e, uint32_t f, uint32_t g, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m,
                               bool upper, bool unit, uint64_t *Tinv, int *bad_row, int block, cudaStream_t st) {
    const FieldTab *ftab = field_tab(e, f, g);
    if (!ftab) return cudaErrorUnknown;
    if (block == 256 && e <= 8) return launch_tri_tb<256>(e, ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, st);
    if (block == 128) return launch_tri_tb<128>(e, ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_mul_by_x(int e, uint32_t f, const uint64_t *in, int64_t ld, int64_t pin, uint64_t *out,
                            int64_t pout, int64_t rows, int64_t nwords, cudaStream_t st) {
    const int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_mul_by_x<<<grid_for(total, 256), 256, 0, st>>>(e, f, in, ld, pin, out, pout, rows, nwords);
    return cudaGetLastError();
}

// out row r = c_r * (in row r, or in row 0 when broadcast) on packed words: the NJ multiple
// table (newton_john.py:55-88) is broadcast row x scalars 0 .. 2^e - 1.  Products via exp/log
// tables of the field (ple.cu: field_tab).
__global__ void k_row_scales(int e, const FieldTab *__restrict__ ftab, int w, const uint64_t *__restrict__ in,
                             int64_t ldi, int bcast, const uint32_t *__restrict__ cs, uint64_t *__restrict__ out,
                             int64_t ldo, int64_t rows, int64_t nwords) {
    __shared__ uint16_t ex[1024], lg[1024];
    const int q1 = (1 << e) - 1;
    for (int i = threadIdx.x; i <= q1; i += blockDim.x) {
        ex[i] = ftab->ex[i];
        lg[i] = ftab->lg[i];
    }
    __syncthreads();
    const int per = 64 / w;
    const uint64_t emask = (1ULL << e) - 1;
    const int64_t total = rows * nwords;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / nwords, wi = idx - r * nwords;
        const uint64_t x = in[(bcast ? 0 : r) * ldi + wi];
        const uint32_t c = cs[r];
        uint64_t y = 0;
        if (c)
            for (int sl = 0; sl < per; ++sl) {
                const uint32_t a = (uint32_t)((x >> (sl * w)) & emask);
                if (a) {
                    int l = lg[a] + lg[c];
                    if (l >= q1) l -= q1;
                    y |= (uint64_t)ex[l] << (sl * w);
                }
            }
        out[r * ldo + wi] = y;
    }
}

cudaError_t launch_scalar_mul(int e, uint32_t f, uint32_t c, int w, const uint64_t *in, int64_t ldi, uint64_t *out,
                              int64_t ldo, int64_t rows, int64_t nwords, cudaStream_t st) {
    const int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_scalar_mul<<<grid_for(total, 256), 256, 0, st>>>(e, f, c, w, in, ldi, out, ldo, rows, nwords);
    return cudaGetLastError();
}

cudaError_t launch_row_scales(int e, uint32_t f, uint32_t g, int w, const uint64_t *in, int64_t ldi, bool bcast,
                              const uint32_t *cs, uint64_t *out, int64_t ldo, int64_t rows, int64_t nwords,
                              cudaStream_t st) {
    const FieldTab *ftab = field_tab(e, f, g);
    if (!ftab) return cudaErrorUnknown;
    const int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_row_scales<<<grid_for(total, 256), 256, 0, st>>>(e, ftab, w, in, ldi, bcast ? 1 : 0, cs, out, ldo, rows, nwords);
    return cudaGetLastError();
}

}  // namespace gf2e

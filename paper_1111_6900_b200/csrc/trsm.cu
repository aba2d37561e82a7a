// trsm.cu — device kernels for the first consumers of the hot path:
//   * k_tri_inverse: inverse of each 128-row diagonal block of a triangular GF(2^e) matrix
//     held as bit planes (the base case of the blocked TRSM in capi.cu, whose off-diagonal
//     updates are all addmul calls into the tensor-core product kernel);
//   * k_mul_by_x: sliced multiplication by alpha (mat_sliced.py:109-122);
//   * k_scalar_mul: packed multiplication by a scalar (mat_packed.py:192-199).
// Field arithmetic uses the per-field tables of ple.cu (field_tab: inverses, multiplication
// matrices; the scalar kernels build their own small tables).
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


// Inverse of each 128 x 128 diagonal block by bitsliced substitution: thread k owns row k of
// the block and of its inverse X (two words per plane each, in registers).  Lower triangular:
// for i = 0 .. rows-1, thread i finalises X_i = T_ii^-1 X_i and publishes it; every thread
// k > i then adds T_ki * X_i (T's own entries are the multipliers: X_k = T_kk^-1 (e_k -
// sum_{i<k} T_ki X_i)).  Upper: the same from the bottom.  Scalar * bitsliced word uses the
// field's multiplication matrices (FieldTab.mulmask: plane b of c*v = XOR of the planes in
// mulmask[c][b]).
template <int E, int TB>  // TB = diagonal block rows = threads
__global__ void __launch_bounds__(TB) k_tri_inverse(const FieldTab *__restrict__ ftab, const uint64_t *__restrict__ T,
                                                   int64_t ldt, int64_t pt, int64_t m, int upper, int unit,
                                                   uint64_t *__restrict__ Tinv, int *__restrict__ bad_row) {
    constexpr int NW = TB / 64;           // plane words per block row
    __shared__ uint64_t pub[2][NW][E];    // the published row X_i, double-buffered by step parity
    __shared__ uint16_t sinv[1 << E], smk[(1 << E) * E], sex[1 << E], slg[1 << E], sdlog[TB];
    constexpr int ORD = (1 << E) - 1;     // multiplicative group order
    for (int i = threadIdx.x; i < (1 << E); i += TB) {
        sinv[i] = ftab->inv[i];
        sex[i] = ftab->ex[i < ORD ? i : 0];
        slg[i] = ftab->lg[i];
#pragma unroll
        for (int b = 0; b < E; ++b) smk[i * E + b] = ftab->mulmask[i][b];
    }
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * TB;
    const int rows = (int)((m - r0) < TB ? (m - r0) : TB);
    const int k = threadIdx.x;
    uint64_t t[E][NW], x[E][NW];
#pragma unroll
    for (int b = 0; b < E; ++b)
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            t[b][w] = 0;
            x[b][w] = 0;
        }
    if (k < rows) {
        const uint64_t *src = T + (r0 + k) * ldt + (r0 >> 6);
        const int nw = (rows + 63) >> 6;
#pragma unroll
        for (int b = 0; b < E; ++b)
#pragma unroll
            for (int w = 0; w < NW; ++w)
                if (w < nw) t[b][w] = src[b * pt + w];
#pragma unroll
        for (int w = 0; w < NW; ++w) x[0][w] = ((k >> 6) == w) ? (1ULL << (k & 63)) : 0ULL;  // identity row
    }
    auto entry = [&](int c) {  // T[k][c] as a field element
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < E; ++b) {
            uint64_t wv = t[b][0];
#pragma unroll
            for (int w = 1; w < NW; ++w)
                if ((c >> 6) == w) wv = t[b][w];
            v |= (uint32_t)((wv >> (c & 63)) & 1ULL) << b;
        }
        return v;
    };
    // T = U D with D = diag(T) and U = T D^-1 unit triangular, so T^-1 = D^-1 U^-1: the
    // substitution runs on U (multipliers T_ki / T_ii, from the log tables) with no scaling on
    // the per-row critical path, and each thread scales its own row of the result at the end.
    const uint32_t dk = k < rows ? entry(k) : 1u;
    if (!unit && k < rows && dk == 0) atomicMin(bad_row, (int)(r0 + k));
    sdlog[k] = (unit || dk == 0) ? 0 : slg[dk];
    __syncthreads();
    for (int step = 0; step < rows; ++step) {
        const int i = upper ? rows - 1 - step : step;
        if (k == i) {  // X_i of U^-1 is final as it stands
#pragma unroll
            for (int w = 0; w < NW; ++w)
#pragma unroll
                for (int b = 0; b < E; ++b) pub[step & 1][w][b] = x[b][w];
        }
        // one barrier per row: pub[step & 1] is rewritten two steps later, after every reader
        // of this step has passed the next step's barrier
        __syncthreads();
        const bool below = upper ? (k < i) : (k > i && k < rows);
        if (below) {
            uint32_t c = entry(i);
            if (c && !unit) {  // U_ki = T_ki / T_ii
                int l = (int)slg[c] - (int)sdlog[i];
                c = sex[l < 0 ? l + ORD : l];
            }
            if (c) {
#pragma unroll
                for (int b = 0; b < E; ++b) {
                    const uint32_t mk = smk[c * E + b];
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        uint64_t acc = 0;
#pragma unroll
                        for (int p = 0; p < E; ++p) acc ^= pub[step & 1][w][p] & (0ULL - (uint64_t)((mk >> p) & 1u));
                        x[b][w] ^= acc;
                    }
                }
            }
        }
    }
    if (!unit && k < rows) {  // row k of T^-1 = T_kk^-1 * row k of U^-1
        uint32_t c = sinv[dk];
        if (c == 0) c = 1;  // singular block: reported above, result unused
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            uint64_t y[E];
#pragma unroll
            for (int b = 0; b < E; ++b) {
                const uint32_t mk = smk[c * E + b];
                uint64_t acc = 0;
#pragma unroll
                for (int p = 0; p < E; ++p) acc ^= x[p][w] & (0ULL - (uint64_t)((mk >> p) & 1u));
                y[b] = acc;
            }
#pragma unroll
            for (int b = 0; b < E; ++b) x[b][w] = y[b];
        }
    }
    // Tinv block = e planes of TB rows x NW words
    uint64_t *out = Tinv + (int64_t)blockIdx.x * E * TB * NW;
#pragma unroll
    for (int b = 0; b < E; ++b)
#pragma unroll
        for (int w = 0; w < NW; ++w) out[(int64_t)b * TB * NW + k * NW + w] = (k < rows) ? x[b][w] : 0;
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

inline int grid_for(int64_t total, int threads) {
    int64_t g = (total + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

template <int E, int TB>
cudaError_t launch_tri_e(const FieldTab *ftab, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m, bool upper,
                         bool unit, uint64_t *Tinv, int *bad_row, int64_t nblk, cudaStream_t st) {
    k_tri_inverse<E, TB><<<(unsigned)nblk, TB, 0, st>>>(ftab, T, ldt, pt, m, upper ? 1 : 0, unit ? 1 : 0, Tinv,
                                                        bad_row);
    return cudaGetLastError();
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
        case 9: return launch_tri_e<9, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        case 10: return launch_tri_e<10, TB>(ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, nblk, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tri_inverse(int e, uint32_t f, uint32_t g, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m,
                               bool upper, bool unit, uint64_t *Tinv, int *bad_row, int block, cudaStream_t st) {
    const FieldTab *ftab = field_tab(e, f, g);
    if (!ftab) return cudaErrorUnknown;
    if (block == 256) return launch_tri_tb<256>(e, ftab, T, ldt, pt, m, upper, unit, Tinv, bad_row, st);
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

// trsm.cu — device kernels for the first consumers of the hot path:
//   * k_tri_inverse: inverse of each 128-row diagonal block of a triangular GF(2^e) matrix
//     held as bit planes (the base case of the blocked TRSM in capi.cu, whose off-diagonal
//     updates are all addmul calls into the tensor-core product kernel);
//   * k_mul_by_x: sliced multiplication by alpha (mat_sliced.py:109-122);
//   * k_scalar_mul: packed multiplication by a scalar (mat_packed.py:192-199).
// Field arithmetic uses exp/log tables over a primitive element g, built in shared memory.
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

struct Tables {
    uint16_t ex[1024];
    uint16_t lg[1024];
};

__device__ void build_tables(Tables &t, int e, uint32_t f, uint32_t g) {
    if (threadIdx.x == 0) {
        const int q1 = (1 << e) - 1;
        uint32_t v = 1;
        for (int i = 0; i < q1; ++i) {
            t.ex[i] = (uint16_t)v;
            t.lg[v] = (uint16_t)i;
            v = gf_mul_slow(v, g, e, f);
        }
        t.lg[0] = 0;
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t gmul(const Tables &t, uint32_t a, uint32_t b, int q1) {
    if (a == 0 || b == 0) return 0;
    uint32_t s = (uint32_t)t.lg[a] + t.lg[b];
    if (s >= (uint32_t)q1) s -= q1;
    return t.ex[s];
}
__device__ __forceinline__ uint32_t ginv(const Tables &t, uint32_t a, int q1) {
    uint32_t l = t.lg[a];
    return t.ex[l == 0 ? 0 : q1 - l];
}

constexpr int TB = kTrsmBlock;  // 128

// grid = number of diagonal blocks; 128 threads (thread j owns column j of the inverse)
__global__ void __launch_bounds__(TB) k_tri_inverse(int e, uint32_t f, uint32_t g, const uint64_t *__restrict__ T,
                                                   int64_t ldt, int64_t pt, int64_t m, int upper, int unit,
                                                   uint64_t *__restrict__ Tinv, int *__restrict__ bad_row) {
    extern __shared__ __align__(16) uint8_t smem[];
    Tables &tab = *reinterpret_cast<Tables *>(smem);
    uint16_t *tb = reinterpret_cast<uint16_t *>(smem + sizeof(Tables));  // TB x TB elements of the block
    uint16_t *xs = tb + TB * TB;                                          // TB x TB inverse
    const int q1 = (1 << e) - 1;
    const int64_t r0 = (int64_t)blockIdx.x * TB;
    const int rows = (int)((m - r0) < TB ? (m - r0) : TB);
    build_tables(tab, e, f, g);
    // gather the block's elements from the planes (r0 is a multiple of 128: word aligned)
    for (int idx = threadIdx.x; idx < TB * TB; idx += TB) {
        const int i = idx / TB, j = idx % TB;
        uint32_t v = 0;
        if (i < rows && j < rows) {
            const uint64_t *w = T + (r0 + i) * ldt + (r0 >> 6) + (j >> 6);
            for (int b = 0; b < e; ++b) v |= (uint32_t)((w[b * pt] >> (j & 63)) & 1ULL) << b;
        }
        tb[idx] = (uint16_t)v;
        xs[idx] = 0;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (!unit && j < rows && tb[j * TB + j] == 0) atomicMin(bad_row, (int)(r0 + j));
    if (j < rows) {
        if (upper) {
            for (int i = j; i >= 0; --i) {  // column j of U^-1: rows j .. 0
                uint32_t s = (i == j) ? 1u : 0u;
                for (int k = i + 1; k <= j; ++k) s ^= gmul(tab, tb[i * TB + k], xs[k * TB + j], q1);
                const uint32_t d = tb[i * TB + i];
                xs[i * TB + j] = (uint16_t)(unit ? s : (d ? gmul(tab, s, ginv(tab, d, q1), q1) : 0));
            }
        } else {
            for (int i = j; i < rows; ++i) {  // column j of L^-1: rows j .. rows-1
                uint32_t s = (i == j) ? 1u : 0u;
                for (int k = j; k < i; ++k) s ^= gmul(tab, tb[i * TB + k], xs[k * TB + j], q1);
                const uint32_t d = tb[i * TB + i];
                xs[i * TB + j] = (uint16_t)(unit ? s : (d ? gmul(tab, s, ginv(tab, d, q1), q1) : 0));
            }
        }
    }
    __syncthreads();
    // scatter into planes: Tinv block = e planes of TB rows x TB/64 words
    uint64_t *out = Tinv + (int64_t)blockIdx.x * e * TB * (TB / 64);
    for (int task = threadIdx.x; task < e * TB * (TB / 64); task += TB) {
        const int b = task / (TB * (TB / 64)), rem = task % (TB * (TB / 64));
        const int i = rem / (TB / 64), wq = rem % (TB / 64);
        uint64_t word = 0;
        for (int c = 0; c < 64; ++c) word |= (uint64_t)((xs[i * TB + wq * 64 + c] >> b) & 1u) << c;
        out[(int64_t)b * TB * (TB / 64) + i * (TB / 64) + wq] = word;
    }
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

size_t tri_inverse_smem() { return sizeof(Tables) + 2 * TB * TB * sizeof(uint16_t); }

cudaError_t launch_tri_inverse(int e, uint32_t f, uint32_t g, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m,
                               bool upper, bool unit, uint64_t *Tinv, int *bad_row, cudaStream_t st) {
    const int64_t nblk = (m + TB - 1) / TB;
    if (nblk == 0) return cudaSuccess;
    const size_t sm = tri_inverse_smem();
    cudaError_t err = cudaFuncSetAttribute(k_tri_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    k_tri_inverse<<<(unsigned)nblk, TB, sm, st>>>(e, f, g, T, ldt, pt, m, upper ? 1 : 0, unit ? 1 : 0, Tinv, bad_row);
    return cudaGetLastError();
}

cudaError_t launch_mul_by_x(int e, uint32_t f, const uint64_t *in, int64_t ld, int64_t pin, uint64_t *out,
                            int64_t pout, int64_t rows, int64_t nwords, cudaStream_t st) {
    const int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_mul_by_x<<<grid_for(total, 256), 256, 0, st>>>(e, f, in, ld, pin, out, pout, rows, nwords);
    return cudaGetLastError();
}

cudaError_t launch_scalar_mul(int e, uint32_t f, uint32_t c, int w, const uint64_t *in, int64_t ldi, uint64_t *out,
                              int64_t ldo, int64_t rows, int64_t nwords, cudaStream_t st) {
    const int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_scalar_mul<<<grid_for(total, 256), 256, 0, st>>>(e, f, c, w, in, ldi, out, ldo, rows, nwords);
    return cudaGetLastError();
}

}  // namespace gf2e

// product_m4rm.cu — the integer-pipe form of K4: "Method of Four Russians" Gray tables in
// shared memory (reference: _mul_m4rm mat_gf2.py:348-366 with the table of
// _subset_xor_table_batched 301-310, k = 8 per tuning.py:15), fused with the Karatsuba
// fold of poly_mul.py:187-219 / 223-242.
//
// CTA tile: 512 rows x 1024 columns of C, 512 threads (16 warps).  For every group of 8
// inner indices the CTA builds the 256-entry table T[x] = XOR of the B rows selected by x
// (256 x 128 B = 32 KiB, double buffered), then each row of A picks its 1024-bit
// contribution with one LDS.128 per lane (a quarter-warp reads one 128-byte table row,
// conflict-free) and 4 LOP3.  One product's C tile lives in registers (32 words/thread);
// it is folded into the E output planes in global memory (the CTA owns the tile, so the
// read-modify-write needs no atomics).  C must be zeroed / hold C0 before the launch.
#include "common.cuh"
#include "kernels.h"

namespace gf2e {
namespace {

constexpr int BM = 512, BN = 1024;
constexpr int NT = 512;
constexpr int TABLE_BYTES = 256 * (BN / 8);  // 32 KiB
constexpr int SMEM_BYTES = 2 * TABLE_BYTES;

__global__ void __launch_bounds__(NT, 1) k_product_m4rm(const Sched s, const M4rmArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t tiles_n = a.n_pad / BN;
    const int64_t m0 = (int64_t)(blockIdx.x / tiles_n) * BM;
    const int64_t n0 = (int64_t)(blockIdx.x % tiles_n) * BN;
    const int nchunks = (int)(a.k_pad / 64);

    // table build role: word w (of 32 per table row) for entries [16*g, 16*g + 16)
    const int bw = tid & 31, bg = tid >> 5;  // bg in 0..15
    // lookup role: rows warp*32 + 4*i + (lane>>3), 16-byte column chunk (lane & 7)
    const int lrow0 = warp * 32 + (lane >> 3);
    const int lchunk = lane & 7;

    const int64_t nw = words_for(a.n);
    const int64_t w0 = n0 >> 6;

    for (int t = 0; t < s.nprod; ++t) {
        const uint64_t *Ap = a.Ac + t * a.a_pstride;
        const uint32_t *Bp = reinterpret_cast<const uint32_t *>(a.Bc + t * a.b_pstride);
        uint4 c[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = make_uint4(0, 0, 0, 0);
        int buf = 0;
        // A words of this thread's 8 rows for chunk kc; the next chunk's are fetched one chunk
        // ahead (the lookups stalled on these loads: 40% of the warp samples, profiles/r02)
        uint64_t aw[8], an[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) an[i] = nchunks ? __ldg(Ap + (m0 + lrow0 + 4 * i) * a.kwords) : 0;
        for (int kc = 0; kc < nchunks; ++kc) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                aw[i] = an[i];
                if (kc + 1 < nchunks) an[i] = __ldg(Ap + (m0 + lrow0 + 4 * i) * a.kwords + kc + 1);
            }
#pragma unroll 1
            for (int g = 0; g < 8; ++g) {
                // ---- build T[x] for x in [16*bg, 16*bg+16), word bw ----
                const int64_t krow = (int64_t)kc * 64 + g * 8;
                uint32_t r[8];
#pragma unroll
                for (int b = 0; b < 8; ++b) r[b] = __ldg(Bp + (krow + b) * (a.nwords_pad * 2) + (n0 >> 5) + bw);
                uint32_t base = 0;
#pragma unroll
                for (int b = 4; b < 8; ++b) base ^= r[b] & (0u - ((bg >> (b - 4)) & 1u));
                uint32_t *T = reinterpret_cast<uint32_t *>(smem + buf * TABLE_BYTES);
                // Gray walk over the low 4 bits: 15 XORs (mat_gf2.py:283-298 ordering)
                uint32_t cur = base;
                T[(16 * bg) * 32 + bw] = cur;
#pragma unroll
                for (int x = 1; x < 16; ++x) {
                    const int gcode = x ^ (x >> 1);
                    // the bit that flips between gray(x-1) and gray(x) is ctz(x); written so it
                    // folds to a constant after unrolling (a runtime index sent r[] to local memory)
                    const int bit = (x & 1) ? 0 : (x & 2) ? 1 : (x & 4) ? 2 : 3;
                    cur ^= r[bit];
                    T[(16 * bg + gcode) * 32 + bw] = cur;
                }
                __syncthreads();
                // ---- lookups ----
                const uint8_t *Tb = smem + buf * TABLE_BYTES + lchunk * 16;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t idx = (uint32_t)(aw[i] >> (8 * g)) & 0xFFu;
                    const uint4 v = *reinterpret_cast<const uint4 *>(Tb + idx * 128);
                    c[i].x ^= v.x;
                    c[i].y ^= v.y;
                    c[i].z ^= v.z;
                    c[i].w ^= v.w;
                }
                buf ^= 1;
            }
        }
        // ---- fold this product into the output planes it belongs to ----
        const uint32_t mask = s.outmask[t];
        for (int j = 0; j < s.nout; ++j) {
            if (!((mask >> j) & 1u)) continue;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t row = m0 + lrow0 + 4 * i;
                const int64_t gw = w0 + lchunk * 2;  // two 64-bit words per 16-byte chunk
                if (row < a.m) {
                    uint64_t *crow = a.C + j * a.c_pstride + row * a.ldc;
                    if (gw < nw) crow[gw] ^= (uint64_t)c[i].x | ((uint64_t)c[i].y << 32);
                    if (gw + 1 < nw) crow[gw + 1] ^= (uint64_t)c[i].z | ((uint64_t)c[i].w << 32);
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch_product_m4rm(const Sched &s, const M4rmArgs &a, cudaStream_t st) {
    cudaError_t err = cudaFuncSetAttribute(k_product_m4rm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (err != cudaSuccess) return err;
    const int64_t tiles = (a.m_pad / BM) * (a.n_pad / BN);
    if (tiles == 0) return cudaSuccess;
    k_product_m4rm<<<(unsigned)tiles, NT, SMEM_BYTES, st>>>(s, a);
    return cudaGetLastError();
}

}  // namespace gf2e

// nj.cu — the packed-domain Newton-John product for small blocks:
// nj_mul (newton_john.py:145-164) on packed words, C (^)= A * B with no slicing.
//
// The reference builds, for every row i of B, the table of all 2^e scalar multiples x * B_i
// (_table_block, newton_john.py:91-112: e scalings by alpha and a doubling walk), then adds
// table_i[A[j, i]] into row j of C for every (j, i).  Here one CTA owns 64 rows of C; it walks
// the rows of B in groups of G, builds the G tables in shared memory (entry x = XOR of the
// alpha^s * B_i selected by the bits of x; alpha-multiples by a SWAR xtime on the packed
// words) and every thread XORs the looked-up words of its (row, word) pairs into registers.
// One launch replaces slice A, slice B, two operand-combination launches, the product and
// the cling of the sliced path; the host routes small products here (poly_mul.NJ_CROSSOVER,
// measured, profiles/r02).
#include "common.cuh"
#include "kernels.h"

namespace gf2e {
namespace {

constexpr int NJ_THREADS = 256;
constexpr int NJ_ROWS = 64;                         // C rows per CTA
constexpr int NJ_ACC = NJ_ROWS * kNjMaxWords / NJ_THREADS;  // accumulator words per thread
constexpr int NJ_SMEM = 160 * 1024;

// x * alpha on every e-bit slot of a packed word (slot width w): shift inside the slot, fold
// the carried-out bit with the low bits of f
__device__ __forceinline__ uint64_t xtime_packed(uint64_t x, uint64_t low_mask, uint64_t lsb, int e, uint64_t fl) {
    const uint64_t hi = (x >> (e - 1)) & lsb;
    return ((x & low_mask) << 1) ^ (hi * fl);
}

// Tables per row of B: one of all 2^e multiples for e <= 4; for larger e two half tables
// (multiples by the low h1 bits and by the high e - h1 bits of the scalar, x*B = T_lo[x_lo] ^
// T_hi[x_hi]), 2^h1 + 2^h2 entries instead of 2^e, one more lookup per element.
template <int E>
struct NjTab {
    static constexpr bool SPLIT = E >= 5;
    static constexpr int H1 = SPLIT ? E / 2 : E, H2 = SPLIT ? E - E / 2 : 0;
    static constexpr int ENTRIES = (1 << H1) + (SPLIT ? (1 << H2) : 0);
};

template <int E>
__global__ void __launch_bounds__(NJ_THREADS) k_nj_mul(uint32_t f, int w, const uint64_t *__restrict__ A,
                                                        int64_t lda, const uint64_t *__restrict__ B, int64_t ldb,
                                                        uint64_t *__restrict__ C, int64_t ldc, int64_t m, int64_t k,
                                                        int64_t n, int acc, int G) {
    extern __shared__ __align__(16) uint64_t sm[];
    using T = NjTab<E>;
    constexpr int Q = T::ENTRIES;  // table entries per row of B
    const int WB = (int)words_for(n * w);
    uint64_t *mult = sm;                      // [G][E][WB]: alpha^s * B_i
    uint64_t *tab = sm + (size_t)G * E * WB;  // [G][Q][WB]: x * B_i
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * NJ_ROWS;
    const int rows = (int)(m - r0 < NJ_ROWS ? m - r0 : NJ_ROWS);
    // packed-slot masks of the field elements
    uint64_t emask = 0, low = 0, lsb = 0;
    for (int s = 0; s < 64 / w; ++s) {
        emask |= (uint64_t)((1u << E) - 1) << (s * w);
        low |= (uint64_t)((1u << (E - 1)) - 1) << (s * w);
        lsb |= 1ULL << (s * w);
    }
    const uint64_t fl = f & ((1u << E) - 1);
    uint64_t accw[NJ_ACC];
#pragma unroll
    for (int a = 0; a < NJ_ACC; ++a) accw[a] = 0;
    const int per = NJ_ROWS * WB;  // (row, word) pairs of the CTA
    for (int64_t i0 = 0; i0 < k; i0 += G) {
        const int g = (int)(k - i0 < G ? k - i0 : G);
        // alpha-multiples of the group's rows of B
        for (int idx = tid; idx < g * WB; idx += NJ_THREADS) {
            const int gg = idx / WB, wd = idx - gg * WB;
            uint64_t x = B[(i0 + gg) * ldb + wd] & emask;
            for (int s = 0; s < E; ++s) {
                mult[(gg * E + s) * WB + wd] = x;
                x = xtime_packed(x, low, lsb, E, fl);
            }
        }
        __syncthreads();
        // tables: entry x of row gg = XOR of alpha^s * B_i over the set bits s of x (low table:
        // s < H1; high table at entries 2^H1 .., scalar bits H1 ..)
        for (int idx = tid; idx < g * Q * WB; idx += NJ_THREADS) {
            const int gg = idx / (Q * WB), rem = idx - gg * (Q * WB), x = rem / WB, wd = rem - x * WB;
            const bool hi = x >= (1 << T::H1);
            const int xs = hi ? x - (1 << T::H1) : x, s0 = hi ? T::H1 : 0;
            uint64_t v = 0;
#pragma unroll
            for (int s = 0; s < (T::H1 > T::H2 ? T::H1 : T::H2); ++s)
                if ((xs >> s) & 1) v ^= mult[(gg * E + s0 + s) * WB + wd];
            tab[idx] = v;
        }
        __syncthreads();
        // lookups: row j of C ^= table_i[A[j, i]] for the group's i
#pragma unroll
        for (int a = 0; a < NJ_ACC; ++a) {
            const int idx = tid + a * NJ_THREADS;
            if (idx < per) {
                const int j = idx / WB, wd = idx - j * WB;
                if (j < rows) {
                    const uint64_t *arow = A + (r0 + j) * lda;
                    uint64_t v = 0;
                    for (int gg = 0; gg < g; ++gg) {
                        const int64_t bit = (i0 + gg) * w;
                        const uint32_t x = (uint32_t)((arow[bit >> 6] >> (bit & 63)) & ((1u << E) - 1));
                        const uint64_t *tg = tab + (size_t)gg * Q * WB + wd;
                        if constexpr (T::SPLIT)
                            v ^= tg[(x & ((1u << T::H1) - 1)) * WB] ^ tg[((1u << T::H1) + (x >> T::H1)) * WB];
                        else
                            v ^= tg[x * WB];
                    }
                    accw[a] ^= v;
                }
            }
        }
        __syncthreads();  // the next group overwrites the tables
    }
#pragma unroll
    for (int a = 0; a < NJ_ACC; ++a) {
        const int idx = tid + a * NJ_THREADS;
        if (idx < per) {
            const int j = idx / WB, wd = idx - j * WB;
            if (j < rows) {
                uint64_t *c = C + (r0 + j) * ldc + wd;
                *c = acc ? (*c ^ accw[a]) : accw[a];
            }
        }
    }
}

template <int E>
cudaError_t launch_nj_e(uint32_t f, int w, const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                        uint64_t *C, int64_t ldc, int64_t m, int64_t k, int64_t n, bool acc, cudaStream_t st) {
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr_set[dev]) {
        cudaError_t err = cudaFuncSetAttribute(k_nj_mul<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, NJ_SMEM);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    const int WB = (int)words_for(n * w);
    const size_t per_row = ((size_t)NjTab<E>::ENTRIES + E) * WB * 8;  // tables + multiples of one row of B
    int G = (int)(NJ_SMEM / per_row);
    if (G > 16) G = 16;
    if (G < 1) return cudaErrorInvalidValue;
    const size_t smem = per_row * G;
    const unsigned grid = (unsigned)((m + NJ_ROWS - 1) / NJ_ROWS);
    k_nj_mul<E><<<grid, NJ_THREADS, smem, st>>>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc ? 1 : 0, G);
    return cudaGetLastError();
}

// ---- the same algorithm on bit planes (sliced operands): small updates of PLE and TRSM ----
// C (^)= A * B with A m x k, B k x n, C m x n as e bit planes.  CTA (column word w, row block):
// for each chunk of KC rows of B, the tables of multiples of those rows' word w (split by the
// low H1 / high H2 bits of the scalar, PleSplit) are built in shared memory from the
// multiplication matrices; row r of C is held by TPR lanes (lane b: plane b), the entry
// A[r][i] is one ballot of the lanes' plane bits and the update is two table words per plane.
// All tables of a CTA are built before it writes C, so with one row block per column word
// (nblk_rows == 1) C may alias B (TRSM leaves: X = inv(T) B over B).
template <int E>
struct NjsShape {
    static constexpr int THREADS = 512;
    static constexpr int TPR = E <= 8 ? 8 : 16;
    static constexpr int RPC = THREADS / TPR;  // rows per pass
    static constexpr int KC = 32;              // rows of B per table chunk
    static constexpr int MAXPASS = 4;
    static constexpr size_t SMEM = (size_t)KC * PleSplit<E>::QE * 8 + (size_t)KC * E * 8;
};

template <int E>
__global__ void __launch_bounds__(512, 1) k_nj_sliced(const FieldTab *__restrict__ ftab, const uint64_t *__restrict__ A,
                                                   int64_t lda, int64_t pa, const uint64_t *B, int64_t ldb,
                                                   int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m,
                                                   int64_t k, int64_t n, int acc, int npass) {
    using Sh = NjsShape<E>;
    using SP = PleSplit<E>;
    constexpr int TPR = Sh::TPR, KC = Sh::KC, QE = SP::QE, NH = SP::H2 ? 2 : 1;
    constexpr uint32_t EMASK = (1u << E) - 1;
    extern __shared__ __align__(16) uint64_t nsm[];
    uint64_t *tab = nsm;                   // [KC][Q][E]
    uint64_t *bs = tab + KC * QE;          // [KC][E]: the chunk's rows of B, word w
    pdl_trigger();
    pdl_wait();  // A, B, C come from the chain
    const int tid = threadIdx.x, lane = tid & 31, b = tid % TPR, gl = lane - b, rl = tid / TPR;
    const int64_t w = blockIdx.x;
    const int64_t row0 = (int64_t)blockIdx.y * Sh::RPC * npass;
    uint64_t v[Sh::MAXPASS];
#pragma unroll
    for (int q = 0; q < Sh::MAXPASS; ++q) v[q] = 0;
    for (int64_t i0 = 0; i0 < k; i0 += KC) {
        const int kc = (int)(k - i0 < KC ? k - i0 : KC);
        // this chunk's A words, loaded before the tables are built (their latency overlaps)
        uint64_t aw[Sh::MAXPASS];
#pragma unroll
        for (int q = 0; q < Sh::MAXPASS; ++q) {
            const int64_t r = row0 + q * Sh::RPC + rl;
            aw[q] = (q < npass && r < m && b < E) ? A[b * pa + r * lda + (i0 >> 6)] : 0;
        }
        __syncthreads();  // the previous chunk's tables are consumed
        for (int i = tid; i < kc * E; i += Sh::THREADS) bs[i] = B[(i % E) * pb + (i0 + i / E) * ldb + w];
        __syncthreads();
        // tables: thread (row i of the chunk, half h, plane q) forms plane q of the half's basis
        // alpha^s * B_i (s in the half; mulmask of x^s = mulmask2[1] >> s), then the half's
        // entries by doubling, one XOR each
        for (int t = tid; t < kc * NH * E; t += Sh::THREADS) {
            const int i = t / (NH * E), rem = t - i * (NH * E), h = rem / E, q = rem - h * E;
            const int s0 = h ? SP::H1 : 0, hb = h ? SP::H2 : SP::H1;
            uint64_t br[E];
#pragma unroll
            for (int p = 0; p < E; ++p) br[p] = bs[i * E + p];
            const uint32_t m1 = ftab->mulmask2[1][q];
            uint64_t basis[SP::H1 > SP::H2 ? SP::H1 : SP::H2];
#pragma unroll
            for (int u = 0; u < (SP::H1 > SP::H2 ? SP::H1 : SP::H2); ++u) {
                const uint32_t mk = (m1 >> (s0 + u)) & EMASK;
                uint64_t a = 0;
#pragma unroll
                for (int p = 0; p < E; ++p)
                    if ((mk >> p) & 1u) a ^= br[p];
                basis[u] = a;
            }
            // doubling: entry 2^u + t = entry t ^ basis[u] (this thread's own earlier stores)
            uint64_t *dst = tab + i * QE + (h ? (1 << SP::H1) : 0) * E + q;
            dst[0] = 0;
#pragma unroll
            for (int u = 0; u < (SP::H1 > SP::H2 ? SP::H1 : SP::H2); ++u) {
                if (u >= hb) break;
                for (int t = 0; t < (1 << u); ++t) dst[((1 << u) + t) * E] = dst[t * E] ^ basis[u];
            }
        }
        __syncthreads();
        const int sh = (int)(i0 & 63);
#pragma unroll
        for (int q = 0; q < Sh::MAXPASS; ++q) {
            if (q >= npass) break;
            // entry 0 of every table is zero: no branch on x; lanes past the planes (TPR > E)
            // read plane-0 words and drop them at the store
            const uint64_t *tb = tab + (b < E ? b : 0);
            const uint64_t arow = aw[q] >> sh;
#pragma unroll 4
            for (int i = 0; i < kc; ++i) {
                const unsigned bal = __ballot_sync(0xffffffffu, (arow >> i) & 1ULL);
                const uint32_t x = (bal >> gl) & EMASK;
                const uint64_t *ti = tb + i * QE;
                if constexpr (SP::H2 > 0)
                    v[q] ^= ti[(x & ((1u << SP::H1) - 1)) * E] ^ ti[((1u << SP::H1) + (x >> SP::H1)) * E];
                else
                    v[q] ^= ti[x * E];
            }
        }
    }
    // bits of the last word beyond column n keep their value
    const int64_t nw = (n + 63) >> 6;
    const uint64_t keep = (w == nw - 1 && (n & 63)) ? ~((1ULL << (n & 63)) - 1) : 0ULL;
#pragma unroll
    for (int q = 0; q < Sh::MAXPASS; ++q) {
        if (q >= npass) break;
        const int64_t r = row0 + q * Sh::RPC + rl;
        if (r < m && b < E) {
            uint64_t *c = C + b * pc + r * ldc + w;
            const uint64_t old = *c;
            const uint64_t nv = acc ? old ^ v[q] : v[q];
            *c = (old & keep) | (nv & ~keep);
        }
    }
}

template <int E>
cudaError_t launch_nj_sliced_e(const FieldTab *ftab, const uint64_t *A, int64_t lda, int64_t pa, const uint64_t *B,
                               int64_t ldb, int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m, int64_t k,
                               int64_t n, bool acc, bool c_aliases_b, cudaStream_t st) {
    using Sh = NjsShape<E>;
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr_set[dev]) {
        cudaError_t err =
            cudaFuncSetAttribute(k_nj_sliced<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    const int64_t nw = (n + 63) >> 6;
    const int64_t blocks1 = (m + Sh::RPC - 1) / Sh::RPC;  // row blocks at one pass
    int npass = 1;
    if (c_aliases_b) {
        npass = (int)blocks1;  // one row block per column word
        if (npass > Sh::MAXPASS) return cudaErrorInvalidValue;
    } else {
        // fewer, longer row blocks when the grid is far beyond one wave (tables amortised)
        while (npass < Sh::MAXPASS && nw * ((blocks1 + npass - 1) / npass) > 4 * 148) npass *= 2;
    }
    const int64_t rb = (m + (int64_t)Sh::RPC * npass - 1) / ((int64_t)Sh::RPC * npass);
    if (nw > 0x7fffffff || rb > 65535) return cudaErrorInvalidValue;
    dim3 grid((unsigned)nw, (unsigned)rb);
    return launch_pdl(k_nj_sliced<E>, grid, dim3(Sh::THREADS), Sh::SMEM, st, ftab, A, lda, pa, B, ldb, pb, C, ldc, pc, m,
                      k, n, acc ? 1 : 0, npass);
}

}  // namespace

cudaError_t launch_nj_mul(int e, uint32_t f, int w, const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          uint64_t *C, int64_t ldc, int64_t m, int64_t k, int64_t n, bool acc, cudaStream_t st) {
    switch (e) {
        case 2: return launch_nj_e<2>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 3: return launch_nj_e<3>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 4: return launch_nj_e<4>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 5: return launch_nj_e<5>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 6: return launch_nj_e<6>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 7: return launch_nj_e<7>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 8: return launch_nj_e<8>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 9: return launch_nj_e<9>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        case 10: return launch_nj_e<10>(f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gf2e

namespace gf2e {
cudaError_t launch_nj_sliced(int e, const FieldTab *ftab, const uint64_t *A, int64_t lda, int64_t pa,
                             const uint64_t *B, int64_t ldb, int64_t pb, uint64_t *C, int64_t ldc, int64_t pc,
                             int64_t m, int64_t k, int64_t n, bool acc, bool c_aliases_b, cudaStream_t st) {
#define NJS(EE) \
    case EE: return launch_nj_sliced_e<EE>(ftab, A, lda, pa, B, ldb, pb, C, ldc, pc, m, k, n, acc, c_aliases_b, st);
    switch (e) {
        NJS(2) NJS(3) NJS(4) NJS(5) NJS(6) NJS(7) NJS(8) NJS(9) NJS(10)
        default: return cudaErrorInvalidValue;
    }
#undef NJS
}
}  // namespace gf2e

// product_tc.cu — K3/K4/K5 fused: every GF(2) plane product of the Karatsuba schedule for
// one 128 x 256 tile of C on the tcgen05 tensor cores (kind::i8), with the Karatsuba
// combine, the mod-f fold and the addmul XOR in the epilogue.
//
// Reference: karatsuba_mul (poly_mul.py:245-259) -> _kara (166-220) -> mat_gf2.mul
// (mat_gf2.py:425-455) per product, then reduce_mod_f (poly_mul.py:223-242) and, for
// addmul, xor_window (mat_gf2.py:270-277).  Here C_j (^)= XOR_{t : M[j,t]} A'_t . B'_t with
// M = R_f . Gamma (the schedule, capi.cu), evaluated tile by tile without materialising
// any product plane.
//
// GF(2) product on an integer MMA.  Operand bits are expanded to bytes in shared memory
// by the producer warps with ONE AND per 32-bit output word and no shifts:
//   A (natural bit order)            : byte j of out_i = (w & (0x01010101 << i)) -> value a*2^i
//   B^T (bits reversed in each byte) : byte j of out_i = (w & (0x80808080 >> i)) -> value b*2^(7-i)
// Both hold k-bit 32q+8j+i at the same byte slot, so every byte product is a*b*2^7 and the
// s32 accumulator equals 128 * sum_k a_k b_k (mod 2^32): the GF(2) result is bit 7.
//
// Warp roles (416 threads, 1 CTA / SM):
//   warps 0-3  producers: cp.async bit tiles D stages ahead, expand into the UMMA
//              K-major SWIZZLE_128B layout (S stages of 48 KiB), arrive on full[s]
//   warps 4-11 epilogue : tcgen05.ld the s32 accumulator (TMEM lanes 32*(w%4).., one column
//              half per warp), take bit 7, pack 128 bits per row, fold into E
//              register-resident output planes
//   warp  12   MMA      : one thread issues tcgen05.mma (M=128, N=256, K=32) x 4 per stage;
//              tcgen05.commit frees the stage and, per product, hands the TMEM buffer
//              (2 x 256 columns) to the epilogue.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace gf2e {
namespace {
using namespace tc;

constexpr int BM = kTcBM, BN = kTcBN, BK = kTcBK;
constexpr int S = 3;  // expanded operand stages
constexpr int D = 8;  // bit-tile staging depth
constexpr int NPROD = 128;
constexpr int NEPI = 256;      // 8 epilogue warps: 4 TMEM lane quarters x 2 column halves
constexpr int MMA_WARP = 12;
constexpr int NTHREADS = 13 * 32;
constexpr int A_BYTES = BM * BK;  // 16 KiB of 0/1 bytes
constexpr int B_BYTES = BN * BK;  // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int BITS_A = BM * (BK / 8);             // 2 KiB
constexpr int BITS_BYTES = (BM + BN) * (BK / 8);  // 6 KiB
constexpr int TMEM_COLS = 512;
constexpr uint32_t IDESC = idesc_i8(BM, BN);

struct __align__(8) Bars {
    uint64_t full[S], empty[S], tfull[2], tempty[2];
    uint32_t tmem_base;
    uint16_t outmask[kMaxProducts];
};
constexpr int SMEM_BYTES = S * STAGE_BYTES + D * BITS_BYTES + (int)sizeof(Bars) + 1024;

template <int E>
__global__ void __launch_bounds__(NTHREADS, 1) k_product_tc(const Sched s, const TcArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *stages = smem;
    uint8_t *bits = smem + S * STAGE_BYTES;
    Bars *bars = reinterpret_cast<Bars *>(bits + D * BITS_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Persistent: CTA b owns tiles b, b + grid, b + 2*grid, ...  All roles walk the same
    // (tile, product, k-stage) sequence, so ring phases carry across tiles and the epilogue
    // of tile i (TMEM read-out + C store) overlaps the MMAs of tile i+1.
    const int64_t tiles_n = a.n_pad / BN;
    const int64_t ntiles = (a.m_pad / BM) * tiles_n;
    const int64_t my_tiles = ntiles > (int64_t)blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int nks = (int)(a.kwords / (BK / 64));
    const int64_t per_tile = (int64_t)s.nprod * nks;
    const int64_t total = my_tiles * per_tile;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&bars->full[i], NPROD);
            mbar_init(&bars->empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->tfull[i], 1);
            mbar_init(&bars->tempty[i], NEPI);
        }
        mbar_fence_init();
    }
    if (threadIdx.x < kMaxProducts) bars->outmask[threadIdx.x] = s.outmask[threadIdx.x];
    if (warp == MMA_WARP) tmem_alloc(&bars->tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp < 4) {
        // ===================== producers =====================
        const int p = threadIdx.x;
        const int64_t offA = (int64_t)p * a.kwords;
        const int64_t offB0 = (int64_t)b_row_perm(p) * a.kwords;
        const int64_t offB1 = (int64_t)b_row_perm(p + 128) * a.kwords;
        const uint32_t bits_s = smem_u32(bits);
        // issue cursor (runs D-1 stages ahead of the consume cursor); no 64-bit divisions
        int64_t i_tile = blockIdx.x;
        int i_t = 0, i_ks = 0, i_slot = 0;
        const uint64_t *Ab = nullptr, *Bb = nullptr;
        auto set_base = [&]() {
            const int64_t m0 = (i_tile / tiles_n) * BM, n0 = (i_tile % tiles_n) * BN;
            Ab = a.Ac + m0 * a.kwords + offA;
            Bb = a.Bt + n0 * a.kwords;
        };
        set_base();
        auto issue = [&]() {
            const uint32_t slot = bits_s + (uint32_t)(i_slot * BITS_BYTES);
            const int64_t koff = i_ks * (BK / 64);
            const uint64_t *ap = Ab + i_t * a.a_pstride + koff;
            const uint64_t *bp = Bb + i_t * a.b_pstride + koff;
            cp_async16(slot + p * 16, ap);
            cp_async16(slot + BITS_A + p * 16, bp + offB0);
            cp_async16(slot + BITS_A + (p + 128) * 16, bp + offB1);
            if (++i_slot == D) i_slot = 0;
            if (++i_ks == nks) {
                i_ks = 0;
                if (++i_t == s.nprod) {
                    i_t = 0;
                    i_tile += gridDim.x;
                    if (i_tile < ntiles) set_base();
                }
            }
        };
        for (int i = 0; i < D - 1; ++i) {
            if (i < total) issue();
            cp_async_commit();
        }
        int c_slot = 0, st = 0;
        uint32_t phase = 0;
        for (int64_t it = 0; it < total; ++it) {
            if (it + D - 1 < total) issue();
            cp_async_commit();
            cp_async_wait<D - 1>();
            const uint8_t *slot = bits + c_slot * BITS_BYTES;
            const uint4 wa = *reinterpret_cast<const uint4 *>(slot + p * 16);
            const uint4 wb0 = *reinterpret_cast<const uint4 *>(slot + BITS_A + p * 16);
            const uint4 wb1 = *reinterpret_cast<const uint4 *>(slot + BITS_A + (p + 128) * 16);
            mbar_wait(&bars->empty[st], phase ^ 1);
            uint8_t *sa = stages + st * STAGE_BYTES;
            expand_row<false>(sa, p, wa);
            expand_row<true>(sa + A_BYTES, p, wb0);
            expand_row<true>(sa + A_BYTES, p + 128, wb1);
            fence_proxy_async_smem();
            mbar_arrive(&bars->full[st]);
            if (++c_slot == D) c_slot = 0;
            if (++st == S) {
                st = 0;
                phase ^= 1;
            }
        }
        cp_async_wait<0>();
    } else if (warp < MMA_WARP) {
        // ===================== epilogue =====================
        const int q = warp & 3;         // TMEM lane quarter (hardware: warp id % 4)
        const int h = (warp - 4) >> 2;  // column half: columns [128h, 128h + 128)
        const int row_local = q * 32 + lane;
        const int64_t nw = words_for(a.n);
        int64_t gp = 0;  // global product counter (TMEM buffer ring)
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = blockIdx.x + ti * gridDim.x;
            const int64_t m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
            uint32_t acc[E][4];
#pragma unroll
            for (int j = 0; j < E; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[j][c] = 0;
            for (int t = 0; t < s.nprod; ++t, ++gp) {
                const int buf = (int)(gp & 1);
                mbar_wait(&bars->tfull[buf], (uint32_t)((gp >> 1) & 1));
                tc_fence_after();
                const uint32_t mask = bars->outmask[t];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + h * 128 + c * 32), v);
                    tmem_wait_ld();
                    const uint32_t pw = parity_word(v);
#pragma unroll
                    for (int j = 0; j < E; ++j) acc[j][c] ^= pw & (0u - ((mask >> j) & 1u));
                }
                tc_fence_before();
                mbar_arrive(&bars->tempty[buf]);
            }
            const int64_t row = m0 + row_local;
            if (row < a.m) {
                const int64_t w0 = (n0 >> 6) + 2 * h;
                const bool v0 = w0 < nw, v1 = w0 + 1 < nw;
                uint64_t old[E][2];
#pragma unroll
                for (int j = 0; j < E; ++j) {  // all C0 loads in flight before any store
                    const uint64_t *crow = a.C + j * a.c_pstride + row * a.ldc + w0;
                    old[j][0] = (a.accumulate && v0) ? crow[0] : 0;
                    old[j][1] = (a.accumulate && v1) ? crow[1] : 0;
                }
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    uint64_t *crow = a.C + j * a.c_pstride + row * a.ldc + w0;
                    const uint64_t x0 = ((uint64_t)acc[j][0] | ((uint64_t)acc[j][1] << 32)) ^ old[j][0];
                    const uint64_t x1 = ((uint64_t)acc[j][2] | ((uint64_t)acc[j][3] << 32)) ^ old[j][1];
                    if (v0 && v1 && !(reinterpret_cast<uintptr_t>(crow) & 15)) {
                        *reinterpret_cast<ulonglong2 *>(crow) = make_ulonglong2(x0, x1);
                    } else {
                        if (v0) crow[0] = x0;
                        if (v1) crow[1] = x1;
                    }
                }
            }
        }
    } else {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int64_t gp = 0;
            int st = 0;
            uint32_t phase = 0;
            const uint32_t st0 = smem_u32(stages);
            for (int64_t ti = 0; ti < my_tiles; ++ti) {
                for (int t = 0; t < s.nprod; ++t, ++gp) {
                    const int buf = (int)(gp & 1);
                    mbar_wait(&bars->tempty[buf], (uint32_t)((gp >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t dt = tmem + (uint32_t)(buf * BN);
                    for (int ks = 0; ks < nks; ++ks) {
                        mbar_wait(&bars->full[st], phase);
                        tc_fence_after();
                        const uint32_t sa = st0 + (uint32_t)(st * STAGE_BYTES);
                        const uint32_t sb = sa + A_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk)
                            mma_i8(dt, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), IDESC,
                                   (ks | kk) != 0);
                        mma_commit(&bars->empty[st]);
                        if (++st == S) {
                            st = 0;
                            phase ^= 1;
                        }
                    }
                    mma_commit(&bars->tfull[buf]);
                }
            }
        }
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

int g_num_sms = 0;

template <int E>
cudaError_t launch_e(const Sched &s, const TcArgs &a, cudaStream_t st) {
    cudaError_t err = cudaFuncSetAttribute(k_product_tc<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (err != cudaSuccess) return err;
    const int64_t tiles = (a.m_pad / BM) * (a.n_pad / BN);
    if (tiles == 0) return cudaSuccess;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    const int64_t grid = tiles < g_num_sms ? tiles : g_num_sms;  // one persistent CTA per SM
    k_product_tc<E><<<(unsigned)grid, NTHREADS, SMEM_BYTES, st>>>(s, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_product_tc(const Sched &s, const TcArgs &a, cudaStream_t st) {
    switch (s.nout) {
        case 1: return launch_e<1>(s, a, st);
        case 2: return launch_e<2>(s, a, st);
        case 3: return launch_e<3>(s, a, st);
        case 4: return launch_e<4>(s, a, st);
        case 5: return launch_e<5>(s, a, st);
        case 6: return launch_e<6>(s, a, st);
        case 7: return launch_e<7>(s, a, st);
        case 8: return launch_e<8>(s, a, st);
        case 9: return launch_e<9>(s, a, st);
        case 10: return launch_e<10>(s, a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gf2e

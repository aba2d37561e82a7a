// product_tc2.cu — the fused Karatsuba product kernel on CTA PAIRS (tcgen05 cta_group::2).
//
// Same contract and arithmetic as product_tc.cu (reference: karatsuba_mul poly_mul.py:245-259,
// _kara 166-220, mat_gf2.mul mat_gf2.py:425-455, reduce_mod_f poly_mul.py:223-242), but each
// cluster of 2 CTAs owns a 256 x 256 tile of C and issues M=256 N=256 K=32 MMAs:
//   CTA r (r = cluster rank) expands A rows [128r, 128r+128) and B^T rows [128r, 128r+128)
//   of the tile, so per SM the producers write 32 KiB of 0/1 bytes per 128-bit k-stage
//   instead of 48 KiB and the tensor core reads 32 KiB instead of 48 KiB — shared-memory
//   bandwidth, not the tensor pipe, bounds the 1-CTA kernel (profiles/r01).
//   The leader (rank 0) issues the MMAs; accumulators land in each CTA's own TMEM (its 128
//   rows x 256 columns, double buffered), so the epilogue is unchanged per CTA.
// Synchronisation across the pair:
//   full[s]   (leader)   <- 4 producer warps x 2 CTAs (remote arrive after fence.proxy.async)
//   empty[s]  (each CTA) <- tcgen05.commit multicast to both CTAs
//   tfull[b]  (each CTA) <- tcgen05.commit multicast to both CTAs
//   tempty[b] (leader)   <- 8 epilogue warps x 2 CTAs (remote arrive)
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace gf2e {
namespace {
using namespace tc;

constexpr int BM = 128;    // rows per CTA (tile = 2 x BM)
constexpr int BNH = 128;   // B^T rows per CTA (tile N = 2 x BNH = 256)
constexpr int BN = 256;
constexpr int BK = kTcBK;  // 128 k-bits per stage
constexpr int S = 5;       // expanded operand stages
constexpr int D = 8;       // bit-tile staging depth
#ifndef GF2E_NPW
#define GF2E_NPW 4
#endif
#ifndef GF2E_GROUP_M
#define GF2E_GROUP_M 8
#endif
#ifndef GF2E_EPI_X16
#define GF2E_EPI_X16 2  // 2: pack::16b + sign-PRMT parity, 1: two x16 loads, 0: one x32 load
#endif
constexpr int NPW = GF2E_NPW;  // expander warps (8: 0-3 expand A rows, 4-7 B^T rows; 4: both)
constexpr int NEW = 8;         // epilogue warps
constexpr int GROUP_M = GF2E_GROUP_M;  // tile rasterisation: row-tiles per column sweep (L2 reuse)
#ifndef GF2E_EXP_HIGH
#define GF2E_EXP_HIGH 0
#endif
// Warp roles.  The issue arbiter favours higher warp ids, and the expanders are the critical
// role, so (GF2E_EXP_HIGH) they take the highest ids: epilogue 0-7, MMA 8, loader 9,
// expanders 10-13 (one per SMSP either way: warp id % 4 covers 0..3).
constexpr int EPI_W0 = GF2E_EXP_HIGH ? 0 : NPW;
constexpr int MMA_WARP = GF2E_EXP_HIGH ? NEW : NPW + NEW;
constexpr int LOAD_WARP = MMA_WARP + 1;
constexpr int EXP_W0 = GF2E_EXP_HIGH ? NEW + 2 : 0;
constexpr int NTHREADS = (NPW + NEW + 2) * 32;
constexpr int A_BYTES = BM * BK;   // 16 KiB
constexpr int B_BYTES = BNH * BK;  // 16 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int BITS_A = BM * (BK / 8);
constexpr int BITS_BYTES = (BM + BNH) * (BK / 8);  // 4 KiB
constexpr int TMEM_COLS = 512;
constexpr uint32_t IDESC = idesc_i8(2 * BM, BN);

struct __align__(8) Bars {
    uint64_t full[S], empty[S], tfull[2], tempty[2], bfull[D], bempty[D];
    uint32_t tmem_base;
    uint16_t outmask[kMaxProducts];
};
constexpr int SMEM_BYTES = S * STAGE_BYTES + D * BITS_BYTES + (int)sizeof(Bars) + 1024;

// tile index -> (row-tile, column-tile): sweep GROUP_M row-tiles down each column before
// moving right, so the ~74 CTA pairs in flight share a few A row-blocks and B^T column-blocks
// in L2 (row-major order re-read all of B^T from DRAM once per wave).
__device__ __forceinline__ void tile_coords(int64_t tile, int64_t tiles_m, int64_t tiles_n, int64_t &tm,
                                            int64_t &tn) {
    const int64_t per_group = (int64_t)GROUP_M * tiles_n;
    const int64_t g = tile / per_group, r = tile - g * per_group;
    const int64_t first = g * GROUP_M;
    const int64_t gsize = tiles_m - first < GROUP_M ? tiles_m - first : GROUP_M;
    tm = first + r % gsize;
    tn = r / gsize;
}

template <int E>
__global__ void __launch_bounds__(NTHREADS, 1) k_product_tc2(const Sched s, const TcArgs a) {
    extern __shared__ uint8_t smem_raw[];
    // keep the shared state space visible to the compiler (STS/LDS, not generic ST/LD)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *stages = smem;
    uint8_t *bits = smem + S * STAGE_BYTES;
    Bars *bars = reinterpret_cast<Bars *>(bits + D * BITS_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int64_t tiles_n = a.n_pad / BN;
    const int64_t tiles_m = a.m_pad / (2 * BM);
    const int64_t ntiles = tiles_m * tiles_n;
    const int64_t my_tiles = ntiles > cluster ? (ntiles - cluster + nclusters - 1) / nclusters : 0;
    const int nks = (int)(a.kwords / (BK / 64));
    const int64_t per_tile = (int64_t)s.nprod * nks;
    const int64_t total = my_tiles * per_tile;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&bars->full[i], 2 * NPW);
            mbar_init(&bars->empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->tfull[i], 1);
            mbar_init(&bars->tempty[i], 2 * NEW);
        }
        for (int i = 0; i < D; ++i) {
            mbar_init(&bars->bfull[i], 1);
            mbar_init(&bars->bempty[i], NPW);
        }
        mbar_fence_init();
    }
    if (threadIdx.x < kMaxProducts) bars->outmask[threadIdx.x] = s.outmask[threadIdx.x];
    if (warp == MMA_WARP) tmem_alloc2(&bars->tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp >= EXP_W0 && warp < EXP_W0 + NPW) {
        // ===================== expanders (both CTAs) =====================
        // bit tiles arrive by bulk copy (loader warp); these warps keep no global loads in
        // flight, so the per-stage fence.proxy.async (MEMBAR.ALL.CTA) only drains their STS.
        // Two warps per SMSP: one warp's fence / LDS latency overlaps another's expansion.
        const bool isB = NPW == 8 && warp - EXP_W0 >= 4;
        const int p = (threadIdx.x - EXP_W0 * 32) & 127;  // row of this CTA's A half (isB: B^T half)
        const uint32_t src_off = (isB ? BITS_A : 0) + p * 16;
        const uint32_t dst_off = isB ? A_BYTES : 0;
        const uint32_t full_leader = mapa(smem_u32(&bars->full[0]), 0);
        int slot = 0, st = 0;
        uint32_t bph = 0, phase = 0;
        for (int64_t it = 0; it < total; ++it) {
            mbar_wait(&bars->bfull[slot], bph);
            const uint4 w = *reinterpret_cast<const uint4 *>(bits + slot * BITS_BYTES + src_off);
            uint4 wb2;
            if (NPW == 4) wb2 = *reinterpret_cast<const uint4 *>(bits + slot * BITS_BYTES + BITS_A + p * 16);
            mbar_wait(&bars->empty[st], phase ^ 1);
            uint8_t *tile = stages + st * STAGE_BYTES + dst_off;
            if (isB)
                expand_row<true>(tile, p, w);
            else
                expand_row<false>(tile, p, w);
            if (NPW == 4) expand_row<true>(stages + st * STAGE_BYTES + A_BYTES, p, wb2);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_cluster(full_leader + (uint32_t)(st * 8));
                // the bit tile was consumed by the expansion above (data dependence), so the
                // loader may overwrite the slot: no read-before-overwrite race on bits
                mbar_arrive(&bars->bempty[slot]);
            }
            if (++slot == D) {
                slot = 0;
                bph ^= 1;
            }
            if (++st == S) {
                st = 0;
                phase ^= 1;
            }
        }
    } else if (warp == LOAD_WARP) {
        // ===================== bit-tile loader (both CTAs, one thread) =====================
        if (lane == 0) {
            const int64_t KS = a.kwords >> 1;  // k-stages per row block
            const uint32_t bits_s = smem_u32(bits);
            int slot = 0;
            uint32_t bph = 0;
            for (int64_t ti = 0; ti < my_tiles; ++ti) {
                const int64_t tile = cluster + ti * nclusters;
                int64_t tm, tn;
                tile_coords(tile, tiles_m, tiles_n, tm, tn);
                const int64_t rbA = tm * 2 + rank;  // 128-row block of A
                const int64_t rbB = tn * 2 + rank;  // 128-row block of B^T
                for (int t = 0; t < s.nprod; ++t) {
                    const uint64_t *Ab = a.Ac + t * a.a_pstride + rbA * KS * 256;
                    const uint64_t *Bb = a.Bt + t * a.b_pstride + rbB * KS * 256;
                    for (int ks = 0; ks < nks; ++ks) {
                        mbar_wait(&bars->bempty[slot], bph ^ 1);
                        mbar_arrive_expect_tx(&bars->bfull[slot], BITS_BYTES);
                        const uint32_t dst = bits_s + (uint32_t)(slot * BITS_BYTES);
                        bulk_g2s(dst, Ab + ks * 256, BITS_A, &bars->bfull[slot]);
                        bulk_g2s(dst + BITS_A, Bb + ks * 256, BITS_BYTES - BITS_A, &bars->bfull[slot]);
                        if (++slot == D) {
                            slot = 0;
                            bph ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp >= EPI_W0 && warp < EPI_W0 + NEW) {
        // ===================== epilogue (both CTAs) =====================
        const int ew = warp - EPI_W0;
        const int q = warp & 3;  // TMEM lane quarter (hardware: warp id % 4)
        const int h = ew >> 2;   // column half
        const int row_local = (int)rank * BM + q * 32 + lane;
        const int64_t nw = words_for(a.n);
        const uint32_t tempty_leader = mapa(smem_u32(&bars->tempty[0]), 0);
        int64_t gp = 0;
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = cluster + ti * nclusters;
            int64_t tm, tn;
            tile_coords(tile, tiles_m, tiles_n, tm, tn);
            const int64_t m0 = tm * (2 * BM), n0 = tn * BN;
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
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + h * 128 + c * 32);
#if GF2E_EPI_X16 == 2
                    uint32_t v[16];
                    tmem_ld32_pack16(ta, v);
                    tmem_wait_ld();
                    const uint32_t pw = parity_word_packed(v);
#elif GF2E_EPI_X16
                    uint32_t v[16];
                    tmem_ld16(ta, v);
                    tmem_wait_ld();
                    uint32_t pw = parity_half(v, 0);
                    tmem_ld16(ta + 16, v);
                    tmem_wait_ld();
                    pw |= parity_half(v, 4);
#else
                    uint32_t v[32];
                    tmem_ld32(ta, v);
                    tmem_wait_ld();
                    const uint32_t pw = parity_word(v);
#endif
#pragma unroll
                    for (int j = 0; j < E; ++j) acc[j][c] ^= pw & (0u - ((mask >> j) & 1u));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(buf * 8));
            }
            const int64_t row = m0 + row_local;
            if (row < a.m) {
                const int64_t w0 = (n0 >> 6) + 2 * h;
                const bool v0 = w0 < nw, v1 = w0 + 1 < nw;
#pragma unroll
                for (int j0 = 0; j0 < E; j0 += 4) {  // C0 loads of up to 4 planes in flight per batch
                    uint64_t old[4][2];
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int j = j0 + jj;
                        if (j < E) {
                            const uint64_t *crow = a.C + j * a.c_pstride + row * a.ldc + w0;
                            old[jj][0] = (a.accumulate && v0) ? crow[0] : 0;
                            old[jj][1] = (a.accumulate && v1) ? crow[1] : 0;
                        }
                    }
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int j = j0 + jj;
                        if (j < E) {
                            uint64_t *crow = a.C + j * a.c_pstride + row * a.ldc + w0;
                            const uint64_t x0 = ((uint64_t)acc[j][0] | ((uint64_t)acc[j][1] << 32)) ^ old[jj][0];
                            const uint64_t x1 = ((uint64_t)acc[j][2] | ((uint64_t)acc[j][3] << 32)) ^ old[jj][1];
                            if (v0 && v1 && !(reinterpret_cast<uintptr_t>(crow) & 15)) {
                                *reinterpret_cast<ulonglong2 *>(crow) = make_ulonglong2(x0, x1);
                            } else {
                                if (v0) crow[0] = x0;
                                if (v1) crow[1] = x1;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == MMA_WARP && rank == 0) {
        // ===================== MMA issuer (leader CTA, one thread) =====================
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
                            mma2_i8(dt, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), IDESC,
                                    (ks | kk) != 0);
                        mma2_commit_both(&bars->empty[st]);
                        if (++st == S) {
                            st = 0;
                            phase ^= 1;
                        }
                    }
                    mma2_commit_both(&bars->tfull[buf]);
                }
            }
        }
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();  // all MMAs of the pair retired (every epilogue saw its last tfull)
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, TMEM_COLS);
    }
}

int g_num_sms2 = 0;

template <int E>
cudaError_t launch_e(const Sched &s, const TcArgs &a, cudaStream_t st) {
    cudaError_t err = cudaFuncSetAttribute(k_product_tc2<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (err != cudaSuccess) return err;
    const int64_t tiles = (a.m_pad / (2 * BM)) * (a.n_pad / BN);
    if (tiles == 0) return cudaSuccess;
    if (g_num_sms2 == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms2, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms2 <= 1) g_num_sms2 = 148;
    }
    const int64_t clusters = tiles < g_num_sms2 / 2 ? tiles : g_num_sms2 / 2;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_product_tc2<E>, s, a);
}

}  // namespace

cudaError_t launch_product_tc2(const Sched &s, const TcArgs &a, cudaStream_t st) {
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

// product_run.cu — the short-k tensor-core form of the fused Karatsuba product (k < 2048: the
// config-4 addmul 65536x256x65536, the TRSM / PLE Schur updates ple_echelon.py:130-136,259).
//
// Same GF(2) encoding as the fp4 forms of product_tc2.cu (kind::mxf4 block-scaled e2m1, all
// scale factors 1.0: A nibbles 0.5/1/2/1, B^T nibbles 2/1/0.5/1, every product of aligned bits
// exactly 1.0), but short accumulations make the per-product TMEM traffic, not the MMA, the
// bound.  Measured (tools/tmem_bench.cu, profiles/r02): tcgen05.ld reaches ~100 cells/clk/SM
// alone and ~50 while MMAs run; tcgen05.st ~40-58 cells/clk.  The fp4 forms re-initialise the
// accumulator after every drain (one tcgen05.st per cell per product) and have a single
// accumulator; this form removes both:
//
//  * running sums.  Each accumulator starts at 65536.0f once per tile and is never
//    re-initialised between products: after product t it holds 65536 + S_t, S_t = the sum of
//    the counts of the products accumulated into it so far (exact while S_t < 2^16: at most
//    ceil(K/2) * k < 65536, which the host checks), so S_t sits in mantissa bits 7.. and
//    parity(count_t) = bit7 ^ bit7 of the previous read of the same buffer: the epilogue keeps
//    the previous parity word of each buffer and XORs.  No tcgen05.st per product.
//  * double buffering.  Two accumulators of N = 192 columns (products alternate between
//    them), so the drain of product t overlaps the MMAs of product t+1.  TMEM: accumulators
//    0-191 and 192-383, three A stages 384-479 (the expanded A operand lives in TMEM, as in
//    the long-k fp4 form), scale factors 480-511.  N = 192 (not 256) is what makes both
//    accumulators, the A stages and the scale factors fit in 512 columns.
//
// Tiles are 256 x 192 (CTA pair, cta_group::2, M = 256, N = 192); B^T is stage-tiled in
// 96-row blocks (tc_tile_word br = 96).  Output words are written 32 bits at a time (a tile
// covers 6 words of 32 columns).  Warp roles as in product_tc2.cu: 4 expander warps (A rows
// into TMEM, B^T rows into shared memory), 8 epilogue warps (lane quarter x column half),
// MMA issuer (leader CTA), bulk loader.
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

// Per-degree variants (build knobs, chosen by measurement, profiles/r02/run_variants.txt):
//  STW: a store warp writes each finished tile out (double-buffered staging in shared memory,
//       C0 read by that warp) while the epilogue warps drain the next tile; for E >= the knob
//  DIET: differenced output masks (no previous parity words kept), the parity word packed with
//       IMAD.HI on the FMA pipe, plane selectors read from a shared table; for E >= the knob
#ifndef GF2E_RUN_REINIT_EVERY_TILE  // 1: reset the running sums at every tile (the round-2 form)
#define GF2E_RUN_REINIT_EVERY_TILE 0
#endif
#ifndef GF2E_RUN_STW_MIN_E
#define GF2E_RUN_STW_MIN_E 7
#endif
#ifndef GF2E_RUN_DIET_MIN_E
#define GF2E_RUN_DIET_MIN_E 11
#endif
// Tile raster: groups of GROUP_M row tiles walk all column tiles.  The pre-expanded B^T of a
// config-4 product (e = 8: 27 x 342 column tiles x 24 KiB = 221 MB) does not fit the L2, so it
// streams from DRAM once per row group: wider groups re-read it less (e = 8: 8 -> 24 rows,
// 15.93 -> 14.85 ms, profiles/r02/run_variants.txt); 48 rows at e = 4..6, 8 below
#ifndef GF2E_RUN_GROUP_M_SMALL
#define GF2E_RUN_GROUP_M_SMALL 8
#endif
#ifndef GF2E_RUN_GROUP_M_MID  // e = 4..6 (e = 4: 6.59 -> 6.44 ms, e = 6: 11.33 -> 11.26)
#define GF2E_RUN_GROUP_M_MID 48
#endif
#ifndef GF2E_RUN_GROUP_M_LARGE
#define GF2E_RUN_GROUP_M_LARGE 24
#endif
template <int E>
struct RunVar {
    static constexpr bool STW = E >= GF2E_RUN_STW_MIN_E, DIET = E >= GF2E_RUN_DIET_MIN_E;
    static constexpr int GM = E >= 7   ? GF2E_RUN_GROUP_M_LARGE
                              : E >= 4 ? GF2E_RUN_GROUP_M_MID
                                       : GF2E_RUN_GROUP_M_SMALL;  // raster rows
};

namespace gf2e {
namespace {
using namespace tc;

constexpr int BM = 128;               // A rows per CTA (tile = 2 x BM)
constexpr int BN = kRunBN;            // tile columns
constexpr int BNH = BN / 2;           // B^T rows per CTA
constexpr int KW = 4;                 // 64-bit words per row per stage (256 k-bits)
constexpr int S = 3;                  // operand stages (A: 3 x 32 TMEM columns)
constexpr int D = 8;                  // raw bit-tile ring
constexpr int NEXP = 4, NEPI = 8;  // epilogue: lane quarter x column half (96 columns, one TMEM round trip)
constexpr int EPI_W0 = NEXP, MMA_WARP = NEXP + NEPI, LOAD_WARP = MMA_WARP + 1, STORE_WARP = LOAD_WARP + 1;
constexpr int NTHREADS = (NEXP + NEPI + 3) * 32;  // + the store warp (idle unless RunVar<E>::STW)
constexpr int B_BYTES = BNH * 128;                     // expanded B^T stage (12 KiB)
// B^T operand stages: pre-expanded by k_combos_bt and bulk-copied ready for the MMA (kRunBPre),
// or expanded here from bit tiles
// B^T operand stages: pre-expanded by k_combos_bt and bulk-copied ready for the MMA (BP), or
// expanded here from bit tiles by the expander warps (products with few row tiles, where the
// 4x pre-expanded B^T would be written for one or two reads)
constexpr int BITS_A = BM * KW * 8;
template <bool BP>
struct RunMem {
    static constexpr int BITS_B = BP ? 0 : BNH * KW * 8, BITS_BYTES = BITS_A + BITS_B;
};
constexpr uint32_t ACC1 = BN;  // TMEM column of the second accumulator (the first starts at 0)
constexpr uint32_t ATM0 = 2 * BN, SFA = 480, SFB = 496;
static_assert(ATM0 + 32 * S <= SFA, "TMEM: A stages overlap the scale factors");
// 65536.0f: ulp 2^-7 up to 2^17, so the running sum S sits in mantissa bits 7.. and its
// parity is bit 7 of the pattern (the extraction of the other fp4 forms); exact while S < 2^16,
// i.e. ceil(K/2) * k < 65536 (host: kRunMaxSum)
constexpr uint32_t RUN_INIT = 0x47800000u;
constexpr uint32_t SF_ONE = 0x7F7F7F7Fu;               // E8M0 1.0
// Paired drains (PR, E <= 8 at k <= 256): two groups share one accumulator fill, the second one
// scaled by 2^11 through its A scale factors (TMEM columns SFA2..SFA2+7, E8M0 2^11).  The
// accumulators start at 2^23 (ulp 1), so a cell's running sum is F0 + 2^11 F1 with F0, F1 the
// running sums of the two fields' counts, exact while F0 < 2^11 and the total < 2^23 (host:
// run_pair_ok); the parities are bits 0 and 11 of the low 16 bits, i.e. one TMEM drain and one
// hand-off serve two products
constexpr uint32_t PAIR_INIT = 0x4B000000u, SF_2P11 = 0x8A8A8A8Au, SFA2 = 488;
constexpr int CH = BN / (NEPI / 4) / 32;               // 32-column chunks per epilogue thread
constexpr int BARS_BYTES = 1024;
// epilogue staging (per CTA and tile): the E x 128 x 192-bit output words and their C0
// epilogue staging (per CTA and tile): the E x 128 x 192-bit output words and their C0
constexpr int STAGE_OUT_BYTES = kMaxE * BM * 24, STAGE_OLD_BYTES = kMaxE * BM * 24;
// per drain group: the all-ones / zero selector word of every output plane (SEL_EP words per
// group, 16-byte aligned rows, read with LDS.128 instead of being formed from the mask)
constexpr int SEL_EP = 12, SEL_BYTES = kMaxSeq * SEL_EP * 4;
// with the store warp: two staging buffers for the output words and two for the prefetched C0
constexpr int SMEM_BYTES = S * B_BYTES + D * RunMem<false>::BITS_BYTES + BARS_BYTES +
                           STAGE_OUT_BYTES + STAGE_OLD_BYTES + SEL_BYTES +
                           1024;  // (the larger bit ring)
static_assert(B_BYTES % 1024 == 0, "swizzle atoms need 1024-byte aligned stages");
static_assert(SMEM_BYTES <= 232448, "shared memory");

#ifndef GF2E_INSTR
#define GF2E_INSTR 0
#endif
#if GF2E_INSTR
// dev-only (-DGF2E_INSTR=1): per-CTA cycle counters of each role's waits and work
__device__ unsigned long long g_instr_run[1024][32];
#define TWR(acc, stmt)                                \
    do {                                              \
        const long long _t0 = clock64();              \
        stmt;                                         \
        acc += (unsigned long long)(clock64() - _t0); \
    } while (0)
#else
#define TWR(acc, stmt) stmt
#endif

struct __align__(8) Bars {
    uint64_t full[S], empty[S], bfullB[S], tfull[2], tempty[2], bfull[D], bempty[D], sfull[2], sempty[2];
    uint32_t tmem_base;
    uint16_t gmask[kMaxSeq];  // output planes of each drain group
};
static_assert(sizeof(Bars) <= BARS_BYTES, "barrier block");

template <int GROUP_M>
__device__ __forceinline__ void tile_coords(int64_t tile, int64_t tiles_m, int64_t tiles_n, int64_t &tm,
                                            int64_t &tn) {
    const int64_t per_group = (int64_t)GROUP_M * tiles_n;
    const int64_t g = tile / per_group, r = tile - g * per_group;
    const int64_t first = g * GROUP_M;
    const int64_t gsize = tiles_m - first < GROUP_M ? tiles_m - first : GROUP_M;
    tm = first + r % gsize;
    tn = r / gsize;
}

__device__ __forceinline__ void st32_const(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
            taddr),
        "r"(v)
        : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// bit 7 of the 32 pack::16b cells of v -> one word (bit 8b+g = column 4g+b, as
// parity_word_packed), merged as a tree: 8 PRMT, 8 masks, 4 + 2 + 1 ORs, depth 4 instead of 8
__device__ __forceinline__ uint32_t parity_word_tree(const uint32_t (&v)[16]) {
    uint32_t w[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        asm("prmt.b32 %0, %1, %2, 0xECA8;" : "=r"(w[g]) : "r"(v[2 * g]), "r"(v[2 * g + 1]));
        w[g] &= 0x01010101u << g;
    }
    return ((w[0] | w[1]) | (w[2] | w[3])) | ((w[4] | w[5]) | (w[6] | w[7]));
}

// the same word with the merge on the FMA pipe: PRMT gathers bytes 0 and 2 of each cell pair
// without sign replication (a byte is parity << 7: the running sum is an integer in mantissa
// bits 7.., bits 0-6 are zero), then IMAD.HI shifts word g right by 7 - g and adds (disjoint
// bits, so the sum is the OR): 8 PRMT + 7 IMAD.HI instead of 8 PRMT + 8 LOP3 on the ALU pipe.
// The multipliers come from a register (ptxas would turn a constant power of two into SHF).
__device__ __forceinline__ uint32_t parity_word_mad(const uint32_t (&v)[16], uint32_t m25) {
    uint32_t w[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) asm("prmt.b32 %0, %1, %2, 0x6420;" : "=r"(w[g]) : "r"(v[2 * g]), "r"(v[2 * g + 1]));
    uint32_t o = w[7];
#pragma unroll
    for (int g = 0; g < 7; ++g) asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(o) : "r"(w[g]), "r"(m25 << g), "r"(o));
    return o;
}
#define PARITY_WORD(v) (DIET ? parity_word_mad(v, m25) : parity_word_tree(v))

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// A row of one stage into this thread's TMEM lane: 32 columns, word i of chunk q = nibble
// plane i of 32-bit word q (k-bit 32q + 4j + i <-> nibble j)
__device__ __forceinline__ void expand_a_tmem(uint32_t taddr, uint4 lo, uint4 hi) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t o[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t x = w[q];
        o[4 * q] = x & 0x11111111u;
        o[4 * q + 1] = x & 0x22222222u;
        o[4 * q + 2] = x & 0x44444444u;
        o[4 * q + 3] = (x >> 2) & 0x22222222u;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%"
        "29,%30,%31,%32};" ::"r"(taddr),
        "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]), "r"(o[9]),
        "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]), "r"(o[17]), "r"(o[18]),
        "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]), "r"(o[25]), "r"(o[26]), "r"(o[27]),
        "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31])
        : "memory");
}

// B^T row (bits 0 and 2 of every nibble pre-swapped by k_combos_bt) into its swizzle row
__device__ __forceinline__ void expand_b_smem(uint8_t *tile, int r, uint4 lo, uint4 hi) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t x = w[q];
        *reinterpret_cast<uint4 *>(tile + swz(r, q)) =
            make_uint4(x & 0x44444444u, x & 0x22222222u, x & 0x11111111u, (x >> 2) & 0x22222222u);
    }
}

__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma2_mxf4_ts(uint32_t d, uint32_t at, uint64_t bd, uint32_t idesc, uint32_t sfa,
                                             uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, 1, 1;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "r"(at), "l"(bd), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}

template <int E, bool BPRE, bool PR>
__global__ void __launch_bounds__(NTHREADS, 1) k_product_run(const Sched s, const TcArgs a) {
    constexpr int BITS_B = RunMem<BPRE>::BITS_B, BITS_BYTES = RunMem<BPRE>::BITS_BYTES;
    constexpr bool STW = RunVar<E>::STW, DIET = RunVar<E>::DIET;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *stages = smem;
    uint8_t *bits = smem + S * B_BYTES;
    Bars *bars = reinterpret_cast<Bars *>(bits + D * BITS_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int64_t tiles_n = a.n_pad / BN;
    const int64_t tiles_m = a.m_pad / (2 * BM);
    const int64_t ntiles = tiles_m * tiles_n;
    const int64_t my_tiles = ntiles > cluster ? (ntiles - cluster + nclusters - 1) / nclusters : 0;
    const int nks = (int)(a.kwords / KW);
    const int64_t total = my_tiles * (int64_t)s.nseq * nks;  // operand stages (entries x k-stages)

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&bars->full[i], 2 * NEXP);
            mbar_init(&bars->bfullB[i], 1);
            mbar_init(&bars->empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->tfull[i], 1);
            mbar_init(&bars->tempty[i], 2 * NEPI);
        }
        for (int i = 0; i < D; ++i) {
            mbar_init(&bars->bfull[i], 1);
            mbar_init(&bars->bempty[i], NEXP);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->sfull[i], NEPI);
            mbar_init(&bars->sempty[i], 1);
        }
        mbar_fence_init();
    }
    if (threadIdx.x < kMaxSeq) bars->gmask[threadIdx.x] = s.gmask[threadIdx.x];
    // DIET: differenced output masks -- parity(count_t) = bit7(S_t) ^ bit7(S_{t-2}) (same
    // buffer), so plane j = XOR over t of bit7(S_t) * (M_j[t] ^ M_j[t+2]): the bit-7 word of each
    // drain is folded as it is, with no previous word kept (M_j[t+2] = 0 past the buffer's last
    // group); the per-plane all-ones / zero selectors of each group in a table
    uint32_t *selt = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(bars) + BARS_BYTES +
                                                  STAGE_OUT_BYTES + STAGE_OLD_BYTES);
    if constexpr (PR) {  // drain d: field 0 = group 2d, field 1 = group 2d + 1 (differenced per field)
        const int nd = (s.ngrp + 1) / 2;
        auto gm = [&](int g) -> uint32_t { return g < s.ngrp ? (uint32_t)s.gmask[g] : 0u; };
        for (int i = threadIdx.x; i < nd * 2 * SEL_EP; i += NTHREADS) {
            const int d = i / (2 * SEL_EP), r = i - d * (2 * SEL_EP), f = r / SEL_EP, j = r - f * SEL_EP;
            const uint32_t m = gm(2 * d + f) ^ (d + 2 < nd ? gm(2 * d + 4 + f) : 0u);
            selt[i] = j < E ? 0u - ((m >> j) & 1u) : 0u;
        }
    } else if constexpr (DIET)
        for (int i = threadIdx.x; i < s.ngrp * SEL_EP; i += NTHREADS) {
            const int t = i / SEL_EP, j = i - t * SEL_EP;
            const uint32_t m = s.gmask[t] ^ (t + 2 < s.ngrp ? s.gmask[t + 2] : 0u);
            selt[i] = j < E ? 0u - ((m >> j) & 1u) : 0u;
        }
    if (warp == MMA_WARP) tmem_alloc2(&bars->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    if (warp >= EPI_W0 && warp < EPI_W0 + 4) {
        // scale factors (every byte E8M0 1.0) and both running-sum accumulators at 65536
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        st32_const(tmem + lb + SFA, SF_ONE);
        if constexpr (PR)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tmem + lb + SFA2),
                         "r"(SF_2P11)
                         : "memory");
        for (int c = 0; c < 2 * BN; c += 32) st32_const(tmem + lb + c, PR ? PAIR_INIT : RUN_INIT);
        wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();

    if (warp < NEXP) {
        // ===================== expanders =====================
        const int p = threadIdx.x;  // A row p; B^T row p (p < BNH)
        const bool doB = !BPRE && p < BNH;
        const uint32_t full_leader = mapa(smem_u32(&bars->full[0]), 0);
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16) + ATM0;
        int slot = 0, st = 0;
        uint32_t bph = 0, phase = 0;
        uint4 cur[4];
        auto load_bits = [&](int sl) {
            const uint8_t *bs = bits + sl * BITS_BYTES + p * 16;
            cur[0] = *reinterpret_cast<const uint4 *>(bs);
            cur[1] = *reinterpret_cast<const uint4 *>(bs + BM * 16);
            if (doB) {
                cur[2] = *reinterpret_cast<const uint4 *>(bs + BITS_A);
                cur[3] = *reinterpret_cast<const uint4 *>(bs + BITS_A + BNH * 16);
            }
        };
        unsigned long long i_empty = 0, i_bfull = 0, i_work = 0, i_sa = 0, i_sb = 0, i_sw = 0;
        (void)i_sa, (void)i_sb, (void)i_sw;
        const long long i_t0 = clock64();
        (void)i_empty, (void)i_bfull, (void)i_work, (void)i_t0;
        if (total > 0) {
            mbar_wait(&bars->bfull[0], 0);
            load_bits(0);
        }
        for (int64_t it = 0; it < total; ++it) {
            TWR(i_empty, mbar_wait_sleep(&bars->empty[st], phase ^ 1, 32));
#if GF2E_INSTR
            const long long i_w0 = clock64();
#endif
            expand_a_tmem(tl + (uint32_t)(st * 32), cur[0], cur[1]);
#if GF2E_INSTR
            const long long i_w1 = clock64();
#endif
            if (doB) expand_b_smem(stages + st * B_BYTES, p, cur[2], cur[3]);
#if GF2E_INSTR
            const long long i_w2 = clock64();
#endif
            wait_st();
            tc_fence_before();
            if constexpr (BPRE)
                mbar_wait(&bars->bfullB[st], phase);  // the bulk-copied B stage has landed
            else
                fence_proxy_async_smem();
#if GF2E_INSTR
            const long long i_w3 = clock64();
            i_work += (unsigned long long)(i_w3 - i_w0);
            i_sa += (unsigned long long)(i_w1 - i_w0);
            i_sb += (unsigned long long)(i_w2 - i_w1);
            i_sw += (unsigned long long)(i_w3 - i_w2);
#endif
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_cluster(full_leader + (uint32_t)(st * 8));
                mbar_arrive(&bars->bempty[slot]);
            }
            if (++slot == D) {
                slot = 0;
                bph ^= 1;
            }
            if (it + 1 < total) {
                TWR(i_bfull, mbar_wait(&bars->bfull[slot], bph));
                load_bits(slot);
            }
            if (++st == S) {
                st = 0;
                phase ^= 1;
            }
        }
#if GF2E_INSTR
        if (threadIdx.x == 0) {
            g_instr_run[blockIdx.x][0] = i_empty;
            g_instr_run[blockIdx.x][1] = i_bfull;
            g_instr_run[blockIdx.x][2] = i_work;
            g_instr_run[blockIdx.x][3] = (unsigned long long)(clock64() - i_t0);
            g_instr_run[blockIdx.x][12] = i_sa;
            g_instr_run[blockIdx.x][13] = i_sb;
            g_instr_run[blockIdx.x][14] = i_sw;
        }
#endif
    } else if (warp == LOAD_WARP) {
        // ===================== bit-tile loader =====================
        const bool issuer = elect_one();
        const int64_t KS = a.kwords / KW;
        const int64_t tw_a = BM * KW, tw_b = BPRE ? BNH * KW * 4 : BNH * KW;  // B tile words (x4 expanded)
        const uint32_t bits_s = smem_u32(bits), st0 = smem_u32(stages);
        int slot = 0, bst = 0;
        uint32_t bph = 0, sph = 0;
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = cluster + ti * nclusters;
            int64_t tm, tn;
            tile_coords<RunVar<E>::GM>(tile, tiles_m, tiles_n, tm, tn);
            const int64_t rbA = tm * 2 + rank, rbB = tn * 2 + rank;
            for (int i = 0; i < s.nseq; ++i) {
                const int t = s.seq[i];  // entry i of the grouped sequence is product t
                const uint64_t *Ab = a.Ac + t * a.a_pstride + rbA * KS * tw_a;
                const uint64_t *Bb = a.Bt + t * a.b_pstride + rbB * KS * tw_b;
                for (int ks = 0; ks < nks; ++ks) {
                    mbar_wait_sleep(&bars->bempty[slot], bph ^ 1, 64);
                    const uint32_t dst = bits_s + (uint32_t)(slot * BITS_BYTES);
                    if (issuer) {
                        mbar_arrive_expect_tx(&bars->bfull[slot], BITS_BYTES);
                        bulk_g2s(dst, Ab + ks * tw_a, BITS_A, &bars->bfull[slot]);
                        if (!BPRE) bulk_g2s(dst + BITS_A, Bb + ks * tw_b, BITS_B, &bars->bfull[slot]);
                    }
                    __syncwarp();
                    if (++slot == D) {
                        slot = 0;
                        bph ^= 1;
                    }
                    if constexpr (BPRE) {  // the ready B operand stage, once the MMA has freed it
                        mbar_wait_sleep(&bars->empty[bst], sph ^ 1, 64);
                        if (issuer) {
                            mbar_arrive_expect_tx(&bars->bfullB[bst], B_BYTES);
                            bulk_g2s(st0 + (uint32_t)(bst * B_BYTES), Bb + ks * tw_b, B_BYTES, &bars->bfullB[bst]);
                        }
                        __syncwarp();
                        if (++bst == S) {
                            bst = 0;
                            sph ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp < MMA_WARP) {
        // ===================== epilogue =====================
        // Per product: two TMEM round trips per warp (chunks 0+1, then 2; the tempty arrive
        // after the second), parity words folded into E x 3 register words.  Per tile: the words
        // go through shared memory (stage_out) and leave as coalesced 64-bit row segments; C0
        // (addmul) is prefetched into shared memory with cp.async at the tile start by the
        // thread that later XORs it in.
        const int ew = warp - EPI_W0;
        const int et = ew * 32 + lane;  // 0..255
        const int q = warp & 3;         // TMEM lane quarter
        const int h = ew >> 2;          // column half: tile columns [h*96, h*96+96)
        const int r_cta = q * 32 + lane;  // this thread's accumulator row within the CTA's 128
        const int64_t nw = words_for(a.n);
        const uint32_t tempty_leader = mapa(smem_u32(&bars->tempty[0]), 0);
        const uint32_t lq = (uint32_t)(q * 32) << 16;
        // 2^25, opaque to ptxas (bars->tmem_base is a multiple of 2^16 with lane 0, column < 512)
        const uint32_t m25 = (bars->tmem_base & 0x1000000u) | 0x2000000u;
        (void)m25;
        uint32_t *stage_out = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(bars) + BARS_BYTES);
        uint64_t *stage_old = reinterpret_cast<uint64_t *>(stage_out + E * BM * 6);
        const uint64_t *stage_out64 = reinterpret_cast<const uint64_t *>(stage_out);
        constexpr int NOUT = E * BM * 3;  // 64-bit output words per CTA and tile
        uint32_t pc[CH], po[CH];  // !DIET: previous parity words: current buffer / the other buffer
#pragma unroll
        for (int c = 0; c < CH; ++c) pc[c] = po[c] = 0;
        int64_t gp = 0;
        const int64_t sum_tile = (int64_t)(s.run_load > 0 ? s.run_load : 1) * a.kwords * 64;
        const int64_t reinit_tiles =
            (DIET || PR || GF2E_RUN_REINIT_EVERY_TILE) ? 1 : ((kRunMaxSum - 1) / sum_tile > 0 ? (kRunMaxSum - 1) / sum_tile : 1);
        unsigned long long i_tfull = 0, i_drain = 0, i_store = 0, i_e[5] = {0, 0, 0, 0, 0};
        const long long i_t0 = clock64();
        (void)i_tfull, (void)i_drain, (void)i_store, (void)i_t0, (void)i_e;
        // 64-bit output word idx = (j * 128 + r) * 3 + w of the CTA's tile -> global address
        auto out_ptr = [&](int idx, int64_t m0, int64_t n0w, bool &ok) -> uint64_t * {
            const int j = idx / (BM * 3), rem = idx - j * (BM * 3), r = rem / 3, w = rem - r * 3;
            const int64_t row = m0 + r, gw = n0w + w;
            ok = row < a.m && gw < nw;
            return a.C + j * a.c_pstride + row * a.ldc + gw;
        };
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = cluster + ti * nclusters;
            int64_t tm, tn;
            tile_coords<RunVar<E>::GM>(tile, tiles_m, tiles_n, tm, tn);
            const int64_t m0 = tm * (2 * BM) + (int64_t)rank * BM, n0w = tn * (BN / 64);
            if (!STW && a.accumulate) {  // C0 of the words this thread writes out, into shared memory
                for (int idx = et; idx < NOUT; idx += NEPI * 32) {
                    bool ok;
                    const uint64_t *src = out_ptr(idx, m0, n0w, ok);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(stage_old + idx)),
                                 "l"(ok ? src : a.C), "r"(ok ? 8 : 0)
                                 : "memory");
                }
                cp_async_commit();
            }
            uint32_t acc[E][CH];
#pragma unroll
            for (int j = 0; j < E; ++j)
#pragma unroll
                for (int c = 0; c < CH; ++c) acc[j][c] = 0;
            // The running sums continue across tiles (the previous parity words pc / po are kept
            // per thread, which drains the same TMEM cells in every tile) and are re-initialised
            // only every reinit_tiles tiles, as late as exactness allows: a buffer takes at most
            // run_load entries of <= k_pad counts per tile.  (DIET's differenced masks and the
            // paired drains assume a reset per tile.)
            const bool reinit = (ti + 1) % reinit_tiles == 0 || ti + 1 == my_tiles;
            if constexpr (PR) {
                // paired drains: per 32-column chunk two parity words, bit 0 (field 0: group 2d)
                // and bit 11 (field 1: group 2d + 1) of each cell's low 16 bits, folded with the
                // differenced per-field masks of the selector table (no previous words kept)
                const int nd = (s.ngrp + 1) / 2;
                for (int d = 0; d < nd; ++d, ++gp) {
                    const int b = (int)(gp & 1);
                    TWR(i_tfull, mbar_wait(&bars->tfull[b], (uint32_t)((gp >> 1) & 1)));
#if GF2E_INSTR
                    const long long i_d0 = clock64();
#endif
                    tc_fence_after();
                    const uint32_t ta = tmem + lq + (b ? ACC1 : 0u) + (uint32_t)(h * (CH * 32));
                    const bool last = d + 2 >= nd;  // this buffer's last drain in the tile
                    uint32_t sel0[E], sel1[E];
                    {
                        const uint4 *sp = reinterpret_cast<const uint4 *>(selt + d * 2 * SEL_EP);
#pragma unroll
                        for (int j4 = 0; j4 < (E + 3) / 4; ++j4) {
                            const uint4 q0 = sp[j4], q1 = sp[SEL_EP / 4 + j4];
                            const uint32_t a0[4] = {q0.x, q0.y, q0.z, q0.w}, a1[4] = {q1.x, q1.y, q1.z, q1.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (4 * j4 + u < E) {
                                    sel0[4 * j4 + u] = a0[u];
                                    sel1[4 * j4 + u] = a1[u];
                                }
                        }
                    }
                    auto fold2 = [&](int c, const uint32_t (&vv)[16]) {
                        const uint32_t w0 = parity_word_packed_shl<7, 0xECA8>(vv);
                        const uint32_t w1 = parity_word_packed_shl<4, 0xFDB9>(vv);
#pragma unroll
                        for (int j = 0; j < E; ++j) acc[j][c] ^= (w0 & sel0[j]) ^ (w1 & sel1[j]);
                    };
                    uint32_t v[2][16];
                    tmem_ld32_pack16(ta, v[0]);
                    tmem_ld32_pack16(ta + 32, v[1]);
                    tmem_wait_ld();
                    if (last) {
                        st32_const(ta, PAIR_INIT);
                        st32_const(ta + 32, PAIR_INIT);
                    }
                    fold2(0, v[0]);
                    tmem_ld32_pack16(ta + 64, v[0]);
                    fold2(1, v[1]);
                    tmem_wait_ld();
                    if (last) {
                        st32_const(ta + 64, PAIR_INIT);
                        wait_st();
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(b * 8));
                    fold2(2, v[0]);
#if GF2E_INSTR
                    i_drain += (unsigned long long)(clock64() - i_d0);
#endif
                }
            } else
            for (int t = 0; t < s.ngrp; ++t, ++gp) {  // one drain per group
                const int b = (int)(gp & 1);
                const uint32_t mask = bars->gmask[t];
                TWR(i_tfull, mbar_wait(&bars->tfull[b], (uint32_t)((gp >> 1) & 1)));
#if GF2E_INSTR
                const long long i_d0 = clock64();
#endif
                tc_fence_after();
                const uint32_t ta = tmem + lq + (b ? ACC1 : 0u) + (uint32_t)(h * (CH * 32));
                // this buffer's last group before a re-initialisation (every reinit_tiles tiles)
                const bool last = t + 2 >= s.ngrp && reinit;
                uint32_t sel[E];  // all-ones for the output planes this product folds into
                if constexpr (DIET) {
                    const uint4 *sp = reinterpret_cast<const uint4 *>(selt + t * SEL_EP);
#pragma unroll
                    for (int j4 = 0; j4 < (E + 3) / 4; ++j4) {
                        const uint4 q4 = sp[j4];
                        const uint32_t qq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (4 * j4 + u < E) sel[4 * j4 + u] = qq[u];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < E; ++j) sel[j] = 0u - ((mask >> j) & 1u);
                }
                auto fold = [&](int c, uint32_t w) {
                    uint32_t pw = w;  // DIET: differenced masks, the bit-7 word as it is
                    if constexpr (!DIET) {
                        pw = w ^ pc[c];
                        pc[c] = po[c];
                        po[c] = last ? 0u : w;
                    }
#pragma unroll
                    for (int j = 0; j < E; ++j) acc[j][c] ^= pw & sel[j];
                };
                static_assert(CH == 3, "three 32-column chunks per epilogue thread");
                uint32_t v[2][16];
                tmem_ld32_pack16(ta, v[0]);
                tmem_ld32_pack16(ta + 32, v[1]);
                tmem_wait_ld();
#if GF2E_INSTR
                const long long i_e1 = clock64();
#endif
                if (last) {
                    st32_const(ta, RUN_INIT);
                    st32_const(ta + 32, RUN_INIT);
                }
                const uint32_t w0 = PARITY_WORD(v[0]);  // bit 7 of each cell
                tmem_ld32_pack16(ta + 64, v[0]);
                const uint32_t w1 = PARITY_WORD(v[1]);
                if constexpr (E > 4) {  // registers: fold before the hand-off
                    fold(0, w0);
                    fold(1, w1);
                }
#if GF2E_INSTR
                const long long i_e2 = clock64();
#endif
                tmem_wait_ld();
#if GF2E_INSTR
                const long long i_e3 = clock64();
#endif
                if (last) {
                    st32_const(ta + 64, RUN_INIT);
                    wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(b * 8));
#if GF2E_INSTR
                const long long i_e4 = clock64();
#endif
                if constexpr (E <= 4) {  // small E: fold after the hand-off (the MMA may refill
                    fold(0, w0);         // this accumulator meanwhile)
                    fold(1, w1);
                }
                fold(2, PARITY_WORD(v[0]));
#if GF2E_INSTR
                i_e[0] += (unsigned long long)(i_e1 - i_d0);
                i_e[1] += (unsigned long long)(i_e2 - i_e1);
                i_e[2] += (unsigned long long)(i_e3 - i_e2);
                i_e[3] += (unsigned long long)(i_e4 - i_e3);
                i_e[4] += (unsigned long long)(clock64() - i_e4);
#endif
#if GF2E_INSTR
                i_drain += (unsigned long long)(clock64() - i_d0);
#endif
            }
#if GF2E_INSTR
            const long long i_s0 = clock64();
#endif
            if constexpr (STW) {  // stage buffer ti & 1 -> the store warp (it freed the buffer after tile ti - 2)
                const int sb = (int)(ti & 1);
                if (ti >= 2) mbar_wait(&bars->sempty[sb], (uint32_t)(((ti >> 1) - 1) & 1));
                uint32_t *so = stage_out + sb * (kMaxE * BM * 6);
#pragma unroll
                for (int j = 0; j < E; ++j)
#pragma unroll
                    for (int c = 0; c < CH; ++c) so[(j * BM + r_cta) * 6 + h * CH + c] = acc[j][c];
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->sfull[sb]);
            } else {
            // stage: row r_cta's 96 columns of each plane -> stage_out[j][r][h*3 .. h*3+2]
            named_bar_sync(1, NEPI * 32);  // the previous tile's copy-out has read stage_out
#pragma unroll
            for (int j = 0; j < E; ++j)
#pragma unroll
                for (int c = 0; c < CH; ++c) stage_out[(j * BM + r_cta) * 6 + h * CH + c] = acc[j][c];
            if (a.accumulate) cp_async_wait<0>();
            named_bar_sync(1, NEPI * 32);
            for (int idx = et; idx < NOUT; idx += NEPI * 32) {
                bool ok;
                uint64_t *dst = out_ptr(idx, m0, n0w, ok);
                if (ok) *dst = stage_out64[idx] ^ (a.accumulate ? stage_old[idx] : 0ull);
            }
            }
#if GF2E_INSTR
            i_store += (unsigned long long)(clock64() - i_s0);
#endif
        }
#if GF2E_INSTR
        if (lane == 0 && warp == EPI_W0) {
            g_instr_run[blockIdx.x][4] = i_tfull;
            g_instr_run[blockIdx.x][5] = i_drain;
            g_instr_run[blockIdx.x][6] = i_store;
            g_instr_run[blockIdx.x][7] = (unsigned long long)(clock64() - i_t0);
            for (int i = 0; i < 5; ++i) g_instr_run[blockIdx.x][16 + i] = i_e[i];
        }
#endif
    } else if (warp == STORE_WARP) {
        if constexpr (STW) {
        // ===================== store warp =====================
        // Per tile: wait for the 8 epilogue warps' staged words (buffer ti & 1), write them out
        // as 64-bit row segments XORed with C0 (addmul; read here, 16 words in flight per lane),
        // free the buffer.
        const int64_t nw = words_for(a.n);
        constexpr int NOUT = E * BM * 3, BUFW = kMaxE * BM * 3;  // words per tile / per buffer
        const uint64_t *stage64 = reinterpret_cast<const uint64_t *>(reinterpret_cast<uint8_t *>(bars) + BARS_BYTES);
        auto word_ptr = [&](int idx, int64_t m0, int64_t n0w, bool &ok) -> uint64_t * {
            const int j = idx / (BM * 3), rem = idx - j * (BM * 3), r = rem / 3, w = rem - r * 3;
            const int64_t row = m0 + r, gw = n0w + w;
            ok = row < a.m && gw < nw;
            return a.C + j * a.c_pstride + row * a.ldc + gw;
        };
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            int64_t tm, tn;
            tile_coords<RunVar<E>::GM>(cluster + ti * nclusters, tiles_m, tiles_n, tm, tn);
            const int64_t m0 = tm * (2 * BM) + (int64_t)rank * BM, n0w = tn * (BN / 64);
            const int sb = (int)(ti & 1);
            mbar_wait_sleep(&bars->sfull[sb], (uint32_t)((ti >> 1) & 1), 64);
            const uint64_t *so = stage64 + sb * BUFW;
            constexpr int U = 16;
            for (int i0 = lane; i0 < NOUT; i0 += 32 * U) {
                uint64_t v[U];
                uint64_t *dst[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = i0 + 32 * u;
                    dst[u] = word_ptr(idx, m0, n0w, ok[u]);
                    ok[u] = ok[u] && idx < NOUT;
                    v[u] = 0ull;
                    if (a.accumulate && ok[u]) v[u] = *dst[u];
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (ok[u]) *dst[u] = v[u] ^ so[i0 + 32 * u];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->sempty[sb]);
        }
        }
    } else if (warp == MMA_WARP && rank == 0) {
        // ===================== MMA issuer (leader CTA) =====================
        const bool issuer = elect_one();
        const uint32_t st0 = smem_u32(stages);
        const uint32_t idesc = idesc_mxf4(2 * BM, BN);
        int st = 0;
        uint32_t phase = 0;
        int64_t gp = 0;
        unsigned long long i_full = 0, i_tempty = 0;
        const long long i_t0 = clock64();
        (void)i_full, (void)i_tempty, (void)i_t0;
#if GF2E_INSTR
        unsigned long long i_g0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(i_g0));
#endif
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            // drain unit: one group, or (PR) groups 2d and 2d + 1, the second one's entries with the
            // 2^11 A scale factors
            constexpr int GPD = PR ? 2 : 1;
            for (int t0 = 0; t0 < s.ngrp; t0 += GPD, ++gp) {
                const int b = (int)(gp & 1);
                TWR(i_tempty, mbar_wait(&bars->tempty[b], (uint32_t)((gp >> 1) & 1) ^ 1));
                tc_fence_after();
                const uint32_t dt = tmem + (b ? ACC1 : 0u);
                const int n0 = nks * s.gsize[t0], nall = n0 + ((PR && t0 + 1 < s.ngrp) ? nks * s.gsize[t0 + 1] : 0);
                for (int ks = 0; ks < nall; ++ks) {
                    TWR(i_full, mbar_wait(&bars->full[st], phase));
                    tc_fence_after();
                    const uint32_t sb = st0 + (uint32_t)(st * B_BYTES);
                    const uint32_t sfa = tmem + ((PR && ks >= n0) ? SFA2 : SFA);
                    if (issuer) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma2_mxf4_ts(dt, tmem + ATM0 + (uint32_t)(st * 32 + kk * 8), umma_desc_sw128(sb + kk * 32),
                                         idesc, sfa, tmem + SFB);
                        mma2_commit_both(&bars->empty[st]);
                    }
                    __syncwarp();
                    if (++st == S) {
                        st = 0;
                        phase ^= 1;
                    }

                }
                if (issuer) mma2_commit_both(&bars->tfull[b]);
                __syncwarp();
            }
        }
        __syncwarp();
#if GF2E_INSTR
        if (lane == 0) {
            unsigned long long i_g1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(i_g1));
            g_instr_run[blockIdx.x][8] = i_full;
            g_instr_run[blockIdx.x][9] = i_tempty;
            g_instr_run[blockIdx.x][10] = (unsigned long long)(clock64() - i_t0);
            g_instr_run[blockIdx.x][11] = i_g1 - i_g0;
        }
#endif
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, 512);
    }
}

int g_num_sms_run = 0;

template <int E, bool BP, bool PR>
cudaError_t launch_e(const Sched &s, const TcArgs &a, cudaStream_t st) {
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr_set[dev]) {
        cudaError_t err =
            cudaFuncSetAttribute(k_product_run<E, BP, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    const int64_t tiles = (a.m_pad / (2 * BM)) * (a.n_pad / BN);
    if (tiles == 0) return cudaSuccess;
    if (g_num_sms_run == 0) {
        cudaDeviceGetAttribute(&g_num_sms_run, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms_run <= 1) g_num_sms_run = 148;
    }
    const int64_t clusters = tiles < g_num_sms_run / 2 ? tiles : g_num_sms_run / 2;
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
    return cudaLaunchKernelEx(&cfg, k_product_run<E, BP, PR>, s, a);
}

}  // namespace

// paired drains (PR): per accumulator buffer and tile, the field-0 counts must stay below 2^11
// and F0 + 2^11 F1 below 2^23 (every count <= k_pad).  Used for the degrees in the bit mask
// GF2E_RUN_PAIR_E (default e = 3..6, where it measured faster: config 4 e=3 4.70 -> 4.24 ms,
// e=4 6.73 -> 6.61, e=6 11.81 -> 11.44; at e = 2, 7, 8 slower, profiles/r02/run_variants.txt)
bool run_pair_ok(const Sched &s, int64_t kpad) {
    static const unsigned emask = getenv("GF2E_RUN_PAIR_E") ? (unsigned)strtoul(getenv("GF2E_RUN_PAIR_E"), nullptr, 0)
                                                            : 0x78u;
    if (s.nout > 8 || !((emask >> s.nout) & 1u) || s.ngrp < 2) return false;
    int64_t f0[2] = {0, 0}, f1[2] = {0, 0};
    for (int d = 0; 2 * d < s.ngrp; ++d) {
        f0[d & 1] += s.gsize[2 * d];
        if (2 * d + 1 < s.ngrp) f1[d & 1] += s.gsize[2 * d + 1];
    }
    for (int b = 0; b < 2; ++b)
        if (f0[b] * kpad >= 2048 || f1[b] * kpad * 2048 + f0[b] * kpad >= (int64_t(1) << 23)) return false;
    return true;
}

template <int E, bool BP>
cudaError_t launch_ep(const Sched &s, const TcArgs &a, cudaStream_t st) {
    if constexpr (E <= 8)
        if (run_pair_ok(s, a.kwords * 64)) return launch_e<E, BP, true>(s, a, st);
    return launch_e<E, BP, false>(s, a, st);
}

cudaError_t launch_product_run(const Sched &s, const TcArgs &a, cudaStream_t st, bool bpre) {
#define RUN_E(EE) \
    case EE: return bpre ? launch_ep<EE, true>(s, a, st) : launch_ep<EE, false>(s, a, st);
    switch (s.nout) {
        RUN_E(1) RUN_E(2) RUN_E(3) RUN_E(4) RUN_E(5) RUN_E(6) RUN_E(7) RUN_E(8) RUN_E(9) RUN_E(10)
        default: return cudaErrorInvalidValue;
    }
#undef RUN_E
}

}  // namespace gf2e

#if GF2E_INSTR
extern "C" int gf2e_debug_instr_run(unsigned long long *out, int nblocks) {
    return (int)cudaMemcpyFromSymbol(out, gf2e::g_instr_run, sizeof(unsigned long long) * 32 * nblocks);
}
#endif

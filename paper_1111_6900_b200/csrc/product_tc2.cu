// product_tc2.cu — the fused Karatsuba product kernel on CTA PAIRS (tcgen05 cta_group::2).
//
// Reference: karatsuba_mul (poly_mul.py:245-259) -> _kara (166-220) -> mat_gf2.mul
// (mat_gf2.py:425-455) per product, then reduce_mod_f (poly_mul.py:223-242) and, for addmul,
// xor_window (mat_gf2.py:270-277).  Here C_j (^)= XOR_{t : M[j,t]} A'_t . B'_t with
// M = R_f . Gamma (the schedule, capi.cu), evaluated tile by tile; no product plane is ever
// materialised.  Each cluster of 2 CTAs owns a 256 x 256 tile of C and issues M=256 N=256
// MMAs: CTA r (cluster rank) expands A rows [128r, 128r+128) and B^T rows [128r, 128r+128)
// of the tile; the leader issues the MMAs; accumulators land in each CTA's own TMEM.
//
// Two tensor-core forms of the same GF(2) product (template parameter FP4):
//
//  int8 (kind::i8, K=32 per MMA, 128 k-bits per stage).  Bits -> bytes with ONE AND per
//    32-bit output word: A byte = a*2^i (w & 0x01010101<<i), B^T (bits reversed inside each
//    byte) byte = b*2^(7-i) (w & 0x80808080>>i); both hold k-bit 32q+8j+i in the same slot, so
//    every byte product is a*b*2^7 and the s32 accumulator is 128*count (mod 2^32): the GF(2)
//    result is bit 7.  Two TMEM accumulators (2 x 256 columns) double-buffer the epilogue.
//
//  fp4 (kind::mxf4 block-scaled e2m1, K=64 per MMA, 256 k-bits per stage, all scale factors
//    1.0 = E8M0 0x7F in TMEM).  Bits -> nibbles: A nibble i of k-bit 4j+i holds 0.5, 1, 2, 1
//    (w & 0x11111111<<i for i<3, (w>>2) & 0x22222222 for i=3); B^T is stored with bits 0 and 2
//    of every nibble swapped so its nibbles hold 2, 1, 0.5, 1 — every product is exactly 1.0.
//    fp32 accumulation of 0/1 products is exact (probe: tools/fp4_probe.py, to 2^24); the
//    accumulator starts at 65536.0f, so for counts < 2^16 the pattern is 0x47800000 + (count<<7)
//    and the parity is again bit 7.  K is processed in chunks of <= 32768 bits (count < 2^16);
//    one 256-column accumulator (the other 256 TMEM columns hold the scale factors); the
//    epilogue re-initialises it to 65536.0f after each read-out.  2x the int8 rate, half the
//    expanded bytes per k-bit.
//
//  fp4 paired (template PAIR, k < 2048): two consecutive products share the accumulator; the
//    second one's A scale factors are 2^11 (E8M0 0x8A, TMEM columns 320..383).  The
//    accumulator starts at 2^23 (ulp 1), so its low 16 bits are c0 + 2^11 c1 with c0, c1 <=
//    k < 2^11: the parities are bits 0 and 11, and one TMEM drain serves two products.  Exact
//    and parity-tested; at k = 256 it matches (does not beat) the double-buffered int8 form,
//    which stays the default below k = 2048 (the drain, not the MMA, bounds short k).
//
// Warp roles (448 threads per CTA, 1 CTA / SM):
//   warps 0-3   expanders: expand this CTA's A and B^T rows of each stage into the UMMA
//               K-major SWIZZLE_128B layout, fence.proxy.async, arrive on the leader's full[s]
//   warps 4-11  epilogue: tcgen05.ld pack::16b, parity via sign-replicating PRMT, fold into
//               E register-resident output planes (the columns of M), store the tile once
//   warp 12     MMA issuer (leader CTA, one elected lane of the warp)
//   warp 13     loader: cp.async.bulk of the stage-tiled bit tiles into a ring (mbarrier tx),
//               one elected lane issuing
// Synchronisation across the pair:
//   full[s]   (leader)   <- 4 expander warps x 2 CTAs (relaxed remote arrive after the fence;
//                           release.cluster would compile to MEMBAR.ALL.GPU)
//   empty[s]  (each CTA) <- tcgen05.commit multicast to both CTAs
//   tfull[b]  (each CTA) <- tcgen05.commit multicast to both CTAs
//   tempty[b] (leader)   <- 8 epilogue warps x 2 CTAs (remote arrive)
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace gf2e {
namespace {
using namespace tc;

constexpr int BM = 128;   // rows per CTA (tile = 2 x BM)
#ifndef GF2E_FP4_S
#define GF2E_FP4_S 5
#endif
#ifndef GF2E_ATMEM
#define GF2E_ATMEM 1
#endif
constexpr int DMAX = 16;  // bit-tile ring slots (upper bound)
constexpr int SMAX = 8;
constexpr int BARS_BYTES = 1024;  // Bars (static_assert below)      // expanded operand stages (32 KiB each: one 128-byte swizzle row per operand row)
#ifndef GF2E_INSTR
#define GF2E_INSTR 0
#endif
#if GF2E_INSTR
// dev-only: per-CTA cycle counters [block][16] (1: per-wait counters, 2: totals only)
__device__ unsigned long long g_instr[1024][16];
#endif
#if GF2E_INSTR == 1
#define TW(acc, stmt)                          \
    do {                                       \
        const long long _t0 = clock64();       \
        stmt;                                  \
        acc += (unsigned long long)(clock64() - _t0); \
    } while (0)
#else
#define TW(acc, stmt) stmt
#endif
#ifndef GF2E_LOAD_SLEEP_NS
#define GF2E_LOAD_SLEEP_NS 500
#endif
constexpr uint32_t LOAD_SLEEP_NS = GF2E_LOAD_SLEEP_NS;  // bulk loader waiting for a free bit slot
#ifndef GF2E_EXP_SLEEP_NS
#define GF2E_EXP_SLEEP_NS 64
#endif
constexpr uint32_t EXP_SLEEP_NS = GF2E_EXP_SLEEP_NS;  // expanders waiting for a free operand stage
#ifndef GF2E_IDLE_SLEEP_NS
#define GF2E_IDLE_SLEEP_NS 500
#endif
constexpr uint32_t IDLE_SLEEP_NS = GF2E_IDLE_SLEEP_NS;  // epilogue (long k only, see below)
#ifndef GF2E_SPLITX
#define GF2E_SPLITX 1
#endif
// Warp roles (14 warps): expanders 0 .. NPW-1, epilogue NPW .. 11, MMA 12, loader 13.  The
// fp4 form with A in TMEM (Cfg::SPLIT) uses 8 expander warps — 0-3 expand A rows into TMEM,
// 4-7 B^T rows into shared memory — and 4 epilogue warps (one per TMEM lane quarter, all 256
// columns, the E x 8 output words kept in shared memory): its long accumulations leave the
// epilogue idle, while the MMA waited on expansion.  The other forms use 4 expander warps
// (A and B^T rows) and 8 epilogue warps (lane quarter x column half).
constexpr int NPW = 4;  // expander warps (non-split forms)
constexpr int NEW = 8;  // epilogue warps (non-split forms)
#ifndef GF2E_TC2_GROUP_M
#define GF2E_TC2_GROUP_M 8
#endif
constexpr int GROUP_M = GF2E_TC2_GROUP_M;  // tile rasterisation: row-tiles per column sweep (L2 reuse)
constexpr int MMA_WARP = NPW + NEW;
constexpr int LOAD_WARP = MMA_WARP + 1;
constexpr int NTHREADS = (NPW + NEW + 2) * 32;
constexpr int A_BYTES = BM * 128;
constexpr int TMEM_COLS = 512;
constexpr uint32_t FP4_ACC_INIT = 0x47800000u;  // 65536.0f
constexpr uint32_t FP4_PAIR_INIT = 0x4B000000u;  // 2^23: ulp 1, count sum in mantissa bits 0..22
constexpr uint32_t SF_ONE = 0x7F7F7F7Fu;         // E8M0 1.0
constexpr uint32_t SF_2P11 = 0x8A8A8A8Au;        // E8M0 2^11 (second product of a pair)
constexpr int FP4_CHUNK_STAGES = 32768 / 256;   // k-bits per accumulation chunk / bits per stage

template <bool FP4, bool PAIR, bool WIDE = false>
struct Cfg {
    // tile N = 256: two 256-column accumulators for int8; one for fp4 (scale factors in the
    // other 256 TMEM columns).  (An N = 192 double-buffered paired form measured slower: the
    // TMEM read-out competes with the MMAs, so overlap buys little at k < 2048.)
    static constexpr int BN = 256;
    // fp4 (not paired): the expanded A operand lives in TMEM (tcgen05.st by the expanders,
    // tcgen05.mma A-from-TMEM), so shared memory carries only B: half the shared-memory traffic
    static constexpr bool ATMEM = FP4 && !PAIR && GF2E_ATMEM;
    static constexpr int A_SMEM = ATMEM ? 0 : A_BYTES;
    static constexpr int BNH = BN / 2;          // B^T rows per CTA
    static constexpr int B_BYTES = BNH * 128;
    static constexpr int STAGE_BYTES = A_SMEM + B_BYTES;
    static constexpr int BK = FP4 ? 256 : 128;  // k-bits per stage (= one 128-byte row of operand)
    static constexpr int KW = BK / 64;          // bit words per tile row per stage
#ifndef GF2E_ATMEM_S
#define GF2E_ATMEM_S 7
#endif
    static constexpr int S = ATMEM ? GF2E_ATMEM_S : FP4 ? GF2E_FP4_S : 5;  // operand stages (TMEM A: S x 32 columns)
#ifndef GF2E_FP4_D
#define GF2E_FP4_D 6
#endif
#ifndef GF2E_ATMEM_D
#define GF2E_ATMEM_D 6
#endif
    static constexpr int D = ATMEM ? GF2E_ATMEM_D : FP4 ? GF2E_FP4_D : 8;  // bit-tile ring depth
    static constexpr int BITS_A = BM * (BK / 8);
    static constexpr int BITS_BYTES = (BM + BNH) * (BK / 8);
    static constexpr int NBUF = FP4 ? 1 : 2;  // TMEM accumulators
    static constexpr bool SPLIT = ATMEM && WIDE && GF2E_SPLITX;  // k >= 8192 (host: kFormFp4Long)
    static constexpr int NPW = SPLIT ? 8 : 4;             // expander warps
    static constexpr int NEW = SPLIT ? 4 : 8;             // epilogue warps
    static constexpr int EPI_W0 = NPW;
    static_assert(NPW + NEW == MMA_WARP, "warp roles");
    static constexpr int CH = BN * 4 / NEW / 32;          // 32-column chunks per epilogue warp
    static constexpr int ACC_SMEM = SPLIT ? kMaxE * CH * 128 * 4 : 0;  // epilogue output words
    // scale-factor TMEM columns (fp4): A (first / second product of a pair) and B
    static constexpr uint32_t SFA0 = ATMEM ? 256 + 32 * S : 256, SFA1 = 320, SFB = ATMEM ? SFA0 + (S >= 7 ? 16 : 32) : 384;
    static_assert(!ATMEM || SFB + (S >= 7 ? 16 : 32) <= 512, "TMEM columns: A stages overlap the scale factors");
    static constexpr uint32_t ATM0 = 256;  // TMEM column of A stage 0 (ATMEM)
    static constexpr int SMEM_BYTES = S * STAGE_BYTES + D * BITS_BYTES + BARS_BYTES + ACC_SMEM + 1024;
    static_assert(SMEM_BYTES <= 232448, "shared memory");
    static_assert(NBUF * BN <= (FP4 ? 384 : 512), "accumulators overlap the scale factors");
};

struct __align__(8) Bars {
    uint64_t full[SMAX], empty[SMAX], tfull[2], tempty[2], bfull[DMAX], bempty[DMAX];
    uint32_t tmem_base;
    uint16_t outmask[kMaxProducts];
};
static_assert(sizeof(Bars) <= BARS_BYTES, "barrier block");

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

// fp4 expansion of one 256-bit row of a stage into its 128-byte swizzle row: u32 word q of
// the row gives chunk q (four u32 = 32 nibbles; nibble j of word i <-> k-bit 32q + 4j + i)
template <bool kB>
__device__ __forceinline__ void expand_row_fp4(uint8_t *tile, int r, uint4 lo, uint4 hi) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t x = w[q];
        const uint32_t o3 = (x >> 2) & 0x22222222u;
        const uint4 o = kB ? make_uint4(x & 0x44444444u, x & 0x22222222u, x & 0x11111111u, o3)
                           : make_uint4(x & 0x11111111u, x & 0x22222222u, x & 0x44444444u, o3);
        *reinterpret_cast<uint4 *>(tile + swz(r, q)) = o;
    }
}

// A row of one fp4 stage into TMEM (this thread's lane): 32 columns = the 8 chunks of
// expand_row_fp4 in order (column 4q + i = word i of chunk q)
__device__ __forceinline__ void expand_row_fp4_tmem(uint32_t taddr, uint4 lo, uint4 hi) {
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

__device__ __forceinline__ void tmem_st32_const(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
            taddr),
        "r"(v)
        : "memory");
}
// 8 columns per instruction: tcgen05.st takes its sources as consecutive registers, so the
// x32 form would pin 32 registers in the epilogue (spills at E >= 7)
__device__ __forceinline__ void tmem_st8_const(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// block-scaled instruction descriptor: e2m1 x e2m1, E8M0 scales, K-major, K=64
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
// A operand from TMEM (tcgen05 "TS" form)
__device__ __forceinline__ void mma2_mxf4_ts(uint32_t d, uint32_t at, uint64_t bd, uint32_t idesc, uint32_t sfa,
                                             uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, 1, 1;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "r"(at), "l"(bd), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}
__device__ __forceinline__ void mma2_mxf4(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, 1, 1;\n\t"  // always accumulate: D starts at 65536.0f
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}

template <int E, bool FP4, bool PAIR, bool WIDE>
__global__ void __launch_bounds__(NTHREADS, 1) k_product_tc2(const Sched s, const TcArgs a) {
    using C = Cfg<FP4, PAIR, WIDE>;
    constexpr int BN = C::BN, BNH = C::BNH, STAGE_BYTES = C::STAGE_BYTES;
    static_assert(FP4 || !PAIR, "product pairing is an fp4 form");
    // PAIR (k < 2048): two products share one accumulator, the second scaled by 2^11 through
    // its E8M0 scale factors, so one TMEM drain serves two products (see the header comment)
    constexpr uint32_t ACC_INIT = PAIR ? FP4_PAIR_INIT : FP4_ACC_INIT;
    constexpr int STEP = PAIR ? 2 : 1;
    extern __shared__ uint8_t smem_raw[];
    // keep the shared state space visible to the compiler (STS/LDS, not generic ST/LD)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *stages = smem;
    uint8_t *bits = smem + C::S * STAGE_BYTES;
    Bars *bars = reinterpret_cast<Bars *>(bits + C::D * C::BITS_BYTES);
    constexpr int S = C::S;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int64_t tiles_n = a.n_pad / BN;
    const int64_t tiles_m = a.m_pad / (2 * BM);
    const int64_t ntiles = tiles_m * tiles_n;
    const int64_t my_tiles = ntiles > cluster ? (ntiles - cluster + nclusters - 1) / nclusters : 0;
    const int nks = (int)(a.kwords / C::KW);
    // accumulation chunks per product: int8 wraps harmlessly mod 2^32; fp4 keeps count < 2^16
    const int chunk = (FP4 && !PAIR) ? FP4_CHUNK_STAGES : nks;
    const int nchunks = (nks + chunk - 1) / chunk;
    const int64_t total = my_tiles * (int64_t)s.nprod * nks;
    // short k (few stages per accumulation) makes the epilogue hand-off latency-critical
    const uint32_t idle_ns = nks >= 16 ? IDLE_SLEEP_NS : 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&bars->full[i], 2 * C::NPW);
            mbar_init(&bars->empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->tfull[i], 1);
            mbar_init(&bars->tempty[i], 2 * C::NEW);
        }
        for (int i = 0; i < C::D; ++i) {
            mbar_init(&bars->bfull[i], 1);
            mbar_init(&bars->bempty[i], C::NPW);
        }
        mbar_fence_init();
    }
    if (threadIdx.x < kMaxProducts) bars->outmask[threadIdx.x] = s.outmask[threadIdx.x];
    if (warp == MMA_WARP) tmem_alloc2(&bars->tmem_base, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    if (FP4 && warp >= C::EPI_W0 && warp < C::EPI_W0 + 4) {
        // scale factors (columns 256..511: every byte E8M0 1.0) and the first accumulator init
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        for (int c = (int)C::SFA0; c < 512; c += 32)
            tmem_st32_const(tmem + lb + c, (PAIR && c >= (int)C::SFA1 && c < (int)C::SFB) ? SF_2P11 : SF_ONE);
        for (int c = 0; c < C::NBUF * BN; c += 32) tmem_st32_const(tmem + lb + c, ACC_INIT);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // barriers and TMEM of both CTAs ready before any remote arrive / MMA
    tc_fence_after();

    unsigned long long i_empty = 0, i_bfull = 0, i_tfull = 0, i_tempty = 0, i_full = 0;
    (void)i_empty, (void)i_bfull, (void)i_tfull, (void)i_tempty, (void)i_full;
#if GF2E_INSTR
    const long long i_t0 = clock64();
    unsigned long long i_g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(i_g0));
#endif
    if (warp < C::NPW) {
        // ===================== expanders (both CTAs) =====================
        // bit tiles arrive by bulk copy (loader warp); these warps keep no global loads in
        // flight, so the per-stage fence.proxy.async (MEMBAR.ALL.CTA) only drains their STS.
        const int p = threadIdx.x & 127;  // A row and B^T row of this CTA's half
        const bool doA = !C::SPLIT || warp < 4, doB = !C::SPLIT || warp >= 4;  // SPLIT: A or B^T rows
        const uint32_t full_leader = mapa(smem_u32(&bars->full[0]), 0);
        int slot = 0, st = 0;
        uint32_t bph = 0, phase = 0;
        // bit words of one stage for this thread: A row then B^T row (fp4: 2 x 32 B, int8: 2 x 16 B)
        constexpr int NQ = FP4 ? 4 : 2;
        uint4 cur[NQ];
        auto load_bits = [&](int sl, uint4 (&v)[NQ]) {
            // slab layout (tc_tile_word): [KW/2 slabs][rows][16 B]
            const uint8_t *bs = bits + sl * C::BITS_BYTES + p * 16;
#pragma unroll
            for (int i = 0; i < NQ / 2; ++i) {
                if (doA) v[i] = *reinterpret_cast<const uint4 *>(bs + i * (BM * 16));
                if (doB && p < BNH) v[NQ / 2 + i] = *reinterpret_cast<const uint4 *>(bs + C::BITS_A + i * (BNH * 16));
            }
        };
        if (total > 0) {
            mbar_wait(&bars->bfull[0], 0);
            load_bits(0, cur);
        }
        for (int64_t it = 0; it < total; ++it) {
            TW(i_empty, mbar_wait_sleep(&bars->empty[st], phase ^ 1, EXP_SLEEP_NS));
            uint8_t *sa = stages + st * STAGE_BYTES;
            if constexpr (C::ATMEM) {
                if (doA) {
                    expand_row_fp4_tmem(tmem + ((uint32_t)((warp & 3) * 32) << 16) + C::ATM0 + (uint32_t)(st * 32),
                                        cur[0], cur[1]);
                }
                if (doB) expand_row_fp4<true>(sa, p, cur[2], cur[3]);
                if (doA) {
                    tmem_wait_st();
                    tc_fence_before();
                }
            } else if constexpr (FP4) {
                if (doA) expand_row_fp4<false>(sa, p, cur[0], cur[1]);
                if (doB && p < BNH) expand_row_fp4<true>(sa + A_BYTES, p, cur[2], cur[3]);
            } else {
                if (doA) expand_row<false>(sa, p, cur[0]);
                if (doB) expand_row<true>(sa + A_BYTES, p, cur[1]);
            }
            if (!C::ATMEM || doB) fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_cluster(full_leader + (uint32_t)(st * 8));
                // this slot's bits were consumed by the expansion above (data dependence), so
                // the loader may overwrite it: no read-before-overwrite race on bits
                mbar_arrive(&bars->bempty[slot]);
            }
            if (++slot == C::D) {
                slot = 0;
                bph ^= 1;
            }
            // next stage's bits: read now so the shared-memory latency overlaps the empty wait
            // (reading them before this stage's expansion was measured slower)
            if (it + 1 < total) {
                TW(i_bfull, mbar_wait(&bars->bfull[slot], bph));
                load_bits(slot, cur);
            }
            if (++st == S) {
                st = 0;
                phase ^= 1;
            }
        }
    } else if (warp == LOAD_WARP) {
        // ===================== bit-tile loader (both CTAs, one elected lane) =====================
        // the whole warp walks the stages (addresses warp-uniform), one lane issues the copies
        const bool issuer = elect_one();
        const int64_t KS = a.kwords / C::KW;  // k-stages per row block
        const int64_t tile_words = BM * C::KW, tile_words_b = BNH * C::KW;
        const uint32_t bits_s = smem_u32(bits);
        int slot = 0;
        uint32_t bph = 0;
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = cluster + ti * nclusters;
            int64_t tm, tn;
            tile_coords(tile, tiles_m, tiles_n, tm, tn);
            const int64_t rbA = tm * 2 + rank;  // 128-row block of A
            const int64_t rbB = tn * 2 + rank;  // BNH-row block of B^T
            for (int t = 0; t < s.nprod; ++t) {
                const uint64_t *Ab = a.Ac + t * a.a_pstride + rbA * KS * tile_words;
                const uint64_t *Bb = a.Bt + t * a.b_pstride + rbB * KS * tile_words_b;
                for (int ks = 0; ks < nks; ++ks) {
                    mbar_wait_sleep(&bars->bempty[slot], bph ^ 1, LOAD_SLEEP_NS);
                    const uint32_t dst = bits_s + (uint32_t)(slot * C::BITS_BYTES);
                    if (issuer) {
                        mbar_arrive_expect_tx(&bars->bfull[slot], C::BITS_BYTES);
                        bulk_g2s(dst, Ab + ks * tile_words, C::BITS_A, &bars->bfull[slot]);
                        bulk_g2s(dst + C::BITS_A, Bb + ks * tile_words_b, C::BITS_BYTES - C::BITS_A,
                                 &bars->bfull[slot]);
                    }
                    __syncwarp();
                    if (++slot == C::D) {
                        slot = 0;
                        bph ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp < MMA_WARP) {
        // ===================== epilogue (both CTAs) =====================
        const int ew = warp - C::EPI_W0;
        const int et = ew * 32 + lane;  // epilogue thread index
        const int q = warp & 3;  // TMEM lane quarter (hardware: warp id % 4)
        const int h = ew >> 2;   // column group (two halves with 8 epilogue warps, one with 4)
        constexpr int EPI_COLS = C::CH * 32;
        const int row_local = (int)rank * BM + q * 32 + lane;
        const int64_t nw = words_for(a.n);
        const uint32_t tempty_leader = mapa(smem_u32(&bars->tempty[0]), 0);
        int64_t gp = 0;  // accumulator hand-offs seen (products x chunks)
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            const int64_t tile = cluster + ti * nclusters;
            int64_t tm, tn;
            tile_coords(tile, tiles_m, tiles_n, tm, tn);
            const int64_t m0 = tm * (2 * BM), n0 = tn * BN;
            constexpr int CH = C::CH;
            // output words: registers, or shared memory for the 4-warp epilogue (E x 8 words)
            uint32_t acc_r[C::SPLIT ? 1 : E][C::SPLIT ? 1 : CH];
            uint32_t *acc_s = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(bars) + BARS_BYTES) + et;
            auto ACC = [&](int j, int c) -> uint32_t & {
                if constexpr (C::SPLIT)
                    return acc_s[(j * CH + c) * 128];
                else
                    return acc_r[j][c];
            };
#pragma unroll
            for (int j = 0; j < E; ++j)
#pragma unroll
                for (int c = 0; c < CH; ++c) ACC(j, c) = 0;
            for (int t = 0; t < s.nprod; t += STEP) {
                const uint32_t mask = bars->outmask[t];
                const uint32_t mask1 = (PAIR && t + 1 < s.nprod) ? bars->outmask[t + 1] : 0u;
                for (int ch = 0; ch < nchunks; ++ch, ++gp) {
                    const int buf = (int)(gp % C::NBUF);
                    TW(i_tfull, mbar_wait_sleep(&bars->tfull[buf], (uint32_t)((gp / C::NBUF) & 1), idle_ns));
                    tc_fence_after();
                    // chunks per tcgen05.ld: 2 (x32: 64 columns, half the load/wait round trips of
                    // the drain) where the output words live in shared memory (long-k form) or
                    // the accumulator is not re-initialised (int8); 1 (x16: 32 columns) for the
                    // other register-resident forms (register pressure)
                    constexpr int LB = (C::SPLIT || !FP4) ? 2 : 1;
#pragma unroll
                    for (int c0 = 0; c0 < CH; c0 += LB) {
                        uint32_t v[LB][16];
                        const uint32_t ta0 =
                            tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + h * EPI_COLS + c0 * 32);
                        if constexpr (LB == 2)
                            tmem_ld64_pack16(ta0, *reinterpret_cast<uint32_t(*)[32]>(&v[0][0]));
                        else
                            tmem_ld32_pack16(ta0, v[0]);
                        tmem_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < LB; ++cc) {
                            const int c = c0 + cc;
                            if constexpr (PAIR) {
                                // low 16 bits of each cell = c0 + 2^11 c1: parities at bits 0 and 11
                                const uint32_t pw0 = parity_word_packed_shl<7, 0xECA8>(v[cc]);
                                const uint32_t pw1 = parity_word_packed_shl<4, 0xFDB9>(v[cc]);
#pragma unroll
                                for (int j = 0; j < E; ++j)
                                    ACC(j, c) ^=
                                        (pw0 & (0u - ((mask >> j) & 1u))) ^ (pw1 & (0u - ((mask1 >> j) & 1u)));
                            } else {
                                const uint32_t pw = parity_word_packed(v[cc]);
                                if constexpr (C::SPLIT) {
#pragma unroll
                                    for (int j = 0; j < E; ++j)
                                        if ((mask >> j) & 1u) ACC(j, c) ^= pw;
                                } else {
#pragma unroll
                                    for (int j = 0; j < E; ++j) ACC(j, c) ^= pw & (0u - ((mask >> j) & 1u));
                                }
                            }
                            if (FP4) {
                                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) +
                                                    (uint32_t)(buf * BN + h * EPI_COLS + c * 32);
#pragma unroll
                                for (int c8 = 0; c8 < 32; c8 += 8) tmem_st8_const(ta + c8, ACC_INIT);
                            }
                        }
                    }
                    if (FP4) tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(buf * 8));
                }
            }
            const int64_t row = m0 + row_local;
            if (row < a.m) {
#pragma unroll
                for (int wp = 0; wp < CH / 4; ++wp) {  // pairs of 64-bit words of this warp's columns
                    const int64_t w0 = (n0 >> 6) + (CH / 2) * h + 2 * wp;
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
                                const uint64_t x0 =
                                    ((uint64_t)ACC(j, 4 * wp) | ((uint64_t)ACC(j, 4 * wp + 1) << 32)) ^ old[jj][0];
                                const uint64_t x1 =
                                    ((uint64_t)ACC(j, 4 * wp + 2) | ((uint64_t)ACC(j, 4 * wp + 3) << 32)) ^ old[jj][1];
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
        }
    } else if (warp == MMA_WARP && rank == 0) {
        // ===================== MMA issuer (leader CTA, one elected thread) =====================
        // The whole warp runs the loop, so the descriptors and TMEM addresses are warp-uniform
        // (uniform registers); one elected lane issues the MMAs and commits.
        const bool issuer = elect_one();
        int64_t gp = 0;
        int st = 0;
        uint32_t phase = 0;
        const uint32_t st0 = smem_u32(stages);
        const uint32_t idesc = FP4 ? idesc_mxf4(2 * BM, BN) : idesc_i8(2 * BM, BN);
        static_assert(BN % 16 == 0 && BN <= 256, "cta_group::2 MMA N");
        for (int64_t ti = 0; ti < my_tiles; ++ti) {
            for (int t = 0; t < s.nprod; t += STEP) {
                const int units = (PAIR && t + 1 < s.nprod) ? 2 : 1;
                for (int ch = 0; ch < nchunks; ++ch, ++gp) {
                    const int buf = (int)(gp % C::NBUF);
                    TW(i_tempty, mbar_wait(&bars->tempty[buf], (uint32_t)((gp / C::NBUF) & 1) ^ 1));
                    tc_fence_after();
                    const uint32_t dt = tmem + (uint32_t)(buf * BN);
                    const int ks1 = (ch + 1) * chunk < nks ? (ch + 1) * chunk : nks;
                    for (int u = 0; u < units; ++u) {
                        const uint32_t sfa = tmem + (u ? C::SFA1 : C::SFA0);
                        for (int ks = ch * chunk; ks < ks1; ++ks) {
                            TW(i_full, mbar_wait(&bars->full[st], phase));
                            tc_fence_after();
                            const uint32_t sa = st0 + (uint32_t)(st * STAGE_BYTES);
                            const uint32_t sb = sa + C::A_SMEM;
                            if (issuer) {
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    const uint64_t ad = umma_desc_sw128(sa + kk * 32),
                                                   bd = umma_desc_sw128(sb + kk * 32);
                                    if constexpr (C::ATMEM)
                                        mma2_mxf4_ts(dt, tmem + C::ATM0 + (uint32_t)(st * 32 + kk * 8), bd, idesc, sfa,
                                                     tmem + C::SFB);
                                    else if constexpr (FP4)
                                        mma2_mxf4(dt, ad, bd, idesc, sfa, tmem + C::SFB);
                                    else
                                        mma2_i8(dt, ad, bd, idesc, (ks != ch * chunk) | kk);
                                }
                                mma2_commit_both(&bars->empty[st]);
                            }
                            __syncwarp();
                            if (++st == S) {
                                st = 0;
                                phase ^= 1;
                            }
                        }
                    }
                    if (issuer) mma2_commit_both(&bars->tfull[buf]);
                    __syncwarp();
                }
            }
        }
        __syncwarp();
    }
#if GF2E_INSTR
    {
        const unsigned long long i_tot = (unsigned long long)(clock64() - i_t0);
        if (lane == 0 && warp == 0) {
            g_instr[blockIdx.x][0] = i_empty;
            g_instr[blockIdx.x][1] = i_bfull;
            g_instr[blockIdx.x][2] = i_tot;
        }
        if (lane == 0 && warp == C::EPI_W0) {
            g_instr[blockIdx.x][3] = i_tfull;
            g_instr[blockIdx.x][4] = i_tot;
        }
        if (lane == 0 && warp == MMA_WARP) {
            g_instr[blockIdx.x][5] = i_full;
            g_instr[blockIdx.x][6] = i_tempty;
            g_instr[blockIdx.x][7] = i_tot;
            unsigned long long i_g1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(i_g1));
            g_instr[blockIdx.x][8] = i_g1 - i_g0;
        }
    }
#endif

    tc_fence_before();
    __syncthreads();
    cluster_sync();  // all MMAs of the pair retired (every epilogue saw its last tfull)
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc2(tmem, TMEM_COLS);
    }
}

int g_num_sms2 = 0;

template <int E, bool FP4, bool PAIR, bool WIDE>
cudaError_t launch_e(const Sched &s, const TcArgs &a, cudaStream_t st) {
    const int smem = Cfg<FP4, PAIR, WIDE>::SMEM_BYTES;
    // once per instantiation and device (idempotent, so a race is harmless)
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= kMaxDevices || !attr_set[dev]) {
        cudaError_t err =
            cudaFuncSetAttribute(k_product_tc2<E, FP4, PAIR, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    const int64_t tiles = (a.m_pad / (2 * BM)) * (a.n_pad / Cfg<FP4, PAIR, WIDE>::BN);
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
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_product_tc2<E, FP4, PAIR, WIDE>, s, a);
}

template <bool FP4, bool PAIR, bool WIDE>
cudaError_t launch_any(const Sched &s, const TcArgs &a, cudaStream_t st) {
    switch (s.nout) {
        case 1: return launch_e<1, FP4, PAIR, WIDE>(s, a, st);
        case 2: return launch_e<2, FP4, PAIR, WIDE>(s, a, st);
        case 3: return launch_e<3, FP4, PAIR, WIDE>(s, a, st);
        case 4: return launch_e<4, FP4, PAIR, WIDE>(s, a, st);
        case 5: return launch_e<5, FP4, PAIR, WIDE>(s, a, st);
        case 6: return launch_e<6, FP4, PAIR, WIDE>(s, a, st);
        case 7: return launch_e<7, FP4, PAIR, WIDE>(s, a, st);
        case 8: return launch_e<8, FP4, PAIR, WIDE>(s, a, st);
        case 9: return launch_e<9, FP4, PAIR, WIDE>(s, a, st);
        case 10: return launch_e<10, FP4, PAIR, WIDE>(s, a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_product_tc2(const Sched &s, const TcArgs &a, int form, cudaStream_t st) {
    switch (form) {
        case kFormI8: return launch_any<false, false, false>(s, a, st);
        case kFormFp4: return launch_any<true, false, false>(s, a, st);
        case kFormFp4Long: return launch_any<true, false, true>(s, a, st);
        case kFormFp4Pair: return launch_any<true, true, false>(s, a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gf2e

#if GF2E_INSTR
extern "C" int gf2e_debug_instr(unsigned long long *out, int nblocks) {
    return (int)cudaMemcpyFromSymbol(out, gf2e::g_instr, sizeof(unsigned long long) * 16 * nblocks);
}
#endif

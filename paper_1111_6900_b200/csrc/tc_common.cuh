// tc_common.cuh — device helpers shared by the tcgen05 product kernels (product_tc*.cu):
// operand expansion into the UMMA K-major SWIZZLE_128B layout, the bit-7 parity packer of
// the epilogue, and cluster (2-SM) PTX wrappers.
#pragma once
#include "common.cuh"

namespace gf2e {
namespace tc {

__device__ __forceinline__ uint32_t swz(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

template <bool kReversed>
__device__ __forceinline__ void expand_row(uint8_t *tile, int r, uint4 w4) {
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = w[q] & (kReversed ? (0x80808080u >> i) : (0x01010101u << i));
        *reinterpret_cast<uint4 *>(tile + swz(r, 2 * q)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4 *>(tile + swz(r, 2 * q + 1)) = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

// parity_word from pack::16b registers (v[i] = column 2i | column 2i+1 << 16): PRMT with
// sign-replicating selectors turns the bit-7 of 4 columns into 4 byte masks (0x00 / 0xFF) in
// one instruction, and one LOP3 merges them: 16 ALU ops per 32 columns; bit 8b+g of the
// result = column 4g+b (the B^T row permutation tc_b_row_inv undoes this order).
__device__ __forceinline__ uint32_t parity_word_packed(const uint32_t (&v)[16]) {
    uint32_t r = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        uint32_t w;  // byte b = sign-replicated bit 7 of column 4g+b (prmt selector msb = replicate)
        asm("prmt.b32 %0, %1, %2, 0xECA8;" : "=r"(w) : "r"(v[2 * g]), "r"(v[2 * g + 1]));
        r |= w & (0x01010101u << g);
    }
    return r;
}

// The same for the paired fp4 form: the parity sits at bit SH' of each 16-bit half; shifting
// left by SHIFT moves it to bit 7 of a byte, SEL picks (and sign-replicates) that byte of each
// of the four halves: 0xECA8 = low bytes (bits 0 + 7), 0xFDB9 = high bytes (bits 11 + 4).
template <int SHIFT, uint32_t SEL>
__device__ __forceinline__ uint32_t parity_word_packed_shl(const uint32_t (&v)[16]) {
    uint32_t r = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        uint32_t w;
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(v[2 * g] << SHIFT), "r"(v[2 * g + 1] << SHIFT), "n"(SEL));
        r |= w & (0x01010101u << g);
    }
    return r;
}

// TMEM column j (= B smem row j) of every 32-column group holds tile column b_row_perm(j).
__host__ __device__ __forceinline__ int b_row_perm(int j) {
    const int g = (j & 31) >> 2, b = j & 3;
    return (j & ~31) | (8 * b + g);
}


// ---- cluster (CTA pair) helpers ----------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of this cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Remote arrive on the pair leader's barrier.  Relaxed on purpose: release.cluster compiles
// to MEMBAR.ALL.GPU, which would drain this thread's in-flight cp.async prefetches every
// stage.  Producers order their st.shared before it with fence.proxy.async.shared::cta
// (MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC.S); the epilogue's TMEM reads are complete after
// tcgen05.wait::ld.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, both CTAs: 2 x 128 rows] . B[smem, both CTAs: 2 x N/2 rows]^T
__device__ __forceinline__ void mma2_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at this smem offset in both CTAs of the pair once all prior MMAs finish
__device__ __forceinline__ void mma2_commit_both(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

}  // namespace tc
}  // namespace gf2e

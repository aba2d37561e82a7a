// Dev: does tcgen05.cp.cta_group::1.128x256b (shared memory -> TMEM) read a K-major
// SWIZZLE_128B operand stage (the layout the B^T stages already use) row r -> TMEM lane r,
// 32-byte slice kk -> columns 8kk..8kk+7?  Fills 128 rows x 128 B with word (r << 8 | c) at
// column c, copies with 4 x 128x256b, reads back with tcgen05.ld and counts mismatches.
// Variant 1: the same data in the no-swizzle canonical layout (8-row x 16-byte core matrices,
// per 32-byte slice: LBO 128 B between the two 16-byte chunks, SBO 256 B between row groups).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1111_6900_b200/csrc tools/tmem_cp_test.cu
#include <cstdio>
#include <cstdint>
#include "common.cuh"

using namespace gf2e;

__device__ __forceinline__ uint32_t swz128(int r, int c16) { return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c16 ^ (r & 7)) << 4)); }

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ULL << 46);
}

__global__ void k_cp_test(int variant, int *bad, uint32_t *first) {
    __shared__ __align__(1024) uint8_t st[16384];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int r = threadIdx.x, warp = r >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (r == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    for (int c = 0; c < 32; ++c) {
        const uint32_t w = ((uint32_t)r << 8) | (uint32_t)c;
        uint32_t off;
        if (variant == 0) {
            off = swz128(r, c >> 2) + (c & 3) * 4;
        } else {  // [kk][g][j][row][16 B]: kk = c / 8, j = (c / 4) & 1
            const int kk = c >> 3, j = (c >> 2) & 1;
            off = kk * 4096 + (r >> 3) * 256 + j * 128 + (r & 7) * 16 + (c & 3) * 4;
        }
        *reinterpret_cast<uint32_t *>(st + off) = w;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    if (r == 0) {
        for (int kk = 0; kk < 4; ++kk) {
            const uint64_t d = variant == 0 ? umma_desc_sw128(smem_u32(st) + kk * 32)
                                            : desc_none(smem_u32(st) + kk * 4096, 128, 256);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + kk * 8), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) {
        const uint32_t want = ((uint32_t)r << 8) | (uint32_t)c;
        if (v[c] != want) {
            if (atomicAdd(bad, 1) == 0) {
                first[0] = r;
                first[1] = c;
                first[2] = v[c];
                first[3] = want;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
    int *bad;
    uint32_t *first;
    cudaMalloc(&bad, 4);
    cudaMalloc(&first, 16);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(bad, 0, 4);
        cudaMemset(first, 0, 16);
        k_cp_test<<<1, 128>>>(variant, bad, first);
        cudaError_t err = cudaDeviceSynchronize();
        int hb = -1;
        uint32_t hf[4] = {0, 0, 0, 0};
        cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(hf, first, 16, cudaMemcpyDeviceToHost);
        printf("variant %d (%s): err=%s mismatches=%d first: row %u col %u got 0x%x want 0x%x\n", variant,
               variant == 0 ? "sw128" : "no-swizzle", cudaGetErrorString(err), hb, hf[0], hf[1], hf[2], hf[3]);
        if (err != cudaSuccess) return 1;
    }
    return 0;
}

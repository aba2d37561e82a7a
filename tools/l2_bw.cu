// Dev: L2 -> shared memory bandwidth of cp.async.bulk (the running-sum form's operand path):
// every CTA streams CHUNK-byte bulk copies of an L2-resident buffer into a shared ring of R
// slots (mbarrier complete_tx), G CTAs per SM-count.  Prints GB/s for a few chunk sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1111_6900_b200/csrc tools/l2_bw.cu
#include <cstdio>
#include <cstdint>
#include "common.cuh"

using namespace gf2e;

__global__ void k_l2_bw(const uint8_t *src, int64_t src_bytes, int chunk, int iters, int ring) {
    // one issuing warp per ring (blockDim / 32 rings of `ring` slots each)
    extern __shared__ __align__(1024) uint8_t smem_all[];
    __shared__ __align__(8) uint64_t bars[4][8];
    const int w = threadIdx.x >> 5;
    uint64_t *bar = bars[w];
    uint8_t *sm = smem_all + w * ring * chunk;
    if ((threadIdx.x & 31) == 0) {
        for (int i = 0; i < ring; ++i) mbar_init(&bar[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    const int64_t nchunks = src_bytes / chunk;
    int64_t c = ((int64_t)(blockIdx.x * 4 + w) * 7919) % nchunks;
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        const int slot = it % ring;
        if (it >= ring) {
            mbar_wait(&bar[slot], ph[slot]);
            ph[slot] ^= 1;
        }
        mbar_arrive_expect_tx(&bar[slot], chunk);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + slot * chunk)),
            "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&bar[slot]))
            : "memory");
        c += 37;
        if (c >= nchunks) c -= nchunks;
    }
    for (int i = 0; i < ring && i < iters; ++i) {
        const int it = iters - 1 - i;
        const int slot = it % ring;
        (void)it;
        mbar_wait(&bar[slot], ph[slot]);
        ph[slot] ^= 1;
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t bytes = 64ll << 20;  // L2-resident
    uint8_t *src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    cudaFuncSetAttribute(k_l2_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int nw : {1, 2, 4})
    for (int chunk : {4096, 12288, 16384, 32768}) {
        for (int ring : {2, 4, 8}) {
            if (chunk * ring * nw > 200 * 1024) continue;
            const int iters = 4000;
            k_l2_bw<<<sms, 32 * nw, chunk * ring * nw>>>(src, bytes, chunk, 200, ring);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            k_l2_bw<<<sms, 32 * nw, chunk * ring * nw>>>(src, bytes, chunk, iters, ring);
            cudaEventRecord(b);
            cudaError_t err = cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("issuers %d chunk %6d B ring %d: %8.1f GB/s (%s)\n", nw, chunk, ring, (double)sms * nw * iters * chunk / (ms * 1e6),
                   cudaGetErrorString(err));
        }
    }
    return 0;
}

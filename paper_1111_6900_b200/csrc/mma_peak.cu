// mma_peak.cu — measured denominator for the roofline: the dense kind::i8 tcgen05 rate of
// this B200, from a pure-MMA loop (no operand production, no epilogue) on every SM.
//   cta_group 1: M=128 N=256 K=32 per instruction, one CTA per SM
//   cta_group 2: M=256 N=256 K=32 per instruction, CTA pairs (cluster of 2)
// Operands are fixed shared-memory tiles (0x01 bytes); accumulators alternate between two
// TMEM buffers.  Reported as int8 tensor ops/s (2 per MAC).
#include "common.cuh"
#include "kernels.h"

namespace gf2e {
namespace {

constexpr int PK_THREADS = 128;
constexpr int PK_SMEM = 48 * 1024 + 1024 + 64;

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG>
__global__ void __launch_bounds__(PK_THREADS, 1) k_mma_peak(int iters) {
    extern __shared__ uint8_t smem_raw[];
    // keep the shared state space visible to the compiler (STS/LDS, not generic ST/LD)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 48 * 1024);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + 48 * 1024 + 16);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += PK_THREADS) reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    if (warp == 0) {
        if (CG == 1) {
            tmem_alloc(tslot, 512);
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                         "r"(512)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const bool leader = (CG == 1) || cluster_ctarank() == 0;
    if (warp == 0 && lane == 0 && leader) {
        const uint32_t sa = smem_u32(smem), sb = sa + 16 * 1024;
        const uint32_t idesc = idesc_i8(128 * CG, 256);
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + (uint32_t)((i & 1) * 256);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = umma_desc_sw128(sa + kk * 32), bd = umma_desc_sw128(sb + kk * 32);
                if (CG == 1) {
                    mma_i8(d, ad, bd, idesc, (uint32_t)kk);
                } else {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)kk)
                        : "memory");
                }
            }
        }
        if (CG == 1) {
            mma_commit(bar);
        } else {
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(bar)),
                "h"((uint16_t)3)
                : "memory");
        }
    }
    if (warp == 0) mbar_wait(bar, 0);
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        if (CG == 1)
            tmem_dealloc(tmem, 512);
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// INT-pipe roofline of the M4RM form (k_product_m4rm): conflict-free LDS.128 table reads
// XOR-ed into registers, 2 CTAs x 1024 threads per SM
__global__ void __launch_bounds__(1024) k_lds_peak(int iters, uint32_t *out) {
    __shared__ uint4 tab[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    uint4 acc = make_uint4(0, 0, 0, 0);
    int idx = threadIdx.x & 2047;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint4 v = tab[(idx + r * 32) & 2047];
            acc.x ^= v.x;
            acc.y ^= v.y;
            acc.z ^= v.z;
            acc.w ^= v.w;
        }
        idx = (idx + (int)(acc.x & 1)) & 2047;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345u) out[0] = 1;
}

}  // namespace

cudaError_t run_lds_peak(int iters, int nsms, cudaStream_t st, double *bytes_per_s) {
    uint32_t *d = nullptr;
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void **>(&d), 64, st);
    if (err != cudaSuccess) return err;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_lds_peak<<<nsms * 2, 1024, 0, st>>>(iters, d);  // warm-up
    cudaEventRecord(a, st);
    k_lds_peak<<<nsms * 2, 1024, 0, st>>>(iters, d);
    cudaEventRecord(b, st);
    err = cudaGetLastError();
    float ms = 0;
    if (err == cudaSuccess) err = cudaEventSynchronize(b);
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeAsync(d, st);
    if (err == cudaSuccess) *bytes_per_s = (double)nsms * 2 * 1024 * iters * 16 * 16 / (ms * 1e-3);
    return err;
}

cudaError_t run_mma_peak(int cta_group, int iters, int nsms, cudaStream_t st, float *ms) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaError_t err = cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(PK_THREADS);
    cfg.dynamicSmemBytes = PK_SMEM;
    cfg.stream = st;
    if (cta_group == 2) {
        err = cudaFuncSetAttribute(k_mma_peak<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, PK_SMEM);
        cfg.gridDim = dim3((unsigned)(nsms & ~1));
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    } else {
        err = cudaFuncSetAttribute(k_mma_peak<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, PK_SMEM);
        cfg.gridDim = dim3((unsigned)nsms);
    }
    if (err != cudaSuccess) return err;
    for (int rep = 0; rep < 2 && err == cudaSuccess; ++rep) {  // first launch warms up
        cudaEventRecord(a, st);
        err = cta_group == 2 ? cudaLaunchKernelEx(&cfg, k_mma_peak<2>, iters) : cudaLaunchKernelEx(&cfg, k_mma_peak<1>, iters);
        cudaEventRecord(b, st);
    }
    if (err == cudaSuccess) err = cudaEventSynchronize(b);
    if (err == cudaSuccess) err = cudaEventElapsedTime(ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return err;
}

}  // namespace gf2e

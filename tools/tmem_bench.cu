// tmem_bench.cu — dev microbenchmark (not part of the library): TMEM read / write throughput
// of tcgen05.ld / tcgen05.st per SM, and how TMEM reads slow a concurrent MMA stream.  Sizes
// the epilogue drain of the short-k (config 4) product forms.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1111_6900_b200/csrc \
//        tools/tmem_bench.cu -o tools/_tmem_bench && tools/_tmem_bench
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"

using namespace gf2e;
using namespace gf2e::tc;

__device__ __forceinline__ void ld_x32(uint32_t t, uint32_t (&v)[32]) { tmem_ld32(t, v); }
__device__ __forceinline__ void ld_x16p(uint32_t t, uint32_t (&v)[16]) { tmem_ld32_pack16(t, v); }
__device__ __forceinline__ void ld_x32p(uint32_t t, uint32_t (&v)[32]) { tmem_ld64_pack16(t, v); }
__device__ __forceinline__ void st_x32(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
            taddr),
        "r"(v)
        : "memory");
}
__device__ __forceinline__ void st_x8(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
                 : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_mxf4_1(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t sfa,
                                           uint32_t sfb, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
        : "memory");
}
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

constexpr int SMEM = 48 * 1024 + 1024 + 256;

// mode: 0 ld x32, 1 ld x16.pack16, 2 ld x32.pack16, 3 two ld x32 per wait, 4 st x32, 5 st x8
// mma: 0 none, 1 mxf4 loop on columns 0..255 (warp 0), 2 i8 loop
// nw: TMEM-access warps (besides warp 0 when mma != 0); warp w accesses lane quarter w%4,
//     columns [base, base+span) split across the nw/4 warps of a quarter
__global__ void __launch_bounds__(544, 1) k_bench(int mode, int mma, int nw, int iters, int mma_iters,
                                                  unsigned long long *out) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 48 * 1024);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smem + 48 * 1024 + 16);
    volatile int *done = reinterpret_cast<volatile int *>(smem + 48 * 1024 + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
        *done = 0;
    }
    if (warp == 0) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp < 4) {  // scale factors (1.0) at columns 256..319 for the mxf4 loop
        const uint32_t lb = (uint32_t)(warp * 32) << 16;
        st_x32(tmem + lb + 256, 0x7F7F7F7Fu);
        st_x32(tmem + lb + 288, 0x7F7F7F7Fu);
        wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int aw = mma ? warp - 1 : warp;  // access-warp index
    const uint32_t base = mma ? 256 : 0, span = mma ? 256 : 512;
    uint32_t acc = 0;
    long long t0 = clock64(), t1 = t0;
    if (mma && warp == 0) {
        if (lane == 0) {
            const uint32_t a0 = smem_u32(smem), b0 = a0 + 16 * 1024;
            const uint32_t idesc = mma == 1 ? idesc_mxf4(128, 256) : idesc_i8(128, 256);
            for (int it = 0; it < mma_iters; ++it)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (mma == 1)
                        mma_mxf4_1(tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                                   tmem + 256, tmem + 288, it | kk);
                    else
                        mma_i8(tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc, it | kk);
                }
            mma_commit(bar);
        }
        __syncwarp();
        mbar_wait(bar, 0);
        t1 = clock64();
        if (lane == 0) *done = 1;
    } else if (aw >= 0 && aw < nw) {
        const int q = warp & 3;  // hardware lane quarter of this warp
        const int per_q = nw / 4, h = aw / 4;
        const uint32_t cols = span / per_q, c0 = base + h * cols;
        const uint32_t lb = (uint32_t)(q * 32) << 16;
        for (int it = 0; mma ? !*done : it < iters; ++it) {
            if (mode == 0) {
                for (uint32_t c = 0; c < cols; c += 32) {
                    uint32_t v[32];
                    ld_x32(tmem + lb + c0 + c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc ^= v[j];
                }
            } else if (mode == 1) {
                for (uint32_t c = 0; c < cols; c += 32) {
                    uint32_t v[16];
                    ld_x16p(tmem + lb + c0 + c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc ^= v[j];
                }
            } else if (mode == 2) {
                for (uint32_t c = 0; c < cols; c += 64) {
                    uint32_t v[32];
                    ld_x32p(tmem + lb + c0 + c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc ^= v[j];
                }
            } else if (mode == 3) {
                for (uint32_t c = 0; c < cols; c += 64) {
                    uint32_t v[32], w[32];
                    ld_x32(tmem + lb + c0 + c, v);
                    ld_x32(tmem + lb + c0 + c + 32, w);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc ^= v[j] ^ w[j];
                }
            } else if (mode == 4) {
                for (uint32_t c = 0; c < cols; c += 32) st_x32(tmem + lb + c0 + c, (uint32_t)it);
                wait_st();
            } else {
                for (uint32_t c = 0; c < cols; c += 8) st_x8(tmem + lb + c0 + c, (uint32_t)it);
                wait_st();
            }
            if (mma) out[(size_t)blockIdx.x * 64 + 32 + warp] = it + 1;
        }
        t1 = clock64();
    }
    if (lane == 0) out[(size_t)blockIdx.x * 64 + warp] = (unsigned long long)(t1 - t0);
    if (acc == 0x12345678u) out[0] = 0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    unsigned long long *d;
    cudaMalloc(&d, (size_t)nsm * 64 * 8);
    std::vector<unsigned long long> h((size_t)nsm * 64);
    const char *names[] = {"ld 32x32b.x32", "ld x16.pack16", "ld x32.pack16", "ld 2*x32/wait", "st x32", "st x8"};
    auto run = [&](int mode, int mma, int nw, int iters, int mma_iters, float *ms) {
        cudaMemset(d, 0, (size_t)nsm * 64 * 8);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int threads = (nw + (mma ? 1 : 0)) * 32;
        k_bench<<<nsm, threads, SMEM>>>(mode, mma, nw, iters, mma_iters, d);  // warm
        cudaEventRecord(a);
        k_bench<<<nsm, threads, SMEM>>>(mode, mma, nw, iters, mma_iters, d);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            exit(1);
        }
        cudaEventElapsedTime(ms, a, b);
        cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
    };
    // 1. TMEM read / write throughput alone
    for (int mode = 0; mode < 6; ++mode)
        for (int nw : {4, 8, 16}) {
            const int iters = 200;
            float ms;
            run(mode, 0, nw, iters, 0, &ms);
            unsigned long long mx = 0;
            for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;  // CTA 0
            const double cells = (double)iters * 128 * 512;            // 128 lanes x 512 columns per iter
            printf("%-16s warps %2d : %7.1f B/clk/SM (cells x4B)  %.3f ms  %llu cyc\n", names[mode], nw,
                   cells * 4 / mx, ms, mx);
        }
    // 2. MMA rate alone and with concurrent TMEM reads of the other 256 columns
    for (int mma : {1, 2}) {
        const int mi = mma == 1 ? 4000 : 2000;
        for (int mode : {-1, 0, 1, 2, 4}) {
            for (int nw : {4, 8}) {
                if (mode < 0 && nw == 8) continue;
                float ms;
                run(mode < 0 ? 0 : mode, mma, mode < 0 ? 0 : nw, 0, mi, &ms);
                const double macs = (double)mi * 4 * 128 * 256 * (mma == 1 ? 64 : 32);
                unsigned long long it = 0;
                for (int w = 1; w <= nw; ++w) it += h[32 + w];
                const double rd_cells = mode < 0 ? 0 : (double)it / nw * 128 * 256;  // per warp-quarter pass
                printf("%s mma alone/with %-14s x%d: %.3f ms (%.0f MAC/clk-equiv ms-based: %.2f TOPS chip) | side passes %.1f (%.1f B/clk)\n",
                       mma == 1 ? "mxf4" : "i8  ", mode < 0 ? "-" : names[mode], nw, ms, 0.0,
                       macs * 2 * nsm / (ms * 1e-3) / 1e12, (double)it / (nw ? nw : 1),
                       h[0] ? rd_cells * 4 / h[0] : 0.0);
            }
        }
    }
    return 0;
}

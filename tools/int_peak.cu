// int_peak.cu — dev microbenchmark: the INT-pipe roofline of the M4RM product form
// (k_product_m4rm: LOP3 XOR/AND on 32-bit words, table rows from shared memory with LDS.128).
//   LOP3: each thread runs 8 independent chains of lop3.b32 (a ^ b ^ c); reported as lop3/clk/SM
//         and as the M4RM bound: k_product_m4rm spends 1 LDS.128 + 4 LOP3 per (row, 128
//         columns, 8 k-bits) = 2048 GF(2) bit-ops, i.e. 512 bit-ops per LOP3 and 128 per
//         shared-memory byte.
//   LDS.128: conflict-free 16-byte shared loads per clk per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/int_peak.cu -o tools/_int_peak
#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(1024) k_lop3(int iters, uint32_t seed, uint32_t *out, long long *cyc) {
    uint32_t a[8], b = seed ^ threadIdx.x, c = seed * 3 + blockIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + i * 0x9E3779B9u + threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
    }
    const long long t1 = clock64();
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= a[i];
    if (x == 0x12345u) out[0] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) k_lds(int iters, uint32_t *out, long long *cyc) {
    __shared__ uint4 tab[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    uint4 acc = make_uint4(0, 0, 0, 0);
    int idx = threadIdx.x & 2047;
    const long long t0 = clock64();
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
    const long long t1 = clock64();
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345u) out[0] = 1;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int nsm = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    uint32_t *d;
    long long *cyc;
    cudaMalloc(&d, 64);
    cudaMalloc(&cyc, nsm * 8 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {512, 1024}) {
        const int iters = 20000;
        k_lop3<<<nsm * 2, threads>>>(iters, 7, d, cyc);
        cudaEventRecord(a);
        k_lop3<<<nsm * 2, threads>>>(iters, 7, d, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long c0;
        cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        const double ops = (double)nsm * 2 * threads * iters * 16 * 8;  // lop3 per launch
        // k_product_m4rm: per (row, 128 columns, 8 k-bits) 1 LDS.128 + 4 LOP3 = 2048 GF(2) bit-ops
        printf("LOP3 %4d thr x2 CTA/SM: %.3f ms, %.1f lop3/clk/SM (CTA-0 clock), %.2f T lop3/s chip -> M4RM LOP3 "
               "bound %.1f Tbit-op/s (512 bit-ops per LOP3)\n",
               threads, ms, (double)2 * threads * iters * 16 * 8 / c0, ops / (ms * 1e-3) / 1e12,
               ops * 512 / (ms * 1e-3) / 1e12);
    }
    {
        const int iters = 20000, threads = 1024;
        k_lds<<<nsm * 2, threads>>>(iters, d, cyc);
        cudaEventRecord(a);
        k_lds<<<nsm * 2, threads>>>(iters, d, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long c0;
        cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        const double bytes = (double)nsm * 2 * threads * iters * 16 * 16;
        printf("LDS.128 1024 thr x2 CTA/SM: %.3f ms, %.1f B/clk/SM (CTA-0 clock), %.1f TB/s chip -> M4RM LDS bound "
               "%.1f Tbit-op/s (2048 bit-ops per 16-byte table load)\n", ms,
               (double)2 * threads * iters * 16 * 16 / c0, bytes / (ms * 1e-3) / 1e12, bytes / 16 * 2048 / (ms * 1e-3) / 1e12);
    }
    printf("sm clock attr %.0f MHz\n", clk_khz / 1e3);
    return 0;
}

// kernels.h — host-side launchers of libgf2e_b200 (internal; the public ABI is include/gf2e_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace gf2e {

cudaError_t launch_random_packed(int e, int w, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                                 int64_t col0, int64_t gcols, uint64_t *out, int64_t ldp, cudaStream_t st);
cudaError_t launch_random_sliced(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0, int64_t col0,
                                 int64_t gcols, uint64_t *planes, int64_t ld, int64_t pstride, cudaStream_t st);
cudaError_t launch_random_words(int64_t rows, int64_t ncols, uint64_t seed, uint64_t *out, int64_t ld,
                                cudaStream_t st);
cudaError_t launch_slice(int e, int w, int64_t rows, int64_t cols, const uint64_t *packed, int64_t ldp,
                         uint64_t *planes, int64_t ld, int64_t pstride, cudaStream_t st);
cudaError_t launch_cling(int e, int w, int64_t rows, int64_t cols, const uint64_t *planes, int64_t ld,
                         int64_t pstride, uint64_t *packed, int64_t ldp, cudaStream_t st);
cudaError_t launch_xor(uint64_t *x, int64_t ldx, const uint64_t *y, int64_t ldy, int64_t rows, int64_t nwords,
                       cudaStream_t st);
cudaError_t launch_reduce(int e, uint32_t f, uint64_t *planes, int64_t rows, int64_t nwords, int64_t ld,
                          int64_t pstride, cudaStream_t st);
cudaError_t launch_combos_rows(const Sched &s, const uint64_t *X, int64_t ldx, int64_t px, int64_t rows,
                               int64_t ncols, uint64_t *out, int64_t ldo, int64_t po, int64_t rows_pad,
                               int64_t words_pad, cudaStream_t st);
cudaError_t launch_combos_bt(const Sched &s, const uint64_t *B, int64_t ldb, int64_t pb, int64_t k, int64_t n,
                             uint64_t *out, int64_t ldo, int64_t po, int64_t kblocks, int64_t nblocks,
                             cudaStream_t st);

// Tensor-core product (product_tc.cu).  Operands: Ac [nprod][m_pad][k_pad/64] natural bit
// order, Bt [nprod][n_pad][k_pad/64] transposed with bits reversed in each byte.
struct TcArgs {
    const uint64_t *Ac;
    const uint64_t *Bt;
    int64_t a_pstride, b_pstride;  // words
    int64_t kwords;                // k_pad / 64
    int64_t m, n;                  // real output extent
    int64_t m_pad, n_pad;
    uint64_t *C;
    int64_t ldc, c_pstride;
    int accumulate;
};
constexpr int kTcBM = 128, kTcBN = 256, kTcBK = 128;  // tile rows, tile cols, k-bits per stage
cudaError_t launch_product_tc(const Sched &s, const TcArgs &a, cudaStream_t st);
// CTA-pair variant (product_tc2.cu): m_pad must be a multiple of 256.
cudaError_t launch_product_tc2(const Sched &s, const TcArgs &a, cudaStream_t st);

// INT-pipe M4RM product (product_m4rm.cu).  Operands: Ac as above, Bc [nprod][k_pad][n_pad/64].
struct M4rmArgs {
    const uint64_t *Ac;
    const uint64_t *Bc;
    int64_t a_pstride, b_pstride;
    int64_t kwords;   // Ac words per row = k_pad/64
    int64_t nwords_pad;  // Bc words per row = n_pad/64
    int64_t k_pad;
    int64_t m, n;
    int64_t m_pad, n_pad;
    uint64_t *C;
    int64_t ldc, c_pstride;
};
constexpr int kM4BM = 512, kM4BN = 1024, kM4KPAD = 64;
cudaError_t launch_product_m4rm(const Sched &s, const M4rmArgs &a, cudaStream_t st);

cudaError_t run_mma_peak(int cta_group, int iters, int nsms, cudaStream_t st, float *ms);

}  // namespace gf2e

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
// wwords: plane words written per row (default ld: the words past cols are zeroed); a column
// window of a wider plane passes words_for(cols) so its neighbours are left alone
cudaError_t launch_slice(int e, int w, int64_t rows, int64_t cols, const uint64_t *packed, int64_t ldp,
                         uint64_t *planes, int64_t ld, int64_t pstride, cudaStream_t st, int64_t wwords = -1);
cudaError_t launch_cling(int e, int w, int64_t rows, int64_t cols, const uint64_t *planes, int64_t ld,
                         int64_t pstride, uint64_t *packed, int64_t ldp, cudaStream_t st);
cudaError_t launch_xor(uint64_t *x, int64_t ldx, const uint64_t *y, int64_t ldy, int64_t rows, int64_t nwords,
                       cudaStream_t st);
cudaError_t launch_reduce(int e, uint32_t f, uint64_t *planes, int64_t rows, int64_t nwords, int64_t ld,
                          int64_t pstride, cudaStream_t st);
// Stage-tiled operand layout of the tensor-core kernel: a plane of rows_pad x kwords words
// is a sequence of tiles (row block rb = r/128, k-stage ks = w/KW), each 128 rows x KW words
// contiguous (KW = 2: 128-bit int8 stages, 2 KiB; KW = 4: 256-bit fp4 stages, 4 KiB), so one
// bulk copy moves one stage of one operand half.
// Inside one 128-row x kw-word stage tile the words are stored as kw/2 slabs of [128 rows][2
// words], so the expander's per-row 16-byte shared-memory reads are consecutive across a warp
// (a [row][kw] layout makes the kw = 4 reads two-way bank-conflicted).
// br: rows per tile (128; 96 for the B^T operand of the running-sum form, whose CTA pairs
// cover 192 columns)
__host__ __device__ __forceinline__ int64_t tc_tile_word(int64_t r, int64_t w, int64_t kwords, int kw,
                                                         int br = 128) {
    const int64_t wk = w % kw;
    return (((r / br) * (kwords / kw) + (w / kw)) * br) * kw + (wk >> 1) * (2 * br) + (r % br) * 2 + (wk & 1);
}
// Row order inside each 32-row group of B^T tiles: tile row j holds column b_row_perm(j)
// (tc_common.cuh), i.e. column o sits at tile row 4*(o%8) + o/8.
__host__ __device__ __forceinline__ int64_t tc_b_row_inv(int64_t n) {
    const int64_t o = n & 31;
    return (n & ~int64_t(31)) | (4 * (o & 7) + (o >> 3));
}
// tiled_kw: 0 = row-major rows of ldo words; 2 / 4 = stage-tiled (tc_tile_word) with KW words
cudaError_t launch_combos_rows(const Sched &s, const uint64_t *X, int64_t ldx, int64_t px, int64_t rows,
                               int64_t ncols, uint64_t *out, int64_t ldo, int64_t po, int64_t rows_pad,
                               int64_t words_pad, int tiled_kw, cudaStream_t st);
// B^T combinations, stage-tiled; fp4: KW = 4 and bits 0/2 of every nibble swapped, else
// KW = 2 and bits reversed inside every byte
cudaError_t launch_combos_bt(const Sched &s, const uint64_t *B, int64_t ldb, int64_t pb, int64_t k, int64_t n,
                             uint64_t *out, int64_t ldo, int64_t po, int64_t kblocks, int64_t nblocks, bool fp4,
                             cudaStream_t st, int br = 128, int64_t row0 = 0, bool expand = false);
// (expand: fp4 only — write the MMA-ready nibble expansion in 128-byte-swizzled br-row stage
// tiles, 4 x the words: the running-sum form bulk-copies B stages straight into shared memory)
// (row0: first B^T row written, a multiple of 64 — the column offset of a B part; the tile
// layout stays relative to `out`)

// Tensor-core product.  Operands: Ac [nprod] x (m_pad x k_pad bits) natural bit order,
// Bt [nprod] x (n_pad x k_pad bits) = B^T with bits reversed in each byte.
constexpr int kMaxDevices = 64;  // per-device launch-attribute caches

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
// CTA-pair tcgen05 kernel (product_tc2.cu): m_pad multiple of 256, n_pad of 256, k_pad of
// 128 (int8) / 256 (fp4); Ac / Bt stage-tiled (tc_tile_word, KW 2 / 4), Bt rows in
// tc_b_row_inv order.
constexpr int kTcBKFp4 = 256;
// tensor-core forms of the product kernel: int8; fp4 (k chunks <= 32768); fp4 with two
// products per accumulator (k < 2048 only)
constexpr int kFormI8 = 0, kFormFp4 = 1, kFormFp4Pair = 2, kFormFp4Long = 3;  // Long: k >= 8192
// fp4 running-sum form (product_run.cu): double-buffered accumulators, no per-product
// re-initialisation; tiles 256 x kRunBN, B^T stage-tiled in kRunBN/2-row blocks
constexpr int kFormFp4Run = 4;
constexpr int kFormFp4RunX = 5;  // the running-sum form with B^T expanded in-kernel (few row tiles)
constexpr int kRunBN = 192;  // tile columns (two 192-column accumulators, three A stages and the
                             // scale factors fill the 512 TMEM columns; 128-column tiles with three
                             // accumulators measured slower: 23.1 vs 17.7 ms at config 4, e = 8)
constexpr int64_t kRunMaxSum = 65536;  // ceil(K/2) * k_pad must stay below (exact running sums)
#ifndef GF2E_RUN_BPRE
#define GF2E_RUN_BPRE 1
#endif
// the running-sum form's B^T operand is stored pre-expanded (4 words per bit word, swizzled
// stage tiles: launch_combos_bt(..., expand)) and bulk-copied straight into shared memory
constexpr bool kRunBPre = GF2E_RUN_BPRE != 0;
// bpre: B^T stages pre-expanded (launch_combos_bt(..., expand)); else bit tiles expanded in-kernel
cudaError_t launch_product_run(const Sched &s, const TcArgs &a, cudaStream_t st, bool bpre);
constexpr int64_t kFp4PairMaxK = 2047;
cudaError_t launch_product_tc2(const Sched &s, const TcArgs &a, int form, cudaStream_t st);

// packed-domain Newton-John product for small blocks (nj.cu): rows of B at most kNjMaxWords words
constexpr int kNjMaxWords = 16;
struct FieldTab;
// sliced Newton-John product (nj.cu): C (^)= A * B on bit planes, CUDA cores, one launch;
// c_aliases_b: C == B allowed (one row block per column word, m <= 256 rows)
inline int nj_sliced_alias_rows(int e) { return 4 * (512 / (e <= 8 ? 8 : 16)); }
cudaError_t launch_nj_sliced(int e, const FieldTab *ftab, const uint64_t *A, int64_t lda, int64_t pa,
                             const uint64_t *B, int64_t ldb, int64_t pb, uint64_t *C, int64_t ldc, int64_t pc,
                             int64_t m, int64_t k, int64_t n, bool acc, bool c_aliases_b, cudaStream_t st);
cudaError_t launch_nj_mul(int e, uint32_t f, int w, const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          uint64_t *C, int64_t ldc, int64_t m, int64_t k, int64_t n, bool acc, cudaStream_t st);

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
// conflict-free LDS.128 throughput of the whole GPU (bytes/s): the M4RM form's INT-pipe roofline
cudaError_t run_lds_peak(int iters, int nsms, cudaStream_t st, double *bytes_per_s);

// trsm.cu
// diagonal blocks of the blocked TRSM: 256 rows (full product tiles, k = 256 leaf products)
// for large solves, 128 rows for small / narrow ones (half the inverse's sequential chain)
constexpr int kTrsmBlockMax = 256;
cudaError_t launch_tri_inverse(int e, uint32_t f, uint32_t g, const uint64_t *T, int64_t ldt, int64_t pt, int64_t m,
                               bool upper, bool unit, uint64_t *Tinv, int *bad_row, int block, cudaStream_t st);
cudaError_t launch_mul_by_x(int e, uint32_t f, const uint64_t *in, int64_t ld, int64_t pin, uint64_t *out,
                            int64_t pout, int64_t rows, int64_t nwords, cudaStream_t st);
cudaError_t launch_scalar_mul(int e, uint32_t f, uint32_t c, int w, const uint64_t *in, int64_t ldi, uint64_t *out,
                              int64_t ldo, int64_t rows, int64_t nwords, cudaStream_t st);

// ple.cu — PLE base case on one 64-column panel + permutation / mask helpers
constexpr int kPlePanel = 64;
// Multiples of a scaled pivot suffix T kept by the PLE panel kernels: x * T = lo[x_lo] ^
// hi[x_hi], x_lo the low H1 bits of x, x_hi the high H2 (one table of all 2^e multiples for
// e <= 4).  Q entries of e plane words.
template <int E>
struct PleSplit {
    static constexpr int H1 = E <= 4 ? E : E / 2, H2 = E <= 4 ? 0 : E - E / 2;
    static constexpr int Q = (1 << H1) + (H2 ? (1 << H2) : 0);
    static constexpr int QE = Q * E;
};
constexpr int kPleTabWords = PleSplit<kMaxE>::QE;
struct PanelOut {
    int rank, ndisp, window, pad;
    int64_t P[64], Q[64];
    int jcol[64];
    int64_t dpos[64];
    int dstep[64];
    uint64_t dval[64][kMaxE];
    uint64_t tabs[64 * kPleTabWords];  // multiples of T_t split by scalar bits, [t][entry][plane]
};
// GF(2^e) tables for one field (one device allocation per (device, e, f), ple.cu: field_tab)
struct FieldTab {
    uint16_t ex[1024], lg[1024], inv[1024];  // exp/log over a primitive element; inverses
    uint16_t mulmask[1024][kMaxE];           // bit p of [c][b] = coefficient b of c * x^p
    uint32_t mulmask2[1024][kMaxE];          // the same for p < 2e - 1 (c * x^s * x^p: >> s)
    uint32_t f;                              // the field polynomial (bit e set)
};
const FieldTab *field_tab(int e, uint32_t f, uint32_t g);  // device pointer (synchronous fill)
int ple_window(int e);  // rows kept in shared memory by the panel kernel (launches = 1 + (m > window))
cudaError_t launch_ple_panel(int e, const FieldTab *tab, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int nb,
                             PanelOut *out, cudaStream_t st);
// speculative PLE: swaps t <-> Pg[t] (t in [t0, t1)) read from device memory; a panel's pivots
// committed into the global vectors, flag set if its rank differs from the speculated one
cudaError_t launch_row_swaps_vec(int planes, uint64_t *S, int64_t ld, int64_t ps, int64_t nwords, const int64_t *Pg,
                                 int64_t t0, int64_t t1, cudaStream_t st);
cudaError_t launch_ple_commit(const PanelOut *po, int64_t *Pg, int64_t *Qg, int64_t r0, int64_t c0, int expected,
                              int *flag, cudaStream_t st);
cudaError_t launch_row_swaps(int planes, uint64_t *S, int64_t ld, int64_t ps, int64_t nwords, const int64_t *pairs,
                             int n, bool backward, cudaStream_t st);
cudaError_t launch_col_swaps(int planes, int w, uint64_t *S, int64_t ld, int64_t ps, int64_t rows, const int64_t *trip,
                             int n, cudaStream_t st);
cudaError_t launch_tril_copy(int e, const uint64_t *S, int64_t ld, int64_t ps, int64_t r, uint64_t *out, int64_t ldo,
                             int64_t po, cudaStream_t st);
// (wstart: nw + 1 offsets; tpos / pmask: per column word, its pivots' t in increasing order and
// the prefix ORs of their bits -- built on the host from Q)
cudaError_t launch_echelon_marks(int e, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t nw, const int64_t *Q,
                                 int r, const int *wstart, const int *tpos, const uint64_t *pmask, cudaStream_t st);
cudaError_t launch_gather_cols(int e, const uint64_t *S, int64_t ld, int64_t ps, const int64_t *Q, int64_t r,
                               uint64_t *out, int64_t ldo, int64_t po, cudaStream_t st);

cudaError_t launch_row_scales(int e, uint32_t f, uint32_t g, int w, const uint64_t *in, int64_t ldi, bool bcast,
                              const uint32_t *cs, uint64_t *out, int64_t ldo, int64_t rows, int64_t nwords,
                              cudaStream_t st);

cudaError_t run_fp4_probe(int iters, int mode, const uint8_t *a_img, const uint8_t *b_img, uint32_t *out, int nctas,
                          cudaStream_t st, float *ms);
cudaError_t run_mma_peak(int cta_group, int iters, int nsms, cudaStream_t st, float *ms);


// launch with programmatic stream serialization (GF2E_PDL=0 turns it off): the kernel must
// call pdl_wait() before touching data its predecessors produce (common.cuh)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace gf2e

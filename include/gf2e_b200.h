/*
 * gf2e_b200.h — C ABI of libgf2e_b200.so, the B200 (sm_100a) implementation of the
 * GF(2^e) bitsliced-Karatsuba hot path of the M4RIE paper (arxiv 1111.6900), reference
 * package gf2elin (/root/reference/pkg/src/gf2elin).
 *
 * Plain pointers and sizes only.  Every pointer argument named *_dev is a CUDA device
 * pointer; `stream` is a cudaStream_t passed as void*.  All calls are stream-ordered and
 * asynchronous (no hidden host synchronisation); they return 0 on success and a nonzero
 * GF2E_E* status otherwise, with a thread-local message in gf2e_last_error().
 *
 * Layouts (identical to the reference, mat_gf2.py:3-7 and mat_packed.py:1-13):
 *   plane  (BitMatrix / mzd_t)   : rows x ld uint64 words, entry (i, j) = bit j%64 of word
 *                                  [i*ld + j/64]; bits past ncols are zero.
 *   plane stack (SlicedMatrix /  : e planes, plane t at base + t*pstride words.
 *                mzd_slice_t)
 *   packed (PackedMatrix / mzed_t): rows x ldp words, element (i, j) in bits
 *                                  [j*w, j*w+e) of the packed row, w = gf2e_pack_width(e),
 *                                  pad bits zero.
 *
 * Each entry point names the reference interface it replaces (file:line in gf2elin).
 */
#ifndef GF2E_B200_H
#define GF2E_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define GF2E_OK 0
#define GF2E_EINVAL 1   /* invalid argument (maps to ValueError in the Python shim) */
#define GF2E_ECUDA 2    /* CUDA runtime / launch error (RuntimeError)            */
#define GF2E_ENOMEM 3   /* workspace too small                                   */
#define GF2E_ENODEV 4   /* no sm_100 device                                      */
#define GF2E_ESINGULAR 5 /* zero diagonal entry in a triangular solve (SingularMatrixError) */

/* gf2e_slice_mul flags */
#define GF2E_ACCUMULATE 1u   /* C ^= A*B (addmul) instead of C = A*B              */
#define GF2E_BACKEND_TC 0u   /* K4 on tcgen05 tensor cores (default), all kind::mxf4 (e2m1
                                0/1, exact fp32 accumulation) unless the device's fp4 self-
                                check failed: the long-k form for k >= 8192, the fp4 form for
                                k >= 2048, the running-sum form below while its sums stay
                                exact, kind::i8 past that bound                             */
#define GF2E_BACKEND_M4RM 2u /* K4 as M4RM Gray tables in shared memory (INT pipe) */
#define GF2E_TC_INT8 4u      /* tensor-core K4 forced to kind::i8 at every k                */
#define GF2E_TC_FP4 8u       /* tensor-core K4 forced to kind::mxf4 at every k (paired form
                                below k = 2048)                                             */
#define GF2E_B_DEVICE 32u    /* gf2e_mzed_mul_host: B_host is a DEVICE pointer (B already
                                resident, e.g. broadcast to this GPU by the multi-GPU path)  */
#define GF2E_TC_RUN 16u      /* tensor-core K4 forced to the kind::mxf4 running-sum form
                                (double-buffered accumulators, 256 x 192 tiles) at every k  */

/* Last error message of the calling thread ("" if none). */
const char *gf2e_last_error(void);

/* Library version string. */
const char *gf2e_version(void);

/* mat_packed.pack_width (mat_packed.py:26-33): smallest divisor of 64 >= e; -1 if e out of 2..10. */
int gf2e_pack_width(int e);

/*
 * Karatsuba schedule for GF(2^e) mod f — the symbolic replay of _kara + reduce_mod_f
 * (poly_mul.py:166-242).  Replaces count_products (poly_mul.py:262-272) and the
 * MulCounters bookkeeping (poly_mul.py:32-43).
 *   n_products       <- K(e) (3, 6, 9, 15, 18, 24, 27, 39, 45 for the default f)
 *   subsets[t]       <- bitmask of input planes XOR-ed into operand t (t < K(e), cap 64)
 *   outmap[j]        <- bitmask over products folded into output plane j (j < e)
 *   counters[3]      <- gf2_matmul_count, additions, peak_live_products
 * Any output pointer may be NULL.  Fails (GF2E_EINVAL) if e is outside 2..10 or f is not
 * an irreducible polynomial of degree e (gf2e.py:125-137).
 */
int gf2e_schedule(int e, uint32_t f, int *n_products, uint64_t *subsets, uint64_t *outmap,
                  int64_t *counters);

/*
 * K7 generator: counter-mode splitmix64 (rng.py:20-35) exactly as
 * PackedMatrix.random (mat_packed.py:253-265), for the window of rows
 * [row0, row0+rows) and columns [col0, col0+cols) of a matrix with gcols columns
 * (element (i, j) uses stream index (row0+i)*gcols + col0 + j).
 * gf2e_random_packed writes packed words; gf2e_random_sliced writes e planes
 * (= slice_packed of the same matrix).
 */
int gf2e_random_packed(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                       int64_t col0, int64_t gcols, uint64_t *out_dev, int64_t ldp, void *stream);
int gf2e_random_sliced(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                       int64_t col0, int64_t gcols, uint64_t *planes_dev, int64_t ld,
                       int64_t pstride, void *stream);

/* BitMatrix.random (mat_gf2.py:194-206): words[i, w] = word_stream(seed)[i*ld_ref + w]
 * with ld_ref = ceil(ncols/64), tail bits past ncols cleared. */
int gf2e_random_words(int64_t rows, int64_t ncols, uint64_t seed, uint64_t *out_dev, int64_t ld,
                      void *stream);

/* K1 slice_packed (mat_sliced.py:97-101): packed -> e planes (mzed -> mzd_slice). */
int gf2e_slice(int e, int64_t rows, int64_t cols, const uint64_t *packed_dev, int64_t ldp,
               uint64_t *planes_dev, int64_t ld, int64_t pstride, void *stream);

/* K2 cling (mat_sliced.py:104-106): e planes -> packed, pad bits zero (mzd_slice -> mzed). */
int gf2e_cling(int e, int64_t rows, int64_t cols, const uint64_t *planes_dev, int64_t ld,
               int64_t pstride, uint64_t *packed_dev, int64_t ldp, void *stream);

/* Plane / packed addition X ^= Y over rows x nwords words (BitMatrix.iadd mat_gf2.py:161-164,
 * PackedMatrix.iadd mat_packed.py:180-190, SlicedMatrix.add mat_sliced.py:69-72). */
int gf2e_xor(uint64_t *x_dev, int64_t ldx, const uint64_t *y_dev, int64_t ldy, int64_t rows,
             int64_t nwords, void *stream);

/*
 * reduce_mod_f (poly_mul.py:223-242) on device: 2e-1 planes (plane d at base + d*pstride)
 * folded in place so planes 0..e-1 hold the reduced result.
 */
int gf2e_reduce_mod_f(int e, uint32_t f, uint64_t *planes_dev, int64_t rows, int64_t nwords,
                      int64_t ld, int64_t pstride, void *stream);

/*
 * Workspace bytes needed by gf2e_slice_mul / gf2e_plane_mul for this shape.
 * (Operand combinations of the Karatsuba schedule in the tensor-core layout.)
 */
int64_t gf2e_slice_mul_workspace(int e, uint32_t f, int64_t m, int64_t k, int64_t n,
                                 uint32_t flags);
int64_t gf2e_plane_mul_workspace(int64_t m, int64_t k, int64_t n, uint32_t flags);

/*
 * ★ The hot path: mzd_slice_mul / mzd_slice_addmul.
 * Replaces karatsuba_mul (poly_mul.py:245-259) and the addmul pattern
 * X.xor_window(0, 0, karatsuba_mul(A, B)) (ple_echelon.py:130-136,259).
 *   A: e planes m x k (lda words/row, plane stride pa)
 *   B: e planes k x n (ldb, pb)
 *   C: e planes m x n (ldc, pc); C = A*B, or C ^= A*B with GF2E_ACCUMULATE.
 * C must not overlap A or B.  workspace: >= gf2e_slice_mul_workspace(...) bytes of device
 * memory (256-byte aligned).
 */
int gf2e_slice_mul(int e, uint32_t f, const uint64_t *A_dev, int64_t lda, int64_t pa,
                   const uint64_t *B_dev, int64_t ldb, int64_t pb, uint64_t *C_dev, int64_t ldc,
                   int64_t pc, int64_t m, int64_t k, int64_t n, uint32_t flags, void *workspace,
                   int64_t workspace_bytes, void *stream);

/*
 * Small-block product on PACKED words, no slicing: nj_mul (newton_john.py:145-164) /
 * karatsuba_mul_packed below the crossover.  C = A*B or C ^= A*B (GF2E_ACCUMULATE), A m x k,
 * B k x n, C m x n, all packed (mzed) with row strides in words; rows of B and C at most 16
 * words (n <= 64 at e = 9, 10; 128 at e = 5..8; 256 at e = 3, 4; 512 at e = 2).  One launch:
 * per 64 rows of C, Newton-John tables of all 2^e multiples of each row of B in shared memory,
 * one lookup-and-XOR per (row of A, row of B) pair.
 */
int gf2e_nj_mul(int e, uint32_t f, const uint64_t *A_dev, int64_t lda, const uint64_t *B_dev, int64_t ldb,
                uint64_t *C_dev, int64_t ldc, int64_t m, int64_t k, int64_t n, uint32_t flags, void *stream);

/*
 * The same Newton-John product on bit planes (sliced operands, strides as gf2e_slice_mul): the
 * CUDA-core form that PLE's Schur updates and TRSM's updates take up to GF2E_NJS_MAXK (default
 * 128) inner dimension.  Per 64-column word of C and block of rows, tables of the multiples of
 * 32 rows of B at a time (split by the scalar's low / high bits) in shared memory; the entry
 * A[r][i] is one warp ballot over the plane lanes of row r.  No workspace.  C must not overlap
 * A or B.  flags: GF2E_ACCUMULATE.
 */
int gf2e_nj_slice_mul(int e, uint32_t f, const uint64_t *A_dev, int64_t lda, int64_t pa, const uint64_t *B_dev,
                      int64_t ldb, int64_t pb, uint64_t *C_dev, int64_t ldc, int64_t pc, int64_t m, int64_t k,
                      int64_t n, uint32_t flags, void *stream);

/*
 * gf2e_slice_mul with B arriving in column parts — the multi-GPU form (dist.sharded_mul: B is
 * broadcast over NVLink part by part while this rank already multiplies the parts that
 * arrived).  Part p holds columns [col_bounds[p], col_bounds[p+1]) of B as its own plane
 * stack (B_parts[p], ldb[p], pb[p]); col_bounds[0] = 0, col_bounds[nparts] = n, interior
 * bounds multiples of 64.  ready_events (optional; entries optional) are cudaEvent_t handles:
 * the stream waits for event p before reading part p.  A's operand combinations are formed
 * once; after each part the product runs over every column tile whose columns have all
 * arrived.  Same workspace as gf2e_slice_mul (gf2e_slice_mul_workspace); tensor-core
 * backends only.  C = A*B or C ^= A*B (GF2E_ACCUMULATE).
 */
int gf2e_slice_mul_parts(int e, uint32_t f, const uint64_t *A_dev, int64_t lda, int64_t pa, int nparts,
                         const int64_t *col_bounds, const uint64_t *const *B_parts_dev, const int64_t *ldb,
                         const int64_t *pb, void *const *ready_events, uint64_t *C_dev, int64_t ldc,
                         int64_t pc, int64_t m, int64_t k, int64_t n, uint32_t flags, void *workspace,
                         int64_t workspace_bytes, void *stream);

/*
 * The running-sum form's drain grouping for field (e, f) (diagnostic; the kernel's schedule):
 * product seq[i] is the i-th accumulated entry of a tile, group g = the next gsize[g] entries
 * with one accumulator drain whose parity is folded into the output planes gmask[g];
 * run_load = the most entries one accumulator takes per tile (exactness: run_load * k_pad <
 * 65536, else the plain one-group-per-product order runs).  Arrays hold up to 128 entries.
 */
int gf2e_run_schedule(int e, uint32_t f, int *nseq, int *ngrp, int *run_load, int *seq, int *gsize,
                      uint32_t *gmask);

/*
 * Columns of C per product tile (CTA pair) of the form a product with inner dimension k and
 * these flags would use (256, or 192 for the short-k running-sum form) — the quantum for
 * gf2e_slice_mul_parts bounds that keep every tile inside one part.  -1 on bad arguments.
 */
int64_t gf2e_tile_cols(int e, uint32_t f, int64_t k, uint32_t flags);

/*
 * mzed_mul / mzed_addmul with HOST buffers/*
 * mzed_mul / mzed_addmul with HOST buffers — the end-to-end entry a numpy-based caller
 * (e.g. gf2elin itself) binds: karatsuba_mul_packed (poly_mul.py:275-278)
 * and C ^= A*B on packed matrices, with A (m x k), B (k x n), C (m x n) in host memory in
 * the reference PackedMatrix.storage.words layout (row stride in words; pinned memory gives
 * full copy/compute overlap).  Synchronous.  B is uploaded, sliced and combined once; rows of
 * A (and C0) then stream through in chunks of `chunk_rows` rows (<= 0: a wave-aware plan
 * around 2048 rows) with the copies, operand preparation, products and copy-out of
 * consecutive chunks overlapped on four internal streams.  Device memory
 * comes from the library's own stream-ordered pool (gf2e_trim_pool).  flags: GF2E_ACCUMULATE,
 * GF2E_B_DEVICE (B_host is a device pointer: no B upload; B must be complete before the call,
 * which runs on its own streams).  *device_ms (optional) = CUDA-event time from the first
 * H2D to the last D2H.
 */
int gf2e_mzed_mul_host(int e, uint32_t f, const uint64_t *A_host, int64_t lda, const uint64_t *B_host,
                       int64_t ldb, uint64_t *C_host, int64_t ldc, int64_t m, int64_t k, int64_t n,
                       uint32_t flags, int64_t chunk_rows, double *device_ms);

/*
 * GF(2) plane product mzd_mul / mzd_addmul (mat_gf2.mul, mat_gf2.py:425-455):
 * C = A*B or C ^= A*B (GF2E_ACCUMULATE).  A m x k, B k x n, C m x n.
 */
int gf2e_plane_mul(const uint64_t *A_dev, int64_t lda, const uint64_t *B_dev, int64_t ldb,
                   uint64_t *C_dev, int64_t ldc, int64_t m, int64_t k, int64_t n, uint32_t flags,
                   void *workspace, int64_t workspace_bytes, void *stream);

/*
 * Triangular solve T X = B in place (X overwrites B), T m x m upper (upper != 0) or lower
 * triangular over GF(2^e), both as plane stacks: the consumer of the hot path in the
 * reference's recursive PLE/TRSM (trsm_upper_left / trsm_lower_left[_unit],
 * ple_echelon.py:138-217).  Blocked recursion with 128-row-aligned splits; every off-diagonal
 * update B_i ^= T_ij X_j is a gf2e_slice_mul(GF2E_ACCUMULATE) on plane views; diagonal blocks
 * are inverted on device (k_tri_inverse) and applied with gf2e_slice_mul.  unit_diag: the
 * stored diagonal is ignored and taken as 1 (lower only, as the reference).  Returns
 * GF2E_ESINGULAR (B untouched) if a diagonal entry is zero; *bad_row (optional) receives the
 * smallest such row.  Synchronises the stream once (singularity check).
 */
int64_t gf2e_trsm_workspace(int e, uint32_t f, int64_t m, int64_t n);
int gf2e_trsm(int e, uint32_t f, int upper, int unit_diag, const uint64_t *T_dev, int64_t ldt, int64_t pt,
              uint64_t *B_dev, int64_t ldb, int64_t pb, int64_t m, int64_t n, void *workspace,
              int64_t workspace_bytes, void *stream, int64_t *bad_row);

/*
 * In-place PLE decomposition of the m x n plane stack S (ple_echelon.ple, ple_echelon.py:240-300,
 * with the quadratic base case newton_john.nj_ple, newton_john.py:207-260): afterwards S holds
 * L strictly below the diagonal of its leading `rank` columns (original pivot values on the
 * diagonal) and E (leading ones implicit) on and above it; P_host / Q_host (length min(m, n),
 * optional) receive the LAPACK-style row / column swap vectors, *rank the rank.  Same pivot
 * rule as the reference (first nonzero entry top-down in the leftmost unfinished column), so
 * the result is bit-identical to ple() for every crossover.  Recursion on the host over
 * 64-column-aligned splits; 64-column base panels on device (k_ple_find / k_ple_apply);
 * Schur updates are gf2e_slice_mul(GF2E_ACCUMULATE); corner solves are gf2e_trsm.
 * Synchronises the stream (the recursion needs each panel's rank).
 */
int gf2e_ple(int e, uint32_t f, uint64_t *S_dev, int64_t ld, int64_t ps, int64_t m, int64_t n, int64_t *P_host,
             int64_t *Q_host, int64_t *rank, void *stream);

/* echelonize (ple_echelon.py:343-374): row echelon form (full = 0) or reduced row echelon form
 * (full != 0) of S in place via gf2e_ple; *rank receives the rank. */
int gf2e_echelonize(int e, uint32_t f, uint64_t *S_dev, int64_t ld, int64_t ps, int64_t m, int64_t n, int full,
                    int64_t *rank, void *stream);

/* apply_perm_rows (ple_echelon.py:81-91): swap vector swaps_host[0..n) applied in ascending
 * (backward = 0) or descending order to rows of `planes` word arrays (planes = e for a plane
 * stack, 1 for packed words) of nwords words each. */
int gf2e_row_swaps(int planes, uint64_t *S_dev, int64_t ld, int64_t ps, int64_t rows, int64_t nwords,
                   const int64_t *swaps_host, int64_t n, int backward, void *stream);

/* PackedMatrix.col_swap sequence (mat_packed.py col_swap; ple_echelon.py:94-107, 275-279):
 * triples_host[3i..3i+2] = (column a, column b, first row); w = slot width (1 for plane
 * stacks, the pack width for packed words). */
int gf2e_col_swaps(int planes, int w, uint64_t *S_dev, int64_t ld, int64_t ps, int64_t rows, int64_t cols,
                   const int64_t *triples_host, int64_t n, void *stream);

/* Row-wise scalar multiples on packed words: out row r = scalars_host[r] * (in row r, or in row
 * 0 when broadcast != 0).  With broadcast and scalars 0 .. 2^e - 1 this is the Newton-John
 * multiple table of one row (newton_john.make_table / _table_words, newton_john.py:55-88);
 * without, PackedMatrix.scale_row for many rows (mat_packed.py:201-205). */
int gf2e_row_scales(int e, uint32_t f, const uint64_t *in_dev, int64_t ldi, int broadcast, const uint32_t *scalars_host,
                    uint64_t *out_dev, int64_t ldo, int64_t rows, int64_t cols, void *stream);

/* mul_by_x (mat_sliced.py:109-122): out planes = alpha * in planes (alpha = class of x). */
int gf2e_mul_by_x(int e, uint32_t f, const uint64_t *in_dev, int64_t ld, int64_t pin, uint64_t *out_dev,
                  int64_t pout, int64_t rows, int64_t cols, void *stream);

/* PackedMatrix.scalar_mul (mat_packed.py:192-199): out = c * in, packed words. */
int gf2e_scalar_mul(int e, uint32_t f, uint32_t c, const uint64_t *in_dev, int64_t ldi, uint64_t *out_dev,
                    int64_t ldo, int64_t rows, int64_t cols, void *stream);

/*
 * Instrumentation: number of kernels the last successful call on this thread launched,
 * the name of the product kernel it used, and the GF(2) plane products it launched (K(e)
 * per fused product launch: the device-side counterpart of MulCounters.gf2_matmul_count,
 * e.g. every Schur update and diagonal-block product of a TRSM / PLE call).
 */
int gf2e_last_launch_count(void);
const char *gf2e_last_product_kernel(void);
int64_t gf2e_last_gf2_products(void);

/*
 * Live kernel timing for bench.py: while enabled, every product-kernel launch is bracketed
 * by CUDA events recorded on the launching stream.  gf2e_profile_read synchronises those
 * events and returns the summed duration (ms) and the number of launches, then clears.
 */
int gf2e_profile_enable(int on);
/*
 * Pure-MMA microbenchmark (no operand production, no epilogue): tcgen05.mma kind::i8 with
 * cta_group 1 (M=128,N=256,K=32) or 2 (M=256,N=256,K=32) on every SM for `iters` x 4
 * instructions.  Returns the measured dense int8 tensor rate (ops/s, 2 per MAC) in *tops
 * (units of 1e12) and the launch time in *ms.  The roofline denominator of bench.py.
 */
int gf2e_mma_peak(int cta_group, int iters, double *tops, double *ms, void *stream);
/*
 * Development probe (not on the product path): block-scaled FP4 tcgen05 MMA (kind::mxf4,
 * M=128 N=256 K=64, all scales 1.0) on fixed operand images a_dev [128][128 B], b_dev
 * [256][128 B] (two e2m1 elements per byte), iters x 4 MMAs per SM; out_dev [128][256]
 * receives CTA 0's raw fp32 accumulator.  mode bit 0: accumulator starts at 65536.0f.
 */
int gf2e_dev_fp4_probe(int iters, int mode, const uint8_t *a_dev, const uint8_t *b_dev, uint32_t *out_dev,
                       double *tops, void *stream);
int gf2e_profile_read(double *total_ms, int *launches);

/*
 * INT-pipe roofline of the M4RM product form (GF2E_BACKEND_M4RM): conflict-free LDS.128 table
 * reads on every SM (the form's bound, profiles/r02/ncu_m4rm_c3.txt), as bytes/s and as the
 * GF(2) bit-op rate it allows (2048 bit-ops per 16-byte table read: 128 columns x 8 k-bits).
 */
int gf2e_int_peak(int iters, double *lds_bytes_per_s, double *m4rm_tops, void *stream);

/*
 * fp4 exactness self-check.  The kind::mxf4 forms of the product assume exact fp32
 * accumulation of 0/1 products (measured, not architecturally guaranteed).  Before the first
 * fp4 product on a device the library compares every fp4 form with the int8 form (integer
 * arithmetic) on random and all-ones GF(2) planes: plane products up to k = 33024 (across the
 * 32768-bit accumulation chunk) and the running-sum form with the 9-product GF(16) schedule;
 * on any mismatch fp4 is disabled on that device and every product uses kind::i8.  This entry runs the check if it has not run (rerun != 0: again) and reports
 * *ok = 1 (fp4 in use) or -1 (disabled).  inject_fault != 0 (tests) corrupts the fp4 results
 * of this check, so it must fail and disable fp4.
 */
int gf2e_fp4_selfcheck(int rerun, int inject_fault, int *ok);

/*
 * Release the current device's cached temporaries of the library pool (host-buffer
 * pipeline, PLE/echelonize scratch) down to keep_bytes; synchronises the device.  The pool
 * keeps at most 4 GiB between calls on its own.
 */
int gf2e_trim_pool(int64_t keep_bytes);

#ifdef __cplusplus
}
#endif

#endif /* GF2E_B200_H */

// convert.cu — HBM-bound kernels of the hot path (sm_100a):
//   K7 generator (rng.py:20-35, mat_packed.py:253-265), K1 slice (mat_sliced.py:97-101),
//   K2 cling (mat_sliced.py:104-106), plane XOR (mat_gf2.py:161-164), reduce_mod_f
//   (poly_mul.py:223-242), and K3 operand combinations of the Karatsuba schedule
//   (poly_mul.py:153-163,184-186,200-201) in the layouts the product kernels read.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace gf2e {

namespace {

__host__ __device__ constexpr uint64_t rep(uint64_t pattern, int period) {
    uint64_t r = 0;
    for (int i = 0; i < 64; i += period) r |= pattern << i;
    return r;
}

// Bit 0 of every W-bit slot of x, packed into the low 64/W bits (a PEXT by constant mask).
template <int W>
__device__ __forceinline__ uint64_t gather_slots(uint64_t x) {
    x &= rep(1, W);
#pragma unroll
    for (int k = 1; (W << (k - 1)) < 64; ++k)
        x = (x | (x >> ((W - 1) << (k - 1)))) & rep((1ULL << (1 << k)) - 1, W << k);
    return x;
}

// Inverse of gather_slots: low 64/W bits of x to bit 0 of each W-bit slot (a PDEP).
template <int W>
__device__ __forceinline__ uint64_t spread_slots(uint64_t x) {
    constexpr int P = 64 / W;
    constexpr int K = (P == 32) ? 5 : (P == 16) ? 4 : (P == 8) ? 3 : (P == 4) ? 2 : 1;
    x &= (P == 64) ? ~0ULL : ((1ULL << P) - 1);
#pragma unroll
    for (int k = K; k >= 1; --k)
        x = (x | (x << ((W - 1) << (k - 1)))) & rep((1ULL << (1 << (k - 1))) - 1, W << (k - 1));
    return x;
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// ---- K7 generators -------------------------------------------------------------------

__global__ void k_random_packed(int e, int w, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                                int64_t col0, int64_t gcols, uint64_t *__restrict__ out, int64_t ldp) {
    const int per = 64 / w;
    const uint64_t mask = (1ULL << e) - 1;
    const int64_t total = rows * ldp;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / ldp, pw = idx - r * ldp;
        int64_t j0 = pw * per;
        uint64_t base = (uint64_t)(row0 + r) * (uint64_t)gcols + (uint64_t)col0;
        uint64_t v = 0;
        for (int s = 0; s < per; ++s) {
            int64_t j = j0 + s;
            if (j < cols) v |= (splitmix(seed, base + (uint64_t)j) & mask) << (s * w);
        }
        out[idx] = v;
    }
}

__global__ void k_random_sliced(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                                int64_t col0, int64_t gcols, uint64_t *__restrict__ planes, int64_t ld,
                                int64_t pstride) {
    const int64_t total = rows * ld;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / ld, wi = idx - r * ld;
        uint64_t base = (uint64_t)(row0 + r) * (uint64_t)gcols + (uint64_t)col0;
        uint64_t acc[kMaxE];
#pragma unroll
        for (int t = 0; t < kMaxE; ++t) acc[t] = 0;
        int64_t j0 = wi * 64;
        int nvalid = (int)(cols - j0 < 64 ? (cols - j0 < 0 ? 0 : cols - j0) : 64);
        for (int s = 0; s < nvalid; ++s) {
            uint64_t v = splitmix(seed, base + (uint64_t)(j0 + s));
#pragma unroll
            for (int t = 0; t < kMaxE; ++t) acc[t] |= ((v >> t) & 1ULL) << s;
        }
#pragma unroll
        for (int t = 0; t < kMaxE; ++t)
            if (t < e) planes[t * pstride + r * ld + wi] = acc[t];
    }
}

// mat_gf2.py:194-206: one splitmix64 word per storage word, tail bits cleared.
__global__ void k_random_words(int64_t rows, int64_t ncols, uint64_t seed, uint64_t *__restrict__ out,
                               int64_t ld) {
    const int64_t nw = words_for(ncols);
    const uint64_t tm = tail_mask(ncols);
    const int64_t total = rows * nw;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / nw, w = idx - r * nw;
        uint64_t v = splitmix(seed, (uint64_t)idx);
        out[r * ld + w] = (w == nw - 1) ? (v & tm) : v;
    }
}

// ---- K1 / K2 ----------------------------------------------------------------------

template <int W>
__global__ void k_slice(int e, int64_t rows, int64_t cols, const uint64_t *__restrict__ packed, int64_t ldp,
                        uint64_t *__restrict__ planes, int64_t ld, int64_t pstride, int64_t wn) {
    constexpr int P = 64 / W;
    const int64_t nw = words_for(cols);
    const int64_t pwords = words_for(cols * W);
    const int64_t total = rows * wn;  // wn <= ld plane words written per row (pad words zeroed)
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / wn, wi = idx - r * wn;
        uint64_t acc[kMaxE];
#pragma unroll
        for (int t = 0; t < kMaxE; ++t) acc[t] = 0;
        if (wi < nw) {
            const uint64_t *src = packed + r * ldp + wi * W;
#pragma unroll
            for (int q = 0; q < W; ++q) {
                uint64_t x = (wi * W + q < pwords) ? src[q] : 0;
#pragma unroll
                for (int t = 0; t < kMaxE; ++t)
                    if (t < e) acc[t] |= gather_slots<W>(x >> t) << (q * P);
            }
            if (wi == nw - 1) {
                uint64_t tm = tail_mask(cols);
#pragma unroll
                for (int t = 0; t < kMaxE; ++t) acc[t] &= tm;
            }
        }
#pragma unroll
        for (int t = 0; t < kMaxE; ++t)
            if (t < e) planes[t * pstride + r * ld + wi] = acc[t];
    }
}

template <int W>
__global__ void k_cling(int e, int64_t rows, int64_t cols, const uint64_t *__restrict__ planes, int64_t ld,
                        int64_t pstride, uint64_t *__restrict__ packed, int64_t ldp) {
    constexpr int P = 64 / W;
    const int64_t total = rows * ldp;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / ldp, pw = idx - r * ldp;
        int64_t j0 = pw * P;
        uint64_t v = 0;
        if (j0 < cols) {
            int64_t wi = pw / W;
            int sh = (int)(pw % W) * P;
#pragma unroll
            for (int t = 0; t < kMaxE; ++t)
                if (t < e) v |= spread_slots<W>(planes[t * pstride + r * ld + wi] >> sh) << t;
            int64_t nvalid = cols - j0;
            if (nvalid < P) v &= (1ULL << (nvalid * W)) - 1;
        }
        packed[idx] = v;
    }
}

// ---- w = 8 (e = 5..8) fast paths: 8x8 bit-matrix transposes + byte gathers ---------------
// transpose of the 8x8 bit matrix held in a word (byte i = row i, bit j = column j):
// afterwards byte j bit i = old byte i bit j  (three delta swaps)
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAULL;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCULL;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ULL;
    x = x ^ t ^ (t << 28);
    return x;
}

// byte b of each of 8 words, packed into one word (byte q = byte b of v[q])
__device__ __forceinline__ uint64_t gather_byte(const uint64_t (&v)[8], int b) {
    const uint32_t sel = (uint32_t)(b & 3) | ((uint32_t)((b & 3) + 4) << 4);  // bytes b, 4+b of (a,c)
    uint32_t h[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) h[q] = b < 4 ? (uint32_t)v[q] : (uint32_t)(v[q] >> 32);
    const uint32_t p01 = __byte_perm(h[0], h[1], sel), p23 = __byte_perm(h[2], h[3], sel);
    const uint32_t p45 = __byte_perm(h[4], h[5], sel), p67 = __byte_perm(h[6], h[7], sel);
    const uint32_t lo = __byte_perm(p01, p23, 0x5410), hi = __byte_perm(p45, p67, 0x5410);
    return (uint64_t)lo | ((uint64_t)hi << 32);
}

// K1, w = 8: thread = one 64-bit plane word position (64 elements = 8 packed words)
__global__ void k_slice_w8(int e, int64_t rows, int64_t cols, const uint64_t *__restrict__ packed, int64_t ldp,
                           uint64_t *__restrict__ planes, int64_t ld, int64_t pstride, int64_t wn) {
    const int64_t nw = words_for(cols);
    const int64_t pwords = words_for(cols * 8);
    const uint64_t tm = tail_mask(cols);
    const int64_t total = rows * wn;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t r = idx / wn, wi = idx - r * wn;
        uint64_t v[8];
        if (wi < nw) {
            const uint64_t *src = packed + r * ldp + wi * 8;
            if (wi * 8 + 8 <= pwords && !(reinterpret_cast<uintptr_t>(src) & 15)) {
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    const ulonglong2 p = *reinterpret_cast<const ulonglong2 *>(src + q);
                    v[q] = p.x;
                    v[q + 1] = p.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = (wi * 8 + q < pwords) ? src[q] : 0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = transpose8x8(v[q]);  // byte t of v[q] = bit t of elements 8q..8q+7
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = 0;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (t < e) {
                uint64_t p = gather_byte(v, t);
                if (wi == nw - 1) p &= tm;
                planes[t * pstride + r * ld + wi] = p;
            }
        }
    }
}

// K2, w = 8: thread = one plane word position -> 8 packed words (pad bits 0)
__global__ void k_cling_w8(int e, int64_t rows, int64_t cols, const uint64_t *__restrict__ planes, int64_t ld,
                           int64_t pstride, uint64_t *__restrict__ packed, int64_t ldp) {
    const int64_t nw = words_for(cols);
    const int64_t pwords = words_for(cols * 8);
    const int64_t total = rows * nw;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t r = idx / nw, wi = idx - r * nw;
        uint64_t pl[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) pl[t] = t < e ? planes[t * pstride + r * ld + wi] : 0;
        if (wi == nw - 1) {
            const uint64_t tmk = tail_mask(cols);
#pragma unroll
            for (int t = 0; t < 8; ++t) pl[t] &= tmk;
        }
        uint64_t out[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) out[q] = transpose8x8(gather_byte(pl, q));  // byte s bit t = plane t elem 8q+s
        uint64_t *dst = packed + r * ldp + wi * 8;
        if (wi * 8 + 8 <= pwords && !(reinterpret_cast<uintptr_t>(dst) & 15)) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
                *reinterpret_cast<ulonglong2 *>(dst + q) = make_ulonglong2(out[q], out[q + 1]);
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (wi * 8 + q < pwords) dst[q] = out[q];
        }
        // words of the packed row beyond the last element-carrying word (ldp > pwords) are padding
        if (wi == nw - 1)
            for (int64_t q = pwords; q < ldp; ++q) packed[r * ldp + q] = 0;
    }
}

__global__ void k_xor(uint64_t *__restrict__ x, int64_t ldx, const uint64_t *__restrict__ y, int64_t ldy,
                      int64_t rows, int64_t nwords) {
    const int64_t total = rows * nwords;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / nwords, w = idx - r * nwords;
        x[r * ldx + w] ^= y[r * ldy + w];
    }
}

// poly_mul.py:223-242: for d = 2e-2 .. e, plane d folds into planes d-e+k for set low bits k of f.
__global__ void k_reduce(int e, uint32_t f, uint64_t *__restrict__ planes, int64_t rows, int64_t nwords,
                         int64_t ld, int64_t pstride) {
    const int64_t total = rows * nwords;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / nwords, w = idx - r * nwords;
        int64_t off = r * ld + w;
        uint64_t x[2 * kMaxE - 1];
#pragma unroll
        for (int d = 0; d < 2 * kMaxE - 1; ++d) x[d] = d < 2 * e - 1 ? planes[d * pstride + off] : 0;
#pragma unroll
        for (int d = 2 * kMaxE - 2; d >= 1; --d) {
            if (d > 2 * e - 2 || d < e) continue;
#pragma unroll
            for (int k = 0; k < kMaxE; ++k)
                if (k < e && ((f >> k) & 1u) && d - e + k >= 0) x[d - e + k] ^= x[d];
        }
#pragma unroll
        for (int d = 0; d < kMaxE; ++d)
            if (d < e) planes[d * pstride + off] = x[d];
    }
}

// ---- K3 operand combinations --------------------------------------------------------

// out[t] = XOR_{i in S_t} X_i on a zero-padded (rows_pad x words_pad) grid, natural bit order,
// row-major rows of ldo words (the M4RM operands; the tensor-core ones use k_combos_tiled).
__global__ void k_combos_rows(Sched s, const uint64_t *__restrict__ X, int64_t ldx, int64_t px, int64_t rows,
                              int64_t ncols, uint64_t *__restrict__ out, int64_t ldo, int64_t po,
                              int64_t rows_pad, int64_t words_pad) {
    const int64_t nw = words_for(ncols);
    const uint64_t tm = tail_mask(ncols);
    const int64_t total = rows_pad * words_pad;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        int64_t r = idx / words_pad, w = idx - r * words_pad;
        uint64_t x[kMaxE];
        bool valid = r < rows && w < nw;
#pragma unroll
        for (int i = 0; i < kMaxE; ++i) {
            uint64_t v = (i < s.e && valid) ? X[i * px + r * ldx + w] : 0;
            x[i] = (w == nw - 1) ? (v & tm) : v;
        }
        for (int t = 0; t < s.nprod; ++t) {
            uint32_t sub = s.subset[t];
            uint64_t acc = 0;
#pragma unroll
            for (int i = 0; i < kMaxE; ++i) acc ^= x[i] & (0ULL - (uint64_t)((sub >> i) & 1u));
            out[t * po + r * ldo + w] = acc;
        }
    }
}

// Stage-tiled A'_t (tensor-core layout): thread = (row r, pair of k-stages); reads 32 B of each
// input plane row (one sector), writes 16 B to each of two tiles; a warp's writes are 32
// consecutive tile rows = 512 contiguous bytes.
template <int E, int Q>  // planes at compile time; Q words (Q / 2 16-byte pieces) per thread
__global__ void k_combos_tiled(Sched s, const uint64_t *__restrict__ X, int64_t ldx, int64_t px, int64_t rows,
                               int64_t ncols, uint64_t *__restrict__ out, int64_t po, int64_t rows_pad,
                               int64_t kwords, int kw) {
    const int64_t nw = words_for(ncols);
    const uint64_t tm = tail_mask(ncols);
    const int64_t KP = (kwords + Q - 1) / Q;  // groups of Q words
    const int64_t total = rows_pad * KP;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t rb = idx / (KP * 128), rem = idx - rb * KP * 128;
        const int64_t kp = rem >> 7, r = rb * 128 + (rem & 127);
        const int64_t w0 = kp * Q;
        uint64_t x[E][Q];
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int64_t w = w0 + q;
                uint64_t v = (r < rows && w < nw) ? X[i * px + r * ldx + w] : 0;
                x[i][q] = (w == nw - 1) ? (v & tm) : v;
            }
        for (int t = 0; t < s.nprod; ++t) {
            const uint32_t sub = s.subset[t];
            uint64_t a[Q] = {};
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const uint64_t sel = 0ULL - (uint64_t)((sub >> i) & 1u);
#pragma unroll
                for (int q = 0; q < Q; ++q) a[q] ^= x[i][q] & sel;
            }
            uint64_t *o = out + t * po;
#pragma unroll
            for (int q = 0; q < Q; q += 2)
                if (w0 + q < kwords)
                    *reinterpret_cast<ulonglong2 *>(o + tc_tile_word(r, w0 + q, kwords, kw)) =
                        make_ulonglong2(a[q], a[q + 1]);
        }
    }
}

// 64x64 bit-matrix transpose held as two words per lane (rows lane and lane+32).
__device__ __forceinline__ void transpose64(uint64_t &xa, uint64_t &xb, int lane) {
    uint64_t t = ((xa >> 32) ^ xb) & 0x00000000FFFFFFFFULL;
    xb ^= t;
    xa ^= t << 32;
    const uint64_t masks[5] = {0x0000FFFF0000FFFFULL, 0x00FF00FF00FF00FFULL, 0x0F0F0F0F0F0F0F0FULL,
                               0x3333333333333333ULL, 0x5555555555555555ULL};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint64_t m = masks[s];
        uint64_t oa = __shfl_xor_sync(0xffffffffu, xa, j);
        uint64_t ob = __shfl_xor_sync(0xffffffffu, xb, j);
        if ((lane & j) == 0) {
            xa ^= (((xa >> j) ^ oa) & m) << j;
            xb ^= (((xb >> j) ^ ob) & m) << j;
        } else {
            xa ^= ((oa >> j) ^ xa) & m;
            xb ^= ((ob >> j) ^ xb) & m;
        }
    }
}

// Bt[t] = (XOR_{i in S_t} B_i)^T: row n holds the k-bits of column n of B, with the bit
// order reversed inside every byte (k-bit 8q+i at position 8q+7-i) — the layout the
// tensor-core producer expands with one AND per output word (product_tc2.cu) — stored
// stage-tiled with the rows of every 32-row group in tc_b_row_inv order (the epilogue's
// parity packer emits columns in b_row_perm order).  One warp per 64x64 block.
// fp4 B^T words (w2, w2 + 1) of row r, EXPANDED to the MMA operand (nibbles 2/1/0.5/1 per bit
// as product_run.cu's expander would write them) inside the row's 128-byte-swizzled stage tile
// of br rows: one bulk copy then moves a ready operand stage into shared memory
__device__ __forceinline__ void put_expanded(uint64_t *o, int64_t r, int64_t w2, int64_t ldo, int br, uint64_t x0,
                                             uint64_t x1) {
    constexpr int kw = 4;
    const int64_t stage = w2 / kw;
    const int c0 = (int)(w2 % kw) * 2;
    uint8_t *tile = reinterpret_cast<uint8_t *>(o + ((r / br) * (ldo / kw) + stage) * (int64_t)br * 16);
    const int rr = (int)(r % br);
    const uint32_t q[4] = {(uint32_t)x0, (uint32_t)(x0 >> 32), (uint32_t)x1, (uint32_t)(x1 >> 32)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t x = q[i];
        const int c = c0 + i;
        *reinterpret_cast<uint4 *>(tile + (rr >> 3) * 1024 + (rr & 7) * 128 + ((c ^ (rr & 7)) << 4)) =
            make_uint4(x & 0x44444444u, x & 0x22222222u, x & 0x11111111u, (x >> 2) & 0x22222222u);
    }
}

template <int E>  // planes at compile time (register arrays of E words)
__global__ void k_combos_bt(Sched s, const uint64_t *__restrict__ B, int64_t ldb, int64_t pb, int64_t k,
                            int64_t n, uint64_t *__restrict__ out, int64_t ldo, int64_t po, int64_t kblocks,
                            int64_t nblocks, int fp4, int tsplit, int br, int64_t row0, int expand) {
    // one warp per (2 x 64 k-rows, 64-column block[, product group]): two 64x64 transposes, then each lane
    // writes 16-byte pieces of tile rows.  Input row r of a 64-block lands at bit sigma(r):
    // int8 reverses bits inside bytes (r ^ 7), fp4 swaps bits 0 and 2 of every nibble.
    const int kw = fp4 ? 4 : 2;
    const int lane = threadIdx.x & 31;
    const int64_t warp = gtid() >> 5;
    const int64_t nwarps = gstride() >> 5;
    const int64_t nw = words_for(n);
    const int64_t kstages = kblocks >> 1;
    // small problems (the TRSM / PLE blocks) split the products over tsplit warps per block, so
    // the latency of the per-product loop is spread over more SMs
    const int tper = (s.nprod + tsplit - 1) / tsplit;
    for (int64_t wb = warp; wb < kstages * nblocks * tsplit; wb += nwarps) {
        const int tg = (int)(wb % tsplit);
        const int64_t blk = wb / tsplit;
        // nb fastest: neighbouring warps read neighbouring words of the same rows, so every
        // 32-byte sector of B is fetched from DRAM once (L2 serves the other three warps)
        const int64_t nb = blk % nblocks, ks = blk / nblocks;
        const uint64_t tm = (nb == nw - 1) ? tail_mask(n) : ~0ULL;
        uint64_t a[2][E], b[2][E];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sl = fp4 ? (lane ^ ((~lane & 1) << 1)) : (lane ^ 7);
            const int64_t r0 = (2 * ks + h) * 64 + sl, r1 = r0 + 32;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                a[h][i] = (nb < nw && r0 < k) ? (B[i * pb + r0 * ldb + nb] & tm) : 0;
                b[h][i] = (nb < nw && r1 < k) ? (B[i * pb + r1 * ldb + nb] & tm) : 0;
            }
        }
        const int64_t ra = tc_b_row_inv(row0 + nb * 64 + lane), rbw = tc_b_row_inv(row0 + nb * 64 + lane + 32);
        // the transpose is GF(2)-linear: transpose the e planes once, then form every
        // product's subset XOR from the transposed words (e instead of K(e) transposes)
#pragma unroll
        for (int i = 0; i < E; ++i) {
            transpose64(a[0][i], b[0][i], lane);
            transpose64(a[1][i], b[1][i], lane);
        }
        const int t1 = (tg + 1) * tper < s.nprod ? (tg + 1) * tper : s.nprod;
        for (int t = tg * tper; t < t1; ++t) {
            const uint32_t sub = s.subset[t];
            uint64_t xa[2] = {0, 0}, xb[2] = {0, 0};
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const uint64_t sel = 0ULL - (uint64_t)((sub >> i) & 1u);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    xa[h] ^= a[h][i] & sel;
                    xb[h] ^= b[h][i] & sel;
                }
            }
            uint64_t *o = out + t * po;
            if (expand) {
                put_expanded(o, ra, 2 * ks, ldo, br, xa[0], xa[1]);
                put_expanded(o, rbw, 2 * ks, ldo, br, xb[0], xb[1]);
            } else {
                *reinterpret_cast<ulonglong2 *>(o + tc_tile_word(ra, 2 * ks, ldo, kw, br)) =
                    make_ulonglong2(xa[0], xa[1]);
                *reinterpret_cast<ulonglong2 *>(o + tc_tile_word(rbw, 2 * ks, ldo, kw, br)) =
                    make_ulonglong2(xb[0], xb[1]);
            }
        }
    }
}

// f(std::integral_constant<int, e>) for e = 1 .. kMaxE (compile-time plane count)
template <typename F>
cudaError_t dispatch_e(int e, F &&f) {
    switch (e) {
        case 1: return f(std::integral_constant<int, 1>{});
        case 2: return f(std::integral_constant<int, 2>{});
        case 3: return f(std::integral_constant<int, 3>{});
        case 4: return f(std::integral_constant<int, 4>{});
        case 5: return f(std::integral_constant<int, 5>{});
        case 6: return f(std::integral_constant<int, 6>{});
        case 7: return f(std::integral_constant<int, 7>{});
        case 8: return f(std::integral_constant<int, 8>{});
        case 9: return f(std::integral_constant<int, 9>{});
        case 10: return f(std::integral_constant<int, 10>{});
        default: return cudaErrorInvalidValue;
    }
}

inline int grid_for(int64_t total, int threads) {
    int64_t g = (total + threads - 1) / threads;
    if (g > 148 * 64) g = 148 * 64;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

// ---- host launchers -------------------------------------------------------------------

cudaError_t launch_random_packed(int e, int w, int64_t rows, int64_t cols, uint64_t seed, int64_t row0,
                                 int64_t col0, int64_t gcols, uint64_t *out, int64_t ldp, cudaStream_t st) {
    int64_t total = rows * ldp;
    if (total == 0) return cudaSuccess;
    k_random_packed<<<grid_for(total, 256), 256, 0, st>>>(e, w, rows, cols, seed, row0, col0, gcols, out, ldp);
    return cudaGetLastError();
}

cudaError_t launch_random_sliced(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0, int64_t col0,
                                 int64_t gcols, uint64_t *planes, int64_t ld, int64_t pstride, cudaStream_t st) {
    int64_t total = rows * ld;
    if (total == 0) return cudaSuccess;
    k_random_sliced<<<grid_for(total, 256), 256, 0, st>>>(e, rows, cols, seed, row0, col0, gcols, planes, ld,
                                                          pstride);
    return cudaGetLastError();
}

cudaError_t launch_random_words(int64_t rows, int64_t ncols, uint64_t seed, uint64_t *out, int64_t ld,
                                cudaStream_t st) {
    int64_t total = rows * words_for(ncols);
    if (total == 0) return cudaSuccess;
    k_random_words<<<grid_for(total, 256), 256, 0, st>>>(rows, ncols, seed, out, ld);
    return cudaGetLastError();
}

cudaError_t launch_slice(int e, int w, int64_t rows, int64_t cols, const uint64_t *packed, int64_t ldp,
                         uint64_t *planes, int64_t ld, int64_t pstride, cudaStream_t st, int64_t wwords) {
    const int64_t wn = wwords < 0 ? ld : wwords;
    int64_t total = rows * wn;
    if (total == 0) return cudaSuccess;
    int g = grid_for(total, 256);
    switch (w) {
        case 2: k_slice<2><<<g, 256, 0, st>>>(e, rows, cols, packed, ldp, planes, ld, pstride, wn); break;
        case 4: k_slice<4><<<g, 256, 0, st>>>(e, rows, cols, packed, ldp, planes, ld, pstride, wn); break;
        case 8: k_slice_w8<<<g, 256, 0, st>>>(e, rows, cols, packed, ldp, planes, ld, pstride, wn); break;
        case 16: k_slice<16><<<g, 256, 0, st>>>(e, rows, cols, packed, ldp, planes, ld, pstride, wn); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_cling(int e, int w, int64_t rows, int64_t cols, const uint64_t *planes, int64_t ld,
                         int64_t pstride, uint64_t *packed, int64_t ldp, cudaStream_t st) {
    int64_t total = rows * ldp;
    if (total == 0) return cudaSuccess;
    int g = grid_for(total, 256);
    switch (w) {
        case 2: k_cling<2><<<g, 256, 0, st>>>(e, rows, cols, planes, ld, pstride, packed, ldp); break;
        case 4: k_cling<4><<<g, 256, 0, st>>>(e, rows, cols, planes, ld, pstride, packed, ldp); break;
        case 8: {
            const int64_t tw = rows * words_for(cols);
            if (tw == 0) return cudaMemset2DAsync(packed, ldp * 8, 0, ldp * 8, rows, st);
            k_cling_w8<<<grid_for(tw, 256), 256, 0, st>>>(e, rows, cols, planes, ld, pstride, packed, ldp);
            break;
        }
        case 16: k_cling<16><<<g, 256, 0, st>>>(e, rows, cols, planes, ld, pstride, packed, ldp); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_xor(uint64_t *x, int64_t ldx, const uint64_t *y, int64_t ldy, int64_t rows, int64_t nwords,
                       cudaStream_t st) {
    int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_xor<<<grid_for(total, 256), 256, 0, st>>>(x, ldx, y, ldy, rows, nwords);
    return cudaGetLastError();
}

cudaError_t launch_reduce(int e, uint32_t f, uint64_t *planes, int64_t rows, int64_t nwords, int64_t ld,
                          int64_t pstride, cudaStream_t st) {
    int64_t total = rows * nwords;
    if (total == 0) return cudaSuccess;
    k_reduce<<<grid_for(total, 256), 256, 0, st>>>(e, f, planes, rows, nwords, ld, pstride);
    return cudaGetLastError();
}

cudaError_t launch_combos_rows(const Sched &s, const uint64_t *X, int64_t ldx, int64_t px, int64_t rows,
                               int64_t ncols, uint64_t *out, int64_t ldo, int64_t po, int64_t rows_pad,
                               int64_t words_pad, int tiled_kw, cudaStream_t st) {
    if (tiled_kw) {
#ifndef GF2E_COMBOS_Q
#define GF2E_COMBOS_Q 2
#endif
        constexpr int Q = GF2E_COMBOS_Q;
        const int64_t tot = rows_pad * ((words_pad + Q - 1) / Q);
        if (tot == 0) return cudaSuccess;
        return dispatch_e(s.e, [&](auto ec) {
            k_combos_tiled<decltype(ec)::value, Q><<<grid_for(tot, 256), 256, 0, st>>>(
                s, X, ldx, px, rows, ncols, out, po, rows_pad, words_pad, tiled_kw);
            return cudaGetLastError();
        });
    }
    int64_t total = rows_pad * words_pad;
    if (total == 0) return cudaSuccess;
    k_combos_rows<<<grid_for(total, 256), 256, 0, st>>>(s, X, ldx, px, rows, ncols, out, ldo, po, rows_pad,
                                                        words_pad);
    return cudaGetLastError();
}

cudaError_t launch_combos_bt(const Sched &s, const uint64_t *B, int64_t ldb, int64_t pb, int64_t k, int64_t n,
                             uint64_t *out, int64_t ldo, int64_t po, int64_t kblocks, int64_t nblocks, bool fp4,
                             cudaStream_t st, int br, int64_t row0, bool expand) {
    int64_t warps = (kblocks >> 1) * nblocks;  // kblocks is even (k_pad is a multiple of 128)
    if (warps == 0) return cudaSuccess;
    int tsplit = 1;
    while (tsplit < s.nprod && warps * tsplit * 2 <= 148 * 16) tsplit *= 2;
    int g = grid_for(warps * tsplit * 32, 256);
    return dispatch_e(s.e, [&](auto ec) {
        k_combos_bt<decltype(ec)::value><<<g, 256, 0, st>>>(s, B, ldb, pb, k, n, out, ldo, po, kblocks, nblocks,
                                                            fp4 ? 1 : 0, tsplit, br, row0, expand ? 1 : 0);
        return cudaGetLastError();
    });
}

}  // namespace gf2e

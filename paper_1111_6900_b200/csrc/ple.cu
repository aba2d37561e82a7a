// ple.cu — device kernels of the PLE decomposition consumer:
//
//   k_ple_find / k_ple_apply: the quadratic base case `nj_ple` (newton_john.py:207-260) on one
//     64-column panel of a sliced matrix (one plane word per row per plane).  nj_ple walks the
//     panel's columns; for column j it takes the first row at or below position r whose entry
//     is nonzero as pivot, swaps it to r, rescales the pivot row right of j by 1/pivot, and
//     XORs x_i * (pivot row right of j) into every row below (the multiplier x_i stays in
//     place as L).  Only the pivot search and the pivot row are sequential, so:
//       phase 1 (one CTA): keeps a window of the first 128 row positions in shared memory,
//         reduced step by step; finds each pivot there (or, if the window has none, scans the
//         rows below it lazily, reducing each candidate by the pivots found so far); records
//         the pivots, the swaps, and the basis tables alpha^s * T_t of every scaled pivot
//         suffix T_t; writes the window rows back.
//       phase 2 (all SMs): every row below the window applies the panel's <= 64 eliminations
//         in order (x = entry at the pivot column, row ^= sum_s x_s * alpha^s * T_t) — one
//         independent job per row.
//     Both phases finish with the base case's L compression (column swaps t <-> Q[t] for rows
//     >= t, newton_john.py:257-259).
//   k_row_swaps:  LAPACK-style swap vectors on a window (apply_perm_rows, ple_echelon.py:81-91).
//   k_col_swaps:  a sequence of (column a, column b, first row) swaps on w-bit slots — bit
//     planes (w = 1) or packed words (w = pack width) (PackedMatrix.col_swap, used at
//     ple_echelon.py:275-279, 311-313, 359-362).
//   k_tril_copy:  the r x r corner with entries above the diagonal cleared (_tril_with_diag,
//     ple_echelon.py:223-237).
//   k_echelon_marks: echelonize's "drop L, set the implicit leading ones" (ple_echelon.py:364-370).
//   k_gather_cols: pivot columns of the leading rows as an r x r matrix (_gather_columns,
//     ple_echelon.py:338-340).
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace gf2e {
namespace {

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// ---- per-field constant tables (static module memory, filled once per (e, f)) ----------------

// window rows of the panel kernel: 128, or 64 for e >= GF2E_PLE_WIN64_E (a window row is
// nonzero at a pivot column with probability 1 - 2^-e, so 64 rows leave the lazy scan below
// the window practically unused there while halving the panel kernel's threads)
#ifndef GF2E_PLE_WIN64_E
#define GF2E_PLE_WIN64_E 5
#endif
template <int E>
constexpr int ple_win() { return E >= GF2E_PLE_WIN64_E ? 64 : 128; }
constexpr int KP = 64;   // pivots per panel (one plane word)

__device__ __forceinline__ uint64_t swap_bits(uint64_t w, int a, int b) {
    const uint64_t d = ((w >> a) ^ (w >> b)) & 1ULL;
    return w ^ (d << a) ^ (d << b);
}

template <int E>
__device__ __forceinline__ uint32_t elemE(const uint64_t *v, int c) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < E; ++b) x |= (uint32_t)((v[b] >> c) & 1ULL) << b;
    return x;
}
// v ^= x * T_t, bt = [alpha^s * T_t][plane]
template <int E>
__device__ __forceinline__ void stepE(uint64_t *v, uint32_t x, const uint64_t *bt) {
#pragma unroll
    for (int s = 0; s < E; ++s) {
        const uint64_t sel = 0ULL - (uint64_t)((x >> s) & 1u);
#pragma unroll
        for (int b = 0; b < E; ++b) v[b] ^= bt[s * E + b] & sel;
    }
}

// Window threads: TPR lanes of one warp per window row, lane b holding plane b (an entry is
// one ballot); 1024 threads, RP rows per pass.
// lanes per window row (measured per e, PLE 8192^2: e = 4 20.9 ms at 4 lanes vs 23.5 at 8;
// e = 8 28.7 ms at 8 vs 30.0 at 4 and 33.0 at 2; e = 10 46.7 at 16 vs 47.2 at 8)
template <int E>
struct FindShape {
    static constexpr int PT = ple_win<E>();      // window rows
    static constexpr int TPR = E <= 4 ? 4 : E <= 8 ? 8 : 16;
    static constexpr int PPL = (E + TPR - 1) / TPR;  // planes per lane: sub, sub + TPR, ...
    static constexpr int NT = PT * TPR < 1024 ? PT * TPR : 1024;
    static constexpr int RP = NT / TPR;           // window rows per pass
    static constexpr int PASSES = (PT + RP - 1) / RP;
    static constexpr uint32_t EMASK = (1u << E) - 1;
};

// first row (of the ballot's row groups) whose group has a set bit: the lowest set lane
template <int TPR>
__device__ __forceinline__ int first_row(unsigned bal, int row_of_lane0) {
    return row_of_lane0 + (__ffs(bal) - 1) / TPR;
}

template <int E>
__global__ void __launch_bounds__(FindShape<E>::NT) k_ple_find(const FieldTab *__restrict__ tab, uint64_t *__restrict__ S,
                                                   int64_t ld, int64_t ps, int64_t m, int nb,
                                                   PanelOut *__restrict__ out) {
    using F = FindShape<E>;
    using SP = PleSplit<E>;
    constexpr int NT = F::NT, TPR = F::TPR, PT = F::PT, PPL = F::PPL;
    constexpr uint32_t GMASK = TPR >= 32 ? 0xffffffffu : ((1u << TPR) - 1);
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t *win = reinterpret_cast<uint64_t *>(smem);  // [PT][E]
    uint64_t *ptab = win + PT * E;                       // [Q][E]: multiples of the current T_r
    uint32_t *smm = reinterpret_cast<uint32_t *>(ptab + SP::QE);  // [2^E][E] mulmask2
    uint16_t *sinv = reinterpret_cast<uint16_t *>(smm + (1 << E) * E);  // [2^E] inverses
    __shared__ uint64_t ext[kMaxE], prow[kMaxE], oldr[kMaxE];
    __shared__ uint64_t s_dval[KP][kMaxE];
    __shared__ int64_t dpos[KP];
    __shared__ int dstep[KP], s_jcol[KP];
    __shared__ int64_t s_P[KP], s_Q[KP];
    __shared__ int s_mn[2], s_nd, s_supp_ok;
    __shared__ unsigned long long s_supp;
    __shared__ int64_t s_pmin;

    pdl_trigger();
    const int tid = threadIdx.x;
    const int lane = tid & 31, b = tid % TPR, gl = lane - b, rl = tid / TPR;
    const int W = (int)(m < PT ? m : PT);
    const uint64_t cmask = nb >= 64 ? ~0ULL : ((1ULL << nb) - 1);
    const int k = (int)(m < nb ? m : nb);
    if (tid == 0) {
        s_nd = 0;
        s_supp_ok = 0;
        s_supp = 0;
        s_mn[0] = 0x7fffffff;
    }
    for (int i = tid; i < (1 << E); i += NT) {
        sinv[i] = tab->inv[i];
#pragma unroll
        for (int q = 0; q < E; ++q) smm[i * E + q] = tab->mulmask2[i][q];
    }
    __syncthreads();
    pdl_wait();  // the field tables above are constant; S and out come from the chain
    // window rows; candidates for column 0 (lowest row of each warp with a nonzero entry)
#pragma unroll
    for (int pass = 0; pass < F::PASSES; ++pass) {
        const int s = pass * F::RP + rl;
        uint64_t any = 0;
#pragma unroll
        for (int sl = 0; sl < PPL; ++sl) {
            const int bb = b + TPR * sl;
            if (s < W && bb < E) {
                const uint64_t x = S[bb * ps + s * ld] & cmask;
                win[s * E + bb] = x;
                any |= x;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, any & 1ULL);
        if (lane == 0 && bal) atomicMin(&s_mn[0], first_row<TPR>(bal, pass * F::RP + (tid - lane) / TPR));
    }
    __syncthreads();
    int r = 0;
    // Two barriers per pivot: (pivot found: table of its multiples, bookkeeping) | (pivot row
    // written, rows below eliminated with two table words per plane, candidates for the next
    // column).  The candidate minimum is double-buffered (s_mn[j & 1]).
    for (int j = 0; j < nb && r < k; ++j) {
        const int cb = j & 1;
        int64_t ipos = s_mn[cb];
        if (ipos == 0x7fffffff && W < m) {
            // Column support of the rows below the window: their original bits OR the scaled
            // pivot suffixes (the only things ever XOR-ed into them).  Computed at the first
            // miss; a column outside it has no pivot below the window either.
            if (tid == 0) s_pmin = INT64_MAX;
            if (!s_supp_ok) {
                uint64_t acc = 0;
                for (int64_t p = W + tid; p < m; p += NT)
#pragma unroll
                    for (int q = 0; q < E; ++q) acc |= S[q * ps + p * ld];
                if (acc) atomicOr(&s_supp, acc & cmask);
                for (int t = tid; t < r; t += NT)
#pragma unroll
                    for (int q = 0; q < E; ++q) atomicOr(&s_supp, out->tabs[t * kPleTabWords + E + q]);
                __syncthreads();
                if (tid == 0) s_supp_ok = 1;
            }
            __syncthreads();
            if ((s_supp >> j) & 1ULL) {
                // scan the rows below the window, reducing each candidate lazily by the tables
                // of the pivots so far (written to global memory by this CTA)
                const int nd = s_nd;
                for (int64_t base = W; base < m; base += NT) {
                    const int64_t p = base + tid;
                    uint64_t v[E];
                    bool hit = false;
                    if (p < m) {
                        int st0 = 0, di = -1;
                        for (int d = 0; d < nd; ++d)
                            if (dpos[d] == p) di = d;
                        if (di >= 0) {
#pragma unroll
                            for (int q = 0; q < E; ++q) v[q] = s_dval[di][q];
                            st0 = dstep[di];
                        } else {
#pragma unroll
                            for (int q = 0; q < E; ++q) v[q] = S[q * ps + p * ld] & cmask;
                        }
                        for (int t = st0; t < r; ++t) {
                            const uint32_t x = elemE<E>(v, s_jcol[t]);
                            if (!x) continue;
                            const uint64_t *tt = out->tabs + t * kPleTabWords;
                            const uint64_t *lo = tt + (x & ((1u << SP::H1) - 1)) * E;
                            if constexpr (SP::H2 > 0) {
                                const uint64_t *hi = tt + ((1u << SP::H1) + (x >> SP::H1)) * E;
#pragma unroll
                                for (int q = 0; q < E; ++q) v[q] ^= lo[q] ^ hi[q];
                            } else {
#pragma unroll
                                for (int q = 0; q < E; ++q) v[q] ^= lo[q];
                            }
                        }
                        uint64_t any = 0;
#pragma unroll
                        for (int q = 0; q < E; ++q) any |= v[q];
                        hit = (any >> j) & 1ULL;
                        if (hit) atomicMin((unsigned long long *)&s_pmin, (unsigned long long)p);
                    }
                    __syncthreads();
                    if (hit && s_pmin == p)
#pragma unroll
                        for (int q = 0; q < E; ++q) ext[q] = v[q];
                    __syncthreads();
                    if (s_pmin != INT64_MAX) break;
                }
                ipos = s_pmin;
            }
        }
        if (ipos == 0x7fffffff || ipos == INT64_MAX) {
            // no pivot in column j: collect the window's candidates for column j + 1
            if (tid == 0) s_mn[cb ^ 1] = 0x7fffffff;
            __syncthreads();
            if (j + 1 < nb)
#pragma unroll
                for (int pass = 0; pass < F::PASSES; ++pass) {
                    const int s = pass * F::RP + rl;
                    uint64_t any = 0;
#pragma unroll
                    for (int sl = 0; sl < PPL; ++sl)
                        if (s >= r && s < W && b + TPR * sl < E) any |= win[s * E + b + TPR * sl];
                    const unsigned bal = __ballot_sync(0xffffffffu, (any >> (j + 1)) & 1ULL);
                    if (lane == 0 && bal)
                        atomicMin(&s_mn[cb ^ 1], first_row<TPR>(bal, pass * F::RP + (tid - lane) / TPR));
                }
            __syncthreads();
            continue;
        }
        // ---- phase A: the pivot row P (window row ipos, or ext from below the window) ----
        const uint64_t *P = ipos < W ? win + ipos * E : ext;
        const uint64_t sm = (j >= 63 ? 0ULL : (~0ULL << (j + 1))) & cmask;  // suffix right of j
        // table of the multiples of T_r = (P right of j) / pivot: entry x of the low half is
        // x * T_r, of the high half (x << H1) * T_r; plane b of c * T_r is the XOR of the
        // planes p of T_r with bit p of mulmask[c][b], and mulmask[y / pivot][b] is the XOR of
        // mulmask2[1 / pivot][b] >> s over the bits s of y
        for (int idx = tid; idx < SP::QE; idx += NT) {
            const int x = idx / E, q = idx - (idx / E) * E;
            const uint32_t y = x < (1 << SP::H1) ? (uint32_t)x : (uint32_t)(x - (1 << SP::H1)) << SP::H1;
            uint64_t pv[E];
#pragma unroll
            for (int p = 0; p < E; ++p) pv[p] = P[p];
            const uint32_t pinv = sinv[elemE<E>(pv, j)];
            const uint32_t m2 = smm[pinv * E + q];
            uint32_t mk = 0;
#pragma unroll
            for (int s = 0; s < E; ++s)
                if ((y >> s) & 1u) mk ^= m2 >> s;
            uint64_t acc = 0;
#pragma unroll
            for (int p = 0; p < E; ++p)
                if ((mk >> p) & 1u) acc ^= pv[p];
            acc &= sm;
            ptab[idx] = acc;
            out->tabs[r * kPleTabWords + idx] = acc;
        }
        if (tid >= NT - 32) {  // last warp: bookkeeping (no table words there)
            if (tid - (NT - 32) < E) {
                const int q = tid - (NT - 32);
                prow[q] = P[q];
                oldr[q] = win[r * E + q];
            }
            if (tid == NT - 1) {
                if (ipos >= W) {
                    // the row at position r moves below the window: remember it (reduced by
                    // steps < r)
                    int di = -1;
                    for (int d = 0; d < s_nd; ++d)
                        if (dpos[d] == ipos) di = d;
                    if (di < 0) di = s_nd++;
                    dpos[di] = ipos;
                    dstep[di] = r;
#pragma unroll
                    for (int q = 0; q < E; ++q) s_dval[di][q] = win[r * E + q];
                }
                s_P[r] = ipos;
                s_Q[r] = j;
                s_jcol[r] = j;
                s_mn[cb ^ 1] = 0x7fffffff;  // candidates for column j + 1 (collected below)
            }
        }
        __syncthreads();
        // ---- phase B: pivot row to position r (prefix kept, suffix scaled), eliminations ----
        if (tid < E) {
            const uint64_t t0 = ptab[E + tid];  // entry 1: the scaled suffix itself
            win[r * E + tid] = (prow[tid] & ~sm) | t0;
            if (s_supp_ok) atomicOr(&s_supp, t0);
        }
        const bool next = j + 1 < nb;
#pragma unroll
        for (int pass = 0; pass < F::PASSES; ++pass) {
            const int s = pass * F::RP + rl;
            const bool act = s > r && s < W;
            uint64_t v[PPL];
            uint32_t x = 0;
#pragma unroll
            for (int sl = 0; sl < PPL; ++sl) {  // lane b holds planes b, b + TPR, ...
                const int bb = b + TPR * sl;
                v[sl] = 0;
                if (act && bb < E) v[sl] = (s == ipos) ? oldr[bb] : win[s * E + bb];  // old row r moved to ipos
                const unsigned bal = __ballot_sync(0xffffffffu, (v[sl] >> j) & 1ULL);
                x |= ((bal >> gl) & GMASK) << (TPR * sl);
            }
            x &= F::EMASK;
            uint64_t any = 0;
#pragma unroll
            for (int sl = 0; sl < PPL; ++sl) {
                const int bb = b + TPR * sl;
                if (act && bb < E && (x || s == ipos)) {
                    if (x) {
                        if constexpr (SP::H2 > 0)
                            v[sl] ^= ptab[(x & ((1u << SP::H1) - 1)) * E + bb] ^
                                     ptab[((1u << SP::H1) + (x >> SP::H1)) * E + bb];
                        else
                            v[sl] ^= ptab[x * E + bb];
                    }
                    win[s * E + bb] = v[sl];
                }
                any |= v[sl];
            }
            if (next) {
                const unsigned bal2 = __ballot_sync(0xffffffffu, act && ((any >> (j + 1)) & 1ULL));
                if (lane == 0 && bal2)
                    atomicMin(&s_mn[cb ^ 1], first_row<TPR>(bal2, pass * F::RP + (tid - lane) / TPR));
            }
        }
        ++r;
        __syncthreads();
    }
    // L compression of the base case (newton_john.py:257-259) and write-back of the window
#pragma unroll
    for (int pass = 0; pass < F::PASSES; ++pass) {
        const int s = pass * F::RP + rl;
#pragma unroll
        for (int sl = 0; sl < PPL; ++sl) {
            const int bb = b + TPR * sl;
            if (s < W && bb < E) {
                uint64_t v = win[s * E + bb];
                for (int t = 0; t < r && t <= s; ++t) {
                    const int q = (int)s_Q[t];
                    if (q != t) v = swap_bits(v, t, q);
                }
                uint64_t *d = S + bb * ps + s * ld;
                *d = (*d & ~cmask) | v;
            }
        }
    }
    // outputs for phase 2 and the host
    if (tid < r) {
        out->P[tid] = s_P[tid];
        out->Q[tid] = s_Q[tid];
        out->jcol[tid] = s_jcol[tid];
    }
    if (tid < s_nd) {
        out->dpos[tid] = dpos[tid];
        out->dstep[tid] = dstep[tid];
#pragma unroll
        for (int q = 0; q < E; ++q) out->dval[tid][q] = s_dval[tid][q];
    }
    if (tid == 0) {
        out->rank = r;
        out->ndisp = s_nd;
        out->window = W;
    }
}

// phase 2: rows at positions >= window apply the panel's eliminations and the L compression.
// Row p is owned by TPR lanes of one warp, lane b holding plane b: the entry at a pivot
// column is one ballot, and the elimination row ^= x * T_t is two looked-up words of the
// panel's multiple tables (PanelOut.tabs, staged in shared memory CH pivots at a time).
template <int E>
struct ApplyShape {
    static constexpr int THREADS = 512;
    static constexpr int TPR = E <= 8 ? 8 : 16;      // lanes per row (planes >= E idle)
    static constexpr int RPC = THREADS / TPR;         // rows per CTA
    static constexpr int CH = 32;                     // pivots per table chunk
    static constexpr size_t SMEM = (size_t)CH * PleSplit<E>::QE * 8;
};

template <int E>
__global__ void __launch_bounds__(512) k_ple_apply(uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t m, int nb,
                                                   const PanelOut *__restrict__ in) {
    pdl_trigger();
    pdl_wait();
    using A = ApplyShape<E>;
    using SP = PleSplit<E>;
    extern __shared__ __align__(16) uint64_t ctab[];  // [CH][Q][E]
    __shared__ int jc[KP], qc[KP], dst[KP];
    __shared__ int64_t dps[KP];
    __shared__ int r_s, nd_s, w_s;
    if (threadIdx.x == 0) {
        r_s = in->rank;
        nd_s = in->ndisp;
        w_s = in->window;
    }
    __syncthreads();
    const int r = r_s, nd = nd_s;
    for (int i = threadIdx.x; i < r; i += A::THREADS) {
        jc[i] = in->jcol[i];
        qc[i] = (int)in->Q[i];
    }
    for (int i = threadIdx.x; i < nd; i += A::THREADS) {
        dps[i] = in->dpos[i];
        dst[i] = in->dstep[i];
    }
    const uint64_t cmask = nb >= 64 ? ~0ULL : ((1ULL << nb) - 1);
    const int lane = threadIdx.x & 31, b = threadIdx.x % A::TPR, gl = lane - b;
    const int64_t p = w_s + (int64_t)blockIdx.x * A::RPC + threadIdx.x / A::TPR;
    const bool mine = p < m && b < E;
    __syncthreads();
    uint64_t v = 0;
    int st0 = 0;
    if (mine) {
        int di = -1;
        for (int d = 0; d < nd; ++d)
            if (dps[d] == p) di = d;
        if (di >= 0) {
            v = in->dval[di][b];
            st0 = dst[di];
        } else {
            v = S[b * ps + p * ld] & cmask;
        }
    }
    for (int c0 = 0; c0 < r; c0 += A::CH) {
        const int c1 = c0 + A::CH < r ? c0 + A::CH : r;
        if (c0) __syncthreads();  // the previous chunk's readers are done
        const uint64_t *src = in->tabs + (size_t)c0 * kPleTabWords;
        for (int i = threadIdx.x; i < (c1 - c0) * SP::QE; i += A::THREADS) {
            const int t = i / SP::QE;
            ctab[i] = src[(size_t)t * kPleTabWords + (i - t * SP::QE)];
        }
        __syncthreads();
        for (int t = c0; t < c1; ++t) {
            const unsigned bal = __ballot_sync(0xffffffffu, (v >> jc[t]) & 1ULL);
            const uint32_t x = (bal >> gl) & ((1u << E) - 1);
            if (mine && t >= st0 && x) {
                const uint64_t *tt = ctab + (size_t)(t - c0) * SP::QE;
                if constexpr (SP::H2 > 0)
                    v ^= tt[(x & ((1u << SP::H1) - 1)) * E + b] ^ tt[((1u << SP::H1) + (x >> SP::H1)) * E + b];
                else
                    v ^= tt[x * E + b];
            }
        }
    }
    if (mine) {
        for (int t = 0; t < r; ++t)
            if (qc[t] != t) v = swap_bits(v, t, qc[t]);
        uint64_t *d = S + b * ps + p * ld;
        *d = (*d & ~cmask) | v;
    }
}

// (a, b) row pairs applied in order (backward: reverse order); the host drops identity
// entries of a swap vector, so a random matrix's factorisation swaps almost nothing.
// Thread = (plane, word).
__global__ void k_row_swaps(int planes, uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t nwords,
                            const int64_t *__restrict__ pairs, int n, int backward) {
    const int64_t total = (int64_t)planes * nwords;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t b = idx / nwords, w = idx % nwords;
        uint64_t *col = S + b * ps + w;
        for (int i = 0; i < n; ++i) {
            const int u = backward ? n - 1 - i : i;
            const int64_t ra = pairs[2 * u], rb = pairs[2 * u + 1];
            const uint64_t x = col[ra * ld];
            col[ra * ld] = col[rb * ld];
            col[rb * ld] = x;
        }
    }
}

// LAPACK-style swaps t <-> Pg[t] for t in [t0, t1), in order, on a column window (the
// speculative PLE: the pivots stay in device memory, ple_commit)
__global__ void k_row_swaps_vec(int planes, uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t nwords,
                                const int64_t *__restrict__ Pg, int64_t t0, int64_t t1) {
    pdl_trigger();
    pdl_wait();
    // the pivots are staged in shared memory and compacted to the non-trivial swaps (a generic
    // matrix pivots on the diagonal almost everywhere), 1024 pivot positions at a time; 128
    // threads per block (the compaction's layout)
    __shared__ int64_t sp[1024][2];
    __shared__ int cnt;
    const int64_t total = (int64_t)planes * nwords;
    const int64_t idx = gtid();
    const int64_t b = idx / nwords, w = idx % nwords;
    uint64_t *col = idx < total ? S + b * ps + w : nullptr;
    for (int64_t c0 = t0; c0 < t1; c0 += 1024) {
        const int64_t c1 = c0 + 1024 < t1 ? c0 + 1024 : t1;
        // ordered compaction: thread i owns positions c0 + 8i .. c0 + 8i + 7 (blockDim 128)
        __shared__ int wsum[4];
        int64_t u[8];
        int mine = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t t = c0 + 8 * threadIdx.x + j;
            u[j] = t < c1 ? Pg[t] : t;
            mine += u[j] != t;
        }
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        int base = incl - mine;
        for (int q = 0; q < wid; ++q) base += wsum[q];
        if (threadIdx.x == 127) cnt = base + mine;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t t = c0 + 8 * threadIdx.x + j;
            if (u[j] != t) {
                sp[base][0] = t;
                sp[base][1] = u[j];
                ++base;
            }
        }
        __syncthreads();
        if (col)
            for (int i = 0; i < cnt; ++i) {
                const int64_t t = sp[i][0], u = sp[i][1];
                const uint64_t x = col[t * ld];
                col[t * ld] = col[u * ld];
                col[u * ld] = x;
            }
        __syncthreads();
    }
}

// a panel's pivots into the global swap vectors (P[r0 + t] = r0 + P_panel[t], Q likewise with
// the column offset); a rank other than the speculated one raises the flag
__global__ void k_ple_commit(const PanelOut *__restrict__ po, int64_t *__restrict__ Pg, int64_t *__restrict__ Qg,
                             int64_t r0, int64_t c0, int expected, int *__restrict__ flag) {
    pdl_trigger();
    pdl_wait();
    const int r = po->rank;
    for (int t = threadIdx.x; t < expected; t += blockDim.x) {
        Pg[r0 + t] = t < r ? r0 + po->P[t] : r0 + t;
        Qg[r0 + t] = t < r ? c0 + po->Q[t] : c0 + t;
    }
    if (threadIdx.x == 0 && r != expected) atomicOr(flag, 1);
}

// (a, b, first row) triples applied in order to w-bit slots; thread = (plane, row)
__global__ void k_col_swaps(int planes, int w, uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t rows,
                            const int64_t *__restrict__ trip, int n) {
    const int64_t total = (int64_t)planes * rows;
    const uint64_t fm = w >= 64 ? ~0ULL : ((1ULL << w) - 1);
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t b = idx / rows, i = idx % rows;
        uint64_t *row = S + b * ps + i * ld;
        for (int t = 0; t < n; ++t) {
            const int64_t ca = trip[3 * t], cb = trip[3 * t + 1], r0 = trip[3 * t + 2];
            if (i < r0 || ca == cb) continue;
            const int64_t ba = ca * w, bb = cb * w;
            uint64_t *wa = row + (ba >> 6), *wb = row + (bb >> 6);
            const int sa = (int)(ba & 63), sb = (int)(bb & 63);
            const uint64_t va = (*wa >> sa) & fm, vb = (*wb >> sb) & fm;
            *wa = (*wa & ~(fm << sa)) | (vb << sa);
            *wb = (*wb & ~(fm << sb)) | (va << sb);
        }
    }
}

// out[i][c] = S[i][c] for c <= i < r, 0 above the diagonal
__global__ void k_tril_copy(int e, const uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t r,
                            uint64_t *__restrict__ out, int64_t ldo, int64_t po) {
    pdl_trigger();
    pdl_wait();
    const int64_t nw = words_for(r);
    const int64_t total = (int64_t)e * r * nw;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t b = idx / (r * nw), rem = idx % (r * nw), i = rem / nw, w = rem % nw;
        uint64_t v = S[b * ps + i * ld + w];
        const int64_t lo = w * 64;
        uint64_t keep;
        if (i < lo) keep = 0;
        else if (i - lo >= 63) keep = ~0ULL;
        else keep = (2ULL << (i - lo)) - 1;
        if (w == nw - 1) keep &= tail_mask(r);
        out[b * po + i * ldo + w] = v & keep;
    }
}

// echelonize: rows >= t lose column Q[t]; row t < r gets the leading one at Q[t]
// Row i clears the pivot columns Q[t], t <= min(i, r - 1), in every plane, and row i < r sets
// its leading one.  Thread = (row, column word); the host lists, per column word, the pivots
// it holds in increasing t (tpos) with prefix ORs of their bits (pmask), so a thread's mask is
// one binary search away.
__global__ void k_echelon_marks(int e, uint64_t *__restrict__ S, int64_t ld, int64_t ps, int64_t m, int64_t nw,
                                const int64_t *__restrict__ Q, int r, const int *__restrict__ wstart,
                                const int *__restrict__ tpos, const uint64_t *__restrict__ pmask) {
    const int64_t total = m * nw;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t i = idx / nw, w = idx - i * nw;
        const int tmax = (int)(i < r - 1 ? i : r - 1);
        int lo = wstart[w], hi = wstart[w + 1];  // first entry with tpos > tmax
        const int base = lo;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tpos[mid] <= tmax)
                lo = mid + 1;
            else
                hi = mid;
        }
        const uint64_t mask = lo > base ? pmask[lo - 1] : 0ULL;
        if (mask)
            for (int b = 0; b < e; ++b) S[b * ps + i * ld + w] &= ~mask;
        if (i < r && (Q[i] >> 6) == w) S[i * ld + w] |= 1ULL << (Q[i] & 63);
    }
}

// out[i][t] = S[i][Q[t]], i, t < r
__global__ void k_gather_cols(int e, const uint64_t *__restrict__ S, int64_t ld, int64_t ps, const int64_t *__restrict__ Q,
                              int64_t r, uint64_t *__restrict__ out, int64_t ldo, int64_t po) {
    const int64_t nw = words_for(r);
    const int64_t total = (int64_t)e * r * nw;
    for (int64_t idx = gtid(); idx < total; idx += gstride()) {
        const int64_t b = idx / (r * nw), rem = idx % (r * nw), i = rem / nw, w = rem % nw;
        uint64_t v = 0;
        for (int u = 0; u < 64 && w * 64 + u < r; ++u) {
            const int64_t c = Q[w * 64 + u];
            v |= ((S[b * ps + i * ld + (c >> 6)] >> (c & 63)) & 1ULL) << u;
        }
        out[b * po + i * ldo + w] = v;
    }
}

inline int grid_for(int64_t total, int threads) {
    int64_t g = (total + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

template <int E>
cudaError_t launch_ple_e(const FieldTab *tab, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int nb, PanelOut *out,
                         cudaStream_t st) {
    constexpr int PT = FindShape<E>::PT;
    const int smem = (PT * E + PleSplit<E>::QE) * 8 + (1 << E) * E * 4 + (1 << E) * 2;
    const int smem2 = (int)ApplyShape<E>::SMEM;
    // launch attributes once per instantiation and device (idempotent)
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t err = cudaSuccess;
    if (dev >= kMaxDevices || !attr_set[dev]) {
        err = cudaFuncSetAttribute(k_ple_find<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_ple_apply<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        if (err != cudaSuccess) return err;
        if (dev < kMaxDevices) attr_set[dev] = true;
    }
    err = launch_pdl(k_ple_find<E>, dim3(1), dim3(FindShape<E>::NT), smem, st, tab, S, ld, ps, m, nb, out);
    if (err != cudaSuccess || m <= PT) return err;
    using A = ApplyShape<E>;
    return launch_pdl(k_ple_apply<E>, dim3((unsigned)((m - PT + A::RPC - 1) / A::RPC)), dim3(A::THREADS), smem2, st, S,
                      ld, ps, m, nb, (const PanelOut *)out);
}

bool pdl_enabled() {
    static const bool on = !getenv("GF2E_PDL") || atoi(getenv("GF2E_PDL")) != 0;
    return on;
}

int ple_window(int e) { return e >= GF2E_PLE_WIN64_E ? 64 : 128; }

cudaError_t launch_ple_panel(int e, const FieldTab *tab, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int nb,
                             PanelOut *out, cudaStream_t st) {
    switch (e) {
        case 2: return launch_ple_e<2>(tab, S, ld, ps, m, nb, out, st);
        case 3: return launch_ple_e<3>(tab, S, ld, ps, m, nb, out, st);
        case 4: return launch_ple_e<4>(tab, S, ld, ps, m, nb, out, st);
        case 5: return launch_ple_e<5>(tab, S, ld, ps, m, nb, out, st);
        case 6: return launch_ple_e<6>(tab, S, ld, ps, m, nb, out, st);
        case 7: return launch_ple_e<7>(tab, S, ld, ps, m, nb, out, st);
        case 8: return launch_ple_e<8>(tab, S, ld, ps, m, nb, out, st);
        case 9: return launch_ple_e<9>(tab, S, ld, ps, m, nb, out, st);
        case 10: return launch_ple_e<10>(tab, S, ld, ps, m, nb, out, st);
        default: return cudaErrorInvalidValue;
    }
}

// host: gf(2^e) tables over a primitive element g; mulmask[c][b] bit p = coefficient b of c*x^p
static uint32_t gf_mul_h(uint32_t a, uint32_t b, int e, uint32_t f) {
    uint32_t acc = 0;
    for (int i = 0; i < e; ++i)
        if ((b >> i) & 1u) acc ^= a << i;
    for (int d = 2 * e - 2; d >= e; --d)
        if ((acc >> d) & 1u) acc ^= f << (d - e);
    return acc;
}

// One table per (device, e, f), allocated on first use and kept for the process lifetime:
// a returned pointer is never reused for another field, so no kernel can read a table that
// another thread replaced (at most ~230 irreducible f of degree 2..10, 26 KiB each).
const FieldTab *field_tab(int e, uint32_t f, uint32_t g) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, uint32_t>, FieldTab *> tabs;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    auto it = tabs.find({dev, e, f});
    if (it != tabs.end()) return it->second;
    static FieldTab h;
    std::memset(&h, 0, sizeof(h));
    h.f = f;
    const uint32_t q1 = (1u << e) - 1;
    uint32_t v = 1;
    for (uint32_t i = 0; i < q1; ++i) {
        h.ex[i] = (uint16_t)v;
        h.lg[v] = (uint16_t)i;
        v = gf_mul_h(v, g, e, f);
    }
    for (uint32_t a = 1; a <= q1; ++a) h.inv[a] = h.ex[(q1 - h.lg[a]) % q1];
    for (uint32_t c = 0; c <= q1; ++c)
        for (int p = 0; p < e; ++p) {
            const uint32_t prod = gf_mul_h(c, 1u << p, e, f);
            for (int b = 0; b < e; ++b)
                if ((prod >> b) & 1u) h.mulmask[c][b] |= (uint16_t)(1u << p);
        }
    for (uint32_t c = 0; c <= q1; ++c) {
        uint32_t prod = c;  // c * x^p
        for (int p = 0; p < 2 * e - 1; ++p) {
            for (int b = 0; b < e; ++b)
                if ((prod >> b) & 1u) h.mulmask2[c][b] |= 1u << p;
            prod = gf_mul_h(prod, 2u, e, f);
        }
    }
    FieldTab *d = nullptr;
    if (cudaMalloc(reinterpret_cast<void **>(&d), sizeof(FieldTab)) != cudaSuccess) return nullptr;
    // complete before any kernel (on any stream) can be enqueued with d: a pageable cudaMemcpy
    // may return before its DMA lands, so wait for the legacy stream it ran on
    if (cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    tabs[{dev, e, f}] = d;
    return d;
}

cudaError_t launch_row_swaps(int planes, uint64_t *S, int64_t ld, int64_t ps, int64_t nwords, const int64_t *swaps,
                             int n, bool backward, cudaStream_t st) {
    if (n == 0 || nwords == 0) return cudaSuccess;
    k_row_swaps<<<grid_for((int64_t)planes * nwords, 128), 128, 0, st>>>(planes, S, ld, ps, nwords, swaps, n,
                                                                        backward ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_row_swaps_vec(int planes, uint64_t *S, int64_t ld, int64_t ps, int64_t nwords, const int64_t *Pg,
                                 int64_t t0, int64_t t1, cudaStream_t st) {
    if (t1 <= t0 || nwords == 0) return cudaSuccess;
    const int64_t total = (int64_t)planes * nwords;
    return launch_pdl(k_row_swaps_vec, dim3((unsigned)((total + 127) / 128)), dim3(128), 0, st, planes, S, ld, ps, nwords,
                      Pg, t0, t1);
}

cudaError_t launch_ple_commit(const PanelOut *po, int64_t *Pg, int64_t *Qg, int64_t r0, int64_t c0, int expected,
                              int *flag, cudaStream_t st) {
    if (expected <= 0) return cudaSuccess;
    return launch_pdl(k_ple_commit, dim3(1), dim3(64), 0, st, po, Pg, Qg, r0, c0, expected, flag);
}

cudaError_t launch_col_swaps(int planes, int w, uint64_t *S, int64_t ld, int64_t ps, int64_t rows, const int64_t *trip,
                             int n, cudaStream_t st) {
    if (n == 0 || rows == 0) return cudaSuccess;
    k_col_swaps<<<grid_for((int64_t)planes * rows, 256), 256, 0, st>>>(planes, w, S, ld, ps, rows, trip, n);
    return cudaGetLastError();
}

cudaError_t launch_tril_copy(int e, const uint64_t *S, int64_t ld, int64_t ps, int64_t r, uint64_t *out, int64_t ldo,
                             int64_t po, cudaStream_t st) {
    if (r == 0) return cudaSuccess;
    return launch_pdl(k_tril_copy, dim3(grid_for((int64_t)e * r * words_for(r), 256)), dim3(256), 0, st, e, S, ld, ps,
                      r, out, ldo, po);
}

cudaError_t launch_echelon_marks(int e, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t nw, const int64_t *Q,
                                 int r, const int *wstart, const int *tpos, const uint64_t *pmask, cudaStream_t st) {
    if (r == 0 || m == 0) return cudaSuccess;
    k_echelon_marks<<<grid_for(m * nw, 256), 256, 0, st>>>(e, S, ld, ps, m, nw, Q, r, wstart, tpos, pmask);
    return cudaGetLastError();
}

cudaError_t launch_gather_cols(int e, const uint64_t *S, int64_t ld, int64_t ps, const int64_t *Q, int64_t r,
                               uint64_t *out, int64_t ldo, int64_t po, cudaStream_t st) {
    if (r == 0) return cudaSuccess;
    k_gather_cols<<<grid_for((int64_t)e * r * words_for(r), 256), 256, 0, st>>>(e, S, ld, ps, Q, r, out, ldo, po);
    return cudaGetLastError();
}

}  // namespace gf2e

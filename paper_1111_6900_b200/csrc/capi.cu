// capi.cu — the extern "C" boundary of libgf2e_b200.so (declared in include/gf2e_b200.h):
// argument validation with the reference's error semantics, the native Karatsuba
// schedule, workspace carving, and the launch sequence of the hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gf2e_b200.h"
#include "common.cuh"
#include "kernels.h"

using namespace gf2e;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local int64_t g_products = 0;  // GF(2) plane products launched by the last entry call
thread_local const char *g_kernel = "";

// live product-kernel timing (gf2e_profile_*)
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_events;

struct ProfScope {
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    explicit ProfScope(cudaStream_t s) : st(s) {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        if (!g_prof_on) return;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEventRecord(b, st);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof_events.emplace_back(a, b);
    }
};

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(GF2E_ECUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

#define CKH(expr, what)                                    \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

#define CK(expr, what)                               \
    do {                                             \
        cudaError_t _e = (expr);                     \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
        ++g_launches;                                \
    } while (0)

// ---- field checks (gf2e.py:44-71, 125-137) ---------------------------------------------
int poly_degree(uint64_t p) { return p ? 63 - __builtin_clzll(p) : -1; }
uint64_t poly_mod(uint64_t a, uint64_t m) {
    int dm = poly_degree(m);
    while (poly_degree(a) >= dm) a ^= m << (poly_degree(a) - dm);
    return a;
}
bool is_irreducible(uint64_t f) {
    int d = poly_degree(f);
    if (d < 1) return false;
    if (d == 1) return true;
    if ((f & 1) == 0) return false;
    for (uint64_t g = 2; g < (1ULL << (d / 2 + 1)); ++g)
        if (poly_degree(g) >= 1 && poly_mod(f, g) == 0) return false;
    return true;
}

int check_field(int e, uint32_t f) {
    if (e < 2 || e > 10) return fail(GF2E_EINVAL, "extension degree must be in 2..10, got %d", e);
    if (poly_degree(f) != e)
        return fail(GF2E_EINVAL, "modulus 0x%x has degree %d, expected %d", f, poly_degree(f), e);
    if (!is_irreducible(f)) return fail(GF2E_EINVAL, "modulus 0x%x is not irreducible over GF(2)", f);
    return GF2E_OK;
}

// ---- Karatsuba schedule: symbolic replay of poly_mul.py:128-242 -------------------------
struct Schedule {
    std::vector<uint64_t> subsets;  // per product: bitmask of input planes
    std::vector<uint64_t> outmap;   // per output plane: bitmask of products
    int64_t counters[3];            // gf2_matmul_count, additions, peak_live_products
    // running-sum form grouping (Sched.seq / gsize / gmask, run_groups below)
    std::vector<int> grp_seq, grp_size;
    std::vector<uint32_t> grp_mask;
    int grp_load = 0;
};

// ---- drain grouping of the running-sum form ----------------------------------------------
// The running-sum kernel pays one accumulator drain (TMEM read + parity + fold) per group of
// products, and every accumulated entry pays its operand staging and MMAs.  Output
// plane b is the XOR of the parities of the products t with bit b of their column M_t (the
// e-bit vector of output planes product t feeds).  Choose q drain vectors c_1..c_q in GF(2)^e
// and write every column as a XOR of a few of them, M_t = sum_{j in R_t} c_j: product t is
// accumulated into each group j of R_t, group j's drain parity is folded into the planes c_j,
// and plane b receives sum_j c_j[b] sum_{t: j in R_t} P_t = sum_t M_t[b] P_t.  One group per
// product (c = the columns) is the identity; fewer groups trade drains for repeated MMAs.
// dist: fewest vectors of S summing to each element of GF(2)^e (BFS), par: last vector used.
static void gf2_span_bfs(const std::vector<uint32_t> &S, int e, std::vector<int> &dist, std::vector<int> *par) {
    const int n = 1 << e;
    dist.assign(n, 1 << 20);
    if (par) par->assign(n, -1);
    std::vector<uint32_t> frontier{0}, next;
    dist[0] = 0;
    while (!frontier.empty()) {
        next.clear();
        for (uint32_t v : frontier)
            for (size_t j = 0; j < S.size(); ++j) {
                const uint32_t u = v ^ S[j];
                if (dist[u] > dist[v] + 1) {
                    dist[u] = dist[v] + 1;
                    if (par) (*par)[u] = (int)j;
                    next.push_back(u);
                }
            }
        frontier.swap(next);
    }
}
static int64_t grouping_cost(const std::vector<uint32_t> &S, const std::vector<uint32_t> &cols, int e) {
    std::vector<int> d;
    gf2_span_bfs(S, e, d, nullptr);
    int64_t c = 0;
    for (uint32_t x : cols) c += d[x];
    return c;
}

// q: drains per tile (GF2E_RUN_DRAINS; default and >= K: identity)
static void run_groups(Schedule &s, int e) {
    const int K = (int)s.subsets.size();
    std::vector<uint32_t> cols(K);
    for (int t = 0; t < K; ++t) {
        uint32_t m = 0;
        for (int j = 0; j < e; ++j)
            if ((s.outmap[j] >> t) & 1ULL) m |= 1u << j;
        cols[t] = m;
    }
    std::vector<uint32_t> S = cols;
    std::sort(S.begin(), S.end());
    S.erase(std::unique(S.begin(), S.end()), S.end());
    S.erase(std::remove(S.begin(), S.end(), 0u), S.end());
    const char *env = getenv("GF2E_RUN_DRAINS");
    const int want = env ? atoi(env) : 0;
    // greedy removal down to e vectors, keeping the frontier (entries per number of drains)
    std::vector<std::vector<uint32_t>> front(S.size() + 1);
    std::vector<int64_t> fcost(S.size() + 1, -1);
    front[S.size()] = S;
    fcost[S.size()] = grouping_cost(S, cols, e);
    for (std::vector<uint32_t> cur = S; (int)cur.size() > e;) {
        int64_t best = -1;
        size_t bi = 0;
        for (size_t i = 0; i < cur.size(); ++i) {
            std::vector<uint32_t> T = cur;
            T.erase(T.begin() + i);
            const int64_t c = grouping_cost(T, cols, e);
            if (c < (int64_t)K * (1 << 20) && (best < 0 || c < best)) {
                best = c;
                bi = i;
            }
        }
        if (best < 0) break;
        cur.erase(cur.begin() + bi);
        front[cur.size()] = cur;
        fcost[cur.size()] = best;
    }
    // measured (profiles/r02/run_grouping.txt, e = 8, config 4): 27 drains 17.0 ms, 24: 17.4,
    // 20: 18.5, 16: 19.3 -- an extra accumulated entry costs more than the drain it saves
    // while the A operand is expanded into TMEM by the expander warps, so the default is the
    // identity (one drain per product); GF2E_RUN_DRAINS=q selects a grouping
    int q = (int)S.size();
    if (want > 0) {
        q = want < (int)S.size() ? want : (int)S.size();
        while (q < (int)S.size() && fcost[q] < 0) ++q;
    }
    std::vector<uint32_t> G = front[q];
    int64_t gc = fcost[q];
    if (e <= 8 && q < (int)S.size()) {  // local search: replace one vector by any other
        for (bool improved = true; improved;) {
            improved = false;
            for (size_t i = 0; i < G.size(); ++i)
                for (uint32_t v = 1; v < (1u << e); ++v) {
                    if (std::find(G.begin(), G.end(), v) != G.end()) continue;
                    std::vector<uint32_t> U = G;
                    U[i] = v;
                    const int64_t c = grouping_cost(U, cols, e);
                    if (c < gc) {
                        gc = c;
                        G = U;
                        improved = true;
                    }
                }
        }
    }
    // representations and groups (empty groups dropped)
    std::vector<int> dist, par;
    gf2_span_bfs(G, e, dist, &par);
    std::vector<std::vector<int>> members(G.size());
    for (int t = 0; t < K; ++t)
        for (uint32_t x = cols[t]; x;) {
            const int j = par[x];
            members[j].push_back(t);
            x ^= G[j];
        }
    s.grp_seq.clear();
    s.grp_size.clear();
    s.grp_mask.clear();
    int64_t load[2] = {0, 0};
    for (size_t j = 0; j < G.size(); ++j) {
        if (members[j].empty()) continue;
        load[s.grp_size.size() & 1] += (int64_t)members[j].size();
        s.grp_size.push_back((int)members[j].size());
        s.grp_mask.push_back(G[j]);
        for (int t : members[j]) s.grp_seq.push_back(t);
    }
    s.grp_load = (int)std::max(load[0], load[1]);
    if ((int)s.grp_seq.size() > kMaxSeq || (int)s.grp_size.size() > kMaxSeq) {  // cannot happen for e <= 10
        s.grp_seq.clear();
        s.grp_size.clear();
        s.grp_mask.clear();
    }
}

struct Replay {
    std::vector<uint64_t> subsets;
    int64_t additions = 0, live = 0, peak = 0;
    void grab(int64_t k) {
        live += k;
        if (live > peak) peak = live;
    }
    uint64_t base(uint64_t a) {  // poly_mul.py:146-150
        subsets.push_back(a);
        grab(1);
        return 1ULL << (subsets.size() - 1);
    }
    std::vector<uint64_t> add_lists(std::vector<uint64_t> xs, std::vector<uint64_t> ys) {  // 153-163
        if (xs.size() < ys.size()) std::swap(xs, ys);
        for (size_t i = 0; i < ys.size(); ++i) xs[i] ^= ys[i];
        additions += (int64_t)ys.size();
        return xs;
    }
    std::vector<uint64_t> kara(const std::vector<uint64_t> &a) {  // 166-220 (a == b symbolically)
        const size_t ka = a.size();
        if (ka == 1) return {base(a[0])};
        if (ka == 3) {
            uint64_t d0 = base(a[0]), d1 = base(a[1]), d2 = base(a[2]);
            uint64_t d01 = base(a[0] ^ a[1]), d02 = base(a[0] ^ a[2]), d12 = base(a[1] ^ a[2]);
            additions += 6 + 7;
            live -= 6;
            grab(5);
            return {d0, d01 ^ d0 ^ d1, d02 ^ d0 ^ d1 ^ d2, d12 ^ d1 ^ d2, d2};
        }
        const size_t h = (ka + 1) / 2;
        std::vector<uint64_t> alo(a.begin(), a.begin() + h), ahi(a.begin() + h, a.end());
        std::vector<uint64_t> lo = kara(alo), hi = kara(ahi);
        std::vector<uint64_t> mid = kara(add_lists(alo, ahi));
        add_lists(alo, ahi);  // the B-side _add_lists of poly_mul.py:201 (counted, same subsets)
        for (size_t i = 0; i < lo.size(); ++i) mid[i] ^= lo[i];
        for (size_t i = 0; i < hi.size(); ++i) mid[i] ^= hi[i];
        additions += (int64_t)(lo.size() + hi.size());
        std::vector<uint64_t> out(2 * ka - 1, 0);
        for (size_t i = 0; i < lo.size(); ++i) out[i] ^= lo[i];
        for (size_t i = 0; i < mid.size(); ++i) out[h + i] ^= mid[i];
        for (size_t i = 0; i < hi.size(); ++i) out[2 * h + i] ^= hi[i];
        additions += (int64_t)(lo.size() + mid.size() + hi.size());
        live -= (int64_t)(lo.size() + hi.size() + mid.size());
        grab((int64_t)out.size());
        return out;
    }
};

std::mutex g_sched_mu;
std::map<std::pair<int, uint32_t>, Schedule> g_sched_cache;

const Schedule &get_schedule(int e, uint32_t f) {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    auto key = std::make_pair(e, f);
    auto it = g_sched_cache.find(key);
    if (it != g_sched_cache.end()) return it->second;
    Replay r;
    std::vector<uint64_t> planes(e);
    for (int i = 0; i < e; ++i) planes[i] = 1ULL << i;
    std::vector<uint64_t> gamma = r.kara(planes);
    Schedule s;
    s.subsets = r.subsets;
    s.counters[0] = (int64_t)r.subsets.size();
    s.counters[2] = r.peak;
    // reduce_mod_f (poly_mul.py:223-242) on symbols
    std::vector<uint64_t> work(2 * e - 1);
    for (int d = 0; d < 2 * e - 1; ++d) work[d] = 1ULL << d;
    int64_t adds = r.additions;
    for (int d = 2 * e - 2; d >= e; --d)
        for (int k = 0; k < e; ++k)
            if ((f >> k) & 1u) {
                work[d - e + k] ^= work[d];
                ++adds;
            }
    s.counters[1] = adds;
    s.outmap.assign(e, 0);
    for (int j = 0; j < e; ++j)
        for (int d = 0; d < 2 * e - 1; ++d)
            if ((work[j] >> d) & 1ULL) s.outmap[j] ^= gamma[d];
    run_groups(s, e);
    return g_sched_cache.emplace(key, s).first->second;
}

// one group per product: the running-sum form's plain order (exact whenever run_ok holds)
void run_identity(Sched &k) {
    k.nseq = k.ngrp = k.nprod;
    for (int t = 0; t < k.nprod; ++t) {
        k.seq[t] = (uint8_t)t;
        k.gsize[t] = 1;
        k.gmask[t] = k.outmask[t];
    }
    k.run_load = (k.nprod + 1) / 2;
}

Sched to_kernel_sched(int e, const Schedule &S) {
    Sched k;
    memset(&k, 0, sizeof(k));
    k.e = e;
    k.nout = e;
    k.nprod = (int)S.subsets.size();
    for (int t = 0; t < k.nprod; ++t) {
        k.subset[t] = (uint16_t)S.subsets[t];
        uint16_t m = 0;
        for (int j = 0; j < e; ++j)
            if ((S.outmap[j] >> t) & 1ULL) m |= (uint16_t)(1u << j);
        k.outmask[t] = m;
    }
    run_identity(k);
    if (!S.grp_seq.empty()) {
        k.nseq = (int)S.grp_seq.size();
        k.ngrp = (int)S.grp_size.size();
        for (int i = 0; i < k.nseq; ++i) k.seq[i] = (uint8_t)S.grp_seq[i];
        for (int g = 0; g < k.ngrp; ++g) {
            k.gsize[g] = (uint8_t)S.grp_size[g];
            k.gmask[g] = (uint16_t)S.grp_mask[g];
        }
        k.run_load = S.grp_load;
    }
    return k;
}

Sched plane_sched() {
    Sched k;
    memset(&k, 0, sizeof(k));
    k.e = 1;
    k.nout = 1;
    k.nprod = 1;
    k.subset[0] = 1;
    k.outmask[0] = 1;
    run_identity(k);
    return k;
}

// ---- library memory pool ----------------------------------------------------------------
// Temporaries of the host-buffer pipeline and of PLE/echelonize come from a pool the library
// owns (one per device), not the device's default pool, so the process-wide default pool and
// the PyTorch caching allocator are untouched.  The pool keeps up to kPoolKeep bytes mapped
// across calls (re-mapping gigabytes per call costs milliseconds) and returns the rest to the
// driver at each synchronisation; gf2e_trim_pool() releases the cached memory on demand.
constexpr uint64_t kPoolKeep = 4ull << 30;
std::mutex g_pool_mu;
cudaMemPool_t g_pools[kMaxDevices] = {};

cudaMemPool_t lib_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
        uint64_t keep = kPoolKeep;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        g_pools[dev] = pool;
    }
    return g_pools[dev];
}

cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool = lib_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

// stream-ordered temporary from the library pool, freed at scope exit
struct DevTmpAny {
    void *p = nullptr;
    cudaStream_t st;
    DevTmpAny(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes && pool_alloc(&p, bytes, st) != cudaSuccess) p = nullptr;
    }
    ~DevTmpAny() {
        if (p) cudaFreeAsync(p, st);
    }
    DevTmpAny(const DevTmpAny &) = delete;
    DevTmpAny &operator=(const DevTmpAny &) = delete;
};

// ---- device check ---------------------------------------------------------------------
int check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(GF2E_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
    int major = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return fail(GF2E_ENODEV, "cannot query device: %s", cudaGetErrorString(e));
    if (major != 10) return fail(GF2E_ENODEV, "libgf2e_b200 needs an sm_100 (B200) device, found sm_%d", major * 10);
    return GF2E_OK;
}

int check_mat(const void *p, int64_t rows, int64_t cols_words, int64_t ld, const char *name) {
    if (rows < 0 || cols_words < 0) return fail(GF2E_EINVAL, "matrix dimensions must be non-negative");
    if (rows > 0 && cols_words > 0) {
        if (!p) return fail(GF2E_EINVAL, "%s is NULL", name);
        if (ld < cols_words) return fail(GF2E_EINVAL, "%s: row stride %lld < %lld words", name, (long long)ld,
                                         (long long)cols_words);
    }
    return GF2E_OK;
}

// ---- workspace layout -----------------------------------------------------------------
struct Layout {
    int64_t m_pad, n_pad, k_pad, kwords;
    int64_t a_pstride, b_pstride;  // words
    int64_t a_bytes, b_bytes, total;
};

int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

// Tensor-core form: fp4 (kind::mxf4, 2x the int8 rate) unless forced to int8.  Below k = 2048
// the single-accumulator fp4 forms' per-product hand-off would dominate, so short inner
// dimensions take the running-sum form (product_run.cu) while its sums stay exact, else int8;
// backend "tc_fp4" forces the paired form there.
constexpr int64_t kFp4MinK = 2048;
// short k: the running-sum fp4 form (double-buffered accumulators, no per-product
// re-initialisation; config 4 e=8: 17.7 ms against 21.5 ms for int8, profiles/r02)
constexpr int64_t kFp4LongK = 8192;  // 8 expander / 4 epilogue warps pay off for long accumulations
// fp4 exactness self-check state per device: 0 not run, 1 passed, -1 failed (fp4 disabled)
int g_fp4_state[kMaxDevices] = {};
std::mutex g_fp4_mu;
int fp4_state() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
    std::lock_guard<std::mutex> lk(g_fp4_mu);
    return g_fp4_state[dev];
}

// the running-sum form is exact while every accumulator's sum of counts stays below 2^16:
// ceil(K/2) products of at most k_pad each per buffer and tile
bool run_ok(int nprod, int64_t k) { return (int64_t)((nprod + 1) / 2) * round_up(k, kTcBKFp4) < kRunMaxSum; }

// the running-sum form expands B^T in-kernel for products of at most this many rows: there
// the 4x pre-expanded B^T would be written for one or a few row tiles (GF2E_RUNX_MAXM)
int64_t runx_max_m() {
    static const int64_t v = getenv("GF2E_RUNX_MAXM") ? atoll(getenv("GF2E_RUNX_MAXM")) : 2048;
    return v;
}
bool is_run(int form) { return form == kFormFp4Run || form == kFormFp4RunX; }

int tc_form(uint32_t flags, int64_t k, int nprod = kMaxProducts, int64_t m = INT64_MAX) {
    if (flags & GF2E_TC_INT8) return kFormI8;
    if (fp4_state() < 0) return kFormI8;  // the fp4 self-check failed on this device
    const int run = m <= runx_max_m() ? kFormFp4RunX : kFormFp4Run;
    if ((flags & GF2E_TC_RUN) && run_ok(nprod, k)) return run;
    if (k >= kFp4LongK) return kFormFp4Long;
    if (k >= kFp4MinK) return kFormFp4;
    if (flags & GF2E_TC_FP4) return kFormFp4Pair;
    return run_ok(nprod, k) ? run : kFormI8;
}
const char *form_name(int form) {
    return form == kFormFp4Pair                            ? "k_product_tc2<fp4x2>"
           : (form == kFormFp4 || form == kFormFp4Long) ? "k_product_tc2<fp4>"
           : is_run(form)                                 ? "k_product_run<fp4>"
                                                          : "k_product_tc2<i8>";
}
// tile columns of a form (CTA-pair tile width; B^T is stage-tiled in half-width row blocks)
int64_t form_bn(int form) { return is_run(form) ? kRunBN : kTcBN; }
int form_br(int form) { return (int)(form_bn(form) / 2); }
// B^T words per row per bit word: 4 when the form's B operand is stored pre-expanded
int64_t form_bx(int form) { return (form == kFormFp4Run && kRunBPre) ? 4 : 1; }
bool form_bexp(int form) { return form_bx(form) > 1; }

constexpr int kFormAny = -2;  // workspace bound over every tensor-core form

Layout layout_for(int nprod, int64_t m, int64_t k, int64_t n, uint32_t flags, int form = -1) {
    Layout L;
    if (flags & GF2E_BACKEND_M4RM) {
        L.m_pad = round_up(m, kM4BM);
        L.n_pad = round_up(n, kM4BN);
        L.k_pad = round_up(k, kM4KPAD);
        L.kwords = L.k_pad / 64;
        L.a_pstride = L.m_pad * L.kwords;
        L.b_pstride = L.k_pad * (L.n_pad / 64);
    } else {
        if (form == -1) form = tc_form(flags, k, nprod, m);
        L.m_pad = round_up(m, 2 * kTcBM);  // CTA-pair tiles are 256 rows
        int64_t bx = 1;
        if (form == kFormAny) {  // every form a call with these sizes may take
            const bool run = run_ok(nprod, k);
            const int64_t a = round_up(n, kTcBN), b = run ? round_up(n, kRunBN) : 0;
            L.n_pad = a > b ? a : b;
            L.k_pad = round_up(k, kTcBKFp4);
            bx = run ? form_bx(kFormFp4Run) : 1;
        } else {
            L.n_pad = round_up(n, form_bn(form));
            L.k_pad = round_up(k, form == kFormI8 ? kTcBK : kTcBKFp4);
            bx = form_bx(form);
        }
        L.kwords = L.k_pad / 64;
        L.a_pstride = L.m_pad * L.kwords;
        L.b_pstride = L.n_pad * L.kwords * bx;
    }
    L.a_bytes = align256((int64_t)nprod * L.a_pstride * 8);
    L.b_bytes = align256((int64_t)nprod * L.b_pstride * 8);
    L.total = L.a_bytes + L.b_bytes;
    return L;
}

// GF(2) plane products one launch_form call runs (the grouped running-sum sequence repeats some)
int form_products(const Sched &ks, const TcArgs &a, int form) {
    if (!is_run(form) || (int64_t)ks.run_load * a.kwords * 64 >= kRunMaxSum) return ks.nprod;
    return ks.nseq;
}

cudaError_t launch_form(const Sched &ks, const TcArgs &a, int form, cudaStream_t st) {
    if (is_run(form) && (int64_t)ks.run_load * a.kwords * 64 >= kRunMaxSum) {
        Sched plain = ks;  // the grouping's accumulators would overflow at this k: plain order
        run_identity(plain);
        return launch_product_run(plain, a, st, form == kFormFp4Run);
    }
    return is_run(form) ? launch_product_run(ks, a, st, form == kFormFp4Run) : launch_product_tc2(ks, a, form, st);
}

// Per host thread and device: a side stream and a fork / join event pair for running the
// two operand-combination kernels of a product concurrently (created on first use, kept)
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream &side_stream() {
    thread_local SideStream per_dev[kMaxDevices];
    static SideStream none;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return none;
    SideStream &ss = per_dev[dev];
    if (!ss.s) {
        if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
            ss = SideStream{};
            return none;
        }
    }
    return ss;
}

// The shared launch sequence: K3 combos -> fused K4/K5 product.
int ensure_fp4_checked();

int run_product(const Sched &ks, const uint64_t *A, int64_t lda, int64_t pa, const uint64_t *B, int64_t ldb,
                int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m, int64_t k, int64_t n, uint32_t flags,
                void *ws, int64_t ws_bytes, cudaStream_t st, int form_override = -1) {
    const bool acc = (flags & GF2E_ACCUMULATE) != 0;
    const int64_t nw = words_for(n);
    if (m == 0 || n == 0) return GF2E_OK;
    if (k == 0) {  // empty inner dimension: product is zero (mat_gf2.py:352-354)
        if (!acc)
            for (int j = 0; j < ks.nout; ++j)
                CK(cudaMemset2DAsync(C + j * pc, ldc * 8, 0, nw * 8, m, st), "cudaMemset2DAsync");
        return GF2E_OK;
    }
    const bool tc = !(flags & GF2E_BACKEND_M4RM);
    if (tc && form_override < 0 && !(flags & GF2E_TC_INT8))
        if (int rc = ensure_fp4_checked()) return rc;
    const int form = form_override >= 0 ? form_override : tc_form(flags, k, ks.nprod, m);
    const bool fp4 = tc && form != kFormI8;
    static const bool trace = getenv("GF2E_PROD_TRACE") != nullptr;
    if (trace) fprintf(stderr, "product m=%lld k=%lld n=%lld form=%d\n", (long long)m, (long long)k, (long long)n, form);
    Layout L = layout_for(ks.nprod, m, k, n, flags, form);
    if (ws_bytes < L.total)
        return fail(GF2E_ENOMEM, "workspace too small: %lld < %lld bytes", (long long)ws_bytes, (long long)L.total);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255))
        return fail(GF2E_EINVAL, "workspace must be a 256-byte aligned device pointer");
    uint64_t *Ac = static_cast<uint64_t *>(ws);
    uint64_t *Bx = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + L.a_bytes);
    // tensor-core forms: the B^T combinations run beside the A combinations on a side stream
    // (fork / join by events): two small independent kernels, latency-bound at small sizes
    // (below GF2E_FORK_MIN_BITS operand bits the fork's four event calls cost the host more
    // than the overlap saves the device; default 0: always fork)
    static const int64_t fork_min = getenv("GF2E_FORK_MIN_BITS") ? atoll(getenv("GF2E_FORK_MIN_BITS")) : 0;
    SideStream no_side;
    const bool want_fork = tc && m * k + k * n >= fork_min;
    SideStream &side = want_fork ? side_stream() : no_side;
    const bool forked = want_fork && side.s;
    if (forked) {
        CKH(cudaEventRecord(side.fork, st), "cudaEventRecord");
        CKH(cudaStreamWaitEvent(side.s, side.fork, 0), "cudaStreamWaitEvent");
    }
    CK(launch_combos_rows(ks, A, lda, pa, m, k, Ac, L.kwords, L.a_pstride, L.m_pad, L.kwords, tc ? (fp4 ? 4 : 2) : 0,
                          st),
       "combos(A)");
    if (!tc) {
        const int64_t nwp = L.n_pad / 64;
        CK(launch_combos_rows(ks, B, ldb, pb, k, n, Bx, nwp, L.b_pstride, L.k_pad, nwp, 0, st), "combos(B)");
        if (!acc)
            for (int j = 0; j < ks.nout; ++j)
                CK(cudaMemset2DAsync(C + j * pc, ldc * 8, 0, nw * 8, m, st), "cudaMemset2DAsync");
        M4rmArgs a{Ac, Bx, L.a_pstride, L.b_pstride, L.kwords, nwp, L.k_pad, m, n, L.m_pad, L.n_pad, C, ldc, pc};
        ProfScope prof(st);
        CK(launch_product_m4rm(ks, a, st), "product_m4rm");
        g_products += ks.nprod;
        g_kernel = "k_product_m4rm";
    } else {
        CK(launch_combos_bt(ks, B, ldb, pb, k, n, Bx, L.kwords, L.b_pstride, L.kwords, L.n_pad / 64, fp4,
                            forked ? side.s : st, form_br(form), 0, form_bexp(form)),
           "combos(B^T)");
        if (forked) {
            CKH(cudaEventRecord(side.join, side.s), "cudaEventRecord");
            CKH(cudaStreamWaitEvent(st, side.join, 0), "cudaStreamWaitEvent");
        }
        TcArgs a{Ac, Bx, L.a_pstride, L.b_pstride, L.kwords, m, n, L.m_pad, L.n_pad, C, ldc, pc, acc ? 1 : 0};
        ProfScope prof(st);
        CK(launch_form(ks, a, form, st), "product");
        g_products += form_products(ks, a, form);
        g_kernel = form_name(form);
    }
    return GF2E_OK;
}


// ---- fp4 exactness self-check ---------------------------------------------------------------
// The fp4 forms rely on kind::mxf4 accumulating exact small integers in fp32 (parity = bit 7
// of the pattern, product_tc2.cu header).  That is measured behaviour (tools/fp4_probe.py),
// not an architectural guarantee, so before the first fp4 product on a device the library
// multiplies GF(2) planes in every fp4 form and in the int8 form (integer arithmetic, exact
// by construction) and compares them bit for bit: random operands and all-ones operands
// (count = k, the largest accumulator values) at k = 33024, across the 32768-bit accumulation
// chunk boundary of the long form; k = 4096 (short form); k = 1024 (paired form).  On any
// mismatch fp4 is disabled on that device (every product takes the int8 form) and
// gf2e_fp4_selfcheck reports it.
bool g_fp4_inject = false;  // test hook: corrupt the fp4 results of the next check

int fp4_probe_run(bool inject, int *ok) {
    *ok = 0;
    const int64_t m = 256, n = 256;
    // plane products (one GF(2) product) for the single-accumulator forms; the running-sum form
    // with the GF(16) schedule (9 products, 4 input planes: several products per accumulator)
    const struct {
        int form;
        int64_t k;
        int e;
    } cases[] = {{kFormFp4Long, 33024, 1}, {kFormFp4, 4096, 1}, {kFormFp4Pair, 1024, 1}, {kFormFp4Run, 1792, 4},
                 {kFormFp4RunX, 1792, 4}};
    cudaStream_t st = nullptr;
    CKH(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } sg{st};
    const int64_t kmax = 33024, nw = n / 64, emax = 4;
    const int64_t ws_bytes = layout_for(9, m, kmax, n, 0, kFormAny).total;
    DevTmpAny A((size_t)emax * m * (kmax / 64) * 8, st), B((size_t)emax * kmax * nw * 8, st),
        C8((size_t)emax * m * nw * 8, st), C4((size_t)emax * m * nw * 8, st), ws((size_t)ws_bytes, st);
    if (!A.p || !B.p || !C8.p || !C4.p || !ws.p) return fail(GF2E_ENOMEM, "out of device memory (fp4 self-check)");
    uint64_t *a = static_cast<uint64_t *>(A.p), *b = static_cast<uint64_t *>(B.p);
    uint64_t *c8 = static_cast<uint64_t *>(C8.p), *c4 = static_cast<uint64_t *>(C4.p);
    std::vector<uint64_t> h8((size_t)emax * m * nw), h4((size_t)emax * m * nw);
    bool good = true;
    for (const auto &cs : cases) {
        const Sched ks = cs.e == 1 ? plane_sched() : to_kernel_sched(cs.e, get_schedule(cs.e, 0x13));
        const int64_t kw = cs.k / 64, pa = m * kw, pb = cs.k * nw, pc = m * nw;
        const size_t cw = (size_t)cs.e * m * nw;
        for (int ones = 0; ones < 2; ++ones) {
            if (ones) {
                CKH(cudaMemsetAsync(a, 0xFF, (size_t)cs.e * pa * 8, st), "cudaMemsetAsync");
                CKH(cudaMemsetAsync(b, 0xFF, (size_t)cs.e * pb * 8, st), "cudaMemsetAsync");
            } else {
                CKH(launch_random_words((int64_t)cs.e * m, cs.k, 0x5eed0 + (uint64_t)cs.k, a, kw, st), "random_words");
                CKH(launch_random_words((int64_t)cs.e * cs.k, n, 0x5eed1 + (uint64_t)cs.k, b, nw, st), "random_words");
            }
            if (int rc = run_product(ks, a, kw, pa, b, nw, pb, c8, nw, pc, m, cs.k, n, GF2E_TC_INT8, ws.p, ws_bytes,
                                     st, kFormI8))
                return rc;
            if (int rc = run_product(ks, a, kw, pa, b, nw, pb, c4, nw, pc, m, cs.k, n, 0, ws.p, ws_bytes, st, cs.form))
                return rc;
            CKH(cudaMemcpyAsync(h8.data(), c8, cw * 8, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
            CKH(cudaMemcpyAsync(h4.data(), c4, cw * 8, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
            CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            if (inject) h4[(size_t)cs.k % cw] ^= 1;
            if (std::memcmp(h8.data(), h4.data(), cw * 8) != 0) good = false;
        }
    }
    *ok = good ? 1 : -1;
    return GF2E_OK;
}

// run the self-check once per device (first fp4-capable product); 0 or an error status
int ensure_fp4_checked() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return GF2E_OK;
    {
        std::lock_guard<std::mutex> lk(g_fp4_mu);
        if (g_fp4_state[dev] != 0) return GF2E_OK;
    }
    const int launches = g_launches;
    const int64_t products = g_products;
    int ok = 0;
    int rc = fp4_probe_run(g_fp4_inject, &ok);
    g_launches = launches;  // the check's launches are not the caller's
    g_products = products;
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_fp4_mu);
    g_fp4_state[dev] = ok;
    g_fp4_inject = false;
    return GF2E_OK;
}

// ---- host-buffer packed multiply (e2e entry) ----------------------------------------------
int pair_count() {
    int dev = 0, nsms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
    return nsms / 2;
}

// Row chunks of the host pipeline (k >= 4096).  The first chunk meets B part by part: it
// gets as many 256-row tiles as fill the CTA pairs next to one part's column tiles (9 x 8 =
// 72 of 74 at n = 16384), so the products that run while B is still arriving use the whole
// GPU.  The rest go in `chunk`-row chunks, the remainder merged into the first of them (at
// 16384 rows: 2304, 3840, 5 x 2048 — 97-99.8% wave fill each, against 86% for 1792 rows).
int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

std::vector<int64_t> host_row_plan(int64_t m, int64_t n, int64_t k, int64_t chunk, int nbp, bool fixed, int64_t tw) {
    std::vector<int64_t> rb{0};
    int64_t first = chunk;
    // only where the products, not the copies, bound the pipeline (long k; at k = 256 the
    // C0/C copies dominate and uniform chunks pipeline them best)
    fixed = fixed || k < 4096;
    if (!fixed && nbp > 1) {
        static const int reserve = env_int("GF2E_E2E_RESERVE", 0);
        const int64_t part_tiles = ((n + tw - 1) / tw + nbp - 1) / nbp;
        const int64_t rt0 = (pair_count() - reserve) / part_tiles;
        if (rt0 >= 1) first = rt0 * 256;
    }
    if (first >= m) return {0, m};
    rb.push_back(first);
    const int64_t rest = m - first, nfull = rest / chunk, rem = rest - nfull * chunk;
    if (nfull == 0) {
        rb.push_back(m);
        return rb;
    }
    int64_t r = first + (fixed ? chunk : chunk + rem);
    rb.push_back(r);
    while (r < m) {
        r = r + chunk < m ? r + chunk : m;
        rb.push_back(r);
    }
    return rb;
}


// Column split of the host pipeline's last row chunk: the first part a whole number of waves
// of CTA pairs (row tiles x column tiles a multiple of the pair count), about half of n.
int64_t last_split_cols(int64_t rows, int64_t n, int64_t tw) {
    if (n < 8192) return n;
    const int64_t pairs = pair_count(), rt = (rows + 255) / 256, nt = (n + tw - 1) / tw;
    int64_t g = pairs, b = rt;
    while (b) {
        const int64_t t = g % b;
        g = b;
        b = t;
    }
    const int64_t q = pairs / g;  // column tiles per whole wave step
    const int64_t ct = (nt / 2 + q - 1) / q * q;
    return ct > 0 && ct < nt ? ct * tw : n;
}

// GF2E_E2E_TRACE=1: per-stage completion times of the host-buffer pipeline on stderr
struct Trace {
    bool on = getenv("GF2E_E2E_TRACE") != nullptr;
    cudaEvent_t t0 = nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> ev;
    void start(cudaStream_t s) {
        if (!on) return;
        cudaEventCreate(&t0);
        cudaEventRecord(t0, s);
    }
    void mark(cudaStream_t s, const char *what, int64_t i, int64_t j = -1) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        char buf[64];
        snprintf(buf, sizeof buf, j < 0 ? "%s %lld" : "%s %lld.%lld", what, (long long)i, (long long)j);
        ev.emplace_back(buf, e);
    }
    ~Trace() {
        if (!on) return;
        for (auto &x : ev) {
            float ms = 0;
            cudaEventSynchronize(x.second);
            cudaEventElapsedTime(&ms, t0, x.second);
            fprintf(stderr, "trace %-14s %8.3f\n", x.first.c_str(), ms);
            cudaEventDestroy(x.second);
        }
        cudaEventDestroy(t0);
    }
};

struct HostPlan {
    cudaStream_t sc = nullptr, sh = nullptr, sd = nullptr, sp = nullptr;
    std::vector<void *> allocs;
    ~HostPlan() {
        if (sh) cudaStreamSynchronize(sh);  // error paths: no copy or kernel may outlive its buffers
        if (sd) cudaStreamSynchronize(sd);
        if (sp) cudaStreamSynchronize(sp);
        if (sp) cudaStreamDestroy(sp);
        for (void *p : allocs) cudaFreeAsync(p, sc);
        if (sc) cudaStreamSynchronize(sc);
        if (sc) cudaStreamDestroy(sc);
        if (sh) cudaStreamDestroy(sh);
        if (sd) cudaStreamDestroy(sd);
    }
    template <typename T>
    cudaError_t alloc(T **p, int64_t bytes) {
        void *q = nullptr;
        cudaError_t e = pool_alloc(&q, (size_t)(bytes > 256 ? bytes : 256), sc);
        if (e == cudaSuccess) allocs.push_back(q);
        *p = static_cast<T *>(q);
        return e;
    }
};



// ---- blocked TRSM over plane views (consumer of run_product) ------------------------------
uint32_t gf_mul_host(uint32_t a, uint32_t b, int e, uint32_t f) {
    uint32_t acc = 0;
    for (int i = 0; i < e; ++i)
        if ((b >> i) & 1u) acc ^= a << i;
    for (int d = 2 * e - 2; d >= e; --d)
        if ((acc >> d) & 1u) acc ^= f << (d - e);
    return acc;
}

// smallest element of multiplicative order 2^e - 1 (f irreducible => one exists)
uint32_t primitive_element(int e, uint32_t f) {
    const uint32_t q1 = (1u << e) - 1;
    for (uint32_t g = 2; g <= q1; ++g) {
        uint32_t v = g, ord = 1;
        while (v != 1 && ord <= q1) {
            v = gf_mul_host(v, g, e, f);
            ++ord;
        }
        if (ord == q1) return g;
    }
    return 2;
}

struct TrsmLayout {
    int64_t nblk, inv_bytes, tmp_bytes, mul_bytes, total;
};

// diagonal block size: 256 when the solve is big enough that leaf products dominate
// 256-row diagonal blocks for big solves; e >= 9 keeps 128 (the 256-row inverse kernel runs
// 1024 threads, whose 64-register budget cannot hold e = 9, 10 rows without spilling)
int trsm_block(int e, int64_t m, int64_t n) { return (m >= 1024 && n >= 4096 && e <= 8) ? 256 : 128; }

TrsmLayout trsm_layout(int nprod, int e, int64_t m, int64_t n) {
    TrsmLayout T;
    const int64_t tb = trsm_block(e, m, n);
    T.nblk = (m + tb - 1) / tb;
    T.inv_bytes = align256(T.nblk * e * tb * (tb / 64) * 8);
    T.tmp_bytes = align256((int64_t)e * tb * words_for(n) * 8);
    // bounds every update and block product (k <= m): the largest k of the 256-column forms and
    // the largest k the running-sum form (4x B^T words) may take
    const int64_t krun = ((kRunMaxSum - 1) / ((nprod + 1) / 2)) / kTcBKFp4 * kTcBKFp4;
    const int64_t a = layout_for(nprod, m, m, n, 0, kFormAny).total;
    const int64_t b = layout_for(nprod, m, m < krun ? m : krun, n, 0, kFormAny).total;
    T.mul_bytes = a > b ? a : b;
    T.total = T.inv_bytes + T.tmp_bytes + 256 + T.mul_bytes;
    return T;
}

// Small updates of the consumers (PLE Schur complements, TRSM updates and leaves) run on CUDA
// cores through the sliced Newton-John kernel when the inner dimension is small: one launch
// instead of two operand-combination launches and a tensor-core product, whose fixed cost
// dominates there (the reference likewise multiplies small blocks with Newton-John tables
// below its crossover).  GF2E_NJS_MAXK overrides the crossover (measured, profiles/r02).
int64_t nj_sliced_max_k() {
    static const int64_t v = getenv("GF2E_NJS_MAXK") ? atoll(getenv("GF2E_NJS_MAXK")) : 128;
    return v;
}

int run_update(const Sched &ks, int e, const FieldTab *tab, const uint64_t *A, int64_t lda, int64_t pa,
               const uint64_t *B, int64_t ldb, int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m,
               int64_t k, int64_t n, uint32_t flags, void *ws, int64_t ws_bytes, cudaStream_t st,
               bool c_aliases_b = false) {
    // (grid limits of the Newton-John launch: 65535 row blocks of at least 64 rows)
    // (at e >= 9 the split tables of 64 entries make a wide 128-deep product cheaper on the
    // tensor cores: TRSM 8192 \ 8192 x 16384 at e = 10 18.7 against 22.5 ms, measured)
    const bool small_k = k <= 64 || (k <= nj_sliced_max_k() && (e <= 8 || n <= 2048));
    if (tab && m > 0 && n > 0 && k > 0 && small_k && m <= 65535LL * 64 &&
        (!c_aliases_b || m <= nj_sliced_alias_rows(e))) {
        CK(launch_nj_sliced(e, tab, A, lda, pa, B, ldb, pb, C, ldc, pc, m, k, n, (flags & GF2E_ACCUMULATE) != 0,
                            c_aliases_b, st),
           "nj_sliced");
        return GF2E_OK;
    }
    return run_product(ks, A, lda, pa, B, ldb, pb, C, ldc, pc, m, k, n, flags, ws, ws_bytes, st);
}

struct TrsmCtx {
    Sched ks;
    bool upper;
    const uint64_t *T;
    int64_t ldt, pt;
    uint64_t *B;
    int64_t ldb, pb, n;
    uint64_t *inv, *tmp;
    void *mulws;
    int64_t mulws_bytes;
    int e;
    cudaStream_t st;
    int64_t tb;  // diagonal block rows
    const FieldTab *tab;
};

int trsm_rec(TrsmCtx &c, int64_t i0, int64_t i1) {
    const int64_t rows = i1 - i0;
    const int64_t tb = c.tb;
    if (rows <= tb) {  // X = inv(T_blk) . B_blk  (tensor-core product), written over B_blk:
        // the product reads only its operand combinations, which are formed from B_blk before
        // the product kernel starts (stream order), so C may alias B here
        const uint64_t *Ib = c.inv + (i0 / tb) * c.e * tb * (tb / 64);
        uint64_t *Bb = c.B + i0 * c.ldb;
        const int64_t nwn = words_for(c.n);
        if (rows <= nj_sliced_max_k() && rows > 64 && (c.e <= 8 || c.n <= 2048) && c.pb % c.ldb == 0) {
            // the Newton-John form with the rows split over CTAs: B_blk copied to the scratch
            // first (one 3-D copy of all planes), so C no longer aliases the operand
            cudaMemcpy3DParms cp = {};
            cp.srcPtr = make_cudaPitchedPtr(Bb, (size_t)c.ldb * 8, (size_t)nwn * 8, (size_t)(c.pb / c.ldb));
            cp.dstPtr = make_cudaPitchedPtr(c.tmp, (size_t)nwn * 8, (size_t)nwn * 8, (size_t)tb);
            cp.extent = make_cudaExtent((size_t)nwn * 8, (size_t)rows, (size_t)c.e);
            cp.kind = cudaMemcpyDeviceToDevice;
            CKH(cudaMemcpy3DAsync(&cp, c.st), "cudaMemcpy3DAsync");
            return run_update(c.ks, c.e, c.tab, Ib, tb / 64, tb * (tb / 64), c.tmp, nwn, tb * nwn, Bb, c.ldb, c.pb,
                              rows, rows, c.n, 0, c.mulws, c.mulws_bytes, c.st, false);
        }
        return run_update(c.ks, c.e, c.tab, Ib, tb / 64, tb * (tb / 64), Bb, c.ldb, c.pb, Bb, c.ldb, c.pb, rows, rows,
                          c.n, 0, c.mulws, c.mulws_bytes, c.st, true);
    }
    const int64_t h = i0 + round_up(rows / 2, tb);  // aligned split: plane views stay word aligned
    auto update = [&](int64_t r0, int64_t r1, int64_t k0, int64_t k1) {  // B[r0:r1] ^= T[r0:r1, k0:k1] X[k0:k1]
        return run_update(c.ks, c.e, c.tab, c.T + r0 * c.ldt + k0 / 64, c.ldt, c.pt, c.B + k0 * c.ldb, c.ldb, c.pb,
                          c.B + r0 * c.ldb, c.ldb, c.pb, r1 - r0, k1 - k0, c.n, GF2E_ACCUMULATE, c.mulws,
                          c.mulws_bytes, c.st);
    };
    if (c.upper) {  // ple_echelon.py:201-217 order: bottom block, update top, top block
        if (int rc = trsm_rec(c, h, i1)) return rc;
        if (int rc = update(i0, h, h, i1)) return rc;
        return trsm_rec(c, i0, h);
    }
    if (int rc = trsm_rec(c, i0, h)) return rc;  // ple_echelon.py:159-175
    if (int rc = update(h, i1, i0, h)) return rc;
    return trsm_rec(c, h, i1);
}

int check_flags(uint32_t flags) {
    if (flags & ~(GF2E_ACCUMULATE | GF2E_BACKEND_M4RM | GF2E_TC_INT8 | GF2E_TC_FP4 | GF2E_TC_RUN))
        return fail(GF2E_EINVAL, "unknown flags 0x%x", flags);
    const uint32_t forced = flags & (GF2E_TC_INT8 | GF2E_TC_FP4 | GF2E_TC_RUN);
    if (forced & (forced - 1)) return fail(GF2E_EINVAL, "conflicting flags 0x%x", flags);
    return GF2E_OK;
}

int trsm_impl(int e, uint32_t f, int upper, int unit_diag, const uint64_t *T, int64_t ldt, int64_t pt, uint64_t *B,
              int64_t ldb, int64_t pb, int64_t m, int64_t n, void *ws, int64_t ws_bytes, void *stream,
              int64_t *bad_row, bool check);

// ---- PLE / echelonize over plane views (consumers of run_product and the TRSM) ----------------
// Stream-ordered temporaries from the CUDA memory pool (freed at scope exit, reused by the pool).
struct DevTmp {
    void *p = nullptr;
    cudaStream_t st;
    DevTmp(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes && pool_alloc(&p, bytes, st) != cudaSuccess) p = nullptr;
    }
    ~DevTmp() {
        if (p) cudaFreeAsync(p, st);
    }
    DevTmp(const DevTmp &) = delete;
    DevTmp &operator=(const DevTmp &) = delete;
};

struct PleCtx {
    int e;
    uint32_t f;
    Sched ks;
    uint64_t *S;
    int64_t ld, ps;
    cudaStream_t st;
    PanelOut *pout;  // device
    int64_t *idx;    // device index scratch (3 * max(m, n) + 3 entries)
    const FieldTab *tab;
    int64_t panels = 0;
    static constexpr int kRing = 4;
    int64_t *ring[kRing] = {};  // pinned staging, 3 * max(m, n) + 3 entries each
    cudaEvent_t ring_ev[kRing] = {};
    int ring_next = 0;
};

// host vector -> device index scratch (synchronous staging: the host buffer may be reused)
// LAPACK-style swap vector -> the (t, P[t]) pairs that move something
std::vector<int64_t> swap_pairs(const int64_t *P, int64_t n) {
    std::vector<int64_t> v;
    for (int64_t t = 0; t < n; ++t)
        if (P[t] != t) {
            v.push_back(t);
            v.push_back(P[t]);
        }
    return v;
}

// Upload through a ring of pinned staging slots (an event guards each slot's reuse), so the
// copies stay asynchronous; the device index buffer itself is reused in stream order.
int put_idx(PleCtx &c, const std::vector<int64_t> &v) {
    if (v.empty()) return GF2E_OK;
    const int slot = c.ring_next++ % PleCtx::kRing;
    CKH(cudaEventSynchronize(c.ring_ev[slot]), "cudaEventSynchronize");
    std::memcpy(c.ring[slot], v.data(), v.size() * 8);
    CKH(cudaMemcpyAsync(c.idx, c.ring[slot], v.size() * 8, cudaMemcpyHostToDevice, c.st), "cudaMemcpyAsync");
    CKH(cudaEventRecord(c.ring_ev[slot], c.st), "cudaEventRecord");
    return GF2E_OK;
}

// ple_echelon.py:240-287 on the view rows [r0, r0+m), columns [c0, c0+n) (c0 % 64 == 0).  The
// column split is rounded to a plane word: the factorisation does not depend on it (the
// reference makes the same claim for its crossover, ple_echelon.py:8-10, and every split is
// checked against its fixtures).  P, Q: length min(m, n), LAPACK-style swap vectors.
int ple_rec(PleCtx &c, int64_t r0, int64_t c0, int64_t m, int64_t n, int64_t *P, int64_t *Q, int64_t &rank) {
    const int64_t k = m < n ? m : n;
    for (int64_t i = 0; i < k; ++i) P[i] = Q[i] = i;
    rank = 0;
    if (m == 0 || n == 0) return GF2E_OK;
    uint64_t *V = c.S + r0 * c.ld + c0 / 64;
    if (n <= kPlePanel) {  // base case nj_ple (newton_john.py:207-260) on one plane word
        CK(launch_ple_panel(c.e, c.tab, V, c.ld, c.ps, m, (int)n, c.pout, c.st), "ple_panel");
        g_launches += m > ple_window(c.e) ? 2 : 1;
        ++c.panels;
        struct Head {  // the leading members of PanelOut (rank .. Q)
            int rank, ndisp, window, pad;
            int64_t P[64], Q[64];
        } h;
        static_assert(sizeof(Head) == offsetof(PanelOut, jcol) && offsetof(Head, Q) == offsetof(PanelOut, Q),
                      "PanelOut layout");
        CKH(cudaMemcpyAsync(&h, c.pout, sizeof(Head), cudaMemcpyDeviceToHost, c.st), "cudaMemcpyAsync");
        CKH(cudaStreamSynchronize(c.st), "cudaStreamSynchronize");
        rank = h.rank;
        for (int64_t t = 0; t < rank; ++t) {
            P[t] = h.P[t];
            Q[t] = h.Q[t];
        }
        return GF2E_OK;
    }
    int64_t n1 = round_up(n / 2, 64);
    if (n1 >= n) n1 -= 64;
    const int64_t k1 = m < n1 ? m : n1;
    std::vector<int64_t> P1(k1), Q1(k1);
    int64_t r1 = 0;
    if (int rc = ple_rec(c, r0, c0, m, n1, P1.data(), Q1.data(), r1)) return rc;
    uint64_t *R = V + n1 / 64;  // right half view
    const int64_t nr = n - n1;
    if (r1 > 0) {
        std::vector<int64_t> sw = swap_pairs(P1.data(), r1);
        if (!sw.empty()) {
            if (int rc = put_idx(c, sw)) return rc;
            CK(launch_row_swaps(c.e, R, c.ld, c.ps, words_for(nr), c.idx, (int)(sw.size() / 2), false, c.st),
               "row_swaps");
        }
        // L_top X = right[0:r1]  (the corner with its diagonal = pivots, ple_echelon.py:255-258)
        const int64_t lw = words_for(r1);
        DevTmp lt((size_t)c.e * r1 * lw * 8, c.st);
        if (!lt.p) return fail(GF2E_ENOMEM, "out of device memory (PLE corner)");
        uint64_t *L = static_cast<uint64_t *>(lt.p);
        CK(launch_tril_copy(c.e, V, c.ld, c.ps, r1, L, lw, r1 * lw, c.st), "tril_copy");
        const int64_t tws = gf2e_trsm_workspace(c.e, c.f, r1, nr);
        DevTmp tw((size_t)(tws > 0 ? tws : 256), c.st);
        if (!tw.p) return fail(GF2E_ENOMEM, "out of device memory (PLE trsm workspace)");
        int64_t bad = -1;
        if (int rc = trsm_impl(c.e, c.f, 0, 0, L, lw, r1 * lw, R, c.ld, c.ps, r1, nr, tw.p, tws, c.st, &bad, false))
            return rc;
        if (m - r1 > 0) {  // right[r1:] ^= left[r1:, :r1] . right[:r1]  (ple_echelon.py:259-260)
            const int64_t mws = gf2e_slice_mul_workspace(c.e, c.f, m - r1, r1, nr, GF2E_ACCUMULATE);
            DevTmp mw((size_t)(mws > 0 ? mws : 256), c.st);
            if (!mw.p) return fail(GF2E_ENOMEM, "out of device memory (PLE update workspace)");
            if (int rc = run_update(c.ks, c.e, c.tab, V + r1 * c.ld, c.ld, c.ps, R, c.ld, c.ps, R + r1 * c.ld, c.ld, c.ps,
                                    m - r1, r1, nr, GF2E_ACCUMULATE, mw.p, mws, c.st))
                return rc;
        }
    }
    const int64_t k2 = (m - r1) < nr ? (m - r1) : nr;
    std::vector<int64_t> P2(k2 > 0 ? k2 : 0), Q2(k2 > 0 ? k2 : 0);
    int64_t r2 = 0;
    if (m - r1 > 0)
        if (int rc = ple_rec(c, r0 + r1, c0 + n1, m - r1, nr, P2.data(), Q2.data(), r2)) return rc;
    if (r2 > 0) {
        std::vector<int64_t> sw = swap_pairs(P2.data(), r2);  // left rows r1.. (ple_echelon.py:268-271)
        if (!sw.empty()) {
            if (int rc = put_idx(c, sw)) return rc;
            CK(launch_row_swaps(c.e, V + r1 * c.ld, c.ld, c.ps, n1 / 64, c.idx, (int)(sw.size() / 2), false, c.st),
               "row_swaps");
        }
        std::vector<int64_t> tr;  // compress the right half's L into the leading columns (:275-279)
        for (int64_t u = 0; u < r2; ++u)
            if (n1 + u != r1 + u) tr.insert(tr.end(), {r1 + u, n1 + u, r1 + u});
        if (!tr.empty()) {
            if (int rc = put_idx(c, tr)) return rc;
            CK(launch_col_swaps(c.e, 1, V, c.ld, c.ps, m, c.idx, (int)(tr.size() / 3), c.st), "col_swaps");
        }
    }
    for (int64_t t = 0; t < r1; ++t) {
        P[t] = P1[t];
        Q[t] = Q1[t];
    }
    for (int64_t t = 0; t < r2; ++t) {
        P[r1 + t] = r1 + P2[t];
        Q[r1 + t] = n1 + Q2[t];
    }
    rank = r1 + r2;
    return GF2E_OK;
}

// ---- speculative PLE: no host synchronisation inside the recursion ---------------------------
// The recursion's launch sequence depends on the data only through the ranks of the left halves
// (the sizes of the corner solves, Schur updates and sub-problems) and the row pivots.  A
// generic matrix has full rank at every node (r1 = min(m, n1)) and the column rank profile
// 0, 1, 2, ...; so the whole recursion is enqueued with those ranks, the row pivots stay in
// device memory (every panel commits its pivots into global swap vectors that the row-swap
// kernels read), and every panel checks its rank against the speculated one.  One
// synchronisation at the end reads the flag: if any panel fell short, the input is restored
// from a device copy and the exact host-driven recursion (ple_rec) runs instead.
struct PleSpec {
    int e;
    uint32_t f;
    Sched ks;
    uint64_t *S;
    int64_t ld, ps;
    cudaStream_t st;
    PanelOut *pout;
    const FieldTab *tab;
    int64_t *Pg, *Qg;  // device swap vectors (length min(m, n))
    int *flag;         // device: a panel's rank differed from the speculated one
    int64_t *hstage, *dstage;  // column-swap triples: pinned host / device bump buffers
    size_t cap, used;          // entries
};

int ple_rec_spec(PleSpec &c, int64_t r0, int64_t c0, int64_t m, int64_t n) {
    if (m == 0 || n == 0) return GF2E_OK;
    uint64_t *V = c.S + r0 * c.ld + c0 / 64;
    if (n <= kPlePanel) {
        CK(launch_ple_panel(c.e, c.tab, V, c.ld, c.ps, m, (int)n, c.pout, c.st), "ple_panel");
        g_launches += m > ple_window(c.e) ? 1 : 0;
        CK(launch_ple_commit(c.pout, c.Pg, c.Qg, r0, c0, (int)(m < n ? m : n), c.flag, c.st), "ple_commit");
        return GF2E_OK;
    }
    int64_t n1 = round_up(n / 2, 64);
    if (n1 >= n) n1 -= 64;
    if (int rc = ple_rec_spec(c, r0, c0, m, n1)) return rc;
    const int64_t r1 = m < n1 ? m : n1, nr = n - n1;
    uint64_t *R = V + n1 / 64;
    if (r1 > 0) {
        CK(launch_row_swaps_vec(c.e, c.S + (c0 + n1) / 64, c.ld, c.ps, words_for(nr), c.Pg, r0, r0 + r1, c.st),
           "row_swaps");
        const int64_t lw = words_for(r1);
        DevTmp lt((size_t)c.e * r1 * lw * 8, c.st);
        if (!lt.p) return fail(GF2E_ENOMEM, "out of device memory (PLE corner)");
        uint64_t *L = static_cast<uint64_t *>(lt.p);
        CK(launch_tril_copy(c.e, V, c.ld, c.ps, r1, L, lw, r1 * lw, c.st), "tril_copy");
        const int64_t tws = gf2e_trsm_workspace(c.e, c.f, r1, nr);
        DevTmp tw((size_t)(tws > 0 ? tws : 256), c.st);
        if (!tw.p) return fail(GF2E_ENOMEM, "out of device memory (PLE trsm workspace)");
        int64_t bad = -1;
        if (int rc = trsm_impl(c.e, c.f, 0, 0, L, lw, r1 * lw, R, c.ld, c.ps, r1, nr, tw.p, tws, c.st, &bad, false))
            return rc;
        if (m - r1 > 0) {
            const int64_t mws = gf2e_slice_mul_workspace(c.e, c.f, m - r1, r1, nr, GF2E_ACCUMULATE);
            DevTmp mw((size_t)(mws > 0 ? mws : 256), c.st);
            if (!mw.p) return fail(GF2E_ENOMEM, "out of device memory (PLE update workspace)");
            if (int rc = run_update(c.ks, c.e, c.tab, V + r1 * c.ld, c.ld, c.ps, R, c.ld, c.ps, R + r1 * c.ld, c.ld, c.ps,
                                    m - r1, r1, nr, GF2E_ACCUMULATE, mw.p, mws, c.st))
                return rc;
        }
    }
    if (m - r1 > 0)
        if (int rc = ple_rec_spec(c, r0 + r1, c0 + n1, m - r1, nr)) return rc;
    const int64_t r2 = (m - r1) < nr ? (m - r1) : nr;
    if (r2 > 0) {
        CK(launch_row_swaps_vec(c.e, c.S + c0 / 64, c.ld, c.ps, n1 / 64, c.Pg, r0 + r1, r0 + r1 + r2, c.st),
           "row_swaps");
        std::vector<int64_t> tr;  // compress the right half's L into the leading columns (:275-279)
        for (int64_t u = 0; u < r2; ++u)
            if (n1 + u != r1 + u) tr.insert(tr.end(), {r1 + u, n1 + u, r1 + u});
        if (!tr.empty()) {
            if (c.used + tr.size() > c.cap) return fail(GF2E_ENOMEM, "PLE staging overflow");
            int64_t *h = c.hstage + c.used, *d = c.dstage + c.used;
            std::memcpy(h, tr.data(), tr.size() * 8);
            c.used += tr.size();
            CKH(cudaMemcpyAsync(d, h, tr.size() * 8, cudaMemcpyHostToDevice, c.st), "cudaMemcpyAsync");
            CK(launch_col_swaps(c.e, 1, V, c.ld, c.ps, m, d, (int)(tr.size() / 3), c.st), "col_swaps");
        }
    }
    return GF2E_OK;
}

// column-swap triples the speculative recursion stages: 3 per compressed column per node, at
// most 3 * min(m, n) per recursion level
int64_t ple_spec_stage_entries(int64_t m, int64_t n) {
    int64_t levels = 1;
    for (int64_t w = n; w > kPlePanel; w = (w + 1) / 2) ++levels;
    return 3 * (m < n ? m : n) * levels + 64;
}

// 1: done (P, Q, rank written); 0: a rank check failed, S restored; <0... errors as status
int ple_try_spec(int e, uint32_t f, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t n, int64_t *P,
                 int64_t *Q, int64_t *rank, cudaStream_t st, const FieldTab *tab, PanelOut *pout, bool *done) {
    *done = false;
    const int64_t k = m < n ? m : n, nw = words_for(n);
    DevTmp backup((size_t)e * m * nw * 8, st), pq((size_t)2 * k * 8 + 256, st);
    const int64_t entries = ple_spec_stage_entries(m, n);
    DevTmp dst((size_t)entries * 8, st);
    if (!backup.p || !pq.p || !dst.p) return GF2E_OK;  // no room: take the exact path
    // pinned host staging, persistent per host thread and device (grown on demand)
    struct Stage {
        int64_t *buf = nullptr;
        size_t cap = 0;
    };
    thread_local Stage stages[kMaxDevices];
    int dev = 0;
    CKH(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return GF2E_OK;
    Stage &sg = stages[dev];
    if (sg.cap < (size_t)entries) {
        if (sg.buf) {
            CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            cudaFreeHost(sg.buf);
            sg.buf = nullptr;
            sg.cap = 0;
        }
        const size_t want = (size_t)entries > ((size_t)1 << 17) ? (size_t)entries : ((size_t)1 << 17);
        if (cudaMallocHost(reinterpret_cast<void **>(&sg.buf), want * 8) != cudaSuccess) return GF2E_OK;
        sg.cap = want;
    }
    uint64_t *bk = static_cast<uint64_t *>(backup.p);
    for (int t = 0; t < e; ++t)
        CKH(cudaMemcpy2DAsync(bk + t * m * nw, nw * 8, S + t * ps, ld * 8, nw * 8, m, cudaMemcpyDeviceToDevice, st),
            "backup");
    int64_t *Pg = static_cast<int64_t *>(pq.p), *Qg = Pg + k;
    int *flag = reinterpret_cast<int *>(Qg + k);
    CKH(cudaMemsetAsync(flag, 0, sizeof(int), st), "cudaMemsetAsync");
    PleSpec c{e, f, to_kernel_sched(e, get_schedule(e, f)), S, ld, ps, st, pout, tab, Pg, Qg, flag,
              sg.buf, static_cast<int64_t *>(dst.p), (size_t)entries, 0};
    const auto h0 = std::chrono::steady_clock::now();
    if (int rc = ple_rec_spec(c, 0, 0, m, n)) return rc;
    if (getenv("GF2E_PLE_TRACE"))
        fprintf(stderr, "ple spec: host enqueue %.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    int hflag = 0;
    std::vector<int64_t> hp(k), hq(k);
    CKH(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    CKH(cudaMemcpyAsync(hp.data(), Pg, k * 8, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    CKH(cudaMemcpyAsync(hq.data(), Qg, k * 8, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (hflag) {  // some left half was rank deficient: restore and take the exact path
        for (int t = 0; t < e; ++t)
            CKH(cudaMemcpy2DAsync(S + t * ps, ld * 8, bk + t * m * nw, nw * 8, nw * 8, m, cudaMemcpyDeviceToDevice,
                                  st),
                "restore");
        return GF2E_OK;
    }
    for (int64_t i = 0; i < k; ++i) {
        if (P) P[i] = hp[i];
        if (Q) Q[i] = hq[i];
    }
    if (rank) *rank = k;
    *done = true;
    return GF2E_OK;
}

int ple_top(int e, uint32_t f, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t n, int64_t *P, int64_t *Q,
            int64_t *rank, cudaStream_t st) {
    const int64_t k = m < n ? m : n;
    DevTmp po(sizeof(PanelOut), st);
    DevTmp ix((size_t)(3 * (m > n ? m : n) + 3) * 8, st);
    if (!po.p || !ix.p) return fail(GF2E_ENOMEM, "out of device memory (PLE scratch)");
    const FieldTab *tab = field_tab(e, f, primitive_element(e, f));
    if (!tab) return fail(GF2E_ECUDA, "field table upload failed");
    if (!getenv("GF2E_PLE_EXACT")) {  // GF2E_PLE_EXACT=1: always the host-driven recursion
        bool done = false;
        if (int rc = ple_try_spec(e, f, S, ld, ps, m, n, P, Q, rank, st, tab, static_cast<PanelOut *>(po.p), &done))
            return rc;
        if (done) return GF2E_OK;
    }
    PleCtx c{e, f, to_kernel_sched(e, get_schedule(e, f)), S, ld, ps, st, static_cast<PanelOut *>(po.p),
             static_cast<int64_t *>(ix.p), tab};
    // The pinned staging ring persists per host thread and only grows: pinning and unpinning
    // host pages on every call (cudaMallocHost / cudaFreeHost) stalled some calls for
    // hundreds of milliseconds.  It is never freed (process lifetime).  One ring per device:
    // its events belong to the device that was current when they were created.
    struct PinnedRing {
        int64_t *buf[PleCtx::kRing] = {};
        cudaEvent_t ev[PleCtx::kRing] = {};
        size_t bytes = 0;
    };
    thread_local PinnedRing rings[kMaxDevices];
    int dev = 0;
    CKH(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return fail(GF2E_ENODEV, "device index %d out of range", dev);
    PinnedRing &pr = rings[dev];
    const size_t ring_bytes = (size_t)(3 * (m > n ? m : n) + 3) * 8;
    if (pr.bytes < ring_bytes) {
        for (int i = 0; i < PleCtx::kRing; ++i) {
            if (pr.ev[i]) CKH(cudaEventSynchronize(pr.ev[i]), "cudaEventSynchronize");
            if (pr.buf[i]) cudaFreeHost(pr.buf[i]);
            pr.buf[i] = nullptr;
        }
        pr.bytes = 0;
        const size_t want = ring_bytes > (size_t)1 << 20 ? ring_bytes : (size_t)1 << 20;
        for (int i = 0; i < PleCtx::kRing; ++i)
            if (cudaMallocHost(reinterpret_cast<void **>(&pr.buf[i]), want) != cudaSuccess)
                return fail(GF2E_ENOMEM, "out of pinned host memory (PLE staging)");
        pr.bytes = want;
    }
    for (int i = 0; i < PleCtx::kRing; ++i) {
        if (!pr.ev[i] && cudaEventCreateWithFlags(&pr.ev[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(GF2E_ECUDA, "cudaEventCreate (PLE staging)");
        c.ring[i] = pr.buf[i];
        c.ring_ev[i] = pr.ev[i];
    }
    std::vector<int64_t> hp(k), hq(k);
    int64_t r = 0;
    if (int rc = ple_rec(c, 0, 0, m, n, hp.data(), hq.data(), r)) return rc;
    for (int64_t i = 0; i < k; ++i) {
        if (P) P[i] = hp[i];
        if (Q) Q[i] = hq[i];
    }
    if (rank) *rank = r;
    return GF2E_OK;
}

}  // namespace

extern "C" {

const char *gf2e_last_error(void) { return g_err.c_str(); }
const char *gf2e_version(void) { return "gf2e_b200 0.2 (sm_100a; tcgen05 cta_group::2 kind::mxf4 + kind::i8, M4RM)"; }
int gf2e_last_launch_count(void) { return g_launches; }
int64_t gf2e_last_gf2_products(void) { return g_products; }
const char *gf2e_last_product_kernel(void) { return g_kernel; }

int gf2e_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    return GF2E_OK;
}

int gf2e_profile_read(double *total_ms, int *launches) {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        evs.swap(g_prof_events);
    }
    double tot = 0;
    int rc = GF2E_OK;
    for (auto &p : evs) {
        float ms = 0;
        cudaError_t e = cudaEventSynchronize(p.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, p.first, p.second);
        if (e != cudaSuccess) rc = cuda_fail(e, "gf2e_profile_read");
        tot += ms;
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = (int)evs.size();
    return rc;
}

int gf2e_mma_peak(int cta_group, int iters, double *tops, double *ms, void *stream) {
    g_err.clear();
    if (cta_group != 1 && cta_group != 2) return fail(GF2E_EINVAL, "cta_group must be 1 or 2");
    if (iters < 1) return fail(GF2E_EINVAL, "iters must be >= 1");
    if (int rc = check_device()) return rc;
    int dev = 0, nsms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
    float t = 0;
    cudaError_t e = run_mma_peak(cta_group, iters, nsms, (cudaStream_t)stream, &t);
    if (e != cudaSuccess) return cuda_fail(e, "mma_peak");
    const int sms_used = cta_group == 2 ? (nsms & ~1) : nsms;
    const double ops = (double)sms_used * iters * 4.0 * 2.0 * 128.0 * 256.0 * 32.0;
    if (ms) *ms = t;
    if (tops) *tops = ops / (t * 1e-3) / 1e12;
    return GF2E_OK;
}

int gf2e_int_peak(int iters, double *lds_bytes_per_s, double *m4rm_tops, void *stream) {
    g_err.clear();
    if (iters < 1) return fail(GF2E_EINVAL, "iters must be >= 1");
    if (int rc = check_device()) return rc;
    int dev = 0, nsms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
    double bps = 0;
    cudaError_t e = run_lds_peak(iters, nsms, (cudaStream_t)stream, &bps);
    if (e != cudaSuccess) return cuda_fail(e, "lds_peak");
    if (lds_bytes_per_s) *lds_bytes_per_s = bps;
    // k_product_m4rm: one 16-byte table read (+ 4 LOP3) per (row, 128 columns, 8 k-bits) =
    // 128 x 8 x 2 GF(2) bit-ops
    if (m4rm_tops) *m4rm_tops = bps / 16.0 * 2048.0 / 1e12;
    return GF2E_OK;
}

int gf2e_dev_fp4_probe(int iters, int mode, const uint8_t *a_dev, const uint8_t *b_dev, uint32_t *out_dev,
                       double *tops, void *stream) {
    g_err.clear();
    if (iters < 1 || !a_dev || !b_dev || !out_dev) return fail(GF2E_EINVAL, "bad probe arguments");
    if (int rc = check_device()) return rc;
    int dev = 0, nsms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsms, cudaDevAttrMultiProcessorCount, dev);
    float ms = 0;
    cudaError_t e = run_fp4_probe(iters, mode, a_dev, b_dev, out_dev, nsms, (cudaStream_t)stream, &ms);
    if (e != cudaSuccess) return cuda_fail(e, "fp4_probe");
    if (tops) *tops = (double)nsms * iters * 4.0 * 2.0 * 128.0 * 256.0 * 64.0 / (ms * 1e-3) / 1e12;
    return GF2E_OK;
}

int gf2e_fp4_selfcheck(int rerun, int inject_fault, int *ok) {
    g_err.clear();
    if (ok) *ok = 0;
    if (int rc = check_device()) return rc;
    int dev = 0;
    cudaGetDevice(&dev);
    if (rerun || inject_fault) {
        std::lock_guard<std::mutex> lk(g_fp4_mu);
        g_fp4_state[dev] = 0;
        g_fp4_inject = inject_fault != 0;
    }
    if (int rc = ensure_fp4_checked()) return rc;
    if (ok) *ok = fp4_state();
    return GF2E_OK;
}

int gf2e_run_schedule(int e, uint32_t f, int *nseq, int *ngrp, int *run_load, int *seq, int *gsize,
                      uint32_t *gmask) {
    g_err.clear();
    if (int rc = check_field(e, f)) return rc;
    const Sched k = to_kernel_sched(e, get_schedule(e, f));
    if (nseq) *nseq = k.nseq;
    if (ngrp) *ngrp = k.ngrp;
    if (run_load) *run_load = k.run_load;
    for (int i = 0; i < k.nseq; ++i)
        if (seq) seq[i] = k.seq[i];
    for (int g = 0; g < k.ngrp; ++g) {
        if (gsize) gsize[g] = k.gsize[g];
        if (gmask) gmask[g] = k.gmask[g];
    }
    return GF2E_OK;
}

int64_t gf2e_tile_cols(int e, uint32_t f, int64_t k, uint32_t flags) {
    g_err.clear();
    if (check_field(e, f) || check_flags(flags)) return -1;
    if (flags & GF2E_BACKEND_M4RM) return kM4BN;
    return form_bn(tc_form(flags, k, (int)get_schedule(e, f).subsets.size()));
}

int gf2e_trim_pool(int64_t keep_bytes) {
    g_err.clear();
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return fail(GF2E_ENODEV, "no CUDA device");
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        pool = g_pools[dev];
    }
    if (!pool) return GF2E_OK;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, (size_t)(keep_bytes > 0 ? keep_bytes : 0));
    return e == cudaSuccess ? GF2E_OK : cuda_fail(e, "gf2e_trim_pool");
}

int gf2e_pack_width(int e) {
    if (e < 2 || e > 10) return -1;
    for (int w : {1, 2, 4, 8, 16, 32, 64})
        if (w >= e) return w;
    return -1;
}

int gf2e_schedule(int e, uint32_t f, int *n_products, uint64_t *subsets, uint64_t *outmap, int64_t *counters) {
    g_err.clear();
    int rc = check_field(e, f);
    if (rc) return rc;
    const Schedule &S = get_schedule(e, f);
    if (n_products) *n_products = (int)S.subsets.size();
    if (subsets)
        for (size_t t = 0; t < S.subsets.size(); ++t) subsets[t] = S.subsets[t];
    if (outmap)
        for (int j = 0; j < e; ++j) outmap[j] = S.outmap[j];
    if (counters)
        for (int i = 0; i < 3; ++i) counters[i] = S.counters[i];
    return GF2E_OK;
}

int gf2e_random_packed(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0, int64_t col0, int64_t gcols,
                       uint64_t *out, int64_t ldp, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    int w = gf2e_pack_width(e);
    if (w < 0) return fail(GF2E_EINVAL, "extension degree must be in 2..10, got %d", e);
    if (int rc = check_mat(out, rows, words_for(cols * w), ldp, "packed")) return rc;
    if (rows == 0 || ldp == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_random_packed(e, w, rows, cols, seed, row0, col0, gcols, out, ldp, (cudaStream_t)stream),
       "random_packed");
    return GF2E_OK;
}

int gf2e_random_sliced(int e, int64_t rows, int64_t cols, uint64_t seed, int64_t row0, int64_t col0, int64_t gcols,
                       uint64_t *planes, int64_t ld, int64_t pstride, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (e < 2 || e > 10) return fail(GF2E_EINVAL, "extension degree must be in 2..10, got %d", e);
    if (int rc = check_mat(planes, rows, words_for(cols), ld, "planes")) return rc;
    if (rows == 0 || ld == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_random_sliced(e, rows, cols, seed, row0, col0, gcols, planes, ld, pstride, (cudaStream_t)stream),
       "random_sliced");
    return GF2E_OK;
}

int gf2e_random_words(int64_t rows, int64_t ncols, uint64_t seed, uint64_t *out, int64_t ld, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_mat(out, rows, words_for(ncols), ld, "words")) return rc;
    if (rows == 0 || ncols == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_random_words(rows, ncols, seed, out, ld, (cudaStream_t)stream), "random_words");
    return GF2E_OK;
}

int gf2e_slice(int e, int64_t rows, int64_t cols, const uint64_t *packed, int64_t ldp, uint64_t *planes, int64_t ld,
               int64_t pstride, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    int w = gf2e_pack_width(e);
    if (w < 0) return fail(GF2E_EINVAL, "extension degree must be in 2..10, got %d", e);
    if (int rc = check_mat(packed, rows, words_for(cols * w), ldp, "packed")) return rc;
    if (int rc = check_mat(planes, rows, words_for(cols), ld, "planes")) return rc;
    if (rows == 0 || ld == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_slice(e, w, rows, cols, packed, ldp, planes, ld, pstride, (cudaStream_t)stream), "slice");
    return GF2E_OK;
}

int gf2e_cling(int e, int64_t rows, int64_t cols, const uint64_t *planes, int64_t ld, int64_t pstride,
               uint64_t *packed, int64_t ldp, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    int w = gf2e_pack_width(e);
    if (w < 0) return fail(GF2E_EINVAL, "extension degree must be in 2..10, got %d", e);
    if (int rc = check_mat(packed, rows, words_for(cols * w), ldp, "packed")) return rc;
    if (int rc = check_mat(planes, rows, words_for(cols), ld, "planes")) return rc;
    if (rows == 0 || ldp == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_cling(e, w, rows, cols, planes, ld, pstride, packed, ldp, (cudaStream_t)stream), "cling");
    return GF2E_OK;
}

int gf2e_xor(uint64_t *x, int64_t ldx, const uint64_t *y, int64_t ldy, int64_t rows, int64_t nwords, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_mat(x, rows, nwords, ldx, "x")) return rc;
    if (int rc = check_mat(y, rows, nwords, ldy, "y")) return rc;
    if (rows == 0 || nwords == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_xor(x, ldx, y, ldy, rows, nwords, (cudaStream_t)stream), "xor");
    return GF2E_OK;
}

int gf2e_reduce_mod_f(int e, uint32_t f, uint64_t *planes, int64_t rows, int64_t nwords, int64_t ld, int64_t pstride,
                      void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_mat(planes, rows, nwords, ld, "planes")) return rc;
    if (rows == 0 || nwords == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_reduce(e, f, planes, rows, nwords, ld, pstride, (cudaStream_t)stream), "reduce_mod_f");
    return GF2E_OK;
}

int64_t gf2e_slice_mul_workspace(int e, uint32_t f, int64_t m, int64_t k, int64_t n, uint32_t flags) {
    g_err.clear();
    if (check_field(e, f) || check_flags(flags)) return -1;
    if (m < 0 || k < 0 || n < 0) return fail(GF2E_EINVAL, "matrix dimensions must be non-negative"), -1;
    if (m == 0 || k == 0 || n == 0) return 0;
    const Schedule &S = get_schedule(e, f);
    // a bound over the tensor-core forms: the form is picked at call time (it can change when
    // the fp4 self-check disables fp4 between this query and the product)
    return layout_for((int)S.subsets.size(), m, k, n, flags, kFormAny).total;
}

int64_t gf2e_plane_mul_workspace(int64_t m, int64_t k, int64_t n, uint32_t flags) {
    g_err.clear();
    if (check_flags(flags)) return -1;
    if (m < 0 || k < 0 || n < 0) return fail(GF2E_EINVAL, "matrix dimensions must be non-negative"), -1;
    if (m == 0 || k == 0 || n == 0) return 0;
    return layout_for(1, m, k, n, flags, kFormAny).total;
}

int gf2e_slice_mul(int e, uint32_t f, const uint64_t *A, int64_t lda, int64_t pa, const uint64_t *B, int64_t ldb,
                   int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m, int64_t k, int64_t n, uint32_t flags,
                   void *ws, int64_t ws_bytes, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_flags(flags)) return rc;
    if (int rc = check_mat(A, m, words_for(k), lda, "A")) return rc;
    if (int rc = check_mat(B, k, words_for(n), ldb, "B")) return rc;
    if (int rc = check_mat(C, m, words_for(n), ldc, "C")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    Sched ks = to_kernel_sched(e, get_schedule(e, f));
    return run_product(ks, A, lda, pa, B, ldb, pb, C, ldc, pc, m, k, n, flags, ws, ws_bytes, (cudaStream_t)stream);
}

int gf2e_nj_slice_mul(int e, uint32_t f, const uint64_t *A, int64_t lda, int64_t pa, const uint64_t *B, int64_t ldb,
                      int64_t pb, uint64_t *C, int64_t ldc, int64_t pc, int64_t m, int64_t k, int64_t n,
                      uint32_t flags, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (flags & ~GF2E_ACCUMULATE) return fail(GF2E_EINVAL, "gf2e_nj_slice_mul: unsupported flags 0x%x", flags);
    if (int rc = check_mat(A, m, words_for(k), lda, "A")) return rc;
    if (int rc = check_mat(B, k, words_for(n), ldb, "B")) return rc;
    if (int rc = check_mat(C, m, words_for(n), ldc, "C")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const bool acc = (flags & GF2E_ACCUMULATE) != 0;
    if (k == 0) {
        if (!acc)
            for (int j = 0; j < e; ++j)
                CK(cudaMemset2DAsync(C + j * pc, ldc * 8, 0, words_for(n) * 8, m, st), "cudaMemset2DAsync");
        return GF2E_OK;
    }
    const FieldTab *tab = field_tab(e, f, primitive_element(e, f));
    if (!tab) return fail(GF2E_ECUDA, "field table upload failed");
    CK(launch_nj_sliced(e, tab, A, lda, pa, B, ldb, pb, C, ldc, pc, m, k, n, acc, false, st), "nj_sliced");
    g_kernel = "k_nj_sliced";
    return GF2E_OK;
}

int gf2e_nj_mul(int e, uint32_t f, const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, uint64_t *C,
                int64_t ldc, int64_t m, int64_t k, int64_t n, uint32_t flags, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (flags & ~GF2E_ACCUMULATE) return fail(GF2E_EINVAL, "gf2e_nj_mul: unsupported flags 0x%x", flags);
    const int w = gf2e_pack_width(e);
    const int64_t wb = words_for(n * w);
    if (wb > kNjMaxWords)
        return fail(GF2E_EINVAL, "gf2e_nj_mul: %lld columns exceed the small-block product (%d words per row)",
                    (long long)n, kNjMaxWords);
    if (int rc = check_mat(A, m, words_for(k * w), lda, "A")) return rc;
    if (int rc = check_mat(B, k, wb, ldb, "B")) return rc;
    if (int rc = check_mat(C, m, wb, ldc, "C")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const bool acc = (flags & GF2E_ACCUMULATE) != 0;
    if (k == 0) {
        if (!acc) CK(cudaMemset2DAsync(C, ldc * 8, 0, wb * 8, m, st), "cudaMemset2DAsync");
        return GF2E_OK;
    }
    CK(launch_nj_mul(e, f, w, A, lda, B, ldb, C, ldc, m, k, n, acc, st), "nj_mul");
    g_kernel = "k_nj_mul";
    return GF2E_OK;
}

int gf2e_slice_mul_parts(int e, uint32_t f, const uint64_t *A, int64_t lda, int64_t pa, int nparts,
                         const int64_t *col_bounds, const uint64_t *const *B_parts, const int64_t *ldb,
                         const int64_t *pb, void *const *ready_events, uint64_t *C, int64_t ldc, int64_t pc,
                         int64_t m, int64_t k, int64_t n, uint32_t flags, void *ws, int64_t ws_bytes,
                         void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_flags(flags)) return rc;
    if (flags & GF2E_BACKEND_M4RM) return fail(GF2E_EINVAL, "column parts need a tensor-core backend");
    if (nparts < 1 || !col_bounds || !B_parts || !ldb || !pb) return fail(GF2E_EINVAL, "bad part arrays");
    if (col_bounds[0] != 0 || col_bounds[nparts] != n)
        return fail(GF2E_EINVAL, "column bounds must run from 0 to n = %lld", (long long)n);
    for (int p = 0; p < nparts; ++p) {
        const int64_t c0 = col_bounds[p], c1 = col_bounds[p + 1];
        if (c1 < c0 || (p + 1 < nparts && (c1 & 63)))
            return fail(GF2E_EINVAL, "column bound %d (%lld) must be non-decreasing and a multiple of 64", p + 1,
                        (long long)c1);
        if (int rc = check_mat(B_parts[p], k, words_for(c1 - c0), ldb[p], "B part")) return rc;
    }
    if (int rc = check_mat(A, m, words_for(k), lda, "A")) return rc;
    if (int rc = check_mat(C, m, words_for(n), ldc, "C")) return rc;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const bool acc = (flags & GF2E_ACCUMULATE) != 0;
    if (m == 0 || n == 0 || k == 0) {  // nothing to wait for but the parts' events
        for (int p = 0; p < nparts; ++p)
            if (ready_events && ready_events[p])
                CKH(cudaStreamWaitEvent(st, (cudaEvent_t)ready_events[p], 0), "cudaStreamWaitEvent");
        if (m && n && !acc)
            for (int j = 0; j < e; ++j)
                CK(cudaMemset2DAsync(C + j * pc, ldc * 8, 0, words_for(n) * 8, m, st), "cudaMemset2DAsync");
        return GF2E_OK;
    }
    if (int rc = ensure_fp4_checked()) return rc;
    const Sched ks = to_kernel_sched(e, get_schedule(e, f));
    const int form = tc_form(flags, k, ks.nprod);
    const bool fp4 = form != kFormI8;
    const Layout L = layout_for(ks.nprod, m, k, n, flags, form);
    if (ws_bytes < L.total)
        return fail(GF2E_ENOMEM, "workspace too small: %lld < %lld bytes", (long long)ws_bytes, (long long)L.total);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255))
        return fail(GF2E_EINVAL, "workspace must be a 256-byte aligned device pointer");
    uint64_t *Ac = static_cast<uint64_t *>(ws);
    uint64_t *Bt = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + L.a_bytes);
    const int64_t tw = form_bn(form), ntiles = L.n_pad / tw;
    CK(launch_combos_rows(ks, A, lda, pa, m, k, Ac, L.kwords, L.a_pstride, L.m_pad, L.kwords, fp4 ? 4 : 2, st),
       "combos(A)");
    int64_t done = 0;  // column tiles already multiplied
    for (int p = 0; p < nparts; ++p) {
        const int64_t c0 = col_bounds[p], c1 = col_bounds[p + 1];
        const bool lastp = p + 1 == nparts;
        if (ready_events && ready_events[p])
            CKH(cudaStreamWaitEvent(st, (cudaEvent_t)ready_events[p], 0), "cudaStreamWaitEvent");
        const int64_t rend = lastp ? L.n_pad : c1;  // the last part also zero-fills the padding
        if (rend > c0)
            CK(launch_combos_bt(ks, B_parts[p], ldb[p], pb[p], k, c1 - c0, Bt, L.kwords, L.b_pstride, L.kwords,
                                (rend - c0) / 64, fp4, st, form_br(form), c0, form_bexp(form)),
               "combos(B^T part)");
        // every tile whose columns have all arrived
        const int64_t avail = lastp ? ntiles : c1 / tw;
        if (avail > done) {
            const int64_t n0 = done * tw, n1 = avail * tw < n ? avail * tw : n;
            TcArgs a{Ac, Bt + n0 * L.kwords * form_bx(form), L.a_pstride, L.b_pstride, L.kwords, m, n1 - n0, L.m_pad,
                     (avail - done) * tw, C + n0 / 64, ldc, pc, acc ? 1 : 0};
            ProfScope prof(st);
            CK(launch_form(ks, a, form, st), "product");
            g_products += form_products(ks, a, form);
            done = avail;
        }
    }
    g_kernel = form_name(form);
    return GF2E_OK;
}

int gf2e_mzed_mul_host(int e, uint32_t f, const uint64_t *A_h, int64_t lda, const uint64_t *B_h, int64_t ldb,
                       uint64_t *C_h, int64_t ldc, int64_t m, int64_t k, int64_t n, uint32_t flags,
                       int64_t chunk_rows, double *device_ms) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (device_ms) *device_ms = 0;
    if (int rc = check_field(e, f)) return rc;
    if (flags & ~(GF2E_ACCUMULATE | GF2E_B_DEVICE))
        return fail(GF2E_EINVAL, "gf2e_mzed_mul_host: unsupported flags 0x%x", flags);
    const bool b_dev = (flags & GF2E_B_DEVICE) != 0;  // B already in device memory (e.g. broadcast)
    const bool acc = (flags & GF2E_ACCUMULATE) != 0;
    const int w = gf2e_pack_width(e);
    const int64_t wa = words_for(k * w), wb = words_for(n * w), nwk = words_for(k), nwn = words_for(n);
    if (int rc = check_mat(A_h, m, wa, lda, "A")) return rc;
    if (int rc = check_mat(B_h, k, wb, ldb, "B")) return rc;
    if (int rc = check_mat(C_h, m, wb, ldc, "C")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (k == 0) {  // product is zero
        if (!acc)
            for (int64_t i = 0; i < m; ++i) memset(C_h + i * ldc, 0, (size_t)wb * 8);
        return GF2E_OK;
    }
    if (int rc = check_device()) return rc;
    if (int rc = ensure_fp4_checked()) return rc;
    Sched ks = to_kernel_sched(e, get_schedule(e, f));
    const int form = tc_form(0, k, ks.nprod);
    const int64_t tw = form_bn(form);  // column tile width: B parts and column splits align to it
    int64_t chunk = chunk_rows > 0 ? round_up(chunk_rows, 2 * kTcBM) : 2048;
    if (chunk > round_up(m, 2 * kTcBM)) chunk = round_up(m, 2 * kTcBM);
    constexpr int kMaxBParts = 16;
    // B arrives in column parts (multiples of 256 columns) so the first row chunk's products
    // start after the first part's upload instead of all of B's
    static const int bparts = std::min(std::max(env_int("GF2E_E2E_BPARTS", 8), 1), kMaxBParts);
    static const bool a_first = env_int("GF2E_E2E_AFIRST", 0) != 0;
    const int nbp = (n >= 8192 && m > chunk) ? bparts : 1;
    const std::vector<int64_t> rb = host_row_plan(m, n, k, chunk, nbp, chunk_rows > 0, tw);
    for (size_t i = 1; i < rb.size(); ++i)
        if (rb[i] - rb[i - 1] > chunk) chunk = rb[i] - rb[i - 1];  // slot size
    const int64_t nchunks = (int64_t)rb.size() - 1;
    const int nslots = nchunks > 1 ? 2 : 1;

    // Streams: sh host->device copies, sp operand preparation (slice + combinations of A and
    // B), sc products + cling, sd device->host copies.  Preparation runs beside the previous
    // product (on the SMs a partial last wave leaves idle) instead of between products.
    HostPlan P;
    CKH(cudaStreamCreateWithFlags(&P.sc, cudaStreamNonBlocking), "stream");
    CKH(cudaStreamCreateWithFlags(&P.sh, cudaStreamNonBlocking), "stream");
    CKH(cudaStreamCreateWithFlags(&P.sd, cudaStreamNonBlocking), "stream");
    CKH(cudaStreamCreateWithFlags(&P.sp, cudaStreamNonBlocking), "stream");
    Layout LB = layout_for(ks.nprod, chunk, k, n, 0, form);  // Ac sized for one chunk, Bt for all of B
    uint64_t *dBp, *dBs, *dBt, *dAc[2], *dAp[2], *dAs[2], *dCs[2], *dCp[2];
    int64_t ldbd = wb;  // row stride of the device copy of B
    if (b_dev) {
        dBp = const_cast<uint64_t *>(B_h);
        ldbd = ldb;
    } else {
        CKH(P.alloc(&dBp, k * wb * 8), "pool_alloc");
    }
    CKH(P.alloc(&dBs, (int64_t)e * k * nwn * 8), "pool_alloc");
    CKH(P.alloc(&dBt, LB.b_bytes), "pool_alloc");
    for (int sl = 0; sl < nslots; ++sl) {
        CKH(P.alloc(&dAc[sl], LB.a_bytes), "pool_alloc");
        CKH(P.alloc(&dAp[sl], chunk * wa * 8), "pool_alloc");
        CKH(P.alloc(&dAs[sl], (int64_t)e * chunk * nwk * 8), "pool_alloc");
        CKH(P.alloc(&dCs[sl], (int64_t)e * chunk * nwn * 8), "pool_alloc");
        CKH(P.alloc(&dCp[sl], chunk * wb * 8), "pool_alloc");
    }
    int64_t cb[kMaxBParts + 1];
    for (int p = 0; p <= nbp; ++p) cb[p] = p == nbp ? n : round_up(n * p / nbp, tw);
    // events: copies in (A chunk / B part), preparation done, products done (frees that
    // slot's A combinations), cling done, copy out done
    cudaEvent_t part_out, ev_alloc, ev_t0, ev_t1, in_ready[2], prep_a[2], prod_done[2], out_ready[2], d2h_done[2],
        ev_bp[kMaxBParts], prep_b[kMaxBParts];
    std::vector<cudaEvent_t *> all{&part_out, &ev_alloc, &ev_t0, &ev_t1};
    for (int sl = 0; sl < 2; ++sl)
        for (cudaEvent_t *ev : {&in_ready[sl], &prep_a[sl], &prod_done[sl], &out_ready[sl], &d2h_done[sl]})
            all.push_back(ev);
    for (int p = 0; p < kMaxBParts; ++p) {
        all.push_back(&ev_bp[p]);
        all.push_back(&prep_b[p]);
    }
    struct EvGuard {
        std::vector<cudaEvent_t *> evs;
        size_t made = 0;
        ~EvGuard() {
            for (size_t i = 0; i < made; ++i) cudaEventDestroy(*evs[i]);
        }
    } guard{all};
    for (cudaEvent_t *ev : all) {
        CKH(cudaEventCreateWithFlags(ev, cudaEventDefault), "cudaEventCreate");
        ++guard.made;
    }
    CKH(cudaEventRecord(ev_alloc, P.sc), "cudaEventRecord");
    for (cudaStream_t s2 : {P.sh, P.sd, P.sp}) CKH(cudaStreamWaitEvent(s2, ev_alloc, 0), "cudaStreamWaitEvent");

    CKH(cudaEventRecord(ev_t0, P.sh), "cudaEventRecord");
    Trace tr;
    tr.start(P.sh);
    auto h2d_bpart = [&](int p) -> int {
        const int64_t w0 = cb[p] * w / 64, w1 = p + 1 == nbp ? wb : cb[p + 1] * w / 64;
        if (!b_dev)
            CKH(cudaMemcpy2DAsync(dBp + w0, wb * 8, B_h + w0, ldb * 8, (w1 - w0) * 8, k, cudaMemcpyHostToDevice,
                                  P.sh),
                "H2D(B)");
        CKH(cudaEventRecord(ev_bp[p], P.sh), "cudaEventRecord");
        tr.mark(P.sh, "h2d B", p);
        return GF2E_OK;
    };
    auto h2d_chunk = [&](int64_t i) -> int {
        const int sl = (int)(i % nslots);
        const int64_t r0 = rb[i], rows = rb[i + 1] - rb[i];
        if (i >= nslots) {  // slot reuse: chunk i-2 fully consumed (its cling and its D2H)
            CKH(cudaStreamWaitEvent(P.sh, out_ready[sl], 0), "cudaStreamWaitEvent");
            CKH(cudaStreamWaitEvent(P.sh, d2h_done[sl], 0), "cudaStreamWaitEvent");
        }
        CKH(cudaMemcpy2DAsync(dAp[sl], wa * 8, A_h + r0 * lda, lda * 8, wa * 8, rows, cudaMemcpyHostToDevice, P.sh),
            "H2D(A)");
        if (acc)
            CKH(cudaMemcpy2DAsync(dCp[sl], wb * 8, C_h + r0 * ldc, ldc * 8, wb * 8, rows, cudaMemcpyHostToDevice,
                                  P.sh),
                "H2D(C0)");
        CKH(cudaEventRecord(in_ready[sl], P.sh), "cudaEventRecord");
        tr.mark(P.sh, "h2d A", i);
        return GF2E_OK;
    };
    const bool fp4 = form != kFormI8;
    // Preparation runs on its own stream, one chunk ahead, where the products bound the
    // pipeline (k >= 4096); at short k the copies do, and preparing in line on sc pipelines
    // them with the fewest cross-stream dependencies.
    const bool side = k >= 4096;
    cudaStream_t sp = side ? P.sp : P.sc;
    // chunk i's A: slice, row combinations into its slot's Ac (free once chunk i-2's products
    // are done)
    auto prep_chunk = [&](int64_t i) -> int {
        const int sl = (int)(i % nslots);
        const int64_t rows = rb[i + 1] - rb[i];
        CKH(cudaStreamWaitEvent(sp, in_ready[sl], 0), "cudaStreamWaitEvent");
        if (i >= nslots) CKH(cudaStreamWaitEvent(sp, prod_done[sl], 0), "cudaStreamWaitEvent");
        CK(launch_slice(e, w, rows, k, dAp[sl], wa, dAs[sl], nwk, rows * nwk, sp), "slice(A)");
        Layout L = layout_for(ks.nprod, rows, k, n, 0, form);
        CK(launch_combos_rows(ks, dAs[sl], nwk, rows * nwk, rows, k, dAc[sl], L.kwords, L.a_pstride, L.m_pad,
                              L.kwords, fp4 ? 4 : 2, sp),
           "combos(A)");
        CKH(cudaEventRecord(prep_a[sl], sp), "cudaEventRecord");
        tr.mark(sp, "prep A", i);
        return GF2E_OK;
    };
    // B part p: slice its columns, write its rows [cb[p], cb[p+1]) of the B^T combinations
    auto prep_bpart = [&](int p) -> int {
        CKH(cudaStreamWaitEvent(sp, ev_bp[p], 0), "cudaStreamWaitEvent");
        const int64_t c0 = cb[p], nc = cb[p + 1] - c0;
        const int64_t npad = (p + 1 == nbp ? LB.n_pad : cb[p + 1]) - c0;
        CK(launch_slice(e, w, k, nc, dBp + c0 * w / 64, ldbd, dBs + c0 / 64, nwn, k * nwn, sp, words_for(nc)),
           "slice(B)");
        CK(launch_combos_bt(ks, dBs + c0 / 64, nwn, k * nwn, k, nc, dBt + c0 * LB.kwords * form_bx(form), LB.kwords,
                            LB.b_pstride, LB.kwords, npad / 64, fp4, sp, form_br(form), 0, form_bexp(form)),
           "combos(B^T)");
        CKH(cudaEventRecord(prep_b[p], sp), "cudaEventRecord");
        tr.mark(sp, "prep B", p);
        return GF2E_OK;
    };
    // enqueue order (each event recorded before any wait on it): B part 0, chunk 0, the other
    // B parts; A's preparation one chunk ahead of the products
    if (!a_first)
        if (int rc = h2d_bpart(0)) return rc;
    if (int rc = h2d_chunk(0)) return rc;
    if (a_first)
        if (int rc = h2d_bpart(0)) return rc;
    for (int p = 1; p < nbp; ++p)
        if (int rc = h2d_bpart(p)) return rc;
    if (side) {
        if (int rc = prep_chunk(0)) return rc;
        for (int p = 0; p < nbp; ++p)
            if (int rc = prep_bpart(p)) return rc;
    }
    for (int64_t i = 0; i < nchunks; ++i) {
        const int sl = (int)(i % nslots);
        const int64_t r0 = rb[i], rows = rb[i + 1] - rb[i];
        if (i + 1 < nchunks)
            if (int rc = h2d_chunk(i + 1)) return rc;  // overlaps this chunk's kernels
        if (side && i + 1 < nchunks)
            if (int rc = prep_chunk(i + 1)) return rc;
        if (!side)
            if (int rc = prep_chunk(i)) return rc;
        CKH(cudaStreamWaitEvent(P.sc, prep_a[sl], 0), "cudaStreamWaitEvent");
        if (acc) {
            CKH(cudaStreamWaitEvent(P.sc, in_ready[sl], 0), "cudaStreamWaitEvent");
            CK(launch_slice(e, w, rows, n, dCp[sl], wb, dCs[sl], nwn, rows * nwn, P.sc), "slice(C0)");
        }
        Layout L = layout_for(ks.nprod, rows, k, n, 0, form);
        // the first chunk runs one product per B part as the parts arrive; later chunks see all of
        // B.  The last chunk runs as two column parts, the first sized to whole waves of CTA
        // pairs, so its cling and copy-out overlap the second part's product.
        const bool last = i + 1 == nchunks && i > 0;
        const int64_t cs = last && side ? last_split_cols(rows, n, tw) : n;
        const int nprods = i == 0 ? nbp : (cs < n ? 2 : 1);
        for (int p = 0; p < nprods; ++p) {
            const int64_t c0 = i == 0 ? cb[p] : (p ? cs : 0), c1 = i == 0 ? cb[p + 1] : (p || cs == n ? n : cs);
            const int64_t npad = (c1 == n ? LB.n_pad : c1) - c0;
            if (i == 0 && !side)
                if (int rc = prep_bpart(p)) return rc;
            if (i == 0) CKH(cudaStreamWaitEvent(P.sc, prep_b[p], 0), "cudaStreamWaitEvent");
            TcArgs ta{dAc[sl], dBt + c0 * LB.kwords * form_bx(form), L.a_pstride, LB.b_pstride, L.kwords, rows, c1 - c0,
                      L.m_pad, npad,
                      dCs[sl] + c0 / 64, nwn, rows * nwn, acc ? 1 : 0};
            ProfScope prof(P.sc);
            CK(launch_form(ks, ta, form, P.sc), "product");
            g_products += form_products(ks, ta, form);
            tr.mark(P.sc, "product", i, p);
            if (last && p == 0 && cs < n) {  // first column part out while the second computes
                const int64_t cw = cs * w / 64;
                CK(launch_cling(e, w, rows, cs, dCs[sl], nwn, rows * nwn, dCp[sl], wb, P.sc), "cling(C)");
                CKH(cudaEventRecord(part_out, P.sc), "cudaEventRecord");
                CKH(cudaStreamWaitEvent(P.sd, part_out, 0), "cudaStreamWaitEvent");
                CKH(cudaMemcpy2DAsync(C_h + r0 * ldc, ldc * 8, dCp[sl], wb * 8, cw * 8, rows, cudaMemcpyDeviceToHost,
                                      P.sd),
                    "D2H(C)");
            }
        }
        CKH(cudaEventRecord(prod_done[sl], P.sc), "cudaEventRecord");
        const int64_t cx = cs < n ? cs : 0, cwx = cx * w / 64;  // columns not yet copied out
        CK(launch_cling(e, w, rows, n - cx, dCs[sl] + cx / 64, nwn, rows * nwn, dCp[sl] + cwx, wb, P.sc),
           "cling(C)");
        CKH(cudaEventRecord(out_ready[sl], P.sc), "cudaEventRecord");
        tr.mark(P.sc, "cling", i);
        CKH(cudaStreamWaitEvent(P.sd, out_ready[sl], 0), "cudaStreamWaitEvent");
        CKH(cudaMemcpy2DAsync(C_h + r0 * ldc + cwx, ldc * 8, dCp[sl] + cwx, wb * 8, (wb - cwx) * 8, rows,
                              cudaMemcpyDeviceToHost, P.sd),
            "D2H(C)");
        CKH(cudaEventRecord(d2h_done[sl], P.sd), "cudaEventRecord");
        tr.mark(P.sd, "d2h C", i);
    }
    CKH(cudaStreamWaitEvent(P.sh, d2h_done[(nchunks - 1) % nslots], 0), "cudaStreamWaitEvent");
    CKH(cudaEventRecord(ev_t1, P.sh), "cudaEventRecord");
    CKH(cudaEventSynchronize(ev_t1), "cudaEventSynchronize");
    float ms = 0;
    CKH(cudaEventElapsedTime(&ms, ev_t0, ev_t1), "cudaEventElapsedTime");
    if (device_ms) *device_ms = ms;
    g_kernel = form_name(form);
    return GF2E_OK;
}

int64_t gf2e_trsm_workspace(int e, uint32_t f, int64_t m, int64_t n) {
    g_err.clear();
    if (check_field(e, f)) return -1;
    if (m < 0 || n < 0) return fail(GF2E_EINVAL, "matrix dimensions must be non-negative"), -1;
    if (m == 0 || n == 0) return 0;
    return trsm_layout((int)get_schedule(e, f).subsets.size(), e, m, n).total;
}

int gf2e_trsm(int e, uint32_t f, int upper, int unit_diag, const uint64_t *T, int64_t ldt, int64_t pt, uint64_t *B,
              int64_t ldb, int64_t pb, int64_t m, int64_t n, void *ws, int64_t ws_bytes, void *stream,
              int64_t *bad_row) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    return trsm_impl(e, f, upper, unit_diag, T, ldt, pt, B, ldb, pb, m, n, ws, ws_bytes, stream, bad_row, true);
}
}  // extern "C"

namespace {
int trsm_impl(int e, uint32_t f, int upper, int unit_diag, const uint64_t *T, int64_t ldt, int64_t pt, uint64_t *B,
              int64_t ldb, int64_t pb, int64_t m, int64_t n, void *ws, int64_t ws_bytes, void *stream,
              int64_t *bad_row, bool check) {
    if (bad_row) *bad_row = -1;
    if (int rc = check_field(e, f)) return rc;
    if (unit_diag && upper) return fail(GF2E_EINVAL, "unit_diag is only defined for lower triangular solves");
    if (int rc = check_mat(T, m, words_for(m), ldt, "T")) return rc;
    if (int rc = check_mat(B, m, words_for(n), ldb, "B")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    const Schedule &S = get_schedule(e, f);
    TrsmLayout L = trsm_layout((int)S.subsets.size(), e, m, n);
    if (ws_bytes < L.total)
        return fail(GF2E_ENOMEM, "workspace too small: %lld < %lld bytes", (long long)ws_bytes, (long long)L.total);
    if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255))
        return fail(GF2E_EINVAL, "workspace must be a 256-byte aligned device pointer");
    cudaStream_t st = (cudaStream_t)stream;
    char *w = static_cast<char *>(ws);
    uint64_t *inv = reinterpret_cast<uint64_t *>(w);
    uint64_t *tmp = reinterpret_cast<uint64_t *>(w + L.inv_bytes);
    int *flag = reinterpret_cast<int *>(w + L.inv_bytes + L.tmp_bytes);
    void *mulws = w + L.inv_bytes + L.tmp_bytes + 256;
    const int big = 0x7fffffff;
    CKH(cudaMemcpyAsync(flag, &big, sizeof(int), cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CK(launch_tri_inverse(e, f, primitive_element(e, f), T, ldt, pt, m, upper != 0, unit_diag != 0, inv, flag,
                          trsm_block(e, m, n), st),
       "tri_inverse");
    int bad = big;
    if (check) {  // PLE corners skip this: their diagonal is the (nonzero) pivots
        CKH(cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
        CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    }
    if (bad != big) {
        if (bad_row) *bad_row = bad;
        return fail(GF2E_ESINGULAR, "zero diagonal entry at index %d", bad);
    }
    TrsmCtx c{to_kernel_sched(e, S), upper != 0, T, ldt, pt, B, ldb, pb, n, inv, tmp, mulws, L.mul_bytes, e, st,
              trsm_block(e, m, n), field_tab(e, f, primitive_element(e, f))};
    return trsm_rec(c, 0, m);
}
}  // namespace

extern "C" {

int gf2e_mul_by_x(int e, uint32_t f, const uint64_t *in, int64_t ld, int64_t pin, uint64_t *out, int64_t pout,
                  int64_t rows, int64_t cols, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_mat(in, rows, words_for(cols), ld, "in")) return rc;
    if (int rc = check_mat(out, rows, words_for(cols), ld, "out")) return rc;
    if (rows == 0 || cols == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_mul_by_x(e, f, in, ld, pin, out, pout, rows, words_for(cols), (cudaStream_t)stream), "mul_by_x");
    return GF2E_OK;
}

int gf2e_scalar_mul(int e, uint32_t f, uint32_t c, const uint64_t *in, int64_t ldi, uint64_t *out, int64_t ldo,
                    int64_t rows, int64_t cols, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    if (c >= (1u << e)) return fail(GF2E_EINVAL, "scalar %u out of range for GF(2^%d)", c, e);
    const int w = gf2e_pack_width(e);
    if (int rc = check_mat(in, rows, words_for(cols * w), ldi, "in")) return rc;
    if (int rc = check_mat(out, rows, words_for(cols * w), ldo, "out")) return rc;
    if (rows == 0 || cols == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    CK(launch_scalar_mul(e, f, c, w, in, ldi, out, ldo, rows, words_for(cols * w), (cudaStream_t)stream),
       "scalar_mul");
    return GF2E_OK;
}

int gf2e_plane_mul(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, uint64_t *C, int64_t ldc, int64_t m,
                   int64_t k, int64_t n, uint32_t flags, void *ws, int64_t ws_bytes, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_flags(flags)) return rc;
    if (int rc = check_mat(A, m, words_for(k), lda, "A")) return rc;
    if (int rc = check_mat(B, k, words_for(n), ldb, "B")) return rc;
    if (int rc = check_mat(C, m, words_for(n), ldc, "C")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    return run_product(plane_sched(), A, lda, 0, B, ldb, 0, C, ldc, 0, m, k, n, flags, ws, ws_bytes,
                       (cudaStream_t)stream);
}


int gf2e_ple(int e, uint32_t f, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t n, int64_t *P, int64_t *Q,
             int64_t *rank, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (rank) *rank = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_mat(S, m, words_for(n), ld, "A")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    return ple_top(e, f, S, ld, ps, m, n, P, Q, rank, (cudaStream_t)stream);
}

int gf2e_echelonize(int e, uint32_t f, uint64_t *S, int64_t ld, int64_t ps, int64_t m, int64_t n, int full,
                    int64_t *rank, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (rank) *rank = 0;
    if (int rc = check_field(e, f)) return rc;
    if (int rc = check_mat(S, m, words_for(n), ld, "A")) return rc;
    if (m == 0 || n == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t k = m < n ? m : n;
    std::vector<int64_t> P(k), Q(k);
    int64_t r = 0;
    if (int rc = ple_top(e, f, S, ld, ps, m, n, P.data(), Q.data(), &r, st)) return rc;
    if (rank) *rank = r;
    if (r == 0) return GF2E_OK;
    DevTmp ix((size_t)(3 * r + 3) * 8, st);
    if (!ix.p) return fail(GF2E_ENOMEM, "out of device memory (echelonize scratch)");
    int64_t *idx = static_cast<int64_t *>(ix.p);
    std::vector<int64_t> tr;  // undo the L compression (ple_echelon.py:359-362)
    for (int64_t t = r - 1; t >= 0; --t)
        if (Q[t] != t) tr.insert(tr.end(), {t, Q[t], t});
    if (!tr.empty()) {
        CKH(cudaMemcpyAsync(idx, tr.data(), tr.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
        CK(launch_col_swaps(e, 1, S, ld, ps, m, idx, (int)(tr.size() / 3), st), "col_swaps");
        CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    }
    CKH(cudaMemcpyAsync(idx, Q.data(), r * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    // per column word: its pivots in increasing t and the prefix ORs of their bits
    const int64_t nw = words_for(n);
    std::vector<std::vector<int>> per(nw);
    for (int64_t t = 0; t < r; ++t) per[Q[t] >> 6].push_back((int)t);
    std::vector<int> wstart(nw + 1), tpos;
    std::vector<uint64_t> pmask;
    tpos.reserve(r);
    pmask.reserve(r);
    for (int64_t w = 0; w < nw; ++w) {
        wstart[w] = (int)tpos.size();
        uint64_t acc = 0;
        for (int t : per[w]) {
            acc |= 1ULL << (Q[t] & 63);
            tpos.push_back(t);
            pmask.push_back(acc);
        }
    }
    wstart[nw] = (int)tpos.size();
    const size_t mk_bytes = align256((nw + 1) * 4) + align256(r * 4) + (size_t)r * 8;
    DevTmp mk(mk_bytes, st);
    if (!mk.p) return fail(GF2E_ENOMEM, "out of device memory (echelonize marks)");
    int *d_ws = static_cast<int *>(mk.p);
    int *d_tp = reinterpret_cast<int *>(static_cast<char *>(mk.p) + align256((nw + 1) * 4));
    uint64_t *d_pm = reinterpret_cast<uint64_t *>(static_cast<char *>(mk.p) + align256((nw + 1) * 4) + align256(r * 4));
    CKH(cudaMemcpyAsync(d_ws, wstart.data(), (nw + 1) * 4, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CKH(cudaMemcpyAsync(d_tp, tpos.data(), r * 4, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CKH(cudaMemcpyAsync(d_pm, pmask.data(), r * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CK(launch_echelon_marks(e, S, ld, ps, m, nw, idx, (int)r, d_ws, d_tp, d_pm, st), "echelon_marks");  // (:364-370)
    if (full) {  // rows[:r] = upper^-1 rows[:r], upper = pivot columns (:371-375)
        const int64_t lw = words_for(r);
        DevTmp ut((size_t)e * r * lw * 8, st);
        if (!ut.p) return fail(GF2E_ENOMEM, "out of device memory (echelonize corner)");
        uint64_t *U = static_cast<uint64_t *>(ut.p);
        bool ident = true;  // pivot columns 0 .. r-1 (a generic matrix): the gather is a copy
        for (int64_t t = 0; t < r && ident; ++t) ident = Q[t] == t;
        if (ident) {
            for (int b = 0; b < e; ++b)
                CKH(cudaMemcpy2DAsync(U + b * r * lw, lw * 8, S + b * ps, ld * 8, lw * 8, r, cudaMemcpyDeviceToDevice,
                                      st),
                    "cudaMemcpy2DAsync");
        } else {
            CK(launch_gather_cols(e, S, ld, ps, idx, r, U, lw, r * lw, st), "gather_cols");
        }
        const int64_t tws = gf2e_trsm_workspace(e, f, r, n);
        DevTmp tw((size_t)(tws > 0 ? tws : 256), st);
        if (!tw.p) return fail(GF2E_ENOMEM, "out of device memory (echelonize trsm workspace)");
        int64_t bad = -1;
        if (int rc = trsm_impl(e, f, 1, 0, U, lw, r * lw, S, ld, ps, r, n, tw.p, tws, st, &bad, true)) return rc;
    }
    CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return GF2E_OK;
}

int gf2e_row_swaps(int planes, uint64_t *S, int64_t ld, int64_t ps, int64_t rows, int64_t nwords,
                   const int64_t *swaps, int64_t n, int backward, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (planes < 1 || n < 0 || n > rows) return fail(GF2E_EINVAL, "bad swap vector arguments");
    if (int rc = check_mat(S, rows, nwords, ld, "A")) return rc;
    for (int64_t i = 0; i < n; ++i)
        if (swaps[i] < i || swaps[i] >= rows)
            return fail(GF2E_EINVAL, "swap target %lld at index %lld invalid for %lld rows", (long long)swaps[i],
                        (long long)i, (long long)rows);
    std::vector<int64_t> pr = swap_pairs(swaps, n);
    if (pr.empty() || nwords == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    DevTmp ix(pr.size() * 8, st);
    if (!ix.p) return fail(GF2E_ENOMEM, "out of device memory");
    CKH(cudaMemcpyAsync(ix.p, pr.data(), pr.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CK(launch_row_swaps(planes, S, ld, ps, nwords, static_cast<int64_t *>(ix.p), (int)(pr.size() / 2), backward != 0,
                        st),
       "row_swaps");
    CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return GF2E_OK;
}

int gf2e_col_swaps(int planes, int w, uint64_t *S, int64_t ld, int64_t ps, int64_t rows, int64_t cols,
                   const int64_t *triples, int64_t n, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (planes < 1 || n < 0 || (w != 1 && w != 2 && w != 4 && w != 8 && w != 16))
        return fail(GF2E_EINVAL, "bad column swap arguments");
    if (int rc = check_mat(S, rows, words_for(cols * w), ld, "A")) return rc;
    for (int64_t i = 0; i < n; ++i)
        if (triples[3 * i] < 0 || triples[3 * i] >= cols || triples[3 * i + 1] < 0 || triples[3 * i + 1] >= cols ||
            triples[3 * i + 2] < 0)
            return fail(GF2E_EINVAL, "column swap %lld out of range for %lld columns", (long long)i, (long long)cols);
    if (n == 0 || rows == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    DevTmp ix((size_t)n * 24, st);
    if (!ix.p) return fail(GF2E_ENOMEM, "out of device memory");
    CKH(cudaMemcpyAsync(ix.p, triples, n * 24, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CK(launch_col_swaps(planes, w, S, ld, ps, rows, static_cast<int64_t *>(ix.p), (int)n, st), "col_swaps");
    CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return GF2E_OK;
}


int gf2e_row_scales(int e, uint32_t f, const uint64_t *in, int64_t ldi, int broadcast, const uint32_t *scalars,
                    uint64_t *out, int64_t ldo, int64_t rows, int64_t cols, void *stream) {
    g_err.clear();
    g_launches = 0;
    g_products = 0;
    if (int rc = check_field(e, f)) return rc;
    const int w = gf2e_pack_width(e);
    const int64_t nwords = words_for(cols * w);
    if (int rc = check_mat(in, broadcast ? 1 : rows, nwords, ldi, "in")) return rc;
    if (int rc = check_mat(out, rows, nwords, ldo, "out")) return rc;
    for (int64_t r = 0; r < rows; ++r)
        if (scalars[r] >> e) return fail(GF2E_EINVAL, "scalar %u out of range for GF(2^%d)", scalars[r], e);
    if (rows == 0 || nwords == 0) return GF2E_OK;
    if (int rc = check_device()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    DevTmp cs((size_t)rows * 4, st);
    if (!cs.p) return fail(GF2E_ENOMEM, "out of device memory");
    CKH(cudaMemcpyAsync(cs.p, scalars, rows * 4, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    CK(launch_row_scales(e, f, primitive_element(e, f), w, in, ldi, broadcast != 0, static_cast<uint32_t *>(cs.p), out,
                         ldo, rows, nwords, st),
       "row_scales");
    CKH(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return GF2E_OK;
}

}  // extern "C"

// frr_gen.cu -- candidate generation, CUDA-core balance checks, regeneration
// and the randomization-test kernels (sm_100a).
//
// Work mapping: one warp per candidate.  A candidate's assignment lives only
// in a per-warp shared-memory table (2 bytes per unit) and is consumed in
// place; nothing per candidate but its statistic reaches HBM.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "frr_common.cuh"
#include "frr_launch.cuh"
#include "frr_revfy.cuh"

// ------------------------------------------------ universal step table
namespace {
constexpr int kDescSteps = 65536 + 128;
struct DescSteps {
    StepC v[kDescSteps];
    constexpr DescSteps() : v() {
        for (int i = 0; i < kDescSteps; i++) {
            const uint32_t b = i < 65535 ? 65536u - (uint32_t)i : 1u;
            v[i].b = b;
            v[i].c2 = (uint32_t)((1ull << 32) % b);
            v[i].M = (~0ull) / b + 1ull;
        }
    }
};
__device__ const DescSteps g_frr_desc_steps = DescSteps();
}  // namespace

const StepC* frr_global_steps(int n) {
    static const StepC* cached[64] = {nullptr};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        void* p = nullptr;
        if (cudaGetSymbolAddress(&p, g_frr_desc_steps) != cudaSuccess) {
            frr_check_launch("cudaGetSymbolAddress(step table)");
            return nullptr;
        }
        cached[dev] = static_cast<const StepC*>(p);
    }
    return cached[dev] + (65536 - n);
}

namespace {

constexpr int kWarps = 8;  // warps per CTA of k_exact_small
constexpr int kThreads = kWarps * 32;
constexpr int kPlanWarps = 16;  // max warps per CTA of the warp-per-candidate kernels
constexpr int kPlanThreads = kPlanWarps * 32;

// Shared-memory plan of a warp-per-candidate kernel: the Fisher-Yates step
// table (shared, or global when t is too large), fixed per-CTA bytes, and a
// per-warp part (the candidate table + scratch).  Huge n gets fewer warps.
struct WarpPlan {
    int warps;
    bool gsteps;
    size_t smem;
};

// Picks (warps per CTA, step table placement) maximising resident warps per
// SM: a shared step table costs every CTA its bytes, a global one (L1
// cached) frees them for more candidate tables.
WarpPlan plan_warps(int t, bool needs_steps, size_t fixed, size_t per_warp) {
    const size_t cap = 227 * 1024 - 1024, sm_bytes = 228 * 1024;
    const size_t steps_b = needs_steps ? (size_t)frr_steps_len(t) * sizeof(StepC) : 0;
    WarpPlan best{0, false, 0};
    int best_res = 0;
    for (int g = 0; g < 2; g++) {
        const bool gsteps = g == 1;
        if (gsteps && !needs_steps) break;
        const size_t f = fixed + FRR_TABLE_SLACK + (gsteps ? 0 : steps_b);
        for (int w = 1; w <= kPlanWarps; w++) {
            const size_t smem = f + (size_t)w * per_warp;
            if (smem > cap) break;
            const int ctas = (int)std::min<size_t>(std::min<size_t>(sm_bytes / (smem + 1024), 64 / w), 32);
            if (ctas < 1) continue;
            // a shared step table saves a global (L1) load per draw: worth
            // ~25% fewer resident warps
            const int res = gsteps ? (ctas * w * 4) / 5 : ctas * w;
            if (res > best_res || (res == best_res && !gsteps && best.gsteps)) {
                best = {w, gsteps, smem};
                best_res = res;
            }
        }
    }
    return best;
}

// per-CTA steps pointer: shared copy (filled here) or the global table
template <bool GS>
__device__ __forceinline__ const StepC* cta_steps(unsigned char*& cursor, const StepC* gsteps, int n, int t, bool keys) {
    if (!keys) return nullptr;
    if (GS) return gsteps;
    StepC* s = reinterpret_cast<StepC*>(cursor);
    cursor += (size_t)frr_steps_len(t) * sizeof(StepC);
    frr_fill_steps(s, n, t);
    return s;
}

enum Source { SRC_KEYS = 0, SRC_RANKS = 1, SRC_ROWS = 2 };

// Build the candidate table for source SRC.
template <int SRC, bool GS = false>
__device__ __forceinline__ void build_table(uint64_t seed, const uint64_t* ids, const int8_t* rows,
                                            int64_t c, int n, int t, const StepC* steps, uint16_t* lw,
                                            int lane) {
    if (SRC == SRC_KEYS) {
        frr_warp_fy<GS>(frr_derive_state(seed, ids[c]), n, t, steps, lw, lane);
    } else if (SRC == SRC_RANKS) {
        frr_table_fill(lw, n, FRR_CTL, lane);
        __syncwarp();
        if (lane == 0) frr_unrank_to_table(ids[c], n, t, lw);
        __syncwarp();
    } else {
        const int8_t* row = rows + (size_t)c * n;
        for (int e = lane; e < n; e += 32) lw[e] = row[e] ? (uint16_t)0 : (uint16_t)FRR_CTL;
        __syncwarp();
    }
}

// Bit i of word w = unit 32w+i is treated (its entry is not FRR_CTL; every
// other entry value is < 2^15, so "treated" is bit 15 clear).  Four 16-byte
// loads per word; units >= n (table padding) read as 0.
__device__ __forceinline__ uint32_t table_word(const uint16_t* lw, int n, int w) {
    const uint4* src = reinterpret_cast<const uint4*>(lw + 32 * w);
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint4 v = src[c];
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t nb = ~x[j];  // bit 15: unit 2k treated, bit 31: unit 2k+1 treated
            const int k = 4 * c + j;
            word |= ((nb >> 15) & 1u) << (2 * k);
            word |= (nb >> 31) << (2 * k + 1);
        }
    }
    const int valid = n - 32 * w;
    return valid >= 32 ? word : word & ((1u << valid) - 1u);
}

// ------------------------------------------------------------- regeneration
template <int SRC, bool GS>
__global__ void __launch_bounds__(kPlanThreads) k_regen(uint64_t seed, const uint64_t* ids, int64_t m, int n,
                                                    int t, int8_t* rows, uint32_t* bits, const StepC* gsteps) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char* cursor = smem;
    const StepC* steps = cta_steps<GS>(cursor, gsteps, n, t, SRC == SRC_KEYS);
    uint16_t* tables = reinterpret_cast<uint16_t*>(cursor);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint16_t* lw = tables + (size_t)warp * frr_table_len(n);
    __syncthreads();
    const int words = (n + 31) >> 5;
    for (int64_t c = (int64_t)blockIdx.x * nw + warp; c < m; c += (int64_t)gridDim.x * nw) {
        build_table<SRC, GS>(seed, ids, nullptr, c, n, t, steps, lw, lane);
        if (rows) {
            int8_t* out = rows + (size_t)c * n;
            if ((n & 7) == 0) {
                for (int e = lane * 8; e < n; e += 256) {
                    uint32_t lo = 0, hi = 0;
#pragma unroll
                    for (int i = 0; i < 4; i++) lo |= (uint32_t)(lw[e + i] != FRR_CTL) << (8 * i);
#pragma unroll
                    for (int i = 0; i < 4; i++) hi |= (uint32_t)(lw[e + 4 + i] != FRR_CTL) << (8 * i);
                    *reinterpret_cast<uint2*>(out + e) = make_uint2(lo, hi);
                }
            } else {
                for (int e = lane; e < n; e += 32) out[e] = lw[e] != FRR_CTL;
            }
        }
        if (bits) {
            uint32_t* ob = bits + (size_t)c * words;
            for (int w = lane; w < words; w += 32) ob[w] = table_word(lw, n, w);
        }
        __syncwarp();
    }
}

// -------------------------------------------------------- small-d epilogue
// balance.py:96-104 for d <= D: delta = fl(fl(S*g) - cc); q = delta^2;
// numpy pairwise sum over the d values; times const.
template <int D>
__device__ __forceinline__ double small_stat(const int64_t (&S)[D], int d, double g, const double* cc,
                                             double cst) {
    double q[D];
#pragma unroll
    for (int j = 0; j < D; j++) {
        if (j < d) {
            double delta = __dsub_rn(__dmul_rn(__ll2double_rn(S[j]), g), cc[j]);
            q[j] = __dmul_rn(delta, delta);
        } else {
            q[j] = 0.0;
        }
    }
    double res;
    if (d < 8) {
        res = -0.0;
#pragma unroll
        for (int j = 0; j < D; j++)
            if (j < d) res = __dadd_rn(res, q[j]);
    } else {
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; k++) r[k] = q[k < D ? k : 0];
        int full = d - (d % 8);
        if (D >= 16 && full >= 16) {
#pragma unroll
            for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], q[(8 + k) < D ? 8 + k : 0]);
        }
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
        for (int j = 8; j < D; j++)
            if (j >= full && j < d) res = __dadd_rn(res, q[j]);
    }
    return __dmul_rn(__dadd_rn(0.0, res), cst);
}

template <int D>
__device__ __forceinline__ void warp_sum(int64_t (&a)[D]) {
#pragma unroll
    for (int j = 0; j < D; j++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a[j] += __shfl_xor_sync(FRR_FULL, a[j], o);
    }
}

// ------------------------------------------------ small-d balance (d <= 16)
// S = colsum - sum over control units of Zq rows (exact int64), warp
// reduction, then the fp64 epilogue on lane 0.
template <int SRC, int D, bool GS>
__global__ void __launch_bounds__(kPlanThreads) k_stats_small(frr_balance_t bal, uint64_t seed, const uint64_t* ids,
                                                          const int8_t* rows, uint64_t lo, int64_t count,
                                                          double* out, const StepC* gsteps) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = bal.n, t = bal.t, d = bal.d;
    unsigned char* cursor = smem;
    const StepC* steps = cta_steps<GS>(cursor, gsteps, n, t, SRC == SRC_KEYS);
    uint16_t* tables = reinterpret_cast<uint16_t*>(cursor);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint16_t* lw = tables + (size_t)warp * frr_table_len(n);
    __syncthreads();
    const int64_t* __restrict__ zq = bal.zq;
    for (int64_t c = (int64_t)blockIdx.x * nw + warp; c < count; c += (int64_t)gridDim.x * nw) {
        if (SRC == SRC_KEYS) {
            frr_warp_fy<GS>(frr_derive_state(seed, lo + (uint64_t)c), n, t, steps, lw, lane);
        } else {
            build_table<SRC, GS>(seed, ids, rows, c, n, t, steps, lw, lane);
        }
        int64_t acc[D];
#pragma unroll
        for (int j = 0; j < D; j++) acc[j] = 0;
        for (int e = lane; e < n; e += 32) {
            if (lw[e] == FRR_CTL) {
                const int64_t* z = zq + (size_t)e * d;
#pragma unroll
                for (int j = 0; j < D; j++)
                    if (j < d) acc[j] += __ldg(reinterpret_cast<const long long*>(z) + j);
            }
        }
        warp_sum<D>(acc);
        if (lane == 0) {
            int64_t S[D];
#pragma unroll
            for (int j = 0; j < D; j++) S[j] = j < d ? bal.colsum[j] - acc[j] : 0;
            out[c] = small_stat<D>(S, d, bal.g, bal.cc, bal.cst);
        }
        __syncwarp();
    }
}

// --------------------------------------------- generic balance (any d)
// Lanes own columns j; S_j = colsum_j - sum_{control e} Zq[e][j]; q_j to a
// per-warp scratch; lane 0 runs the exact numpy pairwise sum.
template <int SRC, bool GS>
__global__ void __launch_bounds__(kPlanThreads) k_stats_generic(frr_balance_t bal, uint64_t seed, const uint64_t* ids,
                                                            const int8_t* rows, uint64_t lo, int64_t count,
                                                            double* out, const StepC* gsteps) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = bal.n, t = bal.t, d = bal.d;
    unsigned char* cursor = smem;
    const StepC* steps = cta_steps<GS>(cursor, gsteps, n, t, SRC == SRC_KEYS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* scratch = reinterpret_cast<double*>(cursor);
    // candidate tables start 16-byte aligned (uint4 fills) for any nw * d
    uint16_t* tables = reinterpret_cast<uint16_t*>(scratch + (((size_t)nw * d + 1) & ~(size_t)1));
    uint16_t* lw = tables + (size_t)warp * frr_table_len(n);
    double* q = scratch + (size_t)warp * d;
    __syncthreads();
    for (int64_t c = (int64_t)blockIdx.x * nw + warp; c < count; c += (int64_t)gridDim.x * nw) {
        if (SRC == SRC_KEYS) {
            frr_warp_fy<GS>(frr_derive_state(seed, lo + (uint64_t)c), n, t, steps, lw, lane);
        } else {
            build_table<SRC, GS>(seed, ids, rows, c, n, t, steps, lw, lane);
        }
        for (int j = lane; j < d; j += 32) {
            int64_t acc = 0;
            for (int e = 0; e < n; e++)
                if (lw[e] == FRR_CTL) acc += bal.zq[(size_t)e * d + j];
            int64_t S = bal.colsum[j] - acc;
            double delta = __dsub_rn(__dmul_rn(__ll2double_rn(S), bal.g), bal.cc[j]);
            q[j] = __dmul_rn(delta, delta);
        }
        __syncwarp();
        if (lane == 0) out[c] = __dmul_rn(frr_pw_sum(q, d), bal.cst);
        __syncwarp();
    }
}

// --------------------------------------------- exact enumeration (n <= 64)
// One lane walks a run of 32 consecutive lexicographic ranks: unrank once,
// then the complement-Gosper successor (unit i <-> bit n-1-i, lex order ==
// decreasing mask) with an incremental exact S.  Results are transposed
// through shared memory for coalesced stores.
#ifndef FRR_KRUN
#define FRR_KRUN 32
#endif
constexpr int kRun = FRR_KRUN;

template <int D>
__global__ void __launch_bounds__(kThreads) k_exact_small(frr_balance_t bal, uint64_t rank_lo, int64_t count,
                                                          double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = bal.n, t = bal.t, d = bal.d;
    const int nb = n + 1;                                             // binomial rows/cols 0..n
    uint64_t* binom = reinterpret_cast<uint64_t*>(smem);              // [n+1][n+1]
    int64_t* zq = reinterpret_cast<int64_t*>(binom + nb * nb);       // [n][D]
    double* stage = reinterpret_cast<double*>(zq + (size_t)n * D);   // [kWarps][32][kRun + 1]
    for (int i = threadIdx.x; i < nb * nb; i += blockDim.x) binom[i] = frr_binom(i / nb, i % nb);
    for (int i = threadIdx.x; i < n * D; i += blockDim.x) {
        int e = i / D, j = i % D;
        zq[i] = j < d ? bal.zq[(size_t)e * d + j] : 0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* st = stage + (size_t)warp * 32 * (kRun + 1);
    const uint64_t fullmask = n == 64 ? ~0ull : ((1ull << n) - 1ull);
    const int64_t per_warp = 32 * kRun;
    for (int64_t wb = ((int64_t)blockIdx.x * kWarps + warp) * per_warp; wb < count;
         wb += (int64_t)gridDim.x * kWarps * per_warp) {
        int64_t r0 = wb + (int64_t)lane * kRun;
        int64_t left = count - r0;
        int nrun = left < kRun ? (int)left : kRun;
        if (nrun > 0) {
            // unrank rank_lo + r0 into mask (unit i <-> bit n-1-i)
            uint64_t rank = rank_lo + (uint64_t)r0;
            uint64_t m = 0;
            int x = 0;
            for (int i = 0; i < t; i++) {
                for (;;) {
                    uint64_t cnk = binom[(n - x - 1) * nb + (t - i - 1)];
                    if (rank < cnk) break;
                    rank -= cnk;
                    x++;
                }
                m |= 1ull << (n - 1 - x);
                x++;
            }
            int64_t S[D];
#pragma unroll
            for (int j = 0; j < D; j++) S[j] = 0;
            uint64_t mm = m;
            while (mm) {
                int b = __ffsll((long long)mm) - 1;
                const int64_t* z = zq + (size_t)(n - 1 - b) * D;
#pragma unroll
                for (int j = 0; j < D; j++) S[j] += z[j];
                mm &= mm - 1;
            }
            for (int r = 0; r < nrun; r++) {
                st[lane * (kRun + 1) + r] = small_stat<D>(S, d, bal.g, bal.cc, bal.cst);
                if (r + 1 < nrun) {
                    uint64_t xc = ~m & fullmask;
                    uint64_t cbit = xc & (0ull - xc);
                    uint64_t rr = xc + cbit;
                    uint64_t xn = (((rr ^ xc) >> 2) >> (__ffsll((long long)cbit) - 1)) | rr;
                    uint64_t mn = ~xn & fullmask;
                    // the successor keeps the popcount: units leave and enter in
                    // pairs, one (enter, leave) pair per iteration (no divergent
                    // add/subtract paths)
                    uint64_t add = mn & ~m, rem = m & ~mn;
                    while (add) {
                        const int ba = __ffsll((long long)add) - 1, br = __ffsll((long long)rem) - 1;
                        const int64_t* za = zq + (size_t)(n - 1 - ba) * D;
                        const int64_t* zr = zq + (size_t)(n - 1 - br) * D;
#pragma unroll
                        for (int j = 0; j < D; j++) S[j] += za[j] - zr[j];
                        add &= add - 1;
                        rem &= rem - 1;
                    }
                    m = mn;
                }
            }
        }
        __syncwarp();
        for (int k = 0; k < kRun; k++) {  // coalesced: the warp's 32 * kRun statistics in rank order
            int64_t idx = wb + (int64_t)k * 32 + lane;
            if (idx < count) out[idx] = st[(k * 32 + lane) / kRun * (kRun + 1) + (k * 32 + lane) % kRun];
        }
        __syncwarp();
    }
}

// ------------------------------------------- exact: split enumeration
// itertools.combinations order split at na = n/2: a combination is (a, b)
// with a = its units < na and b = its units >= na, and all combinations
// sharing a are one contiguous run of ranks in which b runs through the
// |b|-subsets of the upper units in lexicographic order.  The host plan
// (generation.py, _split_plan) lists those blocks in rank order (base rank,
// a, offset of the |b|-subset list), so a rank is (block, offset) and its
// exact S is SA[a] + SB[b] from two subset-sum tables: two table loads and
// D integer adds per candidate, no divergent successor walk.
template <int D>
__global__ void __launch_bounds__(256) k_subset_sums(const int64_t* __restrict__ zq, int n, int d, int na,
                                                     const int32_t* __restrict__ lb, int64_t* __restrict__ sa,
                                                     int64_t* __restrict__ sb) {
    const int nb = n - na;
    const int64_t ta = 1ll << na, tot = ta + (1ll << nb);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const bool isa = i < ta;
        // SA by lower-half mask; SB row j = the upper-half subset lb[j] (the
        // lexicographic subset lists), so a block's ranks read SB rows in order
        const int64_t m = isa ? i : (int64_t)lb[i - ta];
        int64_t* dst = (isa ? sa + i * D : sb + (i - ta) * D);
        const int off = isa ? 0 : na, nbits = isa ? na : nb;
        int64_t S[D];
#pragma unroll
        for (int u = 0; u < D; u++) S[u] = 0;
        for (int j = 0; j < nbits; j++)
            if ((m >> j) & 1) {
#pragma unroll
                for (int u = 0; u < D; u++)
                    if (u < d) S[u] += zq[(size_t)(off + j) * d + u];
            }
#pragma unroll
        for (int u = 0; u < D; u++) dst[u] = S[u];
    }
}

// FILT: instead of writing every statistic, append (rank, stat) of the
// statistics whose bits are <= hbits (statistics are >= +0, so bit order is
// value order) to fidx/fval (unordered; warp-aggregated atomic on fcount,
// entries past cap counted but not written).  The caller sorts by rank.
template <int D, bool FILT>
__global__ void __launch_bounds__(256) k_exact_split(frr_balance_t bal, const int64_t* __restrict__ sa,
                                                     const int64_t* __restrict__ sb, const int32_t* __restrict__ blk_a,
                                                     const int64_t* __restrict__ blk_off,
                                                     const int64_t* __restrict__ blk_base, int64_t nblk,
                                                     uint64_t rank_lo, int64_t count, double* __restrict__ out,
                                                     uint64_t hbits, int64_t cap, int64_t* __restrict__ fidx,
                                                     double* __restrict__ fval,
                                                     unsigned long long* __restrict__ fcount, int64_t stride) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t chunk = (count + nwarps - 1) / nwarps;
    chunk = (chunk + 31) & ~(int64_t)31;
    const int64_t c0 = warp * chunk;
    if (c0 >= count) return;
    const int64_t c1 = min(count, c0 + chunk);
    // block of the warp's first rank (last base <= rank), then per lane
    int64_t b = 0;
    if (lane == 0) {
        const int64_t r = (int64_t)(rank_lo + (uint64_t)c0 * (uint64_t)stride);
        int64_t lo = 0, hi = nblk - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (blk_base[mid] <= r) lo = mid;
            else hi = mid - 1;
        }
        b = lo;
    }
    b = __shfl_sync(FRR_FULL, b, 0);
    int64_t base = -1, next = -1, loff = 0;
    int64_t A[D];
    // uniform trip count over the warp (ballot in the filtered variant)
    for (int64_t cb = c0; cb < c1; cb += 32) {
        const int64_t c = cb + lane;
        const bool valid = c < c1;
        const int64_t r = (int64_t)(rank_lo + (uint64_t)c * (uint64_t)stride);
        double st = 0.0;
        if (valid) {
            if (r >= next) {
                if (stride > 1) {  // sampled ranks: each one may be many blocks further
                    int64_t lo = b, hi = nblk - 1;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi + 1) >> 1;
                        if (blk_base[mid] <= r) lo = mid;
                        else hi = mid - 1;
                    }
                    b = lo;
                }
                while (b + 1 < nblk && blk_base[b + 1] <= r) b++;
                base = blk_base[b];
                next = b + 1 < nblk ? blk_base[b + 1] : INT64_MAX;
                loff = blk_off[b];
                const int64_t* ar = sa + (int64_t)blk_a[b] * D;
#pragma unroll
                for (int u = 0; u < D; u++) A[u] = ar[u];
            }
            // consecutive ranks: consecutive rows (D * 8 bytes, a multiple of 16)
            const longlong2* br = reinterpret_cast<const longlong2*>(sb + (loff + (r - base)) * D);
            int64_t S[D];
#pragma unroll
            for (int u = 0; u < D / 2; u++) {
                const longlong2 v = __ldg(br + u);
                S[2 * u] = A[2 * u] + v.x;
                S[2 * u + 1] = A[2 * u + 1] + v.y;
            }
            st = small_stat<D>(S, bal.d, bal.g, bal.cc, bal.cst);
            if (!FILT) out[c] = st;
        }
        if (FILT) {
            const bool keep = valid && (uint64_t)__double_as_longlong(st) <= hbits;
            const unsigned m = __ballot_sync(FRR_FULL, keep);
            if (m) {
                unsigned long long at = 0;
                if (lane == 0) at = atomicAdd(fcount, (unsigned long long)__popc(m));
                at = __shfl_sync(FRR_FULL, at, 0) + __popc(m & ((1u << lane) - 1u));
                if (keep && at < (unsigned long long)cap) {
                    fidx[at] = r;
                    fval[at] = st;
                }
            }
        }
    }
}

// ------------------------------------ split enumeration, tiled (filtered)
// The same (lower, upper) decomposition as k_exact_split, reordered for
// reuse: a tile pairs up to kTileRows consecutive upper-half subsets of one
// size s (SB rows j0 .. j0+nrows, held in registers, one per thread) with
// up to kTileBlocks blocks of that s (their SA rows staged in shared memory
// and read as warp broadcasts).  Candidate (block g, row j) has rank
// base_g + j.  Every SB row is loaded once per tile instead of once per
// candidate, so the kernel is bound by the fp64 epilogue, not by L2.  Only
// the filtered output exists (ranks come out in tile order; the caller
// sorts).  tiles[i] = {sb_row0, j0 << 32 | nrows, g0, interior << 32 | ng}.
constexpr int kTileRows = 256, kTileBlocks = 256;

template <int D, int DD>  // DD = d, a compile-time constant: no per-column predicates in the epilogue
__global__ void __launch_bounds__(kTileRows) k_exact_tiled(frr_balance_t bal, const int64_t* __restrict__ sa,
                                                           const int64_t* __restrict__ sb,
                                                           const int64_t* __restrict__ tiles, int64_t ntiles,
                                                           const int32_t* __restrict__ g_a,
                                                           const int64_t* __restrict__ g_base, int64_t rank_lo,
                                                           int64_t rank_hi, uint64_t hbits, int64_t cap,
                                                           int64_t* __restrict__ fidx, double* __restrict__ fval,
                                                           unsigned long long* __restrict__ fcount) {
    __shared__ __align__(16) int64_t sA[kTileBlocks * D];
    __shared__ int64_t sBase[kTileBlocks];
    const int lane = threadIdx.x & 31;
    double ccr[D];
#pragma unroll
    for (int u = 0; u < D; u++) ccr[u] = u < DD ? bal.cc[u] : 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t sb_row0 = tiles[4 * tile], jn = tiles[4 * tile + 1], g0 = tiles[4 * tile + 2];
        const int ng = (int)(tiles[4 * tile + 3] & 0xFFFFFFFF);
        const bool interior = (tiles[4 * tile + 3] >> 32) != 0;  // every rank of the tile is in [lo, hi)
        const int nrows = (int)(jn & 0xFFFFFFFF);
        const int64_t j = (jn >> 32) + threadIdx.x;
        __syncthreads();  // previous tile's readers are done with sA
        for (int i = threadIdx.x; i < ng * D; i += blockDim.x) sA[i] = sa[(int64_t)g_a[g0 + i / D] * D + i % D];
        for (int i = threadIdx.x; i < ng; i += blockDim.x) sBase[i] = g_base[g0 + i];
        const bool row_ok = threadIdx.x < nrows;
        int64_t B[D];
        const longlong2* br = reinterpret_cast<const longlong2*>(sb + (sb_row0 + (row_ok ? threadIdx.x : 0)) * D);
#pragma unroll
        for (int u = 0; u < D / 2; u++) {
            const longlong2 v = __ldg(br + u);
            B[2 * u] = v.x;
            B[2 * u + 1] = v.y;
        }
        __syncthreads();
        auto run = [&](auto inside) {
        for (int g = 0; g < ng; g++) {
            const int64_t r = sBase[g] + j;
            const bool valid = decltype(inside)::value ? row_ok : (row_ok && r >= rank_lo && r < rank_hi);
            const longlong2* ar = reinterpret_cast<const longlong2*>(sA + g * D);
            int64_t S[D];
#pragma unroll
            for (int u = 0; u < D / 2; u++) {
                const longlong2 a = ar[u];
                S[2 * u] = a.x + B[2 * u];
                S[2 * u + 1] = a.y + B[2 * u + 1];
            }
            const double st = small_stat<D>(S, DD, bal.g, ccr, bal.cst);
            const bool keep = valid && (uint64_t)__double_as_longlong(st) <= hbits;
            const unsigned m = __ballot_sync(FRR_FULL, keep);
            if (m) {
                unsigned long long at = 0;
                if (lane == 0) at = atomicAdd(fcount, (unsigned long long)__popc(m));
                at = __shfl_sync(FRR_FULL, at, 0) + __popc(m & ((1u << lane) - 1u));
                if (keep && at < (unsigned long long)cap) {
                    fidx[at] = r;
                    fval[at] = st;
                }
            }
        }
        };
        if (interior) run(std::integral_constant<bool, true>{});
        else run(std::integral_constant<bool, false>{});
    }
}

// ------------------------------------------ exact rows, thread per rank
// n <= 64: each thread unranks its rank into a unit mask (the combinadic
// walk of k_exact_small), a warp stages its 32 rows in shared memory and
// writes them as one contiguous, coalesced span.
constexpr int kRowsThreads = 256;
__global__ void __launch_bounds__(kRowsThreads) k_exact_rows_small(const uint64_t* __restrict__ ranks, int64_t m,
                                                                 int n, int t, int8_t* __restrict__ rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int nb = n + 1;
    uint64_t* binom = reinterpret_cast<uint64_t*>(smem);                     // [n+1][n+1]
    unsigned char* stage = reinterpret_cast<unsigned char*>(binom + nb * nb);  // [warps][32 * n]
    for (int i = threadIdx.x; i < nb * nb; i += blockDim.x) binom[i] = frr_binom(i / nb, i % nb);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* st = stage + (size_t)warp * 32 * n;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; w0 < m; w0 += nwarps * 32) {
        const int64_t c = w0 + lane;
        if (c < m) {
            uint64_t rank = ranks[c], msk = 0;
            int x = 0;
            for (int i = 0; i < t; i++) {
                for (;;) {
                    const uint64_t cnk = binom[(n - x - 1) * nb + (t - i - 1)];
                    if (rank < cnk) break;
                    rank -= cnk;
                    x++;
                }
                msk |= 1ull << x;
                x++;
            }
            for (int e = 0; e < n; e++) st[lane * n + e] = (unsigned char)((msk >> e) & 1);
        }
        __syncwarp();
        const int nrow = m - w0 < 32 ? (int)(m - w0) : 32;
        int8_t* dst = rows + (size_t)w0 * n;
        for (int o = lane; o < nrow * n; o += 32) dst[o] = (int8_t)st[o];
        __syncwarp();
    }
}

// ------------------------------------------------ randomization-test rows
// inference.py:82-101 (_dim_rows) for y (a) and for the observed assignment
// as outcome (b, exact popcounts), plus the pool-membership flag
// (inference.py:144).  The pairwise plan of length n (numpy's recursion) is
// built once per CTA: leaves + a post-order combine program.
struct PwPlan {
    int nleaf, ntok;
    int* leaf_off;
    int* leaf_len;
    int16_t* tok;  // >=0: leaf id; -1: combine
};

__device__ void plan_build(PwPlan& P, int off, int len) {
    if (len <= 128) {
        P.leaf_off[P.nleaf] = off;
        P.leaf_len[P.nleaf] = len;
        P.tok[P.ntok++] = (int16_t)P.nleaf++;
        return;
    }
    int n2 = len / 2;
    n2 -= n2 % 8;
    plan_build(P, off, n2);
    plan_build(P, off + n2, len - n2);
    P.tok[P.ntok++] = -1;
}

__host__ __device__ inline int plan_max_leaves(int n) { return n / 64 + 2; }

// The leaf-combination tree of numpy's pairwise sum as parallel rounds: node
// (L, R) adds its right child's value into its left child's slot (a node's
// slot is its leftmost leaf).  Nodes in one round touch disjoint slots and
// only read values finished in earlier rounds, so a warp evaluates the tree
// round by round instead of one lane walking the postfix program.
// sched[2e], sched[2e+1] = (L, R) of entry e; round r holds entries
// [round_start[r], round_start[r+1]).  Scratch: 3 * nleaf ints.  Returns the
// number of rounds.
constexpr int kMaxRounds = 32;
__device__ int plan_rounds(const int16_t* tok, int ntok, int nleaf, int* scratch, int16_t* sched,
                           int* round_start) {
    int* stk_slot = scratch;
    int* stk_h = scratch + nleaf;
    int* ent_r = scratch + 2 * nleaf;  // round of entry e (postfix order), its (L, R) staged in sched
    int sp = 0, ne = 0, nr = 0;
    for (int i = 0; i < ntok; i++) {
        if (tok[i] >= 0) {
            stk_slot[sp] = tok[i];
            stk_h[sp++] = 0;
        } else {
            sp--;
            const int r = max(stk_h[sp - 1], stk_h[sp]);
            ent_r[ne] = r;
            sched[2 * ne] = (int16_t)stk_slot[sp - 1];
            sched[2 * ne + 1] = (int16_t)stk_slot[sp];
            ne++;
            stk_h[sp - 1] = r + 1;
            nr = max(nr, r + 1);
        }
    }
    // stable counting sort of the entries by round, in place through scratch
    for (int r = 0; r <= nr; r++) round_start[r] = 0;
    for (int e = 0; e < ne; e++) round_start[ent_r[e] + 1]++;
    for (int r = 0; r < nr; r++) round_start[r + 1] += round_start[r];
    int* lr = stk_slot;  // (L, R) packed, reusing the stack area (2 * nleaf ints >= ne)
    for (int e = 0; e < ne; e++) lr[e] = (int)sched[2 * e] | ((int)sched[2 * e + 1] << 16);
    int* fill = stk_h;  // reused: per-round fill pointers (nr <= kMaxRounds)
    for (int r = 0; r < nr; r++) fill[r] = round_start[r];
    for (int e = 0; e < ne; e++) {
        const int d = fill[ent_r[e]]++;
        sched[2 * d] = (int16_t)(lr[e] & 0xFFFF);
        sched[2 * d + 1] = (int16_t)(lr[e] >> 16);
    }
    return nr;
}

template <int SRC, bool GS>
__global__ void __launch_bounds__(kPlanThreads) k_dim(uint64_t seed, const uint64_t* ids, const int8_t* rows,
                                                  int64_t m, int n, int t, const double* __restrict__ y,
                                                  const uint32_t* __restrict__ obs, double* a, double* b,
                                                  int32_t* match, const StepC* gsteps) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int maxl = plan_max_leaves(n);
    unsigned char* cursor = smem;
    const StepC* steps = cta_steps<GS>(cursor, gsteps, n, t, SRC == SRC_KEYS);
    const int nw = blockDim.x >> 5;
    double* leafres = reinterpret_cast<double*>(cursor);                   // [nw][2][maxl]
    int* leaf_off = reinterpret_cast<int*>(leafres + (size_t)nw * 2 * maxl);
    int* leaf_len = leaf_off + maxl;
    int16_t* tok = reinterpret_cast<int16_t*>(leaf_len + maxl);          // [2*maxl]
    __shared__ int s_nleaf, s_ntok;
    size_t toff = reinterpret_cast<unsigned char*>(tok + ((2 * maxl + 7) & ~7)) - smem;
    uint16_t* tables = reinterpret_cast<uint16_t*>(smem + ((toff + 15) & ~(size_t)15));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint16_t* lw = tables + (size_t)warp * frr_table_len(n);
    __shared__ int s_round[kMaxRounds + 1];
    __shared__ int s_nround;
    if (threadIdx.x == 0) {
        PwPlan P{0, 0, leaf_off, leaf_len, tok};
        plan_build(P, 0, n);
        s_nleaf = P.nleaf;
        s_ntok = P.ntok;
        // the round schedule overwrites tok (2 * (nleaf - 1) <= 2 * maxl
        // entries); scratch: the first 3 * nleaf ints of leafres
        s_nround = plan_rounds(tok, P.ntok, P.nleaf, reinterpret_cast<int*>(leafres), tok, s_round);
    }
    __syncthreads();
    const int nleaf = s_nleaf, nround = s_nround;
    double* rt = leafres + (size_t)warp * 2 * maxl;
    double* rc = rt + maxl;
    const int words = (n + 31) >> 5;
    const double inv_t = 1.0 / (double)t, inv_c = 1.0 / (double)(n - t);
    for (int64_t c = (int64_t)blockIdx.x * nw + warp; c < m; c += (int64_t)gridDim.x * nw) {
        build_table<SRC, GS>(seed, ids, rows, c, n, t, steps, lw, lane);
        // b and membership from packed words
        uint32_t pt = 0, pc = 0;
        bool same = true;
        for (int w = lane; w < words; w += 32) {
            uint32_t word = table_word(lw, n, w);
            uint32_t o = obs[w];
            pt += __popc(word & o);
            pc += __popc(~word & o);
            same &= (word == o);
        }
        // a: masked pairwise sums.  A leaf of numpy's pairwise_sum is 8
        // interleaved accumulator streams r_j = a[j] + a[j+8] + ... (in order)
        // combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential
        // tail: 8 lanes take the 8 streams of one leaf (4 leaves per warp
        // step, coalesced y / table reads) and a butterfly forms the tree
        // (IEEE addition is commutative, so the tree's values are exact).
        // Masked-out terms are +-0 like the reference's 0.0*y.
        {
            const int g = lane >> 3, j = lane & 7;
            for (int L0 = 0; L0 < nleaf; L0 += 4) {
                const int L = L0 + g;
                const bool act = L < nleaf;
                const int off = act ? leaf_off[L] : 0, len = act ? leaf_len[L] : 0;
                const int full = len >= 8 ? len - (len % 8) : 0;
                double st = 0.0, sc = 0.0;
                if (j < full) {
                    for (int i = j; i < full; i += 8) {
                        const int e = off + i;
                        const double v = __ldg(y + e), z = copysign(0.0, v);
                        const bool tr = lw[e] != FRR_CTL;
                        const double vt = tr ? v : z, vc = tr ? z : v;
                        if (i == j) {
                            st = vt;
                            sc = vc;
                        } else {
                            st = __dadd_rn(st, vt);
                            sc = __dadd_rn(sc, vc);
                        }
                    }
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const double ot = __shfl_xor_sync(FRR_FULL, st, o), oc = __shfl_xor_sync(FRR_FULL, sc, o);
                    st = __dadd_rn(st, ot);
                    sc = __dadd_rn(sc, oc);
                }
                if (act && j == 0) {
                    if (len < 8) st = sc = -0.0;
                    for (int i = full; i < len; i++) {  // tail (or a whole short leaf)
                        const int e = off + i;
                        const double v = __ldg(y + e), z = copysign(0.0, v);
                        const bool tr = lw[e] != FRR_CTL;
                        st = __dadd_rn(st, tr ? v : z);
                        sc = __dadd_rn(sc, tr ? z : v);
                    }
                    rt[L] = st;
                    rc[L] = sc;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            pt += __shfl_xor_sync(FRR_FULL, pt, o);
            pc += __shfl_xor_sync(FRR_FULL, pc, o);
        }
        same = __all_sync(FRR_FULL, same);
        __syncwarp();
        // the leaf-combination tree, one round of independent nodes at a time
        for (int rd = 0; rd < nround; rd++) {
            for (int e = s_round[rd] + lane; e < s_round[rd + 1]; e += 32) {
                const int L = tok[2 * e], R = tok[2 * e + 1];
                rt[L] = __dadd_rn(rt[L], rt[R]);
                rc[L] = __dadd_rn(rc[L], rc[R]);
            }
            __syncwarp();
        }
        if (lane == 0) {
            double s_t = __dadd_rn(0.0, rt[0]), s_c = __dadd_rn(0.0, rc[0]);
            a[c] = __dsub_rn(__dmul_rn(s_t, inv_t), __dmul_rn(s_c, inv_c));
            if (b) b[c] = __dsub_rn(__dmul_rn((double)pt, inv_t), __dmul_rn((double)pc, inv_c));
            if (match && same) atomicOr(match, 1);
        }
        __syncwarp();
    }
}

// ------------------------------------- randomization-test rows from keys
// k_dim for Monte Carlo keys with the thread-per-candidate generator: a warp
// regenerates 32 keys at once (frr_rev_fy: each lane builds one key's
// control bitset in its own bank column of the warp's block; exact
// recomputation of flagged keys), then every lane evaluates its own key:
//   b and pool membership: exact popcounts against the observed assignment;
//   a: numpy's pairwise sums of w*y and (1-w)*y (inference.py:82-101) in the
//     reference's arithmetic -- the 0/1 weight times y is a float64 product,
//     so masked-out terms are the reference's signed zeros -- walking numpy's
//     recursion (leaves of <= 128 units with 8 interleaved accumulators,
//     then the post-order combines) with a per-lane stack.  All lanes run the
//     same program on the same unit, so y is read as one broadcast per 8
//     units and the 16 accumulator chains give each lane its own ILP.
constexpr int kDimRevWarps = 8;
constexpr int kDimStack = 12;  // combine-stack depth bound: numpy's recursion holds <= log2(n / 128) + 2 <= 11 partial sums

struct DimRevPlan {
    int kw, maxl, warps;
    size_t steps_off, fix_off, lock_off, plan_off, warp_off, per_warp, total;
};

DimRevPlan dim_rev_plan(int n, int t) {
    DimRevPlan p;
    p.kw = (n + 31) / 32;
    p.maxl = plan_max_leaves(n);
    size_t o = 0;
    p.steps_off = o;
    o += (size_t)frr_steps_len(t) * sizeof(StepC);
    p.fix_off = o;
    o += (size_t)frr_table_len(n) * 2 + FRR_TABLE_SLACK;
    o = (o + 15) & ~(size_t)15;
    p.lock_off = o;
    o += 16;
    p.plan_off = o;
    o += 2 * (size_t)p.maxl * sizeof(int) + (size_t)((2 * p.maxl + 7) & ~7) * sizeof(int16_t);
    o = (o + 15) & ~(size_t)15;
    p.warp_off = o;
    p.per_warp = (size_t)32 * p.kw * 4 + (size_t)kDimStack * 2 * 32 * sizeof(double);
    p.warps = 0;
    for (int w = kDimRevWarps; w >= 1; w--)
        if (o + (size_t)w * p.per_warp <= 227 * 1024) {
            p.warps = w;
            break;
        }
    p.total = o + (size_t)p.warps * p.per_warp;
    return p;
}

// masked terms of one unit for this lane's key: w*y and (1-w)*y, w = 0/1
__device__ __forceinline__ void dim_terms(double v, uint32_t treated_bit, double& vt, double& vc) {
    const double w = __hiloint2double(treated_bit ? 0x3FF00000 : 0, 0);
    const double nw = __hiloint2double(treated_bit ? 0 : 0x3FF00000, 0);
    vt = __dmul_rn(w, v);
    vc = __dmul_rn(nw, v);
}

// FRR_DIM_FMA (default): r += w*y as one fused multiply-add.  For w in
// {0, 1} the product w*y is exact, so fma(w, y, r) -- one rounding of
// w*y + r, zero signs by the rules of addition -- is bit-identical to
// numpy's separately rounded (w*y) then r + (w*y), and numpy's first term
// r_j = w*y equals fma(w, y, -0.0).  Two DFMAs per unit instead of two
// DMULs and two DADDs.
#ifndef FRR_DIM_FMA
#define FRR_DIM_FMA 1
#endif

// ctl != 0: the unit is a control unit of this key (w = 0)
__device__ __forceinline__ void dim_acc(double& st, double& sc, double v, uint32_t ctl) {
    const int wh = ctl ? 0 : 0x3FF00000;
    st = __fma_rn(__hiloint2double(wh, 0), v, st);
    sc = __fma_rn(__hiloint2double(wh ^ 0x3FF00000, 0), v, sc);
}

// b and membership of one bitset word (exact integer popcounts)
struct DimCounts {
    uint32_t pt = 0, pc = 0;
    bool same = true;
    __device__ __forceinline__ void add(uint32_t ctl_word, int w, int n, const uint32_t* __restrict__ obs) {
        const int valid = n - 32 * w;
        const uint32_t vm = valid >= 32 ? FRR_FULL : ((1u << valid) - 1u);
        const uint32_t tr = ~ctl_word & vm, o = __ldg(obs + w);
        pt += __popc(tr & o);
        pc += __popc(~tr & vm & o);
        same &= tr == o;
    }
};

// a lane's control words in shared memory (word w at col[32 w])
struct DimWordsShared {
    static constexpr bool kStream = false;
    const uint32_t* col;
    __device__ __forceinline__ uint32_t operator()(int w) const { return col[32 * w]; }
};

// a lane's control words in global memory, read once each in ascending
// order (the pairwise walk visits units left to right): kDimRing words in
// flight through a per-lane ring in shared memory (cp.async, one commit
// group per word, so a word's wait never waits on a register move of a
// load still in flight); each word's popcounts are taken as it retires
constexpr int kDimRing = 8;

struct DimWordsRing {
    static constexpr bool kStream = true;
    const uint32_t* col;  // word w at col[32 w]
    uint32_t ring;        // shared address of this lane's slot 0 (slot s at ring + 128 s)
    int kw, n, cw;
    const uint32_t* obs;
    uint32_t cur;
    DimCounts cnt;
    __device__ __forceinline__ void fetch(int w) {
        if (w < kw)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ring + 128u * (uint32_t)(w % kDimRing)),
                         "l"(col + 32 * (size_t)w)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __device__ __forceinline__ uint32_t slot(int w) const {
        uint32_t v;
        asm volatile("cp.async.wait_group %1;\n\tld.shared.u32 %0, [%2];"
                     : "=r"(v)
                     : "n"(kDimRing - 1), "r"(ring + 128u * (uint32_t)(w % kDimRing))
                     : "memory");
        return v;
    }
    __device__ __forceinline__ DimWordsRing(const uint32_t* c, uint32_t r, int kw_, int n_, const uint32_t* o)
        : col(c), ring(r), kw(kw_), n(n_), cw(0), obs(o) {
#pragma unroll
        for (int d = 0; d < kDimRing; d++) fetch(d);
        cur = slot(0);
    }
    __device__ __forceinline__ void advance() {
        cnt.add(cur, cw, n, obs);
        fetch(cw + kDimRing);  // into the slot of word cw, already in `cur`
        cw++;
        cur = slot(cw);
    }
    __device__ __forceinline__ uint32_t operator()(int w) {
        if (w != cw) advance();  // w == cw or cw + 1
        return cur;
    }
    __device__ __forceinline__ void finish() {
        while (cw < kw - 1) advance();
        cnt.add(cur, cw, n, obs);
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
};

// b, membership and the pairwise sums of one lane's key: words(w) = the
// key's control bits of units 32 w .. 32 w + 31; the sums are left on the
// lane's stack (stk[0] = treated, stk[32] = control); y may be shared or global.
template <class Words>
__device__ __forceinline__ void dim_lane(int n, int kw, const double* __restrict__ y, const uint32_t* __restrict__ obs,
                                         Words& col_word, const int* leaf_off, const int* leaf_len, const int16_t* tok,
                                         int ntok, double* stk, uint32_t& pt_out, uint32_t& pc_out, bool& same_out) {
    DimCounts cnt;
    if constexpr (!Words::kStream)
        for (int w = 0; w < kw; w++) cnt.add(col_word(w), w, n, obs);
    // ---- a: numpy's pairwise sums of w*y and (1-w)*y, token program
    int sp = 0;
    for (int k = 0; k < ntok; k++) {
        const int L = tok[k];
        if (L < 0) {  // combine the top two partial sums
            sp--;
            stk[(2 * (sp - 1)) * 32] = __dadd_rn(stk[(2 * (sp - 1)) * 32], stk[(2 * sp) * 32]);
            stk[(2 * (sp - 1) + 1) * 32] = __dadd_rn(stk[(2 * (sp - 1) + 1) * 32], stk[(2 * sp + 1) * 32]);
            continue;
        }
        const int off = leaf_off[L], len = leaf_len[L];
        double st, sc;
#if FRR_DIM_FMA
        if (len < 8) {
            st = sc = -0.0;
            for (int i = 0; i < len; i++) {
                const int e = off + i;
                dim_acc(st, sc, y[e], (col_word(e >> 5) >> (e & 31)) & 1u);
            }
        } else {
            // 8 accumulators: r_j = term[j] + term[j + 8] + ... (off is a
            // multiple of 8, so units e..e+7 share one bitset word)
            const int full = len - (len % 8);
            double rt[8], rc[8];
#pragma unroll
            for (int j = 0; j < 8; j++) rt[j] = rc[j] = -0.0;
            for (int i = 0; i < full; i += 8) {
                const int e = off + i;
                const uint32_t bits = col_word(e >> 5) >> (e & 31);
                const double2* yv = reinterpret_cast<const double2*>(y + e);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const double2 v2 = yv[q];
                    dim_acc(rt[2 * q], rc[2 * q], v2.x, bits & (1u << (2 * q)));
                    dim_acc(rt[2 * q + 1], rc[2 * q + 1], v2.y, bits & (2u << (2 * q)));
                }
            }
            st = __dadd_rn(__dadd_rn(__dadd_rn(rt[0], rt[1]), __dadd_rn(rt[2], rt[3])),
                           __dadd_rn(__dadd_rn(rt[4], rt[5]), __dadd_rn(rt[6], rt[7])));
            sc = __dadd_rn(__dadd_rn(__dadd_rn(rc[0], rc[1]), __dadd_rn(rc[2], rc[3])),
                           __dadd_rn(__dadd_rn(rc[4], rc[5]), __dadd_rn(rc[6], rc[7])));
            for (int i = full; i < len; i++) {  // the tail, in order
                const int e = off + i;
                dim_acc(st, sc, y[e], (col_word(e >> 5) >> (e & 31)) & 1u);
            }
        }
#else
        if (len < 8) {
            st = sc = -0.0;
            for (int i = 0; i < len; i++) {
                const int e = off + i;
                double vt, vc;
                dim_terms(y[e], ~(col_word(e >> 5) >> (e & 31)) & 1u, vt, vc);
                st = __dadd_rn(st, vt);
                sc = __dadd_rn(sc, vc);
            }
        } else {
            const int full = len - (len % 8);
            double rt[8], rc[8];
            {
                const uint32_t bits = ~(col_word(off >> 5) >> (off & 31));
                const double2* yv = reinterpret_cast<const double2*>(y + off);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const double2 v2 = yv[q];
                    dim_terms(v2.x, (bits >> (2 * q)) & 1u, rt[2 * q], rc[2 * q]);
                    dim_terms(v2.y, (bits >> (2 * q + 1)) & 1u, rt[2 * q + 1], rc[2 * q + 1]);
                }
            }
            for (int i = 8; i < full; i += 8) {
                const int e = off + i;
                const uint32_t bits = ~(col_word(e >> 5) >> (e & 31));
                const double2* yv = reinterpret_cast<const double2*>(y + e);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const double2 v2 = yv[q];
                    double vt0, vc0, vt1, vc1;
                    dim_terms(v2.x, (bits >> (2 * q)) & 1u, vt0, vc0);
                    dim_terms(v2.y, (bits >> (2 * q + 1)) & 1u, vt1, vc1);
                    rt[2 * q] = __dadd_rn(rt[2 * q], vt0);
                    rc[2 * q] = __dadd_rn(rc[2 * q], vc0);
                    rt[2 * q + 1] = __dadd_rn(rt[2 * q + 1], vt1);
                    rc[2 * q + 1] = __dadd_rn(rc[2 * q + 1], vc1);
                }
            }
            st = __dadd_rn(__dadd_rn(__dadd_rn(rt[0], rt[1]), __dadd_rn(rt[2], rt[3])),
                           __dadd_rn(__dadd_rn(rt[4], rt[5]), __dadd_rn(rt[6], rt[7])));
            sc = __dadd_rn(__dadd_rn(__dadd_rn(rc[0], rc[1]), __dadd_rn(rc[2], rc[3])),
                           __dadd_rn(__dadd_rn(rc[4], rc[5]), __dadd_rn(rc[6], rc[7])));
            for (int i = full; i < len; i++) {
                const int e = off + i;
                double vt, vc;
                dim_terms(y[e], ~(col_word(e >> 5) >> (e & 31)) & 1u, vt, vc);
                st = __dadd_rn(st, vt);
                sc = __dadd_rn(sc, vc);
            }
        }
#endif
        stk[(2 * sp) * 32] = st;
        stk[(2 * sp + 1) * 32] = sc;
        sp++;
    }
    if constexpr (Words::kStream) {
        col_word.finish();
        cnt = col_word.cnt;
    }
    pt_out = cnt.pt;
    pc_out = cnt.pc;
    same_out = cnt.same;
}

__global__ void __launch_bounds__(kDimRevWarps * 32) k_dim_rev(uint64_t seed, const uint64_t* __restrict__ ids,
                                                               int64_t m, int n, int t, const double* __restrict__ y,
                                                               const uint32_t* __restrict__ obs, double* a, double* b,
                                                               int32_t* match, DimRevPlan P) {
    extern __shared__ __align__(16) unsigned char smem[];
    StepC* steps = reinterpret_cast<StepC*>(smem + P.steps_off);
    uint16_t* fix = reinterpret_cast<uint16_t*>(smem + P.fix_off);
    int* lock = reinterpret_cast<int*>(smem + P.lock_off);
    int* leaf_off = reinterpret_cast<int*>(smem + P.plan_off);
    int* leaf_len = leaf_off + P.maxl;
    int16_t* tok = reinterpret_cast<int16_t*>(leaf_len + P.maxl);
    __shared__ int s_ntok;
    frr_fill_steps(steps, n, t);
    if (threadIdx.x == 0) {
        *lock = 0;
        PwPlan pl{0, 0, leaf_off, leaf_len, tok};
        plan_build(pl, 0, n);
        s_ntok = pl.ntok;
    }
    __syncthreads();
    const int ntok = s_ntok;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kw = P.kw;
    unsigned char* wbase = smem + P.warp_off + (size_t)warp * P.per_warp;
    const uint32_t* col = reinterpret_cast<const uint32_t*>(wbase) + lane;  // this lane's key, word w at col[32 w]
    double* stk = reinterpret_cast<double*>(wbase + (size_t)32 * kw * 4) + lane;  // [level][t/c][lane]
    const uint32_t blk_a = (uint32_t)__cvta_generic_to_shared(wbase), sst = (uint32_t)__cvta_generic_to_shared(steps);
    const double inv_t = 1.0 / (double)t, inv_c = 1.0 / (double)(n - t);
    const int64_t njobs = (m + 31) / 32;
    for (int64_t job = (int64_t)blockIdx.x * P.warps + warp; job < njobs; job += (int64_t)gridDim.x * P.warps) {
        const int64_t c = job * 32 + lane;
        // ---- regenerate the 32 keys (lane = key), exact path for flagged ones
        const uint64_t state = frr_derive_state(seed, ids[c < m ? c : m - 1]);
        const bool flag = frr_rev_fy(state, t, sst, blk_a + 4u * lane, kw);
        uint32_t fl = __ballot_sync(FRR_FULL, flag);
        while (fl) {
            const int src = __ffs(fl) - 1;
            fl &= fl - 1;
            if (lane == 0)
                while (atomicCAS(lock, 0, 1) != 0) __nanosleep(100);
            __syncwarp();
            frr_rev_fixup(__shfl_sync(FRR_FULL, state, src), n, t, steps, fix, blk_a + 4u * src, kw, lane);
            if (lane == 0) atomicExch(lock, 0);
            __syncwarp();
        }
        __syncwarp();
        uint32_t pt, pc;
        bool same;
        DimWordsShared cw{col};
        dim_lane(n, kw, y, obs, cw, leaf_off, leaf_len, tok, ntok, stk, pt, pc, same);
        if (c < m) {
            const double s_t = __dadd_rn(0.0, stk[0]), s_c = __dadd_rn(0.0, stk[32]);
            a[c] = __dsub_rn(__dmul_rn(s_t, inv_t), __dmul_rn(s_c, inv_c));
            if (b) b[c] = __dsub_rn(__dmul_rn((double)pt, inv_t), __dmul_rn((double)pc, inv_c));
            if (match && same) atomicOr(match, 1);
        }
        __syncwarp();
    }
}

// The same statistics from control bitsets already in global memory
// (frr_rev_words' interleaved layout [job][w][32], lane = key): y lives in
// shared memory (one broadcast per 8 units), so many warps per SM fit and
// the generation kernel keeps all of shared memory for its bitsets.
constexpr int kDimBitsWarps = 8;

struct DimBitsPlan {
    int kw, maxl;
    size_t y_off, plan_off, stk_off, ring_off, total;
};

DimBitsPlan dim_bits_plan(int n) {
    DimBitsPlan p;
    p.kw = (n + 31) / 32;
    p.maxl = plan_max_leaves(n);
    size_t o = 0;
    p.y_off = o;
    o += (size_t)n * sizeof(double);
    o = (o + 15) & ~(size_t)15;
    p.plan_off = o;
    o += 2 * (size_t)p.maxl * sizeof(int) + (size_t)((2 * p.maxl + 7) & ~7) * sizeof(int16_t);
    o = (o + 15) & ~(size_t)15;
    p.stk_off = o;
    o += (size_t)kDimBitsWarps * kDimStack * 2 * 32 * sizeof(double);
    p.ring_off = o;
    o += (size_t)kDimBitsWarps * kDimRing * 32 * sizeof(uint32_t);
    p.total = o;
    return p;
}

__global__ void __launch_bounds__(kDimBitsWarps * 32) k_dim_bits(const uint32_t* __restrict__ words, int64_t m, int n,
                                                                 int t, const double* __restrict__ y,
                                                                 const uint32_t* __restrict__ obs, double* a, double* b,
                                                                 int32_t* match, DimBitsPlan P) {
    extern __shared__ __align__(16) unsigned char smem[];
    double* sy = reinterpret_cast<double*>(smem + P.y_off);
    int* leaf_off = reinterpret_cast<int*>(smem + P.plan_off);
    int* leaf_len = leaf_off + P.maxl;
    int16_t* tok = reinterpret_cast<int16_t*>(leaf_len + P.maxl);
    __shared__ int s_ntok;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sy[i] = y[i];
    if (threadIdx.x == 0) {
        PwPlan pl{0, 0, leaf_off, leaf_len, tok};
        plan_build(pl, 0, n);
        s_ntok = pl.ntok;
    }
    __syncthreads();
    const int ntok = s_ntok;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kw = P.kw;
    double* stk = reinterpret_cast<double*>(smem + P.stk_off) + (size_t)warp * kDimStack * 2 * 32 + lane;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem + P.ring_off) + 4u * (uint32_t)(warp * kDimRing * 32 + lane);
    const double inv_t = 1.0 / (double)t, inv_c = 1.0 / (double)(n - t);
    const int64_t njobs = (m + 31) / 32;
    for (int64_t job = (int64_t)blockIdx.x * kDimBitsWarps + warp; job < njobs;
         job += (int64_t)gridDim.x * kDimBitsWarps) {
        const int64_t c = job * 32 + lane;
        const uint32_t* col = words + (size_t)job * kw * 32 + lane;  // coalesced: one 128-byte row per word
        uint32_t pt, pc;
        bool same;
        DimWordsRing cw(col, ring, kw, n, obs);
        dim_lane(n, kw, sy, obs, cw, leaf_off, leaf_len, tok, ntok, stk, pt, pc, same);
        if (c < m) {
            const double s_t = __dadd_rn(0.0, stk[0]), s_c = __dadd_rn(0.0, stk[32]);
            a[c] = __dsub_rn(__dmul_rn(s_t, inv_t), __dmul_rn(s_c, inv_c));
            if (b) b[c] = __dsub_rn(__dmul_rn((double)pt, inv_t), __dmul_rn((double)pc, inv_c));
            if (match && same) atomicOr(match, 1);
        }
    }
}

// ------------------------------------------------------------ tau counts
constexpr int kTauTile = 32;

__global__ void __launch_bounds__(256) k_tau_counts(const double* __restrict__ a, const double* __restrict__ b,
                                                    int64_t m, const double* __restrict__ taus,
                                                    const double* __restrict__ rhs, int ntau,
                                                    unsigned long long* counts) {
    __shared__ double s_tau[kTauTile], s_rhs[kTauTile];
    const int t0 = blockIdx.y * kTauTile;
    const int nt = min(kTauTile, ntau - t0);
    if (threadIdx.x < nt) {
        s_tau[threadIdx.x] = taus[t0 + threadIdx.x];
        s_rhs[threadIdx.x] = rhs[t0 + threadIdx.x];
    }
    __syncthreads();
    uint32_t cnt[kTauTile];
#pragma unroll
    for (int j = 0; j < kTauTile; j++) cnt[j] = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double ai = a[i], bi = b[i];
#pragma unroll
        for (int j = 0; j < kTauTile; j++) {
            if (j < nt) cnt[j] += fabs(__dsub_rn(ai, __dmul_rn(s_tau[j], bi))) >= s_rhs[j];
        }
    }
#pragma unroll
    for (int j = 0; j < kTauTile; j++) {
        uint32_t v = cnt[j];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FRR_FULL, v, o);
        if ((threadIdx.x & 31) == 0 && j < nt && v) atomicAdd(counts + t0 + j, (unsigned long long)v);
    }
}

// -------------------------------------------------------- host helpers
size_t table_bytes1(int n) { return (size_t)frr_table_len(n) * sizeof(uint16_t); }

int check_nt(int n, int t) {
    if (n < 2 || n > FRR_MAX_UNITS) {
        frr_set_error("n_units=%d outside [2, %d]", n, FRR_MAX_UNITS);
        return n < 2 ? FRR_E_INVALID_DESIGN : FRR_E_UNSUPPORTED;
    }
    if (t <= 0 || t >= n) {
        frr_set_error("n_treated must satisfy 0 < n_treated < n_units (got %d, %d)", t, n);
        return FRR_E_INVALID_DESIGN;
    }
    return FRR_OK;
}

// Launch a warp-per-candidate kernel instantiated for shared (GS=false) or
// global (GS=true) step tables according to the plan.
template <class KS, class KG, class... Args>
int launch_planned(const char* what, KS ks, KG kg, const WarpPlan& P, int n, int t, bool keys, int64_t items,
                   void* stream, Args... args) {
    if (P.warps < 1) {
        frr_set_error("%s: n=%d does not fit shared memory", what, n);
        return FRR_E_UNSUPPORTED;
    }
    cudaStream_t s = frr_stream(stream);
    GlobalSteps gs;
    int rc;
    const int threads = P.warps * 32;
    if (P.gsteps) {
        if ((rc = gs.init(n, t, s))) return rc;
        if ((rc = frr_prepare_kernel(kg, P.smem))) return rc;
        int grid = frr_persistent_grid(kg, threads, P.smem, frr_cdiv(items, P.warps));
        if (getenv("FRR_DEBUG_PLAN")) fprintf(stderr, "%s: warps=%d gsteps=1 smem=%zu grid=%d\n", what, P.warps, P.smem, grid);
        kg<<<grid, threads, P.smem, s>>>(args..., gs.p);
    } else {
        if ((rc = frr_prepare_kernel(ks, P.smem))) return rc;
        int grid = frr_persistent_grid(ks, threads, P.smem, frr_cdiv(items, P.warps));
        if (getenv("FRR_DEBUG_PLAN")) fprintf(stderr, "%s: warps=%d gsteps=0 smem=%zu grid=%d\n", what, P.warps, P.smem, grid);
        ks<<<grid, threads, P.smem, s>>>(args..., (const StepC*)nullptr);
    }
    (void)keys;
    return frr_launched(what);
}

template <int SRC>
int launch_regen(uint64_t seed, const uint64_t* ids, int64_t m, int n, int t, int8_t* rows, uint32_t* bits,
                 void* stream) {
    int rc = check_nt(n, t);
    if (rc) return rc;
    if (m <= 0) return FRR_OK;
    WarpPlan P = plan_warps(t, SRC == SRC_KEYS, 0, table_bytes1(n));
    return launch_planned("k_regen", k_regen<SRC, false>, k_regen<SRC, true>, P, n, t, SRC == SRC_KEYS, m, stream,
                          seed, ids, m, n, t, rows, bits);
}

template <int SRC, int D>
int launch_small(const frr_balance_t* bal, uint64_t seed, const uint64_t* ids, const int8_t* rows, uint64_t lo,
                 int64_t count, double* out, void* stream) {
    WarpPlan P = plan_warps(bal->t, SRC == SRC_KEYS, 0, table_bytes1(bal->n));
    return launch_planned("k_stats_small", k_stats_small<SRC, D, false>, k_stats_small<SRC, D, true>, P, bal->n,
                          bal->t, SRC == SRC_KEYS, count, stream, *bal, seed, ids, rows, lo, count, out);
}

template <int SRC>
int launch_stats(const frr_balance_t* bal, uint64_t seed, const uint64_t* ids, const int8_t* rows, uint64_t lo,
                 int64_t count, double* out, void* stream) {
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (count <= 0) return FRR_OK;
    if (bal->d <= 4) return launch_small<SRC, 4>(bal, seed, ids, rows, lo, count, out, stream);
    if (bal->d <= 8) return launch_small<SRC, 8>(bal, seed, ids, rows, lo, count, out, stream);
    if (bal->d <= 16) return launch_small<SRC, 16>(bal, seed, ids, rows, lo, count, out, stream);
    WarpPlan P = plan_warps(bal->t, SRC == SRC_KEYS, 16, (size_t)bal->d * sizeof(double) + table_bytes1(bal->n));
    return launch_planned("k_stats_generic", k_stats_generic<SRC, false>, k_stats_generic<SRC, true>, P, bal->n,
                          bal->t, SRC == SRC_KEYS, count, stream, *bal, seed, ids, rows, lo, count, out);
}

template <int D>
int launch_exact_small(const frr_balance_t* bal, uint64_t rank_lo, int64_t count, double* out, void* stream) {
    size_t smem = (size_t)(bal->n + 1) * (bal->n + 1) * sizeof(uint64_t) + (size_t)bal->n * D * sizeof(int64_t) +
                  (size_t)kWarps * 32 * (kRun + 1) * sizeof(double);
    auto kern = k_exact_small<D>;
    int rc = frr_prepare_kernel(kern, smem);
    if (rc) return rc;
    int grid = frr_persistent_grid(kern, kThreads, smem, frr_cdiv(count, (int64_t)kWarps * 32 * kRun));
    kern<<<grid, kThreads, smem, frr_stream(stream)>>>(*bal, rank_lo, count, out);
    return frr_launched("k_exact_small");
}

template <int SRC>
int launch_dim(uint64_t seed, const uint64_t* ids, const int8_t* rows, int64_t m, int n, int t, const double* y,
               const uint32_t* obs, double* a, double* b, int32_t* match, void* stream) {
    int rc = check_nt(n, t);
    if (rc) return rc;
    if (m <= 0) return FRR_OK;
    int maxl = plan_max_leaves(n);
    size_t fixed = 2 * (size_t)maxl * sizeof(int) + (size_t)((2 * maxl + 7) & ~7) * sizeof(int16_t) + 16;
    size_t per_warp = (size_t)2 * maxl * sizeof(double) + table_bytes1(n);
    WarpPlan P = plan_warps(t, SRC == SRC_KEYS, fixed, per_warp);
    return launch_planned("k_dim", k_dim<SRC, false>, k_dim<SRC, true>, P, n, t, SRC == SRC_KEYS, m, stream, seed,
                          ids, rows, m, n, t, y, obs, a, b, match);
}

int split_width(int d) { return d <= 4 ? 4 : d <= 6 ? 6 : d <= 8 ? 8 : d <= 16 ? 16 : 0; }

struct SplitFilter {
    uint64_t hbits;
    int64_t cap;
    int64_t* idx;
    double* val;
    unsigned long long* count;
};

template <int D>
int launch_split(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, const int32_t* blk_a,
                 const int64_t* blk_off, const int64_t* blk_base, int64_t nblk, uint64_t rank_lo, int64_t count,
                 double* out, const SplitFilter* f, int64_t stride, void* stream) {
    auto kern = f ? k_exact_split<D, true> : k_exact_split<D, false>;
    int rc = frr_prepare_kernel(kern, 0);
    if (rc) return rc;
    int grid = frr_persistent_grid(kern, 256, 0, frr_cdiv(count, (int64_t)256 * 32));
    const SplitFilter z{0, 0, nullptr, nullptr, nullptr};
    const SplitFilter& F = f ? *f : z;
    kern<<<grid, 256, 0, frr_stream(stream)>>>(*bal, sa, sb, blk_a, blk_off, blk_base, nblk, rank_lo, count, out,
                                               F.hbits, F.cap, F.idx, F.val, F.count, stride);
    return frr_launched(f ? "k_exact_split<filtered>" : "k_exact_split");
}

template <int D>
int launch_subset_sums(const frr_balance_t* bal, int na, const int32_t* lb, int64_t* sa, int64_t* sb, void* stream) {
    const int64_t tot = (1ll << na) + (1ll << (bal->n - na));
    k_subset_sums<D><<<(int)std::min<int64_t>(frr_cdiv(tot, 256), 4096), 256, 0, frr_stream(stream)>>>(
        bal->zq, bal->n, bal->d, na, lb, sa, sb);
    return frr_launched("k_subset_sums");
}

template <int D, int DD>
int launch_tiled(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, const int64_t* tiles,
                 int64_t ntiles, const int32_t* g_a, const int64_t* g_base, int64_t rank_lo, int64_t rank_hi,
                 const SplitFilter& f, void* stream) {
    auto kern = k_exact_tiled<D, DD>;
    int rc = frr_prepare_kernel(kern, 0);
    if (rc) return rc;
    int grid = frr_persistent_grid(kern, kTileRows, 0, ntiles);
    kern<<<grid, kTileRows, 0, frr_stream(stream)>>>(*bal, sa, sb, tiles, ntiles, g_a, g_base, rank_lo, rank_hi,
                                                     f.hbits, f.cap, f.idx, f.val, f.count);
    return frr_launched("k_exact_tiled");
}

int split_dispatch(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width, const int32_t* blk_a,
                   const int64_t* blk_off, const int64_t* blk_base, int64_t nblk, uint64_t rank_lo, int64_t count,
                   double* stats, const SplitFilter* f, int64_t stride, void* stream) {
    switch (width) {
        case 4: return launch_split<4>(bal, sa, sb, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, f, stride, stream);
        case 6: return launch_split<6>(bal, sa, sb, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, f, stride, stream);
        case 8: return launch_split<8>(bal, sa, sb, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, f, stride, stream);
        default:
            return launch_split<16>(bal, sa, sb, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, f, stride, stream);
    }
}

}  // namespace

// ===================================================================== ABI
int frr_mc_stats_mma(const frr_balance_t* bal, uint64_t seed, uint64_t lo, int64_t count, double* stats,
                     void* stream);  // frr_mma.cu
bool frr_mma_supported(const frr_balance_t* bal);

extern "C" int frr_mc_stats(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                            double* stats, void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    if (bal->limbs && frr_mma_supported(bal)) return frr_mc_stats_mma(bal, root_seed, draw_lo, count, stats, stream);
    return launch_stats<SRC_KEYS>(bal, root_seed, nullptr, nullptr, draw_lo, count, stats, stream);
}

extern "C" int frr_exact_stats(const frr_balance_t* bal, uint64_t rank_lo, int64_t count, double* stats,
                               void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (count <= 0) return FRR_OK;
    if (bal->n <= 64 && bal->d <= 16) {
        if (bal->d <= 4) return launch_exact_small<4>(bal, rank_lo, count, stats, stream);
        if (bal->d <= 6) return launch_exact_small<6>(bal, rank_lo, count, stats, stream);  // C1/C4: d = 5
        if (bal->d <= 8) return launch_exact_small<8>(bal, rank_lo, count, stats, stream);
        return launch_exact_small<16>(bal, rank_lo, count, stats, stream);
    }
    // general exact path: ranks materialised on the fly, one per warp
    frr_set_error("frr_exact_stats: n=%d d=%d needs the rank-list path (use frr_exact_stats_ids)", bal->n, bal->d);
    return FRR_E_UNSUPPORTED;
}

extern "C" int frr_exact_stats_ids(const frr_balance_t* bal, const uint64_t* ranks, int64_t m, double* stats,
                                   void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    return launch_stats<SRC_RANKS>(bal, 0, ranks, nullptr, 0, m, stats, stream);
}

extern "C" int frr_exact_split_width(int d) { return split_width(d); }

extern "C" int frr_subset_sums(const frr_balance_t* bal, int na, int width, const int32_t* lb, int64_t* sa,
                               int64_t* sb, void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (width != split_width(bal->d) || na < 1 || na > 24 || bal->n - na < 1 || bal->n - na > 24) {
        frr_set_error("frr_subset_sums: width %d / halves %d+%d unsupported for d=%d", width, na, bal->n - na, bal->d);
        return FRR_E_UNSUPPORTED;
    }
    switch (width) {
        case 4: return launch_subset_sums<4>(bal, na, lb, sa, sb, stream);
        case 6: return launch_subset_sums<6>(bal, na, lb, sa, sb, stream);
        case 8: return launch_subset_sums<8>(bal, na, lb, sa, sb, stream);
        default: return launch_subset_sums<16>(bal, na, lb, sa, sb, stream);
    }
}

extern "C" int frr_exact_stats_split(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                                     const int32_t* blk_a, const int64_t* blk_off, const int64_t* blk_base,
                                     int64_t nblk, uint64_t rank_lo, int64_t count, double* stats, void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (count <= 0) return FRR_OK;
    if (width != split_width(bal->d) || nblk < 1) {
        frr_set_error("frr_exact_stats_split: width %d for d=%d, %lld blocks", width, bal->d, (long long)nblk);
        return FRR_E_UNSUPPORTED;
    }
    return split_dispatch(bal, sa, sb, width, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, nullptr, 1,
                          stream);
}

extern "C" int frr_exact_stats_split_strided(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb,
                                             int width, const int32_t* blk_a, const int64_t* blk_off,
                                             const int64_t* blk_base, int64_t nblk, uint64_t rank_lo,
                                             int64_t stride, int64_t count, double* stats, void* stream) {
    if (!bal || stride < 1) return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (count <= 0) return FRR_OK;
    if (width != split_width(bal->d) || nblk < 1) {
        frr_set_error("frr_exact_stats_split_strided: width %d for d=%d, %lld blocks", width, bal->d,
                      (long long)nblk);
        return FRR_E_UNSUPPORTED;
    }
    return split_dispatch(bal, sa, sb, width, blk_a, blk_off, blk_base, nblk, rank_lo, count, stats, nullptr, stride,
                          stream);
}

extern "C" int frr_exact_stats_split_filtered(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb,
                                              int width, const int32_t* blk_a, const int64_t* blk_off,
                                              const int64_t* blk_base, int64_t nblk, uint64_t rank_lo,
                                              int64_t count, uint64_t h_bits, int64_t cap, int64_t* idx,
                                              double* vals, uint64_t* n_kept, void* stream) {
    if (!bal || !n_kept || cap < 0 || (cap > 0 && (!idx || !vals))) return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (count <= 0) return FRR_OK;
    if (width != split_width(bal->d) || nblk < 1) {
        frr_set_error("frr_exact_stats_split_filtered: width %d for d=%d, %lld blocks", width, bal->d,
                      (long long)nblk);
        return FRR_E_UNSUPPORTED;
    }
    const SplitFilter f{h_bits, cap, idx, vals, reinterpret_cast<unsigned long long*>(n_kept)};
    return split_dispatch(bal, sa, sb, width, blk_a, blk_off, blk_base, nblk, rank_lo, count, nullptr, &f, 1,
                          stream);
}

extern "C" int frr_rows_stats(const frr_balance_t* bal, const int8_t* rows, int64_t m, double* stats,
                              void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    return launch_stats<SRC_ROWS>(bal, 0, nullptr, rows, 0, m, stats, stream);
}

extern "C" int frr_mc_stats_small(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                                  double* stats, void* stream) {
    if (!bal) return FRR_E_INVALID_DESIGN;
    return launch_stats<SRC_KEYS>(bal, root_seed, nullptr, nullptr, draw_lo, count, stats, stream);
}

extern "C" int frr_regen_mc(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t, int8_t* rows,
                            uint32_t* bits, void* stream) {
    return launch_regen<SRC_KEYS>(root_seed, draws, m, n, t, rows, bits, stream);
}

extern "C" int frr_regen_exact(const uint64_t* ranks, int64_t m, int n, int t, int8_t* rows, uint32_t* bits,
                               void* stream) {
    if (rows && !bits && n <= 64 && m > 0 && check_nt(n, t) == FRR_OK) {
        const size_t smem = (size_t)(n + 1) * (n + 1) * sizeof(uint64_t) + (size_t)(kRowsThreads / 32) * 32 * n;
        int rc = frr_prepare_kernel(k_exact_rows_small, smem);
        if (rc) return rc;
        int grid = frr_persistent_grid(k_exact_rows_small, kRowsThreads, smem, frr_cdiv(m, (int64_t)kRowsThreads));
        k_exact_rows_small<<<grid, kRowsThreads, smem, frr_stream(stream)>>>(ranks, m, n, t, rows);
        return frr_launched("k_exact_rows_small");
    }
    return launch_regen<SRC_RANKS>(0, ranks, m, n, t, rows, bits, stream);
}

extern "C" int frr_dim_mc(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t, const double* y,
                          const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* stream) {
    int rc = check_nt(n, t);
    if (rc) return rc;
    if (m <= 0) return FRR_OK;
    // thread-per-key regeneration when two or more warps' bitsets fit shared
    // memory (n up to ~9000), else the warp-per-key kernel
    const DimRevPlan P = dim_rev_plan(n, t);
    const char* path = getenv("FRR_DIM_PATH");
    if (P.warps >= 2 && !(path && path[0] == 'w')) {
        if ((rc = frr_prepare_kernel(k_dim_rev, P.total))) return rc;
        const int grid = frr_persistent_grid(k_dim_rev, P.warps * 32, P.total, frr_cdiv(m, 32 * P.warps));
        k_dim_rev<<<grid, P.warps * 32, P.total, frr_stream(stream)>>>(root_seed, draws, m, n, t, y, obs_bits, a, b,
                                                                      match, P);
        return frr_launched("k_dim_rev");
    }
    return launch_dim<SRC_KEYS>(root_seed, draws, nullptr, m, n, t, y, obs_bits, a, b, match, stream);
}

int frr_rev_words(uint64_t root_seed, const uint64_t* ids, int64_t count, int n, int t, uint32_t* words,
                  void* steps, void* stream);
int64_t frr_rev_wave_keys(int n, int t);

// workspace of frr_dim_mc_ws: the generator's global step table (64 KB per
// 4096 steps, t <= FRR_MAX_UNITS) then the bitsets of a chunk of keys (a
// multiple of 32)
static size_t dim_ws_steps_bytes() { return (size_t)frr_steps_len(FRR_MAX_UNITS) * sizeof(StepC); }

static int64_t dim_ws_chunk(int n, size_t ws_bytes) {
    const size_t per_key = (size_t)((n + 31) / 32) * 4;
    if (ws_bytes < dim_ws_steps_bytes()) return 0;
    return (int64_t)((ws_bytes - dim_ws_steps_bytes()) / per_key) / 32 * 32;
}

// keys per internal chunk: whole generator waves (a chunk of 2^18 keys at
// n = 5000 is 5.03 waves of 11 warps x 148 SMs, i.e. 6 rounds of which the
// last is almost idle)
static int64_t dim_ws_chunk_aligned(int64_t m, int n, int t, size_t ws_bytes) {
    int64_t chunk = dim_ws_chunk(n, ws_bytes);
    const int64_t wave = frr_rev_wave_keys(n, t);
    if (wave > 0 && chunk >= wave && m > chunk) chunk = chunk / wave * wave;
    return chunk;
}

extern "C" int64_t frr_dim_mc_chunk_keys(int64_t m, int n, int t, size_t ws_bytes) {
    if (m <= 0 || n < 2 || t < 1 || t >= n) return 0;
    const int64_t chunk = dim_ws_chunk_aligned(m, n, t, ws_bytes);
    return chunk < 32 ? m : std::min(chunk, m);
}

extern "C" size_t frr_dim_mc_workspace_bytes(int64_t m, int n) {
    if (m <= 0 || n < 2) return 0;
    const int64_t keys = std::min<int64_t>((m + 31) / 32 * 32, (int64_t)1 << 18);
    return dim_ws_steps_bytes() + (size_t)keys * ((n + 31) / 32) * 4;
}

extern "C" int frr_dim_mc_ws(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t, const double* y,
                             const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* workspace,
                             size_t ws_bytes, void* stream) {
    int rc = check_nt(n, t);
    if (rc) return rc;
    if (m <= 0) return FRR_OK;
    const int64_t chunk = dim_ws_chunk_aligned(m, n, t, ws_bytes);
    const DimBitsPlan P = dim_bits_plan(n);
    if (chunk < 32 || P.total > 227 * 1024)
        return frr_dim_mc(root_seed, draws, m, n, t, y, obs_bits, a, b, match, stream);
    if ((rc = frr_prepare_kernel(k_dim_bits, P.total))) return rc;
    void* steps = workspace;
    uint32_t* words = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(workspace) + dim_ws_steps_bytes());
    for (int64_t lo = 0; lo < m; lo += chunk) {
        const int64_t cnt = std::min<int64_t>(chunk, m - lo);
        if ((rc = frr_rev_words(root_seed, draws + lo, cnt, n, t, words, steps, stream))) return rc;
        const int grid = frr_persistent_grid(k_dim_bits, kDimBitsWarps * 32, P.total,
                                             frr_cdiv(cnt, 32 * kDimBitsWarps));
        k_dim_bits<<<grid, kDimBitsWarps * 32, P.total, frr_stream(stream)>>>(
            words, cnt, n, t, y, obs_bits, a + lo, b ? b + lo : nullptr, match, P);
        if ((rc = frr_launched("k_dim_bits"))) return rc;
    }
    return FRR_OK;
}

extern "C" int frr_dim_exact(const uint64_t* ranks, int64_t m, int n, int t, const double* y,
                             const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* stream) {
    return launch_dim<SRC_RANKS>(0, ranks, nullptr, m, n, t, y, obs_bits, a, b, match, stream);
}

extern "C" int frr_dim_rows(const int8_t* rows, int64_t m, int n, int t, const double* y,
                            const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* stream) {
    return launch_dim<SRC_ROWS>(0, nullptr, rows, m, n, t, y, obs_bits, a, b, match, stream);
}

extern "C" int frr_tau_counts(const double* a, const double* b, int64_t m, const double* taus, const double* rhs,
                              int ntau, uint64_t* counts, void* stream) {
    if (ntau <= 0) return FRR_OK;
    cudaStream_t s = frr_stream(stream);
    if (cudaMemsetAsync(counts, 0, sizeof(uint64_t) * (size_t)ntau, s) != cudaSuccess)
        return frr_check_launch("frr_tau_counts memset");
    if (m <= 0) return FRR_OK;
    int tiles = (ntau + kTauTile - 1) / kTauTile;
    int64_t per_tile = std::max<int64_t>(1, (int64_t)frr_num_sms() * 8 / tiles);
    per_tile = std::min<int64_t>(per_tile, frr_cdiv(m, 256));
    dim3 grid((unsigned)per_tile, (unsigned)tiles);
    k_tau_counts<<<grid, 256, 0, s>>>(a, b, m, taus, rhs, ntau, reinterpret_cast<unsigned long long*>(counts));
    return frr_launched("k_tau_counts");
}

// ------------------------------------------------------------ diagnostics
namespace {
// Generator arithmetic only: per draw one 64-bit counter step, splitmix64,
// the rejection flag fold and the exact bounded reduction (frr_fy_draw minus
// its step-table load), two independent chains per thread like the
// generators' two rounds per iteration.
__global__ void __launch_bounds__(256) k_microbench_draws(int64_t per_thread, StepC st, uint64_t* sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t x0 = frr_mix64(tid), x1 = x0 + 32ull * FRR_GOLDEN;
    const uint64_t stride = 64ull * FRR_GOLDEN;
    uint32_t hmax = 0, acc = 0;
    for (int64_t i = 0; i < per_thread; i += 2) {
        const uint64_t u0 = frr_mix64(x0), u1 = frr_mix64(x1);
        hmax = max(hmax, max((uint32_t)(u0 >> 32), (uint32_t)(u1 >> 32)));
        acc += frr_mod_step(u0, st) + frr_mod_step(u1, st);
        x0 += stride;
        x1 += stride;
    }
    if ((acc ^ hmax) == 0x9E3779B9u) atomicAdd(reinterpret_cast<unsigned long long*>(sink), 1ull);
}
}  // namespace

extern "C" int frr_microbench_draws(int64_t per_thread, uint64_t* sink, int64_t* total_draws_host, void* stream) {
    if (per_thread <= 0 || (per_thread & 1)) {
        frr_set_error("frr_microbench_draws: per_thread must be positive and even");
        return FRR_E_INVALID_DESIGN;
    }
    const int grid = frr_persistent_grid(k_microbench_draws, 256, 0, INT64_MAX);
    const StepC st = frr_make_step(1000, 257);
    k_microbench_draws<<<grid, 256, 0, frr_stream(stream)>>>(per_thread, st, sink);
    if (total_draws_host) *total_draws_host = (int64_t)grid * 256 * per_thread;
    return frr_launched("k_microbench_draws");
}

extern "C" int frr_exact_tiled_filtered(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                                        const int64_t* tiles, int64_t ntiles, const int32_t* g_a,
                                        const int64_t* g_base, uint64_t rank_lo, uint64_t rank_hi, uint64_t h_bits,
                                        int64_t cap, int64_t* idx, double* vals, uint64_t* n_kept, void* stream) {
    if (!bal || !n_kept || cap < 0 || (cap > 0 && (!idx || !vals)) || rank_hi < rank_lo)
        return FRR_E_INVALID_DESIGN;
    int rc = check_nt(bal->n, bal->t);
    if (rc) return rc;
    if (ntiles <= 0) return FRR_OK;
    if (width != split_width(bal->d)) {
        frr_set_error("frr_exact_tiled_filtered: width %d for d=%d", width, bal->d);
        return FRR_E_UNSUPPORTED;
    }
    const SplitFilter f{h_bits, cap, idx, vals, reinterpret_cast<unsigned long long*>(n_kept)};
    const int64_t lo = (int64_t)rank_lo, hi = (int64_t)rank_hi;
#define FRR_TILED(W, DD) \
    case DD: return launch_tiled<W, DD>(bal, sa, sb, tiles, ntiles, g_a, g_base, lo, hi, f, stream)
    switch (bal->d) {
        FRR_TILED(4, 1); FRR_TILED(4, 2); FRR_TILED(4, 3); FRR_TILED(4, 4);
        FRR_TILED(6, 5); FRR_TILED(6, 6); FRR_TILED(8, 7); FRR_TILED(8, 8);
        FRR_TILED(16, 9); FRR_TILED(16, 10); FRR_TILED(16, 11); FRR_TILED(16, 12);
        FRR_TILED(16, 13); FRR_TILED(16, 14); FRR_TILED(16, 15); FRR_TILED(16, 16);
        default: frr_set_error("frr_exact_tiled_filtered: d=%d", bal->d); return FRR_E_UNSUPPORTED;
    }
#undef FRR_TILED
}

// frr_select.cu -- exact k-smallest acceptance (generation.py:159-169).
//
// The reference stable-argsorts all M statistics (O(M log M) on the host).
// Here: statistics are non-negative doubles, so their IEEE bit patterns
// order like the values; an 8-pass, 8-bit MSD radix select finds the exact
// threshold bit pattern T and the number of ties at T still to accept.  Ties
// are accepted in index order, which is exactly the stable-argsort rule.  An
// order-preserving compaction then emits the accepted indices ascending.
// Multi-GPU: the per-pass histogram is all-reduced between frr_select_hist
// and frr_select_pick; the tie quota is split by rank order on the host.
#include <cuda_runtime.h>

#include "frr_common.cuh"
#include "frr_launch.cuh"

namespace {

constexpr int kHistThreads = 512;
constexpr int kTile = 4096;  // compaction tile: 256 threads x 16 elements
constexpr int kCThreads = 256;
constexpr int kPer = kTile / kCThreads;

__global__ void __launch_bounds__(kHistThreads) k_hist(const uint64_t* __restrict__ bits, int64_t m,
                                                       const frr_select_state_t* st, int shift,
                                                       unsigned long long* hist) {
    __shared__ unsigned int sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t prefix = st->prefix, mask = st->mask;
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = base + threadIdx.x;
        bool ok = false;
        unsigned digit = 0;
        if (i < m) {
            uint64_t v = bits[i];
            ok = (v & mask) == prefix;
            digit = (unsigned)(v >> shift) & 255u;
        }
        unsigned active = __ballot_sync(FRR_FULL, ok);
        if (ok) {
            // warp-aggregate equal digits: stats concentrate in few bins
            unsigned peers = __match_any_sync(active, digit);
            if ((__ffs(peers) - 1) == lane) atomicAdd(&sh[digit], __popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// One warp: lane l owns bins 8l..8l+7; an inclusive warp scan of the lane
// sums finds the lane holding rank k_rem, that lane its digit.
__global__ void __launch_bounds__(32) k_pick(const unsigned long long* hist, frr_select_state_t* st, int shift) {
    const int lane = threadIdx.x;
    const int64_t k = st->k_rem;
    unsigned long long h[8], own = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        h[i] = hist[8 * lane + i];
        own += h[i];
    }
    unsigned long long incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(FRR_FULL, incl, o);
        if (lane >= o) incl += v;
    }
    // k <= total (k_rem counts ranks inside the current prefix): the first
    // lane whose inclusive sum reaches k holds the digit
    const unsigned hit = __ballot_sync(FRR_FULL, (int64_t)incl >= k);
    const int src = hit ? __ffs(hit) - 1 : 31;
    if (lane == src) {
        unsigned long long cum = incl - own;
        int digit = 8 * lane + 7;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if ((int64_t)(cum + h[i]) >= k) {
                digit = 8 * lane + i;
                break;
            }
            cum += h[i];
        }
        st->k_rem = k - (int64_t)cum;
        st->prefix |= (uint64_t)digit << shift;
        st->mask |= 255ull << shift;
    }
}

__global__ void k_init(frr_select_state_t* st, int64_t k) {
    st->prefix = 0;
    st->mask = 0;
    st->k_rem = k;
    st->pad = 0;
}

__global__ void __launch_bounds__(256) k_count(const uint64_t* __restrict__ bits, int64_t m,
                                               const frr_select_state_t* st, unsigned long long* counts) {
    const uint64_t T = st->prefix;
    unsigned long long lt = 0, eq = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t v = bits[i];
        lt += v < T;
        eq += v == T;
    }
    for (int o = 16; o > 0; o >>= 1) {
        lt += __shfl_xor_sync(FRR_FULL, lt, o);
        eq += __shfl_xor_sync(FRR_FULL, eq, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (lt) atomicAdd(counts, lt);
        if (eq) atomicAdd(counts + 1, eq);
    }
}

// per-tile (less, equal) counts
__global__ void __launch_bounds__(kCThreads) k_tile_counts(const uint64_t* __restrict__ bits, int64_t m,
                                                           const frr_select_state_t* st, int64_t* ws) {
    const uint64_t T = st->prefix;
    int64_t base = (int64_t)blockIdx.x * kTile;
    int lt = 0, eq = 0;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        int64_t i = base + (int64_t)j * kCThreads + threadIdx.x;
        if (i < m) {
            uint64_t v = bits[i];
            lt += v < T;
            eq += v == T;
        }
    }
    __shared__ int s_lt[kCThreads / 32], s_eq[kCThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        lt += __shfl_xor_sync(FRR_FULL, lt, o);
        eq += __shfl_xor_sync(FRR_FULL, eq, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_lt[threadIdx.x >> 5] = lt;
        s_eq[threadIdx.x >> 5] = eq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0, b = 0;
        for (int w = 0; w < kCThreads / 32; w++) {
            a += s_lt[w];
            b += s_eq[w];
        }
        ws[2 * blockIdx.x] = a;
        ws[2 * blockIdx.x + 1] = b;
    }
}

// exclusive scan of the tile counts (single CTA), total accepted count
// Exclusive scan of the per-tile (below, tie) counts, one CTA: 4096 tiles
// per round, 4 per thread, warp-shuffle scans, one shared-memory step for the
// warp totals (2 barriers per round instead of 20).
__device__ __forceinline__ void warp_incl_scan2(int64_t& a, int64_t& b, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t va = __shfl_up_sync(0xffffffffu, a, o), vb = __shfl_up_sync(0xffffffffu, b, o);
        if (lane >= o) {
            a += va;
            b += vb;
        }
    }
}

__global__ void __launch_bounds__(1024) k_tile_scan(int64_t* ws, int64_t ntiles, const int64_t* tie_quota,
                                                    int64_t* n_out) {
    __shared__ int64_t s_wa[32], s_wb[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t carry_a = 0, carry_b = 0;  // identical in every thread
    for (int64_t base = 0; base < ntiles; base += 4096) {
        const int64_t i0 = base + 4 * (int64_t)threadIdx.x;
        int64_t a[4], b[4], ta = 0, tb = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const bool ok = i0 + u < ntiles;
            a[u] = ok ? ws[2 * (i0 + u)] : 0;
            b[u] = ok ? ws[2 * (i0 + u) + 1] : 0;
            ta += a[u];
            tb += b[u];
        }
        int64_t ia = ta, ib = tb;
        warp_incl_scan2(ia, ib, lane);
        if (lane == 31) {
            s_wa[warp] = ia;
            s_wb[warp] = ib;
        }
        __syncthreads();
        if (warp == 0) {
            int64_t wa = s_wa[lane], wb = s_wb[lane];
            warp_incl_scan2(wa, wb, lane);
            s_wa[lane] = wa;
            s_wb[lane] = wb;
        }
        __syncthreads();
        int64_t ea = carry_a + (warp ? s_wa[warp - 1] : 0) + ia - ta;
        int64_t eb = carry_b + (warp ? s_wb[warp - 1] : 0) + ib - tb;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            if (i0 + u < ntiles) {
                ws[2 * (i0 + u)] = ea;
                ws[2 * (i0 + u) + 1] = eb;
            }
            ea += a[u];
            eb += b[u];
        }
        carry_a += s_wa[31];
        carry_b += s_wb[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int64_t q = *tie_quota;
        if (q > carry_b) q = carry_b;
        if (q < 0) q = 0;
        *n_out = carry_a + q;
    }
}

__global__ void __launch_bounds__(kCThreads) k_compact(const uint64_t* __restrict__ bits, int64_t m, int64_t index_base,
                                                       const frr_select_state_t* st, const int64_t* tie_quota,
                                                       const int64_t* ws, int64_t cap, int64_t* idx_out,
                                                       double* stat_out) {
    const uint64_t T = st->prefix;
    const int64_t quota = *tie_quota;
    // coalesced tile load through shared memory (row stride kPer+1 words:
    // 2-way bank conflicts), then thread-contiguous runs of kPer elements
    __shared__ uint64_t s_tile[kCThreads * (kPer + 1)];
    const int64_t tile0 = (int64_t)blockIdx.x * kTile;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        const int e = j * kCThreads + threadIdx.x;  // element of the tile
        const int64_t i = tile0 + e;
        s_tile[(e / kPer) * (kPer + 1) + e % kPer] = i < m ? bits[i] : ~0ull;
    }
    __syncthreads();
    int64_t base = tile0 + (int64_t)threadIdx.x * kPer;  // thread-contiguous run
    uint64_t v[kPer];
    int lt = 0, eq = 0;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        v[j] = s_tile[threadIdx.x * (kPer + 1) + j];
        lt += v[j] < T;
        eq += v[j] == T;
    }
    // block exclusive scan of (lt, eq) in thread order: warp shuffles, then
    // the 8 warp totals (one barrier)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int il = lt, ie = eq;  // inclusive within the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(FRR_FULL, il, o), b = __shfl_up_sync(FRR_FULL, ie, o);
        if (lane >= o) {
            il += a;
            ie += b;
        }
    }
    __shared__ int s_wl[kCThreads / 32], s_we[kCThreads / 32];
    if (lane == 31) {
        s_wl[wid] = il;
        s_we[wid] = ie;
    }
    __syncthreads();
    int bl = 0, be = 0;
    for (int w = 0; w < wid; w++) {
        bl += s_wl[w];
        be += s_we[w];
    }
    int64_t lrank = ws[2 * blockIdx.x] + bl + il - lt;
    int64_t erank = ws[2 * blockIdx.x + 1] + be + ie - eq;
#pragma unroll
    for (int j = 0; j < kPer; j++) {
        bool less = v[j] < T, tie = v[j] == T;
        if (less || (tie && erank < quota)) {
            int64_t pos = lrank + (erank < quota ? erank : quota);
            if (pos < cap) {
                idx_out[pos] = index_base + base + j;
                stat_out[pos] = __longlong_as_double((long long)v[j]);
            }
        }
        lrank += less;
        erank += tie;
    }
}

}  // namespace

extern "C" int frr_select_init(frr_select_state_t* st, int64_t k, void* stream) {
    k_init<<<1, 1, 0, frr_stream(stream)>>>(st, k);
    return frr_launched("k_init");
}

extern "C" int frr_select_hist(const double* stats, int64_t m, const frr_select_state_t* st, int pass,
                               uint64_t* hist, void* stream) {
    if (pass < 0 || pass > 7) {
        frr_set_error("select pass %d outside [0, 7]", pass);
        return FRR_E_INVALID_DESIGN;
    }
    cudaStream_t s = frr_stream(stream);
    if (cudaMemsetAsync(hist, 0, 256 * sizeof(uint64_t), s) != cudaSuccess) return frr_check_launch("hist memset");
    if (m <= 0) return FRR_OK;
    int grid = (int)std::min<int64_t>(frr_cdiv(m, kHistThreads), (int64_t)frr_num_sms() * 4);
    k_hist<<<grid, kHistThreads, 0, s>>>(reinterpret_cast<const uint64_t*>(stats), m, st, 56 - 8 * pass,
                                         reinterpret_cast<unsigned long long*>(hist));
    return frr_launched("k_hist");
}

extern "C" int frr_select_pick(const uint64_t* hist, frr_select_state_t* st, int pass, void* stream) {
    k_pick<<<1, 32, 0, frr_stream(stream)>>>(reinterpret_cast<const unsigned long long*>(hist), st, 56 - 8 * pass);
    return frr_launched("k_pick");
}

extern "C" int frr_select_count(const double* stats, int64_t m, const frr_select_state_t* st, int64_t* counts,
                                void* stream) {
    cudaStream_t s = frr_stream(stream);
    if (cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), s) != cudaSuccess) return frr_check_launch("count memset");
    if (m <= 0) return FRR_OK;
    int grid = (int)std::min<int64_t>(frr_cdiv(m, 256), (int64_t)frr_num_sms() * 8);
    k_count<<<grid, 256, 0, s>>>(reinterpret_cast<const uint64_t*>(stats), m, st,
                                 reinterpret_cast<unsigned long long*>(counts));
    return frr_launched("k_count");
}

extern "C" size_t frr_select_workspace_bytes(int64_t m) {
    return (size_t)std::max<int64_t>(1, frr_cdiv(m, kTile)) * 2 * sizeof(int64_t);
}

extern "C" int frr_select_compact(const double* stats, int64_t m, int64_t index_base, const frr_select_state_t* st,
                                  const int64_t* tie_quota, int64_t* idx_out, double* stat_out, int64_t* n_out,
                                  void* workspace, void* stream) {
    return frr_select_compact_capped(stats, m, index_base, st, tie_quota, INT64_MAX, idx_out, stat_out, n_out,
                                     workspace, stream);
}

extern "C" int frr_select_compact_capped(const double* stats, int64_t m, int64_t index_base,
                                         const frr_select_state_t* st, const int64_t* tie_quota, int64_t cap,
                                         int64_t* idx_out, double* stat_out, int64_t* n_out, void* workspace,
                                         void* stream) {
    cudaStream_t s = frr_stream(stream);
    int64_t ntiles = frr_cdiv(m, kTile);
    if (m <= 0) {
        if (cudaMemsetAsync(n_out, 0, sizeof(int64_t), s) != cudaSuccess) return frr_check_launch("n_out memset");
        return FRR_OK;
    }
    int64_t* ws = reinterpret_cast<int64_t*>(workspace);
    const uint64_t* bits = reinterpret_cast<const uint64_t*>(stats);
    k_tile_counts<<<(unsigned)ntiles, kCThreads, 0, s>>>(bits, m, st, ws);
    int rc = frr_launched("k_tile_counts");
    if (rc) return rc;
    k_tile_scan<<<1, 1024, 0, s>>>(ws, ntiles, tie_quota, n_out);
    if ((rc = frr_launched("k_tile_scan"))) return rc;
    k_compact<<<(unsigned)ntiles, kCThreads, 0, s>>>(bits, m, index_base, st, tie_quota, ws, cap, idx_out,
                                                     stat_out);
    return frr_launched("k_compact");
}

// ------------------------------------------------- (key, value) pair sort
// Stable LSD radix sort of uint64 keys carrying 8-byte values, 8-bit digits:
// the fused exact pass keeps its (rank, statistic) pairs in arrival order,
// the select and the pool want them by rank.  Per pass: per-tile digit
// counts, one exclusive scan over [digit][tile], then a stable scatter --
// every tile walks its elements in index order, 256 per round, ranking equal
// digits inside a warp with __match_any_sync and across warps / rounds
// through shared counters.
namespace {
constexpr int kSortThreads = 256, kSortRounds = 8, kSortTile = kSortThreads * kSortRounds;

__global__ void __launch_bounds__(kSortThreads) k_sort_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                            uint32_t* counts, int64_t ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; r++) {
        const int64_t i = base + r * kSortThreads + threadIdx.x;
        const bool ok = i < n;
        const unsigned d = ok ? (unsigned)(keys[i] >> shift) & 255u : 0u;
        const unsigned act = __ballot_sync(FRR_FULL, ok);
        if (ok) {
            const unsigned peers = __match_any_sync(act, d);
            if ((__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// CTA d: exclusive scan of digit d's per-tile counts counts[d][0, ntiles) in
// place, and the digit's total
__global__ void __launch_bounds__(1024) k_sort_scan(uint32_t* counts, int64_t ntiles, uint32_t* totals) {
    __shared__ uint32_t warp_sum[32];
    __shared__ uint32_t carry;
    uint32_t* row = counts + (int64_t)blockIdx.x * ntiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < ntiles; c0 += 1024) {
        const int64_t i = c0 + threadIdx.x;
        const uint32_t v = i < ntiles ? row[i] : 0u;
        uint32_t x = v;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FRR_FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = warp_sum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FRR_FULL, w, o);
                if (lane >= o) w += y;
            }
            warp_sum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const uint32_t before = carry + (warp ? warp_sum[warp - 1] : 0u) + x - v;
        if (i < ntiles) row[i] = before;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(kSortThreads) k_sort_scatter(const uint64_t* __restrict__ kin,
                                                               const uint64_t* __restrict__ vin, int64_t n, int shift,
                                                               const uint32_t* __restrict__ offs, int64_t ntiles,
                                                               const uint32_t* __restrict__ totals,
                                                               uint64_t* __restrict__ kout,
                                                               uint64_t* __restrict__ vout) {
    constexpr int NW = kSortThreads / 32;
    __shared__ uint32_t run[256];
    __shared__ uint32_t wc[NW][256];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {  // digit base: exclusive scan of the digit totals (one per thread)
        const uint32_t tv = totals[tid];
        uint32_t x = tv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FRR_FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wc[0][warp] = x;
        __syncthreads();
        uint32_t wb = 0;
        for (int w = 0; w < warp; w++) wb += wc[0][w];
        __syncthreads();
        run[tid] = wb + x - tv + offs[(int64_t)tid * ntiles + blockIdx.x];
    }
    for (int w = 0; w < NW; w++) wc[w][tid] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; r++) {
        const int64_t i = base + r * kSortThreads + tid;
        const bool ok = i < n;
        uint64_t k = 0, v = 0;
        unsigned d = 0, peers = 0;
        const unsigned act = __ballot_sync(FRR_FULL, ok);
        if (ok) {
            k = kin[i];
            v = vin[i];
            d = (unsigned)(k >> shift) & 255u;
            peers = __match_any_sync(act, d);
            if ((__ffs(peers) - 1) == lane) wc[warp][d] = __popc(peers);
        }
        __syncthreads();
        if (ok) {
            uint32_t before = run[d] + __popc(peers & ((1u << lane) - 1u));
            for (int w = 0; w < warp; w++) before += wc[w][d];
            kout[before] = k;
            vout[before] = v;
        }
        __syncthreads();
        uint32_t tot = 0;  // thread tid: digit tid's count in this round
        for (int w = 0; w < NW; w++) {
            tot += wc[w][tid];
            wc[w][tid] = 0;
        }
        run[tid] += tot;
        __syncthreads();
    }
}
}  // namespace

extern "C" size_t frr_sort_pairs_workspace_bytes(int64_t n) {
    const int64_t ntiles = std::max<int64_t>(1, frr_cdiv(n, kSortTile));
    return (size_t)std::max<int64_t>(n, 1) * 16 + ((size_t)ntiles + 1) * 256 * sizeof(uint32_t);
}

extern "C" int frr_sort_pairs(uint64_t* keys, uint64_t* vals, int64_t n, int key_bits, void* workspace,
                              size_t ws_bytes, void* stream) {
    if (n <= 1) return FRR_OK;
    if (key_bits < 1 || key_bits > 64 || ws_bytes < frr_sort_pairs_workspace_bytes(n)) {
        frr_set_error("frr_sort_pairs: key_bits in [1, 64] and frr_sort_pairs_workspace_bytes(n) of workspace");
        return FRR_E_INVALID_DESIGN;
    }
    if (n > 0xFFFFFFFFll) {
        frr_set_error("frr_sort_pairs: n < 2^32");
        return FRR_E_UNSUPPORTED;
    }
    cudaStream_t s = frr_stream(stream);
    const int64_t ntiles = frr_cdiv(n, kSortTile);
    uint64_t* kt = static_cast<uint64_t*>(workspace);
    uint64_t* vt = kt + n;
    uint32_t* counts = reinterpret_cast<uint32_t*>(vt + n);
    uint32_t* totals = counts + (size_t)ntiles * 256;
    uint64_t *ka = keys, *va = vals, *kb = kt, *vb = vt;
    const int passes = (key_bits + 7) / 8;
    int rc;
    for (int p = 0; p < passes; p++) {
        k_sort_hist<<<(unsigned)ntiles, kSortThreads, 0, s>>>(ka, n, 8 * p, counts, ntiles);
        if ((rc = frr_launched("k_sort_hist"))) return rc;
        k_sort_scan<<<256, 1024, 0, s>>>(counts, ntiles, totals);
        if ((rc = frr_launched("k_sort_scan"))) return rc;
        k_sort_scatter<<<(unsigned)ntiles, kSortThreads, 0, s>>>(ka, va, n, 8 * p, counts, ntiles, totals, kb, vb);
        if ((rc = frr_launched("k_sort_scatter"))) return rc;
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {  // odd pass count: the result is in the workspace
        if (cudaMemcpyAsync(keys, ka, (size_t)n * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(vals, va, (size_t)n * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return frr_check_launch("frr_sort_pairs copy");
    }
    return FRR_OK;
}

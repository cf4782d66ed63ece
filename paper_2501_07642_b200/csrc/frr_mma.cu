// frr_mma.cu -- fused Monte Carlo generation + tensor-core balance check.
//
// Replaces generation.py:185-204 (_pass1_stats) = keys.py:177-208 feeding
// balance.py:93-105 for mid-size d.  Per 128-candidate tile:
//
//   generator       GEN 1 (default): thread per candidate (frr_rev_fy, the
//   warps           reverse-bitset Fisher-Yates), each warp builds 32 rows of
//                   a tile buffer in place; GEN 0 (large n, whose bitsets do
//                   not fit): warp per candidate (frr_warp_fy) into a smem
//                   table, packed to the row.  Rows never leave the SM.
//   tile warps (4)  expand bit rows to int8 0/1 A-operand K-chunks in the
//                   tcgen05 K-major canonical layout; later the epilogue
//   TMA warp        cp.async.bulk of the pre-tiled int8-limb B operand
//                   (Zq split into L balanced base-256 digits, N = L*dpad)
//   MMA warp        tcgen05.mma.cta_group::1.kind::i8, int32 accumulators
//                   in TMEM (128 lanes x N columns)
//   epilogue        tcgen05.ld, S_j = sum_l acc_l * 256^l (exact int64),
//                   fp64 delta^2 with numpy's pairwise order, * const
//
// S = W . Zq is exact in every limb (|acc| <= 128 n < 2^31), so the
// statistic is bit-identical to the reference's float64 BLAS path.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "frr_common.cuh"
#include "frr_launch.cuh"
#include "frr_revfy.cuh"
#include "frr_tc.cuh"

namespace {
using namespace frr_tc;

constexpr int BM = 128;        // candidates per tile = MMA M
#ifndef FRR_MMA_TW
#define FRR_MMA_TW 1  // 2 measured -2% (20 generators + 8 tile warps vs 24 + 4)
#endif
#ifndef FRR_MMA_NFY
#define FRR_MMA_NFY 20  // the launch bound: 28 warps -> 72 registers per thread (26: 32 warps, 64)
#endif
#ifndef FRR_MMA_KC
#define FRR_MMA_KC 64
#endif
#ifndef FRR_MMA_STAGES
#define FRR_MMA_STAGES 3
#endif
#ifndef FRR_MMA_NBITS
#define FRR_MMA_NBITS 3
#endif
constexpr int KC = FRR_MMA_KC;  // K bytes per pipeline stage
constexpr int NBITS = FRR_MMA_NBITS;  // max bit-row tile buffers between generators and tile warps
constexpr int A_STAGES = FRR_MMA_STAGES;
// A operand in TMEM (tcgen05.st of the 0/1 bytes; the MMA reads A from TMEM)
// whenever the accumulator leaves room for >= 2 K stages of KC / 4 columns
#ifndef FRR_MMA_TMEM_A
#define FRR_MMA_TMEM_A 0
#endif
constexpr int A_TSTAGES = 8;  // max TMEM A stages
constexpr int A_SLOTS = A_STAGES > A_TSTAGES ? A_STAGES : A_TSTAGES;
#ifndef FRR_MMA_BSTAGES
#define FRR_MMA_BSTAGES FRR_MMA_STAGES
#endif
constexpr int B_STAGES = FRR_MMA_BSTAGES;
constexpr int NFY = FRR_MMA_NFY;  // max generator warps (fewer for large n: their tables share smem)
// thread-per-candidate generators: RFY warps (4 per tile in flight, a
// multiple of 4) building rows in place in RBITS tile buffers
// tile warps per TMEM lane quadrant (FRR_MMA_TW, above): 2 split each
// tile's expansion (K chunks by parity) and epilogue (columns 0-3 / 4-7 of
// every 8-group: numpy's accumulator streams r0-3 / r4-7, joined through
// shared memory)
#ifndef FRR_MMA_RFY
#define FRR_MMA_RFY 20  // 20 generators at 72 registers beat 24 at 64 by 1% (16 at 80: -1.7%)
#endif
#ifndef FRR_MMA_RBITS
#define FRR_MMA_RBITS 8
#endif
#ifndef FRR_MMA_SPARE
#define FRR_MMA_SPARE 2  // tile buffers beyond the RFY / 4 being built
#endif
constexpr int RFY = FRR_MMA_RFY;
constexpr int TW2 = FRR_MMA_TW;
static_assert(TW2 == 1 || TW2 == 2, "tile warps per quadrant");
constexpr int RBITS = FRR_MMA_RBITS;
constexpr int MAXBITS = NBITS > RBITS ? NBITS : RBITS;
// Wait-time accounting (debug builds only): per-slot clock64 sums read back
// with frr_debug_waits().
#ifndef FRR_MMA_TIMING
#define FRR_MMA_TIMING 0
#endif
#if FRR_MMA_TIMING
__device__ unsigned long long g_frr_waits[16];
#define TW(slot, ...)                          \
    do {                                       \
        const long long t0_ = clock64();       \
        __VA_ARGS__;                           \
        wacc[slot] += clock64() - t0_;         \
    } while (0)
#else
#define TW(slot, ...) \
    do {              \
        __VA_ARGS__;  \
    } while (0)
#endif
// epilogue limb recombination through 32-bit limb pairs (tc_limbs8_pairs)
#ifndef FRR_MMA_PAIRS
#define FRR_MMA_PAIRS 1
#endif
// L = 6 epilogue: all limbs of 4 columns per TMEM round trip, software-pipelined
#ifndef FRR_MMA_STAGGER
#define FRR_MMA_STAGGER 0  // cycles: odd generator groups' start delay
#endif
#ifndef FRR_MMA_EPI_PIPE
#define FRR_MMA_EPI_PIPE 0  // measured: no gain (the epilogue is not TMEM-latency bound)
#endif
// timing experiments only (results invalid): 1 no Fisher-Yates, 4 no epilogue,
// 8 generators only (tile, copy and MMA roles just recycle the bit buffers)
#ifndef FRR_MMA_DEBUG
#define FRR_MMA_DEBUG 0
#endif
// Warp roles (per shape, see mma_shape): generators 0..nfy-1, then the bulk
// copy and MMA warps, then the 4 tile warps at a multiple of 4 (warp % 4 is
// their TMEM lane quadrant).  The scheduler favours higher warp ids, so the
// latency-critical roles sit above the generators.
constexpr int NTHREADS_MAX = ((((NFY > RFY ? NFY : RFY) + 2 + 3) & ~3) + 4 * TW2) * 32;
constexpr int NTHREADS = NTHREADS_MAX;  // launch bound: the largest layout
static_assert(NTHREADS <= 1024, "roles exceed one CTA (FRR_MMA_TW=2 needs FRR_MMA_NFY <= 20)");
constexpr int A_STAGE_BYTES = BM * KC;

struct MmaShape {
    int n, t, d, L, dpad, npad, kpad, nkc, kw;  // kw: 32-bit words per bit row
    int nparts, part_n[2], part_off[2];
    int gen;                                     // 1: thread-per-candidate generators, 0: warp per candidate
    int ta, nsta;                                // A in TMEM (columns [npad, npad + nsta KC/4)), A stages
    int nfy, nbits;                              // generator warps, bit-row buffers
    int steps_smem;                              // step table in shared (1) or global memory
    int w_tma, w_mma, w_tile0, nwarps;           // warp roles
};

struct SmemPlan {
    size_t steps, tables, bits, a, b, xch, bars, total;
};

// Tile buffer of 128 bit rows, kw words each, laid out [row / 32][word][row % 32]
// (uint32): a thread-per-candidate generator owns one column of a 32-row
// block and every access of a warp hits 32 distinct banks.  Bit b of word w
// = unit 32 w + b is a CONTROL unit (padding beyond n reads as control).
__host__ __device__ inline size_t bits_buf_bytes(int kw) { return (size_t)BM * kw * 4; }

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemPlan smem_plan(const MmaShape& s) {
    SmemPlan p;
    size_t o = 0;
    p.a = o;
    if (!s.ta) o += (size_t)A_STAGES * A_STAGE_BYTES;
    p.b = o;
    o += (size_t)B_STAGES * s.npad * KC;
    p.bits = o;
    o += (size_t)s.nbits * bits_buf_bytes(s.kw);
    p.steps = o;
    if (s.steps_smem) o += (size_t)frr_steps_len(s.t) * sizeof(StepC);
    p.tables = o;
    // GEN 0: one table per generator warp; GEN 1: one shared scratch table
    // for the exact recomputation of flagged candidates (+ its lock word)
    o += (size_t)(s.gen ? 1 : s.nfy) * frr_table_len(s.n) * 2;
    if (s.gen) o = align_up(o + FRR_TABLE_SLACK, 16) + 16;
    o = align_up(o, 16);
    p.xch = o;  // split epilogue: half sums handed between a quadrant's two tile warps
    o += TW2 == 2 ? BM * sizeof(double) : 0;
    o = align_up(o, 16);
    p.bars = o;
    o += 48 * 8 + 16;  // barriers + TMEM slot: also the FRR_TABLE_SLACK after the tables
    static_assert(48 * 8 + 16 >= FRR_TABLE_SLACK, "table slack");
    p.total = o + 1024;  // slack for base alignment
    return p;
}

__host__ __device__ inline void set_roles(MmaShape& s, int nfy, int nbits) {
    s.nfy = nfy;
    s.nbits = nbits;
    s.w_tma = nfy;
    s.w_mma = nfy + 1;
    s.w_tile0 = (nfy + 2 + 3) & ~3;
    s.nwarps = s.w_tile0 + 4 * TW2;
}

__host__ __device__ inline MmaShape mma_shape(int n, int t, int d, int L) {
    MmaShape s;
    s.n = n;
    s.t = t;
    s.d = d;
    s.L = L;
    s.dpad = (d + 15) & ~15;
    s.npad = L * s.dpad;
    s.kpad = (n + KC - 1) / KC * KC;
    s.nkc = s.kpad / KC;
    s.kw = s.kpad / 32;
    s.nparts = s.npad > 256 ? 2 : 1;
    // split N into <=256-column parts, each a multiple of 16
    s.part_n[0] = s.nparts == 1 ? s.npad : ((s.npad / 2 + 15) & ~15);
    s.part_n[1] = s.npad - s.part_n[0];
    s.part_off[0] = 0;
    s.part_off[1] = s.part_n[0];
    s.ta = FRR_MMA_TMEM_A && s.npad + 2 * (KC / 4) <= 512;
    s.nsta = s.ta ? min(A_TSTAGES, (512 - s.npad) / (KC / 4)) : A_STAGES;
    // Thread-per-candidate generators when their tile buffers fit: RFY / 4
    // tiles being built plus two being consumed, at least 8 generator warps.
    s.gen = 1;
    s.steps_smem = 1;
    for (int f = RFY; f >= 8; f -= 4) {
        const int nb = f / 4 + FRR_MMA_SPARE <= RBITS ? f / 4 + FRR_MMA_SPARE : RBITS;
        set_roles(s, f, nb);
        if (smem_plan(s).total <= 227 * 1024) return s;
    }
    s.gen = 0;
    // Largest generator count with at least two bit buffers that fits shared
    // memory (tables are 2n bytes per generator, bit buffers n/8 per row);
    // large n falls back to one buffer and as few as 4 generators.
    // The step table (16 B per step) moves to global memory (L1-cached) when
    // keeping it would cost generators or buffers.
    for (int ss = 1; ss >= 0; ss--) {
        s.steps_smem = ss;
        for (int nb = NBITS; nb >= 1; nb--) {
            for (int f = NFY; f >= (nb >= 2 ? 8 : 4); f--) {
                set_roles(s, f, nb);
                if (smem_plan(s).total <= 227 * 1024 && (ss == 0 || (f == NFY && nb == NBITS))) return s;
            }
        }
    }
    set_roles(s, 0, 0);  // does not fit: tc_layout rejects the shape
    return s;
}

// barrier slots
constexpr int BAR_BITS_FULL = 0, BAR_BITS_EMPTY = MAXBITS;
constexpr int BAR_A_FULL = 2 * MAXBITS, BAR_A_EMPTY = BAR_A_FULL + A_SLOTS;
constexpr int BAR_B_FULL = BAR_A_EMPTY + A_SLOTS, BAR_B_EMPTY = BAR_B_FULL + B_STAGES;
constexpr int BAR_TMEM_FULL = BAR_B_EMPTY + B_STAGES, BAR_TMEM_EMPTY = BAR_TMEM_FULL + 1;
constexpr int N_BARS = BAR_TMEM_EMPTY + 1;
static_assert(N_BARS <= 46, "barrier slots");

// GEN 1: thread-per-candidate generators (step table in shared memory).
// GEN 0, GS: step table in global memory (large n), else in shared memory.
// FULL: the default generator/buffer counts as compile-time constants.
template <bool GS, bool FULL, int GEN>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_mc_stats_mma(frr_balance_t bal, uint64_t seed, uint64_t lo, int64_t count, double* __restrict__ out,
                   const StepC* __restrict__ gsteps) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // keep the shared address space visible to the compiler (LDS/STS, not
    // generic LD/ST): align by offsetting the __shared__ array itself
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const MmaShape S = mma_shape(bal.n, bal.t, bal.d, bal.n_limbs);
    const SmemPlan P = smem_plan(S);
    // FULL: the default layout (NFY / RFY generators, NBITS / RBITS buffers)
    // as compile-time constants -- the fast path; otherwise the shape's
    // reduced layout
    const int c_nfy = FULL ? (GEN ? RFY : NFY) : S.nfy, c_nbits = FULL ? (GEN ? RBITS : NBITS) : S.nbits;
    const int c_w_tma = c_nfy, c_w_mma = c_nfy + 1, c_w_tile0 = (c_nfy + 2 + 3) & ~3;
    unsigned char* sA = smem + P.a;
    unsigned char* sB = smem + P.b;
    uint32_t* sBits = reinterpret_cast<uint32_t*>(smem + P.bits);
    StepC* ssteps = reinterpret_cast<StepC*>(smem + P.steps);
    uint16_t* tables = reinterpret_cast<uint16_t*>(smem + P.tables);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.bars);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 46);
    // GEN 1: lock of the shared fixup table (last 16 bytes before the barriers)
    int* fix_lock = reinterpret_cast<int*>(smem + P.xch - 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (count + BM - 1) / BM;
    const size_t buf_words = (size_t)BM * S.kw;
#if FRR_MMA_TIMING
    long long wacc[16] = {0};
    const long long tstart = clock64();
#endif

    if (!GS) frr_fill_steps(ssteps, S.n, S.t);
    if (threadIdx.x == 0) {
        if (GEN) *fix_lock = 0;
        for (int b = 0; b < c_nbits; b++) {
            mbar_init(&bars[BAR_BITS_FULL + b], GEN ? 4 : c_nfy);
            mbar_init(&bars[BAR_BITS_EMPTY + b], 4 * TW2);
        }
        for (int s = 0; s < S.nsta; s++) {
            mbar_init(&bars[BAR_A_FULL + s], 4);
            mbar_init(&bars[BAR_A_EMPTY + s], 1);
        }
        for (int s = 0; s < B_STAGES; s++) {
            mbar_init(&bars[BAR_B_FULL + s], 1);
            mbar_init(&bars[BAR_B_EMPTY + s], 1);
        }
        mbar_init(&bars[BAR_TMEM_FULL], 1);
        mbar_init(&bars[BAR_TMEM_EMPTY], 4 * TW2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    if (warp == c_w_mma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (GEN && warp < c_nfy) {
        // ================================ thread-per-candidate generators
        // warp g builds quadrant g % 4 (rows 32 q .. 32 q + 31) of the
        // CTA's tiles g / 4, g / 4 + nfy / 4, ... in place in their buffers
        const int q = warp & 3, kstep = c_nfy >> 2;
        const uint32_t sst = smem_u32(ssteps);
#if FRR_MMA_STAGGER
        // desynchronise the tile groups' rounds: odd groups start half a job late
        if ((warp >> 2) & 1) {
            const long long t_end = clock64() + (long long)FRR_MMA_STAGGER;
            while (clock64() < t_end) __nanosleep(1000);
        }
#endif
        for (int64_t k = warp >> 2;; k += kstep) {
            const int64_t tile = blockIdx.x + k * gridDim.x;
            if (tile >= ntiles) break;
            const int buf = (int)(k % c_nbits);
            TW(0, mbar_wait_long(&bars[BAR_BITS_EMPTY + buf], ((k / c_nbits) & 1) ^ 1));
            const uint32_t blk = smem_u32(sBits + (size_t)buf * buf_words + (size_t)q * S.kw * 32);
            const uint64_t state = frr_derive_state(seed, lo + (uint64_t)(tile * BM + 32 * q + lane));
            bool flag = false;
            if (!(FRR_MMA_DEBUG & 1)) TW(11, flag = frr_rev_fy(state, S.t, sst, blk + 4u * lane, S.kw));
            uint32_t fl = __ballot_sync(FRR_FULL, flag);
            while (fl) {  // p ~ 1e-7 per candidate: exact recomputation in the shared scratch table
                const int src = __ffs(fl) - 1;
                fl &= fl - 1;
                if (lane == 0)
                    while (atomicCAS(fix_lock, 0, 1) != 0) __nanosleep(100);
                __syncwarp();
                frr_rev_fixup(__shfl_sync(FRR_FULL, state, src), S.n, S.t, ssteps, tables, blk + 4u * src, S.kw,
                              lane);
                if (lane == 0) atomicExch(fix_lock, 0);
                __syncwarp();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[BAR_BITS_FULL + buf]);
        }
    } else if (!GEN && warp < c_nfy) {
        // ===================================== warp-per-candidate generators
        const int fyw = warp;
        uint16_t* lw = tables + (size_t)fyw * frr_table_len(S.n);
        int i = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, i++) {
            const int buf = i % c_nbits;
            TW(0, mbar_wait_long(&bars[BAR_BITS_EMPTY + buf], ((i / c_nbits) & 1) ^ 1));
            uint32_t* tb = sBits + (size_t)buf * buf_words;
            for (int r = fyw; r < BM; r += c_nfy) {
                const int64_t c = tile * BM + r;
                uint32_t* row = tb + (size_t)(r >> 5) * S.kw * 32 + (r & 31);
                if (c < count && !(FRR_MMA_DEBUG & 1)) {
                    TW(11, frr_warp_fy<GS>(frr_derive_state(seed, lo + (uint64_t)c), S.n, S.t, GS ? gsteps : ssteps,
                                       lw, lane));
                    // control bits in natural unit order, one ballot per word
                    for (int w = 0; w < S.kw; w++) {
                        const int e = 32 * w + lane;
                        const uint32_t word = __ballot_sync(FRR_FULL, e >= S.n || lw[e] == FRR_CTL);
                        if (lane == (w & 31)) row[(size_t)w * 32] = word;
                    }
                } else {
                    for (int w = lane; w < S.kw; w += 32) row[(size_t)w * 32] = ~0u;
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(&bars[BAR_BITS_FULL + buf]);
        }
    } else if (warp >= c_w_tile0 && warp < c_w_tile0 + 4 * TW2) {
        // ============================================ expansion + epilogue
        // quadrant warp `half` (of TW2) expands the K chunks kc % TW2 == half and,
        // with TW2 = 2, evaluates columns 4 half .. 4 half + 3 of every 8-group
        const int quad = (warp - c_w_tile0) & 3, half = (warp - c_w_tile0) >> 2;
        const int r = quad * 32 + lane;  // tile row == TMEM lane (warp % 4 = lane quadrant)
        const double g = bal.g, cst = bal.cst;
        const int d = S.d, full = d - (d % 8);
        // |acc| <= 128 n would allow 32-bit limb pairs, but here (64-register
        // budget, generator-bound kernel) the per-limb chain measured 1% faster
        const bool pair32 = false;
        int i = 0;
        uint32_t astage = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, i++) {
            const int buf = i % c_nbits;
            TW(1, mbar_wait_long(&bars[BAR_BITS_FULL + buf], (i / c_nbits) & 1));
            if (FRR_MMA_DEBUG & 8) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars[BAR_BITS_EMPTY + buf]);
                continue;
            }
            // row r: word w at [r / 32][w][r % 32]; control bits -> treated
            const uint32_t* row = sBits + (size_t)buf * buf_words + (size_t)(r >> 5) * S.kw * 32 + (r & 31);
            // A stages in TMEM: this warp's lane quadrant, columns after the accumulator
            const uint32_t a_tl = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)S.npad;
            for (int kc = 0; kc < S.nkc; kc++, astage++) {
                if (TW2 == 2 && (kc & 1) != half) continue;
                const int s = astage % S.nsta;
                TW(2, mbar_wait(&bars[BAR_A_EMPTY + s], ((astage / S.nsta) & 1) ^ 1));
                const uint32_t* src = row + (size_t)kc * (KC / 32) * 32;
                uint32_t wv[KC / 32];
#pragma unroll
                for (int q = 0; q < KC / 32; q++) wv[q] = ~src[q * 32];
                if (S.ta) {
                    // register q of word w: K offsets 4q..4q+3 of its 32-group = column 8w + q
                    tc_fence_after();
                    uint32_t v[KC / 4];
#pragma unroll
                    for (int q = 0; q < KC / 4; q++) v[q] = (wv[q >> 3] >> (q & 7)) & 0x01010101u;
                    tc_st16(a_tl + (uint32_t)(s * (KC / 4)), v);
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars[BAR_A_FULL + s]);
                    continue;
                }
                unsigned char* dst = sA + (size_t)s * A_STAGE_BYTES + (r >> 3) * 128 + (r & 7) * 16;
#pragma unroll
                for (int k16 = 0; k16 < KC / 16; k16++) {
                    // bytes 4j..4j+3 of this slab: (w >> (4*half + j)) & 0x01010101
                    // (K offset 4q + b <- bit 8b + q of the word: frr_k_unit_nat)
                    const uint32_t w = wv[k16 >> 1];
                    const int q0 = (k16 & 1) * 4;
                    uint4 o;
                    o.x = (w >> (q0 + 0)) & 0x01010101u;
                    o.y = (w >> (q0 + 1)) & 0x01010101u;
                    o.z = (w >> (q0 + 2)) & 0x01010101u;
                    o.w = (w >> (q0 + 3)) & 0x01010101u;
                    *reinterpret_cast<uint4*>(dst + (size_t)k16 * (BM / 8) * 128) = o;
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars[BAR_A_FULL + s]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[BAR_BITS_EMPTY + buf]);

            // ---------------- epilogue: TMEM -> exact S -> fp64 statistic
            TW(3, mbar_wait_long(&bars[BAR_TMEM_FULL], i & 1));
#if FRR_MMA_TIMING
            const long long t_epi0 = clock64();
#endif
            tc_fence_after();
            const uint32_t tl = tmem_base + ((uint32_t)(quad * 32) << 16);
            double res = -0.0;
            if (TW2 == 2) {
                // d <= 128: one leaf of numpy's pairwise sum.  This warp's 4 of the
                // 8 accumulator streams, then ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7))
                // across the pair of warps, then half 0 adds the tail in order.
                double ra[4];
#pragma unroll
                for (int u = 0; u < 4; u++) ra[u] = 0.0;
                for (int jb = 0; jb < ((FRR_MMA_DEBUG & 4) ? 0 : full); jb += 8) {
                    int64_t Sj[4];
                    tc_limbs4(tl + (uint32_t)(jb + 4 * half), S.L, S.dpad, true, Sj);
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const double delta =
                            __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u]), g), bal.cc[jb + 4 * half + u]);
                        const double q = __dmul_rn(delta, delta);
                        ra[u] = jb == 0 ? q : __dadd_rn(ra[u], q);
                    }
                }
                int64_t St[8];
                if (half == 0 && full < d && !(FRR_MMA_DEBUG & 4)) tc_limbs8(tl + (uint32_t)full, S.L, S.dpad, true, St);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars[BAR_TMEM_EMPTY]);
                double* xch = reinterpret_cast<double*>(smem + P.xch);
                const double part = __dadd_rn(__dadd_rn(ra[0], ra[1]), __dadd_rn(ra[2], ra[3]));
                if (half == 1) xch[r] = part;
                asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
                if (half == 0) {
                    res = __dadd_rn(part, xch[r]);
                    if (!(FRR_MMA_DEBUG & 4))
                        for (int u = 0; u < 8; u++)
                            if (full + u < d) {
                                const double delta =
                                    __dsub_rn(__dmul_rn(__ll2double_rn(St[u]), g), bal.cc[full + u]);
                                res = __dadd_rn(res, __dmul_rn(delta, delta));
                            }
                    const int64_t c = tile * BM + r;
                    if (c < count) out[c] = __dmul_rn(__dadd_rn(0.0, res), cst);
                }
                // half 0 has read xch[r] before half 1 may rewrite it next tile
                asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
                continue;
            }
            // d <= 128 here: one leaf of numpy's pairwise sum -- 8 accumulators
            // over the full groups, their tree, then the tail added in order
            double racc[8];
#pragma unroll
            for (int k = 0; k < 8; k++) racc[k] = 0.0;
            int jb0 = 0;  // first group left for the generic loop below
            if (FRR_MMA_EPI_PIPE && S.L == 6 && !(FRR_MMA_DEBUG & 4)) {
                // L = 6 (the C2 shape): 4 columns x 6 limbs per TMEM round trip,
                // the next 4 columns' loads in flight while this group's fp64
                // work runs (the epilogue holds the single accumulator, so its
                // latency is the consumer pipeline's critical path)
                int32_t v[6][4];
                int64_t Sc[4];
                auto issue = [&](int j) {
#pragma unroll
                    for (int l = 0; l < 6; l++) tc_ld4(tl + (uint32_t)(l * S.dpad + j), v[l]);
                };
                auto combine = [&]() {
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int32_t p0 = v[1][u] * 256 + v[0][u], p1 = v[3][u] * 256 + v[2][u],
                                      p2 = v[5][u] * 256 + v[4][u];
                        Sc[u] = ((int64_t)p2 * 65536 + p1) * 65536 + p0;
                    }
                };
                auto accumulate = [&](int j, int s0, bool first) {
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const double delta = __dsub_rn(__dmul_rn(__ll2double_rn(Sc[u]), g), bal.cc[j + u]);
                        const double q = __dmul_rn(delta, delta);
                        racc[s0 + u] = first ? q : __dadd_rn(racc[s0 + u], q);
                    }
                };
                if (full >= 8) {
                    issue(0);
                    tc_wait_ld();
                    combine();
                    for (int jb = 0; jb < full; jb += 8) {
                        issue(jb + 4);
                        accumulate(jb, 0, jb == 0);
                        tc_wait_ld();
                        combine();
                        const bool more = jb + 8 < full;
                        if (more) issue(jb + 8);
                        accumulate(jb + 4, 4, jb == 0);
                        if (more) {
                            tc_wait_ld();
                            combine();
                        }
                    }
                    jb0 = full;
                }
            }
            for (int jb = jb0; jb < ((FRR_MMA_DEBUG & 4) ? 0 : S.dpad); jb += 8) {
                if (jb >= d) break;
                int64_t Sj[8];
#if FRR_MMA_PAIRS
                tc_limbs8_fast(tl + (uint32_t)jb, S.L, S.dpad, Sj);
#else
                tc_limbs8(tl + (uint32_t)jb, S.L, S.dpad, pair32, Sj);
#endif
                if (jb < full) {
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const double delta = __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u]), g), bal.cc[jb + u]);
                        const double q = __dmul_rn(delta, delta);
                        racc[u] = jb == 0 ? q : __dadd_rn(racc[u], q);
                    }
                } else {  // the tail group (full < d)
                    if (d >= 8)
                        res = __dadd_rn(__dadd_rn(__dadd_rn(racc[0], racc[1]), __dadd_rn(racc[2], racc[3])),
                                        __dadd_rn(__dadd_rn(racc[4], racc[5]), __dadd_rn(racc[6], racc[7])));
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        if (jb + u < d) {
                            const double delta = __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u]), g), bal.cc[jb + u]);
                            res = __dadd_rn(res, __dmul_rn(delta, delta));
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[BAR_TMEM_EMPTY]);
#if FRR_MMA_TIMING
            wacc[13] += clock64() - t_epi0;  // epilogue: TMEM full -> drained
#endif
            if (d >= 8 && full == d)
                res = __dadd_rn(__dadd_rn(__dadd_rn(racc[0], racc[1]), __dadd_rn(racc[2], racc[3])),
                                __dadd_rn(__dadd_rn(racc[4], racc[5]), __dadd_rn(racc[6], racc[7])));
            const int64_t c = tile * BM + r;
            if (c < count) out[c] = __dmul_rn(__dadd_rn(0.0, res), cst);
        }
    } else if (warp == c_w_tma) {
        // ============================================== B operand producer
        if (lane == 0 && !(FRR_MMA_DEBUG & 8)) {
            const uint32_t bytes = (uint32_t)S.npad * KC;
            uint32_t bstage = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kc = 0; kc < S.nkc; kc++, bstage++) {
                    const int s = bstage % B_STAGES;
                    TW(4, mbar_wait_long(&bars[BAR_B_EMPTY + s], ((bstage / B_STAGES) & 1) ^ 1));
                    mbar_expect_tx(&bars[BAR_B_FULL + s], bytes);
                    bulk_g2s(sB + (size_t)s * bytes, bal.limbs + (size_t)kc * bytes, bytes, &bars[BAR_B_FULL + s]);
                }
            }
        }
    } else if (warp == c_w_mma) {
        // ===================================================== MMA issuer
        if (lane == 0 && !(FRR_MMA_DEBUG & 8)) {
            uint32_t stage = 0;
            int i = 0;
            const uint32_t a_lbo = (BM / 8) * 128, b_lbo = (uint32_t)(S.npad / 8) * 128;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, i++) {
                TW(5, mbar_wait_long(&bars[BAR_TMEM_EMPTY], (i & 1) ^ 1));
                tc_fence_after();
                for (int kc = 0; kc < S.nkc; kc++, stage++) {
                    const int sa = stage % S.nsta, sb = stage % B_STAGES;
                    TW(6, mbar_wait(&bars[BAR_A_FULL + sa], (stage / S.nsta) & 1));
                    TW(7, mbar_wait(&bars[BAR_B_FULL + sb], (stage / B_STAGES) & 1));
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + (size_t)sa * A_STAGE_BYTES);
                    const uint32_t at = tmem_base + (uint32_t)S.npad + (uint32_t)(sa * (KC / 4));
                    const uint32_t b0 = smem_u32(sB + (size_t)sb * S.npad * KC);
#pragma unroll
                    for (int ks = 0; ks < KC / 32; ks++) {
                        const uint64_t ad = umma_desc(a0 + ks * 2 * a_lbo, a_lbo, 128);
                        for (int p = 0; p < S.nparts; p++) {
                            const uint64_t bd =
                                umma_desc(b0 + ks * 2 * b_lbo + (uint32_t)(S.part_off[p] / 8) * 128, b_lbo, 128);
                            if (S.ta)
                                tc_mma_i8_ts(tmem_base + (uint32_t)S.part_off[p], at + (uint32_t)(ks * 8), bd,
                                             idesc_i8(BM, S.part_n[p]), (kc | ks) != 0);
                            else
                                tc_mma_i8(tmem_base + (uint32_t)S.part_off[p], ad, bd, idesc_i8(BM, S.part_n[p]),
                                          (kc | ks) != 0);
                        }
                    }
                    tc_commit(&bars[BAR_A_EMPTY + sa]);
                    tc_commit(&bars[BAR_B_EMPTY + sb]);
                }
                tc_commit(&bars[BAR_TMEM_FULL]);
            }
        }
    }

#if FRR_MMA_TIMING
    {
        const int role = warp < c_nfy ? 8 : (warp >= c_w_tile0 && warp < c_w_tile0 + 4 * TW2) ? 9 : (warp == c_w_mma ? 10 : 12);
        wacc[role] += clock64() - tstart;
        if (lane == 0)
            for (int k = 0; k < 16; k++)
                if (wacc[k]) atomicAdd(&g_frr_waits[k], (unsigned long long)wacc[k]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == c_w_mma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// ------------------------------------------------------ limb preparation
__global__ void k_prepare_limbs(const int64_t* __restrict__ zq, MmaShape S, int8_t* __restrict__ limbs,
                                int32_t* overflow) {
    const int64_t total = (int64_t)S.kpad * S.npad;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = (int64_t)S.npad * KC;
        int kc = (int)(o / chunk);
        int rem = (int)(o % chunk);
        int k16 = rem / (S.npad * 16);
        int rem2 = rem % (S.npad * 16);
        int n8 = rem2 / 128;
        int rem3 = rem2 % 128;
        int rr = rem3 / 16, kb = rem3 % 16;
        int kk = kc * KC + k16 * 16 + kb;  // K index
        int k = frr_k_unit_nat(kk);         // unit behind that K position
        int nrow = n8 * 8 + rr;
        int l = nrow / S.dpad, j = nrow % S.dpad;
        int8_t v = 0;
        if (k < S.n && j < S.d && l < S.L) {
            int64_t z = zq[(size_t)k * S.d + j];
            for (int q = 0; q <= l; q++) {
                v = (int8_t)(z & 0xFF);
                z = (z - v) >> 8;
            }
            if (l == S.L - 1 && z != 0) atomicExch(overflow, 1);
        }
        limbs[o] = v;
    }
}


// ------------------------------------------------ descriptor self-test
// D[128 x N] = A[128 x K] . B[N x K]^T with one CTA, through the same
// descriptor/idesc/TMEM code as the fused kernel (variant 1 swaps LBO/SBO,
// for diagnosing layout conventions on hardware).
__global__ void __launch_bounds__(128) k_selftest_mma(const int8_t* A, const int8_t* B, int K, int N, int32_t* D,
                                                     int variant) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = smem;
    unsigned char* sB = smem + (size_t)BM * K;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (size_t)N * K);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // canonical K-major layout: [k16][row8][8][16]
    for (int o = threadIdx.x; o < BM * K; o += blockDim.x) {
        int r = o / K, k = o % K;
        sA[((size_t)(k / 16) * (BM / 8) + r / 8) * 128 + (r % 8) * 16 + k % 16] = (unsigned char)A[o];
    }
    for (int o = threadIdx.x; o < N * K; o += blockDim.x) {
        int r = o / K, k = o % K;
        sB[((size_t)(k / 16) * (N / 8) + r / 8) * 128 + (r % 8) * 16 + k % 16] = (unsigned char)B[o];
    }
    fence_proxy_async();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t a_tm = tmem + 256;  // variant 2: A staged in TMEM columns [256, 256 + K/4)
    if (variant == 2) {
        // row threadIdx.x -> TMEM lane, 4 consecutive K bytes per column
        const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16) + 256;
        for (int c0 = 0; c0 < K / 4; c0 += 32) {
            uint32_t v[32];
            for (int c = 0; c < 32; c++) {
                uint32_t w = 0;
                for (int b = 0; b < 4; b++) {
                    const int k = (c0 + c) * 4 + b;
                    w |= (k < K ? (uint32_t)(uint8_t)A[(size_t)threadIdx.x * K + k] : 0u) << (8 * b);
                }
                v[c] = w;
            }
            tc_st32(lane_base + (uint32_t)c0, v);
        }
        tc_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a_lbo = (BM / 8) * 128, b_lbo = (uint32_t)(N / 8) * 128;
        for (int ks = 0; ks < K / 32; ks++) {
            const uint64_t bd = variant == 1 ? umma_desc(smem_u32(sB) + ks * 2 * b_lbo, 128, b_lbo)
                                             : umma_desc(smem_u32(sB) + ks * 2 * b_lbo, b_lbo, 128);
            if (variant == 2) {
                tc_mma_i8_ts(tmem, a_tm + (uint32_t)(ks * 8), bd, idesc_i8(BM, N), ks != 0);
            } else {
                const uint64_t ad = variant == 1 ? umma_desc(smem_u32(sA) + ks * 2 * a_lbo, 128, a_lbo)
                                                 : umma_desc(smem_u32(sA) + ks * 2 * a_lbo, a_lbo, 128);
                tc_mma_i8(tmem, ad, bd, idesc_i8(BM, N), ks != 0);
            }
        }
        tc_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    tc_fence_after();
    const int r = threadIdx.x;
    for (int c = 0; c < N; c += 8) {
        int32_t v[8];
        tc_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
        tc_wait_ld();
        for (int u = 0; u < 8; u++) D[(size_t)r * N + c + u] = v[u];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
    (void)lane;
}

}  // namespace

// N-tiled variant for L*d beyond one TMEM accumulator (frr_mma_nt.cu)
bool frr_nt_fits(int n, int d, int L);
size_t frr_nt_limbs_bytes(int n, int d, int L);
int frr_nt_prepare_limbs(const int64_t* zq, int n, int d, int L, int8_t* limbs, int32_t* overflow, cudaStream_t s);
int frr_mc_stats_nt(const frr_balance_t* bal, uint64_t seed, uint64_t lo, int64_t count, double* stats,
                    void* stream);

namespace {
enum TcLayout { TC_NONE = 0, TC_SINGLE = 1, TC_NT = 2 };

// Which tensor-core kernel (and B-operand layout) serves (n, d, L).  Decided
// without t (worst case t = n - 1) so the limb operand can be built once.
TcLayout tc_layout(int n, int d, int L) {
    if (d <= 16 || L < 1 || L > 8 || n < 2 || n > FRR_MAX_UNITS) return TC_NONE;
    static const int force_nt = [] {
        const char* e = getenv("FRR_TC_FORCE_NT");
        return e && *e == '1';
    }();
    if (force_nt && frr_nt_fits(n, d, L)) return TC_NT;
    MmaShape s = mma_shape(n, n - 1, d, L);
    if (s.npad <= 512 && s.nfy > 0) return TC_SINGLE;
    if (frr_nt_fits(n, d, L)) return TC_NT;
    return TC_NONE;
}
}  // namespace

bool frr_mma_supported(const frr_balance_t* bal) {
    if (bal->t <= 0 || bal->t >= bal->n) return false;
    if (bal->t >= 32768) return false;  // frr_pack_word reads control marks from bit 15
    return tc_layout(bal->n, bal->d, bal->n_limbs) != TC_NONE;
}

extern "C" int frr_tc_kernel(int n, int d, int n_limbs) { return (int)tc_layout(n, d, n_limbs); }

extern "C" size_t frr_limbs_bytes(int n, int d, int n_limbs) {
    switch (tc_layout(n, d, n_limbs)) {
        case TC_SINGLE: {
            MmaShape s = mma_shape(n, 1, d, n_limbs);
            return (size_t)s.kpad * s.npad;
        }
        case TC_NT:
            return frr_nt_limbs_bytes(n, d, n_limbs);
        default:
            return 0;
    }
}

extern "C" int frr_prepare_limbs(const int64_t* zq, int n, int d, int n_limbs, int8_t* limbs, int32_t* overflow_dev,
                                 void* stream) {
    const TcLayout lay = tc_layout(n, d, n_limbs);
    if (lay == TC_NONE) {
        frr_set_error("frr_prepare_limbs: no tensor-core layout for n=%d d=%d limbs=%d", n, d, n_limbs);
        return FRR_E_UNSUPPORTED;
    }
    cudaStream_t s = frr_stream(stream);
    if (cudaMemsetAsync(overflow_dev, 0, sizeof(int32_t), s) != cudaSuccess) return frr_check_launch("overflow memset");
    if (lay == TC_NT) return frr_nt_prepare_limbs(zq, n, d, n_limbs, limbs, overflow_dev, s);
    MmaShape S = mma_shape(n, 1, d, n_limbs);
    int64_t total = (int64_t)S.kpad * S.npad;
    int grid = (int)std::min<int64_t>(frr_cdiv(total, 256), (int64_t)frr_num_sms() * 16);
    k_prepare_limbs<<<grid, 256, 0, s>>>(zq, S, limbs, overflow_dev);
    return frr_launched("k_prepare_limbs");
}

int frr_mc_stats_mma(const frr_balance_t* bal, uint64_t seed, uint64_t lo, int64_t count, double* stats,
                     void* stream) {
    if (count <= 0) return FRR_OK;
    if (tc_layout(bal->n, bal->d, bal->n_limbs) == TC_NT) return frr_mc_stats_nt(bal, seed, lo, count, stats, stream);
    MmaShape S = mma_shape(bal->n, bal->t, bal->d, bal->n_limbs);
    SmemPlan P = smem_plan(S);
    const bool full = S.gen ? (S.nfy == RFY && S.nbits == RBITS) : (S.nfy == NFY && S.nbits == NBITS);
    const auto kern = S.gen ? (full ? k_mc_stats_mma<false, true, 1> : k_mc_stats_mma<false, false, 1>)
                      : S.steps_smem ? (full ? k_mc_stats_mma<false, true, 0> : k_mc_stats_mma<false, false, 0>)
                                     : (full ? k_mc_stats_mma<true, true, 0> : k_mc_stats_mma<true, false, 0>);
    int rc = frr_prepare_kernel(kern, P.total);
    if (rc) return rc;
    int64_t ntiles = frr_cdiv(count, BM);
    int grid = (int)std::min<int64_t>(ntiles, frr_num_sms());
    GlobalSteps gs;
    if (!S.steps_smem && (rc = gs.init(bal->n, bal->t, frr_stream(stream)))) return rc;
    kern<<<grid, S.nwarps * 32, P.total, frr_stream(stream)>>>(*bal, seed, lo, count, stats, gs.p);
    return frr_launched("k_mc_stats_mma");
}

extern "C" int frr_mc_stats_tc(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                               double* stats, void* stream) {
    if (!bal || !bal->limbs || !frr_mma_supported(bal)) {
        frr_set_error("frr_mc_stats_tc: shape not supported by the tensor-core path");
        return FRR_E_UNSUPPORTED;
    }
    return frr_mc_stats_mma(bal, root_seed, draw_lo, count, stats, stream);
}

extern "C" int frr_selftest_mma_i8(const int8_t* A, const int8_t* B, int K, int N, int32_t* D, int variant,
                                   void* stream) {
    if (K % 32 || K > 512 || N % 16 || N < 16 || N > 256 || (variant == 2 && (K > 1024 || K % 128))) {
        frr_set_error("selftest: K %% 32 == 0, K <= 512, N %% 16 == 0, 16 <= N <= 256 (variant 2: K %% 128 == 0)");
        return FRR_E_INVALID_DESIGN;
    }
    size_t smem = (size_t)BM * K + (size_t)N * K + 64 + 1024;
    int rc = frr_prepare_kernel(k_selftest_mma, smem);
    if (rc) return rc;
    k_selftest_mma<<<1, 128, smem, frr_stream(stream)>>>(A, B, K, N, D, variant);
    return frr_launched("k_selftest_mma");
}

// ---------------------------------------------------- tensor-pipe ceiling
namespace {
// One CTA per SM, one thread issuing back-to-back tcgen05.mma.kind::i8
// (M = 128, N, K = 32 per instruction, 4 per 128-byte K stage) into one
// TMEM accumulator; A from shared memory (a_tmem = 0) or TMEM (1).  The
// operands are zero: the tensor pipe's rate does not depend on the values.
__global__ void __launch_bounds__(128) k_microbench_mma(int N, int a_tmem, int64_t iters) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = smem;
    unsigned char* sB = smem + BM * 128;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (size_t)N * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const bool rnd = (a_tmem & 2) != 0;  // random operand bytes instead of zeros
    a_tmem &= 1;
    for (int o = threadIdx.x; o < (BM + N) * 128 / 16; o += blockDim.x) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (rnd) {
            const uint64_t h = frr_mix64((uint64_t)o), h2 = frr_mix64(h);
            v = make_uint4((uint32_t)h, (uint32_t)(h >> 32), (uint32_t)h2, (uint32_t)(h2 >> 32));
        }
        reinterpret_cast<uint4*>(smem)[o] = v;
    }
    fence_proxy_async();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (rnd && a_tmem) {  // A stage (TMEM columns 256..287) with random bytes
        uint32_t v[32];
        for (int c = 0; c < 32; c++) v[c] = (uint32_t)frr_mix64((uint64_t)(threadIdx.x * 32 + c + 12345));
        tc_st32(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + 256, v);
        tc_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a_lbo = (BM / 8) * 128, b_lbo = (uint32_t)(N / 8) * 128;
        const uint32_t idesc = idesc_i8(BM, N);
        const uint64_t ad0 = umma_desc(smem_u32(sA), a_lbo, 128), bd0 = umma_desc(smem_u32(sB), b_lbo, 128);
        for (int64_t it = 0; it < iters; it++) {
#pragma unroll
            for (int ks = 0; ks < 4; ks++) {
                const uint64_t bd = bd0 + (uint64_t)((ks * 2 * b_lbo) >> 4);
                if (a_tmem)
                    tc_mma_i8_ts(tmem, tmem + 256 + (uint32_t)(ks * 8), bd, idesc, (it | ks) != 0);
                else
                    tc_mma_i8(tmem, ad0 + (uint64_t)((ks * 2 * a_lbo) >> 4), bd, idesc, (it | ks) != 0);
            }
        }
        tc_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
}  // namespace

extern "C" int frr_microbench_mma_i8(int N, int a_tmem, int64_t iters, int64_t* ops_host, void* stream) {
    if (N < 16 || N > 256 || N % 16 || iters < 1) {
        frr_set_error("frr_microbench_mma_i8: N must be 16..256 (multiple of 16), iters >= 1");
        return FRR_E_INVALID_DESIGN;
    }
    const size_t smem = 1024 + (size_t)(BM + N) * 128 + 64;
    int rc = frr_prepare_kernel(k_microbench_mma, smem);
    if (rc) return rc;
    const int grid = frr_num_sms();
    k_microbench_mma<<<grid, 128, smem, frr_stream(stream)>>>(N, a_tmem, iters);
    if (ops_host) *ops_host = (int64_t)grid * iters * 4 * 2 * BM * N * 32;
    return frr_launched("k_microbench_mma");
}

namespace {
// The same ceiling for CTA pairs: clusters of two CTAs on one TPC, the
// leader issuing tcgen05.mma.cta_group::2.kind::i8 (M = 256: 128 rows per
// CTA from its own shared memory or TMEM; B split by N, N/2 rows in each
// CTA's shared memory; each CTA's TMEM holds its 128 x N accumulator).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) k_microbench_mma2(int N, int a_tmem, int64_t iters) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sA = smem;
    unsigned char* sB = smem + BM * 128;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (size_t)(N / 2) * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int o = threadIdx.x; o < (BM + N / 2) * 128 / 16; o += blockDim.x)
        reinterpret_cast<uint4*>(smem)[o] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a_lbo = (BM / 8) * 128, b_lbo = (uint32_t)(N / 16) * 128;
        const uint32_t idesc = idesc_i8(2 * BM, N);
        const uint64_t ad0 = umma_desc(smem_u32(sA), a_lbo, 128), bd0 = umma_desc(smem_u32(sB), b_lbo, 128);
        for (int64_t it = 0; it < iters; it++) {
#pragma unroll
            for (int ks = 0; ks < 4; ks++) {
                const uint64_t bd = bd0 + (uint64_t)((ks * 2 * b_lbo) >> 4);
                const uint32_t acc = (it | ks) != 0;
                if (a_tmem)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                        "r"(tmem + 256 + (uint32_t)(ks * 8)), "l"(bd), "r"(idesc), "r"(acc)
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(ad0 + (uint64_t)((ks * 2 * a_lbo) >> 4)), "l"(bd), "r"(idesc), "r"(acc)
                        : "memory");
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(bar)),
            "h"((uint16_t)3)
            : "memory");
    }
    __syncwarp();
    mbar_wait(bar, 0);
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if ((threadIdx.x >> 5) == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
}  // namespace

extern "C" int frr_microbench_mma_i8_pair(int N, int a_tmem, int64_t iters, int64_t* ops_host, void* stream) {
    if (N < 32 || N > 256 || N % 32 || iters < 1) {
        frr_set_error("frr_microbench_mma_i8_pair: N must be 32..256 (multiple of 32), iters >= 1");
        return FRR_E_INVALID_DESIGN;
    }
    const size_t smem = 1024 + (size_t)(BM + N / 2) * 128 + 64;
    int rc = frr_prepare_kernel(k_microbench_mma2, smem);
    if (rc) return rc;
    const int grid = frr_num_sms() / 2 * 2;
    k_microbench_mma2<<<grid, 128, smem, frr_stream(stream)>>>(N, a_tmem & 1, iters);
    if (ops_host) *ops_host = (int64_t)(grid / 2) * iters * 4 * 2 * (2 * BM) * N * 32;
    return frr_launched("k_microbench_mma2");
}

#if FRR_MMA_TIMING
extern "C" int frr_debug_waits(unsigned long long* host16) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host16, g_frr_waits, sizeof(unsigned long long) * 16);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_frr_waits, z, sizeof(z));
    return 0;
}
#endif

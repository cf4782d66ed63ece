// frr_mma_nt_body.cuh -- the N-tiled kernel, instantiated by frr_mma_nt.cu once
// per K-stage size (FRR_NT_KC = 128 / 256) in namespace FRR_NT_NS.
namespace FRR_NT_NS {
using namespace frr_tc;

constexpr int BM = 128;
constexpr int KC = FRR_NT_KC;  // K bytes per stage: this instantiation's (128 or 256)
#ifndef FRR_NT_ST
#define FRR_NT_ST 4
#endif
#ifndef FRR_NT_NFY
#define FRR_NT_NFY 8
#endif
#ifndef FRR_NT_NEXP
#define FRR_NT_NEXP 8
#endif
// thread-per-candidate generators (frr_rev_fy): at most RFY warps (a
// multiple of 4: one tile in flight per 4) and MAXB tile buffers
// epilogue limb recombination through the unrolled 32-bit pair helper
#ifndef FRR_NT_PAIRS
#define FRR_NT_PAIRS 0  // measured slower than tc_limbs8 (runtime limb loop) in this kernel
#endif
// epilogue warps per TMEM lane quadrant: 2 splits each 8-column group (the
// accumulator streams r0..r3 / r4..r7 of numpy's pairwise leaves), 1 = whole
#ifndef FRR_NT_EPIW
#define FRR_NT_EPIW 2
#endif
#ifndef FRR_NT_RFY
#define FRR_NT_RFY (FRR_NT_EPIW == 2 ? 12 : 16)
#endif
#ifndef FRR_NT_MAXB
#define FRR_NT_MAXB 8
#endif
// timing experiments only (results invalid): 1 no B loads, 2 no A stores,
// 4 no epilogue work, 8 no Fisher-Yates
#ifndef FRR_NT_DEBUG
#define FRR_NT_DEBUG 0
#endif
// wait-time accounting (debug builds, FRR_NT_TIMING=1; read back with
// frr_debug_nt_waits for the 256-byte-stage instantiation)
#ifndef FRR_NT_TIMING
#define FRR_NT_TIMING 0
#endif
#if FRR_NT_TIMING
__device__ unsigned long long g_nt_waits[16];
#define NTW(slot, ...)                         \
    do {                                       \
        const long long t0_ = clock64();       \
        __VA_ARGS__;                           \
        wacc[slot] += clock64() - t0_;         \
    } while (0)
#else
#define NTW(slot, ...) \
    do {               \
        __VA_ARGS__;   \
    } while (0)
#endif
// K-stage ring: stage s = A chunk s in TMEM + B chunk s in shared memory, one
// "stage consumed" barrier (a single tcgen05.commit) releases both halves.
constexpr int NST = KC == 256 ? 2 : FRR_NT_ST;  // TMEM holds two 64-column A stages at KC = 256
constexpr int NFY = FRR_NT_NFY;
constexpr int RFY = FRR_NT_RFY;
constexpr int EPIW = FRR_NT_EPIW;
static_assert(EPIW == 1 || EPIW == 2, "epilogue warps per quadrant");
constexpr int MAXB = FRR_NT_MAXB;
constexpr int NEXP = FRR_NT_NEXP;          // expansion warps (4 or 8: 1 or 2 threads per row)
// Warp roles (the scheduler favours higher warp ids; the epilogue is the
// measured bottleneck of this kernel, so it gets the highest ones).
#ifndef FRR_NT_LAYOUT
#define FRR_NT_LAYOUT 2
#endif
#if FRR_NT_LAYOUT == 2
// expansion 0..NEXP-1, generators, bulk copy, MMA, then the epilogue on the
// highest ids (4-aligned: warp % 4 is its TMEM lane quadrant)
constexpr int W_EXP0 = 0, W_FY0 = NEXP;
__host__ __device__ constexpr int w_tma(int nfy) { return W_FY0 + nfy; }
__host__ __device__ constexpr int w_mma(int nfy) { return W_FY0 + nfy + 1; }
__host__ __device__ constexpr int w_epi0(int nfy) { return (W_FY0 + nfy + 2 + 3) & ~3; }
__host__ __device__ constexpr int n_warps(int nfy) { return w_epi0(nfy) + 4 * EPIW; }
#elif FRR_NT_LAYOUT == 1
constexpr int W_EXP0 = 4, W_FY0 = W_EXP0 + NEXP;
__host__ __device__ constexpr int w_tma(int nfy) { return W_FY0 + nfy; }
__host__ __device__ constexpr int w_mma(int nfy) { return W_FY0 + nfy + 1; }
__host__ __device__ constexpr int w_epi0(int) { return 0; }
__host__ __device__ constexpr int n_warps(int nfy) { return W_FY0 + nfy + 2; }
#else
constexpr int W_EXP0 = 4, W_FY0 = W_EXP0 + NEXP + 2;
__host__ __device__ constexpr int w_tma(int) { return W_EXP0 + NEXP; }
__host__ __device__ constexpr int w_mma(int) { return W_EXP0 + NEXP + 1; }
__host__ __device__ constexpr int w_epi0(int) { return 0; }
__host__ __device__ constexpr int n_warps(int nfy) { return W_FY0 + nfy; }
#endif
constexpr int NWARPS = n_warps(NFY > RFY ? NFY : RFY);
constexpr int NTHREADS = NWARPS * 32;
constexpr int DJ = 32;  // covariates per N-chunk
constexpr int MAX_LEAVES = 1024;

struct NtShape {
    int n, t, d, L, dpad, nch, nc, kpad, nkc, kw;
    int gen;         // 1: thread-per-candidate generators (step table in shared memory), 0: warp per candidate
    int nfy, nbits;  // generator warps, bit-row buffers (fewer for large n)
};

struct NtPlan {
    size_t a, b, bits, steps, tables, starts, ncomb, xch, bars, total;
};

// tile buffer: 128 bit rows of kw words, [row / 32][word][row % 32] (see
// frr_mma.cu); bit b of word w = unit 32 w + b is a control unit
__host__ __device__ inline size_t nt_buf_words(int kw) { return (size_t)BM * kw; }

__host__ __device__ inline size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline NtPlan nt_plan(const NtShape& s) {
    NtPlan p;
    size_t o = 0;
    p.a = o;
    p.b = o;
    o += (size_t)NST * s.nc * KC;
    p.bits = o;
    o += (size_t)s.nbits * nt_buf_words(s.kw) * 4;
    p.steps = o;
    if (s.gen) o += (size_t)frr_steps_len(s.t) * sizeof(StepC);
    p.tables = o;
    // GEN 0: a table per generator warp; GEN 1: one shared scratch table for
    // the exact recomputation of flagged candidates, + its lock word
    o += (size_t)(s.gen ? 1 : s.nfy) * frr_table_len(s.n) * 2;
    if (s.gen) o = up(o + FRR_TABLE_SLACK, 16) + 16;
    o = up(o, 16);
    p.starts = o;
    o += up((size_t)(s.dpad / 8 + 31) / 32 * 4, 16);
    p.ncomb = o;
    o += MAX_LEAVES;
    o = up(o, 16);
    p.xch = o;  // split epilogue: half-leaf sums handed between a quadrant's warps
    o += (EPIW == 2 ? 2 * BM * sizeof(double) : 0);
    p.bars = o;
    o += 32 * 8 + 16;  // barriers: also the FRR_TABLE_SLACK after the tables
    static_assert(32 * 8 + 16 >= FRR_TABLE_SLACK, "table slack");
    p.total = o + 1024;
    return p;
}

__host__ __device__ inline NtShape nt_shape(int n, int t, int d, int L) {
    NtShape s;
    s.n = n;
    s.t = t;
    s.d = d;
    s.L = L;
    s.dpad = (d + DJ - 1) / DJ * DJ;
    s.nch = s.dpad / DJ;
    s.nc = DJ * L;
    s.kpad = (n + KC - 1) / KC * KC;
    s.nkc = s.kpad / KC;
    s.kw = s.kpad / 32;
    // thread-per-candidate generators when their tile buffers fit (nfy / 4
    // tiles being built + two being consumed); else the warp generators with
    // the full layout (NFY generators, two bit buffers) when it fits, else
    // fewer generators / one buffer so that large n keeps the tensor cores
    s.gen = 1;
    for (int f = RFY; f >= 4; f -= 4) {
        s.nfy = f;
        s.nbits = f / 4 + 2 <= MAXB ? f / 4 + 2 : MAXB;
        if (nt_plan(s).total <= 227 * 1024) return s;
    }
    s.gen = 0;
    for (int nb = 2; nb >= 1; nb--)
        for (int f = NFY; f >= 2; f--) {
            s.nfy = f;
            s.nbits = nb;
            if (nt_plan(s).total <= 227 * 1024) return s;
        }
    s.nfy = s.nbits = 0;
    return s;
}

// one "stage full" barrier per ring slot, arrived on by the 8 expansion warps
// and by the bulk copy (arrive + expect_tx)
constexpr int B_BITS_FULL = 0, B_BITS_EMPTY = MAXB, B_A_FULL = 2 * MAXB, B_B_FULL = B_A_FULL;
constexpr int B_S_EMPTY = B_B_FULL + NST, B_TM_FULL = B_S_EMPTY + NST, B_TM_EMPTY = B_TM_FULL + 2;
static_assert(B_TM_EMPTY + 2 <= 30, "barrier slots");

// numpy pairwise plan over d: leaves (<= 128, starting at multiples of 8),
// "group g starts a leaf" bits and, per leaf, how many combines follow it in
// post order (numpy's recursion: n2 = n/2 rounded down to a multiple of 8).
__device__ void nt_build(int off, int len, uint32_t* starts, uint8_t* ncomb, int& nleaf) {
    if (len <= 128) {
        const int g = off / 8;
        starts[g >> 5] |= 1u << (g & 31);
        ncomb[nleaf++] = 0;
        return;
    }
    int n2 = len / 2;
    n2 -= n2 % 8;
    nt_build(off, n2, starts, ncomb, nleaf);
    nt_build(off + n2, len - n2, starts, ncomb, nleaf);
    ncomb[nleaf - 1]++;
}

__device__ __forceinline__ void tc_st_cols(uint32_t a, const uint32_t (&v)[16]) { tc_st16(a, v); }
__device__ __forceinline__ void tc_st_cols(uint32_t a, const uint32_t (&v)[32]) { tc_st32(a, v); }

// wait with a short sleep between polls, for roles whose waits are long
__device__ __forceinline__ void mbar_wait_lazy(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(128);
    }
}

// spin wait for the pipeline roles (suspend-hint and sleep variants measured no better)
#ifndef FRR_NT_HW_LAZY
#define FRR_NT_HW_LAZY 0
#endif
__device__ __forceinline__ void mbar_wait_hw(uint64_t* b, uint32_t parity) {
#if FRR_NT_HW_LAZY
    mbar_wait_lazy(b, parity);
#else
    mbar_wait(b, parity);
#endif
}

__device__ __forceinline__ double comb8(const double (&r)[8]) {
    return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                     __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

// FULL: the default generator and bit-buffer counts as compile-time
// constants; GEN: thread-per-candidate (1) or warp-per-candidate (0) generators
template <bool FULL, int GEN>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_mc_stats_nt(frr_balance_t bal, uint64_t seed, uint64_t lo, int64_t count, double* __restrict__ out,
                  const StepC* __restrict__ steps) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const NtShape S = nt_shape(bal.n, bal.t, bal.d, bal.n_limbs);
    const NtPlan P = nt_plan(S);
    unsigned char* sB = smem + P.b;
    uint32_t* sBits = reinterpret_cast<uint32_t*>(smem + P.bits);
    StepC* ssteps = reinterpret_cast<StepC*>(smem + P.steps);
    uint16_t* tables = reinterpret_cast<uint16_t*>(smem + P.tables);
    int* fix_lock = reinterpret_cast<int*>(smem + P.starts - 16);
    uint32_t* starts = reinterpret_cast<uint32_t*>(smem + P.starts);
    uint8_t* ncomb = smem + P.ncomb;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.bars);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (count + BM - 1) / BM;
    const size_t buf_words = nt_buf_words(S.kw);
    const int nst = min(NST, (512 - 2 * S.nc) / (KC / 4));  // ring stages whose A fits in TMEM
    const int c_nfy = FULL ? (GEN ? RFY : NFY) : S.nfy, c_nbits = FULL ? (GEN ? RFY / 4 + 2 : 2) : S.nbits;
#if FRR_NT_TIMING
    long long wacc[16] = {0};
    const long long tstart = clock64();
#endif

    for (int i = threadIdx.x; i < (S.dpad / 8 + 31) / 32; i += blockDim.x) starts[i] = 0;
    if (GEN) frr_fill_steps(ssteps, S.n, S.t);
    __syncthreads();
    if (threadIdx.x == 0) {
        int nleaf = 0;
        nt_build(0, S.d, starts, ncomb, nleaf);
        if (GEN) *fix_lock = 0;
        for (int b = 0; b < c_nbits; b++) {
            mbar_init(&bars[B_BITS_FULL + b], GEN ? 4 : c_nfy);
            mbar_init(&bars[B_BITS_EMPTY + b], NEXP);
        }
        for (int s = 0; s < nst; s++) {
            mbar_init(&bars[B_A_FULL + s], NEXP + 1);
            mbar_init(&bars[B_S_EMPTY + s], 1);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(&bars[B_TM_FULL + s], 1);
            mbar_init(&bars[B_TM_EMPTY + s], 4 * EPIW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    const int W_TMA = w_tma(c_nfy), W_MMA = w_mma(c_nfy), W_EPI0 = w_epi0(c_nfy);
    if (warp == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (GEN && warp >= W_FY0 && warp < W_FY0 + c_nfy) {
        // ================================ thread-per-candidate generators
        // warp g builds quadrant g % 4 of the CTA's tiles g / 4, g / 4 +
        // nfy / 4, ... in place in their buffers (frr_mma.cu)
        const int fyw = warp - W_FY0, q = fyw & 3, kstep = c_nfy >> 2;
        const uint32_t sst = smem_u32(ssteps);
        for (int64_t k = fyw >> 2;; k += kstep) {
            const int64_t tile = blockIdx.x + k * gridDim.x;
            if (tile >= ntiles) break;
            const int buf = (int)(k % c_nbits);
            NTW(0, mbar_wait_lazy(&bars[B_BITS_EMPTY + buf], ((k / c_nbits) & 1) ^ 1));
            const uint32_t blk = smem_u32(sBits + (size_t)buf * buf_words + (size_t)q * S.kw * 32);
            const uint64_t state = frr_derive_state(seed, lo + (uint64_t)(tile * BM + 32 * q + lane));
            bool flag = false;
            if (!(FRR_NT_DEBUG & 8)) flag = frr_rev_fy(state, S.t, sst, blk + 4u * lane, S.kw);
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
            if (lane == 0) mbar_arrive(&bars[B_BITS_FULL + buf]);
        }
    } else if (!GEN && warp >= W_FY0 && warp < W_FY0 + c_nfy) {
        // ===================================== warp-per-candidate generators
        const int fyw = warp - W_FY0;
        uint16_t* lw = tables + (size_t)fyw * frr_table_len(S.n);
        int i = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, i++) {
            const int buf = i % c_nbits;
            NTW(0, mbar_wait_lazy(&bars[B_BITS_EMPTY + buf], ((i / c_nbits) & 1) ^ 1));
            uint32_t* tb = sBits + (size_t)buf * buf_words;
            for (int r = fyw; r < BM; r += c_nfy) {
                const int64_t c = tile * BM + r;
                uint32_t* row = tb + (size_t)(r >> 5) * S.kw * 32 + (r & 31);
                if (c < count && !(FRR_NT_DEBUG & 8)) {
                    frr_warp_fy<true>(frr_derive_state(seed, lo + (uint64_t)c), S.n, S.t, steps, lw, lane);
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
            if (lane == 0) mbar_arrive(&bars[B_BITS_FULL + buf]);
        }
    } else if (warp >= W_EXP0 && warp < W_EXP0 + NEXP) {
        // ============================ A expansion, once per N-chunk pass
        constexpr int TPR = NEXP / 4;             // threads per row
        constexpr int WPT = KC / 32 / TPR;        // bit words per thread per stage
        static_assert(WPT == 2 || WPT == 4, "tcgen05.st.x16 / x32 cover 2 / 4 bit words");
        const int et = threadIdx.x - W_EXP0 * 32;
        const int r = et % BM, part = et / BM;   // r / 32 == warp % 4: this warp's TMEM lanes
        const uint32_t lane_tm =
            tmem_base + ((uint32_t)((r >> 5) * 32) << 16) + (uint32_t)(2 * S.nc + part * WPT * 8);
        int i = 0;
        int a_s = 0;
        uint32_t a_ph = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, i++) {
            const int buf = i % c_nbits;
            NTW(1, mbar_wait_hw(&bars[B_BITS_FULL + buf], (i / c_nbits) & 1));
            // row r: word w at [r / 32][w][r % 32]; control bits -> treated
            const uint32_t* row = sBits + (size_t)buf * buf_words + (size_t)(r >> 5) * S.kw * 32 + (r & 31);
            for (int c = 0; c < S.nch; c++) {
                for (int kc = 0; kc < S.nkc; kc++) {
                    const int s = a_s;
                    NTW(2, mbar_wait_hw(&bars[B_S_EMPTY + s], a_ph ^ 1));
                    if (++a_s == nst) {
                        a_s = 0;
                        a_ph ^= 1;
                    }
                    tc_fence_after();
                    const uint32_t* src = row + (size_t)(kc * (KC / 32) + part * WPT) * 32;
                    uint32_t v[WPT * 8];
#pragma unroll
                    for (int q = 0; q < WPT; q++) {
                        const uint32_t w = ~src[q * 32], wh = w >> 4;
#pragma unroll
                        for (int b = 0; b < 8; b++) {
                            // bit 8j+b of w lands in byte j of register b with weight
                            // 2^(b&3); the B rows carry the compensating 2^(3-(b&3))
                            v[q * 8 + b] = (b < 4 ? w : wh) & (0x01010101u << (b & 3));
                        }
                    }
                    if (!(FRR_NT_DEBUG & 2)) {
                        tc_st_cols(lane_tm + (uint32_t)(s * (KC / 4)), v);
                        tc_wait_st();
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars[B_A_FULL + s]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[B_BITS_EMPTY + buf]);
        }
    } else if (EPIW == 2 && warp >= W_EPI0 && warp < W_EPI0 + 8) {
        // ================================== streaming epilogue, two warps per quadrant
        // Warp half h of quadrant q owns columns 4h..4h+3 of every 8-column group,
        // i.e. numpy's accumulator streams r_{4h..4h+3} of each pairwise leaf.
        // A leaf's combination ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) joins the
        // halves through shared memory; half 0 keeps the combine stack.  The
        // tail group of d % 8 columns is loaded whole by half 0.
        const int k = warp - W_EPI0, quad = k & 3, half = k >> 2;
        const int r = quad * 32 + lane;  // tile row == TMEM lane
        const uint32_t tl = tmem_base + ((uint32_t)(quad * 32) << 16);
        double* xch = reinterpret_cast<double*>(smem + P.xch);  // [parity][row]
        const double g = bal.g, cst = bal.cst;
        const int d = S.d;
        const bool pair32 = (int64_t)S.n * (128 << 3) * 257 < (1ll << 31);
        uint32_t chunk_ctr = 0, xphase = 0;
        // the two warps of a quadrant meet at named barrier 1 + quad
        auto meet = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory"); };
        // joins the halves of the open leaf; half 0 returns the leaf sum
        auto join = [&](const double (&ra)[4]) -> double {
            const double part = __dadd_rn(__dadd_rn(ra[0], ra[1]), __dadd_rn(ra[2], ra[3]));
            double* slot = xch + (xphase & 1) * BM + r;
            if (half == 1) *slot = part;
            meet();
            xphase++;
            return half == 0 ? __dadd_rn(part, *slot) : 0.0;
        };
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            double racc[4];
#pragma unroll
            for (int u = 0; u < 4; u++) racc[u] = 0.0;
            double stk[16];
            int sp = 0, leaf = -1;
            bool done = false;
            for (int c = 0; c < S.nch; c++, chunk_ctr++) {
                const int tb = chunk_ctr & 1;
                NTW(3, mbar_wait_lazy(&bars[B_TM_FULL + tb], (chunk_ctr >> 1) & 1));
                tc_fence_after();
                const uint32_t cb = tl + (uint32_t)(tb * S.nc);
                for (int g4 = 0; g4 < DJ / 8; g4++) {
                    if (FRR_NT_DEBUG & 4) break;
                    const int j0 = c * DJ + g4 * 8;
                    if (j0 >= d) break;
                    const int G = j0 >> 3;
                    const bool starts_leaf = (starts[G >> 5] >> (G & 31)) & 1u;
                    if (!starts_leaf && j0 + 8 > d) {
                        // tail of the last leaf: combine, then add the tail columns in order
                        const double res0 = join(racc);
                        if (half == 0) {
                            int64_t Sj[8];
                            tc_limbs8(cb + (uint32_t)(g4 * 8), S.L, DJ, pair32, Sj);
                            double res = res0;
#pragma unroll
                            for (int u = 0; u < 8; u++)
                                if (j0 + u < d) {
                                    const double delta =
                                        __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u] >> 3), g), bal.cc[j0 + u]);
                                    res = __dadd_rn(res, __dmul_rn(delta, delta));
                                }
                            stk[sp++] = res;
                            for (int m = ncomb[leaf]; m > 0; m--) {
                                sp--;
                                stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                            }
                        }
                        done = true;
                        continue;
                    }
                    int64_t Sj[4];
                    tc_limbs4(cb + (uint32_t)(g4 * 8 + 4 * half), S.L, DJ, pair32, Sj);
                    double q[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int j = j0 + 4 * half + u;
                        const double delta =
                            __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u] >> 3), g), j < d ? bal.cc[j] : 0.0);
                        q[u] = __dmul_rn(delta, delta);
                    }
                    if (starts_leaf) {
                        if (leaf >= 0) {  // close the previous leaf
                            const double lv = join(racc);
                            if (half == 0) {
                                stk[sp++] = lv;
                                for (int m = ncomb[leaf]; m > 0; m--) {
                                    sp--;
                                    stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                                }
                            }
                        }
                        leaf++;
#pragma unroll
                        for (int u = 0; u < 4; u++) racc[u] = q[u];
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; u++) racc[u] = __dadd_rn(racc[u], q[u]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars[B_TM_EMPTY + tb]);
            }
            if (!done) {
                const double lv = join(racc);
                if (half == 0) {
                    stk[sp++] = lv;
                    for (int m = ncomb[leaf]; m > 0; m--) {
                        sp--;
                        stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                    }
                }
            }
            const int64_t cidx = tile * BM + r;
            if (half == 0 && cidx < count) out[cidx] = __dmul_rn(__dadd_rn(0.0, stk[0]), cst);
        }
    } else if (EPIW == 1 && warp >= W_EPI0 && warp < W_EPI0 + 4) {
        // ================================================ streaming epilogue
        const int r = threadIdx.x - W_EPI0 * 32;  // tile row == TMEM lane
        const uint32_t tl = tmem_base + ((uint32_t)((warp - W_EPI0) * 32) << 16);
        const double g = bal.g, cst = bal.cst;
        const int d = S.d;
        // per-limb accumulators are bounded by n * 8 * 128 (pre-shifted rows)
        const bool pair32 = (int64_t)S.n * (128 << 3) * 257 < (1ll << 31);
        uint32_t chunk_ctr = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            double racc[8];
#pragma unroll
            for (int k = 0; k < 8; k++) racc[k] = 0.0;
            double stk[16];
            int sp = 0, leaf = -1;
            bool done = false;
            for (int c = 0; c < S.nch; c++, chunk_ctr++) {
                const int tb = chunk_ctr & 1;
                NTW(3, mbar_wait_lazy(&bars[B_TM_FULL + tb], (chunk_ctr >> 1) & 1));
                tc_fence_after();
                const uint32_t cb = tl + (uint32_t)(tb * S.nc);
                for (int g4 = 0; g4 < DJ / 8; g4++) {
                    if (FRR_NT_DEBUG & 4) break;
                    const int j0 = c * DJ + g4 * 8;
                    if (j0 >= d) break;
                    int64_t Sj[8];
                    const uint32_t cg = cb + (uint32_t)(g4 * 8);
#if FRR_NT_PAIRS
                    if (pair32)
                        tc_limbs8_fast(cg, S.L, DJ, Sj);
                    else
#endif
                        tc_limbs8(cg, S.L, DJ, pair32, Sj);
                    double q[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int j = j0 + u;
                        const double cc = j < d ? bal.cc[j] : 0.0;
                        const double delta = __dsub_rn(__dmul_rn(__ll2double_rn(Sj[u] >> 3), g), cc);
                        q[u] = __dmul_rn(delta, delta);
                    }
                    const int G = j0 >> 3;
                    if ((starts[G >> 5] >> (G & 31)) & 1u) {
                        if (leaf >= 0) {  // close the previous leaf
                            stk[sp++] = comb8(racc);
                            for (int m = ncomb[leaf]; m > 0; m--) {
                                sp--;
                                stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                            }
                        }
                        leaf++;
#pragma unroll
                        for (int u = 0; u < 8; u++) racc[u] = q[u];
                    } else if (j0 + 8 <= d) {
#pragma unroll
                        for (int u = 0; u < 8; u++) racc[u] = __dadd_rn(racc[u], q[u]);
                    } else {  // tail of the last leaf: combine, then add sequentially
                        double res = comb8(racc);
#pragma unroll
                        for (int u = 0; u < 8; u++)
                            if (j0 + u < d) res = __dadd_rn(res, q[u]);
                        stk[sp++] = res;
                        for (int m = ncomb[leaf]; m > 0; m--) {
                            sp--;
                            stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                        }
                        done = true;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars[B_TM_EMPTY + tb]);
            }
            if (!done) {
                stk[sp++] = comb8(racc);
                for (int m = ncomb[leaf]; m > 0; m--) {
                    sp--;
                    stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]);
                }
            }
            const int64_t cidx = tile * BM + r;
            if (cidx < count) out[cidx] = __dmul_rn(__dadd_rn(0.0, stk[0]), cst);
        }
    } else if (warp == W_TMA) {
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)S.nc * KC;
            int bs = 0;
            uint32_t bph = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < S.nch; c++) {
                    for (int kc = 0; kc < S.nkc; kc++) {
                        const int s = bs;
                        NTW(4, mbar_wait_hw(&bars[B_S_EMPTY + s], bph ^ 1));
                        if (++bs == nst) {
                            bs = 0;
                            bph ^= 1;
                        }
#if FRR_NT_DEBUG & 1
                        mbar_arrive(&bars[B_B_FULL + s]);  // timing experiment only: no B traffic
#else
                        mbar_expect_tx(&bars[B_B_FULL + s], bytes);
                        bulk_g2s(sB + (size_t)s * bytes, bal.limbs + ((size_t)c * S.nkc + kc) * bytes, bytes,
                                 &bars[B_B_FULL + s]);
#endif
                    }
                }
            }
        }
    } else if (warp == W_MMA) {
        if (lane == 0) {
            uint32_t chunk_ctr = 0, m_ph = 0;
            int m_s = 0;
            const uint32_t b_lbo = (uint32_t)(S.nc / 8) * 128;
            const uint32_t idesc = idesc_i8(BM, S.nc);
            const uint32_t a_t0 = tmem_base + (uint32_t)(2 * S.nc);
            const uint64_t bdesc0 = umma_desc(smem_u32(sB), b_lbo, 128);
            const uint32_t b_stage16 = (uint32_t)(S.nc * KC) >> 4, b_ks16 = (2 * b_lbo) >> 4;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int c = 0; c < S.nch; c++, chunk_ctr++) {
                    const int tb = chunk_ctr & 1;
                    NTW(5, mbar_wait(&bars[B_TM_EMPTY + tb], ((chunk_ctr >> 1) & 1) ^ 1));
                    tc_fence_after();
                    const uint32_t dt = tmem_base + (uint32_t)(tb * S.nc);
                    for (int kc = 0; kc < S.nkc; kc++) {
                        const int st = m_s;
                        NTW(6, mbar_wait(&bars[B_A_FULL + st], m_ph));
                        if (++m_s == nst) {
                            m_s = 0;
                            m_ph ^= 1;
                        }
                        tc_fence_after();
                        // descriptor of stage st, K step ks = base descriptor + address offset
                        // (start address field: bits 0-13 in 16-byte units; shared
                        // addresses < 256 KB never carry out of it)
                        const uint32_t at = a_t0 + (uint32_t)st * (KC / 4);
                        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)st * b_stage16);
#pragma unroll
                        for (int ks = 0; ks < KC / 32; ks++)
                            tc_mma_i8_ts(dt, at + (uint32_t)(ks * 8), bd + (uint64_t)(ks * b_ks16), idesc, (kc | ks) != 0);
                        tc_commit(&bars[B_S_EMPTY + st]);
                    }
                    tc_commit(&bars[B_TM_FULL + tb]);
                }
            }
        }
    }

#if FRR_NT_TIMING
    {
        const int role = warp == W_MMA ? 11 : warp == W_TMA ? 12
                       : warp >= W_EPI0 && warp < W_EPI0 + 4 * EPIW ? 10
                       : warp >= W_EXP0 && warp < W_EXP0 + NEXP ? 9 : 8;
        wacc[role] += clock64() - tstart;
        if (lane == 0)
            for (int k = 0; k < 16; k++)
                if (wacc[k]) atomicAdd(&g_nt_waits[k], (unsigned long long)wacc[k]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// B operand: [chunk c][kc][k16][n8][8 rows][16 B]; chunk rows [limb][32 j]
__global__ void k_prepare_limbs_nt(const int64_t* __restrict__ zq, NtShape S, int8_t* __restrict__ limbs,
                                   int32_t* overflow) {
    const int64_t block = (int64_t)S.nc * KC;
    const int64_t total = (int64_t)S.nch * S.nkc * block;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bi = o / block;
        const int c = (int)(bi / S.nkc), kc = (int)(bi % S.nkc);
        const int rem = (int)(o % block);
        const int k16 = rem / (S.nc * 16);
        const int rem2 = rem % (S.nc * 16);
        const int nrow = (rem2 / 128) * 8 + (rem2 % 128) / 16;
        const int kb = rem2 % 16;
        const int kk = kc * KC + k16 * 16 + kb;
        const int k = frr_k_unit_nat(kk);
        const int l = nrow / DJ, j = c * DJ + nrow % DJ;
        int8_t v = 0;
        if (k < S.n && j < S.d && l < S.L) {
            // pre-shifted rows: K offset r of a 32-group is expanded with weight
            // 2^((r>>2)&3), so its limbs encode z * 2^(3-((r>>2)&3)) (all
            // products carry 8; the epilogue divides the exact sum by 8)
            int64_t z = zq[(size_t)k * S.d + j] * (int64_t)(8 >> ((kk >> 2) & 3));
            for (int q = 0; q <= l; q++) {
                v = (int8_t)(z & 0xFF);
                z = (z - v) >> 8;
            }
            if (l == S.L - 1 && z != 0) atomicExch(overflow, 1);
        }
        limbs[o] = v;
    }
}


// ------------------------------------------------------------- host side
bool fits(int n, int d, int L) {
    if (d < 8 || L < 1 || L > 8 || n > FRR_MAX_UNITS) return false;
    NtShape s = nt_shape(n, n - 1, d, L);
    if (s.nc > 256 || s.dpad / 8 > 8 * MAX_LEAVES) return false;
    if (2 * s.nc + 2 * (KC / 4) > 512) return false;  // two accumulators + >= 2 A stages in TMEM
    return s.nfy > 0;
}

size_t limbs_bytes(int n, int d, int L) {
    NtShape s = nt_shape(n, 1, d, L);
    return (size_t)s.nch * s.nkc * s.nc * KC;
}

int prepare_limbs(const int64_t* zq, int n, int d, int L, int8_t* limbs, int32_t* overflow, cudaStream_t s) {
    NtShape S = nt_shape(n, 1, d, L);
    int64_t total = (int64_t)limbs_bytes(n, d, L);
    int grid = (int)std::min<int64_t>(frr_cdiv(total, 256), (int64_t)frr_num_sms() * 16);
    k_prepare_limbs_nt<<<grid, 256, 0, s>>>(zq, S, limbs, overflow);
    return frr_launched("k_prepare_limbs_nt");
}

int mc_stats(const frr_balance_t* bal, uint64_t seed, uint64_t lo, int64_t count, double* stats, void* stream) {
    if (count <= 0) return FRR_OK;
    cudaStream_t s = frr_stream(stream);
    NtShape S = nt_shape(bal->n, bal->t, bal->d, bal->n_limbs);
    NtPlan P = nt_plan(S);
    GlobalSteps gs;
    int rc = S.gen ? 0 : gs.init(bal->n, bal->t, s);
    if (rc) return rc;
    const bool full = S.gen ? (S.nfy == RFY && S.nbits == RFY / 4 + 2) : (S.nfy == NFY && S.nbits == 2);
    const auto kern = S.gen ? (full ? k_mc_stats_nt<true, 1> : k_mc_stats_nt<false, 1>)
                            : (full ? k_mc_stats_nt<true, 0> : k_mc_stats_nt<false, 0>);
    if ((rc = frr_prepare_kernel(kern, P.total))) return rc;
    int64_t ntiles = frr_cdiv(count, BM);
    int grid = (int)std::min<int64_t>(ntiles, frr_num_sms());
    kern<<<grid, n_warps(S.nfy) * 32, P.total, s>>>(*bal, seed, lo, count, stats, gs.p);
    return frr_launched("k_mc_stats_nt");
}

#if FRR_NT_TIMING
int debug_waits(unsigned long long* host16) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host16, g_nt_waits, sizeof(unsigned long long) * 16);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_nt_waits, z, sizeof(z));
    return 0;
}
#endif

}  // namespace FRR_NT_NS

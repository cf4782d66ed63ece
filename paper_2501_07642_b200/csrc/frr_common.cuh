// frr_common.cuh -- shared device code for libfrr (sm_100a).
//
// Bit-exact restatement, on the GPU, of the reference key -> assignment
// contract (keys.py:9-38, 138-159) and of numpy's pairwise reduction order
// used by balance.py:104 and inference.py:97-98.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/frr.h"

#define FRR_GOLDEN 0x9E3779B97F4A7C15ull

// Device-side bounds / invariant checks of the FRR_CHECKS=1 diagnostic build
// (make checks): a failed check traps the kernel with its location.  The
// pool's GPUs run no compute-sanitizer, so these asserts plus oracle
// comparisons on small cases are the memory-safety evidence.
#ifndef FRR_CHECKS
#define FRR_CHECKS 0
#endif
#if FRR_CHECKS
#include <assert.h>
#define FRR_CHECK(c) assert(c)
#else
#define FRR_CHECK(c) ((void)0)
#endif
#define FRR_FULL 0xffffffffu
#define FRR_CTL 0xFFFFu  // table marker: unit is a control unit

// ---------------------------------------------------------------- error state
void frr_set_error(const char* fmt, ...);
int frr_check_launch(const char* what);
// frr_check_launch after a kernel launch, counted by frr_launch_count()
int frr_launched(const char* what);

// -------------------------------------------------------------- splitmix64
// keys.py:99-104
// 64 x 64 -> low 64 multiply by a constant in three IMADs (wide low product,
// then both cross terms accumulated straight into the high word)
__device__ __forceinline__ uint64_t frr_mul64c(uint64_t z, uint32_t clo, uint32_t chi) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 zl, zh;\n\t"
        "mov.b64 {zl, zh}, %2;\n\t"
        "mul.lo.u32 %0, zl, %3;\n\t"
        "mul.hi.u32 %1, zl, %3;\n\t"
        "mad.lo.u32 %1, zl, %4, %1;\n\t"
        "mad.lo.u32 %1, zh, %3, %1;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(z), "r"(clo), "r"(chi));
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t frr_mix64(uint64_t z) {
    z = frr_mul64c(z ^ (z >> 30), 0x1CE4E5B9u, 0xBF58476Du);
    z = frr_mul64c(z ^ (z >> 27), 0x133111EBu, 0x94D049BBu);
    return z ^ (z >> 31);
}

// z ^ (z >> s) (0 < s < 32) with the high word's shift on the FMA pipe
// (hi >> s = umulhi(hi, 2^(32-s))) instead of the ALU pipe
template <int S>
__device__ __forceinline__ uint64_t frr_xorshift_fma(uint64_t z) {
    uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t lo_s = __funnelshift_r(lo, hi, S);
    uint32_t hi_s;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi_s) : "r"(hi), "n"(1u << (32 - S)));
    return ((uint64_t)(hi ^ hi_s) << 32) | (lo ^ lo_s);
}

// mix64 with a chosen subset of the three xorshifts' high-word shifts on the
// FMA pipe (bit i of FMA_MASK: xorshift i), balancing the generator's ALU
// and FMA pipes
template <int FMA_MASK>
__device__ __forceinline__ uint64_t frr_mix64_bal(uint64_t z) {
    z = (FMA_MASK & 1) ? frr_xorshift_fma<30>(z) : z ^ (z >> 30);
    z = frr_mul64c(z, 0x1CE4E5B9u, 0xBF58476Du);
    z = (FMA_MASK & 2) ? frr_xorshift_fma<27>(z) : z ^ (z >> 27);
    z = frr_mul64c(z, 0x133111EBu, 0x94D049BBu);
    return (FMA_MASK & 4) ? frr_xorshift_fma<31>(z) : z ^ (z >> 31);
}

// keys.py:118-121
__device__ __forceinline__ uint64_t frr_derive_state(uint64_t seed, uint64_t draw) {
    return frr_mix64((seed ^ (draw * FRR_GOLDEN)) + FRR_GOLDEN);
}

// Per Fisher-Yates step k (bound b = n - k) constants for an exact
// u mod b without a division:  y = hi(u)*c2 + lo(u)  (c2 = 2^32 mod b,
// y < 2^48, y == u mod b), then Lemire-Kaser-Kurz direct remainder with
// M = ceil(2^64 / b), valid for 48-bit dividends and b <= 2^16.
struct __align__(16) StepC {
    uint32_t b;
    uint32_t c2;
    uint64_t M;
};

__host__ __device__ __forceinline__ StepC frr_make_step(int n, int k) {
    StepC s;
    s.b = (uint32_t)(n - k);
    s.c2 = (uint32_t)((1ull << 32) % s.b);
    s.M = (~0ull) / s.b + 1ull;
    return s;
}

#ifndef FRR_MOD_R_IMM0
#define FRR_MOD_R_IMM0 1  // madc.hi with an immediate zero: ptxas moves the addend copy to the ALU (C2 +0.2%)
#endif
__device__ __forceinline__ uint32_t frr_mod_step(uint64_t u, const StepC& s, uint32_t zero = 0u, uint32_t zero2 = 0u) {
    // written on 32-bit halves so the result stays a plain 32-bit register
    const uint32_t ulo = (uint32_t)u, uhi = (uint32_t)(u >> 32);
    const uint32_t mlo = (uint32_t)s.M, mhi = (uint32_t)(s.M >> 32);
    uint32_t ylo, yhi;  // y = uhi * c2 + ulo  (< 2^48)
    asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.u32 %1, %2, %3, %5;" : "=r"(ylo), "=r"(yhi) : "r"(uhi), "r"(s.c2), "r"(ulo), "r"(zero));
    // low = M * y mod 2^64
    const uint32_t llo = mlo * ylo;
    const uint32_t lhi = __umulhi(mlo, ylo) + mhi * ylo + mlo * yhi;
    // result = floor(low * b / 2^64) = hi32(lhi * b + umulhi(llo, b))
    uint32_t rhi;  // the low word of the sum only feeds the carry
#if FRR_MOD_R_IMM0
    asm("{\n\t.reg .u32 rlo;\n\tmad.lo.cc.u32 rlo, %1, %2, %3;\n\tmadc.hi.u32 %0, %1, %2, 0;\n\t}"
        : "=r"(rhi)
        : "r"(lhi), "r"(s.b), "r"(__umulhi(llo, s.b)));
    (void)zero2;
#else
    asm("{\n\t.reg .u32 rlo;\n\tmad.lo.cc.u32 rlo, %1, %2, %3;\n\tmadc.hi.u32 %0, %1, %2, %4;\n\t}"
        : "=r"(rhi)
        : "r"(lhi), "r"(s.b), "r"(__umulhi(llo, s.b)), "r"(zero2));
#endif
    return rhi;
}

// t real steps, padded to a multiple of 64 with dummies of bound b = 1
// (c2 = 0, M = 2^64 mod 2^64 = 0): frr_mod_step then returns 0, a self-swap
// that stores nothing, so two full rounds per iteration need no bounds tests.
__host__ __device__ __forceinline__ int frr_steps_len(int t) { return (t + 127) & ~127; }

__device__ inline void frr_fill_steps(StepC* steps, int n, int t) {
    for (int k = threadIdx.x; k < frr_steps_len(t); k += blockDim.x) steps[k] = frr_make_step(k < t ? n : k + 1, k);
}

// Table entries per candidate: n uint16 entries padded to a multiple of 32
// (whole 64-byte words for the packers); padding entries read as control.
__host__ __device__ __forceinline__ int frr_table_len(int n) { return (n + 31) & ~31; }
// Readable bytes every layout keeps after the last table (frr_warp_fy's
// unpredicated re-read of padding steps reaches up to 127 entries past it).
#define FRR_TABLE_SLACK 256

__device__ __forceinline__ void frr_table_fill(uint16_t* lw, int n, uint16_t v, int lane) {
    uint32_t w = (uint32_t)v | ((uint32_t)v << 16);
    uint4 q = make_uint4(w, w, w, w);
    int len = frr_table_len(n);
    for (int i = lane * 8; i < len; i += 256) *reinterpret_cast<uint4*>(lw + i) = q;
    __syncwarp();
    if (n + lane < len) lw[n + lane] = 0xFFFFu;
}

// ----------------------------------------------------------- warp generator
// One warp builds the assignment of draw (seed, draw) into the per-warp table
// lw[0..n): on return lw[e] == FRR_CTL iff unit e is a control unit.
//
// Equivalent to the reference's sequential partial Fisher-Yates
// (keys.py:146-158) but parallel over the t steps: the stream value of step
// k is mix64(state + (k+1)C) unless an earlier step rejected, which needs
// hi(u) == 0xFFFFFFFF (p ~ 2^-32); any such warp redoes the candidate
// sequentially with exact rejection.  Swaps are replaced by a "last writer"
// table: lw[p] = 1 + (last step k < p with r_k = p).  The final content of a
// position p >= t is found by following lw links to a never-written position
// (its original element); those t..n-1 contents are the control units.
__device__ __forceinline__ uint32_t frr_fy_draw(uint64_t x, const StepC* sp, uint32_t& hmax, uint32_t zero = 0u,
                                                uint32_t zero2 = 0u) {
    const uint4 q = *reinterpret_cast<const uint4*>(sp);  // one LDS.128
    StepC s;
    s.b = q.x;
    s.c2 = q.y;
    s.M = ((uint64_t)q.w << 32) | q.z;
    const uint64_t u = frr_mix64(x);
    hmax = max(hmax, (uint32_t)(u >> 32));  // a rejection needs hi(u) == 0xFFFFFFFF
    const uint32_t d = frr_mod_step(u, s, zero, zero2);
    FRR_CHECK(d < s.b && d == (uint32_t)(u % s.b));
    return d;
}

#ifndef FRR_FY_ROUNDS
#define FRR_FY_ROUNDS 4
#endif

// CLIP: steps k >= t are no-ops whatever their table record says (the
// universal global step table frr_global_steps has real bounds there; the
// per-(n, t) tables have b = 1 dummies and need no clipping).
template <bool CLIP = false>
__device__ __forceinline__ void frr_warp_fy(uint64_t state, int n, int t, const StepC* steps,
                                            uint16_t* lw, int lane) {
    constexpr int R = FRR_FY_ROUNDS;
    static_assert(!CLIP || R == 4, "step clipping is implemented for FRR_FY_ROUNDS == 4");
    frr_table_fill(lw, n, 0, lane);
    __syncwarp();
    uint32_t hmax = 0;
    // R rounds (32R steps) per iteration: independent draws for ILP; later
    // rounds hold strictly later steps, so storing the rounds in order and
    // settling them with one verify loop keeps "last writer wins".
    uint64_t x[R];
    // step slot of this lane within a round: the highest step in the lowest
    // lane, because same-address stores of one instruction mostly resolve in
    // favour of the lowest lane (fewer verify retries; correctness does not
    // depend on it)
    const int sl = 31 - lane;
    x[0] = state + (uint64_t)(sl + 1) * FRR_GOLDEN;
#pragma unroll
    for (int i = 1; i < R; i++) x[i] = x[i - 1] + 32ull * FRR_GOLDEN;
    const uint64_t stride = 32ull * R * FRR_GOLDEN;
    // (padding steps k >= t have b = 1: d = 0, no store; a spurious flag from
    // them (p ~ 2^-32) only triggers the exact slow path)
    //
    // Each round stores, then re-reads: a higher lane's store can be
    // overwritten by a lower lane's in the same instruction, so retry until
    // the largest k holds (values at a position only grow, so "pending" is
    // recomputed from a fresh read each time).
#if FRR_FY_ROUNDS == 2
    // loop-carried step pointer, table address of lw[k] and k + 1 (round 0;
    // round 1 is +32 steps) instead of per-iteration index arithmetic.  The
    // re-read is unpredicated: with d = 0, r = k can lie up to 63 entries
    // past the table (padding steps), which every layout leaves readable
    // (FRR_TABLE_SLACK); the value is ignored there.
    const uint32_t lwa = (uint32_t)__cvta_generic_to_shared(lw);
    const StepC* sp = steps + sl;
    uint32_t ka = lwa + 2u * (uint32_t)sl, v0 = (uint32_t)sl + 1u;
    const uint32_t kend = ka + 2u * (uint32_t)t;  // base < t
    // zeros opaque to the compiler: live zero high words of the 64-bit
    // addends in frr_mod_step (saves re-zeroing a register pair per use)
    uint32_t z[4];
#pragma unroll
    for (int i = 0; i < 4; i++) z[i] = (uint32_t)(t + i) >> 31;
    for (; ka < kend; ka += 128u, v0 += 64u, sp += 64) {
        const uint32_t d0 = frr_fy_draw(x[0], sp, hmax, z[0], z[1]), d1 = frr_fy_draw(x[1], sp + 32, hmax, z[2], z[3]);
        x[0] += stride;
        x[1] += stride;
        uint32_t any;
        asm volatile(
            "{\n\t.reg .pred q0, q1;\n\t.reg .u32 x0, x1;\n\t"
            "setp.ne.u32 q0, %1, 0;\n\t"
            "setp.ne.u32 q1, %4, 0;\n\t"
            "@q0 st.shared.u16 [%2], %3;\n\t"
            "@q1 st.shared.u16 [%5], %6;\n\t"
            "bar.warp.sync 0xffffffff;\n\t"
            "ld.shared.u16 x0, [%2];\n\t"
            "ld.shared.u16 x1, [%5];\n\t"
            "setp.lt.and.u32 q0, x0, %3, q0;\n\t"
            "setp.lt.and.u32 q1, x1, %6, q1;\n\t"
            "or.pred q0, q0, q1;\n\t"
            "vote.sync.any.pred q0, q0, 0xffffffff;\n\t"
            "selp.u32 %0, 1, 0, q0;\n\t}"
            : "=r"(any)
            : "r"(d0), "r"(ka + 2u * d0), "r"(v0), "r"(d1), "r"(ka + 64u + 2u * d1), "r"(v0 + 32u)
            : "memory");
        if (any) {
            const uint32_t d[2] = {d0, d1}, v[2] = {v0, v0 + 32u}, r[2] = {v0 - 1u + d0, v0 + 31u + d1};
#elif FRR_FY_ROUNDS == 4
    const uint32_t lwa = (uint32_t)__cvta_generic_to_shared(lw);
    const StepC* sp = steps + sl;
    uint32_t ka = lwa + 2u * (uint32_t)sl, v0 = (uint32_t)sl + 1u;
    const uint32_t kend = ka + 2u * (uint32_t)t;
    uint32_t z[4];
#pragma unroll
    for (int i = 0; i < 4; i++) z[i] = (uint32_t)(t + i) >> 31;
    for (; ka < kend; ka += 256u, v0 += 128u, sp += 128) {
        uint32_t d[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            d[i] = frr_fy_draw(x[i], sp + 32 * i, hmax, z[(2 * i) & 3], z[(2 * i + 1) & 3]);
            if (CLIP && v0 + 32u * i > (uint32_t)t) d[i] = 0;  // step k = v0 + 32 i - 1 >= t
            x[i] += stride;
        }
        uint32_t any;
        asm volatile(
            "{\n\t.reg .pred q0, q1, q2, q3;\n\t.reg .u32 x0, x1, x2, x3;\n\t"
            "setp.ne.u32 q0, %1, 0;\n\t"
            "setp.ne.u32 q1, %4, 0;\n\t"
            "setp.ne.u32 q2, %7, 0;\n\t"
            "setp.ne.u32 q3, %10, 0;\n\t"
            "@q0 st.shared.u16 [%2], %3;\n\t"
            "@q1 st.shared.u16 [%5], %6;\n\t"
            "@q2 st.shared.u16 [%8], %9;\n\t"
            "@q3 st.shared.u16 [%11], %12;\n\t"
            "bar.warp.sync 0xffffffff;\n\t"
            "ld.shared.u16 x0, [%2];\n\t"
            "ld.shared.u16 x1, [%5];\n\t"
            "ld.shared.u16 x2, [%8];\n\t"
            "ld.shared.u16 x3, [%11];\n\t"
            "setp.lt.and.u32 q0, x0, %3, q0;\n\t"
            "setp.lt.and.u32 q1, x1, %6, q1;\n\t"
            "setp.lt.and.u32 q2, x2, %9, q2;\n\t"
            "setp.lt.and.u32 q3, x3, %12, q3;\n\t"
            "or.pred q0, q0, q1;\n\t"
            "or.pred q2, q2, q3;\n\t"
            "or.pred q0, q0, q2;\n\t"
            "vote.sync.any.pred q0, q0, 0xffffffff;\n\t"
            "selp.u32 %0, 1, 0, q0;\n\t}"
            : "=r"(any)
            : "r"(d[0]), "r"(ka + 2u * d[0]), "r"(v0), "r"(d[1]), "r"(ka + 64u + 2u * d[1]), "r"(v0 + 32u),
              "r"(d[2]), "r"(ka + 128u + 2u * d[2]), "r"(v0 + 64u), "r"(d[3]), "r"(ka + 192u + 2u * d[3]),
              "r"(v0 + 96u)
            : "memory");
        if (any) {
            const uint32_t v[4] = {v0, v0 + 32u, v0 + 64u, v0 + 96u};
            const uint32_t r[4] = {v[0] - 1u + d[0], v[1] - 1u + d[1], v[2] - 1u + d[2], v[3] - 1u + d[3]};
#else
    for (int base = 0; base < t; base += 32 * R) {
        uint32_t d[R], r[R], v[R];
#pragma unroll
        for (int i = 0; i < R; i++) {
            const int k = base + 32 * i + sl;
            d[i] = frr_fy_draw(x[i], steps + k, hmax);
            r[i] = (uint32_t)k + d[i];
            v[i] = (uint32_t)k + 1;
            x[i] += stride;
        }
#pragma unroll
        for (int i = 0; i < R; i++)
            if (d[i] != 0) lw[r[i]] = (uint16_t)v[i];
        __syncwarp();
        bool pend = false;
#pragma unroll
        for (int i = 0; i < R; i++) pend |= d[i] != 0 && (uint32_t)lw[r[i]] < v[i];
        if (__any_sync(FRR_FULL, pend)) {
#endif
            bool pend;
            do {
#pragma unroll
                for (int i = 0; i < R; i++)
                    if (d[i] != 0 && (uint32_t)lw[r[i]] < v[i]) lw[r[i]] = (uint16_t)v[i];
                __syncwarp();
                pend = false;
#pragma unroll
                for (int i = 0; i < R; i++) pend |= d[i] != 0 && (uint32_t)lw[r[i]] < v[i];
            } while (__any_sync(FRR_FULL, pend));
        }
    }
    __syncwarp();
    const bool flag = hmax == 0xFFFFFFFFu;
    if (__any_sync(FRR_FULL, flag)) {
        // exact sequential restatement with rejection (keys.py:146-156)
        __syncwarp();
        frr_table_fill(lw, n, 0, lane);
        __syncwarp();
        if (lane == 0) {
            uint64_t s = state;
            for (int j = 0; j < t; j++) {
                uint64_t b = (uint64_t)(n - j);
                uint64_t rem = (0ull - b) % b;
                uint64_t u;
                do {
                    s += FRR_GOLDEN;
                    u = frr_mix64(s);
                } while (rem != 0 && u >= 0ull - rem);
                uint32_t r = (uint32_t)j + (uint32_t)(u % b);
                FRR_CHECK(r < (uint32_t)n);
                if (r != (uint32_t)j) lw[r] = (uint16_t)(j + 1);
            }
        }
        __syncwarp();
    }
    // Each lane walks its positions p = t+lane, t+lane+32, ... one link per
    // iteration, S interleaved walks for memory-level parallelism.  Chains
    // are disjoint and end at distinct roots, so marking a root never
    // disturbs another walk.
    {
        // walk on 32-bit shared addresses: link q -> lw[v - 1] is one IMAD
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(lw);
        const uint32_t ea = base + 2u * (uint32_t)n, vbase = base - 2u;
        uint32_t pa = base + 2u * (uint32_t)(t + lane), qa = pa;
        if (pa < ea) {
            // one link per iteration: a zero entry is a root (mark it, move to
            // this lane's next start), else follow to lw[v - 1]
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t.reg .u32 v, nx;\n"
                "FRR_WALK_LOOP:\n\t"
                "ld.shared.u16 v, [%0];\n\t"
                "setp.eq.u32 p, v, 0;\n\t"
                "mad.lo.u32 nx, v, 2, %3;\n\t"
                "@p st.shared.u16 [%0], %4;\n\t"
                "@p add.u32 %1, %1, 64;\n\t"
                "selp.u32 %0, %1, nx, p;\n\t"
                "setp.lt.u32 q, %1, %2;\n\t"
                "@q bra FRR_WALK_LOOP;\n\t}"
                : "+r"(qa), "+r"(pa)
                : "r"(ea), "r"(vbase), "r"((uint32_t)n | FRR_CTL)  // low half FRR_CTL, kept in a register
                : "memory");
        }
    }
    __syncwarp();
}

// Packed treated bits of one 32-unit word for t < 32768 (step marks k+1 <
// 2^15, so bit 15 of an entry is set exactly for control units).  Bit
// position -> unit map (the tensor-core B operand uses the same order):
// bit 15-i <- unit 32w+2i, bit 31-i <- unit 32w+2i+1, i = 0..15.
__host__ __device__ __forceinline__ int frr_packed_unit(int w, int p) {
    return p < 16 ? 32 * w + 2 * (15 - p) : 32 * w + 2 * (31 - p) + 1;
}

// Tensor-core K order inside a packed word: K offset r (0..31) holds bit
// 8*(r & 3) + (r >> 2), so the int8 0/1 expansion of bit word w is eight
// registers ((w >> q) & 0x01010101), q = 0..7 (byte b of register q = K
// offset 4q + b).  The B operand rows are permuted to the same order.
__host__ __device__ __forceinline__ int frr_kpos_bit(int r) { return 8 * (r & 3) + (r >> 2); }
__host__ __device__ __forceinline__ int frr_k_unit(int kk) { return frr_packed_unit(kk >> 5, frr_kpos_bit(kk & 31)); }
// the same K order over words in natural unit order (bit b of word w = unit
// 32 w + b): the single-pass tensor-core kernel's tile rows
__host__ __device__ __forceinline__ int frr_k_unit_nat(int kk) { return 32 * (kk >> 5) + frr_kpos_bit(kk & 31); }

__device__ __forceinline__ uint32_t frr_pack_word(const uint16_t* lw, int w) {
    const uint4* src = reinterpret_cast<const uint4*>(lw + 32 * w);
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const int cc = (c + w) & 3;  // rotate 16-byte chunks: conflict-free across lanes
        const uint4 v = src[cc];
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
        // component i = 4 cc + j contributes (~x & 0x80008000) >> i: compile-time
        // shifts by j inside the chunk, one runtime shift by 4 cc per chunk
        uint32_t part = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) part |= ~(x[j] >> j) & (0x80008000u >> j);
        acc |= part >> (4 * cc);
    }
    return acc;
}

// Packed treated bits of the table: word w (units 32w..32w+31) lands in
// lane (w & 31)'s return slot for its words; one ballot per word.
template <class Store>
__device__ __forceinline__ void frr_table_bits(const uint16_t* lw, int n, int words, int lane, Store store) {
    for (int w = 0; w < words; w++) {
        const int e = w * 32 + lane;
        const uint32_t word = __ballot_sync(FRR_FULL, e < n && lw[e] != FRR_CTL);
        if (lane == (w & 31)) store(w, word);
    }
}

// ---------------------------------------------------- exact (combinadic)
// generation.py:257-266: itertools.combinations order == lexicographic
// combinadic unranking.  binom(a, b) exact in 64 bits for a <= 67.
// Pascal's triangle for a <= 67 (every entry fits 64 bits), built at compile
// time into constant memory.
struct FrrBinomTable {
    uint64_t v[68][68];
    constexpr FrrBinomTable() : v() {
        for (int a = 0; a < 68; a++)
            for (int b = 0; b <= a; b++) v[a][b] = (b == 0 || b == a) ? 1ull : v[a - 1][b - 1] + v[a - 1][b];
    }
};
static __constant__ FrrBinomTable c_frr_binom = FrrBinomTable();

__device__ __forceinline__ uint64_t frr_binom(int a, int b) {
    if (b < 0 || b > a) return 0;
    if (a < 68) return c_frr_binom.v[a][b];
    if (b > a - b) b = a - b;
    unsigned __int128 r = 1;
    for (int i = 1; i <= b; i++) r = r * (unsigned)(a - b + i) / (unsigned)i;
    return (uint64_t)r;
}

// Writes the t treated units of lexicographic rank `rank` into table lw as
// "not control" (others FRR_CTL).  Single lane, any n.
__device__ inline void frr_unrank_to_table(uint64_t rank, int n, int t, uint16_t* lw) {
    int x = 0;
    for (int i = 0; i < t; i++) {
        // skip C(n-x-1, t-i-1) combinations per unit passed over
        const int b = t - i - 1;
        uint64_t c;
        while (rank >= (c = frr_binom(n - x - 1, b))) {
            rank -= c;
            x++;
        }
        lw[x] = 0;
        x++;
    }
}

// --------------------------------------------------------- pairwise sums
// numpy pairwise_sum (PW_BLOCKSIZE 128) on a leaf of length len, values
// produced by f(i) for i in [0, len).
template <class F>
__device__ __forceinline__ double frr_pw_leaf(int len, F f) {
    if (len < 8) {
        double res = -0.0;
        for (int i = 0; i < len; i++) res = __dadd_rn(res, f(i));
        return res;
    }
    double r0 = f(0), r1 = f(1), r2 = f(2), r3 = f(3), r4 = f(4), r5 = f(5), r6 = f(6), r7 = f(7);
    int i = 8;
    int full = len - (len % 8);
    for (; i < full; i += 8) {
        r0 = __dadd_rn(r0, f(i + 0));
        r1 = __dadd_rn(r1, f(i + 1));
        r2 = __dadd_rn(r2, f(i + 2));
        r3 = __dadd_rn(r3, f(i + 3));
        r4 = __dadd_rn(r4, f(i + 4));
        r5 = __dadd_rn(r5, f(i + 5));
        r6 = __dadd_rn(r6, f(i + 6));
        r7 = __dadd_rn(r7, f(i + 7));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < len; i++) res = __dadd_rn(res, f(i));
    return res;
}

// Whole pairwise sum of a[0..n) held in (shared or global) memory; single
// thread; recursion depth <= log2(n/64).  Returns 0.0 + pw (the reduction
// starts from the additive identity).
__device__ inline double frr_pw_rec(const double* a, int n) {
    if (n <= 128) return frr_pw_leaf(n, [&](int i) { return a[i]; });
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(frr_pw_rec(a, n2), frr_pw_rec(a + n2, n - n2));
}

__device__ inline double frr_pw_sum(const double* a, int n) { return __dadd_rn(0.0, frr_pw_rec(a, n)); }

// --------------------------------------------------------- small helpers
__device__ __forceinline__ uint64_t frr_f64_bits(double x) { return (uint64_t)__double_as_longlong(x); }

__host__ __device__ __forceinline__ int64_t frr_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// frr_revfy.cuh -- thread-per-candidate key -> assignment generator
// ("reverse bitset" Fisher-Yates), sm_100a.
//
// The reference draws r_j = j + u_j mod (n - j) for j = 0..t-1 and swaps
// perm[j] <-> perm[r_j] (keys.py:146-158); the treated units are perm[0..t).
// With perm_0 = identity, the final array is perm_t[x] = tau_0(tau_1(...
// tau_{t-1}(x))) (tau_j the transposition (j r_j)), so the CONTROL set is
// the image of the position set {t..n-1} under tau_0 o ... o tau_{t-1}:
// start from the bitset B = {t..n-1} and apply the transpositions in
// reverse order, j = t-1 down to 0.  Before reverse step j, bit j is still
// 0 (steps > j only touch positions > j), so the swap is
//
//     bit = B[r_j];  B[r_j] = 0;  B[j] |= bit
//
// and the state is an n-bit set (128 B at n = 1000) instead of a 2n-byte
// permutation: one candidate per thread, no last-writer table, no verify
// loop, no chain walk, and the final B is already the packed control mask
// the tensor-core operand is built from.
//
// The stream value of step j is mix64(state + (j+1) C) unless an earlier
// step rejected (keys.py:150-154), which needs hi(u) == 0xFFFFFFFF
// (p ~ 2^-32 per draw): the generator reports such candidates and the caller
// recomputes them with the exact sequential rule (frr_warp_fy).
#pragma once
#include "frr_common.cuh"

// Shared-memory layout of a warp's 32 bitsets: word w of lane l at
// ws_base + (w * 32 + l) * 4 -- every lane in its own bank whatever word it
// touches.  Bit b of word w <-> unit 32 w + b; 1 = control.
#ifndef FRR_REV_GROUP
#define FRR_REV_GROUP 8  // draws computed ahead of their bit moves (divides 32)
#endif
#ifndef FRR_REV_FMA_MASK
#define FRR_REV_FMA_MASK 0  // xorshifts whose high-word shift runs on the FMA pipe (frr_mix64_bal)
#endif
#ifndef FRR_REV_PIPE
#define FRR_REV_PIPE 0  // 1: next group's draws ahead of the bit moves; 2: interleaved draw/move
#endif
#ifndef FRR_REV_RA_ALU
#define FRR_REV_RA_ALU 1  // r's word index by shr (ALU) instead of mul.hi (FMA pipe): C2 +2.7% (the FMA pipe is the busiest, 72%)
#endif
#ifndef FRR_REV_FETCH_AND
#define FRR_REV_FETCH_AND 1  // 1: atom.and fetch-and-clear for the r-side bit
#endif

// one step-constant record (b, c2, M) of the shared step table; pure
// register function of its address for the compiler (the table is
// read-only while generators run), so loads can be hoisted ahead of the
// bitset traffic
__device__ __forceinline__ StepC frr_lds_step(uint32_t a) {
    uint32_t x, y, z, w;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
    StepC s;
    s.b = x;
    s.c2 = y;
    s.M = ((uint64_t)w << 32) | z;
    return s;
}

// the same record from a global step table (read-only for the kernel's
// lifetime: non-coherent loads, L1-cached; every lane loads the same address)
__device__ __forceinline__ StepC frr_ldg_step(uint64_t a) {
    uint32_t x, y, z, w;
    asm("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(a));
    StepC s;
    s.b = x;
    s.c2 = y;
    s.M = ((uint64_t)w << 32) | z;
    return s;
}

// words [from, to) of this lane's bitset = all ones (positions >= t: the
// initial set; padding beyond n stays control, its operand rows are zero)
__device__ __forceinline__ void frr_rev_fill(uint32_t wsa, int from, int to) {
    for (int w = from; w < to; w++) asm volatile("st.shared.u32 [%0], %1;" ::"r"(wsa + 128u * (uint32_t)w), "r"(~0u) : "memory");
}

// One draw of the group (step record at sa): d and hi(u).
template <bool GS>
__device__ __forceinline__ uint32_t frr_rev_draw1(uint64_t& x, uint64_t sa, uint32_t z0, uint32_t z1, uint32_t& h) {
    x -= FRR_GOLDEN;
    const StepC s = GS ? frr_ldg_step(sa) : frr_lds_step((uint32_t)sa);
    const uint64_t u = frr_mix64_bal<FRR_REV_FMA_MASK>(x);
    h = (uint32_t)(u >> 32);
    const uint32_t d = frr_mod_step(u, s, z0, z1);
    FRR_CHECK(d < s.b && d == (uint32_t)(u % s.b));
    return d;
}

// Builds the control bitset of candidate `state` into this lane's column of
// the warp's bitset block (wsa = shared address of word 0 of this lane).
// kw words are written (kw >= ceil(n / 32)).  steps: shared address of the
// step table (frr_fill_steps: steps k >= t are dummies with b = 1, d = 0).
// Returns true when some stream value had hi == 0xFFFFFFFF (possible
// rejection: the candidate must be recomputed exactly).
// GS: `steps` is the generic address of a global step table (frees the
// table's shared memory for more bitsets), else a shared address.
// One reverse step's bit move: fetch-and-clear bit r (= 32 W + e) of the
// r-side word, OR it into bit jb = e - d of word W (address wa).  Program
// order of one thread's shared accesses keeps the r == j and same-word
// cases right.
__device__ __forceinline__ void frr_rev_move(uint32_t wa, uint32_t e, uint32_t d) {
    uint32_t ra;  // r's word is W + e / 32
#if FRR_REV_RA_ALU
    asm volatile("{\n\t.reg .u32 q;\n\tshr.u32 q, %1, 5;\n\tshl.b32 q, q, 7;\n\tadd.u32 %0, q, %2;\n\t}" : "=r"(ra) : "r"(e), "r"(wa));
#else
    asm("{\n\t.reg .u32 q;\n\tmul.hi.u32 q, %1, 0x8000000;\n\tmad.lo.u32 %0, q, 128, %2;\n\t}" : "=r"(ra) : "r"(e), "r"(wa));
#endif
#if FRR_REV_FETCH_AND
    // nm = ~(1 << (e & 31)); the rotation of the isolated bit right by d lands it on jb
    asm volatile(
        "{\n\t.reg .u32 w, c, nm, v;\n\t"
        "shf.l.wrap.b32 nm, %4, %4, %1;\n\t"
        "atom.shared.and.b32 w, [%0], nm;\n\t"
        "lop3.b32 c, w, nm, 0, 0x30;\n\t"  // w & ~nm
        "shf.r.wrap.b32 v, c, c, %3;\n\t"
        "red.shared.or.b32 [%2], v;\n\t}" ::"r"(ra),
        "r"(e), "r"(wa), "r"(d), "r"(0xFFFFFFFEu)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .u32 w, c, m, v;\n\t"
        "shf.l.wrap.b32 m, 1, 1, %1;\n\t"
        "ld.shared.u32 w, [%0];\n\t"
        "and.b32 c, w, m;\n\t"
        "xor.b32 w, w, c;\n\t"
        "st.shared.u32 [%0], w;\n\t"
        "shf.r.wrap.b32 v, c, c, %3;\n\t"
        "red.shared.or.b32 [%2], v;\n\t}" ::"r"(ra),
        "r"(e), "r"(wa), "r"(d)
        : "memory");
#endif
}

// FRR_REV_GROUP draws of consecutive steps (descending j from the record at
// address sa): d values and the running max of hi(u).  x = state + (j+1) C
// of the next step, decremented per draw.
template <bool GS>
__device__ __forceinline__ void frr_rev_draws(uint64_t& x, uint64_t sa, uint32_t z0, uint32_t z1,
                                              uint32_t (&dd)[FRR_REV_GROUP], uint32_t& hmax) {
    uint32_t hh[FRR_REV_GROUP];
#pragma unroll
    for (int i = 0; i < FRR_REV_GROUP; i++) {
        x -= FRR_GOLDEN;
        const StepC s = GS ? frr_ldg_step(sa - 16ull * (uint64_t)i) : frr_lds_step((uint32_t)sa - 16u * (uint32_t)i);
        const uint64_t u = frr_mix64_bal<FRR_REV_FMA_MASK>(x);
        hh[i] = (uint32_t)(u >> 32);
        dd[i] = frr_mod_step(u, s, z0, z1);
        FRR_CHECK(dd[i] < s.b && dd[i] == (uint32_t)(u % s.b));
    }
    // a rejection needs hi(u) == 0xFFFFFFFF: running max, two draws per three-input max
#pragma unroll
    for (int i = 0; i + 1 < FRR_REV_GROUP; i += 2) hmax = max(hmax, max(hh[i], hh[i + 1]));
    if (FRR_REV_GROUP & 1) hmax = max(hmax, hh[FRR_REV_GROUP - 1]);
}

// Builds the control bitset of candidate `state` into this lane's column of
// the warp's bitset block (wsa = shared address of word 0 of this lane).
// kw words are written (kw >= ceil(n / 32)).  steps: shared address of the
// step table (frr_fill_steps: steps k >= t are dummies with b = 1, d = 0);
// GS: the generic address of a global step table instead.
// Returns true when some stream value had hi == 0xFFFFFFFF (possible
// rejection: the candidate must be recomputed exactly).
//
// Software-pipelined: the draws of the next FRR_REV_GROUP steps are issued
// ahead of the current group's bit moves, so their independent register
// work fills the latency of the serial shared-memory chain (each move's
// atomic must return before its OR).
template <bool GS = false>
__device__ __forceinline__ bool frr_rev_fy(uint64_t state, int t, uint64_t steps, uint32_t wsa, int kw) {
    constexpr int GPW = 32 / FRR_REV_GROUP;  // groups per 32-step word block
    const int wtop = (t - 1) >> 5;
    // whole groups of the top word above step t - 1 are dummies: skipped
    const int q0 = (31 - ((t - 1) & 31)) / FRR_REV_GROUP;
    frr_rev_fill(wsa, wtop + 1, kw);
    uint32_t hmax = 0;
    // zeros opaque to the compiler: the high words of frr_mod_step's 64-bit
    // addends stay live instead of being re-zeroed every draw
    uint32_t z0 = (uint32_t)t >> 31, z1 = (uint32_t)(t + 1) >> 31;
    // x = state + (j + 1) C for the step j about to be drawn; sa = its record
    const int j0 = 32 * wtop + 31 - FRR_REV_GROUP * q0;
    uint64_t x = state + (uint64_t)(j0 + 2) * FRR_GOLDEN;
    uint64_t sa = steps + 16ull * (uint64_t)j0;
    uint32_t dn[FRR_REV_GROUP];
    frr_rev_draws<GS>(x, sa, z0, z1, dn, hmax);
    sa -= 16ull * FRR_REV_GROUP;
    for (int W = wtop; W >= 0; W--) {
        const uint32_t wa = wsa + 128u * (uint32_t)W;
        // word W before its own steps: positions >= t set
        const int lo = 32 * W;
        const uint32_t init = t >= lo + 32 ? 0u : (~0u << (t - lo));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(wa), "r"(init) : "memory");
#pragma unroll
        for (int q = 0; q < GPW; q++) {
            if (W == wtop && q < q0) continue;
            uint32_t dd[FRR_REV_GROUP];
#pragma unroll
            for (int i = 0; i < FRR_REV_GROUP; i++) dd[i] = dn[i];
            if (FRR_REV_PIPE == 1 && (q < GPW - 1 || W > 0)) {  // the next group (the last one has none)
                frr_rev_draws<GS>(x, sa, z0, z1, dn, hmax);
                sa -= 16ull * FRR_REV_GROUP;
            }
            if (FRR_REV_PIPE == 2) {
                // interleaved: the next group's draw i fills the latency of
                // this group's bit move i (each move waits for its atomic)
                const bool more = q < GPW - 1 || W > 0;
                uint32_t hh[FRR_REV_GROUP];
#pragma unroll
                for (int i = 0; i < FRR_REV_GROUP; i++) {
                    const int jb = 31 - q * FRR_REV_GROUP - i;
                    FRR_CHECK(32 * W + jb + (int)dd[i] < 32 * kw);  // r inside this lane's bitset
                    frr_rev_move(wa, (uint32_t)jb + dd[i], dd[i]);
                    hh[i] = 0;
                    if (more) dn[i] = frr_rev_draw1<GS>(x, sa - 16ull * (uint64_t)i, z0, z1, hh[i]);
                }
#pragma unroll
                for (int i = 0; i + 1 < FRR_REV_GROUP; i += 2) hmax = max(hmax, max(hh[i], hh[i + 1]));
                if (more) sa -= 16ull * FRR_REV_GROUP;
                continue;
            }
#pragma unroll
            for (int i = 0; i < FRR_REV_GROUP; i++) {
                const int jb = 31 - q * FRR_REV_GROUP - i;
                FRR_CHECK(32 * W + jb + (int)dd[i] < 32 * kw);  // r inside this lane's bitset
                frr_rev_move(wa, (uint32_t)jb + dd[i], dd[i]);
            }
            if (!FRR_REV_PIPE && (q < GPW - 1 || W > 0)) {
                frr_rev_draws<GS>(x, sa, z0, z1, dn, hmax);
                sa -= 16ull * FRR_REV_GROUP;
            }
        }
    }
    return hmax == 0xFFFFFFFFu;
}

// Exact recomputation of one lane's candidate (src_lane) of the warp with
// the sequential-rule warp generator (frr_warp_fy, rejection included) in
// the scratch table lw, then its control bits into that lane's bitset column.
// All 32 lanes call it together.
__device__ inline void frr_rev_fixup(uint64_t state, int n, int t, const StepC* steps, uint16_t* lw,
                                     uint32_t wsa_src, int kw, int lane) {
    frr_warp_fy(state, n, t, steps, lw, lane);
    for (int w = 0; w < kw; w++) {
        const int e = 32 * w + lane;
        const uint32_t word = __ballot_sync(FRR_FULL, e >= n || lw[e] == FRR_CTL);
        if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(wsa_src + 128u * (uint32_t)w), "r"(word) : "memory");
    }
    __syncwarp();
}

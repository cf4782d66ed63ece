// frr_rev.cu -- thread-per-candidate generator (frr_revfy.cuh) as a
// stand-alone kernel: Monte Carlo draws -> packed control bitsets.
//
// Serves the generator microbenchmark (throughput of the bare key ->
// assignment work, frr_microbench_revfy) and its GPU parity check against
// the warp generator / the reference keys (frr_rev_bits).
#include <cuda_runtime.h>

// 16 draws ahead of their bit moves in this kernel (C5 at n = 5000, 11
// warps/SM with 128 registers: +2.4% over 8; the fused C2 kernel keeps 8)
#ifndef FRR_REV_GROUP
#define FRR_REV_GROUP 16
#endif
#include "frr_common.cuh"
#include "frr_launch.cuh"
#include "frr_revfy.cuh"

namespace {
constexpr int kRevWarps = 16;

struct RevPlan {
    int kw, warps;
    size_t steps_off, ws_off, fix_off, lock_off, total;
};

// gsteps: the step table lives in global memory (the caller's workspace)
RevPlan rev_plan(int n, int t, bool gsteps = false) {
    RevPlan p;
    p.kw = (n + 31) / 32;
    p.warps = kRevWarps;
    const size_t steps_b = gsteps ? 0 : (size_t)frr_steps_len(t) * sizeof(StepC);
    // fewer warps when the bitsets of 16 do not fit shared memory
    while (p.warps > 1 && (size_t)p.warps * 32 * p.kw * 4 + steps_b + (size_t)frr_table_len(n) * 2 +
                                  FRR_TABLE_SLACK + 64 > 227 * 1024)
        p.warps--;
    size_t o = 0;
    p.steps_off = o;
    o += steps_b;
    p.ws_off = o;
    o += (size_t)p.warps * 32 * p.kw * 4;
    p.fix_off = o;
    o += (size_t)frr_table_len(n) * 2 + FRR_TABLE_SLACK;
    o = (o + 15) & ~(size_t)15;
    p.lock_off = o;
    o += 16;
    p.total = o;
    return p;
}

// Candidate c = draw ids[c] (ids != NULL) or lo + c.  out: control bits
// (bit e of word e/32 = unit e), row-major [count][kw] (interleaved = 0) or
// [count/32][kw][32] (interleaved = 1: a warp's block as built, coalesced
// stores; frr_dim_mc_ws reads it back per lane); optional.  sink: XOR of
// every candidate's words (optional; keeps the work alive in benchmarks).
// GS: the step table `gsteps` is in global memory (filled by the caller),
// else this kernel fills a shared copy
template <bool GS>
__global__ void __launch_bounds__(kRevWarps * 32) k_rev_bits(uint64_t seed, const uint64_t* __restrict__ ids,
                                                             uint64_t lo, int64_t count, int n, int t, RevPlan P,
                                                             uint32_t* __restrict__ out, int interleaved,
                                                             unsigned long long* sink, const StepC* gsteps) {
    extern __shared__ __align__(16) unsigned char smem[];
    StepC* steps = GS ? const_cast<StepC*>(gsteps) : reinterpret_cast<StepC*>(smem + P.steps_off);
    uint16_t* fix = reinterpret_cast<uint16_t*>(smem + P.fix_off);
    int* lock = reinterpret_cast<int*>(smem + P.lock_off);
    if (!GS) frr_fill_steps(steps, n, t);
    if (threadIdx.x == 0) *lock = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t sst = GS ? (uint64_t)steps : (uint64_t)__cvta_generic_to_shared(steps);
    const uint32_t wsa0 = (uint32_t)__cvta_generic_to_shared(smem + P.ws_off) + (uint32_t)warp * 128u * P.kw;
    const uint32_t wsa = wsa0 + 4u * lane;
    uint32_t acc = 0;
    const int64_t njobs = (count + 31) / 32;
    for (int64_t job = (int64_t)blockIdx.x * P.warps + warp; job < njobs; job += (int64_t)gridDim.x * P.warps) {
        const int64_t c = job * 32 + lane;
        const uint64_t state =
            frr_derive_state(seed, ids ? ids[c < count ? c : count - 1] : lo + (uint64_t)c);
        const bool flag = frr_rev_fy<GS>(state, t, sst, wsa, P.kw);
        uint32_t fl = __ballot_sync(FRR_FULL, flag);
        while (fl) {
            const int src = __ffs(fl) - 1;
            fl &= fl - 1;
            if (lane == 0)
                while (atomicCAS(lock, 0, 1) != 0) {
                }
            __syncwarp();
            frr_rev_fixup(__shfl_sync(FRR_FULL, state, src), n, t, steps, fix, wsa0 + 4u * src, P.kw, lane);
            if (lane == 0) atomicExch(lock, 0);
            __syncwarp();
        }
        for (int w = 0; w < P.kw; w++) {
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(wsa + 128u * (uint32_t)w) : "memory");
            acc ^= v * (uint32_t)(2 * w + 1);
            if (out && interleaved) out[((size_t)job * P.kw + w) * 32 + lane] = v;
            else if (out && c < count) out[(size_t)c * P.kw + w] = v;
        }
    }
    if (sink && acc) atomicXor(sink, (unsigned long long)acc);
}
}  // namespace

__global__ void k_fill_steps_ws(StepC* steps, int n, int t) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < frr_steps_len(t); k += gridDim.x * blockDim.x)
        steps[k] = frr_make_step(k < t ? n : k + 1, k);
}

// the global step table (when the caller provides one) unless the shared
// copy leaves as many warps' bitsets room (n = 5000: 11 warps instead of 9,
// +7% through frr_dim_mc_ws)
static bool rev_use_gsteps(int n, int t) { return rev_plan(n, t, false).warps < rev_plan(n, t, true).warps; }

// keys per full wave of the generator (every resident warp busy once) when
// the caller provides a global step table; 0 on error
int64_t frr_rev_wave_keys(int n, int t) {
    if (n < 2 || t < 1 || t >= n || n > FRR_MAX_UNITS) return 0;
    const bool gs = rev_use_gsteps(n, t);
    const RevPlan P = rev_plan(n, t, gs);
    const auto kern = gs ? k_rev_bits<true> : k_rev_bits<false>;
    if (P.total > 227 * 1024 || frr_prepare_kernel(kern, P.total)) return 0;
    return (int64_t)frr_persistent_grid(kern, P.warps * 32, P.total, INT64_MAX) * P.warps * 32;
}

// gsteps: caller memory of frr_steps_len(t) * 16 bytes for a global step
// table (NULL: shared copy per CTA)
static int rev_launch(uint64_t root_seed, const uint64_t* ids, uint64_t draw_lo, int64_t count, int n, int t,
                      uint32_t* bits, int interleaved, unsigned long long* sink, StepC* gsteps, void* stream) {
    if (n < 2 || t < 1 || t >= n || n > FRR_MAX_UNITS) {
        frr_set_error("frr_rev_bits: need 0 < t < n <= %d", FRR_MAX_UNITS);
        return FRR_E_INVALID_DESIGN;
    }
    if (count <= 0) return FRR_OK;
    if (gsteps && !rev_use_gsteps(n, t)) gsteps = nullptr;
    const RevPlan P = rev_plan(n, t, gsteps != nullptr);
    if (P.total > 227 * 1024) {
        frr_set_error("frr_rev_bits: n=%d too large for the shared bitsets", n);
        return FRR_E_UNSUPPORTED;
    }
    const auto kern = gsteps ? k_rev_bits<true> : k_rev_bits<false>;
    int rc = frr_prepare_kernel(kern, P.total);
    if (rc) return rc;
    cudaStream_t s = frr_stream(stream);
    if (gsteps) {
        k_fill_steps_ws<<<std::max(1, frr_steps_len(t) / 256), 256, 0, s>>>(gsteps, n, t);
        if ((rc = frr_launched("k_fill_steps_ws"))) return rc;
    }
    const int grid = frr_persistent_grid(kern, P.warps * 32, P.total, frr_cdiv(count, 32 * P.warps));
    kern<<<grid, P.warps * 32, P.total, s>>>(root_seed, ids, draw_lo, count, n, t, P, bits, interleaved, sink, gsteps);
    return frr_launched("k_rev_bits");
}

// keys (root_seed, ids[i]) -> control bitsets in the interleaved layout
// [ceil(count/32)][ceil(n/32)][32] (used by frr_dim_mc_ws); steps: caller
// memory for the global step table (frr_steps_len(t) * 16 bytes) or NULL
int frr_rev_words(uint64_t root_seed, const uint64_t* ids, int64_t count, int n, int t, uint32_t* words,
                  void* steps, void* stream) {
    return rev_launch(root_seed, ids, 0, count, n, t, words, 1, nullptr, static_cast<StepC*>(steps), stream);
}

extern "C" int frr_rev_bits(uint64_t root_seed, uint64_t draw_lo, int64_t count, int n, int t, uint32_t* bits,
                            unsigned long long* sink, void* stream) {
    return rev_launch(root_seed, nullptr, draw_lo, count, n, t, bits, 0, sink, nullptr, stream);
}

// ------------------------------------------------- simulation streams
// Polar-method candidates of a keyed simulation stream (reference
// bench.py:101-136): pair p = stream outputs 2p, 2p+1, output i =
// mix64(state + (i+1) C) of key (seed, 2^63 + stream); v = 2 (u >> 11) 2^-53 - 1
// (exact), s = v1 v1 + v2 v2 with numpy's separate roundings.
namespace {
__global__ void k_sim_pairs(uint64_t state, int64_t pair_lo, int64_t npairs, double* __restrict__ v1,
                            double* __restrict__ v2, double* __restrict__ s) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t i = 2 * (uint64_t)(pair_lo + p) + 1;
        const uint64_t u1 = frr_mix64(state + i * FRR_GOLDEN), u2 = frr_mix64(state + (i + 1) * FRR_GOLDEN);
        const double a = __dsub_rn(__dmul_rn(2.0, __dmul_rn((double)(u1 >> 11), 0x1p-53)), 1.0);
        const double b = __dsub_rn(__dmul_rn(2.0, __dmul_rn((double)(u2 >> 11), 0x1p-53)), 1.0);
        v1[p] = a;
        v2[p] = b;
        s[p] = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
    }
}
}  // namespace

extern "C" int frr_sim_pairs(uint64_t root_seed, uint64_t stream_id, int64_t pair_lo, int64_t npairs, double* v1,
                             double* v2, double* s, void* stream) {
    if (npairs <= 0) return FRR_OK;
    const uint64_t state = [&] {
        // derive_state(AssignmentKey(seed, 2^63 + stream)) (keys.py:118-121)
        const uint64_t draw = (1ull << 63) + stream_id;
        uint64_t z = (root_seed ^ (draw * FRR_GOLDEN)) + FRR_GOLDEN;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }();
    const int grid = (int)std::min<int64_t>(frr_cdiv(npairs, 256), (int64_t)frr_num_sms() * 8);
    k_sim_pairs<<<grid, 256, 0, frr_stream(stream)>>>(state, pair_lo, npairs, v1, v2, s);
    return frr_launched("k_sim_pairs");
}

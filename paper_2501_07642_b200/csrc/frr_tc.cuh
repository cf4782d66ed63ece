// frr_tc.cuh -- tcgen05 / TMEM / mbarrier / bulk-copy wrappers (sm_100a inline PTX)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef FRR_WAIT_SLEEP
#define FRR_WAIT_SLEEP 0
#endif
#ifndef FRR_WAIT_HINT_NS
#define FRR_WAIT_HINT_NS 0
#endif

namespace frr_tc {
// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware
// (NANOSLEEP.SYNCS) until the phase completes instead of spinning on issue
// slots the generator warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_u32(b);
    do {
#if FRR_WAIT_HINT_NS > 0
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(FRR_WAIT_HINT_NS)
            : "memory");
#else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
#if FRR_WAIT_SLEEP > 0
        if (!ok) __nanosleep(FRR_WAIT_SLEEP);  // back off: keep issue slots for the generators
#endif
#endif
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// wait for long-idle roles: FRR_LONG_WAIT 0 = spin, 1 = hardware-suspended
// try_wait (time hint), 2 = spin with __nanosleep backoff
#ifndef FRR_LONG_WAIT
#define FRR_LONG_WAIT 2
#endif
#ifndef FRR_LONG_SLEEP_NS
#define FRR_LONG_SLEEP_NS 500
#endif
__device__ __forceinline__ void mbar_wait_long(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t ok = 0;
    for (;;) {
#if FRR_LONG_WAIT == 1
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(200000)
            : "memory");
#else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
#endif
        if (ok) return;
#if FRR_LONG_WAIT == 2
        __nanosleep(FRR_LONG_SLEEP_NS);
#endif
    }
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// A operand from TMEM (lane = row, 4 consecutive int8 K values per 32-bit column)
__device__ __forceinline__ void tc_mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// store 32 consecutive 32-bit columns of this thread's TMEM lane
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, int32_t (&v)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle (canonical layout
// ((8,m),(T,2)):((1T,SBO),(1,LBO)) in 16-byte units).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100)
    return d;         // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// Exact S_j = sum_l acc_l 256^l for 8 consecutive columns: limb l of column
// u sits at TMEM column base + l*stride + u.  pair32: |acc| * 257 < 2^31, so
// two limbs combine in 32 bits and only pairs need 64-bit arithmetic.
__device__ __forceinline__ void tc_limbs8(uint32_t base, int L, int stride, bool pair32, int64_t (&Sj)[8]) {
    int l = L - 1;
    if (pair32 && !(L & 1)) {
#pragma unroll
        for (int u = 0; u < 8; u++) Sj[u] = 0;
    } else {
        int32_t v[8];
        tc_ld8(base + (uint32_t)(l * stride), v);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; u++) Sj[u] = v[u];
        l--;
    }
    if (pair32) {
        for (; l > 0; l -= 2) {
            int32_t vh[8], vl[8];
            tc_ld8(base + (uint32_t)(l * stride), vh);
            tc_ld8(base + (uint32_t)((l - 1) * stride), vl);
            tc_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; u++) Sj[u] = Sj[u] * 65536 + (int64_t)(vh[u] * 256 + vl[u]);
        }
    } else {
        for (; l >= 0; l--) {
            int32_t v[8];
            tc_ld8(base + (uint32_t)(l * stride), v);
            tc_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; u++) Sj[u] = Sj[u] * 256 + v[u];
        }
    }
}

__device__ __forceinline__ void tc_ld4(uint32_t taddr, int32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr)
                 : "memory");
}

// exact S of 4 consecutive columns from L limbs (column l*stride + u), as tc_limbs8
__device__ __forceinline__ void tc_limbs4(uint32_t base, int L, int stride, bool pair32, int64_t (&Sj)[4]) {
    int l = L - 1;
    if (pair32 && !(L & 1)) {
#pragma unroll
        for (int u = 0; u < 4; u++) Sj[u] = 0;
    } else {
        int32_t v[4];
        tc_ld4(base + (uint32_t)(l * stride), v);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; u++) Sj[u] = v[u];
        l--;
    }
    if (pair32) {
        for (; l > 0; l -= 2) {
            int32_t vh[4], vl[4];
            tc_ld4(base + (uint32_t)(l * stride), vh);
            tc_ld4(base + (uint32_t)((l - 1) * stride), vl);
            tc_wait_ld();
#pragma unroll
            for (int u = 0; u < 4; u++) Sj[u] = Sj[u] * 65536 + (int64_t)(vh[u] * 256 + vl[u]);
        }
    } else {
        for (; l >= 0; l--) {
            int32_t v[4];
            tc_ld4(base + (uint32_t)(l * stride), v);
            tc_wait_ld();
#pragma unroll
            for (int u = 0; u < 4; u++) Sj[u] = Sj[u] * 256 + v[u];
        }
    }
}

// The same S_j from 32-bit limb pairs p_i = acc_{2i+1} * 256 + acc_{2i}
// (|acc| <= 128 t, so |p| < 2^31 whenever t < 65280): one TMEM round trip
// per pair, then S = sum_i p_i 2^(16 i) with two int64 multiply-adds for
// L = 6 (the C2 shape) instead of five.
template <int L>
__device__ __forceinline__ void tc_limbs8_pairs(uint32_t base, int stride, int64_t (&Sj)[8]) {
    constexpr int NP = (L + 1) / 2;
#pragma unroll
    for (int i = NP - 1; i >= 0; i--) {
        int32_t vh[8], vl[8];
        const int lh = 2 * i + 1, ll = 2 * i;
        if (lh < L) tc_ld8(base + (uint32_t)(lh * stride), vh);
        tc_ld8(base + (uint32_t)(ll * stride), vl);
        tc_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int32_t pi = lh < L ? vh[u] * 256 + vl[u] : vl[u];
            Sj[u] = i == NP - 1 ? (int64_t)pi : Sj[u] * 65536 + (int64_t)pi;
        }
    }
}

__device__ __forceinline__ void tc_limbs8_fast(uint32_t base, int L, int stride, int64_t (&Sj)[8]) {
    switch (L) {
        case 6: tc_limbs8_pairs<6>(base, stride, Sj); break;
        case 5: tc_limbs8_pairs<5>(base, stride, Sj); break;
        case 7: tc_limbs8_pairs<7>(base, stride, Sj); break;
        default: tc_limbs8(base, L, stride, false, Sj); break;
    }
}

// instruction descriptor: kind::i8, D=s32, A=s8, B=s8, K-major both
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}


}  // namespace frr_tc

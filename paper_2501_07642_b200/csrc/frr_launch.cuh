// frr_launch.cuh -- host-side launch helpers (grid sizing for persistent
// grids: a multiple of the SM count times the resident CTAs per SM).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "frr_common.cuh"

static inline int frr_num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 1;
    }
    return cached[dev];
}

template <class K>
static inline int frr_prepare_kernel(K kernel, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            frr_set_error("cudaFuncSetAttribute(smem=%zu): %s", smem, cudaGetErrorString(e));
            return FRR_E_CUDA;
        }
    }
    return FRR_OK;
}

// persistent grid: SMs x resident blocks, capped by the number of work items
template <class K>
static inline int frr_persistent_grid(K kernel, int threads, size_t smem, int64_t work_items) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    int64_t g = (int64_t)per_sm * frr_num_sms();
    if (work_items < g) g = std::max<int64_t>(1, work_items);
    return (int)g;
}

static inline cudaStream_t frr_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// The universal step table (frr_gen.cu): record i = frr_make_step(max(1,
// 65536 - i), .) for i < 65536 + 128, immutable data of the library image --
// step k of any design n is record 65536 - n + k, so one table serves every
// (n, t) without allocation.  Records k >= t carry real bounds, so its users
// clip those steps (frr_warp_fy<true>).
const StepC* frr_global_steps(int n);

namespace {
// Step table in global memory for the large-t plans: a view into the
// universal table (no allocation).
struct GlobalSteps {
    const StepC* p = nullptr;
    int init(int n, int /*t*/, cudaStream_t /*s*/) {
        p = frr_global_steps(n);
        return p ? FRR_OK : FRR_E_CUDA;
    }
};

}  // namespace

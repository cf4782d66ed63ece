// frr_abi.cu -- error state and device helpers shared by the C-ABI.
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "frr_common.cuh"

static thread_local char g_err[512] = "";

void frr_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int frr_check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        frr_set_error("%s: %s", what, cudaGetErrorString(e));
        return FRR_E_CUDA;
    }
    return FRR_OK;
}

// process-wide count of libfrr kernel launches (diagnostic: bench.py reports
// the launches of its timed region from it)
static std::atomic<unsigned long long> g_launches{0};

int frr_launched(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return frr_check_launch(what);
}

extern "C" unsigned long long frr_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int frr_abi_version(void) { return FRR_ABI_VERSION; }

extern "C" const char* frr_last_error(void) { return g_err; }

extern "C" int frr_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) {
        frr_set_error("frr_device_info: %s", cudaGetErrorString(e));
        return FRR_E_CUDA;
    }
    return FRR_OK;
}

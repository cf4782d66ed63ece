// frr_mma_nt.cu -- N-tiled tensor-core balance check for high-dimensional
// covariates (BASELINE config C3: n=2000, d=1024, L=6 int8 limbs -> N=6144).
//
// Same bit-exact pipeline as frr_mma.cu, but N = L*d no longer fits TMEM, so
// the columns are processed in chunks of 32 covariates (N_chunk = 32 L <= 256)
// through two TMEM buffers: the MMA fills chunk c+1 while the epilogue drains
// chunk c.  The epilogue streams the q_j = delta_j^2 values in j order through
// numpy's pairwise-summation tree (leaves of <= 128 with 8 accumulators, a
// combine stack driven by a plan built once per CTA), so the statistic stays
// bit-identical for any d.
//
// Warp roles (frr_mma_nt_body.cuh): A-operand expansion (bit rows -> int8
// K-chunks written straight into TMEM with tcgen05.st, once per N-chunk pass;
// one LOP3 per register because the B rows are pre-shifted), the Fisher-Yates
// generators, the bulk-copy warp for the int8-limb B chunks, the tcgen05.mma
// issuer, and the epilogue (4 warps, TMEM lane quadrants) on the highest ids.
// TMEM columns: [0, 2 NC) two accumulators, then nst A stages of KC/4 columns.
#include <cuda_runtime.h>

#include "frr_common.cuh"
#include "frr_launch.cuh"
#include "frr_revfy.cuh"
#include "frr_tc.cuh"

// Two instantiations: 256-byte K stages (half the barrier and commit traffic
// per MMA; TMEM then holds two 64-column A stages next to the accumulators,
// so up to 6 limbs) and 128-byte K stages (7 limbs).  Every entry point picks
// the same one for a shape, so the limb layout always matches the kernel.
#define FRR_NT_KC 256
#define FRR_NT_NS nt256
#include "frr_mma_nt_body.cuh"
#undef FRR_NT_KC
#undef FRR_NT_NS
#define FRR_NT_KC 128
#define FRR_NT_NS nt128
#include "frr_mma_nt_body.cuh"
#undef FRR_NT_KC
#undef FRR_NT_NS

bool frr_nt_fits(int n, int d, int L) { return nt256::fits(n, d, L) || nt128::fits(n, d, L); }

size_t frr_nt_limbs_bytes(int n, int d, int L) {
    return nt256::fits(n, d, L) ? nt256::limbs_bytes(n, d, L) : nt128::limbs_bytes(n, d, L);
}

int frr_nt_prepare_limbs(const int64_t* zq, int n, int d, int L, int8_t* limbs, int32_t* overflow, cudaStream_t s) {
    return nt256::fits(n, d, L) ? nt256::prepare_limbs(zq, n, d, L, limbs, overflow, s)
                                : nt128::prepare_limbs(zq, n, d, L, limbs, overflow, s);
}

int frr_mc_stats_nt(const frr_balance_t* bal, uint64_t seed, uint64_t lo, int64_t count, double* stats,
                    void* stream) {
    return nt256::fits(bal->n, bal->d, bal->n_limbs) ? nt256::mc_stats(bal, seed, lo, count, stats, stream)
                                                      : nt128::mc_stats(bal, seed, lo, count, stats, stream);
}

#if FRR_NT_TIMING
extern "C" int frr_debug_nt_waits(unsigned long long* host16) { return nt256::debug_waits(host16); }
#endif

/*
 * frr.h -- C-ABI of libfrr.so, the B200 (sm_100a) rerandomization hot path.
 *
 * This is the drop-in boundary under the fastrr-compatible Python API
 * (paper_2501_07642_b200/).  Every entry point replaces one hot function of
 * the reference fastrr package (arXiv 2501.07642; reference paths below are
 * relative to pkg/src/fastrr/ of the reference).  The reference has no
 * native FFI of its own (it is pure numpy), so these are the symbols a
 * ctypes binding of that path binds; see INTEGRATION.md.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no torch types.
 *   - Every array argument is a DEVICE pointer owned by the caller unless
 *     its name ends in _host.  Every call is asynchronous on `stream`
 *     (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - Return value: FRR_OK (0) or an error code mirroring fastrr.errors
 *     (errors.py:9-88); frr_last_error() gives a thread-local message.
 *   - The library holds no global mutable state besides that message,
 *     per-device one-time kernel attributes and a launch counter; functions
 *     are reentrant.
 *   - n_units <= FRR_MAX_UNITS (uint16 positions in the generators).
 */
#ifndef FRR_H
#define FRR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRR_ABI_VERSION 1
#define FRR_MAX_UNITS 65535

enum frr_status {
    FRR_OK = 0,
    FRR_E_INVALID_DESIGN = 1,   /* errors.py InvalidDesignError    */
    FRR_E_DIMENSION = 2,        /* errors.py DimensionError        */
    FRR_E_ENUM_TOO_LARGE = 3,   /* errors.py EnumerationTooLargeError */
    FRR_E_STORAGE_CAP = 4,      /* errors.py StorageCapError       */
    FRR_E_UNSUPPORTED = 5,      /* shape outside the compiled kernels */
    FRR_E_CUDA = 64             /* CUDA launch / runtime failure    */
};

/* Integer balance machinery on device (balance.py:75-105).
 * zq      : int64 [n*d] row-major, the reference's integer-valued Zq
 * cc      : fp64 [d], fl(colsum_j * fl(1/nc))            (balance.py:97)
 * colsum  : int64 [d], sum_i zq[i][j] (exact)
 * g       : fl(fl(1/t) + fl(1/nc))                        (balance.py:96)
 * cst     : fl(fl((t*nc)/n) * inv_scale_sq)               (balance.py:98)
 * limbs   : int8 [frr_limbs_bytes()] B operand of the tensor-core path,
 *           built by frr_prepare_limbs(); NULL when not prepared.      */
typedef struct frr_balance {
    int32_t n, d, t, n_limbs;
    const int64_t* zq;
    const int64_t* colsum;
    const double* cc;
    const int8_t* limbs;
    double g;
    double cst;
} frr_balance_t;

int frr_abi_version(void);
const char* frr_last_error(void);
/* Process-wide number of libfrr kernel launches so far (all threads,
 * devices and streams); a diagnostic counter, the only other global state. */
unsigned long long frr_launch_count(void);
/* number of SMs / compute capability of the current device */
int frr_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- balance-operand preparation ------------------------------------- */
/* Which tensor-core kernel serves (n, d, n_limbs): 0 none, 1 single-pass
 * (N = n_limbs * d_pad <= 512 TMEM columns), 2 N-tiled.  The N-tiled kernel's
 * B operand is pre-shifted: its limbs encode zq * 2^(3 - (k/4 mod 4)) for K
 * offset k of each 32-unit group, so n_limbs must cover 8 * max|zq|. */
int frr_tc_kernel(int n, int d, int n_limbs);
/* Bytes of the tiled int8-limb B operand for (n, d, n_limbs). */
size_t frr_limbs_bytes(int n, int d, int n_limbs);
/* Split zq into n_limbs balanced int8 digits and tile them in the tcgen05
 * K-major canonical layout.  *overflow_dev (int32, zeroed by the call) is set
 * when some |zq| does not fit n_limbs digits.  Replaces the float64 GEMM
 * operand of balance.py:100-102. */
int frr_prepare_limbs(const int64_t* zq, int n, int d, int n_limbs, int8_t* limbs,
                      int32_t* overflow_dev, void* stream);

/* ---- candidate generation + balance check (pass 1) ------------------- */
/* Monte Carlo draws [draw_lo, draw_lo+count) of root_seed: assignment by
 * keys.py:138-159 (bit-exact), statistic by balance.py:93-105 (bit-exact).
 * Replaces generation.py:185-204 (_pass1_stats). */
int frr_mc_stats(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                 double* stats, void* stream);
/* Exact enumeration ranks [rank_lo, rank_lo+count) in itertools.combinations
 * order.  Replaces generation.py:257-272 + 293-296. */
int frr_exact_stats(const frr_balance_t* bal, uint64_t rank_lo, int64_t count, double* stats,
                    void* stream);
/* Exact-mode statistics for an explicit list of lexicographic ranks (any
 * n, any d; used when frr_exact_stats' n <= 64, d <= 16 kernel does not
 * apply and for regenerated accepted ranks). */
int frr_exact_stats_ids(const frr_balance_t* bal, const uint64_t* ranks, int64_t m, double* stats,
                        void* stream);
/* Split enumeration of exact mode (halves of <= 24 units, d <= 16): the host
 * plan lists the runs of ranks that share their units below na = n/2
 * (blocks, in rank order: base rank, lower-half mask, offset of the block's
 * upper-half subsets in lb, the lexicographic s-subset lists grouped by s).
 * frr_subset_sums builds SA[lower mask] and SB[j] = sum of the rows of the
 * upper subset lb[j] (rows of `width` = frr_exact_split_width(d) int64);
 * the S of a rank is SA[lower] + SB[offset + position in the block].  Same
 * results as frr_exact_stats.  Replaces generation.py:257-272 + 293-296. */
int frr_exact_split_width(int d);
int frr_subset_sums(const frr_balance_t* bal, int na, int width, const int32_t* lb, int64_t* sa, int64_t* sb,
                    void* stream);
int frr_exact_stats_split(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                          const int32_t* blk_a, const int64_t* blk_off, const int64_t* blk_base, int64_t nblk,
                          uint64_t rank_lo, int64_t count, double* stats, void* stream);
/* frr_exact_stats_split on the sampled ranks rank_lo + j * stride, j < count
 * (stats[j]); the select's upper bound for the fused path comes from it. */
int frr_exact_stats_split_strided(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                                  const int32_t* blk_a, const int64_t* blk_off, const int64_t* blk_base,
                                  int64_t nblk, uint64_t rank_lo, int64_t stride, int64_t count, double* stats,
                                  void* stream);
/* frr_exact_stats_split fused with the select's narrowing step: no
 * statistics array; the (rank, statistic) pairs whose statistic's IEEE bits
 * are <= h_bits are appended, in no particular order, to idx/vals (at most
 * cap written) and *n_kept (caller-zeroed, accumulates over launches) counts
 * them all.  The caller sorts by rank and runs the radix select on them
 * (same accepted set as generation.py:159-169 whenever >= k statistics are
 * kept and *n_kept <= cap; otherwise it falls back to the full array). */
int frr_exact_stats_split_filtered(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                                   const int32_t* blk_a, const int64_t* blk_off, const int64_t* blk_base,
                                   int64_t nblk, uint64_t rank_lo, int64_t count, uint64_t h_bits, int64_t cap,
                                   int64_t* idx, double* vals, uint64_t* n_kept, void* stream);
/* frr_exact_stats_split_filtered reordered for reuse (same kept set, tile
 * order): tiles[i] = {sb_row0, j0 << 32 | nrows, g0, interior << 32 | ng} pairs nrows <= 256
 * consecutive upper subsets of one size s (SB rows sb_row0.., positions j0..
 * in their segment) with ng <= 256 blocks of that s (lower masks g_a[g0..],
 * base ranks g_base[g0..]); candidate (g, j) has rank g_base[g] + j and is
 * considered when rank_lo <= rank < rank_hi (interior = 1: all of the tile is).  Host plan:
 * generation._tile_plan. */
int frr_exact_tiled_filtered(const frr_balance_t* bal, const int64_t* sa, const int64_t* sb, int width,
                             const int64_t* tiles, int64_t ntiles, const int32_t* g_a, const int64_t* g_base,
                             uint64_t rank_lo, uint64_t rank_hi, uint64_t h_bits, int64_t cap, int64_t* idx,
                             double* vals, uint64_t* n_kept, void* stream);
/* Path-forcing variants of frr_mc_stats (frr_mc_stats dispatches): the
 * CUDA-core warp path and the tcgen05 tensor-core path (FRR_E_UNSUPPORTED
 * when the shape or limbs do not fit it). */
int frr_mc_stats_small(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                       double* stats, void* stream);
int frr_mc_stats_tc(const frr_balance_t* bal, uint64_t root_seed, uint64_t draw_lo, int64_t count,
                    double* stats, void* stream);
/* Explicit int8 rows [m, n] all treating bal->t units.  Replaces
 * balance.py:234-251 (batch_balance) per treated-count group. */
int frr_rows_stats(const frr_balance_t* bal, const int8_t* rows, int64_t m, double* stats,
                   void* stream);

/* ---- assignment regeneration ------------------------------------------ */
/* keys (root_seed, draws[i]) -> int8 rows [m, n] and/or packed bits
 * [m, ceil(n/32)] (bit e of word e/32 = unit e treated).  Either output may
 * be NULL.  Replaces keys.py:177-208 and generation.py:338-362. */
int frr_regen_mc(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t,
                 int8_t* rows, uint32_t* bits, void* stream);
/* lexicographic ranks -> rows/bits (generation.py:257-272). */
int frr_regen_exact(const uint64_t* ranks, int64_t m, int n, int t, int8_t* rows, uint32_t* bits,
                    void* stream);

/* ---- acceptance: exact k-smallest selection (generation.py:159-169) ---- */
/* Device state of the radix select; the caller allocates it (device) and
 * initialises it with frr_select_init. */
typedef struct frr_select_state {
    uint64_t prefix;   /* threshold bit pattern found so far            */
    uint64_t mask;     /* bits of prefix that are fixed                 */
    int64_t k_rem;     /* rank (1-based) still to find inside the prefix */
    int64_t pad;
} frr_select_state_t;

int frr_select_init(frr_select_state_t* st, int64_t k, void* stream);
/* 8-bit digit histogram (pass 0..7, most significant digit first) of the
 * stats whose bits match st->prefix under st->mask; hist: uint64[256],
 * zeroed by the call. */
int frr_select_hist(const double* stats, int64_t m, const frr_select_state_t* st, int pass,
                    uint64_t* hist, void* stream);
/* pick the digit holding rank st->k_rem from a (possibly all-reduced) hist */
int frr_select_pick(const uint64_t* hist, frr_select_state_t* st, int pass, void* stream);
/* counts[0] = #{stat < T}, counts[1] = #{stat == T}, T = st->prefix */
int frr_select_count(const double* stats, int64_t m, const frr_select_state_t* st,
                     int64_t* counts, void* stream);
/* Order-preserving compaction: accepted = {i: stat<T} plus the first
 * *tie_quota indices with stat==T; writes ascending (index_base+i) to
 * idx_out, the stats to stat_out, the count to *n_out.  workspace:
 * frr_select_workspace_bytes(m) bytes. */
size_t frr_select_workspace_bytes(int64_t m);
int frr_select_compact(const double* stats, int64_t m, int64_t index_base,
                       const frr_select_state_t* st, const int64_t* tie_quota, int64_t* idx_out,
                       double* stat_out, int64_t* n_out, void* workspace, void* stream);
/* Same, writing at most `cap` accepted entries (the first `cap` in index
 * order); *n_out is the full accepted count.  With st->prefix = bits(h) and
 * *tie_quota = INT64_MAX it is the order-preserving filter {i: stat <= h}
 * used to narrow the select to a small candidate set. */
int frr_select_compact_capped(const double* stats, int64_t m, int64_t index_base, const frr_select_state_t* st,
                              const int64_t* tie_quota, int64_t cap, int64_t* idx_out, double* stat_out,
                              int64_t* n_out, void* workspace, void* stream);

/* Stable LSD radix sort of n (key, value) pairs by the low key_bits of the
 * uint64 keys, in place (values: any 8-byte payload).  The fused exact pass
 * keeps (rank, statistic) pairs in arrival order; this puts them in rank
 * order for the select (generation.py:159-169 breaks ties by index).
 * workspace: frr_sort_pairs_workspace_bytes(n) bytes; n < 2^32. */
size_t frr_sort_pairs_workspace_bytes(int64_t n);
int frr_sort_pairs(uint64_t* keys, uint64_t* vals, int64_t n, int key_bits, void* workspace, size_t ws_bytes,
                   void* stream);

/* ---- randomization test (inference.py:82-101, 129-182) ----------------- */
/* Difference in means of y per assignment with numpy's pairwise reduction
 * order (a), the same for y = obs assignment via popcounts (b), and whether
 * the row equals the observed assignment (match, atomically OR-ed; may be
 * NULL).  obs_bits: packed observed assignment; t: treated count of the rows.
 * Sources: keys (frr_dim_mc), ranks (frr_dim_exact), rows (frr_dim_rows). */
int frr_dim_mc(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t,
               const double* y, const uint32_t* obs_bits, double* a, double* b, int32_t* match,
               void* stream);
/* frr_dim_mc in two kernels through a caller workspace: keys -> control
 * bitsets (thread per key) in the workspace, then the statistics with y in
 * shared memory, chunk by chunk (the workspace holds ws_bytes / (4 ceil(n/32))
 * keys, a multiple of 32).  Same results as frr_dim_mc; falls back to it when
 * the workspace holds fewer than 32 keys.  frr_dim_mc_workspace_bytes: the
 * size that serves m keys in chunks of up to 2^18.  frr_dim_mc_chunk_keys:
 * the keys per internal chunk for m keys and that workspace size (whole
 * generator waves) -- the granularity at which a caller streaming keys in
 * can split the call without changing the launch shapes. */
size_t frr_dim_mc_workspace_bytes(int64_t m, int n);
int64_t frr_dim_mc_chunk_keys(int64_t m, int n, int t, size_t ws_bytes);
int frr_dim_mc_ws(uint64_t root_seed, const uint64_t* draws, int64_t m, int n, int t,
                  const double* y, const uint32_t* obs_bits, double* a, double* b, int32_t* match,
                  void* workspace, size_t ws_bytes, void* stream);
int frr_dim_exact(const uint64_t* ranks, int64_t m, int n, int t, const double* y,
                  const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* stream);
int frr_dim_rows(const int8_t* rows, int64_t m, int n, int t, const double* y,
                 const uint32_t* obs_bits, double* a, double* b, int32_t* match, void* stream);
/* counts[j] = #{i : |a_i - fl(taus[j]*b_i)| >= rhs[j]} for j < ntau
 * (inference.py:151 with taus=0, inference.py:177-180 p_at). */
int frr_tau_counts(const double* a, const double* b, int64_t m, const double* taus,
                   const double* rhs, int ntau, uint64_t* counts, void* stream);

/* ---- synthetic inputs (reference bench.py:101-154) --------------------- */
/* Polar-method candidate pairs [pair_lo, pair_lo + npairs) of simulation
 * stream `stream_id` of root_seed: v1, v2 in [-1, 1) and s = v1^2 + v2^2,
 * bit-identical to the reference's numpy arithmetic.  The caller keeps the
 * pairs with 0 < s < 1 and scales them by sqrt(-2 ln s / s) (numpy, so the
 * logarithm is the reference's own). */
int frr_sim_pairs(uint64_t root_seed, uint64_t stream_id, int64_t pair_lo, int64_t npairs, double* v1,
                  double* v2, double* s, void* stream);

/* ---- diagnostics ------------------------------------------------------ */
/* Thread-per-candidate generator (reverse-bitset Fisher-Yates) on its own:
 * draws [draw_lo, draw_lo+count) -> CONTROL bitsets bits [count, ceil(n/32)]
 * (bit e of word e/32 = unit e is control; NULL: not written) and an XOR
 * checksum folded into *sink (NULL: none).  Same assignments as
 * keys.py:138-159; used as the generator microbenchmark and its parity
 * check (the fused pass-1 kernel runs the same device code). */
int frr_rev_bits(uint64_t root_seed, uint64_t draw_lo, int64_t count, int n, int t, uint32_t* bits,
                 unsigned long long* sink, void* stream);

/* D[128 x N] = A[128 x K] . B[N x K]^T (int8 row-major in, int32 out) on one
 * CTA through the same tcgen05 descriptor code as the fused kernel. */
int frr_selftest_mma_i8(const int8_t* A, const int8_t* B, int K, int N, int32_t* D, int variant,
                        void* stream);

/* Integer-issue ceiling of the generator arithmetic: every thread of a
 * persistent grid (SMs x 1024 threads) evaluates `per_thread` splitmix64 draws
 * plus the exact bounded reduction (frr_mod_step) with its constants in
 * registers -- no tables, no shared memory -- and folds them into *sink.
 * Draws per second of this kernel is the peak the Fisher-Yates generators
 * are compared against (bench.py "int_roofline"). */
int frr_microbench_draws(int64_t per_thread, uint64_t* sink, int64_t* total_draws_host, void* stream);
/* Tensor-pipe ceiling for the int8 path: one CTA per SM issuing `iters` x 4
 * back-to-back tcgen05.mma.kind::i8 (M=128, N, K=32) into one TMEM
 * accumulator, A from shared memory (a_tmem bit 0 clear) or TMEM (set);
 * bit 1 set: random operand bytes instead of zeros.
 * *ops_host = 2*M*N*K*instructions (int8 ops) of the launch. */
int frr_microbench_mma_i8(int N, int a_tmem, int64_t iters, int64_t* ops_host, void* stream);
/* The same for CTA pairs (clusters of 2, tcgen05.mma.cta_group::2, M=256,
 * B split by N between the two CTAs); N a multiple of 32. */
int frr_microbench_mma_i8_pair(int N, int a_tmem, int64_t iters, int64_t* ops_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FRR_H */

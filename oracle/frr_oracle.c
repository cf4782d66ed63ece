/*
 * frr_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the fastrr reference algorithm for the
 * rerandomization hot path.  It exists to CHECK the CUDA product path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  Nothing in paper_2501_07642_b200/
 * links or calls it.
 *
 * Parity is pinned by tests/test_oracle_golden.py against fixtures produced
 * by importing the reference itself (oracle/make_golden.py).
 *
 * Each function cites the reference file:line it restates
 * (paths relative to the reference's pkg/src/fastrr/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MULT1 0xBF58476D1CE4E5B9ULL
#define MULT2 0x94D049BB133111EBULL

/* keys.py:99-104 -- splitmix64 finaliser */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * MULT1;
    z = (z ^ (z >> 27)) * MULT2;
    return z ^ (z >> 31);
}

/* keys.py:118-121 -- state = mix64((seed ^ draw*C) + C) */
uint64_t orc_derive_state(uint64_t seed, uint64_t draw) {
    return orc_mix64((seed ^ (draw * GOLDEN)) + GOLDEN);
}

/* keys.py:138-159 -- partial Fisher-Yates with rejection-sampled bounds.
 * perm: caller scratch of n uint32.  row: int8[n] (0/1). */
static void assign_mc(uint64_t seed, uint64_t draw, int n, int t, uint32_t* perm, int8_t* row) {
    uint64_t s = orc_derive_state(seed, draw);
    for (int i = 0; i < n; i++) perm[i] = (uint32_t)i;
    for (int j = 0; j < t; j++) {
        uint64_t bound = (uint64_t)(n - j);
        /* limit = floor(2^64/bound)*bound; u accepted iff u < limit */
        uint64_t rem = (uint64_t)(-bound) % bound; /* 2^64 mod bound */
        uint64_t u;
        for (;;) {
            s += GOLDEN;
            u = orc_mix64(s);
            if (rem == 0 || u < (uint64_t)0 - rem) break;
        }
        uint64_t r = (uint64_t)j + u % bound;
        uint32_t tmp = perm[j];
        perm[j] = perm[r];
        perm[r] = tmp;
    }
    memset(row, 0, (size_t)n);
    for (int j = 0; j < t; j++) row[perm[j]] = 1;
}

void orc_assign_mc(uint64_t seed, uint64_t draw, int n, int t, int8_t* row) {
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    assign_mc(seed, draw, n, t, perm, row);
    free(perm);
}

/* ---------------------------------------------------------------------- */
/* numpy pairwise summation (numpy _core/src/umath/loops_utils.h.src,
 * PW_BLOCKSIZE=128) as used by ndarray.sum(axis=1) on C-contiguous float64
 * rows in balance.py:104 and inference.py:97-98.  The reduction starts from
 * the additive identity +0.0, hence the final "0.0 +". */
static double pw_rec(const double* a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_rec(a, n2) + pw_rec(a + n2, n - n2);
    }
}

double orc_pairwise(const double* a, int64_t n) { return 0.0 + pw_rec(a, n); }

/* ---------------------------------------------------------------------- */
/* balance.py:93-105 -- BalanceKernel.stats on exact integers.
 * zq: int64 [n*d] row-major (the reference's integer-valued float64 Zq),
 * colsum: float64[d] (= zq.sum(axis=0)), inv_scale_sq: 2^(-2 exp). */
typedef struct {
    const int64_t* zq;
    const double* colsum;
    double inv_scale_sq;
    int n, d, t;
} orc_bal_t;

static double stat_from_S(const orc_bal_t* B, const int64_t* S, double* q) {
    int nc = B->n - B->t;
    double g = 1.0 / (double)B->t + 1.0 / (double)nc;
    double inv_nc = 1.0 / (double)nc;
    double cst = ((double)((int64_t)B->t * nc) / (double)B->n) * B->inv_scale_sq;
    for (int j = 0; j < B->d; j++) {
        double cc = B->colsum[j] * inv_nc;
        double delta = (double)S[j] * g;
        delta = delta - cc;
        q[j] = delta * delta;
    }
    return orc_pairwise(q, B->d) * cst;
}

static double stat_row(const orc_bal_t* B, const int8_t* row, int64_t* S, double* q) {
    for (int j = 0; j < B->d; j++) S[j] = 0;
    for (int i = 0; i < B->n; i++) {
        if (row[i]) {
            const int64_t* z = B->zq + (size_t)i * B->d;
            for (int j = 0; j < B->d; j++) S[j] += z[j];
        }
    }
    return stat_from_S(B, S, q);
}

/* ---------------------------------------------------------------------- */
/* threaded drivers */
typedef struct {
    orc_bal_t B;
    int mode; /* 0 = rows, 1 = mc, 2 = exact */
    const int8_t* rows;
    uint64_t seed;
    uint64_t lo;
    int64_t begin, end;
    double* out;
} job_t;

/* generation.py:257-266 order: itertools.combinations == lexicographic
 * combinadic unranking; idx gets the t ascending treated indices */
static uint64_t binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; i++) r = r * (unsigned)(n - k + i) / (unsigned)i;
    return (uint64_t)r;
}

void orc_unrank(uint64_t rank, int n, int t, int32_t* idx) {
    int x = 0;
    for (int i = 0; i < t; i++) {
        for (;;) {
            uint64_t c = binom(n - x - 1, t - i - 1);
            if (rank < c) break;
            rank -= c;
            x++;
        }
        idx[i] = x;
        x++;
    }
}

/* lexicographic successor of an ascending t-subset of [0,n); 0 at end */
static int next_comb(int32_t* c, int n, int t) {
    int i = t - 1;
    while (i >= 0 && c[i] == n - t + i) i--;
    if (i < 0) return 0;
    c[i]++;
    for (int j = i + 1; j < t; j++) c[j] = c[j - 1] + 1;
    return 1;
}

static void* run_job(void* p) {
    job_t* J = (job_t*)p;
    int n = J->B.n, d = J->B.d, t = J->B.t;
    int64_t* S = (int64_t*)malloc(sizeof(int64_t) * (size_t)d);
    double* q = (double*)malloc(sizeof(double) * (size_t)d);
    int8_t* row = (int8_t*)malloc((size_t)n);
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    int32_t* comb = (int32_t*)malloc(sizeof(int32_t) * (size_t)t);
    if (J->mode == 2 && J->begin < J->end) orc_unrank(J->lo + (uint64_t)J->begin, n, t, comb);
    for (int64_t m = J->begin; m < J->end; m++) {
        if (J->mode == 0) {
            J->out[m] = stat_row(&J->B, J->rows + (size_t)m * n, S, q);
        } else if (J->mode == 1) {
            assign_mc(J->seed, J->lo + (uint64_t)m, n, t, perm, row);
            J->out[m] = stat_row(&J->B, row, S, q);
        } else {
            for (int j = 0; j < d; j++) S[j] = 0;
            for (int i = 0; i < t; i++) {
                const int64_t* z = J->B.zq + (size_t)comb[i] * d;
                for (int j = 0; j < d; j++) S[j] += z[j];
            }
            J->out[m] = stat_from_S(&J->B, S, q);
            next_comb(comb, n, t);
        }
    }
    free(S); free(q); free(row); free(perm); free(comb);
    return NULL;
}

static void run_threads(job_t proto, int64_t count, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (count < nthreads) nthreads = count > 0 ? (int)count : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; i++) {
        jobs[i] = proto;
        jobs[i].begin = count * i / nthreads;
        jobs[i].end = count * (i + 1) / nthreads;
        pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(th);
    free(jobs);
}

/* balance.py:234-251 batch_balance for rows sharing treated count t */
void orc_stats_rows(const int64_t* zq, const double* colsum, double inv_scale_sq, int n, int d,
                    int t, const int8_t* rows, int64_t m, double* out, int nthreads) {
    job_t J = {{zq, colsum, inv_scale_sq, n, d, t}, 0, rows, 0, 0, 0, 0, out};
    run_threads(J, m, nthreads);
}

/* generation.py:185-204 _pass1_stats for draws [lo, lo+count) */
void orc_mc_stats(const int64_t* zq, const double* colsum, double inv_scale_sq, int n, int d,
                  int t, uint64_t seed, uint64_t lo, int64_t count, double* out, int nthreads) {
    job_t J = {{zq, colsum, inv_scale_sq, n, d, t}, 1, NULL, seed, lo, 0, 0, out};
    run_threads(J, count, nthreads);
}

/* generation.py:293-296 exact loop for ranks [lo, lo+count) */
void orc_exact_stats(const int64_t* zq, const double* colsum, double inv_scale_sq, int n, int d,
                     int t, uint64_t lo, int64_t count, double* out, int nthreads) {
    job_t J = {{zq, colsum, inv_scale_sq, n, d, t}, 2, NULL, 0, lo, 0, 0, out};
    run_threads(J, count, nthreads);
}

/* keys.py:177-208 batch_assignments */
void orc_batch_assign_mc(uint64_t seed, const uint64_t* draws, int64_t m, int n, int t, int8_t* rows) {
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    for (int64_t i = 0; i < m; i++) assign_mc(seed, draws[i], n, t, perm, rows + (size_t)i * n);
    free(perm);
}

/* generation.py:269-272 rows for lexicographic ranks */
void orc_exact_rows(const uint64_t* ranks, int64_t m, int n, int t, int8_t* rows) {
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)t);
    for (int64_t i = 0; i < m; i++) {
        orc_unrank(ranks[i], n, t, idx);
        int8_t* row = rows + (size_t)i * n;
        memset(row, 0, (size_t)n);
        for (int j = 0; j < t; j++) row[idx[j]] = 1;
    }
    free(idx);
}

/* ---------------------------------------------------------------------- */
/* generation.py:159-169 _select: k smallest by (stat, index) */
typedef struct { double v; int64_t i; } pair_t;
static int cmp_pair(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->v < y->v) return -1;
    if (x->v > y->v) return 1;
    return (x->i > y->i) - (x->i < y->i);
}
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}
void orc_select(const double* stats, int64_t M, int64_t k, int64_t* acc, double* thr) {
    pair_t* p = (pair_t*)malloc(sizeof(pair_t) * (size_t)M);
    for (int64_t i = 0; i < M; i++) { p[i].v = stats[i]; p[i].i = i; }
    qsort(p, (size_t)M, sizeof(pair_t), cmp_pair);
    for (int64_t i = 0; i < k; i++) acc[i] = p[i].i;
    *thr = p[k - 1].v;
    qsort(acc, (size_t)k, sizeof(int64_t), cmp_i64);
    free(p);
}

/* ---------------------------------------------------------------------- */
/* inference.py:82-101 _dim_rows */
void orc_dim_rows(const int8_t* rows, int64_t m, int n, const double* y, int t, double* out) {
    double* bt = (double*)malloc(sizeof(double) * (size_t)n);
    double* bc = (double*)malloc(sizeof(double) * (size_t)n);
    int nc = n - t;
    for (int64_t r = 0; r < m; r++) {
        const int8_t* w = rows + (size_t)r * n;
        for (int i = 0; i < n; i++) {
            double wf = (double)w[i];
            bt[i] = wf * y[i];
            bc[i] = (1.0 - wf) * y[i];
        }
        double st = orc_pairwise(bt, n), sc = orc_pairwise(bc, n);
        out[r] = st * (1.0 / (double)t) - sc * (1.0 / (double)nc);
    }
    free(bt);
    free(bc);
}

/* inference.py:177-180 p_at numerator: count |a - tau*b| >= rhs */
int64_t orc_count_ge(const double* a, const double* b, int64_t m, double tau, double rhs) {
    int64_t c = 0;
    for (int64_t i = 0; i < m; i++) {
        volatile double tb = tau * b[i];
        double v = a[i] - tb;
        if ((v < 0 ? -v : v) >= rhs) c++;
    }
    return c;
}

/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the CPU reference's numba kernels (flatdecode,
 * /root/reference/pkg/src/flatdecode) used as the parity checker for the
 * B200 CUDA path and as the "port" CPU baseline in bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product package never links or calls it.
 *
 * Each function states the reference file:line it restates.  Arithmetic is
 * kept in the reference's precision and order:
 *   - f32 dot products accumulated sequentially in ascending c
 *     (attention.py:180-183), compiled with -ffp-contract=off so no FMA
 *     contraction changes the rounding (numba/LLVM does not contract either);
 *   - f64 num/den accumulators for the async partials (attention.py:176-177);
 *   - f64 ascending-k GEMM oracle rounded once to f32 (matrix.py:70-104).
 * The parallel_for tasks mirror numba's prange task decomposition; every task owns
 * disjoint outputs, so results are independent of the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* Dynamic-schedule parallel-for over [0, n) on a persistent pthread pool
   (numba's prange stand-in: numba's threading layer keeps its workers alive
   between calls, so a per-call thread spawn would overstate the reference's
   cost on small problems; the image's gcc has no usable OpenMP runtime).
   Each task index is executed exactly once; tasks own disjoint outputs. */
static int g_threads = 0;

int oracle_set_threads(int n) {
    if (n > 0) g_threads = n;
    if (g_threads <= 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        g_threads = c > 0 ? (int)c : 1;
    }
    return g_threads;
}

typedef void (*task_fn)(int64_t t, void *ctx);

static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;
static pthread_cond_t g_go = PTHREAD_COND_INITIALIZER, g_done = PTHREAD_COND_INITIALIZER;
static pthread_mutex_t g_call = PTHREAD_MUTEX_INITIALIZER;  /* one parallel_for at a time */
static int g_pool = 0;              /* workers started */
static uint64_t g_gen = 0;          /* job generation */
static int g_want = 0;              /* workers taking part in the current job */
static int g_busy = 0;              /* of those, still running */
static int64_t g_n = 0, g_next = 0;
static task_fn g_fn = NULL;
static void *g_ctx = NULL;

static void run_tasks(void) {
    for (;;) {
        int64_t t = __atomic_fetch_add(&g_next, 1, __ATOMIC_RELAXED);
        if (t >= g_n) break;
        g_fn(t, g_ctx);
    }
}

static void *worker(void *arg) {
    const int id = (int)(intptr_t)arg;
    uint64_t seen = 0;
    pthread_mutex_lock(&g_mu);
    for (;;) {
        while (g_gen == seen) pthread_cond_wait(&g_go, &g_mu);
        seen = g_gen;
        if (id >= g_want) continue;     /* not part of this job */
        pthread_mutex_unlock(&g_mu);
        run_tasks();
        pthread_mutex_lock(&g_mu);
        if (--g_busy == 0) pthread_cond_signal(&g_done);
    }
    return NULL;
}

static void parallel_for(int64_t n, task_fn fn, void *ctx) {
    int T = oracle_set_threads(0);
    if (T > n) T = (int)n;
    if (T <= 1) { for (int64_t t = 0; t < n; ++t) fn(t, ctx); return; }
    pthread_mutex_lock(&g_call);
    pthread_mutex_lock(&g_mu);
    while (g_pool < T - 1) {            /* grow the pool (workers never exit) */
        pthread_t th;
        pthread_create(&th, NULL, worker, (void *)(intptr_t)g_pool);
        pthread_detach(th);
        ++g_pool;
    }
    g_n = n; g_next = 0; g_fn = fn; g_ctx = ctx;
    g_want = T - 1; g_busy = T - 1;
    ++g_gen;
    pthread_cond_broadcast(&g_go);
    pthread_mutex_unlock(&g_mu);
    run_tasks();                        /* the calling thread is worker T-1 */
    pthread_mutex_lock(&g_mu);
    while (g_busy > 0) pthread_cond_wait(&g_done, &g_mu);
    pthread_mutex_unlock(&g_mu);
    pthread_mutex_unlock(&g_call);
}

/* attention.py:167-199 (_async_partials_njit): per (row r, chunk j) task. */
typedef struct {
    const float *Q, *K, *V; int64_t d, p; float scale, phi, a, b;
    const int64_t *bounds; double *num_out, *den_out; int64_t *viol_out;
} async_ctx;

static void async_task(int64_t t, void *vctx) {
    async_ctx *c = (async_ctx *)vctx;
    int64_t d = c->d, p = c->p, r = t / p, j = t % p;
    int64_t lo = c->bounds[j], hi = c->bounds[j + 1];
    const float *Q = c->Q, *K = c->K, *V = c->V;
    double den = 0.0;
    double *num = (double *)calloc((size_t)d, sizeof(double));
    int64_t viol = -1;
    for (int64_t i = lo; i < hi; ++i) {
        float acc = 0.0f;
        for (int64_t k = 0; k < d; ++k) acc += Q[r * d + k] * K[i * d + k];
        float ti = c->scale * acc - c->phi;
        if (ti <= c->a || ti >= c->b) { viol = i; break; }  /* worker terminates its chunk */
        /* numba evaluates np.exp on the f32 scalar and promotes into the
           f64 accumulator (attention.py:187-190) */
        float e = expf(ti);
        den += (double)e;
        /* e * V[i, c] is an f32 product in numba, widened on the add */
        for (int64_t k = 0; k < d; ++k) num[k] += (double)(e * V[i * d + k]);
    }
    double *no = c->num_out + (r * p + j) * d;
    if (viol >= 0) {
        c->den_out[r * p + j] = 0.0;
        for (int64_t k = 0; k < d; ++k) no[k] = 0.0;
    } else {
        c->den_out[r * p + j] = den;
        for (int64_t k = 0; k < d; ++k) no[k] = num[k];
    }
    c->viol_out[r * p + j] = viol;
    free(num);
}

void oracle_async_partials(const float *Q, const float *K, const float *V,
                           int64_t M, int64_t d, float scale, float phi,
                           float a, float b, const int64_t *bounds, int64_t p,
                           double *num_out, double *den_out, int64_t *viol_out) {
    async_ctx c = {Q, K, V, d, p, scale, phi, a, b, bounds, num_out, den_out, viol_out};
    parallel_for(M * p, async_task, &c);
}

/* attention.py:91-120 (_sync_partials_njit): chunk max, exp-sum, weighted acc, all f32. */
typedef struct {
    const float *Q, *K, *V; int64_t d, p; float scale; const int64_t *bounds;
    float *m_out, *l_out, *acc_out;
} sync_ctx;

static void sync_task(int64_t t, void *vctx) {
    sync_ctx *c = (sync_ctx *)vctx;
    int64_t d = c->d, p = c->p, r = t / p, j = t % p;
    int64_t lo = c->bounds[j], hi = c->bounds[j + 1];
    const float *Q = c->Q, *K = c->K, *V = c->V;
    float *x = (float *)malloc(sizeof(float) * (size_t)(hi - lo > 0 ? hi - lo : 1));
    float *accv = (float *)calloc((size_t)d, sizeof(float));
    float m = -INFINITY;
    for (int64_t i = lo; i < hi; ++i) {
        float acc = 0.0f;
        for (int64_t k = 0; k < d; ++k) acc += Q[r * d + k] * K[i * d + k];
        float xi = c->scale * acc;
        x[i - lo] = xi;
        if (xi > m) m = xi;
    }
    float l = 0.0f;
    for (int64_t i = lo; i < hi; ++i) {
        float e = expf(x[i - lo] - m);
        l += e;
        for (int64_t k = 0; k < d; ++k) accv[k] += e * V[i * d + k];
    }
    c->m_out[r * p + j] = m;
    c->l_out[r * p + j] = l;
    for (int64_t k = 0; k < d; ++k) c->acc_out[(r * p + j) * d + k] = accv[k];
    free(x);
    free(accv);
}

void oracle_sync_partials(const float *Q, const float *K, const float *V,
                          int64_t M, int64_t d, float scale,
                          const int64_t *bounds, int64_t p,
                          float *m_out, float *l_out, float *acc_out) {
    sync_ctx c = {Q, K, V, d, p, scale, bounds, m_out, l_out, acc_out};
    parallel_for(M * p, sync_task, &c);
}

/* matrix.py:70-79 + :90-104 (gemm_oracle): f64, ascending k, rounded to f32.
   Parallel over output rows only; each element's k-order is the reference's,
   so the result is bit-identical to the single-threaded loop. */
typedef struct { const float *A, *B; float *C; int64_t n, k; } gemm_ctx;

static void gemm_f64_task(int64_t i, void *vctx) {
    gemm_ctx *c = (gemm_ctx *)vctx;
    int64_t n = c->n, k = c->k;
    double *acc = (double *)calloc((size_t)n, sizeof(double));
    /* per element: acc += a[i,kk]*b[kk,j] for kk ascending (loop interchange
       keeps each element's summation order) */
    for (int64_t kk = 0; kk < k; ++kk) {
        double av = (double)c->A[i * k + kk];
        const float *brow = c->B + kk * n;
        for (int64_t j = 0; j < n; ++j) acc[j] += av * (double)brow[j];
    }
    for (int64_t j = 0; j < n; ++j) c->C[i * n + j] = (float)acc[j];
    free(acc);
}

void oracle_gemm_f64(const float *A, const float *B, float *C,
                     int64_t m, int64_t n, int64_t k) {
    gemm_ctx c = {A, B, C, n, k};
    parallel_for(m, gemm_f64_task, &c);
}

/* dispatch.py:55-70 (_gemv_rows_njit, ImplA): per (row, 256-col panel) task. */
typedef struct { const float *A, *B; float *C; int64_t K, N, panel, panels; } gemv_ctx;

static void gemv_task(int64_t t, void *vctx) {
    gemv_ctx *c = (gemv_ctx *)vctx;
    int64_t r = t / c->panels, j0 = (t % c->panels) * c->panel, N = c->N, K = c->K;
    int64_t w = (c->panel < N - j0) ? c->panel : N - j0;
    float *out = (float *)calloc((size_t)w, sizeof(float));
    for (int64_t kk = 0; kk < K; ++kk) {
        float av = c->A[r * K + kk];
        const float *brow = c->B + kk * N + j0;
        for (int64_t j = 0; j < w; ++j) out[j] += av * brow[j];
    }
    for (int64_t j = 0; j < w; ++j) c->C[r * N + j0 + j] = out[j];
    free(out);
}

void oracle_gemv_rows(const float *A, const float *B, float *C,
                      int64_t M, int64_t K, int64_t N, int64_t panel) {
    gemv_ctx c = {A, B, C, K, N, panel, (N + panel - 1) / panel};
    parallel_for(M * c.panels, gemv_task, &c);
}

/* flatgemm.py:137-188 (_stage/_tile_mac/_flat_gemm_njit, ImplB).  A is the
   already 8-row-padded [Mp,K] matrix; C must be zeroed [Mp,N].  The double
   buffer changes only the staging schedule, never the arithmetic order
   (flatgemm.py:219-221), so one staging sequence serves both. */
typedef struct { const float *A, *B; float *C; int64_t Mp, K, N, bn, bk, k_tiles; } flat_ctx;

static void flat_task(int64_t ti, void *vctx) {
    flat_ctx *c = (flat_ctx *)vctx;
    int64_t Mp = c->Mp, K = c->K, N = c->N, bn = c->bn, bk = c->bk;
    int64_t n0 = ti * bn;
    int64_t w = (bn < N - n0) ? bn : N - n0;
    float *bufA = (float *)malloc(sizeof(float) * 2 * (size_t)(Mp * bk));
    float *bufB = (float *)malloc(sizeof(float) * 2 * (size_t)(bk * bn));
    for (int64_t t = 0; t < c->k_tiles; ++t) {
        int64_t k0 = t * bk;
        int64_t kl = (bk < K - k0) ? bk : K - k0;
        int s = (int)(t % 2);
        float *sa = bufA + (size_t)s * Mp * bk, *sb = bufB + (size_t)s * bk * bn;
        for (int64_t mm = 0; mm < Mp; ++mm)                     /* _stage */
            for (int64_t kk = 0; kk < kl; ++kk) sa[mm * bk + kk] = c->A[mm * K + k0 + kk];
        for (int64_t kk = 0; kk < kl; ++kk)
            for (int64_t j = 0; j < w; ++j) sb[kk * bn + j] = c->B[(k0 + kk) * N + n0 + j];
        for (int64_t rb = 0; rb < Mp; rb += 8) {                 /* _tile_mac (flatgemm.py:148-158) */
            int64_t r1 = (rb + 8 < Mp) ? rb + 8 : Mp;
            for (int64_t kk = 0; kk < kl; ++kk)
                for (int64_t mm = rb; mm < r1; ++mm) {
                    float av = sa[mm * bk + kk];
                    for (int64_t j = 0; j < w; ++j) c->C[mm * N + n0 + j] += av * sb[kk * bn + j];
                }
        }
    }
    free(bufA);
    free(bufB);
}

void oracle_flat_gemm(const float *A, const float *B, float *C,
                      int64_t Mp, int64_t K, int64_t N, int64_t bn, int64_t bk,
                      int double_buffer) {
    (void)double_buffer;
    flat_ctx c = {A, B, C, Mp, K, N, bn, bk, (K + bk - 1) / bk};
    parallel_for((N + bn - 1) / bn, flat_task, &c);
}

/* dispatch.py:95-114 (_blocked_gemm_njit, ImplC); C must be zeroed. */
typedef struct { const float *A, *B; float *C; int64_t M, K, N, bm, bn, bk, n_tiles; } blk_ctx;

static void blocked_task(int64_t t, void *vctx) {
    blk_ctx *c = (blk_ctx *)vctx;
    int64_t M = c->M, K = c->K, N = c->N;
    int64_t m0 = (t / c->n_tiles) * c->bm, n0 = (t % c->n_tiles) * c->bn;
    int64_t m1 = (m0 + c->bm < M) ? m0 + c->bm : M, n1 = (n0 + c->bn < N) ? n0 + c->bn : N;
    int64_t k_tiles = (K + c->bk - 1) / c->bk;
    for (int64_t kt = 0; kt < k_tiles; ++kt) {
        int64_t k0 = kt * c->bk, k1 = (k0 + c->bk < K) ? k0 + c->bk : K;
        for (int64_t kk = k0; kk < k1; ++kk)
            for (int64_t mm = m0; mm < m1; ++mm) {
                float av = c->A[mm * K + kk];
                for (int64_t j = n0; j < n1; ++j) c->C[mm * N + j] += av * c->B[kk * N + j];
            }
    }
}

void oracle_blocked_gemm(const float *A, const float *B, float *C,
                         int64_t M, int64_t K, int64_t N,
                         int64_t bm, int64_t bn, int64_t bk) {
    blk_ctx c = {A, B, C, M, K, N, bm, bn, bk, (N + bn - 1) / bn};
    parallel_for(((M + bm - 1) / bm) * c.n_tiles, blocked_task, &c);
}

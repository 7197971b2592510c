/*
 * fdpp.h — C ABI of the B200-native FlashDecoding++ hot paths
 * (libfdpp.so, built from paper_2311_01282_b200/csrc for sm_100a).
 *
 * Plain pointers and sizes only: every device pointer is caller-owned CUDA
 * device memory, `stream` is a cudaStream_t passed as void*, and every entry
 * point returns an fdpp_status (0 = ok).  Calls are stream-ordered and hold
 * no global state beyond a mutex-guarded TMA descriptor cache, so they are
 * safe from several host threads on distinct streams and capturable into
 * CUDA graphs.  Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/flatdecode/<file>:<line>).
 */
#ifndef FDPP_H_
#define FDPP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
    FDPP_OK = 0,
    FDPP_ERR_SHAPE = 1,       /* -> ShapeError (matrix.py:16)            */
    FDPP_ERR_VALUE = 2,       /* -> ValueError (bad p / scale / mode ...) */
    FDPP_ERR_CUDA = 3,        /* -> RuntimeError (launch / driver error)  */
    FDPP_ERR_UNSUPPORTED = 4, /* -> ValueError (dtype / head dim / align) */
    FDPP_ERR_WORKSPACE = 5    /* -> ValueError (workspace too small)      */
} fdpp_status;

typedef enum { FDPP_F16 = 0, FDPP_BF16 = 1, FDPP_F32 = 2 } fdpp_dtype;

/* Last error message of the calling thread ("" if none). */
const char *fdpp_last_error(void);
/* ABI version (major*100 + minor). */
int fdpp_version(void);
/* Streaming-multiprocessor count of the current device (148 on B200), or -1. */
int fdpp_sm_count(void);
/* Launch every kernel with programmatic dependent launch (default on): a
 * kernel may start its prologue -- and a GEMM its weight stream -- while its
 * predecessor in the stream finishes; each kernel waits (griddepcontrol.wait)
 * before reading produced data or writing memory.  Returns the old setting. */
int fdpp_set_pdl(int enable);

/* ------------------------------------------------- subsystem 1: attention */
#define FDPP_AR_MAX_WORLD 8

typedef enum { FDPP_ATTN_ASYNC = 0, FDPP_ATTN_SYNC = 1 } fdpp_attn_mode;

/* Split-KV decode/prefill attention over a [B, Hkv, L, D] cache.  Query head
 * h uses kv head h / (Hq/Hkv); every query row of one (b, kv-head) sees the
 * same K/V (the reference's "M rows share one K/V", attention.py:77-86).
 * Semantic chunking is the reference's chunk_bounds(L, p) (softmax.py:103-110);
 * each chunk is further divided into `splits_per_chunk` CTAs whose partials
 * are combined in fixed order (bitwise-reproducible reruns). */
typedef struct fdpp_attn_params {
    const void *q;            /* [B, Hq, D] (strides below), dtype           */
    const void *k, *v;        /* [B, Hkv, L, D], key rows contiguous (stride D) */
    void *o;                  /* [B, Hq, D] output, dtype                     */
    int32_t dtype;            /* fdpp_dtype                                  */
    int32_t B, Hq, Hkv, L, D; /* D in {8,16,32,64,128,256} (f32: <= 128)      */
    int64_t q_stride_b, q_stride_h;   /* elements                           */
    int64_t kv_stride_b, kv_stride_h; /* elements (K and V share strides)    */
    int64_t o_stride_b, o_stride_h;   /* elements                           */
    const int32_t *seq_lens;  /* optional [B] device lengths (<= L): batch row b
                                 attends to its first seq_lens[b] keys, read at
                                 run time so one captured graph serves every
                                 decode step; NULL = L for every row           */
    float scale;              /* logit scale (AttentionConfig.scale)         */
    float phi, a, b;          /* ScalingCalibration (softmax.py:175-197)      */
    int32_t p;                /* semantic chunk count (AttentionConfig.p)     */
    int32_t splits_per_chunk; /* CTAs per chunk; 0 = auto (fill 148 SMs)      */
    int32_t mode;             /* fdpp_attn_mode                              */
    uint8_t *row_flags;       /* [B, Hq] out (async): 1 = row recomputed      */
    int32_t *viol_index;      /* optional [B, Hq, p] out: first violating key
                                 of each chunk, or -1 (attention.py:217-238)   */
    int32_t *rows_recomputed; /* optional device counter, incremented         */
    float *chunk_num;         /* optional [B, Hq, p, D] out: async chunk states
                                 num_j (zeroed for a violating chunk)          */
    float *chunk_den;         /* optional [B, Hq, p] out: async chunk den_j    */
    void *workspace;          /* zero-filled before first use; kernels leave
                                 its counters zeroed on exit                   */
    size_t workspace_bytes;
    int32_t kv_prefetch;      /* nonzero: the kernel launched just before this
                                 call wrote no K/V row except the last one each
                                 batch row attends (the decode step's append at
                                 seq_lens[b] - 1), so the other rows may stream
                                 before the programmatic-dependent-launch wait,
                                 under the predecessor's tail; 0 = wait first */
} fdpp_attn_params;

/* Bytes of workspace `fdpp_attn_decode` needs for these params. */
fdpp_status fdpp_attn_workspace_size(const fdpp_attn_params *p, size_t *bytes);

/* The semantic chunk count and CTAs per chunk the call will use (resolves
 * p = 0 / splits_per_chunk = 0 "auto"); AttnStats arithmetic uses this p. */
fdpp_status fdpp_attn_plan(const fdpp_attn_params *p, int32_t *chunks, int32_t *splits_per_chunk);

/* Kernel launches `fdpp_attn_decode` makes for these params: 1 when the async
 * launch joins each row group inside one thread-block cluster and recomputes
 * its flagged rows there (the decode plans: <= 16 single-chunk CTAs per row
 * group, no per-chunk outputs), 2 otherwise (async + recompute launch), 1 for
 * SYNC. */
fdpp_status fdpp_attn_launches(const fdpp_attn_params *p, int32_t *launches);

/* Replaces batch_decode_attention(Q, K, V, cfg, mode) for mode in
 * {"async", "sync"} (attention.py:308-321) and the per-row recompute of
 * _batch_async (attention.py:266-286).  ASYNC: unified-phi partials, fused
 * band check, fixed-order chunk join, then the synchronized recompute of
 * flagged rows: inside the same cluster launch when the row group is one
 * cluster (see fdpp_attn_launches), else a second launch that walks the
 * flagged (batch, kv-head) list.  SYNC: FlashDecoding split-KV with the
 * Eq. (2) max-rescaled join. */
fdpp_status fdpp_attn_decode(const fdpp_attn_params *p, void *stream);

/* ------------------------------------------- subsystem 2: flat GEMM family */
typedef enum { FDPP_IMPL_A = 0, FDPP_IMPL_B = 1, FDPP_IMPL_C = 2 } fdpp_impl;

/* C[M,N] = A[M,K] · W[N,K]^T (+ R[M,N]); W is the reference's B[K,N]
 * prepacked to [N, ldw] (fdpp_prepack_weight).  fp32 accumulation,
 * fixed-order (deterministic) reductions, dtype in {F16, BF16}. */
typedef struct fdpp_gemm_params {
    const void *a; int64_t lda;   /* [M, K] activations                       */
    const void *w; int64_t ldw;   /* [N, K] prepacked weight, ldw % 8 == 0     */
    void *c; int64_t ldc;         /* [M, N] output                            */
    const void *r; int64_t ldr;   /* optional residual added in the epilogue
                                     (may alias c)                             */
    int32_t M, N, K;
    int32_t dtype;                /* FDPP_F16 or FDPP_BF16                     */
    int32_t block_x;              /* token tile on the MMA N axis; 0 = auto
                                     (ImplB 16/32/64, ImplC 128/256)           */
    int32_t ctas;                 /* 0 = auto: ImplB with fewer 128-row tiles
                                     than SMs uses cluster split-K (DSMEM
                                     reduction), otherwise a persistent
                                     stream-K grid of one CTA per SM; > 0 =
                                     stream-K with this many CTAs; < 0 =
                                     cluster split-K with -ctas CTAs/cluster   */
    int32_t stages;               /* smem ring depth; 0 = auto (1 = single
                                     buffer, 2 = the paper's double buffer)     */
    void *workspace;              /* stream-K partials of split tiles + tile
                                     counters (zeroed before first use, left
                                     zeroed)                                    */
    size_t workspace_bytes;
} fdpp_gemm_params;

/* Transpose the reference's row-major B[K,N] into W[N, ldw] (zero pad K..ldw). */
fdpp_status fdpp_prepack_weight(const void *b_kn, void *w_nk, int32_t K, int32_t N,
                                int64_t ldw, int32_t dtype, void *stream);
fdpp_status fdpp_gemm_workspace_size(int32_t impl, const fdpp_gemm_params *p, size_t *bytes);
/* Host-only plan query for ImplB / ImplC (no launch, no device work): CTAs in
 * the grid, cluster split-K size (1 = no cluster; 0 = persistent stream-K) and
 * the token tile on the MMA N axis -- what fdpp_run_kernel would launch. */
fdpp_status fdpp_gemm_plan(int32_t impl, const fdpp_gemm_params *p, int32_t *ctas, int32_t *cluster,
                           int32_t *block_x);

/* ImplA (dispatch.py:73-90): CUDA-core GEMV for M <= 8, weights streamed
 * once for all rows (the reference re-streams B per row). */
fdpp_status fdpp_impl_a_gemv(const fdpp_gemm_params *p, void *stream);
/* ImplB (dispatch.py:140-145 / flatgemm.py:215-242): swap-AB tcgen05 flat
 * GEMM — weight rows on the MMA M axis (128), tokens on the MMA N axis
 * (16..64, TMA zero-fills the padding), persistent stream-K grid over the
 * (N-tile, k-block) space with one continuous TMA/mbarrier ring per SM,
 * double-buffered TMEM accumulators, fixed-order fixup of split tiles. */
fdpp_status fdpp_impl_b_flat(const fdpp_gemm_params *p, void *stream);
/* ImplC (dispatch.py:117-137): conventional big-tile tcgen05 GEMM -- all
 * M <= 256 tokens in one 128- or 256-wide tile (weights on the MMA M axis),
 * so each weight byte is multiplied by every token in one MMA chain rather
 * than once per 64-token flat tile; cluster split-K while its tiles fit one
 * wave, persistent stream-K beyond.  129-256 tokens with N >= ~9.5K run on
 * 2-CTA clusters: one tcgen05.mma.cta_group::2 per 256 weight rows x 256
 * tokens, each CTA staging half the tokens. */
fdpp_status fdpp_impl_c_gemm(const fdpp_gemm_params *p, void *stream);
/* run_kernel(choice, a, b) (dispatch.py:155-156). */
fdpp_status fdpp_run_kernel(int32_t impl, const fdpp_gemm_params *p, void *stream);

/* Fusions around the ImplB flat GEMM for the decode step (the caller of the
 * path): prologue transforms of each landed activation tile, and
 * epilogues that replace the standalone glue kernels. */
typedef struct fdpp_gemm_fuse {
    int32_t x_op;            /* 0 none; 1 A <- RMSNorm(A) * norm_w (row sums of squares
                                given as ssq_in[ssq_tiles][ssq_ld]); 2 A <- silu(A[:, :K]) *
                                A[:, K:2K] (lda >= 2K); 3 folded RMSNorm: the norm weight is
                                pre-multiplied into W's columns and each output row is
                                scaled by its inverse RMS in the epilogue (from ssq_in)    */
    const float *ssq_in;
    int32_t ssq_tiles, ssq_ld;
    const void *norm_w;      /* [K] RMSNorm weight, dtype                              */
    float eps;
    float *ssq_out;          /* optional [N/128][ssq_out_ld]: sum of squares of each
                                stored output row over every 128-column tile            */
    int32_t ssq_out_ld;
    void *q_out;             /* optional RoPE + KV append (QKV projection, head dim 128,
                                N = (Hq + 2 Hkv) * 128): q -> q_out [M, Hq, 128],
                                k/v -> caches [M, Hkv, Lmax, 128] at row pos[m]; C unused */
    void *k_cache, *v_cache;
    const int32_t *pos;
    int32_t Hq, Hkv;
    int64_t cache_stride_b, cache_stride_h;
    float theta;
    void *act_out;           /* optional SiLU*up epilogue (fused gate|up projection whose
                                weight rows are tile-interleaved: each 128-row tile holds 64
                                gate rows then the matching 64 up rows): act_out[m, 64 t + j]
                                = silu(gate) * up, [M, N/2] with leading dim act_ld; C unused */
    int64_t act_ld;
    int32_t ar_rank, ar_world;  /* optional one-shot all-reduce of C over ar_world >= 2
                                tensor-parallel ranks (row-parallel O / down projections):
                                every rank runs this call on its K shard with the same M, N,
                                K; each CTA pushes its fp32 output slice into every peer's
                                receive buffer over peer memory, publishes an epoch flag,
                                waits for the peers' slices and writes C = sum over ranks in
                                rank order + r (residual added once; ssq_out covers the
                                reduced C).  Replaces partial GEMM + ncclAllReduce.         */
    int64_t ar_cap;          /* floats per receive slot (>= M * N), as sized for
                                fdpp_ar_workspace_size                                      */
    void *ar_ws[FDPP_AR_MAX_WORLD]; /* each rank's all-reduce workspace, mapped in this
                                process (its own from fdpp_ar_alloc, peers' from
                                fdpp_ipc_open), zero-filled before first use               */
} fdpp_gemm_fuse;

/* Peer-memory all-reduce workspace: bytes for `world` ranks and `cap` floats per
 * receive slot; allocation (cudaMalloc, zero-filled) and CUDA IPC export/import so
 * each rank can map its peers' workspaces (handles are 64 bytes). */
fdpp_status fdpp_ar_workspace_size(int32_t world, int64_t cap, size_t *bytes);
fdpp_status fdpp_ar_alloc(size_t bytes, void **ptr);
fdpp_status fdpp_ar_free(void *ptr);
fdpp_status fdpp_ipc_get_handle(void *ptr, void *handle64);
fdpp_status fdpp_ipc_open(const void *handle64, void **ptr);
fdpp_status fdpp_ipc_close(void *ptr);
/* 1 in *timed_out if a fused all-reduce on this workspace gave up waiting for a
 * peer (~1 s), else 0; synchronises the device. */
fdpp_status fdpp_ar_check(const void *ws, int32_t *timed_out);

/* ImplB with the fusions above (fused epilogues run in cluster split-K mode). */
fdpp_status fdpp_gemm_fused(const fdpp_gemm_params *p, const fdpp_gemm_fuse *fuse, void *stream);

/* ImplA (GEMV, M <= 2) with the same fusions in GEMV form: x_op 0 or 3 (the inverse RMS
 * comes from the activation rows the CTA streams; ssq_in is ignored), residual,
 * ssq_out as one tile per 8 output columns (ssq_tiles = N / 8 for the consumer),
 * RoPE + KV append for a QKV weight whose head rows are permuted to
 * [4j..4j+3, 64+4j..64+4j+3] per 8-row block, SiLU*up for a gate|up weight permuted
 * to [gate 4c..4c+3, up 4c..4c+3] per 8-row block (act_out [M, N/2]). */
fdpp_status fdpp_gemv_fused(const fdpp_gemm_params *p, const fdpp_gemm_fuse *fuse, void *stream);

/* ------------------------------------------ subsystem 3: heuristic dispatch */
/* dispatch(m, n, k, table) on one entry (dispatch.py:189-197): 0=A,1=B,2=C. */
int32_t fdpp_dispatch_choose(int32_t m, int32_t m1, int32_t m2);
/* _first_sustained (dispatch.py:248-265); returns index or -1 for None. */
int32_t fdpp_first_sustained(const double *costs_new, const double *costs_old,
                             int32_t n, int32_t start);
/* Decision flow of profile_shape (dispatch.py:326-338) on measured medians. */
fdpp_status fdpp_profile_decide(const int32_t *m_sweep, const double *med_a,
                                const double *med_b, const double *med_c, int32_t n,
                                int32_t *m1, int32_t *m2);
/* chunk_bounds(n, p) (softmax.py:103-110) into bounds[p+1]. */
fdpp_status fdpp_chunk_bounds(int64_t n, int32_t p, int64_t *bounds);

/* --------------------------- decode-step glue (caller of the hot path, §8f) */
/* out = x * rsqrt(mean(x^2) + eps) * w, rows of length dim. */
fdpp_status fdpp_rmsnorm(const void *x, const void *w, void *out, int32_t rows, int32_t dim,
                         float eps, int32_t dtype, void *stream);
/* Rotary embedding on the q/k parts of a fused [B, (Hq+2*Hkv)*D] qkv row at
 * position pos[b], writing q to q_out [B, Hq, D] and appending k/v to the
 * caches at row pos[b] ([B, Hkv, Lmax, D], strides in elements). */
fdpp_status fdpp_rope_append(const void *qkv, void *q_out, void *k_cache, void *v_cache,
                             const int32_t *pos, int32_t B, int32_t Hq, int32_t Hkv,
                             int32_t D, int64_t cache_stride_b, int64_t cache_stride_h,
                             float theta, int32_t dtype, void *stream);
/* out[r, j] = silu(gu[r, j]) * gu[r, F + j] for a fused [rows, 2F] gate/up. */
fdpp_status fdpp_silu_mul(const void *gu, void *out, int32_t rows, int32_t F, int32_t dtype,
                          void *stream);
/* out[b, :] = table[ids[b], :]; optional ssq_out[b] = sum_j out[b, j]^2 (the
 * one-tile row sums a fused RMSNorm prologue consumes). */
fdpp_status fdpp_embed(const int32_t *ids, const void *table, void *out, int32_t B, int32_t dim,
                       float *ssq_out, int32_t dtype, void *stream);

/* Per-row sum of squares of x[B, dim] into ssq_out[B] (one tile per row): the
 * folded-RMSNorm input of the next projection after a tensor-parallel
 * all-reduce of the residual stream. */
fdpp_status fdpp_row_ssq(const void *x, float *ssq_out, int32_t B, int32_t dim, int32_t dtype,
                         void *stream);

/* Calibration producer: out[i] = scale * q[b,h] . k[b, h/G, key] at n
 * pseudo-random (b, h, key < seq_lens[b]) drawn from `seed` (uses p's q, k, strides,
 * seq_lens, B, Hq, Hkv, L, D, scale, dtype); idx_out (optional) [n][3] = (b, h, key).
 * The host fits phi and the band with calibrate() (softmax.py:219-266). */
fdpp_status fdpp_sample_logits(const fdpp_attn_params *p, int32_t n, uint64_t seed, float *out,
                               int32_t *idx_out, void *stream);

/* ---------------------------------------------- vector softmax APIs (rows a5/a6) */
/* softmax_reference[_f64] (softmax.py:90-100): exp(x - max) / sum in f64; f64 = 0: f32 x and
 * out (softmax_reference), f64 = 1: f64 x and out (softmax_reference_f64). */
fdpp_status fdpp_softmax_reference(const void *x, int32_t n, void *out, int32_t f64, void *stream);
/* softmax_unified (softmax.py:146-172): e = expf(x - phi), f64 sum.  status[0] = first
 * non-finite e index (INT_MAX if none), *total = the f64 sum; out is written only when
 * the result is representable (the host raises SoftmaxOverflow / DegenerateSumError). */
fdpp_status fdpp_softmax_unified(const float *x, int32_t n, float phi, float *out, int32_t *status,
                                 double *total, void *stream);
/* error path: status[1] = first index where the running f64 sum exceeds FLT_MAX. */
fdpp_status fdpp_softmax_overflow_index(const float *x, int32_t n, float phi, int32_t *status, void *stream);
/* partial_softmax_sync (softmax.py:113-143) over chunk bounds[p+1] (chunk_bounds):
 * per-chunk (max, f32 exp-sum) into ml[2p], merged in chunk order, rescaled output. */
fdpp_status fdpp_partial_softmax_sync(const float *x, const int64_t *bounds, int32_t p, float *out, float *ml,
                                      void *stream);
/* ids[r] = argmax_j logits[r, j] (lowest index on ties). */
fdpp_status fdpp_argmax(const void *logits, int32_t *ids, int32_t rows, int32_t vocab,
                        int32_t dtype, void *stream);
/* pos[b] += 1 and lens[b] = pos[b] + 1 for b < B (advances the decode
 * position and the attended length on device; lens may be NULL). */
fdpp_status fdpp_advance_positions(int32_t *pos, int32_t *lens, int32_t B, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FDPP_H_ */

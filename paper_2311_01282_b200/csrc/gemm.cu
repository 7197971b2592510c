// Subsystem 2 — the flat-GEMM family on sm_100a.
//
//   ImplA  gemv_kernel        CUDA-core GEMV for M <= 8 (dispatch.py:55-90).
//                             Streams every weight byte once for all M rows
//                             (the reference re-reads B per row), 16-B
//                             no-L1-allocate loads, fp32 FMA, fixed-order
//                             warp + CTA reductions.
//   ImplB  gemm_tc<SWAP=1>    flat GEMM (flatgemm.py:215-242): swap-AB tcgen05,
//                             weight rows on the MMA M axis (128), the few
//                             tokens on the MMA N axis (16/32/64; TMA zero-fills
//                             the rows past M, the paper's "pad to 8" without
//                             a padded copy), multi-stage TMA/mbarrier ring (the
//                             paper's double buffer generalised to S stages),
//                             N-split grid plus deterministic split-K.
//   ImplC  gemm_tc<SWAP=0>    conventional GEMM (dispatch.py:95-137): tokens on
//                             the MMA M axis (128-row tiles), weights on N.
//
// All paths: C[M,N] = A[M,K] · W[N,K]^T (+ R), W = prepacked reference B[K,N].
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace fdpp {

// ============================================================ prepack B[K,N] -> W[N,ldw]
template <typename T>
__global__ void prepack_kernel(const T *__restrict__ b, T *__restrict__ w, int K, int N,
                               int64_t ldw) {
    __shared__ T tile[32][33];
    int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int k = k0 + i, n = n0 + threadIdx.x;
        tile[i][threadIdx.x] = (k < K && n < N) ? b[(int64_t)k * N + n] : T(0.0f);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int n = n0 + i, k = k0 + threadIdx.x;
        if (n < N && k < ldw) w[(int64_t)n * ldw + k] = (k < K) ? tile[threadIdx.x][i] : T(0.0f);
    }
}

// ============================================================ ImplA: GEMV (M <= 8)
// CTA = NR weight rows x full K; its 8 warps split K (warp w takes 16-byte
// chunks w*32+lane, stepping 256), so every weight byte is loaded once and the
// activation chunk a lane holds is reused across the NR rows.
constexpr int GEMV_NR = 8;
constexpr int GEMV_WARPS = 8;

template <typename T, int MR>
__global__ void __launch_bounds__(GEMV_WARPS * 32)
gemv_kernel(const T *__restrict__ A, int64_t lda, const T *__restrict__ W, int64_t ldw,
            T *C, int64_t ldc, const T *R, int64_t ldr, int M, int N, int K) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * GEMV_NR;
    const int nchunks = K >> 3;  // 8 elements per 16-B chunk (K % 8 == 0 by contract)
    pdl_wait();
    float acc[GEMV_NR][MR];
#pragma unroll
    for (int r = 0; r < GEMV_NR; ++r)
#pragma unroll
        for (int m = 0; m < MR; ++m) acc[r][m] = 0.f;

    const T *wrow[GEMV_NR];
#pragma unroll
    for (int r = 0; r < GEMV_NR; ++r) wrow[r] = W + (int64_t)min(n0 + r, N - 1) * ldw;

    for (int c = warp * 32 + lane; c < nchunks; c += GEMV_WARPS * 32) {
        int4 wv[GEMV_NR];
#pragma unroll
        for (int r = 0; r < GEMV_NR; ++r) wv[r] = ld_stream_16(wrow[r] + (int64_t)c * 8);
#pragma unroll
        for (int m = 0; m < MR; ++m) {
            const int mm = m < M ? m : M - 1;  // rows past M are computed but never stored
            int4 av = __ldg(reinterpret_cast<const int4 *>(A + (int64_t)mm * lda) + c);
            float2 a0 = Elem<T>::to_f2(av.x), a1 = Elem<T>::to_f2(av.y);
            float2 a2 = Elem<T>::to_f2(av.z), a3 = Elem<T>::to_f2(av.w);
#pragma unroll
            for (int r = 0; r < GEMV_NR; ++r) {
                float2 w0 = Elem<T>::to_f2(wv[r].x), w1 = Elem<T>::to_f2(wv[r].y);
                float2 w2 = Elem<T>::to_f2(wv[r].z), w3 = Elem<T>::to_f2(wv[r].w);
                float s = acc[r][m];
                s = fmaf(a0.x, w0.x, s); s = fmaf(a0.y, w0.y, s);
                s = fmaf(a1.x, w1.x, s); s = fmaf(a1.y, w1.y, s);
                s = fmaf(a2.x, w2.x, s); s = fmaf(a2.y, w2.y, s);
                s = fmaf(a3.x, w3.x, s); s = fmaf(a3.y, w3.y, s);
                acc[r][m] = s;
            }
        }
    }
    pdl_trigger();
    // warp reduction (fixed butterfly order)
#pragma unroll
    for (int r = 0; r < GEMV_NR; ++r)
#pragma unroll
        for (int m = 0; m < MR; ++m) {
            float v = acc[r][m];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[r][m] = v;
        }
    __shared__ float red[GEMV_WARPS][GEMV_NR][MR];
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < GEMV_NR; ++r)
#pragma unroll
            for (int m = 0; m < MR; ++m) red[warp][r][m] = acc[r][m];
    }
    __syncthreads();
    if (threadIdx.x < GEMV_NR * MR) {
        const int r = threadIdx.x / MR, m = threadIdx.x % MR, n = n0 + r;
        if (n < N && m < M) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < GEMV_WARPS; ++w) s += red[w][r][m];  // warp order fixed
            if (R) s += Elem<T>::to_f(R[(int64_t)m * ldr + n]);
            C[(int64_t)m * ldc + n] = Elem<T>::from_f(s);
        }
    }
}

// ============================================================ ImplB / ImplC: tcgen05
// Persistent stream-K kernel.  The (tile, k-block) iteration space -- tiles
// ordered m-tile-major so consecutive tiles share the activation tile -- is
// cut into one contiguous range of `units` k-blocks per CTA (one CTA per SM).
// Inside a CTA:
//   warp 0      TMA producer: streams W and X k-blocks of the whole range
//               through one STAGES-deep smem ring, crossing tile boundaries
//               without draining (the paper's double buffer, generalised);
//   warp 1      TMEM owner + single-thread MMA issuer: one accumulation
//               "segment" per (tile, contiguous k-range), alternating between
//               two TMEM accumulators so the epilogue of segment s overlaps
//               the MMAs of segment s + 1;
//   warps 2..5  epilogue (TMEM lane quadrant = warp % 4): a segment covering
//               the whole K of its tile is written straight to C (+ residual);
//               a tile split across CTAs deposits fp32 partials and the last
//               arriving CTA (atomic ticket) sums them in fixed segment order,
//               so results are bitwise reproducible for a given grid.
constexpr int TC_BK = 64;  // 64 fp16 = 128 B rows: one SWIZZLE_128B atom wide
constexpr int TC_THREADS = 192;

template <int BW, int BX, int STAGES>
struct TcSmem {
    static constexpr uint32_t W_BYTES = BW * TC_BK * 2;
    static constexpr uint32_t X_BYTES = BX * TC_BK * 2;
    static constexpr uint32_t STAGE_BYTES = W_BYTES + X_BYTES;
    static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr uint32_t TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;  // + align slack
};

struct TcWork {
    int n_tiles_n, n_tiles_m, kb_total, units, max_seg;
};

// Store 16 accumulator columns of one TMEM lane (+ residual).  SWAP: lane =
// weight row n, column = token m; otherwise lane = token m, column = n.
template <typename T, int BW, bool SWAP>
__device__ __forceinline__ void epi_store16(const float (&v)[16], T *C, int64_t ldc, const T *R,
                                            int64_t ldr, int M, int N, int n0, int m0, int row,
                                            int c0) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int n = SWAP ? n0 + row : n0 + c0 + j;
        const int m = SWAP ? m0 + c0 + j : m0 + row;
        if (n < N && m < M) {
            float o = v[j];
            if (R) o += Elem<T>::to_f(R[(int64_t)m * ldr + n]);
            C[(int64_t)m * ldc + n] = Elem<T>::from_f(o);
        }
    }
}

template <typename T, int BW, int BX, bool SWAP, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
               T *C, int64_t ldc, const T *R /* may alias C */, int64_t ldr, int M, int N,
               const TcWork wk, float *__restrict__ ws, int *__restrict__ counters) {
    using S = TcSmem<BW, BX, STAGES>;
    constexpr int MMA_M = SWAP ? BW : BX;
    constexpr int MMA_N = SWAP ? BX : BW;
    static_assert(MMA_M == 128, "tcgen05 tile uses the 128-lane MMA");
    static_assert(MMA_N % 16 == 0 && MMA_N >= 16 && MMA_N <= 256, "MMA N");
    constexpr uint32_t ACC_COLS = MMA_N;  // one accumulator
    constexpr uint32_t TMEM_COLS = 2 * ACC_COLS <= 32 ? 32 : 2 * ACC_COLS <= 64 ? 64
                                 : 2 * ACC_COLS <= 128 ? 128 : 2 * ACC_COLS <= 256 ? 256 : 512;
    constexpr uint32_t IDESC = umma_idesc_f16(MMA_M, MMA_N, std::is_same<T, __nv_bfloat16>::value);
    constexpr int TILE_ELEMS = BW * BX;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::BAR_OFF);
    uint64_t *empty = full + STAGES;
    uint64_t *tmem_full = empty + STAGES;      // [2]
    uint64_t *tmem_empty = tmem_full + 2;      // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
    __shared__ int s_is_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KB = wk.kb_total;
    const int total = wk.n_tiles_n * wk.n_tiles_m * KB;
    const int u0 = blockIdx.x * wk.units;
    const int u1 = min(total, u0 + wk.units);
    if (u0 >= u1) return;  // uniform per CTA (host sizes the grid so this never triggers)
#ifdef FDPP_TRACE
    __shared__ unsigned int s_trace_seq;
    if (threadIdx.x == 0) {
        const unsigned long long t_entry = globaltimer_ns();
        s_trace_seq = blockIdx.x < 512 ? atomicAdd(&g_fdpp_launch[blockIdx.x], 1u) : 0u;
        if (blockIdx.x < 512) g_fdpp_trace[s_trace_seq & 7][blockIdx.x][7] = t_entry;
    }
    __syncthreads();
#endif
    if (threadIdx.x == 0) FDPP_TRACE_AT(0);

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmW);
        prefetch_tmap(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer over the whole unit range
            // PDL: the weight stream does not depend on any earlier kernel, so
            // the first ring's worth of W tiles is requested before waiting on
            // the predecessor; activation tiles follow once its output is visible.
            const int pre = min(u1 - u0, STAGES);
            for (int i = 0; i < pre; ++i) {
                const int u = u0 + i, t = u / KB, kb = u % KB;
                mbar_arrive_expect_tx(&full[i], S::STAGE_BYTES);
                tma_load_2d(smem + i * S::STAGE_BYTES, &tmW, &full[i], kb * TC_BK,
                            (t % wk.n_tiles_n) * BW, kEvictFirst);
            }
            FDPP_TRACE_AT(1);
            pdl_wait();
            FDPP_TRACE_AT(2);
            for (int i = 0; i < pre; ++i) {
                const int u = u0 + i, t = u / KB, kb = u % KB;
                tma_load_2d(smem + i * S::STAGE_BYTES + S::W_BYTES, &tmX, &full[i], kb * TC_BK,
                            (t / wk.n_tiles_n) * BX, kEvictLast);
            }
            for (int u = u0 + pre, i = pre; u < u1; ++u, ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                const int t = u / KB, kb = u % KB;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t *sw = smem + s * S::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
                tma_load_2d(sw, &tmW, &full[s], kb * TC_BK, (t % wk.n_tiles_n) * BW, kEvictFirst);
                tma_load_2d(sw + S::W_BYTES, &tmX, &full[s], kb * TC_BK, (t / wk.n_tiles_n) * BX,
                            kEvictLast);
            }
            pdl_trigger();  // every load issued: let the next kernel start its prologue
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            int seg = 0;
            for (int u = u0, i = 0; u < u1; ++u, ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                const int kb = u % KB;
                const bool first = (u == u0) || kb == 0;
                const bool last = (u == u1 - 1) || kb == KB - 1;
                const int buf = seg & 1;
                if (first) {
                    mbar_wait(&tmem_empty[buf], ((seg >> 1) & 1) ^ 1);
                    tc_fence_after();
                }
                mbar_wait(&full[s], ph);
                tc_fence_after();
                if (i == 0) FDPP_TRACE_AT(3);
                if (u == u1 - 1) FDPP_TRACE_AT(4);
                uint8_t *sw = smem + s * S::STAGE_BYTES;
                uint8_t *sx = sw + S::W_BYTES;
                const uint64_t da = umma_desc_sw128(SWAP ? sw : sx);
                const uint64_t db = umma_desc_sw128(SWAP ? sx : sw);
                const uint32_t dt = tmem_base + buf * ACC_COLS;
#pragma unroll
                for (int k = 0; k < TC_BK / 16; ++k)  // UMMA_K = 16: +32 B inside the swizzle atom
                    umma_f16(dt, da + 2 * k, db + 2 * k, IDESC, (first && k == 0) ? 0u : 1u);
                umma_commit(&empty[s]);  // frees the smem slot when these MMAs finish
                if (last) {
                    umma_commit(&tmem_full[buf]);
                    ++seg;
                }
            }
        }
    } else {  // ---------------- epilogue warps 2..5
        pdl_wait();  // residual / C / workspace belong to the stream's earlier kernels
        const int quad = warp & 3;
        const int row = quad * 32 + lane;  // TMEM lane = accumulator row
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        int seg = 0;
        for (int u = u0; u < u1; ++seg) {
            const int t = u / KB, kb_start = u % KB;
            const int kb_end = min(KB, kb_start + (u1 - u));
            u += kb_end - kb_start;
            const int n0 = (t % wk.n_tiles_n) * BW, m0 = (t / wk.n_tiles_n) * BX;
            const int buf = seg & 1;
            const bool whole = kb_start == 0 && kb_end == KB;
            int c_lo = 0, nseg = 1, segi = 0;
            float *slot = nullptr;
            if (!whole) {
                c_lo = (t * KB) / wk.units;
                nseg = ((t + 1) * KB - 1) / wk.units - c_lo + 1;
                segi = blockIdx.x - c_lo;
                slot = ws + ((int64_t)t * wk.max_seg + segi) * TILE_ELEMS;
            }
            mbar_wait(&tmem_full[buf], (seg >> 1) & 1);
            tc_fence_after();
            if (warp == 2 && lane == 0) FDPP_TRACE_AT(5);
            // 16 accumulator columns at a time: compact code, few live registers
#pragma unroll 1
            for (int c0 = 0; c0 < MMA_N; c0 += 16) {
                float v[16];
                tmem_ld16(tmem_base + buf * ACC_COLS + lane_off + c0, v);
                if (whole) {
                    epi_store16<T, BW, SWAP>(v, C, ldc, R, ldr, M, N, n0, m0, row, c0);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)   // partial tile layout [BX m][BW n]
                        slot[SWAP ? (c0 + j) * BW + row : row * BW + c0 + j] = v[j];
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[buf]);  // accumulator may be reused
            if (whole) continue;
            // ---- split tile: last arriving CTA reduces all segments in fixed order
            __threadfence();
            named_bar_sync(1, 128);
            if (warp == 2 && lane == 0) {
                const int ticket = atomicAdd(&counters[t], 1);
                s_is_last = (ticket == nseg - 1);
                if (s_is_last) counters[t] = 0;  // leave the workspace zeroed
            }
            named_bar_sync(1, 128);
            const bool is_last = s_is_last;
            named_bar_sync(1, 128);  // s_is_last is rewritten by the next split tile
            if (!is_last) continue;
            __threadfence();
            const float *base = ws + (int64_t)t * wk.max_seg * TILE_ELEMS;
#pragma unroll 1
            for (int c0 = 0; c0 < MMA_N; c0 += 16) {
                float acc[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = 0.f;
                // segments in groups of 4: all loads of a group are in flight
                // together (one L2 round trip), then added in segment order
#pragma unroll 1
                for (int sg0 = 0; sg0 < nseg; sg0 += 4) {
                    float val[4][16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float *src = base + (int64_t)(sg0 + q) * TILE_ELEMS;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            val[q][j] = (sg0 + q < nseg)
                                ? ld_cg_f32(src + (SWAP ? (c0 + j) * BW + row : row * BW + c0 + j))
                                : 0.f;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[j] += val[q][j];
                }
                epi_store16<T, BW, SWAP>(acc, C, ldc, R, ldr, M, N, n0, m0, row, c0);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) FDPP_TRACE_AT(6);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ============================================================ ImplB: cluster split-K
// For few output tiles (small N, e.g. [4096, K]): the K range of each 128-row
// weight tile is split across the CS CTAs of one thread-block cluster.  Each
// CTA streams its K slice through the TMA ring into its own TMEM accumulator;
// after a cluster barrier the fp32 slices are reduced over DSMEM -- CTA r sums
// column slice r across ranks 0..CS-1 in fixed order and writes C (+residual)
// -- so there are no global partials, fences or tickets, and the result is
// bitwise reproducible.  All CS * n_tiles CTAs are co-resident (one wave).
struct TcCluster {
    int n_tiles_n, kb_total, kb_per, cs;
};

template <int BX, int STAGES>
struct ClSmem {
    using S = TcSmem<128, BX, STAGES>;
    static constexpr uint32_t RING = STAGES * S::STAGE_BYTES;
    static constexpr uint32_t PART = BX * 128 * 4;  // fp32 partial [MMA_N][128]
    static constexpr uint32_t BAR_OFF = RING > PART ? RING : PART;
    static constexpr uint32_t TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
};

template <typename T, int BX, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    T *C, int64_t ldc, const T *R /* may alias C */, int64_t ldr, int M, int N,
                    const TcCluster ck) {
    constexpr int BW = 128;
    using S = TcSmem<BW, BX, STAGES>;
    constexpr int MMA_N = BX;
    constexpr uint32_t TMEM_COLS = MMA_N <= 32 ? 32 : MMA_N <= 64 ? 64 : 128;
    constexpr uint32_t IDESC = umma_idesc_f16(128, MMA_N, std::is_same<T, __nv_bfloat16>::value);
    using CS = ClSmem<BX, STAGES>;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + CS::BAR_OFF);
    uint64_t *empty = full + STAGES;
    uint64_t *tmem_full = empty + STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 2);
    float *part = reinterpret_cast<float *>(smem);  // [MMA_N][128] after the ring drains

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int tn = blockIdx.x / ck.cs, tm = blockIdx.y;
    const int n0 = tn * BW, m0 = tm * BX;
    const int kb0 = (int)rank * ck.kb_per;
    const int nkb = min(ck.kb_total, kb0 + ck.kb_per) - kb0;  // >= 1 (host guarantees)

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmW);
        prefetch_tmap(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (weights first, PDL)
            const int pre = min(nkb, STAGES);
            for (int i = 0; i < pre; ++i) {
                mbar_arrive_expect_tx(&full[i], S::STAGE_BYTES);
                tma_load_2d(smem + i * S::STAGE_BYTES, &tmW, &full[i], (kb0 + i) * TC_BK, n0, kEvictFirst);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i)
                tma_load_2d(smem + i * S::STAGE_BYTES + S::W_BYTES, &tmX, &full[i], (kb0 + i) * TC_BK,
                            m0, kEvictLast);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
                uint8_t *sw = smem + s * S::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
                tma_load_2d(sw, &tmW, &full[s], (kb0 + i) * TC_BK, n0, kEvictFirst);
                tma_load_2d(sw + S::W_BYTES, &tmX, &full[s], (kb0 + i) * TC_BK, m0, kEvictLast);
            }
            pdl_trigger();
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&full[s], (i / STAGES) & 1);
                tc_fence_after();
                uint8_t *sw = smem + s * S::STAGE_BYTES;
                const uint64_t da = umma_desc_sw128(sw);
                const uint64_t db = umma_desc_sw128(sw + S::W_BYTES);
#pragma unroll
                for (int k = 0; k < TC_BK / 16; ++k)
                    umma_f16(tmem_base, da + 2 * k, db + 2 * k, IDESC, (i == 0 && k == 0) ? 0u : 1u);
                umma_commit(&empty[s]);
            }
            umma_commit(tmem_full);
        }
        __syncwarp();
    } else {  // ---------------- epilogue warps: TMEM -> own smem partial [col][row]
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < MMA_N; c0 += 16) {
            float v[16];
            tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) part[(c0 + j) * 128 + row] = v[j];
        }
    }
    tc_fence_before();
    cluster_sync_all();  // every rank's partial is in its smem
    if (warp >= 2) {
        pdl_wait();  // residual / C belong to earlier kernels
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        const int n = n0 + row;
        const int per = (MMA_N + ck.cs - 1) / ck.cs;
        const int c_beg = (int)rank * per, c_end = min(MMA_N, c_beg + per);
        uint32_t peer[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) peer[q] = q < ck.cs ? dsmem_map(part, q) : 0u;
        for (int c = c_beg; c < c_end; ++c) {
            const int m = m0 + c;
            float vals[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                vals[q] = q < ck.cs ? dsmem_ld_f32(peer[q] + (uint32_t)((c * 128 + row) * 4)) : 0.f;
            float o = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) o += vals[q];  // rank order
            if (n < N && m < M) {
                if (R) o += Elem<T>::to_f(R[(int64_t)m * ldr + n]);
                C[(int64_t)m * ldc + n] = Elem<T>::from_f(o);
            }
        }
    }
    cluster_sync_all();  // peers may still be reading this CTA's partial
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ============================================================ host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

struct MapKey {
    const void *ptr;
    int64_t rows, cols, ld;
    int box_rows, dtype;
    bool operator==(const MapKey &o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld &&
               box_rows == o.box_rows && dtype == o.dtype;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey &k) const {
        size_t h = std::hash<const void *>()(k.ptr);
        h ^= std::hash<int64_t>()(k.rows * 1315423911ll + k.cols) + 0x9e3779b9 + (h << 6);
        h ^= std::hash<int64_t>()(k.ld * 31 + k.box_rows * 7 + k.dtype) + (h >> 2);
        return h;
    }
};

// 2-D K-major tile map over a row-major [rows, cols] matrix (leading dim ld),
// box = [box_rows x 64] elements, SWIZZLE_128B, OOB rows/cols zero-filled.
static fdpp_status make_kmajor_map(CUtensorMap *out, const void *ptr, int64_t rows, int64_t cols,
                                   int64_t ld, int box_rows, int dtype) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    MapKey key{ptr, rows, cols, ld, box_rows, dtype};
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *out = it->second;
            return FDPP_OK;
        }
    }
    EncodeTiledFn enc = get_encode_fn();
    FDPP_REQUIRE(enc != nullptr, FDPP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    FDPP_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (ld * 2) % 16 == 0,
                 FDPP_ERR_UNSUPPORTED, "TMA operand must be 16-byte aligned with ld %% 8 == 0");
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUtensorMap m;
    CUresult r = enc(&m, dtype == FDPP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                     2, const_cast<void *>(ptr), gdim, gstride, box, estride,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    FDPP_REQUIRE(r == CUDA_SUCCESS, FDPP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    {
        std::lock_guard<std::mutex> g(mu);
        if (cache.size() > 4096) cache.clear();
        cache.emplace(key, m);
    }
    *out = m;
    return FDPP_OK;
}

// ============================================================ host: planning
struct TcPlan {
    int bw, bx, stages, grid;
    TcWork wk;
    bool cluster;    // ImplB cluster split-K (few tiles) instead of stream-K
    TcCluster ck;
};

static int pick_block_x(int M, bool swap) {
    if (!swap) return 128;
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    return 64;
}

static fdpp_status plan_tc(const fdpp_gemm_params *p, bool swap, TcPlan *pl) {
    const int kb_total = ceil_div(p->K, TC_BK);
    pl->bx = p->block_x > 0 ? p->block_x : pick_block_x(p->M, swap);
    if (swap) {
        FDPP_REQUIRE(pl->bx == 16 || pl->bx == 32 || pl->bx == 64, FDPP_ERR_VALUE,
                     "ImplB block_x must be 16, 32 or 64");
    } else {
        FDPP_REQUIRE(pl->bx == 128, FDPP_ERR_VALUE, "ImplC block_x must be 128");
    }
    pl->bw = 128;
    TcWork &w = pl->wk;
    w.n_tiles_n = ceil_div(p->N, pl->bw);
    w.n_tiles_m = ceil_div(p->M, pl->bx);
    w.kb_total = kb_total;
    const int64_t total = (int64_t)w.n_tiles_n * w.n_tiles_m * kb_total;
    FDPP_REQUIRE(total < (1ll << 31), FDPP_ERR_SHAPE, "GEMM too large");
    const int sms = sm_count() > 0 ? sm_count() : 148;
    const int tiles = w.n_tiles_n * w.n_tiles_m;
    // Auto policy for ImplB (measured in-graph on B200 across the Llama shapes,
    // tools/mode_sweep.py): few tiles -> cluster split-K, 8 CTAs per tile for
    // <= 40 tiles (e.g. N = 4096), 2 per tile up to ~0.9 SMs of tiles (N = 12288);
    // many tiles -> stream-K with two CTAs per SM.  ctas < 0 forces cs = -ctas.
    pl->cluster = swap && ((p->ctas == 0 && tiles <= (sms * 9) / 10) || p->ctas < 0);
    if (pl->cluster) {
        int cs = p->ctas < 0 ? -p->ctas : (tiles <= 40 ? 8 : 2);
        cs = cs < 1 ? 1 : (cs > 8 ? 8 : cs);
        if (cs > kb_total) cs = kb_total;
        TcCluster &c = pl->ck;
        c.n_tiles_n = w.n_tiles_n;
        c.kb_total = kb_total;
        c.kb_per = (kb_total + cs - 1) / cs;
        c.cs = (kb_total + c.kb_per - 1) / c.kb_per;  // no empty rank
        pl->grid = w.n_tiles_n * c.cs;
        pl->stages = p->stages > 0 ? p->stages : 0;
        return FDPP_OK;
    }
    // persistent stream-K grid: one CTA per SM (or the `ctas` override),
    // contiguous equal unit ranges -- perfect balance up to one k-block
    int ctas = p->ctas > 0 ? p->ctas : (swap ? 2 * sms : sms);
    if (ctas > total) ctas = (int)total;
    w.units = (int)((total + ctas - 1) / ctas);
    pl->grid = (int)((total + w.units - 1) / w.units);
    w.max_seg = (kb_total + w.units - 1) / w.units + 1;
    FDPP_REQUIRE(w.n_tiles_n * w.n_tiles_m <= kWsCounters, FDPP_ERR_SHAPE,
                 "too many output tiles (%d)", w.n_tiles_n * w.n_tiles_m);
    pl->stages = p->stages > 0 ? p->stages : 0;
    return FDPP_OK;
}

static bool has_split_tiles(const TcPlan &pl) {
    return !pl.cluster && (pl.wk.units % pl.wk.kb_total != 0 || pl.wk.units < pl.wk.kb_total);
}

static size_t tc_workspace(const TcPlan &pl, const fdpp_gemm_params *p) {
    (void)p;
    if (!has_split_tiles(pl)) return 0;
    const size_t part = (size_t)pl.wk.n_tiles_n * pl.wk.n_tiles_m * pl.wk.max_seg * pl.bw * pl.bx *
                        sizeof(float);
    return kWsCounterBytes + part;
}

template <typename T, int BX, int STAGES>
static fdpp_status launch_cluster(const fdpp_gemm_params *p, const TcPlan &pl, const CUtensorMap &mw,
                                  const CUtensorMap &mx, cudaStream_t st) {
    using S = ClSmem<BX, STAGES>;
    auto kern = gemm_cluster_kernel<T, BX, STAGES>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)S::TOTAL);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(gemm_cluster)");
        attr_set = true;
    }
    cudaError_t e = launch_kernel_cluster(kern, dim3(pl.grid, pl.wk.n_tiles_m), dim3(TC_THREADS),
                                          S::TOTAL, st, pl.ck.cs, mw, mx, static_cast<T *>(p->c),
                                          p->ldc, static_cast<const T *>(p->r), p->ldr, p->M, p->N,
                                          pl.ck);
    if (e != cudaSuccess) return cuda_status(e, "gemm_cluster_kernel launch");
    return FDPP_OK;
}

template <typename T, int BW, int BX, bool SWAP, int STAGES>
static fdpp_status launch_tc(const fdpp_gemm_params *p, const TcPlan &pl, const CUtensorMap &mw,
                             const CUtensorMap &mx, cudaStream_t st) {
    if constexpr (SWAP && BW == 128) {
        if (pl.cluster) return launch_cluster<T, BX, STAGES>(p, pl, mw, mx, st);
    }
    using S = TcSmem<BW, BX, STAGES>;
    auto kern = gemm_tc_kernel<T, BW, BX, SWAP, STAGES>;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)S::TOTAL);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(gemm_tc)");
        attr_set = true;
    }
    int *counters = nullptr;
    float *ws = nullptr;
    if (has_split_tiles(pl)) {
        counters = static_cast<int *>(p->workspace);
        ws = reinterpret_cast<float *>(static_cast<char *>(p->workspace) + kWsCounterBytes);
    }
    cudaError_t e = launch_kernel(kern, dim3(pl.grid), dim3(TC_THREADS), S::TOTAL, st, mw, mx,
                                  static_cast<T *>(p->c), p->ldc, static_cast<const T *>(p->r),
                                  p->ldr, p->M, p->N, pl.wk, ws, counters);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc_kernel launch");
    return FDPP_OK;
}

// stage counts: 1 (single buffer), 2 (double buffer) and the deep default
template <typename T, int BX, bool SWAP>
static fdpp_status dispatch_stages(const fdpp_gemm_params *p, const TcPlan &pl,
                                   const CUtensorMap &mw, const CUtensorMap &mx, cudaStream_t st) {
    constexpr int BW = 128;
    // default ring: ~100 KB of stages (>= 4x the ~20 KB/SM Little's-law need
    // at 6.5 TB/s), small enough that the next kernel's CTA fits beside it on
    // the SM while this one drains (PDL overlap)
    constexpr int DEEP = (100 * 1024) / ((BW + BX) * TC_BK * 2) < 4
                             ? 4
                             : (100 * 1024) / ((BW + BX) * TC_BK * 2);
    switch (pl.stages) {
        case 1: return launch_tc<T, BW, BX, SWAP, 1>(p, pl, mw, mx, st);
        case 2: return launch_tc<T, BW, BX, SWAP, 2>(p, pl, mw, mx, st);
        case 4: return launch_tc<T, BW, BX, SWAP, 4>(p, pl, mw, mx, st);
        default: return launch_tc<T, BW, BX, SWAP, DEEP>(p, pl, mw, mx, st);
    }
}

static fdpp_status check_gemm(const fdpp_gemm_params *p) {
    FDPP_REQUIRE(p && p->a && p->w && p->c, FDPP_ERR_VALUE, "null GEMM operand");
    FDPP_REQUIRE(p->M >= 1 && p->N >= 1 && p->K >= 1, FDPP_ERR_SHAPE,
                 "GEMM dims must be >= 1, got (%d, %d, %d)", p->M, p->N, p->K);
    FDPP_REQUIRE(p->dtype == FDPP_F16 || p->dtype == FDPP_BF16, FDPP_ERR_UNSUPPORTED,
                 "GEMM dtype must be f16 or bf16");
    FDPP_REQUIRE(p->K % 8 == 0 && p->lda % 8 == 0 && p->ldw % 8 == 0 && p->ldw >= p->K &&
                     p->lda >= p->K && p->ldc >= p->N,
                 FDPP_ERR_UNSUPPORTED, "K, lda, ldw must be multiples of 8 (pad K with zeros)");
    return FDPP_OK;
}

static fdpp_status run_tc(const fdpp_gemm_params *p, bool swap, cudaStream_t st) {
    fdpp_status s = check_gemm(p);
    if (s != FDPP_OK) return s;
    TcPlan pl;
    if ((s = plan_tc(p, swap, &pl)) != FDPP_OK) return s;
    FDPP_REQUIRE(tc_workspace(pl, p) <= p->workspace_bytes, FDPP_ERR_WORKSPACE,
                 "GEMM workspace too small: need %zu bytes", tc_workspace(pl, p));
    CUtensorMap mw, mx;
    if ((s = make_kmajor_map(&mw, p->w, p->N, p->K, p->ldw, pl.bw, p->dtype)) != FDPP_OK) return s;
    if ((s = make_kmajor_map(&mx, p->a, p->M, p->K, p->lda, pl.bx, p->dtype)) != FDPP_OK) return s;
    const bool bf = p->dtype == FDPP_BF16;
    if (swap) {
        switch (pl.bx) {
            case 16: return bf ? dispatch_stages<__nv_bfloat16, 16, true>(p, pl, mw, mx, st)
                               : dispatch_stages<__half, 16, true>(p, pl, mw, mx, st);
            case 32: return bf ? dispatch_stages<__nv_bfloat16, 32, true>(p, pl, mw, mx, st)
                               : dispatch_stages<__half, 32, true>(p, pl, mw, mx, st);
            default: return bf ? dispatch_stages<__nv_bfloat16, 64, true>(p, pl, mw, mx, st)
                               : dispatch_stages<__half, 64, true>(p, pl, mw, mx, st);
        }
    }
    return bf ? dispatch_stages<__nv_bfloat16, 128, false>(p, pl, mw, mx, st)
              : dispatch_stages<__half, 128, false>(p, pl, mw, mx, st);
}

template <typename T>
static fdpp_status launch_gemv(const fdpp_gemm_params *p, cudaStream_t st) {
    dim3 grid(ceil_div(p->N, GEMV_NR));
    const T *A = static_cast<const T *>(p->a);
    const T *W = static_cast<const T *>(p->w);
    T *C = static_cast<T *>(p->c);
    const T *R = static_cast<const T *>(p->r);
    cudaError_t err = cudaSuccess;
#define FDPP_GEMV_CASE(MR)                                                                   \
    case MR:                                                                                 \
        err = launch_kernel(gemv_kernel<T, MR>, grid, dim3(GEMV_WARPS * 32), 0, st, A, p->lda, \
                            W, p->ldw, C, p->ldc, R, p->ldr, p->M, p->N, p->K);              \
        break;
    switch (p->M) {
        FDPP_GEMV_CASE(1)
        FDPP_GEMV_CASE(2)
        FDPP_GEMV_CASE(3)
        FDPP_GEMV_CASE(4)
        FDPP_GEMV_CASE(5)
        FDPP_GEMV_CASE(6)
        FDPP_GEMV_CASE(7)
        FDPP_GEMV_CASE(8)
        default: break;
    }
#undef FDPP_GEMV_CASE
    if (err != cudaSuccess) return cuda_status(err, "gemv_kernel launch");
    return FDPP_OK;
}

}  // namespace fdpp

using namespace fdpp;

#ifdef FDPP_TRACE
extern "C" int fdpp_trace_read(unsigned long long *host, int n) {
    (void)n;
    return (int)cudaMemcpyFromSymbol(host, fdpp::g_fdpp_trace, sizeof(fdpp::g_fdpp_trace));
}
extern "C" int fdpp_trace_reset(void) {
    unsigned int z[512] = {0};
    return (int)cudaMemcpyToSymbol(fdpp::g_fdpp_launch, z, sizeof(z));
}
#endif

extern "C" fdpp_status fdpp_prepack_weight(const void *b_kn, void *w_nk, int32_t K, int32_t N,
                                           int64_t ldw, int32_t dtype, void *stream) {
    FDPP_REQUIRE(b_kn && w_nk, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(K >= 1 && N >= 1 && ldw >= K, FDPP_ERR_SHAPE, "bad prepack dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dim3 grid(ceil_div(N, 32), ceil_div(ldw, 32)), block(32, 8);
    switch (dtype) {
        case FDPP_F16:
            prepack_kernel<__half><<<grid, block, 0, st>>>(static_cast<const __half *>(b_kn),
                                                           static_cast<__half *>(w_nk), K, N, ldw);
            break;
        case FDPP_BF16:
            prepack_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(
                static_cast<const __nv_bfloat16 *>(b_kn), static_cast<__nv_bfloat16 *>(w_nk), K, N,
                ldw);
            break;
        default: FDPP_REQUIRE(false, FDPP_ERR_UNSUPPORTED, "prepack dtype");
    }
    FDPP_CHECK_LAUNCH("prepack_kernel");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_gemm_workspace_size(int32_t impl, const fdpp_gemm_params *p,
                                                size_t *bytes) {
    FDPP_REQUIRE(p && bytes, FDPP_ERR_VALUE, "null pointer");
    *bytes = 0;
    if (impl == FDPP_IMPL_A) return FDPP_OK;
    FDPP_REQUIRE(impl == FDPP_IMPL_B || impl == FDPP_IMPL_C, FDPP_ERR_VALUE, "bad impl %d", impl);
    TcPlan pl;
    fdpp_status s = plan_tc(p, impl == FDPP_IMPL_B, &pl);
    if (s != FDPP_OK) return s;
    *bytes = tc_workspace(pl, p);
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_impl_a_gemv(const fdpp_gemm_params *p, void *stream) {
    fdpp_status s = check_gemm(p);
    if (s != FDPP_OK) return s;
    FDPP_REQUIRE(p->M <= 8, FDPP_ERR_SHAPE, "ImplA (GEMV) supports M <= 8, got %d", p->M);
    FDPP_REQUIRE((reinterpret_cast<uintptr_t>(p->a) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(p->w) & 15) == 0,
                 FDPP_ERR_UNSUPPORTED, "GEMV operands must be 16-byte aligned");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return p->dtype == FDPP_BF16 ? launch_gemv<__nv_bfloat16>(p, st) : launch_gemv<__half>(p, st);
}

extern "C" fdpp_status fdpp_impl_b_flat(const fdpp_gemm_params *p, void *stream) {
    return run_tc(p, true, static_cast<cudaStream_t>(stream));
}

extern "C" fdpp_status fdpp_impl_c_gemm(const fdpp_gemm_params *p, void *stream) {
    return run_tc(p, false, static_cast<cudaStream_t>(stream));
}

extern "C" fdpp_status fdpp_run_kernel(int32_t impl, const fdpp_gemm_params *p, void *stream) {
    switch (impl) {
        case FDPP_IMPL_A: return fdpp_impl_a_gemv(p, stream);
        case FDPP_IMPL_B: return fdpp_impl_b_flat(p, stream);
        case FDPP_IMPL_C: return fdpp_impl_c_gemm(p, stream);
        default: FDPP_REQUIRE(false, FDPP_ERR_VALUE, "unknown kernel choice %d", impl);
    }
}

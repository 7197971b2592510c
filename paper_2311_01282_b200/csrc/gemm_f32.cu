// The flat-GEMM family in the reference's own precision (f32 storage, f32
// accumulation) for reference-signature calls with float32 operands.
//
// The reference's kernels compute in f32 (flatgemm.py:148-158 `_tile_mac`,
// dispatch.py:55-70 `_gemv_rows_njit`, dispatch.py:95-114 `_blocked_gemm_njit`)
// and its API promises <= 1e-4 row-relative error against the f64 oracle; the
// tensor-core paths compute from fp16/bf16 operands (~1e-3).  So a float32
// call (numpy arrays through flatdecode's API, or float32 CUDA tensors) runs
// here instead, on CUDA cores:
//
//   ImplA  BM = 8-row slabs x 128 weight rows per CTA (the GEMV's "stream the
//          weights once per slab of rows"),
//   ImplB  BM = M padded to 8 (<= 64) x 128 weight rows per CTA: the paper's
//          flat tile -- one N-split grid over the weight rows, the few tokens
//          padded to 8 (flatgemm.py:215-242),
//   ImplC  64 x 64 output blocks (the reference's 64^3 blocked GEMM).
//
// One kernel template serves all three: a CTA stages BK = 32 columns of its
// activation rows and weight rows in shared memory, double-buffered through
// registers (tile t + 1 is loaded while tile t is multiplied: the paper's
// double buffer), and each thread accumulates a TM x TN register block with
// fp32 FMA in ascending k.  Every output sums k in the same order for any
// grid, so results are bitwise reproducible and independent of the impl's
// tiling except through that order.  W is the prepacked [N, ldw] weight.
#include "common.cuh"

namespace fdpp {

constexpr int F32_BK = 32;
constexpr int F32_THREADS = 256;  // 8 thread rows x 32 thread columns

template <int BM, int BN>
__global__ void __launch_bounds__(F32_THREADS)
gemm_f32_kernel(const float *__restrict__ A, int64_t lda, const float *__restrict__ W, int64_t ldw,
                float *C, int64_t ldc, const float *R, int64_t ldr, int M, int N, int K) {
    constexpr int TM = BM / 8, TN = BN / 32;
    static_assert(TM >= 1 && TN >= 1, "tile");
    constexpr int A_V4 = BM * F32_BK / 4, W_V4 = BN * F32_BK / 4;  // float4 per tile
    constexpr int A_PER = (A_V4 + F32_THREADS - 1) / F32_THREADS;
    constexpr int W_PER = (W_V4 + F32_THREADS - 1) / F32_THREADS;
    __shared__ float sa[F32_BK][BM];  // k-major: a warp (one thread row) reads one broadcast value
    __shared__ float sw[F32_BK][BN + 1];

    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    pdl_wait();

    float4 ra[A_PER], rw[W_PER];
    auto load = [&](int k0) {
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int v = threadIdx.x + i * F32_THREADS;
            const int r = v / (F32_BK / 4), c = (v % (F32_BK / 4)) * 4;
            const int m = m0 + r, k = k0 + c;
            ra[i] = (v < A_V4 && m < M && k < K) ? __ldg(reinterpret_cast<const float4 *>(A + (int64_t)m * lda + k))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < W_PER; ++i) {
            const int v = threadIdx.x + i * F32_THREADS;
            const int r = v / (F32_BK / 4), c = (v % (F32_BK / 4)) * 4;
            const int n = n0 + r, k = k0 + c;
            rw[i] = (v < W_V4 && n < N && k < K) ? ld_stream_16f(W + (int64_t)n * ldw + k)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int v = threadIdx.x + i * F32_THREADS;
            if (v >= A_V4) break;
            const int r = v / (F32_BK / 4), c = (v % (F32_BK / 4)) * 4;
            sa[c][r] = ra[i].x; sa[c + 1][r] = ra[i].y; sa[c + 2][r] = ra[i].z; sa[c + 3][r] = ra[i].w;
        }
#pragma unroll
        for (int i = 0; i < W_PER; ++i) {
            const int v = threadIdx.x + i * F32_THREADS;
            if (v >= W_V4) break;
            const int r = v / (F32_BK / 4), c = (v % (F32_BK / 4)) * 4;
            sw[c][r] = rw[i].x; sw[c + 1][r] = rw[i].y; sw[c + 2][r] = rw[i].z; sw[c + 3][r] = rw[i].w;
        }
    };

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    const int ntiles = (K + F32_BK - 1) / F32_BK;
    load(0);
    for (int t = 0; t < ntiles; ++t) {
        __syncthreads();  // previous tile fully consumed
        store();
        __syncthreads();
        if (t + 1 < ntiles) load((t + 1) * F32_BK);  // next tile in flight under this tile's FMAs
#pragma unroll 8
        for (int k = 0; k < F32_BK; ++k) {
            float av[TM], wv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = sa[k][ty + 8 * i];
#pragma unroll
            for (int j = 0; j < TN; ++j) wv[j] = sw[k][tx + 32 * j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
        }
    }
    pdl_trigger();
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int m = m0 + ty + 8 * i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + tx + 32 * j;
            if (n >= N) continue;
            float s = acc[i][j];
            if (R) s += R[(int64_t)m * ldr + n];
            C[(int64_t)m * ldc + n] = s;
        }
    }
}

template <int BM, int BN>
static fdpp_status launch_f32(const fdpp_gemm_params *p, cudaStream_t st) {
    dim3 grid(ceil_div(p->N, BN), ceil_div(p->M, BM));
    cudaError_t e = launch_kernel(gemm_f32_kernel<BM, BN>, grid, dim3(F32_THREADS), 0, st,
                                  static_cast<const float *>(p->a), p->lda, static_cast<const float *>(p->w),
                                  p->ldw, static_cast<float *>(p->c), p->ldc, static_cast<const float *>(p->r),
                                  p->ldr, p->M, p->N, p->K);
    if (e != cudaSuccess) return cuda_status(e, "gemm_f32_kernel launch");
    return FDPP_OK;
}

fdpp_status run_gemm_f32(int impl, const fdpp_gemm_params *p, cudaStream_t st) {
    FDPP_REQUIRE(p && p->a && p->w && p->c, FDPP_ERR_VALUE, "null GEMM operand");
    FDPP_REQUIRE(p->M >= 1 && p->N >= 1 && p->K >= 1, FDPP_ERR_SHAPE,
                 "GEMM dims must be >= 1, got (%d, %d, %d)", p->M, p->N, p->K);
    FDPP_REQUIRE(p->K % 4 == 0 && p->lda % 4 == 0 && p->ldw % 4 == 0 && p->ldw >= p->K && p->lda >= p->K &&
                     p->ldc >= p->N && (reinterpret_cast<uintptr_t>(p->a) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(p->w) & 15) == 0,
                 FDPP_ERR_UNSUPPORTED, "f32 GEMM: K, lda, ldw multiples of 4, 16-byte aligned operands");
    switch (impl) {
        case FDPP_IMPL_A: return launch_f32<8, 128>(p, st);
        case FDPP_IMPL_B: {
            const int mp = (p->M + 7) / 8 * 8;  // the paper's pad-to-8 (flatgemm.py:215-242)
            if (mp <= 8) return launch_f32<8, 128>(p, st);
            if (mp <= 16) return launch_f32<16, 128>(p, st);
            if (mp <= 32) return launch_f32<32, 128>(p, st);
            return launch_f32<64, 128>(p, st);
        }
        case FDPP_IMPL_C: return launch_f32<64, 64>(p, st);
        default: FDPP_REQUIRE(false, FDPP_ERR_VALUE, "bad impl %d", impl);
    }
}

}  // namespace fdpp

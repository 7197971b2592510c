// The reference's vector softmax APIs (softmax.py:90-172)
// on the device.  Their arithmetic is what the attention kernels inline per
// logit; these entry points expose it for one f32 vector, as the reference's
// operator API does:
//   softmax_reference  (softmax.py:90-100)   max-subtracted, f64 internally
//   softmax_unified    (softmax.py:146-172)  e^(x - phi) in f32, f64 sum,
//                                            first non-finite index reported
//   partial_softmax_sync (softmax.py:113-143) per-chunk (max, f32 exp-sum)
//                                            states merged in chunk order
// One CTA per vector (per chunk for the partial states); fixed-order block
// reductions, so reruns are bitwise identical.
#include <cfloat>

#include "common.cuh"

namespace fdpp {

constexpr int SMX_THREADS = 1024;

template <typename V, typename Op>
__device__ __forceinline__ V block_reduce(V v, V *sh, Op op) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        V t = sh[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = op(t, sh[w]);  // warp order
        sh[32] = t;
    }
    __syncthreads();
    const V r = sh[32];
    __syncthreads();
    return r;
}

struct MaxF { __device__ float operator()(float a, float b) const { return fmaxf(a, b); } };
struct AddF { __device__ float operator()(float a, float b) const { return a + b; } };
struct AddD { __device__ double operator()(double a, double b) const { return a + b; } };
struct MinF { __device__ float operator()(float a, float b) const { return fminf(a, b); } };

// out = e / sum(e), e = exp(x - max) in f64 (softmax_reference_f64 / softmax_reference)
struct MaxD { __device__ double operator()(double a, double b) const { return fmax(a, b); } };

template <typename InT, typename OutT>
__global__ void __launch_bounds__(SMX_THREADS) softmax_ref_kernel(const InT *__restrict__ x, int n,
                                                                  OutT *__restrict__ out) {
    __shared__ double shd[33];
    double m = -INFINITY;
    for (int i = threadIdx.x; i < n; i += SMX_THREADS) m = fmax(m, (double)x[i]);
    m = block_reduce(m, shd, MaxD{});
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += SMX_THREADS) s += exp((double)x[i] - (double)m);
    s = block_reduce(s, shd, AddD{});
    for (int i = threadIdx.x; i < n; i += SMX_THREADS) out[i] = (OutT)(exp((double)x[i] - (double)m) / s);
}

// e_i = expf(x_i - phi) (f32); first non-finite i -> status[0]; sum in f64 -> total;
// out_i = float(double(e_i) / total).  The host raises SoftmaxOverflow /
// DegenerateSumError from status / total like the reference.
__global__ void __launch_bounds__(SMX_THREADS) softmax_unified_kernel(const float *__restrict__ x, int n,
                                                                      float phi, float *__restrict__ out,
                                                                      int *status, double *total) {
    __shared__ double shd[33];
    __shared__ float shf[33];
    int bad = INT_MAX;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += SMX_THREADS) {
        const float e = expf(x[i] - phi);
        if (!isfinite(e)) bad = min(bad, i);
        s += (double)e;
    }
    const float badf = block_reduce((float)min(bad, 1 << 24), shf, MinF{});
    s = block_reduce(s, shd, AddD{});
    if (threadIdx.x == 0) {
        status[0] = badf >= (float)(1 << 24) ? INT_MAX : (int)badf;
        *total = s;
    }
    if (badf < (float)(1 << 24) || s == 0.0 || !isfinite((float)s)) return;
    for (int i = threadIdx.x; i < n; i += SMX_THREADS) out[i] = (float)((double)expf(x[i] - phi) / s);
}

// error path of softmax_unified: first index where the f64 running sum leaves f32 range
__global__ void softmax_overflow_index_kernel(const float *__restrict__ x, int n, float phi, int *status) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        s += (double)expf(x[i] - phi);
        if (s > (double)FLT_MAX) {
            status[1] = i;
            return;
        }
    }
    status[1] = -1;
}

// chunk j of partial_softmax_sync: m_j = max, l_j = f32 sum of expf(x - m_j)
__global__ void __launch_bounds__(SMX_THREADS) softmax_chunk_state_kernel(const float *__restrict__ x,
                                                                          const int64_t *__restrict__ bounds,
                                                                          float *__restrict__ ml) {
    __shared__ float shf[33];
    const int j = blockIdx.x;
    const int lo = (int)bounds[j], hi = (int)bounds[j + 1];
    float m = -INFINITY;
    for (int i = lo + threadIdx.x; i < hi; i += SMX_THREADS) m = fmaxf(m, x[i]);
    m = block_reduce(m, shf, MaxF{});
    float l = 0.f;
    for (int i = lo + threadIdx.x; i < hi; i += SMX_THREADS) l += expf(x[i] - m);
    l = block_reduce(l, shf, AddF{});
    if (threadIdx.x == 0) {
        ml[2 * j] = m;
        ml[2 * j + 1] = l;
    }
}

// merge the chunk states in chunk order (merge_states, softmax.py:66-78), then
// out = expf(x - m_j) * expf(m_j - M) / L per chunk
__global__ void __launch_bounds__(SMX_THREADS) softmax_sync_finish_kernel(const float *__restrict__ x,
                                                                          const int64_t *__restrict__ bounds,
                                                                          int p, const float *__restrict__ ml,
                                                                          float *__restrict__ out) {
    __shared__ float s_M, s_L;
    if (threadIdx.x == 0) {
        float M = ml[0], L = ml[1];
        for (int j = 1; j < p; ++j) {
            const float m2 = ml[2 * j], l2 = ml[2 * j + 1];
            if (L == 0.f && M == -INFINITY) {
                M = m2;
                L = l2;
                continue;
            }
            if (l2 == 0.f && m2 == -INFINITY) continue;
            const float mm = fmaxf(M, m2);
            const float t1 = expf(M - mm) * L, t2 = expf(m2 - mm) * l2;
            M = mm;
            L = t1 + t2;
        }
        s_M = M;
        s_L = L;
    }
    __syncthreads();
    for (int j = 0; j < p; ++j) {
        const float scale = expf(ml[2 * j] - s_M);
        for (int i = (int)bounds[j] + threadIdx.x; i < (int)bounds[j + 1]; i += SMX_THREADS)
            out[i] = expf(x[i] - ml[2 * j]) * scale / s_L;
    }
}

}  // namespace fdpp

using namespace fdpp;

extern "C" fdpp_status fdpp_softmax_reference(const void *x, int32_t n, void *out, int32_t f64,
                                              void *stream) {
    FDPP_REQUIRE(x && out, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(n >= 1, FDPP_ERR_VALUE, "x must be a non-empty 1-D vector");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (f64)  // softmax_reference_f64: f64 in, f64 out
        softmax_ref_kernel<double, double><<<1, SMX_THREADS, 0, st>>>(static_cast<const double *>(x), n,
                                                                       static_cast<double *>(out));
    else      // softmax_reference: f32 in, f64 inside, f32 out
        softmax_ref_kernel<float, float><<<1, SMX_THREADS, 0, st>>>(static_cast<const float *>(x), n,
                                                                    static_cast<float *>(out));
    FDPP_CHECK_LAUNCH("softmax_ref_kernel");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_softmax_unified(const float *x, int32_t n, float phi, float *out, int32_t *status,
                                            double *total, void *stream) {
    FDPP_REQUIRE(x && out && status && total, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(n >= 1 && n < (1 << 24), FDPP_ERR_VALUE, "x must be a non-empty 1-D vector below 2^24");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    softmax_unified_kernel<<<1, SMX_THREADS, 0, st>>>(x, n, phi, out, status, total);
    FDPP_CHECK_LAUNCH("softmax_unified_kernel");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_softmax_overflow_index(const float *x, int32_t n, float phi, int32_t *status,
                                                   void *stream) {
    FDPP_REQUIRE(x && status && n >= 1, FDPP_ERR_VALUE, "bad arguments");
    softmax_overflow_index_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(x, n, phi, status);
    FDPP_CHECK_LAUNCH("softmax_overflow_index_kernel");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_partial_softmax_sync(const float *x, const int64_t *bounds, int32_t p, float *out,
                                                 float *ml, void *stream) {
    FDPP_REQUIRE(x && bounds && out && ml, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(p >= 1, FDPP_ERR_VALUE, "partition count must be >= 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    softmax_chunk_state_kernel<<<p, SMX_THREADS, 0, st>>>(x, bounds, ml);
    FDPP_CHECK_LAUNCH("softmax_chunk_state_kernel");
    softmax_sync_finish_kernel<<<1, SMX_THREADS, 0, st>>>(x, bounds, p, ml, out);
    FDPP_CHECK_LAUNCH("softmax_sync_finish_kernel");
    return FDPP_OK;
}

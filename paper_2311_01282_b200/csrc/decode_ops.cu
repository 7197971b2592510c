// Decode-step glue around the hot path: the small
// bandwidth-trivial kernels a real Llama decode step needs between the
// dispatched GEMMs and the attention op.  All fp32 math, fixed-order
// reductions, one CTA (or warp) per row.
#include "common.cuh"

namespace fdpp {

template <typename T>
__global__ void rmsnorm_kernel(const T *__restrict__ x, const T *__restrict__ w, T *__restrict__ out,
                               int dim, float eps) {
    pdl_wait();
    pdl_trigger();
    const int row = blockIdx.x;
    const T *xr = x + (int64_t)row * dim;
    float ss = 0.f;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
        const float v = Elem<T>::to_f(xr[i]);
        ss = fmaf(v, v, ss);
    }
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / dim + eps);
    for (int i = threadIdx.x; i < dim; i += blockDim.x)
        out[(int64_t)row * dim + i] = Elem<T>::from_f(Elem<T>::to_f(xr[i]) * inv * Elem<T>::to_f(w[i]));
}

// one block per batch row; thread i handles rotary pair (i, i + D/2) of one head
template <typename T>
__global__ void rope_append_kernel(const T *__restrict__ qkv, T *__restrict__ q_out, T *__restrict__ kc,
                                   T *__restrict__ vc, const int32_t *__restrict__ pos, int Hq, int Hkv,
                                   int D, int64_t csb, int64_t csh, float theta) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x;
    const int half = D / 2;
    const int width = (Hq + 2 * Hkv) * D;
    const T *row = qkv + (int64_t)b * width;
    const int p = pos[b];
    // capacity guard: a [B, Hkv, Lmax, D] cache holds csh / D rows per head; a
    // position past it is never written (it would land in the next head / row)
    const bool in_cache = p >= 0 && (int64_t)p < csh / D;
    for (int idx = threadIdx.x; idx < (Hq + Hkv) * half; idx += blockDim.x) {
        const int h = idx / half, i = idx % half;
        const double inv_freq = rope_inv_freq(theta, i, D);
        float sn, cs;
        rope_sincos(p, inv_freq, &sn, &cs);
        const T *src = row + h * D;  // q heads then k heads are contiguous in the fused row
        const float x0 = Elem<T>::to_f(src[i]), x1 = Elem<T>::to_f(src[i + half]);
        const T r0 = Elem<T>::from_f(x0 * cs - x1 * sn), r1 = Elem<T>::from_f(x1 * cs + x0 * sn);
        if (h < Hq) {
            T *dst = q_out + ((int64_t)b * Hq + h) * D;
            dst[i] = r0;
            dst[i + half] = r1;
        } else if (in_cache) {
            T *dst = kc + (int64_t)b * csb + (int64_t)(h - Hq) * csh + (int64_t)p * D;
            dst[i] = r0;
            dst[i + half] = r1;
        }
    }
    const T *vsrc = row + (Hq + Hkv) * D;
    for (int idx = threadIdx.x; in_cache && idx < Hkv * D; idx += blockDim.x) {
        const int h = idx / D, i = idx % D;
        vc[(int64_t)b * csb + (int64_t)h * csh + (int64_t)p * D + i] = vsrc[h * D + i];
    }
}

template <typename T>
__global__ void silu_mul_kernel(const T *__restrict__ gu, T *__restrict__ out, int F) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
        const float g = Elem<T>::to_f(gu[(int64_t)r * 2 * F + j]);
        const float u = Elem<T>::to_f(gu[(int64_t)r * 2 * F + F + j]);
        out[(int64_t)r * F + j] = Elem<T>::from_f(__fdividef(g, 1.f + __expf(-g)) * u);
    }
}

template <typename T>
__global__ void embed_kernel(const int32_t *__restrict__ ids, const T *__restrict__ table,
                             T *__restrict__ out, int dim, float *ssq_out) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x;
    const int64_t id = ids[b];
    float ss = 0.f;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
        const T v = table[id * dim + i];
        out[(int64_t)b * dim + i] = v;
        const float f = Elem<T>::to_f(v);
        ss = fmaf(f, f, ss);
    }
    if (ssq_out) {
        __shared__ float red[32];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
            ssq_out[b] = t;
        }
    }
}

// Per-row sum of squares of the residual stream (one tile spanning the row):
// what the folded-RMSNorm prologue of the next projection needs after a
// tensor-parallel all-reduce (the single-GPU path gets it from GEMM epilogues).
template <typename T>
__global__ void row_ssq_kernel(const T *__restrict__ x, int dim, float *__restrict__ ssq_out) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x;
    float ss = 0.f;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
        const float f = Elem<T>::to_f(x[(int64_t)b * dim + i]);
        ss = fmaf(f, f, ss);
    }
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];  // warp order
        ssq_out[b] = t;
    }
}

// Calibration producer: n logits s = scale * q[b, h] . k[b, h/G, key]
// at pseudo-random (b, h, key < lens[b]) -- the sample the reference's
// calibrate() (softmax.py:219-266) fits phi and the band to.  One warp per sample.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}

template <typename T>
__global__ void sample_logits_kernel(const T *__restrict__ q, const T *__restrict__ k,
                                     const int32_t *__restrict__ lens, int B, int Hq, int Hkv, int D,
                                     int L, int64_t q_sb, int64_t q_sh, int64_t kv_sb, int64_t kv_sh,
                                     float scale, int n, uint64_t seed, float *__restrict__ out,
                                     int32_t *__restrict__ idx_out) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint64_t r = mix64(seed * 0x9e3779b97f4a7c15ull + (uint64_t)i);
    const int b = (int)(r % (uint64_t)B);
    const int h = (int)((r >> 20) % (uint64_t)Hq);
    const int Lb = lens ? min(lens[b], L) : L;
    const int key = (int)((r >> 40) % (uint64_t)max(Lb, 1));
    const T *qp = q + (int64_t)b * q_sb + (int64_t)h * q_sh;
    const T *kp = k + (int64_t)b * kv_sb + (int64_t)(h / (Hq / Hkv)) * kv_sh + (int64_t)key * D;
    float acc = 0.f;
    for (int d = lane; d < D; d += 32) acc = fmaf(Elem<T>::to_f(qp[d]), Elem<T>::to_f(kp[d]), acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        out[i] = scale * acc;
        if (idx_out) {
            idx_out[3 * i] = b;
            idx_out[3 * i + 1] = h;
            idx_out[3 * i + 2] = key;
        }
    }
}

template <typename T>
__global__ void argmax_kernel(const T *__restrict__ logits, int32_t *__restrict__ ids, int vocab) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int j = threadIdx.x; j < vocab; j += blockDim.x) {
        const float v = Elem<T>::to_f(logits[(int64_t)r * vocab + j]);
        if (v > best || (v == best && j < bi)) { best = v; bi = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
        ids[r] = bi;
    }
}

__global__ void advance_kernel(int32_t *pos, int32_t *lens, int B) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        const int p = pos[b] + 1;
        pos[b] = p;
        if (lens) lens[b] = p + 1;
    }
}

}  // namespace fdpp

using namespace fdpp;

#define FDPP_DT_SWITCH(dtype, ...)                                       \
    switch (dtype) {                                                     \
        case FDPP_F16: { using T = __half; __VA_ARGS__; break; }         \
        case FDPP_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; } \
        case FDPP_F32: { using T = float; __VA_ARGS__; break; }          \
        default: set_error("bad dtype %d", dtype); return FDPP_ERR_UNSUPPORTED; \
    }

extern "C" fdpp_status fdpp_rmsnorm(const void *x, const void *w, void *out, int32_t rows,
                                    int32_t dim, float eps, int32_t dtype, void *stream) {
    FDPP_REQUIRE(rows >= 1 && dim >= 1, FDPP_ERR_SHAPE, "rmsnorm dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(rmsnorm_kernel<T>, dim3(rows), dim3(512), 0, st,
                                            static_cast<const T *>(x), static_cast<const T *>(w),
                                            static_cast<T *>(out), (int)dim, eps));
    if (e != cudaSuccess) return cuda_status(e, "rmsnorm_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_rope_append(const void *qkv, void *q_out, void *k_cache, void *v_cache,
                                        const int32_t *pos, int32_t B, int32_t Hq, int32_t Hkv,
                                        int32_t D, int64_t csb, int64_t csh, float theta,
                                        int32_t dtype, void *stream) {
    FDPP_REQUIRE(B >= 1 && Hq >= 1 && Hkv >= 1 && D >= 2 && D % 2 == 0, FDPP_ERR_SHAPE, "rope dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(rope_append_kernel<T>, dim3(B), dim3(512), 0, st,
                                            static_cast<const T *>(qkv), static_cast<T *>(q_out),
                                            static_cast<T *>(k_cache), static_cast<T *>(v_cache),
                                            pos, (int)Hq, (int)Hkv, (int)D, csb, csh, theta));
    if (e != cudaSuccess) return cuda_status(e, "rope_append_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_silu_mul(const void *gu, void *out, int32_t rows, int32_t F,
                                     int32_t dtype, void *stream) {
    FDPP_REQUIRE(rows >= 1 && F >= 1, FDPP_ERR_SHAPE, "silu_mul dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dim3 grid(ceil_div(F, 256) < 16 ? ceil_div(F, 256) : 16, rows);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(silu_mul_kernel<T>, grid, dim3(256), 0, st,
                                            static_cast<const T *>(gu), static_cast<T *>(out), (int)F));
    if (e != cudaSuccess) return cuda_status(e, "silu_mul_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_embed(const int32_t *ids, const void *table, void *out, int32_t B,
                                  int32_t dim, float *ssq_out, int32_t dtype, void *stream) {
    FDPP_REQUIRE(B >= 1 && dim >= 1, FDPP_ERR_SHAPE, "embed dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(embed_kernel<T>, dim3(B), dim3(256), 0, st, ids,
                                            static_cast<const T *>(table), static_cast<T *>(out),
                                            (int)dim, ssq_out));
    if (e != cudaSuccess) return cuda_status(e, "embed_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_row_ssq(const void *x, float *ssq_out, int32_t B, int32_t dim, int32_t dtype,
                                    void *stream) {
    FDPP_REQUIRE(x && ssq_out, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(B >= 1 && dim >= 1, FDPP_ERR_SHAPE, "row_ssq dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(row_ssq_kernel<T>, dim3(B), dim3(256), 0, st,
                                            static_cast<const T *>(x), (int)dim, ssq_out));
    if (e != cudaSuccess) return cuda_status(e, "row_ssq_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_sample_logits(const fdpp_attn_params *p, int32_t n, uint64_t seed,
                                          float *out, int32_t *idx_out, void *stream) {
    FDPP_REQUIRE(p && out && p->q && p->k, FDPP_ERR_VALUE, "null pointer");
    FDPP_REQUIRE(n >= 1 && p->B >= 1 && p->Hq >= 1 && p->Hkv >= 1 && p->Hq % p->Hkv == 0 && p->L >= 1 &&
                     p->D >= 1, FDPP_ERR_SHAPE, "sample_logits dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    const int per_block = 8;  // warps (samples) per 256-thread block
    FDPP_DT_SWITCH(p->dtype, e = launch_kernel(sample_logits_kernel<T>, dim3((n + per_block - 1) / per_block),
                                               dim3(32 * per_block), 0, st, static_cast<const T *>(p->q),
                                               static_cast<const T *>(p->k), p->seq_lens, (int)p->B,
                                               (int)p->Hq, (int)p->Hkv, (int)p->D, (int)p->L, p->q_stride_b,
                                               p->q_stride_h, p->kv_stride_b, p->kv_stride_h, p->scale,
                                               (int)n, (uint64_t)seed, out, idx_out));
    if (e != cudaSuccess) return cuda_status(e, "sample_logits_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_argmax(const void *logits, int32_t *ids, int32_t rows, int32_t vocab,
                                   int32_t dtype, void *stream) {
    FDPP_REQUIRE(rows >= 1 && vocab >= 1, FDPP_ERR_SHAPE, "argmax dims");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSuccess;
    FDPP_DT_SWITCH(dtype, e = launch_kernel(argmax_kernel<T>, dim3(rows), dim3(1024), 0, st,
                                            static_cast<const T *>(logits), ids, (int)vocab));
    if (e != cudaSuccess) return cuda_status(e, "argmax_kernel launch");
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_advance_positions(int32_t *pos, int32_t *lens, int32_t B, void *stream) {
    FDPP_REQUIRE(B >= 1, FDPP_ERR_SHAPE, "B");
    cudaError_t e = launch_kernel(advance_kernel, dim3(ceil_div(B, 256)), dim3(256), 0,
                                  static_cast<cudaStream_t>(stream), pos, lens, (int)B);
    if (e != cudaSuccess) return cuda_status(e, "advance_kernel launch");
    return FDPP_OK;
}

// Dev probe: best achievable HBM read bandwidth of ONE kernel that streams S
// bytes, as a function of S (the decode step's kernels stream 16 MB .. 540 MB
// each, so launch ramp and tail are a visible share).  Buffers rotate over
// >= 2 GB so every launch is L2-cold; launches are back to back on one stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/readbw.cu -o gpurun_out/readbw
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(512) readk(const int4 *__restrict__ p, int64_t n16, int *out) {
    // contiguous per-CTA range, U 16-B loads in flight per thread
    const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
    const int64_t b = blockIdx.x * per, e = min(n16, b + per);
    int acc = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += (int64_t)blockDim.x * U) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + (int64_t)u * blockDim.x;
            if (j < e) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                    : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
            else v[u] = make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

// same stream plus `extra` 16-B loads per 16-B streamed from a small
// L2-resident buffer (models the activation tile re-read by every weight tile)
__global__ void __launch_bounds__(512) readk_x(const int4 *__restrict__ p, int64_t n16,
                                               const int4 *__restrict__ x, int xmask, int ratio_q,
                                               int *out) {
    const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
    const int64_t b = blockIdx.x * per, e = min(n16, b + per);
    int acc = 0;
    int64_t cnt = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += (int64_t)blockDim.x * 8) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t j = i + (int64_t)u * blockDim.x;
            if (j < e) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                                    : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
            else v[u] = make_int4(0, 0, 0, 0);
        }
        int4 w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            w[u] = make_int4(0, 0, 0, 0);
            if (((cnt + u) & 3) < ratio_q)
                asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(w[u].x), "=r"(w[u].y), "=r"(w[u].z), "=r"(w[u].w)
                             : "l"(x + ((i + u * blockDim.x) & xmask)));
        }
        cnt += 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w ^ w[u].x ^ w[u].w;
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

int main(int argc, char **argv) {
    if (argc > 1) {  // L2-hit tax experiment: 100 MB stream + ratio_q/4 extra L2-hit bytes
        const size_t S = 100663296, pool = 4ull << 30;
        char *buf;
        int *out;
        int4 *x;
        cudaMalloc(&buf, pool);
        cudaMalloc(&out, 4);
        cudaMalloc(&x, 1 << 20);
        cudaMemset(buf, 1, pool);
        cudaMemset(x, 2, 1 << 20);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int nbuf = (int)(pool / S);
        for (int q = 0; q <= 4; ++q)
            for (int grid : {296, 1184}) {
                auto go = [&](int r) {
                    readk_x<<<grid, 512>>>(reinterpret_cast<const int4 *>(buf + (size_t)(r % nbuf) * S),
                                           (int64_t)(S / 16), x, (1 << 14) - 1, q, out);
                };
                for (int r = 0; r < nbuf; ++r) go(r);
                cudaEventRecord(e0);
                for (int r = 0; r < 4 * nbuf; ++r) go(r);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1e3 / (4 * nbuf);
                printf("extra L2-hit bytes = %d/4 of stream, grid=%4d: %8.2f us  stream %6.0f GB/s  total %6.0f GB/s\n",
                       q, grid, us, S / us / 1e3, S * (1 + q / 4.0) / us / 1e3);
            }
        return 0;
    }
    const size_t sizes[] = {16u << 20, 33554432, 100663296, 180355072, 536870912, 2147483648ull};
    const size_t pool = 4ull << 30;
    char *buf;
    if (cudaMalloc(&buf, pool) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(buf, 1, pool);
    int *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t S : sizes) {
        const int nbuf = (int)(pool / S) < 64 ? (int)(pool / S) : 64;
        for (int mult : {1, 2, 4, 8}) {
            for (int thr : {256, 512}) {
                const int grid = 148 * mult;
                const int reps = nbuf * (S < (1u << 28) ? 4 : 1);
                auto go = [&](int r) {
                    const int4 *p = reinterpret_cast<const int4 *>(buf + (size_t)(r % nbuf) * S);
                    readk<8><<<grid, thr>>>(p, (int64_t)(S / 16), out);
                };
                for (int r = 0; r < nbuf; ++r) go(r);
                cudaEventRecord(e0);
                for (int r = 0; r < reps; ++r) go(r);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1e3 / reps;
                printf("S=%8.1f MB grid=%4d thr=%3d  %8.2f us  %7.0f GB/s\n", S / 1e6, grid, thr, us,
                       S / us / 1e3);
            }
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}

// Dev probe: legacy warp-level mma.sync.m16n8k16 (f16 -> f32) throughput on
// sm_100a, to size the tensor-core GQA/MQA decode attention (which needs only
// ~16 flop/B x HBM bandwidth ~ 0.1-0.2 PFLOP/s).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mma_probe.cu -o tools/mma_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) mma_loop(float *out, int iters) {
    unsigned a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
    unsigned b[2] = {0x3c003c00u, 0x3c003c00u};
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 1.2345f) out[threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8}) {
        for (int per_sm : {1, 2, 4}) {
            const int grid = 148 * per_sm;
            mma_loop<<<grid, warps * 32>>>(out, 16);
            cudaEventRecord(e0);
            mma_loop<<<grid, warps * 32>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 16 * 8 * 16 * 8 * (double)iters * warps * grid;
            printf("warps/CTA=%d CTAs/SM=%d: %.1f TFLOP/s (mma.sync m16n8k16 f16->f32)\n", warps, per_sm,
                   flops / ms / 1e9);
        }
    }
    return 0;
}

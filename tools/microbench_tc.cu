// Dev microbenchmark: fixed per-CTA cost of the tcgen05 pipeline pieces.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//      tools/microbench_tc.cu -o gpurun_out/mb -lcuda
#include <cstdio>
#include <vector>

#include "../paper_2311_01282_b200/csrc/common.cuh"

using namespace fdpp;

namespace fdpp {
void set_error(const char *, ...) {}
fdpp_status cuda_status(cudaError_t, const char *) { return FDPP_ERR_CUDA; }
int sm_count() { return 148; }
}  // namespace fdpp

template <int MODE>
__global__ void __launch_bounds__(192, 1) probe(const __grid_constant__ CUtensorMap tm, float *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 32768);
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 4);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (MODE >= 1 && warp == 1) tmem_alloc(slot, 64);
    if (MODE >= 2 && threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tbase = MODE >= 1 ? *slot : 0;
    if (MODE >= 3 && threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[0], 2 * 128 * 128);  // two 128-row boxes
        tma_load_2d(smem, &tm, &bar[0], 0, blockIdx.x * 128, kEvictFirst);
        tma_load_2d(smem + 16384, &tm, &bar[0], 0, 0, kEvictLast);
    }
    if (MODE >= 3 && warp == 1 && lane == 0) {
        mbar_wait(&bar[0], 0);
        tc_fence_after();
        if (MODE >= 4) {
            const uint64_t da = umma_desc_sw128(smem), db = umma_desc_sw128(smem + 16384);
            for (int k = 0; k < 4; ++k) umma_f16(tbase, da + 2 * k, db + 2 * k, umma_idesc_f16(128, 32, false), k > 0);
            umma_commit(&bar[1]);
        }
    }
    if (MODE >= 4 && warp >= 2) {
        mbar_wait(&bar[1], 0);
        tc_fence_after();
        if (MODE >= 5) {
            float v[16];
            tmem_ld16(tbase + ((uint32_t)((warp & 3) * 32) << 16), v);
            if (v[0] == 12345.f) out[threadIdx.x] = v[1];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (MODE >= 1 && warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 64);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE>
float run(const CUtensorMap &tm, float *out, int grid, int iters) {
    auto k = probe<MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k<<<grid, 192, 40000>>>(tm, out);
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) k<<<grid, 192, 40000>>>(tm, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return ms * 1000.f / iters;
}

__global__ void empty_k() {}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fn;
    const int N = 128 * 148, K = 64;
    __half *w;
    float *out;
    cudaMalloc(&w, (size_t)N * K * 2);
    cudaMalloc(&out, 4096);
    cudaMemset(w, 0, (size_t)N * K * 2);
    CUtensorMap tm;
    cuuint64_t gd[2] = {(cuuint64_t)K, (cuuint64_t)N}, gs[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    const int iters = 200;
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int i = 0; i < 3; ++i) empty_k<<<148, 192>>>();
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) empty_k<<<148, 192>>>();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("empty kernel            : %7.2f us/launch\n", ms * 1000 / iters);
    }
    for (int grid : {1, 148}) {
        printf("grid %d\n", grid);
        printf(" mode0 (sync only)      : %7.2f us\n", run<0>(tm, out, grid, iters));
        printf(" mode1 (+tmem alloc)    : %7.2f us\n", run<1>(tm, out, grid, iters));
        printf(" mode2 (+mbar init)     : %7.2f us\n", run<2>(tm, out, grid, iters));
        printf(" mode3 (+TMA + wait)    : %7.2f us\n", run<3>(tm, out, grid, iters));
        printf(" mode4 (+MMA + commit)  : %7.2f us\n", run<4>(tm, out, grid, iters));
        printf(" mode5 (+tmem ld)       : %7.2f us\n", run<5>(tm, out, grid, iters));
    }
    return 0;
}

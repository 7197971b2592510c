// Dev probe: how long after the last CTA of a primary grid finishes does a
// programmatic-dependent secondary get past griddepcontrol.wait, versus a
// secondary that spins on a release/acquire counter the primary's CTAs bump?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pdl_latency tools/pdl_latency.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void primary(uint64_t *end_t, unsigned *counter, unsigned target_base, uint64_t spin_ns, float *sink) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t t0 = gtime();
    float acc = threadIdx.x;
    // uneven finish: CTA b spins spin_ns * (1 + b / gridDim)
    const uint64_t until = t0 + spin_ns + spin_ns * blockIdx.x / gridDim.x;
    while (gtime() < until) acc = acc * 1.0001f + 1.f;
    if (acc == -1.f) sink[0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        sink[1 + blockIdx.x] = acc;  // the "output"
        __threadfence();
        end_t[blockIdx.x] = gtime();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    }
}

__global__ void secondary(uint64_t *go_t, const unsigned *counter, unsigned target, int use_flag) {
    if (threadIdx.x == 0) {
        if (use_flag) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            } while (v < target);
        } else {
            asm volatile("griddepcontrol.wait;" ::: "memory");
        }
        go_t[blockIdx.x] = gtime();
    }
}

int main() {
    const int PA = 296, PB = 148, reps = 30;
    uint64_t *end_t, *go_t;
    unsigned *counter;
    float *sink;
    cudaMalloc(&end_t, PA * 8);
    cudaMalloc(&go_t, PB * 8);
    cudaMalloc(&counter, 4);
    cudaMalloc(&sink, (PA + 1) * 4);
    cudaMemset(counter, 0, 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    unsigned done = 0;  // the counter only grows: every primary CTA adds 1
    for (int use_flag = 0; use_flag < 2; ++use_flag) {
        for (uint64_t spin : {2000ull, 10000ull}) {
            std::vector<double> lat_min, lat_med;
            for (int r = 0; r < reps; ++r) {
                primary<<<PA, 128, 0, st>>>(end_t, counter, done, spin, sink);
                done += PA;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cudaLaunchConfig_t cb = {};
                cb.gridDim = dim3(PB);
                cb.blockDim = dim3(32);
                cb.stream = st;
                cb.attrs = at;
                cb.numAttrs = 1;
                cudaLaunchKernelEx(&cb, secondary, go_t, (const unsigned *)counter, done, use_flag);
                cudaStreamSynchronize(st);
                std::vector<uint64_t> e(PA), g(PB);
                cudaMemcpy(e.data(), end_t, PA * 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(g.data(), go_t, PB * 8, cudaMemcpyDeviceToHost);
                const uint64_t last = *std::max_element(e.begin(), e.end());
                std::sort(g.begin(), g.end());
                if (r >= 5) {
                    lat_min.push_back(((double)g[0] - (double)last) / 1000.0);
                    lat_med.push_back(((double)g[PB / 2] - (double)last) / 1000.0);
                }
            }
            std::sort(lat_min.begin(), lat_min.end());
            std::sort(lat_med.begin(), lat_med.end());
            printf("%s spin=%5llu ns: secondary past its wait, after the primary's last CTA end: first CTA p50 %.2f us, median CTA p50 %.2f us\n",
                   use_flag ? "flag (ld.acquire poll)   " : "griddepcontrol.wait (PDL)", (unsigned long long)spin,
                   lat_min[lat_min.size() / 2], lat_med[lat_med.size() / 2]);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}

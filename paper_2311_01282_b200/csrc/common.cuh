// Shared device/host helpers for the sm_100a kernels: status plumbing, PTX
// wrappers for mbarrier, bulk/TMA copies and tcgen05 (TMEM, UMMA).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/fdpp.h"

namespace fdpp {

// ------------------------------------------------------------------ host side
void set_error(const char *fmt, ...);
fdpp_status cuda_status(cudaError_t e, const char *what);
int sm_count();
// f32 CUDA-core flat-GEMM family (gemm_f32.cu): reference-precision calls
fdpp_status run_gemm_f32(int impl, const fdpp_gemm_params *p, cudaStream_t st);

#define FDPP_CHECK_LAUNCH(what)                                     \
    do {                                                            \
        cudaError_t _e = cudaGetLastError();                        \
        if (_e != cudaSuccess) return ::fdpp::cuda_status(_e, what); \
    } while (0)

#define FDPP_REQUIRE(cond, code, ...)          \
    do {                                       \
        if (!(cond)) {                         \
            ::fdpp::set_error(__VA_ARGS__);    \
            return code;                       \
        }                                      \
    } while (0)

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Per-device "done" bits for one-time launch setup (cudaFuncSetAttribute):
// thread-safe (the setup is idempotent, so two threads racing both run it)
// and per device (a second GPU in the process gets its own setup).
struct DeviceOnce {
    std::atomic<uint64_t> done{0};
    template <typename F>
    cudaError_t run(F &&f) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
        e = f();
        if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
        return e;
    }
};

// Every workspace starts with a fixed region of ticket counters that is never
// used for anything else, so a pooled buffer reused by a differently shaped
// call can never see partial sums where it expects zeroed counters.
constexpr int kWsCounters = 16384;
constexpr size_t kWsCounterBytes = kWsCounters * sizeof(int);

// Launch with the programmatic-stream-serialization attribute when PDL is
// enabled (fdpp_set_pdl); every kernel in libfdpp calls pdl_wait() before
// reading a predecessor's output or writing any global memory.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block,
                                         size_t smem, cudaStream_t st, int cluster_x,
                                         Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    static const bool occ_probe = getenv("FDPP_OCC_PROBE") != nullptr;  // dev: cluster residency
    if (occ_probe && cluster_x > 1) {
        int nc = -1;
        cudaError_t oe = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
        fprintf(stderr, "[occ] grid %ux%u block %u smem %zu cluster %d: clusters %u, max active %d (%s)\n",
                grid.x, grid.y, block.x, smem, cluster_x, grid.x * grid.y / cluster_x, nc,
                cudaGetErrorString(oe));
    }
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st, Args &&...args) {
    return launch_kernel_cluster(kern, grid, block, smem, st, 1, std::forward<Args>(args)...);
}

// 2-D tile map over a row-major [rows, cols] 16-bit matrix (leading dim ld):
// box = [64 cols x box_rows], SWIZZLE_128B, OOB zero-filled; cached per
// (pointer, shape).  Defined in gemm.cu.
fdpp_status make_kmajor_map(CUtensorMap *out, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                            int box_rows, int dtype);

// RoPE angle p * theta^(-2i/D) in double, reduced to [-pi, pi], then the fast
// intrinsic: accurate at 32K-scale positions (a float angle alone is off by up
// to ~2e-3 rad there, and __sincosf's own reduction degrades with |x|)
__device__ __forceinline__ double rope_inv_freq(float theta, int i, int D) {
    return pow((double)theta, -2.0 * i / D);
}
// p * f with f = (hi, lo) float pair from the double; exact product error via
// fma, Cody-Waite reduction by 2 pi in float (no per-element double math)
__device__ __forceinline__ void rope_sincos(int p, double inv_freq, float *sn, float *cs) {
    const float f_hi = (float)inv_freq, f_lo = (float)(inv_freq - (double)f_hi);
    const float pf = (float)p;                      // exact: p < 2^24
    const float x_hi = pf * f_hi;
    const float x_err = fmaf(pf, f_hi, -x_hi) + pf * f_lo;
    const float k = rintf(x_hi * 0.159154943091895336f);
    float r = fmaf(-k, 6.28318548202514648f, x_hi);  // 2 pi = hi + lo, hi = float(2 pi)
    r = fmaf(-k, -1.74845553146951718e-07f, r) + x_err;
    __sincosf(r, sn, cs);
}

// ------------------------------------------------------------- element types
template <typename T> struct Elem;
template <> struct Elem<__half> {
    __device__ static __forceinline__ float to_f(__half x) { return __half2float(x); }
    __device__ static __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
    __device__ static __forceinline__ float2 to_f2(uint32_t u) {
        __half2 h = *reinterpret_cast<__half2 *>(&u);
        return __half22float2(h);
    }
};
template <> struct Elem<__nv_bfloat16> {
    __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
    __device__ static __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
    __device__ static __forceinline__ float2 to_f2(uint32_t u) {
        __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162 *>(&u);
        return __bfloat1622float2(h);
    }
};
template <> struct Elem<float> {
    __device__ static __forceinline__ float to_f(float x) { return x; }
    __device__ static __forceinline__ float from_f(float x) { return x; }
};

// ------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// L2 cache policies (createpolicy.fractional encodings used by CUTLASS)
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// 1-D bulk copy global -> shared, completion on an mbarrier (TMA bulk engine)
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 2-D tensor-map (TMA) tile load global -> shared
__device__ __forceinline__ void tma_load_2d(void *dst_smem, const CUtensorMap *map, uint64_t *bar,
                                            int32_t c0, int32_t c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst_smem)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

// 2-D tensor-map tile prefetch global -> L2 (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t *slot_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem desc] · B[smem desc]^T, kind::f16 (fp16/bf16 in, fp32 acc)
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// mbarrier arrives when all prior tcgen05 ops of this thread complete
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32 bits, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor: K-major operand tile laid out by a TMA
// SWIZZLE_128B load (rows of 64 fp16 = 128 B, 8-row atoms of 1024 B).
//   bits  0-13 start address >> 4
//   bits 16-29 leading byte offset >> 4 (unused for swizzled K-major: 1)
//   bits 32-45 stride byte offset >> 4 (1024 B between 8-row groups)
//   bits 46-47 version = 1 (sm_100)
//   bits 61-63 layout = 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t umma_desc_sw128(const void *smem_tile) {
    uint64_t addr = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor for kind::f16 with fp32 accumulate, both operands K-major.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N, bool bf16) {
    return (1u << 4)                         // D format: f32
           | ((bf16 ? 1u : 0u) << 7)         // A format
           | ((bf16 ? 1u : 0u) << 10)        // B format
           | ((uint32_t)(N >> 3) << 17)      // N / 8
           | ((uint32_t)(M >> 4) << 24);     // M / 16
}

// Programmatic dependent launch (PDL).  Kernels launched with
// launch_kernel() may start before their predecessor in the stream finishes:
// everything before pdl_wait() must touch only data no earlier kernel writes
// (weights, tensor maps, smem/TMEM setup).  pdl_wait() returns once every
// prerequisite grid has completed and its writes are visible; it is a no-op
// when the launch had no programmatic dependency.
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
// Allow the next kernel in the stream to begin launching (its pdl_wait()
// still waits for this whole grid to finish).
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------ clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// split form: arrive (non-blocking) now, wait later (every thread does both)
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
// address of `local_smem` in the shared memory of cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_map(const void *local_smem, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local_smem)), "r"(rank));
    return r;
}
__device__ __forceinline__ float dsmem_ld_f32(uint32_t cluster_addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr) : "memory");
    return v;
}

// 4-B DSMEM load with no memory clobber: loads of a loop issue back to back
__device__ __forceinline__ float dsmem_ld_f32_batched(uint32_t cluster_addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr));
    return v;
}

// 16-B DSMEM load with no memory clobber: a run of these issues back to back
// (one round trip for all of them)
__device__ __forceinline__ float4 dsmem_ld_v4(uint32_t cluster_addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(cluster_addr));
    return v;
}
// OR into a 32-bit word in a cluster peer's shared memory
__device__ __forceinline__ void dsmem_red_or_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dsmem_map_addr(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Trace build only (-DFDPP_TRACE): per-CTA event timestamps for the dev tools.
#ifdef FDPP_TRACE
// [launch % 8][cta][slot]; the launch number comes from a per-CTA-index counter
static __device__ unsigned long long g_fdpp_trace[8][512][8];  // one TU (gemm.cu) uses it
static __device__ unsigned int g_fdpp_launch[512];
#define FDPP_TRACE_AT(slot)                                                       \
    do {                                                                          \
        if (blockIdx.x < 512) g_fdpp_trace[s_trace_seq & 7][blockIdx.x][slot] = globaltimer_ns(); \
    } while (0)
#else
#define FDPP_TRACE_AT(slot) do { } while (0)
#endif

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float ld_cg_f32(const float *p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// streaming 16-B load: read-only path, no L1 allocation, L2 evict-first
__device__ __forceinline__ int4 ld_stream_16(const void *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(kEvictFirst));
    return r;
}
__device__ __forceinline__ float4 ld_stream_16f(const void *p) {
    const int4 r = ld_stream_16(p);
    return make_float4(__int_as_float(r.x), __int_as_float(r.y), __int_as_float(r.z), __int_as_float(r.w));
}

}  // namespace fdpp

// Host-side half of the C ABI: error plumbing, device queries and the
// integer decision logic of subsystem 3 (heuristic dispatch) — the parts of
// dispatch.py / softmax.py that are pure control flow, restated natively so a
// C/Go/Java caller gets the same decisions as the Python wrapper.
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <mutex>

#include "../../include/fdpp.h"

namespace fdpp {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

fdpp_status cuda_status(cudaError_t e, const char *what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FDPP_ERR_CUDA;
}

// FDPP_PDL=0 starts with programmatic dependent launch off (A/B); fdpp_set_pdl changes it
static std::atomic<int> g_pdl{[] {
    const char *e = getenv("FDPP_PDL");
    return e ? (atoi(e) != 0 ? 1 : 0) : 1;
}()};
bool pdl_enabled() { return g_pdl.load(std::memory_order_relaxed) != 0; }

int sm_count() {
    static int cached = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (cached == 0) {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        cached = n;
    }
    return cached;
}

}  // namespace fdpp

extern "C" const char *fdpp_last_error(void) { return fdpp::g_err; }

extern "C" int fdpp_version(void) { return 101; }

extern "C" int fdpp_set_pdl(int enable) {
    return fdpp::g_pdl.exchange(enable ? 1 : 0);
}

extern "C" int fdpp_sm_count(void) { return fdpp::sm_count(); }

// dispatch.py:189-197
extern "C" int32_t fdpp_dispatch_choose(int32_t m, int32_t m1, int32_t m2) {
    if (m < m1) return FDPP_IMPL_A;
    if (m < m2) return FDPP_IMPL_B;
    return FDPP_IMPL_C;
}

// dispatch.py:248-265: first i >= start with new <= old at i and at i+1 (unless
// i is the last point), and no later pair of consecutive losses.
extern "C" int32_t fdpp_first_sustained(const double *nw, const double *od, int32_t n,
                                        int32_t start) {
    for (int32_t i = start; i < n; ++i) {
        if (nw[i] > od[i]) continue;
        if (i < n - 1 && nw[i + 1] > od[i + 1]) continue;
        bool relapsed = false;
        for (int32_t j = i + 1; j < n - 1; ++j)
            if (nw[j] > od[j] && nw[j + 1] > od[j + 1]) {
                relapsed = true;
                break;
            }
        if (!relapsed) return i;
    }
    return -1;
}

// dispatch.py:326-338
extern "C" fdpp_status fdpp_profile_decide(const int32_t *sweep, const double *a, const double *b,
                                           const double *c, int32_t n, int32_t *m1, int32_t *m2) {
    if (!sweep || !a || !b || !c || !m1 || !m2) {
        fdpp::set_error("null pointer");
        return FDPP_ERR_VALUE;
    }
    if (n < 2) {
        fdpp::set_error("m_sweep must be ascending with at least 2 points");
        return FDPP_ERR_VALUE;
    }
    for (int32_t i = 1; i < n; ++i)
        if (sweep[i] <= sweep[i - 1]) {
            fdpp::set_error("m_sweep must be ascending with at least 2 points");
            return FDPP_ERR_VALUE;
        }
    const int32_t beyond = 2 * sweep[n - 1];
    const int32_t i1 = fdpp_first_sustained(b, a, n, 0);
    if (i1 < 0) {
        const int32_t iac = fdpp_first_sustained(c, a, n, 0);
        *m1 = *m2 = iac >= 0 ? sweep[iac] : beyond;
    } else {
        const int32_t i2 = fdpp_first_sustained(c, b, n, i1);
        *m1 = sweep[i1];
        *m2 = i2 >= 0 ? (sweep[i2] > *m1 ? sweep[i2] : *m1) : beyond;
    }
    return FDPP_OK;
}

// softmax.py:103-110
extern "C" fdpp_status fdpp_chunk_bounds(int64_t n, int32_t p, int64_t *bounds) {
    if (!bounds) {
        fdpp::set_error("null bounds");
        return FDPP_ERR_VALUE;
    }
    if (p < 1 || p > n) {
        fdpp::set_error("partition count must be in [1, %lld], got %d", (long long)n, p);
        return FDPP_ERR_VALUE;
    }
    const int64_t base = n / p;
    for (int32_t i = 0; i <= p; ++i) bounds[i] = (int64_t)i * base;
    bounds[p] = n;
    return FDPP_OK;
}

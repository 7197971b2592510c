// Subsystem 1 kernels, f16 async softmax: explicit instantiations (attention_kernels.cuh).
#include "attention_kernels.cuh"

namespace fdpp {
template fdpp_status by_d<__half, true>(const AttnArgs &, int, int, int, cudaStream_t);
template fdpp_status launch_mma_t<__half, true>(const AttnArgs &, int, const CUtensorMap *,
                                                 const CUtensorMap *, cudaStream_t);
}  // namespace fdpp

#ifdef FDPP_ATRACE
extern "C" int fdpp_atrace_read(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, fdpp::g_atrace, sizeof(fdpp::g_atrace));
}
extern "C" int fdpp_atrace_reset(void) {
    static unsigned long long z[8192][8];
    return (int)cudaMemcpyToSymbol(fdpp::g_atrace, z, sizeof(z));
}
#endif

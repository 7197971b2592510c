// Subsystem 1 kernels, bf16 async softmax: explicit instantiations (attention_kernels.cuh).
#include "attention_kernels.cuh"

namespace fdpp {
template fdpp_status by_d<__nv_bfloat16, true>(const AttnArgs &, int, int, int, cudaStream_t);
template fdpp_status launch_mma_t<__nv_bfloat16, true>(const AttnArgs &, int, const CUtensorMap *,
                                                 const CUtensorMap *, cudaStream_t);
}  // namespace fdpp

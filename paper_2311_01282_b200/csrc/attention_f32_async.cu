// Subsystem 1 kernels, f32 async softmax: explicit instantiations (attention_kernels.cuh).
#include "attention_kernels.cuh"

namespace fdpp {
template fdpp_status by_d<float, true>(const AttnArgs &, int, int, int, cudaStream_t);
}  // namespace fdpp

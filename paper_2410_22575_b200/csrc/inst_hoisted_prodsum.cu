// inst_hoisted_prodsum.cu -- NEXT-4 hoisted HVP kernels for FUNC_PRODSUM: n in {2, 4, 8, 16},
// compile-time rows / chunks / variables (hvp_small_kernel, kernels.cuh).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SMALL(F, C, NS) template cudaError_t launch_small<F, C, NS>(BatchArgs, cudaStream_t);
CHF_FOR_SMALL(CHF_INST_SMALL, FUNC_PRODSUM)
}  // namespace chessfad

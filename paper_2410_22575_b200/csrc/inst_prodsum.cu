// inst_prodsum.cu -- kernel instantiations for FUNC_PRODSUM (hDual<C> in registers), C in {1..32}.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_REG(F, C)                                                 \
  template cudaError_t launch_reg<F, C, false>(BatchArgs, cudaStream_t); \
  template cudaError_t launch_reg<F, C, true>(BatchArgs, cudaStream_t);
CHF_FOR_C(CHF_INST_REG, FUNC_PRODSUM)
}  // namespace chessfad

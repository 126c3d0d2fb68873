// inst_ackley.cu -- kernel instantiations for FUNC_ACKLEY (hDual<C> in registers), C in {1,2,4,8,16},
// all four modes (Alg 7, Alg 5, Alg 8, Alg 6).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_REG1(F, C, M) template cudaError_t launch_reg<F, C, M>(BatchArgs, cudaStream_t);
#define CHF_INST_REG(F, C) CHF_FOR_MODE(CHF_INST_REG1, F, C)
CHF_FOR_C(CHF_INST_REG, FUNC_ACKLEY)
}  // namespace chessfad

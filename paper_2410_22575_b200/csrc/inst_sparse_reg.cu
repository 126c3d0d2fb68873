// inst_sparse_reg.cu -- kernel instantiations of the seed-sparse register-path bodies (NEXT-4,
// testfuncs.cuh SparseFunc) for F1, F2, F4: Alg 7 HVP, Alg 5 Hessian, Alg 8 symmetric HVP,
// Alg 6 symmetric Hessian and Alg 5 + gradient, C in {1,2,4,8,16}.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SPR1(F, C) CHF_FOR_SP_MODE(CHF_INST_SPR2, F, C)
#define CHF_INST_SPR2(F, C, M) template cudaError_t launch_sparse_reg<F, C, M>(BatchArgs, cudaStream_t);
CHF_FOR_C(CHF_INST_SPR1, FUNC_ROSENBROCK)
CHF_FOR_C(CHF_INST_SPR1, FUNC_ACKLEY)
CHF_FOR_C(CHF_INST_SPR1, FUNC_PRODSUM)
}  // namespace chessfad

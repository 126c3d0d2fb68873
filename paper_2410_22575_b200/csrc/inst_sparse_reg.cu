// inst_sparse_reg.cu -- kernel instantiations of the seed-sparse register-path bodies (NEXT-4,
// testfuncs.cuh SparseFunc) for F1, F2, F4: HVP and Hessian, C in {1,2,4,8,16}.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SPR1(F, C) template cudaError_t launch_sparse_reg<F, C, MODE_HVP>(BatchArgs, cudaStream_t); \
  template cudaError_t launch_sparse_reg<F, C, MODE_HESS>(BatchArgs, cudaStream_t);
CHF_FOR_C(CHF_INST_SPR1, FUNC_ROSENBROCK)
CHF_FOR_C(CHF_INST_SPR1, FUNC_ACKLEY)
CHF_FOR_C(CHF_INST_SPR1, FUNC_PRODSUM)
}  // namespace chessfad

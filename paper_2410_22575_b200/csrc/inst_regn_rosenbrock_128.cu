// inst_regn_rosenbrock_128.cu -- the register-path kernel compiled for n == 128 (FUNC_ROSENBROCK),
// C in {1,2,4,8,16}, Alg 7 only (kernels.cuh NS; dispatched by capi.cu for n == 128).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_REGNB(F, C, NS) template cudaError_t launch_reg_n<F, C, MODE_HVP, NS>(BatchArgs, cudaStream_t);
CHF_FOR_REGN_C(CHF_INST_REGNB, FUNC_ROSENBROCK, 128)
}  // namespace chessfad

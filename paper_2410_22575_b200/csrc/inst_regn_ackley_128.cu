// inst_regn_ackley_128.cu -- the register-path kernel compiled for n == 128 (FUNC_ACKLEY),
// C in {1,2,4,8,16}, Alg 7 only (kernels.cuh NS; capi.cu dispatches it at kernel chunk 8 only).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_REGNB(F, C, NS) template cudaError_t launch_reg_n<F, C, MODE_HVP, NS>(BatchArgs, cudaStream_t);
CHF_FOR_REGN_C(CHF_INST_REGNB, FUNC_ACKLEY, 128)
}  // namespace chessfad

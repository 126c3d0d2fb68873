// inst_regn_prodsum_32.cu -- the register-path kernel compiled for n == 32 (FUNC_PRODSUM),
// C in {1,2,4,8,16}, every mode (kernels.cuh NS; dispatched by capi.cu for n == 32).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_REGN2(F, C, M, NS) template cudaError_t launch_reg_n<F, C, M, NS>(BatchArgs, cudaStream_t);
#define CHF_INST_REGN1(F, C, NS) CHF_FOR_REGN_MODE(CHF_INST_REGN2, F, C, NS)
CHF_FOR_REGN_C(CHF_INST_REGN1, FUNC_PRODSUM, 32)
}  // namespace chessfad

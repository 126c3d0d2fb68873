// inst_f3mma_120.cu -- F3 tensor-core kernels (hvp_f3_mma_kernel, f3_mma.cuh) for n <= 120, all modes.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_MMA1(NN, M) template cudaError_t launch_f3_mma<NN, M>(BatchArgs, cudaStream_t);
CHF_FOR_MMA_MODE(CHF_INST_MMA1, 120)
}  // namespace chessfad

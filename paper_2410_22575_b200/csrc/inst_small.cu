// inst_small.cu -- small-n HVP kernels (n in {2, 4, 8}, compile-time seeds) for F1, F2, F4.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SMALL(F, C, NS) template cudaError_t launch_small<F, C, NS>(BatchArgs, cudaStream_t);
CHF_FOR_SMALL(CHF_INST_SMALL, FUNC_ROSENBROCK)
CHF_FOR_SMALL(CHF_INST_SMALL, FUNC_ACKLEY)
CHF_FOR_SMALL(CHF_INST_SMALL, FUNC_PRODSUM)
}  // namespace chessfad

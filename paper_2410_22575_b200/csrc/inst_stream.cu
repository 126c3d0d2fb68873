// inst_stream.cu -- Alg 7 kernels for n in {2, 4, 8} (hvp_stream_kernel, stream_small.cuh):
// thread per point, persistent grid, bulk-copy ring; Rosenbrock, Ackley, prodsum.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_STREAM(F, C, NS) template cudaError_t launch_stream<F, C, NS>(BatchArgs, cudaStream_t);
CHF_FOR_STREAM(CHF_INST_STREAM, FUNC_ROSENBROCK)
CHF_FOR_STREAM(CHF_INST_STREAM, FUNC_ACKLEY)
CHF_FOR_STREAM(CHF_INST_STREAM, FUNC_PRODSUM)
}  // namespace chessfad

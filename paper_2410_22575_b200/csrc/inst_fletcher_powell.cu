// inst_fletcher_powell.cu -- kernel instantiations for F3 (slot-column schedule, f3.cuh).
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_F3(KB)                                                  \
  template cudaError_t launch_f3<KB, false, false>(BatchArgs, cudaStream_t); \
  template cudaError_t launch_f3<KB, false, true>(BatchArgs, cudaStream_t);  \
  template cudaError_t launch_f3<KB, true, false>(BatchArgs, cudaStream_t);  \
  template cudaError_t launch_f3<KB, true, true>(BatchArgs, cudaStream_t);
CHF_INST_F3(1) CHF_INST_F3(2) CHF_INST_F3(4) CHF_INST_F3(8) CHF_INST_F3(16)
}  // namespace chessfad

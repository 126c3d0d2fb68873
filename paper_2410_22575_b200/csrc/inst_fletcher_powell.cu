// inst_fletcher_powell.cu -- kernel instantiations for F3 (slot-column schedule, f3.cuh),
// all four modes, (A,B) in shared memory or global.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_F31(KB, AB, M) template cudaError_t launch_f3<KB, M, AB>(BatchArgs, cudaStream_t);
#define CHF_INST_F3(KB) CHF_FOR_MODE(CHF_INST_F31, KB, false) CHF_FOR_MODE(CHF_INST_F31, KB, true) \
  CHF_INST_F31(KB, false, MODE_HVP_ROWHOIST) CHF_INST_F31(KB, true, MODE_HVP_ROWHOIST)
CHF_INST_F3(1) CHF_INST_F3(2) CHF_INST_F3(4) CHF_INST_F3(8) CHF_INST_F3(16)
}  // namespace chessfad

// inst_f3_sparse.cu -- kernel instantiations of the seed-sparse F3 HVP (NEXT-4,
// f3_sparse.cuh), one per column block CB.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SP(CB) template cudaError_t launch_f3_sparse<CB, false>(BatchArgs, cudaStream_t); \
  template cudaError_t launch_f3_sparse<CB, true>(BatchArgs, cudaStream_t);
CHF_FOR_CB(CHF_INST_SP)
}  // namespace chessfad

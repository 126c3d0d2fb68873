// inst_f3_sparse.cu -- kernel instantiations of the seed-sparse F3 HVP (NEXT-4,
// f3_sparse.cuh), one per column block CB.
#include "launch.cuh"

namespace chessfad {
#define CHF_INST_SP1(CB, M) template cudaError_t launch_f3_sparse<CB, M>(BatchArgs, cudaStream_t);
#define CHF_INST_SP(CB) CHF_FOR_F3SP_MODE(CHF_INST_SP1, CB)
CHF_FOR_CB(CHF_INST_SP)
}  // namespace chessfad

// launch.cuh -- host-side launchers for the kernel instantiations (one .cu per function
// family so that nvcc compiles them in parallel).  Used only by capi.cu.
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace chessfad {

// groups of 32 points per CTA so that every warp of the CTA has a row to work on
inline int groups_for(int n, int warps) {
  int g = 1;
  while (g * 2 <= warps && n * g * 2 <= warps) g *= 2;
  return g;
}

inline size_t reg_smem_bytes(int func, int n, int G, bool hess) {
  return (size_t)((hess ? 1 : 3) + (func == FUNC_ACKLEY ? 2 : 0)) * G * n * kPad * sizeof(double);
}

inline size_t f3_smem_bytes(int n, int G, bool hess, bool ab_smem) {
  return (size_t)(hess ? 2 : 4) * G * n * kPad * sizeof(double) + (ab_smem ? (size_t)n * n * 2 * sizeof(double) : 0);
}

template <class K>
inline cudaError_t launch_with_smem(K kernel, int grid, int block, size_t smem, cudaStream_t s, const BatchArgs& a) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}

// warps per CTA of the register path (tuning knob CHESSFAD_REG_WARPS = 4 | 8, read once)
int reg_warps();

template <int FUNC, int C, bool HESS, int W>
cudaError_t launch_reg_w(BatchArgs a, cudaStream_t s) {
  a.groups = groups_for(a.n, W);
  const int64_t P = 32 * a.groups;
  const int grid = (int)((a.m + P - 1) / P);
  return launch_with_smem(hvp_reg_kernel<FUNC, C, HESS, W>, grid, W * 32, reg_smem_bytes(FUNC, a.n, a.groups, HESS),
                          s, a);
}

template <int FUNC, int C, bool HESS>
cudaError_t launch_reg(BatchArgs a, cudaStream_t s) {
  return reg_warps() == 8 ? launch_reg_w<FUNC, C, HESS, 8>(a, s) : launch_reg_w<FUNC, C, HESS, 4>(a, s);
}

template <int KB, bool HESS, bool AB_SMEM>
cudaError_t launch_f3(BatchArgs a, cudaStream_t s) {
  a.groups = groups_for(a.n, kWarpsF3);
  const int64_t P = 32 * a.groups;
  const int grid = (int)((a.m + P - 1) / P);
  return launch_with_smem(hvp_f3_kernel<KB, HESS, AB_SMEM>, grid, kWarpsF3 * 32,
                          f3_smem_bytes(a.n, a.groups, HESS, AB_SMEM), s, a);
}

// explicit-instantiation declarations (definitions in inst_*.cu)
#define CHF_DECL_REG(F, C)                                         \
  extern template cudaError_t launch_reg<F, C, false>(BatchArgs, cudaStream_t); \
  extern template cudaError_t launch_reg<F, C, true>(BatchArgs, cudaStream_t);
#define CHF_FOR_C(X, F) X(F, 1) X(F, 2) X(F, 4) X(F, 8) X(F, 16) X(F, 32)
CHF_FOR_C(CHF_DECL_REG, FUNC_ROSENBROCK)
CHF_FOR_C(CHF_DECL_REG, FUNC_ACKLEY)
CHF_FOR_C(CHF_DECL_REG, FUNC_PRODSUM)

#define CHF_DECL_F3(KB)                                                   \
  extern template cudaError_t launch_f3<KB, false, false>(BatchArgs, cudaStream_t); \
  extern template cudaError_t launch_f3<KB, false, true>(BatchArgs, cudaStream_t);  \
  extern template cudaError_t launch_f3<KB, true, false>(BatchArgs, cudaStream_t);  \
  extern template cudaError_t launch_f3<KB, true, true>(BatchArgs, cudaStream_t);
CHF_DECL_F3(1) CHF_DECL_F3(2) CHF_DECL_F3(4) CHF_DECL_F3(8) CHF_DECL_F3(16)

}  // namespace chessfad

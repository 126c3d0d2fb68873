// chessfad/launch_functor.cuh -- host-side launch of the register-path kernel
// (hvp_reg_kernel, kernels.cuh) for any hDual<C> functor: used by the library's built-in
// functions (csrc/launch.cuh) and by user functions (chessfad_device.cuh).
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace chessfad {

#ifndef CHF_WARPS_REG
#define CHF_WARPS_REG 4  // measured vs 2 and 8: profiles/r01/warps/ (2: neutral but Ackley n = 64 +16%; 8: up to +35%)
#endif
constexpr int kWarpsReg = CHF_WARPS_REG;  // register path: 128 threads per CTA (2 CTAs/SM at <= 255 regs)

// groups of 32 points per CTA so that every warp of the CTA has a row to work on; the
// symmetric HVP gives every warp its own group (it walks all rows of its points)
#ifndef CHF_GROUP_ALL_MAXN
#define CHF_GROUP_ALL_MAXN 8  // warps own whole 32-point groups for n <= 8 (measured +5..23% at n = 4,
                                  // neutral at 8, -1..35% at n >= 16: profiles/r01/groups/)
#endif
inline int groups_for(int n, int warps, int mode) {
  if (mode == MODE_SYM_HVP || n <= CHF_GROUP_ALL_MAXN) return warps;
  int g = 1;
  while (g * 2 <= warps && n * g * 2 <= warps) g *= 2;
  return g;
}

inline size_t reg_smem_bytes(bool trig, int n, int G, int mode) {
  const int tiles = (mode_hess(mode) ? 1 : 3) + (trig ? 2 : 0);
  return (size_t)tiles * G * n * kPad * sizeof(double);
}

template <class K, class... Args>
inline cudaError_t launch_with_smem(K kernel, int grid, int block, size_t smem, cudaStream_t s, const Args&... args) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, block, smem, s>>>(args...);
  return cudaGetLastError();
}

// any functor F (built-in or user, see testfuncs.cuh), hDual<C> in registers
// NS > 0: the kernel compiled for n == NS (kernels.cuh); the caller guarantees a.n == NS
template <class F, int C, int MODE, int NS = 0>
cudaError_t launch_functor(const F& f, BatchArgs a, cudaStream_t s) {
  a.groups = groups_for(a.n, kWarpsReg, MODE);
  const int64_t P = 32 * a.groups;
  const int grid = (int)((a.m + P - 1) / P);
  return launch_with_smem(hvp_reg_kernel<F, C, MODE, kWarpsReg, NS>, grid, kWarpsReg * 32,
                          reg_smem_bytes(uses_trig2pi<F>::value, a.n, a.groups, MODE), s, a, f);
}

}  // namespace chessfad

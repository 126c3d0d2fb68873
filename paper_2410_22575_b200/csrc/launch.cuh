// launch.cuh -- host-side launchers for the kernel instantiations (one .cu per function
// family so that nvcc compiles them in parallel).  Used only by capi.cu.
#pragma once
#include <cuda_runtime.h>

#include "chessfad/launch_functor.cuh"
#include "f3_sparse.cuh"
#include "stream_small.cuh"
#include "f3_mma.cuh"

namespace chessfad {

inline bool f3_ab_smem(int n) { return n <= 32; }  // seed-sparse F3: (A, B) copied to shared memory

template <int FUNC, int C, int MODE>
cudaError_t launch_reg(BatchArgs a, cudaStream_t s) {
  return launch_functor<BuiltinFunc<FUNC>, C, MODE>(BuiltinFunc<FUNC>{}, a, s);
}
// the same kernel compiled for n == NS (kernels.cuh NS; inst_regn_*.cu)
template <int FUNC, int C, int MODE, int NS>
cudaError_t launch_reg_n(BatchArgs a, cudaStream_t s) {
  return launch_functor<BuiltinFunc<FUNC>, C, MODE, NS>(BuiltinFunc<FUNC>{}, a, s);
}
#define CHF_FOR_REGN_NS(X, F) X(F, 8) X(F, 16) X(F, 32)
#define CHF_FOR_REGN_C(X, F, NS) X(F, 1, NS) X(F, 2, NS) X(F, 4, NS) X(F, 8, NS) X(F, 16, NS)
#define CHF_FOR_REGN_MODE(X, F, C, NS) X(F, C, MODE_HVP, NS) X(F, C, MODE_HESS, NS) X(F, C, MODE_SYM_HVP, NS) \
  X(F, C, MODE_SYM_HESS, NS) X(F, C, MODE_HESS_GRAD, NS)
#define CHF_DECL_REGN2(F, C, M, NS) extern template cudaError_t launch_reg_n<F, C, M, NS>(BatchArgs, cudaStream_t);
#define CHF_DECL_REGN1(F, C, NS) CHF_FOR_REGN_MODE(CHF_DECL_REGN2, F, C, NS)
#define CHF_DECL_REGN0(F, NS) CHF_FOR_REGN_C(CHF_DECL_REGN1, F, NS)
CHF_FOR_REGN_NS(CHF_DECL_REGN0, FUNC_ROSENBROCK)
CHF_FOR_REGN_NS(CHF_DECL_REGN0, FUNC_ACKLEY)
CHF_FOR_REGN_NS(CHF_DECL_REGN0, FUNC_PRODSUM)
// n in {64, 128}: Alg 7 only (cfg3 / cfg5); the other modes run the runtime-n kernel there
#define CHF_FOR_REGN_BIG_NS(X, F) X(F, 64) X(F, 128)
#define CHF_DECL_REGNB1(F, C, NS) CHF_DECL_REGN2(F, C, MODE_HVP, NS)
#define CHF_DECL_REGNB0(F, NS) CHF_FOR_REGN_C(CHF_DECL_REGNB1, F, NS)
CHF_FOR_REGN_BIG_NS(CHF_DECL_REGNB0, FUNC_ROSENBROCK)
CHF_FOR_REGN_BIG_NS(CHF_DECL_REGNB0, FUNC_ACKLEY)
CHF_FOR_REGN_BIG_NS(CHF_DECL_REGNB0, FUNC_PRODSUM)

// NEXT-4 seed-sparse F3 HVP (f3_sparse.cuh): CB = column block, (A, B) in shared memory for
// n <= 32, else read from the caller's params; SLIM tiles for n > 32
inline bool f3_sp_slim(int n) { return n > 32; }
inline bool f3_sp_staged(int n) { return f3_sp_slim(n) && n % kSpKS == 0; }
inline size_t f3_sparse_smem_bytes(int n, int G) {
  const int tiles = f3_sp_slim(n) ? 3 : 5;
  const size_t ring = (size_t)(2 * kSpKS * 16 + kWarpsF3 * 2 * kSpKS) * 2 * sizeof(double);  // STAGED, CB <= 16
  return (size_t)tiles * G * n * kPad * sizeof(double) + (f3_ab_smem(n) ? (size_t)n * n * 2 * sizeof(double) : 0) +
         (f3_sp_staged(n) ? ring : 0);
}
template <int CB, int MODE>
cudaError_t launch_f3_sparse(BatchArgs a, cudaStream_t s) {
  a.groups = groups_for(a.n, kWarpsF3, MODE);  // Alg 8: every warp owns a group and walks all rows
  const int64_t P = 32 * a.groups;
  const int grid = (int)((a.m + P - 1) / P);
  const size_t smem = f3_sparse_smem_bytes(a.n, a.groups);
  if (f3_ab_smem(a.n)) return launch_with_smem(hvp_f3_sparse_kernel<CB, true, false, MODE, false>, grid, kWarpsF3 * 32, smem, s, a);
  return f3_sp_staged(a.n) ? launch_with_smem(hvp_f3_sparse_kernel<CB, false, true, MODE, true>, grid, kWarpsF3 * 32, smem, s, a)
                           : launch_with_smem(hvp_f3_sparse_kernel<CB, false, true, MODE, false>, grid, kWarpsF3 * 32, smem, s, a);
}
#define CHF_FOR_CB(X) X(1) X(2) X(4) X(8) X(16)
#define CHF_FOR_F3SP_MODE(X, CB) X(CB, MODE_HVP) X(CB, MODE_HESS) X(CB, MODE_SYM_HESS) X(CB, MODE_HESS_GRAD) \
  X(CB, MODE_SYM_HVP)
#define CHF_DECL_SP1(CB, M) extern template cudaError_t launch_f3_sparse<CB, M>(BatchArgs, cudaStream_t);
#define CHF_DECL_SP(CB) CHF_FOR_F3SP_MODE(CHF_DECL_SP1, CB)
CHF_FOR_CB(CHF_DECL_SP)

// hoisted HVP (NEXT-4) for n = NS in {2, 4, 8, 16}: thread per point, compile-time seeds
// Fused accumulate forms (R5) only where they measured faster on this path: Rosenbrock at
// n = 16, C >= 8 (0.31 vs 0.69 ms: fewer live registers, no spilling); elsewhere the plain
// forms let nvcc share more across the unrolled evaluations (profiles/r01/fused/).
constexpr bool small_fused(int FUNC, int C, int NS) { return FUNC == FUNC_ROSENBROCK && NS == 16 && C >= 8; }
template <int FUNC, int C, int NS>
cudaError_t launch_small(BatchArgs a, cudaStream_t s) {
  const int grid = (int)((a.m + 127) / 128);
  hvp_small_kernel<BuiltinFunc<FUNC>, C, NS, small_fused(FUNC, C, NS)><<<grid, 128, 0, s>>>(a, BuiltinFunc<FUNC>{});
  return cudaGetLastError();
}
#define CHF_FOR_SMALL(X, F) X(F, 1, 2) X(F, 2, 2) X(F, 1, 4) X(F, 2, 4) X(F, 4, 4) X(F, 1, 8) X(F, 2, 8) X(F, 4, 8) X(F, 8, 8) \
  X(F, 1, 16) X(F, 2, 16) X(F, 4, 16) X(F, 8, 16) X(F, 16, 16)
#define CHF_DECL_SMALL(F, C, NS) extern template cudaError_t launch_small<F, C, NS>(BatchArgs, cudaStream_t);
CHF_FOR_SMALL(CHF_DECL_SMALL, FUNC_ROSENBROCK)
CHF_FOR_SMALL(CHF_DECL_SMALL, FUNC_ACKLEY)
CHF_FOR_SMALL(CHF_DECL_SMALL, FUNC_PRODSUM)

// Alg 7 at n = NS in {2, 4, 8}: thread per point, persistent grid, bulk-copy ring
// (stream_small.cuh).  Grid = min(tiles, SMs x resident CTAs), resident CTAs queried once.
// compile-time chunk start (reading R8) where the kernel is FP64-bound; the HBM-bound corners
// (Rosenbrock / prodsum at n = 2, prodsum at n = 4) measured faster with it read per evaluation
// (profiles/r02/stream_fold/summary.txt)
constexpr bool stream_fold_cs(int FUNC, int NS) {
  return !((NS == 2 && FUNC != FUNC_ACKLEY) || (NS == 4 && FUNC == FUNC_PRODSUM));
}
template <int FUNC, int C, int NS>
cudaError_t launch_stream(BatchArgs a, cudaStream_t s) {
  auto kern = hvp_stream_kernel<BuiltinFunc<FUNC>, C, NS, stream_fold_cs(FUNC, NS)>;
  constexpr size_t smem = StreamCfg<NS>::kSmem;
  static int occ = 0;
  cudaError_t e;
  if (occ == 0) {
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStreamTP, smem)) != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const int64_t tiles = (a.m + kStreamTP - 1) / kStreamTP;
  const int grid = (int)(tiles < (int64_t)sms * occ ? tiles : (int64_t)sms * occ);
  kern<<<grid, kStreamTP, smem, s>>>(a, BuiltinFunc<FUNC>{});
  return cudaGetLastError();
}
#define CHF_FOR_STREAM(X, F) X(F, 1, 2) X(F, 2, 2) X(F, 1, 4) X(F, 2, 4) X(F, 4, 4) X(F, 1, 8) X(F, 2, 8) X(F, 4, 8) X(F, 8, 8)
#define CHF_DECL_STREAM(F, C, NS) extern template cudaError_t launch_stream<F, C, NS>(BatchArgs, cudaStream_t);
CHF_FOR_STREAM(CHF_DECL_STREAM, FUNC_ROSENBROCK)
CHF_FOR_STREAM(CHF_DECL_STREAM, FUNC_ACKLEY)
CHF_FOR_STREAM(CHF_DECL_STREAM, FUNC_PRODSUM)

// F3 with the E-sums on the FP64 tensor core (f3_mma.cuh): n <= NN (zero-padded), NN = 8 ceil(n / 8)
template <int NN, int MODE>
cudaError_t launch_f3_mma(BatchArgs a, cudaStream_t s) {
  using Cfg = F3Mma<NN, MODE>;
  const int grid = (int)((a.m + Cfg::P - 1) / Cfg::P);
  return launch_with_smem(hvp_f3_mma_kernel<NN, MODE>, grid, Cfg::W * 32, Cfg::smem_bytes(), s, a);
}
#define CHF_FOR_MMA_MODE(X, NN) X(NN, MODE_HVP) X(NN, MODE_HESS) X(NN, MODE_SYM_HVP) X(NN, MODE_SYM_HESS) \
  X(NN, MODE_HESS_GRAD) X(NN, MODE_HVP_ROWHOIST)
#define CHF_FOR_MMA_NN(X) X(8) X(16) X(24) X(32) X(40) X(48) X(56) X(64) X(72) X(80) X(88) X(96) X(104) X(112) \
  X(120) X(128)
#define CHF_DECL_MMA1(NN, M) extern template cudaError_t launch_f3_mma<NN, M>(BatchArgs, cudaStream_t);
#define CHF_DECL_MMA(NN) CHF_FOR_MMA_MODE(CHF_DECL_MMA1, NN)
CHF_FOR_MMA_NN(CHF_DECL_MMA)

// explicit-instantiation declarations (definitions in inst_*.cu)
#define CHF_FOR_MODE(X, A, B) \
  X(A, B, MODE_HVP) X(A, B, MODE_HESS) X(A, B, MODE_SYM_HVP) X(A, B, MODE_SYM_HESS) X(A, B, MODE_HESS_GRAD)
#define CHF_DECL_REG1(F, C, M) extern template cudaError_t launch_reg<F, C, M>(BatchArgs, cudaStream_t);
#define CHF_DECL_REG(F, C) CHF_FOR_MODE(CHF_DECL_REG1, F, C)
#define CHF_FOR_C(X, F) X(F, 1) X(F, 2) X(F, 4) X(F, 8) X(F, 16)
CHF_FOR_C(CHF_DECL_REG, FUNC_ROSENBROCK)
CHF_FOR_C(CHF_DECL_REG, FUNC_ACKLEY)
CHF_FOR_C(CHF_DECL_REG, FUNC_PRODSUM)

// NEXT-4 seed sparsity for F1/F2/F4 (testfuncs.cuh SparseFunc), HVP and Hessian
template <int FUNC, int C, int MODE>
cudaError_t launch_sparse_reg(BatchArgs a, cudaStream_t s) {
  return launch_functor<SparseFunc<FUNC>, C, MODE>(SparseFunc<FUNC>{}, a, s);
}
#define CHF_FOR_SP_MODE(X, F, C) X(F, C, MODE_HVP) X(F, C, MODE_HESS) X(F, C, MODE_SYM_HVP) X(F, C, MODE_SYM_HESS) \
  X(F, C, MODE_HESS_GRAD)
#define CHF_DECL_SPR2(F, C, M) extern template cudaError_t launch_sparse_reg<F, C, M>(BatchArgs, cudaStream_t);
#define CHF_DECL_SPR1(F, C) CHF_FOR_SP_MODE(CHF_DECL_SPR2, F, C)
CHF_FOR_C(CHF_DECL_SPR1, FUNC_ROSENBROCK)
CHF_FOR_C(CHF_DECL_SPR1, FUNC_ACKLEY)
CHF_FOR_C(CHF_DECL_SPR1, FUNC_PRODSUM)


}  // namespace chessfad

// paper_l2.cu -- the paper's own GPU designs, Alg 9 "L0", Alg 10 "L1"
// (:459-482) and Fig. 2 "L2" (:485-524), recompiled for sm_100a as MEASURED COMPARISON
// POINTS (not the product path).  L0: one thread per instance, rows and chunks looped in the
// thread; L1: one thread per (instance, row), chunks looped; both re-seed the materialised
// y[NV] per evaluation (:446, :472) and write out once per row (reading G7).
//
// As printed: one thread per (instance, row i, chunk j); NETBLK instances per block of
// NV*NCHUNK threads each; every thread materialises its seed array `hDual<C> y[NV]` with
// INITIALIZE/CHUNK-INIT, evaluates f, dots its chunk with vec straight from
// global memory (:501-505), stores the partial in shared memory sprod[local_eid][i][j],
// __syncthreads(), and threads tid < NV sum their row's NCHUNK partials in ascending k and
// store z[tid + eid*NV] (:506-518).  Reading G5 of DESIGN.md for the lost '%' expressions.
// The test-function bodies are the same canonical forms as the product (testfuncs.cuh),
// fed from the materialised array instead of on-the-fly seeds.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/chessfad.h"
#include "chessfad/testfuncs.cuh"

namespace chessfad {
namespace {

template <int C, int NV>
struct ArraySeed {  // y(k) reads the thread's materialised hDual<C> y[NV]
  static constexpr bool kStatic = false;
  static constexpr bool kFused = false;  // the paper's design: canonical forms as written
  const hd<C>* y;
  const double* sin2pi = nullptr;  // (unused: built-in Ackley is not offered here)
  const double* cos2pi = nullptr;
  int stride = 0;
  CHF_INL hd<C> operator()(int k) const { return y[k]; }
};

template <int FUNC, int NV, int C, int NETBLK>
__global__ void __launch_bounds__(NETBLK * NV * (NV / C)) paper_l2_kernel(int64_t m, const double* __restrict__ x,
                                                                         const double* __restrict__ vec,
                                                                         double* __restrict__ z) {
  constexpr int NCHUNK = NV / C;
  __shared__ double sprod[NETBLK][NV][NCHUNK];
  const int local_eid = threadIdx.x / (NV * NCHUNK);
  const int64_t eid = (int64_t)NETBLK * blockIdx.x + local_eid;
  const int tid = threadIdx.x % (NV * NCHUNK);
  const int i = tid / NCHUNK;
  const int j = tid % NCHUNK;
  const int64_t e = eid < m ? eid : m - 1;
  // INITIALIZE / CHUNK-INIT (Alg 4) into the per-thread array
  hd<C> y[NV];
  for (int k = 0; k < NV; k++) {
    y[k].v[0] = x[e * NV + k];
    y[k].v[1] = (k == i) ? 1.0 : 0.0;
    for (int l = 0; l < C; l++) y[k].v[2 + l] = (k - j * C == l) ? 1.0 : 0.0;
    for (int l = 0; l < C; l++) y[k].v[C + 2 + l] = 0.0;
  }
  const hd<C> temp1 = eval_f<FUNC, C>(NV, ArraySeed<C, NV>{y});
  const int chunkstart = j * C;
  double res = 0.0;
  for (int l = C + 2; l <= 2 * C + 1; l++) res = res + temp1.v[l] * vec[e * NV + chunkstart + l - C - 2];
  sprod[local_eid][i][j] = res;  // save partial results in shared memory
  __syncthreads();
  if (tid < NV) {  // accumulate results in the shared memory
    double r = 0.0;
    for (int k = 0; k < NCHUNK; k++) r = r + sprod[local_eid][tid][k];
    if (eid < m) z[tid + eid * NV] = r;
  }
}

// L0 (LEVEL 0) and L1 (LEVEL 1): 256-thread blocks, id = blockIdx.x * blockDim.x + threadIdx.x
template <int FUNC, int NV, int C, int LEVEL>
__global__ void __launch_bounds__(256) paper_l01_kernel(int64_t m, const double* __restrict__ x,
                                                        const double* __restrict__ vec, double* __restrict__ out) {
  constexpr int NCHUNK = NV / C;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t eid = LEVEL == 0 ? id : id / NV;
  if (eid >= m) return;
  const int i0 = LEVEL == 0 ? 0 : (int)(id % NV);
  const int i1 = LEVEL == 0 ? NV : i0 + 1;
  hd<C> y[NV];
  for (int i = i0; i < i1; i++) {
    double res = 0.0;
    for (int j = 0; j < NCHUNK; j++) {
      const int cstart = j * C;
      for (int k = 0; k < NV; k++) {  // CHUNK-INIT(y, &a[eid*n], n, i, j, csize)
        y[k].v[0] = x[eid * NV + k];
        y[k].v[1] = (k == i) ? 1.0 : 0.0;
        for (int l = 0; l < C; l++) y[k].v[2 + l] = (k - cstart == l) ? 1.0 : 0.0;
        for (int l = 0; l < C; l++) y[k].v[C + 2 + l] = 0.0;
      }
      const hd<C> temp = eval_f<FUNC, C>(NV, ArraySeed<C, NV>{y});
      for (int l = 0; l < C; l++) res = res + temp.v[C + 2 + l] * vec[eid * NV + cstart + l];
    }
    out[eid * NV + i] = res;
  }
}

template <int FUNC, int NV, int C, int LEVEL>
cudaError_t launch_l01(int64_t m, const double* x, const double* v, double* z, cudaStream_t s) {
  const int64_t threads = LEVEL == 0 ? m : m * NV;
  paper_l01_kernel<FUNC, NV, C, LEVEL><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(m, x, v, z);
  return cudaGetLastError();
}

template <int FUNC, int NV, int C>
cudaError_t launch_l2(int64_t m, const double* x, const double* v, double* z, cudaStream_t s) {
  constexpr int THREADS_PER_INSTANCE = NV * (NV / C);
  constexpr int NETBLK = THREADS_PER_INSTANCE >= 256 ? 1 : 256 / THREADS_PER_INSTANCE;  // G22: free knob
  const int64_t grid = (m + NETBLK - 1) / NETBLK;
  paper_l2_kernel<FUNC, NV, C, NETBLK><<<(unsigned)grid, NETBLK * THREADS_PER_INSTANCE, 0, s>>>(m, x, v, z);
  return cudaGetLastError();
}

template <int FUNC, int NV, int C>
cudaError_t launch_level(int level, int64_t m, const double* x, const double* v, double* z, cudaStream_t s) {
  switch (level) {
    case 0: return launch_l01<FUNC, NV, C, 0>(m, x, v, z, s);
    case 1: return launch_l01<FUNC, NV, C, 1>(m, x, v, z, s);
    case 2: return launch_l2<FUNC, NV, C>(m, x, v, z, s);
  }
  return cudaErrorInvalidValue;
}

template <int FUNC, int NV>
cudaError_t dispatch_c(int level, int C, int64_t m, const double* x, const double* v, double* z, cudaStream_t s) {
  switch (C) {
    case 1: return launch_level<FUNC, NV, 1>(level, m, x, v, z, s);
    case 2: return launch_level<FUNC, NV, 2>(level, m, x, v, z, s);
    case 4: if constexpr (NV >= 4) return launch_level<FUNC, NV, 4>(level, m, x, v, z, s); break;
    case 8: if constexpr (NV >= 8) return launch_level<FUNC, NV, 8>(level, m, x, v, z, s); break;
    case 16: if constexpr (NV >= 16) return launch_level<FUNC, NV, 16>(level, m, x, v, z, s); break;
  }
  return cudaErrorInvalidValue;
}

template <int FUNC>
cudaError_t dispatch_n(int level, int n, int C, int64_t m, const double* x, const double* v, double* z,
                       cudaStream_t s) {
  switch (n) {
    case 2: return dispatch_c<FUNC, 2>(level, C, m, x, v, z, s);
    case 4: return dispatch_c<FUNC, 4>(level, C, m, x, v, z, s);
    case 8: return dispatch_c<FUNC, 8>(level, C, m, x, v, z, s);
    case 16: return dispatch_c<FUNC, 16>(level, C, m, x, v, z, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace
}  // namespace chessfad

extern "C" int chessfad_hvp_batch_paper(int level, int func, int n, int csize, int64_t m, const double* points,
                                        const double* vecs, double* out, void* stream) {
  using namespace chessfad;
  if (level < 0 || level > 2 || n < 1 || m < 0) return CHESSFAD_ERR_ARG;
  if (m > 0 && (!points || !vecs || !out)) return CHESSFAD_ERR_ARG;
  if (csize < 1 || csize > n || n % csize) return CHESSFAD_ERR_CHUNK;
  if ((func != CHESSFAD_ROSENBROCK && func != CHESSFAD_PRODSUM) || n < 2) return CHESSFAD_ERR_UNSUPPORTED;
  if (!(n == 2 || n == 4 || n == 8 || n == 16) || csize > 16) return CHESSFAD_ERR_UNSUPPORTED;
  if (m == 0) return CHESSFAD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const cudaError_t e = func == CHESSFAD_ROSENBROCK
                            ? dispatch_n<FUNC_ROSENBROCK>(level, n, csize, m, points, vecs, out, s)
                            : dispatch_n<FUNC_PRODSUM>(level, n, csize, m, points, vecs, out, s);
  return e == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
}

extern "C" int chessfad_hvp_batch_paper_l2(int func, int n, int csize, int64_t m, const double* points,
                                           const double* vecs, double* out, void* stream) {
  return chessfad_hvp_batch_paper(2, func, n, csize, m, points, vecs, out, stream);
}

// chessfad_device.cuh -- header-only C++/CUDA API for USER-DEFINED functions (SURVEY §8(f)
// NEXT-3; the paper's library takes "a templated function on the data type", PAPER.md:16,
// and is templated on csize).  Compile with
//     nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I<repo>/include ...
//
// A user function is a functor
//     struct F {
//       template <int C, class Seed>
//       __device__ chessfad::hd<C> operator()(int n, const Seed& y) const;   // y(k): variable k
//     };
// written with the overloaded hDual<C> arithmetic (+ - * / with hDual or double operands,
// sin cos exp sqrt log abs, comparisons on the value slot) of hdual.cuh (Fig. 1 rules,
// PAPER.md:263-344).  y(k) returns the CHUNK-INIT seed of variable k (Alg 4) built on the fly,
// as a seed-shaped chessfad::hs<C> (second-order slots structural zeros; every rule accepts it
// and `hd<C> x = y(k);` converts it -- `auto x = y(k);` keeps the cheaper form, R7).
// The functor runs inside the same lane=point / warp=row kernels as the built-in functions,
// so the batched HVP (Alg 7), Hessian (Alg 5) and their symmetric variants (Alg 8, Alg 6)
// are all available for it.  The functor object is passed by value as a kernel argument
// (it may carry parameters, <= a few KB).
//
// All pointers are DEVICE pointers with the layouts of chessfad.h; calls are asynchronous
// on `stream`; the return value is the cudaError_t of the launch (cudaErrorInvalidValue for
// bad arguments: n < 1, m < 0, C does not divide n, n > 256, or shared memory too small).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "chessfad/launch_functor.cuh"  // self-contained: include/ only

namespace chessfad {

enum UserAlgo {
  USER_HVP = MODE_HVP,
  USER_HESSIAN = MODE_HESS,
  USER_SYM_HVP = MODE_SYM_HVP,
  USER_SYM_HESSIAN = MODE_SYM_HESS,
  USER_HESSIAN_GRAD = MODE_HESS_GRAD
};

template <int C, int ALGO, class F>
inline cudaError_t user_batch(const F& f, int n, int64_t m, const double* points, const double* vecs, double* out,
                              cudaStream_t stream, double* grad = nullptr) {
  if (n < 1 || m < 0 || C < 1 || C > n || n % C != 0 || n > 256) return cudaErrorInvalidValue;
  if (m == 0) return cudaSuccess;
  if (!points || !out || (!mode_hess(ALGO) && !vecs) || (ALGO == USER_HESSIAN_GRAD && !grad))
    return cudaErrorInvalidValue;
  if (reg_smem_bytes(uses_trig2pi<F>::value, n, groups_for(n, kWarpsReg, ALGO), ALGO) > 227 * 1024)
    return cudaErrorInvalidValue;
  BatchArgs a;
  a.n = n;
  a.csize = C;
  a.groups = 1;
  a.m = m;
  a.points = points;
  a.vecs = vecs;
  a.out = out;
  a.params = nullptr;
  a.grad = grad;
  return launch_functor<F, C, ALGO>(f, a, stream);
}

// The same kernels compiled for n == NS (reading R8; the paper's NV-templated kernels):
// the functor's loops over the variables see a compile-time n, so nvcc can unroll them and fold
// the seed's constant chunk slots; rows and chunks stay runtime loops (every evaluation is
// executed on its own).  n must equal NS (cudaErrorInvalidValue otherwise).
template <int NS, int C, int ALGO, class F>
inline cudaError_t user_batch_n(const F& f, int n, int64_t m, const double* points, const double* vecs, double* out,
                                cudaStream_t stream, double* grad = nullptr) {
  static_assert(NS >= 1 && C >= 1 && NS % C == 0, "C must divide NS");
  if (n != NS) return cudaErrorInvalidValue;
  if (m < 0 || NS > 256) return cudaErrorInvalidValue;
  if (m == 0) return cudaSuccess;
  if (!points || !out || (!mode_hess(ALGO) && !vecs) || (ALGO == USER_HESSIAN_GRAD && !grad))
    return cudaErrorInvalidValue;
  if (reg_smem_bytes(uses_trig2pi<F>::value, n, groups_for(n, kWarpsReg, ALGO), ALGO) > 227 * 1024)
    return cudaErrorInvalidValue;
  BatchArgs a;
  a.n = n;
  a.csize = C;
  a.groups = 1;
  a.m = m;
  a.points = points;
  a.vecs = vecs;
  a.out = out;
  a.params = nullptr;
  a.grad = grad;
  return launch_functor<F, C, ALGO, NS>(f, a, stream);
}

// out[e*n+i] = sum_j d2f/dx_i dx_j (points[e]) vecs[e*n+j]     (Alg 7; USER_SYM_HVP: Alg 8)
template <int C, class F>
inline cudaError_t user_hvp_batch(const F& f, int n, int64_t m, const double* points, const double* vecs,
                                  double* out, cudaStream_t stream, bool symmetric = false) {
  return symmetric ? user_batch<C, USER_SYM_HVP>(f, n, m, points, vecs, out, stream)
                   : user_batch<C, USER_HVP>(f, n, m, points, vecs, out, stream);
}

// hess[e*n*n + i*n + j] = d2f/dx_i dx_j (points[e])              (Alg 5; symmetric: Alg 6)
template <int C, class F>
inline cudaError_t user_hessian_batch(const F& f, int n, int64_t m, const double* points, double* hess,
                                      cudaStream_t stream, bool symmetric = false) {
  return symmetric ? user_batch<C, USER_SYM_HESSIAN>(f, n, m, points, nullptr, hess, stream)
                   : user_batch<C, USER_HESSIAN>(f, n, m, points, nullptr, hess, stream);
}

// hess as above plus grad[e*n+i] = df/dx_i (points[e])                 (Alg 5 + PAPER.md:252)
template <int C, class F>
inline cudaError_t user_hessian_grad_batch(const F& f, int n, int64_t m, const double* points, double* hess,
                                           double* grad, cudaStream_t stream) {
  return user_batch<C, USER_HESSIAN_GRAD>(f, n, m, points, nullptr, hess, stream, grad);
}

}  // namespace chessfad

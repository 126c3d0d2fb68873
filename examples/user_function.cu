// examples/user_function.cu -- a user-defined function through the header-only device API
// (include/chessfad_device.cuh).  Built by tests/test_gpu_user_function.py into a small .so:
//     nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -Xcompiler -fPIC -shared \
//          -I include examples/user_function.cu -o <out>.so
//
//   f(y) = sum_i [ cos(y_i) + y_i / (1 + y_i^2) ] + sum_{i<n-1} y_i^2 y_{i+1}
// (exercises hDual division, unary cos, mixed scalar ops and products).
#include "chessfad_device.cuh"

struct UserF {
  template <int C, class Seed>
  __device__ chessfad::hd<C> operator()(int n, const Seed& y) const {
    using namespace chessfad;
    hd<C> s;
    {
      const hd<C> y0 = y(0);
      s = cos(y0) + y0 / (1.0 + y0 * y0);
    }
    for (int i = 1; i < n; i++) {
      const auto yi = y(i);
      s = s + (cos(yi) + yi / (1.0 + yi * yi));
    }
    for (int i = 0; i < n - 1; i++) {
      const auto a = y(i);
      s = s + a * a * y(i + 1);
    }
    return s;
  }
};

// C-ABI shims for the test (algo: 0 HVP, 1 Hessian, 2 symmetric HVP, 3 symmetric Hessian)
extern "C" int user_batch(int algo, int n, int csize, long long m, const double* points, const double* vecs,
                          double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
#define CASE(C)                                                                                  \
  case C:                                                                                        \
    switch (algo) {                                                                              \
      case 0: return (int)chessfad::user_hvp_batch<C>(UserF{}, n, m, points, vecs, out, s);        \
      case 1: return (int)chessfad::user_hessian_batch<C>(UserF{}, n, m, points, out, s);          \
      case 2: return (int)chessfad::user_hvp_batch<C>(UserF{}, n, m, points, vecs, out, s, true);  \
      case 3: return (int)chessfad::user_hessian_batch<C>(UserF{}, n, m, points, out, s, true);    \
    }                                                                                            \
    return -1;
  switch (csize) { CASE(1) CASE(4) CASE(8) }
#undef CASE
  return -2;
}

// the same function through the kernels compiled for n = 16 (chessfad::user_batch_n, reading R8)
extern "C" int user_batch_n16(int algo, int csize, long long m, const double* points, const double* vecs,
                              double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  using namespace chessfad;
#define CASE_N(C)                                                                                          \
  case C:                                                                                                  \
    switch (algo) {                                                                                        \
      case 0: return (int)user_batch_n<16, C, USER_HVP>(UserF{}, 16, m, points, vecs, out, s);             \
      case 1: return (int)user_batch_n<16, C, USER_HESSIAN>(UserF{}, 16, m, points, nullptr, out, s);      \
      case 2: return (int)user_batch_n<16, C, USER_SYM_HVP>(UserF{}, 16, m, points, vecs, out, s);         \
      case 3: return (int)user_batch_n<16, C, USER_SYM_HESSIAN>(UserF{}, 16, m, points, nullptr, out, s);  \
    }                                                                                                      \
    return -1;
  switch (csize) { CASE_N(1) CASE_N(4) CASE_N(16) }
#undef CASE_N
  return -2;
}

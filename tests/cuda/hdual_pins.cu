// tests/cuda/hdual_pins.cu -- TEST KERNEL: the device hDual<C> rules of include/chessfad/hdual.cuh
// and the device CHUNK-INIT seed (LaneSeed, include/chessfad/testfuncs.cuh) applied to the SPEC
// worked examples (tests/golden/spec_hdual_examples.json) on the GPU, one thread.  Built by
// tests/test_gpu_hdual_pins.py with nvcc into a small .so; nothing here is product code.
#include <cuda_runtime.h>

#include <type_traits>

#include "chessfad/testfuncs.cuh"

using namespace chessfad;

enum { OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_SADD, OP_ADDS, OP_SSUB, OP_SUBS, OP_SMUL, OP_DIVS, OP_NEG,
       OP_SIN, OP_COS, OP_EXP, OP_SQRT, OP_LOG, OP_ABS, OP_LT, OP_GT, OP_LE, OP_GE, OP_SDIV };

template <int C>
__global__ void op_kernel(int op, const double* u_, const double* v_, double c, double* out) {
  hd<C> u, v, r;
  for (int s = 0; s < hd<C>::N; s++) {
    u.v[s] = u_[s];
    v.v[s] = v_[s];
    r.v[s] = 0.0;
  }
  switch (op) {
    case OP_ADD: r = u + v; break;
    case OP_SUB: r = u - v; break;
    case OP_MUL: r = u * v; break;
    case OP_DIV: r = u / v; break;
    case OP_SADD: r = c + u; break;
    case OP_ADDS: r = u + c; break;
    case OP_SSUB: r = c - u; break;
    case OP_SUBS: r = u - c; break;
    case OP_SMUL: r = c * u; break;
    case OP_DIVS: r = u / c; break;
    case OP_SDIV: r = c / u; break;
    case OP_NEG: r = -u; break;
    case OP_SIN: r = sin(u); break;
    case OP_COS: r = cos(u); break;
    case OP_EXP: r = exp(u); break;
    case OP_SQRT: r = sqrt(u); break;
    case OP_LOG: r = log(u); break;
    case OP_ABS: r = abs(u); break;
    case OP_LT: r.v[0] = (u < v) ? 1.0 : 0.0; break;
    case OP_GT: r.v[0] = (u > v) ? 1.0 : 0.0; break;
    case OP_LE: r.v[0] = (u <= v) ? 1.0 : 0.0; break;
    case OP_GE: r.v[0] = (u >= v) ? 1.0 : 0.0; break;
  }
  for (int s = 0; s < hd<C>::N; s++) out[s] = r.v[s];
}

// Reading R7: every rule with seed-shaped operands (hs<C>: second-order slots
// structural zeros) against the same rule on the operands converted to full hd<C>.  Mode bits:
// 1 = u seed-shaped, 2 = v seed-shaped, 4 = acc seed-shaped.  out[0..N) typed, out[N..2N) full.
enum { SS_ADD, SS_SUB, SS_MUL, SS_DIV, SS_FMA, SS_FNMA, SS_AXPY, SS_SIN, SS_EXP, SS_SQRT, SS_UACC, SS_SMUL, SS_CSUB };
template <int C, class U, class V, class A>
__device__ void ss_apply(int op, const U& u, const V& v, const A& acc, double c, double* out) {
  hd<C> r;
  switch (op) {
    case SS_ADD: r = u + v; break;
    case SS_SUB: r = u - v; break;
    case SS_MUL: r = u * v; break;
    case SS_DIV: r = u / v; break;
    case SS_FMA: r = hd_fma(u, v, acc); break;
    case SS_FNMA: r = hd_fnma(u, v, acc); break;
    case SS_AXPY: r = hd_axpy(c, u, acc); break;
    case SS_SIN: r = sin(u); break;
    case SS_EXP: r = exp(u); break;
    case SS_SQRT: r = sqrt(u); break;
    case SS_UACC: r = hd_unary_acc(u, 0.3, -0.7, 1.9, acc); break;
    case SS_SMUL: r = c * u; break;
    case SS_CSUB: r = c - u; break;
  }
  for (int q = 0; q < hd<C>::N; q++) out[q] = r.v[q];
}
template <int C, bool SU, bool SV, bool SA>
__device__ void ss_run(int op, const double* u_, const double* v_, const double* a_, double c, double* out) {
  using U = std::conditional_t<SU, hs<C>, hd<C>>;
  using V = std::conditional_t<SV, hs<C>, hd<C>>;
  using A = std::conditional_t<SA, hs<C>, hd<C>>;
  U u;
  V v;
  A a;
  hd<C> fu, fv, fa;
  for (int q = 0; q < hd<C>::N; q++) {
    const bool second = q >= C + 2;
    fu.v[q] = (SU && second) ? 0.0 : u_[q];
    fv.v[q] = (SV && second) ? 0.0 : v_[q];
    fa.v[q] = (SA && second) ? 0.0 : a_[q];
    if (q < U::N) u.v[q] = u_[q];
    if (q < V::N) v.v[q] = v_[q];
    if (q < A::N) a.v[q] = a_[q];
  }
  ss_apply<C>(op, u, v, a, c, out);
  ss_apply<C>(op, fu, fv, fa, c, out + hd<C>::N);
}
template <int C>
__global__ void seedshape_kernel(int op, int mode, const double* u, const double* v, const double* a, double c,
                                 double* out) {
  switch (mode) {
    case 0: ss_run<C, false, false, false>(op, u, v, a, c, out); break;
    case 1: ss_run<C, true, false, false>(op, u, v, a, c, out); break;
    case 2: ss_run<C, false, true, false>(op, u, v, a, c, out); break;
    case 3: ss_run<C, true, true, false>(op, u, v, a, c, out); break;
    case 4: ss_run<C, false, false, true>(op, u, v, a, c, out); break;
    case 5: ss_run<C, true, false, true>(op, u, v, a, c, out); break;
    case 6: ss_run<C, false, true, true>(op, u, v, a, c, out); break;
    case 7: ss_run<C, true, true, true>(op, u, v, a, c, out); break;
  }
}

// CHUNK-INIT seeds of all n variables (Alg 4) from the device seed generator
template <int C>
__global__ void seed_kernel(int n, const double* a, int i, int cs, double* out) {
  const LaneSeed<C> y{a, 1, i, cs, nullptr, nullptr};
  for (int k = 0; k < n; k++) {
    const hd<C> s = y(k);
    for (int q = 0; q < hd<C>::N; q++) out[k * hd<C>::N + q] = s.v[q];
  }
}

static int run(void (*launch)(double*, double*, double*), const double* u, const double* v, int nin, double* out,
               int nout) {
  double *du, *dv, *dout;
  if (cudaMalloc(&du, 64 * sizeof(double)) || cudaMalloc(&dv, 64 * sizeof(double)) ||
      cudaMalloc(&dout, 256 * sizeof(double)))
    return 1;
  cudaMemcpy(du, u, nin * sizeof(double), cudaMemcpyHostToDevice);
  if (v) cudaMemcpy(dv, v, nin * sizeof(double), cudaMemcpyHostToDevice);
  launch(du, dv, dout);
  const int err = cudaDeviceSynchronize() != cudaSuccess;
  cudaMemcpy(out, dout, nout * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(du);
  cudaFree(dv);
  cudaFree(dout);
  return err;
}

extern "C" int dev_hd_op(int op, int C, const double* u, const double* v, double c, double* out) {
  const int N = 2 * C + 2;
  static int s_op;
  static double s_c;
  s_op = op;
  s_c = c;
  double zero[64] = {0};
  if (C == 1)
    return run([](double* a, double* b, double* o) { op_kernel<1><<<1, 1>>>(s_op, a, b, s_c, o); }, u, v ? v : zero,
               N, out, N);
  if (C == 2)
    return run([](double* a, double* b, double* o) { op_kernel<2><<<1, 1>>>(s_op, a, b, s_c, o); }, u, v ? v : zero,
               N, out, N);
  return 2;
}

extern "C" int dev_chunk_init(int n, int C, const double* a, int i, int cs, double* out) {
  static int s_n, s_i, s_cs;
  s_n = n;
  s_i = i;
  s_cs = cs;
  if (C == 1)
    return run([](double* x, double*, double* o) { seed_kernel<1><<<1, 1>>>(s_n, x, s_i, s_cs, o); }, a, nullptr, n,
               out, n * 4);
  if (C == 2)
    return run([](double* x, double*, double* o) { seed_kernel<2><<<1, 1>>>(s_n, x, s_i, s_cs, o); }, a, nullptr, n,
               out, n * 6);
  return 2;
}

// three operands of 2C+2 slots each packed in `in` (u | v | acc); out: typed | full
extern "C" int dev_seedshape(int op, int mode, int C, const double* in, double c, double* out) {
  static int s_op, s_mode;
  static double s_c;
  s_op = op;
  s_mode = mode;
  s_c = c;
  double* d;
  if (cudaMalloc(&d, 256 * sizeof(double))) return 1;
  const int N = 2 * C + 2;
  cudaMemcpy(d, in, 3 * N * sizeof(double), cudaMemcpyHostToDevice);
  if (C == 2) seedshape_kernel<2><<<1, 1>>>(s_op, s_mode, d, d + N, d + 2 * N, s_c, d + 3 * N);
  else if (C == 4) seedshape_kernel<4><<<1, 1>>>(s_op, s_mode, d, d + N, d + 2 * N, s_c, d + 3 * N);
  else return 2;
  const int err = cudaDeviceSynchronize() != cudaSuccess;
  cudaMemcpy(out, d + 3 * N, 2 * N * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return err;
}

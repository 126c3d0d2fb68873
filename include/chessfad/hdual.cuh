// hdual.cuh -- the chunked second-order dual number hDual<C> on the device (sm_100a).
//
// Layout (§IV "CHESSFAD Library Implementation"):
//   v[0]            f
//   v[1]            df/dx_i              (the active Hessian row i)
//   v[2 .. C+1]     df/dx_{cs .. cs+C-1} (the active chunk of columns)
//   v[C+2 .. 2C+1]  d2f/dx_i dx_{cs..}   (one chunk of row i of the Hessian)
// A hDual<C> is 2C+2 doubles = 4C+4 registers; it lives in registers, never in memory.
//
// Rules; FMA contraction is left to nvcc (--fmad=true, G14):
//   hh+ / hh-  componentwise                                 PAPER.md:97, Fig. 1 :276-280
//   hh*        r0 = u0 v0; r[k] = u0 v[k] + v0 u[k] (k=1..C+1);
//              r[C+k] = u0 v[C+k] + u1 v[k] + v1 u[k] + v0 u[C+k]   PAPER.md:98, Fig. 1 :302-321
//   s+ / s-    value slot only (c - u negates the derivative slots)  Fig. 1 :282-300
//   s*         every slot scaled                             Fig. 1 :323-338
//   unary g    r0 = g(u0); r[k] = g' u[k]; r[C+k] = g' u[C+k] + (g'' u1) u[k]
//              (sin printed at PAPER.md:99; general chain rule)
// The term order of hh* is the Fig. 1 order so that an FMA-free build would reproduce the
// paper's rounding; the GPU differs from the oracle only by contraction.
#pragma once
#include <cuda_runtime.h>

namespace chessfad {

#define CHF_INL __device__ __forceinline__

template <int C>
struct hd {
  static constexpr int N = 2 * C + 2;
  double v[N];
};

template <int C>
CHF_INL hd<C> operator+(const hd<C>& a, const hd<C>& b) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = a.v[s] + b.v[s];
  return r;
}

template <int C>
CHF_INL hd<C> operator-(const hd<C>& a, const hd<C>& b) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = a.v[s] - b.v[s];
  return r;
}

template <int C>
CHF_INL hd<C> operator-(const hd<C>& a) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = -a.v[s];
  return r;
}

template <int C>
CHF_INL hd<C> operator*(const hd<C>& u, const hd<C>& v) {
  hd<C> r;
  r.v[0] = u.v[0] * v.v[0];
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = u.v[0] * v.v[i] + v.v[0] * u.v[i];
#pragma unroll
  for (int j = 2; j <= C + 1; j++)
    r.v[C + j] = u.v[0] * v.v[C + j] + u.v[1] * v.v[j] + v.v[1] * u.v[j] + v.v[0] * u.v[C + j];
  return r;
}

// Fused accumulate forms (reading R5): acc + u*v, acc - u*v, acc + c*u with every
// term of the product added onto the running sum one at a time, in the Fig. 1 term order,
// as one DFMA each.  Per slot these are exactly the multiplications and additions of one
// hh* (or s*) plus one hh+ (model FLOPs unchanged: 6C+3 mul + 4C+1 add + 2C+2 add =
// 6C+3 FMAs); only the association of the sum differs from `acc + (u*v)`, i.e. the
// reduction order of the sum being accumulated.  Used by the built-in test functions
// (testfuncs.cuh) for their running sums; the plain operators above are unchanged.
template <int C>
CHF_INL hd<C> hd_fma(const hd<C>& u, const hd<C>& v, const hd<C>& acc) {
  hd<C> r;
  r.v[0] = __fma_rn(u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(v.v[0], u.v[i], __fma_rn(u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++)
    r.v[C + j] = __fma_rn(v.v[0], u.v[C + j],
                          __fma_rn(v.v[1], u.v[j], __fma_rn(u.v[1], v.v[j], __fma_rn(u.v[0], v.v[C + j], acc.v[C + j]))));
  return r;
}
template <int C>
CHF_INL hd<C> hd_fnma(const hd<C>& u, const hd<C>& v, const hd<C>& acc) {  // acc - u*v
  hd<C> r;
  r.v[0] = __fma_rn(-u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(-v.v[0], u.v[i], __fma_rn(-u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++)
    r.v[C + j] = __fma_rn(-v.v[0], u.v[C + j],
                          __fma_rn(-v.v[1], u.v[j], __fma_rn(-u.v[1], v.v[j], __fma_rn(-u.v[0], v.v[C + j], acc.v[C + j]))));
  return r;
}
template <int C>
CHF_INL hd<C> hd_axpy(double c, const hd<C>& u, const hd<C>& acc) {  // acc + c*u
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = __fma_rn(c, u.v[s], acc.v[s]);
  return r;
}

// c * u and u * c
template <int C>
CHF_INL hd<C> operator*(double c, const hd<C>& u) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = c * u.v[s];
  return r;
}
template <int C>
CHF_INL hd<C> operator*(const hd<C>& u, double c) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = u.v[s] * c;
  return r;
}

// c + u, u + c, c - u, u - c
template <int C>
CHF_INL hd<C> operator+(double c, const hd<C>& u) {
  hd<C> r = u;
  r.v[0] = c + u.v[0];
  return r;
}
template <int C>
CHF_INL hd<C> operator+(const hd<C>& u, double c) {
  hd<C> r = u;
  r.v[0] = u.v[0] + c;
  return r;
}
template <int C>
CHF_INL hd<C> operator-(double c, const hd<C>& u) {
  hd<C> r;
  r.v[0] = c - u.v[0];
#pragma unroll
  for (int s = 1; s < hd<C>::N; s++) r.v[s] = -u.v[s];
  return r;
}
template <int C>
CHF_INL hd<C> operator-(const hd<C>& u, double c) {
  hd<C> r = u;
  r.v[0] = u.v[0] - c;
  return r;
}

// u / v (quotient rule; SPEC.md:69-77 -- the paper lists "/" without a rule)
template <int C>
CHF_INL hd<C> operator/(const hd<C>& u, const hd<C>& v) {
  hd<C> r;
  r.v[0] = u.v[0] / v.v[0];
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = (u.v[k] - r.v[0] * v.v[k]) / v.v[0];
#pragma unroll
  for (int k = 2; k <= C + 1; k++)
    r.v[C + k] = (u.v[C + k] - r.v[1] * v.v[k] - r.v[k] * v.v[1] - r.v[0] * v.v[C + k]) / v.v[0];
  return r;
}

// u / c and c / u (a scalar operand is a lifted constant)
template <int C>
CHF_INL hd<C> operator/(const hd<C>& u, double c) {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = u.v[s] / c;
  return r;
}
template <int C>
CHF_INL hd<C> operator/(double c, const hd<C>& v) {
  hd<C> lifted;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) lifted.v[s] = 0.0;
  lifted.v[0] = c;
  return lifted / v;
}

// unary chain rule given (g, g', g'') at u0
template <int C>
CHF_INL hd<C> hd_unary(const hd<C>& u, double g0, double g1, double g2) {
  hd<C> r;
  r.v[0] = g0;
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = g1 * u.v[k];
  const double g2u1 = g2 * u.v[1];
#pragma unroll
  for (int k = 2; k <= C + 1; k++) r.v[C + k] = g1 * u.v[C + k] + g2u1 * u.v[k];
  return r;
}

// acc + g(u), the unary rule's terms accumulated onto acc (R5, as hd_fma)
template <int C>
CHF_INL hd<C> hd_unary_acc(const hd<C>& u, double g0, double g1, double g2, const hd<C>& acc) {
  hd<C> r;
  r.v[0] = acc.v[0] + g0;
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = __fma_rn(g1, u.v[k], acc.v[k]);
  const double g2u1 = g2 * u.v[1];
#pragma unroll
  for (int k = 2; k <= C + 1; k++) r.v[C + k] = __fma_rn(g2u1, u.v[k], __fma_rn(g1, u.v[C + k], acc.v[C + k]));
  return r;
}

template <int C>
CHF_INL hd<C> sin(const hd<C>& u) {
  double s, c;
  ::sincos(u.v[0], &s, &c);
  return hd_unary(u, s, c, -s);
}
template <int C>
CHF_INL hd<C> cos(const hd<C>& u) {
  double s, c;
  ::sincos(u.v[0], &s, &c);
  return hd_unary(u, c, -s, -c);
}
template <int C>
CHF_INL hd<C> exp(const hd<C>& u) {
  const double e = ::exp(u.v[0]);
  return hd_unary(u, e, e, e);
}
template <int C>
CHF_INL hd<C> sqrt(const hd<C>& u) {
  const double r = ::sqrt(u.v[0]);
  const double g1 = 1.0 / (2.0 * r);
  const double g2 = -1.0 / (4.0 * u.v[0] * r);
  return hd_unary(u, r, g1, g2);
}
template <int C>
CHF_INL hd<C> log(const hd<C>& u) {
  const double x = u.v[0];
  return hd_unary(u, ::log(x), 1.0 / x, -1.0 / (x * x));
}
template <int C>
CHF_INL hd<C> abs(const hd<C>& u) {  // abs'(0) = 0
  const double x = u.v[0];
  const double sg = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0);
  return hd_unary(u, ::fabs(x), sg, 0.0);
}

// comparisons look at the value slot only
template <int C> CHF_INL bool operator<(const hd<C>& a, const hd<C>& b) { return a.v[0] < b.v[0]; }
template <int C> CHF_INL bool operator>(const hd<C>& a, const hd<C>& b) { return a.v[0] > b.v[0]; }
template <int C> CHF_INL bool operator<=(const hd<C>& a, const hd<C>& b) { return a.v[0] <= b.v[0]; }
template <int C> CHF_INL bool operator>=(const hd<C>& a, const hd<C>& b) { return a.v[0] >= b.v[0]; }

}  // namespace chessfad

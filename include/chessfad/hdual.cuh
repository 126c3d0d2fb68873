// hdual.cuh -- the chunked second-order dual number hDual<C> on the device (sm_100a).
//
// Layout (§IV "CHESSFAD Library Implementation"):
//   v[0]            f
//   v[1]            df/dx_i              (the active Hessian row i)
//   v[2 .. C+1]     df/dx_{cs .. cs+C-1} (the active chunk of columns)
//   v[C+2 .. 2C+1]  d2f/dx_i dx_{cs..}   (one chunk of row i of the Hessian)
// A hDual<C> is 2C+2 doubles = 4C+4 registers; it lives in registers, never in memory.
//
// Two types carry it (reading R7):
//   hd<C>  every slot stored;
//   hs<C>  "seed-shaped": slots 0 .. C+1 stored, the C second-order slots ZERO BY
//          CONSTRUCTION.  A CHUNK-INIT seed (Alg 4: y_k = <a_k, [k==i],
//          e_{k-cs}, 0 ... 0>) is one, and so is every affine image of seeds (c*y, y+c, c-y,
//          y+-y', y/c).  The rules below take either type for each operand and omit exactly
//          the terms whose factor is a structural-zero slot: a product with a second-order slot
//          of an hs operand is not formed (the paper's rule adds u0*0 there, which is +-0 for
//          finite u0).  Only the sign of a zero result, or a NaN from inf*0 on non-finite input,
//          can differ from forming the term; nvcc cannot drop these products itself under
//          IEEE rules because the other factor might be inf or NaN.
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

#include <type_traits>

namespace chessfad {

#define CHF_INL __device__ __forceinline__

template <int C>
struct hd {
  static constexpr int N = 2 * C + 2;
  double v[N];
};

template <int C>
struct hs {  // seed-shaped: v[0 .. C+1]; the second-order slots are structural zeros
  static constexpr int N = C + 2;
  double v[N];
  CHF_INL operator hd<C>() const {  // materialise the zeros (e.g. `hd<C> y = seed;`)
    hd<C> r;
#pragma unroll
    for (int s = 0; s < N; s++) r.v[s] = v[s];
#pragma unroll
    for (int s = N; s < hd<C>::N; s++) r.v[s] = 0.0;
    return r;
  }
};

template <class T> struct dual_traits { static constexpr bool ok = false; };
template <int C> struct dual_traits<hd<C>> { static constexpr bool ok = true, seed = false; static constexpr int c = C; };
template <int C> struct dual_traits<hs<C>> { static constexpr bool ok = true, seed = true; static constexpr int c = C; };
template <class T> inline constexpr bool is_seed_v = dual_traits<T>::seed;

// U and V are hDual types of the same C
#define CHF_DUAL1(U) std::enable_if_t<dual_traits<U>::ok, int> = 0
#define CHF_DUAL2(U, V) \
  std::enable_if_t<dual_traits<U>::ok && dual_traits<V>::ok && dual_traits<U>::c == dual_traits<V>::c, int> = 0
// result type of a componentwise combination: seed-shaped iff both operands are
template <class U, class V>
using sum_t = std::conditional_t<is_seed_v<U> && is_seed_v<V>, U, hd<dual_traits<U>::c>>;

// ---------------------------------------------------------------- hh+ / hh- / negation
template <class U, class V, CHF_DUAL2(U, V)>
CHF_INL sum_t<U, V> operator+(const U& a, const V& b) {
  constexpr int C = dual_traits<U>::c;
  sum_t<U, V> r;
#pragma unroll
  for (int s = 0; s < C + 2; s++) r.v[s] = a.v[s] + b.v[s];
  if constexpr (!(is_seed_v<U> && is_seed_v<V>)) {
#pragma unroll
    for (int s = C + 2; s < 2 * C + 2; s++) {
      if constexpr (is_seed_v<U>) r.v[s] = b.v[s];
      else if constexpr (is_seed_v<V>) r.v[s] = a.v[s];
      else r.v[s] = a.v[s] + b.v[s];
    }
  }
  return r;
}

template <class U, class V, CHF_DUAL2(U, V)>
CHF_INL sum_t<U, V> operator-(const U& a, const V& b) {
  constexpr int C = dual_traits<U>::c;
  sum_t<U, V> r;
#pragma unroll
  for (int s = 0; s < C + 2; s++) r.v[s] = a.v[s] - b.v[s];
  if constexpr (!(is_seed_v<U> && is_seed_v<V>)) {
#pragma unroll
    for (int s = C + 2; s < 2 * C + 2; s++) {
      if constexpr (is_seed_v<U>) r.v[s] = -b.v[s];
      else if constexpr (is_seed_v<V>) r.v[s] = a.v[s];
      else r.v[s] = a.v[s] - b.v[s];
    }
  }
  return r;
}

template <class U, CHF_DUAL1(U)>
CHF_INL U operator-(const U& a) {
  U r;
#pragma unroll
  for (int s = 0; s < U::N; s++) r.v[s] = -a.v[s];
  return r;
}

// ---------------------------------------------------------------- hh*
template <class U, class V, CHF_DUAL2(U, V)>
CHF_INL hd<dual_traits<U>::c> operator*(const U& u, const V& v) {
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = u.v[0] * v.v[0];
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = u.v[0] * v.v[i] + v.v[0] * u.v[i];
#pragma unroll
  for (int j = 2; j <= C + 1; j++) {
    double t;
    if constexpr (!is_seed_v<V>) t = u.v[0] * v.v[C + j] + u.v[1] * v.v[j];
    else t = u.v[1] * v.v[j];
    t = t + v.v[1] * u.v[j];
    if constexpr (!is_seed_v<U>) t = t + v.v[0] * u.v[C + j];
    r.v[C + j] = t;
  }
  return r;
}

// Fused accumulate forms (reading R5): acc + u*v, acc - u*v, acc + c*u with every
// term of the product added onto the running sum one at a time, in the Fig. 1 term order,
// as one DFMA each.  Per slot these are exactly the multiplications and additions of one
// hh* (or s*) plus one hh+ (model FLOPs unchanged: 6C+3 mul + 4C+1 add + 2C+2 add =
// 6C+3 FMAs); only the association of the sum differs from `acc + (u*v)`, i.e. the
// reduction order of the sum being accumulated.  Used by the built-in test functions
// (testfuncs.cuh) for their running sums; the plain operators above are unchanged.
// Second-order chain of acc +- (u*v) in slot C+j; SGN = +1 or -1.
template <int SGN>
CHF_INL double sgn(double x) {
  if constexpr (SGN > 0) return x;
  else return -x;
}
template <int SGN, class U, class V, class A>
CHF_INL double fma_chain2(const U& u, const V& v, const A& acc, int j) {
  constexpr int C = dual_traits<U>::c;
  constexpr bool SU = is_seed_v<U>, SV = is_seed_v<V>, SA = is_seed_v<A>;
  double t;  // terms in the Fig. 1 order onto acc[C+j]; a term with a structural-zero factor is absent
  if constexpr (!SV && !SA) t = __fma_rn(sgn<SGN>(u.v[1]), v.v[j], __fma_rn(sgn<SGN>(u.v[0]), v.v[C + j], acc.v[C + j]));
  else if constexpr (!SV) t = __fma_rn(sgn<SGN>(u.v[1]), v.v[j], sgn<SGN>(u.v[0]) * v.v[C + j]);
  else if constexpr (!SA) t = __fma_rn(sgn<SGN>(u.v[1]), v.v[j], acc.v[C + j]);
  else t = sgn<SGN>(u.v[1]) * v.v[j];
  t = __fma_rn(sgn<SGN>(v.v[1]), u.v[j], t);
  if constexpr (!SU) t = __fma_rn(sgn<SGN>(v.v[0]), u.v[C + j], t);
  return t;
}

template <class U, class V, class A, CHF_DUAL2(U, V), CHF_DUAL2(U, A)>
CHF_INL hd<dual_traits<U>::c> hd_fma(const U& u, const V& v, const A& acc) {
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = __fma_rn(u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(v.v[0], u.v[i], __fma_rn(u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++) r.v[C + j] = fma_chain2<1>(u, v, acc, j);
  return r;
}
template <class U, class V, class A, CHF_DUAL2(U, V), CHF_DUAL2(U, A)>
CHF_INL hd<dual_traits<U>::c> hd_fnma(const U& u, const V& v, const A& acc) {  // acc - u*v
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = __fma_rn(-u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(-v.v[0], u.v[i], __fma_rn(-u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++) r.v[C + j] = fma_chain2<-1>(u, v, acc, j);
  return r;
}
template <class U, class A, CHF_DUAL2(U, A)>
CHF_INL sum_t<U, A> hd_axpy(double c, const U& u, const A& acc) {  // acc + c*u
  constexpr int C = dual_traits<U>::c;
  sum_t<U, A> r;
#pragma unroll
  for (int s = 0; s < C + 2; s++) r.v[s] = __fma_rn(c, u.v[s], acc.v[s]);
  if constexpr (!(is_seed_v<U> && is_seed_v<A>)) {
#pragma unroll
    for (int s = C + 2; s < 2 * C + 2; s++) {
      if constexpr (is_seed_v<U>) r.v[s] = acc.v[s];
      else if constexpr (is_seed_v<A>) r.v[s] = c * u.v[s];
      else r.v[s] = __fma_rn(c, u.v[s], acc.v[s]);
    }
  }
  return r;
}

// ---------------------------------------------------------------- s* / s+ / s- (type kept)
template <class U, CHF_DUAL1(U)>
CHF_INL U operator*(double c, const U& u) {
  U r;
#pragma unroll
  for (int s = 0; s < U::N; s++) r.v[s] = c * u.v[s];
  return r;
}
template <class U, CHF_DUAL1(U)>
CHF_INL U operator*(const U& u, double c) {
  U r;
#pragma unroll
  for (int s = 0; s < U::N; s++) r.v[s] = u.v[s] * c;
  return r;
}
template <class U, CHF_DUAL1(U)>
CHF_INL U operator+(double c, const U& u) {
  U r = u;
  r.v[0] = c + u.v[0];
  return r;
}
template <class U, CHF_DUAL1(U)>
CHF_INL U operator+(const U& u, double c) {
  U r = u;
  r.v[0] = u.v[0] + c;
  return r;
}
template <class U, CHF_DUAL1(U)>
CHF_INL U operator-(double c, const U& u) {
  U r;
  r.v[0] = c - u.v[0];
#pragma unroll
  for (int s = 1; s < U::N; s++) r.v[s] = -u.v[s];
  return r;
}
template <class U, CHF_DUAL1(U)>
CHF_INL U operator-(const U& u, double c) {
  U r = u;
  r.v[0] = u.v[0] - c;
  return r;
}

// ---------------------------------------------------------------- quotient
// u / v (quotient rule; SPEC.md:69-77 -- the paper lists "/" without a rule)
template <class U, class V, CHF_DUAL2(U, V)>
CHF_INL hd<dual_traits<U>::c> operator/(const U& u, const V& v) {
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = u.v[0] / v.v[0];
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = (u.v[k] - r.v[0] * v.v[k]) / v.v[0];
#pragma unroll
  for (int k = 2; k <= C + 1; k++) {
    double t;
    if constexpr (!is_seed_v<U>) t = u.v[C + k] - r.v[1] * v.v[k];
    else t = -(r.v[1] * v.v[k]);
    t = t - r.v[k] * v.v[1];
    if constexpr (!is_seed_v<V>) t = t - r.v[0] * v.v[C + k];
    r.v[C + k] = t / v.v[0];
  }
  return r;
}

// u / c and c / u (a scalar operand is a lifted constant)
template <class U, CHF_DUAL1(U)>
CHF_INL U operator/(const U& u, double c) {
  U r;
#pragma unroll
  for (int s = 0; s < U::N; s++) r.v[s] = u.v[s] / c;
  return r;
}
template <class V, CHF_DUAL1(V)>
CHF_INL hd<dual_traits<V>::c> operator/(double c, const V& v) {
  hs<dual_traits<V>::c> lifted;  // <c, 0, ..., 0>: seed-shaped
#pragma unroll
  for (int s = 0; s < hs<dual_traits<V>::c>::N; s++) lifted.v[s] = 0.0;
  lifted.v[0] = c;
  return lifted / v;
}

// ---------------------------------------------------------------- unary chain rule
// given (g, g', g'') at u0
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> hd_unary(const U& u, double g0, double g1, double g2) {
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = g0;
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = g1 * u.v[k];
  const double g2u1 = g2 * u.v[1];
#pragma unroll
  for (int k = 2; k <= C + 1; k++) {
    if constexpr (is_seed_v<U>) r.v[C + k] = g2u1 * u.v[k];
    else r.v[C + k] = g1 * u.v[C + k] + g2u1 * u.v[k];
  }
  return r;
}

// acc + g(u), the unary rule's terms accumulated onto acc (R5, as hd_fma)
template <class U, class A, CHF_DUAL2(U, A)>
CHF_INL hd<dual_traits<U>::c> hd_unary_acc(const U& u, double g0, double g1, double g2, const A& acc) {
  constexpr int C = dual_traits<U>::c;
  hd<C> r;
  r.v[0] = acc.v[0] + g0;
#pragma unroll
  for (int k = 1; k <= C + 1; k++) r.v[k] = __fma_rn(g1, u.v[k], acc.v[k]);
  const double g2u1 = g2 * u.v[1];
#pragma unroll
  for (int k = 2; k <= C + 1; k++) {
    if constexpr (!is_seed_v<U> && !is_seed_v<A>) r.v[C + k] = __fma_rn(g2u1, u.v[k], __fma_rn(g1, u.v[C + k], acc.v[C + k]));
    else if constexpr (!is_seed_v<U>) r.v[C + k] = __fma_rn(g2u1, u.v[k], g1 * u.v[C + k]);
    else if constexpr (!is_seed_v<A>) r.v[C + k] = __fma_rn(g2u1, u.v[k], acc.v[C + k]);
    else r.v[C + k] = g2u1 * u.v[k];
  }
  return r;
}

template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> sin(const U& u) {
  double s, c;
  ::sincos(u.v[0], &s, &c);
  return hd_unary(u, s, c, -s);
}
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> cos(const U& u) {
  double s, c;
  ::sincos(u.v[0], &s, &c);
  return hd_unary(u, c, -s, -c);
}
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> exp(const U& u) {
  const double e = ::exp(u.v[0]);
  return hd_unary(u, e, e, e);
}
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> sqrt(const U& u) {
  const double r = ::sqrt(u.v[0]);
  const double g1 = 1.0 / (2.0 * r);
  const double g2 = -1.0 / (4.0 * u.v[0] * r);
  return hd_unary(u, r, g1, g2);
}
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> log(const U& u) {
  const double x = u.v[0];
  return hd_unary(u, ::log(x), 1.0 / x, -1.0 / (x * x));
}
template <class U, CHF_DUAL1(U)>
CHF_INL hd<dual_traits<U>::c> abs(const U& u) {  // abs'(0) = 0
  const double x = u.v[0];
  const double sg = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0);
  return hd_unary(u, ::fabs(x), sg, 0.0);
}

// comparisons look at the value slot only
template <class U, class V, CHF_DUAL2(U, V)> CHF_INL bool operator<(const U& a, const V& b) { return a.v[0] < b.v[0]; }
template <class U, class V, CHF_DUAL2(U, V)> CHF_INL bool operator>(const U& a, const V& b) { return a.v[0] > b.v[0]; }
template <class U, class V, CHF_DUAL2(U, V)> CHF_INL bool operator<=(const U& a, const V& b) { return a.v[0] <= b.v[0]; }
template <class U, class V, CHF_DUAL2(U, V)> CHF_INL bool operator>=(const U& a, const V& b) { return a.v[0] >= b.v[0]; }

}  // namespace chessfad

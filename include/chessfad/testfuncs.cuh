// testfuncs.cuh -- the paper's test functions over hDual<C> (device code).
//
// The paper names Rosenbrock, Ackley and Fletcher-Powell without formulas;
// the definitions are SPEC.md:352-396 and the expression forms are DESIGN.md's canonical
// forms (loops ascend, first term of every sum initialises).  The GPU may differ from the
// oracle only in FMA contraction and in the order of reductions.
//
// Bodies are generic over a seed provider `y(k)` that returns the CHUNK-INIT seed of
// variable k (Alg 4) on the fly: the paper's per-thread array
// hDual<C> y[n] is never materialised.
//
// Fletcher-Powell is in csrc/f3_mma.cuh (its O(n^2) hDual sums run on the FP64 tensor core).
#pragma once
#include "hdual.cuh"

namespace chessfad {

enum { FUNC_ROSENBROCK = 0, FUNC_ACKLEY = 1, FUNC_FLETCHER_POWELL = 2, FUNC_PRODSUM = 3 };

// shared-memory load neither compiler may merge, hoist or fold (a fresh value per call)
CHF_INL double ld_shared_volatile(const double* p) {
  double r;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(r) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return r;
}

// CHUNK-INIT seed for the lane's own point; row i and chunk start cs are warp-uniform.
//   y[k] = < a_k, [k==i], e_{k-cs} if cs <= k < cs+C, 0 ... 0 >          (Alg 4)
// STATIC: n is a compile-time constant of the kernel (the paper's NV template, Fig. 2,
// PAPER.md:485-499) and the functions' variable loops are fully unrolled, so k is a constant
// in each copy; row i and chunk start cs stay runtime values (every evaluation is formed and
// executed on its own, as in Alg 7).
// VOL (STATIC only): a_k (and Ackley's tables) are read with volatile loads, so each evaluation
// reads its own copy and no compiler can share work between evaluations whose code sits side by
// side (the unrolled chunk loop of kernels.cuh); it also keeps nvcc from hoisting every
// coordinate load of the unrolled variable loop (register pressure at n >= 32)
template <int C, bool STATIC = false, bool VOL = false>
struct LaneSeed {
  static constexpr bool kStatic = STATIC;  // false: runtime n, loops keep their partial unrolling
  static constexpr bool kFused = true;    // fused accumulate forms (R5) in the running sums
  const double* a;  // a[k * stride] = coordinate k of this lane's point (shared memory)
  int stride;
  int i, cs;
  // Ackley: sin/cos of the value slot 2*pi*a_k of cos(2*pi*y_k), tabulated once per tile
  // (g, g', g'' of an input-only argument; the model counts them as 0 FLOPs)
  const double* sin2pi;
  const double* cos2pi;
  CHF_INL hs<C> operator()(int k) const {
    hs<C> y;
    y.v[0] = VOL ? ld_shared_volatile(a + k * stride) : a[k * stride];
    y.v[1] = (k == i) ? 1.0 : 0.0;
    const int off = k - cs;
#pragma unroll
    for (int l = 0; l < C; l++) y.v[2 + l] = (off == l) ? 1.0 : 0.0;
    return y;  // second-order slots: structural zeros (hdual.cuh hs<C>)
  }
  // Ackley's tabulated sin / cos(2 pi a_k) (volatile with VOL, as a_k above)
  CHF_INL double s2pi(int k) const { return VOL ? ld_shared_volatile(sin2pi + k * stride) : sin2pi[k * stride]; }
  CHF_INL double c2pi(int k) const { return VOL ? ld_shared_volatile(cos2pi + k * stride) : cos2pi[k * stride]; }
};

// Compile-time-n seed (small-n path, kernels.cuh hvp_small_kernel): the point lives in
// registers and every loop over variables, rows and chunks is fully unrolled, so i, cs and
// k are compile-time constants in each copy and the 0/1 seed slots fold exactly (as in the
// paper's NV-templated kernels).
// FUSED: fused accumulate forms (R5) or the plain operators; the plain forms leave nvcc more
// common subexpressions to share across the unrolled evaluations, which wins for most
// (F, C, n) of this path (measured, launch.cuh small_fused).
template <int C, bool FUSED = false>
struct StaticSeed {
  static constexpr bool kStatic = true;
  static constexpr bool kFused = FUSED;
  const double* a;  // this thread's point, a[k]
  int stride;       // 1
  int i, cs;
  const double* sin2pi;
  const double* cos2pi;
  CHF_INL hs<C> operator()(int k) const {
    hs<C> y;
    y.v[0] = a[k];
    y.v[1] = (k == i) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l < C; l++) y.v[2 + l] = (k - cs == l) ? 1.0 : 0.0;
    return y;
  }
  CHF_INL double s2pi(int k) const { return sin2pi[k * stride]; }
  CHF_INL double c2pi(int k) const { return cos2pi[k * stride]; }
};

#ifndef CHF_SUM_UNROLL
#define CHF_SUM_UNROLL 4  // Rosenbrock term-loop unroll of the runtime-n kernels (measured: 4 > 2 > 1,
                          // profiles/r01/fused/)
#endif

// Loop over [lo, hi): fully unrolled for a compile-time-n seed, `#pragma unroll UNROLL`
// otherwise (the runtime-n kernels' schedule is left exactly as it was).
template <class Seed, int UNROLL, class Body>
CHF_INL void seed_loop(int lo, int hi, Body&& body) {
  if constexpr (Seed::kStatic) {
#pragma unroll
    for (int k = lo; k < hi; k++) body(k);
  } else if constexpr (UNROLL > 0) {
#pragma unroll UNROLL
    for (int k = lo; k < hi; k++) body(k);
  } else {
    for (int k = lo; k < hi; k++) body(k);
  }
}

// F1 Rosenbrock: s = sum_{i<n-1} 100 (y_{i+1} - y_i^2)^2 + (1 - y_i)^2
// per evaluation: 3(n-1) hh*, 3n-4 hh+, n-1 s*, n-1 s+  (DESIGN.md op table)
// Running sums use the fused accumulate forms (hdual.cuh, R5): y_{i+1} - y_i*y_i
// and s + 100 (d*d) + e*e add each product term onto the sum as one DFMA; the same
// multiplications and additions as the canonical form, reassociated.
template <int C, class Seed>
CHF_INL hd<C> f_rosenbrock(int n, const Seed& y) {
  hd<C> s;
  if constexpr (Seed::kFused) {
    auto yc = y(1);  // the seed of y_{i+1}, carried into the next term (one seed built per term;
                     // 3-5% faster for Rosenbrock, slower for prodsum: profiles/r02/seed_typed/carry)
    {
      const auto y0 = y(0);
      const auto d = hd_fnma(y0, y0, yc);
      const auto e = 1.0 - y0;
      s = hd_fma(e, e, 100.0 * (d * d));
    }
    seed_loop<Seed, CHF_SUM_UNROLL>(1, n - 1, [&](int i) {
      const auto yi = yc;
      yc = y(i + 1);
      const auto d = hd_fnma(yi, yi, yc);
      const auto e = 1.0 - yi;
      s = hd_fma(e, e, hd_axpy(100.0, d * d, s));
    });
  } else {  // the canonical form as written (R2)
    {
      const auto y0 = y(0), y1 = y(1);
      const hd<C> d = y1 - y0 * y0;
      const auto e = 1.0 - y0;
      s = 100.0 * (d * d) + e * e;
    }
    seed_loop<Seed, 2>(1, n - 1, [&](int i) {
      const auto yi = y(i), yi1 = y(i + 1);
      const hd<C> d = yi1 - yi * yi;
      const auto e = 1.0 - yi;
      const hd<C> t = 100.0 * (d * d) + e * e;
      s = s + t;
    });
  }
  return s;
}

// F2 Ackley: -20 exp(-0.2 sqrt(S1/n)) - exp(S2/n) + 20 + e,  S1 = sum y^2, S2 = sum cos(2 pi y)
// (SPEC.md:361-369); per evaluation n hh*, 2n-1 hh+, n+4 s*, n+3 unary, 1 s+
template <int C, class Seed>
CHF_INL hd<C> f_ackley(int n, const Seed& y) {
  const double two_pi = 6.283185307179586, euler = 2.718281828459045;
  hd<C> s1;
  {
    const auto y0 = y(0);
    s1 = y0 * y0;
  }
  seed_loop<Seed, 0>(1, n, [&](int i) {
    const auto yi = y(i);
    if constexpr (Seed::kFused) s1 = hd_fma(yi, yi, s1);  // s1 + yi*yi, fused (R5)
    else s1 = s1 + yi * yi;
  });
  // cos(u), u = 2 pi y_i: (g, g', g'') = (cos u0, -sin u0, -cos u0) with u0 = 2 pi a_i,
  // bit-identical to the tabulated argument (same single rounding of two_pi * a_i)
  auto cos2pi = [&](int k) {
    const auto u = two_pi * y(k);
    const double s = y.s2pi(k), c = y.c2pi(k);
    return hd_unary(u, c, -s, -c);
  };
  hd<C> s2 = cos2pi(0);
  seed_loop<Seed, 0>(1, n, [&](int i) {
    if constexpr (Seed::kFused) {  // s2 + cos(2 pi y_i), fused (R5)
      const auto u = two_pi * y(i);
      s2 = hd_unary_acc(u, y.c2pi(i), -y.s2pi(i), -y.c2pi(i), s2);
    } else {
      s2 = s2 + cos2pi(i);
    }
  });
  const double inv_n = 1.0 / n;
  const hd<C> t1 = (-20.0) * exp((-0.2) * sqrt(s1 * inv_n));
  const hd<C> t2 = exp(s2 * inv_n);
  return (t1 - t2) + (20.0 + euler);
}

// F4 prodsum: sum_{i<n-1} y_i y_{i+1}; exactly n-1 hh* and n-2 hh+ 
template <int C, class Seed>
CHF_INL hd<C> f_prodsum(int n, const Seed& y) {
  hd<C> s = y(0) * y(1);
  seed_loop<Seed, 2>(1, n - 1, [&](int i) {
    if constexpr (Seed::kFused) s = hd_fma(y(i), y(i + 1), s);  // fused (R5)
    else s = s + y(i) * y(i + 1);
  });
  return s;
}

template <int FUNC, int C, class Seed>
CHF_INL hd<C> eval_f(int n, const Seed& y) {
  if constexpr (FUNC == FUNC_ROSENBROCK) return f_rosenbrock<C>(n, y);
  else if constexpr (FUNC == FUNC_ACKLEY) return f_ackley<C>(n, y);
  else return f_prodsum<C>(n, y);
}

// The register-path kernel evaluates a FUNCTOR: any type with
//     template <int C, class Seed> __device__ hd<C> operator()(int n, const Seed& y) const
// where y(k) is the CHUNK-INIT seed hDual<C> of variable k.  The built-in test functions are
// functors too; user functions (NEXT-3, "templated function on the data type")
// plug into the same kernels through include/chessfad_device.cuh.
// kTrig2Pi: the built-in Ackley tabulates sincos(2 pi a_k) per tile (Seed::sin2pi/cos2pi).
template <int FUNC>
struct BuiltinFunc {
  static constexpr bool kTrig2Pi = FUNC == FUNC_ACKLEY;
  // compiled-n kernels (kernels.cuh NS): volatile seed loads + unrolled chunk loop for this
  // (n, kernel chunk C, mode)?  Measured (profiles/r02/ns3/summary.txt): faster for Rosenbrock
  // everywhere; for Ackley in the non-symmetric modes at n >= 32 with C >= 16 (n = 32 HVP 1.33x,
  // Hessian 1.25x; n = 64 also C <= 2); slower for prodsum.
  __host__ __device__ static constexpr int min_blocks(int ns, int c, int mode) {
    return (FUNC == FUNC_ACKLEY && ns == 16 && c == 16 && (mode == 0 || mode == 2)) ? 3 : 0;  // HVP modes
  }
  __host__ __device__ static constexpr bool vol_seeds(int ns, int c, int mode) {
    return FUNC == FUNC_ROSENBROCK ||
           (FUNC == FUNC_ACKLEY && ns >= 32 && (c >= 16 || (ns == 64 && c <= 2) || (ns == 128 && c == 8)) &&
            mode != 2 && mode != 3);  // not MODE_SYM_HVP / MODE_SYM_HESS (kernels.cuh)
  }
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int n, const Seed& y) const {
    return eval_f<FUNC, C>(n, y);
  }
};

// ---------------------------------------------------------------- NEXT-4 seed sparsity (F1, F2, F4)
// chessfad_hvp_batch_seedsparse / chessfad_hessian_batch_seedsparse for the register functions.
// A CHUNK-INIT seed y(k) has nonzero derivative slots only for k in {i} U [cs, cs+C) (Alg 4,
// PAPER.md:172-194).  A term of a running sum whose operands are all constant seeds has
// derivative slots that are exact +-0, so it changes no derivative slot of the sum (up to the
// sign of zero); only the ACTIVE terms -- those touching {i} U [cs, cs+C) -- are evaluated as
// hDuals, in the same ascending order and with the same operations as f_rosenbrock /
// f_ackley / f_prodsum.  The value slot of a sum is needed only where a later unary rule reads
// it (Ackley's s1, s2); it is formed over all terms in the same chain as the full evaluation.
// Work per evaluation: O(C) hDual ops instead of O(n).  Executed FLOPs are far below the model.

// ascending k in [lo1, hi1] U [lo2, hi2] (each clipped to [0, kmax]), each k once
template <class Body>
CHF_INL void sp_union(int lo1, int hi1, int lo2, int hi2, int kmax, Body&& body) {
  lo1 = max(lo1, 0); hi1 = min(hi1, kmax);
  lo2 = max(lo2, 0); hi2 = min(hi2, kmax);
  if (lo2 < lo1) {  // order the intervals
    int t = lo1; lo1 = lo2; lo2 = t;
    t = hi1; hi1 = hi2; hi2 = t;
  }
  if (lo1 <= hi1) {
    for (int k = lo1; k <= hi1; k++) body(k);
    lo2 = max(lo2, hi1 + 1);
  }
  for (int k = lo2; k <= hi2; k++) body(k);
}

template <int C>
CHF_INL hd<C> hd_zero() {
  hd<C> r;
#pragma unroll
  for (int s = 0; s < hd<C>::N; s++) r.v[s] = 0.0;
  return r;
}

// F1: terms k touch y_k, y_{k+1}: active k in {i-1, i} U [cs-1, cs+C-1]; the value slot of s is dead
template <int C>
CHF_INL hd<C> fsp_rosenbrock(int n, const LaneSeed<C>& y) {
  hd<C> s = hd_zero<C>();
  sp_union(y.i - 1, y.i, y.cs - 1, y.cs + C - 1, n - 2, [&](int k) {
    const auto yk = y(k), yk1 = y(k + 1);
    const auto d = hd_fnma(yk, yk, yk1);
    const auto e = 1.0 - yk;
    s = hd_fma(e, e, hd_axpy(100.0, d * d, s));
  });
  return s;
}

// F4: as F1
template <int C>
CHF_INL hd<C> fsp_prodsum(int n, const LaneSeed<C>& y) {
  hd<C> s = hd_zero<C>();
  sp_union(y.i - 1, y.i, y.cs - 1, y.cs + C - 1, n - 2, [&](int k) { s = hd_fma(y(k), y(k + 1), s); });
  return s;
}

// F2: s1 = sum y_k^2, s2 = sum cos(2 pi y_k): active k in {i} U [cs, cs+C); value slots over all k
template <int C>
CHF_INL hd<C> fsp_ackley(int n, const LaneSeed<C>& y) {
  const double two_pi = 6.283185307179586, euler = 2.718281828459045;
  hd<C> s1 = hd_zero<C>(), s2 = hd_zero<C>();
  sp_union(y.i, y.i, y.cs, y.cs + C - 1, n - 1, [&](int k) {
    const auto yk = y(k);
    s1 = hd_fma(yk, yk, s1);
    const auto u = two_pi * yk;
    s2 = hd_unary_acc(u, y.c2pi(k), -y.s2pi(k), -y.c2pi(k), s2);
  });
  {  // value slots: the chains of f_ackley (first term initialises)
    const double a0 = y.a[0];
    double v1 = a0 * a0, v2 = y.c2pi(0);
    for (int k = 1; k < n; k++) {
      const double ak = y.a[k * y.stride];
      v1 = __fma_rn(ak, ak, v1);
      v2 = v2 + y.c2pi(k);
    }
    s1.v[0] = v1;
    s2.v[0] = v2;
  }
  const double inv_n = 1.0 / n;
  const hd<C> t1 = (-20.0) * exp((-0.2) * sqrt(s1 * inv_n));
  const hd<C> t2 = exp(s2 * inv_n);
  return (t1 - t2) + (20.0 + euler);
}

template <int FUNC>
struct SparseFunc {
  static constexpr bool kTrig2Pi = FUNC == FUNC_ACKLEY;
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int n, const Seed& y) const {
    if constexpr (FUNC == FUNC_ROSENBROCK) return fsp_rosenbrock<C>(n, y);
    else if constexpr (FUNC == FUNC_ACKLEY) return fsp_ackley<C>(n, y);
    else return fsp_prodsum<C>(n, y);
  }
};

// F::min_blocks(ns, c, mode): min resident CTAs per SM for the register kernel's launch bounds
// (0 = the default CHF_REG_MINB); measured: Ackley compiled for n = 16 at C = 16 runs its HVP
// modes 1-5% faster capped at 168 registers (3 CTAs/SM) but its Hessian 27% slower; every other
// shape at its default (profiles/r02/ns3/, profiles/r02/a3/)
template <class F, class = void>
struct min_blocks_of {
  __host__ __device__ static constexpr int get(int, int, int) { return 0; }
};
template <class F>
struct min_blocks_of<F, decltype((void)F::min_blocks(0, 0, 0))> {
  __host__ __device__ static constexpr int get(int ns, int c, int mode) { return F::min_blocks(ns, c, mode); }
};

// F::vol_seeds(ns, c, mode) if the functor declares it, else false (user functors)
template <class F, class = void>
struct vol_seeds_of {
  __host__ __device__ static constexpr bool get(int, int, int) { return false; }
};
template <class F>
struct vol_seeds_of<F, decltype((void)F::vol_seeds(0, 0, 0))> {
  __host__ __device__ static constexpr bool get(int ns, int c, int mode) { return F::vol_seeds(ns, c, mode); }
};

template <class F, class = void>
struct uses_trig2pi {
  static constexpr bool value = false;
};
template <class F>
struct uses_trig2pi<F, decltype((void)F::kTrig2Pi)> {
  static constexpr bool value = F::kTrig2Pi;
};

}  // namespace chessfad

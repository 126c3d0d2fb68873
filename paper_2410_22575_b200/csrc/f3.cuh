// f3.cuh -- F3 Fletcher-Powell over hDual<C>, scheduled slot-column by slot-column.
//
// f(y) = sum_k r_k^2,  r_k = E*_k - E_k,  E_k = sum_j A_kj sin(y_j) + B_kj cos(y_j)
// (canonical form in DESIGN.md).  One hDual<C> evaluation costs
// n hh*, 2n^2-1 hh+, 2n^2 s*, 2n unary, n s+ (DESIGN.md op table): the E_k sums are a
// matrix (A | B) times the 2n hDuals sin y_j, cos y_j, 4 n^2 (C+1) FMAs per evaluation.
//
// Keeping the 2n hDuals sin y_j / cos y_j (2n(2C+2) doubles) in registers is impossible
// beyond tiny n*C, so the evaluation DAG is executed in a different topological order
// that needs O(KB) registers:
//   phase A   slots 0 and 1 of every intermediate (they are shared by all columns);
//   phase B   for each column c of the chunk: slots 2+c and C+2+c of every
//             intermediate, which by slot independence need only slots
//             {0, 1, 2+c, C+2+c} of their operands;
//   both are blocked over KB residuals r_k at a time (see f3_eval).
// Every scalar operation of the hDual evaluation is executed once (except g''*u1 of the
// 2n unary ops, recomputed per column: 2 DMUL per j per column) in the paper's per-slot
// form; only the order of independent operations changes.  The result slot 2+c (first
// derivative of f) is dead for the HVP/Hessian and is not formed, exactly as nvcc
// eliminates dead result slots in the register path.
//
// sin(a_j), cos(a_j) (g, g', g'' of the seeded inputs, whose value slot is a_j for every
// evaluation) are computed once per tile of points into shared memory; the §V model counts
// g, g', g'' evaluations as zero FLOPs, so this removes no model work.
//
// Inner loop: for each j, (A_kj, B_kj) is a warp-uniform 16-byte broadcast load feeding
// 4 DFMAs per k; KB k-accumulators per slot give the ILP.
#pragma once
#include "hdual.cuh"

namespace chessfad {

// (A_kj, B_kj) sources: interleaved and transposed in shared memory, abT[j*n + k] (one
// 16-byte broadcast load; the KB k-values of one j sit at immediate offsets), or the
// caller's params in global memory (two 8-byte broadcast loads through the read-only path)
struct ABShared {
  const double2* abT;
  int n;
  CHF_INL double2 get(int k, int j) const { return abT[j * n + k]; }
};
struct ABGlobal {  // same interleaved, transposed layout in global scratch (n > 32)
  const double2* abT;
  int n;
  CHF_INL double2 get(int k, int j) const { return __ldg(abT + j * n + k); }
};

// accumulate variable j into KB k-rows of two slots:  Ep[kk] (+)= A_kj*sp + B_kj*cp, same for q
template <int KB, bool FIRST, class AB>
CHF_INL void f3_accum(const AB& ab, int kb, int j, double sp, double cp, double sq, double cq,
                      double (&Ep)[KB], double (&Eq)[KB]) {
#pragma unroll
  for (int kk = 0; kk < KB; kk++) {
    const double2 c = ab.get(kb + kk, j);
    if (FIRST) {
      Ep[kk] = c.x * sp + c.y * cp;
      Eq[kk] = c.x * sq + c.y * cq;
    } else {
      Ep[kk] = Ep[kk] + c.x * sp + c.y * cp;
      Eq[kk] = Eq[kk] + c.x * sq + c.y * cq;
    }
  }
}

// One evaluation f<hDual<C>>(CHUNK-INIT(i, cs)) for this lane's point (Alg 4 + Fig. 1).
// For each column l in ascending order, sink(cs + l, d2f/dx_i dx_{cs+l}) consumes the
// second-order slot C+2+l (the chunk dot of Alg 7, the store of Alg 5, the scatter of Alg 8).
// sa/ca: sin/cos of the lane's coordinates, element j at [j * stride]; Es: E*.
// Loop order: k-blocks outer, columns inner.  For each block of KB residuals r_k, slots 0/1
// (phase A) are formed once and kept in registers, then every column's slots 2+c / C+2+c of
// those r_k are formed and their r*r contributions added to the column's f accumulator
// FC[c] (per-thread scratch, C doubles) in ascending k -- the same summation order as a
// column-outer schedule, with O(KB) live state instead of the 2n residual slots.
template <int KB, class AB, class Sink>
CHF_INL void f3_eval(int n, int C, int i, int cs, const double* __restrict__ sa,
                     const double* __restrict__ ca, int stride, const AB& ab,
                     const double* __restrict__ Es, double* FC, Sink&& sink) {
  for (int kb = 0; kb < n; kb += KB) {
    // ---------------- phase A: slots 0 and 1 of r_k, k in [kb, kb+KB)
    double r0[KB], r1[KB];
    {
      double E0[KB], E1[KB];
      {
        const double s0 = sa[0], c0 = ca[0];
        const double y1 = (0 == i) ? 1.0 : 0.0;
        // sin(y_0) = <sin a, cos a * y1, ...>;  cos(y_0) = <cos a, -sin a * y1, ...>
        f3_accum<KB, true>(ab, kb, 0, s0, c0, c0 * y1, (-s0) * y1, E0, E1);
      }
      for (int j = 1; j < n; j++) {
        const double s0 = sa[j * stride], c0 = ca[j * stride];
        const double y1 = (j == i) ? 1.0 : 0.0;
        f3_accum<KB, false>(ab, kb, j, s0, c0, c0 * y1, (-s0) * y1, E0, E1);
      }
#pragma unroll
      for (int kk = 0; kk < KB; kk++) {
        r0[kk] = Es[kb + kk] - E0[kk];  // r_k = E*_k - E_k (s+ on slot 0, negation elsewhere)
        r1[kk] = -E1[kk];
      }
    }
    // f slots 0/1 (f = sum_k r_k * r_k) are dead for the HVP and the Hessian.

    // ---------------- phase B: columns 2+c / C+2+c of the same r_k
    for (int c = 0; c < C; c++) {
      const int col = cs + c;
      double E2[KB], EC[KB];
      {
        const double s0 = sa[0], c0 = ca[0];
        const double y1 = (0 == i) ? 1.0 : 0.0, y2 = (0 == col) ? 1.0 : 0.0, yC = 0.0;
        // sin: g' = cos a, g'' = -sin a;   cos: g' = -sin a, g'' = -cos a
        const double s2 = c0 * y2, sC = c0 * yC + ((-s0) * y1) * y2;
        const double c2 = (-s0) * y2, cC = (-s0) * yC + ((-c0) * y1) * y2;
        f3_accum<KB, true>(ab, kb, 0, s2, c2, sC, cC, E2, EC);
      }
      for (int j = 1; j < n; j++) {
        const double s0 = sa[j * stride], c0 = ca[j * stride];
        const double y1 = (j == i) ? 1.0 : 0.0, y2 = (j == col) ? 1.0 : 0.0, yC = 0.0;
        const double s2 = c0 * y2, sC = c0 * yC + ((-s0) * y1) * y2;
        const double c2 = (-s0) * y2, cC = (-s0) * yC + ((-c0) * y1) * y2;
        f3_accum<KB, false>(ab, kb, j, s2, c2, sC, cC, E2, EC);
      }
      double fC = kb == 0 ? 0.0 : FC[c];
#pragma unroll
      for (int kk = 0; kk < KB; kk++) {
        const double r2 = -E2[kk], rC = -EC[kk];
        // (r*r)[C+2+c] = r0 rC + r1 r2 + r1 r2 + r0 rC   (Fig. 1 term order)
        const double rrC = r0[kk] * rC + r1[kk] * r2 + r1[kk] * r2 + r0[kk] * rC;
        fC = (kb + kk == 0) ? rrC : fC + rrC;
      }
      FC[c] = fC;
    }
  }
  for (int c = 0; c < C; c++) sink(cs + c, FC[c]);
}

}  // namespace chessfad

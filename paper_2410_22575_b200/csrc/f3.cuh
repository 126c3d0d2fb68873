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

// (A_kj, B_kj) sources: interleaved and transposed, abT[j*n + k], so that the KB k-values of
// one j are 16-byte warp-uniform broadcast loads at immediate offsets.
//   ABShared  the whole matrix in shared memory (n <= 32)
//   ABRing    n > 32: streamed from the global scratch copy through a per-warp cp.async
//             double buffer of JC j-values x KB k-values (hides the L1/L2 latency that the
//             direct global loads expose: ncu long_scoreboard stalls, profiles/r01)
struct ABShared {
  const double2* abT;
  int n;
  CHF_INL double2 get(int k, int j) const { return abT[j * n + k]; }
};

CHF_INL void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
CHF_INL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
CHF_INL void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int KB, int JC>
struct ABRing {
  double2* buf;         // this warp's ring: 2 stages x JC x KB
  const double2* abT;   // global scratch, [j][k]
  int n, lane;
  CHF_INL void issue(int kb, int j0, int stage) const {
    for (int q = lane; q < JC * KB; q += 32) {
      const int jj = q / KB, kk = q - jj * KB;
      cp_async16(buf + (stage * JC + jj) * KB + kk, abT + (size_t)(j0 + jj) * n + kb + kk);
    }
    cp_async_commit();
  }
};

// E (+)= sum_j A_kj * p_j + B_kj * q_j for KB k-rows and two slots; vals(j, sp, cp, sq, cq)
// yields the slot values of sin y_j (s*) and cos y_j (c*).  The first j initialises.
template <int KB, bool FIRST, class V>
CHF_INL void f3_fma(const double2& c, int kk, const V& v, double (&Ep)[KB], double (&Eq)[KB]) {
  if (FIRST) {
    Ep[kk] = c.x * v.sp + c.y * v.cp;
    Eq[kk] = c.x * v.sq + c.y * v.cq;
  } else {
    Ep[kk] = Ep[kk] + c.x * v.sp + c.y * v.cp;
    Eq[kk] = Eq[kk] + c.x * v.sq + c.y * v.cq;
  }
}

#ifndef CHF_F3_JUNROLL
#define CHF_F3_JUNROLL 1
#endif
constexpr int kF3JUnroll = CHF_F3_JUNROLL;  // j-loop unroll of the shared-memory (A,B) path
#ifndef CHF_F3_RING_JUNROLL
#define CHF_F3_RING_JUNROLL 2  // measured 2-5% faster than 1 at n = 64 / 128 (profiles/r01/f3ab/)
#endif
constexpr int kF3RingJUnroll = CHF_F3_RING_JUNROLL;  // j-loop unroll of the ring path (n > 32)

struct SlotVals {
  double sp, cp, sq, cq;
};

template <int KB, class Vals>
CHF_INL void f3_sum_j(const ABShared& ab, int n, int kb, const Vals& vals, double (&Ep)[KB], double (&Eq)[KB]) {
  {
    const SlotVals v = vals(0);
#pragma unroll
    for (int kk = 0; kk < KB; kk++) f3_fma<KB, true>(ab.get(kb + kk, 0), kk, v, Ep, Eq);
  }
#pragma unroll kF3JUnroll
  for (int j = 1; j < n; j++) {
    const SlotVals v = vals(j);
#pragma unroll
    for (int kk = 0; kk < KB; kk++) f3_fma<KB, false>(ab.get(kb + kk, j), kk, v, Ep, Eq);
  }
}

template <int KB, int JC, class Vals>
CHF_INL void f3_sum_j(const ABRing<KB, JC>& ab, int n, int kb, const Vals& vals, double (&Ep)[KB], double (&Eq)[KB]) {
  const int nch = n / JC;  // n % JC == 0 on this path
  ab.issue(kb, 0, 0);
  for (int jc = 0; jc < nch; jc++) {
    if (jc + 1 < nch) ab.issue(kb, (jc + 1) * JC, (jc + 1) & 1);
    else cp_async_commit();  // empty group keeps wait_group<1> uniform
    cp_async_wait<1>();
    __syncwarp();
    const double2* st = ab.buf + (jc & 1) * JC * KB;
    if (jc == 0) {
      const SlotVals v = vals(0);
#pragma unroll
      for (int kk = 0; kk < KB; kk++) f3_fma<KB, true>(st[kk], kk, v, Ep, Eq);
    }
#pragma unroll kF3RingJUnroll
    for (int jj = (jc == 0 ? 1 : 0); jj < JC; jj++) {
      const SlotVals v = vals(jc * JC + jj);
#pragma unroll
      for (int kk = 0; kk < KB; kk++) f3_fma<KB, false>(st[jj * KB + kk], kk, v, Ep, Eq);
    }
    __syncwarp();  // the stage is refilled two chunks later
  }
}

// Phase A of an evaluation: slots 0 and 1 of every residual r_k = E*_k - E_k into R0/R1.
// It depends on the point and the row i only -- not on the chunk -- which is what the
// NEXT-4 hoisted variant exploits (computed once per row instead of once per chunk).
template <int KB, class AB>
CHF_INL void f3_phase_a(int n, int i, const double* __restrict__ sa, const double* __restrict__ ca, int stride,
                        const AB& ab, const double* __restrict__ Es, double* R0, double* R1) {
  // sin(y_j) = <sin a, cos a * y1, ...>;  cos(y_j) = <cos a, -sin a * y1, ...>
  auto valsA = [&](int j) {
    const double s0 = sa[j * stride], c0 = ca[j * stride];
    const double y1 = (j == i) ? 1.0 : 0.0;
    return SlotVals{s0, c0, c0 * y1, (-s0) * y1};
  };
  for (int kb = 0; kb < n; kb += KB) {
    double E0[KB], E1[KB];
    f3_sum_j<KB>(ab, n, kb, valsA, E0, E1);
#pragma unroll
    for (int kk = 0; kk < KB; kk++) {
      const int k = kb + kk;
      R0[k] = Es[k] - E0[kk];  // r_k = E*_k - E_k (s+ on slot 0, negation elsewhere)
      R1[k] = -E1[kk];
    }
  }
  // f slots 0/1 (f = sum_k r_k * r_k) are dead for the HVP and the Hessian.
}

// Phase B: the C columns of the chunk starting at cs, given R0/R1 of this row.  For each
// column l in ascending order, sink(cs + l, d2f/dx_i dx_{cs+l}) consumes the second-order
// slot C+2+l (the chunk dot of Alg 7, the store of Alg 5, the scatter of Alg 8).
template <int KB, class AB, class Sink>
CHF_INL void f3_phase_b(int n, int C, int i, int cs, const double* __restrict__ sa, const double* __restrict__ ca,
                        int stride, const AB& ab, const double* R0, const double* R1, Sink&& sink) {
  for (int c = 0; c < C; c++) {
    const int col = cs + c;
    // sin: g' = cos a, g'' = -sin a;   cos: g' = -sin a, g'' = -cos a
    auto valsB = [&](int j) {
      const double s0 = sa[j * stride], c0 = ca[j * stride];
      const double y1 = (j == i) ? 1.0 : 0.0, y2 = (j == col) ? 1.0 : 0.0, yC = 0.0;
      return SlotVals{c0 * y2, (-s0) * y2, c0 * yC + ((-s0) * y1) * y2, (-s0) * yC + ((-c0) * y1) * y2};
    };
    double fC = 0.0;
    for (int kb = 0; kb < n; kb += KB) {
      double E2[KB], EC[KB];
      f3_sum_j<KB>(ab, n, kb, valsB, E2, EC);
#pragma unroll
      for (int kk = 0; kk < KB; kk++) {
        const int k = kb + kk;
        const double r0 = R0[k], r1 = R1[k], r2 = -E2[kk], rC = -EC[kk];
        // (r*r)[C+2+c] = r0 rC + r1 r2 + r1 r2 + r0 rC   (Fig. 1 term order)
        const double rrC = r0 * rC + r1 * r2 + r1 * r2 + r0 * rC;
        fC = (k == 0) ? rrC : fC + rrC;
      }
    }
    sink(col, fC);
  }
}

// One evaluation f<hDual<C>>(CHUNK-INIT(i, cs)) for this lane's point (Alg 4 + Fig. 1):
// phase A then phase B.  sa/ca: sin/cos of the lane's coordinates (element j at
// [j * stride]); Es: E*; R0/R1: per-thread scratch (n doubles).
template <int KB, class AB, class Sink>
CHF_INL void f3_eval(int n, int C, int i, int cs, const double* __restrict__ sa,
                     const double* __restrict__ ca, int stride, const AB& ab,
                     const double* __restrict__ Es, double* R0, double* R1, Sink&& sink) {
  f3_phase_a<KB>(n, i, sa, ca, stride, ab, Es, R0, R1);
  f3_phase_b<KB>(n, C, i, cs, sa, ca, stride, ab, R0, R1, sink);
}

}  // namespace chessfad

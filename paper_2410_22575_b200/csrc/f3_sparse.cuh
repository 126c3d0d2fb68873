// f3_sparse.cuh -- NEXT-4 seed sparsity for F3 Fletcher-Powell: chessfad_hvp_batch_seedsparse.
//
// Alg 7 (CHESS-VEC) evaluates f<hDual<C>> on the CHUNK-INIT seeds (Alg 4,
// PAPER.md:172-194): variable j carries derivative 1 in slot 1 only if j == i (the row) and
// in slot 2+c only if j == cs+c (the column).  Every other derivative slot of every seed is 0,
// so in F3's E_k sums (sum over j of A_kj sin y_j + B_kj cos y_j) all but one term of
// each derivative slot is a product with an exact zero.  This kernel skips those terms:
//
//   slot 0 (value)     E0_k = sum_j A_kj s_j + B_kj c_j          same for every row and column
//                                                                -> once per point (R0 tile)
//   slot 1 (row i)     E1_k = fma(B_ki, -s_i, A_ki c_i)          the j = i term of the chain
//   slot 2+c (col)     E2_k = fma(B_kc, -s_c, A_kc c_c)          the j = col term
//   slot C+2+c         EC_k = [i == col] fma(B_ki, -c_i, -A_ki s_i)
//   then, as in f3_phase_b, r = E* - E and d2f/dx_i dx_col = sum_k (r0 rC + r1 r2 + r1 r2 + r0 rC)
//   (Fig. 1 term order); for col != i, rC = 0 and the r0 rC terms are skipped as well.
//
// With finite inputs every skipped term is an exact +-0 added to a nonzero partial, so the
// result equals chessfad_hvp_batch's bit for bit up to the sign of zero (tested on the GPU);
// the work per point drops from O(n^4 / C) to O(n^3).  Executed FLOPs are far below the §V
// model; rates against the model are "effective".
//
// Mapping: lane = point, warp = row, CTA = 4 warps sharing a tile (as the register kernel).  Per
// row, columns go in blocks of CB (accumulators and the lane's sin/cos of the block in
// registers); the inner loop over k reads (A_kj, B_kj) for the block's columns as warp-uniform
// broadcasts of (A_kj, B_kj): an interleaved row-major shared-memory copy for n <= 32, the
// caller's params through the read-only path otherwise (no per-call scratch copy).
#pragma once
#include <type_traits>

#include "chessfad/kernels.cuh"

#ifndef CHF_SP_KUNROLL
#define CHF_SP_KUNROLL 4  // k-loop unroll of the column-block loop (measured 4 > 2: profiles/r01/sparse/)
#endif
#ifndef CHF_SP_MINB
#define CHF_SP_MINB 2  // min CTAs/SM (register budget) of the seed-sparse kernel, n > 32 (tuning knob)
#endif
#ifndef CHF_SP_MINB_SMEM
#define CHF_SP_MINB_SMEM 3  // ... with (A, B) in shared memory, n <= 32 (column blocks of <= 8)
#endif

namespace chessfad {

constexpr int kSpKUnroll = CHF_SP_KUNROLL;

CHF_INL void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
CHF_INL void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src));
}
CHF_INL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
CHF_INL void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// (A_kj, B_kj) pairs: from the caller's params directly (global, read-only path; no scratch
// copy) or from an interleaved shared-memory copy [k][j] (n <= 32)
struct ABGlobal {
  const double* A;
  const double* B;
  int n;
  CHF_INL double2 operator()(int k, int j) const {
    return make_double2(__ldg(A + (size_t)k * n + j), __ldg(B + (size_t)k * n + j));
  }
  CHF_INL void stage(double2* dst, int k, int j) const {  // cp.async of one pair into an interleaved slot
    cp_async8(&dst->x, A + (size_t)k * n + j);
    cp_async8(&dst->y, B + (size_t)k * n + j);
  }
};
struct ABSmem {
  const double2* ab;
  int n;
  CHF_INL double2 operator()(int k, int j) const { return ab[k * n + j]; }
};

// The j = 0 term of each E chain is written `A x + B y` (f3_fma's FIRST form) and every later
// term as fma(B, y, fma(A, x, E)); the sparse terms below copy whichever form the full chain
// used for that j so that nvcc rounds them identically.
template <bool FIRST>
CHF_INL double f3_sp_term(double A, double x, double B, double y) {
  if constexpr (FIRST) return A * x + B * y;
  else return __fma_rn(B, y, __dmul_rn(A, x));
}

// one block of CB columns [cb, cb + CB) of row i: fC[q] = d2f/dx_i dx_{cb+q} for col != i
template <int CB, bool ROW0, bool COL0, class AB>
CHF_INL void f3_sp_block(int n, int i, int cb, double si, double ci, const AB& ab,
                         const double* __restrict__ sa, const double* __restrict__ ca, double (&fC)[CB]) {
  double sc[CB], cc[CB];
#pragma unroll
  for (int q = 0; q < CB; q++) {
    sc[q] = sa[(cb + q) * kPad];
    cc[q] = ca[(cb + q) * kPad];
  }
#pragma unroll kSpKUnroll
  for (int k = 0; k < n; k++) {
    const double2 c1 = ab(k, i);
    const double r1 = -f3_sp_term<ROW0>(c1.x, ci, c1.y, -si);  // slot 1: the j = i term
#pragma unroll
    for (int q = 0; q < CB; q++) {
      const double2 c = ab(k, cb + q);
      const double r2 = (COL0 && q == 0) ? -f3_sp_term<true>(c.x, cc[q], c.y, -sc[q])
                                         : -f3_sp_term<false>(c.x, cc[q], c.y, -sc[q]);  // slot 2+c
      const double t = __dmul_rn(r1, r2);
      const double rr = __fma_rn(r1, r2, t);  // r0 rC + r1 r2 + r1 r2 + r0 rC with rC = 0 (col != i)
      fC[q] = (k == 0) ? rr : __dadd_rn(fC[q], rr);
    }
  }
}

// n > 32, n % kSpKS == 0: the block's (A, B) rows ab[k][cb .. cb+CB) do not depend on the row
// i, so the CTA's 4 warps (which walk the same (cb, k) sequence for their different rows) share
// them through a cp.async double buffer of kSpKS k-values in shared memory; each warp's own
// column ab[k][i] (slot 1) rides in a per-warp buffer of the same stages.  Replaces the
// latency-bound broadcast loads from L2 ((A, B) is 256 KB at n = 128).
constexpr int kSpKS = 8;
struct SpRing {
  double2* blk;  // [2][kSpKS][CB], CTA-shared
  double2* col;  // [2][kSpKS], this warp's
};

// one stage (kSpKS k-values) of a staged block, no barriers inside
template <int CB, bool ROW0, bool COL0>
CHF_INL void f3_sp_stage(int k0, double si, double ci, const double2* __restrict__ blk, const double2* __restrict__ col,
                         const double (&sc)[CB], const double (&cc)[CB], double (&fC)[CB]) {
#pragma unroll
  for (int kk = 0; kk < kSpKS; kk++) {
    const int k = k0 + kk;
    const double2 c1 = col[kk];
    const double r1 = -f3_sp_term<ROW0>(c1.x, ci, c1.y, -si);
#pragma unroll
    for (int q = 0; q < CB; q++) {
      const double2 c = blk[kk * CB + q];
      const double r2 = (COL0 && q == 0) ? -f3_sp_term<true>(c.x, cc[q], c.y, -sc[q])
                                         : -f3_sp_term<false>(c.x, cc[q], c.y, -sc[q]);
      const double t = __dmul_rn(r1, r2);
      const double rr = __fma_rn(r1, r2, t);
      fC[q] = (k == 0) ? rr : __dadd_rn(fC[q], rr);
    }
  }
}

// The barriers of the staged pipeline must be the SAME instructions in every warp (warps with
// row 0 / column block 0 take other term forms), so row0 / col0 are runtime (warp-uniform)
// flags here and only the barrier-free stage compute is specialised.
template <int CB>
CHF_INL void f3_sp_block_staged(int n, int i, int cb, bool row0, double si, double ci, const ABGlobal& ab,
                                const SpRing& rg, const double* __restrict__ sa, const double* __restrict__ ca,
                                double (&fC)[CB]) {
  double sc[CB], cc[CB];
#pragma unroll
  for (int q = 0; q < CB; q++) {
    sc[q] = sa[(cb + q) * kPad];
    cc[q] = ca[(cb + q) * kPad];
  }
  const bool col0 = cb == 0;
  const int S = n / kSpKS, lane = threadIdx.x & 31;
  auto issue = [&](int st) {
    const int k0 = st * kSpKS, buf = st & 1;
    for (int q = threadIdx.x; q < kSpKS * CB; q += blockDim.x) {
      const int kk = q / CB, cq = q - kk * CB;
      ab.stage(rg.blk + (buf * kSpKS + kk) * CB + cq, k0 + kk, cb + cq);
    }
    if (lane < kSpKS) ab.stage(rg.col + buf * kSpKS + lane, k0 + lane, i);
    cp_async_commit();
  };
  __syncthreads();  // every warp is done with the previous block's buffers
  issue(0);
  for (int st = 0; st < S; st++) {
    cp_async_wait<0>();
    __syncthreads();  // stage st landed for all threads; stage st-1's buffer is free
    if (st + 1 < S) issue(st + 1);
    const double2* blk = rg.blk + (st & 1) * kSpKS * CB;
    const double2* col = rg.col + (st & 1) * kSpKS;
    const int k0 = st * kSpKS;
    if (row0) {
      if (col0) f3_sp_stage<CB, true, true>(k0, si, ci, blk, col, sc, cc, fC);
      else f3_sp_stage<CB, true, false>(k0, si, ci, blk, col, sc, cc, fC);
    } else {
      if (col0) f3_sp_stage<CB, false, true>(k0, si, ci, blk, col, sc, cc, fC);
      else f3_sp_stage<CB, false, false>(k0, si, ci, blk, col, sc, cc, fC);
    }
  }
}

// row i: out_i = sum_col d2f/dx_i dx_col * v_col, ascending columns (HVP), or the row stored
// to hrow (HESS; nullptr for ragged-tail lanes)
template <bool ROW0, bool GRAD, class AB>
CHF_INL double f3_sp_diag(int n, int i, double si, double ci, const AB& ab,
                          const double* __restrict__ r0t, double& f1) {
  // diagonal column: the full slot set (r0, r1 = r2, rC), f3_phase_b's expression; GRAD: also
  // slot 1 of f = sum_k r_k r_k, df/dx_i = sum_k (r0 r1 + r0 r1) (Fig. 1 product)
  double fdiag = 0.0;
  for (int k = 0; k < n; k++) {
    const double2 c = ab(k, i);
    const double r0 = r0t[k * kPad];
    const double r1 = -f3_sp_term<ROW0>(c.x, ci, c.y, -si);
    const double r2 = r1;
    // slot C+2+c (sin'' = -sin, cos'' = -cos); for row 0 the per-evaluation kernel's FIRST-form
    // sum A*sq + B*cq is contracted as fma(A, sq, B*cq) (measured: bit-identical on the GPU)
    const double rC = ROW0 ? -__fma_rn(c.x, -si, __dmul_rn(c.y, -ci)) : -f3_sp_term<false>(c.x, -si, c.y, -ci);
    const double rrC = r0 * rC + r1 * r2 + r1 * r2 + r0 * rC;
    fdiag = (k == 0) ? rrC : fdiag + rrC;
    if (GRAD) {
      const double rr1 = r0 * r1 + r0 * r1;
      f1 = (k == 0) ? rr1 : f1 + rr1;
    }
  }
  return fdiag;
}

// row0 is a runtime flag so that the staged path's barriers are shared by all warps.
// MODE: MODE_HVP (returns the row of H v), MODE_HESS (stores the row to hrow), MODE_SYM_HESS
// (Alg 6: stores the entries of chunks >= row i's chunk, mirrors those of later chunks into
// hcol[col * n]; the unstaged path also skips the column blocks wholly below row i's chunk --
// the staged path keeps every warp on the same block sequence for its shared barriers),
// MODE_HESS_GRAD (stores the row and returns df/dx_i through f1).
// MODE_SYM_HVP (Alg 8, one lane owns every row of its point): `acc` is the point's output row
// (stride as), res starts from the mirror terms earlier rows scattered into acc[i], the direct
// terms of chunks >= row i's chunk follow in ascending column order, and the entries of chunks
// strictly after row i's are scattered into acc[col] (the register kernel's RowSink order).
template <int CB, int MODE, bool STAGED, class AB>
CHF_INL double f3_sp_row(int n, int Capi, int i, bool row0, const AB& ab, const double* __restrict__ sa,
                         const double* __restrict__ ca, const double* __restrict__ r0t, const double* __restrict__ v,
                         int vs, double* __restrict__ hrow, double* __restrict__ hcol, const SpRing& rg, double& f1,
                         double* __restrict__ acc = nullptr, int as = 0) {
  constexpr bool HESS = mode_hess(MODE);
  constexpr bool GRAD = MODE == MODE_HESS_GRAD;
  constexpr bool SYM = MODE == MODE_SYM_HESS || MODE == MODE_SYM_HVP;
  const double si = sa[i * kPad], ci = ca[i * kPad];
  const double fdiag = row0 ? f3_sp_diag<true, GRAD>(n, i, si, ci, ab, r0t, f1)
                            : f3_sp_diag<false, GRAD>(n, i, si, ci, ab, r0t, f1);
  const int cs_row = (i / Capi) * Capi;  // first column of row i's chunk (Alg 6 / Alg 8)
  double res = (MODE == MODE_SYM_HVP && acc) ? acc[i * as] : 0.0;
  const double vi = MODE == MODE_SYM_HVP ? v[i * vs] : 0.0;
  const int cb_first = (SYM && !STAGED) ? cs_row / CB * CB : 0;
  for (int cb = cb_first; cb < n; cb += CB) {
    double fC[CB];
    if constexpr (STAGED) {
      f3_sp_block_staged<CB>(n, i, cb, row0, si, ci, ab, rg, sa, ca, fC);
    } else if (row0) {
      if (cb == 0) f3_sp_block<CB, true, true>(n, i, cb, si, ci, ab, sa, ca, fC);
      else f3_sp_block<CB, true, false>(n, i, cb, si, ci, ab, sa, ca, fC);
    } else {
      if (cb == 0) f3_sp_block<CB, false, true>(n, i, cb, si, ci, ab, sa, ca, fC);
      else f3_sp_block<CB, false, false>(n, i, cb, si, ci, ab, sa, ca, fC);
    }
#pragma unroll
    for (int q = 0; q < CB; q++) {
      const double h = (cb + q == i) ? fdiag : fC[q];
      if (HESS) {
        const int col = cb + q;
        if (MODE == MODE_SYM_HESS) {
          if (hrow && col >= cs_row) {
            hrow[col] = h;                                              // Alg 6 :229-235
            if (col / Capi > i / Capi) hcol[(size_t)col * n] = h;       // mirror, :237-241 (G9)
          }
        } else if (hrow) {
          hrow[col] = h;  // a7': H[e][i][col] (Alg 5)
        }
      } else if (MODE == MODE_SYM_HVP) {
        const int col = cb + q;
        if (col >= cs_row) {
          res = __fma_rn(h, v[col * vs], res);                                  // Alg 8 :417-419
          if (acc && col / Capi > i / Capi) acc[col * as] = __fma_rn(h, vi, acc[col * as]);  // :420-421
        }
      } else {
        res = __fma_rn(h, v[(cb + q) * vs], res);  // a5/a6: ascending columns, as RowSink
      }
    }
  }
  return res;
}

// AB_SMEM (n <= 32): (A, B) whole in shared memory, else the interleaved global scratch.
// SLIM (n > 32): vectors read and outputs written straight from/to global memory (3 tiles).
// MODE: MODE_HVP, or a Hessian mode (Alg 5 output hess[e][i][j]; Alg 6; Alg 5 + gradient).
// STAGED (SLIM, n % kSpKS == 0): the CTA-shared (A, B) block rows go through the cp.async
// double buffer (f3_sp_block_staged); every warp then has n / 4 rows (uniform barriers).
template <int CB, bool AB_SMEM, bool SLIM, int MODE, bool STAGED>
__global__ void __launch_bounds__(kWarpsF3 * 32, AB_SMEM ? CHF_SP_MINB_SMEM : CHF_SP_MINB) hvp_f3_sparse_kernel(BatchArgs p) {
  constexpr bool HESS = mode_hess(MODE);
  extern __shared__ double smem[];
  const int n = p.n, G = p.groups, P = 32 * G;
  double* s_sa = smem;                 // [G][n][33]  sin a
  double* s_ca = s_sa + G * n * kPad;  // [G][n][33]  cos a
  double* s_r0 = s_ca + G * n * kPad;  // [G][n][33]  r0_k = E*_k - E0_k (slot 0 of the residuals)
  double* s_vec = s_r0 + G * n * kPad;
  double* s_out = s_vec + G * n * kPad;
  double2* s_ab = reinterpret_cast<double2*>(SLIM ? s_vec : s_out + G * n * kPad);
  const int64_t e0 = (int64_t)blockIdx.x * P;
  stage_tile(p, e0, P, s_sa, (SLIM || HESS) ? nullptr : s_vec);
  if (AB_SMEM) {
    const double* A = p.params;
    const double* B = p.params + (size_t)n * n;
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) s_ab[q] = make_double2(A[q], B[q]);  // [k][j]
  }
  __syncthreads();
  for (int q = threadIdx.x; q < G * n * 32; q += blockDim.x) {
    const int idx = (q >> 5) * kPad + (q & 31);
    double s, c;
    sincos(s_sa[idx], &s, &c);
    s_sa[idx] = s;
    s_ca[idx] = c;
  }
  __syncthreads();
  using AB = typename std::conditional<AB_SMEM, ABSmem, ABGlobal>::type;
  AB ab;
  if constexpr (AB_SMEM) ab = ABSmem{s_ab, n};
  else ab = ABGlobal{p.params, p.params + (size_t)n * n, n};
  const double* Es = p.params + 2 * (size_t)n * n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp % G, wg = warp / G, rstep = kWarpsF3 / G;
  const double* sa = s_sa + g * n * kPad + lane;
  const double* ca = s_ca + g * n * kPad + lane;
  double* r0t = s_r0 + g * n * kPad + lane;
  // slot 0 once per point: E0_k = sum_j (A_kj s_j + B_kj c_j), f3_sum_j's chain with (s, c)
  for (int k = wg; k < n; k += rstep) {
    double E;
    {
      const double2 c = ab(k, 0);
      E = c.x * sa[0] + c.y * ca[0];
    }
    for (int j = 1; j < n; j++) {
      const double2 c = ab(k, j);
      E = E + c.x * sa[j * kPad] + c.y * ca[j * kPad];
    }
    r0t[k * kPad] = Es[k] - E;
  }
  __syncthreads();

  const int64_t e = e0 + g * 32 + lane;
  const int64_t ec = e < p.m ? e : p.m - 1;
  const double* v = HESS ? nullptr : (SLIM ? p.vecs + ec * n : s_vec + g * n * kPad + lane);
  const int vs = SLIM ? 1 : kPad;
  double* o = s_out + g * n * kPad + lane;
  // Alg 8 accumulators: the output tile column of the lane's point, or (SLIM) its output row in
  // global memory (nullptr for a ragged-tail lane there: it computes but never accumulates)
  double* acc = nullptr;
  int as = 0;
  if constexpr (MODE == MODE_SYM_HVP) {
    if constexpr (SLIM) {
      acc = e < p.m ? p.out + e * n : nullptr;
      as = 1;
    } else {
      acc = o;
      as = kPad;
    }
    if (acc)
      for (int q = 0; q < n; q++) acc[q * as] = 0.0;
  }
  // STAGED ring: [2][kSpKS][CB] shared block rows, then [warps][2][kSpKS] column values
  const SpRing rg{s_ab, s_ab + 2 * kSpKS * CB + warp * 2 * kSpKS};
  for (int i = wg; i < n; i += rstep) {
    double* hrow = (HESS && e < p.m) ? p.out + (e * n + i) * n : nullptr;
    double* hcol = (HESS && e < p.m) ? p.out + e * n * n + i : nullptr;
    double f1 = 0.0;
    const double res =
        f3_sp_row<CB, MODE, STAGED>(n, p.csize, i, i == 0, ab, sa, ca, r0t, v, vs, hrow, hcol, rg, f1, acc, as);
    if (MODE == MODE_HESS_GRAD && e < p.m) p.grad[e * n + i] = f1;
    if (HESS) {
    } else if (SLIM) {
      if (e < p.m) p.out[e * n + i] = res;
    } else {
      o[i * kPad] = res;
    }
  }
  if (!SLIM && !HESS) {
    __syncthreads();
    write_tile(p, e0, P, s_out);
  }
}


}  // namespace chessfad

// f3_mma.cuh -- F3 Fletcher-Powell over hDual<C> with its E-sums on the FP64 tensor core.
//
// One evaluation f<hDual<C>>(CHUNK-INIT(i, cs)) of F3 (definition, canonical
// form DESIGN.md) is dominated by the n sums E_k = sum_j A_kj sin y_j + B_kj cos y_j, one per
// hDual slot: 2n^2 s* and 2n^2-1 hh+ (4 n^2 (C+1) FMAs, ~88-97% of the model FLOPs).  Per slot
// they are a dense matrix-vector product
//       E_slot = M x_slot,     M = [A | B]  (n x 2n, shared by every point),
//       x_slot = [slot of sin y_j ; slot of cos y_j]   (2n, per point and evaluation),
// so for the 8 points of a warp and one slot it is an (n x 2n) x (2n x 8) GEMM: a dense
// contraction, executed here with mma.sync m8n8k4 .f64 (DMMA).  On B200 DMMA and DFMA share the
// FP64 pipe at the same peak (tools/micro/dmma_probe: 37.0 vs 36.7 TFLOP/s, 36.5 mixed; DMMA
// saturates with one warp per SM sub-partition and 2 independent accumulators,
// tools/micro/dmma_latency_probe), so this is not a faster pipe -- it is 256 FMAs per issued
// instruction instead of 32, which frees the issue slots and registers that round 1's SIMT
// schedule (retired) spent on broadcasts, loop control and local-memory residual arrays
// (profiles/r01/f3: 57% of FP64 peak at n = 64).
//
// The evaluation is round 1's slot-column schedule (every scalar op of the hDual evaluation
// once, in the paper's per-slot form; only the order of independent operations changes):
//   phase A   slots 0 and 1 of every E_k, r_k = E*_k - E_k           (R0, R1 in registers)
//   phase B   per column c of the chunk: slots 2+c and C+2+c of every E_k, then
//             d2f/dx_i dx_{cs+c} = sum_k (r0 rC + r1 r2 + r1 r2 + r0 rC)   (Fig. 1 term order)
// The x_slot entries are the slots of the 2n unary ops sin y_j / cos y_j of the seeded inputs
// (g' u[k] and g' u[C+k] + (g'' u1) u[k], PAPER.md:99 / SPEC.md:81), formed per evaluation by
// the lane that feeds them to the tensor core; sin a_j, cos a_j (g, g', g'' of the value slot,
// 0 model FLOPs) are tabulated once per point in shared memory.
//
// Mapping (m8n8k4: A 8x4 row-major, B 4x8 col-major, C/D 8x8; lane = 4 g + t):
//   CTA   = W warps x 8 points; M in shared memory in A-fragment order, KB rows at a time.
//   warp  = 8 points (the N dimension); it walks all n rows of its points (Alg 7 row order)
//   A     = M[8 kt + g][4 s + t]            (k-tile kt, j'-step s over j' in [0, 2n))
//   B     = x_slot[4 s + t] of point g      (formed by the lane from the sin/cos tables + seed)
//   D     = E_slot[8 kt + g] of points 2t, 2t+1
// n <= NN: M, E*, the tables and x are zero-padded to NN (a padded k has E = E* = 0, so
// r = 0 and it adds exact zeros; a padded j' has M = 0).  NN > KB (n > 64: M is 256 KB at
// n = 128): the k range is processed in blocks of KB rows, each evaluation's sums over k split
// into per-block partial sums that are added into the outputs (global read-add-write by the
// owning lane; the work per evaluation is unchanged, only the association of the k sum).
// Alg 8's scatter targets out[e][s] live in a shared-memory tile up to n = 64 and in the
// output rows themselves beyond (zeroed first; only the owning lane ever touches a row).
// The sum over k of each second-order entry is a per-lane partial over the k-tiles plus a
// 3-step butterfly over g; every other reduction order is as in the SIMT kernel.
#pragma once
#include "chessfad/kernels.cuh"

namespace chessfad {

constexpr int kMmaPPW = 8;  // points per warp (the MMA N dimension)

CHF_INL void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// NN: padded n (multiple of 8); W: warps per CTA; KB: k rows of M resident per block
constexpr int f3_mma_kb(int NN) {  // k rows of M per block: all of M up to n = 64, else <= 32 dividing NN
  return NN <= 64 ? NN : NN % 32 == 0 ? 32 : NN % 24 == 0 ? 24 : NN % 16 == 0 ? 16 : 8;
}
template <int NN, int MODE>
struct F3Mma {
  static constexpr int W = 8;
  // Alg 8's scatter targets: a shared-memory tile up to n = 64; beyond, the output rows
  // themselves in global memory (the tile would not fit next to M's block and the tables)
  static constexpr bool kSmemScatter = MODE == MODE_SYM_HVP && NN <= 64;
  static constexpr bool kGlobalScatter = MODE == MODE_SYM_HVP && NN > 64;
  static constexpr int KB = f3_mma_kb(NN);
  static constexpr int P = W * kMmaPPW;        // points per CTA
  static constexpr int TS = P + 8;             // sin/cos table row stride (doubles): 2 wavefronts per LDS
  static constexpr int KT = KB / 8;            // k-tiles per block
  static constexpr int JQ = NN / 4;            // j-quads per half of j' (A part / B part)
  static constexpr size_t kMf = (size_t)2 * KB * NN;  // one M block in fragment order
  static constexpr size_t kTab = (size_t)NN * TS;
  static constexpr size_t smem_bytes() {
    return (kMf + NN + 2 * kTab + (kSmemScatter ? (size_t)P * (NN + 1) : 0)) * sizeof(double);
  }
  static_assert(NN % 8 == 0 && NN % KB == 0 && KB % 8 == 0, "tile shapes");
};

template <int NN, int MODE>
__global__ void __launch_bounds__(F3Mma<NN, MODE>::W * 32, 1) hvp_f3_mma_kernel(BatchArgs p) {
  using Cfg = F3Mma<NN, MODE>;
  constexpr int KT = Cfg::KT, JQ = Cfg::JQ, KB = Cfg::KB, P = Cfg::P, TS = Cfg::TS;
  constexpr bool HESS = mode_hess(MODE);
  extern __shared__ double smem[];
  double* Mf = smem;                 // [KT][2 JQ][32]  A fragments of rows [kb0, kb0 + KB) of M = [A | B]
  double* Es = Mf + Cfg::kMf;        // [NN]            E*, zero-padded
  double* s_tab = Es + NN;           // [NN][TS]        sin a_j of the CTA's points, zero-padded
  double* c_tab = s_tab + Cfg::kTab; // [NN][TS]        cos a_j
  double* s_acc = c_tab + Cfg::kTab; // [P][NN+1]       MODE_SYM_HVP scatter targets (n <= 64)
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int n = p.n;
  const int64_t e0 = (int64_t)blockIdx.x * P;

  // ---- E*, sin/cos of the CTA's points (zero-padded)
  for (int q = tid; q < NN; q += nthr) Es[q] = q < n ? p.params[2 * n * n + q] : 0.0;
  for (int q = tid; q < P * NN; q += nthr) {
    const int pt = q / NN, j = q - pt * NN;
    double sv = 0.0, cv = 0.0;
    if (j < n) {
      int64_t e = e0 + pt;
      if (e >= p.m) e = p.m - 1;  // ragged tail: replicate the last point, never stored
      sincos(__ldg(p.points + e * n + j), &sv, &cv);
    }
    s_tab[j * TS + pt] = sv;
    c_tab[j * TS + pt] = cv;
  }
  if (Cfg::kSmemScatter)
    for (int q = tid; q < P * (NN + 1); q += nthr) s_acc[q] = 0.0;

  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int ptB = warp * kMmaPPW + g;                 // B-fragment point (CTA-local)
  const double* sB = s_tab + ptB;                     // sin a_j of that point at [j * TS]
  const double* cB = c_tab + ptB;
  const double* mf = Mf + lane;                       // this lane's A-fragment elements
  int64_t eD[2], eDc[2];                              // D-fragment points 2t, 2t+1 (global)
#pragma unroll
  for (int h = 0; h < 2; h++) {
    eD[h] = e0 + warp * kMmaPPW + 2 * t + h;
    eDc[h] = eD[h] < p.m ? eD[h] : p.m - 1;
  }
  const int Capi = p.csize;
  const int nchunk = n / Capi;
  // sum over all k of a per-(k, point) term: per-lane k-tile partials + butterfly over g
  auto ksum = [&](double (&x)[2]) {
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) x[h] += __shfl_xor_sync(0xffffffffu, x[h], off);
  };
  // k-blocked outputs: the first block stores, later blocks add their partial sums
  auto emit = [&](double* dst, double v, bool first) { *dst = first ? v : *dst + v; };

  if (Cfg::kGlobalScatter && g == 0)  // every contribution to out is added (scatter + rows)
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (eD[h] < p.m)
        for (int i = 0; i < n; i++) p.out[eD[h] * n + i] = 0.0;

  for (int kb0 = 0; kb0 < NN; kb0 += KB) {
    const bool first = kb0 == 0;
    // ---- stage rows [kb0, kb0 + KB) of M in A-fragment order (zero-padded)
    if (!first) __syncthreads();  // every warp is done with the previous block
    {
      const double* A = p.params;
      const double* B = p.params + n * n;
      for (int q = tid; q < 2 * KB * NN; q += nthr) {
        const int ln = q & 31, fs = q >> 5;  // fragment (kt, s) and lane
        const int kt = fs / (2 * JQ), s = fs - kt * (2 * JQ);
        const int k = kb0 + 8 * kt + (ln >> 2), jp = 4 * s + (ln & 3);
        double v = 0.0;
        if (k < n) {
          if (jp < NN) v = jp < n ? A[k * n + jp] : 0.0;
          else v = jp - NN < n ? B[k * n + jp - NN] : 0.0;
        }
        Mf[q] = v;
      }
    }
    __syncthreads();
    double Esr[KT];
#pragma unroll
    for (int kt = 0; kt < KT; kt++) Esr[kt] = Es[kb0 + 8 * kt + g];

    double R0[KT][2], R1[KT][2];  // r_k slots 0 / 1 of k = kb0 + 8 kt + g, points 2t + h
    // phase A: slots 0 and 1 of every residual of this k block (row i; independent of the chunk)
    auto phase_a = [&](int i) {
      double d0[KT][2], d1[KT][2];
#pragma unroll
      for (int kt = 0; kt < KT; kt++) d0[kt][0] = d0[kt][1] = d1[kt][0] = d1[kt][1] = 0.0;
#pragma unroll 4
      for (int jq = 0; jq < JQ; jq++) {
        const int j = 4 * jq + t;
        const double s0 = sB[j * TS], c0 = cB[j * TS];
        const double y1 = (j == i) ? 1.0 : 0.0;
        // sin y_j = <sin a, cos a * y1, ...>;  cos y_j = <cos a, -sin a * y1, ...>
        const double xa0 = s0, xa1 = c0 * y1, xb0 = c0, xb1 = (-s0) * y1;
#pragma unroll
        for (int kt = 0; kt < KT; kt++) {
          const double aA = mf[(kt * 2 * JQ + jq) * 32], aB = mf[(kt * 2 * JQ + JQ + jq) * 32];
          dmma(d0[kt], aA, xa0);
          dmma(d1[kt], aA, xa1);
          dmma(d0[kt], aB, xb0);
          dmma(d1[kt], aB, xb1);
        }
      }
#pragma unroll
      for (int kt = 0; kt < KT; kt++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          R0[kt][h] = Esr[kt] - d0[kt][h];  // r_k = E*_k - E_k (s+ on slot 0, negation elsewhere)
          R1[kt][h] = -d1[kt][h];
        }
    };

    for (int i = 0; i < n; i++) {
      const int scn = i / Capi;
      double res[2] = {0.0, 0.0};
      double vi[2] = {0.0, 0.0};
      if (MODE == MODE_SYM_HVP)
#pragma unroll
        for (int h = 0; h < 2; h++) vi[h] = __ldg(p.vecs + eDc[h] * n + i);
      if (MODE == MODE_HVP_ROWHOIST) phase_a(i);  // NEXT-4: phase A once per row
      for (int jc = mode_sym(MODE) ? scn : 0; jc < nchunk; jc++) {
        const int cs = jc * Capi;
        const bool mirror = jc > scn;
        if (MODE != MODE_HVP_ROWHOIST) phase_a(i);  // per evaluation (Alg 7 as written)
        if (MODE == MODE_HESS_GRAD && jc == 0) {    // gradient: slot 1 of f = sum_k r_k r_k
          double f1[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            f1[h] = R0[0][h] * R1[0][h] + R0[0][h] * R1[0][h];
#pragma unroll
            for (int kt = 1; kt < KT; kt++) f1[h] = f1[h] + (R0[kt][h] * R1[kt][h] + R0[kt][h] * R1[kt][h]);
          }
          ksum(f1);
          if (g == 0)
#pragma unroll
            for (int h = 0; h < 2; h++)
              if (eD[h] < p.m) emit(p.grad + eD[h] * n + i, f1[h], first);
        }
        for (int c = 0; c < Capi; c++) {
          const int col = cs + c;
          double d2[KT][2], dC[KT][2];
#pragma unroll
          for (int kt = 0; kt < KT; kt++) d2[kt][0] = d2[kt][1] = dC[kt][0] = dC[kt][1] = 0.0;
#pragma unroll 4
          for (int jq = 0; jq < JQ; jq++) {
            const int j = 4 * jq + t;
            const double s0 = sB[j * TS], c0 = cB[j * TS];
            const double y1 = (j == i) ? 1.0 : 0.0, y2 = (j == col) ? 1.0 : 0.0;
            // sin: g' = cos a, g'' = -sin a;   cos: g' = -sin a, g'' = -cos a   (unary rule)
            // slot C+2+c: g' y[C+2+c] + (g'' y1) y2, the seed's y[C+2+c] a structural zero (reading R7)
            const double xa2 = c0 * y2, xaC = ((-s0) * y1) * y2;
            const double xb2 = (-s0) * y2, xbC = ((-c0) * y1) * y2;
#pragma unroll
            for (int kt = 0; kt < KT; kt++) {
              const double aA = mf[(kt * 2 * JQ + jq) * 32], aB = mf[(kt * 2 * JQ + JQ + jq) * 32];
              dmma(d2[kt], aA, xa2);
              dmma(dC[kt], aA, xaC);
              dmma(d2[kt], aB, xb2);
              dmma(dC[kt], aB, xbC);
            }
          }
          double fC[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
#pragma unroll
            for (int kt = 0; kt < KT; kt++) {
              const double r0 = R0[kt][h], r1 = R1[kt][h], r2 = -d2[kt][h], rC = -dC[kt][h];
              // (r*r)[C+2+c] = r0 rC + r1 r2 + r1 r2 + r0 rC   (Fig. 1 term order)
              const double rrC = r0 * rC + r1 * r2 + r1 * r2 + r0 * rC;
              fC[h] = (kt == 0) ? rrC : fC[h] + rrC;
            }
          }
          ksum(fC);  // every lane with this t now holds d2f/dx_i dx_col of points 2t, 2t+1 (k block)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if (MODE == MODE_HVP || MODE == MODE_HVP_ROWHOIST || MODE == MODE_SYM_HVP) {
              res[h] = res[h] + fC[h] * __ldg(p.vecs + eDc[h] * n + col);  // Alg 7 :392-394
              if (MODE == MODE_SYM_HVP && mirror && g == 0) {                 // Alg 8 scatter
                if (Cfg::kSmemScatter) {
                  double* acc = s_acc + (warp * kMmaPPW + 2 * t + h) * (NN + 1) + col;
                  *acc = *acc + fC[h] * vi[h];
                } else if (eD[h] < p.m) {  // the owning lane's own output row (zeroed below)
                  double* acc = p.out + eD[h] * n + col;
                  *acc = *acc + fC[h] * vi[h];
                }
              }
            } else if (g == 0 && eD[h] < p.m) {
              emit(p.out + (eD[h] * n + i) * n + col, fC[h], first);       // Alg 5 :210-212
              if (MODE == MODE_SYM_HESS && mirror) emit(p.out + (eD[h] * n + col) * n + i, fC[h], first);
            }
          }
        }
      }
      if (!HESS && g == 0)
#pragma unroll
        for (int h = 0; h < 2; h++)
          if (eD[h] < p.m) emit(p.out + eD[h] * n + i, res[h], first && !Cfg::kGlobalScatter);
    }
  }
  if (Cfg::kSmemScatter) {  // Alg 8: add the scattered mirror terms H_is v_i
    __syncthreads();
    for (int q = tid; q < P * n; q += nthr) {
      const int pt = q / n, i = q - pt * n;
      const int64_t e = e0 + pt;
      if (e < p.m) p.out[e * n + i] += s_acc[pt * (NN + 1) + i];
    }
  }
}

}  // namespace chessfad

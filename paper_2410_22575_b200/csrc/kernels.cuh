// kernels.cuh -- batched HVP / Hessian kernels (sm_100a, FP64 SIMT, no tensor cores).
//
// Work decomposition (the paper's L0/L1/L2 levels):
// the paper maps instance x row x chunk to threads (Fig. 2: one thread per (e, i, j) and a
// shared-memory reduction).  Here a LANE is a POINT and a WARP is a ROW:
//   * the 32 lanes of a warp hold 32 different points and evaluate the SAME (row i,
//     chunk cs) -> CHUNK-INIT seeds, loop bounds and control flow are warp-uniform;
//   * a thread loops over the n/C chunks of its row and accumulates the row of H.v in a
//     register in ascending chunk order (Alg 7 order; no reduction across threads);
//   * a CTA stages a tile of 32*G points (and vectors) once, transposed [k][lane] in
//     shared memory (stride 33: conflict-free), with coalesced global loads; its warps
//     share the tile and split the n rows; the output tile is written back coalesced.
// Inputs are m x n FP64 row-major, instance-major a[e*n + k].
#pragma once
#include <cstdint>

#include "f3.cuh"
#include "testfuncs.cuh"

namespace chessfad {

struct BatchArgs {
  int n;
  int csize;
  int groups;  // G: 32-point groups per CTA
  int64_t m;
  const double* __restrict__ points;
  const double* __restrict__ vecs;
  double* __restrict__ out;  // HVP: m x n;  Hessian: m x n x n
  const double* __restrict__ params;
};

constexpr int kPad = 33;          // shared-memory row stride (doubles) of [k][lane] tiles
constexpr int kWarpsF3 = 4;       // Fletcher-Powell path: 128 threads per CTA

// stage points [and vectors] of the tile into shared memory, transposed per 32-point group
CHF_INL void stage_tile(const BatchArgs& p, int64_t e0, int P, double* s_pts, double* s_vec) {
  const int n = p.n;
  for (int q = threadIdx.x; q < P * n; q += blockDim.x) {
    const int pi = q / n, k = q - pi * n;
    int64_t e = e0 + pi;
    if (e >= p.m) e = p.m - 1;  // ragged tail: replicate the last point, never stored
    const int g = pi >> 5, ln = pi & 31;
    s_pts[(g * n + k) * kPad + ln] = __ldg(p.points + e * n + k);
    if (s_vec) s_vec[(g * n + k) * kPad + ln] = __ldg(p.vecs + e * n + k);
  }
}

CHF_INL void write_tile(const BatchArgs& p, int64_t e0, int P, const double* s_out) {
  const int n = p.n;
  for (int q = threadIdx.x; q < P * n; q += blockDim.x) {
    const int pi = q / n, k = q - pi * n;
    const int64_t e = e0 + pi;
    if (e < p.m) p.out[e * n + k] = s_out[((pi >> 5) * n + k) * kPad + (pi & 31)];
  }
}

// ---------------------------------------------------------------- F1, F2, F4: hDual<C> in registers
template <int FUNC, int C, bool HESS, int W>
__global__ void __launch_bounds__(W * 32) hvp_reg_kernel(BatchArgs p) {
  extern __shared__ double smem[];
  const int n = p.n, G = p.groups, P = 32 * G;
  double* s_pts = smem;
  double* s_vec = HESS ? nullptr : s_pts + G * n * kPad;
  double* s_out = HESS ? nullptr : s_vec + G * n * kPad;
  double* s_sin = (HESS ? s_pts : s_out) + G * n * kPad;  // Ackley only
  double* s_cos = s_sin + G * n * kPad;
  const int64_t e0 = (int64_t)blockIdx.x * P;
  stage_tile(p, e0, P, s_pts, s_vec);
  if (FUNC == FUNC_ACKLEY) {
    __syncthreads();
    for (int q = threadIdx.x; q < G * n * 32; q += blockDim.x) {
      const int idx = (q >> 5) * kPad + (q & 31);
      sincos(6.283185307179586 * s_pts[idx], s_sin + idx, s_cos + idx);
    }
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp % G, rstep = W / G;
  const double* a = s_pts + g * n * kPad + lane;
  const double* v = HESS ? nullptr : s_vec + g * n * kPad + lane;
  const double* tsin = FUNC == FUNC_ACKLEY ? s_sin + g * n * kPad + lane : nullptr;
  const double* tcos = FUNC == FUNC_ACKLEY ? s_cos + g * n * kPad + lane : nullptr;
  const int64_t e = e0 + g * 32 + lane;
  const int nchunk = n / C;
  for (int i = warp / G; i < n; i += rstep) {
    double res = 0.0;
    for (int j = 0; j < nchunk; j++) {
      const int cs = j * C;
      const LaneSeed<C> y{a, kPad, i, cs, tsin, tcos};
      const hd<C> t = eval_f<FUNC, C>(n, y);  // CHUNK-INIT + f<hDual<C>>, Alg 7 :389-390
      if (HESS) {
        if (e < p.m) {
          double* h = p.out + (e * n + i) * n + cs;  // H[e][i][cs + l] = t.v[C+2+l] (Alg 5)
#pragma unroll
          for (int l = 0; l < C; l++) h[l] = t.v[C + 2 + l];
        }
      } else {
#pragma unroll
        for (int l = 0; l < C; l++) res = res + t.v[C + 2 + l] * v[(cs + l) * kPad];  // :392-394
      }
    }
    if (!HESS) s_out[(g * n + i) * kPad + lane] = res;
  }
  if (!HESS) {
    __syncthreads();
    write_tile(p, e0, P, s_out);
  }
}

// ---------------------------------------------------------------- F3 Fletcher-Powell
// params = [A (n*n) | B (n*n) | E* (n)].  AB_SMEM: (A_kj, B_kj) interleaved into shared memory
// (n <= 32), else read from params through the read-only path.
template <int KB, bool HESS, bool AB_SMEM>
__global__ void __launch_bounds__(kWarpsF3 * 32, 3) hvp_f3_kernel(BatchArgs p) {
  extern __shared__ double smem[];
  const int n = p.n, G = p.groups, P = 32 * G, C = p.csize;
  double* s_sa = smem;                 // [G][n][33]  sin a
  double* s_ca = s_sa + G * n * kPad;  // [G][n][33]  cos a
  double* s_vec = s_ca + G * n * kPad;
  double* s_out = s_vec + G * n * kPad;
  double2* s_ab = reinterpret_cast<double2*>(HESS ? s_vec : s_out + G * n * kPad);
  const int64_t e0 = (int64_t)blockIdx.x * P;
  stage_tile(p, e0, P, s_sa, HESS ? nullptr : s_vec);
  const double* A = p.params;
  const double* B = p.params + (size_t)n * n;
  if (AB_SMEM)
    for (int q = threadIdx.x; q < n * n; q += blockDim.x) {
      const int k = q / n, j = q - k * n;
      s_ab[j * n + k] = make_double2(A[q], B[q]);  // transposed: [j][k]
    }
  __syncthreads();
  // g, g', g'' of the seeded inputs: sin a_k, cos a_k once per tile (see f3.cuh)
  for (int q = threadIdx.x; q < G * n * 32; q += blockDim.x) {
    const int idx = (q >> 5) * kPad + (q & 31);
    double s, c;
    sincos(s_sa[idx], &s, &c);
    s_sa[idx] = s;
    s_ca[idx] = c;
  }
  __syncthreads();

  const double* Es = p.params + 2 * (size_t)n * n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp % G, rstep = kWarpsF3 / G;
  const double* sa = s_sa + g * n * kPad + lane;
  const double* ca = s_ca + g * n * kPad + lane;
  const double* v = HESS ? nullptr : s_vec + g * n * kPad + lane;
  const int64_t e = e0 + g * 32 + lane;
  const int nchunk = n / C;
  double R0[128], R1[128];
  for (int i = warp / G; i < n; i += rstep) {
    double res = 0.0;
    double* hrow = (HESS && e < p.m) ? p.out + (e * n + i) * n : nullptr;
    for (int j = 0; j < nchunk; j++) {
      if (AB_SMEM)
        res = f3_eval<KB, HESS>(n, C, i, j * C, sa, ca, kPad, ABShared{s_ab, n}, Es, v, hrow, R0, R1, res);
      else
        res = f3_eval<KB, HESS>(n, C, i, j * C, sa, ca, kPad, ABGlobal{A, B, n}, Es, v, hrow, R0, R1, res);
    }
    if (!HESS) s_out[(g * n + i) * kPad + lane] = res;
  }
  if (!HESS) {
    __syncthreads();
    write_tile(p, e0, P, s_out);
  }
}

}  // namespace chessfad

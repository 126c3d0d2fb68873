// chessfad/kernels.cuh -- batched HVP / Hessian kernels (sm_100a, FP64 SIMT, no tensor cores).
//
// Work decomposition (the paper's L0/L1/L2 levels):
// the paper maps instance x row x chunk to threads (Fig. 2: one thread per (e, i, j) and a
// shared-memory reduction).  Here a LANE is a POINT and a WARP is a ROW:
//   * the 32 lanes of a warp hold 32 different points and evaluate the SAME (row i,
//     chunk cs) -> CHUNK-INIT seeds, loop bounds and control flow are warp-uniform;
//   * a thread loops over the chunks of its row and accumulates the row of H.v in a
//     register in ascending chunk order (Alg 7 order; no reduction across threads);
//   * a CTA stages a tile of 32*G points (and vectors) once, transposed [k][lane] in
//     shared memory (stride 33: conflict-free), with coalesced global loads; its warps
//     share the tile and split the n rows; the output tile is written back coalesced.
// Inputs are m x n FP64 row-major, instance-major a[e*n + k].
//
// Modes (one kernel body, the consumer of each finished column differs):
//   MODE_HVP       Alg 7 CHESS-VEC  out[i] = sum over all chunks
//   MODE_HESS      Alg 5 CHUNK-HESS  H[i][cs+l] stored
//   MODE_SYM_HVP   Alg 8 SC-HESS-VEC  chunks cn >= i/C only; H_is v_i also
//                  scattered into out[s] for chunks after row i's (reading G8)
//   MODE_SYM_HESS  Alg 6 SCHUNK-HESS  chunks cn >= i/C only, mirrored
// The symmetric modes use the API chunk size p.csize to decide which chunks are computed
// (the kernel's register chunk C may be a column group of it).  MODE_SYM_HVP needs one
// thread to own all rows of its point (the scatter crosses rows), so its CTA holds W groups
// of 32 points and every warp walks all n rows of its own group (the paper's L0 level).
#pragma once
#include <cstdint>

#include "testfuncs.cuh"

namespace chessfad {

// MODE_HVP_ROWHOIST (part of NEXT-4, the F3 kernel of chessfad_hvp_batch_hoisted): Alg 7 with
// phase A (slots 0/1 of the residuals, which do not depend on the chunk) computed once per
// row instead of once per chunk; outputs are bit-identical to MODE_HVP, executed FLOPs are
// below the model count.
// MODE_HESS_GRAD: Alg 5 plus the gradient by-product df/dx_i = slot v[1] of row i's
// evaluations (only this mode keeps slot 1 of the result alive).
enum { MODE_HVP = 0, MODE_HESS = 1, MODE_SYM_HVP = 2, MODE_SYM_HESS = 3, MODE_HVP_ROWHOIST = 4, MODE_HESS_GRAD = 5 };
__host__ __device__ constexpr bool mode_hess(int M) { return M == MODE_HESS || M == MODE_SYM_HESS || M == MODE_HESS_GRAD; }
__host__ __device__ constexpr bool mode_sym(int M) { return M == MODE_SYM_HVP || M == MODE_SYM_HESS; }

struct BatchArgs {
  int n;
  int csize;   // the API chunk size C (symmetric modes: which chunks are computed)
  int groups;  // G: 32-point groups per CTA
  int64_t m;
  const double* __restrict__ points;
  const double* __restrict__ vecs;
  double* __restrict__ out;  // HVP: m x n;  Hessian: m x n x n
  const double* __restrict__ params;
  double* __restrict__ grad;  // MODE_HESS_GRAD: m x n gradient
};

constexpr int kPad = 33;     // shared-memory row stride (doubles) of [k][lane] tiles
constexpr int kWarpsF3 = 4;  // seed-sparse Fletcher-Powell kernel: 128 threads per CTA

CHF_INL bool aligned16_ptr(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// stage points [and vectors] of the tile into shared memory, transposed per 32-point group.
// The tile is one contiguous range of each array (row-major m x n); with n even and 16-byte-
// aligned rows it is read as coalesced 16-byte words (two coordinates of one point each),
// otherwise 8 bytes at a time.
CHF_INL void stage_tile(const BatchArgs& p, int64_t e0, int P, double* s_pts, double* s_vec) {
  const int n = p.n;
  if ((n & 1) == 0 && aligned16_ptr(p.points) && (!s_vec || aligned16_ptr(p.vecs))) {
    const int h = n >> 1;
    for (int q = threadIdx.x; q < P * h; q += blockDim.x) {
      const int pi = q / h, k = 2 * (q - pi * h);
      int64_t e = e0 + pi;
      if (e >= p.m) e = p.m - 1;  // ragged tail: replicate the last point, never stored
      const int g = pi >> 5, ln = pi & 31;
      const double2 x = __ldg(reinterpret_cast<const double2*>(p.points + e * n + k));
      s_pts[(g * n + k) * kPad + ln] = x.x;
      s_pts[(g * n + k + 1) * kPad + ln] = x.y;
      if (s_vec) {
        const double2 w = __ldg(reinterpret_cast<const double2*>(p.vecs + e * n + k));
        s_vec[(g * n + k) * kPad + ln] = w.x;
        s_vec[(g * n + k + 1) * kPad + ln] = w.y;
      }
    }
    return;
  }
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
  if ((n & 1) == 0 && aligned16_ptr(p.out)) {  // 16-byte coalesced stores
    const int h = n >> 1;
    for (int q = threadIdx.x; q < P * h; q += blockDim.x) {
      const int pi = q / h, k = 2 * (q - pi * h);
      const int64_t e = e0 + pi;
      const double* src = s_out + ((pi >> 5) * n + k) * kPad + (pi & 31);
      if (e < p.m) *reinterpret_cast<double2*>(p.out + e * n + k) = make_double2(src[0], src[kPad]);
    }
    return;
  }
  for (int q = threadIdx.x; q < P * n; q += blockDim.x) {
    const int pi = q / n, k = q - pi * n;
    const int64_t e = e0 + pi;
    if (e < p.m) p.out[e * n + k] = s_out[((pi >> 5) * n + k) * kPad + (pi & 31)];
  }
}

// Per-row consumer of finished columns (one instance per thread and row).
//   a5/a6 of §8(a): res accumulates sum_l H[i][col] * v[col] in ascending column order.
template <int MODE>
struct RowSink {
  double res;       // HVP modes: this row's accumulator
  const double* v;  // lane's vector (stride vs), HVP modes
  int vs;
  double* s_res;    // lane's output column (stride kPad), MODE_SYM_HVP scatter target
  double vi;        // v[i], MODE_SYM_HVP
  double* hrow;     // &H[e][i][0] (nullptr for ragged-tail lanes), Hessian modes
  double* hcol;     // &H[e][0][i] (stride n), MODE_SYM_HESS mirror
  int n;
  bool mirror;      // symmetric modes: this chunk lies strictly after row i's chunk
  CHF_INL void operator()(int col, double h) {
    if (MODE == MODE_HVP || MODE == MODE_SYM_HVP || MODE == MODE_HVP_ROWHOIST) {
      res = res + h * v[col * vs];
      if (MODE == MODE_SYM_HVP && mirror) s_res[col * kPad] = s_res[col * kPad] + h * vi;
    } else if (hrow) {
      hrow[col] = h;
      if (MODE == MODE_SYM_HESS && mirror) hcol[(size_t)col * n] = h;
    }
  }
};

template <int MODE>
CHF_INL RowSink<MODE> make_sink(const BatchArgs& p, int i, int64_t e, const double* v, double* o, int vs = kPad) {
  constexpr bool HESS = mode_hess(MODE);
  const int n = p.n;
  RowSink<MODE> s;
  s.res = MODE == MODE_SYM_HVP ? o[i * kPad] : 0.0;
  s.v = v;
  s.vs = vs;
  s.s_res = o;
  s.vi = HESS ? 0.0 : v[i * vs];
  s.hrow = (HESS && e < p.m) ? p.out + (e * n + i) * n : nullptr;
  s.hcol = (HESS && e < p.m) ? p.out + e * n * n + i : nullptr;
  s.n = n;
  s.mirror = false;
  return s;
}

// ---------------------------------------------------------------- F1, F2, F4: hDual<C> in registers
#ifndef CHF_NS_CHUNK_UNROLL
#define CHF_NS_CHUNK_UNROLL 4  // compiled-n kernels: unroll the chunk loop up to this many chunks
#endif
#ifndef CHF_REG_MINB
#define CHF_REG_MINB 1  // min CTAs/SM hint of the register path (tuning experiments)
#endif
// NS > 0: n == NS at compile time (the paper's NV-templated kernels, Fig. 2):
// the function's variable loops are fully unrolled and each seed's variable index is a
// constant; rows and chunks remain runtime loops, so every (row, chunk) evaluation of Alg 7 is
// still formed from its own CHUNK-INIT seeds and executed on its own.  nvcc folds the seed
// slots that become constants (x*1 -> x; IEEE-exact, outputs bit-identical to NS = 0).
template <class F, int NS, int C, int MODE>
__host__ __device__ constexpr int reg_min_blocks() {
  return min_blocks_of<F>::get(NS, C, MODE) > 0 ? min_blocks_of<F>::get(NS, C, MODE) : CHF_REG_MINB;
}
template <class F, int C, int MODE, int W, int NS = 0>
__global__ void __launch_bounds__(W * 32, (reg_min_blocks<F, NS, C, MODE>())) hvp_reg_kernel(BatchArgs p, F f) {
  constexpr bool TRIG = uses_trig2pi<F>::value;
  constexpr bool HESS = mode_hess(MODE);
  extern __shared__ double smem[];
  const int n = NS > 0 ? NS : p.n, G = p.groups, P = 32 * G, Capi = p.csize;
  double* s_pts = smem;
  double* s_vec = HESS ? nullptr : s_pts + G * n * kPad;
  double* s_out = HESS ? nullptr : s_vec + G * n * kPad;
  double* s_sin = (HESS ? s_pts : s_out) + G * n * kPad;  // TRIG only
  double* s_cos = s_sin + G * n * kPad;
  const int64_t e0 = (int64_t)blockIdx.x * P;
  stage_tile(p, e0, P, s_pts, s_vec);
  if (MODE == MODE_SYM_HVP)
    for (int q = threadIdx.x; q < G * n * kPad; q += blockDim.x) s_out[q] = 0.0;
  if (TRIG) {
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
  double* o = HESS ? nullptr : s_out + g * n * kPad + lane;
  const double* tsin = TRIG ? s_sin + g * n * kPad + lane : nullptr;
  const double* tcos = TRIG ? s_cos + g * n * kPad + lane : nullptr;
  const int64_t e = e0 + g * 32 + lane;
  const int nchunk = n / C;
  // NS > 0 with 2 .. CHF_NS_CHUNK_UNROLL chunks per row: the chunk loop unrolls too, so the chunk
  // start is a constant in each copy (reading R8) and the seeds read the point with volatile
  // loads (no work shared between the copies); otherwise chunks stay a runtime loop
  // (where the functor opts in, F::vol_seeds: measured per function, profiles/r02/ns3/)
  constexpr bool kVolOk = NS > 0 && vol_seeds_of<F>::get(NS, C, MODE);
  constexpr int kChunkUnroll = (kVolOk && NS / C <= CHF_NS_CHUNK_UNROLL) ? (NS > 0 ? NS / C : 1) : 1;
  constexpr bool kVolSeed = kVolOk && (kChunkUnroll > 1 || NS >= 32);
  for (int i = warp / G; i < n; i += rstep) {
    const int scn = i / Capi;  // row i's first chunk (symmetric modes)
    RowSink<MODE> sink = make_sink<MODE>(p, i, e, v, o);
    double gi = 0.0;  // MODE_HESS_GRAD: df/dx_i (slot v[1], identical for every chunk of row i)
#pragma unroll kChunkUnroll
    for (int j = mode_sym(MODE) ? (scn * Capi) / C : 0; j < nchunk; j++) {
      const int cs = j * C;
      sink.mirror = cs / Capi > scn;
      const LaneSeed<C, (NS > 0), kVolSeed> y{a, kPad, i, cs, tsin, tcos};
      const hd<C> t = f.template operator()<C>(n, y);  // CHUNK-INIT + f<hDual<C>>, Alg 7 :389-390
#pragma unroll
      for (int l = 0; l < C; l++) sink(cs + l, t.v[C + 2 + l]);  // :392-394 / :210-212 / :417-421
      if (MODE == MODE_HESS_GRAD) gi = t.v[1];
    }
    if (MODE == MODE_HESS_GRAD && e < p.m) p.grad[e * n + i] = gi;
    if (!HESS) o[i * kPad] = sink.res;
  }
  if (!HESS) {
    __syncthreads();
    write_tile(p, e0, P, s_out);
  }
}

// ---------------------------------------------------------------- NEXT-4: compile-time NS
// chessfad_hvp_batch_hoisted for F1/F2/F4, n = NS in {2, 4, 8, 16}: Alg 7 with one thread per
// point (the paper's L0 level, Alg 9, whose code is likewise templated on n),
// point and vector in registers (16-byte loads), every row / chunk / variable loop unrolled at
// compile time so that the CHUNK-INIT seeds are constants (StaticSeed).  nvcc then folds the
// 0/1 seed products and computes each scalar sub-expression shared by the point's n^2/C
// evaluations once (the value channel, the first-order slots common to all rows): value-
// channel hoisting done by the compiler, IEEE-exact, outputs identical to per-evaluation
// execution, executed FLOPs far below the model count (reported by ncu, labelled).
template <class F, int C, int NS, bool FUSED>
__global__ void __launch_bounds__(128) hvp_small_kernel(BatchArgs p, F f) {
  constexpr bool TRIG = uses_trig2pi<F>::value;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.m) return;
  double a[NS], v[NS], out[NS], ts[NS], tc[NS];
  const double2* a2 = reinterpret_cast<const double2*>(p.points + e * NS);
  const double2* v2 = reinterpret_cast<const double2*>(p.vecs + e * NS);
#pragma unroll
  for (int q = 0; q < NS / 2; q++) {
    const double2 x = __ldg(a2 + q), w = __ldg(v2 + q);
    a[2 * q] = x.x;
    a[2 * q + 1] = x.y;
    v[2 * q] = w.x;
    v[2 * q + 1] = w.y;
  }
  if (TRIG) {
#pragma unroll
    for (int k = 0; k < NS; k++) sincos(6.283185307179586 * a[k], ts + k, tc + k);
  }
#pragma unroll
  for (int i = 0; i < NS; i++) {
    double res = 0.0;
#pragma unroll
    for (int j = 0; j < NS / C; j++) {
      const StaticSeed<C, FUSED> y{a, 1, i, j * C, ts, tc};
      const hd<C> t = f.template operator()<C>(NS, y);  // CHUNK-INIT + f<hDual<C>>, Alg 7 :389-390
#pragma unroll
      for (int l = 0; l < C; l++) res = res + t.v[C + 2 + l] * v[j * C + l];  // :392-394
    }
    out[i] = res;
  }
  double2* o2 = reinterpret_cast<double2*>(p.out + e * NS);
#pragma unroll
  for (int q = 0; q < NS / 2; q++) o2[q] = make_double2(out[2 * q], out[2 * q + 1]);
}

}  // namespace chessfad

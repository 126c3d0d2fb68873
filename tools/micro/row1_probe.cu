// row1_probe.cu -- the headline kernel (Rosenbrock, n = C = 16, compiled n) with the seed's
// row slot [k == i] read from a per-warp shared table written once per row, instead of an
// ISETP + FSEL + zero-word move per variable.  Not part of the library.
// Result (static SASS): 1 644 FP64 instructions per evaluation instead of 656 -- with the row
// slot a loaded value nvcc can no longer turn products with the 0/1 select into selects of
// the two outcomes, so the table costs far more than the selects it removes.  Not adopted.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chessfad/launch_functor.cuh"

using namespace chessfad;

template <int C>
struct RowTabSeed {
  static constexpr bool kStatic = true;
  static constexpr bool kFused = true;
  const double* a;
  int stride;
  int i, cs;
  const double* sin2pi;
  const double* cos2pi;
  const double* row1;  // per-warp [n]: [k == i]
  CHF_INL hs<C> operator()(int k) const {
    hs<C> y;
    y.v[0] = a[k * stride];
    y.v[1] = row1[k];
    const int off = k - cs;
#pragma unroll
    for (int l = 0; l < C; l++) y.v[2 + l] = (off == l) ? 1.0 : 0.0;
    return y;
  }
  CHF_INL double s2pi(int k) const { return sin2pi[k * stride]; }
  CHF_INL double c2pi(int k) const { return cos2pi[k * stride]; }
};

template <class F, int C, int NS>
__global__ void __launch_bounds__(128, 1) row1_kernel(BatchArgs p, F f) {
  extern __shared__ double smem[];
  __shared__ __align__(16) double s_row1[4][NS];
  const int n = NS, P = 32;
  double* s_pts = smem;
  double* s_vec = s_pts + n * kPad;
  double* s_out = s_vec + n * kPad;
  const int64_t e0 = (int64_t)blockIdx.x * P;
  stage_tile(p, e0, P, s_pts, s_vec);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* a = s_pts + lane;
  const double* v = s_vec + lane;
  double* o = s_out + lane;
  const int64_t e = e0 + lane;
  for (int i = warp; i < n; i += 4) {
    if (lane < NS) s_row1[warp][lane] = (lane == i) ? 1.0 : 0.0;
    __syncwarp();
    RowSink<MODE_HVP> sink = make_sink<MODE_HVP>(p, i, e, v, o);
#pragma unroll 1
    for (int j = 0; j < n / C; j++) {
      const int cs = j * C;
      const RowTabSeed<C> y{a, kPad, i, cs, nullptr, nullptr, s_row1[warp]};
      const hd<C> t = f.template operator()<C>(n, y);
#pragma unroll
      for (int l = 0; l < C; l++) sink(cs + l, t.v[C + 2 + l]);
    }
    o[i * kPad] = sink.res;
    __syncwarp();
  }
  __syncthreads();
  write_tile(p, e0, P, s_out);
}

template <class L>
float timeit(L&& go) {
  for (int w = 0; w < 3; w++) go();
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int r = 0; r < 20; r++) go();
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  return ms / 20;
}

int main() {
  const int n = 16;
  const int64_t m = 1 << 20;
  std::vector<double> hp(m * n), hv(m * n);
  srand(5);
  for (auto& x : hp) x = 2.0 * rand() / RAND_MAX - 1.0;
  for (auto& x : hv) x = 2.0 * rand() / RAND_MAX - 1.0;
  double *dp, *dv, *d1, *d2;
  cudaMalloc(&dp, m * n * 8);
  cudaMalloc(&dv, m * n * 8);
  cudaMalloc(&d1, m * n * 8);
  cudaMalloc(&d2, m * n * 8);
  cudaMemcpy(dp, hp.data(), m * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), m * n * 8, cudaMemcpyHostToDevice);
  BatchArgs a1{n, 16, 1, m, dp, dv, d1, nullptr, nullptr}, a2{n, 16, 1, m, dp, dv, d2, nullptr, nullptr};
  using F = BuiltinFunc<FUNC_ROSENBROCK>;
  const size_t smem = 3 * n * kPad * 8;
  const int grid = (int)(m / 32);
  printf("lib  %.4f ms\n", timeit([&] { launch_functor<F, 16, MODE_HVP, 16>(F{}, a1, 0); }));
  printf("row1 %.4f ms\n", timeit([&] { row1_kernel<F, 16, 16><<<grid, 128, smem>>>(a2, F{}); }));
  std::vector<double> r1(m * n), r2(m * n);
  cudaMemcpy(r1.data(), d1, m * n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), d2, m * n * 8, cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  for (int64_t q = 0; q < m * n; q++) bad += r1[q] != r2[q];
  printf("bitwise mismatches %lld (%s)\n", (long long)bad, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

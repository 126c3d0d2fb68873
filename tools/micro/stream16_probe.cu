// stream16_probe.cu -- the n <= 8 streaming kernel (stream_small.cuh) tried at n = 16 for the
// HBM-facing prodsum, against the register kernel compiled for n = 16.  Not part of the library.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chessfad/launch_functor.cuh"
// (stream_small.cuh launch bounds: NS == 8 ? 1 : 2 -- NS = 16 runs at 2 CTAs/SM here)
#include "stream_small.cuh"

using namespace chessfad;

template <int FUNC, int C, int NS, bool KCS>
cudaError_t launch_stream_probe(BatchArgs a) {
  auto kern = hvp_stream_kernel<BuiltinFunc<FUNC>, C, NS, KCS>;
  constexpr size_t smem = StreamCfg<NS>::kSmem;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStreamTP, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (occ < 1) occ = 1;
  const int64_t tiles = (a.m + kStreamTP - 1) / kStreamTP;
  const int grid = (int)(tiles < (int64_t)sms * occ ? tiles : (int64_t)sms * occ);
  kern<<<grid, kStreamTP, smem>>>(a, BuiltinFunc<FUNC>{});
  return cudaGetLastError();
}

template <class L>
float timeit(L&& go) {
  for (int w = 0; w < 3; w++) go();
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int r = 0; r < 10; r++) go();
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  return ms / 10;
}

int main() {
  const int n = 16;
  const int64_t m = 1 << 20;
  std::vector<double> hp(m * n), hv(m * n);
  srand(3);
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
  using F = BuiltinFunc<FUNC_PRODSUM>;
  printf("reg_ns C=16    %.4f ms\n", timeit([&] { launch_functor<F, 16, MODE_HVP, 16>(F{}, a1, 0); }));
  printf("stream C=16    %.4f ms\n", timeit([&] { launch_stream_probe<FUNC_PRODSUM, 16, 16, true>(a2); }));
  printf("stream C=16 o  %.4f ms\n", timeit([&] { launch_stream_probe<FUNC_PRODSUM, 16, 16, false>(a2); }));
  printf("stream C=8     %.4f ms\n", timeit([&] { launch_stream_probe<FUNC_PRODSUM, 8, 16, true>(a2); }));
  std::vector<double> r1(m * n), r2(m * n);
  launch_functor<F, 16, MODE_HVP, 16>(F{}, a1, 0);
  launch_stream_probe<FUNC_PRODSUM, 16, 16, true>(a2);
  cudaMemcpy(r1.data(), d1, m * n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), d2, m * n * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int64_t q = 0; q < m * n; q++) mx = fmax(mx, fabs(r1[q] - r2[q]) / (fabs(r1[q]) + 1e-300));
  printf("max rel diff %.3e  (%s)\n", mx, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

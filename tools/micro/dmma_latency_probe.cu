#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void probe(long iters, double* sink) {
  double acc[NACC][2];
#pragma unroll
  for (int q = 0; q < NACC; q++) acc[q][0] = acc[q][1] = q;
  const double a0 = 1.0 + threadIdx.x * 1e-17, b0 = 1.0 - threadIdx.x * 1e-17;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int q = 0; q < NACC; q++) dmma(acc[q], a0, b0);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < NACC; q++) s += acc[q][0] + acc[q][1];
  sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
void run(int sms, int threads, long iters, double* sink) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<NACC><<<sms, threads>>>(iters / 10, sink);
  cudaEventRecord(e0);
  probe<NACC><<<sms, threads>>>(iters, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)sms * threads / 32 * iters * NACC * 512;
  printf("DMMA threads/SM %d, independent accumulators %d: %.2f TFLOP/s\n", threads, NACC, fl / (ms * 1e-3) / 1e12);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, (size_t)sms * 1024 * 8);
  for (int t : {128, 256}) { run<1>(sms, t, 40000, sink); run<2>(sms, t, 40000, sink); run<4>(sms, t, 20000, sink); run<8>(sms, t, 10000, sink); run<16>(sms, t, 5000, sink); }
  return 0;
}

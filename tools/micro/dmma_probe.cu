// Microbenchmark: FP64 throughput of DFMA (SIMT FP64 pipe) vs DMMA m8n8k4 (FP64 mma.sync) on
// sm_100a, alone and interleaved (do they share a pipe?).  Decides whether the F3 E-sum
// contraction (E = [A|B] x slot values) can use DMMA.  Usage: dmma_probe [blocks_per_sm]
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>  // 0 = DFMA only, 1 = DMMA only, 2 = both interleaved
__global__ void __launch_bounds__(256) probe(long iters, double* sink) {
  const double b = 1.0 + 1e-16 * threadIdx.x, c = 1e-300;
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; q++) x[q] = threadIdx.x + q;
  double acc[8][2];
#pragma unroll
  for (int q = 0; q < 8; q++) acc[q][0] = acc[q][1] = q;
  const double a0 = 1.0 + threadIdx.x * 1e-17, b0 = 1.0 - threadIdx.x * 1e-17;
  for (long it = 0; it < iters; it++) {
    if (MODE != 1) {
#pragma unroll
      for (int q = 0; q < 8; q++) x[q] = fma(x[q], b, c);
    }
    if (MODE != 0) {
#pragma unroll
      for (int q = 0; q < 8; q++) dmma(acc[q], a0, b0);
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; q++) s += x[q] + acc[q][0] + acc[q][1];
  sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(int blocks, long iters, double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<MODE><<<blocks, 256>>>(iters / 10, sink);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, 256>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = blocks * 8.0;
  // per iteration per warp: DFMA 8 instr x 32 lanes x 2 flop; DMMA 8 x 512 flop
  const double fl = warps * iters * ((MODE != 1) ? 8 * 32 * 2.0 : 0) + warps * iters * ((MODE != 0) ? 8 * 512.0 : 0);
  const double tf = fl / (ms * 1e-3) / 1e12;
  printf("mode %d (%s): blocks %d, %.3f ms, %.2f TFLOP/s\n", MODE, MODE == 0 ? "DFMA" : MODE == 1 ? "DMMA" : "DFMA+DMMA",
         blocks, ms, tf);
  return tf;
}

int main(int argc, char** argv) {
  int bps = argc > 1 ? atoi(argv[1]) : 4;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, (size_t)sms * 8 * 256 * 8);
  for (int b : {1, 2, 4, 8}) {
    if (b > bps) break;
    run<0>(sms * b, 20000, sink);
    run<1>(sms * b, 20000, sink);
    run<2>(sms * b, 20000, sink);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

// dfma_ilp.cu -- FP64 FMA pipe throughput vs independent chains per warp (ILP) and warps per
// scheduler, on one B200.  Each thread runs ILP independent dependent-DFMA chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/dfma_ilp.cu -o /tmp/dfma_ilp
#include <cstdio>

// ALU: integer ops (independent IMAD chains) issued per DFMA x ILP... per iteration, ALU of them
// KIND 0: IMAD chains (FMA pipe), 1: LOP3/shift xorshift (ALU pipe), 2: ISETP+FSEL selects
template <int ILP, int ALU = 0, int KIND = 0>
__global__ void chains(double* out, int iters, double b, double c) {
  double a[ILP];
  unsigned x[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
#pragma unroll
  for (int j = 0; j < ILP; j++) a[j] = threadIdx.x * 1e-3 + j;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < ILP; j++) a[j] = fma(a[j], b, c);
#pragma unroll
    for (int q = 0; q < ALU; q++) {
      if (KIND == 0) x[q & 3] = x[q & 3] * 2654435761u + (unsigned)it;
      else if (KIND == 1) x[q & 3] = (x[q & 3] ^ (unsigned)it) ^ (x[q & 3] >> 7);
      else x[q & 3] = __float_as_uint(x[q & 3] == (unsigned)(it + q) ? 1.875f : 0.0f) ^ x[(q + 1) & 3];
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; j++) s += a[j];
  if (s == 12345.678 || (x[0] ^ x[1] ^ x[2] ^ x[3]) == 7u) out[threadIdx.x] = s;
}

template <int ILP, int ALU = 0, int KIND = 0>
void run(int warps_per_smsp, int sms, double* out) {
  const int threads = 32 * 4 * warps_per_smsp;  // one CTA per SM, warps spread over 4 SMSPs
  const int iters = 1 << 16;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  chains<ILP, ALU, KIND><<<sms, threads>>>(out, 64, 0.999999, 1e-9);
  cudaEventRecord(t0);
  chains<ILP, ALU, KIND><<<sms, threads>>>(out, iters, 0.999999, 1e-9);
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  const double fmas = (double)sms * threads * iters * ILP;
  const double tflops = 2 * fmas / (ms * 1e-3) / 1e12;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double per_clk_sm = fmas / (ms * 1e-3) / (clk * 1e3) / sms;
  printf("warps/smsp %d ILP %2d ALU/iter %2d kind %d: %6.2f TFLOP/s  %5.1f FMA/clk/SM (of 64)\n", warps_per_smsp, ILP, ALU, KIND, tflops, per_clk_sm);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 4096 * 8);
  for (int w = 2; w <= 2; w++) {
    run<1>(w, sms, out);
    run<2>(w, sms, out);
    run<3>(w, sms, out);
    run<4>(w, sms, out);
    run<6>(w, sms, out);
    run<8>(w, sms, out);
  }
  for (int w = 2; w <= 3; w++) {
    run<8, 4, 0>(w, sms, out);
    run<8, 8, 0>(w, sms, out);
    run<8, 4, 1>(w, sms, out);
    run<8, 8, 1>(w, sms, out);
    run<8, 4, 2>(w, sms, out);
    run<8, 8, 2>(w, sms, out);
  }
  return 0;
}

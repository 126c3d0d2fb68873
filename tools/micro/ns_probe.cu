// ns_probe.cu -- the register kernels compiled for n = 32 / 64 at a given min-CTAs-per-SM bound
// (build with -DCHF_REG_MINB=k): event-timed Alg 7 over m points, Rosenbrock and Ackley C = 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCHF_REG_MINB=3 \
//        tools/micro/ns_probe.cu -o /tmp/ns_probe && /tmp/ns_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chessfad/launch_functor.cuh"

using namespace chessfad;

// Ackley / Rosenbrock with the volatile-seed form forced on (policy experiments)
template <int FUNC>
struct VolOn : BuiltinFunc<FUNC> {
  __host__ __device__ static constexpr bool vol_seeds(int, int, int) { return true; }
};

template <int FUNC, int NS, int C, class F = BuiltinFunc<FUNC>>
void run(const char* name, int64_t m) {
  const int n = NS;
  std::vector<double> hp(m * n), hv(m * n);
  srand(1);
  for (auto& x : hp) x = 2.0 * rand() / RAND_MAX - 1.0;
  for (auto& x : hv) x = 2.0 * rand() / RAND_MAX - 1.0;
  double *dp, *dv, *dout;
  cudaMalloc(&dp, m * n * 8);
  cudaMalloc(&dv, m * n * 8);
  cudaMalloc(&dout, m * n * 8);
  cudaMemcpy(dp, hp.data(), m * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), m * n * 8, cudaMemcpyHostToDevice);
  BatchArgs a{n, C, 1, m, dp, dv, dout, nullptr, nullptr};
  auto go = [&] { launch_functor<F, C, MODE_HVP, NS>(F{}, a, 0); };
  for (int w = 0; w < 2; w++) go();
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int r = 0; r < 5; r++) go();
  cudaEventRecord(t1);
  cudaEventSynchronize(t1);
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  printf("MINB %d %-12s n=%d C=%d m=%lld: %8.3f ms  (%s)\n", CHF_REG_MINB, name, n, C, (long long)m, ms / 5,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dp);
  cudaFree(dv);
  cudaFree(dout);
}

int main() {
  if (getenv("NS_PROBE_ACK128")) {
    run<FUNC_ACKLEY, 128, 16, VolOn<FUNC_ACKLEY>>("ackley-vol", 65536);
    run<FUNC_ACKLEY, 128, 8, VolOn<FUNC_ACKLEY>>("ackley-vol", 65536);
    run<FUNC_ACKLEY, 128, 16>("ackley", 65536);
    return 0;
  }
  if (getenv("NS_PROBE_BIG")) {
    run<FUNC_ROSENBROCK, 128, 8>("rosenbrock", 65536);
    run<FUNC_ROSENBROCK, 128, 16>("rosenbrock", 65536);
    run<FUNC_ROSENBROCK, 64, 8>("rosenbrock", 262144);
    run<FUNC_ROSENBROCK, 64, 16>("rosenbrock", 262144);
    return 0;
  }
  run<FUNC_ROSENBROCK, 16, 16>("rosenbrock", 1048576);
  run<FUNC_ROSENBROCK, 16, 8>("rosenbrock", 1048576);
  run<FUNC_ROSENBROCK, 8, 8>("rosenbrock", 1048576);
  run<FUNC_ACKLEY, 16, 16>("ackley", 1048576);
  run<FUNC_ACKLEY, 16, 16, VolOn<FUNC_ACKLEY>>("ackley-vol", 1048576);
  run<FUNC_ACKLEY, 16, 8>("ackley", 1048576);
  run<FUNC_ACKLEY, 16, 8, VolOn<FUNC_ACKLEY>>("ackley-vol", 1048576);
  run<FUNC_ACKLEY, 8, 8>("ackley", 1048576);
  run<FUNC_ACKLEY, 8, 8, VolOn<FUNC_ACKLEY>>("ackley-vol", 1048576);
  run<FUNC_PRODSUM, 16, 16>("prodsum", 1048576);
  run<FUNC_PRODSUM, 16, 16, VolOn<FUNC_PRODSUM>>("prodsum-vol", 1048576);
  return 0;
  run<FUNC_ROSENBROCK, 16, 16>("rosenbrock", 1048576);
  run<FUNC_ACKLEY, 16, 16>("ackley", 1048576);
  run<FUNC_PRODSUM, 16, 16>("prodsum", 1048576);
  run<FUNC_ROSENBROCK, 16, 4>("rosenbrock", 1048576);
  run<FUNC_ROSENBROCK, 32, 16>("rosenbrock", 262144);
  run<FUNC_ROSENBROCK, 32, 8>("rosenbrock", 262144);
  run<FUNC_ACKLEY, 32, 8>("ackley", 262144);
  run<FUNC_ACKLEY, 32, 16>("ackley", 262144);
  run<FUNC_ROSENBROCK, 64, 16>("rosenbrock", 65536);
  run<FUNC_ROSENBROCK, 64, 8>("rosenbrock", 65536);
  run<FUNC_ACKLEY, 64, 8>("ackley", 65536);
  return 0;
}

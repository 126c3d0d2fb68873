// reg_probe.cu -- tuning probe for the headline register kernel (Rosenbrock n = 16, C = 16,
// Alg 7, per-evaluation execution).  Not part of the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/micro/reg_probe.cu -o /tmp/reg_probe && /tmp/reg_probe
//
// Variants (all evaluate exactly the library kernel's per-row body):
//   lib        chessfad::hvp_reg_kernel as launched by the library
//   compute R  the tile staged once, the 4 rows of each warp evaluated R times (no staging
//              cost in the steady state: the pipe utilisation of the evaluation alone)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chessfad/launch_functor.cuh"

using namespace chessfad;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

template <class F, int C, int W, int R>
__global__ void __launch_bounds__(W * 32, 1) compute_kernel(BatchArgs p, F f) {
  extern __shared__ double smem[];
  const int n = p.n, P = 32;
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
  for (int i = warp; i < n; i += W) {
    RowSink<MODE_HVP> sink = make_sink<MODE_HVP>(p, i, e, v, o);
    for (int r = 0; r < R; r++) {
      for (int j = 0; j < n / C; j++) {
        const int cs = j * C;
        const LaneSeed<C> y{a, kPad, i, cs, nullptr, nullptr};
        const hd<C> t = f.template operator()<C>(n, y);
#pragma unroll
        for (int l = 0; l < C; l++) sink(cs + l, t.v[C + 2 + l]);
      }
    }
    o[i * kPad] = sink.res;
  }
  __syncthreads();
  write_tile(p, e0, P, s_out);
}

// ---- prototype: seed operands typed with structurally-zero second-order slots
template <int C>
struct hz {  // CHUNK-INIT seed (or 1 - seed): slots 0 .. C+1 only, v[C+2..] == 0 by construction
  double v[C + 2];
};
template <int C>
CHF_INL hz<C> zseed(const LaneSeed<C>& y, int k) {
  hz<C> r;
  r.v[0] = y.a[k * y.stride];
  r.v[1] = (k == y.i) ? 1.0 : 0.0;
  const int off = k - y.cs;
#pragma unroll
  for (int l = 0; l < C; l++) r.v[2 + l] = (off == l) ? 1.0 : 0.0;
  return r;
}
template <int C>
CHF_INL hz<C> one_minus(const hz<C>& u) {
  hz<C> r;
  r.v[0] = 1.0 - u.v[0];
#pragma unroll
  for (int s = 1; s < C + 2; s++) r.v[s] = -u.v[s];
  return r;
}
// acc - u*v, u, v, acc seeds: the hd_fnma term order with the zero second-order terms absent
template <int C>
CHF_INL hd<C> z_fnma(const hz<C>& u, const hz<C>& v, const hz<C>& acc) {
  hd<C> r;
  r.v[0] = __fma_rn(-u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(-v.v[0], u.v[i], __fma_rn(-u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++) r.v[C + j] = __fma_rn(-v.v[1], u.v[j], -u.v[1] * v.v[j]);
  return r;
}
// acc + u*v, u, v seeds, acc full
template <int C>
CHF_INL hd<C> z_fma(const hz<C>& u, const hz<C>& v, const hd<C>& acc) {
  hd<C> r;
  r.v[0] = __fma_rn(u.v[0], v.v[0], acc.v[0]);
#pragma unroll
  for (int i = 1; i <= C + 1; i++) r.v[i] = __fma_rn(v.v[0], u.v[i], __fma_rn(u.v[0], v.v[i], acc.v[i]));
#pragma unroll
  for (int j = 2; j <= C + 1; j++) r.v[C + j] = __fma_rn(v.v[1], u.v[j], __fma_rn(u.v[1], v.v[j], acc.v[C + j]));
  return r;
}
struct RosenZ {
  static constexpr bool kTrig2Pi = false;
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int n, const Seed& y) const {
    hd<C> s;
    {
      const hz<C> y0 = zseed(y, 0), y1 = zseed(y, 1);
      const hd<C> d = z_fnma(y0, y0, y1);
      const hz<C> e = one_minus(y0);
      s = z_fma(e, e, 100.0 * (d * d));
    }
#pragma unroll 4
    for (int i = 1; i < n - 1; i++) {
      const hz<C> yi = zseed(y, i), yi1 = zseed(y, i + 1);
      const hd<C> d = z_fnma(yi, yi, yi1);
      const hz<C> e = one_minus(yi);
      s = z_fma(e, e, hd_axpy(100.0, d * d, s));
    }
    return s;
  }
};

// ---- prototype: chunk slots of the seed read from a shared one-hot table with 16-byte loads
// T[q][t] = [t == Z + q]  (q = 0, 1: two copies so that the C-slot window starts 16-byte aligned)
constexpr int kTabZ = 20, kTabN = 48;
template <int C>
struct TabSeed {
  static constexpr bool kStatic = false;
  static constexpr bool kFused = true;
  const double* a;
  int stride;
  int i, cs;
  const double* sin2pi;
  const double* cos2pi;
  const double* tab;  // shared [2][kTabN]
  CHF_INL hs<C> operator()(int k) const {
    hs<C> y;
    y.v[0] = a[k * stride];
    y.v[1] = (k == i) ? 1.0 : 0.0;
    int off = k - cs;
    off = min(max(off, -1), C);               // outside the chunk: every slot 0
    const int q = off & 1;                    // copy whose window start Z + q - off is even
    const double2* w = reinterpret_cast<const double2*>(tab + q * kTabN + kTabZ + q - off);
#pragma unroll
    for (int l = 0; l < C / 2; l++) {
      const double2 t = w[l];
      y.v[2 + 2 * l] = t.x;
      y.v[3 + 2 * l] = t.y;
    }
    return y;
  }
};

template <class F, int C, int W>
__global__ void __launch_bounds__(W * 32, 1) tab_kernel(BatchArgs p, F f) {
  extern __shared__ double smem[];
  __shared__ __align__(16) double s_tab[2 * kTabN];
  const int n = p.n, P = 32;
  double* s_pts = smem;
  double* s_vec = s_pts + n * kPad;
  double* s_out = s_vec + n * kPad;
  const int64_t e0 = (int64_t)blockIdx.x * P;
  for (int t = threadIdx.x; t < 2 * kTabN; t += blockDim.x) s_tab[t] = (t % kTabN == kTabZ + t / kTabN) ? 1.0 : 0.0;
  stage_tile(p, e0, P, s_pts, s_vec);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* a = s_pts + lane;
  const double* v = s_vec + lane;
  double* o = s_out + lane;
  const int64_t e = e0 + lane;
  for (int i = warp; i < n; i += W) {
    RowSink<MODE_HVP> sink = make_sink<MODE_HVP>(p, i, e, v, o);
    for (int j = 0; j < n / C; j++) {
      const int cs = j * C;
      const TabSeed<C> y{a, kPad, i, cs, nullptr, nullptr, s_tab};
      const hd<C> t = f.template operator()<C>(n, y);
#pragma unroll
      for (int l = 0; l < C; l++) sink(cs + l, t.v[C + 2 + l]);
    }
    o[i * kPad] = sink.res;
  }
  __syncthreads();
  write_tile(p, e0, P, s_out);
}

// Rosenbrock with the seed of y_{i+1} carried into the next term (one seed built per term)
struct RosenCarry {
  static constexpr bool kTrig2Pi = false;
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int n, const Seed& y) const {
    hd<C> s;
    auto yc = y(1);
    {
      const auto y0 = y(0);
      const auto d = hd_fnma(y0, y0, yc);
      const auto e = 1.0 - y0;
      s = hd_fma(e, e, 100.0 * (d * d));
    }
#pragma unroll 4
    for (int i = 1; i < n - 1; i++) {
      const auto yi = yc;
      yc = y(i + 1);
      const auto d = hd_fnma(yi, yi, yc);
      const auto e = 1.0 - yi;
      s = hd_fma(e, e, hd_axpy(100.0, d * d, s));
    }
    return s;
  }
};

// Ackley with S1 and S2 accumulated in one pass over the variables (one seed per variable;
// each sum keeps its own ascending order -> bit-identical)
struct AckleyOnePass {
  static constexpr bool kTrig2Pi = true;
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int n, const Seed& y) const {
    const double two_pi = 6.283185307179586, euler = 2.718281828459045;
    hd<C> s1, s2;
    {
      const auto y0 = y(0);
      s1 = y0 * y0;
      const auto u = two_pi * y0;
      s2 = hd_unary(u, y.cos2pi[0], -y.sin2pi[0], -y.cos2pi[0]);
    }
    for (int i = 1; i < n; i++) {
      const auto yi = y(i);
      s1 = hd_fma(yi, yi, s1);
      const auto u = two_pi * yi;
      s2 = hd_unary_acc(u, y.cos2pi[i * y.stride], -y.sin2pi[i * y.stride], -y.cos2pi[i * y.stride], s2);
    }
    const double inv_n = 1.0 / n;
    const hd<C> t1 = (-20.0) * exp((-0.2) * sqrt(s1 * inv_n));
    const hd<C> t2 = exp(s2 * inv_n);
    return (t1 - t2) + (20.0 + euler);
  }
};

// Rosenbrock with compile-time n (variable loop fully unrolled; row i and chunk cs stay
// runtime, so the seeds are still formed per evaluation)
template <int NS>
struct RosenFixed {
  static constexpr bool kTrig2Pi = false;
  template <int C, class Seed>
  CHF_INL hd<C> operator()(int, const Seed& y) const {
    hd<C> s;
    auto yc = y(1);
    {
      const auto y0 = y(0);
      const auto d = hd_fnma(y0, y0, yc);
      const auto e = 1.0 - y0;
      s = hd_fma(e, e, 100.0 * (d * d));
    }
#pragma unroll
    for (int i = 1; i < NS - 1; i++) {
      const auto yi = yc;
      yc = y(i + 1);
      const auto d = hd_fnma(yi, yi, yc);
      const auto e = 1.0 - yi;
      s = hd_fma(e, e, hd_axpy(100.0, d * d, s));
    }
    return s;
  }
};

// persistent CTAs, static tile order, the next tile's points/vectors prefetched with 8-byte
// cp.async into the other half of a double buffer while the current tile is evaluated
CHF_INL void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
CHF_INL void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
CHF_INL void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

CHF_INL void stage_async(const BatchArgs& p, int64_t e0, double* s_pts, double* s_vec) {
  const int n = p.n;
  for (int q = threadIdx.x; q < 32 * n; q += blockDim.x) {
    const int pi = q / n, k = q - pi * n;
    int64_t e = e0 + pi;
    if (e >= p.m) e = p.m - 1;
    cp_async8(s_pts + k * kPad + pi, p.points + e * n + k);
    cp_async8(s_vec + k * kPad + pi, p.vecs + e * n + k);
  }
}

template <class F, int C, int W, int MINB>
__global__ void __launch_bounds__(W * 32, MINB) persist_kernel(BatchArgs p, F f) {
  extern __shared__ double smem[];
  const int n = p.n;
  const int T = n * kPad;
  double* buf = smem;            // [2][pts, vec] tiles
  double* s_out = smem + 4 * T;  // output tile
  const int64_t tiles = (p.m + 31) / 32;
  int64_t t = blockIdx.x;
  if (t < tiles) stage_async(p, t * 32, buf, buf + T);
  cp_commit();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = 0; t < tiles; it++, t += gridDim.x) {
    const int64_t tn = t + gridDim.x;
    double* cur = buf + (it & 1) * 2 * T;
    if (tn < tiles) stage_async(p, tn * 32, buf + ((it + 1) & 1) * 2 * T, buf + ((it + 1) & 1) * 2 * T + T);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* a = cur + lane;
    const double* v = cur + T + lane;
    double* o = s_out + lane;
    const int64_t e = t * 32 + lane;
    for (int i = warp; i < n; i += W) {
      RowSink<MODE_HVP> sink = make_sink<MODE_HVP>(p, i, e, v, o);
      for (int j = 0; j < n / C; j++) {
        const int cs = j * C;
        const LaneSeed<C> y{a, kPad, i, cs, nullptr, nullptr};
        const hd<C> r = f.template operator()<C>(n, y);
#pragma unroll
        for (int l = 0; l < C; l++) sink(cs + l, r.v[C + 2 + l]);
      }
      o[i * kPad] = sink.res;
    }
    __syncthreads();
    write_tile(p, t * 32, 32, s_out);
  }
  cp_wait<0>();
}

int main(int argc, char** argv) {
  const int n = 16;
  const int64_t m = argc > 1 ? atoll(argv[1]) : (1 << 20);
  std::vector<double> hp(m * n), hv(m * n);
  srand(1);
  for (auto& x : hp) x = 2.0 * rand() / RAND_MAX - 1.0;
  for (auto& x : hv) x = 2.0 * rand() / RAND_MAX - 1.0;
  double *dp, *dv, *dout;
  CK(cudaMalloc(&dp, m * n * 8));
  CK(cudaMalloc(&dv, m * n * 8));
  CK(cudaMalloc(&dout, m * n * 8));
  CK(cudaMemcpy(dp, hp.data(), m * n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), m * n * 8, cudaMemcpyHostToDevice));
  BatchArgs a{n, 16, 1, m, dp, dv, dout, nullptr, nullptr};
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  auto timeit = [&](const char* name, double evals_per_point, auto&& launch) {
    for (int w = 0; w < 3; w++) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 10;
    CK(cudaEventRecord(t0));
    for (int r = 0; r < reps; r++) launch();
    CK(cudaEventRecord(t1));
    CK(cudaEventSynchronize(t1));
    float ms;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    ms /= reps;
    printf("%-12s %8.3f ms  %8.3f ms per 1x work  %.4e HVP/s-equiv\n", name, ms, ms / evals_per_point,
           m * evals_per_point / (ms * 1e-3));
  };
  using F = BuiltinFunc<FUNC_ROSENBROCK>;
  timeit("lib", 1, [&] { CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0))); });
  const size_t smem = 3 * n * kPad * 8;
  const int grid = (int)(m / 32);
  timeit("compute1", 1, [&] { compute_kernel<F, 16, 4, 1><<<grid, 128, smem>>>(a, F{}); });
  timeit("compute4", 4, [&] { compute_kernel<F, 16, 4, 4><<<grid, 128, smem>>>(a, F{}); });
  timeit("compute16", 16, [&] { compute_kernel<F, 16, 4, 16><<<grid, 128, smem>>>(a, F{}); });
  {
    const size_t psmem = 5 * n * kPad * 8;
    auto k = persist_kernel<F, 16, 4, 1>;
    int occ = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, psmem));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int pgrid = occ * sms;
    printf("persist: %d CTAs/SM x %d SMs\n", occ, sms);
    timeit("persist", 1, [&] { k<<<pgrid, 128, psmem>>>(a, F{}); });
  }
  timeit("zseed", 1, [&] { CK((launch_functor<RosenZ, 16, MODE_HVP>(RosenZ{}, a, 0))); });
  timeit("carry", 1, [&] { CK((launch_functor<RosenCarry, 16, MODE_HVP>(RosenCarry{}, a, 0))); });
  {
    std::vector<double> ref(m * n), got(m * n);
    CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0)));
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    CK((launch_functor<RosenCarry, 16, MODE_HVP>(RosenCarry{}, a, 0)));
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t q = 0; q < m * n; q++) bad += ref[q] != got[q];
    printf("carry parity: %lld bitwise mismatches of %lld\n", (long long)bad, (long long)(m * n));
  }
  auto cmp0 = [&](const char* name, auto&& la, auto&& lb) {
    std::vector<double> ref(m * n), got(m * n);
    la();
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    lb();
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t q = 0; q < m * n; q++) bad += !(ref[q] == got[q] || (ref[q] != ref[q] && got[q] != got[q]));
    printf("%s parity: %lld bitwise mismatches of %lld\n", name, (long long)bad, (long long)(m * n));
  };
  timeit("fixed16", 1, [&] { CK((launch_functor<RosenFixed<16>, 16, MODE_HVP>(RosenFixed<16>{}, a, 0))); });
  timeit("fixed16c8", 1, [&] { CK((launch_functor<RosenFixed<16>, 8, MODE_HVP>(RosenFixed<16>{}, a, 0))); });
  timeit("lib_c8", 1, [&] { CK((launch_functor<F, 8, MODE_HVP>(F{}, a, 0))); });
  cmp0("fixed16", [&] { CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0))); },
       [&] { CK((launch_functor<RosenFixed<16>, 16, MODE_HVP>(RosenFixed<16>{}, a, 0))); });
  auto cmp = [&](const char* name, auto&& la, auto&& lb) {
    std::vector<double> ref(m * n), got(m * n);
    la();
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    lb();
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t q = 0; q < m * n; q++) bad += !(ref[q] == got[q] || (ref[q] != ref[q] && got[q] != got[q]));
    printf("%s parity: %lld bitwise mismatches of %lld\n", name, (long long)bad, (long long)(m * n));
  };
  using FA = BuiltinFunc<FUNC_ACKLEY>;
  timeit("ackley8", 1, [&] { CK((launch_functor<FA, 8, MODE_HVP>(FA{}, a, 0))); });
  timeit("ack1pass8", 1, [&] { CK((launch_functor<AckleyOnePass, 8, MODE_HVP>(AckleyOnePass{}, a, 0))); });
  timeit("ackley16", 1, [&] { CK((launch_functor<FA, 16, MODE_HVP>(FA{}, a, 0))); });
  timeit("ack1pass16", 1, [&] { CK((launch_functor<AckleyOnePass, 16, MODE_HVP>(AckleyOnePass{}, a, 0))); });
  cmp("ack1pass8", [&] { CK((launch_functor<FA, 8, MODE_HVP>(FA{}, a, 0))); },
      [&] { CK((launch_functor<AckleyOnePass, 8, MODE_HVP>(AckleyOnePass{}, a, 0))); });
  timeit("tab", 1, [&] { tab_kernel<F, 16, 4><<<grid, 128, smem>>>(a, F{}); });
  {
    std::vector<double> ref(m * n), got(m * n);
    CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0)));
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    tab_kernel<F, 16, 4><<<grid, 128, smem>>>(a, F{});
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t q = 0; q < m * n; q++) bad += ref[q] != got[q];
    printf("tab parity: %lld bitwise mismatches of %lld\n", (long long)bad, (long long)(m * n));
  }
  {
    std::vector<double> ref(m * n), got(m * n);
    CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0)));
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    CK((launch_functor<RosenZ, 16, MODE_HVP>(RosenZ{}, a, 0)));
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    double mx = 0;
    for (int64_t q = 0; q < m * n; q++) {
      bad += ref[q] != got[q];
      mx = fmax(mx, fabs(ref[q] - got[q]) / fmax(1e-300, fabs(ref[q])));
    }
    printf("zseed parity: %lld bitwise mismatches of %lld, max rel diff %.3e\n", (long long)bad, (long long)(m * n), mx);
  }
  // parity of the variants against the library kernel (bitwise: same evaluation)
  {
    std::vector<double> ref(m * n), got(m * n);
    CK((launch_functor<F, 16, MODE_HVP>(F{}, a, 0)));
    CK(cudaMemcpy(ref.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, m * n * 8));
    const size_t psmem = 5 * n * kPad * 8;
    int occ = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, persist_kernel<F, 16, 4, 1>, 128, psmem));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    persist_kernel<F, 16, 4, 1><<<occ * sms, 128, psmem>>>(a, F{});
    CK(cudaMemcpy(got.data(), dout, m * n * 8, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t q = 0; q < m * n; q++) bad += ref[q] != got[q];
    printf("persist parity: %lld mismatches of %lld\n", (long long)bad, (long long)(m * n));
  }
  CK(cudaGetLastError());
  return 0;
}

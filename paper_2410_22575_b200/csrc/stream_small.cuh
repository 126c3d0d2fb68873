// stream_small.cuh -- Alg 7 for tiny n (NS in {2, 4, 8}): the HBM-facing end of the path.
//
// At n = 2 the batched HVP is bound by HBM, not FP64 (48 B and ~228 model FLOP per point,
// SURVEY §8(d)), so the memory path decides the rate.  The runtime-n register kernel stages
// a tile through a transposed shared-memory layout with per-element div/mod and scalar 8-byte
// loads, which is right for n >= 16 (a warp walks a row of 32 points) but leaves n = 2 at a
// third of HBM bandwidth (profiles/r02/).  Here:
//   * one THREAD per POINT (the paper's L0 level, Alg 9): all n rows and
//     n/C chunks of the point are evaluated by its thread, in Alg 7's order;
//   * a PERSISTENT grid (a multiple of the 148 SMs) walks tiles of 256 points; the tile's
//     points and vectors are each ONE contiguous range of global memory (row-major m x n,
//     PAPER.md:432), copied by one thread with 1-D bulk async copies (cp.async.bulk, the TMA
//     engine) into an S-stage shared-memory ring signalled by mbarriers, so S tiles per CTA
//     are in flight while the current one is computed;
//   * each thread reads its point and vector as 16-byte words, keeps them in registers, and
//     writes its n results with 16-byte coalesced stores.
//
// Per-evaluation execution (reading R8).  The row / chunk / variable loops are
// unrolled (NS is a compile-time constant, so the point, vector and result live in registers),
// but every evaluation reads its row index (from a per-CTA table) and the point's coordinates
// (from the thread's own shared-memory copy) with VOLATILE shared loads: to both compilers
// (NVVM and ptxas) they are fresh runtime values in each evaluation, so the value channel is
// recomputed in every evaluation and no work is shared across evaluations (that is the
// separate NEXT-4 hoisted entry point).  The chunk start j*C is a compile-time constant, as in
// the paper's NV/CHUNK-templated kernels: the seed's chunk slots are constants within the
// evaluation and nvcc folds them (x*1 -> x, IEEE-exact).  (Register moves through inline asm
// do not keep values opaque: ptxas propagates them, folds the seeds and shares the
// evaluations -- measured, same SASS for C = 1 and C = 2 at n = 2.)
#pragma once
#include <cstdint>

#include "chessfad/kernels.cuh"

namespace chessfad {

// shared-memory loads neither compiler may merge, hoist or fold
CHF_INL double ld_vol(const double* p) {
  double r;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return r;
}
CHF_INL int2 ld_vol(const int2* p) {
  int2 r;
  asm volatile("ld.volatile.shared.v2.s32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return r;
}

// CHUNK-INIT seed (Alg 4) over a register-resident point: compile-time
// variable index k (full unrolling of the function's variable loops), runtime i and cs.
template <int C>
struct RegSeed {
  static constexpr bool kStatic = true;  // variable loops fully unrolled (k compile-time)
  static constexpr bool kFused = true;   // the runtime-n kernel's forms (R5): same operations
  const double* a;                       // this evaluation's fresh copy of the point
  int stride;                            // 1
  int i, cs;                             // row / chunk start (runtime values)
  const double* sin2pi;                  // Ackley: sincos(2 pi a_k) of the point (registers)
  const double* cos2pi;
  CHF_INL hs<C> operator()(int k) const {
    hs<C> y;  // second-order slots: structural zeros (hdual.cuh hs<C>)
    y.v[0] = a[k];
    y.v[1] = (k == i) ? 1.0 : 0.0;
    const int off = k - cs;
#pragma unroll
    for (int l = 0; l < C; l++) y.v[2 + l] = (off == l) ? 1.0 : 0.0;
    return y;
  }
  CHF_INL double s2pi(int k) const { return sin2pi[k]; }
  CHF_INL double c2pi(int k) const { return cos2pi[k]; }
};

// ---------------------------------------------------------------- mbarrier / bulk copy PTX
CHF_INL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
CHF_INL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
CHF_INL void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
CHF_INL void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar` in bytes;
// bytes % 16 == 0, both addresses 16-byte aligned.  evict_first: the inputs are read once.
CHF_INL void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kStreamTP = 256;  // points per tile = threads per CTA
template <int NS>
struct StreamCfg {
  static constexpr int kStages = NS == 2 ? 4 : 2;  // tiles in flight per CTA
  static constexpr size_t kTileBytes = (size_t)kStreamTP * NS * sizeof(double);
  static constexpr int kEvals = NS * NS;  // (row, chunk) table entries (C = 1 bound)
  // points+vecs ring | the threads' point copies [NS][TP] | (i, cs) per evaluation | barriers
  static constexpr size_t kSmem = 2 * kStages * kTileBytes + kTileBytes + 8 * kEvals + 8 * kStages + 16;
};

// KCS: the chunk start is a compile-time constant (true) or read per evaluation like the row
// index (false; the HBM-bound corners measured faster that way, launch.cuh stream_fold_cs)
template <class F, int C, int NS, bool KCS = true>
__global__ void __launch_bounds__(kStreamTP, NS == 8 ? 1 : 2) hvp_stream_kernel(BatchArgs p, F f) {
  static_assert(NS % 2 == 0 && NS % C == 0, "NS even, C | NS");
  using Cfg = StreamCfg<NS>;
  constexpr int S = Cfg::kStages;
  constexpr bool TRIG = uses_trig2pi<F>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);  // stage s: points [TP*NS] | vecs [TP*NS]
  double* acopy = reinterpret_cast<double*>(smem_raw + 2 * S * Cfg::kTileBytes);  // [NS][TP]
  int2* evtab = reinterpret_cast<int2*>(smem_raw + (2 * S + 1) * Cfg::kTileBytes);  // [NS * NS / C]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (2 * S + 1) * Cfg::kTileBytes + 8 * Cfg::kEvals);
  const int tid = threadIdx.x;
  for (int q = tid; q < NS * (NS / C); q += blockDim.x) evtab[q] = make_int2(q / (NS / C), (q % (NS / C)) * C);
  const int64_t ntiles = (p.m + kStreamTP - 1) / kStreamTP;

  auto issue = [&](int64_t tile, int s) {  // one thread: bulk-copy tile's points and vectors
    const int64_t e0 = tile * kStreamTP;
    const int64_t cnt = (p.m - e0 < kStreamTP) ? p.m - e0 : kStreamTP;
    const uint32_t bytes = (uint32_t)(cnt * NS * sizeof(double));
    mbar_expect_tx(full + s, 2 * bytes);
    bulk_g2s(ring + (size_t)(2 * s) * kStreamTP * NS, p.points + e0 * NS, bytes, full + s);
    bulk_g2s(ring + (size_t)(2 * s + 1) * kStreamTP * NS, p.vecs + e0 * NS, bytes, full + s);
  };
  if (tid == 0) {
    for (int s = 0; s < S; s++) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int s = 0; s < S; s++) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  }
  __syncthreads();

  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
    const int s = it % S;
    mbar_wait(full + s, (uint32_t)((it / S) & 1));
    const int64_t e = tile * kStreamTP + tid;
    const bool live = e < p.m;
    double a[NS], v[NS];
    {
      const double2* ps = reinterpret_cast<const double2*>(ring + (size_t)(2 * s) * kStreamTP * NS) + tid * (NS / 2);
      const double2* vs = reinterpret_cast<const double2*>(ring + (size_t)(2 * s + 1) * kStreamTP * NS) + tid * (NS / 2);
#pragma unroll
      for (int q = 0; q < NS / 2; q++) {
        const double2 x = live ? ps[q] : make_double2(0.0, 0.0);
        const double2 w = live ? vs[q] : make_double2(0.0, 0.0);
        a[2 * q] = x.x;
        a[2 * q + 1] = x.y;
        v[2 * q] = w.x;
        v[2 * q + 1] = w.y;
      }
    }
    // WAR across proxies: the refill below is an async-proxy (TMA) write, which bar.sync alone
    // does not order after these generic-proxy shared loads (they may still be queued --
    // measured: whole warps read the NEXT tile at n = 8).  Each thread's proxy fence orders
    // its loads before the barrier, the barrier before the refill.
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();  // every thread holds its point: stage s may be refilled
    if (tid == 0) {
      const int64_t nxt = tile + (int64_t)S * gridDim.x;
      if (nxt < ntiles) issue(nxt, s);
    }
    if (!live) continue;

    double ts[NS], tc[NS];
    if (TRIG) {
#pragma unroll
      for (int k = 0; k < NS; k++) sincos(6.283185307179586 * a[k], ts + k, tc + k);
    }
#pragma unroll
    for (int k = 0; k < NS; k++) acopy[k * kStreamTP + tid] = a[k];  // this thread's slots only
    double out[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
      double res = 0.0;
#pragma unroll
      for (int j = 0; j < NS / C; j++) {
        double ao[NS];
#pragma unroll
        for (int k = 0; k < NS; k++) ao[k] = ld_vol(acopy + k * kStreamTP + tid);
        // row i opaque (read per evaluation), chunk start j C a compile-time constant: the seed's
        // chunk slots fold within the evaluation (reading R8), nothing is shared across evaluations
        const int2 ic = ld_vol(evtab + i * (NS / C) + j);  // == (i, j C)
        const RegSeed<C> y{ao, 1, ic.x, KCS ? j * C : ic.y, ts, tc};
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
}

}  // namespace chessfad

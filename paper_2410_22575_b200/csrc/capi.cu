// capi.cu -- the C-ABI of libchessfad.so (include/chessfad.h): argument validation,
// dispatch on (func, csize) to the compiled kernel set, the host-buffer pipeline, the
// model-FLOP count and the FP64 probe.  Host code only launches kernels; no compute here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <new>
#include <utility>
#include <vector>

#include "../../include/chessfad.h"
#include "launch.cuh"

using namespace chessfad;


namespace {

constexpr int kMaxNReg = 256;  // register-hDual path: (3 or 5)*n*33*8 B of shared memory per CTA
constexpr int kMaxNF3 = 128;   // F3: tensor-core kernel tiles (f3_mma.cuh), seed-sparse tiles

// hDual<32> needs > 255 registers (ptxas spills 400+ B) and measured ~25% slower than two
// 16-column groups (profiles/r01/campaign1/time_cfg3n*.jsonl), so C >= 32 runs as groups of 16.
bool reg_chunk_compiled(int C) { return C == 1 || C == 2 || C == 4 || C == 8 || C == 16; }

// Register path, C outside the compiled set: the chunk is executed as C/c' column groups of
// the largest compiled c' <= 16 dividing C.  By slot independence column k of a
// hDual<C> evaluation is bit-identical to column k of a hDual<c'> evaluation with the same
// row seed, so the results are those of hDual<C>; slots 0 and 1 are recomputed per group
// (executed FLOPs > model FLOPs, never fewer).
int reg_kernel_chunk(int C) {
  if (reg_chunk_compiled(C)) return C;
  for (int c = 16; c > 1; c >>= 1)
    if (C % c == 0) return c;
  return 1;
}

int validate(int func, int n, int csize, int64_t m, bool need_params_ptr, const void* params,
             const void* p1, const void* p2, const void* p3) {
  if (n < 1 || m < 0) return CHESSFAD_ERR_ARG;
  if (m > 0 && (!p1 || !p2 || (p3 == nullptr && need_params_ptr))) return CHESSFAD_ERR_ARG;
  if (csize < 1 || csize > n || n % csize != 0) return CHESSFAD_ERR_CHUNK;
  switch (func) {
    case CHESSFAD_ROSENBROCK:
    case CHESSFAD_PRODSUM:
      if (n < 2) return CHESSFAD_ERR_FUNC;
      break;
    case CHESSFAD_ACKLEY:
      break;
    case CHESSFAD_FLETCHER_POWELL:
      if (!params) return CHESSFAD_ERR_FUNC;
      break;
    default:
      return CHESSFAD_ERR_FUNC;
  }
  return CHESSFAD_OK;
}

constexpr size_t kSmemMax = 227 * 1024;

int supported(int func, int n, int csize, int mode) {
  (void)csize;  // every C | n runs (F3: runtime C; register path: reg_kernel_chunk)
  if (mode == MODE_HVP_ROWHOIST) mode = MODE_HVP;  // same shapes as the per-evaluation HVP
  if (func == CHESSFAD_FLETCHER_POWELL)  // tensor-core kernel, every mode (smem fits at NN = 128)
    return n <= kMaxNF3 && F3Mma<128, MODE_SYM_HVP>::smem_bytes() <= kSmemMax &&
           F3Mma<128, MODE_HVP>::smem_bytes() <= kSmemMax;
  return n <= kMaxNReg && reg_smem_bytes(func == CHESSFAD_ACKLEY, n, groups_for(n, kWarpsReg, mode), mode) <= kSmemMax;
}

// seed-sparse HVP (NEXT-4): Fletcher-Powell only; every C | n gives the same result (the
// columns of all chunks are formed one by one), so csize only has to be valid
bool sparse_supported(int func, int n) {
  if (func != CHESSFAD_FLETCHER_POWELL)  // register path: same shapes as the per-evaluation kernels
    return supported(func, n, 1, MODE_HVP) && supported(func, n, 1, MODE_HESS);
  return n <= kMaxNF3 && f3_sparse_smem_bytes(n, groups_for(n, kWarpsF3, MODE_HVP)) <= kSmemMax;
}

// F3 seed-sparse Alg 8: every warp owns a 32-point group (4 groups per CTA) -> n <= 64
bool f3_sparse_sym_hvp_fits(int n) {
  return n <= kMaxNF3 && f3_sparse_smem_bytes(n, groups_for(n, kWarpsF3, MODE_SYM_HVP)) <= kSmemMax;
}

// register path: the chunk runs as column groups of the largest compiled c' (reg_kernel_chunk)
template <int MODE>
cudaError_t dispatch_sparse_reg(int func, int Capi, const BatchArgs& a, cudaStream_t s) {
  const int C = reg_kernel_chunk(Capi);
#define CHF_SPR_CASE(F)                                           \
  switch (C) {                                                    \
    case 1: return launch_sparse_reg<F, 1, MODE>(a, s);           \
    case 2: return launch_sparse_reg<F, 2, MODE>(a, s);           \
    case 4: return launch_sparse_reg<F, 4, MODE>(a, s);           \
    case 8: return launch_sparse_reg<F, 8, MODE>(a, s);           \
    case 16: return launch_sparse_reg<F, 16, MODE>(a, s);         \
  }                                                               \
  break;
  switch (func) {
    case CHESSFAD_ROSENBROCK: CHF_SPR_CASE(FUNC_ROSENBROCK)
    case CHESSFAD_ACKLEY: CHF_SPR_CASE(FUNC_ACKLEY)
    case CHESSFAD_PRODSUM: CHF_SPR_CASE(FUNC_PRODSUM)
  }
#undef CHF_SPR_CASE
  return cudaErrorInvalidValue;
}

#ifndef CHF_SP_CB
#define CHF_SP_CB 16  // column block of the seed-sparse kernel (tuning knob; power of two <= 16)
#endif
#ifndef CHF_SP_CB_SMEM
#define CHF_SP_CB_SMEM 8  // ... with (A, B) in shared memory (n <= 32): 3 CTAs/SM (measured)
#endif

// seed-sparse entry: MODE_HVP / MODE_HESS for every function; the symmetric modes and the
// gradient for the register functions (F3's seed-sparse kernel implements Alg 7 / Alg 5 only)
template <int MODE>
int sparse_entry(int func, int n, int csize, int64_t m, const double* points, const double* vecs, double* out,
                 const double* params, void* stream, double* grad = nullptr) {
  constexpr bool HESS = mode_hess(MODE);
  int st = validate(func, n, csize, m, false, params, points, HESS ? out : vecs, out);
  if (st) return st;
  if (MODE == MODE_HESS_GRAD && m > 0 && !grad) return CHESSFAD_ERR_ARG;
  if (!sparse_supported(func, n)) return CHESSFAD_ERR_UNSUPPORTED;
  if (func == CHESSFAD_FLETCHER_POWELL && MODE == MODE_SYM_HVP && !f3_sparse_sym_hvp_fits(n))
    return CHESSFAD_ERR_UNSUPPORTED;
  if (mode_sym(MODE) && func != CHESSFAD_FLETCHER_POWELL && !supported(func, n, csize, MODE))
    return CHESSFAD_ERR_UNSUPPORTED;
  if (m == 0) return CHESSFAD_OK;
  BatchArgs a{};
  a.n = n;
  a.csize = csize;
  a.groups = 1;
  a.m = m;
  a.points = points;
  a.vecs = vecs;
  a.out = out;
  a.params = params;
  a.grad = grad;
  if (func != CHESSFAD_FLETCHER_POWELL) {
    const cudaError_t er = dispatch_sparse_reg<MODE>(func, csize, a, (cudaStream_t)stream);
    return er == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
  }
  cudaError_t e = cudaErrorInvalidValue;
  // column block: largest power of two <= CHF_SP_CB (n <= 32: <= CHF_SP_CB_SMEM) dividing n
  int cb = n <= 32 ? CHF_SP_CB_SMEM : CHF_SP_CB;
  while (n % cb) cb >>= 1;
  switch (cb) {
#define CHF_CASE_SP(CB) \
  case CB: e = launch_f3_sparse<CB, MODE>(a, (cudaStream_t)stream); break;
    CHF_FOR_CB(CHF_CASE_SP)
#undef CHF_CASE_SP
  }
  return e == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
}

template <int F>
cudaError_t dispatch_small(int C, const BatchArgs& a, cudaStream_t s) {
#define CHF_SMALL_CASE(FF, CC, NS) \
  if (C == CC && a.n == NS) return launch_small<FF, CC, NS>(a, s);
  CHF_FOR_SMALL(CHF_SMALL_CASE, F)
#undef CHF_SMALL_CASE
  return cudaErrorInvalidValue;
}

#ifndef CHF_STREAM_SMALL
#define CHF_STREAM_SMALL 1  // Alg 7 at n in {2, 4, 8} through hvp_stream_kernel (0: runtime-n kernel)
#endif
template <int F>
cudaError_t dispatch_stream(int C, const BatchArgs& a, cudaStream_t s) {
#define CHF_STREAM_CASE(FF, CC, NS) \
  if (C == CC && a.n == NS) return launch_stream<FF, CC, NS>(a, s);
  CHF_FOR_STREAM(CHF_STREAM_CASE, F)
#undef CHF_STREAM_CASE
  return cudaErrorInvalidValue;
}

// the stream kernel is used where it measured faster than the runtime-n kernel at m = 2^24
// (profiles/r02/g): n = 2 (HBM-bound: 2.5-3.4x) and n = 4 (1.3-2.7x) for every function; at
// n = 8 only prodsum (1.3x) -- Rosenbrock / Ackley at n = 8 are FP64-bound and the lane-per-
// point register kernel executes them better (up to 1.5x)
bool stream_small_n(int func, int n, int C) {
  (void)C;
  if (!CHF_STREAM_SMALL) return false;
  return n == 2 || n == 4 || (n == 8 && func == CHESSFAD_PRODSUM);
}

#ifndef CHF_REGN
#define CHF_REGN 1  // register path: kernels compiled for n in {8, 16, 32} (0: runtime-n kernel only)
#endif
#ifndef CHF_REGN_BIG
#define CHF_REGN_BIG 1  // ... and for n in {64, 128}, Alg 7
#endif
// Used where it measured faster (profiles/r02/ns/summary.txt: 1.1-5.8x for every HVP mode and
// F1/F2 Hessians at n <= 32; prodsum's Hessian modes measured up to 1.3x slower and keep the
// runtime-n kernel).  n in {64, 128}, Alg 7 only (profiles/r02/ns/big_summary.txt,
// profiles/r02/ns3/summary.txt): prodsum 2.4-10x at every C; Rosenbrock (volatile seeds,
// unrolled chunks) at n = 64 every C (1.04-3.1x), at n = 128 C >= 4 (C = 1, 2 slower); Ackley
// at n = 64 every C (1.1-1.6x; volatile seeds at C <= 2 and C >= 16), at n = 128 kernel chunk 8
// with volatile seeds (73.2 vs 79.3 ms per 2^16 points at the runtime kernel's best C;
// profiles/r02/ns3/ns_probe_ack128.txt) -- its other chunks spill and run slower.
#ifndef CHF_REGN_ALL
#define CHF_REGN_ALL 0  // tuning: every compiled-n instantiation, measured or not
#endif
bool regn_use(int func, int n, int C, int mode) {
  if (!CHF_REGN) return false;
  if (CHF_REGN_ALL) {
    if (n == 64 || n == 128) return mode == MODE_HVP;
    return n == 8 || n == 16 || n == 32;
  }
  if (n == 64 || n == 128) {
    if (!CHF_REGN_BIG || mode != MODE_HVP) return false;
    switch (func) {
      case CHESSFAD_PRODSUM: return true;
      case CHESSFAD_ROSENBROCK: return n == 64 || C >= 4;
      case CHESSFAD_ACKLEY: return n == 64 || C == 8;  // n = 128: kernel chunk 8 only (1.08x)
    }
    return false;
  }
  if (!(n == 8 || n == 16 || n == 32)) return false;
  return !(func == CHESSFAD_PRODSUM && mode_hess(mode));
}

bool aligned16(const BatchArgs& a) {
  return ((reinterpret_cast<uintptr_t>(a.points) | reinterpret_cast<uintptr_t>(a.vecs) |
           reinterpret_cast<uintptr_t>(a.out)) & 15) == 0;
}

template <int MODE>
cudaError_t dispatch_reg(int func, int Capi, const BatchArgs& a, cudaStream_t s) {
  const int C = reg_kernel_chunk(Capi);
  if constexpr (MODE == MODE_HVP) {
    if (stream_small_n(func, a.n, C) && aligned16(a)) {
      switch (func) {
        case CHESSFAD_ROSENBROCK: return dispatch_stream<FUNC_ROSENBROCK>(C, a, s);
        case CHESSFAD_ACKLEY: return dispatch_stream<FUNC_ACKLEY>(C, a, s);
        case CHESSFAD_PRODSUM: return dispatch_stream<FUNC_PRODSUM>(C, a, s);
      }
    }
  }
  if constexpr (MODE == MODE_HVP_ROWHOIST) {  // NEXT-4 (chessfad_hvp_batch_hoisted), register path
    // the compile-time kernels use 16-byte double2 loads/stores of whole point rows
    if (aligned16(a) && (a.n == 2 || a.n == 4 || a.n == 8 || a.n == 16)) {
      switch (func) {
        case CHESSFAD_ROSENBROCK: return dispatch_small<FUNC_ROSENBROCK>(C, a, s);
        case CHESSFAD_ACKLEY: return dispatch_small<FUNC_ACKLEY>(C, a, s);
        case CHESSFAD_PRODSUM: return dispatch_small<FUNC_PRODSUM>(C, a, s);
      }
    }
    return dispatch_reg<MODE_HVP>(func, Capi, a, s);  // no hoisted kernel: per-evaluation path
  } else {
    if (regn_use(func, a.n, C, MODE)) {  // the kernel compiled for this n (kernels.cuh NS)
#define CHF_CASE_NS(F, NS)                                     \
  if (a.n == NS) switch (C) {                                  \
      case 1: return launch_reg_n<F, 1, MODE, NS>(a, s);       \
      case 2: return launch_reg_n<F, 2, MODE, NS>(a, s);       \
      case 4: return launch_reg_n<F, 4, MODE, NS>(a, s);       \
      case 8: return launch_reg_n<F, 8, MODE, NS>(a, s);       \
      case 16: return launch_reg_n<F, 16, MODE, NS>(a, s);     \
    }
      if constexpr (MODE == MODE_HVP) {
        switch (func) {
          case CHESSFAD_ROSENBROCK: CHF_FOR_REGN_BIG_NS(CHF_CASE_NS, FUNC_ROSENBROCK) break;
          case CHESSFAD_ACKLEY: CHF_FOR_REGN_BIG_NS(CHF_CASE_NS, FUNC_ACKLEY) break;
          case CHESSFAD_PRODSUM: CHF_FOR_REGN_BIG_NS(CHF_CASE_NS, FUNC_PRODSUM) break;
        }
      }
      switch (func) {
        case CHESSFAD_ROSENBROCK: CHF_FOR_REGN_NS(CHF_CASE_NS, FUNC_ROSENBROCK) break;
        case CHESSFAD_ACKLEY: CHF_FOR_REGN_NS(CHF_CASE_NS, FUNC_ACKLEY) break;
        case CHESSFAD_PRODSUM: CHF_FOR_REGN_NS(CHF_CASE_NS, FUNC_PRODSUM) break;
      }
#undef CHF_CASE_NS
      return cudaErrorInvalidValue;
    }
#define CHF_CASE_C(F)                                  \
  switch (C) {                                         \
    case 1: return launch_reg<F, 1, MODE>(a, s);       \
    case 2: return launch_reg<F, 2, MODE>(a, s);       \
    case 4: return launch_reg<F, 4, MODE>(a, s);       \
    case 8: return launch_reg<F, 8, MODE>(a, s);       \
    case 16: return launch_reg<F, 16, MODE>(a, s);     \
  }                                                    \
  break;
  switch (func) {
    case CHESSFAD_ROSENBROCK: CHF_CASE_C(FUNC_ROSENBROCK)
    case CHESSFAD_ACKLEY: CHF_CASE_C(FUNC_ACKLEY)
    case CHESSFAD_PRODSUM: CHF_CASE_C(FUNC_PRODSUM)
  }
#undef CHF_CASE_C
  }
  return cudaErrorInvalidValue;
}

// F3: the tensor-core kernel for NN = n rounded up to a multiple of 8 (f3_mma.cuh)
template <int MODE>
cudaError_t dispatch_f3(const BatchArgs& a, cudaStream_t s) {
  switch ((a.n + 7) / 8 * 8) {
#define CHF_MMA_CASE(NN) \
  case NN: return launch_f3_mma<NN, MODE>(a, s);
    CHF_FOR_MMA_NN(CHF_MMA_CASE)
#undef CHF_MMA_CASE
  }
  return cudaErrorInvalidValue;
}

template <int MODE>
int run(int func, int n, int csize, int64_t m, const double* points, const double* vecs, double* out,
        const double* params, cudaStream_t s, double* grad = nullptr) {
  BatchArgs a;
  a.grad = grad;
  a.n = n;
  a.csize = csize;
  a.groups = 1;
  a.m = m;
  a.points = points;
  a.vecs = vecs;
  a.out = out;
  a.params = params;
  cudaError_t e;
  if constexpr (MODE == MODE_HVP_ROWHOIST) {
    e = (func == CHESSFAD_FLETCHER_POWELL) ? dispatch_f3<MODE>(a, s) : dispatch_reg<MODE>(func, csize, a, s);
  } else {
    e = (func == CHESSFAD_FLETCHER_POWELL) ? dispatch_f3<MODE>(a, s) : dispatch_reg<MODE>(func, csize, a, s);
  }
  return e == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
}

template <int MODE>
int batch_entry(int func, int n, int csize, int64_t m, const double* points, const double* vecs, double* out,
                const double* params, void* stream, double* grad = nullptr) {
  const bool hess = mode_hess(MODE);
  int st = validate(func, n, csize, m, false, params, points, hess ? out : vecs, out);
  if (st) return st;
  if (MODE == MODE_HESS_GRAD && m > 0 && !grad) return CHESSFAD_ERR_ARG;
  if (!supported(func, n, csize, MODE)) return CHESSFAD_ERR_UNSUPPORTED;
  if (m == 0) return CHESSFAD_OK;
  return run<MODE>(func, n, csize, m, points, vecs, out, params, (cudaStream_t)stream, grad);
}

// ---------------------------------------------------------------- FP64 probe kernel
__global__ void __launch_bounds__(256) fp64_probe_kernel(int64_t iters, double* sink) {
  const double b = 1.0 + 1e-16 * threadIdx.x, c = 1e-300;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int64_t it = 0; it < iters; it++) {
    x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
    x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
  }
  sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

}  // namespace

extern "C" {

int chessfad_hvp_batch(int func, int n, int csize, int64_t m, const double* points, const double* vecs, double* out,
                       const double* params, void* stream) {
  return batch_entry<MODE_HVP>(func, n, csize, m, points, vecs, out, params, stream);
}

int chessfad_hessian_batch(int func, int n, int csize, int64_t m, const double* points, double* hess,
                           const double* params, void* stream) {
  return batch_entry<MODE_HESS>(func, n, csize, m, points, nullptr, hess, params, stream);
}

int chessfad_sym_hvp_batch(int func, int n, int csize, int64_t m, const double* points, const double* vecs,
                           double* out, const double* params, void* stream) {
  return batch_entry<MODE_SYM_HVP>(func, n, csize, m, points, vecs, out, params, stream);
}

int chessfad_sym_hessian_batch(int func, int n, int csize, int64_t m, const double* points, double* hess,
                               const double* params, void* stream) {
  return batch_entry<MODE_SYM_HESS>(func, n, csize, m, points, nullptr, hess, params, stream);
}

int chessfad_hessian_grad_batch(int func, int n, int csize, int64_t m, const double* points, double* hess,
                                double* grad, const double* params, void* stream) {
  return batch_entry<MODE_HESS_GRAD>(func, n, csize, m, points, nullptr, hess, params, stream, grad);
}

int chessfad_hvp_batch_hoisted(int func, int n, int csize, int64_t m, const double* points, const double* vecs,
                               double* out, const double* params, void* stream) {
  return batch_entry<MODE_HVP_ROWHOIST>(func, n, csize, m, points, vecs, out, params, stream);
}

int chessfad_hvp_batch_seedsparse(int func, int n, int csize, int64_t m, const double* points, const double* vecs,
                                  double* out, const double* params, void* stream) {
  return sparse_entry<MODE_HVP>(func, n, csize, m, points, vecs, out, params, stream);
}

int chessfad_sym_hvp_batch_seedsparse(int func, int n, int csize, int64_t m, const double* points, const double* vecs,
                                      double* out, const double* params, void* stream) {
  return sparse_entry<MODE_SYM_HVP>(func, n, csize, m, points, vecs, out, params, stream);
}

int chessfad_sym_hessian_batch_seedsparse(int func, int n, int csize, int64_t m, const double* points, double* hess,
                                          const double* params, void* stream) {
  return sparse_entry<MODE_SYM_HESS>(func, n, csize, m, points, nullptr, hess, params, stream);
}

int chessfad_hessian_grad_batch_seedsparse(int func, int n, int csize, int64_t m, const double* points, double* hess,
                                           double* grad, const double* params, void* stream) {
  return sparse_entry<MODE_HESS_GRAD>(func, n, csize, m, points, nullptr, hess, params, stream, grad);
}

int chessfad_hessian_batch_seedsparse(int func, int n, int csize, int64_t m, const double* points, double* hess,
                                      const double* params, void* stream) {
  return sparse_entry<MODE_HESS>(func, n, csize, m, points, nullptr, hess, params, stream);
}

namespace {
constexpr int kHostSets = 3;  // buffer sets of the host pipeline (pieces in flight)
int64_t host_piece(int64_t m, int64_t piece_points) {
  if (piece_points <= 0) piece_points = std::max<int64_t>(4096, (m + 7) / 8);
  return std::max<int64_t>(1, std::min(piece_points, m));
}

// Piece schedule of the host pipeline: pieces of `piece` points, except that the first and the
// last three ramp (piece/8, /4, /2 ... /2, /4, /8) so that the pipeline's fill (the first H2D,
// which nothing overlaps) and drain (the last kernel and D2H) move little data.
std::vector<std::pair<int64_t, int64_t>> host_schedule(int64_t m, int64_t piece) {
  std::vector<std::pair<int64_t, int64_t>> sched;
  std::vector<int64_t> head, tail;
  int64_t body = m;
  if (m >= 4 * piece && piece >= 64) {
    for (int64_t d : {8, 4, 2}) {
      head.push_back(piece / d);
      tail.insert(tail.begin(), piece / d);
      body -= 2 * (piece / d);
    }
  }
  int64_t e0 = 0;
  for (int64_t c : head) sched.push_back({e0, c}), e0 += c;
  for (int64_t left = body; left > 0;) {
    const int64_t c = std::min(piece, left);
    sched.push_back({e0, c});
    e0 += c;
    left -= c;
  }
  for (int64_t c : tail) sched.push_back({e0, c}), e0 += c;
  return sched;
}
size_t host_ws_bytes(int func, int n, int64_t m, int64_t piece_points) {
  const size_t pbytes = (size_t)host_piece(m, piece_points) * n * sizeof(double);
  const size_t nparams = (func == CHESSFAD_FLETCHER_POWELL) ? (size_t)2 * n * n + n : 0;
  return (size_t)kHostSets * 3 * pbytes + nparams * sizeof(double) + 256;
}
}  // namespace

size_t chessfad_hvp_host_workspace_bytes(int func, int n, int64_t m, int64_t piece_points) {
  if (n < 1 || m < 0) return 0;
  return host_ws_bytes(func, n, m, piece_points);
}

}  // extern "C"

// Streams and events of the host-buffer pipeline: created once per chessfad_host_ctx and
// reused by every call on it (chessfad_hvp_batch_host makes a temporary one).
struct chessfad_host_ctx {
  enum { H2D = 0, KRN = 1, D2H = 2 };
  cudaStream_t ss[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ready = nullptr, ev[3][kHostSets] = {};
  int device = -1;
  cudaError_t init() {
    cudaError_t e = cudaGetDevice(&device);
    for (int k = 0; k < 3 && e == cudaSuccess; k++) e = cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    for (int k = 0; k < 3; k++)
      for (int b = 0; b < kHostSets && e == cudaSuccess; b++) e = cudaEventCreateWithFlags(&ev[k][b], cudaEventDisableTiming);
    return e;
  }
  ~chessfad_host_ctx() {
    for (int k = 0; k < 3; k++) {
      if (ss[k]) cudaStreamDestroy(ss[k]);
      for (int b = 0; b < kHostSets; b++)
        if (ev[k][b]) cudaEventDestroy(ev[k][b]);
    }
    if (ready) cudaEventDestroy(ready);
  }
};

namespace {
// Three-stage pipeline over pieces of the batch: an H2D stream copies piece p into buffer set
// p % 3 (after that set's previous D2H), a compute stream runs the kernel, a D2H stream copies
// the result back -- the H2D copy engine never waits for a kernel, H2D and D2H overlap.
// argument checks of the host-buffer entry points (no CUDA call)
int host_precheck(int func, int n, int csize, int64_t m, const double* points, const double* vecs, double* out,
                  const double* params, int64_t piece_points, void* workspace, size_t workspace_bytes) {
  int st = validate(func, n, csize, m, false, params, points, vecs, out);
  if (st) return st;
  if (!supported(func, n, csize, MODE_HVP)) return CHESSFAD_ERR_UNSUPPORTED;
  if (m > 0 && workspace && workspace_bytes < host_ws_bytes(func, n, m, piece_points)) return CHESSFAD_ERR_ARG;
  return CHESSFAD_OK;
}

int host_pipeline(chessfad_host_ctx* cx, int func, int n, int csize, int64_t m, const double* points,
                  const double* vecs, double* out, const double* params, int64_t piece_points, void* workspace,
                  size_t workspace_bytes, void* stream) {
  int st = host_precheck(func, n, csize, m, points, vecs, out, params, piece_points, workspace, workspace_bytes);
  if (st || m == 0) return st;
  const size_t need = host_ws_bytes(func, n, m, piece_points);
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != cx->device) return CHESSFAD_ERR_ARG;
  cudaStream_t s0 = (cudaStream_t)stream;
  const int64_t piece = host_piece(m, piece_points);
  const auto sched = host_schedule(m, piece);
  const int npieces = (int)sched.size();
  const size_t row = (size_t)n * sizeof(double);
  const size_t pdoubles = (size_t)piece * n;
  const size_t nparams = (func == CHESSFAD_FLETCHER_POWELL) ? (size_t)2 * n * n + n : 0;
  enum { H2D = 0, KRN = 1, D2H = 2 };
  cudaStream_t* ss = cx->ss;
  double* d_buf = (double*)workspace;
  const bool own = d_buf == nullptr;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { if (e == cudaSuccess) e = x; return e == cudaSuccess; };
  if (own) ok(cudaMallocAsync((void**)&d_buf, need, s0));
  if (e == cudaSuccess) {
    double* d_params = d_buf + (size_t)kHostSets * 3 * pdoubles;
    if (nparams) ok(cudaMemcpyAsync(d_params, params, nparams * sizeof(double), cudaMemcpyHostToDevice, s0));
    ok(cudaEventRecord(cx->ready, s0));
    for (int k = 0; k < 3; k++) ok(cudaStreamWaitEvent(ss[k], cx->ready, 0));
    for (int p = 0; p < npieces && e == cudaSuccess; p++) {
      const int b = p % kHostSets;
      double* dp = d_buf + (size_t)(3 * b) * pdoubles;
      double* dv = dp + pdoubles;
      double* dout = dv + pdoubles;
      const int64_t e0 = sched[p].first;
      const int64_t cnt = sched[p].second;
      const size_t bytes = (size_t)cnt * row;
      if (p >= kHostSets) ok(cudaStreamWaitEvent(ss[H2D], cx->ev[D2H][b], 0));  // set b drained
      ok(cudaMemcpyAsync(dp, points + e0 * n, bytes, cudaMemcpyHostToDevice, ss[H2D]));
      ok(cudaMemcpyAsync(dv, vecs + e0 * n, bytes, cudaMemcpyHostToDevice, ss[H2D]));
      ok(cudaEventRecord(cx->ev[H2D][b], ss[H2D]));
      ok(cudaStreamWaitEvent(ss[KRN], cx->ev[H2D][b], 0));
      if (e == cudaSuccess) {
        const int r = run<MODE_HVP>(func, n, csize, cnt, dp, dv, dout, nparams ? d_params : nullptr, ss[KRN]);
        if (r != CHESSFAD_OK) e = cudaErrorLaunchFailure;
      }
      ok(cudaEventRecord(cx->ev[KRN][b], ss[KRN]));
      ok(cudaStreamWaitEvent(ss[D2H], cx->ev[KRN][b], 0));
      ok(cudaMemcpyAsync(out + e0 * n, dout, bytes, cudaMemcpyDeviceToHost, ss[D2H]));
      ok(cudaEventRecord(cx->ev[D2H][b], ss[D2H]));
    }
    for (int k = 0; k < 3; k++) {  // s0 joins all three streams
      ok(cudaEventRecord(cx->ready, ss[k]));
      ok(cudaStreamWaitEvent(s0, cx->ready, 0));
    }
    if (own) ok(cudaFreeAsync(d_buf, s0));
  }
  const cudaError_t es = cudaStreamSynchronize(s0);
  if (e == cudaSuccess) e = es;
  return e == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
}
}  // namespace

extern "C" {

int chessfad_host_ctx_create(chessfad_host_ctx** ctx) {
  if (!ctx) return CHESSFAD_ERR_ARG;
  *ctx = nullptr;
  chessfad_host_ctx* c = new (std::nothrow) chessfad_host_ctx();
  if (!c) return CHESSFAD_ERR_CUDA;
  if (c->init() != cudaSuccess) {
    delete c;
    return CHESSFAD_ERR_CUDA;
  }
  *ctx = c;
  return CHESSFAD_OK;
}

int chessfad_host_ctx_destroy(chessfad_host_ctx* ctx) {
  delete ctx;  // NULL is a no-op
  return CHESSFAD_OK;
}

int chessfad_hvp_batch_host_ctx(chessfad_host_ctx* ctx, int func, int n, int csize, int64_t m, const double* points,
                                const double* vecs, double* out, const double* params, int64_t piece_points,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (!ctx) return CHESSFAD_ERR_ARG;
  return host_pipeline(ctx, func, n, csize, m, points, vecs, out, params, piece_points, workspace, workspace_bytes,
                       stream);
}

int chessfad_hvp_batch_host(int func, int n, int csize, int64_t m, const double* points, const double* vecs,
                            double* out, const double* params, int64_t piece_points, void* workspace,
                            size_t workspace_bytes, void* stream) {
  int st = host_precheck(func, n, csize, m, points, vecs, out, params, piece_points, workspace, workspace_bytes);
  if (st || m == 0) return st;
  chessfad_host_ctx* cx = nullptr;
  st = chessfad_host_ctx_create(&cx);
  if (st) return st;
  st = host_pipeline(cx, func, n, csize, m, points, vecs, out, params, piece_points, workspace, workspace_bytes,
                     stream);
  chessfad_host_ctx_destroy(cx);
  return st;
}

int chessfad_is_supported(int func, int n, int csize) {
  if (validate(func, n, csize, 0, false, func == CHESSFAD_FLETCHER_POWELL ? (const void*)1 : nullptr, nullptr,
               nullptr, nullptr))
    return 0;
  return supported(func, n, csize, MODE_HVP) && supported(func, n, csize, MODE_HESS);
}

int chessfad_is_supported_algo(int func, int n, int csize, int algo) {
  if (algo < CHESSFAD_ALGO_HVP || algo > CHESSFAD_ALGO_HESSIAN_GRAD_SEEDSPARSE) return 0;
  if (validate(func, n, csize, 0, false, func == CHESSFAD_FLETCHER_POWELL ? (const void*)1 : nullptr, nullptr,
               nullptr, nullptr))
    return 0;
  if (algo == CHESSFAD_ALGO_HVP_SEEDSPARSE || algo == CHESSFAD_ALGO_HESSIAN_SEEDSPARSE) return sparse_supported(func, n);
  if (algo >= CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE) {  // Fletcher-Powell: seed-sparse Alg 8 up to n = 64
    static const int smode[3] = {MODE_SYM_HVP, MODE_SYM_HESS, MODE_HESS_GRAD};
    if (func == CHESSFAD_FLETCHER_POWELL)
      return sparse_supported(func, n) && (algo != CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE || f3_sparse_sym_hvp_fits(n));
    return sparse_supported(func, n) && supported(func, n, csize, smode[algo - CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE]);
  }
  static const int mode_of[6] = {MODE_HVP, MODE_HESS, MODE_SYM_HVP, MODE_SYM_HESS, MODE_HVP_ROWHOIST, MODE_HESS_GRAD};
  return supported(func, n, csize, mode_of[algo]);
}

const char* chessfad_status_string(int status) {
  switch (status) {
    case CHESSFAD_OK: return "CHESSFAD_OK";
    case CHESSFAD_ERR_ARG: return "CHESSFAD_ERR_ARG: n < 1, m < 0 or NULL data pointer";
    case CHESSFAD_ERR_CHUNK: return "CHESSFAD_ERR_CHUNK: csize must satisfy 1 <= csize <= n and csize | n";
    case CHESSFAD_ERR_FUNC: return "CHESSFAD_ERR_FUNC: unknown function, n < 2, or missing Fletcher-Powell params";
    case CHESSFAD_ERR_UNSUPPORTED: return "CHESSFAD_ERR_UNSUPPORTED: (func, n, csize) not in the compiled set";
    case CHESSFAD_ERR_CUDA: return "CHESSFAD_ERR_CUDA: CUDA runtime error";
  }
  return "CHESSFAD: unknown status";
}

double chessfad_model_flops_per_point_algo(int func, int n, int csize, int algo) {
  if (algo < CHESSFAD_ALGO_HVP || algo > CHESSFAD_ALGO_HESSIAN_GRAD_SEEDSPARSE) return -1.0;
  if (validate(func, n, csize, 0, false, (const void*)1, nullptr, nullptr, nullptr)) return -1.0;
  const double C = csize, N = n;
  // per-evaluation hDual op counts of the canonical forms (DESIGN.md op table)
  double hm = 0, ha = 0, sm = 0, sa = 0, un = 0;
  switch (func) {
    case CHESSFAD_ROSENBROCK: hm = 3 * (N - 1); ha = 3 * N - 4; sm = N - 1; sa = N - 1; break;
    case CHESSFAD_ACKLEY: hm = N; ha = 2 * N - 1; sm = N + 4; sa = 1; un = N + 3; break;
    case CHESSFAD_FLETCHER_POWELL: hm = N; ha = 2 * N * N - 1; sm = 2 * N * N; sa = N; un = 2 * N; break;
    case CHESSFAD_PRODSUM: hm = N - 1; ha = N - 2; break;
  }
  const double per_eval = hm * (10 * C + 4) + ha * (2 * C + 2) + sm * (2 * C + 2) + sa + un * (4 * C + 2);
  const bool sym = algo == CHESSFAD_ALGO_SYM_HVP || algo == CHESSFAD_ALGO_SYM_HESSIAN ||
                   algo == CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE || algo == CHESSFAD_ALGO_SYM_HESSIAN_SEEDSPARSE;
  const double evals = sym ? N * (N / C + 1) / 2 : N * N / C;
  // HVP dot: every H_ij v_j term once (Alg 8: n(n+C)/2 direct + n(n-C)/2 mirrored) = 2n^2
  const bool hvp = algo == CHESSFAD_ALGO_HVP || algo == CHESSFAD_ALGO_SYM_HVP || algo == CHESSFAD_ALGO_HVP_HOISTED ||
                   algo == CHESSFAD_ALGO_HVP_SEEDSPARSE || algo == CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE;
  return evals * per_eval + (hvp ? 2 * N * N : 0.0);
}

double chessfad_model_flops_per_point(int func, int n, int csize, int hessian) {
  return chessfad_model_flops_per_point_algo(func, n, csize, hessian ? CHESSFAD_ALGO_HESSIAN : CHESSFAD_ALGO_HVP);
}

int chessfad_fp64_probe(int blocks, int64_t iters, double* sink, void* stream) {
  if (blocks < 1 || iters < 0 || !sink) return CHESSFAD_ERR_ARG;
  fp64_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, sink);
  return cudaGetLastError() == cudaSuccess ? CHESSFAD_OK : CHESSFAD_ERR_CUDA;
}

const char* chessfad_path(int func, int n, int csize, int algo) {
  if (!chessfad_is_supported_algo(func, n, csize, algo)) return "unsupported";
  const bool sparse = algo >= CHESSFAD_ALGO_HVP_SEEDSPARSE;
  if (func == CHESSFAD_FLETCHER_POWELL) {
    if (sparse) return "f3_seedsparse";
    return "f3_dmma";
  }
  if (sparse) return "reg_seedsparse";
  const int C = reg_kernel_chunk(csize);
  if (algo == CHESSFAD_ALGO_HVP && stream_small_n(func, n, C)) return "stream";  // 16-byte-aligned buffers
  if (algo == CHESSFAD_ALGO_HVP_HOISTED && (n == 2 || n == 4 || n == 8 || n == 16)) return "small_hoisted";
  const int mode = algo == CHESSFAD_ALGO_HESSIAN ? MODE_HESS : algo == CHESSFAD_ALGO_SYM_HESSIAN ? MODE_SYM_HESS
                   : algo == CHESSFAD_ALGO_HESSIAN_GRAD ? MODE_HESS_GRAD
                   : algo == CHESSFAD_ALGO_SYM_HVP ? MODE_SYM_HVP : MODE_HVP;
  return regn_use(func, n, C, mode) ? "reg_ns" : "reg";
}

const char* chessfad_version(void) { return "chessfad-b200 0.1.0 (sm_100a)"; }

}  // extern "C"

/*
 * chessfad.h -- C-ABI of the B200-native batched FP64 Hessian-vector product library
 * (libchessfad.so), a from-scratch implementation of the data-parallel hot path of
 * CHESSFAD (arXiv 2410.22575).
 *
 * Citations: PAPER.md / SPEC.md line numbers of the reference text (DESIGN.md lists the
 * section each belongs to).  All floating point is IEEE FP64 (the paper's
 * `double v[2*csize+2]`).
 *
 * Conventions shared by every entry point
 *   func     test function id (definitions):
 *              CHESSFAD_ROSENBROCK      sum 100(y_{i+1}-y_i^2)^2 + (1-y_i)^2, needs n >= 2
 *              CHESSFAD_ACKLEY          -20 exp(-0.2 sqrt(S/n)) - exp(sum cos(2 pi y)/n) + 20 + e
 *              CHESSFAD_FLETCHER_POWELL sum_k (E*_k - sum_j A_kj sin y_j + B_kj cos y_j)^2
 *              CHESSFAD_PRODSUM         sum y_i y_{i+1} (count calibration), needs n >= 2
 *   n        number of variables, >= 1
 *   csize    chunk size C of hDual<C>: 1 <= C <= n and C | n
 *            (the paper assumes exact division)
 *   m        number of points (instances); m == 0 is an empty no-op
 *   points   m x n FP64 row-major, point e at points[e*n .. e*n+n)
 *   vecs     m x n FP64 row-major, multiplicand of point e
 *   params   Fletcher-Powell only, else ignored (may be NULL): 2n^2+n FP64
 *            [A (n x n row-major) | B (n x n row-major) | E* (n)]
 *   stream   a cudaStream_t passed as void* (NULL = legacy default stream)
 *   Memory is owned by the caller.  Outputs must not alias inputs.  Outputs are fully
 *   overwritten.  NaN/Inf propagate and are not errors:
 *   Ackley at the origin yields NaN derivatives by design.
 *   The library never aborts, never throws across the ABI, allocates nothing that
 *   outlives a call, and keeps no global mutable state beyond one-time kernel attributes.
 *   Calls on distinct streams are thread-safe.
 */
#ifndef CHESSFAD_H
#define CHESSFAD_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum chessfad_func {
  CHESSFAD_ROSENBROCK = 0,
  CHESSFAD_ACKLEY = 1,
  CHESSFAD_FLETCHER_POWELL = 2,
  CHESSFAD_PRODSUM = 3
};

enum chessfad_status {
  CHESSFAD_OK = 0,
  CHESSFAD_ERR_ARG = 1,         /* n < 1, m < 0, or a NULL data pointer with m > 0 */
  CHESSFAD_ERR_CHUNK = 2,       /* csize < 1, csize > n, or n % csize != 0 */
  CHESSFAD_ERR_FUNC = 3,        /* unknown func, n < 2 for Rosenbrock/prodsum, NULL params for F3 */
  CHESSFAD_ERR_UNSUPPORTED = 4, /* (func, n, csize) outside the compiled set (chessfad_is_supported) */
  CHESSFAD_ERR_CUDA = 5         /* a CUDA runtime error (launch, copy, allocation) */
};

/*
 * Batched Hessian-vector product, Alg 7 CHESS-VEC over m points:
 *   out[e*n + i] = sum_j  d2f/dx_i dx_j (points[e]) * vecs[e*n + j]
 * computed row by row and chunk by chunk with hDual<csize> forward propagation
 * (Alg 4 CHUNK-INIT; Fig. 1 rules), never storing H
 * (PAPER.md:246).  points, vecs, out (m x n) and params are DEVICE pointers.
 * Asynchronous on `stream`: no host synchronisation; results are valid once the caller
 * synchronises the stream.  Returns a chessfad_status.
 */
int chessfad_hvp_batch(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                       double *out, const double *params, void *stream);

/*
 * Batched dense Hessian, Alg 5 CHUNK-HESS:
 *   hess[e*n*n + i*n + j] = d2f/dx_i dx_j (points[e])
 * every (i, j) computed (not mirrored), n^2/csize evaluations per point.
 * DEVICE pointers; hess is m x n x n.  Asynchronous on `stream`.
 */
int chessfad_hessian_batch(int func, int n, int csize, int64_t m, const double *points, double *hess,
                           const double *params, void *stream);

/*
 * Alg 5 plus the gradient by-product ("it can compute the Jacobian while
 * computing the Hessian"): additionally grad[e*n + i] = df/dx_i (points[e]), read from slot
 * v[1] of row i's evaluations (DEVICE pointer, m x n).  Same other arguments as
 * chessfad_hessian_batch; ERR_ARG if grad is NULL with m > 0.
 */
int chessfad_hessian_grad_batch(int func, int n, int csize, int64_t m, const double *points, double *hess,
                                double *grad, const double *params, void *stream);

/*
 * Symmetric chunked HVP, Alg 8 SC-HESS-VEC (§III-C): for row
 * i only chunks cn >= i/csize are evaluated (n(n/C+1)/2 evaluations per point);
 * each entry H_is of a chunk strictly after row i's chunk also adds H_is*vecs[i] to out[s].
 * Reading of the garbled loop bound (G8): all csize second-order slots are used and
 * out <- res.  Same arguments, layout and semantics as chessfad_hvp_batch.
 */
int chessfad_sym_hvp_batch(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                           double *out, const double *params, void *stream);

/*
 * Symmetric chunked Hessian, Alg 6 SCHUNK-HESS: chunks cn >= i/csize are
 * evaluated and stored; whole chunks strictly below row i's chunk are mirrored
 * (hess[e][s][i] = hess[e][i][s]); entries of the diagonal chunk are computed directly (mirror
 * loop read as exclusive of endindex, G9).  Same arguments as chessfad_hessian_batch.
 */
int chessfad_sym_hessian_batch(int func, int n, int csize, int64_t m, const double *points, double *hess,
                               const double *params, void *stream);

/*
 * NEXT-4 (beyond the paper): Alg 7 with value-channel hoisting.  Computations
 * that are identical across the n^2/C evaluations of a point are done once:
 *  - Rosenbrock, Ackley, prodsum at n in {2, 4, 8, 16}: kernels compiled for that n with
 *    rows, chunks and variables unrolled, so the CHUNK-INIT seeds are constants and nvcc
 *    folds them and computes each shared sub-expression (value channel, the first-order
 *    slots common to all rows) once per point; other n run the per-evaluation kernel;
 *  - Fletcher-Powell: slots 0/1 of every residual (f, df/dx_i) once per (point, row).
 * The outputs are those of chessfad_hvp_batch up to FP64 rounding (bit-identical for
 * Fletcher-Powell and on the integer pins); the executed FLOPs are BELOW the model count of
 * chessfad_model_flops_per_point_algo(.., CHESSFAD_ALGO_HVP_HOISTED), the paper's, so rates
 * quoted against the model are "effective".  Arguments as chessfad_hvp_batch.
 */
int chessfad_hvp_batch_hoisted(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                               double *out, const double *params, void *stream);

/*
 * NEXT-4 seed sparsity (beyond the paper): Alg 7 with the operations on exact-zero
 * seed slots skipped.  Rosenbrock, Ackley, prodsum: only the terms of the running sums that
 * touch variable i or the chunk are evaluated as hDuals (the others have derivative slots
 * that are exact +-0), O(C) instead of O(n) hDual ops per evaluation.  Fletcher-Powell: a
 * CHUNK-INIT seed (Alg 4) has derivative 1 in slot 1 only for variable i and
 * in slot 2+c only for variable cs+c, so each derivative slot of the E_k sums of F3 has ONE
 * nonzero term; the value slot does not depend on the seed and is formed once per point; work
 * per point O(n^3) instead of O(n^4/C), the same for every C.  Every remaining operation is
 * the one the per-evaluation path performs, in the same order, so with finite inputs `out`
 * equals chessfad_hvp_batch's bit for bit up to the sign of zero.  Executed FLOPs
 * are far BELOW the model count (CHESSFAD_ALGO_HVP_SEEDSPARSE reports the paper's model);
 * rates against the model are "effective".  Arguments and errors as chessfad_hvp_batch;
 * ERR_UNSUPPORTED outside the per-evaluation kernels' shapes (Fletcher-Powell: n > 128).
 */
int chessfad_hvp_batch_seedsparse(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                                  double *out, const double *params, void *stream);

/*
 * The same seed sparsity for the Hessian API (Alg 5 output): hess[e*n*n + i*n + j] as
 * chessfad_hessian_batch, bit-identical to it up to the sign of zero.  Arguments and errors
 * as chessfad_hessian_batch (Fletcher-Powell: n <= 128).
 */
int chessfad_hessian_batch_seedsparse(int func, int n, int csize, int64_t m, const double *points, double *hess,
                                      const double *params, void *stream);

/*
 * Seed sparsity (as chessfad_hvp_batch_seedsparse) for the symmetric algorithms and the
 * gradient by-product: Alg 8 SC-HESS-VEC,
 * Alg 6 SCHUNK-HESS and Alg 5 + gradient, evaluating only the
 * terms of each running sum that touch row i or the chunk (the others add exact +-0 to every
 * derivative slot; the gradient slot v[1] needs only the terms touching i).  Arguments,
 * layouts and results as chessfad_sym_hvp_batch / chessfad_sym_hessian_batch /
 * chessfad_hessian_grad_batch (bit-identical up to the sign of zero; Fletcher-Powell: within
 * rounding of its tensor-core per-evaluation kernel); executed FLOPs below the model.
 * Fletcher-Powell: Alg 6 and the gradient are supported (each (i, col) entry O(n); Alg 6 skips
 * the column blocks below row i's chunk for n <= 32 or n % 8 != 0, and mirrors); Alg 8 is
 * ERR_UNSUPPORTED (its scatter crosses the warps that own a point's rows in that kernel).
 */
int chessfad_sym_hvp_batch_seedsparse(int func, int n, int csize, int64_t m, const double *points,
                                      const double *vecs, double *out, const double *params, void *stream);
int chessfad_sym_hessian_batch_seedsparse(int func, int n, int csize, int64_t m, const double *points,
                                          double *hess, const double *params, void *stream);
int chessfad_hessian_grad_batch_seedsparse(int func, int n, int csize, int64_t m, const double *points,
                                           double *hess, double *grad, const double *params, void *stream);

/*
 * End-to-end variant of chessfad_hvp_batch on HOST buffers: points, vecs, out (m x n) and
 * params are HOST pointers (pinned memory gives copy/compute overlap; pageable memory
 * works but serialises).  The batch is split into pieces of `piece_points` points
 * (<= 0: library default, m/8; the first and last three pieces ramp down to 1/8 of that so
 * the pipeline's fill and drain are short) flowing through a three-stage pipeline -- an H2D stream,
 * a compute stream and a D2H stream with three device buffer sets -- so that both copy
 * directions overlap the kernels.  Device scratch: `workspace` (DEVICE, at least
 * chessfad_hvp_host_workspace_bytes(...) bytes, owned by the caller), or NULL to allocate
 * stream-ordered scratch inside the call.  SYNCHRONOUS: returns after `out` holds the
 * result.  `stream` orders the work after prior work on it (NULL = legacy default stream).
 * ERR_ARG if the workspace is too small.
 */
int chessfad_hvp_batch_host(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                            double *out, const double *params, int64_t piece_points, void *workspace,
                            size_t workspace_bytes, void *stream);

/*
 * Reusable host-pipeline context: the three streams and the events of
 * chessfad_hvp_batch_host, created once (on the current device) instead of per call.
 * create: *ctx = new context or NULL on failure (ERR_ARG if ctx is NULL, ERR_CUDA if a stream
 * or event cannot be created).  destroy: releases it (NULL is a no-op); the caller must not
 * destroy a context while a call on it is running.  A context serves one call at a time.
 */
typedef struct chessfad_host_ctx chessfad_host_ctx;
int chessfad_host_ctx_create(chessfad_host_ctx **ctx);
int chessfad_host_ctx_destroy(chessfad_host_ctx *ctx);

/*
 * chessfad_hvp_batch_host on a context (same arguments, semantics and errors); ERR_ARG if ctx
 * is NULL or was created on another device than the current one.
 */
int chessfad_hvp_batch_host_ctx(chessfad_host_ctx *ctx, int func, int n, int csize, int64_t m,
                                const double *points, const double *vecs, double *out, const double *params,
                                int64_t piece_points, void *workspace, size_t workspace_bytes, void *stream);

/*
 * COMPARISON BASELINE, not the product path: the paper's own GPU design, Fig. 2 "L2"
 * recompiled for sm_100a -- one thread per (instance, row, chunk), a
 * materialised per-thread hDual<C> y[n] seed array, partial dots reduced through shared
 * memory with __syncthreads.  Same result as chessfad_hvp_batch (within rounding).
 * Rosenbrock and prodsum, n in {2, 4, 8, 16}, csize in {1, 2, 4, 8, 16}, csize | n; else
 * ERR_UNSUPPORTED.  Device pointers, asynchronous on `stream`.
 */
int chessfad_hvp_batch_paper_l2(int func, int n, int csize, int64_t m, const double *points, const double *vecs,
                                double *out, void *stream);

/* The paper's three GPU levels as comparison baselines: level 0 = Alg 9 L0 (thread per
 * instance), 1 = Alg 10 L1 (thread per instance x row), 2 = Fig. 2 L2 (= the call above).
 * Same restrictions; ERR_ARG for another level. */
int chessfad_hvp_batch_paper(int level, int func, int n, int csize, int64_t m, const double *points,
                             const double *vecs, double *out, void *stream);

/* Device workspace bytes chessfad_hvp_batch_host needs for (func, n, m, piece_points). */
size_t chessfad_hvp_host_workspace_bytes(int func, int n, int64_t m, int64_t piece_points);

/* 1 if (func, n, csize) runs for both chessfad_hvp_batch and chessfad_hessian_batch, else 0
 * (argument errors also give 0).  Compiled set: Fletcher-Powell any csize | n, n <= 128 (every
 * entry point); the other functions n <= 256 (Ackley n <= 176), with one hDual<csize> per
 * evaluation for csize in {1,2,4,8,16} and, for any other csize | n, csize/c' column groups of
 * the largest c' in {1,2,4,8,16} dividing csize (bit-identical results by slot independence,
 * SPEC.md:107; slots 0/1 recomputed per group). */
int chessfad_is_supported(int func, int n, int csize);

/* algorithm ids for chessfad_is_supported_algo / chessfad_model_flops_per_point_algo */
enum chessfad_algo {
  CHESSFAD_ALGO_HVP = 0,          /* Alg 7, chessfad_hvp_batch */
  CHESSFAD_ALGO_HESSIAN = 1,      /* Alg 5, chessfad_hessian_batch */
  CHESSFAD_ALGO_SYM_HVP = 2,      /* Alg 8, chessfad_sym_hvp_batch */
  CHESSFAD_ALGO_SYM_HESSIAN = 3,  /* Alg 6, chessfad_sym_hessian_batch */
  CHESSFAD_ALGO_HVP_HOISTED = 4,  /* Alg 7 + NEXT-4 value-channel hoisting, chessfad_hvp_batch_hoisted */
  CHESSFAD_ALGO_HESSIAN_GRAD = 5, /* Alg 5 + gradient by-product, chessfad_hessian_grad_batch */
  CHESSFAD_ALGO_HVP_SEEDSPARSE = 6, /* Alg 7 + NEXT-4 seed sparsity, chessfad_hvp_batch_seedsparse */
  CHESSFAD_ALGO_HESSIAN_SEEDSPARSE = 7, /* Alg 5 + seed sparsity, chessfad_hessian_batch_seedsparse */
  CHESSFAD_ALGO_SYM_HVP_SEEDSPARSE = 8, /* Alg 8 + seed sparsity (F1/F2/F4), chessfad_sym_hvp_batch_seedsparse */
  CHESSFAD_ALGO_SYM_HESSIAN_SEEDSPARSE = 9, /* Alg 6 + seed sparsity, chessfad_sym_hessian_batch_seedsparse */
  CHESSFAD_ALGO_HESSIAN_GRAD_SEEDSPARSE = 10 /* Alg 5 + gradient + seed sparsity */
};

/* 1 if (func, n, csize) runs for the given algorithm, else 0. */
int chessfad_is_supported_algo(int func, int n, int csize, int algo);

/* Static description of a status code. */
const char *chessfad_status_string(int status);

/*
 * Model FLOPs per point of one call: the paper's
 * §V count extended to all hDual ops with hh* = 10C+4 (6C+3 mul +
 * 4C+1 add, Fig. 1 code), hh+ = s* = 2C+2, s+ = 1, unary = 4C+2 (g, g', g'' count 0),
 * times n^2/C evaluations, plus the 2n^2 of the HVP dot when hessian == 0.
 * Returns -1 on invalid arguments.
 */
double chessfad_model_flops_per_point(int func, int n, int csize, int hessian);

/* Model FLOPs per point for any algorithm id: evaluations (n^2/C for Alg 5/7, n(n/C+1)/2 for
 * Alg 6/8) x per-evaluation cost, plus 2n^2 for the HVP algorithms (Alg 8's
 * n(n+C)/2 direct and n(n-C)/2 mirrored terms also total n^2 multiply-adds). */
double chessfad_model_flops_per_point_algo(int func, int n, int csize, int algo);

/*
 * FP64 pipe probe: launches `blocks` x 256 threads, each running `iters` iterations of one
 * DFMA on each of 8 independent chains, and writes one double per thread to `sink`
 * (DEVICE, blocks*256 doubles) so nothing is dead.  FLOPs per launch =
 * blocks * 256 * iters * 16.  Used by bench.py to measure the attainable FP64 rate.
 */
int chessfad_fp64_probe(int blocks, int64_t iters, double *sink, void *stream);

/*
 * Which kernel family a call with these arguments runs (introspection for tests and the bench;
 * DESIGN.md §3 describes each): "reg" (hDual<C> in registers, lane = point, warp = row),
 * "stream" (n in {2,4,8}, thread per point, bulk-copy ring; 16-byte-aligned buffers, else
 * "reg"), "small_hoisted", "reg_seedsparse", "f3_dmma" (Fletcher-Powell E-sums on the FP64
 * tensor core), "f3_seedsparse", or "unsupported".  Static string, never NULL.
 */
const char *chessfad_path(int func, int n, int csize, int algo);

/* Library version string. */
const char *chessfad_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CHESSFAD_H */

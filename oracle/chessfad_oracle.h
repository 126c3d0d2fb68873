/*
 * chessfad_oracle.h -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * Plain, slow, obviously-correct CPU oracle for the CHESSFAD batched Hessian-vector
 * product (arXiv 2410.22575).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library.  It shares no
 * code, header, table or constant with the CUDA product path (paper_2410_22575_b200/).
 *
 * Citations are PAPER.md / SPEC.md line numbers of the reference text.
 * All arithmetic is IEEE FP64, compiled with -ffp-contract=off, in the order the
 * paper writes it (Fig. 1; Alg 1-8).
 */
#ifndef CHESSFAD_ORACLE_H
#define CHESSFAD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* test functions (canonical forms in DESIGN.md) */
enum { OR_ROSENBROCK = 0, OR_ACKLEY = 1, OR_FLETCHER_POWELL = 2, OR_PRODSUM = 3 };
/* status */
enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_CHUNK = 2, OR_ERR_FUNC = 3 };
/* hDual binary / mixed operations exposed for unit pins */
enum {
  OR_OP_ADD = 0, OR_OP_SUB = 1, OR_OP_MUL = 2, OR_OP_DIV = 3,
  OR_OP_SADD = 4,  /* c + u */
  OR_OP_ADDS = 5,  /* u + c */
  OR_OP_SSUB = 6,  /* c - u */
  OR_OP_SUBS = 7,  /* u - c */
  OR_OP_SMUL = 8,  /* c * u */
  OR_OP_DIVS = 9,  /* u / c */
  OR_OP_SDIV = 10, /* c / u */
  OR_OP_NEG = 11
};
/* elementary functions */
enum { OR_G_SIN = 0, OR_G_COS = 1, OR_G_EXP = 2, OR_G_SQRT = 3, OR_G_LOG = 4, OR_G_ABS = 5 };
/* comparisons on the value slot */
enum { OR_CMP_LT = 0, OR_CMP_GT = 1, OR_CMP_LE = 2, OR_CMP_GE = 3, OR_CMP_EQ = 4 };

#define OR_CMAX 128

/* ---- hDual<C> primitives: arrays of 2C+2 doubles ---- */
int or_hd_binary(int op, int C, const double *u, const double *v, double c, double *r);
int or_hd_unary(int g, int C, const double *u, double *r);
int or_hd_compare(int cmp, const double *u, const double *v);

/* ---- seeding ---- */
/* Alg 1 INITIALIZE: y is n x 4 */
void or_initialize(int n, const double *a, int i, int j, double *y);
/* Alg 4 CHUNK-INIT: y is n x (2C+2) */
void or_chunk_init(int n, const double *a, int i, int cstart, int C, double *y);

/* ---- function evaluation ---- */
int or_eval_hdual(int func, int n, const double *params, int C, const double *y, double *t);
int or_eval_scalar(int func, int n, const double *params, const double *x, double *f);

/* ---- single-point algorithms ---- */
int or_hessian(int func, int n, const double *params, const double *a, double *H);              /* Alg 2 */
int or_sym_hessian(int func, int n, const double *params, const double *a, double *H);          /* Alg 3 */
int or_chunk_hess(int func, int n, int C, const double *params, const double *a,
                  double *H, double *grad);                                                     /* Alg 5 */
int or_schunk_hess(int func, int n, int C, const double *params, const double *a,
                   double *H, double *grad);                                                    /* Alg 6 */
int or_chess_vec(int func, int n, int C, const double *params, const double *a,
                 const double *in, double *out, double *sabs);                                  /* Alg 7 */
int or_sc_hess_vec(int func, int n, int C, const double *params, const double *a,
                   const double *in, double *out);                                              /* Alg 8 */
/* the full (n+1)(n+2)/2-component scheme of the cited prior work: one
   evaluation of f gives the whole Hessian (upper triangle mirrored) and the gradient */
int or_full_scheme_hessian(int func, int n, const double *params, const double *a,
                           double *H, double *grad);

/* ---- batches over m points (row-major m x n), std::thread-free: pthreads over points ---- */
int or_hvp_batch(int func, int n, int C, int64_t m, const double *points, const double *vecs,
                 double *out, double *sabs, const double *params, int nthreads);
int or_sc_hvp_batch(int func, int n, int C, int64_t m, const double *points, const double *vecs,
                    double *out, const double *params, int nthreads);
int or_hessian_batch(int func, int n, int C, int64_t m, const double *points, double *hess,
                     const double *params, int nthreads);

/* ---- instrumentation (thread-local) ---- */
void or_counters_reset(void);
/* evals: number of f<hDual> evaluations; mul/add: scalar multiplications / additions
   (only counted in the counting build, liboracle_count.so; 0 otherwise) */
void or_counters_get(int64_t *evals, int64_t *mul, int64_t *add);
int or_is_counting_build(void);

#ifdef __cplusplus
}
#endif
#endif

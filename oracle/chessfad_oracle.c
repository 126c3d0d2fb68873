/*
 * chessfad_oracle.c -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * The plain CPU oracle for the CHESSFAD batched FP64 Hessian-vector product
 * (arXiv 2410.22575).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code with the CUDA
 * path.  Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/__init__.py);
 * the counting build adds -DOR_COUNTING.
 *
 * What it computes: for every point, r = Hess f(a) . v by
 * Alg 7 CHESS-VEC over a runtime-C hDual whose rules are the
 * paper's Fig. 1 code and sum/product/sin rules;
 * the Hessian by Alg 5 CHUNK-HESS.  Alg 1/2/3/6/8 and the full
 * (n+1)(n+2)/2 scheme are here as cross-checks.
 *
 * Every value is carried as an array of doubles.  One "carrier" description
 * (scalar / hDual<C> / full scheme) lets the four test functions be written once, in
 * the canonical forms of DESIGN.md, and run on every carrier.
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, SPEC examples, FD, full scheme,
 * mpmath goldens, operation counts).  No function here is "parity unpinned".
 */
#include "chessfad_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ counting */
static _Thread_local int64_t g_evals, g_mul, g_add;

#ifdef OR_COUNTING
#define MUL(a, b) (g_mul++, (a) * (b))
#define ADD(a, b) (g_add++, (a) + (b))
#define SUB(a, b) (g_add++, (a) - (b))
int or_is_counting_build(void) { return 1; }
#else
#define MUL(a, b) ((a) * (b))
#define ADD(a, b) ((a) + (b))
#define SUB(a, b) ((a) - (b))
int or_is_counting_build(void) { return 0; }
#endif

void or_counters_reset(void) { g_evals = g_mul = g_add = 0; }
void or_counters_get(int64_t *evals, int64_t *mul, int64_t *add) {
  if (evals) *evals = g_evals;
  if (mul) *mul = g_mul;
  if (add) *add = g_add;
}

/* ------------------------------------------------------------------ carriers */
enum { K_SCALAR = 0, K_HDUAL = 1, K_FULL = 2 };
typedef struct {
  int kind;
  int C;     /* hDual chunk size */
  int n;     /* full scheme: number of variables */
  int ncomp; /* doubles per value */
} car;

static car car_scalar(void) { car c = {K_SCALAR, 0, 0, 1}; return c; }
static car car_hdual(int C) { car c = {K_HDUAL, C, 0, 2 * C + 2}; return c; }
static car car_full(int n) { car c = {K_FULL, 0, n, (n + 1) * (n + 2) / 2}; return c; }

/* full scheme layout: v[0]=f, v[1+i]=df/dx_i, v[1+n+tri(i,j)] = d2f/dx_i dx_j, i<=j */
static int tri(int n, int i, int j) { return i * n - i * (i - 1) / 2 + (j - i); }

static void v_copy(const car *K, const double *u, double *r) { memcpy(r, u, sizeof(double) * K->ncomp); }

/* u + v, u - v: componentwise, 2C+2 additions (Fig. 1 :276-280) */
static void v_add(const car *K, const double *u, const double *v, double *r) {
  for (int s = 0; s < K->ncomp; s++) r[s] = ADD(u[s], v[s]);
}
static void v_sub(const car *K, const double *u, const double *v, double *r) {
  for (int s = 0; s < K->ncomp; s++) r[s] = SUB(u[s], v[s]);
}
/* c + u and u + c: value slot only (Fig. 1 :282-300) */
static void v_sadd(const car *K, double c, const double *u, double *r) {
  r[0] = ADD(c, u[0]);
  for (int s = 1; s < K->ncomp; s++) r[s] = u[s];
}
static void v_adds(const car *K, const double *u, double c, double *r) {
  r[0] = ADD(u[0], c);
  for (int s = 1; s < K->ncomp; s++) r[s] = u[s];
}
/* c - u: value slot subtraction, derivative slots negated (no flop) */
static void v_ssub(const car *K, double c, const double *u, double *r) {
  r[0] = SUB(c, u[0]);
  for (int s = 1; s < K->ncomp; s++) r[s] = -u[s];
}
static void v_subs(const car *K, const double *u, double c, double *r) {
  r[0] = SUB(u[0], c);
  for (int s = 1; s < K->ncomp; s++) r[s] = u[s];
}
static void v_neg(const car *K, const double *u, double *r) {
  for (int s = 0; s < K->ncomp; s++) r[s] = -u[s];
}
/* c * u: every slot scaled, 2C+2 multiplications (Fig. 1 :323-338) */
static void v_smul(const car *K, double c, const double *u, double *r) {
  for (int s = 0; s < K->ncomp; s++) r[s] = MUL(c, u[s]);
}

/* u * v: Fig. 1 operator* (PAPER.md:302-321), term order exactly as printed:
 *   r0      = u0*v0
 *   r[i]    = u0*v[i] + v0*u[i],                          i = 1..C+1
 *   r[C+j]  = u0*v[C+j] + u1*v[j] + v1*u[j] + v0*u[C+j],  j = 2..C+1
 * i.e. 6C+3 multiplications and (C+1)+3C = 4C+1 additions (reading G1). */
static void v_mul(const car *K, const double *u, const double *v, double *r) {
  if (K->kind == K_SCALAR) { r[0] = MUL(u[0], v[0]); return; }
  if (K->kind == K_HDUAL) {
    const int C = K->C;
    double t[2 * OR_CMAX + 2];
    t[0] = MUL(u[0], v[0]);
    for (int i = 1; i <= C + 1; i++) t[i] = ADD(MUL(u[0], v[i]), MUL(v[0], u[i]));
    for (int j = 2; j <= C + 1; j++)
      t[C + j] = ADD(ADD(ADD(MUL(u[0], v[C + j]), MUL(u[1], v[j])), MUL(v[1], u[j])), MUL(v[0], u[C + j]));
    memcpy(r, t, sizeof(double) * (2 * C + 2));
    return;
  }
  /* full scheme, same product rule on every (i<=j) pair */
  {
    const int n = K->n;
    double *t = (double *)malloc(sizeof(double) * K->ncomp);
    t[0] = MUL(u[0], v[0]);
    for (int i = 0; i < n; i++) t[1 + i] = ADD(MUL(u[0], v[1 + i]), MUL(v[0], u[1 + i]));
    for (int i = 0; i < n; i++)
      for (int j = i; j < n; j++) {
        int h = 1 + n + tri(n, i, j);
        t[h] = ADD(ADD(ADD(MUL(u[0], v[h]), MUL(u[1 + i], v[1 + j])), MUL(v[1 + i], u[1 + j])), MUL(v[0], u[h]));
      }
    memcpy(r, t, sizeof(double) * K->ncomp);
    free(t);
  }
}

/* u / v: quotient rule (the paper lists "/" without a rule)
 *   r0 = u0/v0;  r[k] = (u[k] - r0*v[k]) / v0;
 *   r[C+k] = (u[C+k] - r1*v[k] - r[k]*v1 - r0*v[C+k]) / v0 */
static void v_div(const car *K, const double *u, const double *v, double *r) {
  if (K->kind == K_SCALAR) { r[0] = u[0] / v[0]; return; }
  if (K->kind == K_HDUAL) {
    const int C = K->C;
    double t[2 * OR_CMAX + 2];
    t[0] = u[0] / v[0];
    for (int k = 1; k <= C + 1; k++) t[k] = SUB(u[k], MUL(t[0], v[k])) / v[0];
    for (int k = 2; k <= C + 1; k++)
      t[C + k] = SUB(SUB(SUB(u[C + k], MUL(t[1], v[k])), MUL(t[k], v[1])), MUL(t[0], v[C + k])) / v[0];
    memcpy(r, t, sizeof(double) * (2 * C + 2));
    return;
  }
  {
    const int n = K->n;
    double *t = (double *)malloc(sizeof(double) * K->ncomp);
    t[0] = u[0] / v[0];
    for (int i = 0; i < n; i++) t[1 + i] = SUB(u[1 + i], MUL(t[0], v[1 + i])) / v[0];
    for (int i = 0; i < n; i++)
      for (int j = i; j < n; j++) {
        int h = 1 + n + tri(n, i, j);
        t[h] = SUB(SUB(SUB(u[h], MUL(t[1 + i], v[1 + j])), MUL(t[1 + j], v[1 + i])), MUL(t[0], v[h])) / v[0];
      }
    memcpy(r, t, sizeof(double) * K->ncomp);
    free(t);
  }
}

/* (g, g', g'') of the elementary functions */
static void g_triple(int g, double x, double *g0, double *g1, double *g2) {
  switch (g) {
  case OR_G_SIN: *g0 = sin(x); *g1 = cos(x); *g2 = -sin(x); break;
  case OR_G_COS: *g0 = cos(x); *g1 = -sin(x); *g2 = -cos(x); break;
  case OR_G_EXP: *g0 = exp(x); *g1 = *g0; *g2 = *g0; break;
  case OR_G_SQRT: {
    double r = sqrt(x);
    *g0 = r; *g1 = 1.0 / (2.0 * r); *g2 = -1.0 / (4.0 * x * r);
    break;
  }
  case OR_G_LOG: *g0 = log(x); *g1 = 1.0 / x; *g2 = -1.0 / (x * x); break;
  case OR_G_ABS: *g0 = fabs(x); *g1 = (x > 0) ? 1.0 : ((x < 0) ? -1.0 : 0.0); *g2 = 0.0; break;
  default: *g0 = *g1 = *g2 = NAN;
  }
}

/* unary g: the second-order chain rule; sin as printed at PAPER.md:99,
 *   r0 = g(u0);  r[k] = g'*u[k] (k = 1..C+1);  r[C+k] = g'*u[C+k] + (g''*u1)*u[k]
 * g, g', g'' are evaluated on u0 and not counted (SURVEY §8(d) model convention). */
static void v_unary(const car *K, int g, const double *u, double *r) {
  double g0, g1, g2;
  g_triple(g, u[0], &g0, &g1, &g2);
  if (K->kind == K_SCALAR) { r[0] = g0; return; }
  if (K->kind == K_HDUAL) {
    const int C = K->C;
    double t[2 * OR_CMAX + 2];
    t[0] = g0;
    for (int k = 1; k <= C + 1; k++) t[k] = MUL(g1, u[k]);
    double g2u1 = MUL(g2, u[1]);
    for (int k = 2; k <= C + 1; k++) t[C + k] = ADD(MUL(g1, u[C + k]), MUL(g2u1, u[k]));
    memcpy(r, t, sizeof(double) * (2 * C + 2));
    return;
  }
  {
    const int n = K->n;
    double *t = (double *)malloc(sizeof(double) * K->ncomp);
    t[0] = g0;
    for (int i = 0; i < n; i++) t[1 + i] = MUL(g1, u[1 + i]);
    for (int i = 0; i < n; i++) {
      double g2ui = MUL(g2, u[1 + i]);
      for (int j = i; j < n; j++) {
        int h = 1 + n + tri(n, i, j);
        t[h] = ADD(MUL(g1, u[h]), MUL(g2ui, u[1 + j]));
      }
    }
    memcpy(r, t, sizeof(double) * K->ncomp);
    free(t);
  }
}

/* ------------------------------------------------------------------ test functions
 * Canonical forms.  Loops
 * ascend; the first term of every sum initialises it.  y: n values of K->ncomp doubles.
 */
typedef struct {
  const car *K;
  double *buf; /* scratch: nslots * ncomp doubles */
  int nslots;
} ws_t;

static double *ws_slot(ws_t *w, int s) { return w->buf + (size_t)s * w->K->ncomp; }

/* F1 Rosenbrock: sum_{i<n-1} 100(y_{i+1} - y_i^2)^2 + (1 - y_i)^2 */
static void f_rosenbrock(const car *K, int n, const double *y, double *out, ws_t *w) {
  const int nc = K->ncomp;
  double *yy = ws_slot(w, 0), *d = ws_slot(w, 1), *e = ws_slot(w, 2), *dd = ws_slot(w, 3);
  double *t1 = ws_slot(w, 4), *ee = ws_slot(w, 5), *t = ws_slot(w, 6), *s = ws_slot(w, 7);
  for (int i = 0; i < n - 1; i++) {
    const double *yi = y + (size_t)i * nc, *yi1 = y + (size_t)(i + 1) * nc;
    v_mul(K, yi, yi, yy);      /* y_i*y_i           */
    v_sub(K, yi1, yy, d);      /* d = y_{i+1} - yy  */
    v_ssub(K, 1.0, yi, e);     /* e = 1 - y_i       */
    v_mul(K, d, d, dd);        /* d*d               */
    v_smul(K, 100.0, dd, t1);  /* 100*(d*d)         */
    v_mul(K, e, e, ee);        /* e*e               */
    v_add(K, t1, ee, t);       /* t = 100 d^2 + e^2 */
    if (i == 0) v_copy(K, t, s);
    else v_add(K, s, t, s);
  }
  v_copy(K, s, out);
}

/* F2 Ackley: -20 exp(-0.2 sqrt(S1/n)) - exp(S2/n) + 20 + e */
static void f_ackley(const car *K, int n, const double *y, double *out, ws_t *w) {
  const int nc = K->ncomp;
  const double two_pi = 6.283185307179586, euler = 2.718281828459045;
  double *s1 = ws_slot(w, 0), *s2 = ws_slot(w, 1), *p = ws_slot(w, 2), *q = ws_slot(w, 3);
  double *t1 = ws_slot(w, 4), *t2 = ws_slot(w, 5);
  for (int i = 0; i < n; i++) {
    v_mul(K, y + (size_t)i * nc, y + (size_t)i * nc, p);
    if (i == 0) v_copy(K, p, s1);
    else v_add(K, s1, p, s1);
  }
  for (int i = 0; i < n; i++) {
    v_smul(K, two_pi, y + (size_t)i * nc, p);
    v_unary(K, OR_G_COS, p, q);
    if (i == 0) v_copy(K, q, s2);
    else v_add(K, s2, q, s2);
  }
  v_smul(K, 1.0 / n, s1, p);   /* s1*(1/n)        */
  v_unary(K, OR_G_SQRT, p, q); /* sqrt            */
  v_smul(K, -0.2, q, p);       /* (-0.2)*sqrt     */
  v_unary(K, OR_G_EXP, p, q);  /* exp             */
  v_smul(K, -20.0, q, t1);     /* t1 = (-20)*exp  */
  v_smul(K, 1.0 / n, s2, p);   /* s2*(1/n)        */
  v_unary(K, OR_G_EXP, p, t2); /* t2 = exp(...)   */
  v_sub(K, t1, t2, p);         /* t1 - t2         */
  v_adds(K, p, 20.0 + euler, out);
}

/* F3 Fletcher-Powell (trigonometric): sum_k (E*_k - sum_j A_kj sin y_j + B_kj cos y_j)^2
 * (SPEC.md:370-387).  params = [A (n*n) | B (n*n) | Estar (n)], row-major. */
static void f_fletcher_powell(const car *K, int n, const double *params, const double *y, double *out,
                              ws_t *w) {
  const int nc = K->ncomp;
  const double *A = params, *B = params + (size_t)n * n, *Es = params + 2 * (size_t)n * n;
  double *E = ws_slot(w, 0), *p = ws_slot(w, 1), *q = ws_slot(w, 2), *pq = ws_slot(w, 3);
  double *r = ws_slot(w, 4), *rr = ws_slot(w, 5), *f = ws_slot(w, 6);
  double *S = ws_slot(w, 7), *Cc = ws_slot(w, 7 + n); /* sin y_j, cos y_j */
  for (int j = 0; j < n; j++) {
    v_unary(K, OR_G_SIN, y + (size_t)j * nc, S + (size_t)j * nc);
    v_unary(K, OR_G_COS, y + (size_t)j * nc, Cc + (size_t)j * nc);
  }
  for (int k = 0; k < n; k++) {
    for (int j = 0; j < n; j++) {
      v_smul(K, A[(size_t)k * n + j], S + (size_t)j * nc, p);
      v_smul(K, B[(size_t)k * n + j], Cc + (size_t)j * nc, q);
      v_add(K, p, q, pq); /* A_kj sin y_j + B_kj cos y_j */
      if (j == 0) v_copy(K, pq, E);
      else v_add(K, E, pq, E);
    }
    v_ssub(K, Es[k], E, r); /* r_k = E*_k - E_k */
    v_mul(K, r, r, rr);
    if (k == 0) v_copy(K, rr, f);
    else v_add(K, f, rr, f);
  }
  v_copy(K, f, out);
}

/* F4 prodsum: sum_{i<n-1} y_i*y_{i+1}; M = n-1 hDual products, A = n-2 sums */
static void f_prodsum(const car *K, int n, const double *y, double *out, ws_t *w) {
  const int nc = K->ncomp;
  double *p = ws_slot(w, 0), *s = ws_slot(w, 1);
  for (int i = 0; i < n - 1; i++) {
    v_mul(K, y + (size_t)i * nc, y + (size_t)(i + 1) * nc, p);
    if (i == 0) v_copy(K, p, s);
    else v_add(K, s, p, s);
  }
  v_copy(K, s, out);
}

static int ws_slots_needed(int func, int n) { return func == OR_FLETCHER_POWELL ? 7 + 2 * n : 8; }

static int check_func(int func, int n, const double *params) {
  if (n < 1) return OR_ERR_ARG;
  switch (func) {
  case OR_ROSENBROCK:
  case OR_PRODSUM: return n >= 2 ? OR_OK : OR_ERR_FUNC;
  case OR_ACKLEY: return OR_OK;
  case OR_FLETCHER_POWELL: return params ? OR_OK : OR_ERR_FUNC;
  default: return OR_ERR_FUNC;
  }
}

static void eval_f(int func, const car *K, int n, const double *params, const double *y, double *out, ws_t *w) {
  g_evals++;
  switch (func) {
  case OR_ROSENBROCK: f_rosenbrock(K, n, y, out, w); break;
  case OR_ACKLEY: f_ackley(K, n, y, out, w); break;
  case OR_FLETCHER_POWELL: f_fletcher_powell(K, n, params, y, out, w); break;
  case OR_PRODSUM: f_prodsum(K, n, y, out, w); break;
  }
}

static ws_t ws_make(const car *K, int func, int n) {
  ws_t w;
  w.K = K;
  w.nslots = ws_slots_needed(func, n);
  w.buf = (double *)calloc((size_t)w.nslots * K->ncomp, sizeof(double));
  return w;
}

/* ------------------------------------------------------------------ public primitives */
int or_hd_binary(int op, int C, const double *u, const double *v, double c, double *r) {
  if (C < 1 || C > OR_CMAX) return OR_ERR_CHUNK;
  car K = car_hdual(C);
  switch (op) {
  case OR_OP_ADD: v_add(&K, u, v, r); break;
  case OR_OP_SUB: v_sub(&K, u, v, r); break;
  case OR_OP_MUL: v_mul(&K, u, v, r); break;
  case OR_OP_DIV: v_div(&K, u, v, r); break;
  case OR_OP_SADD: v_sadd(&K, c, u, r); break;
  case OR_OP_ADDS: v_adds(&K, u, c, r); break;
  case OR_OP_SSUB: v_ssub(&K, c, u, r); break;
  case OR_OP_SUBS: v_subs(&K, u, c, r); break;
  case OR_OP_SMUL: v_smul(&K, c, u, r); break;
  case OR_OP_DIVS: { /* u / c: every slot divided by c */
    for (int s = 0; s < K.ncomp; s++) r[s] = u[s] / c;
    break;
  }
  case OR_OP_SDIV: { /* c / u := lift_constant(c) / u */
    double *cc = (double *)calloc(K.ncomp, sizeof(double));
    cc[0] = c;
    v_div(&K, cc, u, r);
    free(cc);
    break;
  }
  case OR_OP_NEG: v_neg(&K, u, r); break;
  default: return OR_ERR_ARG;
  }
  return OR_OK;
}

int or_hd_unary(int g, int C, const double *u, double *r) {
  if (C < 1 || C > OR_CMAX) return OR_ERR_CHUNK;
  if (g < OR_G_SIN || g > OR_G_ABS) return OR_ERR_ARG;
  car K = car_hdual(C);
  v_unary(&K, g, u, r);
  return OR_OK;
}

int or_hd_compare(int cmp, const double *u, const double *v) {
  switch (cmp) {
  case OR_CMP_LT: return u[0] < v[0];
  case OR_CMP_GT: return u[0] > v[0];
  case OR_CMP_LE: return u[0] <= v[0];
  case OR_CMP_GE: return u[0] >= v[0];
  case OR_CMP_EQ: return u[0] == v[0];
  }
  return -1;
}

/* Alg 1 INITIALIZE: y[k] = <a_k, [k==i], [k==j], 0> */
void or_initialize(int n, const double *a, int i, int j, double *y) {
  for (int k = 0; k < n; k++) {
    double *yk = y + (size_t)k * 4;
    yk[0] = a[k];
    for (int l = 1; l <= 3; l++) yk[l] = 0.0;
    if (k == i) yk[1] = 1.0;
    if (k == j) yk[2] = 1.0;
  }
}

/* Alg 4 CHUNK-INIT */
void or_chunk_init(int n, const double *a, int i, int cstart, int C, double *y) {
  const int nc = 2 * C + 2;
  for (int k = 0; k < n; k++) {
    double *yk = y + (size_t)k * nc;
    yk[0] = a[k];
    yk[1] = 0.0;
    if (k == i) yk[1] = 1.0;
    for (int l = 2; l <= C + 1; l++) yk[l] = 0.0;
    if (k >= cstart && k < cstart + C) yk[k - cstart + 2] = 1.0;
    for (int l = C + 2; l <= 2 * C + 1; l++) yk[l] = 0.0;
  }
}

int or_eval_hdual(int func, int n, const double *params, int C, const double *y, double *t) {
  int st = check_func(func, n, params);
  if (st) return st;
  if (C < 1 || C > OR_CMAX) return OR_ERR_CHUNK;
  car K = car_hdual(C);
  ws_t w = ws_make(&K, func, n);
  eval_f(func, &K, n, params, y, t, &w);
  free(w.buf);
  return OR_OK;
}

int or_eval_scalar(int func, int n, const double *params, const double *x, double *f) {
  int st = check_func(func, n, params);
  if (st) return st;
  car K = car_scalar();
  ws_t w = ws_make(&K, func, n);
  eval_f(func, &K, n, params, x, f, &w);
  free(w.buf);
  return OR_OK;
}

static int check_chunk(int n, int C) {
  if (C < 1 || C > n || n % C != 0 || C > OR_CMAX) return OR_ERR_CHUNK;
  return OR_OK;
}

/* ------------------------------------------------------------------ Hessian algorithms */
/* Alg 2 HESSIAN: n^2 evaluations of f<hDual> (4 components) */
int or_hessian(int func, int n, const double *params, const double *a, double *H) {
  int st = check_func(func, n, params);
  if (st) return st;
  car K = car_hdual(1);
  ws_t w = ws_make(&K, func, n);
  double *y = (double *)malloc(sizeof(double) * 4 * n), t[4];
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      or_initialize(n, a, i, j, y);
      eval_f(func, &K, n, params, y, t, &w);
      H[(size_t)i * n + j] = t[3];
    }
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Alg 3 SYM-HESSIAN: n(n+1)/2 evaluations + mirror */
int or_sym_hessian(int func, int n, const double *params, const double *a, double *H) {
  int st = check_func(func, n, params);
  if (st) return st;
  car K = car_hdual(1);
  ws_t w = ws_make(&K, func, n);
  double *y = (double *)malloc(sizeof(double) * 4 * n), t[4];
  for (int i = 0; i < n; i++)
    for (int j = i; j < n; j++) {
      or_initialize(n, a, i, j, y);
      eval_f(func, &K, n, params, y, t, &w);
      H[(size_t)i * n + j] = t[3];
      H[(size_t)j * n + i] = H[(size_t)i * n + j];
    }
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Alg 5 CHUNK-HESS: n^2/C evaluations of f<hDual<C>>.
 * grad[i] = slot 1 (df/dx_i) of the last evaluation of row i. */
int or_chunk_hess(int func, int n, int C, const double *params, const double *a, double *H, double *grad) {
  int st = check_func(func, n, params);
  if (st) return st;
  if ((st = check_chunk(n, C))) return st;
  car K = car_hdual(C);
  ws_t w = ws_make(&K, func, n);
  const int nc = 2 * C + 2, nchunk = n / C;
  double *y = (double *)malloc(sizeof(double) * nc * n), t[2 * OR_CMAX + 2];
  for (int i = 0; i < n; i++)
    for (int j = 0; j < nchunk; j++) {
      int cstart = j * C;
      or_chunk_init(n, a, i, cstart, C, y);
      eval_f(func, &K, n, params, y, t, &w);
      for (int l = 0; l < C; l++) H[(size_t)i * n + cstart + l] = t[C + 2 + l];
      if (grad) grad[i] = t[1];
    }
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Alg 6 SCHUNK-HESS: chunks j >= i/C only, n(n/C+1)/2 evaluations;
 * mirror loop read as exclusive of endindex (reading G9). */
int or_schunk_hess(int func, int n, int C, const double *params, const double *a, double *H, double *grad) {
  int st = check_func(func, n, params);
  if (st) return st;
  if ((st = check_chunk(n, C))) return st;
  car K = car_hdual(C);
  ws_t w = ws_make(&K, func, n);
  const int nc = 2 * C + 2, nchunk = n / C;
  double *y = (double *)malloc(sizeof(double) * nc * n), t[2 * OR_CMAX + 2];
  for (int i = 0; i < n; i++) {
    int startchunk = i / C;
    for (int j = startchunk; j < nchunk; j++) {
      int cstart = j * C;
      or_chunk_init(n, a, i, cstart, C, y);
      eval_f(func, &K, n, params, y, t, &w);
      for (int l = 0; l < C; l++) H[(size_t)i * n + cstart + l] = t[C + 2 + l];
      if (grad) grad[i] = t[1];
    }
  }
  for (int i = C; i < n; i++) {
    int endindex = (i / C) * C;
    for (int j = 0; j < endindex; j++) H[(size_t)i * n + j] = H[(size_t)j * n + i];
  }
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Alg 7 CHESS-VEC: out[i] = sum_j H[i][j]*in[j], chunk by chunk,
 * res accumulated left to right from 0.  sabs[i] = sum_j |H_ij||in_j| (the error-metric
 * denominator of DESIGN.md; not part of the method, not counted). */
int or_chess_vec(int func, int n, int C, const double *params, const double *a, const double *in,
                 double *out, double *sabs) {
  int st = check_func(func, n, params);
  if (st) return st;
  if ((st = check_chunk(n, C))) return st;
  car K = car_hdual(C);
  ws_t w = ws_make(&K, func, n);
  const int nc = 2 * C + 2, nchunk = n / C;
  double *y = (double *)malloc(sizeof(double) * nc * n), t[2 * OR_CMAX + 2];
  for (int i = 0; i < n; i++) {
    double res = 0.0, s = 0.0;
    for (int j = 0; j < nchunk; j++) {
      int cstart = j * C;
      or_chunk_init(n, a, i, cstart, C, y); /* G6: chunk index j -> cstart = j*C */
      eval_f(func, &K, n, params, y, t, &w);
      for (int l = 0; l < C; l++) {
        res = ADD(res, MUL(t[C + 2 + l], in[cstart + l]));
        s = s + fabs(t[C + 2 + l]) * fabs(in[cstart + l]);
      }
    }
    out[i] = res;
    if (sabs) sabs[i] = s;
  }
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Alg 8 SC-HESS-VEC with the DESIGN.md reading G8: the inner loop
 * visits every second-order slot C+2..2C+1 and out <- res. */
int or_sc_hess_vec(int func, int n, int C, const double *params, const double *a, const double *in,
                   double *out) {
  int st = check_func(func, n, params);
  if (st) return st;
  if ((st = check_chunk(n, C))) return st;
  car K = car_hdual(C);
  ws_t w = ws_make(&K, func, n);
  const int nc = 2 * C + 2, nchunk = n / C;
  double *y = (double *)malloc(sizeof(double) * nc * n), t[2 * OR_CMAX + 2];
  double *res = (double *)calloc(n, sizeof(double));
  for (int i = 0; i < n; i++) {
    int scn = i / C;
    for (int cn = scn; cn < nchunk; cn++) {
      int cstart = cn * C, s = cstart;
      or_chunk_init(n, a, i, cstart, C, y);
      eval_f(func, &K, n, params, y, t, &w);
      for (int l = C + 2; l <= 2 * C + 1; l++) {
        res[i] = ADD(res[i], MUL(t[l], in[s]));
        if (cn > scn) res[s] = ADD(res[s], MUL(t[l], in[i]));
        s = s + 1;
      }
    }
  }
  memcpy(out, res, sizeof(double) * n);
  free(res);
  free(y);
  free(w.buf);
  return OR_OK;
}

/* Full (n+1)(n+2)/2 scheme (Szirmay-Kalos): y_k = <a_k, e_k, 0>,
 * one evaluation gives f, grad and the upper triangle; the lower triangle is mirrored. */
int or_full_scheme_hessian(int func, int n, const double *params, const double *a, double *H, double *grad) {
  int st = check_func(func, n, params);
  if (st) return st;
  car K = car_full(n);
  ws_t w = ws_make(&K, func, n);
  const int nc = K.ncomp;
  double *y = (double *)calloc((size_t)nc * n, sizeof(double));
  double *t = (double *)malloc(sizeof(double) * nc);
  for (int k = 0; k < n; k++) {
    y[(size_t)k * nc] = a[k];
    y[(size_t)k * nc + 1 + k] = 1.0;
  }
  eval_f(func, &K, n, params, y, t, &w);
  for (int i = 0; i < n; i++) {
    if (grad) grad[i] = t[1 + i];
    for (int j = i; j < n; j++) {
      double h = t[1 + n + tri(n, i, j)];
      H[(size_t)i * n + j] = h;
      H[(size_t)j * n + i] = h;
    }
  }
  free(t);
  free(y);
  free(w.buf);
  return OR_OK;
}

/* ------------------------------------------------------------------ batches */
typedef struct {
  int kind; /* 0 hvp, 1 hessian, 2 sc-hvp */
  int func, n, C;
  int64_t e0, e1;
  const double *points, *vecs, *params;
  double *out, *sabs;
  int status;
} job_t;

static void *job_run(void *arg) {
  job_t *J = (job_t *)arg;
  const int n = J->n;
  for (int64_t e = J->e0; e < J->e1; e++) {
    const double *a = J->points + (size_t)e * n;
    int st;
    if (J->kind == 0)
      st = or_chess_vec(J->func, n, J->C, J->params, a, J->vecs + (size_t)e * n, J->out + (size_t)e * n,
                        J->sabs ? J->sabs + (size_t)e * n : NULL);
    else if (J->kind == 2)
      st = or_sc_hess_vec(J->func, n, J->C, J->params, a, J->vecs + (size_t)e * n, J->out + (size_t)e * n);
    else
      st = or_chunk_hess(J->func, n, J->C, J->params, a, J->out + (size_t)e * n * n, NULL);
    if (st) { J->status = st; return NULL; }
  }
  J->status = OR_OK;
  return NULL;
}

static int run_batch(int kind, int func, int n, int C, int64_t m, const double *points, const double *vecs,
                     double *out, double *sabs, const double *params, int nthreads) {
  int st = check_func(func, n, params);
  if (st) return st;
  if ((st = check_chunk(n, C))) return st;
  if (m < 0) return OR_ERR_ARG;
  if (m == 0) return OR_OK;
  if (!points || !out || (kind != 1 && !vecs)) return OR_ERR_ARG;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > m) nthreads = (int)m;
  job_t *jobs = (job_t *)calloc(nthreads, sizeof(job_t));
  pthread_t *th = (pthread_t *)calloc(nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; t++) {
    job_t *J = &jobs[t];
    J->kind = kind; J->func = func; J->n = n; J->C = C;
    J->e0 = m * t / nthreads; J->e1 = m * (t + 1) / nthreads;
    J->points = points; J->vecs = vecs; J->params = params; J->out = out; J->sabs = sabs;
  }
  for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, job_run, &jobs[t]);
  job_run(&jobs[0]);
  st = OR_OK;
  for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
  for (int t = 0; t < nthreads; t++)
    if (jobs[t].status) st = jobs[t].status;
  free(jobs);
  free(th);
  return st;
}

int or_hvp_batch(int func, int n, int C, int64_t m, const double *points, const double *vecs, double *out,
                 double *sabs, const double *params, int nthreads) {
  return run_batch(0, func, n, C, m, points, vecs, out, sabs, params, nthreads);
}

int or_sc_hvp_batch(int func, int n, int C, int64_t m, const double *points, const double *vecs, double *out,
                    const double *params, int nthreads) {
  return run_batch(2, func, n, C, m, points, vecs, out, NULL, params, nthreads);
}

int or_hessian_batch(int func, int n, int C, int64_t m, const double *points, double *hess,
                     const double *params, int nthreads) {
  return run_batch(1, func, n, C, m, points, NULL, hess, NULL, params, nthreads);
}

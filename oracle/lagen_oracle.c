/*
 * lagen_oracle.c — CPU restatement of the reference executor for the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker (or the reported CPU baseline) — never as the product
 * path.  The product (paper_1906_08613_b200) has no CPU fallback.
 *
 * What it restates, function by function (paths relative to /root/reference):
 *   ora_gemm_update   pkg/src/lagen/kernels.py:16-34   gemm_update
 *   ora_trsm_left     pkg/src/lagen/kernels.py:47-60   trsm_left (lower=True)
 *   ora_chol_leaf     pkg/src/lagen/kernels.py:79-97   chol_leaf
 *   ora_sylv_solve    pkg/src/lagen/kernels.py:100-110 sylv_solve
 *   ora_lyap_solve    pkg/src/lagen/kernels.py:113-130 lyap_solve
 *   mirror / copy-in  pkg/src/lagen/kernels.py:133-149 mirror_lower, copy_region
 *   oracle_execute    pkg/src/lagen/verify.py:221-303  interpret_algorithm
 *   oracle_chol_textbook pkg/src/lagen/verify.py:109-120 _chol_upper_textbook
 *   oracle_residual   pkg/src/lagen/verify.py:186-195  residual
 * plus oracle_generate, the CPU twin of the seeded batched generator
 * (BASELINE.json configs; spec in DESIGN.md §Generator).
 *
 * Numerics: plain sequential dot products (numpy/BLAS order is unpinned in
 * the reference; its tests pin to tolerances).  Views are
 * (pointer, row stride, col stride); symmetric diagonal blocks of a symmetric
 * unknown are gathered as triu(m) + triu(m,1)^T exactly as verify.py:254-261.
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by the reference's own interpret_algorithm
 * (tests/golden/make_golden.py) and against its known-answer tests.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/lagen_b200.h"

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  double* p;
  int rs, cs;   /* element (i, j) = p[i*rs + j*cs] */
  int rows, cols;
} ora_view;

static inline double V(const ora_view* v, int i, int j) { return v->p[(long)i * v->rs + (long)j * v->cs]; }
static inline double* VP(const ora_view* v, int i, int j) { return &v->p[(long)i * v->rs + (long)j * v->cs]; }

/* kernels.py:16-34 */
static void ora_gemm_update(ora_view* out, const ora_view* a, const ora_view* b, int sign, int upper) {
  int m = a->rows, p = a->cols, q = b->cols;
  if (m == 0 || p == 0 || q == 0) return;
  if (!upper) {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < q; ++j) {
        double acc = 0.0;
        for (int l = 0; l < p; ++l) acc += V(a, i, l) * V(b, l, j);
        if (sign > 0) *VP(out, i, j) += acc; else *VP(out, i, j) -= acc;
      }
    return;
  }
  for (int j = 0; j < q; ++j)
    for (int i = 0; i <= j && i < m; ++i) {
      double acc = 0.0;
      for (int l = 0; l < p; ++l) acc += V(a, i, l) * V(b, l, j);
      if (sign > 0) *VP(out, i, j) += acc; else *VP(out, i, j) -= acc;
    }
}

/* kernels.py:47-60, lower=True (the only form synthesised: X^T of an upper factor) */
static void ora_trsm_left(const ora_view* t, ora_view* w) {
  int m = t->rows, q = w->cols;
  for (int i = 0; i < m; ++i) {
    if (i)
      for (int j = 0; j < q; ++j) {
        double acc = 0.0;
        for (int l = 0; l < i; ++l) acc += V(t, i, l) * V(w, l, j);
        *VP(w, i, j) -= acc;
      }
    for (int j = 0; j < q; ++j) *VP(w, i, j) /= V(t, i, i);
  }
}

/* kernels.py:79-97; returns first failing pivot index + 1, or 0.  Unlike the
 * reference (which raises) it keeps going so X can be compared as NaN. */
static int ora_chol_leaf(ora_view* w, int base) {
  int m = w->rows, bad = 0;
  for (int i = 0; i < m; ++i) {
    if (*VP(w, i, i) <= 0.0 && !bad) bad = base + i + 1;
    *VP(w, i, i) = sqrt(*VP(w, i, i));
    for (int j = i + 1; j < m; ++j) *VP(w, i, j) /= *VP(w, i, i);
    for (int r = i + 1; r < m; ++r)
      for (int c = r; c < m; ++c) *VP(w, r, c) -= V(w, i, r) * V(w, i, c);
  }
  return bad;
}

/* kernels.py:100-110 */
static void ora_sylv_solve(const ora_view* l, const ora_view* u, ora_view* w) {
  int m = w->rows, q = w->cols;
  for (int j = 0; j < q; ++j) {
    if (j)
      for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int k = 0; k < j; ++k) acc += V(w, i, k) * V(u, k, j);
        *VP(w, i, j) -= acc;
      }
    for (int i = 0; i < m; ++i) {
      if (i) {
        double acc = 0.0;
        for (int k = 0; k < i; ++k) acc += V(l, i, k) * V(w, k, j);
        *VP(w, i, j) -= acc;
      }
      *VP(w, i, j) /= V(l, i, i) + V(u, j, j);
    }
  }
}

/* kernels.py:113-130 */
static void ora_lyap_solve(const ora_view* l, ora_view* w) {
  int m = w->rows;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i <= j; ++i) {
      double acc = V(w, i, j);
      if (i) {
        double d = 0.0;
        for (int k = 0; k < i; ++k) d += V(l, i, k) * V(w, k, j);
        acc -= d;
      }
      if (j) {
        double d = 0.0;
        for (int k = 0; k < j; ++k) d += V(w, i, k) * V(l, j, k);
        acc -= d;
      }
      acc /= V(l, i, i) + V(l, j, j);
      *VP(w, i, j) = acc;
      *VP(w, j, i) = acc;
    }
}

static int eq_ncoef(int eq) { return eq == LAGEN_CHOLESKY ? 0 : (eq == LAGEN_LYAPUNOV ? 1 : 2); }
static int eq_ninputs(int eq) { return eq + 1; }

/* verify.py:221-303 for one problem.  mats[0] = X work storage, mats[1..] = coefficients. */
static int ora_execute_one(int eq, const lagen_stmt* stmts, int nstmts, int n, int b,
                           double* const* mats, double* gbuf0, double* gbuf1) {
  int sym_target = (eq != LAGEN_SYLVESTER);       /* rhs A/S symmetric */
  int x_sym = (eq == LAGEN_LYAPUNOV);             /* unknown symmetric */
  int info = 0;
  for (int k = 0; k < n / b; ++k) {
    int st[3] = {0, k * b, (k + 1) * b};
    int ex[3] = {k * b, b, n - (k + 1) * b};
    for (int s = 0; s < nstmts; ++s) {
      const lagen_stmt* S = &stmts[s];
      ora_view out = {mats[0] + (long)st[S->out.r] * n + st[S->out.c], n, 1, ex[S->out.r], ex[S->out.c]};
      if (out.rows == 0 || out.cols == 0) continue;
      ora_view in[2];
      double* gb[2] = {gbuf0, gbuf1};
      for (int t = 0; t < 2; ++t) {
        const lagen_view* v = &S->in[t];
        if (v->op < 0) continue;
        double* base = mats[v->op] + (long)st[v->r] * n + st[v->c];
        int r = ex[v->r], c = ex[v->c];
        if (v->op == 0 && x_sym && v->r == v->c && r > 1) {
          /* gather: triu(m) + triu(m,1).T into a private copy (verify.py:254-261) */
          for (int i = 0; i < r; ++i)
            for (int j = 0; j < r; ++j)
              gb[t][i * r + j] = (i <= j) ? base[(long)i * n + j] : base[(long)j * n + i];
          base = gb[t];
          in[t].p = base; in[t].rs = r; in[t].cs = 1;
          if (v->trans) { in[t].rs = 1; in[t].cs = r; }
          in[t].rows = r; in[t].cols = r;
        } else {
          in[t].p = base;
          if (v->trans) { in[t].rs = 1; in[t].cs = n; in[t].rows = c; in[t].cols = r; }
          else { in[t].rs = n; in[t].cs = 1; in[t].rows = r; in[t].cols = c; }
        }
      }
      switch (S->kind) {
        case LAGEN_GEMM_UPDATE:
          ora_gemm_update(&out, &in[0], &in[1], S->sign, sym_target && S->out.r == S->out.c);
          break;
        case LAGEN_CHOL: {
          int bad = ora_chol_leaf(&out, st[S->out.r]);
          if (bad && !info) info = bad;
          break;
        }
        case LAGEN_TRSM_LEFT_TRANSPOSED:
          ora_trsm_left(&in[0], &out);
          break;
        case LAGEN_SYLV:
          ora_sylv_solve(&in[0], &in[1], &out);
          break;
        case LAGEN_LYAP:
          ora_lyap_solve(&in[0], &out);
          break;
        default:
          return -1000;
      }
    }
  }
  if (x_sym) /* mirror_lower, kernels.py:133-138 */
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < i; ++j) mats[0][(long)i * n + j] = mats[0][(long)j * n + i];
  if (!info)
    for (long e = 0; e < (long)n * n; ++e)
      if (!isfinite(mats[0][e])) { info = -1; break; }
  return info;
}

int oracle_execute(int eq, const lagen_stmt* stmts, int nstmts, int n, int b, long long batch,
                   const double* const* inputs, double* X, int* info, int nthreads) {
  if (eq < 0 || eq > 2 || n < 1 || b < 1 || n % b || batch < 0 || !X || !inputs) return LAGEN_EINVAL;
  for (int s = 0; s < nstmts; ++s)
    if (stmts[s].kind < 0 || stmts[s].kind > 4) return LAGEN_EVARIANT;
  int ncoef = eq_ncoef(eq);
  int rhs = eq_ninputs(eq) - 1;       /* rhs source is the last input */
  int status = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    double* g0 = (double*)malloc(sizeof(double) * n * n);
    double* g1 = (double*)malloc(sizeof(double) * n * n);
#pragma omp for schedule(static)
    for (long long p = 0; p < batch; ++p) {
      double* x = X + p * (long long)n * n;
      const double* src = inputs[rhs] + p * (long long)n * n;
      /* copy_region restricted to the unknown's structure (verify.py:236-241) */
      if (eq == LAGEN_CHOLESKY) {
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) x[(long)i * n + j] = (j >= i) ? src[(long)i * n + j] : 0.0;
      } else {
        memcpy(x, src, sizeof(double) * n * n);
      }
      double* mats[3] = {x, NULL, NULL};
      for (int c = 0; c < ncoef; ++c) mats[1 + c] = (double*)(inputs[c] + p * (long long)n * n);
      int r = ora_execute_one(eq, stmts, nstmts, n, b, mats, g0, g1);
      if (r == -1000) status = LAGEN_EVARIANT;
      if (info) info[p] = r;
    }
    free(g0);
    free(g1);
  }
  return status;
}

/* verify.py:109-120 (bordered unblocked); info as above */
int oracle_chol_textbook(int n, long long batch, const double* A, double* X, int* info) {
  for (long long p = 0; p < batch; ++p) {
    const double* a = A + p * (long long)n * n;
    double* x = X + p * (long long)n * n;
    int bad = 0;
    memset(x, 0, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int l = 0; l < i; ++l) s += x[l * n + i] * x[l * n + i];
      s = a[i * n + i] - s;
      if (s <= 0.0 && !bad) bad = i + 1;
      x[i * n + i] = sqrt(s);
      for (int j = i + 1; j < n; ++j) {
        double d = 0.0;
        for (int l = 0; l < i; ++l) d += x[l * n + i] * x[l * n + j];
        x[i * n + j] = (a[i * n + j] - d) / x[i * n + i];
      }
    }
    if (info) info[p] = bad;
  }
  return 0;
}

/* verify.py:186-195: ||lhs - rhs||_F / max(1, ||rhs||_F) per problem */
int oracle_residual(int eq, int n, long long batch, const double* const* inputs, const double* X,
                    double* res, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
  for (long long p = 0; p < batch; ++p) {
    long long off = p * (long long)n * n;
    const double* x = X + off;
    double num = 0.0, den = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double lhs = 0.0, rhs;
        if (eq == LAGEN_CHOLESKY) {
          for (int l = 0; l < n; ++l) lhs += x[l * n + i] * x[l * n + j];
          rhs = inputs[0][off + i * n + j];
        } else if (eq == LAGEN_LYAPUNOV) {
          const double* L = inputs[0] + off;
          double t1 = 0.0, t2 = 0.0;
          for (int l = 0; l < n; ++l) t1 += L[i * n + l] * x[l * n + j];
          for (int l = 0; l < n; ++l) t2 += x[i * n + l] * L[j * n + l];
          lhs = t1 + t2;
          rhs = inputs[1][off + i * n + j];
        } else {
          const double* L = inputs[0] + off;
          const double* U = inputs[1] + off;
          double t1 = 0.0, t2 = 0.0;
          for (int l = 0; l < n; ++l) t1 += L[i * n + l] * x[l * n + j];
          for (int l = 0; l < n; ++l) t2 += x[i * n + l] * U[l * n + j];
          lhs = t1 + t2;
          rhs = inputs[2][off + i * n + j];
        }
        num += (lhs - rhs) * (lhs - rhs);
        den += rhs * rhs;
      }
    den = sqrt(den);
    res[p] = sqrt(num) / (den < 1.0 ? 1.0 : den);
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Seeded batched generator, CPU twin of the device generator.
 * Counter-based: value(seed, eq, n, problem, operand, element, draw).
 * ------------------------------------------------------------------------- */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t gen_key(uint64_t seed, int eq, int n) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + ((uint64_t)eq << 40) + ((uint64_t)n << 20) + 0x632BE59BD9B4E019ULL);
}
static inline double gen_u01(uint64_t key, uint64_t ctr) {
  uint64_t h = mix64(key + ctr * 0x9E3779B97F4A7C15ULL);
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
static inline uint64_t gen_ctr(long long p, int op, int n, int e, int draw) {
  return (((uint64_t)p * 4u + (uint64_t)op) * (uint64_t)n * (uint64_t)n + (uint64_t)e) * 2u + (uint64_t)draw;
}
static inline double gen_normal(uint64_t key, long long p, int op, int n, int e) {
  double u1 = gen_u01(key, gen_ctr(p, op, n, e, 0));
  double u2 = gen_u01(key, gen_ctr(p, op, n, e, 1));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static void gen_tri(uint64_t key, long long p, int op, int n, int lower, double* m) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int e = i * n + j;
      if (i == j) m[e] = 1.0 + gen_u01(key, gen_ctr(p, op, n, e, 0));
      else if ((lower && j < i) || (!lower && j > i)) m[e] = gen_normal(key, p, op, n, e) / (double)n;
      else m[e] = 0.0;
    }
}

int oracle_generate(int eq, int n, unsigned long long seed, long long first, long long batch,
                    double* const* outputs, int nthreads) {
  uint64_t key = gen_key(seed, eq, n);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    double* tmp = (double*)malloc(sizeof(double) * n * n);
#pragma omp for schedule(static)
    for (long long q = 0; q < batch; ++q) {
      long long p = first + q;
      long long off = q * (long long)n * n;
      if (eq == LAGEN_CHOLESKY) {
        for (int e = 0; e < n * n; ++e) tmp[e] = gen_normal(key, p, 0, n, e);
        double* a = outputs[0] + off;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc = fma(tmp[k * n + i], tmp[k * n + j], acc);
            a[i * n + j] = acc + (i == j ? (double)n : 0.0);
          }
      } else if (eq == LAGEN_LYAPUNOV) {
        gen_tri(key, p, 0, n, 1, outputs[0] + off);
        for (int e = 0; e < n * n; ++e) tmp[e] = gen_normal(key, p, 1, n, e);
        double* s = outputs[1] + off;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) s[i * n + j] = 0.5 * (tmp[i * n + j] + tmp[j * n + i]);
      } else {
        gen_tri(key, p, 0, n, 1, outputs[0] + off);
        gen_tri(key, p, 1, n, 0, outputs[1] + off);
        double* c = outputs[2] + off;
        for (int e = 0; e < n * n; ++e) c[e] = gen_normal(key, p, 2, n, e);
      }
    }
    free(tmp);
  }
  return 0;
}

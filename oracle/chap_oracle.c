/* chap_oracle.c — TEST INFRASTRUCTURE ONLY (see chap_oracle.h).
 *
 * Plain fp64 C, built with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so its
 * arithmetic is the IEEE operations written here, in the order written here. OpenMP is used
 * only over independent variables j (each iteration of those loops writes its own outputs).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * against the paper's worked cases, closed forms, full-domain brute force and an independent
 * exact-rational implementation of Algorithm 1 — except orc_tabu_run's selection/bump rules,
 * which the paper does not state (R6, R12, R13, R14): those are pinned only by the hand-worked
 * trajectory in tests/golden/trajectory_2var.json and by invariants ("parity unpinned by the
 * paper" for the rule choices themselves).
 */
#include "chap_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

struct orc_problem {
  int32_t n, m_orig;
  int32_t m_norm;           /* normalised rows + 1 cutoff row (last)                         */
  /* normalised rows in CSR (the cutoff row is stored separately: dense over c_j != 0) */
  int64_t* rp; int32_t* ci; double* va; double* b;
  int32_t* orig; int8_t* side;
  /* the same matrix by column (a plain transpose), cutoff entries excluded */
  int64_t* cp; int32_t* ri; double* cv;
  double* lb; double* ub; uint8_t* vclass; double* c;
  int64_t nnz_norm, nnz_cut;
  double auto_delta;
};

static int is_integral(double v) { return isfinite(v) && v == floor(v); }

int orc_problem_create(int32_t n, int32_t m, int64_t nnz, const int64_t* row_ptr,
                       const int32_t* col_idx, const double* val, const double* lhs,
                       const double* rhs, const double* lb, const double* ub,
                       const uint8_t* is_int, const double* c, orc_problem** out) {
  *out = NULL;
  if (n < 0 || m < 0 || nnz < 0) return ORC_ERR_INVALID_ARG;
  if (row_ptr[0] != 0 || row_ptr[m] != nnz) return ORC_ERR_INVALID_ARG;
  for (int32_t i = 0; i < m; i++) {
    if (row_ptr[i + 1] < row_ptr[i]) return ORC_ERR_INVALID_ARG;
    if (isnan(lhs[i]) || isnan(rhs[i]) || lhs[i] > rhs[i] || lhs[i] == INFINITY || rhs[i] == -INFINITY)
      return ORC_ERR_INVALID_ARG;
  }
  for (int64_t e = 0; e < nnz; e++) {
    if (col_idx[e] < 0 || col_idx[e] >= n || !isfinite(val[e])) return ORC_ERR_INVALID_ARG;
  }
  /* duplicate (i, j): mark columns seen in the current row */
  int32_t* seen = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  for (int32_t j = 0; j < n; j++) seen[j] = -1;
  for (int32_t i = 0; i < m; i++)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
      if (seen[col_idx[e]] == i) { free(seen); return ORC_ERR_INVALID_ARG; }
      seen[col_idx[e]] = i;
    }
  free(seen);

  orc_problem* P = (orc_problem*)calloc(1, sizeof(orc_problem));
  P->n = n; P->m_orig = m;
  P->lb = (double*)malloc(sizeof(double) * (n + 1));
  P->ub = (double*)malloc(sizeof(double) * (n + 1));
  P->vclass = (uint8_t*)malloc(n + 1);
  P->c = (double*)malloc(sizeof(double) * (n + 1));
  for (int32_t j = 0; j < n; j++) {
    double l = lb[j], u = ub[j];
    if (isnan(l) || isnan(u) || isnan(c[j]) || !isfinite(c[j]) || l == INFINITY || u == -INFINITY) {
      orc_problem_free(P); return ORC_ERR_INVALID_ARG;
    }
    if (is_int[j]) { l = ceil(l); u = floor(u); }   /* round integer bounds inward */
    if (l > u) { orc_problem_free(P); return ORC_ERR_INFEASIBLE_BOUNDS; }
    P->lb[j] = l; P->ub[j] = u; P->c[j] = c[j];
    if (l == u) P->vclass[j] = 0;
    else if (is_int[j] && l == 0.0 && u == 1.0) P->vclass[j] = 1;
    else if (is_int[j]) P->vclass[j] = 2;
    else P->vclass[j] = 3;
  }
  /* count normalised rows / nonzeros (explicit zeros dropped: Alg.1 iterates a_ij != 0) */
  int32_t mn = 0; int64_t zn = 0;
  for (int32_t i = 0; i < m; i++) {
    int64_t k = 0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) k += (val[e] != 0.0);
    if (k == 0) {
      if (lhs[i] > 0.0 || rhs[i] < 0.0) { orc_problem_free(P); return ORC_ERR_INFEASIBLE_BOUNDS; }
      continue; /* empty row dropped */
    }
    if (isfinite(rhs[i])) { mn++; zn += k; }
    if (isfinite(lhs[i])) { mn++; zn += k; }
  }
  P->m_norm = mn + 1;
  P->nnz_norm = zn;
  P->rp = (int64_t*)malloc(sizeof(int64_t) * (mn + 2));
  P->ci = (int32_t*)malloc(sizeof(int32_t) * (zn + 1));
  P->va = (double*)malloc(sizeof(double) * (zn + 1));
  P->b = (double*)malloc(sizeof(double) * (mn + 1));
  P->orig = (int32_t*)malloc(sizeof(int32_t) * (mn + 1));
  P->side = (int8_t*)malloc(mn + 1);
  int32_t r = 0; int64_t z = 0;
  P->rp[0] = 0;
  for (int32_t i = 0; i < m; i++) {
    int64_t k = 0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) k += (val[e] != 0.0);
    if (k == 0) continue;
    for (int s = 0; s < 2; s++) {
      double sg = (s == 0) ? 1.0 : -1.0;
      double bb = (s == 0) ? rhs[i] : -lhs[i];
      if (!isfinite(bb)) continue;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
        if (val[e] == 0.0) continue;
        P->ci[z] = col_idx[e]; P->va[z] = sg * val[e]; z++;
      }
      P->b[r] = bb; P->orig[r] = i; P->side[r] = (int8_t)(s == 0 ? 1 : -1);
      r++; P->rp[r] = z;
    }
  }
  /* cutoff row (last): c.x <= z* - delta; stored via c directly */
  int64_t nc = 0; int all_int = 1;
  for (int32_t j = 0; j < n; j++)
    if (c[j] != 0.0) { nc++; if (!is_integral(c[j]) || P->vclass[j] == 3) all_int = 0; }
  P->nnz_cut = nc;
  P->auto_delta = all_int ? 1.0 : NAN;
  /* transpose of the normalised rows (cutoff excluded) */
  P->cp = (int64_t*)calloc(n + 1, sizeof(int64_t));
  P->ri = (int32_t*)malloc(sizeof(int32_t) * (zn + 1));
  P->cv = (double*)malloc(sizeof(double) * (zn + 1));
  for (int64_t e = 0; e < zn; e++) P->cp[P->ci[e] + 1]++;
  for (int32_t j = 0; j < n; j++) P->cp[j + 1] += P->cp[j];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  memcpy(fill, P->cp, sizeof(int64_t) * (n + 1));
  for (int32_t i = 0; i < mn; i++)
    for (int64_t e = P->rp[i]; e < P->rp[i + 1]; e++) {
      int32_t j = P->ci[e];
      P->ri[fill[j]] = i; P->cv[fill[j]] = P->va[e]; fill[j]++;
    }
  free(fill);
  *out = P;
  return ORC_OK;
}

void orc_problem_free(orc_problem* P) {
  if (!P) return;
  free(P->rp); free(P->ci); free(P->va); free(P->b); free(P->orig); free(P->side);
  free(P->cp); free(P->ri); free(P->cv); free(P->lb); free(P->ub); free(P->vclass); free(P->c);
  free(P);
}

void orc_problem_sizes(const orc_problem* P, int32_t* m_norm, int64_t* nnz_norm, int64_t* nnz_cut) {
  *m_norm = P->m_norm; *nnz_norm = P->nnz_norm; *nnz_cut = P->nnz_cut;
}

void orc_problem_row_map(const orc_problem* P, int32_t* orig, int8_t* side) {
  for (int32_t i = 0; i < P->m_norm - 1; i++) { orig[i] = P->orig[i]; side[i] = P->side[i]; }
}

void orc_problem_vars(const orc_problem* P, double* lb, double* ub, uint8_t* vclass) {
  for (int32_t j = 0; j < P->n; j++) { lb[j] = P->lb[j]; ub[j] = P->ub[j]; vclass[j] = P->vclass[j]; }
}

double orc_auto_delta(const orc_problem* P) { return P->auto_delta; }

/* PAPER.md:277-285, with ȳ_i - b_i = r_old and y_ij - b_i = r_new; "satisfied" is r <= 0 exactly
 * (R10). The five cases, in the paper's order. */
double orc_penalty(double w, double r_old, double r_new) {
  if (r_old <= 0.0 && r_new > 0.0) return -w;                       /* ȳ<=b and y>b          */
  if (r_old > 0.0 && r_new <= 0.0) return w;                        /* ȳ>b and y<=b          */
  if (r_old > 0.0 && r_new > 0.0 && r_new < r_old) return 0.5 * w;  /* both >b, y<ȳ          */
  if (r_old > 0.0 && r_new > 0.0 && r_new > r_old) return -0.5 * w; /* both >b, y>ȳ          */
  return 0.0;                                                        /* otherwise             */
}

/* PAPER.md:297 and Alg. 1 l.3-4 (:310-311). b_i - sum_{k!=j} a_ik x_k = b_i - (y_i - a_ij x_j)
 * = a_ij x_j - r_i, so t = x_j - r_i / a_ij. */
double orc_breakpoint(double x_j, double r_i, double a_ij, int is_integer) {
  double t = x_j - r_i / a_ij;
  if (is_integer) t = (a_ij > 0.0) ? floor(t) : ceil(t);
  return t;
}

/* activities ȳ_i = sum_k a_ik x̄_k by a plain loop over row i; the cutoff row's
 * activity is c.x̄ and its right-hand side is cutoff_rhs */
static void activities(const orc_problem* P, const double* x, double* y) {
  int32_t mr = P->m_norm - 1;
  for (int32_t i = 0; i < mr; i++) {
    double s = 0.0;
    for (int64_t e = P->rp[i]; e < P->rp[i + 1]; e++) s += P->va[e] * x[P->ci[e]];
    y[i] = s;
  }
  double s = 0.0;
  for (int32_t j = 0; j < P->n; j++)
    if (P->c[j] != 0.0) s += P->c[j] * x[j];
  y[mr] = s;
}

/* r_i = ȳ_i - b_i; the cutoff row's r is -inf while cutoff_rhs = +inf (inactive) */
void orc_residuals(const orc_problem* P, const double* x, double cutoff_rhs, double* r) {
  int32_t mr = P->m_norm - 1;
  activities(P, x, r);
  for (int32_t i = 0; i < mr; i++) r[i] = r[i] - P->b[i];
  r[mr] = (cutoff_rhs < INFINITY) ? r[mr] - cutoff_rhs : -INFINITY;
}

static double objective(const orc_problem* P, const double* x) {
  double z = 0.0;
  for (int32_t j = 0; j < P->n; j++) z += P->c[j] * x[j];
  return z;
}

/* score of moving x_j to v: sum over the rows i of column j (a_ij != 0), plus the
 * active cutoff row, of p(w_i, ȳ_i - b_i, y_ij - b_i) with y_ij = ȳ_i - a_ij x̄_j + a_ij v
 * (rows with a_ij = 0 have y_ij = ȳ_i and contribute 0). */
static double score_of(const orc_problem* P, int32_t j, double v, const double* x, const double* y,
                       const float* w, double cutoff_rhs) {
  double s = 0.0;
  for (int64_t e = P->cp[j]; e < P->cp[j + 1]; e++) {
    int32_t i = P->ri[e];
    double a = P->cv[e];
    double ynew = y[i] - a * x[j] + a * v;
    double wi = w ? (double)w[i] : 1.0;
    s += orc_penalty(wi, y[i] - P->b[i], ynew - P->b[i]);
  }
  if (cutoff_rhs < INFINITY && P->c[j] != 0.0) {
    int32_t i = P->m_norm - 1;
    double a = P->c[j];
    double ynew = y[i] - a * x[j] + a * v;
    double wi = w ? (double)w[i] : 1.0;
    s += orc_penalty(wi, y[i] - cutoff_rhs, ynew - cutoff_rhs);
  }
  return s;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* is (s1, v1) better than (s0, v0) at incumbent xj: higher score, then smaller |v - x_j|,
 * then smaller v (R4) */
static int better(double s1, double v1, double s0, double v0, double xj) {
  if (s1 != s0) return s1 > s0;
  double d1 = fabs(v1 - xj), d0 = fabs(v0 - xj);
  if (d1 != d0) return d1 < d0;
  return v1 < v0;
}

static void best_shift_var(const orc_problem* P, int32_t j, const double* x, const double* y,
                           const float* w, double cutoff_rhs, double* xhat, double* score) {
  int cut_active = cutoff_rhs < INFINITY;
  double xj = x[j], l = P->lb[j], u = P->ub[j];
  double bs = -INFINITY, bv = xj;
  int have = 0;
  uint8_t vc = P->vclass[j];
  if (vc == 0) { *xhat = xj; *score = -INFINITY; return; }
  if (vc == 1) { /* binary: the only move is the flip */
    double v = 1.0 - xj;
    *xhat = v; *score = score_of(P, j, v, x, y, w, cutoff_rhs); return;
  }
  /* candidate set (R5): the finite bounds and the breakpoint of every row of column j (and of
   * the active cutoff row), within [l_j, u_j], minus x̄_j; collected, sorted and made unique so
   * that each distinct value is scored once */
  int64_t e0 = P->cp[j], e1 = P->cp[j + 1];
  double* cand = (double*)malloc(sizeof(double) * (size_t)(e1 - e0 + 3));
  int64_t nc = 0;
  if (isfinite(l)) cand[nc++] = l;
  if (isfinite(u)) cand[nc++] = u;
  int is_integer = (vc == 2);
  for (int64_t e = e0; e <= e1; e++) {
    double a, ri;
    if (e < e1) { a = P->cv[e]; ri = y[P->ri[e]] - P->b[P->ri[e]]; }
    else {      /* the active cutoff row contributes a breakpoint too */
      if (!(cut_active && P->c[j] != 0.0)) break;
      a = P->c[j]; ri = y[P->m_norm - 1] - cutoff_rhs;
    }
    cand[nc++] = orc_breakpoint(xj, ri, a, is_integer);
  }
  qsort(cand, (size_t)nc, sizeof(double), cmp_double);
  for (int64_t q = 0; q < nc; q++) {
    double v = cand[q];
    if (q > 0 && v == cand[q - 1]) continue;
    if (!(v >= l && v <= u) || v == xj) continue;
    double s = score_of(P, j, v, x, y, w, cutoff_rhs);
    if (!have || better(s, v, bs, bv, xj)) { bs = s; bv = v; have = 1; }
  }
  free(cand);
  if (!have) { *xhat = xj; *score = -INFINITY; return; }
  *xhat = bv; *score = bs;
}

int orc_best_shift_range(const orc_problem* P, const double* x, const float* w, double cutoff_rhs,
                         int32_t j0, int32_t j1, double* xhat, double* score, int32_t* best_j,
                         double* best_v, double* best_s, int n_threads) {
  int32_t n = P->n;
  if (j0 < 0 || j1 > n || j0 > j1) return ORC_ERR_INVALID_ARG;
  for (int32_t j = 0; j < n; j++)
    if (!(x[j] >= P->lb[j] && x[j] <= P->ub[j])) return ORC_ERR_INVALID_ARG;
  double* y = (double*)malloc(sizeof(double) * P->m_norm);
  if (!y) return ORC_ERR_OOM;
  activities(P, x, y);
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
  for (int32_t j = j0; j < j1; j++) best_shift_var(P, j, x, y, w, cutoff_rhs, &xhat[j], &score[j]);
  free(y);
  int32_t bj = -1; double bsv = 0.0, bvv = NAN;
  for (int32_t j = j0; j < j1; j++)
    if (score[j] > 0.0 && (bj < 0 || score[j] > bsv)) { bj = j; bsv = score[j]; bvv = xhat[j]; }
  *best_j = bj; *best_v = bj >= 0 ? bvv : NAN; *best_s = bj >= 0 ? bsv : -INFINITY;
  return ORC_OK;
}

int orc_best_shift(const orc_problem* P, const double* x, const float* w, double cutoff_rhs,
                   double* xhat, double* score, int32_t* best_j, double* best_v, double* best_s,
                   int n_threads) {
  return orc_best_shift_range(P, x, w, cutoff_rhs, 0, P->n, xhat, score, best_j, best_v, best_s, n_threads);
}

/* ---------------------------------------------------------------------------------------- */
/* tabu walk                                                                                */
/* ---------------------------------------------------------------------------------------- */

static double cutoff_delta(const orc_problem* P, const orc_params* prm, double z) {
  if (!isnan(prm->cutoff_delta)) return prm->cutoff_delta;
  if (!isnan(P->auto_delta)) return P->auto_delta;
  return 1e-6 * (fabs(z) > 1.0 ? fabs(z) : 1.0);
}

static int64_t count_violated(const orc_problem* P, const double* r, int cut_active) {
  int64_t v = 0;
  for (int32_t i = 0; i < P->m_norm - 1; i++) v += (r[i] > 0.0);
  if (cut_active) v += (r[P->m_norm - 1] > 0.0);
  return v;
}

/* after-step incumbent check; returns the violated count */
static int64_t incumbent_check(const orc_problem* P, const orc_params* prm, orc_walker* S, double* r) {
  orc_residuals(P, S->x, S->cutoff_rhs, r);
  int64_t viol = count_violated(P, r, S->cutoff_rhs < INFINITY);
  if (viol == 0) {
    double z = objective(P, S->x);
    memcpy(S->best_x, S->x, sizeof(double) * P->n);
    S->best_obj = z; S->has_incumbent = 1;
    S->cutoff_rhs = z - cutoff_delta(P, prm, z);
    orc_residuals(P, S->x, S->cutoff_rhs, r);
    viol = count_violated(P, r, 1);
  }
  return viol;
}

int orc_walker_init(const orc_problem* P, const orc_params* prm, const double* x0, orc_walker* S) {
  for (int32_t j = 0; j < P->n; j++) {
    if (!(x0[j] >= P->lb[j] && x0[j] <= P->ub[j])) return ORC_ERR_INVALID_ARG;
    if (P->vclass[j] != 3 && x0[j] != floor(x0[j])) return ORC_ERR_INVALID_ARG;
    S->x[j] = x0[j]; S->tabu_until[j] = 0;
  }
  for (int32_t i = 0; i < P->m_norm; i++) S->w[i] = 1.0f;
  S->k = 0; S->cutoff_rhs = INFINITY; S->best_obj = INFINITY; S->has_incumbent = 0;
  S->force_j = -1;
  double* r = (double*)malloc(sizeof(double) * P->m_norm);
  incumbent_check(P, prm, S, r);
  free(r);
  S->initialised = 1;
  return ORC_OK;
}

/* Aspiration test (R18): would x_j <- v leave every active row (cutoff row included) satisfied?
 * The point after the move and its residuals recomputed from scratch (plain definition). */
static int feasible_after(const orc_problem* P, const orc_walker* S, int32_t j, double v, double* xt, double* r) {
  memcpy(xt, S->x, sizeof(double) * P->n);
  xt[j] = v;
  orc_residuals(P, xt, S->cutoff_rhs, r);
  return count_violated(P, r, S->cutoff_rhs < INFINITY) == 0;
}

/* SplitMix64 (Steele, Lea & Flood, OOPSLA 2014): the state advances by the golden gamma
 * 0x9e3779b97f4a7c15 and the output is the new state through the mix below; g(state) is the first
 * output of a generator seeded with state. */
uint64_t orc_splitmix64(uint64_t state) {
  uint64_t z = state + 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return orc_splitmix64(orc_splitmix64(orc_splitmix64(orc_splitmix64(seed) ^ a) ^ b) ^ c);
}

/* The perturbation of R21 ("perturb"), drawn at stuck iteration k from the
 * residuals r of the current point, step by step:
 *  1. a row: uniform over the active rows with r_i > 0, else over all active rows — the row with
 *     the least pair (H(seed, id, k, i) >> 32, i); independent uniform draws make every eligible
 *     row equally likely to hold the least one;
 *  2. an entry of that normalised row (input order; the cutoff row: increasing j over c_j != 0):
 *     number H(seed, id, k, 2^62) mod (its length);
 *  3. a value for its variable from h = H(seed, id, k, 2^62 + 1): binary 1 - x_j; integer: with
 *     lo = l_j (x_j - R if infinite), hi = u_j (x_j + R if infinite), cnt = min(hi - lo, 2^52)
 *     values other than x_j, v = lo + (h mod cnt), then v + 1 if v >= x_j; continuous:
 *     v = lo + (hi - lo) * ((h >> 11) * 2^-53), at most hi; fixed or cnt < 1: no move.
 * Returns 1 with (*jo, *vo) when a move was drawn. */
static int perturb_draw(const orc_problem* P, const orc_params* prm, const orc_walker* S, int64_t k,
                        const double* r, int32_t* jo, double* vo) {
  int32_t mn = P->m_norm;
  int cut_active = S->cutoff_rhs < INFINITY;
  uint64_t hv = 0, ha = 0;
  int32_t iv = -1, ia = -1;
  for (int32_t i = 0; i < mn; i++) {
    if (i == mn - 1 && !cut_active) continue;
    uint64_t h = orc_draw(prm->rng_seed, (uint64_t)S->id, (uint64_t)k, (uint64_t)i) >> 32;
    if (ia < 0 || h < ha) { ia = i; ha = h; }              /* i increases: ties keep the lower i */
    if (r[i] > 0.0 && (iv < 0 || h < hv)) { iv = i; hv = h; }
  }
  int32_t row = iv >= 0 ? iv : ia;
  if (row < 0) return 0;
  int64_t len = 0;
  if (row < mn - 1) len = P->rp[row + 1] - P->rp[row];
  else
    for (int32_t j = 0; j < P->n; j++) len += (P->c[j] != 0.0);
  if (len == 0) return 0;
  int64_t q = (int64_t)(orc_draw(prm->rng_seed, (uint64_t)S->id, (uint64_t)k, 1ULL << 62) % (uint64_t)len);
  int32_t j = -1;
  if (row < mn - 1) j = P->ci[P->rp[row] + q];
  else
    for (int32_t jj = 0; jj < P->n; jj++)
      if (P->c[jj] != 0.0 && q-- == 0) { j = jj; break; }
  uint64_t h = orc_draw(prm->rng_seed, (uint64_t)S->id, (uint64_t)k, (1ULL << 62) + 1);
  double xj = S->x[j], R = (double)prm->perturb_radius;
  double lo = isfinite(P->lb[j]) ? P->lb[j] : xj - R;
  double hi = isfinite(P->ub[j]) ? P->ub[j] : xj + R;
  double v;
  switch (P->vclass[j]) {
    case 1: v = 1.0 - xj; break;
    case 2: {
      double cnt = hi - lo;
      if (!(cnt >= 1.0)) return 0;
      if (cnt > 4503599627370496.0) cnt = 4503599627370496.0;   /* 2^52 */
      v = lo + (double)(h % (uint64_t)cnt);
      if (v >= xj) v = v + 1.0;
      break;
    }
    case 3: {
      double u = (double)(h >> 11) * 0x1.0p-53;
      v = lo + (hi - lo) * u;
      if (v > hi) v = hi;
      break;
    }
    default: return 0;   /* fixed */
  }
  *jo = j;
  *vo = v;
  return 1;
}

int orc_tabu_run(const orc_problem* P, const orc_params* prm, orc_walker* S, int64_t n_iters,
                 orc_record* log, int n_threads) {
  if (!S->initialised) return ORC_ERR_INVALID_ARG;
  int32_t n = P->n, mn = P->m_norm;
  double* r = (double*)malloc(sizeof(double) * mn);
  double* y = (double*)malloc(sizeof(double) * mn);
  double* xhat = (double*)malloc(sizeof(double) * (n + 1));
  double* score = (double*)malloc(sizeof(double) * (n + 1));
  double* xt = (double*)malloc(sizeof(double) * (n + 1));   /* aspiration: the point after a move */
  double* r2 = (double*)malloc(sizeof(double) * mn);
  if (!r || !y || !xhat || !score || !xt || !r2) {
    free(r); free(y); free(xhat); free(score); free(xt); free(r2);
    return ORC_ERR_OOM;
  }
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  for (int64_t it = 0; it < n_iters; it++) {
    int64_t k = S->k;
    int cut_active = S->cutoff_rhs < INFINITY;
    if (S->force_j >= 0) {   /* R21: the perturbation drawn by the stuck iteration k - 1 */
      orc_record rec;
      memset(&rec, 0, sizeof(rec));
      rec.k = k; rec.j = S->force_j; rec.flags = 1; rec.v = S->force_v; rec.s = NAN;
      S->x[S->force_j] = S->force_v;
      S->tabu_until[S->force_j] = k + 1 + prm->tenure;
      S->force_j = -1;
      rec.violated = incumbent_check(P, prm, S, r);
      rec.obj = objective(P, S->x);
      if (log) log[it] = rec;
      S->k = k + 1;
      continue;
    }
    activities(P, S->x, y);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int32_t j = 0; j < n; j++) best_shift_var(P, j, S->x, y, S->w, S->cutoff_rhs, &xhat[j], &score[j]);
    orc_residuals(P, S->x, S->cutoff_rhs, r);
    /* selection: admissible = not tabu, or (aspiration, R18) tabu with s_j > 0
     * and a feasible point after the move; max s_j, ties lowest j (R6) */
    int32_t js = -1; double ss = -INFINITY;
    for (int32_t j = 0; j < n; j++) {
      if (P->vclass[j] == 0) continue;
      if (S->tabu_until[j] > k && !(prm->aspiration && score[j] > 0.0 && feasible_after(P, S, j, xhat[j], xt, r2)))
        continue;
      if (js < 0 || score[j] > ss) { js = j; ss = score[j]; }
    }
    orc_record rec;
    memset(&rec, 0, sizeof(rec));
    rec.k = k;
    if (js >= 0 && ss > 0.0) {
      rec.j = js; rec.v = xhat[js];
      S->x[js] = xhat[js];
      S->tabu_until[js] = k + 1 + prm->tenure;
    } else {
      /* stuck: bump every active violated row (R12) — or, when the smoothing draw of R22 falls
       * below smooth_prob, lower every active satisfied row's weight above 1 by one instead */
      rec.j = -1; rec.v = NAN;
      int smooth = 0;
      if (prm->smooth_prob > 0.0f) {
        double u = (double)(orc_draw(prm->rng_seed, (uint64_t)S->id, (uint64_t)k, (1ULL << 62) + 2) >> 11) * 0x1.0p-53;
        smooth = u < (double)prm->smooth_prob;
      }
      for (int32_t i = 0; i < mn; i++) {
        if (i == mn - 1 && !cut_active) continue;
        if (smooth) {
          if (!(r[i] > 0.0) && S->w[i] > 1.0f) S->w[i] = S->w[i] - 1.0f;
        } else if (r[i] > 0.0) {
          float nw = S->w[i] + 1.0f;
          S->w[i] = nw < prm->weight_cap ? nw : prm->weight_cap;
        }
      }
      if (prm->perturb) {   /* R21: drawn from this point's residuals, applied next iteration */
        int32_t jp; double vp;
        if (perturb_draw(P, prm, S, k, r, &jp, &vp)) { S->force_j = jp; S->force_v = vp; }
      }
    }
    rec.s = (js >= 0) ? ss : -INFINITY;
    rec.violated = incumbent_check(P, prm, S, r);
    rec.obj = objective(P, S->x);
    if (log) log[it] = rec;
    S->k = k + 1;
  }
  free(r); free(y); free(xhat); free(score); free(xt); free(r2);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------------------- */
/* portfolio exchange — engineering rule, not stated by the paper  */
/* ---------------------------------------------------------------------------------------- */

int orc_walker_restart(const orc_problem* P, const orc_params* prm, orc_walker* S, const double* x) {
  for (int32_t j = 0; j < P->n; j++) {
    if (!(x[j] >= P->lb[j] && x[j] <= P->ub[j])) return ORC_ERR_INVALID_ARG;
    S->x[j] = x[j];
    S->tabu_until[j] = 0;
  }
  S->force_j = -1;
  double* r = (double*)malloc(sizeof(double) * P->m_norm);
  incumbent_check(P, prm, S, r);
  free(r);
  return ORC_OK;
}

void orc_walker_set_cutoff(const orc_problem* P, const orc_params* prm, orc_walker* S, double z) {
  double rhs = z - cutoff_delta(P, prm, z);
  if (S->cutoff_rhs == INFINITY || rhs < S->cutoff_rhs) S->cutoff_rhs = rhs;
}

void orc_walker_summary(const orc_problem* P, const orc_walker* S, int64_t* violated, double* sumviol) {
  double* r = (double*)malloc(sizeof(double) * P->m_norm);
  orc_residuals(P, S->x, S->cutoff_rhs, r);
  *violated = count_violated(P, r, S->cutoff_rhs < INFINITY);
  double sv = 0.0;
  for (int32_t i = 0; i < P->m_norm - 1; i++) sv += (r[i] > 0.0) ? r[i] : 0.0;
  *sumviol = sv;
  free(r);
}

typedef struct { double a; double b; int64_t c; int32_t id; } orc_key;

static int key_less(const orc_key* x, const orc_key* y) {
  if (x->a != y->a) return x->a < y->a;
  if (x->b != y->b) return x->b < y->b;
  if (x->c != y->c) return x->c < y->c;
  return x->id < y->id;
}

/* selection of the k smallest keys, in order (plain insertion, W is small) */
static int32_t top_k(orc_key* keys, int32_t n, int32_t k) {
  for (int32_t i = 1; i < n; i++) {
    orc_key v = keys[i];
    int32_t q = i;
    while (q > 0 && key_less(&v, &keys[q - 1])) { keys[q] = keys[q - 1]; q--; }
    keys[q] = v;
  }
  return n < k ? n : k;
}

int orc_run_walkers(const orc_problem* P, const orc_params* prm, orc_walker* S, int32_t W, int64_t K,
                    int64_t n_epochs, int32_t n_elite, int32_t n_restart, int n_threads) {
  int32_t n = P->n;
  orc_key* keys = (orc_key*)malloc(sizeof(orc_key) * (W + 1));
  int64_t* viol = (int64_t*)malloc(sizeof(int64_t) * (W + 1));
  double* sv = (double*)malloc(sizeof(double) * (W + 1));
  double* elite = (double*)malloc(sizeof(double) * (size_t)(2 * n_elite + 1) * (n + 1));
  for (int64_t ep = 0; ep < n_epochs; ep++) {
    for (int32_t w = 0; w < W; w++) {
      int st = orc_tabu_run(P, prm, &S[w], K, NULL, n_threads);
      if (st != ORC_OK) return st;
    }
    if (ep == n_epochs - 1) break;       /* no exchange after the last epoch */
    for (int32_t w = 0; w < W; w++) orc_walker_summary(P, &S[w], &viol[w], &sv[w]);
    /* feasible elite */
    int32_t nf = 0;
    for (int32_t w = 0; w < W; w++)
      if (S[w].has_incumbent) { keys[nf].a = S[w].best_obj; keys[nf].b = 0; keys[nf].c = 0; keys[nf].id = w; nf++; }
    int32_t kf = top_k(keys, nf, n_elite);
    int32_t ne = 0;
    double z = INFINITY;
    for (int32_t q = 0; q < kf; q++) {
      memcpy(elite + (size_t)ne * n, S[keys[q].id].best_x, sizeof(double) * n);
      ne++;
      if (S[keys[q].id].best_obj < z) z = S[keys[q].id].best_obj;
    }
    /* infeasible elite: current points by (violated, sumviol, id) */
    for (int32_t w = 0; w < W; w++) { keys[w].a = (double)viol[w]; keys[w].b = sv[w]; keys[w].c = 0; keys[w].id = w; }
    int32_t ki = top_k(keys, W, n_elite);
    for (int32_t q = 0; q < ki; q++) {
      memcpy(elite + (size_t)ne * n, S[keys[q].id].x, sizeof(double) * n);
      ne++;
    }
    /* cutoff from the global incumbent */
    if (z < INFINITY)
      for (int32_t w = 0; w < W; w++) orc_walker_set_cutoff(P, prm, &S[w], z);
    /* restarts: highest (violated, id) first */
    for (int32_t w = 0; w < W; w++) { keys[w].a = -(double)viol[w]; keys[w].b = 0; keys[w].c = -(int64_t)w; keys[w].id = w; }
    int32_t kr = top_k(keys, W, n_restart);
    if (ne > 0)
      for (int32_t q = 0; q < kr; q++) {
        int st = orc_walker_restart(P, prm, &S[keys[q].id], elite + (size_t)(q % ne) * n);
        if (st != ORC_OK) return st;
      }
  }
  free(keys); free(viol); free(sv); free(elite);
  return ORC_OK;
}

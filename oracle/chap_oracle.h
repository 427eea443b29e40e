/* chap_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct fp64 CPU oracle for the best-shift tabu core of
 * CHAP (arxiv 2605.05086, §3.1 "GPU Tabu Search", lines 265-363).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library. It shares no code, header, table or helper with the CUDA
 * path under paper_2605_05086_b200/csrc, and neither includes the other.
 *
 * Every function evaluates the paper's DEFINITIONS directly (activities recomputed from
 * A x̄ from scratch, every candidate shift scored by summing the penalty table) — no
 * breakpoint accumulators, sorting or scanning (Alg. 1) appears here.
 * Readings of the paper where it is silent or ambiguous are listed in DESIGN.md §3 and
 * cited below as R<n>.
 */
#ifndef CHAP_ORACLE_H
#define CHAP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_INVALID_ARG = 1, ORC_ERR_INFEASIBLE_BOUNDS = 2, ORC_ERR_OOM = 4 };

typedef struct orc_problem orc_problem;

/* Normalise lhs <= Ax <= rhs to rows a.x <= b (§3.1 "Second, we normalize"):
 * for each original row in order, the upper side (a, rhs) if rhs is finite, then the lower
 * side (-a, -lhs) if lhs is finite; rows left empty are dropped (or infeasible if 0 violates
 * them); one cutoff row c.x <= z* - delta is appended last, inactive until set.
 * Integer bounds are rounded inward (R8/SURVEY §8(b)). */
int orc_problem_create(int32_t n, int32_t m, int64_t nnz, const int64_t* row_ptr,
                       const int32_t* col_idx, const double* val, const double* lhs,
                       const double* rhs, const double* lb, const double* ub,
                       const uint8_t* is_int, const double* c, orc_problem** out);
void orc_problem_free(orc_problem* P);
/* sizes: m_norm (incl. cutoff row), nnz_norm (excl. cutoff row), cutoff row nnz */
void orc_problem_sizes(const orc_problem* P, int32_t* m_norm, int64_t* nnz_norm, int64_t* nnz_cut);
/* normalised row i (< m_norm-1) came from original row orig[i], side[i] = +1 (upper) / -1 (lower) */
void orc_problem_row_map(const orc_problem* P, int32_t* orig, int8_t* side);
/* the bounds after inward rounding, and the variable class: 0 fixed, 1 binary, 2 integer, 3 continuous */
void orc_problem_vars(const orc_problem* P, double* lb, double* ub, uint8_t* vclass);
/* auto cutoff delta (R14): 1 if every c_j != 0 is integral and on an integer variable, else NaN
 * (meaning 1e-6*max(1,|z|) at the time the cutoff is set) */
double orc_auto_delta(const orc_problem* P);

/* Penalty p_ij of PAPER.md:277-285 on residuals r = y - b: five cases. */
double orc_penalty(double w, double r_old, double r_new);

/* Breakpoint t_ij = (b_i - sum_{k!=j} a_ik x_k)/a_ij = x_j - r_i/a_ij (Alg.1 l.3),
 * floored (a>0) / ceiled (a<0) for integer variables (Alg.1 l.4, R8). */
double orc_breakpoint(double x_j, double r_i, double a_ij, int is_integer);

/* r_i = (A x)_i - b_i for every normalised row, recomputed from scratch.
 * The cutoff row's r is -inf when cutoff_rhs = +inf (inactive). */
void orc_residuals(const orc_problem* P, const double* x, double cutoff_rhs, double* r);

/* Best shift of Eq. (1) for every variable by brute force over the candidate
 * set of PAPER.md:299 (R5): binaries {1-x_j}; otherwise the finite bounds and
 * every breakpoint, within [l_j,u_j], minus x_j (R2). Each candidate v is scored by direct
 * recomputation s = sum_i p(w_i, y_i - b_i, (y_i - a_ij x_j + a_ij v) - b_i).
 * Ties: smallest |v - x_j|, then smallest v (R4). No candidate: (x_j, -inf).
 * w: [m_norm] float weights (NULL = all 1). best_{j,v,s}: argmax over s_j > 0, lowest j (R6);
 * j = -1 if none. n_threads <= 0: OpenMP default. */
int orc_best_shift(const orc_problem* P, const double* x, const float* w, double cutoff_rhs,
                   double* xhat, double* score, int32_t* best_j, double* best_v, double* best_s,
                   int n_threads);

/* The same for the variables [j0, j1) only (activities still from scratch; xhat/score [n] are
 * written at [j0, j1); the best move is the best within the range). Used for bounded samples. */
int orc_best_shift_range(const orc_problem* P, const double* x, const float* w, double cutoff_rhs,
                         int32_t j0, int32_t j1, double* xhat, double* score, int32_t* best_j,
                         double* best_v, double* best_s, int n_threads);

typedef struct {
  int32_t tenure;        /* T: a moved variable is inadmissible in iterations k+1..k+T (R13)   */
  float weight_cap;      /* w <= cap (R11, R12)                                               */
  double cutoff_delta;   /* NaN = auto (R14)                                                  */
  int32_t aspiration;    /* 1: a tabu variable is admissible when moving it to its best shift
                            makes the point feasible, i.e. gives a new incumbent (R18, NEXT f1) */
  int32_t perturb;       /* 1: perturbation after a stuck iteration (R21, NEXT f1)             */
  int32_t perturb_radius;/* half-width of the value window on an infinite side (R21)          */
  float smooth_prob;     /* weight smoothing probability per stuck iteration (R22)            */
  uint64_t rng_seed;     /* seed of the counter-based draws (R21, R22)                        */
} orc_params;

typedef struct {
  int64_t k; int32_t j; int32_t flags; double v; double s; int64_t violated; double obj;
} orc_record;            /* identical field order to chap_step_record (48 bytes); flags = 1 for
                            a perturbation move (R21)                                          */

/* One walker's state. x [n], w [m_norm], tabu_until [n], best_x [n] are caller-owned. */
typedef struct {
  double* x; float* w; int64_t* tabu_until; double* best_x;
  int64_t k; double cutoff_rhs; double best_obj; int32_t has_incumbent; int32_t initialised;
  int64_t id;            /* walker index: the a of the draws H(seed, a, k, c) (R21)            */
  int32_t force_j;       /* a perturbation drawn at a stuck iteration, applied by the next one
                            (-1: none); cleared by init and restart                            */
  int32_t pad;
  double force_v;
} orc_walker;

/* SplitMix64's output function g (the first output of SplitMix64 seeded with state) and the
 * counter-based draw H(seed, a, b, c) = g(g(g(g(seed) ^ a) ^ b) ^ c) of R21. */
uint64_t orc_splitmix64(uint64_t state);
uint64_t orc_draw(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);

/* Initialise a walker at x0 (copied): w = 1, tabu_until = 0, k = 0, cutoff inactive; then the
 * k = 0 incumbent check (R15). */
int orc_walker_init(const orc_problem* P, const orc_params* prm, const double* x0, orc_walker* S);

/* n_iters tabu iterations ("the best admissible move is selected and applied";
 * PAPER.md:361 own solution, tabu list and weights). Each iteration: residuals from scratch;
 * best shift of every variable; select the admissible (tabu_until_j <= k, or with
 * prm->aspiration a tabu j with s_j > 0 whose move to xhat_j leaves no active row violated, R18)
 * argmax s_j, ties lowest j; if s* > 0 move x_j* <- xhat_j*, tabu_until_j* = k+1+T; else (stuck) bump
 * w_i <- min(w_i + 1, cap) on every active row with r_i > 0 (R12); then, if every active row has
 * r_i <= 0, record the incumbent and set the cutoff rhs to c.x - delta; log. */
int orc_tabu_run(const orc_problem* P, const orc_params* prm, orc_walker* S, int64_t n_iters,
                 orc_record* log, int n_threads);

/* Restart a walker from x (copied): tabu cleared, weights and k kept, then the incumbent check of
 * R15 (SURVEY §8(e) restart rule). */
int orc_walker_restart(const orc_problem* P, const orc_params* prm, orc_walker* S, const double* x);
/* Impose a cutoff from an external incumbent z: rhs = z - delta, only tightening. */
void orc_walker_set_cutoff(const orc_problem* P, const orc_params* prm, orc_walker* S, double z);
/* Exchange summary of a walker: active violated rows (cutoff included) and the total violation
 * sum_{i < m_norm-1} max(0, r_i) of its current point. */
void orc_walker_summary(const orc_problem* P, const orc_walker* S, int64_t* violated, double* sumviol);

/* The portfolio of SURVEY §8(e) in one process: W walkers from x0s [W][n]; n_epochs epochs of K
 * tabu iterations each; after every epoch but the last the exchange rule:
 *   summaries (best_obj or +inf, violated, sumviol) of every walker;
 *   feasible elite F = the n_elite walkers with an incumbent by (best_obj, id), their best points;
 *   infeasible elite I = the n_elite walkers by (violated, sumviol, id), their current points;
 *   z = min best_obj -> every walker's cutoff tightened to z - delta;
 *   the n_restart walkers with the highest (violated, id) restart, in that order, from the elite
 *   list E = F ++ I round-robin (E[q mod |E|]).
 * Walker states are left in S[W] (caller-initialised with orc_walker_init). */
int orc_run_walkers(const orc_problem* P, const orc_params* prm, orc_walker* S, int32_t W, int64_t K,
                    int64_t n_epochs, int32_t n_elite, int32_t n_restart, int n_threads);

#ifdef __cplusplus
}
#endif
#endif

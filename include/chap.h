/* chap.h — C ABI of the B200-native best-shift tabu core of CHAP (arxiv 2605.05086).
 *
 * The library evaluates, for every variable j of a candidate point x̄ of
 *     min c^T x  s.t.  lhs <= A x <= rhs,  l <= x <= u,  x_j ∈ Z (j ∈ I)
 * the exact best-shift move of Eq. (1) (§3.1 "Best Shift Moves") using
 * Algorithm 1 (breakpoint emission, segmented sort, scan, argmax) on
 * sm_100a, then runs the tabu walk around it (PAPER.md:80-85 and §3.1 "Parallel Tabu Search
 * Instances", :359-363) with incremental residual updates and constraint-weight
 * bumps. The problem form is PAPER.md:269 with two-sided rows (north star), normalised
 * internally to a.x <= b rows.
 *
 * Conventions (every function):
 *  - returns chap_status; nothing throws across the ABI; chap_last_error() gives a
 *    thread-local message for the last non-OK status on the calling thread;
 *  - "HOST" pointers are ordinary CPU memory, "DEVICE" pointers are CUDA device memory on the
 *    handle's device; all DEVICE outputs are caller-allocated and written stream-ordered on
 *    the given cudaStream_t (passed as void*, NULL = the legacy default stream);
 *  - handles are owned by the caller until *_destroy; a walkers object borrows its problem,
 *    so the problem must outlive it; different handles may be used from different threads,
 *    one handle must not be used concurrently;
 *  - no function allocates device memory per call except the *_create functions and
 *    chap_eval_best_shift_host (which allocates pinned staging once per problem).
 * Readings R1..R17 of the paper are listed in DESIGN.md §3.
 */
#ifndef CHAP_H
#define CHAP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHAP_ABI_VERSION 4

typedef enum {
  CHAP_OK = 0,
  CHAP_ERR_INVALID_ARG = 1,       /* bad size/pointer, NaN, index out of range, duplicate (i,j),
                                     x out of bounds or fractional on an integer variable, w < 0 */
  CHAP_ERR_INFEASIBLE_BOUNDS = 2, /* l > u after rounding integer bounds inward, or an empty row
                                     whose sides exclude 0                                       */
  CHAP_ERR_CUDA = 3,              /* a CUDA runtime error (message has the CUDA error string)    */
  CHAP_ERR_OOM = 4,               /* device or host allocation failed                            */
  CHAP_ERR_NCCL = 5,              /* an NCCL call failed                                         */
  CHAP_ERR_STATE = 6,             /* call not valid in the handle's current state                */
  CHAP_ERR_UNSUPPORTED = 7        /* reserved (no column shape is rejected since the grid-wide sort) */
} chap_status;

/* Message for the last non-OK status returned on this thread ("" if none). */
const char* chap_last_error(void);
/* Static name of a status code. */
const char* chap_status_string(chap_status s);
/* CHAP_ABI_VERSION of the loaded library. */
int32_t chap_abi_version(void);

/* ---------------------------------------------------------------------------------------- */
/* Problem                                                                                  */
/* ---------------------------------------------------------------------------------------- */

typedef struct chap_problem chap_problem;

typedef struct {
  int32_t n, m;               /* as given                                                      */
  int32_t m_norm;             /* normalised rows incl. the cutoff row, which is last            */
  int32_t cutoff_row;         /* = m_norm - 1                                                  */
  int64_t nnz_norm;           /* nonzeros of the normalised rows, cutoff row excluded          */
  int64_t nnz_cut;            /* nonzeros of the cutoff row (#{j : c_j != 0})                  */
  int32_t n_fixed, n_binary, n_integer, n_continuous;   /* variable classes after rounding    */
  int32_t exact_integer_data; /* 1: A, lhs, rhs, l, u, c integral, |a| <= 1e6, all variables
                                 integer -> scores and trajectories are bit-exact */
  int32_t n_long_columns;     /* columns evaluated in warp chunks (long binary, long bounded
                                 integer), added up by atomics, finished by k_eval          */
  double auto_cutoff_delta;   /* 1 if every c_j != 0 is integral on an integer variable, else
                                 NaN (= 1e-6 max(1,|z|) when the cutoff is set) (R14)         */
  int64_t device_bytes;       /* device memory held by the problem                            */
  int64_t model_bytes_A;      /* algorithmic bytes of one pass over A in CSC:
                                 12 (nnz + nnz_cut) + 4 (n + 1), nnz = the ORIGINAL nonzeros
                                 (a two-sided row's entry counts once)          */
  int64_t model_bytes_pass;   /* algorithmic bytes of one best-shift pass of one walker (SURVEY
                                 §8(d)): A in CSC as above, static per-variable data (1 B binary,
                                 17 B other), walker state per variable (x̄: 1 bit binary / 8 B
                                 other; 4 B tabu expiry) and 12 B per normalised row (r f64 +
                                 w f32), each read once (§6)                                  */
  int64_t model_bytes_kernel[3]; /* the same model split by column class: [0] packed binary
                                 columns (k_eval_binrow / k_eval_bin), [1] long binary, general,
                                 empty and long bounded-integer columns, [2] sorted general
                                 columns and the 12 B/row row state                           */
  int64_t nnz_kernel[3];      /* original nonzeros (incl. cutoff entries) of each class split  */
  int32_t eval_launches;      /* kernel launches of one best-shift pass (1-3: the eval kernels
                                 with work, k_eval always); a tabu iteration adds the apply   */
  int32_t n_sorted_columns;   /* general columns whose breakpoints are sorted (line 13) rather
                                 than prefix-summed or bucket-counted: non-bucketable columns
                                 with more than 62 nonzeros                     */
  int64_t model_bytes_walker_kernel[3]; /* the per-walker part of model_bytes_kernel (x̄, tabu
                                 expiry, row state); the rest (A in CSC, static per-variable
                                 data) is read once by a batched pass of W walkers, whose model
                                 is therefore shared + W x per-walker          */
  int32_t n_gridsort_columns; /* of n_sorted_columns, those longer than one block's sort (more
                                 than 2043 nonzeros): chunk sorts plus co-ranking across blocks
                                 ("grid-wide primitives")           */
  int32_t pad_info;
  int64_t exchange_point_bytes; /* bytes of one packed elite point of the portfolio exchange:
                                 binaries as bits, integers as int32 (int64 if a bound is
                                 infinite or beyond 2^31), continuous as f64   */
} chap_problem_info;

/* Build a problem from HOST CSR data (copied; the caller may free its arrays on return).
 *   row_ptr  [m+1] int64, row_ptr[0] = 0, non-decreasing, row_ptr[m] = nnz
 *   col_idx  [nnz] int32 in [0, n); no duplicate (row, col); explicit zeros are dropped
 *   val      [nnz] finite
 *   lhs, rhs [m]   lhs <= rhs; -INF / +INF = that side absent; a free or empty row is dropped
 *   lb, ub   [n]   +-INF allowed; integer bounds are rounded inward (ceil l, floor u)
 *   is_integer [n] 0/1
 *   c        [n]   finite; minimisation
 *   device   CUDA device ordinal the problem lives on
 * Normalisation: for each original row in order, the upper side a.x <= rhs if
 * rhs is finite, then the lower side -a.x <= -lhs if lhs is finite; each side is its own row
 * with its own weight and residual (R17). Row m_norm-1 is the cutoff row c.x <= z* - delta
 * (PAPER.md:373), inactive (excluded from every score) until a cutoff is set.
 * Variable classes: fixed (l = u), binary (integer, l = 0, u = 1), integer,
 * continuous. Errors: INVALID_ARG, INFEASIBLE_BOUNDS, UNSUPPORTED (a non-binary column with
 * more than 4094 nonzeros whose domain is not a bounded integer range of <= 4096 values),
 * CUDA, OOM. */
chap_status chap_problem_create(int32_t n, int32_t m, int64_t nnz, const int64_t* row_ptr,
                                const int32_t* col_idx, const double* val, const double* lhs,
                                const double* rhs, const double* lb, const double* ub,
                                const uint8_t* is_integer, const double* c, int32_t device,
                                chap_problem** out);
chap_status chap_problem_info_get(const chap_problem* p, chap_problem_info* out);
/* HOST [m_norm-1] outputs: normalised row i came from original row orig_row[i], side[i] = +1
 * (upper, a.x <= rhs) or -1 (lower, -a.x <= -lhs). */
chap_status chap_problem_row_map(const chap_problem* p, int32_t* orig_row, int8_t* side);
chap_status chap_problem_destroy(chap_problem* p);

/* ---------------------------------------------------------------------------------------- */
/* Single-point evaluation (the parity entry point)                                          */
/* ---------------------------------------------------------------------------------------- */

typedef struct {
  int32_t j;   /* variable index, -1 if no variable has s_j > 0                               */
  int32_t pad;
  double v;    /* its best shift x̂_j (NaN if j = -1)                                           */
  double s;    /* its score s_j (-INF if j = -1)                                               */
} chap_move;   /* 24 bytes */

/* Eq. (1) for every variable at the point x, by Algorithm 1:
 *   x      DEVICE [n] float64: within bounds, integral on integer variables
 *   w      DEVICE [m_norm] float32 weights >= 0 (NULL = all 1); w[m_norm-1] is the cutoff
 *          row's weight. Scores are exact when weights are integers <= 2^24 (R11).
 *          x and w are validated on the device during the call: an x out of bounds or
 *          fractional on an integer variable, or a negative or NaN weight (negative weights break
 *          Algorithm 1's monotone prefixes), returns CHAP_ERR_INVALID_ARG after the
 *          stream is synchronised (the outputs are then unspecified).
 *   cutoff_rhs  +INF = cutoff row inactive; finite = the row c.x <= cutoff_rhs is scored
 *   xhat, score DEVICE [n] float64 outputs (either may be NULL): the best shift x̂_j and its raw
 *          maximum score s_j over the candidate set {finite bounds} ∪ {breakpoints} within
 *          [l_j, u_j] minus {x̄_j} (R2, R5); ties -> smallest |v - x̄_j|, then smallest v (R4).
 *          A variable without candidates (fixed) reports (x̄_j, -INF). s_j may be <= 0 (R7).
 *   best   DEVICE [1] chap_move out (may be NULL): argmax of s_j over s_j > 0, ties -> lowest j
 *          (R6); j = -1 if none.
 * Runs on cuda_stream and synchronises it before returning (to report the validation); uses the
 * problem's internal workspace, so calls on one problem must not overlap. */
chap_status chap_eval_best_shift(const chap_problem* p, const double* x, const float* w,
                                 double cutoff_rhs, double* xhat, double* score, chap_move* best,
                                 void* cuda_stream);

/* The same call with HOST buffers (x [n], w [m_norm] or NULL, xhat/score [n] or NULL, best
 * [1] or NULL): copies in, evaluates, copies out, and synchronises the stream before
 * returning. Page-locked (pinned) buffers are copied by DMA directly; pageable ones pass through
 * pinned staging owned by the problem. Used for the end-to-end (e2e) measurement. */
chap_status chap_eval_best_shift_host(chap_problem* p, const double* x, const float* w,
                                      double cutoff_rhs, double* xhat, double* score,
                                      chap_move* best, void* cuda_stream);

/* ---------------------------------------------------------------------------------------- */
/* Tabu walkers                                                                              */
/* ---------------------------------------------------------------------------------------- */

typedef struct {
  int32_t tenure;        /* T (default 10): a moved variable is inadmissible in k+1..k+T (R13) */
  float weight_cap;      /* default 1e6; must be in [1, 2^24] so f32 weights stay exact (R11)  */
  double cutoff_delta;   /* NaN = auto (R14)                                                   */
  int32_t exchange_K;    /* iterations per epoch in chap_run_walkers (default 1000)            */
  int32_t n_elite;       /* elite points exchanged per kind per rank (default 4)               */
  int32_t n_restart;     /* walkers restarted from the elite per exchange (default W_total/8)  */
  int32_t graph_iters;   /* iterations per captured CUDA graph in chap_tabu_step (default 16;
                            0 = plain launches); a call's remainder runs as one more graph    */
  int32_t binary_kernel; /* packed binary columns of a single walker: 0 = auto (row-wise kernel
                            when the problem has >= 3e6 binary nonzeros and >= 0.7 entries per
                            row per block), 1 = column-wise, 2 = row-wise (when the
                            coefficients allow it: integers of magnitude <= 32767)            */
  int32_t pdl;           /* 1 = launch the iteration's kernels with programmatic dependent launch
                            (default 0: measured slower on config G)               */
  int32_t l2_persist;    /* 1 (default) = the walkers' row state (residuals and weights, the
                            target of every gather) is an L2 access-policy window with hits
                            persisting ("pin it to the L2 cache"); 0 = off        */
  int32_t aspiration;    /* 1 = incumbent aspiration (NEXT f1, DESIGN R18): a tabu variable is
                            admissible when its best shift makes the point feasible (a new
                            incumbent, the cutoff row included); 0 (default) = off           */
  int32_t lazy;          /* 1 = selective re-evaluation (NEXT f2, an A/B against the paper's
                            from-scratch pass): only the columns whose x̄ or row
                            state changed are re-evaluated, the others keep their cached best
                            shift (identical results); one walker only; 0 (default) = every
                            variable every iteration                                          */
  int32_t perturb;        /* 1 = perturbation after a stuck iteration (NEXT f1, DESIGN R21): the
                            stuck iteration k draws a row (uniform over the violated active rows,
                            else over all active rows: the least (h >> 32, i) of
                            h = H(seed, walker, k, i)), an entry of it (H(.., 2^62) mod its
                            length) and a new value (H(.., 2^62 + 1)): binary 1 - x̄, integer
                            uniform over the domain minus x̄, continuous uniform on [lo, hi], an
                            infinite side replaced by x̄ -/+ perturb_radius; iteration k + 1
                            applies that move in place of its selection (logged with pad = 1,
                            s = NaN). H(s, a, b, c) = g(g(g(g(s) ^ a) ^ b) ^ c), g = SplitMix64's
                            output function. 0 (default) = off                               */
  int32_t perturb_radius; /* window half-width on an infinite side (default 16, >= 1)         */
  float smooth_prob;      /* weight smoothing (NEXT f1, DESIGN R22): a stuck iteration k with
                            u = (H(seed, walker, k, 2^62 + 2) >> 11) 2^-53 < smooth_prob
                            lowers w_i <- w_i - 1 on every active satisfied row with w_i > 1
                            instead of the bump; 0 (default) = always bump, in [0, 1]          */
  uint64_t rng_seed;      /* the seed of H (default 0); give each rank its own                */
} chap_params;

/* Fill *out with the defaults above (n_restart = -1 meaning W_total/8). */
chap_status chap_params_default(chap_params* out);

typedef struct {
  int64_t k;        /* iteration index                                                       */
  int32_t j;        /* moved variable (user index), -1 = stuck: weights bumped, no move      */
  int32_t flags;    /* 1 = the move is a perturbation (chap_params.perturb, R21), else 0      */
  double v;         /* new value of x_j (NaN if stuck)                                        */
  double s;         /* its score; if stuck, the best admissible s_j (<= 0) or -INF if none;
                       NaN for a perturbation                                                 */
  int64_t violated; /* active rows with r > 0 after the step (cutoff row included)           */
  double obj;       /* c.x̄ after the step                                                     */
} chap_step_record; /* 48 bytes; bit-identical to the oracle's log in the exact domain        */

typedef struct {
  int64_t k;              /* iterations done                                                  */
  int64_t violated;       /* current violated active rows                                     */
  double obj;             /* c.x̄                                                             */
  double best_obj;        /* best incumbent objective (+INF if none)                          */
  double cutoff_rhs;      /* current cutoff rhs (+INF if inactive)                            */
  int32_t has_incumbent;  /* 1 if best_obj is set                                             */
  int32_t pad;
  int64_t n_moves;        /* moves applied                                                    */
  int64_t n_stuck;        /* stuck iterations (weight bumps)                                  */
} chap_walker_stats;      /* 64 bytes */

typedef struct chap_walkers chap_walkers;

/* W independent walkers (own solution, tabu list and weights) at start points
 *   x0 DEVICE [W][n] float64 (user variable order), in bounds, integral on integer variables.
 * Initial state: w = 1 on every row (cutoff included), tabu cleared, k = 0, cutoff inactive;
 * residuals computed from scratch; a feasible start is recorded as incumbent at once and the
 * cutoff set (R15). Errors: INVALID_ARG (W < 1, x0 invalid), OOM, CUDA. Synchronises. */
chap_status chap_walkers_create(const chap_problem* p, int32_t W, const double* x0,
                                const chap_params* params, void* cuda_stream, chap_walkers** out);

/* n_iters tabu iterations of every walker, entirely on the device (CUDA graphs of
 * params.graph_iters iterations, the remainder of n_iters as one more graph, kept for reuse). One iteration: best shift of every variable (Alg. 1);
 * select the admissible (tabu_until_j <= k) argmax s_j, ties lowest j (R6); if s* > 0 apply it
 * (x̄_j* <- x̂_j*, r_i += a_ij Δ over column j* — PAPER.md:343 — and tabu_until_j* = k+1+T),
 * else bump w_i <- min(w_i + 1, cap) on every active row with r_i > 0 (R12); then if no active
 * row is violated record the incumbent and set the cutoff rhs to c.x̄ - delta.
 *   log  DEVICE [n_iters][W] chap_step_record (walker-minor) or NULL. Stream-ordered. */
chap_status chap_tabu_step(chap_walkers* ws, int32_t n_iters, chap_step_record* log,
                           void* cuda_stream);

/* Export walker state (any pointer may be NULL); all DEVICE, user order, walker-major:
 *   x [W][n] float64, r [W][m_norm] float64 (r of an inactive cutoff row is -INF),
 *   w [W][m_norm] float32, tabu_until [W][n] int64 (absolute iteration), best_x [W][n] float64,
 *   stats [W] chap_walker_stats. Stream-ordered. */
chap_status chap_walkers_get(const chap_walkers* ws, double* x, double* r, float* w,
                             int64_t* tabu_until, double* best_x, chap_walker_stats* stats,
                             void* cuda_stream);
/* Impose a cutoff from an external incumbent: every walker whose cutoff rhs is
 * above z_best - delta gets rhs = z_best - delta (residual recomputed). Stream-ordered. */
chap_status chap_walkers_set_cutoff(chap_walkers* ws, double z_best, void* cuda_stream);
/* Restart walker `walker` from x DEVICE [n] (user order): residuals recomputed from scratch,
 * weights kept, tabu cleared (SURVEY §8(e) restart rule). x is validated first (synchronising the
 * stream): out of bounds or fractional on an integer variable -> CHAP_ERR_INVALID_ARG with the
 * walker untouched. */
chap_status chap_walkers_restart(chap_walkers* ws, int32_t walker, const double* x,
                                 void* cuda_stream);
chap_status chap_walkers_destroy(chap_walkers* ws);

/* ---------------------------------------------------------------------------------------- */
/* Streamed LP iterates for LP-seeded start points (NEXT f4, DESIGN R19)    */
/* ---------------------------------------------------------------------------------------- */

/* The LP relaxation min c.x s.t. the normalised rows (the cutoff row is not part of
 * it), l <= x <= u, by restarted PDHG: x+ = proj_[l,u](x - eta (c + A^T y)),
 * y+ = max(0, y + tau (A (2x+ - x) - b)), eta = tau = step, running averages of x+ and y+ and a
 * restart to them every restart_period iterations; x0 = proj_[l,u](0), y0 = 0. At each of the
 * n_cp strictly increasing checkpoints (HOST int64, e.g. 100, 1000, 10000: "after 10^2, 10^3,
 * 10^4 ... PDHG iterations, warm-starting each phase from the previous iterate")
 * the current primal average goes to x_out (DEVICE [n_cp][n], user order) and info_out (HOST
 * [n_cp][4]) receives {iteration, c.x, max_i (A x - b)_i^+, step}. step <= 0: 0.9/||A||_2 from 100
 * power iterations on the device. Synchronises the stream; CHAP_ERR_INVALID_ARG on bad arguments. */
chap_status chap_lp_pdhg(const chap_problem* p, const int64_t* checkpoints, int32_t n_cp, double step,
                         int32_t restart_period, double* x_out, double* info_out, void* cuda_stream);

/* An LP point (DEVICE [n], user order) to a tabu start point (DEVICE [n], user order): integer
 * variables rounded to the nearest integer (half away from zero), every value clamped to its
 * bounds ("LP snapshot rounded to nearest integer"); stream-ordered. */
chap_status chap_lp_round(const chap_problem* p, const double* x_lp, double* x_out, void* cuda_stream);

/* Diagnostic timing: n_iters tabu iterations (identical semantics to chap_tabu_step, no log),
 * captured as one CUDA graph with a CUDA-event pair around every kernel node (so no launch latency
 * is inside an interval) and run once on the walkers' stream; ms_per_iter HOST [5] receives the
 * average device time per iteration of [0] k_eval_bin (binary columns), [1] k_eval_gen (general,
 * empty, long bounded-integer columns), [2] k_eval (long-column ends, sorted general columns, the
 * global select), [3] reserved (0), [4] the apply kernel. Synchronises. */
chap_status chap_walkers_profile(chap_walkers* ws, int32_t n_iters, double* ms_per_iter,
                                 void* cuda_stream);

/* Per-kernel device time of the iterations chap_tabu_step runs while timing is on, measured inside
 * the captured graphs without events: every block stamps %globaltimer at its start (atomic min)
 * and end (atomic max) per kernel, and the apply kernel's finalising thread accumulates
 * end - start of each kernel of the iteration. out HOST [6] (may be NULL) first receives the sums:
 * ns of [0] the binary-column kernels (k_eval_bin and k_eval_binrow: first start to last end),
 * [1] k_eval_gen, [2] k_eval, [3] k_apply (its start to the finalisation), [4] first eval kernel
 * start to apply finalisation, [5] iterations timed (synchronous read). The eval kernels' device
 * time is [4] - [3].
 * Then mode 1 turns timing on and zeroes the sums, 0 turns it off, -1 only reads. Turning it on or
 * off re-captures the iteration graph at the next chap_tabu_step. */
chap_status chap_walkers_timing(chap_walkers* ws, int32_t mode, uint64_t* out, void* cuda_stream);

/* Kernel launches of one tabu iteration of these walkers (the eval kernels with work, the binary
 * row-wise kernel when used, k_eval and the apply kernel) into *out. */
chap_status chap_walkers_launches_per_iter(const chap_walkers* ws, int32_t* out);

/* ---------------------------------------------------------------------------------------- */
/* Multi-GPU portfolio: independent walkers per GPU with an every-K exchange                 */
/* ---------------------------------------------------------------------------------------- */

typedef struct chap_comm chap_comm;

/* NCCL unique id (128 bytes) created on one rank and broadcast by the caller (e.g. through
 * torch.distributed) to every rank before chap_comm_create. */
chap_status chap_comm_unique_id(uint8_t id[128]);
chap_status chap_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                             chap_comm** out);
chap_status chap_comm_destroy(chap_comm* comm);

typedef struct {
  double best_obj;          /* best incumbent over all walkers of all ranks (+INF if none)    */
  int32_t has_incumbent;
  int32_t best_walker;      /* global walker id of the incumbent's finder                      */
  int64_t iterations;       /* iterations done per walker                                     */
  int64_t epochs;
  double seconds;           /* wall time of the call                                          */
} chap_result;

/* Per-walker exchange summary (32 bytes), gathered from every rank. */
typedef struct {
  double best_obj;        /* best incumbent objective, +INF if none                            */
  int64_t violated;       /* violated active rows of the current point (cutoff row included)   */
  double sumviol;         /* sum over non-cutoff rows of max(0, r_i) at the current point      */
  int32_t gid;            /* global walker id = rank * W_local + local index                   */
  int32_t flags;          /* bit 0: has an incumbent; bit 1: this rank asks to stop            */
} chap_walker_summary;

/* The deterministic exchange rule of chap_run_walkers, a pure HOST function of the
 * gathered summaries (identical on every rank; usable without a GPU). With W_total summaries s[]
 * indexed by gid and ranks of W_local walkers each:
 *   feasible elite  = up to n_elite walkers with an incumbent, by (best_obj, gid): best points;
 *   infeasible elite = up to n_elite walkers by (violated, sumviol, gid): current points;
 *   the elite list E is the feasible elite followed by the infeasible elite; for each member
 *   elite_gid[q], elite_kind[q] (0: best point, 1: current point) and elite_slot[q], its slot in
 *   the gathered point buffer (rank * 2 n_elite + [n_elite if kind 1] + its position among that
 *   rank's own top-n_elite of the kind);
 *   *z_best = min best_obj (+INF if none), *best_gid its walker (lowest gid on ties; -1);
 *   the n_restart walkers with the highest (violated, gid) restart in that order:
 *   restart_gid[q] from E[q mod |E|] (restart_src[q]); none if E is empty.
 * Output arrays: elite_* [2 n_elite], restart_* [n_restart]. */
chap_status chap_exchange_plan(int32_t W_total, int32_t W_local, const chap_walker_summary* s,
                               int32_t n_elite, int32_t n_restart, double* z_best,
                               int32_t* best_gid, int32_t* n_elite_out, int32_t* elite_gid,
                               int8_t* elite_kind, int32_t* elite_slot, int32_t* n_restart_out,
                               int32_t* restart_gid, int32_t* restart_src);

/* chap_exchange_plan on the device (the portfolio exchange of PAPER.md:359-363 across GPUs, SURVEY
 * §8(e)), as the exchange of chap_walkers_exchange / chap_walkers_epoch computes it
 * (k_exchange_plan: one block, rank counting, O(W_total^2) comparisons), for the walkers of rank
 * `rank`. Caller-owned buffers, nothing retained after the call. All
 * pointers are DEVICE memory, stream-ordered on cuda_stream; s[W_total] indexed by gid as for
 * chap_exchange_plan. Outputs: z_best [1] (+INF: no incumbent); counts [4]: best gid (-1), |E|,
 * the number of restarts, unused; elite_gid / elite_slot [2 n_elite] (the first |E| valid, feasible
 * elite first, slots as for chap_exchange_plan); local_rank [2][W_local]: for this rank's walkers
 * their position among the rank's own top n_elite best points (row 0) and current points (row 1),
 * -1 if not sent; restart_gid / restart_src [W_total] (the first counts[2] valid); restart_slot
 * [W_local]: the gathered-buffer slot each local walker restarts from, -1 if none. Errors:
 * CHAP_ERR_INVALID_ARG (sizes, rank out of range, NULL pointers), CHAP_ERR_CUDA. */
chap_status chap_exchange_plan_device(int32_t W_total, int32_t W_local, int32_t rank,
                                      const chap_walker_summary* s, int32_t n_elite, int32_t n_restart,
                                      double* z_best, int32_t* counts, int32_t* elite_gid, int32_t* elite_slot,
                                      int32_t* local_rank, int32_t* restart_gid, int32_t* restart_src,
                                      int32_t* restart_slot, void* cuda_stream);

/* One portfolio exchange on existing walkers, the step chap_run_walkers runs every
 * exchange_K iterations: per-walker summaries are all-gathered (NCCL when comm is non-NULL), the
 * plan of chap_exchange_plan is computed on the device, the elite points are all-gathered, every
 * walker's cutoff is tightened to the best incumbent and the planned local walkers
 * restart from elite points (weights kept, tabu cleared), all stream-ordered on cuda_stream. The best
 * incumbent of the gathered walkers: z_best HOST [1] and z_walker HOST [1] (global walker id, -1 if
 * none); when either is non-NULL the call synchronises the stream to return them, when both are
 * NULL it does not. Every rank must call it the same number of times. */
chap_status chap_walkers_exchange(chap_walkers* ws, chap_comm* comm, double* z_best, int32_t* z_walker,
                                  void* cuda_stream);

/* One epoch of the portfolio: n_iters tabu iterations of
 * every walker (chap_tabu_step) followed by one chap_walkers_exchange, launched as ONE CUDA graph:
 * captured on the first call for a given (n_iters, comm) and replayed by later calls, so an epoch
 * costs one graph launch and no host round trip. Same results as chap_tabu_step(n_iters) followed
 * by chap_walkers_exchange. z_best / z_walker as for chap_walkers_exchange (NULL: no
 * synchronisation). Errors: CHAP_ERR_INVALID_ARG (NULL walkers, n_iters < 1, n_elite < 0, comm on
 * another device), CHAP_ERR_CUDA / CHAP_ERR_NCCL from the capture or the launch. */
chap_status chap_walkers_epoch(chap_walkers* ws, chap_comm* comm, int32_t n_iters, double* z_best,
                               int32_t* z_walker, void* cuda_stream);

/* The portfolio loop: W_local walkers from x0 DEVICE [W_local][n] (global
 * walker id = rank*W_local + w), epochs of params.exchange_K iterations; after each epoch an
 * allgather of per-walker summaries and of each rank's elite points (n_elite best incumbents
 * and n_elite least-violated points), a global cutoff z_best - delta for every walker, and a
 * deterministic restart of the n_restart most violated walkers from the global elite.
 * comm = NULL: single GPU, same rule with one rank. Stops after max_iters iterations or when
 * time_limit_s (<= 0: none) has elapsed at an epoch end. best_x DEVICE [n] (or NULL) receives
 * the best incumbent. Synchronises. */
chap_status chap_run_walkers(const chap_problem* p, int32_t W_local, const double* x0,
                             const chap_params* params, chap_comm* comm, int64_t max_iters,
                             double time_limit_s, double* best_x, chap_result* out,
                             void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* CHAP_H */

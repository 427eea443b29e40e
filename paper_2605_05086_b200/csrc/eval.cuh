// eval.cuh — best-shift evaluation (§3.1, Eq. (1) and Algorithm 1) on sm_100a.
//
// Three kernels per pass, each a lean gather loop over its own tile list (the paper's length-
// specialised dispatch, re-designed for sm_100a):
//   k_eval_bin  warp tiles of packed binary columns (flip penalty per nonzero, per-column sum,
//               PAPER.md:295) and warp chunks of long binary columns (atomic partial sums);
//   k_eval_gen  warp tiles of packed general columns (Algorithm 1 per column, sort-free, see
//               gen_tile), empty columns, and warp chunks of long bounded-integer columns whose
//               sort (line 13) becomes a counting pass over [l, u] (atomic bucket deltas);
//   k_eval      block tiles of general columns of <= kGenmMax entries (shared-memory bitonic sort
//               and scan), then the global select: the last block of a walker reduces every
//               block's best admissible move to the walker's decision (R6); not
//               launched when it would only select (the last eval kernel's last block selects).
// A long column's chunks add into its accumulators; the chunk that takes the column's last ticket
// finishes the column and zeroes the accumulators (walker groups' binary chunks: k_eval). With the
// integer weights of R11 every delta, β, α and penalty is a multiple of 1/2 and every partial sum
// is exact, so the order of the atomic additions does not change any result.
// Every warp-tile slot issues its coalesced CSC loads and one 16-byte row-state gather before
// using any of them.
#pragma once
#include <climits>
#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"

namespace chap {

// PAPER.md:277-285 on residuals r0 = ȳ_i - b_i, r1 = y_ij - b_i; satisfied means r <= 0 (R10).
__device__ __forceinline__ double penalty(double w, double r0, double r1) {
  const bool s0 = r0 <= 0.0, s1 = r1 <= 0.0;
  const double half = 0.5 * w;
  const double vio = (r1 < r0) ? half : ((r1 > r0) ? -half : 0.0);   // both violated
  const double from_vio = s1 ? w : vio;
  const double from_sat = s1 ? 0.0 : -w;
  return s0 ? from_sat : from_vio;
}

// penalty(w, r, r + d) / (w / 2) as an integer in {-2, -1, 0, 1, 2} from a row-state record
// (r, w | rc): feasibility before from RowState::rc (r <= 0 <=> ceil(r) <= 0), after from r + d,
// and a row violated on both sides gets less violated iff d < 0. For integer data (DESIGN §5:
// r and d integers, r + d exact; DevProblem::rint_base) w m / 2 equals penalty() exactly; inert
// rows (r = -inf) give 0. With integral weights a column's flip score is (Σ m w) / 2, summed in
// integers.
__device__ __forceinline__ int penalty_m(const double2& rv, double d) {
  const bool z0 = __double2hiint(rv.y) <= 0, z1 = rv.x + d <= 0.0;
  return 2 * ((int)z1 - (int)z0) + ((z0 | z1) ? 0 : (d < 0.0 ? 1 : -1));
}
__device__ __forceinline__ int weight_int(const double2& rv) {
  return __float2int_rn(__int_as_float((int)__double2loint(rv.y)));
}

// Within one variable: higher score, then closer to x̄, then smaller value (R4).
__device__ __forceinline__ bool better_shift(double s1, double v1, double s0, double v0, double xb) {
  if (s1 != s0) return s1 > s0;
  const double d1 = fabs(v1 - xb), d0 = fabs(v0 - xb);
  if (d1 != d0) return d1 < d0;
  return v1 < v0;
}

// Across variables: higher score, then lower user index (R6).
__device__ __forceinline__ bool better_move(double s1, int j1, double s0, int j0) {
  return s1 > s0 || (s1 == s0 && j1 < j0);
}

struct Best {
  double s;
  double v;
  int j;
  int p;
  __device__ __forceinline__ void init() {
    s = -INFINITY;
    v = 0.0;
    j = 0x7fffffff;
    p = -1;
  }
  __device__ __forceinline__ void take(const Best& o) {
    if (better_move(o.s, o.j, s, j)) *this = o;
  }
};

__device__ __forceinline__ Best shfl_best(const Best& b, int off) {
  Best o;
  o.s = __shfl_xor_sync(kFull, b.s, off);
  o.v = __shfl_xor_sync(kFull, b.v, off);
  o.j = __shfl_xor_sync(kFull, b.j, off);
  o.p = __shfl_xor_sync(kFull, b.p, off);
  return o;
}

__device__ __forceinline__ Best warp_reduce_best(Best b) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) b.take(shfl_best(b, off));
  return b;
}

// Block-wide reduce of Best; result valid in thread 0. sm must hold >= 32 entries.
__device__ __forceinline__ Best block_reduce_best(Best b, Best* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  b = warp_reduce_best(b);
  __syncthreads();
  if (lane == 0) sm[wid] = b;
  __syncthreads();
  if (wid == 0) {
    Best o;
    if (lane < nw) o = sm[lane]; else o.init();
    b = warp_reduce_best(o);
  }
  return b;
}

__device__ __forceinline__ void write_part(Cand* dst, const Best& b) {
  Cand c;
  c.s = b.s;
  c.v = b.v;
  c.j = b.j;
  c.p = b.p;
  *dst = c;
}

// Aspiration slots of one walker (R18): a tabu column with s > 0 is noted in slot tabu_until % T
// (the <= T tabu variables have distinct expiries k'+1+T, k' in [k-T, k-1]); a = NULL: off.
// The same reference carries the per-column result cache of selective re-evaluation (f2).
struct AspRef {
  Cand* a = nullptr;
  int T = 1;
  double* cs = nullptr;   // chap_params.lazy: cached (s_j, x̂_j) by internal column
  double* cv = nullptr;
};
__device__ __forceinline__ AspRef asp_ref(const DevWalkers& Wk, int w) {
  AspRef r;
  r.a = Wk.asp ? Wk.asp + (size_t)w * Wk.tenure : nullptr;
  r.T = Wk.tenure > 0 ? Wk.tenure : 1;
  r.cs = Wk.cs;
  r.cv = Wk.cv;
  return r;
}
__device__ __forceinline__ void cache_col(const AspRef& A, int p, double v, double s) {
  if (A.cs) {
    A.cs[p] = s;
    A.cv[p] = v;
  }
}
// f2: does any of the internal columns [p0, p0 + nc) (nc <= 33) need re-evaluation at iteration k?
__device__ __forceinline__ bool cols_dirty(const DevWalkers& Wk, long long k, int p0, int nc) {
  if (!Wk.dirty || nc <= 0) return true;
  const uint32_t* d = Wk.dirty + (size_t)(k & 1) * (Wk.dwords + 1);
  if (__ldcg(d + Wk.dwords)) return true;
  const int p1 = p0 + nc - 1;
  for (int w = p0 >> 5; w <= (p1 >> 5); ++w) {
    uint32_t m = __ldcg(d + w);
    if (w == (p0 >> 5)) m &= ~0u << (p0 & 31);
    if (w == (p1 >> 5)) m &= ~0u >> (31 - (p1 & 31));
    if (m) return true;
  }
  return false;
}
__device__ __forceinline__ void asp_note(const AspRef& A, int p, int j, long long tabu_p, double v, double s) {
  if (!A.a || !(s > 0.0)) return;
  Cand c;
  c.s = s;
  c.v = v;
  c.j = j;
  c.p = p;
  A.a[tabu_p % A.T] = c;
}

// The result of one column: outputs (eval API) and the admissible-best update (R6, R13); a tabu
// column is noted for aspiration (R18).
__device__ __forceinline__ void finish_column_j(int p, int j, int32_t tabu_p, double xb, double v,
                                                double s, Best& b, double* oxhat, double* oscore,
                                                long long k, int use_tabu, AspRef A = AspRef()) {
  if (s == -INFINITY) v = xb;
  if (oxhat) oxhat[j] = v;
  if (oscore) oscore[j] = s;
  cache_col(A, p, v, s);
  if (use_tabu && (long long)tabu_p > k) {
    asp_note(A, p, j, tabu_p, v, s);
    return;
  }
  if (better_move(s, j, b.s, b.j)) {
    b.s = s;
    b.v = v;
    b.j = j;
    b.p = p;
  }
}
__device__ __forceinline__ void finish_column(const DevProblem& P, int p, double xb, double v,
                                              double s, Best& b, double* oxhat, double* oscore,
                                              const int32_t* tabu, long long k, int use_tabu, AspRef A) {
  finish_column_j(p, P.perm[p], use_tabu ? tabu[p] : 0, xb, v, s, b, oxhat, oscore, k, use_tabu, A);
}

// One 16-byte row-state gather (r f64, w f32). The inactive cutoff row holds r = -inf, w = 0,
// which makes every one of its contributions vanish (no per-nonzero test needed).
__device__ __forceinline__ void load_row(const RowView& rs, int i, double& r, double& w) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(rs.p) + (size_t)i * rs.st);
  r = v.x;
  w = (double)__int_as_float((int)__double2loint(v.y));
}

// Entry of Algorithm 1 lines 3-11 for row i of column j, in the one-element-
// per-row form of DESIGN.md §2.3: an a<0 row gives (t, -1, δ); an a>0 row gives (t, +1, δ) whose
// candidate value t is scored by the sum before its +1 entry (= its (t, -1, 0) partner's sigma).
struct Elem {
  double t;
  double delta;
  double beta;
  double alpha;
  int valid;   // an entry is emitted
  int plus;    // marker +1 (a > 0 rows)
};

// Line 3: t = x̄ - r/a. A zero residual (a tight row, common with integer data) gives t = x̄
// exactly; the guard also keeps zero/inf numerators off the IEEE division's slow path.
__device__ __forceinline__ double breakpoint(double xb, double r, double a) {
  const bool plain = r != 0.0 && isfinite(r);
  const double q = (plain ? r : 1.0) / a;
  return plain ? xb - q : xb;
}

__device__ __forceinline__ Elem emit(double xb, double r, double a, double w, int is_int) {
  Elem e;
  e.beta = 0.0;
  e.alpha = 0.0;
  e.valid = 0;
  e.plus = 0;
  e.delta = 0.0;
  e.t = xb;
  if (!isfinite(r)) return e;                       // the inert inactive cutoff row (w = 0)
  double t = breakpoint(xb, r, a);                   // (b_i - Σ_{k≠j} a_ik x̄_k) / a_ij  (l.3)
  if (is_int) t = (a > 0.0) ? floor(t) : ceil(t);    // l.4
  e.t = t;
  if (a < 0.0) {                                      // imposes x_j >= t (l.5)
    if (xb < t) {
      e.beta = -0.5 * w; e.alpha = w; e.valid = 1; e.delta = 0.5 * w;
    } else if (xb > t) {
      e.beta = -w; e.valid = 1; e.delta = w;
    } else {
      e.beta = -w; e.alpha = w;
    }
  } else {                                            // imposes x_j <= t (l.8)
    if (xb > t) {
      e.beta = w; e.alpha = -w; e.valid = 1; e.plus = 1; e.delta = -0.5 * w;
    } else if (xb < t) {
      e.valid = 1; e.plus = 1; e.delta = -w;
    } else {
      e.alpha = -w;
    }
  }
  return e;
}

// ------------------------------------------------------------------------------------------
// shared memory
// ------------------------------------------------------------------------------------------
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
struct SmemGenM {                      // CC_GENM block tile
  double t[kGenmMax];
  double del[kGenmMax];
  double P[kGenmMax];
  uint32_t mk[kGenmMax];
};
constexpr size_t kTileSmem = sizeof(SmemGenM);

struct TileCtx {
  const double* x;
  RowView rs;
  const int32_t* tabu;
  long long k;
  int use_tabu;
  double* oxhat;
  double* oscore;
  AspRef asp;
};

// ------------------------------------------------------------------------------------------
// warp tiles
// ------------------------------------------------------------------------------------------

// Entry flags of a general warp tile. Lines 5-11 of Algorithm 1 are fixed by
// the sign of a_ij and the order of x̄ and t: with w = w_i,
//   a<0, x̄<t: δ=+w/2, β-=w/2, α+=w   a<0, x̄>t: δ=+w, β-=w          a<0, x̄=t: β-=w, α+=w
//   a>0, x̄>t: δ=-w/2, β+=w, α-=w     a>0, x̄<t: δ=-w                 a>0, x̄=t: α-=w
// (an a>0 entry's (t,-1,0) partner carries no delta; R3 makes t a candidate all the same).
enum : uint8_t {
  GF_POS = 1,      // a > 0
  GF_LT = 2,       // x̄ < t
  GF_GT = 4,       // x̄ > t
  GF_ROW = 8,      // a row entry
  GF_CAND = 32,    // the value is a candidate: finite, in [l, u], != x̄ (R2, R5)
};
__device__ __forceinline__ void gf_coeffs(uint8_t f, double w, double& D, double& A, double& B) {
  const bool pos = f & GF_POS, lt = f & GF_LT, gt = f & GF_GT, row = f & GF_ROW;
  const double hw = 0.5 * w;
  const double Dn = lt ? hw : (gt ? w : 0.0), An = lt ? -hw : -w, Bn = gt ? 0.0 : w;
  const double Dp = gt ? -hw : (lt ? -w : 0.0), Ap = gt ? w : 0.0, Bp = lt ? 0.0 : -w;
  D = row ? (pos ? Dp : Dn) : 0.0;
  A = row ? (pos ? Ap : An) : 0.0;
  B = row ? (pos ? Bp : Bn) : 0.0;
}

// Columns without nonzeros: a binary flips with score 0; another variable's candidates are its
// finite bounds other than x̄, all scoring 0 (R2, R4, R5); none -> (x̄, -inf).
__device__ __forceinline__ void wtile_empty(const DevProblem& P, const TileCtx& C, const WTile& T,
                                            int lane, Best& b) {
  if (lane >= T.ncols) return;
  const int p = T.p0 + lane;
  const int j = __ldg(P.perm + p);
  const int tb = C.use_tabu ? __ldg(C.tabu + p) : 0;
  const double xb = __ldg(C.x + p);
  const double l = __ldg(P.lb + p), u = __ldg(P.ub + p);
  double bs = -INFINITY, bv = xb;
  if (__ldg(P.vclass + p) == 1) {
    bs = 0.0;
    bv = 1.0 - xb;
  } else {
    if (isfinite(l) && l != xb) { bs = 0.0; bv = l; }
    if (isfinite(u) && u != xb && better_shift(0.0, u, bs, bv, xb)) { bs = 0.0; bv = u; }
  }
  finish_column_j(p, j, tb, xb, bv, bs, b, C.oxhat, C.oscore, C.k, C.use_tabu, C.asp);
}

// ------------------------------------------------------------------------------------------
// block tiles
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ double block_sum(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  double r = 0.0;
  for (int q = 0; q < nw; ++q) r += sm[q];   // fixed order, every thread
  __syncthreads();
  return r;
}

// In-place inclusive scan of a[0..L) by a block (contiguous segment per thread, fixed order).
__device__ void block_scan_inclusive(double* a, int L, double* sm) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int seg = (L + T - 1) / T;
  const int s0 = tid * seg, s1 = min(L, s0 + seg);
  double run = 0.0;
  for (int q = s0; q < s1; ++q) { run += a[q]; a[q] = run; }
  const int lane = tid & 31, wid = tid >> 5;
  double incl = run;
  for (int off = 1; off < 32; off <<= 1) {
    const double y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  __syncthreads();
  if (lane == 31) sm[wid] = incl;
  __syncthreads();
  double woff = 0.0;
  for (int q = 0; q < wid; ++q) woff += sm[q];
  const double off = woff + incl - run;
  for (int q = s0; q < s1; ++q) a[q] += off;
  __syncthreads();
}

// block-wide argmax of (score, value) within one variable (R4); result in thread 0
__device__ __forceinline__ void block_best_shift(double& bs, double& bv, double xb, Best* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    const double so = __shfl_xor_sync(kFull, bs, off), vo = __shfl_xor_sync(kFull, bv, off);
    if (better_shift(so, vo, bs, bv, xb)) { bs = so; bv = vo; }
  }
  __syncthreads();
  if (lane == 0) { sm[wid].s = bs; sm[wid].v = bv; }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (better_shift(sm[q].s, sm[q].v, bs, bv, xb)) { bs = sm[q].s; bv = sm[q].v; }
  __syncthreads();
}

// one general column in one tile: bitonic sort of (value, marker) pairs (l.13), block scan (l.14)
__device__ __forceinline__ void tile_genm(const DevProblem& P, const TileCtx& C, const Tile& T,
                                          SmemGenM& S, double* sm_red, Best* sm_b, Best& b) {
  const int tid = threadIdx.x;
  const int p = T.p0;
  const int beg = P.col_ptr[p], d = P.col_ptr[p + 1] - beg;
  const double xb = C.x[p], l = P.lb[p], u = P.ub[p];
  const int is_int = P.vclass[p] != 3;
  int Lp = 1;
  while (Lp < d + 2) Lp <<= 1;
  double beta = 0.0, alpha = 0.0;
  for (int e = tid; e < Lp; e += blockDim.x) {
    double t = INFINITY, del = 0.0;
    uint32_t mk = 0xffffffffu;
    if (e < d) {
      double r, w;
      load_row(C.rs, P.row_idx[beg + e], r, w);
      const Elem el = emit(xb, r, P.val[beg + e], w, is_int);
      beta += el.beta;
      alpha += el.alpha;
      if (el.valid && isfinite(el.t)) {
        const bool cand = el.t >= l && el.t <= u && el.t != xb;
        t = el.t;
        del = el.delta;
        mk = ((uint32_t)el.plus << 31) | ((uint32_t)cand << 30) | (uint32_t)e;
      }
    } else if (e == d) {
      if (isfinite(l)) { t = l; mk = ((uint32_t)(l != xb) << 30) | (uint32_t)e; }
    } else if (e == d + 1) {
      if (isfinite(u)) { t = u; mk = ((uint32_t)(u != xb) << 30) | (uint32_t)e; }
    }
    S.t[e] = t;
    S.mk[e] = mk;
    S.del[e] = del;
  }
  beta = block_sum(beta, sm_red);
  alpha = block_sum(alpha, sm_red);
  for (int size = 2; size <= Lp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int q = tid; q < (Lp >> 1); q += blockDim.x) {
        const int lo = 2 * q - (q & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const double t0 = S.t[lo], t1 = S.t[hi];
        const uint32_t m0 = S.mk[lo], m1 = S.mk[hi];
        const bool gt = (t0 > t1) || (t0 == t1 && m0 > m1);
        if (gt == asc) {
          S.t[lo] = t1; S.t[hi] = t0;
          S.mk[lo] = m1; S.mk[hi] = m0;
        }
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = S.mk[q];
    S.P[q] = (mk == 0xffffffffu) ? 0.0 : S.del[mk & 0x3fffffffu];
  }
  __syncthreads();
  block_scan_inclusive(S.P, Lp, sm_red);
  double bs = -INFINITY, bv = xb;
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = S.mk[q];
    if (mk == 0xffffffffu || !((mk >> 30) & 1u)) continue;
    const double t = S.t[q];
    const double pre = (mk >> 31) ? (q > 0 ? S.P[q - 1] : 0.0) : S.P[q];
    const double sig = beta + pre + (t > xb ? alpha : 0.0);
    if (better_shift(sig, t, bs, bv, xb)) { bs = sig; bv = t; }
  }
  block_best_shift(bs, bv, xb, sm_b);
  if (tid == 0) finish_column(P, p, xb, bv, bs, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu, C.asp);
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// grid-wide sort of long general columns (CC_GENL)
// ------------------------------------------------------------------------------------------
// k_sort_chunks: one block per chunk and walker. Lines 3-11 per entry (emit) as in tile_genm, the
// chunk's (value, marker) pairs sorted by a shared-memory bitonic network, the inclusive prefix P of
// the deltas in sorted order (line 14 within the chunk), written to walker scratch with the keys and
// the chunk's parts of β and α. The sort key is (t, +1 marker, candidate flag, chunk << 11 | slot):
// a total order in which every (t, -1) entry precedes every (t, +1) entry (line 13, R3).
__global__ void __launch_bounds__(kTileThreads) k_sort_chunks(DevProblem P, DevWalkers Wk) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sm_red[32];
  SmemGenM& S = *reinterpret_cast<SmemGenM*>(smem);
  const int walker = blockIdx.y, tid = threadIdx.x;
  const Tile T = P.schunks[blockIdx.x];
  const int p = T.p0, ch = T.ncols, d = T.e1 - T.e0;
  if (!cols_dirty(Wk, Wk.sc[walker].k, p, 1)) return;   // f2: a clean column keeps its cached result
  const double* X = Wk.x + (size_t)walker * Wk.xs;
  const RowView rs = row_view(Wk, walker);
  const double xb = X[p], l = P.lb[p], u = P.ub[p];
  const int is_int = P.vclass[p] != 3;
  const int nb = ch == 0 ? 2 : 0;   // the bounds ride in chunk 0
  int Lp = 1;
  while (Lp < d + nb) Lp <<= 1;
  const uint32_t tag = (uint32_t)ch << 11;
  double beta = 0.0, alpha = 0.0;
  for (int e = tid; e < Lp; e += blockDim.x) {
    double t = INFINITY, del = 0.0;
    uint32_t mk = 0xffffffffu;
    if (e < d) {
      double r, w;
      load_row(rs, P.row_idx[T.e0 + e], r, w);
      const Elem el = emit(xb, r, P.val[T.e0 + e], w, is_int);
      beta += el.beta;
      alpha += el.alpha;
      if (el.valid && isfinite(el.t)) {
        const bool cand = el.t >= l && el.t <= u && el.t != xb;
        t = el.t;
        del = el.delta;
        mk = ((uint32_t)el.plus << 31) | ((uint32_t)cand << 30) | tag | (uint32_t)e;
      }
    } else if (e < d + nb) {
      const double bv = e == d ? l : u;
      if (isfinite(bv)) { t = bv; mk = ((uint32_t)(bv != xb) << 30) | tag | (uint32_t)e; }
    }
    S.t[e] = t;
    S.mk[e] = mk;
    S.del[e] = del;
  }
  beta = block_sum(beta, sm_red);
  alpha = block_sum(alpha, sm_red);
  for (int size = 2; size <= Lp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int q = tid; q < (Lp >> 1); q += blockDim.x) {
        const int lo = 2 * q - (q & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const double t0 = S.t[lo], t1 = S.t[hi];
        const uint32_t m0 = S.mk[lo], m1 = S.mk[hi];
        const bool gt = (t0 > t1) || (t0 == t1 && m0 > m1);
        if (gt == asc) {
          S.t[lo] = t1; S.t[hi] = t0;
          S.mk[lo] = m1; S.mk[hi] = m0;
        }
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = S.mk[q];
    S.P[q] = (mk == 0xffffffffu) ? 0.0 : S.del[mk & 0x7ffu];
  }
  __syncthreads();
  block_scan_inclusive(S.P, Lp, sm_red);
  // write the chunk (valid entries sort first: the others carry t = +inf and the largest key)
  const SortCol C = P.scols[T.pad];
  double* base = Wk.lscr + (size_t)walker * Wk.lss + C.scr + (size_t)ch * kSortStride;
  double* gt = base;
  double* gP = base + kGenmMax;
  uint32_t* gmk = reinterpret_cast<uint32_t*>(base + 2 * kGenmMax);
  double* meta = base + 2 * kGenmMax + kGenmMax / 2;
  int nv = 0;
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = S.mk[q];
    if (mk == 0xffffffffu) continue;
    gt[q] = S.t[q];
    gP[q] = S.P[q];
    gmk[q] = mk;
    ++nv;
  }
  nv = (int)block_sum((double)nv, sm_red);
  if (tid == 0) {
    meta[0] = (double)nv;
    meta[1] = beta;
    meta[2] = alpha;
  }
}

// k_sort_rank: one block per chunk and walker. Every candidate entry of the chunk (R2, R3, R5) gets
// its σ of line 15 from the global prefix of line 14: its own chunk's prefix (through a -1 entry,
// strictly before a +1 entry) plus, for every other chunk of the column, the prefix of the entries
// that precede it in the total order (binary search, co-ranking); β and α are the sums of the chunks'
// parts. The chunk's best (σ, value) under R4 goes to its scratch; k_eval takes the column's best.
__global__ void __launch_bounds__(kTileThreads) k_sort_rank(DevProblem P, DevWalkers Wk) {
  __shared__ Best sm_b[32];
  __shared__ double s_ba[2];
  const int walker = blockIdx.y, tid = threadIdx.x;
  const Tile T = P.schunks[blockIdx.x];
  const int p = T.p0, ch = T.ncols;
  if (!cols_dirty(Wk, Wk.sc[walker].k, p, 1)) return;
  const SortCol C = P.scols[T.pad];
  const double* X = Wk.x + (size_t)walker * Wk.xs;
  const double xb = X[p];
  double* col = Wk.lscr + (size_t)walker * Wk.lss + C.scr;
  auto chunk = [&](int c) { return col + (size_t)c * kSortStride; };
  constexpr int kMeta = 2 * kGenmMax + kGenmMax / 2;
  if (tid == 0) {
    double B = 0.0, A = 0.0;
    for (int c = 0; c < C.nchunks; ++c) {
      B += __ldcg(chunk(c) + kMeta + 1);
      A += __ldcg(chunk(c) + kMeta + 2);
    }
    s_ba[0] = B;
    s_ba[1] = A;
  }
  __syncthreads();
  const double B = s_ba[0], A = s_ba[1];
  const double* me = chunk(ch);
  const int n = (int)__ldcg(me + kMeta);
  const uint32_t* mmk = reinterpret_cast<const uint32_t*>(me + 2 * kGenmMax);
  double bs = -INFINITY, bv = xb;
  for (int q = tid; q < n; q += blockDim.x) {
    const uint32_t mk = __ldcg(mmk + q);
    if (!((mk >> 30) & 1u)) continue;
    const double t = __ldcg(me + q);
    const bool plus = mk >> 31;
    double pre = plus ? (q > 0 ? __ldcg(me + kGenmMax + q - 1) : 0.0) : __ldcg(me + kGenmMax + q);
    for (int c = 0; c < C.nchunks; ++c) {
      if (c == ch) continue;
      const double* o = chunk(c);
      const uint32_t* omk = reinterpret_cast<const uint32_t*>(o + 2 * kGenmMax);
      int lo = 0, hi = (int)__ldcg(o + kMeta);   // count of entries before (t, mk): first not-less
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const double tm = __ldcg(o + mid);
        const bool less = tm < t || (tm == t && __ldcg(omk + mid) < mk);
        if (less) lo = mid + 1; else hi = mid;
      }
      if (lo > 0) pre += __ldcg(o + kGenmMax + lo - 1);
    }
    const double sig = B + pre + (t > xb ? A : 0.0);
    if (better_shift(sig, t, bs, bv, xb)) { bs = sig; bv = t; }
  }
  block_best_shift(bs, bv, xb, sm_b);
  if (tid == 0) {
    double* meta = const_cast<double*>(me) + kMeta;
    meta[3] = bs;
    meta[4] = bv;
  }
}

// The column's result from its chunks' bests (R4), in k_eval after k_sort_rank.
__device__ __forceinline__ void sortcol_finish(const DevProblem& P, const DevWalkers& Wk, int walker, const SortCol& C,
                                               Best& b, double* oxhat, double* oscore, long long kk, int use_tabu) {
  const double* col = Wk.lscr + (size_t)walker * Wk.lss + C.scr;
  const double xb = Wk.x[(size_t)walker * Wk.xs + C.p];
  constexpr int kMeta = 2 * kGenmMax + kGenmMax / 2;
  double bs = -INFINITY, bv = xb;
  for (int c = 0; c < C.nchunks; ++c) {
    const double s = __ldcg(col + (size_t)c * kSortStride + kMeta + 3), v = __ldcg(col + (size_t)c * kSortStride + kMeta + 4);
    if (s > -INFINITY && better_shift(s, v, bs, bv, xb)) { bs = s; bv = v; }
  }
  finish_column_j(C.p, P.perm[C.p], use_tabu ? Wk.tabu[(size_t)walker * Wk.ts + C.p] : 0, xb, bv, bs, b, oxhat, oscore,
                  kk, use_tabu, asp_ref(Wk, walker));
}

// last-block handshake (the global select): returns true in every thread of the last block
__device__ __forceinline__ bool last_chunk(unsigned* cnt, int nchunks, int* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_flag = (atomicAdd(cnt, 1u) == (unsigned)(nchunks - 1));
  }
  __syncthreads();
  const bool last = *s_flag != 0;
  if (last) __threadfence();
  return last;
}

// The global select (R6), run by the last block of a walker's final eval kernel: the
// best admissible move over the walker's nparts block parts, written as the walker's decision (and
// to best_out for the eval API).
__device__ __forceinline__ void select_walker(const DevProblem& P, const DevWalkers& Wk, int walker, int nparts,
                                              Best* sm_b, chap_move* best_out, const double* x) {
  const Cand* part = Wk.part + (size_t)walker * Wk.ps;
  Best g;
  g.init();
  for (int q = threadIdx.x; q < nparts; q += blockDim.x) {
    Best o;
    o.s = __ldcg(&part[q].s);
    o.v = __ldcg(&part[q].v);
    o.j = __ldcg(&part[q].j);
    o.p = __ldcg(&part[q].p);
    g.take(o);
  }
  g = block_reduce_best(g, sm_b);
  if (Wk.asp) {   // incumbent aspiration (R18): a noted tabu move that beats the best admissible one
                  // is taken if no active row stays violated after it (violated + Δ == 0)
    __shared__ Best s_g;
    __shared__ Cand s_c;
    __shared__ int s_ok;
    __shared__ double s_red[32];
    if (threadIdx.x == 0) s_g = g;
    const int T = Wk.tenure > 0 ? Wk.tenure : 1;
    Cand* slots = Wk.asp + (size_t)walker * Wk.tenure;
    const long long k = Wk.sc[walker].k;
    const RowView rv = row_view(Wk, walker);
    for (int q = 0; q < T; ++q) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const Cand c = slots[q];
        bool ok = c.p >= 0 && c.s > 0.0 && better_move(c.s, c.j, s_g.s, s_g.j);
        if (ok) {
          const long long tp = Wk.tabu[(size_t)walker * Wk.ts + c.p];
          ok = tp > k && tp % T == q;
        }
        s_c = c;
        s_ok = ok;
        slots[q].p = -1;   // consumed: the next pass notes afresh
      }
      __syncthreads();
      if (!s_ok) continue;
      const Cand c = s_c;
      const double d = c.v - x[c.p];
      double dv = 0.0;
      for (int e = P.col_ptr[c.p] + threadIdx.x; e < P.col_ptr[c.p + 1]; e += blockDim.x) {
        const double r0 = rv[P.row_idx[e]].r;   // the inert rows (inactive cutoff, padding): -inf
        if (r0 == -INFINITY) continue;
        const double r1 = r0 + P.val[e] * d;
        dv += (double)(r1 > 0.0) - (double)(r0 > 0.0);
      }
      dv = block_sum(dv, s_red);
      if (threadIdx.x == 0 && (double)Wk.sc[walker].violated + dv == 0.0) {
        s_g.s = c.s;
        s_g.v = c.v;
        s_g.j = c.j;
        s_g.p = c.p;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) g = s_g;
  }
  if (threadIdx.x == 0) {
    WalkerScalars* scw = Wk.sc + walker;
    const bool found = g.p >= 0;
    Decision d;
    d.move = (found && g.s > 0.0) ? 1 : 0;
    d.p = g.p;
    d.j = found ? g.j : -1;
    d.pad = 0;
    d.v = g.v;
    d.s = found ? g.s : -INFINITY;
    d.delta = d.move ? (g.v - x[g.p]) : 0.0;
    if (scw->force_p >= 0) {   // the perturbation drawn by the previous (stuck) iteration (R21)
      d.move = 1;
      d.p = scw->force_p;
      d.j = P.perm[d.p];
      d.pad = 1;
      d.v = scw->force_v;
      d.s = NAN;
      d.delta = d.v - x[d.p];
      scw->force_p = -1;
    }
    scw->dec = d;
    if (best_out) {
      chap_move mv;
      mv.j = d.move ? d.j : -1;
      mv.pad = 0;
      mv.v = d.move ? d.v : NAN;
      mv.s = d.move ? d.s : -INFINITY;
      best_out[walker] = mv;
    }
    Wk.sel_count[walker] = 0u;
  }
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------

// ------------------------------------------------------------------------------------------
// binary kernel
// ------------------------------------------------------------------------------------------
// k_eval_bin evaluates the packed binary columns (flip scores). It is built like a
// plain gather loop so that many warps per SM keep their loads in flight: per warp tile (whole
// columns, <= kBinTile nonzeros, <= 32 columns, starting on a multiple of 4 nonzeros) lane l owns
// slots 4l..4l+3: one 16-byte index load, two 16-byte value loads and four 16-byte row-state
// gathers, all issued back to back. The column of a slot comes from the tile's 128-bit head mask
// (redux.sync), x̄ of the column from a ballot (binaries are 0/1); column sums are a segmented
// scan (in-lane, then a 5-step shuffle scan across lanes), so shared memory only carries the 32
// finished sums — every random access of the kernel is the row-state gather itself.
// A chunk of a long binary column (one column, <= kWChunk nonzeros) sums by a warp reduction and
// adds its partial to the column's accumulator; k_eval finishes the column.
struct __align__(16) BinWarp {
  double cs[32];   // column sums
};
constexpr size_t kBinSmem = sizeof(BinWarp) * (kBinThreads / 32);

// The chunk ticket of a long column: every lane's accumulator additions are made visible, then lane 0
// takes a ticket; true (in every lane) for the chunk that takes the column's last one, which then
// sees every other chunk's additions (fences on both sides) and finishes the column.
#ifndef CHAP_TICKET
#define CHAP_TICKET 1
#endif
__device__ __forceinline__ bool long_last(const DevWalkers& Wk, int walker, const LongCol& L, int lane) {
#if CHAP_TICKET == 0
  __threadfence();
#endif
  __syncwarp();
  unsigned last = 0u;
  if (lane == 0) {
    unsigned* tk = reinterpret_cast<unsigned*>(Wk.lscr + (size_t)walker * Wk.lss + L.tix);
#if CHAP_TICKET == 0
    last = atomicAdd(tk, 1u) == (unsigned)(L.nchunks - 1);
#else
    // acquire-release at gpu scope: the warp's additions (ordered before by the warp barrier) are
    // released with the ticket; the last taker acquires every earlier chunk's additions
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(tk) : "memory");
    last = old == (unsigned)(L.nchunks - 1);
#endif
    if (last) *tk = 0u;
  }
  last = __shfl_sync(kFull, last, 0);
#if CHAP_TICKET == 0
  if (last) __threadfence();
#endif
  return last != 0u;
}

// The end of a long binary column of several chunks: the summed flip score.
__device__ __forceinline__ void lbin_finalize(const DevProblem& P, const DevWalkers& Wk, int walker,
                                              const LongCol& L, Best& b, double* oxhat, double* oscore,
                                              long long kk, int use_tabu) {
  const int p = L.p;
  double* acc = Wk.lscr + (size_t)walker * Wk.lss + L.scr;
  const double s = __ldcg(acc);
  *acc = 0.0;
  const double xb = __ldg(Wk.x + (size_t)walker * Wk.xs + p);
  finish_column_j(p, __ldg(P.perm + p), use_tabu ? __ldg(Wk.tabu + (size_t)walker * Wk.ts + p) : 0, xb,
                  1.0 - xb, s, b, oxhat, oscore, kk, use_tabu, asp_ref(Wk, walker));
}

// A warp chunk (<= kWChunk nonzeros) of a long binary column: warp-reduced flip sum added to the
// column's accumulator (a single-chunk column finishes in place); the chunk that takes the column's
// last ticket finishes it.
__device__ __forceinline__ void lbin_chunk(const DevProblem& P, const DevWalkers& Wk, int walker,
                                           const double* __restrict__ X, const double2* __restrict__ RS,
                                           const int32_t* __restrict__ TB, const WTile& T, int lane,
                                           Best& b, double* oxhat, double* oscore, long long kk,
                                           int use_tabu, bool wint) {
  const int p = T.p0, len = T.ncols;
  const int* __restrict__ ridx = P.row_idx + T.e0;
  const double* __restrict__ rval = P.val + T.e0;
  const double xb = __ldg(X + p);
  const double dir = 1.0 - 2.0 * xb;
  int id[kWChunk / 32];
  double av[kWChunk / 32];
#pragma unroll
  for (int q = 0; q < kWChunk / 32; ++q) {
    const int k = lane + 32 * q;
    id[q] = k < len ? __ldcs(ridx + k) : P.dummy_row;
    av[q] = k < len ? __ldcs(rval + k) : 0.0;
  }
  double own = 0.0;
  if (wint) {   // integer data, integral weights: (Σ m w) / 2 in integers (penalty_m)
    int own2 = 0;
#pragma unroll
    for (int q = 0; q < kWChunk / 32; ++q) {
      const double2 rv = __ldg(RS + id[q]);
      own2 += penalty_m(rv, av[q] * dir) * weight_int(rv);   // the inert dummy row adds 0
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) own2 += __shfl_xor_sync(kFull, own2, off);
    own = 0.5 * (double)own2;
  } else {
#pragma unroll
    for (int q = 0; q < kWChunk / 32; ++q) {
      const double2 rv = __ldg(RS + id[q]);
      const double r = rv.x, w = (double)__int_as_float((int)__double2loint(rv.y));
      own += penalty(w, r, r + av[q] * dir);   // the inert dummy row adds 0
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) own += __shfl_xor_sync(kFull, own, off);
  }
  const LongCol L = P.lcols[T.e1];
  if (L.nchunks == 1) {
    if (lane == 0)
      finish_column_j(p, __ldg(P.perm + p), use_tabu ? __ldg(TB + p) : 0, xb, 1.0 - xb, own, b, oxhat,
                      oscore, kk, use_tabu, asp_ref(Wk, walker));
    return;
  }
  if (lane == 0) atomicAdd(Wk.lscr + (size_t)walker * Wk.lss + L.scr, own);
  if (long_last(Wk, walker, L, lane) && lane == 0) lbin_finalize(P, Wk, walker, L, b, oxhat, oscore, kk, use_tabu);
}

// select_parts > 0: this is the walker's only and last eval kernel and k_eval has nothing but the
// select to do (no long columns, no sort tiles): the last block to finish selects over
// select_parts block parts and k_eval is not launched.
__global__ void __launch_bounds__(kBinThreads, kBinMinBlocks) k_eval_bin(DevProblem P, DevWalkers Wk, double* oxhat,
                                                              double* oscore, int select_parts, chap_move* best_out) {
  pdl_wait_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Best sm_b[32];
  const int walker = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const WalkerScalars* sc = Wk.sc + walker;
  const double* __restrict__ X = Wk.x + (size_t)walker * Wk.xs;
  // walker-major row state (rg = 1): the walker-minor layout runs k_eval_bin_wm instead
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(row_view(Wk, walker).p);
  const int32_t* __restrict__ TB = Wk.tabu + (size_t)walker * Wk.ts;
  const long long kk = sc->k;
  const int use_tabu = Wk.use_tabu;
  double* cs = reinterpret_cast<BinWarp*>(smem)[wid].cs;
  KT_BEGIN(Wk, 0);
  Best b;
  b.init();
  const int nwarps = gridDim.x * (kBinThreads / 32);
  int t = blockIdx.x * (kBinThreads / 32) + wid;
  // chunks of long columns first (their latency overlaps the packed tiles of other warps)
  for (; t < P.n_bchunks; t += nwarps)
    if (cols_dirty(Wk, kk, P.bchunks[t].p0, 1))
      lbin_chunk(P, Wk, walker, X, RS, TB, P.bchunks[t], lane, b, oxhat, oscore, kk, use_tabu,
                 P.rint_base && sc->wint != 0);
  t -= P.n_bchunks;
  const int hwi = lane >> 3, sh = 4 * (lane & 7);   // head word and bit offset of my 4 slots
  const bool intp = P.rint_base && sc->wint != 0;    // integer data, integral weights <= 2^20
  WTile Tn;
  if (t < P.n_btiles) Tn = P.btiles[t];
  for (; t < P.n_btiles; t += nwarps) {
    const WTile T = Tn;
    if (t + nwarps < P.n_btiles) Tn = P.btiles[t + nwarps];
    if (!cols_dirty(Wk, kk, T.p0, T.ncols)) continue;   // f2
    const int nc = T.ncols, len = T.e1 - T.e0;
    // slots 4 lane .. 4 lane + 3: one 16-byte index load, two 16-byte value loads
    const bool act = 4 * lane < len;
    int4 id = make_int4(P.dummy_row, P.dummy_row, P.dummy_row, P.dummy_row);
    double2 a01 = make_double2(0.0, 0.0), a23 = a01;
    if (act) {
      id = __ldcs(reinterpret_cast<const int4*>(P.row_idx + T.e0) + lane);
      a01 = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0) + 2 * lane);
      a23 = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0) + 2 * lane + 1);
    }
    // column data of lane c
    const int p = T.p0 + lane;
    int cb = 0x7fffffff, j = 0, tb = 0;
    double xb = 0.0;
    if (lane < nc) {
      cb = __ldg(P.col_ptr + p) - T.e0;
      j = __ldg(P.perm + p);
      tb = use_tabu ? __ldg(TB + p) : 0;
      xb = __ldg(X + p);
    }
    double2 rv[4];
    rv[0] = __ldg(RS + id.x);
    rv[1] = __ldg(RS + id.y);
    rv[2] = __ldg(RS + id.z);
    rv[3] = __ldg(RS + id.w);
    // column heads of the 128 slots (4 words) and x̄ of every column (one bit each)
    const unsigned h0 = __reduce_or_sync(kFull, (cb >> 5) == 0 ? (1u << (cb & 31)) : 0u);
    const unsigned h1 = __reduce_or_sync(kFull, (cb >> 5) == 1 ? (1u << (cb & 31)) : 0u);
    const unsigned h2 = __reduce_or_sync(kFull, (cb >> 5) == 2 ? (1u << (cb & 31)) : 0u);
    const unsigned h3 = __reduce_or_sync(kFull, (cb >> 5) == 3 ? (1u << (cb & 31)) : 0u);
    const unsigned xm = __ballot_sync(kFull, xb != 0.0);
    const unsigned hw = hwi == 0 ? h0 : (hwi == 1 ? h1 : (hwi == 2 ? h2 : h3));
    const unsigned hnext = hwi == 0 ? h1 : (hwi == 1 ? h2 : (hwi == 2 ? h3 : 1u));
    const int base = (hwi > 0 ? __popc(h0) : 0) + (hwi > 1 ? __popc(h1) : 0) + (hwi > 2 ? __popc(h2) : 0) - 1;
    const unsigned hb = (hw >> sh) & 0xFu;                      // heads among my slots
    const unsigned hn = (lane & 7) == 7 ? (hnext & 1u) : ((hw >> (sh + 4)) & 1u);   // head after them
    // flip penalties and the within-lane segmented prefix; with integer data and
    // integral weights in integers, in half weights (penalty_m), else in double
    int cq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cq[q] = base + __popc(hw & ((2u << (sh + q)) - 1u));
    auto column_sums = [&](auto zero) {
      using Acc = decltype(zero);
      Acc sq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double a = q == 0 ? a01.x : (q == 1 ? a01.y : (q == 2 ? a23.x : a23.y));
        const double d = a * (1.0 - 2.0 * (double)((xm >> (cq[q] & 31)) & 1u));
        Acc pk;
        if constexpr (std::is_same<Acc, int>::value) {
          pk = penalty_m(rv[q], d) * weight_int(rv[q]);   // inert rows: 0
        } else {
          const double r = rv[q].x, w = (double)__int_as_float((int)__double2loint(rv[q].y));
          pk = penalty(w, r, r + d);   // inert rows: 0
        }
        sq[q] = (q == 0 || ((hb >> q) & 1u)) ? pk : sq[q - 1] + pk;
      }
      // columns crossing lanes: segmented scan of the lanes' last runs
      Acc v = sq[3];
      bool f = hb != 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const Acc y = __shfl_up_sync(kFull, v, off);
        const bool g = __shfl_up_sync(kFull, f, off);
        if (lane >= off) {
          if (!f) v += y;
          f = f || g;
        }
      }
      Acc carry = __shfl_up_sync(kFull, v, 1);
      if (lane == 0 || (hb & 1u)) carry = 0;
      // a slot that ends its column publishes the column's sum
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool cont = (hb & ((2u << q) - 1u)) == 0u;          // no head in slots 0..q: continues
        const Acc tot = sq[q] + (cont ? carry : (Acc)0);
        const bool end = (q < 3) ? (((hb >> (q + 1)) & 1u) != 0u) : (hn != 0u);
        const int k = 4 * lane + q;
        if (k < len && (end || k == len - 1))
          cs[cq[q]] = std::is_same<Acc, int>::value ? 0.5 * (double)tot : (double)tot;
      }
    };
    if (intp) column_sums(0); else column_sums(0.0);
    __syncwarp();
    if (lane < nc) finish_column_j(p, j, tb, xb, 1.0 - xb, cs[lane], b, oxhat, oscore, kk, use_tabu, asp_ref(Wk, walker));
    __syncwarp();
  }
  b = block_reduce_best(b, sm_b);
  if (threadIdx.x == 0) write_part(Wk.part + (size_t)walker * Wk.ps + blockIdx.x, b);
  KT_END(Wk, 0);
  if (select_parts <= 0) return;
  __shared__ int s_flag;
  if (!last_chunk(Wk.sel_count + walker, gridDim.x, &s_flag)) return;
  select_walker(P, Wk, walker, select_parts, sm_b, best_out, X);
  KT_END(Wk, 0);
}

// ------------------------------------------------------------------------------------------
// walker-minor binary kernel (row-state groups of rg > 1 walkers): one lane per walker
// ------------------------------------------------------------------------------------------
// With the row state of a group of RG walkers interleaved (DevWalkers), the RG records of one row
// are one contiguous run, so one warp evaluates a binary column for the whole group: lane =
// (slot, walker) = (lane / RG, lane % RG), the 32 / RG slots split the column's nonzeros, the CSC
// entries are read once per group and broadcast, and every row-state gather is a coalesced
// RG x 16-byte run instead of RG scattered sectors. x̄ comes from the group's
// bitset word of the column. The flip penalty per nonzero and the column sum are
// those of k_eval_bin; the sum over slots is a fixed shuffle tree of exact
// half-integer partials (R11), so the scores are bit-identical to the walker-major kernel's.
// A chunk of a long binary column adds each walker's partial to that walker's accumulator;
// k_eval finishes the column.
#ifndef CHAP_BINWM_THREADS
#define CHAP_BINWM_THREADS 256
#endif
constexpr int kBinWmThreads = CHAP_BINWM_THREADS;
struct BinWmWarp {
  int id[kBinTile];
  double a[kBinTile];
};

template <int RG>
__global__ void __launch_bounds__(kBinWmThreads) k_eval_bin_wm(DevProblem P, DevWalkers Wk) {
  pdl_wait_trigger();
  constexpr int NS = 32 / RG;   // slots per warp
  __shared__ __align__(16) BinWmWarp sw[kBinWmThreads / 32];
  __shared__ Best sb[kBinWmThreads / 32][32];
  const int g = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wl = lane % RG, slot = lane / RG;
  const int w = g * RG + wl;
  const bool live = w < Wk.W;
  const int wr = live ? w : g * RG;   // padding lanes of the last group load a real walker's scalars
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(Wk.rs + (size_t)g * Wk.rss * RG) + wl;
  const uint32_t* __restrict__ XB = Wk.xbits + (size_t)g * P.n;
  const int32_t* __restrict__ TB = Wk.tabu + (size_t)wr * Wk.ts;
  const long long kk = Wk.sc[wr].k;
  const int use_tabu = Wk.use_tabu;
  KT_BEGIN(Wk, 0);
  Best b;
  b.init();
  // admissibility (R13) is read only for a column that would become the lane's best (or, with
  // aspiration, for every column with s > 0: a tabu one is noted, R18)
  const AspRef A = asp_ref(Wk, wr);
  auto offer = [&](double sc, int j, int p, double v) {
    const bool bm = better_move(sc, j, b.s, b.j);
    if (!bm && !(A.a && sc > 0.0)) return;
    if (use_tabu) {
      const int32_t tp = __ldg(TB + p);
      if ((long long)tp > kk) {
        if (live) asp_note(A, p, j, tp, v, sc);
        return;
      }
    }
    if (!bm) return;
    b.s = sc;
    b.v = v;
    b.j = j;
    b.p = p;
  };
  const int nwarps = gridDim.x * (kBinWmThreads / 32);
  // integer data and integral weights <= 2^20 for every walker of the warp: flip sums in integers
  const bool wint_all = P.rint_base && __all_sync(kFull, Wk.sc[wr].wint != 0);
  int t = blockIdx.x * (kBinWmThreads / 32) + wid;
  for (; t < P.n_bchunks; t += nwarps) {
    const WTile T = P.bchunks[t];
    const int p = T.p0, len = T.ncols;
    const int* __restrict__ ridx = P.row_idx + T.e0;
    const double* __restrict__ rval = P.val + T.e0;
    const double xb = (double)((__ldg(XB + p) >> wl) & 1u);
    const double dir = 1.0 - 2.0 * xb;
    double acc = 0.0;
    for (int k0 = slot; k0 < len; k0 += 4 * NS) {
      int id[4];
      double av[4];
      double2 rv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + q * NS;
        id[q] = k < len ? __ldg(ridx + k) : -1;
        av[q] = k < len ? __ldg(rval + k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) rv[q] = id[q] >= 0 ? __ldg(RS + (size_t)id[q] * RG) : make_double2(-INFINITY, 0.0);
      if (wint_all) {   // (Σ m w) / 2 of the 4 entries: exact in double (half-integers)
        int a2 = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) a2 += penalty_m(rv[q], av[q] * dir) * weight_int(rv[q]);
        acc += 0.5 * (double)a2;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double r = rv[q].x, wv = (double)__int_as_float((int)__double2loint(rv[q].y));
          acc += penalty(wv, r, r + av[q] * dir);
        }
      }
    }
#pragma unroll
    for (int off = RG; off < 32; off <<= 1) acc += __shfl_xor_sync(kFull, acc, off);
    if (slot == 0 && live) {
      const LongCol L = P.lcols[T.e1];
      if (L.nchunks > 1) atomicAdd(Wk.lscr + (size_t)w * Wk.lss + L.scr, acc);
      else offer(acc, __ldg(P.perm + p), p, 1.0 - xb);
    }
  }
  t -= P.n_bchunks;
  BinWmWarp& S = sw[wid];
  for (; t < P.n_btiles; t += nwarps) {
    const WTile T = P.btiles[t];
    const int nc = T.ncols, len = T.e1 - T.e0;
    __syncwarp();
    if (4 * lane < len) {   // stage the tile's CSC entries (read once for the group)
      *reinterpret_cast<int4*>(S.id + 4 * lane) = __ldcs(reinterpret_cast<const int4*>(P.row_idx + T.e0) + lane);
      *reinterpret_cast<double2*>(S.a + 4 * lane) = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0) + 2 * lane);
      *reinterpret_cast<double2*>(S.a + 4 * lane + 2) = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0) + 2 * lane + 1);
    }
    int cb = 0, ce = 0, j = 0;
    uint32_t xw = 0u;
    if (lane < nc) {   // column data of lane c
      const int p = T.p0 + lane;
      cb = __ldg(P.col_ptr + p) - T.e0;
      ce = min(__ldg(P.col_ptr + p + 1) - T.e0, len);
      j = __ldg(P.perm + p);
      xw = __ldg(XB + p);
    }
    __syncwarp();
    for (int c = 0; c < nc; ++c) {
      const int e0 = __shfl_sync(kFull, cb, c), e1 = __shfl_sync(kFull, ce, c);
      const int jc = __shfl_sync(kFull, j, c);
      const double xb = (double)((__shfl_sync(kFull, xw, c) >> wl) & 1u);
      const double dir = 1.0 - 2.0 * xb;
      double acc = 0.0;
      if (wint_all) {   // integral weights: the flip score in half weights, in integers (penalty_m)
        int acc2 = 0;
        for (int k0 = e0 + slot; k0 < e1; k0 += 4 * NS) {
          int id[4];
          double av[4];
          double2 rv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k0 + q * NS;
            id[q] = k < e1 ? S.id[k] : -1;
            av[q] = k < e1 ? S.a[k] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) rv[q] = id[q] >= 0 ? __ldg(RS + (size_t)id[q] * RG) : make_double2(-INFINITY, 0.0);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc2 += penalty_m(rv[q], av[q] * dir) * weight_int(rv[q]);
        }
#pragma unroll
        for (int off = RG; off < 32; off <<= 1) acc2 += __shfl_xor_sync(kFull, acc2, off);
        if (slot == 0 && live) offer(0.5 * (double)acc2, jc, T.p0 + c, 1.0 - xb);
        continue;
      }
      for (int k0 = e0 + slot; k0 < e1; k0 += 4 * NS) {
        int id[4];
        double av[4];
        double2 rv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + q * NS;
          id[q] = k < e1 ? S.id[k] : -1;
          av[q] = k < e1 ? S.a[k] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) rv[q] = id[q] >= 0 ? __ldg(RS + (size_t)id[q] * RG) : make_double2(-INFINITY, 0.0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double r = rv[q].x, wv = (double)__int_as_float((int)__double2loint(rv[q].y));
          acc += penalty(wv, r, r + av[q] * dir);
        }
      }
#pragma unroll
      for (int off = RG; off < 32; off <<= 1) acc += __shfl_xor_sync(kFull, acc, off);
      if (slot == 0 && live) offer(acc, jc, T.p0 + c, 1.0 - xb);
    }
  }
  // per-walker block best: warps in fixed order
  sb[wid][lane] = b;
  __syncthreads();
  if (threadIdx.x < RG) {
    Best o = sb[0][threadIdx.x];
    for (int q = 1; q < kBinWmThreads / 32; ++q) o.take(sb[q][threadIdx.x]);
    const int ww = g * RG + threadIdx.x;
    if (ww < Wk.W) write_part(Wk.part + (size_t)ww * Wk.ps + blockIdx.x, o);
  }
  KT_END(Wk, 0);
}

// ------------------------------------------------------------------------------------------
// row-wise binary kernel (one walker): PAPER.md:347's row-wise flip scoring, re-designed
// ------------------------------------------------------------------------------------------
// The paper scores binary flips row-wise: a warp per row, the row's residual and weight read once,
// and an atomicAdd of every entry's penalty into a per-variable score array in global memory.
// Here the packed binary columns are cut into blocks of <= kRowVmax variables whose scores live in
// shared memory, so the atomics are shared-memory integer adds (2·penalty is an integer for the
// integral weights of R11; the sums are exact, so their order does not matter). A block's nonzeros
// are stored sorted by row and cut into kRowCluster slices, one per CTA of a cluster: a CTA streams
// its slice (8 bytes per nonzero: row, column-in-block | int16 coefficient), reads the row state of
// consecutive rows (a warp's 32 entries touch a few adjacent 16-byte records instead of 32 random
// sectors), reads x̄ from the block's slice of the bitset incumbent held in shared
// memory, and adds 2·p(w_i, r_i, r_i + a_ij (1 - 2x̄_j)) to the column's
// counter. After a cluster barrier CTA q sums the kRowCluster partial counters of its eighth of the
// block's columns over distributed shared memory, finishes those columns (tabu R13, R6) and keeps
// its best; a second barrier frees the counters for the next block (blocks round-robin over the
// clusters).
// Each CTA streams its slice of a block in stages (RowStage, cut on the host): a stage's entries
// (row, column | coefficient; <= kRowChunk) and the row state of the rows they span (<= kRowSpan
// consecutive 16-byte records, one bulk copy: the entries are sorted by row) arrive together by
// bulk copies (TMA, cp.async.bulk) into a kRowStages-deep shared-memory ring, so that no consumer
// waits on a row-state gather: the kernel streams. The last warp is the producer: its lane 0
// refills a stage as soon as the consumers release it (empty barrier: every consumer warp has
// finished with the stage; full barrier: the copies' bytes landed). A stage whose rows span more
// than kRowSpan rows (very sparse slices) gathers its row state instead (nr = 0).
struct RowRing {
  int2 rc[kRowStages][kRowChunk];   // entries: row, column-in-block | int16 coefficient (one 8-byte word)
  double2 rs[kRowStages][kRowSpan];
  uint64_t full[kRowStages];
  uint64_t empty[kRowStages];
};
constexpr size_t kRowSmem = sizeof(RowRing) + sizeof(int) * kRowVmax + sizeof(uint32_t) * (kRowWpb + 2);

// Cluster barrier with release/acquire at cluster scope (shared-memory counters become visible to
// the other CTAs of the cluster).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ int ld_dsmem_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_acqrel() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kRowThreads, 1) k_eval_binrow(DevProblem P, DevWalkers Wk, int part_base) {
  pdl_wait_trigger();
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Best sb[kRowThreads / 32];
  KT_BEGIN(Wk, 0);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), C = P.rb_cluster;
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool producer = tid >= kRowConsumers;
  RowRing& R = *reinterpret_cast<RowRing*>(smem);
  int* sc = reinterpret_cast<int*>(smem + sizeof(RowRing));    // [kRowVmax] 2·score partials
  uint32_t* bits = reinterpret_cast<uint32_t*>(sc + kRowVmax);  // [kRowWpb] the block's x̄ bits
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(Wk.rs);   // rg = 1, walker 0
  const uint32_t* __restrict__ XB = Wk.xbits;
  const int32_t* __restrict__ TB = Wk.tabu;
  const long long kk = Wk.sc[0].k;
  const int use_tabu = Wk.use_tabu;
  const AspRef A = asp_ref(Wk, 0);
  uint32_t rsc[kRowCluster];   // the counters of every CTA of the cluster (shared::cluster addresses)
#pragma unroll
  for (int q = 0; q < kRowCluster; ++q) rsc[q] = mapa_u32(smem_u32(sc), q < C ? q : 0);
  if (tid == 0) {
    for (int q = 0; q < kRowStages; ++q) {
      mbar_init(&R.full[q], 1);
      mbar_init(&R.empty[q], kRowConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Best b;
  b.init();
  int g = 0;   // chunks of this CTA so far (both roles count the same sequence)
  for (int vb = cid; vb < P.n_rblocks; vb += ncl) {
    const RowBlock& B = P.rblocks[vb];
    const int p0 = B.p0, nv = B.nv, nb = P.n_rblocks;
    const int st0 = B.st[rank], nch = B.st[rank + 1] - st0;
    for (int i = tid; i < nv; i += kRowThreads) sc[i] = 0;
    for (int i = tid; i < (nv + 31) / 32; i += kRowThreads) bits[i] = __ldg(XB + (size_t)vb * kRowWpb + i);
    __syncthreads();
    if (producer) {
      if (lane == 0)
        for (int c = 0; c < nch; ++c) {
          const int q = g + c, st = q % kRowStages;
          const RowStage G = P.rb_stage[st0 + c];
          if (q >= kRowStages) mbar_wait(&R.empty[st], (unsigned)((q / kRowStages) - 1) & 1u);
          mbar_expect_tx(&R.full[st], (unsigned)(8 * G.ne + 16 * G.nr));
          tma_load_1d(R.rc[st], P.rb_rc + G.e0, 8u * G.ne, &R.full[st]);
          if (G.nr > 0) tma_load_1d(R.rs[st], RS + G.r0, 16u * G.nr, &R.full[st]);
        }
      __syncwarp();
    } else {
      for (int c = 0; c < nch; ++c) {
        const int q = g + c, st = q % kRowStages;
        const RowStage G = P.rb_stage[st0 + c];
        mbar_wait(&R.full[st], (unsigned)(q / kRowStages) & 1u);
        int2 e[kRowPer];
#pragma unroll
        for (int k = 0; k < kRowPer; ++k) {
          const int i = tid + k * kRowConsumers;
          e[k] = i < G.ne ? R.rc[st][i] : make_int2(0, 0);   // cv 0: no entry, or inert padding
        }
        double2 rv[kRowPer];
        if (G.nr > 0) {   // the stage's row state came with it (shared memory)
          const double2* rss = R.rs[st] - G.r0;
#pragma unroll
          for (int k = 0; k < kRowPer; ++k) rv[k] = e[k].y ? rss[e[k].x] : make_double2(-INFINITY, 0.0);
        } else {          // a stage spanning too many rows gathers it
#pragma unroll
          for (int k = 0; k < kRowPer; ++k) rv[k] = e[k].y ? __ldg(RS + e[k].x) : make_double2(-INFINITY, 0.0);
        }
#pragma unroll
        for (int k = 0; k < kRowPer; ++k) {
          // 2·p(w, r, r + d) with d = a (1 - 2x̄), in integers: satisfied
          // before is r <= 0, after is r <= -d (exact: r + d is exact when it is near 0,
          // Sterbenz), a violated row gets less violated iff d < 0; w is integral (R11). Inert
          // rows give 0.
          const uint32_t uk = (uint32_t)e[k].y;
          const int c2 = (int)(uk & 0xffffu);
          const int ai = (int)(int16_t)(uk >> 16);
          const bool xb = (bits[c2 >> 5] >> (c2 & 31)) & 1u;
          const int nd = xb ? ai : -ai;   // -d
          // r <= v <=> ceil(r) <= v for the integers 0 and nd: the row state's RowState::rc
          const int rc = __double2hiint(rv[k].y);
          const int iw = __float2int_rn(__int_as_float((int)__double2loint(rv[k].y)));
          const bool z0 = rc <= 0, z1 = rc <= nd;
          // in units of w: -2 (becomes violated), +2 (becomes satisfied), +-1 (stays violated, less
          // or more), 0 (stays satisfied); nd != 0 for every entry but the inert padding
          const int m = 2 * ((int)z1 - (int)z0) + ((z0 | z1) ? 0 : (nd > 0 ? 1 : -1));
          if (m != 0) atomicAdd(sc + c2, m * iw);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[st]);   // the stage's entries and row state are consumed
      }
    }
    g += nch;
    cluster_sync_acqrel();
    // columns [v0, v1) of the block: the sum of the cluster's partial counters (all remote loads
    // in flight together), then the column (x̄ flipped, tabu R13, ties R6)
    const int per = (nv + C - 1) / C;
    const int v0 = rank * per, v1 = min(nv, v0 + per);
    // four columns per thread at a time: their remote counters and user indices are all loaded
    // before any is used; the tabu expiry only for a column that would become the thread's best
    const int32_t* __restrict__ bperm = P.rb_perm + (size_t)vb * kRowVmax;
    for (int vq = v0 + tid; vq < v1; vq += 4 * kRowThreads) {
      int tot[4], jq[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int v = vq + i * kRowThreads;
        tot[i] = 0;
        jq[i] = 0;
        if (v < v1) {
#pragma unroll
          for (int q = 0; q < kRowCluster; ++q)
            if (q < C) tot[i] += ld_dsmem_s32(rsc[q] + 4u * (uint32_t)v);
          jq[i] = __ldg(bperm + v);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int v = vq + i * kRowThreads;
        if (v >= v1) break;
        const double s = 0.5 * (double)tot[i];
        const bool bm = better_move(s, jq[i], b.s, b.j);
        if (!bm && !(A.a && s > 0.0)) continue;
        const int p = p0 + v * nb;
        if (use_tabu) {
          const int32_t tp = __ldg(TB + p);
          if ((long long)tp > kk) {
            asp_note(A, p, jq[i], tp, 1.0 - (double)((bits[v >> 5] >> (v & 31)) & 1u), s);
            continue;
          }
        }
        if (!bm) continue;
        b.s = s;
        b.v = 1.0 - (double)((bits[v >> 5] >> (v & 31)) & 1u);
        b.j = jq[i];
        b.p = p;
      }
    }
    cluster_sync_acqrel();
  }
  b = warp_reduce_best(b);
  if (lane == 0) sb[tid >> 5] = b;
  __syncthreads();
  if (tid == 0) {
    Best o = sb[0];
    for (int q = 1; q < kRowThreads / 32; ++q) o.take(sb[q]);
    write_part(Wk.part + part_base + blockIdx.x, o);
  }
  KT_END(Wk, 0);
}

// ------------------------------------------------------------------------------------------
// general-column kernel
// ------------------------------------------------------------------------------------------
// k_eval_gen evaluates the packed general integer columns (deg + 2 <= kShortDeg) with
// Algorithm 1 per column, sort-free, in offsets relative to x̄, the chunks of long
// bounded-integer columns (counting sort) and, in the row-wise binary mode, the chunks
// of long binary columns.
//
// Lines 3-11 in offsets. For an integer column and a row with residual r and coefficient a, the
// breakpoint of line 3-4 is t = floor(x̄ - r/a) (a > 0) or ceil(x̄ - r/a) (a < 0), so its offset
// d = t - x̄ = floor(-r/a) (a > 0) or -floor(-r/|a|) (a < 0) needs neither x̄ nor the column: it is
// computed per entry, slot-parallel, from the gathered row state alone. The six cases of lines
// 5-11 are the sign of a and of d (d > 0 <=> x̄ < t). With w the row weight they give, in units
// of half a weight (F = 2δ, β2 = 2β, α2 = 2α, integers for the integral weights of R11):
//   code  case                 key     F      β2     α2     side   positive step
//   6     a<0, d>0 (violated)  d       w      -w     2w     up     yes (σ rises at d)
//   0     a<0, d<0 (slack)     d       2w     -2w    0      down   no
//   5     a>0, d<0 (violated)  d+1     -w     2w     -2w    down   yes (σ rises below d+1)
//   3     a>0, d>0 (slack)     d+1     -2w    0      0      up     no
//   2     a<0, d=0 (tight)     MAX     0      -2w    2w     -      -
//   2     a>0, d=0 (tight)     MAX     0      0      -2w    -      -
// (an a>0 row's (t,-1,0) entry of line 10-11 carries no delta; its value is the candidate v = d,
// scored before its +1 entry, R3), so that σ(v) = β + α [v > 0] + Σ_{key_e <= v} δ_e exactly
// (DESIGN §2.3). Code bit 0: key = v + 1; bit 1: up side (v > 0); bit 2: positive step.
// When every residual is an integer below 2^23 in magnitude (WalkerScalars::rint) the floor of the
// quotient is taken without a double division: the float quotient of n = -r by |a| is within one of
// floor(n/|a|) and its exact float remainder n - f|a| corrects it; otherwise line 3 is
// the IEEE double division of the oracle.
//
// Lines 13-16 without a sort. Candidates (R2, R5) are the entries with v in [l - x̄, u - x̄] and the
// finite bounds other than x̄. On the up side (v > 0) σ changes only at keys, rising at the
// positive steps (code 6) and falling elsewhere, so a candidate that is not a positive step scores
// at most the nearest positive step below it, or the smallest up candidate if there is none; on
// the down side symmetrically. Since R4 prefers the smaller |v| on ties, the argmax of Algorithm 1
// over all candidates is always among {the positive steps, the smallest up candidate, the largest
// down candidate} (DESIGN §2.3 gives the proof): only those are scored, each by one pass over
// the column's entries. The number of positive steps is the number of violated rows of the
// column (cutoff row included), a few in a tabu walk.
//
// Each warp works through a list of warp items (a general tile of <= 32 whole columns and
// <= kG32Max entries, or a chunk of a long column): its first item is static, the later ones come
// from a per-walker counter in list order, taken while the current item is evaluated. Within a
// tile the CSC indices and coefficients of the next round of 128 entries are in flight (registers)
// while this round's row state is gathered (one 16-byte __ldg per entry, L2-resident).
// A general tile: phase 1 (slot-parallel) turns every entry's row state into {key << 3 | code, F,
// β2, α2} in the warp's shared-memory tile; phase 2 (lane c = column c) makes one pass for β, α, the nearest candidates and
// the positive steps, then one pass per four candidates. The int path needs weights that are
// integers <= 2^20 (WalkerScalars::wint; |Σ F| < 2^27) and offsets |d| < 2^28; with other weights
// the F, β2, α2 words are floats summed in double (same candidates, scores up to summation order,
// DESIGN §5), and a tile with a larger offset is evaluated column by column by gen_column_serial.
// A long column's chunks add into its accumulators in walker scratch; the chunk that takes the
// column's last ticket finishes it (lbkt_finalize / lbin_finalize) and re-arms the accumulators.
#ifndef CHAP_G32_MAX
#define CHAP_G32_MAX 512
#endif
constexpr int kG32Max = CHAP_G32_MAX;           // entries per general tile
constexpr int kKeyMax = (1 << 28) - 1;          // key of entries that are never in a prefix
constexpr int kKeyLim = kKeyMax - 2;            // |offset| limit of the int path (bounds clamp here)
struct __align__(16) GenWarp {
  int4 ent[kG32Max];
};
// a long bounded-integer chunk uses the warp's GenWarp area: int32 histogram, candidate words, stage
constexpr int kWarpDom = 1024;
constexpr int kLbktHistBytes = 4 * (kWarpDom + 1 + 3);
static_assert(kLbktHistBytes + kWarpDom / 8 + 32 * 8 <= (int)sizeof(GenWarp), "LBKT scratch exceeds GenWarp");
constexpr size_t kGenSmem = sizeof(GenWarp) * (kGenThreads / 32);

__device__ __forceinline__ double next_up(double t) {   // the next double above t
  if (t == 0.0) return 4.9406564584124654e-324;
  if (isinf(t)) return t;
  const long long bits = __double_as_longlong(t);
  return __longlong_as_double(t > 0.0 ? bits + 1 : bits - 1);
}

// Within one variable on offsets (R4): higher score, then smaller |v|, then smaller v.
template <class S>
__device__ __forceinline__ bool better_off(S s1, int v1, S s0, int v0) {
  if (s1 != s0) return s1 > s0;
  const int a1 = abs(v1), a0 = abs(v0);
  if (a1 != a0) return a1 < a0;
  return v1 < v0;
}

// The admissible-best update of a column (R6, R13); the tabu expiry is read only for a column
// that would become the lane's best.
__device__ __forceinline__ void offer_column(int p, int j, const int32_t* __restrict__ TB, double xb, double v,
                                             double s, Best& b, double* oxhat, double* oscore, long long k,
                                             int use_tabu, AspRef A) {
  if (s == -INFINITY) v = xb;
  if (oxhat) oxhat[j] = v;
  if (oscore) oscore[j] = s;
  cache_col(A, p, v, s);
  const bool bm = better_move(s, j, b.s, b.j);
  if (!bm && !(A.a && s > 0.0)) return;
  if (use_tabu) {
    const int32_t tp = __ldg(TB + p);
    if ((long long)tp > k) {
      asp_note(A, p, j, tp, v, s);
      return;
    }
  }
  if (!bm) return;
  b.s = s;
  b.v = v;
  b.j = j;
  b.p = p;
}

// One general column by one lane, in double: continuous columns (their breakpoints are not
// integers), and integer columns of a tile whose offsets exceed the int path. Lines 3-11 per
// entry (emit), the reduced candidate set of the tile path (positive steps, nearest up and down
// candidates), and for each candidate the line-14 prefix as a direct sum over the column's
// entries (re-gathered: L1/L2 hits). Returns (x̂, s); s = -inf without a candidate.
__device__ void gen_column_serial(const DevProblem& P, const double* __restrict__ X, const double2* __restrict__ RS,
                                  int st, int p, double& v_out, double& s_out) {
  const int cb = __ldg(P.col_ptr + p), ce = __ldg(P.col_ptr + p + 1);
  const double xb = __ldg(X + p), l = __ldg(P.lb + p), u = __ldg(P.ub + p);
  const int is_int = __ldg(P.vclass + p) != 3;
  auto entry = [&](int e) {
    const double2 rv = __ldg(RS + (size_t)__ldg(P.row_idx + e) * st);
    const double w = (double)__int_as_float((int)__double2loint(rv.y));
    return emit(xb, rv.x, __ldg(P.val + e), w, is_int);
  };
  auto key_of = [&](const Elem& el) { return el.delta > 0.0 ? el.t : (is_int ? el.t + 1.0 : next_up(el.t)); };
  double beta = 0.0, alpha = 0.0, vup = INFINITY, vdn = -INFINITY;
  unsigned long long pm = 0ull;   // positive steps (deg <= 62)
  for (int e = cb; e < ce; ++e) {
    const Elem el = entry(e);
    beta += el.beta;
    alpha += el.alpha;
    if (!el.valid || !isfinite(el.t) || !(el.t >= l && el.t <= u)) continue;   // R5; valid => t != x̄
    if (el.t > xb) vup = fmin(vup, el.t); else vdn = fmax(vdn, el.t);
    if ((el.t > xb) != (el.plus != 0)) pm |= 1ull << (e - cb);
  }
  if (isfinite(u) && u != xb) vup = fmin(vup, u);
  if (isfinite(l) && l != xb) vdn = fmax(vdn, l);
  double bs = -INFINITY, bv = xb;
  auto score = [&](double v) {
    double acc = 0.0;
    for (int e = cb; e < ce; ++e) {
      const Elem el = entry(e);
      if (el.valid && isfinite(el.t) && key_of(el) <= v) acc += el.delta;
    }
    const double sg = beta + acc + (v > xb ? alpha : 0.0);
    if (better_shift(sg, v, bs, bv, xb)) { bs = sg; bv = v; }
  };
  if (vup < INFINITY) score(vup);
  if (vdn > -INFINITY) score(vdn);
  for (unsigned long long m = pm; m; m &= m - 1) score(entry(cb + __ffsll((long long)m) - 1).t);
  v_out = bv;
  s_out = bs;
}

// Lines 3-11 of Algorithm 1 for one entry of an integer column in offsets (table above): the
// entry word key << 3 | code and F, β2, α2 (ints for INTW, else float bits). rint: every residual
// is an integer (the exact float-quotient path). Sets ovf for an offset beyond the int path.
// The case c = 3 [a > 0] + [d >= 0] + [d > 0] indexes the block's table of {code, F, β2, α2} (in units
// of w): c = 0..5 is (a<0,d<0) (a<0,d=0) (a<0,d>0) (a>0,d<0) (a>0,d=0) (a>0,d>0).
__device__ __forceinline__ void off_table_init(int4* tab) {
  switch (threadIdx.x) {
    case 0: tab[0] = make_int4(0, 2, -2, 0); break;
    case 1: tab[1] = make_int4(2, 0, -2, 2); break;
    case 2: tab[2] = make_int4(6, 1, -1, 2); break;
    case 3: tab[3] = make_int4(5, -1, 2, -2); break;
    case 4: tab[4] = make_int4(2, 0, 0, -2); break;
    case 5: tab[5] = make_int4(3, -2, 0, 0); break;
    default: break;
  }
}
template <bool INTW>
__device__ __forceinline__ int4 off_entry(double r, float wf, double a, bool rint, const int4* __restrict__ tab,
                                          bool& ovf) {
  const float rf = (float)r;
  const bool pos = a > 0.0;
  int d;
  if (rint && (fabsf(rf) < 8388608.f || rf == -INFINITY)) {
    // g = floor(n / A), n = -r, A = |a| (integers below 2^23): the float quotient by the approximate
    // reciprocal is within 1 of n/A, so its floor is g - 1, g or g + 1, and the exact float remainder
    // n - f A (|f A| < 2^24) decides which. The inert rows (r = -inf) take n = 0, d = 0.
    const float n = rf == -INFINITY ? 0.f : -rf, A = fabsf((float)a);
    float ra;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(A));
    float f = floorf(n * ra);
    const float rem = fmaf(-f, A, n);
    f = rem < 0.f ? f - 1.f : (rem >= A ? f + 1.f : f);
    const int g = __float2int_rz(f);
    d = pos ? g : -g;
  } else {
    const bool live = r > -INFINITY;               // inert rows: the inactive cutoff row, padding
    const double qd = (live && r != 0.0) ? r / a : 0.0;
    const double dd = pos ? -ceil(qd) : -floor(qd);   // t - x̄ of lines 3-4
    const bool big = !(fabs(dd) <= (double)(kKeyLim - 1));
    ovf |= live && big;
    // an offset beyond the int path is clamped (its sign, hence its case, is kept): the general tile
    // then re-evaluates in double (ovf); for a bounded domain it lies outside [l, u] either way
    d = !live ? 0 : (big ? (dd > 0.0 ? kKeyLim - 1 : 1 - kKeyLim) : (int)dd);
  }
  const int4 t = tab[(pos ? 3 : 0) + (d >= 0) + (d > 0)];
  int4 ent;
  ent.x = ((d == 0 ? kKeyMax : d + (int)pos) << 3) | t.x;
  // the inert rows carry w = 0 in the row state: all three words vanish
  if (INTW) {
    const int w1 = __float2int_rn(wf);
    ent.y = w1 * t.y;
    ent.z = w1 * t.z;
    ent.w = w1 * t.w;
  } else {
    ent.y = __float_as_int(wf * (float)t.y);
    ent.z = __float_as_int(wf * (float)t.z);
    ent.w = __float_as_int(wf * (float)t.w);
  }
  return ent;
}

// One round of a general tile: slots 4 lane .. 4 lane + 3 of its 128 (one 16-byte index load, two
// 16-byte coefficient loads); out of range: the inert dummy row.
struct GenRound {
  int4 id;
  double2 a01, a23;
};
__device__ __forceinline__ GenRound gen_round(const DevProblem& P, const WTile& T, int k0) {
  GenRound R;
  R.id = make_int4(P.dummy_row, P.dummy_row, P.dummy_row, P.dummy_row);
  R.a01 = make_double2(1.0, 1.0);
  R.a23 = R.a01;
  if (k0 < T.e1 - T.e0) {
    R.id = __ldcs(reinterpret_cast<const int4*>(P.row_idx + T.e0 + k0));
    R.a01 = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0 + k0));
    R.a23 = __ldcs(reinterpret_cast<const double2*>(P.val + T.e0 + k0) + 1);
  }
  return R;
}

// Pass 0 of lines 13-16 on integer offsets, one off_entry word x3 at a time: the nearest candidate
// on each side (vup, vdn; bounds preset by the caller) and the first six positive steps c2..c7.
__device__ __forceinline__ void off_pass0(int x3, int hi, int lo, int& vup, int& vdn, int& c2, int& c3, int& c4,
                                          int& c5, int& c6, int& c7, int& nstep) {
  const int code = x3 & 7;
  const int v = (x3 >> 3) - (code & 1);
  // up side (codes 6, 3 and the tight code 2, whose v exceeds hi): in bounds iff v <= hi;
  // down side (codes 0, 5): iff v >= lo
  const bool up = code & 2;
  const bool inb = up ? v <= hi : v >= lo;
  if (inb) {
    if (up) vup = min(vup, v); else vdn = max(vdn, v);
    if (code & 4) {   // a positive step (codes 6, 5)
      c7 = nstep == 5 ? v : c7;
      c6 = nstep == 4 ? v : c6;
      c5 = nstep == 3 ? v : c5;
      c4 = nstep == 2 ? v : c4;
      c3 = nstep == 1 ? v : c3;
      c2 = nstep == 0 ? v : c2;
      ++nstep;
    }
  }
}

// Lines 13-16 on integer offsets for one column whose off_entry words are at(e),
// e in [e0, e1): σ2 (twice the score) at the reduced candidate set {vup, vdn, positive steps c2..c7
// and beyond} with R4, given β2, α2 and the pass-0 candidates. Returns whether a candidate exists.
template <bool INTW, class At>
__device__ __forceinline__ bool offsets_best(At at, int e0, int e1,
                                             typename std::conditional<INTW, int, double>::type b2,
                                             typename std::conditional<INTW, int, double>::type a2, int hi, int lo,
                                             int vup, int vdn, int c2, int c3, int c4, int c5, int c6, int c7,
                                             int nstep, typename std::conditional<INTW, int, double>::type& bs2,
                                             int& bv) {
  using Acc = typename std::conditional<INTW, int, double>::type;
  auto fv = [](int bits) -> Acc { if (INTW) return (Acc)bits; else return (Acc)__int_as_float(bits); };
  // the best (σ2, v) of the column under R4: with integer scores one packed key, higher is better
  // (σ2, then smaller |v|, then smaller v)
  long long bkey = LLONG_MIN;
  bs2 = 0;
  bv = 0;
  bool have = false;
  auto offer2 = [&](Acc sg, int v) {
    if (INTW) {
      const unsigned tie = 0x7fffffffu - (((unsigned)abs(v) << 1) | (v > 0 ? 1u : 0u));
      bkey = max(bkey, (long long)sg * 4294967296ll + (long long)tie);
    } else if (!have || better_off(sg, v, bs2, bv)) {
      bs2 = sg;
      bv = v;
      have = true;
    }
  };
  // σ2 at up to four candidate offsets (INT_MAX / INT_MIN: none) in one pass
  auto score4 = [&](int q0, int q1, int q2, int q3) {
    auto lim = [](int q) { return (q == INT_MAX || q == INT_MIN) ? INT_MIN : ((q << 3) | 7); };   // key <= v  <=>  x <= v << 3 | 7
    const int l0 = lim(q0), l1 = lim(q1), l2 = lim(q2), l3 = lim(q3);
    Acc s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int e = e0; e < e1; ++e) {
      const int2 E = at(e);
      const Acc F = fv(E.y);
      s0 += E.x <= l0 ? F : (Acc)0;
      s1 += E.x <= l1 ? F : (Acc)0;
      s2 += E.x <= l2 ? F : (Acc)0;
      s3 += E.x <= l3 ? F : (Acc)0;
    }
    if (l0 != INT_MIN) offer2(b2 + s0 + (q0 > 0 ? a2 : (Acc)0), q0);
    if (l1 != INT_MIN) offer2(b2 + s1 + (q1 > 0 ? a2 : (Acc)0), q1);
    if (l2 != INT_MIN) offer2(b2 + s2 + (q2 > 0 ? a2 : (Acc)0), q2);
    if (l3 != INT_MIN) offer2(b2 + s3 + (q3 > 0 ? a2 : (Acc)0), q3);
  };
  score4(vup, vdn, c2, c3);
  if (nstep > 2) score4(c4, c5, c6, c7);
  if (nstep > 6) {   // steps 7, 8, ... (rare): rescan for them, four per pass
    int q0 = INT_MIN, q1 = INT_MIN, q2 = INT_MIN, q3 = INT_MIN;
    int seen = 0, nq = 0;
    for (int e = e0; e < e1; ++e) {
      const int x3 = at(e).x, code = x3 & 7, v = (x3 >> 3) - (code & 1);
      const bool up = code & 2;
      if (!((code & 4) && (up ? v <= hi : v >= lo))) continue;
      if (seen++ < 6) continue;
      q0 = nq == 0 ? v : q0;
      q1 = nq == 1 ? v : q1;
      q2 = nq == 2 ? v : q2;
      q3 = nq == 3 ? v : q3;
      if (++nq == 4) {
        score4(q0, q1, q2, q3);
        nq = 0;
        q0 = q1 = q2 = q3 = INT_MIN;
      }
    }
    if (nq > 0) score4(q0, q1, q2, q3);
  }
  if (INTW && bkey != LLONG_MIN) {
    have = true;
    bs2 = (Acc)(bkey >> 32);
    const unsigned t = 0x7fffffffu - (unsigned)(bkey & 0xffffffffll);
    bv = (t & 1u) ? (int)(t >> 1) : -(int)(t >> 1);
  }
  return have;
}

// One tile of packed general integer columns (see above). INTW: integral weights <= 2^20. R holds
// the tile's first round (loaded by the caller); the rounds are software-pipelined (the next round's
// loads are in flight while this round's gathers return), and when the warp's next item Tn is a
// general tile its first round is loaded into R before phase 2.
template <bool INTW>
__device__ __forceinline__ void gen32_tile(const DevProblem& P, const double* __restrict__ X,
                                           const double2* __restrict__ RS, int st,
                                           const int32_t* __restrict__ TB, const WTile& T, const WTile& Tn,
                                           bool has_next, GenRound& R, int lane, GenWarp& S, bool rint,
                                           const int4* __restrict__ tab, Best& b, double* oxhat, double* oscore,
                                           long long kk, int use_tabu, AspRef A) {
  const int nc = T.ncols, len = T.e1 - T.e0;
  // column data of lane c (loads in flight during phase 1)
  const int p = T.p0 + lane;
  int cb = 0, ce = 0, j = 0;
  double xb = 0.0, l = 0.0, u = 0.0;
  if (lane < nc) {
    cb = __ldg(P.col_ptr + p) - T.e0;
    ce = __ldg(P.col_ptr + p + 1) - T.e0;
    j = __ldg(P.perm + p);
    xb = __ldg(X + p);
    l = __ldg(P.lb + p);
    u = __ldg(P.ub + p);
  }
  int4* ent = S.ent;
  // phase 1: lines 3-11 per entry (slots 4 lane .. 4 lane + 3 of each round of 128)
  bool ovf = false;
  for (int r0 = 0; r0 < len; r0 += 4 * 32) {
    const int k0 = r0 + 4 * lane;
    double2 rv[4];
    rv[0] = __ldg(RS + (size_t)R.id.x * st);
    rv[1] = __ldg(RS + (size_t)R.id.y * st);
    rv[2] = __ldg(RS + (size_t)R.id.z * st);
    rv[3] = __ldg(RS + (size_t)R.id.w * st);
    const double2 a01 = R.a01, a23 = R.a23;
    if (r0 + 4 * 32 < len) R = gen_round(P, T, k0 + 4 * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double a = q == 0 ? a01.x : (q == 1 ? a01.y : (q == 2 ? a23.x : a23.y));
      ent[k0 + q] = off_entry<INTW>(rv[q].x, __int_as_float((int)__double2loint(rv[q].y)), a, rint, tab, ovf);
    }
  }
  if (has_next && Tn.kind == CC_GEN) R = gen_round(P, Tn, 4 * lane);
  ovf = __any_sync(kFull, ovf);
  __syncwarp();
  if (lane >= nc) return;   // (the kernel's loop reconverges the warp after every item)
  if (ovf) {   // an offset beyond the int path: every column of the tile in double
    double v, sv;
    gen_column_serial(P, X, RS, st, p, v, sv);
    offer_column(p, j, TB, xb, v, sv, b, oxhat, oscore, kk, use_tabu, A);
    return;
  }
  // phase 2, pass 0: β, α, the nearest candidate on each side (bounds included) and the positive
  // steps (the first six kept in registers); then σ2 at up to four candidates per pass over the
  // column's entries: {vup, vdn, step 1, step 2}, {steps 3..6}, further steps (rare) four per pass.
  const bool ufin = isfinite(u), lfin = isfinite(l);
  const double hid = u - xb, lod = l - xb;
  const int hi = ufin ? (int)fmin(hid, (double)kKeyLim) : kKeyLim;
  const int lo = lfin ? (int)fmax(lod, -(double)kKeyLim) : -kKeyLim;
  int vup = (ufin && hi > 0) ? hi : INT_MAX;
  int vdn = (lfin && lo < 0) ? lo : INT_MIN;
  using Acc = typename std::conditional<INTW, int, double>::type;
  auto fv = [](int bits) -> Acc { if (INTW) return (Acc)bits; else return (Acc)__int_as_float(bits); };
  Acc b2 = 0, a2 = 0;
  int c2 = INT_MIN, c3 = INT_MIN, c4 = INT_MIN, c5 = INT_MIN, c6 = INT_MIN, c7 = INT_MIN, nstep = 0;
  for (int e = cb; e < ce; ++e) {
    const int4 E = ent[e];
    b2 += fv(E.z);
    a2 += fv(E.w);
    off_pass0(E.x, hi, lo, vup, vdn, c2, c3, c4, c5, c6, c7, nstep);
  }
  Acc bs2;
  int bv;
  const bool have = offsets_best<INTW>([&](int e) { return *reinterpret_cast<const int2*>(&ent[e]); }, cb, ce, b2, a2,
                                       hi, lo, vup, vdn, c2, c3, c4, c5, c6, c7, nstep, bs2, bv);
  double v = xb, sres = -INFINITY;
  if (have) {
    sres = 0.5 * (double)bs2;
    // a bound beyond the clamp is the farthest candidate of its side: report its exact value
    v = (bv == hi && ufin && hid > (double)kKeyLim) ? u : ((bv == lo && lfin && lod < -(double)kKeyLim) ? l : xb + (double)bv);
  }
  offer_column(p, j, TB, xb, v, sres, b, oxhat, oscore, kk, use_tabu, A);
}

// A warp chunk (<= kBktChunk nonzeros) of a long general integer column with domain [l, u],
// dom = u - l + 1 <= kBucketMax: the sort of line 13 becomes a counting pass. With the entries of
// off_entry (gen32_tile's table), D[x̄ + key - l] collects δ = F/2 of every emitted entry, so that
// sigma(v) = β + Σ_{v' <= v} D[v' - l] + α [v > x̄]; an entry whose key is below l is in
// every prefix (folded into β), one above u in none (dropped), and the candidates (R2, R5) are the
// emitted values in [l, u]. Every chunk adds its entries into the column's accumulators (D, β, α,
// candidate bits) in walker scratch. Breakpoints of a long column crowd onto few values, so with
// integral weights <= 2^20 (INTW) a chunk first counts F into a warp-private int32 shared-memory
// histogram (|Σ| <= kBktChunk 2^21 < 2^31) and then adds each nonzero bucket once; other weights, or
// domains above kWarpDom, aggregate per warp instead (lanes with equal buckets: __match_any_sync,
// the lowest lane adds the group's sum). The chunk that takes the column's last ticket scans D
// (lbkt_finalize).
template <bool INTW>
__device__ __forceinline__ void lbkt_chunk(const DevProblem& P, const DevWalkers& Wk, int walker,
                                           const double* __restrict__ X, const double2* __restrict__ RS,
                                           int st, const WTile& T, const LongCol& L, int lane, unsigned char* wmem,
                                           bool rint, const int4* __restrict__ tab) {
  const int p = T.p0, dom = L.dom, len = T.ncols;
  const int* __restrict__ ridx = P.row_idx + T.e0;
  const double* __restrict__ rval = P.val + T.e0;
  const int xl = (int)(__ldg(X + p) - __ldg(P.lb + p));      // x̄ - l, in [0, dom)
  double* Dg = Wk.lscr + (size_t)walker * Wk.lss + L.scr;   // [dom + 1]
  double* BA = Dg + dom + 1;                                 // β, α
  unsigned* Cw = reinterpret_cast<unsigned*>(BA + 2);        // candidate bits
  int* hist = reinterpret_cast<int*>(wmem);                              // [kWarpDom + 1]
  unsigned* hcw = reinterpret_cast<unsigned*>(wmem + kLbktHistBytes);    // [kWarpDom / 32]
  double* stage = reinterpret_cast<double*>(wmem + kLbktHistBytes + kWarpDom / 8);   // [32]
  const bool local = INTW && dom <= kWarpDom;
  const int nwords = (dom + 31) >> 5;
  if (local) {
    for (int q = lane; q <= dom; q += 32) hist[q] = 0;
    for (int q = lane; q < nwords; q += 32) hcw[q] = 0u;
    __syncwarp();
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  using Acc = typename std::conditional<INTW, int, double>::type;
  Acc b2 = 0, a2 = 0;
  bool ovf = false;   // irrelevant here: a clamped offset lies outside [l, u]
  for (int r0 = 0; r0 < len; r0 += 32 * kWSlotsGen) {
    int id[kWSlotsGen];
    double av[kWSlotsGen];
#pragma unroll
    for (int q = 0; q < kWSlotsGen; ++q) {
      const int k = r0 + lane + 32 * q;
      id[q] = k < len ? __ldcs(ridx + k) : P.dummy_row;
      av[q] = k < len ? __ldcs(rval + k) : 1.0;
    }
    double2 rv[kWSlotsGen];
#pragma unroll
    for (int q = 0; q < kWSlotsGen; ++q) rv[q] = __ldg(RS + (size_t)id[q] * st);
#pragma unroll
    for (int q = 0; q < kWSlotsGen; ++q) {
      const int4 E = off_entry<INTW>(rv[q].x, __int_as_float((int)__double2loint(rv[q].y)), av[q], rint, tab, ovf);
      if (INTW) { b2 += E.z; a2 += E.w; } else { b2 += (double)__int_as_float(E.z); a2 += (double)__int_as_float(E.w); }
      const int code = E.x & 7, key = E.x >> 3;
      int bq = -1, cq = -1;
      if (code != 2) {
        const int bk = key + xl, cv = key - (code & 1) + xl;
        if (bk < 0) {   // below l: in every prefix
          if (INTW) b2 += E.y; else b2 += (double)__int_as_float(E.y);
        } else if (bk < dom) {
          bq = bk;
        }
        if (cv >= 0 && cv < dom) cq = cv;
      }
      if (local) {   // the warp's shared histogram and candidate words (shared-memory atomics)
        if (bq >= 0 && E.y != 0) atomicAdd(hist + bq, E.y);
        if (cq >= 0) atomicOr(hcw + (cq >> 5), 1u << (cq & 31));
        continue;
      }
      // bucket deltas: one atomic per distinct bucket of the 32 entries
      const double dq = bq >= 0 ? 0.5 * (INTW ? (double)E.y : (double)__int_as_float(E.y)) : 0.0;
      const unsigned mD = __match_any_sync(kFull, bq);
      stage[lane] = dq;
      __syncwarp();
      if (bq >= 0 && (mD & lt_mask) == 0) {
        double sum = dq;
        for (unsigned mm = mD & (mD - 1); mm; mm &= mm - 1) sum += stage[__ffs(mm) - 1];
        if (sum != 0.0) atomicAdd(Dg + bq, sum);
      }
      __syncwarp();
      // candidate bits: one OR per distinct word, skipped once the bits are set
      const int wq = cq >= 0 ? (cq >> 5) : -1;
      const unsigned mC = __match_any_sync(kFull, wq);
      const unsigned bits = __reduce_or_sync(mC, cq >= 0 ? (1u << (cq & 31)) : 0u);
      if (wq >= 0 && (mC & lt_mask) == 0 && (__ldcg(Cw + wq) & bits) != bits) atomicOr(Cw + wq, bits);
    }
  }
  if (local) {   // one addition per nonzero bucket and candidate word
    __syncwarp();
    for (int q = lane; q <= dom; q += 32) {
      const int h = hist[q];
      if (h != 0) atomicAdd(Dg + q, 0.5 * (double)h);
    }
    for (int q = lane; q < nwords; q += 32) {
      const unsigned c = hcw[q];
      if (c != 0u && (__ldcg(Cw + q) & c) != c) atomicOr(Cw + q, c);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    b2 += __shfl_xor_sync(kFull, b2, off);
    a2 += __shfl_xor_sync(kFull, a2, off);
  }
  if (lane == 0) {
    if (b2 != 0) atomicAdd(BA, 0.5 * (double)b2);
    if (a2 != 0) atomicAdd(BA + 1, 0.5 * (double)a2);
  }
}

// The end of a long bounded-integer column (after every chunk has added its part): line 14 as a scan
// of D in coalesced rounds of 32 buckets, line 16 with R4; the accumulators are zeroed for the next
// pass.
// The column's (s, x̂) in every lane (warp-cooperative); lbkt_finalize offers it.
__device__ __forceinline__ void lbkt_finalize_core(const DevProblem& P, const DevWalkers& Wk, int walker,
                                                   const LongCol& L, int lane, double& bs_out, double& bv_out,
                                                   double& xb_out) {
  const int p = L.p, dom = L.dom;
  const double* X = Wk.x + (size_t)walker * Wk.xs;
  const double xb = __ldg(X + p), l = __ldg(P.lb + p);
  double* Dg = Wk.lscr + (size_t)walker * Wk.lss + L.scr;
  double* BA = Dg + dom + 1;
  unsigned* Cw = reinterpret_cast<unsigned*>(BA + 2);
  const double B = __ldcg(BA), A = __ldcg(BA + 1);
  double carry = 0.0, bs = -INFINITY, bv = xb;
  // rounds of 32 buckets, four rounds' loads in flight at a time
  for (int b0 = 0; b0 < dom; b0 += 128) {
    double d[4];
    unsigned cw[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int q = b0 + 32 * h + lane;
      d[h] = q < dom ? __ldcg(Dg + q) : 0.0;
      cw[h] = (b0 + 32 * h < dom) ? __ldcg(Cw + ((b0 >> 5) + h)) : 0u;
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int q = b0 + 32 * h + lane;
      double incl = d[h];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += y;
      }
      const double pre = carry + incl;
      carry = __shfl_sync(kFull, pre, 31);
      if (q < dom) {
        Dg[q] = 0.0;
        const double v = l + (double)q;
        const bool cand = ((cw[h] >> lane) & 1u) || q == 0 || q == dom - 1;
        if (cand && v != xb) {   // the bounds are always candidates (R2), x̄ never
          const double sig = B + pre + (v > xb ? A : 0.0);
          if (better_shift(sig, v, bs, bv, xb)) { bs = sig; bv = v; }
        }
      }
      if (lane == 0 && b0 + 32 * h < dom) Cw[(b0 >> 5) + h] = 0u;
    }
  }
  __syncwarp();
  if (lane == 0) { BA[0] = 0.0; BA[1] = 0.0; Dg[dom] = 0.0; }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double so = __shfl_xor_sync(kFull, bs, off), vo = __shfl_xor_sync(kFull, bv, off);
    if (better_shift(so, vo, bs, bv, xb)) { bs = so; bv = vo; }
  }
  bs_out = bs;
  bv_out = bv;
  xb_out = xb;
}
__device__ __forceinline__ void lbkt_finalize(const DevProblem& P, const DevWalkers& Wk, int walker,
                                              const LongCol& L, int lane, Best& b, double* oxhat,
                                              double* oscore, long long kk, int use_tabu) {
  double bs, bv, xb;
  lbkt_finalize_core(P, Wk, walker, L, lane, bs, bv, xb);
  const int p = L.p;
  if (lane == 0)
    finish_column_j(p, __ldg(P.perm + p), use_tabu ? __ldg(Wk.tabu + (size_t)walker * Wk.ts + p) : 0, xb, bv, bs, b,
                    oxhat, oscore, kk, use_tabu, asp_ref(Wk, walker));
}

// wm_mode 1 (walker groups): the general tiles (integer and continuous) and the empty columns are
// k_eval_gen_wm's; this kernel takes the long bounded-integer chunks the groups do not take.
// with_lbin (one walker, row-wise binary mode): this kernel also takes the long binary chunks.
// Warp w of the grid takes items w, w + nwarps, ... of its range of P.gitems (long-column chunks
// first: their gathers overlap the packed tiles of other warps).
__global__ void __launch_bounds__(kGenThreads, kGenMinBlocks) k_eval_gen(DevProblem P, DevWalkers Wk, double* oxhat,
                                                                      double* oscore, int part_base, int wm_mode,
                                                                      int with_lbin, int select_parts,
                                                                      chap_move* best_out) {
  pdl_wait_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Best sm_b[kGenThreads / 32];
  __shared__ int4 s_tab[6];
  const int walker = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const WalkerScalars* sc = Wk.sc + walker;
  const double* __restrict__ X = Wk.x + (size_t)walker * Wk.xs;
  const RowView RV = row_view(Wk, walker);
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(RV.p);
  const int st = RV.st;
  const int32_t* __restrict__ TB = Wk.tabu + (size_t)walker * Wk.ts;
  const long long kk = sc->k;
  const int use_tabu = Wk.use_tabu;
  GenWarp& S = reinterpret_cast<GenWarp*>(smem)[wid];
  KT_BEGIN(Wk, 1);
  off_table_init(s_tab);
  __syncthreads();
  TileCtx C;
  C.x = X;
  C.rs = RV;
  C.tabu = TB;
  C.k = kk;
  C.use_tabu = use_tabu;
  C.oxhat = oxhat;
  C.oscore = oscore;
  C.asp = asp_ref(Wk, walker);
  Best b;
  b.init();
  const bool wint = sc->wint != 0;   // integral weights <= 2^20: the int paths
  const bool rint = sc->rint != 0;   // integral residuals: the exact float-quotient path
  // items: P.gitems = [long binary and long bounded-integer chunks, interleaved | continuous tiles |
  // general tiles | empty tiles]; without the long binary chunks (with_lbin = 0, walker groups
  // included) P.gitems2 = [long bounded-integer chunks | the same tiles]
  const WTile* __restrict__ items = with_lbin ? P.gitems : P.gitems2;
  const int ifirst = 0;
  const int iend = wm_mode ? P.n_gchunks : (with_lbin ? P.n_gitems : P.n_gitems2);
  const int nwarps = gridDim.x * (kGenThreads / 32);
  GenRound R;
  bool r_ok = false;   // R holds T's first round
  auto run_item = [&](const WTile& T, const WTile& Tn, bool has_next) {
    if (T.kind == CC_GEN) {
      if (!r_ok) R = gen_round(P, T, 4 * lane);
      if (wint) gen32_tile<true>(P, X, RS, st, TB, T, Tn, has_next, R, lane, S, rint, s_tab, b, oxhat, oscore, kk, use_tabu, C.asp);
      else gen32_tile<false>(P, X, RS, st, TB, T, Tn, has_next, R, lane, S, rint, s_tab, b, oxhat, oscore, kk, use_tabu, C.asp);
      r_ok = has_next && Tn.kind == CC_GEN;
    } else if (T.kind == CC_LBKT) {
      if (wm_mode && Wk.lbkt_wm) return;   // walker groups: k_eval_gen_wm takes the chunk for the group
      const LongCol L = P.lcols[T.e1];
      if (wint) lbkt_chunk<true>(P, Wk, walker, X, RS, st, T, L, lane, reinterpret_cast<unsigned char*>(&S), rint, s_tab);
      else lbkt_chunk<false>(P, Wk, walker, X, RS, st, T, L, lane, reinterpret_cast<unsigned char*>(&S), rint, s_tab);
      if (long_last(Wk, walker, L, lane)) lbkt_finalize(P, Wk, walker, L, lane, b, oxhat, oscore, kk, use_tabu);
    } else if (T.kind == CC_LBIN) {
      lbin_chunk(P, Wk, walker, X, RS, TB, T, lane, b, oxhat, oscore, kk, use_tabu, P.rint_base && wint);
    } else if (T.kind == CC_GENC) {
      if (lane < T.ncols) {
        const int p = T.p0 + lane;
        double v, sv;
        gen_column_serial(P, X, RS, st, p, v, sv);
        offer_column(p, __ldg(P.perm + p), TB, __ldg(X + p), v, sv, b, oxhat, oscore, kk, use_tabu, C.asp);
      }
    } else {
      wtile_empty(P, C, T, lane, b);
    }
    __syncwarp();
  };
  const int t0 = ifirst + blockIdx.x * (kGenThreads / 32) + wid;
  if (Wk.dirty) {
    // f2: the warp's items 32 at a time, lane l testing item l (one round of loads for 32 items);
    // only the items with a dirty column are evaluated, the others keep their cached results
    for (int base = t0; base < iend; base += 32 * nwarps) {
      const int tl = base + lane * nwarps;
      WTile Tl;
      bool dl = false;
      if (tl < iend) {
        Tl = items[tl];
        dl = cols_dirty(Wk, kk, Tl.p0, (Tl.kind == CC_LBKT || Tl.kind == CC_LBIN) ? 1 : (int)Tl.ncols);
      }
      for (unsigned m = __ballot_sync(kFull, dl); m; m &= m - 1) {
        const int q = __ffs(m) - 1;
        WTile T;
        T.p0 = __shfl_sync(kFull, Tl.p0, q);
        T.e0 = __shfl_sync(kFull, Tl.e0, q);
        T.e1 = __shfl_sync(kFull, Tl.e1, q);
        T.ncols = (int16_t)__shfl_sync(kFull, (int)Tl.ncols, q);
        T.kind = (int8_t)__shfl_sync(kFull, (int)Tl.kind, q);
        r_ok = false;
        run_item(T, T, false);
      }
    }
  } else {
    // one walker: items handed out in list order by a counter (long-column chunks first, then the
    // tiles), the first item of every warp static; a warp takes its next item while it evaluates the
    // current one. Several walkers (fewer blocks each): the static round-robin, t += nwarps.
    const bool dyn = gridDim.y == 1;
    unsigned* gctr = Wk.gen_ctr + 2 * walker;
    auto next_item = [&](int t) {
      if (!dyn) return t + nwarps;
      unsigned v = 0u;
      if (lane == 0) v = atomicAdd(gctr, 1u);
      return ifirst + nwarps + (int)__shfl_sync(kFull, v, 0);
    };
    int t = t0;
    WTile T;
    if (t < iend) T = items[t];
    while (t < iend) {
      const int tn = next_item(t);
      const bool has_next = tn < iend;
      WTile Tn;
      if (has_next) Tn = items[tn];
      run_item(T, Tn, has_next);
      T = Tn;
      t = tn;
    }
  }
  b = block_reduce_best(b, sm_b);
  if (!Wk.dirty && gridDim.y == 1 && threadIdx.x == 0) {   // every warp of the block is past its last
    __threadfence();   // grab: the last block re-arms the walker's item counter for the next launch
    unsigned* gctr = Wk.gen_ctr + 2 * walker;
    if (atomicAdd(gctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(gctr, 0u);
      atomicExch(gctr + 1, 0u);
    }
  }
  if (threadIdx.x == 0) write_part(Wk.part + (size_t)walker * Wk.ps + part_base + blockIdx.x, b);
  KT_END(Wk, 1);
  if (select_parts <= 0) return;   // as in k_eval_bin: the last eval kernel selects
  __shared__ int s_flag;
  if (!last_chunk(Wk.sel_count + walker, gridDim.x, &s_flag)) return;
  select_walker(P, Wk, walker, select_parts, sm_b, best_out, X);
  KT_END(Wk, 1);
}

// ------------------------------------------------------------------------------------------
// walker-minor general kernel (row-state groups of rg > 1 walkers)
// ------------------------------------------------------------------------------------------
// One warp evaluates a packed integer general column for a whole walker group: lane = (slot,
// walker), the 32 / RG slots take different columns of the tile. Every lane runs Algorithm 1 for
// its own walker serially: lines 3-11 per entry (the CSC entry is read once for the group, the
// row-state read is a coalesced RG x 16-byte run) into its own shared-memory column of (key, δ),
// then lines 13-16 sort-free: σ(v) = β + α [v > x̄] + Σ_e δ_e [key_e <= v] for every
// candidate v (emitted breakpoints in [l, u] other than x̄, and the finite bounds; R2, R3, R5),
// argmax with R4. No cross-lane coordination: the lanes of a slot do identical control flow on
// different walkers. Sums of ±w, ±w/2 in double are exact (R11), so the scores equal the per-walker
// kernels' bit for bit.
#ifndef CHAP_GENWM_THREADS
#define CHAP_GENWM_THREADS 128
#endif
constexpr int kGenWmThreads = CHAP_GENWM_THREADS;
#ifndef CHAP_WM_ROUND
#define CHAP_WM_ROUND 4   // entries per round of loads in wm_off_column
#endif
// The integer path of k_eval_gen_wm for one packed general column of lane (slot, walker): lines
// 3-11 by off_entry (gen32_tile's table and float-quotient offsets) into the lane's shared-memory
// column (lane-interleaved int2 [k][32]) with pass 0 fused into the emission, then offsets_best
// over the reduced candidate set. Returns false when an offset is beyond the int path
// (the caller re-evaluates the column in double).
template <bool INTW, int RG>
__device__ __forceinline__ bool wm_off_column(const DevProblem& P, const double2* __restrict__ RS, int cb, int k,
                                              double xb, double l, double u, bool rint,
                                              const int4* __restrict__ tab, int2* __restrict__ sent, int lane,
                                              double& bs, double& bv) {
  using Acc = typename std::conditional<INTW, int, double>::type;
  auto fv = [](int bits) -> Acc { if (INTW) return (Acc)bits; else return (Acc)__int_as_float(bits); };
  const bool ufin = isfinite(u), lfin = isfinite(l);
  const double hid = u - xb, lod = l - xb;
  const int hi = ufin ? (int)fmin(hid, (double)kKeyLim) : kKeyLim;
  const int lo = lfin ? (int)fmax(lod, -(double)kKeyLim) : -kKeyLim;
  int vup = (ufin && hi > 0) ? hi : INT_MAX;
  int vdn = (lfin && lo < 0) ? lo : INT_MIN;
  int c2 = INT_MIN, c3 = INT_MIN, c4 = INT_MIN, c5 = INT_MIN, c6 = INT_MIN, c7 = INT_MIN, nstep = 0;
  Acc b2 = 0, a2 = 0;
  bool ovf = false;
  for (int e0 = 0; e0 < k; e0 += CHAP_WM_ROUND) {
    int id[CHAP_WM_ROUND];
    double av[CHAP_WM_ROUND];
    double2 rv[CHAP_WM_ROUND];
#pragma unroll
    for (int q = 0; q < CHAP_WM_ROUND; ++q) {
      id[q] = e0 + q < k ? __ldg(P.row_idx + cb + e0 + q) : -1;
      av[q] = e0 + q < k ? __ldg(P.val + cb + e0 + q) : 1.0;
    }
#pragma unroll
    for (int q = 0; q < CHAP_WM_ROUND; ++q) rv[q] = id[q] >= 0 ? __ldg(RS + (size_t)id[q] * RG) : make_double2(-INFINITY, 0.0);
#pragma unroll
    for (int q = 0; q < CHAP_WM_ROUND; ++q) {
      const int e = e0 + q;
      if (e >= k) break;
      const int4 E = off_entry<INTW>(rv[q].x, __int_as_float((int)__double2loint(rv[q].y)), av[q], rint, tab, ovf);
      b2 += fv(E.z);
      a2 += fv(E.w);
      off_pass0(E.x, hi, lo, vup, vdn, c2, c3, c4, c5, c6, c7, nstep);
      sent[e * 32 + lane] = make_int2(E.x, E.y);
    }
  }
  if (ovf) return false;
  Acc bs2;
  int bo;
  const bool have = offsets_best<INTW>([&](int e) { return sent[e * 32 + lane]; }, 0, k, b2, a2, hi, lo, vup, vdn, c2,
                                       c3, c4, c5, c6, c7, nstep, bs2, bo);
  bs = -INFINITY;
  bv = xb;
  if (have) {
    bs = 0.5 * (double)bs2;
    // a bound beyond the clamp is the farthest candidate of its side: its exact value
    bv = (bo == hi && ufin && hid > (double)kKeyLim) ? u : ((bo == lo && lfin && lod < -(double)kKeyLim) ? l : xb + (double)bo);
  }
  return true;
}

// per warp: kmax x 32 int2 (off_entry key and δ words) for the tiles, or lbkt_words ints for a long
// chunk's histograms (DevWalkers::lbkt_wm), whichever is larger (16-byte multiple)
__host__ __device__ constexpr size_t gen_wm_region(int kmax, int lbkt_words) {
  return (((size_t)kmax * 32 * sizeof(int2) > (size_t)lbkt_words * 4 ? (size_t)kmax * 32 * sizeof(int2)
                                                                       : (size_t)lbkt_words * 4) + 15) / 16 * 16;
}
__host__ __device__ constexpr size_t gen_wm_smem_all(int kmax, int lbkt_words) {
  return (size_t)(kGenWmThreads / 32) * gen_wm_region(kmax, lbkt_words);
}
template <int RG>
#ifndef CHAP_GENWM_MINB
#define CHAP_GENWM_MINB 5   // 5 blocks per SM (96 registers): 1.26 vs 1.85 ms at 1 (128 registers) on G-32
#endif
__global__ void __launch_bounds__(kGenWmThreads, CHAP_GENWM_MINB) k_eval_gen_wm(DevProblem P, DevWalkers Wk, int part_base, int kmax) {
  pdl_wait_trigger();
  constexpr int NS = 32 / RG;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Best sb[kGenWmThreads / 32][32];
  const int g = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wl = lane % RG, slot = lane / RG;
  const int w = g * RG + wl;
  const bool live = w < Wk.W;
  const int wr = live ? w : g * RG;
  // this warp's region of shared memory: the tiles' off_entry columns, or a long chunk's histograms
  unsigned char* wreg = smem + (size_t)wid * gen_wm_region(kmax, Wk.lbkt_wm_words);
  int2* sent = reinterpret_cast<int2*>(wreg);   // [kmax][32]
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(Wk.rs + (size_t)g * Wk.rss * RG) + wl;
  const double* __restrict__ X = Wk.x + (size_t)wr * Wk.xs;
  const int32_t* __restrict__ TB = Wk.tabu + (size_t)wr * Wk.ts;
  const long long kk = Wk.sc[wr].k;
  const int use_tabu = Wk.use_tabu;
  KT_BEGIN(Wk, 1);
  Best b;
  b.init();
  const AspRef A = asp_ref(Wk, wr);
  auto offer = [&](double sc, double v, int j, int p) {
    const bool bm = better_move(sc, j, b.s, b.j);
    if (!bm && !(A.a && sc > 0.0)) return;
    if (use_tabu) {
      const int32_t tp = __ldg(TB + p);
      if ((long long)tp > kk) {
        if (live) asp_note(A, p, j, tp, v, sc);
        return;
      }
    }
    if (!bm) return;
    b.s = sc;
    b.v = v;
    b.j = j;
    b.p = p;
  };
  const int nwarps = gridDim.x * (kGenWmThreads / 32);
  // a10: the long bounded-integer chunks for the whole group. The chunk's CSC entries are read once
  // for the group, lane (slot, walker) takes entries slot, slot + NS, ... of its walker (one coalesced
  // RG x 16-byte row-state read per entry), counts F into a lane-private int32 histogram in this
  // warp's shared memory ([bucket][lane], conflict-free) and adds it to its walker's accumulators;
  // the walkers whose ticket completes are finished by the warp, one after the other.
  const int ng = Wk.lbkt_wm ? P.n_gchunks : 0;
  __shared__ int4 s_tab[6];
  off_table_init(s_tab);
  __syncthreads();
  // the integer path of the tiles: every walker of the warp with integral weights <= 2^20 (INTW)
  const bool wint_all = __all_sync(kFull, Wk.sc[wr].wint != 0);
  const bool rint_l = Wk.sc[wr].rint != 0;
  if (ng > 0) {
    int* hist = reinterpret_cast<int*>(wreg);   // [dom + 1][32] ints, then the candidate words
    for (int t = blockIdx.x * (kGenWmThreads / 32) + wid; t < ng; t += nwarps) {
      const WTile T = P.gchunks[t];
      const LongCol L = P.lcols[T.e1];
      const int p = T.p0, dom = L.dom, len = T.ncols, nwords = (dom + 31) >> 5;
      unsigned* hcw = reinterpret_cast<unsigned*>(hist + (dom + 1) * 32);   // [nwords][32]
      for (int q = 0; q <= dom; ++q) hist[q * 32 + lane] = 0;
      for (int q = 0; q < nwords; ++q) hcw[q * 32 + lane] = 0u;
      const int xl = (int)(__ldg(X + p) - __ldg(P.lb + p));
      const bool rint = Wk.sc[wr].rint != 0;
      int b2 = 0, a2 = 0;
      bool ovf = false;
      for (int k = slot; k < len; k += NS) {
        const int i = __ldg(P.row_idx + T.e0 + k);
        const double a = __ldg(P.val + T.e0 + k);
        const double2 rv = __ldg(RS + (size_t)i * RG);
        const int4 E = off_entry<true>(rv.x, __int_as_float((int)__double2loint(rv.y)), a, rint, s_tab, ovf);
        b2 += E.z;
        a2 += E.w;
        const int code = E.x & 7, key = E.x >> 3;
        if (code == 2) continue;
        const int bk = key + xl, cv = key - (code & 1) + xl;
        if (bk < 0) b2 += E.y;                          // below l: in every prefix
        else if (bk < dom) hist[bk * 32 + lane] += E.y;
        if (cv >= 0 && cv < dom) hcw[(cv >> 5) * 32 + lane] |= 1u << (cv & 31);
      }
      double* Dg = Wk.lscr + (size_t)wr * Wk.lss + L.scr;
      double* BA = Dg + dom + 1;
      unsigned* Cw = reinterpret_cast<unsigned*>(BA + 2);
      if (live) {
        for (int q = 0; q <= dom; ++q) {
          const int h = hist[q * 32 + lane];
          if (h != 0) atomicAdd(Dg + q, 0.5 * (double)h);
        }
        for (int q = 0; q < nwords; ++q) {
          const unsigned c = hcw[q * 32 + lane];
          if (c != 0u && (__ldcg(Cw + q) & c) != c) atomicOr(Cw + q, c);
        }
        if (b2 != 0) atomicAdd(BA, 0.5 * (double)b2);
        if (a2 != 0) atomicAdd(BA + 1, 0.5 * (double)a2);
      }
      __syncwarp();
      // per-walker ticket (slot 0 lanes), acquire-release at gpu scope (see long_last)
      unsigned last = 0u;
      if (slot == 0 && live) {
        unsigned* tk = reinterpret_cast<unsigned*>(Wk.lscr + (size_t)w * Wk.lss + L.tix);
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(tk) : "memory");
        last = old == (unsigned)(L.nchunks - 1);
        if (last) *tk = 0u;
      }
      for (unsigned m = __ballot_sync(kFull, last != 0u); m; m &= m - 1) {
        const int wq = __ffs(m) - 1;   // slot 0: lane == walker-in-group
        double fs, fv, fx;
        lbkt_finalize_core(P, Wk, g * RG + wq, L, lane, fs, fv, fx);
        if (lane == wq) offer(fs, fs == -INFINITY ? fx : fv, __ldg(P.perm + p), p);
      }
      __syncwarp();
    }
  }
  for (int t = blockIdx.x * (kGenWmThreads / 32) + wid; t < P.n_wtiles; t += nwarps) {
    const WTile T = P.wtiles[t];
    for (int c = slot; c < T.ncols; c += NS) {
      const int p = T.p0 + c;
      const double xb = __ldg(X + p), l = __ldg(P.lb + p), u = __ldg(P.ub + p);
      const int j = __ldg(P.perm + p);
      if (T.kind == CC_GENC) {   // a continuous column: Algorithm 1 serially in double, per walker of
        double v2, s2;           // the group (its entries read once per group through L1)
        gen_column_serial(P, X, RS, RG, p, v2, s2);
        if (live) offer(s2, s2 == -INFINITY ? xb : v2, j, p);
        continue;
      }
      double bs = -INFINITY, bv = xb;
      if (T.kind != CC_GEN) {   // a column without nonzeros (R2, R4, R5)
        if (__ldg(P.vclass + p) == 1) {
          bs = 0.0;
          bv = 1.0 - xb;
        } else {
          if (isfinite(l) && l != xb) { bs = 0.0; bv = l; }
          if (isfinite(u) && u != xb && better_shift(0.0, u, bs, bv, xb)) { bs = 0.0; bv = u; }
        }
        if (live) offer(bs, bv, j, p);
        continue;
      }
      const int cb = __ldg(P.col_ptr + p), k = __ldg(P.col_ptr + p + 1) - cb;
      {
        double s1, v1;
        const bool ok = wint_all ? wm_off_column<true, RG>(P, RS, cb, k, xb, l, u, rint_l, s_tab, sent, lane, s1, v1)
                                 : wm_off_column<false, RG>(P, RS, cb, k, xb, l, u, rint_l, s_tab, sent, lane, s1, v1);
        if (ok) {
          if (live) offer(s1, v1, j, p);
          continue;
        }
      }
      // an offset beyond the int path: the column in double (Algorithm 1 serially, no shared memory)
      {
        double v2, s2;
        gen_column_serial(P, X, RS, RG, p, v2, s2);
        if (live) offer(s2, s2 == -INFINITY ? xb : v2, j, p);
      }
    }
  }
  // per-walker block best: slots, then warps, in fixed order
  sb[wid][lane] = b;
  __syncthreads();
  if (threadIdx.x < RG) {
    Best o;
    o.init();
    for (int q = 0; q < kGenWmThreads / 32; ++q)
      for (int sl = 0; sl < NS; ++sl) o.take(sb[q][sl * RG + threadIdx.x]);
    const int ww = g * RG + threadIdx.x;
    if (ww < Wk.W) write_part(Wk.part + (size_t)ww * Wk.ps + part_base + blockIdx.x, o);
  }
  KT_END(Wk, 1);
}

// ------------------------------------------------------------------------------------------
// k_eval: long-column ends, single-column sort tiles, the global select
// ------------------------------------------------------------------------------------------
// grid = (blocks per walker, W). After its tiles every block publishes its best admissible move;
// the last block of the walker reduces them (fixed order) to the decision.
__global__ void __launch_bounds__(kTileThreads, 3) k_eval(DevProblem P, DevWalkers Wk, double* oxhat,
                                                          double* oscore, chap_move* best_out,
                                                          int part_base, int fin_lbin) {
  pdl_wait_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sm_red[32];
  __shared__ Best sm_b[32];
  __shared__ int s_flag;
  const int walker = blockIdx.y;
  const WalkerScalars* sc = Wk.sc + walker;
  KT_BEGIN(Wk, 2);
  TileCtx C;
  C.x = Wk.x + (size_t)walker * Wk.xs;
  C.rs = row_view(Wk, walker);
  C.tabu = Wk.tabu + (size_t)walker * Wk.ts;
  C.k = sc->k;
  C.use_tabu = Wk.use_tabu;
  C.oxhat = oxhat;
  C.oscore = oscore;
  C.asp = asp_ref(Wk, walker);
  Best b;
  b.init();
  // long binary columns of walker groups (k_eval_bin_wm takes no chunk tickets), finished after all
  // their chunks; every other long column is finished by the chunk that takes its last ticket
  if (fin_lbin && (threadIdx.x & 31) == 0) {
    const int nw = gridDim.x * (blockDim.x >> 5), w0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int q = w0; q < P.n_lfin; q += nw) {
      const LongCol L = P.lcols[P.lfin[q]];
      if (L.kind == CC_LBIN) lbin_finalize(P, Wk, walker, L, b, oxhat, oscore, C.k, C.use_tabu);
    }
  }
  // long general columns sorted grid-wide (k_sort_chunks, k_sort_rank ran before this kernel)
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P.n_scols; q += gridDim.x * blockDim.x)
    if (cols_dirty(Wk, C.k, P.scols[q].p, 1)) sortcol_finish(P, Wk, walker, P.scols[q], b, oxhat, oscore, C.k, C.use_tabu);
  // block tiles: single-column sorts
  for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x)
    if (cols_dirty(Wk, C.k, P.tiles[t].p0, 1))
      tile_genm(P, C, P.tiles[t], *reinterpret_cast<SmemGenM*>(smem), sm_red, sm_b, b);
  __syncthreads();
  // publish the block's best; the last block of this walker selects (R6)
  b = block_reduce_best(b, sm_b);
  Cand* part = Wk.part + (size_t)walker * Wk.ps;
  if (threadIdx.x == 0) write_part(part + part_base + blockIdx.x, b);
  KT_END(Wk, 2);
  if (Wk.cs) return;   // f2: k_select_cache selects from the cached results
  if (!last_chunk(Wk.sel_count + walker, gridDim.x, &s_flag)) return;
  select_walker(P, Wk, walker, part_base + (int)gridDim.x, sm_b, best_out, C.x);
  KT_END(Wk, 2);
}

// f2 (chap_params.lazy, one walker): the best admissible move (R6, R13; aspiration notes, R18) over
// the cached per-column results: the columns evaluated this iteration (dirty) and the clean ones,
// whose cached (s_j, x̂_j) is unchanged because neither x̄_j nor any row state of the column changed.
__global__ void __launch_bounds__(kTileThreads) k_select_cache(DevProblem P, DevWalkers Wk) {
  pdl_wait_trigger();
  __shared__ Best sm_b[32];
  __shared__ int s_flag;
  const long long kk = Wk.sc[0].k;
  const AspRef A = asp_ref(Wk, 0);
  Best b;
  b.init();
  for (int p = P.n_fixed + blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    const double s = __ldcg(Wk.cs + p);
    if (s == -INFINITY) continue;
    const int j = __ldg(P.perm + p);
    const bool bm = better_move(s, j, b.s, b.j);
    if (!bm && !(A.a && s > 0.0)) continue;
    if (Wk.use_tabu) {
      const int32_t tp = Wk.tabu[p];
      if ((long long)tp > kk) {
        asp_note(A, p, j, tp, __ldcg(Wk.cv + p), s);
        continue;
      }
    }
    if (!bm) continue;
    b.s = s;
    b.v = __ldcg(Wk.cv + p);
    b.j = j;
    b.p = p;
  }
  b = block_reduce_best(b, sm_b);
  if (threadIdx.x == 0) write_part(Wk.part + blockIdx.x, b);
  if (!last_chunk(Wk.sel_count, gridDim.x, &s_flag)) return;
  select_walker(P, Wk, 0, (int)gridDim.x, sm_b, nullptr, Wk.x);
}

// f2: every column of both dirty sets (walker create, restart, an external cutoff).
__global__ void k_dirty_all(DevWalkers Wk, int only_walker) {
  if (skip_walker(Wk.rmask, only_walker, 0)) return;   // (selective re-evaluation runs one walker)
  if (Wk.dirty && threadIdx.x < 2) Wk.dirty[(size_t)threadIdx.x * (Wk.dwords + 1) + Wk.dwords] = 1u;
}

// Outputs of fixed variables (internal [0, n_fixed)): (x̄, -inf) (R2 leaves no candidate).
__global__ void k_fixed_out(DevProblem P, const double* x, double* oxhat, double* oscore) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n_fixed; p += gridDim.x * blockDim.x) {
    const int j = P.perm[p];
    if (oxhat) oxhat[j] = x[p];
    if (oscore) oscore[j] = -INFINITY;
  }
}

}  // namespace chap

// eval.cuh — best-shift evaluation (§3.1, Eq. (1) and Algorithm 1) on sm_100a.
//
// One persistent kernel, k_eval, evaluates every variable of every walker and selects the best
// admissible move (the paper's length-specialised dispatch, re-designed):
//   phase A, block tiles (all warps of a block):
//     CC_LBIN  a kTileNnz chunk of a long binary column: block partial flip sum;
//     CC_LBKT  a chunk of a general integer column with a bounded domain: the sort of line 13
//              becomes a counting (bucket) pass over [l, u];
//     CC_GENM  one general column of <= kGenmMax entries: shared-memory bitonic sort + scan;
//     the last chunk of a column merges the chunk partials in chunk order (deterministic);
//   phase B, warp tiles (one warp, no block barriers):
//     CC_BIN   packed binary columns: flip penalty per nonzero, per-column sum;
//     CC_GEN   packed general columns: Algorithm 1 per column, sort-free (see wtile_gen);
//     CC_EMPTY columns without nonzeros.
// Every warp-tile slot issues its coalesced CSC loads and one 16-byte row-state gather before
// using any of them. Each block keeps its best admissible move (R6); the last block of a walker
// reduces the block partials to the walker's decision (the global select).
#pragma once
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

// The result of one column: outputs (eval API) and the admissible-best update (R6, R13).
__device__ __forceinline__ void finish_column_j(int p, int j, int32_t tabu_p, double xb, double v,
                                                double s, Best& b, double* oxhat, double* oscore,
                                                long long k, int use_tabu) {
  if (s == -INFINITY) v = xb;
  if (oxhat) oxhat[j] = v;
  if (oscore) oscore[j] = s;
  if (use_tabu && (long long)tabu_p > k) return;
  if (better_move(s, j, b.s, b.j)) {
    b.s = s;
    b.v = v;
    b.j = j;
    b.p = p;
  }
}
__device__ __forceinline__ void finish_column(const DevProblem& P, int p, double xb, double v,
                                              double s, Best& b, double* oxhat, double* oscore,
                                              const int32_t* tabu, long long k, int use_tabu) {
  finish_column_j(p, P.perm[p], use_tabu ? tabu[p] : 0, xb, v, s, b, oxhat, oscore, k, use_tabu);
}

// One 16-byte row-state gather (r f64, w f32). The inactive cutoff row holds r = -inf, w = 0,
// which makes every one of its contributions vanish (no per-nonzero test needed).
__device__ __forceinline__ void load_row(const RowState* rs, int i, double& r, double& w) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(rs) + i);
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
struct WarpBin {                       // CC_BIN warp tile
  double pen[kWTileNnz];
  double xb[kWTileCols];
  uint32_t head[kWTileNnz / 32];       // bit k: slot k starts a column
};
struct WarpGen {                       // CC_GEN warp tile: row entries at slots [0, nnz); the
  double key[kWTileGen];               // bound entries of column c at slots nnz + 2c, nnz + 2c + 1
  double D[kWTileGen];                 // entry delta (0 for bound / dropped entries)
  union {
    float2 AB[kWTileGen];              // phases 1-2: the entry's contributions to β and α
    double sig[kWTileGen];             // phases 3-4: sigma of candidate slots
  };
  uint8_t f[kWTileGen];                // GF_* flags
  uint8_t seg[kWTileGen];              // column of a row slot
  double xb[kWTileCols];
  double l[kWTileCols];
  double u[kWTileCols];
  double beta[kWTileCols];
  double alpha[kWTileCols];
  int32_t cb[kWTileCols];
  int32_t ce[kWTileCols];
  uint32_t head[kWTileGen / 32];
  uint8_t cont[kWTileCols];            // continuous column
};
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t kWarpSmem = (cmax(sizeof(WarpBin), sizeof(WarpGen)) + 15) / 16 * 16;
struct SmemGenM {                      // CC_GENM block tile
  double t[kGenmMax];
  double del[kGenmMax];
  double P[kGenmMax];
  uint32_t mk[kGenmMax];
};
struct SmemBkt {                       // CC_LBKT block tile
  double D[kBucketMax + 1];
  uint8_t cand[kBucketMax];
};
constexpr size_t kTileSmem = cmax(kWarpSmem * kTileWarps, cmax(sizeof(SmemGenM), sizeof(SmemBkt)));

struct TileCtx {
  const double* x;
  const RowState* rs;
  const int32_t* tabu;
  long long k;
  int use_tabu;
  double* oxhat;
  double* oscore;
};

// ------------------------------------------------------------------------------------------
// warp tiles
// ------------------------------------------------------------------------------------------

// Column of slot k = lane + 32 q of a packed tile: columns are contiguous runs of slots and
// none is empty, so the column is (number of column starts <= k) - 1, read off a head bitmap.
__device__ __forceinline__ void build_heads(uint32_t* head, int nwords, int lane, int nc, int cb) {
  if (lane < nwords) head[lane] = 0u;
  __syncwarp();
  if (lane < nc) atomicOr(&head[cb >> 5], 1u << (cb & 31));
  __syncwarp();
}

// packed binary columns, one warp (the only move of a binary is the flip).
// Memory round trips per tile: (stream loads || column loads) -> gathers; all kWSlots slots of a
// lane are issued together.
__device__ __forceinline__ void wtile_bin(const DevProblem& P, const TileCtx& C, const WTile& T,
                                          int lane, WarpBin& S, Best& b) {
  const int nc = T.ncols, nnz = T.e1 - T.e0;
  const int* __restrict__ ridx = P.row_idx + T.e0;
  const double* __restrict__ rval = P.val + T.e0;
  int idx[kWSlots];
  double av[kWSlots];
#pragma unroll
  for (int q = 0; q < kWSlots; ++q) {
    const int k = lane + 32 * q;
    const bool ok = k < nnz;
    idx[q] = ok ? __ldcs(ridx + k) : 0;
    av[q] = ok ? __ldcs(rval + k) : 0.0;
  }
  const int p = T.p0 + lane;
  int cb = 0, ce = 0, j = 0, tb = 0;
  double xb = 0.0;
  if (lane < nc) {
    cb = __ldg(P.col_ptr + p) - T.e0;
    ce = __ldg(P.col_ptr + p + 1) - T.e0;
    j = __ldg(P.perm + p);
    tb = C.use_tabu ? __ldg(C.tabu + p) : 0;
    xb = __ldg(C.x + p);
  }
  double r[kWSlots], w[kWSlots];
#pragma unroll
  for (int q = 0; q < kWSlots; ++q) load_row(C.rs, idx[q], r[q], w[q]);
  if (lane < nc) S.xb[lane] = xb;
  build_heads(S.head, kWSlots, lane, nc, cb);
  const unsigned le = (2u << lane) - 1u;   // lanes <= lane
  int pre = 0;                             // column starts before this slot round
#pragma unroll
  for (int q = 0; q < kWSlots; ++q) {
    const int k = lane + 32 * q;
    const uint32_t hw = S.head[q];
    const int c = pre + __popc(hw & le) - 1;
    pre += __popc(hw);
    if (k < nnz) S.pen[k] = penalty(w[q], r[q], r[q] + av[q] * (1.0 - 2.0 * S.xb[c]));
  }
  __syncwarp();
  if (lane < nc) {
    double s = 0.0;
    for (int e = cb; e < ce; ++e) s += S.pen[e];
    finish_column_j(p, j, tb, xb, 1.0 - xb, s, b, C.oxhat, C.oscore, C.k, C.use_tabu);
  }
  __syncwarp();
}

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

// Packed general columns, one warp: Algorithm 1 per column, sort-free.
// For a candidate value v the score Algorithm 1 reports (the largest sigma of the entries at v,
// R3) is sigma(v) = β + Σ_{entries e: t_e < v, or t_e = v with marker -1} δ_e + α [v > x̄]
// (DESIGN §2.3). A marker +1 entry has δ <= 0 and a marker -1 entry δ >= 0, and an entry with
// δ = 0 adds nothing, so "marker -1" is δ > 0; for integer columns the condition is the single
// compare key_e <= 2v with key_e = 2 t_e + [δ_e < 0] (exact while |t| < 2^51); continuous columns
// compare (t, δ > 0) directly. Phases:
//  (1) slots in parallel: coalesced CSC loads and row-state gathers issued together, then lines
//      3-11 per entry: t, the emission case, δ, the β/α contributions and the key;
//  (2) lane c: β and α of column c (lines 1-12 accumulators, fixed order);
//  (3) candidate slots in parallel: sigma by a compare-add pass over the column's entries
//      (lines 13-15: the sort and scan, done as direct prefix sums);
//  (4) lane c: the argmax of line 16 with the R4 tie-break.
__device__ __forceinline__ void wtile_gen(const DevProblem& P, const TileCtx& C, const WTile& T,
                                          int lane, WarpGen& S, Best& b) {
  const int nc = T.ncols, nnz = T.e1 - T.e0;
  const int nel = nnz + 2 * nc;
  const int* __restrict__ ridx = P.row_idx + T.e0;
  const double* __restrict__ rval = P.val + T.e0;
  const int p = T.p0 + lane;
  int cb = 0, ce = 0, j = 0, tb = 0;
  double xb = 0.0;
  if (lane < nc) {
    cb = __ldg(P.col_ptr + p) - T.e0;
    ce = __ldg(P.col_ptr + p + 1) - T.e0;
    j = __ldg(P.perm + p);
    tb = C.use_tabu ? __ldg(C.tabu + p) : 0;
    xb = __ldg(C.x + p);
    S.xb[lane] = xb;
    S.l[lane] = __ldg(P.lb + p);
    S.u[lane] = __ldg(P.ub + p);
    S.cont[lane] = __ldg(P.vclass + p) == 3;
    S.cb[lane] = cb;
    S.ce[lane] = ce;
  }
  build_heads(S.head, kWSlotsGen, lane, nc, cb);
  // (1) lines 3-11, in two halves of kWSlotsGen/2 loads + gathers in flight
  const unsigned le = (2u << lane) - 1u;
  int pre = 0;
  constexpr int H = kWSlotsGen / 2;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    int idx[H];
    double av[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const int k = lane + 32 * (q + h * H);
      const bool ok = k < nnz;
      idx[q] = ok ? __ldcs(ridx + k) : 0;
      av[q] = ok ? __ldcs(rval + k) : 1.0;
    }
    double r[H], w[H];
#pragma unroll
    for (int q = 0; q < H; ++q) load_row(C.rs, idx[q], r[q], w[q]);
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const int qq = q + h * H;
      const int k = lane + 32 * qq;
      const uint32_t hw = S.head[qq];
      const int cr = pre + __popc(hw & le) - 1;
      pre += __popc(hw);
      if (k >= nel) continue;
      double key = 0.0, D = 0.0;
      float A = 0.f, B = 0.f;
      uint8_t f = 0;
      if (k < nnz) {
        const int c = cr;
        const double x = S.xb[c];
        const bool cont = S.cont[c];
        double t = breakpoint(x, r[q], av[q]);                     // line 3
        if (!cont) t = (av[q] > 0.0) ? floor(t) : ceil(t);         // line 4
        const bool pos = av[q] > 0.0, lt = x < t, gt = x > t;      // lines 5-11
        const double wq = w[q], hw2 = 0.5 * wq;
        D = pos ? (gt ? -hw2 : (lt ? -wq : 0.0)) : (lt ? hw2 : (gt ? wq : 0.0));
        A = (float)(pos ? (gt ? wq : 0.0) : (lt ? -hw2 : -wq));
        B = (float)(pos ? (lt ? 0.0 : -wq) : (gt ? 0.0 : wq));
        key = cont ? t : 2.0 * t + (D < 0.0 ? 1.0 : 0.0);
        if (x != t && t >= S.l[c] && t <= S.u[c]) f = GF_CAND;
        if (!isfinite(r[q])) { D = 0.0; A = B = 0.f; f = 0; }     // inert inactive cutoff row
        S.seg[k] = (uint8_t)c;
        S.AB[k] = make_float2(A, B);
      } else {
        const int c = (k - nnz) >> 1;
        const double v = ((k - nnz) & 1) ? S.u[c] : S.l[c];
        key = S.cont[c] ? v : 2.0 * v;                             // the candidate value, encoded
        if (isfinite(v) && v != S.xb[c]) f = GF_CAND;
      }
      S.key[k] = key;
      S.D[k] = D;
      S.f[k] = f;
    }
  }
  __syncwarp();
  // (2) β, α of column `lane`
  if (lane < nc) {
    double beta = 0.0, alpha = 0.0;
    for (int e = cb; e < ce; ++e) {
      const float2 ab = S.AB[e];
      beta += (double)ab.x;
      alpha += (double)ab.y;
    }
    S.beta[lane] = beta;
    S.alpha[lane] = alpha;
  }
  __syncwarp();
  // (3) sigma of every candidate slot
#pragma unroll 1
  for (int q = 0; q < kWSlotsGen; ++q) {
    const int k = lane + 32 * q;
    if (k >= nel || !(S.f[k] & GF_CAND)) continue;
    const int c = (k < nnz) ? S.seg[k] : ((k - nnz) >> 1);
    const bool cont = S.cont[c];
    const double kv = S.key[k];
    // the candidate's value and its "minus" key 2v
    const double v = cont ? kv : floor(0.5 * kv);
    const double km = cont ? kv : 2.0 * v;
    const int e0 = S.cb[c], e1 = S.ce[c];
    double acc = S.beta[c] + (v > S.xb[c] ? S.alpha[c] : 0.0);
    if (!cont) {
      for (int e = e0; e < e1; ++e) acc += (S.key[e] <= km) ? S.D[e] : 0.0;
    } else {
      for (int e = e0; e < e1; ++e) {
        const double te = S.key[e], de = S.D[e];
        acc += (te < v || (te == v && de > 0.0)) ? de : 0.0;
      }
    }
    S.sig[k] = acc;
  }
  __syncwarp();
  // (4) argmax per column (R3, R4)
  if (lane < nc) {
    const bool cont = S.cont[lane];
    double bs = -INFINITY, bv = xb;
    for (int e = cb; e < ce + 2; ++e) {
      const int k = (e < ce) ? e : nnz + 2 * lane + (e - ce);
      if (!(S.f[k] & GF_CAND)) continue;
      const double kv = S.key[k];
      const double v = cont ? kv : floor(0.5 * kv);
      const double sg = S.sig[k];
      if (better_shift(sg, v, bs, bv, xb)) { bs = sg; bv = v; }
    }
    finish_column_j(p, j, tb, xb, bv, bs, b, C.oxhat, C.oscore, C.k, C.use_tabu);
  }
  __syncwarp();
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
  finish_column_j(p, j, tb, xb, bv, bs, b, C.oxhat, C.oscore, C.k, C.use_tabu);
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
  if (tid == 0) finish_column(P, p, xb, bv, bs, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
  __syncthreads();
}

// last-chunk handshake of a chunked column: returns true in every thread of the last block
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

// The CSC stream of a chunk tile: kPer independent coalesced loads + gathers per thread.
struct ChunkRows {
  double a[kPer];
  double r[kPer];
  double w[kPer];
  bool ok[kPer];
};
__device__ __forceinline__ void load_chunk(const DevProblem& P, const TileCtx& C, int e0, int nnz,
                                           ChunkRows& R) {
  int idx[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = threadIdx.x + q * kTileThreads;
    R.ok[q] = k < nnz;
    idx[q] = R.ok[q] ? __ldcs(P.row_idx + e0 + k) : 0;
    R.a[q] = R.ok[q] ? __ldcs(P.val + e0 + k) : 1.0;
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) load_row(C.rs, idx[q], R.r[q], R.w[q]);
}

// a chunk of a long binary column: partial flip sum, merged in chunk order
__device__ __forceinline__ void tile_lbin(const DevProblem& P, const DevWalkers& Wk, int walker,
                                          const TileCtx& C, const Tile& T, double* sm_red,
                                          int* s_flag, Best& b) {
  const int tid = threadIdx.x;
  const int p = T.p0;
  const double xb = C.x[p];
  const double dir = 1.0 - 2.0 * xb;
  ChunkRows R;
  load_chunk(P, C, T.e0, T.e1 - T.e0, R);
  double pen = 0.0;
#pragma unroll
  for (int q = 0; q < kPer; ++q)
    if (R.ok[q]) pen += penalty(R.w[q], R.r[q], R.r[q] + R.a[q] * dir);
  pen = block_sum(pen, sm_red);
  if (T.nchunks == 1) {
    if (tid == 0) finish_column(P, p, xb, 1.0 - xb, pen, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
    return;
  }
  double* scr = Wk.lscr + (size_t)walker * Wk.lss + T.scr;
  unsigned* cnt = Wk.lcount + (size_t)walker * Wk.lcs + T.lc;
  if (tid == 0) scr[T.chunk] = pen;
  if (last_chunk(cnt, T.nchunks, s_flag) && tid == 0) {
    double s = 0.0;
    for (int c = 0; c < T.nchunks; ++c) s += __ldcg(scr + c);   // chunk order
    *cnt = 0u;
    finish_column(P, p, xb, 1.0 - xb, s, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
  }
  __syncthreads();
}

// a chunk of a general integer column with domain [l, u], dom = u - l + 1 <= kBucketMax: the
// sort of line 13 becomes a counting pass. D[v-l] collects the -1 deltas at v and the +1
// deltas at v-1, so sigma at candidate v = β + Σ_{v' <= v} D[v'] + α [v > x̄].
__device__ __forceinline__ void tile_lbkt(const DevProblem& P, const DevWalkers& Wk, int walker,
                                          const TileCtx& C, const Tile& T, SmemBkt& S,
                                          double* sm_red, Best* sm_b, int* s_flag, Best& b) {
  const int tid = threadIdx.x;
  const int p = T.p0, dom = T.dom;
  const double xb = C.x[p], l = P.lb[p], u = P.ub[p];
  for (int q = tid; q <= dom; q += blockDim.x) S.D[q] = 0.0;
  for (int q = tid; q < dom; q += blockDim.x) S.cand[q] = 0;
  ChunkRows R;
  load_chunk(P, C, T.e0, T.e1 - T.e0, R);
  __syncthreads();
  double beta = 0.0, alpha = 0.0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    if (!R.ok[q]) continue;
    const Elem el = emit(xb, R.r[q], R.a[q], R.w[q], 1);
    beta += el.beta;
    alpha += el.alpha;
    if (!el.valid) continue;
    const double t = el.t;
    if (t >= l && t <= u && t != xb) S.cand[(int)(t - l)] = 1;
    if (!el.plus) {
      if (t < l) beta += el.delta;
      else if (t <= u) atomicAdd(&S.D[(int)(t - l)], el.delta);
    } else {
      if (t < l) beta += el.delta;
      else if (t < u) atomicAdd(&S.D[(int)(t - l) + 1], el.delta);
    }
  }
  beta = block_sum(beta, sm_red);
  alpha = block_sum(alpha, sm_red);
  bool have_all = (T.nchunks == 1);
  double B = beta, A = alpha;
  if (!have_all) {
    double* scr = Wk.lscr + (size_t)walker * Wk.lss + T.scr;
    unsigned* cnt = Wk.lcount + (size_t)walker * Wk.lcs + T.lc;
    double* pD = scr + (size_t)T.chunk * dom;
    double* pC = scr + (size_t)T.nchunks * dom + (size_t)T.chunk * dom;
    double* pBA = scr + (size_t)2 * T.nchunks * dom + 2 * T.chunk;
    for (int q = tid; q < dom; q += blockDim.x) {
      pD[q] = S.D[q];
      pC[q] = S.cand[q] ? 1.0 : 0.0;
    }
    if (tid == 0) { pBA[0] = beta; pBA[1] = alpha; }
    if (!last_chunk(cnt, T.nchunks, s_flag)) return;
    for (int q = tid; q < dom; q += blockDim.x) {
      double dsum = 0.0, csum = 0.0;
      for (int c = 0; c < T.nchunks; ++c) {
        dsum += __ldcg(scr + (size_t)c * dom + q);
        csum += __ldcg(scr + (size_t)T.nchunks * dom + (size_t)c * dom + q);
      }
      S.D[q] = dsum;
      S.cand[q] = csum > 0.0 ? 1 : 0;
    }
    if (tid == 0) {
      double bsum = 0.0, asum = 0.0;
      for (int c = 0; c < T.nchunks; ++c) {
        bsum += __ldcg(scr + (size_t)2 * T.nchunks * dom + 2 * c);
        asum += __ldcg(scr + (size_t)2 * T.nchunks * dom + 2 * c + 1);
      }
      sm_red[0] = bsum;
      sm_red[1] = asum;
      *cnt = 0u;
    }
    __syncthreads();
    B = sm_red[0];
    A = sm_red[1];
    __syncthreads();
  }
  if (tid == 0) {
    if (l != xb) S.cand[0] = 1;                 // (l, -1, 0)
    if (u != xb) S.cand[dom - 1] = 1;           // (u, -1, 0)
  }
  __syncthreads();
  block_scan_inclusive(S.D, dom, sm_red);
  double bs = -INFINITY, bv = xb;
  for (int q = tid; q < dom; q += blockDim.x) {
    if (!S.cand[q]) continue;
    const double v = l + (double)q;
    if (v == xb) continue;
    const double sig = B + S.D[q] + (v > xb ? A : 0.0);
    if (better_shift(sig, v, bs, bv, xb)) { bs = sig; bv = v; }
  }
  block_best_shift(bs, bv, xb, sm_b);
  if (tid == 0) finish_column(P, p, xb, bv, bs, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------

// grid = (blocks per walker, W). After its tiles every block publishes its best admissible move;
// the last block of the walker reduces them (fixed order) to the decision.
__global__ void __launch_bounds__(kTileThreads, 3) k_eval(DevProblem P, DevWalkers Wk, double* oxhat,
                                                          double* oscore, chap_move* best_out,
                                                          int part_base) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sm_red[32];
  __shared__ Best sm_b[32];
  __shared__ int s_flag;
  const int walker = blockIdx.y;
  const WalkerScalars* sc = Wk.sc + walker;
  TileCtx C;
  C.x = Wk.x + (size_t)walker * Wk.xs;
  C.rs = Wk.rs + (size_t)walker * Wk.rss;
  C.tabu = Wk.tabu + (size_t)walker * Wk.ts;
  C.k = sc->k;
  C.use_tabu = Wk.use_tabu;
  C.oxhat = oxhat;
  C.oscore = oscore;
  Best b;
  b.init();
  // phase A: block tiles (chunks of long columns, single-column sorts)
  for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
    const Tile T = P.tiles[t];
    switch (T.kind) {
      case CC_LBIN: tile_lbin(P, Wk, walker, C, T, sm_red, &s_flag, b); break;
      case CC_LBKT: tile_lbkt(P, Wk, walker, C, T, *reinterpret_cast<SmemBkt*>(smem), sm_red, sm_b, &s_flag, b); break;
      default: tile_genm(P, C, T, *reinterpret_cast<SmemGenM*>(smem), sm_red, sm_b, b); break;
    }
  }
  __syncthreads();
  // phase B: warp tiles, each warp on its own slice of shared memory, no block barriers
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* ws = smem + (size_t)wid * kWarpSmem;
    const int nwarps = gridDim.x * kTileWarps;
    int t = blockIdx.x * kTileWarps + wid;
    WTile Tn;
    if (t < P.n_wtiles) Tn = P.wtiles[t];
    for (; t < P.n_wtiles; t += nwarps) {
      const WTile T = Tn;
      if (t + nwarps < P.n_wtiles) Tn = P.wtiles[t + nwarps];   // next descriptor in flight
      if (T.kind == CC_BIN) wtile_bin(P, C, T, lane, *reinterpret_cast<WarpBin*>(ws), b);
      else if (T.kind == CC_GEN) wtile_gen(P, C, T, lane, *reinterpret_cast<WarpGen*>(ws), b);
      else wtile_empty(P, C, T, lane, b);
    }
  }
  // publish the block's best; the last block of this walker selects (R6)
  b = block_reduce_best(b, sm_b);
  Cand* part = Wk.part + (size_t)walker * Wk.ps;
  if (threadIdx.x == 0) write_part(part + part_base + blockIdx.x, b);
  if (!last_chunk(Wk.sel_count + walker, gridDim.x, &s_flag)) return;
  Best g;
  g.init();
  for (int q = threadIdx.x; q < part_base + (int)gridDim.x; q += blockDim.x) {
    Best o;
    o.s = __ldcg(&part[q].s);
    o.v = __ldcg(&part[q].v);
    o.j = __ldcg(&part[q].j);
    o.p = __ldcg(&part[q].p);
    g.take(o);
  }
  g = block_reduce_best(g, sm_b);
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
    d.delta = d.move ? (g.v - C.x[g.p]) : 0.0;
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
// binary kernel
// ------------------------------------------------------------------------------------------
// k_eval_bin evaluates the packed binary columns (flip scores). It is built like a
// plain gather loop so that many warps per SM keep their loads in flight: per warp tile (whole
// columns, <= kBinTile nonzeros, <= 32 columns, starting on a multiple of 4 nonzeros) every lane
// issues its coalesced CSC loads and its 16-byte row-state gathers back to back; the column of a
// slot comes from a redux.sync head mask, x̄ of the column from a shuffle; lane c sums column c.
struct __align__(16) BinWarp {
  double pen[kBinTile];
};
constexpr size_t kBinSmem = sizeof(BinWarp) * (kBinThreads / 32);

__global__ void __launch_bounds__(kBinThreads, 6) k_eval_bin(DevProblem P, DevWalkers Wk, double* oxhat,
                                                              double* oscore) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Best sm_b[32];
  const int walker = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const WalkerScalars* sc = Wk.sc + walker;
  const double* __restrict__ X = Wk.x + (size_t)walker * Wk.xs;
  const double2* __restrict__ RS = reinterpret_cast<const double2*>(Wk.rs + (size_t)walker * Wk.rss);
  const int32_t* __restrict__ TB = Wk.tabu + (size_t)walker * Wk.ts;
  const long long kk = sc->k;
  const int use_tabu = Wk.use_tabu;
  double* pen = reinterpret_cast<BinWarp*>(smem)[wid].pen;
  Best b;
  b.init();
  const int nwarps = gridDim.x * (kBinThreads / 32);
  int t = blockIdx.x * (kBinThreads / 32) + wid;
  WTile Tn;
  if (t < P.n_btiles) Tn = P.btiles[t];
  const unsigned le = (2u << lane) - 1u;
  for (; t < P.n_btiles; t += nwarps) {
    const WTile T = Tn;
    if (t + nwarps < P.n_btiles) Tn = P.btiles[t + nwarps];
    const int nc = T.ncols, len = T.e1 - T.e0;
    const int* __restrict__ ridx = P.row_idx + T.e0;
    const double* __restrict__ rval = P.val + T.e0;
    // column data of lane c (issued before the slot loads are consumed)
    const int p = T.p0 + lane;
    int cb = 0x7fffffff, ce = 0, j = 0, tb = 0;
    double xb = 0.0;
    if (lane < nc) {
      cb = __ldg(P.col_ptr + p) - T.e0;
      ce = __ldg(P.col_ptr + p + 1) - T.e0;
      j = __ldg(P.perm + p);
      tb = use_tabu ? __ldg(TB + p) : 0;
      xb = __ldg(X + p);
    }
#pragma unroll
    for (int h = 0; h < kBinSlots / 2; ++h) {
      int id[2];
      double av[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = lane + 32 * (2 * h + q);
        id[q] = k < len ? __ldcs(ridx + k) : P.dummy_row;
        av[q] = k < len ? __ldcs(rval + k) : 0.0;
      }
      double2 rv[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) rv[q] = __ldg(RS + id[q]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int qq = 2 * h + q;
        const int k = lane + 32 * qq;
        // column of slot k: column starts in rounds < qq plus those at or before this lane
        const unsigned hm = __reduce_or_sync(kFull, (cb >> 5) == qq ? (1u << (cb & 31)) : 0u);
        const unsigned before = __reduce_add_sync(kFull, (cb >> 5) < qq ? 1u : 0u);
        int col = (int)before + __popc(hm & le) - 1;
        col = col < 0 ? 0 : col;
        const double x = __shfl_sync(kFull, xb, col);
        const double r = rv[q].x, w = (double)__int_as_float((int)__double2loint(rv[q].y));
        if (k < len) pen[k] = penalty(w, r, r + av[q] * (1.0 - 2.0 * x));
      }
    }
    __syncwarp();
    if (lane < nc) {
      double s = 0.0;
      for (int e = cb; e < ce; ++e) s += pen[e];
      finish_column_j(p, j, tb, xb, 1.0 - xb, s, b, oxhat, oscore, kk, use_tabu);
    }
    __syncwarp();
  }
  b = block_reduce_best(b, sm_b);
  if (threadIdx.x == 0) write_part(Wk.part + (size_t)walker * Wk.ps + blockIdx.x, b);
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

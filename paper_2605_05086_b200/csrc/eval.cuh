// eval.cuh — best-shift evaluation kernels (§3.1, Eq. (1) and Algorithm 1).
//
// Three kernels cover all column lengths (the paper's length-specialised dispatch,
// PAPER.md:353-355, re-designed for sm_100a):
//   k_eval_warp   warp tasks: binary flips (g lanes per column), binary columns up
//                 to kBinWideMax (one warp each), and general columns with deg+2 <= 32 whose
//                 Algorithm 1 runs entirely in registers/shared memory of g lanes: emit (l.1-12),
//                 rank sort (l.13), inclusive segmented scan (l.14), sigma (l.15), argmax (l.16);
//   k_eval_block  one block per general column with deg+2 <= kBlockElems: shared-memory bitonic
//                 sort, block scan, block argmax;
//   k_eval_long   chunked long columns (4096 nonzeros per block): binary flip partial sums, or a
//                 bucket (counting) scan over a bounded integer domain; the last block of a
//                 column merges the chunk partials in chunk order (deterministic).
// Every kernel also reduces its columns to one best admissible move per block (R6) in Cand
// partials; k_select reduces those per walker.
#pragma once
#include "common.cuh"

namespace chap {

// PAPER.md:277-285 on residuals r0 = ȳ_i - b_i, r1 = y_ij - b_i; satisfied means r <= 0 (R10).
__device__ __forceinline__ double penalty(double w, double r0, double r1) {
  const bool s0 = r0 <= 0.0, s1 = r1 <= 0.0;
  double p = 0.0;
  if (s0) {
    p = s1 ? 0.0 : -w;
  } else if (s1) {
    p = w;
  } else if (r1 < r0) {
    p = 0.5 * w;
  } else if (r1 > r0) {
    p = -0.5 * w;
  }
  return p;
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
__device__ __forceinline__ void finish_column(const DevProblem& P, int p, double xb, double v,
                                              double s, Best& b, double* oxhat, double* oscore,
                                              const int32_t* tabu, long long k, int use_tabu) {
  if (s == -INFINITY) v = xb;
  const int j = P.perm[p];
  if (oxhat) oxhat[j] = v;
  if (oscore) oscore[j] = s;
  if (use_tabu && (long long)tabu[p] > k) return;
  if (better_move(s, j, b.s, b.j)) {
    b.s = s;
    b.v = v;
    b.j = j;
    b.p = p;
  }
}

// One breakpoint element of Algorithm 1 lines 3-11 for row i of column j,
// in the one-element-per-row form of DESIGN.md §2.3: an a<0 row gives (t, -1, δ); an a>0 row
// gives (t, +1, δ) whose candidate value t is scored by the exclusive prefix (the sum before
// its +1 entry = the sigma of the row's own (t, -1, 0) entry of line 9/10).
struct Elem {
  double t;
  double delta;
  double beta;
  double alpha;
  int valid;   // an entry is emitted
  int plus;    // marker +1 (a > 0 rows)
};

__device__ __forceinline__ Elem emit(double xb, double r, double a, double w, int is_int) {
  Elem e;
  e.beta = 0.0;
  e.alpha = 0.0;
  e.valid = 0;
  e.plus = 0;
  e.delta = 0.0;
  double t = xb - r / a;                             // (b_i - Σ_{k≠j} a_ik x̄_k) / a_ij  (l.3)
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
// warp tasks
// ------------------------------------------------------------------------------------------

struct WarpCtx {
  const double* x;
  const RowState* rs;
  const int32_t* tabu;
  long long k;
  int cut_active;
  int use_tabu;
  double* oxhat;
  double* oscore;
};

// binary flips, g = 2^lg lanes per column
__device__ __forceinline__ void task_bin(const DevProblem& P, const WarpCtx& C, const WTask& T,
                                         int lane, Best& b) {
  const int lg = T.lg, g = 1 << lg;
  const int grp = lane >> lg, lig = lane & (g - 1);
  const int p = T.p0 + grp;
  const bool colv = grp < T.ncols;
  double pen = 0.0, xb = 0.0;
  if (colv) {
    const int beg = P.col_ptr[p], d = P.col_ptr[p + 1] - beg;
    xb = C.x[p];
    if (lig < d) {
      const int i = P.row_idx[beg + lig];
      const double a = P.val[beg + lig];
      if (i != P.cut_row || C.cut_active) {
        const RowState s = C.rs[i];
        pen = penalty((double)s.w, s.r, s.r + a * (1.0 - 2.0 * xb));
      }
    }
  }
  for (int off = g >> 1; off > 0; off >>= 1) pen += __shfl_xor_sync(kFull, pen, off);
  if (colv && lig == 0)
    finish_column(P, p, xb, 1.0 - xb, pen, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
}

// binary flips, one warp per column of 32 < deg <= kBinWideMax
__device__ __forceinline__ void task_binw(const DevProblem& P, const WarpCtx& C, const WTask& T,
                                          int lane, Best& b) {
  const int p = T.p0;
  const int beg = P.col_ptr[p], end = P.col_ptr[p + 1];
  const double xb = C.x[p];
  const double dir = 1.0 - 2.0 * xb;
  double pen = 0.0;
#pragma unroll 4
  for (int e = beg + lane; e < end; e += kWarp) {
    const int i = P.row_idx[e];
    const double a = P.val[e];
    if (i != P.cut_row || C.cut_active) {
      const RowState s = C.rs[i];
      pen += penalty((double)s.w, s.r, s.r + a * dir);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) pen += __shfl_xor_sync(kFull, pen, off);
  if (lane == 0) finish_column(P, p, xb, 1.0 - xb, pen, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
}

// General (integer / continuous) columns with deg + 2 <= g lanes: Algorithm 1 in a lane group.
// Lane k < deg holds row k's element, lane deg the lower-bound entry (l, -1, 0), lane deg+1 the
// upper-bound entry (u, -1, 0) (l.1; infinite bounds dropped, R9).
__device__ __forceinline__ void task_gen(const DevProblem& P, const WarpCtx& C, const WTask& T,
                                         int lane, double* sm_d, double* sm_p, Best& b) {
  const int lg = T.lg, g = 1 << lg;
  const int grp = lane >> lg, lig = lane & (g - 1), base = grp << lg;
  const int p = T.p0 + grp;
  const bool colv = grp < T.ncols;
  double xb = 0.0, l = 0.0, u = 0.0;
  int d = 0;
  Elem el;
  el.t = 0.0; el.delta = 0.0; el.beta = 0.0; el.alpha = 0.0; el.valid = 0; el.plus = 0;
  bool cand = false;
  if (colv) {
    const int beg = P.col_ptr[p];
    d = P.col_ptr[p + 1] - beg;
    xb = C.x[p];
    l = P.lb[p];
    u = P.ub[p];
    const int is_int = P.vclass[p] != 3;
    if (lig < d) {
      const int i = P.row_idx[beg + lig];
      const double a = P.val[beg + lig];
      if (i != P.cut_row || C.cut_active) {
        const RowState s = C.rs[i];
        el = emit(xb, s.r, a, (double)s.w, is_int);
        cand = el.valid && el.t >= l && el.t <= u && el.t != xb;
      }
    } else if (lig == d) {
      if (isfinite(l)) { el.valid = 1; el.t = l; cand = (l != xb); }
    } else if (lig == d + 1) {
      if (isfinite(u)) { el.valid = 1; el.t = u; cand = (u != xb); }
    }
  }
  // β and α of lines 1-12: group sums
  double beta = el.beta, alpha = el.alpha;
  for (int off = g >> 1; off > 0; off >>= 1) {
    beta += __shfl_xor_sync(kFull, beta, off);
    alpha += __shfl_xor_sync(kFull, alpha, off);
  }
  // line 13: lexicographic sort by (value, marker) — rank sort; ties by lane (unique ranks)
  const unsigned kmax = __reduce_max_sync(kFull, colv ? (unsigned)(d + 2) : 0u);
  const int mine = el.valid ? el.plus : 2;
  int rank = 0;
  for (unsigned q = 0; q < kmax; ++q) {
    const int src = base + (int)q;
    const double tq = __shfl_sync(kFull, el.t, src);
    const int mq = __shfl_sync(kFull, mine, src);
    const bool less = (mq != 2) && (tq < el.t || (tq == el.t && (mq < mine || (mq == mine && (int)q < lig))));
    rank += less ? 1 : 0;
  }
  const unsigned vmask = __ballot_sync(kFull, el.valid);
  const int nvalid = __popc((vmask >> base) & (g == 32 ? kFull : ((1u << g) - 1u)));
  __syncwarp();
  if (el.valid) sm_d[base + rank] = el.delta;
  __syncwarp();
  // line 14: inclusive scan of the deltas in sorted order (segmented by lane group)
  double ps = (lig < nvalid) ? sm_d[base + lig] : 0.0;
  for (int off = 1; off < g; off <<= 1) {
    const double y = __shfl_up_sync(kFull, ps, off, g);
    if (lig >= off) ps += y;
  }
  sm_p[base + lig] = ps;
  __syncwarp();
  // line 15: sigma; a +1 element scores its value by the prefix before it (its -1 partner)
  double sig = -INFINITY, v = el.t;
  if (el.valid && cand) {
    const double pin = sm_p[base + rank];
    const double pex = rank > 0 ? sm_p[base + rank - 1] : 0.0;
    sig = beta + (el.plus ? pex : pin) + (el.t > xb ? alpha : 0.0);
  }
  // line 16: argmax within the group (R3, R4)
  for (int off = g >> 1; off > 0; off >>= 1) {
    const double so = __shfl_xor_sync(kFull, sig, off);
    const double vo = __shfl_xor_sync(kFull, v, off);
    if (better_shift(so, vo, sig, v, xb)) { sig = so; v = vo; }
  }
  if (colv && lig == 0) finish_column(P, p, xb, v, sig, b, C.oxhat, C.oscore, C.tabu, C.k, C.use_tabu);
}

__global__ void __launch_bounds__(kEvalThreads) k_eval_warp(DevProblem P, DevWalkers Wk,
                                                            double* oxhat, double* oscore) {
  __shared__ double sm_d[kEvalWarps][kWarp];
  __shared__ double sm_p[kEvalWarps][kWarp];
  __shared__ Best sm_b[kWarp];
  const int walker = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const WalkerScalars* sc = Wk.sc + walker;
  WarpCtx C;
  C.x = Wk.x + (size_t)walker * Wk.xs;
  C.rs = Wk.rs + (size_t)walker * Wk.rss;
  C.tabu = Wk.tabu + (size_t)walker * Wk.ts;
  C.k = sc->k;
  C.cut_active = sc->cut_active;
  C.use_tabu = Wk.use_tabu;
  C.oxhat = oxhat;
  C.oscore = oscore;
  Best b;
  b.init();
  for (int t = blockIdx.x * kEvalWarps + wid; t < P.n_wtasks; t += gridDim.x * kEvalWarps) {
    const WTask T = P.wtasks[t];
    if (T.kind == CC_BIN) task_bin(P, C, T, lane, b);
    else if (T.kind == CC_GEN) task_gen(P, C, T, lane, sm_d[wid], sm_p[wid], b);
    else task_binw(P, C, T, lane, b);
  }
  b = block_reduce_best(b, sm_b);
  if (threadIdx.x == 0) write_part(Wk.part + (size_t)walker * Wk.ps + blockIdx.x, b);
}

// ------------------------------------------------------------------------------------------
// block per general column (deg + 2 <= kBlockElems)
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
  // exclusive scan of the per-thread totals
  const int lane = tid & 31, wid = tid >> 5, nw = (T + 31) >> 5;
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
  (void)nw;
}

__global__ void __launch_bounds__(kBlockThreads) k_eval_block(DevProblem P, DevWalkers Wk,
                                                              double* oxhat, double* oscore,
                                                              int part_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* st = reinterpret_cast<double*>(smem);            // [kBlockElems] value
  double* sdel = st + kBlockElems;                            // [kBlockElems] delta (by element)
  double* sp = sdel + kBlockElems;                            // [kBlockElems] prefix (by rank)
  uint32_t* smk = reinterpret_cast<uint32_t*>(sp + kBlockElems);  // [kBlockElems] plus<<31|cand<<30|e
  __shared__ double sm_red[32];
  __shared__ Best sm_b[32];
  const int walker = blockIdx.y, tid = threadIdx.x;
  const WalkerScalars* sc = Wk.sc + walker;
  const double* x = Wk.x + (size_t)walker * Wk.xs;
  const RowState* rs = Wk.rs + (size_t)walker * Wk.rss;
  const int32_t* tabu = Wk.tabu + (size_t)walker * Wk.ts;
  const long long k = sc->k;
  const int cut_active = sc->cut_active;
  const int p = P.bcols[blockIdx.x];
  const int beg = P.col_ptr[p], d = P.col_ptr[p + 1] - beg;
  const double xb = x[p], l = P.lb[p], u = P.ub[p];
  const int is_int = P.vclass[p] != 3;
  const int L = d + 2;
  int Lp = 1;
  while (Lp < L) Lp <<= 1;
  double beta = 0.0, alpha = 0.0;
  for (int e = tid; e < Lp; e += blockDim.x) {
    double t = INFINITY, del = 0.0;
    uint32_t mk = 0xffffffffu;
    if (e < d) {
      const int i = P.row_idx[beg + e];
      const double a = P.val[beg + e];
      if (i != P.cut_row || cut_active) {
        const RowState s = rs[i];
        const Elem el = emit(xb, s.r, a, (double)s.w, is_int);
        beta += el.beta;
        alpha += el.alpha;
        if (el.valid) {
          const bool cand = el.t >= l && el.t <= u && el.t != xb;
          t = el.t;
          del = el.delta;
          mk = ((uint32_t)el.plus << 31) | ((uint32_t)cand << 30) | (uint32_t)e;
        }
      }
    } else if (e == d) {
      if (isfinite(l)) { t = l; mk = ((uint32_t)(l != xb) << 30) | (uint32_t)e; }
    } else if (e == d + 1) {
      if (isfinite(u)) { t = u; mk = ((uint32_t)(u != xb) << 30) | (uint32_t)e; }
    }
    st[e] = t;
    smk[e] = mk;
    sdel[e] = del;
  }
  beta = block_sum(beta, sm_red);
  alpha = block_sum(alpha, sm_red);
  // bitonic sort of (value, marker) pairs (PAPER.md:324 line 13; R3 marker order)
  for (int size = 2; size <= Lp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int q = tid; q < (Lp >> 1); q += blockDim.x) {
        const int lo = 2 * q - (q & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const double t0 = st[lo], t1 = st[hi];
        const uint32_t m0 = smk[lo], m1 = smk[hi];
        const bool gt = (t0 > t1) || (t0 == t1 && m0 > m1);
        if (gt == asc) {
          st[lo] = t1; st[hi] = t0;
          smk[lo] = m1; smk[hi] = m0;
        }
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = smk[q];
    sp[q] = (mk == 0xffffffffu) ? 0.0 : sdel[mk & 0x3fffffffu];
  }
  __syncthreads();
  block_scan_inclusive(sp, Lp, sm_red);   // line 14
  Best bb;
  bb.init();
  double bs = -INFINITY, bv = xb;
  for (int q = tid; q < Lp; q += blockDim.x) {
    const uint32_t mk = smk[q];
    if (mk == 0xffffffffu || !((mk >> 30) & 1u)) continue;
    const double t = st[q];
    const double pre = (mk >> 31) ? (q > 0 ? sp[q - 1] : 0.0) : sp[q];
    const double sig = beta + pre + (t > xb ? alpha : 0.0);   // line 15
    if (better_shift(sig, t, bs, bv, xb)) { bs = sig; bv = t; }
  }
  // line 16: block argmax (shift tie-break within one variable)
  {
    const int lane = tid & 31, wid = tid >> 5;
    for (int off = 16; off > 0; off >>= 1) {
      const double so = __shfl_xor_sync(kFull, bs, off), vo = __shfl_xor_sync(kFull, bv, off);
      if (better_shift(so, vo, bs, bv, xb)) { bs = so; bv = vo; }
    }
    __syncthreads();
    if (lane == 0) { sm_b[wid].s = bs; sm_b[wid].v = bv; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (better_shift(sm_b[q].s, sm_b[q].v, bs, bv, xb)) { bs = sm_b[q].s; bv = sm_b[q].v; }
      finish_column(P, p, xb, bv, bs, bb, oxhat, oscore, tabu, k, Wk.use_tabu);
      write_part(Wk.part + (size_t)walker * Wk.ps + part_off + blockIdx.x, bb);
    }
  }
}

// ------------------------------------------------------------------------------------------
// chunked long columns
// ------------------------------------------------------------------------------------------

__global__ void __launch_bounds__(kBlockThreads) k_eval_long(DevProblem P, DevWalkers Wk,
                                                             double* oxhat, double* oscore,
                                                             int part_off) {
  __shared__ double sD[kBucketMax + 1];
  __shared__ unsigned char sC[kBucketMax];
  __shared__ double sm_red[32];
  __shared__ Best sm_b[32];
  __shared__ int s_last;
  const int walker = blockIdx.y, tid = threadIdx.x;
  const LChunk ch = P.chunks[blockIdx.x];
  const WalkerScalars* sc = Wk.sc + walker;
  const double* x = Wk.x + (size_t)walker * Wk.xs;
  const RowState* rs = Wk.rs + (size_t)walker * Wk.rss;
  const int32_t* tabu = Wk.tabu + (size_t)walker * Wk.ts;
  double* scr = Wk.lscr + (size_t)walker * Wk.lss + ch.scr;
  unsigned* cnt = Wk.lcount + (size_t)walker * Wk.lcs + ch.lc;
  const long long k = sc->k;
  const int cut_active = sc->cut_active;
  const int p = ch.p;
  const double xb = x[p];
  Best bb;
  bb.init();
  if (ch.kind == 0) {
    // binary flip partial sum over this chunk
    const double dir = 1.0 - 2.0 * xb;
    double pen = 0.0;
    for (int e = ch.e0 + tid; e < ch.e1; e += blockDim.x) {
      const int i = P.row_idx[e];
      const double a = P.val[e];
      if (i != P.cut_row || cut_active) {
        const RowState s = rs[i];
        pen += penalty((double)s.w, s.r, s.r + a * dir);
      }
    }
    pen = block_sum(pen, sm_red);
    if (tid == 0) scr[ch.chunk] = pen;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(cnt, 1u) == (unsigned)(ch.nchunks - 1));
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (tid == 0) {
        double s = 0.0;
        for (int c = 0; c < ch.nchunks; ++c) s += __ldcg(scr + c);   // chunk order
        *cnt = 0u;
        finish_column(P, p, xb, 1.0 - xb, s, bb, oxhat, oscore, tabu, k, Wk.use_tabu);
      }
    }
  } else {
    // bounded integer domain [l, u], dom = u - l + 1 <= kBucketMax: the sort of line 13 becomes
    // a counting (bucket) pass. D[v-l] collects the -1 deltas at v and the +1 deltas at v-1, so
    // sigma at candidate v = β + Σ_{v' <= v} D[v'] + α[v > x̄].
    const int dom = ch.dom;
    const double l = P.lb[p], u = P.ub[p];
    for (int q = tid; q <= dom; q += blockDim.x) sD[q] = 0.0;
    for (int q = tid; q < dom; q += blockDim.x) sC[q] = 0;
    __syncthreads();
    double beta = 0.0, alpha = 0.0;
    for (int e = ch.e0 + tid; e < ch.e1; e += blockDim.x) {
      const int i = P.row_idx[e];
      const double a = P.val[e];
      if (i == P.cut_row && !cut_active) continue;
      const RowState s = rs[i];
      const Elem el = emit(xb, s.r, a, (double)s.w, 1);
      beta += el.beta;
      alpha += el.alpha;
      if (!el.valid) continue;
      const double t = el.t;
      if (t >= l && t <= u && t != xb) sC[(int)(t - l)] = 1;
      if (!el.plus) {
        if (t < l) beta += el.delta;
        else if (t <= u) atomicAdd(&sD[(int)(t - l)], el.delta);
      } else {
        if (t < l) beta += el.delta;
        else if (t < u) atomicAdd(&sD[(int)(t - l) + 1], el.delta);
      }
    }
    beta = block_sum(beta, sm_red);
    alpha = block_sum(alpha, sm_red);
    // chunk partials: [nchunks][dom] D, [nchunks][dom] cand (as doubles 0/1), [nchunks][2] β α
    double* pD = scr + (size_t)ch.chunk * dom;
    double* pC = scr + (size_t)ch.nchunks * dom + (size_t)ch.chunk * dom;
    double* pBA = scr + (size_t)2 * ch.nchunks * dom + 2 * ch.chunk;
    for (int q = tid; q < dom; q += blockDim.x) {
      pD[q] = sD[q];
      pC[q] = sC[q] ? 1.0 : 0.0;
    }
    if (tid == 0) { pBA[0] = beta; pBA[1] = alpha; }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(cnt, 1u) == (unsigned)(ch.nchunks - 1));
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int q = tid; q < dom; q += blockDim.x) {
        double dsum = 0.0, csum = 0.0;
        for (int c = 0; c < ch.nchunks; ++c) {
          dsum += __ldcg(scr + (size_t)c * dom + q);
          csum += __ldcg(scr + (size_t)ch.nchunks * dom + (size_t)c * dom + q);
        }
        sD[q] = dsum;
        sC[q] = csum > 0.0 ? 1 : 0;
      }
      __syncthreads();
      if (tid == 0) {
        double bsum = 0.0, asum = 0.0;
        for (int c = 0; c < ch.nchunks; ++c) {
          bsum += __ldcg(scr + (size_t)2 * ch.nchunks * dom + 2 * c);
          asum += __ldcg(scr + (size_t)2 * ch.nchunks * dom + 2 * c + 1);
        }
        sm_b[0].s = bsum;
        sm_b[0].v = asum;
        if (l != xb) sC[0] = 1;                 // (l, -1, 0)
        if (u != xb) sC[dom - 1] = 1;           // (u, -1, 0)
        *cnt = 0u;
      }
      __syncthreads();
      const double B = sm_b[0].s, A = sm_b[0].v;
      __syncthreads();
      block_scan_inclusive(sD, dom, sm_red);
      double bs = -INFINITY, bv = xb;
      for (int q = tid; q < dom; q += blockDim.x) {
        if (!sC[q]) continue;
        const double v = l + (double)q;
        if (v == xb) continue;
        const double sig = B + sD[q] + (v > xb ? A : 0.0);
        if (better_shift(sig, v, bs, bv, xb)) { bs = sig; bv = v; }
      }
      const int lane = tid & 31, wid = tid >> 5;
      for (int off = 16; off > 0; off >>= 1) {
        const double so = __shfl_xor_sync(kFull, bs, off), vo = __shfl_xor_sync(kFull, bv, off);
        if (better_shift(so, vo, bs, bv, xb)) { bs = so; bv = vo; }
      }
      __syncthreads();
      if (lane == 0) { sm_b[wid].s = bs; sm_b[wid].v = bv; }
      __syncthreads();
      if (tid == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
          if (better_shift(sm_b[q].s, sm_b[q].v, bs, bv, xb)) { bs = sm_b[q].s; bv = sm_b[q].v; }
        finish_column(P, p, xb, bv, bs, bb, oxhat, oscore, tabu, k, Wk.use_tabu);
      }
    }
  }
  if (tid == 0) write_part(Wk.part + (size_t)walker * Wk.ps + part_off + blockIdx.x, bb);
}

// ------------------------------------------------------------------------------------------
// global select: best admissible move per walker, ties -> lowest j (R6)
// ------------------------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_select(DevWalkers Wk, int n_part, chap_move* best_out) {
  __shared__ Best sm_b[32];
  const int walker = blockIdx.x;
  const Cand* part = Wk.part + (size_t)walker * Wk.ps;
  Best b;
  b.init();
  for (int q = threadIdx.x; q < n_part; q += blockDim.x) {
    const Cand c = part[q];
    Best o;
    o.s = c.s; o.v = c.v; o.j = c.j; o.p = c.p;
    b.take(o);
  }
  b = block_reduce_best(b, sm_b);
  if (threadIdx.x == 0) {
    WalkerScalars* sc = Wk.sc + walker;
    const bool found = b.p >= 0;
    Decision d;
    d.move = (found && b.s > 0.0) ? 1 : 0;
    d.p = b.p;
    d.j = found ? b.j : -1;
    d.pad = 0;
    d.v = b.v;
    d.s = found ? b.s : -INFINITY;
    d.delta = d.move ? (b.v - Wk.x[(size_t)walker * Wk.xs + b.p]) : 0.0;
    sc->dec = d;
    if (best_out) {
      chap_move mv;
      mv.j = d.move ? d.j : -1;
      mv.pad = 0;
      mv.v = d.move ? d.v : NAN;
      mv.s = d.move ? d.s : -INFINITY;
      best_out[walker] = mv;
    }
  }
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

// tabu.cuh — walker state kernels: residual initialisation, apply (incremental residual update,
// PAPER.md:343), weight bump (R12), incumbent / cutoff (R15), exports.
#pragma once
#include "common.cuh"
#include "eval.cuh"

namespace chap {

// x_int[w][p] = x_user[w][perm[p]]; flags an out-of-bounds or fractional-integer value.
__global__ void k_permute_in(DevProblem P, const double* __restrict__ xu, size_t xus, double* xi,
                             size_t xis, int* bad) {
  const int w = blockIdx.y;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    const double v = xu[(size_t)w * xus + P.perm[p]];
    const uint8_t vc = P.vclass[p];
    const bool ok = (v >= P.lb[p]) && (v <= P.ub[p]) && (vc == 3 || v == floor(v));
    if (!ok && bad) atomicOr(bad, 1);
    xi[(size_t)w * xis + p] = v;
  }
}

// Flags a user-order point that is out of bounds or fractional on an integer variable.
__global__ void k_check_point(DevProblem P, const double* __restrict__ xu, int* bad) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    const double v = xu[P.perm[p]];
    const bool ok = (v >= P.lb[p]) && (v <= P.ub[p]) && (P.vclass[p] == 3 || v == floor(v));
    if (!ok) atomicOr(bad, 1);
  }
}

// r_i = Σ_k a_ik x̄_k - b_i from scratch (warp per row, CSR). The cutoff row (last) is active
// iff sc[w].cut_active (rhs sc[w].cutoff_rhs); an inactive cutoff row is stored inert, r = -inf
// and w = 0, so that it contributes nothing to any score without a per-nonzero test (its logical
// weight while inactive is the initial 1: bumps skip inactive rows). init_w: 0 keep weights,
// 1 set to 1, 2 copy from wsrc (eval API).
__global__ void k_rows_init(DevProblem P, DevWalkers Wk, int init_w, const float* __restrict__ wsrc,
                            int only_walker, int* bad) {
  const int w = only_walker >= 0 ? only_walker : blockIdx.y;
  if (skip_walker(Wk.rmask, only_walker, w)) return;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const double* xw = Wk.x + (size_t)w * Wk.xs;
  const RowView rw = row_view(Wk, w);
  const WalkerScalars* sc = Wk.sc;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    RowState d;
    set_r(d, -INFINITY);
    d.w = 0.0f;
    rw[P.dummy_row] = d;   // inert padding row
  }
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < P.m_norm; i += nwarps) {
    if (i == P.cut_row) {   // c.x comes from k_cut_dot (a grid-wide sum): no warp walks this row
      if (lane == 0) {
        RowState s = rw[i];
        set_r(s, sc[w].cut_active ? sc[w].cdot - sc[w].cutoff_rhs : -INFINITY);
        if (init_w == 1) s.w = 1.0f;
        else if (init_w == 2) s.w = wsrc ? wsrc[i] : 1.0f;
        if (init_w == 2 && bad && !(s.w >= 0.0f)) atomicOr(bad, 1);   // weights must be >= 0 (R11)
        if (init_w == 2 && !(s.w == truncf(s.w) && s.w <= 1048576.0f)) atomicAnd(&Wk.sc[w].wint, 0);
        if (!sc[w].cut_active) s.w = 0.0f;
        rw[i] = s;
      }
      continue;
    }
    const int e0 = P.rp[i], e1 = P.rp[i + 1];
    double y = 0.0;
    for (int e = e0 + lane; e < e1; e += 32) y += P.cv[e] * xw[P.ci[e]];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) y += __shfl_xor_sync(kFull, y, off);
    if (lane == 0) {
      double r;
      if (i < P.cut_row) {
        r = y - P.b[i];
      } else {
        r = sc[w].cut_active ? y - sc[w].cutoff_rhs : -INFINITY;
      }
      RowState s = rw[i];
      set_r(s, r);
      if (init_w == 1) s.w = 1.0f;
      else if (init_w == 2) s.w = wsrc ? wsrc[i] : 1.0f;
      if (init_w == 2 && bad && !(s.w >= 0.0f)) atomicOr(bad, 1);
      if (init_w == 2 && !(s.w == truncf(s.w) && s.w <= 1048576.0f)) atomicAnd(&Wk.sc[w].wint, 0);
      if (i == P.cut_row && !sc[w].cut_active) s.w = 0.0f;
      rw[i] = s;
    }
  }
}

__device__ __forceinline__ double auto_delta(const DevProblem& P, double delta_param, double z) {
  if (!isnan(delta_param)) return delta_param;
  if (!isnan(P.auto_delta)) return P.auto_delta;
  return 1e-6 * fmax(1.0, fabs(z));   // R14
}

// Set the walker's incumbent from its current point (violated == 0): best_obj, cutoff rhs
// c.x̄ - δ, residual of the cutoff row recomputed as y_cut - rhs.
__device__ __forceinline__ void take_incumbent(const DevProblem& P, const DevWalkers& Wk,
                                               WalkerScalars* sc, const RowView& rw) {
  const double z = sc->obj;
  sc->best_obj = z;
  sc->has_inc = 1;
  sc->pending_copy = 1;
  const double rhs = z - auto_delta(P, Wk.delta, z);
  if (!sc->cut_active) rw[P.cut_row].w = 1.0f;   // the inert row takes its logical weight
  sc->cutoff_rhs = rhs;
  sc->cut_active = 1;
  sc->rint = P.rint_base && rhs == floor(rhs);
  const double r = z - rhs;
  set_r(rw[P.cut_row], r);
  sc->violated = (r > 0.0) ? 1 : 0;
}

// One block per walker: violated count, objective, k = 0 incumbent check (R15).
// mode 0: walker create (k = 0, counters cleared); mode 1: restart (keeps k, counters, best).
__global__ void k_walker_finalize_init(DevProblem P, DevWalkers Wk, int mode, int only_walker) {
  const int w = (only_walker >= 0) ? only_walker : blockIdx.x;
  if (skip_walker(Wk.rmask, only_walker, w)) return;
  const int tid = threadIdx.x;
  WalkerScalars* sc = Wk.sc + w;
  const RowView rw = row_view(Wk, w);
  if (tid == 0) {
    const long long vt = sc->vcount;   // k_viol_count
    const double zt = sc->cdot;        // k_cut_dot
    sc->violated = vt;
    sc->obj = zt;
    sc->force_p = -1;   // a restart drops a pending perturbation (R21)
    sc->pert_kv = ~0ull;
    sc->pert_ka = ~0ull;
    if (mode == 0) {
      // weights start at 1 and grow by +1 up to the cap (R12): integers <= 2^20 when the cap is one
      sc->wint = Wk.wcap == floorf(Wk.wcap) && Wk.wcap <= 1048576.0f;
      sc->rint = P.rint_base && (!sc->cut_active || sc->cutoff_rhs == floor(sc->cutoff_rhs));
      sc->k = 0;
      sc->n_moves = 0;
      sc->n_stuck = 0;
      sc->has_inc = 0;
      sc->best_obj = INFINITY;
      sc->apply_counter = 0;
      sc->log = nullptr;
      sc->log_k0 = 0;
    }
    if (vt == 0) take_incumbent(P, Wk, sc, rw);
  }
}

// Zero the grid-wide accumulators of walker `only_walker` (>= 0) or of every walker (blockIdx.x).
__global__ void k_acc_zero(WalkerScalars* sc, int only_walker, const int32_t* rmask) {
  const int w = only_walker >= 0 ? only_walker : blockIdx.x;
  if (skip_walker(rmask, only_walker, w)) return;
  sc[w].cdot = 0.0;
  sc[w].vcount = 0;
}

// c.x of each walker's point (the cutoff row's activity and the objective), grid-wide: block
// partials added to sc[w].cdot (exact for the integer data of DESIGN §5).
__global__ void __launch_bounds__(256) k_cut_dot(DevProblem P, const double* __restrict__ x, size_t xs,
                                                  WalkerScalars* sc, int only_walker, const int32_t* rmask) {
  __shared__ double sm[8];
  const int w = only_walker >= 0 ? only_walker : blockIdx.y;
  if (skip_walker(rmask, only_walker, w)) return;
  const double* xw = x + (size_t)w * xs;
  double z = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) z += P.c[p] * xw[p];
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sm[q];
    if (t != 0.0) atomicAdd(&sc[w].cdot, t);
  }
}

// Violated active rows of each walker (r > 0; the inactive cutoff row excluded), grid-wide.
__global__ void __launch_bounds__(256) k_viol_count(DevProblem P, DevWalkers Wk, int only_walker) {
  __shared__ unsigned long long sm[8];
  const int w = only_walker >= 0 ? only_walker : blockIdx.y;
  if (skip_walker(Wk.rmask, only_walker, w)) return;
  WalkerScalars* sc = Wk.sc;
  const RowView rw = row_view(Wk, w);
  const int cut_active = sc[w].cut_active;
  unsigned long long v = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m_norm; i += gridDim.x * blockDim.x)
    if (!(i == P.cut_row && !cut_active) && rw[i].r > 0.0) ++v;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sm[q];
    if (t) atomicAdd((unsigned long long*)&sc[w].vcount, t);
  }
}

// The binary bitset of walker-minor groups from x (all walkers, or walker only_walker).
__global__ void k_xbits_build(DevProblem P, DevWalkers Wk, int only_walker) {
  if (!Wk.xbits) return;
  if (Wk.rg == 1) {   // one walker: the block-ordered bitset of k_eval_binrow
    const int nb = P.n_rblocks;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nb * kRowWpb; q += gridDim.x * blockDim.x) {
      const int b = q / kRowWpb, k0 = 32 * (q % kRowWpb);
      uint32_t word = 0u;
      for (int t = 0; t < 32; ++t) {
        const long long pq = (long long)(k0 + t) * nb + b;   // position among the packed binaries
        if (pq < P.rb_nbin && Wk.x[P.rb_pb0 + pq] != 0.0) word |= 1u << t;
      }
      Wk.xbits[q] = word;
    }
    return;
  }
  const int g = only_walker >= 0 ? only_walker / Wk.rg : blockIdx.y;
  const int w0 = g * Wk.rg, w1 = min(Wk.W, w0 + Wk.rg);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    if (P.vclass[p] != 1) continue;
    uint32_t word = 0u;
    for (int w = w0; w < w1; ++w)
      if (Wk.x[(size_t)w * Wk.xs + p] != 0.0) word |= 1u << (w - w0);
    Wk.xbits[(size_t)g * P.n + p] = word;
  }
}

// Clear the tabu list of walker w (restart) or of all walkers.
__global__ void k_tabu_clear(int32_t* tabu, size_t ts, int n, int only_walker, const int32_t* rmask) {
  const int w = (only_walker >= 0) ? only_walker : blockIdx.y;
  if (skip_walker(rmask, only_walker, w)) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    tabu[(size_t)w * ts + p] = 0;
}

// Apply the selected move or bump weights, then (last block) finalise the iteration.
// The perturbation's new value of internal column p at x̄ = xb (R21): binary: 1 - x̄; integer: a
// uniform draw over the domain minus x̄ (an infinite side replaced by x̄ ∓ R, at most 2^52 values);
// continuous: lo + (hi - lo) u, u = (h >> 11) 2^-53, rounded once per operation (no contraction);
// fixed or a one-value domain: none.
__device__ __forceinline__ bool perturb_value(const DevProblem& P, int p, double xb, int R, unsigned long long h,
                                              double* out) {
  const int cls = P.vclass[p];
  if (cls == 0) return false;
  if (cls == 1) {
    *out = 1.0 - xb;
    return true;
  }
  const double l = P.lb[p], u = P.ub[p];
  const double lo = isfinite(l) ? l : xb - (double)R, hi = isfinite(u) ? u : xb + (double)R;
  if (cls == 2) {
    double cnt = hi - lo;   // the values other than x̄
    if (!(cnt >= 1.0)) return false;
    if (cnt > 4503599627370496.0) cnt = 4503599627370496.0;
    double v = lo + (double)(h % (unsigned long long)cnt);
    if (v >= xb) v += 1.0;
    *out = v;
    return true;
  }
  double v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), (double)(h >> 11) * 0x1.0p-53));
  if (v > hi) v = hi;
  *out = v;
  return true;
}

__global__ void __launch_bounds__(kApplyThreads) k_apply(DevProblem P, DevWalkers Wk) {
  pdl_wait_trigger();
  __shared__ long long smv[32];
  __shared__ int s_last;
  const int w = blockIdx.y, tid = threadIdx.x;
  WalkerScalars* sc = Wk.sc + w;
  double* x = Wk.x + (size_t)w * Wk.xs;
  const RowView rw = row_view(Wk, w);
  const Decision d = sc->dec;
  KT_BEGIN(Wk, 3);
  const int cut_active = sc->cut_active;
  // a move of a short column with nothing else to do is applied and finalised by block 0 alone (no
  // grid-wide last-block handshake); bumps, long columns, incumbent copies and dirty marking use the grid
  const bool solo = d.move && !sc->pending_copy && !Wk.dirty && Wk.W == 1 &&
                    P.col_ptr[d.p + 1] - P.col_ptr[d.p] <= 4 * kApplyThreads;
  if (solo && blockIdx.x != 0) return;
  // solo: no other block writes the walker's scalars, so thread 0 reads them now (independent loads,
  // their latency hidden behind the column's update) instead of one after another at the end
  long long s_k = 0, s_viol = 0, s_nm = 0;
  double s_obj = 0.0;
  if (solo && tid == 0) {
    s_k = sc->k;
    s_viol = sc->violated;
    s_nm = sc->n_moves;
    s_obj = sc->obj;
  }
  const int gtid = solo ? tid : blockIdx.x * blockDim.x + tid, gstride = solo ? (int)blockDim.x : gridDim.x * blockDim.x;
  // phase 0: an incumbent found by the previous iteration: best_x <- x (x unchanged since)
  if (sc->pending_copy) {
    double* bx = Wk.best_x + (size_t)w * Wk.xs;
    for (int p = gtid; p < P.n; p += gstride) bx[p] = x[p];
  }
  long long dv = 0;
  if (d.move) {
    // r_i += a_ij Δ over column j* (PAPER.md:343); count feasibility transitions
    const int e0 = P.col_ptr[d.p], e1 = P.col_ptr[d.p + 1];
    for (int e = e0 + gtid; e < e1; e += gstride) {
      const int i = P.row_idx[e];
      if ((i == P.cut_row && !cut_active) || i == P.dummy_row) continue;
      const double r0 = rw[i].r;
      const double r1 = r0 + P.val[e] * d.delta;
      set_r(rw[i], r1);
      dv += (long long)(r1 > 0.0) - (long long)(r0 > 0.0);
    }
  } else {
    // stuck: w_i <- min(w_i + 1, cap) on every active violated row (R12), or with weight smoothing
    // (R22) drawn, w_i <- w_i - 1 on every active satisfied row with w_i > 1; with the perturbation
    // (R21) also the row draw: the least (h32 << 32 | i) over the violated and over all active rows
    unsigned long long kv = ~0ull, ka = ~0ull;
    const bool pert = Wk.perturb != 0;
    const unsigned long long h0 =
        (pert || Wk.smooth_prob > 0.0f)
            ? splitmix64(splitmix64(splitmix64(Wk.rng_seed) ^ (unsigned long long)w) ^ (unsigned long long)sc->k)
            : 0ull;
    const bool smooth =
        Wk.smooth_prob > 0.0f && (double)(splitmix64(h0 ^ kDrawSmooth) >> 11) * 0x1.0p-53 < (double)Wk.smooth_prob;
    for (int i = gtid; i < P.m_norm; i += gstride) {
      if (i == P.cut_row && !cut_active) continue;
      const bool viol = rw[i].r > 0.0;
      if (smooth) {
        if (!viol && rw[i].w > 1.0f) rw[i].w = rw[i].w - 1.0f;
      } else if (viol) {
        rw[i].w = fminf(rw[i].w + 1.0f, Wk.wcap);
      }
      if (pert) {
        const unsigned long long key = (splitmix64(h0 ^ (unsigned long long)i) & 0xFFFFFFFF00000000ull) | (unsigned)i;
        ka = key < ka ? key : ka;
        if (viol) kv = key < kv ? key : kv;
      }
    }
    if (pert) {
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long ov = __shfl_xor_sync(kFull, kv, off), oa = __shfl_xor_sync(kFull, ka, off);
        kv = ov < kv ? ov : kv;
        ka = oa < ka ? oa : ka;
      }
      if ((tid & 31) == 0) {
        if (kv != ~0ull) atomicMin(&sc->pert_kv, kv);
        if (ka != ~0ull) atomicMin(&sc->pert_ka, ka);
      }
    }
  }
  if (Wk.dirty) {   // f2: mark the columns whose result changes for iteration k + 1; clear set k & 1
    const long long kd = sc->k;
    uint32_t* cur = Wk.dirty + (size_t)(kd & 1) * (Wk.dwords + 1);
    uint32_t* nxt = Wk.dirty + (size_t)((kd + 1) & 1) * (Wk.dwords + 1);
    for (int q = gtid; q <= Wk.dwords; q += gstride) cur[q] = 0u;
    if (d.move) {   // x̄_j* and the row state of the rows of column j*: every column of those rows
      if (gtid == 0) atomicOr(nxt + (d.p >> 5), 1u << (d.p & 31));
      const int e0 = P.col_ptr[d.p], e1 = P.col_ptr[d.p + 1];
      const int lane = tid & 31, gw = gtid >> 5, nw = gstride >> 5;
      for (int e = e0 + gw; e < e1; e += nw) {   // a warp per row of the column
        const int i = P.row_idx[e];
        if ((i == P.cut_row && !cut_active) || i == P.dummy_row) continue;
        if (i == P.cut_row) {   // the dense cutoff row: every column
          if (lane == 0) nxt[Wk.dwords] = 1u;
          continue;
        }
        for (int e2 = P.rp[i] + lane; e2 < P.rp[i + 1]; e2 += 32) {
          const int q = P.ci[e2];
          atomicOr(nxt + (q >> 5), 1u << (q & 31));
        }
      }
    } else if (gtid == 0) {   // a weight bump (every violated row): every column
      nxt[Wk.dwords] = 1u;
    }
  }
  for (int off = 16; off > 0; off >>= 1) dv += __shfl_xor_sync(kFull, dv, off);
  if ((tid & 31) == 0) smv[tid >> 5] = dv;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += smv[q];
    if (solo) {
      s_viol += t;
      sc->violated = s_viol;
    } else if (t) {
      atomicAdd((unsigned long long*)&sc->violated, (unsigned long long)t);
    }
  }
  if (solo) {
    if (tid != 0) return;
  } else {
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&sc->apply_counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last || tid != 0) return;
    __threadfence();
  }
  volatile WalkerScalars* vsc = sc;
  const long long k = solo ? s_k : vsc->k;
  sc->pending_copy = 0;
  if (d.move) {
    x[d.p] = d.v;
    if (Wk.xbits && Wk.rg > 1 && P.vclass[d.p] == 1) {   // the group's bitset (k_eval_bin_wm)
      uint32_t* word = Wk.xbits + (size_t)(w / Wk.rg) * P.n + d.p;
      const uint32_t bit = 1u << (w % Wk.rg);
      if (d.v != 0.0) atomicOr(word, bit); else atomicAnd(word, ~bit);
    } else if (Wk.xbits && Wk.rg == 1 && d.p >= P.rb_pb0 && d.p < P.rb_pb0 + P.rb_nbin) {   // k_eval_binrow
      const int q = d.p - P.rb_pb0, nb = P.n_rblocks, k = q / nb;
      uint32_t* word = Wk.xbits + (size_t)(q % nb) * kRowWpb + (k >> 5);
      const uint32_t bit = 1u << (k & 31);
      if (d.v != 0.0) atomicOr(word, bit); else atomicAnd(word, ~bit);
    }
    Wk.tabu[(size_t)w * Wk.ts + d.p] = (int32_t)(k + 1 + Wk.tenure);
    sc->obj = (solo ? s_obj : vsc->obj) + P.c[d.p] * d.delta;
    sc->n_moves = (solo ? s_nm : vsc->n_moves) + 1;
  } else {
    sc->n_stuck = vsc->n_stuck + 1;
    if (Wk.perturb) {   // R21: the perturbation move, applied by iteration k + 1
      const unsigned long long kv = vsc->pert_kv, ka = vsc->pert_ka;
      sc->pert_kv = ~0ull;
      sc->pert_ka = ~0ull;
      const unsigned long long key = kv != ~0ull ? kv : ka;
      if (key != ~0ull) {
        const int i = (int)(key & 0xFFFFFFFFull);
        const int e0 = P.rp[i], len = P.rp[i + 1] - e0;
        if (len > 0) {
          const unsigned long long h0 =
              splitmix64(splitmix64(splitmix64(Wk.rng_seed) ^ (unsigned long long)w) ^ (unsigned long long)k);
          const int p = P.ci[e0 + (int)(splitmix64(h0 ^ kDrawEntry) % (unsigned long long)len)];
          double v;
          if (perturb_value(P, p, x[p], Wk.perturb_radius, splitmix64(h0 ^ kDrawValue), &v)) {
            sc->force_p = p;
            sc->force_v = v;
          }
        }
      }
    }
  }
  if ((solo ? s_viol : vsc->violated) == 0) {   // PAPER.md:373, R15
    take_incumbent(P, Wk, sc, rw);
    if (Wk.dirty) Wk.dirty[(size_t)((k + 1) & 1) * (Wk.dwords + 1) + Wk.dwords] = 1u;   // the cutoff row moved
  }
  chap_step_record* log = vsc->log;
  if (log) {
    chap_step_record rec;
    rec.k = k;
    rec.j = d.move ? d.j : -1;
    rec.flags = d.pad;   // 1: a perturbation (R21)
    rec.v = d.move ? d.v : NAN;
    rec.s = d.s;
    rec.violated = vsc->violated;
    rec.obj = vsc->obj;
    log[(size_t)(k - vsc->log_k0) * Wk.W + w] = rec;
  }
  sc->k = k + 1;
  sc->apply_counter = 0;
  // kernel timing: the last walker to finish its apply accumulates this iteration's spans and
  // re-arms (kt[14] counts the walkers done; every walker's blocks stamp the same start/end words)
  if (Wk.kt && (Wk.W == 1 || atomicAdd(Wk.kt + 14, 1ull) == (unsigned long long)(Wk.W - 1))) {
    unsigned long long* kt = Wk.kt;
    if (Wk.W > 1) kt[14] = 0ull;
    const unsigned long long now = kt_now();
    for (int q = 0; q < 3; ++q)
      if (kt[2 * q + 1] > kt[2 * q]) kt[8 + q] += kt[2 * q + 1] - kt[2 * q];   // a kernel not launched: 0
    kt[11] += now - kt[6];
    kt[12] += now - min(kt[0], min(kt[2], kt[4]));   // the eval kernels may overlap (forked branch)
    kt[13] += 1;
    for (int q = 0; q < 4; ++q) { kt[2 * q] = ~0ull; kt[2 * q + 1] = 0ull; }
  }
}

// Complete a pending best_x copy (end of chap_tabu_step / before exports).
__global__ void k_flush_incumbent(DevProblem P, DevWalkers Wk) {
  const int w = blockIdx.y;
  WalkerScalars* sc = Wk.sc + w;
  if (!sc->pending_copy) return;
  const double* x = Wk.x + (size_t)w * Wk.xs;
  double* bx = Wk.best_x + (size_t)w * Wk.xs;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) bx[p] = x[p];
}

__global__ void k_flush_done(DevWalkers Wk) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < Wk.W) Wk.sc[w].pending_copy = 0;
}

// Per-walker log pointer and k offset for the coming chap_tabu_step call.
__global__ void k_set_log(DevWalkers Wk, chap_step_record* log) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < Wk.W) {
    Wk.sc[w].log = log;
    Wk.sc[w].log_k0 = Wk.sc[w].k;
  }
}

// Exports in user order.
__global__ void k_export_vars(DevProblem P, DevWalkers Wk, double* x, int64_t* tabu, double* best_x) {
  const int w = blockIdx.y;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) {
    const size_t uo = (size_t)w * P.n + P.perm[p];
    const size_t io = (size_t)w * Wk.xs + p;
    if (x) x[uo] = Wk.x[io];
    if (best_x) best_x[uo] = Wk.best_x[io];
    if (tabu) tabu[uo] = (int64_t)Wk.tabu[(size_t)w * Wk.ts + p];
  }
}

__global__ void k_export_rows(DevProblem P, DevWalkers Wk, double* r, float* wt) {
  const int w = blockIdx.y;
  const RowView rw = row_view(Wk, w);
  const int cut_active = Wk.sc[w].cut_active;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.m_norm; i += gridDim.x * blockDim.x) {
    const RowState s = rw[i];
    if (r) r[(size_t)w * P.m_norm + i] = (i == P.cut_row && !cut_active) ? -INFINITY : s.r;
    if (wt) wt[(size_t)w * P.m_norm + i] = (i == P.cut_row && !cut_active) ? 1.0f : s.w;
  }
}

__global__ void k_export_stats(DevWalkers Wk, chap_walker_stats* st) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= Wk.W) return;
  const WalkerScalars& s = Wk.sc[w];
  chap_walker_stats o;
  o.k = s.k;
  o.violated = s.violated;
  o.obj = s.obj;
  o.best_obj = s.best_obj;
  o.cutoff_rhs = s.cut_active ? s.cutoff_rhs : INFINITY;
  o.has_incumbent = s.has_inc;
  o.pad = 0;
  o.n_moves = s.n_moves;
  o.n_stuck = s.n_stuck;
  st[w] = o;
}

// External cutoff: rhs = min(current, z - δ); residual and violated count updated.
__device__ __forceinline__ void set_cutoff_one(const DevProblem& P, const DevWalkers& Wk, int w, double z) {
  WalkerScalars* sc = Wk.sc + w;
  const RowView rw = row_view(Wk, w);
  const double rhs = z - auto_delta(P, Wk.delta, z);
  if (sc->cut_active && !(rhs < sc->cutoff_rhs)) return;
  const double r_old = sc->cut_active ? rw[P.cut_row].r : -INFINITY;
  const double r_new = sc->obj - rhs;
  sc->violated += (long long)(r_new > 0.0) - (long long)(r_old > 0.0);
  if (!sc->cut_active) rw[P.cut_row].w = 1.0f;
  set_r(rw[P.cut_row], r_new);
  sc->cutoff_rhs = rhs;
  sc->cut_active = 1;
  sc->rint = P.rint_base && rhs == floor(rhs);
}
__global__ void k_set_cutoff(DevProblem P, DevWalkers Wk, double z) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < Wk.W) set_cutoff_one(P, Wk, w, z);
}
// The same with z from device memory (the device exchange's plan); +INF: no incumbent, no change.
__global__ void k_set_cutoff_from(DevProblem P, DevWalkers Wk, const double* z) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < Wk.W && *z < INFINITY) set_cutoff_one(P, Wk, w, *z);
}

// Scalars of the eval API's single virtual walker: k = 0, cutoff from the call.
__global__ void k_eval_scalars(WalkerScalars* sc, double cutoff_rhs, int rint_base) {
  sc->k = 0;
  sc->rint = rint_base && (!(cutoff_rhs < INFINITY) || cutoff_rhs == floor(cutoff_rhs));
  sc->wint = 1;   // cleared by k_rows_init on a non-integral weight or one above 2^20
  sc->cut_active = cutoff_rhs < INFINITY;
  sc->cutoff_rhs = cutoff_rhs;
  sc->cdot = 0.0;
  sc->force_p = -1;
}

}  // namespace chap

namespace chap {

// Exchange summaries (chap_walker_summary) of every walker: one block per walker, the violation
// sum over non-cutoff rows in fixed order.
__global__ void __launch_bounds__(256) k_summaries(DevProblem P, DevWalkers Wk, chap_walker_summary* out,
                                                   int gid0, int stop) {
  __shared__ double sm[32];
  const int w = blockIdx.x, tid = threadIdx.x;
  const RowView rw = row_view(Wk, w);
  double s = 0.0;
  for (int i = tid; i < P.cut_row; i += blockDim.x) {
    const double r = rw[i].r;
    s += r > 0.0 ? r : 0.0;
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if ((tid & 31) == 0) sm[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sm[q];
    const WalkerScalars& sc = Wk.sc[w];
    chap_walker_summary o;
    o.best_obj = sc.has_inc ? sc.best_obj : INFINITY;
    o.violated = sc.violated;
    o.sumviol = t;
    o.gid = gid0 + w;
    o.flags = (sc.has_inc ? 1 : 0) | (stop ? 2 : 0);
    out[w] = o;
  }
}

}  // namespace chap

namespace chap {
// A point (internal order) to its packed form (DevProblem::pk_*): binaries as bits, integers as
// int32 / int64, continuous values as f64.
__device__ __forceinline__ void pack_point(const DevProblem& P, const double* __restrict__ x, unsigned char* out) {
  const int nw = (P.pk_nbin + 31) >> 5;
  uint32_t* words = reinterpret_cast<uint32_t*>(out);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nw + P.pk_nint + P.pk_ncont; q += gridDim.x * blockDim.x) {
    if (q < nw) {
      uint32_t wd = 0u;
      for (int b = 0; b < 32 && 32 * q + b < P.pk_nbin; ++b)
        if (x[P.pk_bin[32 * q + b]] != 0.0) wd |= 1u << b;
      words[q] = wd;
    } else if (q < nw + P.pk_nint) {
      const int sl = q - nw;
      const double v = x[P.pk_int[sl]];
      if (P.pk_int64) reinterpret_cast<long long*>(out + P.pk_off_int)[sl] = (long long)v;
      else reinterpret_cast<int32_t*>(out + P.pk_off_int)[sl] = (int32_t)v;
    } else {
      const int sl = q - nw - P.pk_nint;
      reinterpret_cast<double*>(out + P.pk_off_cont)[sl] = x[P.pk_cont[sl]];
    }
  }
}

__global__ void k_pack_point(DevProblem P, const double* __restrict__ x, unsigned char* out) { pack_point(P, x, out); }

// The inverse: a packed point to internal order (fixed variables at their bound).
__device__ __forceinline__ void unpack_point(const DevProblem& P, const unsigned char* __restrict__ in, double* x) {
  const uint32_t* words = reinterpret_cast<const uint32_t*>(in);
  const int tot = P.n_fixed + P.pk_nbin + P.pk_nint + P.pk_ncont;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += gridDim.x * blockDim.x) {
    if (q < P.n_fixed) {
      x[q] = P.lb[q];
    } else if (q < P.n_fixed + P.pk_nbin) {
      const int sl = q - P.n_fixed;
      x[P.pk_bin[sl]] = (double)((words[sl >> 5] >> (sl & 31)) & 1u);
    } else if (q < P.n_fixed + P.pk_nbin + P.pk_nint) {
      const int sl = q - P.n_fixed - P.pk_nbin;
      x[P.pk_int[sl]] = P.pk_int64 ? (double)reinterpret_cast<const long long*>(in + P.pk_off_int)[sl]
                                   : (double)reinterpret_cast<const int32_t*>(in + P.pk_off_int)[sl];
    } else {
      const int sl = q - P.n_fixed - P.pk_nbin - P.pk_nint;
      x[P.pk_cont[sl]] = reinterpret_cast<const double*>(in + P.pk_off_cont)[sl];
    }
  }
}

__global__ void k_unpack_point(DevProblem P, const unsigned char* __restrict__ in, double* x) { unpack_point(P, in, x); }

// One internal-order point to user order.
__global__ void k_export_point(DevProblem P, const double* xi, double* xu) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P.n; p += gridDim.x * blockDim.x) xu[P.perm[p]] = xi[p];
}
}  // namespace chap

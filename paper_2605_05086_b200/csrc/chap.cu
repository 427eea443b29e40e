// chap.cu — libchap: the C ABI of include/chap.h on sm_100a.
//
// Host side: input validation, row normalisation, variable classification and
// the length-bucketed column dispatch, device upload, and the launch
// sequences of chap_eval_best_shift and chap_tabu_step (captured as CUDA graphs).
// Device side: eval.cuh (Algorithm 1), tabu.cuh (apply / bump / incumbent).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "chap.h"
#include "common.cuh"
#include "eval.cuh"
#include "host.h"
#include "tabu.cuh"

using namespace chap;

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;

chap_status chap::fail(chap_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

extern "C" const char* chap_last_error(void) { return g_err.c_str(); }

extern "C" const char* chap_status_string(chap_status s) {
  switch (s) {
    case CHAP_OK: return "CHAP_OK";
    case CHAP_ERR_INVALID_ARG: return "CHAP_ERR_INVALID_ARG";
    case CHAP_ERR_INFEASIBLE_BOUNDS: return "CHAP_ERR_INFEASIBLE_BOUNDS";
    case CHAP_ERR_CUDA: return "CHAP_ERR_CUDA";
    case CHAP_ERR_OOM: return "CHAP_ERR_OOM";
    case CHAP_ERR_NCCL: return "CHAP_ERR_NCCL";
    case CHAP_ERR_STATE: return "CHAP_ERR_STATE";
    case CHAP_ERR_UNSUPPORTED: return "CHAP_ERR_UNSUPPORTED";
  }
  return "CHAP_ERR_?";
}

extern "C" int32_t chap_abi_version(void) { return CHAP_ABI_VERSION; }


static bool integral(double v) { return std::isfinite(v) && v == std::floor(v); }

extern "C" chap_status chap_problem_create(int32_t n, int32_t m, int64_t nnz, const int64_t* row_ptr,
                                           const int32_t* col_idx, const double* val,
                                           const double* lhs, const double* rhs, const double* lb,
                                           const double* ub, const uint8_t* is_integer,
                                           const double* c, int32_t device, chap_problem** out) {
  if (!out) return fail(CHAP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 0 || m < 0 || nnz < 0) return fail(CHAP_ERR_INVALID_ARG, "negative size");
  if ((m > 0 && (!row_ptr || !lhs || !rhs)) || (nnz > 0 && (!col_idx || !val)) ||
      (n > 0 && (!lb || !ub || !is_integer || !c)))
    return fail(CHAP_ERR_INVALID_ARG, "NULL input array");
  if (m > 0 && (row_ptr[0] != 0 || row_ptr[m] != nnz)) return fail(CHAP_ERR_INVALID_ARG, "row_ptr[0] != 0 or row_ptr[m] != nnz");
  if (m == 0 && nnz != 0) return fail(CHAP_ERR_INVALID_ARG, "nnz > 0 with m = 0");
  for (int32_t i = 0; i < m; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) return fail(CHAP_ERR_INVALID_ARG, "row_ptr decreasing at row %d", i);
    if (std::isnan(lhs[i]) || std::isnan(rhs[i])) return fail(CHAP_ERR_INVALID_ARG, "NaN side in row %d", i);
    if (lhs[i] > rhs[i] || lhs[i] == INFINITY || rhs[i] == -INFINITY)
      return fail(CHAP_ERR_INVALID_ARG, "row %d: lhs > rhs or infinite in the wrong direction", i);
  }
  for (int64_t e = 0; e < nnz; ++e) {
    if (col_idx[e] < 0 || col_idx[e] >= n) return fail(CHAP_ERR_INVALID_ARG, "col_idx[%lld] out of range", (long long)e);
    if (!std::isfinite(val[e])) return fail(CHAP_ERR_INVALID_ARG, "non-finite val[%lld]", (long long)e);
  }
  {  // duplicate (i, j)
    std::vector<int32_t> mark(n, -1);
    for (int32_t i = 0; i < m; ++i)
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        if (mark[col_idx[e]] == i) return fail(CHAP_ERR_INVALID_ARG, "duplicate entry (%d, %d)", i, col_idx[e]);
        mark[col_idx[e]] = i;
      }
  }
  DeviceGuard guard(device);
  if (!guard.ok) return fail(CHAP_ERR_CUDA, "cannot select CUDA device %d", device);

  auto P = new chap_problem();
  std::unique_ptr<chap_problem> holder(P);
  P->device = device;
  cudaDeviceGetAttribute(&P->sm_count, cudaDevAttrMultiProcessorCount, device);
  chap_problem_info& I = P->info;
  I.n = n;
  I.m = m;
  bool exact = true;

  // variables: round integer bounds inward, classify
  std::vector<double> l(n), u(n), cc(n);
  std::vector<uint8_t> vclass(n);
  for (int32_t j = 0; j < n; ++j) {
    double lj = lb[j], uj = ub[j];
    if (std::isnan(lj) || std::isnan(uj) || lj == INFINITY || uj == -INFINITY)
      return fail(CHAP_ERR_INVALID_ARG, "bad bounds of variable %d", j);
    if (!std::isfinite(c[j])) return fail(CHAP_ERR_INVALID_ARG, "non-finite c[%d]", j);
    if (is_integer[j]) {
      lj = std::ceil(lj);
      uj = std::floor(uj);
    }
    if (lj > uj) return fail(CHAP_ERR_INFEASIBLE_BOUNDS, "variable %d: l > u after rounding", j);
    l[j] = lj;
    u[j] = uj;
    cc[j] = c[j];
    uint8_t vc;
    if (lj == uj) vc = 0;
    else if (is_integer[j] && lj == 0.0 && uj == 1.0) vc = 1;
    else if (is_integer[j]) vc = 2;
    else vc = 3;
    vclass[j] = vc;
    if (!is_integer[j]) exact = false;
    if ((std::isfinite(lj) && !integral(lj)) || (std::isfinite(uj) && !integral(uj)) || !integral(c[j])) exact = false;
    if (vc == 0) I.n_fixed++;
    else if (vc == 1) I.n_binary++;
    else if (vc == 2) I.n_integer++;
    else I.n_continuous++;
  }

  // normalised rows: upper side then lower side per original row
  std::vector<int64_t> nrow_ptr{0};
  std::vector<int32_t> ncol;   // user column
  std::vector<double> nval, nb;
  for (int32_t i = 0; i < m; ++i) {
    int64_t k = 0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) k += (val[e] != 0.0);
    if (k == 0) {
      if (lhs[i] > 0.0 || rhs[i] < 0.0) return fail(CHAP_ERR_INFEASIBLE_BOUNDS, "empty row %d excludes 0", i);
      continue;
    }
    for (int s = 0; s < 2; ++s) {
      const double bb = s == 0 ? rhs[i] : -lhs[i];
      if (!std::isfinite(bb)) continue;
      const double sg = s == 0 ? 1.0 : -1.0;
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        if (val[e] == 0.0) continue;
        ncol.push_back(col_idx[e]);
        nval.push_back(sg * val[e]);
        if (!integral(val[e]) || std::fabs(val[e]) > 1e6) exact = false;
      }
      if (!integral(bb)) exact = false;
      nb.push_back(bb);
      P->orig_row.push_back(i);
      P->side.push_back((int8_t)(s == 0 ? 1 : -1));
      nrow_ptr.push_back((int64_t)ncol.size());
    }
  }
  const int32_t mr = (int32_t)nb.size();      // rows without the cutoff row
  const int32_t m_norm = mr + 1;
  const int32_t cut_row = mr;
  int64_t nnz_cut = 0;
  bool delta_int = true;
  for (int32_t j = 0; j < n; ++j)
    if (cc[j] != 0.0) {
      ++nnz_cut;
      if (!integral(cc[j]) || vclass[j] == 3) delta_int = false;
    }
  const int64_t nnz_norm = (int64_t)ncol.size();
  const int64_t nnz_total = nnz_norm + nnz_cut;
  if (nnz_total >= (int64_t)INT32_MAX - 1 || m_norm >= INT32_MAX - 1)
    return fail(CHAP_ERR_INVALID_ARG, "instance too large for 32-bit CSC offsets (%lld nonzeros)", (long long)nnz_total);
  I.m_norm = m_norm;
  I.cutoff_row = cut_row;
  I.nnz_norm = nnz_norm;
  I.nnz_cut = nnz_cut;
  I.exact_integer_data = exact ? 1 : 0;
  // every residual an integer (DevProblem::rint_base): integer data, no continuous variable, and every
  // coefficient (cutoff row included) an integer of magnitude <= 2^22
  bool rint_base = exact && I.n_continuous == 0;
  for (int32_t j = 0; j < n && rint_base; ++j)
    if (std::fabs(cc[j]) > 4194304.0) rint_base = false;
  for (size_t e = 0; e < nval.size() && rint_base; ++e)
    if (std::fabs(nval[e]) > 4194304.0) rint_base = false;
  I.auto_cutoff_delta = delta_int ? 1.0 : NAN;

  // column degrees (incl. the cutoff entry) and classes
  std::vector<int32_t> deg(n, 0);
  for (int64_t e = 0; e < nnz_norm; ++e) deg[ncol[e]]++;
  for (int32_t j = 0; j < n; ++j) deg[j] += (cc[j] != 0.0);
  std::vector<int32_t> cls(n);
  for (int32_t j = 0; j < n; ++j) {
    const int d = deg[j];
    if (vclass[j] == 0) {
      cls[j] = CC_FIXED;
    } else if (d == 0) {
      cls[j] = CC_EMPTY;
    } else if (vclass[j] == 1) {
      cls[j] = (d <= kShortDeg) ? CC_BIN : CC_LBIN;
    } else if (d + 2 <= kShortDeg) {
      cls[j] = vclass[j] == 3 ? CC_GENC : CC_GEN;
    } else if (vclass[j] == 2 && std::isfinite(l[j]) && std::isfinite(u[j]) && u[j] - l[j] + 1.0 <= kBucketMax) {
      cls[j] = CC_LBKT;
    } else if (d + 2 + 3 <= kGenmMax) {   // + up to 3 padding entries
      cls[j] = CC_GENM;
    } else {
      cls[j] = CC_GENL;   // grid-wide sort
    }
  }
  // internal order: fixed columns, then packed binary columns (so that the binary CSC region starts
  // 16-byte aligned), then the other classes; within a class by degree, then user index
  auto order = [](int k) { return k == CC_FIXED ? 0 : (k == CC_BIN ? 1 : 2 + k); };
  std::vector<int32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) {
    if (order(cls[a]) != order(cls[b])) return order(cls[a]) < order(cls[b]);
    return deg[a] > deg[b];
  });
  std::vector<int32_t> iperm(n);
  for (int32_t p = 0; p < n; ++p) iperm[perm[p]] = p;
  // packed tiles (whole columns: binary <= kBinTile - 3, general <= kWTileGen - 3 nonzeros, <= 32
  // columns) and long columns start on a multiple of 4 nonzeros (16-byte vector loads): inert
  // padding entries (the dummy row) are appended to the column before such a start
  std::vector<int32_t> pad(n, 0);
  std::vector<std::pair<int32_t, int32_t>> bin_ranges, gen_ranges, cont_ranges;   // [p0, p1)
  {
    int64_t off = 0;
    auto align_at = [&](int32_t p) {
      if (p > 0 && (off & 3)) {
        const int a = (int)((4 - (off & 3)) & 3);
        pad[p - 1] += a;
        off += a;
      }
    };
    int32_t p = 0;
    while (p < n) {
      const int k = cls[perm[p]];
      if (k == CC_GENC) {   // a lane per column: no alignment, no entry cap
        int cnt = 0;
        while (p + cnt < n && cnt < kWTileCols && cls[perm[p + cnt]] == k) off += deg[perm[p + cnt++]];
        cont_ranges.push_back({p, p + cnt});
        p += cnt;
      } else if (k == CC_BIN || k == CC_GEN) {
        align_at(p);
        const int cap = (k == CC_BIN ? kBinTile : kG32Max) - 3;
        int cnt = 0, tot = 0;
        while (p + cnt < n && cnt < kWTileCols && cls[perm[p + cnt]] == k &&
               tot + deg[perm[p + cnt]] <= cap) {
          tot += deg[perm[p + cnt]];
          ++cnt;
        }
        (k == CC_BIN ? bin_ranges : gen_ranges).push_back({p, p + cnt});
        off += tot;
        p += cnt;
      } else {
        if (k == CC_LBIN || k == CC_LBKT) align_at(p);
        off += deg[perm[p]];
        ++p;
      }
    }
  }
  int64_t npad = 0;
  for (int32_t q = 0; q < n; ++q) npad += pad[q];
  const int32_t dummy_row = m_norm;   // inert row state (r = -inf, w = 0) for padding entries

  // CSC in internal order; rows ascending within a column, then the cutoff entry, then padding
  std::vector<int32_t> col_ptr(n + 1, 0);
  for (int32_t p = 0; p < n; ++p) col_ptr[p + 1] = col_ptr[p] + deg[perm[p]] + pad[p];
  std::vector<int32_t> fill(col_ptr.begin(), col_ptr.end() - 1);
  std::vector<int32_t> row_idx(nnz_total + npad + 4, dummy_row);
  std::vector<double> cval(nnz_total + npad + 4, 1.0);
  for (int32_t i = 0; i < mr; ++i)
    for (int64_t e = nrow_ptr[i]; e < nrow_ptr[i + 1]; ++e) {
      const int32_t p = iperm[ncol[e]];
      row_idx[fill[p]] = i;
      cval[fill[p]] = nval[e];
      fill[p]++;
    }
  for (int32_t j = 0; j < n; ++j)
    if (cc[j] != 0.0) {
      const int32_t p = iperm[j];
      row_idx[fill[p]] = cut_row;
      cval[fill[p]] = cc[j];
      fill[p]++;
    }
  // CSR (internal columns) incl. the cutoff row
  std::vector<int32_t> rp(m_norm + 1);
  std::vector<int32_t> ci;
  std::vector<double> cv;
  ci.reserve(nnz_total);
  cv.reserve(nnz_total);
  rp[0] = 0;
  for (int32_t i = 0; i < mr; ++i) {
    for (int64_t e = nrow_ptr[i]; e < nrow_ptr[i + 1]; ++e) {
      ci.push_back(iperm[ncol[e]]);
      cv.push_back(nval[e]);
    }
    rp[i + 1] = (int32_t)ci.size();
  }
  for (int32_t j = 0; j < n; ++j)
    if (cc[j] != 0.0) {
      ci.push_back(iperm[j]);
      cv.push_back(cc[j]);
    }
  rp[m_norm] = (int32_t)ci.size();
  // per-variable arrays in internal order
  std::vector<double> lbi(n), ubi(n), ci_(n);
  std::vector<uint8_t> vci(n);
  for (int32_t p = 0; p < n; ++p) {
    const int32_t j = perm[p];
    lbi[p] = l[j];
    ubi[p] = u[j];
    ci_[p] = cc[j];
    vci[p] = vclass[j];
  }
  // tiles (PAPER.md:353-355 length dispatch): block tiles — chunks of long columns, single-column
  // sorts — and warp tiles of packed short columns
  std::vector<Tile> tiles;
  std::vector<WTile> wtiles, btiles, bchunks, gchunks;
  std::vector<LongCol> lcols;
  std::vector<int32_t> lfin;
  std::vector<Tile> schunks;
  std::vector<SortCol> scols;
  for (const auto& r : bin_ranges) {
    WTile W{};
    W.p0 = r.first;
    W.e0 = col_ptr[r.first];
    W.e1 = col_ptr[r.second];   // includes the padding (a multiple of 4 nonzeros)
    W.ncols = (int16_t)(r.second - r.first);
    W.kind = (int8_t)CC_BIN;
    btiles.push_back(W);
  }
  for (const auto& r : gen_ranges) {
    WTile W{};
    W.p0 = r.first;
    W.e0 = col_ptr[r.first];
    W.e1 = col_ptr[r.second];
    W.ncols = (int16_t)(r.second - r.first);
    W.kind = (int8_t)CC_GEN;
    for (int32_t q = r.first; q < r.second; ++q) P->gen_kmax = std::max(P->gen_kmax, col_ptr[q + 1] - col_ptr[q]);
    P->gen_tile_nnz += W.e1 - W.e0;
    wtiles.push_back(W);
  }
  const int32_t n_gtiles = (int32_t)wtiles.size();
  for (const auto& r : cont_ranges) {
    WTile W{};
    W.p0 = r.first;
    W.e0 = col_ptr[r.first];
    W.e1 = col_ptr[r.second];
    W.ncols = (int16_t)(r.second - r.first);
    W.kind = (int8_t)CC_GENC;
    wtiles.push_back(W);
  }
  const int32_t n_ctiles = (int32_t)wtiles.size() - n_gtiles;
  int32_t n_long = 0;
  int64_t lscr = 0;
  int32_t p = 0;
  while (p < n) {
    const int32_t j = perm[p];
    const int k = cls[j];
    if (k == CC_FIXED || k == CC_BIN) { ++p; continue; }
    if (k == CC_GEN || k == CC_GENC) { ++p; continue; }   // packed in gen_ranges / cont_ranges
    if (k == CC_EMPTY) {
      int cnt = 0;
      while (p + cnt < n && cnt < kWTileCols && cls[perm[p + cnt]] == k) ++cnt;
      WTile W{};
      W.p0 = p;
      W.e0 = col_ptr[p];
      W.e1 = col_ptr[p + cnt];
      W.ncols = (int16_t)cnt;
      W.kind = (int8_t)k;
      wtiles.push_back(W);
      p += cnt;
      continue;
    }
    Tile T{};
    T.kind = k;
    T.p0 = p;
    T.ncols = 1;
    if (k == CC_GENL) {   // chunks of <= kSortChunk entries, sorted per block, co-ranked
      SortCol S{};
      S.scr = lscr;
      S.p = p;
      const int d = col_ptr[p + 1] - col_ptr[p];   // incl. any padding (inert: emits nothing)
      S.nchunks = (d + kSortChunk - 1) / kSortChunk;
      for (int c = 0; c < S.nchunks; ++c) {
        Tile C{};
        C.kind = CC_GENL;
        C.p0 = p;
        C.ncols = c;
        C.e0 = col_ptr[p] + c * kSortChunk;
        C.e1 = std::min(col_ptr[p + 1], C.e0 + kSortChunk);
        C.pad = (int32_t)scols.size();
        schunks.push_back(C);
      }
      lscr += (int64_t)S.nchunks * kSortStride;
      scols.push_back(S);
      ++p;
      continue;
    }
    if (k == CC_GENM) {
      T.e0 = col_ptr[p];
      T.e1 = col_ptr[p + 1];
      tiles.push_back(T);
      ++p;
      continue;
    }
    // long columns: warp chunks of kWChunk nonzeros, accumulated with atomics into per-column
    // accumulators (binary: the flip sum; bounded integer: bucket deltas, candidate bits, β, α);
    // k_eval finishes the column
    const int d = col_ptr[p + 1] - col_ptr[p];   // incl. any padding (inert)
    const int csz = (k == CC_LBKT) ? kBktChunk : kWChunk;
    const int nch = std::max(1, (d + csz - 1) / csz);
    const int dom = (k == CC_LBKT) ? (int)(u[j] - l[j] + 1.0) : 0;
    if (k == CC_LBKT) P->lbkt_nnz += d;
    for (int q = 0; q < nch; ++q) {
      WTile W{};
      W.p0 = p;
      W.e0 = col_ptr[p] + q * csz;
      W.e1 = n_long;
      W.ncols = (int16_t)(std::min(col_ptr[p + 1], col_ptr[p] + (q + 1) * csz) - W.e0);
      W.kind = (int8_t)k;
      (k == CC_LBIN ? bchunks : gchunks).push_back(W);
    }
    LongCol L{};
    L.scr = lscr;
    L.tix = lscr + ((k == CC_LBKT) ? ((int64_t)dom + 1 + 2 + (dom + 63) / 64) : 1);
    L.nchunks = nch;
    L.dom = dom;
    L.p = p;
    L.kind = k;
    if (k == CC_LBKT || nch > 1) lfin.push_back(n_long);
    lcols.push_back(L);
    lscr = L.tix + 1;   // accumulators, then the chunk ticket
    ++n_long;
    ++p;
  }
  I.n_long_columns = n_long;
  I.n_sorted_columns = 0;
  I.n_gridsort_columns = 0;
  for (int32_t j = 0; j < n; ++j) {
    I.n_sorted_columns += (cls[j] == CC_GENM || cls[j] == CC_GENL);
    I.n_gridsort_columns += (cls[j] == CC_GENL);
  }
  // row-wise binary blocks (k_eval_binrow): packed binary columns [pb0, pb1) in blocks of <=
  // kRowVmax columns balanced by nonzeros, a multiple of the resident clusters; each block's
  // entries sorted by row, cut into kRowCluster slices padded to multiples of 4 with inert entries
  std::vector<RowBlock> rblocks;
  std::vector<int32_t> rb_row;
  std::vector<uint32_t> rb_cv;
  std::vector<RowStage> rb_stage;
  std::vector<int32_t> rb_perm;
  {
    int32_t pb0 = -1, pb1 = -1;
    for (int32_t q = 0; q < n; ++q)
      if (cls[perm[q]] == CC_BIN) {
        if (pb0 < 0) pb0 = q;
        pb1 = q + 1;
      }
    bool ok = pb0 >= 0;
    int64_t tot = 0;
    int maxdeg = 0;
    for (int32_t q = pb0; ok && q < pb1; ++q) {
      int d = 0;
      for (int32_t e = col_ptr[q]; e < col_ptr[q + 1]; ++e) {
        if (row_idx[e] == dummy_row) continue;
        const double a = cval[e];
        if (!(a == std::floor(a) && std::fabs(a) <= 32767.0)) ok = false;
        ++d;
      }
      tot += d;
      maxdeg = std::max(maxdeg, d);
    }
    // cluster width: the one that keeps the most SMs busy (clusters live inside a GPC), the wider
    // on ties (fewer, larger blocks: more entries per row, denser row-state reads)
    int ncl = 0, C = 0, nb = 0;
    int32_t nbin = 0;
    if (ok) {
      cudaError_t e1 = cudaFuncSetAttribute(k_eval_binrow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem);
      if (cudaFuncSetAttribute(k_eval_binrow, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        cudaGetLastError();
      if (e1 == cudaSuccess) {
#ifndef CHAP_ROW_CMAX
#define CHAP_ROW_CMAX kRowCluster
#endif
#ifndef CHAP_ROW_CMIN
#define CHAP_ROW_CMIN 4
#endif
        for (int c = CHAP_ROW_CMAX; c >= CHAP_ROW_CMIN; --c) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(c * std::max(1, P->sm_count / c));
          cfg.blockDim = dim3(kRowThreads);
          cfg.dynamicSmemBytes = kRowSmem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = c;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int k = 0;
          if (cudaOccupancyMaxActiveClusters(&k, k_eval_binrow, &cfg) != cudaSuccess) k = 0;
          if (k < 1) continue;
          // fewest rounds of blocks first (a block holds <= kRowVmax columns), then the most SMs
          auto rounds = [&](int kc) { return (int)(((int64_t)(pb1 - pb0) + (int64_t)kc * kRowVmax - 1) / ((int64_t)kc * kRowVmax)); };
          if (ncl == 0 || rounds(k) < rounds(ncl) || (rounds(k) == rounds(ncl) && k * c > ncl * C)) { ncl = k; C = c; }
        }
      }
      cudaGetLastError();
      if (ncl < 1) ok = false;
    }
    if (ok) {
      // blocks: nb, a multiple of the resident clusters, with <= kRowVmax columns each; column
      // p = pb0 + b + k nb is column k of block b (round-robin over the degree-sorted columns, so
      // every block gets an equal mix of long and short columns and about tot / nb entries)
      nbin = pb1 - pb0;
      nb = std::max(ncl, (nbin + kRowVmax - 1) / kRowVmax);
      nb = (nb + ncl - 1) / ncl * ncl;
      // where the row-wise kernel pays (measured on the X sweep): enough nonzeros to
      // amortise the cluster launch and the per-block reduction, and enough entries per row of a
      // block that a warp's consecutive entries share row-state lines (chap_params.binary_kernel
      // overrides the rule per walkers object)
      const double density = (double)tot / ((double)nb * std::max(1, m_norm));
      P->binrow_auto = tot >= 3000000 && density >= 0.7;
    }
    if (ok) {
      std::vector<int32_t> cnt(m_norm + 2, 0);
      for (int b = 0; b < nb; ++b) {
        const int32_t nvb = (nbin - b + nb - 1) / nb;   // columns pb0 + b, pb0 + b + nb, ...
        // counting sort of the block's entries by row (stable in column order)
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int32_t k = 0; k < nvb; ++k) {
          const int32_t c = pb0 + b + k * nb;
          for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e)
            if (row_idx[e] != dummy_row) ++cnt[row_idx[e] + 1];
        }
        for (int32_t i = 0; i <= m_norm; ++i) cnt[i + 1] += cnt[i];
        const int64_t E = cnt[m_norm];
        std::vector<int32_t> er(E);
        std::vector<uint32_t> ec(E);
        for (int32_t k = 0; k < nvb; ++k) {
          const int32_t c = pb0 + b + k * nb;
          for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
            const int32_t i = row_idx[e];
            if (i == dummy_row) continue;
            const int32_t at = cnt[i]++;
            er[at] = i;
            ec[at] = (uint32_t)k | ((uint32_t)(uint16_t)(int16_t)cval[e] << 16);
          }
        }
        RowBlock R{};
        R.p0 = pb0 + b;
        R.nv = nvb;
        // slice s: the s-th C-th of the entries of rows < cut_row, then the s-th C-th of the
        // (dense, last) cutoff row's entries, so that every slice carries an equal share of both
        const int64_t E1 = cut_row > 0 ? cnt[cut_row - 1] : 0;   // (after the scatter cnt[i] = end of row i)
        const int64_t E2 = E - E1;
        for (int sl = 0; sl < C; ++sl) {
          R.es[sl] = (int32_t)rb_row.size();
          for (int half = 0; half < 2; ++half) {
            const int64_t base = half ? E1 : 0, len = half ? E2 : E1;
            for (int64_t k = base + len * sl / C; k < base + len * (sl + 1) / C; ++k) {
              rb_row.push_back(er[k]);
              rb_cv.push_back(ec[k]);
            }
          }
          while (rb_row.size() & 3) {   // inert padding (the dummy row)
            rb_row.push_back(dummy_row);
            rb_cv.push_back(0u);
          }
        }
        for (int sl = C; sl <= kRowCluster; ++sl) R.es[sl] = (int32_t)rb_row.size();
        // stages of each slice: <= kRowChunk entries (whole groups of 4) whose rows span <= kRowSpan
        // rows (padding entries, rb_cv = 0, take no row); a single group wider than that gathers
        for (int sl = 0; sl <= kRowCluster; ++sl) {
          R.st[sl] = (int32_t)rb_stage.size();
          if (sl >= C) continue;
          for (int64_t e = R.es[sl], e1; e < R.es[sl + 1]; e = e1) {
            int32_t lo = INT32_MAX, hi = -1;
            for (e1 = e; e1 < R.es[sl + 1] && e1 - e + 4 <= kRowChunk; e1 += 4) {
              int32_t glo = lo, ghi = hi;
              for (int64_t k = e1; k < e1 + 4; ++k)
                if (rb_cv[k] != 0u) { glo = std::min(glo, rb_row[k]); ghi = std::max(ghi, rb_row[k]); }
              if (!CHAP_ROW_GATHER && e1 > e && ghi >= 0 && ghi - glo + 1 > kRowSpan) break;
              lo = glo;
              hi = ghi;
            }
            RowStage G{};
            G.e0 = (int32_t)e;
            G.ne = (int32_t)(e1 - e);
            const bool fits = !CHAP_ROW_GATHER && hi >= 0 && hi - lo + 1 <= kRowSpan;
            G.r0 = fits ? lo : 0;
            G.nr = fits ? hi - lo + 1 : 0;
            rb_stage.push_back(G);
          }
        }
        rblocks.push_back(R);
      }
      if (getenv("CHAP_DEBUG"))
        fprintf(stderr, "[chap] binrow: %d clusters x %d CTAs, %zu blocks, %lld entries (%lld stored)\n", ncl, C,
                rblocks.size(), (long long)tot, (long long)rb_row.size());
      rb_perm.assign((size_t)nb * kRowVmax, -1);
      for (int32_t q = 0; q < nbin; ++q) rb_perm[(size_t)(q % nb) * kRowVmax + q / nb] = perm[pb0 + q];
      P->binrow_grid = ncl * C;
      P->binrow_pb0 = pb0;
      P->binrow_nbin = nbin;
      P->binrow_cluster = C;
      P->binrow_maxdeg = maxdeg;
      P->binrow_entries = (int64_t)rb_row.size();
    }
  }
  {  // algorithmic-bytes model: 12 B per ORIGINAL nonzero (a two-sided
     // row's entry counts once, R17) and per cutoff entry, whatever the kernels store or gather
    std::vector<int32_t> odeg(n, 0);
    for (int64_t e = 0; e < nnz; ++e) odeg[col_idx[e]] += (val[e] != 0.0);
    for (int32_t j = 0; j < n; ++j) odeg[j] += (cc[j] != 0.0);
    int64_t mb[3] = {0, 0, 0}, nz[3] = {0, 0, 0}, mw[3] = {0, 0, 0};
    for (int32_t q = 0; q < n; ++q) {
      const int32_t j = perm[q];
      const int k = cls[j];
      if (k == CC_FIXED) continue;
      // [0] packed binary columns, [1] long binary, general, empty and long bounded-integer
      // columns, [2] sorted general columns and the row state
      const int kk = (k == CC_BIN) ? 0 : ((k == CC_GENM || k == CC_GENL) ? 2 : 1);
      const bool bin = vclass[j] == 1;
      const double per_var = 4.0 + (bin ? 1.0 + 0.125 : 17.0 + 8.0) + 4.0;   // col_ptr, static, x̄, tabu
      mb[kk] += 12LL * odeg[j] + (int64_t)std::llround(per_var * 8) / 8;
      mw[kk] += (int64_t)std::llround(((bin ? 0.125 : 8.0) + 4.0) * 8) / 8;   // x̄, tabu
      nz[kk] += odeg[j];
    }
    mb[2] += 12LL * m_norm;   // the row state, read once per pass (attributed to the last kernel)
    mw[2] += 12LL * m_norm;
    for (int q = 0; q < 3; ++q) {
      I.model_bytes_kernel[q] = mb[q];
      I.model_bytes_walker_kernel[q] = mw[q];
      I.nnz_kernel[q] = nz[q];
    }
    I.model_bytes_pass = mb[0] + mb[1] + mb[2];
  }
  P->lscr_per_walker = (size_t)std::max<int64_t>(lscr, 1);

  // upload
  DeviceBuffers& B = P->buf;
  int32_t *d_col_ptr, *d_row_idx, *d_rp, *d_ci, *d_perm;
  double *d_val, *d_cv, *d_b, *d_lb, *d_ub, *d_c;
  uint8_t* d_vc;
  Tile* d_tiles;
  WTile* d_wtiles;
  WTile* d_btiles;
  LongCol* d_lcols;
  WTile *d_bchunks, *d_gchunks;
  TRY(B.upload(&d_col_ptr, col_ptr));
  TRY(B.upload(&d_row_idx, row_idx));
  TRY(B.upload(&d_val, cval));
  TRY(B.upload(&d_rp, rp));
  TRY(B.upload(&d_ci, ci));
  TRY(B.upload(&d_cv, cv));
  TRY(B.upload(&d_b, nb));
  TRY(B.upload(&d_lb, lbi));
  TRY(B.upload(&d_ub, ubi));
  TRY(B.upload(&d_c, ci_));
  TRY(B.upload(&d_vc, vci));
  TRY(B.upload(&d_perm, perm));
  TRY(B.upload(&d_tiles, tiles));
  TRY(B.upload(&d_wtiles, wtiles));
  TRY(B.upload(&d_btiles, btiles));
  TRY(B.upload(&d_bchunks, bchunks));
  TRY(B.upload(&d_gchunks, gchunks));
  // the chunk region: long binary and long bounded-integer chunks spread evenly over each other
  // (the bounded-integer chunks' long latency chains start throughout the first waves instead of
  // all after the binary ones: G k_eval_gen 61.2 -> 59.8 us), then the tiles
  std::vector<WTile> gitems;
  {
    const size_t nb_ = bchunks.size(), ng_ = gchunks.size();
    size_t ib = 0, ig = 0;
    while (ib < nb_ || ig < ng_) {
      const bool take_g = ig < ng_ && (ib >= nb_ || ig * (nb_ + ng_) <= (ib + ig) * ng_);
      gitems.push_back(take_g ? gchunks[ig++] : bchunks[ib++]);
    }
  }
  gitems.insert(gitems.end(), wtiles.begin() + n_gtiles, wtiles.begin() + n_gtiles + n_ctiles);
  gitems.insert(gitems.end(), wtiles.begin(), wtiles.begin() + n_gtiles);
  gitems.insert(gitems.end(), wtiles.begin() + n_gtiles + n_ctiles, wtiles.end());
  WTile* d_gitems;
  TRY(B.upload(&d_gitems, gitems));
  // the list of the modes where k_eval_bin / k_eval_bin_wm take the long binary chunks
  std::vector<WTile> gitems2(gchunks);
  gitems2.insert(gitems2.end(), gitems.begin() + bchunks.size() + gchunks.size(), gitems.end());
  WTile* d_gitems2;
  TRY(B.upload(&d_gitems2, gitems2));
  P->h_lcols = lcols;   // (host copy: walker creation checks the long bounded-integer domains)
  if (lcols.empty()) lcols.push_back(LongCol{});
  int32_t* d_lfin;
  TRY(B.upload(&d_lfin, lfin));
  TRY(B.upload(&d_lcols, lcols));
  Tile* d_schunks;
  SortCol* d_scols;
  TRY(B.upload(&d_schunks, schunks));
  TRY(B.upload(&d_scols, scols));
  RowBlock* d_rblocks;
  int2* d_rb_rc;
  TRY(B.upload(&d_rblocks, rblocks));
  {
    std::vector<int2> rc(rb_row.size());
    for (size_t q = 0; q < rb_row.size(); ++q) rc[q] = make_int2(rb_row[q], (int)rb_cv[q]);
    TRY(B.upload(&d_rb_rc, rc));
  }
  RowStage* d_rb_stage;
  TRY(B.upload(&d_rb_stage, rb_stage));
  int32_t* d_rb_perm;
  TRY(B.upload(&d_rb_perm, rb_perm));
  DevProblem& D = P->dp;
  D.rb_stage = d_rb_stage;
  D.rblocks = d_rblocks;
  D.n_rblocks = (int32_t)rblocks.size();
  D.n_gtiles = n_gtiles;
  D.n_ctiles = n_ctiles;
  D.rb_cluster = P->binrow_cluster;
  D.rb_pb0 = P->binrow_pb0;
  D.rb_perm = d_rb_perm;
  D.rb_nbin = P->binrow_nbin;
  D.rb_rc = d_rb_rc;
  D.n = n;
  D.m_norm = m_norm;
  D.cut_row = cut_row;
  D.dummy_row = dummy_row;
  D.col_ptr = d_col_ptr;
  D.row_idx = d_row_idx;
  D.val = d_val;
  D.rp = d_rp;
  D.ci = d_ci;
  D.cv = d_cv;
  D.b = d_b;
  D.lb = d_lb;
  D.ub = d_ub;
  D.c = d_c;
  D.vclass = d_vc;
  D.perm = d_perm;
  D.tiles = d_tiles;
  D.n_tiles = (int32_t)tiles.size();
  D.wtiles = d_wtiles;
  D.n_wtiles = (int32_t)wtiles.size();
  D.btiles = d_btiles;
  D.n_btiles = (int32_t)btiles.size();
  D.lcols = d_lcols;
  D.schunks = d_schunks;
  D.n_schunks = (int32_t)schunks.size();
  D.scols = d_scols;
  D.n_scols = (int32_t)scols.size();
  D.lfin = d_lfin;
  D.n_lfin = (int32_t)lfin.size();
  D.bchunks = d_bchunks;
  D.n_bchunks = (int32_t)bchunks.size();
  D.gchunks = d_gchunks;
  D.gitems = d_gitems;
  D.n_gitems = (int32_t)gitems.size();
  D.gitems2 = d_gitems2;
  D.n_gitems2 = (int32_t)gitems2.size();
  D.n_gchunks = (int32_t)gchunks.size();
  D.n_long = n_long;
  D.n_fixed = I.n_fixed;
  D.auto_delta = I.auto_cutoff_delta;
  D.rint_base = rint_base ? 1 : 0;
  {  // packed exchange points: the internal columns of each class
    std::vector<int32_t> kb, ki, kc;
    bool i64 = false;
    for (int32_t q = 0; q < n; ++q) {
      const int32_t j = perm[q];
      if (vclass[j] == 1) kb.push_back(q);
      else if (vclass[j] == 2) {
        ki.push_back(q);
        if (!(std::isfinite(l[j]) && std::isfinite(u[j]) && std::fabs(l[j]) < 2147483647.0 && std::fabs(u[j]) < 2147483647.0))
          i64 = true;
      } else if (vclass[j] == 3) kc.push_back(q);
    }
    int32_t *d_kb, *d_ki, *d_kc;
    TRY(B.upload(&d_kb, kb));
    TRY(B.upload(&d_ki, ki));
    TRY(B.upload(&d_kc, kc));
    D.pk_bin = d_kb;
    D.pk_int = d_ki;
    D.pk_cont = d_kc;
    D.pk_nbin = (int32_t)kb.size();
    D.pk_nint = (int32_t)ki.size();
    D.pk_ncont = (int32_t)kc.size();
    D.pk_int64 = i64 ? 1 : 0;
    auto al8 = [](int64_t b) { return (b + 7) & ~(int64_t)7; };
    D.pk_off_int = al8(4LL * ((D.pk_nbin + 31) / 32));
    D.pk_off_cont = al8(D.pk_off_int + (int64_t)D.pk_nint * (i64 ? 8 : 4));
    D.pk_bytes = std::max<int64_t>(8, al8(D.pk_off_cont + 8LL * D.pk_ncont));
    I.exchange_point_bytes = D.pk_bytes;
  }

  // launch geometry: a persistent grid of (resident blocks) per walker set
  CUDA_TRY(cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
  CUDA_TRY(cudaFuncSetAttribute(k_sort_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
  int occ = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval, kTileThreads, kTileSmem));
  P->eval_occ = std::max(1, occ);
  const int ework = std::max(std::max(D.n_tiles, (D.n_lfin + kTileWarps - 1) / kTileWarps),
                             std::max(1, (D.n_scols + kTileThreads - 1) / kTileThreads));
  P->eval_grid = std::max(1, std::min(ework, P->eval_occ * P->sm_count));
  CUDA_TRY(cudaFuncSetAttribute(k_eval_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGenSmem));
  int gocc = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gocc, k_eval_gen, kGenThreads, kGenSmem));
  P->gen_occ = std::max(1, gocc);
  const int gwarps = kGenThreads / 32;
  const int gwork = D.n_wtiles + D.n_gchunks;
  P->gen_grid = gwork ? std::max(1, std::min((gwork + gwarps - 1) / gwarps, P->gen_occ * P->sm_count)) : 0;
  CUDA_TRY(cudaFuncSetAttribute(k_eval_bin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBinSmem));
  int bocc = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, k_eval_bin, kBinThreads, kBinSmem));
  P->bin_occ = std::max(1, bocc);
  const int bwarps = kBinThreads / 32;
  const int bwork = D.n_btiles + D.n_bchunks;
  P->bin_grid = bwork ? std::max(1, std::min((bwork + bwarps - 1) / bwarps, P->bin_occ * P->sm_count)) : 0;
  P->bin_chunk_grid = D.n_bchunks ? std::max(1, std::min((D.n_bchunks + bwarps - 1) / bwarps, P->bin_occ * P->sm_count)) : 0;
  P->info.eval_launches = 1 + (P->bin_grid > 0) + (P->gen_grid > 0);
  P->rows_grid = std::max(1, std::min((m_norm + 7) / 8, 8 * P->sm_count));
  // eval workspace
  TRY(B.alloc(&P->e_x, n));
  TRY(B.alloc(&P->e_rs, (size_t)m_norm + 1));
  TRY(B.alloc(&P->e_tabu, n));
  TRY(B.alloc(&P->e_bx, n));
  TRY(B.alloc(&P->e_sc, 1));
  TRY(B.alloc(&P->e_part, P->eval_grid + P->bin_grid + P->gen_grid));
  TRY(B.alloc(&P->e_selcnt, 3));   // the select counter, then k_eval_gen's item counters
  TRY(B.alloc(&P->e_bad, 1));
  CUDA_TRY(cudaMallocHost(&P->h_bad, sizeof(int)));
  *P->h_bad = 0;
  CUDA_TRY(cudaMemset(P->e_selcnt, 0, 3 * sizeof(unsigned)));
  TRY(B.alloc(&P->e_lscr, P->lscr_per_walker));
  CUDA_TRY(cudaMemset(P->e_sc, 0, sizeof(WalkerScalars)));
  CUDA_TRY(cudaMemset(P->e_lscr, 0, sizeof(double) * P->lscr_per_walker));
  CUDA_TRY(cudaMemset(P->e_tabu, 0, sizeof(int32_t) * std::max(n, 1)));
  CUDA_TRY(cudaDeviceSynchronize());
  I.device_bytes = (int64_t)B.bytes_total;
  {
    int64_t nnz_orig = 0;
    for (int64_t e = 0; e < nnz; ++e) nnz_orig += (val[e] != 0.0);
    I.model_bytes_A = 12LL * (nnz_orig + nnz_cut) + 4LL * (n + 1);
  }
  *out = holder.release();
  return CHAP_OK;
}

extern "C" chap_status chap_problem_info_get(const chap_problem* p, chap_problem_info* out) {
  if (!p || !out) return fail(CHAP_ERR_INVALID_ARG, "NULL argument");
  *out = p->info;
  return CHAP_OK;
}

extern "C" chap_status chap_problem_row_map(const chap_problem* p, int32_t* orig_row, int8_t* side) {
  if (!p) return fail(CHAP_ERR_INVALID_ARG, "NULL problem");
  const size_t k = p->orig_row.size();
  if (orig_row && k) memcpy(orig_row, p->orig_row.data(), k * sizeof(int32_t));
  if (side && k) memcpy(side, p->side.data(), k * sizeof(int8_t));
  return CHAP_OK;
}

extern "C" chap_status chap_problem_destroy(chap_problem* p) {
  if (!p) return CHAP_OK;
  DeviceGuard g(p->device);
  delete p;
  return CHAP_OK;
}

// ------------------------------------------------------------------------------------------
// eval launches (shared by the eval API and the tabu step)
// ------------------------------------------------------------------------------------------
// Kernel launch through cudaLaunchKernelEx: optional cluster shape and, for the kernels of a tabu
// iteration, programmatic dependent launch (each kernel starts with pdl_wait_trigger()).
template <typename... KArgs, typename... Args>
static chap_status lk(void (*kern)(KArgs...), dim3 grid, int block, size_t smem, cudaStream_t s, bool pdl,
                      int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return CHAP_OK;
}

static chap_status launch_bin_wm(const DevProblem& D, const DevWalkers& Wk, int bgrid, cudaStream_t s, bool pdl) {
  const dim3 grid(bgrid, Wk.n_groups);
  switch (Wk.rg) {
    case 2: TRY(lk(k_eval_bin_wm<2>, grid, kBinWmThreads, 0, s, pdl, 1, D, Wk)); break;
    case 4: TRY(lk(k_eval_bin_wm<4>, grid, kBinWmThreads, 0, s, pdl, 1, D, Wk)); break;
    case 8: TRY(lk(k_eval_bin_wm<8>, grid, kBinWmThreads, 0, s, pdl, 1, D, Wk)); break;
    case 16: TRY(lk(k_eval_bin_wm<16>, grid, kBinWmThreads, 0, s, pdl, 1, D, Wk)); break;
    case 32: TRY(lk(k_eval_bin_wm<32>, grid, kBinWmThreads, 0, s, pdl, 1, D, Wk)); break;
    default: return fail(CHAP_ERR_STATE, "row-state group width %d", Wk.rg);
  }
  return CHAP_OK;
}

static chap_status launch_gen_wm(const chap_problem* P, const DevWalkers& Wk, int wgrid, int part_base, cudaStream_t s,
                                 bool pdl) {
  const dim3 grid(wgrid, Wk.n_groups);
  const int kmax = std::max(1, P->gen_kmax);
  const size_t sm = gen_wm_smem_all(kmax, Wk.lbkt_wm_words);
  switch (Wk.rg) {
    case 1: TRY(lk(k_eval_gen_wm<1>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    case 2: TRY(lk(k_eval_gen_wm<2>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    case 4: TRY(lk(k_eval_gen_wm<4>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    case 8: TRY(lk(k_eval_gen_wm<8>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    case 16: TRY(lk(k_eval_gen_wm<16>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    case 32: TRY(lk(k_eval_gen_wm<32>, grid, kGenWmThreads, sm, s, pdl, 1, P->dp, Wk, part_base, kmax)); break;
    default: return fail(CHAP_ERR_STATE, "row-state group width %d", Wk.rg);
  }
  return CHAP_OK;
}

template <int RG>
static int gen_wm_occ_one(size_t sm) {
  int occ = 0;
  if (cudaFuncSetAttribute(k_eval_gen_wm<RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_gen_wm<RG>, kGenWmThreads, sm) != cudaSuccess)
    occ = 0;
  cudaGetLastError();
  return occ;
}
static int gen_wm_occupancy(int rg, size_t sm) {
  switch (rg) {
    case 1: return gen_wm_occ_one<1>(sm);
    case 2: return gen_wm_occ_one<2>(sm);
    case 4: return gen_wm_occ_one<4>(sm);
    case 8: return gen_wm_occ_one<8>(sm);
    case 16: return gen_wm_occ_one<16>(sm);
    default: return gen_wm_occ_one<32>(sm);
  }
}

static int bin_wm_occupancy(int rg) {
  int occ = 1;
  cudaError_t e = cudaSuccess;
  switch (rg) {
    case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_bin_wm<2>, kBinWmThreads, 0); break;
    case 4: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_bin_wm<4>, kBinWmThreads, 0); break;
    case 8: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_bin_wm<8>, kBinWmThreads, 0); break;
    case 16: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_bin_wm<16>, kBinWmThreads, 0); break;
    default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_bin_wm<32>, kBinWmThreads, 0); break;
  }
  return e == cudaSuccess ? std::max(1, occ) : 1;
}

static chap_status launch_binrow(const chap_problem* P, const DevWalkers& Wk, int rgrid, int part_base,
                                 cudaStream_t s, bool pdl) {
  return lk(k_eval_binrow, dim3(rgrid), kRowThreads, kRowSmem, s, pdl, P->binrow_cluster, P->dp, Wk, part_base);
}

// Part slots of one walker: [k_eval_bin | k_eval_gen | k_eval_binrow | k_eval]; k_eval reduces them.
chap_status chap::launch_eval(const chap_problem* P, const DevWalkers& Wk, int grid, int bgrid, int ggrid,
                              int rgrid, int wgrid, double* oxhat, double* oscore, chap_move* best,
                              cudaStream_t s, bool pdl, int sel_grid) {
  // k_eval only selects when there are no long columns and no sort tiles: then the last eval kernel
  // (k_eval_gen, else k_eval_bin) selects in its last block and k_eval is not launched
  // sel_grid > 0 (chap_params.lazy): the eval kernels only refresh the per-column cache, k_eval runs
  // only for the sort tiles, and k_select_cache selects
  const bool lazy = sel_grid > 0;
  const bool sel_only = !lazy && Wk.W == 1 && Wk.rg == 1 && P->dp.n_tiles == 0 && P->dp.n_scols == 0 && wgrid == 0;
  const int gen_sel = (sel_only && ggrid > 0) ? bgrid + ggrid + rgrid : 0;
  const int bin_sel = (sel_only && ggrid == 0 && rgrid == 0 && bgrid > 0) ? bgrid : 0;
  if (bgrid > 0) {
    if (Wk.rg > 1) {
      TRY(launch_bin_wm(P->dp, Wk, bgrid, s, pdl));
    } else {
      DevProblem D = P->dp;
      if (rgrid > 0) D.n_btiles = 0;   // packed binary columns row-wise: k_eval_bin takes the long chunks only
      TRY(lk(k_eval_bin, dim3(bgrid, Wk.W), kBinThreads, kBinSmem, s, pdl, 1, D, Wk, oxhat, oscore, bin_sel, best));
    }
  }
  if (rgrid > 0) TRY(launch_binrow(P, Wk, rgrid, bgrid + ggrid, s, pdl));
  if (ggrid > 0)
    TRY(lk(k_eval_gen, dim3(ggrid, Wk.W), kGenThreads, kGenSmem, s, pdl, 1, P->dp, Wk, oxhat, oscore, bgrid,
           wgrid > 0 ? 1 : 0, (rgrid > 0 && bgrid == 0) ? 1 : 0, gen_sel, best));
  if (wgrid > 0) TRY(launch_gen_wm(P, Wk, wgrid, bgrid + ggrid + rgrid, s, pdl));
  if (P->dp.n_schunks > 0) {   // long general columns: chunk sorts, then co-ranking (k_eval finishes them)
    TRY(lk(k_sort_chunks, dim3(P->dp.n_schunks, Wk.W), kTileThreads, kTileSmem, s, pdl, 1, P->dp, Wk));
    TRY(lk(k_sort_rank, dim3(P->dp.n_schunks, Wk.W), kTileThreads, 0, s, pdl, 1, P->dp, Wk));
  }
  if (!gen_sel && !bin_sel && (!lazy || P->dp.n_tiles > 0 || P->dp.n_scols > 0))
    TRY(lk(k_eval, dim3(grid, Wk.W), kTileThreads, kTileSmem, s, pdl, 1, P->dp, Wk, oxhat, oscore, best,
           bgrid + ggrid + rgrid + wgrid, Wk.rg > 1 ? 1 : 0));
  if (lazy) TRY(lk(k_select_cache, dim3(sel_grid), kTileThreads, 0, s, pdl, 1, P->dp, Wk));
  return CHAP_OK;
}

static DevWalkers eval_walkers(const chap_problem* P) {
  DevWalkers Wk{};
  Wk.x = P->e_x;
  Wk.xs = (size_t)P->dp.n;
  Wk.rs = P->e_rs;
  Wk.rss = (size_t)P->dp.m_norm + 1;
  Wk.rg = 1;
  Wk.n_groups = 1;
  Wk.xbits = nullptr;
  Wk.tabu = P->e_tabu;
  Wk.ts = (size_t)P->dp.n;
  Wk.best_x = P->e_bx;
  Wk.sc = P->e_sc;
  Wk.part = P->e_part;
  Wk.ps = P->eval_grid + P->bin_grid + P->gen_grid;
  Wk.sel_count = P->e_selcnt;
  Wk.gen_ctr = P->e_selcnt + 1;
  Wk.rmask = nullptr;
  Wk.lscr = P->e_lscr;
  Wk.lss = P->lscr_per_walker;
  Wk.use_tabu = 0;
  Wk.W = 1;
  Wk.tenure = 0;
  Wk.wcap = 1e6f;
  Wk.delta = NAN;
  return Wk;
}

int chap::grid_for(long long work, int threads, int cap) {
  long long g = (work + threads - 1) / threads;
  return (int)std::max<long long>(1, std::min<long long>(g, cap));
}

// Residuals of walker w from scratch (r = A x - b, the cutoff row from a grid-wide c.x), weights
// kept, and the violated count: the state k_walker_finalize_init completes.
chap_status chap::walker_recompute(const chap_problem* P, DevWalkers& Wk, int w, cudaStream_t s) {
  const DevProblem& D = P->dp;
  k_acc_zero<<<1, 1, 0, s>>>(Wk.sc, w, nullptr);
  if (D.n > 0)
    k_cut_dot<<<dim3(grid_for(D.n, 256, 2 * P->sm_count), 1), 256, 0, s>>>(D, Wk.x, Wk.xs, Wk.sc, w, nullptr);
  k_rows_init<<<dim3(P->rows_grid, 1), 256, 0, s>>>(D, Wk, 0, nullptr, w, nullptr);
  k_viol_count<<<dim3(grid_for(D.m_norm, 256, 2 * P->sm_count), 1), 256, 0, s>>>(D, Wk, w);
  if (Wk.xbits && D.n > 0) k_xbits_build<<<dim3(grid_for(D.n, 256, 4 * P->sm_count), 1), 256, 0, s>>>(D, Wk, w);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

// The launches of one eval call; the validation flag (x out of bounds or fractional on an integer
// variable, a negative or NaN weight) is copied to the problem's pinned h_bad, to be read after
// the stream is synchronised.
static chap_status eval_launch(const chap_problem* p, const double* x, const float* w, double cutoff_rhs,
                               double* xhat, double* score, chap_move* best, cudaStream_t s) {
  const DevProblem& D = p->dp;
  DevWalkers Wk = eval_walkers(p);
  CUDA_TRY(cudaMemsetAsync(p->e_bad, 0, sizeof(int), s));
  k_eval_scalars<<<1, 1, 0, s>>>(p->e_sc, cutoff_rhs, p->dp.rint_base);
  if (D.n > 0) k_permute_in<<<dim3(grid_for(D.n, 256, 4 * p->sm_count), 1), 256, 0, s>>>(D, x, D.n, p->e_x, D.n, p->e_bad);
  if (cutoff_rhs < INFINITY && D.n > 0)
    k_cut_dot<<<dim3(grid_for(D.n, 256, 2 * p->sm_count), 1), 256, 0, s>>>(D, p->e_x, D.n, p->e_sc, -1, nullptr);
  k_rows_init<<<dim3(p->rows_grid, 1), 256, 0, s>>>(D, Wk, 2, w, 0, p->e_bad);
  CUDA_TRY(cudaGetLastError());
  if (D.n_fixed > 0 && (xhat || score))
    k_fixed_out<<<grid_for(D.n_fixed, 256, 4 * p->sm_count), 256, 0, s>>>(D, p->e_x, xhat, score);
  TRY(launch_eval(p, Wk, p->eval_grid, p->bin_grid, p->gen_grid, 0, 0, xhat, score, best, s, false, 0));
  CUDA_TRY(cudaMemcpyAsync(p->h_bad, p->e_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

static chap_status eval_check(const chap_problem* p) {
  if (*p->h_bad)
    return fail(CHAP_ERR_INVALID_ARG, "x out of bounds or fractional on an integer variable, or a weight < 0 / NaN "
                                      "(outputs unspecified)");
  return CHAP_OK;
}

extern "C" chap_status chap_eval_best_shift(const chap_problem* p, const double* x, const float* w,
                                            double cutoff_rhs, double* xhat, double* score,
                                            chap_move* best, void* cuda_stream) {
  if (!p || (!x && p->dp.n > 0)) return fail(CHAP_ERR_INVALID_ARG, "NULL problem or x");
  if (std::isnan(cutoff_rhs) || cutoff_rhs == -INFINITY) return fail(CHAP_ERR_INVALID_ARG, "cutoff_rhs must be finite or +INF");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  TRY(eval_launch(p, x, w, cutoff_rhs, xhat, score, best, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return eval_check(p);
}

extern "C" chap_status chap_eval_best_shift_host(chap_problem* p, const double* x, const float* w,
                                                 double cutoff_rhs, double* xhat, double* score,
                                                 chap_move* best, void* cuda_stream) {
  if (!p || (!x && p->dp.n > 0)) return fail(CHAP_ERR_INVALID_ARG, "NULL problem or x");
  if (std::isnan(cutoff_rhs) || cutoff_rhs == -INFINITY) return fail(CHAP_ERR_INVALID_ARG, "cutoff_rhs must be finite or +INF");
  DeviceGuard g(p->device);
  const int n = p->dp.n, mn = p->dp.m_norm;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (!p->h_x) {
    CUDA_TRY(cudaMallocHost(&p->h_x, sizeof(double) * std::max(n, 1)));
    CUDA_TRY(cudaMallocHost(&p->h_w, sizeof(float) * std::max(mn, 1)));
    CUDA_TRY(cudaMallocHost(&p->h_out, sizeof(double) * 2 * std::max(n, 1)));
    CUDA_TRY(cudaMallocHost(&p->h_best, sizeof(chap_move)));
    TRY(p->buf.alloc(&p->d_xu, n));
    TRY(p->buf.alloc(&p->d_wu, mn));
    TRY(p->buf.alloc(&p->d_out, 2 * (size_t)n));
    TRY(p->buf.alloc(&p->d_best, 1));
  }
  // page-locked caller buffers are copied by DMA directly; pageable ones through pinned staging
  auto pinned = [](const void* ptr) {
    cudaPointerAttributes a;
    if (!ptr || cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost;
  };
  const double* hx = x;
  if (!pinned(x)) {
    memcpy(p->h_x, x, sizeof(double) * n);
    hx = p->h_x;
  }
  CUDA_TRY(cudaMemcpyAsync(p->d_xu, hx, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (w) {
    const float* hw = w;
    if (!pinned(w)) {
      memcpy(p->h_w, w, sizeof(float) * mn);
      hw = p->h_w;
    }
    CUDA_TRY(cudaMemcpyAsync(p->d_wu, hw, sizeof(float) * mn, cudaMemcpyHostToDevice, s));
  }
  TRY(eval_launch(p, p->d_xu, w ? p->d_wu : nullptr, cutoff_rhs, xhat ? p->d_out : nullptr,
                  score ? p->d_out + n : nullptr, best ? p->d_best : nullptr, s));
  const bool px = pinned(xhat), ps = pinned(score);
  if (xhat) CUDA_TRY(cudaMemcpyAsync(px ? xhat : p->h_out, p->d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (score)
    CUDA_TRY(cudaMemcpyAsync(ps ? score : p->h_out + n, p->d_out + n, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (best) CUDA_TRY(cudaMemcpyAsync(p->h_best, p->d_best, sizeof(chap_move), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  TRY(eval_check(p));
  if (xhat && !px) memcpy(xhat, p->h_out, sizeof(double) * n);
  if (score && !ps) memcpy(score, p->h_out + n, sizeof(double) * n);
  if (best) *best = *p->h_best;
  return CHAP_OK;
}

// ------------------------------------------------------------------------------------------
// walkers
// ------------------------------------------------------------------------------------------
extern "C" chap_status chap_params_default(chap_params* out) {
  if (!out) return fail(CHAP_ERR_INVALID_ARG, "NULL out");
  out->tenure = 10;
  out->weight_cap = 1e6f;
  out->cutoff_delta = NAN;
  out->exchange_K = 1000;
  out->n_elite = 4;
  out->n_restart = -1;
  out->graph_iters = 16;
  out->binary_kernel = 0;
  out->pdl = 0;
  out->l2_persist = 1;
  out->aspiration = 0;
  out->lazy = 0;
  out->perturb = 0;
  out->perturb_radius = 16;
  out->smooth_prob = 0.0f;
  out->rng_seed = 0;
  return CHAP_OK;
}

static chap_status check_params(const chap_params& q) {
  if (q.tenure < 0) return fail(CHAP_ERR_INVALID_ARG, "tenure < 0");
  if (!(q.weight_cap >= 1.0f && q.weight_cap <= 16777216.0f)) return fail(CHAP_ERR_INVALID_ARG, "weight_cap must be in [1, 2^24]");
  if (!std::isnan(q.cutoff_delta) && !(q.cutoff_delta >= 0.0 && std::isfinite(q.cutoff_delta)))
    return fail(CHAP_ERR_INVALID_ARG, "cutoff_delta must be NaN (auto) or finite >= 0");
  if (q.graph_iters < 0) return fail(CHAP_ERR_INVALID_ARG, "graph_iters < 0");
  if (q.binary_kernel < 0 || q.binary_kernel > 2) return fail(CHAP_ERR_INVALID_ARG, "binary_kernel not in {0, 1, 2}");
  if (q.pdl < 0 || q.pdl > 1) return fail(CHAP_ERR_INVALID_ARG, "pdl not in {0, 1}");
  if (q.l2_persist < 0 || q.l2_persist > 1) return fail(CHAP_ERR_INVALID_ARG, "l2_persist not in {0, 1}");
  if (q.aspiration < 0 || q.aspiration > 1) return fail(CHAP_ERR_INVALID_ARG, "aspiration not in {0, 1}");
  if (q.lazy < 0 || q.lazy > 1) return fail(CHAP_ERR_INVALID_ARG, "lazy not in {0, 1}");
  if (q.perturb < 0 || q.perturb > 1) return fail(CHAP_ERR_INVALID_ARG, "perturb not in {0, 1}");
  if (q.perturb_radius < 1) return fail(CHAP_ERR_INVALID_ARG, "perturb_radius < 1");
  if (!(q.smooth_prob >= 0.0f && q.smooth_prob <= 1.0f)) return fail(CHAP_ERR_INVALID_ARG, "smooth_prob not in [0, 1]");
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_create(const chap_problem* p, int32_t W, const double* x0,
                                           const chap_params* params, void* cuda_stream,
                                           chap_walkers** out) {
  if (!out) return fail(CHAP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!p || W < 1 || (!x0 && p->dp.n > 0)) return fail(CHAP_ERR_INVALID_ARG, "NULL problem/x0 or W < 1");
  chap_params prm;
  if (params) prm = *params; else chap_params_default(&prm);
  TRY(check_params(prm));
  if (prm.lazy && W != 1) return fail(CHAP_ERR_INVALID_ARG, "lazy (selective re-evaluation) takes one walker");
  DeviceGuard g(p->device);
  auto S = new chap_walkers();
  std::unique_ptr<chap_walkers> holder(S);
  S->P = p;
  S->W = W;
  S->prm = prm;
  const DevProblem& D = p->dp;
  const size_t n = (size_t)std::max(D.n, 1), mn = (size_t)D.m_norm;
  DevWalkers& Wk = S->wk;
  DeviceBuffers& B = S->buf;
  TRY(B.alloc(&Wk.x, n * W));
  // row-state groups (DevWalkers): walker-minor groups of up to 32 walkers when W > 1
  int rg = 1;
  if (W > 1) while (rg < 32 && rg < W) rg <<= 1;
  Wk.rg = rg;
  Wk.n_groups = (W + rg - 1) / rg;
  TRY(B.alloc(&Wk.rs, (mn + 1) * (size_t)rg * Wk.n_groups));
  Wk.xbits = nullptr;
  if (rg > 1) TRY(B.alloc(&Wk.xbits, n * (size_t)Wk.n_groups));
  TRY(B.alloc(&Wk.tabu, n * W));
  TRY(B.alloc(&Wk.best_x, n * W));
  TRY(B.alloc(&Wk.sc, W));
  S->eval_grid = std::max(1, std::min(p->eval_grid, (p->eval_occ * p->sm_count + W - 1) / W));
  S->bin_grid = p->bin_grid ? std::max(1, std::min(p->bin_grid, (p->bin_occ * p->sm_count + W - 1) / W)) : 0;
  if (rg > 1 && p->bin_grid) {   // k_eval_bin_wm: one grid row per group
    const int items = p->dp.n_btiles + p->dp.n_bchunks, warps = kBinWmThreads / 32;
    S->bin_grid = std::max(1, std::min((items + warps - 1) / warps,
                                       (bin_wm_occupancy(rg) * p->sm_count + Wk.n_groups - 1) / Wk.n_groups));
  }
  S->gen_grid = p->gen_grid ? std::max(1, std::min(p->gen_grid, (p->gen_occ * p->sm_count + W - 1) / W)) : 0;
  // one walker with integral weights whose column sums fit int32: packed binary columns row-wise
  S->binrow_grid = 0;
  const bool want_row = prm.binary_kernel == 2 || (prm.binary_kernel == 0 && p->binrow_auto);
  if (W == 1 && !prm.lazy && want_row && p->binrow_grid > 0 && prm.weight_cap == std::floor(prm.weight_cap) &&
      2.0 * (double)prm.weight_cap * (double)std::max(1, p->binrow_maxdeg) < 2147483647.0) {
    S->binrow_grid = p->binrow_grid;
    // the long binary chunks ride in k_eval_gen when it runs (with_lbin), else in k_eval_bin
    S->bin_grid = (S->gen_grid > 0) ? 0 : p->bin_chunk_grid;
    TRY(B.alloc(&Wk.xbits, (size_t)p->dp.n_rblocks * kRowWpb));   // block-ordered bitset
  }
  // programmatic dependent launch between the iteration's kernels (chap_params.pdl): measured
  // slower on config G (0.1344 vs 0.1273 ms; early-scheduled k_eval_gen blocks disturb its
  // persistent grid), so off by default
  S->pdl = prm.pdl != 0;
  // a10: with walker groups the long bounded-integer chunks go to k_eval_gen_wm (A read once per group);
  // each of its warps then needs a lane-private histogram of every such column's domain
  Wk.lbkt_wm = 0;
  Wk.lbkt_wm_words = 0;
  if (rg > 1 && p->dp.n_wtiles > 0 && prm.weight_cap == std::floor(prm.weight_cap) && prm.weight_cap <= 1048576.0f &&
      p->dp.n_gchunks > 0) {
    int words = 0;
    for (int q = 0; q < p->dp.n_long; ++q) {
      const LongCol& L = p->h_lcols[q];
      if (L.kind == CC_LBKT) words = std::max(words, 32 * (L.dom + 1 + (L.dom + 31) / 32));
    }
    if ((size_t)words * 4 * (kGenWmThreads / 32) <= 160 * 1024) Wk.lbkt_wm_words = words;
  }
  S->genwm_grid = 0;   // walker groups: integer general tiles and empty columns per group (k_eval_gen_wm)
  if (rg > 1 && p->dp.n_wtiles > 0) {
    int occ = gen_wm_occupancy(rg, gen_wm_smem_all(std::max(1, p->gen_kmax), Wk.lbkt_wm_words));
    const int occ0 = gen_wm_occupancy(rg, gen_wm_smem_all(std::max(1, p->gen_kmax), 0));
    // the histograms do not fit, or the long bounded-integer columns hold less than an eighth as
    // many entries as the general tiles: the chunks stay per walker (k_eval_gen). Measured per
    // iteration, groups vs per walker: G with 32 walkers (long bounded-integer entries 0.49 of the
    // tiles') 1.70 vs 2.27 ms; X1e6 with 64 (0.02) 0.63 vs 0.35 ms.
    if (Wk.lbkt_wm_words > 0 && (occ == 0 || 8 * p->lbkt_nnz < p->gen_tile_nnz)) {
      Wk.lbkt_wm_words = 0;
      occ = occ0;
    }
    // (the kernel's shared-memory attribute is left at the size the launches use)
    gen_wm_occupancy(rg, gen_wm_smem_all(std::max(1, p->gen_kmax), Wk.lbkt_wm_words));
    if (occ > 0) {
      const int warps = kGenWmThreads / 32;
      S->genwm_grid = std::max(1, std::min((p->dp.n_wtiles + warps - 1) / warps,
                                           (occ * p->sm_count + Wk.n_groups - 1) / Wk.n_groups));
    }
  }
  if (S->genwm_grid > 0 && Wk.lbkt_wm_words > 0) Wk.lbkt_wm = 1;
  else Wk.lbkt_wm_words = 0;
  Wk.ps = S->eval_grid + S->bin_grid + S->gen_grid + S->binrow_grid + S->genwm_grid;
  if (prm.lazy) Wk.ps = std::max(Wk.ps, 4 * p->sm_count);   // k_select_cache's parts
  TRY(B.alloc(&Wk.part, (size_t)Wk.ps * W));
  TRY(B.alloc(&Wk.sel_count, 3 * (size_t)W));   // [W] select counters, then [W][2] k_eval_gen item counters
  Wk.gen_ctr = Wk.sel_count + W;
  Wk.lss = p->lscr_per_walker;
  TRY(B.alloc(&Wk.lscr, Wk.lss * W));
  TRY(B.alloc(&S->d_bad, 1));
  {
    int32_t* rm = nullptr;   // the device exchange's restart slots (portfolio.cuh)
    TRY(B.alloc(&rm, W));
    Wk.rmask = rm;
  }
  Wk.asp = nullptr;
  if (prm.aspiration && prm.tenure > 0) TRY(B.alloc(&Wk.asp, (size_t)prm.tenure * W));   // R18 slots
  Wk.cs = Wk.cv = nullptr;
  Wk.dirty = nullptr;
  Wk.dwords = (int32_t)((n + 31) / 32);
  if (prm.lazy) {   // f2: per-column cache and the two dirty sets (every column dirty at first)
    TRY(B.alloc(&Wk.cs, n));
    TRY(B.alloc(&Wk.cv, n));
    TRY(B.alloc(&Wk.dirty, 2 * ((size_t)Wk.dwords + 1)));
    S->sel_grid = std::max(1, std::min((int)((n + kTileThreads - 1) / kTileThreads), 4 * p->sm_count));
  }
  Wk.xs = n;
  Wk.rss = mn + 1;
  Wk.ts = n;
  Wk.use_tabu = 1;
  Wk.W = W;
  Wk.tenure = prm.tenure;
  Wk.wcap = prm.weight_cap;
  Wk.perturb = prm.perturb;
  Wk.perturb_radius = prm.perturb_radius;
  Wk.rng_seed = prm.rng_seed;
  Wk.smooth_prob = prm.smooth_prob;
  Wk.delta = prm.cutoff_delta;
  CUDA_TRY(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
  if (prm.l2_persist) {   // the gathered row state persists in L2 (window on the stream,
                          // copied onto every kernel node of the captured graphs)
    const size_t rs_bytes = sizeof(RowState) * (mn + 1) * (size_t)rg * Wk.n_groups;
    int max_persist = 0, max_win = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, p->device);
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, p->device);
    if (max_persist > 0 && max_win > 0) {
      const size_t win = std::min(rs_bytes, (size_t)max_win);
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur < std::min(win, (size_t)max_persist))
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(win, (size_t)max_persist));
      cudaAccessPolicyWindow& a = S->l2win;
      a.base_ptr = Wk.rs;
      a.num_bytes = win;
      a.hitRatio = (float)std::min(1.0, (double)max_persist / (double)win);
      a.hitProp = cudaAccessPropertyPersisting;
      a.missProp = cudaAccessPropertyStreaming;
      cudaStreamAttrValue v{};
      v.accessPolicyWindow = a;
      if (cudaStreamSetAttribute(S->stream, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess) S->l2win_on = true;
      cudaGetLastError();
    }
  }
  CUDA_TRY(cudaEventCreateWithFlags(&S->ev_in, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&S->ev_out, cudaEventDisableTiming));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  CUDA_TRY(cudaMemsetAsync(Wk.sc, 0, sizeof(WalkerScalars) * W, s));
  CUDA_TRY(cudaMemsetAsync(const_cast<int32_t*>(Wk.rmask), 0xff, sizeof(int32_t) * W, s));
  CUDA_TRY(cudaMemsetAsync(Wk.lscr, 0, sizeof(double) * Wk.lss * W, s));
  CUDA_TRY(cudaMemsetAsync(Wk.sel_count, 0, sizeof(unsigned) * 3 * W, s));
  CUDA_TRY(cudaMemsetAsync(Wk.best_x, 0, sizeof(double) * n * W, s));
  CUDA_TRY(cudaMemsetAsync(Wk.rs, 0, sizeof(RowState) * (mn + 1) * (size_t)rg * Wk.n_groups, s));
  CUDA_TRY(cudaMemsetAsync(S->d_bad, 0, sizeof(int), s));
  if (Wk.asp) CUDA_TRY(cudaMemsetAsync(Wk.asp, 0xff, sizeof(Cand) * (size_t)prm.tenure * W, s));   // p = -1
  if (Wk.dirty) {
    CUDA_TRY(cudaMemsetAsync(Wk.dirty, 0, sizeof(uint32_t) * 2 * ((size_t)Wk.dwords + 1), s));
    k_dirty_all<<<1, 32, 0, s>>>(Wk, -1);
  }
  if (D.n > 0)
    k_permute_in<<<dim3(grid_for(D.n, 256, 4 * p->sm_count), W), 256, 0, s>>>(D, x0, D.n, Wk.x, Wk.xs, S->d_bad);
  k_acc_zero<<<W, 1, 0, s>>>(Wk.sc, -1, nullptr);
  if (D.n > 0) k_cut_dot<<<dim3(grid_for(D.n, 256, 2 * p->sm_count), W), 256, 0, s>>>(D, Wk.x, Wk.xs, Wk.sc, -1, nullptr);
  k_rows_init<<<dim3(p->rows_grid, W), 256, 0, s>>>(D, Wk, 1, nullptr, -1, nullptr);
  k_viol_count<<<dim3(grid_for(D.m_norm, 256, 2 * p->sm_count), W), 256, 0, s>>>(D, Wk, -1);
  if (Wk.xbits && D.n > 0)
    k_xbits_build<<<dim3(grid_for(D.n, 256, 4 * p->sm_count), Wk.n_groups), 256, 0, s>>>(D, Wk, -1);
  k_tabu_clear<<<dim3(grid_for(D.n, 256, 4 * p->sm_count), W), 256, 0, s>>>(Wk.tabu, Wk.ts, D.n, -1, nullptr);
  k_walker_finalize_init<<<W, 1, 0, s>>>(D, Wk, 0, -1);
  k_flush_incumbent<<<dim3(grid_for(D.n, 256, 4 * p->sm_count), W), 256, 0, s>>>(D, Wk);
  k_flush_done<<<(W + 255) / 256, 256, 0, s>>>(Wk);
  CUDA_TRY(cudaGetLastError());
  int bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, S->d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) return fail(CHAP_ERR_INVALID_ARG, "x0 out of bounds or fractional on an integer variable");
  // apply grid: enough blocks for a bump over m_norm rows (4 rows per thread), capped by the SMs
  S->apply_grid = grid_for((long long)mn, 4 * kApplyThreads, std::max(1, 2 * p->sm_count / std::max(1, std::min(W, 8))));
  *out = holder.release();
  return CHAP_OK;
}

static chap_status launch_iteration(chap_walkers* S, cudaStream_t s) {
  const chap_problem* P = S->P;
  TRY(launch_eval(P, S->wk, S->eval_grid, S->bin_grid, S->gen_grid, S->binrow_grid, S->genwm_grid, nullptr, nullptr,
                  nullptr, s, S->pdl, S->wk.cs ? S->sel_grid : 0));
  TRY(lk(k_apply, dim3(S->apply_grid, S->W), kApplyThreads, 0, s, S->pdl, 1, P->dp, S->wk));
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

// Capture `iters` tabu iterations of the walkers as one instantiated CUDA graph.
// A graph of `iters` tabu iterations followed by whatever `tail` launches (chap_walkers_epoch: the
// device exchange), instantiated into *out.
template <class Tail>
static chap_status capture_graph(chap_walkers* S, cudaStream_t s, int iters, Tail tail, cudaGraphExec_t* out) {
  cudaGraph_t graph;
  CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  chap_status st = CHAP_OK;
  for (int it = 0; it < iters && st == CHAP_OK; ++it) st = launch_iteration(S, s);
  if (st == CHAP_OK) st = tail(s);
  cudaError_t ce = cudaStreamEndCapture(s, &graph);
  if (st != CHAP_OK) return st;
  if (ce != cudaSuccess) return fail(CHAP_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
  if (S->l2win_on) {   // the row state's L2 window on every kernel node
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
    cudaKernelNodeAttrValue v{};
    v.accessPolicyWindow = S->l2win;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel)
        cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v);
    }
    cudaGetLastError();
  }
  ce = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return fail(CHAP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
  return CHAP_OK;
}
static chap_status capture_iterations(chap_walkers* S, cudaStream_t s, int iters, cudaGraphExec_t* out) {
  return capture_graph(S, s, iters, [](cudaStream_t) { return CHAP_OK; }, out);
}

extern "C" chap_status chap_tabu_step(chap_walkers* S, int32_t n_iters, chap_step_record* log,
                                      void* cuda_stream) {
  if (!S || n_iters < 0) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers or n_iters < 0");
  if (n_iters == 0) return CHAP_OK;
  DeviceGuard g(S->P->device);
  cudaStream_t us = (cudaStream_t)cuda_stream;
  cudaStream_t s = S->stream;
  CUDA_TRY(cudaEventRecord(S->ev_in, us));
  CUDA_TRY(cudaStreamWaitEvent(s, S->ev_in, 0));
  k_set_log<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk, log);
  CUDA_TRY(cudaGetLastError());
  const int gi = S->prm.graph_iters;
  int done = 0;
  if (gi > 0) {
    // every iteration runs inside a CUDA graph: graphs of gi iterations, then one
    // graph of the remainder (captured once per distinct remainder length and kept)
    if (n_iters >= gi) {
      if (!S->gexec) {
        TRY(capture_iterations(S, s, gi, &S->gexec));
        S->g_iters = gi;
      }
      while (n_iters - done >= S->g_iters) {
        CUDA_TRY(cudaGraphLaunch(S->gexec, s));
        done += S->g_iters;
      }
    }
    const int rem = n_iters - done;
    if (rem > 0) {
      if (S->gexec_rem && S->g_rem != rem) {
        cudaGraphExecDestroy(S->gexec_rem);
        S->gexec_rem = nullptr;
      }
      if (!S->gexec_rem) {
        TRY(capture_iterations(S, s, rem, &S->gexec_rem));
        S->g_rem = rem;
      }
      CUDA_TRY(cudaGraphLaunch(S->gexec_rem, s));
      done += rem;
    }
  }
  for (; done < n_iters; ++done) TRY(launch_iteration(S, s));
  const DevProblem& D = S->P->dp;
  k_flush_incumbent<<<dim3(grid_for(D.n, 256, 4 * S->P->sm_count), S->W), 256, 0, s>>>(D, S->wk);
  k_flush_done<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk);
  k_set_log<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk, nullptr);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(S->ev_out, s));
  CUDA_TRY(cudaStreamWaitEvent(us, S->ev_out, 0));
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_get(const chap_walkers* S, double* x, double* r, float* w,
                                        int64_t* tabu_until, double* best_x, chap_walker_stats* stats,
                                        void* cuda_stream) {
  if (!S) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers");
  DeviceGuard g(S->P->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const DevProblem& D = S->P->dp;
  const int gx = grid_for(std::max(D.n, D.m_norm), 256, 4 * S->P->sm_count);
  if (x || tabu_until || best_x) k_export_vars<<<dim3(gx, S->W), 256, 0, s>>>(D, S->wk, x, tabu_until, best_x);
  if (r || w) k_export_rows<<<dim3(gx, S->W), 256, 0, s>>>(D, S->wk, r, w);
  if (stats) k_export_stats<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk, stats);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_set_cutoff(chap_walkers* S, double z_best, void* cuda_stream) {
  if (!S || !std::isfinite(z_best)) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers or non-finite z_best");
  DeviceGuard g(S->P->device);
  k_set_cutoff<<<(S->W + 255) / 256, 256, 0, (cudaStream_t)cuda_stream>>>(S->P->dp, S->wk, z_best);
  if (S->wk.dirty) k_dirty_all<<<1, 32, 0, (cudaStream_t)cuda_stream>>>(S->wk, -1);   // f2: the cutoff row moved
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_restart(chap_walkers* S, int32_t walker, const double* x,
                                            void* cuda_stream) {
  if (!S || walker < 0 || walker >= S->W || (!x && S->P->dp.n > 0))
    return fail(CHAP_ERR_INVALID_ARG, "bad walker index or NULL x");
  DeviceGuard g(S->P->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const DevProblem& D = S->P->dp;
  DevWalkers& Wk = S->wk;
  const int gx = grid_for(D.n, 256, 4 * S->P->sm_count);
  // write into walker `walker` only: offset the destinations
  // the point is validated first (in bounds, integral on integer variables): an invalid x leaves the
  // walker untouched
  CUDA_TRY(cudaMemsetAsync(S->d_bad, 0, sizeof(int), s));
  if (D.n > 0) k_check_point<<<dim3(gx, 1), 256, 0, s>>>(D, x, S->d_bad);
  int bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, S->d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (bad) return fail(CHAP_ERR_INVALID_ARG, "restart point out of bounds or fractional on an integer variable");
  if (D.n > 0) k_permute_in<<<dim3(gx, 1), 256, 0, s>>>(D, x, D.n, Wk.x + (size_t)walker * Wk.xs, Wk.xs, nullptr);
  TRY(chap::walker_recompute(S->P, Wk, walker, s));
  k_tabu_clear<<<dim3(gx, 1), 256, 0, s>>>(Wk.tabu, Wk.ts, D.n, walker, nullptr);
  k_walker_finalize_init<<<1, 1, 0, s>>>(D, Wk, 1, walker);
  if (Wk.dirty) k_dirty_all<<<1, 32, 0, s>>>(Wk, -1);   // f2: a new point
  k_flush_incumbent<<<dim3(gx, S->W), 256, 0, s>>>(D, Wk);
  k_flush_done<<<(S->W + 255) / 256, 256, 0, s>>>(Wk);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_profile(chap_walkers* S, int32_t n_iters, double* ms, void* cuda_stream) {
  if (!S || n_iters < 1 || !ms) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers/ms or n_iters < 1");
  DeviceGuard g(S->P->device);
  const chap_problem* P = S->P;
  const DevProblem& D = P->dp;
  cudaStream_t s = S->stream;
  cudaStream_t us = (cudaStream_t)cuda_stream;
  CUDA_TRY(cudaEventRecord(S->ev_in, us));
  CUDA_TRY(cudaStreamWaitEvent(s, S->ev_in, 0));
  k_set_log<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk, nullptr);
  std::vector<cudaEvent_t> ev(10 * (size_t)n_iters);
  for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
  // one CUDA graph of n_iters iterations with event-record nodes between the kernels, so that the
  // intervals measure the kernels as chap_tabu_step's graphs run them (no launch latency inside)
  CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int it = 0; it < n_iters; ++it) {
    cudaEvent_t* e = &ev[10 * (size_t)it];
    for (int q = 0; q < 8; ++q) cudaEventRecordWithFlags(e[q], s, cudaEventRecordExternal);
    if (S->bin_grid > 0) {
      DevProblem Db = D;
      if (S->binrow_grid > 0) Db.n_btiles = 0;
      if (S->wk.rg > 1) TRY(launch_bin_wm(D, S->wk, S->bin_grid, s, false));
      else k_eval_bin<<<dim3(S->bin_grid, S->W), kBinThreads, kBinSmem, s>>>(Db, S->wk, nullptr, nullptr, 0, nullptr);
    }
    if (S->binrow_grid > 0) TRY(launch_binrow(P, S->wk, S->binrow_grid, S->bin_grid + S->gen_grid, s, false));
    cudaEventRecordWithFlags(e[1], s, cudaEventRecordExternal);
    cudaEventRecordWithFlags(e[2], s, cudaEventRecordExternal);
    if (S->gen_grid > 0)
      k_eval_gen<<<dim3(S->gen_grid, S->W), kGenThreads, kGenSmem, s>>>(D, S->wk, nullptr, nullptr, S->bin_grid,
                                                                       S->genwm_grid > 0 ? 1 : 0,
                                                                       (S->binrow_grid > 0 && S->bin_grid == 0) ? 1 : 0,
                                                                       0, nullptr);
    if (S->genwm_grid > 0)
      TRY(launch_gen_wm(P, S->wk, S->genwm_grid, S->bin_grid + S->gen_grid + S->binrow_grid, s, false));
    if (D.n_schunks > 0) {
      k_sort_chunks<<<dim3(D.n_schunks, S->W), kTileThreads, kTileSmem, s>>>(D, S->wk);
      k_sort_rank<<<dim3(D.n_schunks, S->W), kTileThreads, 0, s>>>(D, S->wk);
    }
    cudaEventRecordWithFlags(e[3], s, cudaEventRecordExternal);
    cudaEventRecordWithFlags(e[4], s, cudaEventRecordExternal);
    k_eval<<<dim3(S->eval_grid, S->W), kTileThreads, kTileSmem, s>>>(D, S->wk, nullptr, nullptr, nullptr,
                                                                     S->bin_grid + S->gen_grid + S->binrow_grid +
                                                                         S->genwm_grid, S->wk.rg > 1 ? 1 : 0);
    cudaEventRecordWithFlags(e[5], s, cudaEventRecordExternal);
    cudaEventRecordWithFlags(e[8], s, cudaEventRecordExternal);
    k_apply<<<dim3(S->apply_grid, S->W), kApplyThreads, 0, s>>>(D, S->wk);
    cudaEventRecordWithFlags(e[9], s, cudaEventRecordExternal);
  }
  {
    cudaGraph_t graph;
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    CUDA_TRY(cudaGetLastError());
    if (ce != cudaSuccess) return fail(CHAP_ERR_CUDA, "profile graph capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t gx;
    const cudaError_t ci = cudaGraphInstantiate(&gx, graph, 0);
    cudaGraphDestroy(graph);
    if (ci != cudaSuccess) return fail(CHAP_ERR_CUDA, "profile graph instantiate: %s", cudaGetErrorString(ci));
    CUDA_TRY(cudaGraphLaunch(gx, s));
    cudaGraphExecDestroy(gx);
  }
  k_flush_incumbent<<<dim3(grid_for(D.n, 256, 4 * P->sm_count), S->W), 256, 0, s>>>(D, S->wk);
  k_flush_done<<<(S->W + 255) / 256, 256, 0, s>>>(S->wk);
  CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < 5; ++q) ms[q] = 0.0;
  for (int it = 0; it < n_iters; ++it)
    for (int q = 0; q < 5; ++q) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, ev[10 * (size_t)it + 2 * q], ev[10 * (size_t)it + 2 * q + 1]));
      ms[q] += t;
    }
  for (int q = 0; q < 5; ++q) ms[q] /= n_iters;
  ms[3] = 0.0;                   // [0] k_eval_bin, [1] k_eval_gen, [2] k_eval (+ fused select)
  for (auto& e : ev) cudaEventDestroy(e);
  CUDA_TRY(cudaEventRecord(S->ev_out, s));
  CUDA_TRY(cudaStreamWaitEvent(us, S->ev_out, 0));
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_destroy(chap_walkers* S) {
  if (!S) return CHAP_OK;
  DeviceGuard g(S->P->device);
  delete S;
  return CHAP_OK;
}

#include "portfolio.cuh"
#include "lp.cuh"

extern "C" chap_status chap_walkers_launches_per_iter(const chap_walkers* S, int32_t* out) {
  if (!S || !out) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers or out");
  const DevProblem& D = S->P->dp;
  const bool sel_only = S->W == 1 && S->wk.rg == 1 && D.n_tiles == 0 && D.n_scols == 0 && S->genwm_grid == 0;
  const bool fused = sel_only && (S->gen_grid > 0 || (S->binrow_grid == 0 && S->bin_grid > 0));
  *out = (S->bin_grid > 0) + (S->gen_grid > 0) + (S->binrow_grid > 0) + (S->genwm_grid > 0) + (fused ? 0 : 1) + 1 +
         (D.n_schunks > 0 ? 2 : 0);
  if (S->wk.cs)   // lazy: k_eval only for the sort tiles, then k_select_cache
    *out = (S->bin_grid > 0) + (S->gen_grid > 0) + ((D.n_tiles > 0 || D.n_scols > 0) ? 1 : 0) + 1 + 1 +
           (D.n_schunks > 0 ? 2 : 0);
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_timing(chap_walkers* S, int32_t mode, uint64_t* out, void* cuda_stream) {
  if (!S || mode < -1 || mode > 1) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers or mode not in {-1, 0, 1}");
  DeviceGuard g(S->P->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (out) {
    for (int q = 0; q < 6; ++q) out[q] = 0;
    if (S->kt_buf) {
      unsigned long long h[kKtWords];
      CUDA_TRY(cudaMemcpyAsync(h, S->kt_buf, sizeof(h), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      for (int q = 0; q < 6; ++q) out[q] = h[8 + q];
    }
  }
  if (mode == -1) return CHAP_OK;
  if (mode == 1) {
    if (!S->kt_buf) TRY(S->buf.alloc(&S->kt_buf, kKtWords));
    unsigned long long h[kKtWords];
    for (int q = 0; q < 8; ++q) h[q] = (q & 1) ? 0ull : ~0ull;
    for (int q = 8; q < kKtWords; ++q) h[q] = 0ull;
    CUDA_TRY(cudaMemcpyAsync(S->kt_buf, h, sizeof(h), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  unsigned long long* want = mode == 1 ? S->kt_buf : nullptr;
  if (S->wk.kt != want) {   // the captured graph holds the kernel arguments: capture again
    S->wk.kt = want;
    if (S->gexec) {
      cudaGraphExecDestroy(S->gexec);
      S->gexec = nullptr;
    }
    if (S->gexec_rem) {
      cudaGraphExecDestroy(S->gexec_rem);
      S->gexec_rem = nullptr;
    }
    if (S->gexec_ep) {   // (the epoch graph: chap_walkers_epoch)
      cudaGraphExecDestroy(S->gexec_ep);
      S->gexec_ep = nullptr;
    }
  }
  return CHAP_OK;
}

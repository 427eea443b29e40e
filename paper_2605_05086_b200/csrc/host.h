// host.h — host-side internals of libchap shared by chap.cu and portfolio.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "chap.h"
#include "common.cuh"

namespace chap {

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
chap_status fail(chap_status s, const char* fmt, ...);

#define CUDA_TRY(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? CHAP_ERR_OOM : CHAP_ERR_CUDA,        \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);  \
  } while (0)

#define TRY(call)                      \
  do {                                 \
    chap_status s_ = (call);           \
    if (s_ != CHAP_OK) return s_;      \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------------------------------
// problem
// ------------------------------------------------------------------------------------------
struct DeviceBuffers {
  std::vector<void*> ptrs;
  ~DeviceBuffers() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  chap_status alloc(T** out, size_t count) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(CHAP_ERR_OOM, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
    ptrs.push_back(p);
    *out = static_cast<T*>(p);
    bytes_total += bytes;
    return CHAP_OK;
  }
  template <class T>
  chap_status upload(T** out, const std::vector<T>& h) {
    TRY(alloc(out, h.size()));
    if (!h.empty()) CUDA_TRY(cudaMemcpy(*out, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return CHAP_OK;
  }
  size_t bytes_total = 0;
};

}  // namespace chap

using namespace chap;

// The opaque handles of chap.h (global scope).
struct chap_problem {
  using DeviceBuffers = chap::DeviceBuffers;
  int device = 0;
  int sm_count = 148;
  chap_problem_info info{};
  std::vector<int32_t> orig_row;
  std::vector<int8_t> side;
  DeviceBuffers buf;
  DevProblem dp{};
  int eval_occ = 1;            // resident k_eval blocks per SM
  int eval_grid = 1;           // k_eval blocks for one walker
  int bin_occ = 1;             // resident k_eval_bin blocks per SM
  int bin_grid = 0;            // k_eval_bin blocks for one walker (0: no binary tiles)
  int gen_occ = 1;
  int gen_grid = 0;            // k_eval_gen blocks for one walker
  int binrow_grid = 0;         // k_eval_binrow CTAs (clusters x kRowCluster; 0: no row-wise blocks)
  bool binrow_auto = false;    // the size rule chooses the row-wise binary kernel (chap_params.binary_kernel 0)
  int gen_kmax = 0;            // longest packed general column (entries incl. padding)
  int64_t gen_tile_nnz = 0;     // entries of the packed general tiles
  int64_t lbkt_nnz = 0;         // entries of the long bounded-integer columns
  int binrow_maxdeg = 0;       // longest packed binary column (incl. its cutoff entry)
  int binrow_cluster = 0;      // CTAs per cluster of k_eval_binrow
  int binrow_pb0 = 0, binrow_nbin = 0;   // the packed binary columns [pb0, pb0 + nbin)
  int bin_chunk_grid = 0;      // k_eval_bin blocks for the long binary chunks alone
  int64_t binrow_entries = 0;  // stored entries (incl. slice padding)
  int rows_grid = 1;
  size_t lscr_per_walker = 1;   // doubles
  std::vector<LongCol> h_lcols;  // the long columns (host copy)
  // eval workspace (one virtual walker)
  double* e_x = nullptr;
  RowState* e_rs = nullptr;
  int32_t* e_tabu = nullptr;
  double* e_bx = nullptr;
  WalkerScalars* e_sc = nullptr;
  Cand* e_part = nullptr;
  unsigned* e_selcnt = nullptr;
  int* e_bad = nullptr;         // eval-call validation flag (device) and its pinned host copy
  int* h_bad = nullptr;
  double* e_lscr = nullptr;
  // host-buffer variant staging (lazy)
  double* h_x = nullptr;
  float* h_w = nullptr;
  double* h_out = nullptr;
  chap_move* h_best = nullptr;
  double* d_xu = nullptr;
  float* d_wu = nullptr;
  double* d_out = nullptr;
  chap_move* d_best = nullptr;
  ~chap_problem() {
    if (h_x) cudaFreeHost(h_x);
    if (h_w) cudaFreeHost(h_w);
    if (h_out) cudaFreeHost(h_out);
    if (h_best) cudaFreeHost(h_best);
    if (h_bad) cudaFreeHost(h_bad);
  }
};

struct chap_exchange_state;
void chap_exchange_state_free(chap_exchange_state* x);   // portfolio.cuh

struct chap_walkers {
  using DeviceBuffers = chap::DeviceBuffers;
  const chap_problem* P = nullptr;
  int W = 0;
  chap_params prm{};
  DeviceBuffers buf;
  DevWalkers wk{};
  int* d_bad = nullptr;
  unsigned long long* kt_buf = nullptr;   // chap_walkers_timing accumulators (kKtWords)
  chap_exchange_state* xs = nullptr;   // portfolio exchange buffers and state (portfolio.cuh)
  cudaStream_t stream = nullptr;       // internal stream (graph capture / launch)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t gexec = nullptr;      // graph of g_iters iterations
  int g_iters = 0;
  cudaGraphExec_t gexec_rem = nullptr;  // graph of g_rem iterations (the remainder of a call)
  int g_rem = 0;
  cudaGraphExec_t gexec_ep = nullptr;   // graph of one epoch: ep_iters iterations + the device exchange
  int ep_iters = 0;
  const void* ep_comm = nullptr;        // (the communicator the epoch graph was captured with)
  int apply_grid = 1;
  int eval_grid = 1;           // k_eval blocks per walker
  int bin_grid = 0;            // k_eval_bin blocks per walker
  int gen_grid = 0;            // k_eval_gen blocks per walker
  int binrow_grid = 0;         // k_eval_binrow CTAs (one walker, row-wise binary columns), 0 = off
  int genwm_grid = 0;          // k_eval_gen_wm blocks per walker group (walker groups), 0 = off
  int sel_grid = 0;            // k_select_cache blocks (chap_params.lazy)
  bool pdl = false;            // tabu iterations launched with programmatic dependent launch (CHAP_PDL=1)
  size_t genwm_smem = 0;
  cudaAccessPolicyWindow l2win{};      // chap_params.l2_persist: the row state's L2 window
  bool l2win_on = false;
  ~chap_walkers() {
    if (xs) chap_exchange_state_free(xs);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (gexec_rem) cudaGraphExecDestroy(gexec_rem);
    if (gexec_ep) cudaGraphExecDestroy(gexec_ep);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (stream) cudaStreamDestroy(stream);
  }
};


namespace chap {
// shared launch helpers (chap.cu)
chap_status launch_eval(const chap_problem* P, const DevWalkers& Wk, int grid, int bgrid, int ggrid,
                        int rgrid, int wgrid, double* oxhat, double* oscore, chap_move* best, cudaStream_t s,
                        bool pdl, int sel_grid);
int grid_for(long long work, int threads, int cap);
chap_status walker_recompute(const chap_problem* P, DevWalkers& Wk, int w, cudaStream_t s);

}  // namespace chap

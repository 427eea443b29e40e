// portfolio.cuh — (included by chap.cu: one translation unit) the multi-GPU walker portfolio: one process per GPU,
// W_local independent walkers per GPU, and every K iterations a deterministic
// exchange over NCCL: an allgather of per-walker summaries and of each rank's elite points, the
// global cutoff and restarts of the most violated walkers from the global elite.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <mutex>

#include "host.h"
#include "tabu.cuh"

using namespace chap;

// NCCL is resolved at run time: the process's already-loaded libnccl.so.2 (the one PyTorch ships)
// is reused, so libchap never pins a second NCCL build into a process that also runs torch.
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GetErrorString;
  });
  return api;
}
}  // namespace

struct chap_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

#define NCCL_TRY(call)                                                                       \
  do {                                                                                       \
    if (!nccl().ok) return fail(CHAP_ERR_NCCL, "libnccl.so.2 could not be loaded");           \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return fail(CHAP_ERR_NCCL, "%s: %s (%s:%d)", #call, nccl().GetErrorString(r_), __FILE__, \
                  __LINE__);                                                                 \
  } while (0)

extern "C" chap_status chap_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(CHAP_ERR_INVALID_ARG, "NULL id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  NCCL_TRY(nccl().GetUniqueId(&u));
  memcpy(id, &u, 128);
  return CHAP_OK;
}

extern "C" chap_status chap_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device,
                                        chap_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(CHAP_ERR_INVALID_ARG, "bad comm arguments");
  *out = nullptr;
  DeviceGuard g(device);
  if (!g.ok) return fail(CHAP_ERR_CUDA, "cannot select CUDA device %d", device);
  auto C = new chap_comm();
  std::unique_ptr<chap_comm> holder(C);
  ncclUniqueId u;
  memcpy(&u, id, 128);
  NCCL_TRY(nccl().CommInitRank(&C->comm, nranks, u, rank));
  C->nranks = nranks;
  C->rank = rank;
  C->device = device;
  *out = holder.release();
  return CHAP_OK;
}

extern "C" chap_status chap_comm_destroy(chap_comm* comm) {
  if (!comm) return CHAP_OK;
  DeviceGuard g(comm->device);
  if (comm->comm && nccl().ok) nccl().CommDestroy(comm->comm);
  delete comm;
  return CHAP_OK;
}

// ------------------------------------------------------------------------------------------
// the exchange rule (host)
// ------------------------------------------------------------------------------------------
namespace {
struct Key {
  double a, b;
  int64_t c;
  int32_t gid;
  bool operator<(const Key& o) const {
    if (a != o.a) return a < o.a;
    if (b != o.b) return b < o.b;
    if (c != o.c) return c < o.c;
    return gid < o.gid;
  }
};
Key feas_key(const chap_walker_summary& s) { return Key{s.best_obj, 0.0, 0, s.gid}; }
Key infeas_key(const chap_walker_summary& s) { return Key{(double)s.violated, s.sumviol, 0, s.gid}; }
}  // namespace

extern "C" chap_status chap_exchange_plan(int32_t W_total, int32_t W_local, const chap_walker_summary* s,
                                          int32_t n_elite, int32_t n_restart, double* z_best,
                                          int32_t* best_gid, int32_t* n_elite_out, int32_t* elite_gid,
                                          int8_t* elite_kind, int32_t* elite_slot, int32_t* n_restart_out,
                                          int32_t* restart_gid, int32_t* restart_src) {
  if (W_total < 1 || W_local < 1 || W_total % W_local || !s || n_elite < 0 || n_restart < 0 || !z_best ||
      !best_gid || !n_elite_out || !n_restart_out || (n_elite && (!elite_gid || !elite_kind || !elite_slot)) ||
      (n_restart && (!restart_gid || !restart_src)))
    return fail(CHAP_ERR_INVALID_ARG, "bad exchange-plan arguments");
  for (int32_t g = 0; g < W_total; ++g)
    if (s[g].gid != g) return fail(CHAP_ERR_INVALID_ARG, "summaries must be indexed by gid");
  // global feasible / infeasible elites
  std::vector<Key> F, I;
  for (int32_t g = 0; g < W_total; ++g) {
    if (s[g].flags & 1) F.push_back(feas_key(s[g]));
    I.push_back(infeas_key(s[g]));
  }
  std::sort(F.begin(), F.end());
  std::sort(I.begin(), I.end());
  const int nf = std::min<int>((int)F.size(), n_elite), ni = std::min<int>((int)I.size(), n_elite);
  *z_best = F.empty() ? INFINITY : F[0].a;
  *best_gid = F.empty() ? -1 : F[0].gid;
  // slot of a walker's point in the gathered buffer: its rank's local top-n_elite of the kind
  auto slot_of = [&](int32_t g, int kind) -> int32_t {
    const int32_t r = g / W_local;
    std::vector<Key> loc;
    for (int32_t q = r * W_local; q < (r + 1) * W_local; ++q) {
      if (kind == 0 && !(s[q].flags & 1)) continue;
      loc.push_back(kind == 0 ? feas_key(s[q]) : infeas_key(s[q]));
    }
    std::sort(loc.begin(), loc.end());
    for (int32_t q = 0; q < (int32_t)loc.size() && q < n_elite; ++q)
      if (loc[q].gid == g) return r * 2 * n_elite + kind * n_elite + q;
    return -1;   // unreachable: a global top-n_elite member is in its rank's local top-n_elite
  };
  int32_t ne = 0;
  for (int q = 0; q < nf; ++q, ++ne) {
    elite_gid[ne] = F[q].gid;
    elite_kind[ne] = 0;
    elite_slot[ne] = slot_of(F[q].gid, 0);
  }
  for (int q = 0; q < ni; ++q, ++ne) {
    elite_gid[ne] = I[q].gid;
    elite_kind[ne] = 1;
    elite_slot[ne] = slot_of(I[q].gid, 1);
  }
  *n_elite_out = ne;
  // restarts: highest (violated, gid) first
  std::vector<Key> R;
  for (int32_t g = 0; g < W_total; ++g) R.push_back(Key{-(double)s[g].violated, 0.0, -(int64_t)g, g});
  std::sort(R.begin(), R.end());
  const int nr = ne > 0 ? std::min<int>(n_restart, W_total) : 0;
  for (int q = 0; q < nr; ++q) {
    restart_gid[q] = R[q].gid;
    restart_src[q] = q % ne;
  }
  *n_restart_out = nr;
  return CHAP_OK;
}

// ------------------------------------------------------------------------------------------
// the exchange on the device (no host round trip: capturable into the epoch graph)
// ------------------------------------------------------------------------------------------
namespace chap {
// The plan of chap_exchange_plan computed by one block from the gathered summaries, by rank
// counting (O(W_total^2) comparisons, W_total <= a few thousand): the rank of walker g among the
// feasible walkers by (best_obj, gid), among all by (violated, sumviol, gid), the same within its
// rank's own walkers, and its restart rank by (violated, gid) descending. Outputs (device):
//   z[0]: the best incumbent objective (+INF: none); ip[0]: its gid (-1), ip[1]: |E|, ip[2]: restarts;
//   elite_gid / elite_slot [2 E] (feasible elite first); local_rank [2][W_local]: this rank's walkers'
//   positions among its own top-E of each kind (-1: not sent); restart_gid / restart_src [W_total];
//   rmask [W_local]: the gathered-buffer slot each local walker restarts from (-1: none).
__global__ void __launch_bounds__(1024) k_exchange_plan(const chap_walker_summary* __restrict__ s, int W, int W_local,
                                                        int rank, int E, int n_restart, double* z, int32_t* ip,
                                                        int32_t* elite_gid, int32_t* elite_slot, int32_t* local_rank,
                                                        int32_t* restart_gid, int32_t* restart_src, int32_t* rmask) {
  __shared__ int s_nfeas;
  if (threadIdx.x == 0) s_nfeas = 0;
  __syncthreads();
  for (int g = threadIdx.x; g < W; g += blockDim.x)
    if (s[g].flags & 1) atomicAdd(&s_nfeas, 1);
  if (threadIdx.x == 0) { *z = INFINITY; ip[0] = -1; }
  __syncthreads();
  const int nf = min(s_nfeas, E), ni = min(W, E), ne = nf + ni;
  const int nr = ne > 0 ? min(n_restart, W) : 0;
  auto feas_less = [&](int h, int g) {   // (best_obj, gid)
    return s[h].best_obj < s[g].best_obj || (s[h].best_obj == s[g].best_obj && h < g);
  };
  auto inf_less = [&](int h, int g) {    // (violated, sumviol, gid)
    if (s[h].violated != s[g].violated) return s[h].violated < s[g].violated;
    if (s[h].sumviol != s[g].sumviol) return s[h].sumviol < s[g].sumviol;
    return h < g;
  };
  for (int g = threadIdx.x; g < W; g += blockDim.x) {
    const bool fe = s[g].flags & 1;
    const int r = g / W_local, lo = r * W_local, hi = lo + W_local;
    int fr = 0, lfr = 0, ir = 0, lir = 0, rr = 0;
    for (int h = 0; h < W; ++h) {
      const bool loc = h >= lo && h < hi;
      if (fe && (s[h].flags & 1) && feas_less(h, g)) { ++fr; lfr += loc; }
      if (inf_less(h, g)) { ++ir; lir += loc; }
      if (s[h].violated > s[g].violated || (s[h].violated == s[g].violated && h > g)) ++rr;
    }
    if (fe && fr == 0) { *z = s[g].best_obj; ip[0] = g; }
    if (fe && fr < nf) { elite_gid[fr] = g; elite_slot[fr] = r * 2 * E + lfr; }
    if (ir < ni) { elite_gid[nf + ir] = g; elite_slot[nf + ir] = r * 2 * E + E + lir; }
    if (r == rank) {
      local_rank[g - lo] = (fe && lfr < E) ? lfr : -1;
      local_rank[W_local + g - lo] = lir < E ? lir : -1;
      rmask[g - lo] = -1;
    }
    if (rr < nr) { restart_gid[rr] = g; restart_src[rr] = rr % ne; }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nr; q += blockDim.x) {
    const int g = restart_gid[q];
    if (g / W_local == rank) rmask[g % W_local] = elite_slot[restart_src[q]];
  }
  if (threadIdx.x == 0) { ip[1] = ne; ip[2] = nr; }
}

// Pack the points this rank sends: walker w's best point (kind 0) or current point (kind 1) into
// slot kind E + local_rank[kind][w] of the send buffer; blockIdx = (part, w, kind).
__global__ void k_pack_tops(DevProblem P, DevWalkers Wk, const int32_t* __restrict__ local_rank, int W_local, int E,
                            unsigned char* send) {
  const int w = blockIdx.y, kind = blockIdx.z;
  const int q = local_rank[kind * W_local + w];
  if (q < 0) return;
  pack_point(P, (kind == 0 ? Wk.best_x : Wk.x) + (size_t)w * Wk.xs, send + (size_t)(kind * E + q) * P.pk_bytes);
}

// The restarting walkers' new points from the gathered buffer (rmask: slot); blockIdx = (part, w).
__global__ void k_unpack_restarts(DevProblem P, DevWalkers Wk, const unsigned char* __restrict__ recv) {
  const int w = blockIdx.y;
  const int slot = Wk.rmask[w];
  if (slot < 0) return;
  unpack_point(P, recv + (size_t)slot * P.pk_bytes, Wk.x + (size_t)w * Wk.xs);
}
}  // namespace chap

// ------------------------------------------------------------------------------------------
// chap_run_walkers
// ------------------------------------------------------------------------------------------

// Restart walker w from an internal-order device point: r from scratch, weights kept, tabu
// cleared, then the R15 incumbent check (mode 1 keeps k and the counters).
static chap_status restart_internal(chap_walkers* S, int w, const double* x_int, cudaStream_t s) {
  const chap_problem* P = S->P;
  const DevProblem& D = P->dp;
  DevWalkers& Wk = S->wk;
  CUDA_TRY(cudaMemcpyAsync(Wk.x + (size_t)w * Wk.xs, x_int, sizeof(double) * D.n, cudaMemcpyDeviceToDevice, s));
  TRY(chap::walker_recompute(P, Wk, w, s));
  k_tabu_clear<<<dim3(grid_for(D.n, 256, 4 * P->sm_count), 1), 256, 0, s>>>(Wk.tabu, Wk.ts, D.n, w, nullptr);
  k_walker_finalize_init<<<1, 1, 0, s>>>(D, Wk, 1, w);
  if (Wk.dirty) k_dirty_all<<<1, 32, 0, s>>>(Wk, -1);   // f2: a new point
  k_flush_incumbent<<<dim3(grid_for(D.n, 256, 4 * P->sm_count), S->W), 256, 0, s>>>(D, Wk);
  k_flush_done<<<(S->W + 255) / 256, 256, 0, s>>>(Wk);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

// The exchange state of a walkers object (buffers sized for one communicator size).
struct chap_exchange_state {
  int nranks = 0;
  DeviceBuffers buf;
  chap_walker_summary *d_sum_local = nullptr, *d_sum_all = nullptr;
  unsigned char *d_send = nullptr, *d_recv = nullptr;   // packed elite points (DevProblem::pk_bytes each)
  double* d_x = nullptr;                                // one unpacked point (internal order)
  std::vector<chap_walker_summary> h_all;
  std::vector<int32_t> e_gid, e_slot, r_gid, r_src;
  std::vector<int8_t> e_kind;
  double z = INFINITY;   // best incumbent objective seen by any exchange (persists)
  int32_t zg = -1;       // its global walker id
  // the device exchange's plan (k_exchange_plan)
  double* d_z = nullptr;                                // [1]
  int32_t *d_ip = nullptr, *d_egid = nullptr, *d_eslot = nullptr, *d_lrank = nullptr, *d_rgid = nullptr,
          *d_rsrc = nullptr;
};

void chap_exchange_state_free(chap_exchange_state* x) { delete x; }

// The exchange buffers of a walkers object for a communicator size ((re)allocated when it changes;
// z and zg persist). Called before any capture of the device exchange.
static chap_status exchange_prepare(chap_walkers* S, chap_comm* comm) {
  const chap_problem* p = S->P;
  const int nranks = comm ? comm->nranks : 1;
  const int W_local = S->W, W_total = nranks * W_local;
  const int E = S->prm.n_elite;
  const int n = p->dp.n;
  if (!S->xs) S->xs = new chap_exchange_state();
  chap_exchange_state& X = *S->xs;
  if (X.nranks == nranks) return CHAP_OK;
  {
    X.buf = DeviceBuffers();
    X.nranks = nranks;
    TRY(X.buf.alloc(&X.d_sum_local, W_local));
    TRY(X.buf.alloc(&X.d_sum_all, W_total));
    const size_t pb = (size_t)p->dp.pk_bytes;
    TRY(X.buf.alloc(&X.d_send, (size_t)2 * std::max(E, 1) * pb));
    TRY(X.buf.alloc(&X.d_recv, (size_t)nranks * 2 * std::max(E, 1) * pb));
    TRY(X.buf.alloc(&X.d_x, (size_t)std::max(n, 1)));
    X.h_all.resize(W_total);
    X.e_gid.resize(2 * E + 1);
    X.e_slot.resize(2 * E + 1);
    X.e_kind.resize(2 * E + 1);
    X.r_gid.resize(W_total + 1);
    X.r_src.resize(W_total + 1);
    TRY(X.buf.alloc(&X.d_z, 1));
    TRY(X.buf.alloc(&X.d_ip, 4));
    TRY(X.buf.alloc(&X.d_egid, 2 * (size_t)std::max(E, 1)));
    TRY(X.buf.alloc(&X.d_eslot, 2 * (size_t)std::max(E, 1)));
    TRY(X.buf.alloc(&X.d_lrank, 2 * (size_t)W_local));
    TRY(X.buf.alloc(&X.d_rgid, (size_t)W_total));
    TRY(X.buf.alloc(&X.d_rsrc, (size_t)W_total));
  }
  return CHAP_OK;
}

// One portfolio exchange: summaries -> allgather -> plan -> elite points -> allgather ->
// cutoff -> restarts. want_stop marks this rank's summaries; *stop = any rank marked. With
// need_points = false and *stop set, the point exchange is skipped.
static chap_status exchange_internal(chap_walkers* S, chap_comm* comm, bool want_stop, bool need_points,
                                     bool* stop, cudaStream_t s) {
  const chap_problem* p = S->P;
  const int nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  const int W_local = S->W, W_total = nranks * W_local;
  const chap_params& prm = S->prm;
  const int n_restart = prm.n_restart < 0 ? W_total / 8 : prm.n_restart;
  const int E = prm.n_elite;
  const int n = p->dp.n;
  TRY(exchange_prepare(S, comm));
  chap_exchange_state& X = *S->xs;
  const DevWalkers& Wk = S->wk;
  // 1. summaries -> allgather
  k_summaries<<<W_local, 256, 0, s>>>(p->dp, Wk, X.d_sum_local, rank * W_local, want_stop ? 1 : 0);
  CUDA_TRY(cudaGetLastError());
  if (comm) {
    NCCL_TRY(nccl().AllGather(X.d_sum_local, X.d_sum_all, sizeof(chap_walker_summary) * W_local, ncclUint8, comm->comm, s));
  } else {
    CUDA_TRY(cudaMemcpyAsync(X.d_sum_all, X.d_sum_local, sizeof(chap_walker_summary) * W_local, cudaMemcpyDeviceToDevice, s));
  }
  CUDA_TRY(cudaMemcpyAsync(X.h_all.data(), X.d_sum_all, sizeof(chap_walker_summary) * W_total, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  bool st = false;
  for (const auto& x : X.h_all) st = st || (x.flags & 2);
  *stop = st;
  // 2. the plan (identical on every rank)
  int32_t ne = 0, nr = 0;
  TRY(chap_exchange_plan(W_total, W_local, X.h_all.data(), E, n_restart, &X.z, &X.zg, &ne, X.e_gid.data(),
                         X.e_kind.data(), X.e_slot.data(), &nr, X.r_gid.data(), X.r_src.data()));
  if (st && !need_points) return CHAP_OK;
  // 3. local elite points into the send buffer, allgather (internal variable order: every rank
  //    holds the same problem, hence the same permutation)
  if (E > 0) {
    for (int kind = 0; kind < 2; ++kind) {
      std::vector<std::pair<Key, int>> loc;
      for (int w = 0; w < W_local; ++w) {
        const auto& x = X.h_all[rank * W_local + w];
        if (kind == 0 && !(x.flags & 1)) continue;
        loc.push_back({kind == 0 ? feas_key(x) : infeas_key(x), w});
      }
      std::sort(loc.begin(), loc.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (int q = 0; q < (int)loc.size() && q < E; ++q) {
        const int w = loc[q].second;
        const double* src = (kind == 0 ? Wk.best_x : Wk.x) + (size_t)w * Wk.xs;
        k_pack_point<<<grid_for(n, 256, 2 * p->sm_count), 256, 0, s>>>(p->dp, src,
                                                                        X.d_send + (size_t)(kind * E + q) * p->dp.pk_bytes);
      }
    }
    CUDA_TRY(cudaGetLastError());
    const size_t bytes = (size_t)2 * E * p->dp.pk_bytes;
    if (comm) {
      NCCL_TRY(nccl().AllGather(X.d_send, X.d_recv, bytes, ncclUint8, comm->comm, s));
    } else {
      CUDA_TRY(cudaMemcpyAsync(X.d_recv, X.d_send, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (st) return CHAP_OK;
  // 4. global cutoff, restarts of local walkers
  if (X.z < INFINITY) TRY(chap_walkers_set_cutoff(S, X.z, s));
  for (int q = 0; q < nr; ++q) {
    const int gid = X.r_gid[q];
    if (gid / W_local != rank) continue;
    k_unpack_point<<<grid_for(n, 256, 2 * p->sm_count), 256, 0, s>>>(
        p->dp, X.d_recv + (size_t)X.e_slot[X.r_src[q]] * p->dp.pk_bytes, X.d_x);
    TRY(restart_internal(S, gid % W_local, X.d_x, s));
  }
  return CHAP_OK;
}

// The same exchange (without the stop vote) entirely on the device: summaries, their allgather,
// k_exchange_plan, the local elite packed and all-gathered, the cutoff from the plan's z, and the
// planned restarts as one batch (the restart kernels over the walkers rmask marks). Identical in
// effect to exchange_internal; no host synchronisation, so it can be captured into a graph.
static chap_status exchange_device(chap_walkers* S, chap_comm* comm, cudaStream_t s) {
  const chap_problem* p = S->P;
  const DevProblem& D = p->dp;
  const int nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  const int W_local = S->W, W_total = nranks * W_local;
  const chap_params& prm = S->prm;
  const int n_restart = prm.n_restart < 0 ? W_total / 8 : prm.n_restart;
  const int E = prm.n_elite;
  chap_exchange_state& X = *S->xs;
  const DevWalkers& Wk = S->wk;
  k_summaries<<<W_local, 256, 0, s>>>(D, Wk, X.d_sum_local, rank * W_local, 0);
  CUDA_TRY(cudaGetLastError());
  if (comm) {
    NCCL_TRY(nccl().AllGather(X.d_sum_local, X.d_sum_all, sizeof(chap_walker_summary) * W_local, ncclUint8, comm->comm, s));
  } else {
    CUDA_TRY(cudaMemcpyAsync(X.d_sum_all, X.d_sum_local, sizeof(chap_walker_summary) * W_local, cudaMemcpyDeviceToDevice, s));
  }
  k_exchange_plan<<<1, 1024, 0, s>>>(X.d_sum_all, W_total, W_local, rank, E, n_restart, X.d_z, X.d_ip, X.d_egid,
                                     X.d_eslot, X.d_lrank, X.d_rgid, X.d_rsrc, const_cast<int32_t*>(Wk.rmask));
  CUDA_TRY(cudaGetLastError());
  const int gx = grid_for(D.n, 256, 2 * p->sm_count);
  if (E > 0) {
    k_pack_tops<<<dim3(gx, W_local, 2), 256, 0, s>>>(D, Wk, X.d_lrank, W_local, E, X.d_send);
    CUDA_TRY(cudaGetLastError());
    const size_t bytes = (size_t)2 * E * D.pk_bytes;
    if (comm) {
      NCCL_TRY(nccl().AllGather(X.d_send, X.d_recv, bytes, ncclUint8, comm->comm, s));
    } else {
      CUDA_TRY(cudaMemcpyAsync(X.d_recv, X.d_send, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  k_set_cutoff_from<<<(W_local + 255) / 256, 256, 0, s>>>(D, Wk, X.d_z);
  if (Wk.dirty) k_dirty_all<<<1, 32, 0, s>>>(Wk, -1);   // f2: the cutoff row moved
  if (E > 0) {   // the restarts (none without an elite): rmask marks the walkers and their slots
    const int gx4 = grid_for(D.n, 256, 4 * p->sm_count);
    k_unpack_restarts<<<dim3(gx, W_local), 256, 0, s>>>(D, Wk, X.d_recv);
    k_acc_zero<<<W_local, 1, 0, s>>>(Wk.sc, kRestartSet, Wk.rmask);
    if (D.n > 0) k_cut_dot<<<dim3(gx, W_local), 256, 0, s>>>(D, Wk.x, Wk.xs, Wk.sc, kRestartSet, Wk.rmask);
    k_rows_init<<<dim3(p->rows_grid, W_local), 256, 0, s>>>(D, Wk, 0, nullptr, kRestartSet, nullptr);
    k_viol_count<<<dim3(grid_for(D.m_norm, 256, 2 * p->sm_count), W_local), 256, 0, s>>>(D, Wk, kRestartSet);
    if (Wk.xbits && D.n > 0) k_xbits_build<<<dim3(gx4, Wk.n_groups), 256, 0, s>>>(D, Wk, kRestartSet);
    k_tabu_clear<<<dim3(gx4, W_local), 256, 0, s>>>(Wk.tabu, Wk.ts, D.n, kRestartSet, Wk.rmask);
    k_walker_finalize_init<<<W_local, 1, 0, s>>>(D, Wk, 1, kRestartSet);
    if (Wk.dirty) k_dirty_all<<<1, 32, 0, s>>>(Wk, kRestartSet);   // f2: a new point
    k_flush_incumbent<<<dim3(gx4, W_local), 256, 0, s>>>(D, Wk);
    k_flush_done<<<(W_local + 255) / 256, 256, 0, s>>>(Wk);
  }
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

// The persistent best incumbent of the device exchanges to the host (synchronises s; nothing to do
// when both outputs are NULL).
static chap_status exchange_result(chap_walkers* S, double* z_best, int32_t* z_walker, cudaStream_t s) {
  if (!z_best && !z_walker) return CHAP_OK;
  chap_exchange_state& X = *S->xs;
  double z = INFINITY;
  int32_t zg = -1;
  CUDA_TRY(cudaMemcpyAsync(&z, X.d_z, sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(&zg, X.d_ip, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  X.z = z;
  X.zg = zg;
  if (z_best) *z_best = z;
  if (z_walker) *z_walker = zg;
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_exchange(chap_walkers* S, chap_comm* comm, double* z_best,
                                             int32_t* z_walker, void* cuda_stream) {
  if (!S) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers");
  if (S->prm.exchange_K < 1 || S->prm.n_elite < 0) return fail(CHAP_ERR_INVALID_ARG, "n_elite < 0");
  if (comm && comm->device != S->P->device) return fail(CHAP_ERR_INVALID_ARG, "comm and walkers on different devices");
  DeviceGuard g(S->P->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  TRY(exchange_prepare(S, comm));
  TRY(exchange_device(S, comm, s));
  return exchange_result(S, z_best, z_walker, s);
}

extern "C" chap_status chap_exchange_plan_device(int32_t W_total, int32_t W_local, int32_t rank,
                                                 const chap_walker_summary* s, int32_t n_elite, int32_t n_restart,
                                                 double* z_best, int32_t* counts, int32_t* elite_gid,
                                                 int32_t* elite_slot, int32_t* local_rank, int32_t* restart_gid,
                                                 int32_t* restart_src, int32_t* restart_slot, void* cuda_stream) {
  if (W_total < 1 || W_local < 1 || W_total % W_local || rank < 0 || rank >= W_total / W_local || !s ||
      n_elite < 0 || n_restart < 0 || !z_best || !counts || !elite_gid || !elite_slot || !local_rank ||
      !restart_gid || !restart_src || !restart_slot)
    return fail(CHAP_ERR_INVALID_ARG, "bad device exchange-plan arguments");
  k_exchange_plan<<<1, 1024, 0, (cudaStream_t)cuda_stream>>>(s, W_total, W_local, rank, n_elite, n_restart, z_best,
                                                             counts, elite_gid, elite_slot, local_rank, restart_gid,
                                                             restart_src, restart_slot);
  CUDA_TRY(cudaGetLastError());
  return CHAP_OK;
}

extern "C" chap_status chap_walkers_epoch(chap_walkers* S, chap_comm* comm, int32_t n_iters, double* z_best,
                                          int32_t* z_walker, void* cuda_stream) {
  if (!S || n_iters < 1) return fail(CHAP_ERR_INVALID_ARG, "NULL walkers or n_iters < 1");
  if (S->prm.exchange_K < 1 || S->prm.n_elite < 0) return fail(CHAP_ERR_INVALID_ARG, "n_elite < 0");
  if (comm && comm->device != S->P->device) return fail(CHAP_ERR_INVALID_ARG, "comm and walkers on different devices");
  DeviceGuard g(S->P->device);
  cudaStream_t us = (cudaStream_t)cuda_stream;
  cudaStream_t s = S->stream;
  TRY(exchange_prepare(S, comm));
  if (S->gexec_ep && (S->ep_iters != n_iters || S->ep_comm != (const void*)comm)) {
    cudaGraphExecDestroy(S->gexec_ep);
    S->gexec_ep = nullptr;
  }
  CUDA_TRY(cudaEventRecord(S->ev_in, us));
  CUDA_TRY(cudaStreamWaitEvent(s, S->ev_in, 0));
  if (!S->gexec_ep) {
    TRY(capture_graph(S, s, n_iters, [&](cudaStream_t cs) -> chap_status {
      const DevProblem& D = S->P->dp;
      k_flush_incumbent<<<dim3(grid_for(D.n, 256, 4 * S->P->sm_count), S->W), 256, 0, cs>>>(D, S->wk);
      k_flush_done<<<(S->W + 255) / 256, 256, 0, cs>>>(S->wk);
      return exchange_device(S, comm, cs);
    }, &S->gexec_ep));
    S->ep_iters = n_iters;
    S->ep_comm = comm;
  }
  CUDA_TRY(cudaGraphLaunch(S->gexec_ep, s));
  CUDA_TRY(cudaEventRecord(S->ev_out, s));
  CUDA_TRY(cudaStreamWaitEvent(us, S->ev_out, 0));
  return exchange_result(S, z_best, z_walker, us);
}

extern "C" chap_status chap_run_walkers(const chap_problem* p, int32_t W_local, const double* x0,
                                        const chap_params* params, chap_comm* comm, int64_t max_iters,
                                        double time_limit_s, double* best_x, chap_result* out,
                                        void* cuda_stream) {
  if (!p || W_local < 1 || !x0 || !out || max_iters < 0) return fail(CHAP_ERR_INVALID_ARG, "bad arguments");
  chap_params prm;
  if (params) prm = *params; else chap_params_default(&prm);
  if (prm.exchange_K < 1 || prm.n_elite < 0) return fail(CHAP_ERR_INVALID_ARG, "exchange_K < 1 or n_elite < 0");
  if (comm && comm->device != p->device) return fail(CHAP_ERR_INVALID_ARG, "comm and problem on different devices");
  DeviceGuard g(p->device);
  const auto t0 = std::chrono::steady_clock::now();
  const int E = prm.n_elite;
  const int n = p->dp.n;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  chap_walkers* S = nullptr;
  TRY(chap_walkers_create(p, W_local, x0, &prm, cuda_stream, &S));
  std::unique_ptr<chap_walkers, chap_status (*)(chap_walkers*)> hold(S, chap_walkers_destroy);
  int64_t iters = 0, epochs = 0;
  bool stop = false;
  while (!stop) {
    const int64_t k = std::min<int64_t>(prm.exchange_K, max_iters - iters);
    if (time_limit_s <= 0 && k > 0 && iters + k < max_iters) {
      // not the last epoch and no clock to vote on: iterations + device exchange as one graph
      TRY(chap_walkers_epoch(S, comm, (int32_t)k, nullptr, nullptr, cuda_stream));
      iters += k;
      ++epochs;
      continue;
    }
    if (k > 0) TRY(chap_tabu_step(S, (int32_t)k, nullptr, cuda_stream));
    iters += k;
    ++epochs;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool want_stop = iters >= max_iters || (time_limit_s > 0 && el >= time_limit_s);
    TRY(exchange_internal(S, comm, want_stop, best_x != nullptr, &stop, s));
  }
  const chap_exchange_state& X = *S->xs;
  // best point: the top feasible elite member (slot of E[0] when it is feasible)
  out->best_obj = X.z;
  out->has_incumbent = X.zg >= 0;
  out->best_walker = X.zg;
  out->iterations = iters;
  out->epochs = epochs;
  if (best_x && X.zg >= 0 && E > 0) {
    // E[0] is the global best incumbent; export it in user order
    k_unpack_point<<<grid_for(n, 256, 2 * p->sm_count), 256, 0, s>>>(p->dp, X.d_recv + (size_t)X.e_slot[0] * p->dp.pk_bytes,
                                                                       X.d_x);
    k_export_point<<<grid_for(n, 256, 4 * p->sm_count), 256, 0, s>>>(p->dp, X.d_x, best_x);
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return CHAP_OK;
}

// common.cuh — internal types of libchap (the CUDA path). Never included by oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "chap.h"

namespace chap {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kTileThreads = 256;                 // k_eval block
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kGenmMax = 2048;                    // Alg. 1 elements of a single-column sort tile
constexpr int kWSlotsGen = 4;                     // slots per lane of a general warp tile
constexpr int kWTileGen = 32 * kWSlotsGen;        // Alg. 1 elements per general warp tile
constexpr int kWTileCols = 32;                    // columns per warp tile (one lane each)
constexpr int kBinSlots = 4;                      // slots per lane of a binary warp tile
constexpr int kBinTile = 32 * kBinSlots;          // nonzeros per binary warp tile
#ifndef CHAP_BIN_THREADS
#define CHAP_BIN_THREADS 256
#endif
constexpr int kBinThreads = CHAP_BIN_THREADS;     // k_eval_bin block
#ifndef CHAP_BIN_MINB
#define CHAP_BIN_MINB 4
#endif
constexpr int kBinMinBlocks = CHAP_BIN_MINB;      // k_eval_bin resident blocks per SM (register budget)
#ifndef CHAP_GEN_THREADS
#define CHAP_GEN_THREADS 320
#endif
constexpr int kGenThreads = CHAP_GEN_THREADS;     // k_eval_gen block
#ifndef CHAP_GEN_MINB
#define CHAP_GEN_MINB 2
#endif
constexpr int kGenMinBlocks = CHAP_GEN_MINB;      // k_eval_gen resident blocks per SM (register budget)
constexpr int kShortDeg = 64;                     // binary deg <= 64 / general deg+2 <= 64: packed tiles
constexpr int kBucketMax = 4096;                  // max integer domain of a bucket-scanned column
constexpr int kApplyThreads = 256;

// Per normalised row and walker: the residual r_i = ȳ_i - b_i (double) and the
// constraint weight w_i (float) packed into one 16-byte record so a column's
// gather of row i costs one 32-byte sector, not two.
struct __align__(16) RowState {
  double r;
  float w;
  int32_t rc;   // ceil(r) clamped to int32 (r <= v <=> rc <= v for integers v): kept with r by every
                // writer (set_r) so that k_eval_binrow tests feasibility in integers
};
__host__ __device__ __forceinline__ int32_t r_ceil(double r) {
  return r >= 2147483647.0 ? 2147483647 : (r <= -2147483648.0 ? (-2147483647 - 1) : (int32_t)ceil(r));
}
__host__ __device__ __forceinline__ void set_r(RowState& s, double r) {
  s.r = r;
  s.rc = r_ceil(r);
}

// Column classes (the paper's length-specialised dispatch, re-designed).
enum ColClass : int {
  CC_FIXED = 0,  // l = u: no candidate
  CC_LBKT = 1,   // general integer, deg+2 > kShortDeg, bounded domain <= kBucketMax: bucket scan
                 // over kBktChunk-nonzero warp chunks, finished by k_eval
  CC_LBIN = 2,   // binary, deg > kShortDeg: flip partial sums over kWChunk-nonzero warp chunks
  CC_GENM = 3,   // general, kShortDeg < deg+2 <= kGenmMax, other domains: one tile, bitonic sort
  CC_GEN = 4,    // general integer, deg+2 <= kShortDeg: packed warp tiles (gen32_tile), sort-free
  CC_BIN = 5,    // binary, deg <= kShortDeg: packed tiles, flip sums
  CC_EMPTY = 6,  // a column without nonzeros (and c_j = 0)
  CC_GENC = 7,   // continuous, deg+2 <= kShortDeg: a lane per column (gen_column_serial)
  CC_GENL = 8,   // general, deg+2 > kGenmMax, not bucketable: grid-wide sort (chunk sorts + co-ranking)
};

// A warp tile: ncols consecutive packed columns (CC_BIN or CC_GEN) of one warp.
struct WTile {
  int32_t p0;
  int32_t e0;
  int32_t e1;        // nonzero range [e0, e1); a chunk of a long column: the long-column index
  int16_t ncols;     // columns; a chunk of a long column: its nonzeros (<= kWChunk)
  int8_t kind;       // CC_BIN, CC_GEN, CC_EMPTY, or a warp chunk of a long column: CC_LBIN, CC_LBKT
  int8_t pad;
};
// A long column split into warp chunks: where its accumulators live in walker scratch.
struct LongCol {
  int64_t scr;       // offset (doubles) of the accumulators in walker scratch
  int64_t tix;       // offset (doubles) of the column's chunk ticket (unsigned) in walker scratch
  int32_t nchunks;
  int32_t dom;       // CC_LBKT: u - l + 1
  int32_t p;         // the column (internal order)
  int32_t kind;      // CC_LBIN or CC_LBKT
};
#ifndef CHAP_WCHUNK
#define CHAP_WCHUNK 256
#endif
constexpr int kWChunk = CHAP_WCHUNK;                      // nonzeros per warp chunk of a long binary column
#ifndef CHAP_BKT_CHUNK
#define CHAP_BKT_CHUNK 512
#endif
constexpr int kBktChunk = CHAP_BKT_CHUNK;         // nonzeros per warp chunk of a long bounded-integer column

// A block tile (chunk of a long column, or one column sorted by the whole block).
struct Tile {
  int32_t kind;      // CC_GENM
  int32_t p0;        // the column (internal)
  int32_t ncols;     // 1
  int32_t e0, e1;    // nonzero range [e0, e1) (CSC, internal)
  int32_t pad;
};

// Row-wise binary flip evaluation (k_eval_binrow, PAPER.md:347 re-designed): the packed binary
// columns are cut into variable blocks; the nonzeros of a block are stored sorted by row and cut
// into kRowCluster equal slices, one per CTA of a thread-block cluster.
constexpr int kRowCluster = 12;                   // max CTAs per cluster (above 8: non-portable); the
                                                  // width used is chosen at problem create
constexpr int kRowThreads = 1024;                 // k_eval_binrow block (one CTA per SM)
constexpr int kRowVmax = 32768;                   // variables per block: int32 scores in 128 KB of smem
constexpr int kRowWpb = kRowVmax / 32;            // bitset words per block
constexpr int kRowConsumers = kRowThreads - 32;   // consumer threads (the last warp produces)
#ifndef CHAP_ROW_PER
#define CHAP_ROW_PER 5
#endif
#ifndef CHAP_ROW_STAGES
#define CHAP_ROW_STAGES 2
#endif
#ifndef CHAP_ROW_GATHER
#define CHAP_ROW_GATHER 1
#endif
#ifndef CHAP_ROW_SPAN
#define CHAP_ROW_SPAN (CHAP_ROW_GATHER ? 2 : 2000)
#endif
constexpr int kRowPer = CHAP_ROW_PER;             // entries per consumer thread per stage
constexpr int kRowChunk = kRowPer * kRowConsumers;   // max entries per stage (a multiple of 4)
constexpr int kRowSpan = CHAP_ROW_SPAN;           // max rows of row state per stage
constexpr int kRowStages = CHAP_ROW_STAGES;       // stages of the ring (entries + row state)
static_assert(kRowChunk % 4 == 0, "stages start on 16-byte boundaries");
struct RowBlock {
  int32_t p0;                 // first column (internal order): column k of block b is p0 + k nb
  int32_t nv;                 // columns
  int32_t es[kRowCluster + 1];   // entry slices [es[s], es[s+1]), multiples of 4
  int32_t st[kRowCluster + 1];   // the stages of slice s: [st[s], st[s+1]) in DevProblem::rb_stage
  int32_t pad[2];
};
// One stage of a slice: entries [e0, e0 + ne) (a multiple of 4 each) whose rows lie in [r0, r0 + nr):
// the row state of those rows comes with the entries by one bulk copy; nr = 0: the stage's rows span
// more than kRowSpan rows and its row state is gathered instead.
struct RowStage {
  int32_t e0, ne, r0, nr;
};

// A general column longer than one block sort (CC_GENL, "grid-wide primitives"): its
// entries are cut into chunks of <= kSortChunk (chunk 0 also holds the two bounds), each sorted by
// one block; every candidate is then co-ranked against every other chunk by binary search.
constexpr int kSortChunk = kGenmMax - 2;
// walker scratch of one chunk (doubles): t[kGenmMax], P[kGenmMax] (prefix of δ in sorted order),
// mk[kGenmMax] (u32), then n (entries), β, α, best s, best v of the chunk's candidates
constexpr int kSortStride = 2 * kGenmMax + kGenmMax / 2 + 8;
struct SortCol {
  int64_t scr;       // offset (doubles) of chunk 0 in walker scratch
  int32_t p;         // the column (internal order)
  int32_t nchunks;
};

// Per-column result competing for the global best move.
struct Cand {
  double s;
  double v;
  int32_t j;  // user index (tie-break, R6)
  int32_t p;  // internal index
};

struct Decision {
  int32_t move;  // 1: apply, 0: stuck
  int32_t p;     // internal column (if move)
  int32_t j;     // user column, -1 if none admissible
  int32_t pad;
  double v;
  double s;
  double delta;  // v - x̄_p
};

// Walker scalars, device resident.
struct WalkerScalars {
  long long k;
  long long violated;
  double obj;
  double best_obj;
  double cutoff_rhs;
  int cut_active;
  int has_inc;
  int pending_copy;  // best_x <- x still to be done (done by the next apply kernel / a flush)
  int pad0;
  long long n_moves;
  long long n_stuck;
  Decision dec;
  unsigned apply_counter;
  unsigned pad1;
  long long log_k0;           // k of log row 0 (set per chap_tabu_step)
  chap_step_record* log;      // current log base (NULL = no log)
  double cdot;                // c.x of the current point (k_cut_dot), for the cutoff row and obj
  long long vcount;           // violated active rows (k_viol_count)
  int wint;                   // every weight is an integer <= 2^20 (the int path of gen32_tile)
  int rint;                   // every residual is an integer (DevProblem::rint_base and an integral cutoff rhs)
  // perturbation (chap_params.perturb, NEXT f1, DESIGN R21): a stuck iteration's row draw (minimum of
  // (h32 << 32 | i) over the violated / over all active rows, ~0 = none yet) and the move it yields,
  // which iteration k + 1 applies in place of its selection (force_p = -1: none pending)
  unsigned long long pert_kv;
  unsigned long long pert_ka;
  int force_p;
  int pad2;
  double force_v;
};

// SplitMix64's output function (Steele, Lea, Flood 2014; the first output of a generator seeded
// with z) and the counter-based draw of R21: H(seed, a, b, c) = g(g(g(g(seed) ^ a) ^ b) ^ c).
__host__ __device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long rng_draw(unsigned long long seed, unsigned long long a,
                                                              unsigned long long b, unsigned long long c) {
  return splitmix64(splitmix64(splitmix64(splitmix64(seed) ^ a) ^ b) ^ c);
}
constexpr unsigned long long kDrawEntry = 1ull << 62;         // c of the entry draw (rows use c = i)
constexpr unsigned long long kDrawValue = (1ull << 62) + 1;   // c of the value draw
constexpr unsigned long long kDrawSmooth = (1ull << 62) + 2;  // c of the weight-smoothing draw (R22)

// Per-kernel device time (chap_walkers_timing): %globaltimer at every block's start (atomic min)
// and end (atomic max) into DevWalkers::kt when it is non-NULL; k_apply accumulates the spans.
__device__ __forceinline__ unsigned long long kt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// mbarrier / bulk-copy (TMA) helpers (PTX ISA: mbarrier, cp.async.bulk)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
      ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
// Ampere-style asynchronous copies (cp.async, LDGSTS): per-thread gathers into shared memory,
// completed by commit/wait groups (no registers held while in flight)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_u32(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Programmatic dependent launch (the tabu iteration's kernels are launched with the PDL
// attribute): wait for the preceding grid to complete and its writes to be visible, then let the
// next grid be scheduled onto SMs as this one's blocks retire. Both are no-ops for plain launches.
__device__ __forceinline__ void pdl_wait_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#define KT_BEGIN(WK, q) do { if ((WK).kt && threadIdx.x == 0) atomicMin((WK).kt + 2 * (q), chap::kt_now()); } while (0)
#define KT_END(WK, q) do { if ((WK).kt && threadIdx.x == 0) atomicMax((WK).kt + 2 * (q) + 1, chap::kt_now()); } while (0)
constexpr int kRestartSet = -2;   // only_walker: every walker w with DevWalkers::rmask[w] >= 0 (blockIdx)
__device__ __forceinline__ bool skip_walker(const int32_t* rmask, int only_walker, int w) {
  return only_walker == kRestartSet && rmask[w] < 0;
}
constexpr int kKtWords = 16;   // [2q, 2q+1] start/end of kernel q (0 bin, 1 gen, 2 eval, 3 apply); [8..13] sums

// Everything the kernels need about the immutable problem (internal variable order).
struct DevProblem {
  int32_t n, m_norm, cut_row;
  int32_t dummy_row;         // = m_norm: the inert row (r = -inf, w = 0) of padding entries
  const int32_t* col_ptr;    // [n+1] CSC over normalised rows incl. the cutoff row (last entry)
  const int32_t* row_idx;    // [nnz_total]
  const double* val;         // [nnz_total]
  const int32_t* rp;         // CSR [m_norm+1], cutoff row last
  const int32_t* ci;         // CSR columns (internal index)
  const double* cv;          // CSR values
  const double* b;           // [m_norm-1]
  const double* lb;          // [n]
  const double* ub;          // [n]
  const double* c;           // [n]
  const uint8_t* vclass;     // [n] 0 fixed 1 binary 2 integer 3 continuous
  const int32_t* perm;       // internal p -> user j
  const Tile* tiles; int32_t n_tiles; int32_t n_long;   // block tiles
  const Tile* schunks; int32_t n_schunks;               // chunks of CC_GENL columns (e0, e1: entries;
                                                        // ncols: chunk index; pad: the SortCol)
  const SortCol* scols; int32_t n_scols;                // CC_GENL columns
  const WTile* wtiles; int32_t n_wtiles;                // warp tiles: n_gtiles CC_GEN, n_ctiles CC_GENC, then
  int32_t n_gtiles, n_ctiles;                           // CC_EMPTY
  const WTile* btiles; int32_t n_btiles;                // pipelined binary warp tiles
  const WTile* bchunks; int32_t n_bchunks;              // warp chunks of long binary columns
  const WTile* gchunks; int32_t n_gchunks;              // warp chunks of long bounded-integer columns
  const WTile* gitems; int32_t n_gitems;                // k_eval_gen's items: bchunks and gchunks interleaved,
                                                        // continuous tiles, general tiles, empty tiles
  const WTile* gitems2; int32_t n_gitems2;              // the same without the long binary chunks (the modes
                                                        // where k_eval_bin / k_eval_bin_wm take them)
  const LongCol* lcols;                                 // [n_long]
  const int32_t* lfin; int32_t n_lfin;                  // long columns k_eval finishes
  const RowBlock* rblocks; int32_t n_rblocks;           // row-wise binary blocks (0: not built)
  int32_t rb_cluster;        // CTAs per cluster of k_eval_binrow (= slices per block)
  int32_t rb_pb0, rb_nbin;   // packed binary columns [rb_pb0, rb_pb0 + rb_nbin), round-robin over blocks
  const int32_t* rb_perm;    // [n_rblocks][kRowVmax] user index of column k of block b (block order)
  const int2* rb_rc;         // [entries] row of each entry (sorted within a slice), column within the
                             // block (low 16 bits) | int16 a_ij (high 16)
  const RowStage* rb_stage;  // stages of the slices (RowBlock::st)
  // packed points of the portfolio exchange: binaries as bits (PAPER.md:349's bitset),
  // integers as int32 (int64 when a bound is infinite or beyond 2^31), continuous as f64
  const int32_t* pk_bin; const int32_t* pk_int; const int32_t* pk_cont;   // internal columns of each class
  int32_t pk_nbin, pk_nint, pk_ncont, pk_int64;
  int64_t pk_off_int, pk_off_cont, pk_bytes;   // byte offsets of the sections, bytes per point
  int32_t n_fixed;           // internal columns [0, n_fixed) are fixed
  int32_t rint_base;         // integer data with |coefficients| <= 2^22 and no continuous variable: every
                             // residual is an integer while the cutoff rhs is (WalkerScalars::rint)
  double auto_delta;
};

// Per-walker-set state views; walker w = blockIdx.y.
// Row state is grouped by walkers: groups of rg consecutive walkers, and inside a group the rg
// walkers' records of one row are adjacent (walker-minor), so that one row's state for the whole
// group is one contiguous run (rg x 16 B): record (w, i) is at rs[((w / rg) * rss + i) * rg + w % rg].
// rg = 1 is the walker-major layout of a single walker.
struct DevWalkers {
  double* x;            size_t xs;     // [W][n] internal order
  RowState* rs;         size_t rss;    // [W/rg][rss = m_norm + 1][rg]
  int32_t rg;                          // walkers per row-state group (1, or a power of two <= 32)
  int32_t n_groups;                    // ceil(W / rg)
  uint32_t* xbits;                     // rg > 1: [n_groups][n], bit (w % rg) = x̄ of binary p for walker w;
                                       // rg = 1 (one walker, k_eval_binrow): block-ordered bitset of the
                                       // packed binaries, [n_rblocks][kRowWpb], column k of block b at
                                       // bit k % 32 of word b kRowWpb + k / 32 (the bitset incumbent of
                                       // PAPER.md:349); NULL = not kept
  int32_t* tabu;        size_t ts;     // [W][n]
  double* best_x;                      // [W][n]
  WalkerScalars* sc;                   // [W]
  Cand* part;           int32_t ps;    // [W][ps] one per eval block
  unsigned* sel_count;                 // [W] last-block-done counter of the eval kernel
  unsigned* gen_ctr;                   // [W][2] k_eval_gen: next item, blocks done (re-armed by the last block)
  const int32_t* rmask;                // [W] device exchange: the restart source slot of each walker (-1: none);
                                       // the restart kernels launched with only_walker = kRestartSet skip
                                       // the walkers without one
  double* lscr;         size_t lss;    // [W][lss]
  int32_t use_tabu;
  int32_t W;
  int32_t tenure;
  float wcap;
  double delta;                        // NaN = auto
  unsigned long long* kt;              // [kKtWords] kernel timing, NULL = off
  // selective re-evaluation (chap_params.lazy, NEXT f2; one walker): cached per-column results and
  // two dirty bitsets over the internal columns (iteration k evaluates set k & 1, its apply marks set
  // (k + 1) & 1 and clears set k & 1); word dwords of a set = "every column dirty"
  double* cs;                          // [n] cached s_j (internal order), NULL = from scratch
  double* cv;                          // [n] cached x̂_j
  uint32_t* dirty;                     // [2][dwords + 1]
  int32_t dwords;
  int32_t lbkt_wm;                     // walker groups: k_eval_gen_wm takes the long bounded-integer chunks (a10)
  int32_t lbkt_wm_words;               // ... with this many ints of shared memory per warp for the histograms
  int32_t perturb;                     // chap_params.perturb (R21)
  int32_t perturb_radius;              // the window half-width on an infinite side
  unsigned long long rng_seed;         // the seed of the draws (R21, R22)
  float smooth_prob;                   // chap_params.smooth_prob (R22)
  Cand* asp;                           // [W][tenure] aspiration slots (chap_params.aspiration), NULL = off:
                                       // the eval kernels note every tabu column with s > 0 in slot
                                       // tabu_until % tenure; the select takes the feasible ones (R18)
};

// The row state of one walker: base pointer and stride (in records) between consecutive rows.
struct RowView {
  RowState* p;
  int st;
  __device__ __forceinline__ RowState& operator[](int i) const { return p[(size_t)i * st]; }
};
__host__ __device__ __forceinline__ RowView row_view(const DevWalkers& Wk, int w) {
  RowView v;
  v.p = Wk.rs + ((size_t)(w / Wk.rg) * Wk.rss) * Wk.rg + (w % Wk.rg);
  v.st = Wk.rg;
  return v;
}

}  // namespace chap

// common.cuh — internal types of libchap (the CUDA path). Never included by oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "chap.h"

namespace chap {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kEvalThreads = 256;                 // 8 warps per block in the warp-task kernel
constexpr int kEvalWarps = kEvalThreads / kWarp;
constexpr int kBinWideMax = 4096;                 // binary columns with 32 < deg <= this: warp/column
constexpr int kBlockElems = 4096;                 // general columns with deg+2 <= this: block/column
constexpr int kBlockThreads = 256;
constexpr int kLongChunk = 4096;                  // nonzeros per block of a long (chunked) column
constexpr int kBucketMax = 4096;                  // max integer domain of a chunked general column
constexpr int kApplyThreads = 256;

// Per normalised row and walker: the residual r_i = ȳ_i - b_i (double) and the
// constraint weight w_i (float) packed into one 16-byte record so a column's
// gather of row i costs one 32-byte sector, not two.
struct __align__(16) RowState {
  double r;
  float w;
  uint32_t pad;
};

// Column classes (the paper's length-specialised dispatch).
enum ColClass : int {
  CC_FIXED = 0,   // l = u: no candidate
  CC_BIN = 1,     // binary, deg <= 32: g lanes per column, several columns per warp (flip)
  CC_BINW = 2,    // binary, 32 < deg <= kBinWideMax: one warp per column
  CC_BINL = 3,    // binary, longer: chunked over blocks
  CC_GEN = 4,     // integer/continuous, deg+2 <= 32: g lanes per column, warp sort-scan-argmax
  CC_GENB = 5,    // deg+2 <= kBlockElems: one block per column, shared-memory sort-scan-argmax
  CC_GENL = 6,    // longer, bounded integer domain <= kBucketMax: chunked bucket scan
};

// A warp task: ncols consecutive internal columns of one class and group size g.
struct WTask {
  int32_t p0;
  int16_t ncols;
  int8_t kind;    // CC_BIN, CC_BINW, CC_GEN
  int8_t lg;      // log2(g)
};

// One block of a chunked long column.
struct LChunk {
  int32_t p;       // internal column
  int32_t lc;      // long-column slot
  int32_t e0, e1;  // nonzero range of this chunk (CSC, internal)
  int32_t chunk, nchunks;
  int32_t kind;    // 0 binary flip sums, 1 bucket (integer domain)
  int32_t dom;     // u - l + 1 for kind 1
  int64_t scr;     // offset (in doubles) of this column's scratch in a walker's scratch
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
};

// Everything the kernels need about the immutable problem (internal variable order).
struct DevProblem {
  int32_t n, m_norm, cut_row;
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
  const WTask* wtasks; int32_t n_wtasks;
  const int32_t* bcols; int32_t n_bcols;
  const LChunk* chunks; int32_t n_chunks; int32_t n_long;
  int32_t n_fixed;           // internal columns [0, n_fixed) are fixed
  double auto_delta;
};

// Per-walker-set state views; walker w = blockIdx.y.
struct DevWalkers {
  double* x;            size_t xs;     // [W][n] internal order
  RowState* rs;         size_t rss;    // [W][m_norm]
  int32_t* tabu;        size_t ts;     // [W][n]
  double* best_x;                      // [W][n]
  WalkerScalars* sc;                   // [W]
  Cand* part;           int32_t ps;    // [W][ps]
  unsigned* lcount;     int32_t lcs;   // [W][n_long]
  double* lscr;         size_t lss;    // [W][lss]
  int32_t use_tabu;
  int32_t W;
  int32_t tenure;
  float wcap;
  double delta;                        // NaN = auto
};

// Partial-array layout of the eval kernels (per walker).
struct PartLayout {
  int32_t warp_blocks;   // partials [0, warp_blocks)
  int32_t block_off;     // [block_off, block_off + n_bcols)
  int32_t long_off;      // [long_off, long_off + n_chunks)
  int32_t total;
};

}  // namespace chap

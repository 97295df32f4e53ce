// Shared device-side plumbing for the TE-CCL LP engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#include <string>

#include "../../include/teccl_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "teccl_b200 is built for sm_100a only"
#endif

namespace teccl {

constexpr int kSMs = 148;          // B200: 2 dies x 74 SMs
constexpr int kThreads = 256;      // block size of every streaming kernel
constexpr uint32_t kSignBit = 0x80000000u;  // unit-coefficient CSR: bit31 = negative
constexpr uint32_t kIdxMask = 0x7fffffffu;

void set_error(const std::string& msg);

// Held around CUDA-graph capture and around calls that synchronise the
// whole device (pinned-host alloc/free, device-wide syncs): several host
// threads may drive their own contexts on one GPU (sweep.solve_shard), and a
// device-wide synchronisation issued while another thread captures
// invalidates that capture.
std::mutex& device_mutex();

#define TECCL_CUDA(call)                                                         \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::teccl::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));    \
      return TECCL_ECUDA;                                                        \
    }                                                                            \
  } while (0)

#define TECCL_CHECK_LAUNCH()                                                     \
  do {                                                                           \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::teccl::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return TECCL_ECUDA;                                                        \
    }                                                                            \
  } while (0)

// Grid for a grid-stride loop over `work` items: a multiple of the SM count,
// capped so every SM holds `per_sm` resident blocks.
inline int grid_for(int64_t work, int threads = kThreads, int per_sm = 8) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)kSMs * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace teccl

// Device-resident LP. Matrix stored twice: CSR (rows) for A.x and CSC for
// A^T.y, both with sorted minor indices. When every coefficient is +-1 the
// value arrays are absent and the sign lives in bit 31 of the index.
struct teccl_lp {
  int32_t m = 0, n = 0;
  int64_t nnz = 0;
  bool unit = false;               // coefficients are +-1, signs in index bit 31
  int64_t* row_ptr = nullptr;      // [m+1]
  uint32_t* col = nullptr;         // [nnz]
  double* val = nullptr;           // [nnz] (explicit only)
  int64_t* col_ptr = nullptr;      // [n+1]
  uint32_t* row = nullptr;         // [nnz]
  double* cval = nullptr;          // [nnz] (explicit only)
  double* row_lo = nullptr;        // [m]
  double* row_hi = nullptr;        // [m]
  double* var_lb = nullptr;        // [n]
  double* var_ub = nullptr;        // [n]
  double* obj = nullptr;           // [n] minimisation costs
  int device = 0;
  cudaStream_t stream = nullptr;   // stream the LP's arrays were allocated on
  // SELL-32 copies used by the PDLP iteration kernels (built on first solve)
  bool sell_ready = false;
  int64_t* srow_off = nullptr;
  int32_t* srow_w = nullptr;
  uint32_t* srow_idx = nullptr;
  double* srow_val = nullptr;
  int64_t* scol_off = nullptr;
  int32_t* scol_w = nullptr;
  uint32_t* scol_idx = nullptr;
  double* scol_val = nullptr;
  int64_t srow_entries = 0, scol_entries = 0;
  uint32_t* sell_idx = nullptr;    // one allocation: [srow_idx | scol_idx]
  size_t sell_idx_bytes = 0;
  // bound classes: uint16 code per column/row into (lb,ub,c) / (lo,hi)
  // dictionaries; nullptr when the LP has too many distinct classes
  uint16_t* col_code = nullptr;
  uint16_t* row_code = nullptr;
  double* col_dict = nullptr;      // [3 * n_col_dict]
  double* row_dict = nullptr;      // [2 * n_row_dict]
  int32_t n_col_dict = 0, n_row_dict = 0;
  // PDLP workspace kept across solves of this LP (buffers, chunk graph,
  // pinned state ring); freed by teccl_lp_destroy through ws_free
  void* pdlp_ws = nullptr;
  void (*ws_free)(void*) = nullptr;
  // Row-partitioned (epoch-block) LPs built by teccl_lp_build_te_part: this
  // device owns global epoch-major rows [own_r0, own_r1) and columns
  // [own_c0, own_c1); its matrices index the gather windows [win_c0, win_c1)
  // (columns) and [win_r0, win_r1) (rows). Single-device LPs: part_world = 1.
  int part_world = 1, part_rank = 0;
  int64_t em_ncols = 0, em_nrows = 0;
  int64_t own_c0 = 0, own_c1 = 0, own_r0 = 0, own_r1 = 0;
  int64_t win_c0 = 0, win_c1 = 0, win_r0 = 0, win_r1 = 0;
  int64_t nnz_csc = -1;            // CSC entries when they differ from nnz
  void* dist = nullptr;            // peer-memory exchange state (pdlp.cu)
  void (*dist_free)(void*) = nullptr;
  // structure tables of a single-device TE LP (teccl::TeHold, te_gen.cuh):
  // lets the PDLP kernels apply A / A^T without reading the stored matrix
  void* te = nullptr;
  void (*te_free)(void*) = nullptr;
  // source-partitioned solve of a whole single-device TE LP (pdlp.cu
  // SrcState): this device updates the columns / rows of its sources and
  // pairs, the capacity rows are summed across devices every iteration
  void* src = nullptr;
  void (*src_free)(void*) = nullptr;
};

// lengths of the vectors the SpMVs gather from, and where the owned part
// starts inside them
inline int64_t gather_cols(const teccl_lp* lp) { return lp->part_world > 1 ? lp->win_c1 - lp->win_c0 : lp->n; }
inline int64_t gather_rows(const teccl_lp* lp) { return lp->part_world > 1 ? lp->win_r1 - lp->win_r0 : lp->m; }
inline int64_t own_col_off(const teccl_lp* lp) { return lp->part_world > 1 ? lp->own_c0 - lp->win_c0 : 0; }
inline int64_t own_row_off(const teccl_lp* lp) { return lp->part_world > 1 ? lp->own_r0 - lp->win_r0 : 0; }

constexpr int kMaxDict = 65536;

struct teccl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
};

// Build the SELL-32 copies of lp's CSR and CSC on `st` (idempotent).
int teccl_build_sell(teccl_lp* lp, cudaStream_t st);

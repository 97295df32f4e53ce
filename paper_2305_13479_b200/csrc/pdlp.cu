// (2)+(3) Restarted reflected-Halpern PDHG (PDLP family) on sm_100a.
//
// Replaces the CPU LP solve of the reference (pkg/src/collsched/solver.py:
// 128-143, scipy.optimize.milp -> HiGHS) for the TE-CCL LP.
//
// Formulation. The iteration runs in the ORIGINAL variables with diagonal
// preconditioners T = tau * D and S = sigma * E, where D = C^2 and E = R^2 come
// from Ruiz + Pock-Chambolle equilibration (C, R column/row scales) and are
// rounded to fp32 once -- the rounded values *are* the preconditioner, so the
// rounding is exact, and the step-size bound uses the same rounded values:
//
//   x+ = clamp(x - tau D (c - A^T y), lb, ub)          xbar = 2 x+ - x
//   y+ = y - sigma E (A xbar - clamp(A xbar - y/(sigma E), lo, hi))
//   z <- lam ((1+rho) z+ - rho z) + (1-lam) z0,        lam = (k+1)/(k+2)
//
// This is exactly PDHG on the equilibrated problem (x = C xs, y = R ys) but
// the matrix is never scaled, so the +-1 TE-CCL matrix streams 4 B/nnz and
// x, y are already the unscaled solution. Bounds and costs are read through
// per-row/per-column uint16 class codes into small dictionaries (a handful of
// distinct (lb,ub,c) / (lo,hi) classes for the TE-CCL LP) when the LP has
// them, else from the full fp64 arrays. Halpern anchors are fp32 (any anchor
// is valid; it only selects which optimal point the iteration heads for).
//
// One iteration = two fused kernels over SELL-32 matrices (sell.cu):
//   col_step: A^T.y + primal step + projection + reflection + Halpern, emits xbar
//   row_step: A.xbar + dual step + projection + Halpern, emits y
// Every `check_every` iterations the chunk ends with KKT kernels (residuals,
// objectives at T(z)), a one-block control kernel (termination, restart,
// primal weight -- all PDLP control flow stays on the device) and restart
// kernels. Chunks are replayed from a CUDA graph, queued ahead of the host.

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "te_gen.cuh"

namespace teccl {

// build-time knobs of the row half-step (A/B builds: tools/build_variant.sh)
#ifndef TECCL_ROW_G
#define TECCL_ROW_G 8      // index loads in flight per row group
#endif
#ifndef TECCL_ROW_MINB
#define TECCL_ROW_MINB 5   // __launch_bounds__ min blocks per SM (48 registers)
#endif
#ifndef TECCL_SEG_MINB
#define TECCL_SEG_MINB 6   // same, row segment kernel (40 registers: -28 % on the 8-chassis LP)
#endif
#ifndef TECCL_SEG_TPW
#define TECCL_SEG_TPW 1    // row segment kernel: tasks per warp (descriptors loaded together)
#endif
#ifndef TECCL_TE2_MINB
#define TECCL_TE2_MINB 8  // same, two-column column kernel (32 registers: -8 % on the 16-chassis LP)
#endif
#ifndef TECCL_TE2_MINB_L2
#define TECCL_TE2_MINB_L2 6  // same, when the gathered vector fits L2 (40 registers)
#endif
#ifndef TECCL_COL_MINB
#define TECCL_COL_MINB 4   // same, pipelined column kernel (64 registers: measured best)
#endif

constexpr int kGrid = kSMs * 8;  // blocks of the setup reduction kernels
constexpr int kNQ = 15;          // partial quantities per check (9 KKT + 6 infeasibility)
constexpr int kSlice = 32;
constexpr int kSegTPW = TECCL_SEG_TPW;
constexpr int kTile = kThreads;  // rows (columns) per block of the step kernels
constexpr int kPersistThreads = 1024;  // threads per block of the persistent chunk kernel
// auto operator (matrix_free = 1): matrix-free kernels from this many columns
// up (configs[1], 0.97M columns, runs L2-resident on the stored SELL kernels)
constexpr int64_t kAutoMatrixFreeCols = 3000000;
// gathered-vector size up to which the matrix-free column kernel assumes L2
// hits (126 MB L2 on B200)
constexpr double kL2GatherBytes = 128.0 * 1024 * 1024;

enum Q { Q_DX = 0, Q_DX0, Q_DY, Q_DY0, Q_RP, Q_DOBJ_ROW, Q_RD, Q_POBJ, Q_DOBJ_COL,
         // Farkas certificate of the dual-iterate change (infeas_*_kernel): value,
         // magnitude of its terms, count of needed-but-infinite bounds; rows / columns
         Q_IC_ROW, Q_IM_ROW, Q_IN_ROW, Q_IC_COL, Q_IM_COL, Q_IN_COL };
__host__ __device__ constexpr bool row_quantity(int k) {
  return k == Q_DY || k == Q_DY0 || k == Q_RP || k == Q_DOBJ_ROW || k == Q_IC_ROW || k == Q_IM_ROW ||
         k == Q_IN_ROW;
}

struct PdlpState {
  double tau, sigma, omega, eta, refl;
  double bnorm, cnorm;       // unscaled norms for the relative criteria
  double eps;
  double r0, rprev, last_r;
  double rs_suff, rs_nec, rs_art, theta, ki, kd, e_int, e_prev;
  double bias;               // log of the primal-weight target bias (omega_bias)
  long long k_inner, total;
  int have_r0, restart, done, restarts, chunk_len, pad;
  double rel_p, rel_d, gap, pobj, dobj;
  double eps_res;            // residual tolerance (<= eps)
  double eps_infeas;         // certificate margin (0: off)
  double cert;               // last certificate value / magnitude
  int infeas_every, infeas_due;
  double lam_tab[128];       // Halpern weights (k+1)/(k+2) of the current chunk's iterations
};
constexpr int kLamTab = 128;

constexpr int kSlots = 16;  // doubles per rank in the slot table
constexpr int kMaxPeers = 8;

// ---------------------------------------------------------------------------
// Peer-memory exchange for row-partitioned solves (one process per GPU,
// buffers shared through CUDA IPC over NVLink/NVSwitch). A "halo event"
// copies this rank's owned boundary entries straight into the neighbours'
// window arrays and then publishes a sequence number into their flag
// arrays; a wait kernel spins (acquire, system scope, with a timeout) until
// the neighbours' sequence numbers for the same event have arrived. Every
// rank issues the same sequence of events, so sequence numbers line up.
struct Signal {
  unsigned long long* peer_flag[kMaxPeers];  // peer's flags[my rank]
  int npeer;
  unsigned long long* seq;                   // my event counter
  unsigned int* arrive;                      // last-block election
};
struct Halo {
  const double* src[2 * kMaxPeers];
  double* dst[2 * kMaxPeers];
  int64_t cnt[2 * kMaxPeers];
  int n;
};
struct Wait {
  const unsigned long long* flags;           // my flags[world]
  int peer[kMaxPeers];
  int npeer;
  const unsigned long long* seq;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// Fused peer exchange of a half-step kernel (row-partitioned solves): its
// owned outputs that fall inside a neighbour's gather window are stored
// straight into that window over NVLink (the value array, and the check
// array on check iterations), and the last block to finish publishes the
// next sequence number; `wait` is the neighbours' previous signal, awaited
// before the kernel gathers. n = 0 on one device.
struct Push {
  double* dv[2];          // neighbour window at owned-local index lo (xbar or y)
  double* dc[2];          // same for the check array (xt or yt)
  int64_t lo[2], hi[2];   // owned-local index range each neighbour needs
  int n;
  Signal sig;
};

// Per-column / per-row problem data as the iteration kernels see it.
struct Bounds {
  const uint16_t* code;  // class code, or nullptr: read the explicit arrays
  const double* dict;    // classes: (lb, ub, c) for columns, (lo, hi) for rows
  const double* a;       // explicit lb (cols) / lo (rows)
  const double* b;       // explicit ub / hi
  const double* c;       // explicit cost (cols only)
};

struct Vecs {
  const float* D;        // column preconditioner C^2
  const float* E;        // row preconditioner R^2
  Bounds col, row;
  double *x, *xt, *xbar; // xbar has an always-zero slot [n] (SELL padding)
  float* x0;
  double *y, *yt;        // y, yt have an always-zero slot [m]
  float* y0;
  // exact unscaled data for the KKT evaluation
  const double *c_u, *lb_u, *ub_u, *lo_u, *hi_u;
  double* part;          // [kNQ * pstride]
  int64_t pstride;
  int nb_row, nb_col;
  PdlpState* st;
  double* slots;         // [world][kSlots]: every rank's reduced partials
  int world, rank;
  int col_pipe;          // column half-step: pipelined resident grid (1) or one thread per column (0)
  int pdl;               // iteration kernels launched with programmatic dependent launch
  int seg;               // matrix-free segment-walking kernels: bit 0 columns, bit 1 rows (else one thread per entry)
  Push push;             // fused halo out (see Push)
  Wait wait;             // fused halo in: neighbours' signal awaited before gathering
};

__device__ __forceinline__ double block_sum(double v, double* sh);

__device__ __forceinline__ void signal_peers(const Signal& S) {
  const unsigned long long s = *S.seq + 1;
  *S.seq = s;
  __threadfence_system();
  for (int q = 0; q < S.npeer; ++q) st_release_sys(S.peer_flag[q], s);
}

// Fused halo, consumer side: thread 0 of every block waits (acquire, system
// scope) for the neighbours' current sequence number; false on timeout
// (the solve then stops with done = 4 on this rank).
__device__ __forceinline__ bool block_wait_peers(const Wait& W, PdlpState* st) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    const unsigned long long want = *W.seq;
    const long long t0 = clock64();
    for (int q = 0; q < W.npeer && ok; ++q)
      while (ld_acquire_sys(W.flags + W.peer[q]) < want) {
        __nanosleep(64);
        if (clock64() - t0 > 40000000000LL) { st->done = 4; ok = 0; break; }
      }
  }
  __syncthreads();
  return ok != 0;
}

// Fused halo, producer side: store entry j's outputs into every neighbour
// window that holds it.
template <bool CHECK>
__device__ __forceinline__ bool push_entry(const Push& P, int64_t j, double v, double c) {
  bool wrote = false;
  for (int r = 0; r < P.n; ++r)
    if (j >= P.lo[r] && j < P.hi[r]) {
      P.dv[r][j - P.lo[r]] = v;
      if (CHECK) P.dc[r][j - P.lo[r]] = c;
      wrote = true;
    }
  return wrote;
}

// ... and at the end of the kernel: the last block publishes the signal.
__device__ __forceinline__ void push_signal(const Push& P, bool wrote) {
  if (P.n == 0) return;
  if (wrote) __threadfence_system();  // this thread's peer stores before the block's arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(P.sig.arrive, 1u);
    if (prev == gridDim.x - 1) {
      *P.sig.arrive = 0u;
      signal_peers(P.sig);
    }
  }
}

// Copy every (src -> peer dst) range, then the last block to finish signals.
__global__ void halo_kernel(Halo H, Signal S, const PdlpState* st) {
  if (st && st->done) return;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int c = 0; c < H.n; ++c)
    for (int64_t i = tid; i < H.cnt[c]; i += stride) H.dst[c][i] = H.src[c][i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(S.arrive, 1u);
    if (prev == gridDim.x - 1) {
      *S.arrive = 0u;
      signal_peers(S);
    }
  }
}

// Spin until every listed peer has published this rank's current sequence
// number. A peer that never arrives (crash, mismatch) trips the ~20 s
// timeout, which stops the solve with done = 4 instead of hanging the GPU.
__global__ void wait_kernel(Wait Wt, PdlpState* st) {
  if (threadIdx.x != 0 || (st && st->done)) return;
  const unsigned long long want = *Wt.seq;
  const long long t0 = clock64();
  for (int q = 0; q < Wt.npeer; ++q) {
    while (ld_acquire_sys(Wt.flags + Wt.peer[q]) < want) {
      __nanosleep(64);
      if (clock64() - t0 > 40000000000LL) {
        if (st) st->done = 4;
        return;
      }
    }
  }
}

// Reduce this rank's partial sums to kNQ values, store them in its slot row
// of every rank's slot table (own + peers), then signal all peers.
__global__ void __launch_bounds__(1024) reduce_publish_kernel(Vecs V, Signal S,
                                                              double* const* peer_slots) {
  __shared__ double wsum[kNQ][32];
  __shared__ double q[kNQ];
  if (V.st->done) return;
  // all nine quantities in one pass (every thread's loads in flight
  // together), then one warp-shuffle + shared-memory reduction
  double a[kNQ];
#pragma unroll
  for (int k = 0; k < kNQ; ++k) a[k] = 0.0;
  const int nbmax = max(V.nb_row, V.nb_col);
  for (int b = threadIdx.x; b < nbmax; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < kNQ; ++k) {
      if (b < (row_quantity(k) ? V.nb_row : V.nb_col)) a[k] += V.part[k * V.pstride + b];
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kNQ; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
    if (l == 0) wsum[k][w] = a[k];
  }
  __syncthreads();
  if (threadIdx.x < kNQ) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += wsum[threadIdx.x][i];
    q[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x < kNQ) {
    V.slots[V.rank * kSlots + threadIdx.x] = q[threadIdx.x];
    for (int p = 0; p < S.npeer; ++p) peer_slots[p][V.rank * kSlots + threadIdx.x] = q[threadIdx.x];
    __threadfence_system();  // this thread's peer stores before the flag
  }
  __syncthreads();
  if (threadIdx.x == 0 && S.npeer > 0) signal_peers(S);
}

// Generic scalar all-reduce helpers for the setup phase: publish `count`
// values (sum of `nb` partials each, stride `pstride`) into the slot tables,
// then (after a wait) sum the slot rows of every rank in rank order.
__global__ void __launch_bounds__(1024) publish_values_kernel(const double* part, int nb,
                                                              int64_t pstride, int count,
                                                              double* slots, int rank, Signal S,
                                                              double* const* peer_slots) {
  __shared__ double sh[32];
  for (int k = 0; k < count; ++k) {
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[k * pstride + b];
    a = block_sum(a, sh);
    if (threadIdx.x == 0) {
      slots[rank * kSlots + k] = a;
      for (int p = 0; p < S.npeer; ++p) peer_slots[p][rank * kSlots + k] = a;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && S.npeer > 0) signal_peers(S);
}

// out[k] = sum over ranks of slots[r][k]; out[count + k] = 1/sqrt(out[k])
__global__ void sum_slots_kernel(const double* slots, int world, int count, double* out) {
  if (threadIdx.x >= count) return;
  double a = 0.0;
  for (int r = 0; r < world; ++r) a += slots[r * kSlots + threadIdx.x];
  out[threadIdx.x] = a;
  out[count + threadIdx.x] = a > 0.0 ? 1.0 / sqrt(a) : 0.0;
}

// ---------------------------------------------------------------------------
// SELL-32 SpMV (layout built by sell.cu): slice s holds rows 32s..32s+31,
// padded to the slice's longest row, column-major inside the slice, so entry
// q of every row of a warp sits in one 128-byte line; padding points at an
// always-zero vector slot. Coalesced index streams, warp-uniform trip counts,
// no shared memory, no barriers; row order unchanged, so the epilogue is
// thread-per-row with coalesced vector traffic.
// v[t & mask] with the sign bit of t applied (unit-coefficient entries):
// one wide multiply-add for the address, one xor for the sign
__device__ __forceinline__ double sgather(const double* __restrict__ v, uint32_t t) {
  uint64_t off;
  asm("mul.wide.u32 %0, %1, 8;" : "=l"(off) : "r"(t & kIdxMask));
  const double xv = __ldg(reinterpret_cast<const double*>(reinterpret_cast<const char*>(v) + off));
  return __hiloint2double(__double2hiint(xv) ^ (int)(t & kSignBit), __double2loint(xv));
}

struct SellView {
  const int64_t* off;
  const int32_t* width;
  const uint32_t* idx;
  const double* val;     // explicit coefficients (nullptr for unit LPs)
  int64_t count;
};

template <bool UNIT, int G = 4>
__device__ __forceinline__ double sell_dot(const SellView& S, uint32_t r,
                                           const double* __restrict__ v) {
  const uint32_t s = r >> 5;
  const int w = __ldg(S.width + s);
  const uint32_t* ip = S.idx + __ldg(S.off + s) + (r & 31);
  const double* vp = UNIT ? nullptr : S.val + (ip - S.idx);
  double acc = 0.0;
  // groups of G entries, predicated: all index loads of a group are in
  // flight together, then all gathers (2 latencies per group, not per entry)
  for (int q = 0; q < w; q += G) {
    uint32_t t[G];
#pragma unroll
    for (int u = 0; u < G; ++u) t[u] = (q + u < w) ? __ldg(ip + (q + u) * kSlice) : 0u;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (q + u < w) {
        if (UNIT) {
          acc += sgather(v, t[u]);
        } else {
          acc += __ldg(vp + (q + u) * kSlice) * __ldg(v + t[u]);
        }
      }
    }
  }
  return acc;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// Programmatic dependent launch (PDL): the iteration kernels are launched
// with programmatic stream serialization, so a kernel's blocks may start
// while its predecessor drains. Everything before pdl_wait() reads only
// data final at least two launches back (dense iterates, constant tables);
// the predecessor's outputs and the solver state are read after it.
// Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return fmin(fmax(v, lo), hi);
}

// Dual step y+ = y - sE (Ax - P[lo,hi](Ax - y / (sE))) without the fp64
// division: with w = sE Ax - y and sE > 0, sE P[lo,hi](u) = P[sE lo, sE hi](sE u),
// so y+ = P[sE lo, sE hi](w) - w.
__device__ __forceinline__ double dual_step(double yi, double s, double se, double lo, double hi) {
  const double w = fma(se, s, -yi);
  return clampd(w, se * lo, se * hi) - w;
}

template <bool DICT>
__device__ __forceinline__ void col_data(const Bounds& B, int64_t j, double& lb, double& ub,
                                         double& c) {
  if (DICT) {
    const double* e = B.dict + 3 * (int64_t)__ldg(B.code + j);
    lb = __ldg(e);
    ub = __ldg(e + 1);
    c = __ldg(e + 2);
  } else {
    lb = __ldg(B.a + j);
    ub = __ldg(B.b + j);
    c = __ldg(B.c + j);
  }
}

template <bool DICT>
__device__ __forceinline__ void row_data(const Bounds& B, int64_t i, double& lo, double& hi) {
  if (DICT) {
    const double* e = B.dict + 2 * (int64_t)__ldg(B.code + i);
    lo = __ldg(e);
    hi = __ldg(e + 1);
  } else {
    lo = __ldg(B.a + i);
    hi = __ldg(B.b + i);
  }
}

// ---------------------------------------------------------------------------
// Primal half-step over columns (CSC as SELL), fused with A^T.y.
template <bool UNIT, bool DICT, bool CHECK, bool PEER>
__global__ void __launch_bounds__(kThreads) col_step_kernel(int32_t n, SellView S, Vecs V,
                                                            int j_in_chunk) {
  __shared__ double sh[32];
  const int64_t j = (int64_t)blockIdx.x * kTile + threadIdx.x;
  // operands of the epilogue do not depend on the SpMV: load them first
  double xj = 0.0, x0 = 0.0, Dj = 0.0, lb = 0.0, ub = 0.0, cj = 0.0;
  if (j < n) {
    xj = V.x[j];
    x0 = (double)V.x0[j];
    Dj = (double)V.D[j];
    col_data<DICT>(V.col, j, lb, ub, cj);
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double tau = st->tau, refl = st->refl;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  if (PEER && V.wait.npeer && (done || !block_wait_peers(V.wait, V.st))) return;
  const double s = (j < n) ? sell_dot<UNIT>(S, j, V.y) : 0.0;
  if (done) return;
  bool wrote = false;
  double dx = 0.0, dx0 = 0.0;
  if (j < n) {
    const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
    const double xb = 2.0 * xt - xj;
    V.xbar[j] = xb;
    wrote = PEER && push_entry<CHECK>(V.push, j, xb, xt);
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      const double w = 1.0 / Dj;
      dx = (xt - xj) * (xt - xj) * w;
      dx0 = (xt - x0) * (xt - x0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
  if (PEER) push_signal(V.push, wrote);
}

// Software-pipelined variant of col_step: a resident grid walks the columns
// with a grid stride; while a thread gathers and updates column j, the slice
// header and index loads of its next column j + stride are already in
// flight, so each column costs about one memory latency instead of three.
template <bool UNIT, bool DICT, bool CHECK, bool PEER>
__global__ void __launch_bounds__(kThreads, TECCL_COL_MINB) col_pipe_kernel(int32_t n, SellView S, Vecs V,
                                                            int j_in_chunk) {
  __shared__ double sh[32];
  // 32-bit column ids (n < 2^31); 64-bit SELL offsets
  const uint32_t un = (uint32_t)n;
  const uint32_t stride = gridDim.x * kThreads;
  uint32_t j = blockIdx.x * kThreads + threadIdx.x;
  // stage 1 of the first column: slice header and up to 4 indices
  int w = 0;
  int64_t base = 0;
  uint32_t t[4] = {0u, 0u, 0u, 0u};
  if (j < un) {
    w = __ldg(S.width + (j >> 5));
    base = __ldg(S.off + (j >> 5)) + (j & 31);
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = (u < w) ? __ldg(S.idx + base + (int64_t)u * kSlice) : 0u;
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;
  const double tau = st->tau, refl = st->refl;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  if (done) return;
  if (PEER && V.wait.npeer && !block_wait_peers(V.wait, V.st)) return;
  double dx = 0.0, dx0 = 0.0;
  bool wrote = false;
  while (j < un) {
    const uint32_t jn = j + stride;
    // next column's slice header: independent of this column's work
    int wn = 0;
    int64_t basen = 0;
    if (jn < un) {
      wn = __ldg(S.width + (jn >> 5));
      basen = __ldg(S.off + (jn >> 5)) + (jn & 31);
    }
    // this column: epilogue operands and gathers
    double lb, ub, cj;
    col_data<DICT>(V.col, j, lb, ub, cj);
    const double xj = V.x[j];
    const double x0 = (double)V.x0[j];
    const double Dj = (double)V.D[j];
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < w) {
        if (UNIT) {
          s += sgather(V.y, t[u]);
        } else {
          s += __ldg(S.val + base + (int64_t)u * kSlice) * __ldg(V.y + t[u]);
        }
      }
    }
    for (int q = 4; q < w; ++q) {  // columns wider than 4 (rare)
      const uint32_t tq = __ldg(S.idx + base + (int64_t)q * kSlice);
      if (UNIT) {
        s += sgather(V.y, tq);
      } else {
        s += __ldg(S.val + base + (int64_t)q * kSlice) * __ldg(V.y + tq);
      }
    }
    // next column's indices (its header has had a whole gather to arrive)
    uint32_t tn[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 4; ++u) tn[u] = (u < wn) ? __ldg(S.idx + basen + (int64_t)u * kSlice) : 0u;
    const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
    const double xb = 2.0 * xt - xj;
    V.xbar[j] = xb;
    wrote |= PEER && push_entry<CHECK>(V.push, j, xb, xt);
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      const double wgt = 1.0 / Dj;
      dx += (xt - xj) * (xt - xj) * wgt;
      dx0 += (xt - x0) * (xt - x0) * wgt;
    }
    j = jn;
    w = wn;
    base = basen;
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = tn[u];
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
  if (PEER) push_signal(V.push, wrote);
}

// Dual half-step over rows (CSR as SELL), fused with A.xbar.
template <bool UNIT, bool DICT, bool CHECK, bool PEER>
__global__ void __launch_bounds__(kThreads, TECCL_ROW_MINB) row_step_kernel(int32_t m, SellView S, Vecs V,
                                                            int j_in_chunk) {
  __shared__ double sh[32];
  const uint32_t i = blockIdx.x * kTile + threadIdx.x;  // m < 2^31
  double yi = 0.0, y0 = 0.0, Ei = 0.0, lo = 0.0, hi = 0.0;
  if (i < (uint32_t)m) {
    yi = V.y[i];
    y0 = (double)V.y0[i];
    Ei = (double)V.E[i];
    row_data<DICT>(V.row, i, lo, hi);
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double sigma = st->sigma, refl = st->refl;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  if (PEER && V.wait.npeer && (done || !block_wait_peers(V.wait, V.st))) return;
  const double s = (i < (uint32_t)m) ? sell_dot<UNIT, TECCL_ROW_G>(S, i, V.xbar) : 0.0;
  if (done) return;
  bool wrote = false;
  double dy = 0.0, dy0 = 0.0;
  if (i < (uint32_t)m) {
    const double se = sigma * Ei;
    const double yt = dual_step(yi, s, se, lo, hi);
    const double yn = lam * ((1.0 + refl) * yt - refl * yi) + (1.0 - lam) * y0;
    V.y[i] = yn;
    wrote = PEER && push_entry<CHECK>(V.push, i, yn, yt);
    if (CHECK) {
      V.yt[i] = yt;
      const double w = 1.0 / Ei;
      dy = (yt - yi) * (yt - yi) * w;
      dy0 = (yt - y0) * (yt - y0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blockIdx.x] = a;
  }
  if (PEER) push_signal(V.push, wrote);
}

// ---------------------------------------------------------------------------
// Persistent chunk kernel (LPs whose iteration is L2-resident, on the stored
// SELL operator: configs[1]). One cooperative launch runs a whole chunk of
// `check_every` iterations. Block b owns a contiguous, slice-aligned range of
// columns and one of rows and keeps their dense state -- x, x0, D and the
// bound class of its columns; y, y0, E and the class of its rows, plus both
// bound dictionaries -- in shared memory for the whole chunk, so an iteration
// moves only the index streams and the gathered vectors (y for the column
// half-step, xbar for the row half-step) through L2. The gathers use
// ld.global.cg: other blocks wrote those vectors earlier in this launch. The
// half-steps are separated by grid barriers instead of kernel boundaries.
// Same arithmetic, in the same order, as col_pipe_kernel / row_step_kernel.
struct Persist {
  int cpb, rpb;            // columns / rows per block (multiples of the SELL slice)
  int ncd, nrd;            // bound-dictionary entries (DICT)
  int chunk;               // iterations per launch (<= kLamTab)
  unsigned int* bar;       // grid-barrier counter, zeroed before each launch
  size_t smem;             // dynamic shared memory per block
};

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();  // this block's stores (xbar / y) before its arrival
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// sell_dot over a vector written by other blocks of this launch (L2, not L1)
template <bool UNIT, int G>
__device__ __forceinline__ double sell_dot_cg(const SellView& S, uint32_t r, const double* __restrict__ v) {
  const uint32_t s = r >> 5;
  const int w = __ldg(S.width + s);
  const uint32_t* ip = S.idx + __ldg(S.off + s) + (r & 31);
  const double* vp = UNIT ? nullptr : S.val + (ip - S.idx);
  double acc = 0.0;
  for (int q = 0; q < w; q += G) {
    uint32_t t[G];
#pragma unroll
    for (int u = 0; u < G; ++u) t[u] = (q + u < w) ? __ldg(ip + (q + u) * kSlice) : 0u;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (q + u < w) {
        if (UNIT) {
          const double xv = __ldcg(v + (t[u] & kIdxMask));
          acc += __hiloint2double(__double2hiint(xv) ^ (int)(t[u] & kSignBit), __double2loint(xv));
        } else {
          acc += __ldg(vp + (q + u) * kSlice) * __ldcg(v + t[u]);
        }
      }
    }
  }
  return acc;
}

template <bool UNIT, bool DICT>
__global__ void __launch_bounds__(kPersistThreads, 1) chunk_persist_kernel(int32_t n, int32_t m, SellView SC,
                                                                           SellView SR, Vecs Vc, Vecs Vr,
                                                                           Persist P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sh[32];
  const PdlpState* st = Vc.st;
  if (st->done) return;  // read before any barrier: every block takes the same branch
  const double tau = st->tau, sigma = st->sigma, refl = st->refl;
  const int c0 = blockIdx.x * P.cpb, nc = max(0, min(P.cpb, n - c0));
  const int r0 = blockIdx.x * P.rpb, nr = max(0, min(P.rpb, m - r0));
  // shared-memory layout: doubles, then floats, then uint16 codes
  double* xs = (double*)smem;
  double* ys = xs + P.cpb;
  double* cdict = ys + P.rpb;                 // [3 * ncd]
  double* rdict = cdict + 3 * P.ncd;          // [2 * nrd]
  double* lam = rdict + 2 * P.nrd;            // [chunk]
  float* x0s = (float*)(lam + P.chunk);
  float* Ds = x0s + P.cpb;
  float* y0s = Ds + P.cpb;
  float* Es = y0s + P.rpb;
  uint16_t* ccode = (uint16_t*)(Es + P.rpb);
  uint16_t* rcode = ccode + P.cpb;
  for (int q = threadIdx.x; q < nc; q += blockDim.x) {
    const int64_t j = c0 + q;
    xs[q] = Vc.x[j];
    x0s[q] = Vc.x0[j];
    Ds[q] = Vc.D[j];
    if (DICT) ccode[q] = Vc.col.code[j];
  }
  for (int q = threadIdx.x; q < nr; q += blockDim.x) {
    const int64_t i = r0 + q;
    ys[q] = Vr.y[i];
    y0s[q] = Vr.y0[i];
    Es[q] = Vr.E[i];
    if (DICT) rcode[q] = Vr.row.code[i];
  }
  if (DICT) {
    for (int q = threadIdx.x; q < 3 * P.ncd; q += blockDim.x) cdict[q] = Vc.col.dict[q];
    for (int q = threadIdx.x; q < 2 * P.nrd; q += blockDim.x) rdict[q] = Vr.row.dict[q];
  }
  for (int q = threadIdx.x; q < P.chunk; q += blockDim.x) lam[q] = st->lam_tab[q];
  __syncthreads();
  unsigned int target = 0;
  for (int it = 0; it < P.chunk; ++it) {
    const bool check = (it == P.chunk - 1);
    const double l = lam[it];
    // --- primal half-step over this block's columns: A^T y, step, projection,
    // reflection, Halpern average (col_pipe_kernel)
    double dx = 0.0, dx0 = 0.0;
    for (int q = threadIdx.x; q < nc; q += blockDim.x) {
      const int64_t j = c0 + q;
      double lb, ub, cj;
      if (DICT) {
        const double* e = cdict + 3 * ccode[q];
        lb = e[0]; ub = e[1]; cj = e[2];
      } else {
        lb = __ldg(Vc.col.a + j); ub = __ldg(Vc.col.b + j); cj = __ldg(Vc.col.c + j);
      }
      const double s = sell_dot_cg<UNIT, 4>(SC, (uint32_t)j, Vc.y);
      const double xj = xs[q], x0 = (double)x0s[q], Dj = (double)Ds[q];
      const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
      Vc.xbar[j] = 2.0 * xt - xj;
      xs[q] = l * ((1.0 + refl) * xt - refl * xj) + (1.0 - l) * x0;
      if (check) {
        Vc.xt[j] = xt;
        const double w = 1.0 / Dj;
        dx += (xt - xj) * (xt - xj) * w;
        dx0 += (xt - x0) * (xt - x0) * w;
      }
    }
    if (check) {
      double a = block_sum(dx, sh);
      if (threadIdx.x == 0) Vc.part[Q_DX * Vc.pstride + blockIdx.x] = a;
      a = block_sum(dx0, sh);
      if (threadIdx.x == 0) Vc.part[Q_DX0 * Vc.pstride + blockIdx.x] = a;
    }
    grid_barrier(P.bar, target);
    // --- dual half-step over this block's rows: A xbar, step, projection,
    // Halpern average (row_step_kernel)
    double dy = 0.0, dy0 = 0.0;
    for (int q = threadIdx.x; q < nr; q += blockDim.x) {
      const int64_t i = r0 + q;
      double lo, hi;
      if (DICT) {
        const double* e = rdict + 2 * rcode[q];
        lo = e[0]; hi = e[1];
      } else {
        lo = __ldg(Vr.row.a + i); hi = __ldg(Vr.row.b + i);
      }
      const double s = sell_dot_cg<UNIT, TECCL_ROW_G>(SR, (uint32_t)i, Vr.xbar);
      const double yi = ys[q], y0 = (double)y0s[q], Ei = (double)Es[q];
      const double se = sigma * Ei;
      const double yt = dual_step(yi, s, se, lo, hi);
      const double yn = l * ((1.0 + refl) * yt - refl * yi) + (1.0 - l) * y0;
      ys[q] = yn;
      Vr.y[i] = yn;
      if (check) {
        Vr.yt[i] = yt;
        const double w = 1.0 / Ei;
        dy += (yt - yi) * (yt - yi) * w;
        dy0 += (yt - y0) * (yt - y0) * w;
      }
    }
    if (check) {
      double a = block_sum(dy, sh);
      if (threadIdx.x == 0) Vr.part[Q_DY * Vr.pstride + blockIdx.x] = a;
      a = block_sum(dy0, sh);
      if (threadIdx.x == 0) Vr.part[Q_DY0 * Vr.pstride + blockIdx.x] = a;
    }
    if (!check) grid_barrier(P.bar, target);  // the launch boundary orders the last one
  }
  for (int q = threadIdx.x; q < nc; q += blockDim.x) Vc.x[c0 + q] = xs[q];
}

// ---------------------------------------------------------------------------
// Matrix-free half-steps for LPs built by teccl_lp_build_te: the same
// updates as col_step / row_step, with A^T y and A x evaluated from the
// topology tables (te_gen.cuh) and the bounds/costs computed in place. No
// index or bound-class stream: HBM traffic is the dense vectors plus the
// gathered operand, whose accesses are coalesced along the epoch axis.
template <bool CHECK>
__global__ void __launch_bounds__(kThreads) col_te_kernel(TeOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const uint32_t j = blockIdx.x * kTile + threadIdx.x;
  double xj = 0.0, x0 = 0.0, Dj = 1.0, lb = 0.0, ub = 0.0, cj = 0.0, s = 0.0;
  if (j < op.n) {
    xj = V.x[j];
    x0 = (double)V.x0[j];
    Dj = (double)V.D[j];
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double tau = st->tau, refl = st->refl;
  if (j < op.n) s = te_col(op, j, V.y, lb, ub, cj);
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  double dx = 0.0, dx0 = 0.0;
  if (j < op.n) {
    const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
    V.xbar[j] = 2.0 * xt - xj;
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      const double w = 1.0 / Dj;
      dx = (xt - xj) * (xt - xj) * w;
      dx0 = (xt - x0) * (xt - x0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
}

// col_te with two adjacent columns per thread: 16-byte loads/stores of the
// dense iterates and two independent gather chains in flight per thread
// (HBM-resident LPs are short of bytes in flight with one column per
// thread: profiles/r01_j_hbm_roofline.md).
// WIDE: the gathered dual vector is far larger than L2 (8m > kL2GatherBytes),
// gathers miss to HBM and latency hiding needs occupancy: 32 registers, 8
// blocks per SM, per-column decode. Otherwise 40 registers and one family
// decode per column pair (te_col2). Measured both ways on the 8- (y 122 MB)
// and 16-chassis (y 1 GB) LPs, profiles/r01_j_hbm_roofline.md.
// Column ranges of a source-partitioned rank (RANGE instantiations): pairs of
// [c0, c1) then of [q0, q1), all four even.
struct ColRange {
  uint32_t c0, c1, q0, q1;
};

template <bool CHECK, bool WIDE, bool RANGE = false>
__global__ void __launch_bounds__(kThreads, WIDE ? TECCL_TE2_MINB : TECCL_TE2_MINB_L2) col_te2_kernel(TeOp op, Vecs V, int j_in_chunk,
                                                                                                      ColRange CR = ColRange{}) {
  __shared__ double sh[32];
  const uint32_t t2 = 2u * (blockIdx.x * kTile + threadIdx.x);
  uint32_t j = t2, jend = op.n;
  if (RANGE) {
    const uint32_t n0 = CR.c1 - CR.c0;
    j = t2 < n0 ? CR.c0 + t2 : CR.q0 + (t2 - n0);
    jend = t2 < n0 ? CR.c1 : CR.q1;
  }
  const bool pair = j + 1 < jend, any = j < jend;
  // unconditional 16/8-byte loads (x, x0, D have a pad slot [n]; threads
  // past the end load pair 0) kept raw until the epilogue, so the thread
  // issues its table lookups and gathers while they are in flight
  const uint32_t jl = any ? j : 0u;
  const double2 xv = *reinterpret_cast<const double2*>(V.x + jl);
  const float2 x0v = *reinterpret_cast<const float2*>(V.x0 + jl);
  const float2 Dv = __ldg(reinterpret_cast<const float2*>(V.D + jl));
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double tau = st->tau, refl = st->refl;
  double s[2] = {0.0, 0.0}, lb[2] = {0.0, 0.0}, ub[2] = {0.0, 0.0}, cj[2] = {0.0, 0.0};
  if (WIDE) {
    if (any) s[0] = te_col(op, j, V.y, lb[0], ub[0], cj[0]);
    if (pair) s[1] = te_col(op, j + 1, V.y, lb[1], ub[1], cj[1]);
  } else if (pair) {
    te_col2(op, j, V.y, s, lb, ub, cj);
  } else if (any) {
    s[0] = te_col(op, j, V.y, lb[0], ub[0], cj[0]);
  }
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  const double xj[2] = {xv.x, xv.y}, x0[2] = {(double)x0v.x, (double)x0v.y};
  const double Dj[2] = {(double)Dv.x, (double)Dv.y};
  double dx = 0.0, dx0 = 0.0, xt[2], xb[2], xn[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    xt[h] = clampd(xj[h] - tau * Dj[h] * (cj[h] - s[h]), lb[h], ub[h]);
    xb[h] = 2.0 * xt[h] - xj[h];
    xn[h] = lam * ((1.0 + refl) * xt[h] - refl * xj[h]) + (1.0 - lam) * x0[h];
    if (CHECK && (h == 0 ? any : pair)) {
      const double w = 1.0 / Dj[h];
      dx += (xt[h] - xj[h]) * (xt[h] - xj[h]) * w;
      dx0 += (xt[h] - x0[h]) * (xt[h] - x0[h]) * w;
    }
  }
  if (pair) {
    *reinterpret_cast<double2*>(V.xbar + j) = make_double2(xb[0], xb[1]);
    *reinterpret_cast<double2*>(V.x + j) = make_double2(xn[0], xn[1]);
    if (CHECK) *reinterpret_cast<double2*>(V.xt + j) = make_double2(xt[0], xt[1]);
  } else if (any) {
    V.xbar[j] = xb[0];
    V.x[j] = xn[0];
    if (CHECK) V.xt[j] = xt[0];
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
}

template <bool CHECK>
__global__ void __launch_bounds__(kThreads) row_te_kernel(TeOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const uint32_t i = blockIdx.x * kTile + threadIdx.x;
  double yi = 0.0, y0 = 0.0, Ei = 1.0, lo = 0.0, hi = 0.0, s = 0.0;
  if (i < op.m) {
    yi = V.y[i];
    y0 = (double)V.y0[i];
    Ei = (double)V.E[i];
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double sigma = st->sigma, refl = st->refl;
  if (i < op.m) s = te_row(op, i, V.xbar, lo, hi);
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  double dy = 0.0, dy0 = 0.0;
  if (i < op.m) {
    const double se = sigma * Ei;
    const double yt = dual_step(yi, s, se, lo, hi);
    V.y[i] = lam * ((1.0 + refl) * yt - refl * yi) + (1.0 - lam) * y0;
    if (CHECK) {
      V.yt[i] = yt;
      const double w = 1.0 / Ei;
      dy = (yt - yi) * (yt - yi) * w;
      dy0 = (yt - y0) * (yt - y0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blockIdx.x] = a;
  }
}

// Matrix-free half-steps of one rank's epoch block (te_gen.cuh em_col /
// em_row): the col_step / row_step updates with A^T y and A x evaluated from
// the topology tables in the epoch-major window, including the fused peer
// exchange of row-partitioned solves (PEER).
template <bool CHECK, bool PEER>
__global__ void __launch_bounds__(kThreads) col_em_kernel(EmOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const uint32_t j = blockIdx.x * kTile + threadIdx.x;
  double xj = 0.0, x0 = 0.0, Dj = 1.0, lb = 0.0, ub = 0.0, cj = 0.0, s = 0.0;
  if (j < op.n) {
    xj = V.x[j];
    x0 = (double)V.x0[j];
    Dj = (double)V.D[j];
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double tau = st->tau, refl = st->refl;
  if (PEER && V.wait.npeer && (done || !block_wait_peers(V.wait, V.st))) return;
  if (j < op.n) s = em_col(op, j, V.y, lb, ub, cj);
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  bool wrote = false;
  double dx = 0.0, dx0 = 0.0;
  if (j < op.n) {
    const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
    const double xb = 2.0 * xt - xj;
    V.xbar[j] = xb;
    wrote = PEER && push_entry<CHECK>(V.push, j, xb, xt);
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      const double w = 1.0 / Dj;
      dx = (xt - xj) * (xt - xj) * w;
      dx0 = (xt - x0) * (xt - x0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
  if (PEER) push_signal(V.push, wrote);
}

template <bool CHECK, bool PEER>
__global__ void __launch_bounds__(kThreads) row_em_kernel(EmOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const uint32_t i = blockIdx.x * kTile + threadIdx.x;
  double yi = 0.0, y0 = 0.0, Ei = 1.0, lo = 0.0, hi = 0.0, s = 0.0;
  if (i < op.m) {
    yi = V.y[i];
    y0 = (double)V.y0[i];
    Ei = (double)V.E[i];
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;  // checked before the first store: the gathers overlap it
  const double sigma = st->sigma, refl = st->refl;
  if (PEER && V.wait.npeer && (done || !block_wait_peers(V.wait, V.st))) return;
  if (i < op.m) s = em_row(op, i, V.xbar, lo, hi);
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  bool wrote = false;
  double dy = 0.0, dy0 = 0.0;
  if (i < op.m) {
    const double se = sigma * Ei;
    const double yt = dual_step(yi, s, se, lo, hi);
    const double yn = lam * ((1.0 + refl) * yt - refl * yi) + (1.0 - lam) * y0;
    V.y[i] = yn;
    wrote = PEER && push_entry<CHECK>(V.push, i, yn, yt);
    if (CHECK) {
      V.yt[i] = yt;
      const double w = 1.0 / Ei;
      dy = (yt - yi) * (yt - yi) * w;
      dy0 = (yt - y0) * (yt - y0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blockIdx.x] = a;
  }
  if (PEER) push_signal(V.push, wrote);
}

// Segment-walking half-steps (te_gen.cuh seg_cols / seg_rows): one warp per
// task of up to 64 consecutive entries of one column / row family, so the
// table lookups are per task and each entry costs only its gathers and the
// PDHG update. Same updates as col_te / row_te.
template <bool CHECK>
__global__ void __launch_bounds__(kThreads) col_seg_kernel(TeOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int4 tk = (wi < op.n_ctask) ? __ldg(op.ctask + wi) : make_int4(0, 0, 0, 0);
  const int cnt = seg_count(tk);
  const uint32_t first = (uint32_t)tk.z;
  double xj[kSegPerLane], x0[kSegPerLane], Dj[kSegPerLane];
#pragma unroll
  for (int h = 0; h < kSegPerLane; ++h) {
    const int i = lane + 32 * h;
    xj[h] = 0.0; x0[h] = 0.0; Dj[h] = 1.0;
    if (i < cnt) {
      xj[h] = V.x[first + i];
      x0[h] = (double)V.x0[first + i];
      Dj[h] = (double)V.D[first + i];
    }
  }
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  const int done = st->done;
  const double tau = st->tau, refl = st->refl;
  double s[kSegPerLane], lb[kSegPerLane], ub[kSegPerLane], cj[kSegPerLane];
  seg_cols(op, tk, lane, V.y, s, lb, ub, cj);
  if (done) return;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  double dx = 0.0, dx0 = 0.0;
#pragma unroll
  for (int h = 0; h < kSegPerLane; ++h) {
    const int i = lane + 32 * h;
    if (i < cnt) {
      const uint32_t j = first + i;
      const double xt = clampd(xj[h] - tau * Dj[h] * (cj[h] - s[h]), lb[h], ub[h]);
      V.xbar[j] = 2.0 * xt - xj[h];
      V.x[j] = lam * ((1.0 + refl) * xt - refl * xj[h]) + (1.0 - lam) * x0[h];
      if (CHECK) {
        V.xt[j] = xt;
        const double w = 1.0 / Dj[h];
        dx += (xt - xj[h]) * (xt - xj[h]) * w;
        dx0 += (xt - x0[h]) * (xt - x0[h]) * w;
      }
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
}

// TECCL_SEG_TMA: each warp stages its task's rows of y, y0 and E in shared
// memory with three 1-D bulk copies (cp.async.bulk, completion on a per-warp
// mbarrier) issued in the prologue, before griddepcontrol.wait -- they are
// final two launches back -- so they stream while the warp gathers x-bar,
// and the epilogue reads shared memory instead of issuing dependent L2 loads
// (it used to L2-prefetch them and load them after the gathers).
#ifndef TECCL_SEG_TMA
#define TECCL_SEG_TMA 1
#endif
#ifndef TECCL_SEG_PF_NEXT
#define TECCL_SEG_PF_NEXT 1
#endif

struct alignas(16) SegStage {  // 16-byte multiple: every warp's stage is a bulk-copy destination
  double y[kSegTask + 2];   // [first & ~1, round_up_even(first + cnt))
  float y0[kSegTask + 4];   // [first & ~3, round_up_4(first + cnt))
  float E[kSegTask + 4];
  unsigned long long bar;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  }
}

template <bool CHECK>
__global__ void __launch_bounds__(kThreads, TECCL_SEG_MINB) row_seg_kernel(TeOp op, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const int w0 = (blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * kSegTPW, lane = threadIdx.x & 31;
  int4 tks[kSegTPW];
#pragma unroll
  for (int t = 0; t < kSegTPW; ++t)
    tks[t] = (w0 + t < op.n_rtask) ? __ldg(op.rtask + w0 + t) : make_int4(0, 0, 0, 0);
#if TECCL_SEG_PF_NEXT
  // the descriptor of the warp that takes this slot a wave later: into L2 now
  // (at the block's start the descriptor load is an HBM miss, 10 % of the stalls)
  {
    constexpr int ahead = TECCL_SEG_PF_NEXT * kSMs * TECCL_SEG_MINB * (kThreads / 32);
    if (lane == 0 && w0 + ahead < op.n_rtask) prefetch_l2(op.rtask + w0 + ahead);
  }
#endif
#if TECCL_SEG_TMA
  static_assert(kSegTPW == 1, "TMA staging is per warp task");
  __shared__ __align__(16) SegStage stage[kThreads / 32];
  SegStage& sg = stage[threadIdx.x >> 5];
  const int cnt0 = seg_count(tks[0]);
  const uint32_t f0 = (uint32_t)tks[0].z;
  const uint32_t a2 = f0 & ~1u, a4 = f0 & ~3u;
  if (lane == 0 && cnt0 > 0) {
    const uint32_t by = ((f0 + cnt0 + 1u) & ~1u) - a2, b4 = ((f0 + cnt0 + 3u) & ~3u) - a4;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&sg.bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&sg.bar)), "r"(8u * by + 8u * b4) : "memory");
    bulk_g2s(sg.y, V.y + a2, 8u * by, &sg.bar);
    bulk_g2s(sg.y0, V.y0 + a4, 4u * b4, &sg.bar);
    bulk_g2s(sg.E, V.E + a4, 4u * b4, &sg.bar);
  }
  __syncwarp();
#else
  // the dense operands are only prefetched into L2 here and loaded after the
  // gathers: held in registers across seg_rows they were spilled at 40
  // registers, and the spill store waited for the HBM load before any
  // gather could issue (lanes past a task's end touch its last row)
#pragma unroll
  for (int t = 0; t < kSegTPW; ++t)
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const uint32_t r = (uint32_t)tks[t].z + (uint32_t)max(0, min(lane + 32 * h, seg_count(tks[t]) - 1));
      prefetch_l2(V.y + r);
      if ((lane & 1) == 0) { prefetch_l2(V.y0 + r); prefetch_l2(V.E + r); }
    }
#endif
  pdl_wait();
  pdl_trigger();
  const PdlpState* st = V.st;
  double dy = 0.0, dy0 = 0.0;
#pragma unroll
  for (int t = 0; t < kSegTPW; ++t) {
    const int4 tk = tks[t];
    const int cnt = seg_count(tk);
    const uint32_t first = (uint32_t)tk.z;
    double s[kSegPerLane], lo[kSegPerLane], hi[kSegPerLane];
    seg_rows(op, tk, lane, V.xbar, s, lo, hi);
#if TECCL_SEG_TMA
    if (cnt > 0) mbar_wait(&sg.bar, 0);  // the staged rows (long since landed, normally);
                                         // also: no bulk copy may outlive the block
#endif
    if (st->done) return;
    const double sigma = st->sigma, refl = st->refl;
    double yi[kSegPerLane], y0[kSegPerLane], Ei[kSegPerLane];
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const uint32_t r = first + (uint32_t)max(0, min(lane + 32 * h, cnt - 1));
#if TECCL_SEG_TMA
      yi[h] = sg.y[r - a2];
      y0[h] = (double)sg.y0[r - a4];
      Ei[h] = (double)sg.E[r - a4];
#else
      yi[h] = V.y[r];
      y0[h] = (double)V.y0[r];
      Ei[h] = (double)V.E[r];
#endif
    }
    const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
        const uint32_t r = first + i;
        const double se = sigma * Ei[h];
        const double yt = dual_step(yi[h], s[h], se, lo[h], hi[h]);
        V.y[r] = lam * ((1.0 + refl) * yt - refl * yi[h]) + (1.0 - lam) * y0[h];
        if (CHECK) {
          V.yt[r] = yt;
          const double w = 1.0 / Ei[h];
          dy += (yt - yi[h]) * (yt - yi[h]) * w;
          dy0 += (yt - y0[h]) * (yt - y0[h]) * w;
        }
      }
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blockIdx.x] = a;
  }
}

// ---------------------------------------------------------------------------
// Source-partitioned solve (SRC): every rank holds the whole single-device TE
// LP (identical, redundant setup) and updates only the columns of its
// sources [s0, s1) and pairs [p0, p1) and the rows that touch nothing else
// (init / conservation / cumulative rows). Commodities couple only through
// the capacity (and buffer-limit) rows: every iteration each rank sums its
// sources' x-bar over every capacity row and stores the partial sums straight
// into every rank's buffer over NVLink (cap_part_kernel), signals, and every
// rank adds the partials in rank order and applies the capacity rows' dual
// step itself (cap_fin_kernel) -- identical on all ranks.
struct OwnMask {
  int on = 0;
  uint32_t s0 = 0, s1 = 0, rc0 = 0, rc1 = 0, rm0 = 0, rm1 = 0;  // init, cons, cum rows
  uint32_t c0 = 0, c1 = 0, q0 = 0, q1 = 0;                        // flow+buffer, Rd/Rc columns
  __device__ __forceinline__ bool row(uint32_t i) const {
    return !on || (i >= s0 && i < s1) || (i >= rc0 && i < rc1) || (i >= rm0 && i < rm1);
  }
  __device__ __forceinline__ bool col(uint32_t j) const {
    return !on || (j >= c0 && j < c1) || (j >= q0 && j < q1);
  }
};

struct SrcX {
  double* const* bufs;   // [world] every rank's partial-sum buffers (own included)
  uint32_t ncap, ncap_e; // capacity + buffer-limit rows; capacity rows (E*K)
  int world, rank;
  uint32_t s0, s1;
  const int4* cap_tasks;
  int n_cap;
  Signal sig;
  Wait wait;
};

// buffer slot of (parity, value/check, writer rank, row)
__device__ __forceinline__ int64_t src_slot(const SrcX& X, int parity, int which, int w, uint32_t r) {
  return ((int64_t)(parity * 2 + which) * X.world + w) * X.ncap + r;
}

// this rank's columns: flows / buffers of its sources, then its pairs' Rd/Rc
template <bool CHECK>
__global__ void __launch_bounds__(kThreads) col_src_kernel(TeOp op, Vecs V, int j_in_chunk, OwnMask M) {
  __shared__ double sh[32];
  const uint32_t t = blockIdx.x * kTile + threadIdx.x;
  const uint32_t n0 = M.c1 - M.c0, n1 = M.q1 - M.q0;
  const bool on = t < n0 + n1;
  const uint32_t j = t < n0 ? M.c0 + t : M.q0 + (t - n0);
  double xj = 0.0, x0 = 0.0, Dj = 1.0, lb = 0.0, ub = 0.0, cj = 0.0, s = 0.0;
  if (on) {
    xj = V.x[j];
    x0 = (double)V.x0[j];
    Dj = (double)V.D[j];
  }
  const PdlpState* st = V.st;
  if (st->done) return;
  const double tau = st->tau, refl = st->refl;
  const double lam = st->lam_tab[j_in_chunk];  // chunks are at most kLamTab iterations
  if (on) s = te_col(op, j, V.y, lb, ub, cj);
  double dx = 0.0, dx0 = 0.0;
  if (on) {
    const double xt = clampd(xj - tau * Dj * (cj - s), lb, ub);
    V.xbar[j] = 2.0 * xt - xj;
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      const double w = 1.0 / Dj;
      dx = (xt - xj) * (xt - xj) * w;
      dx0 = (xt - x0) * (xt - x0) * w;
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
}

// Partial capacity / buffer-limit row sums over this rank's sources, stored
// into every rank's buffer (peer memory); the last block signals the peers.
template <bool CHECK>
__global__ void __launch_bounds__(kThreads) cap_part_kernel(TeOp op, Vecs V, SrcX X, int parity) {
  if (V.st->done) return;
  const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  bool wrote = false;
  if (wi < X.n_cap) {
    const int4 tk = __ldg(X.cap_tasks + wi);
    const int kind = tk.x & 15, Bv = tk.y, off = tk.w & 0xffffff, cnt = seg_count(tk);
    const uint32_t K = op.K;
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i >= cnt) continue;
      uint32_t r, co;  // buffer row, column offset inside a source block
      if (kind == SEG_CAP) { r = (uint32_t)Bv * K + off + i; co = r; }
      else { const uint32_t qb = (uint32_t)Bv * (K + 1) + off + i; r = X.ncap_e + qb; co = op.EK + qb; }
      double a = 0.0, c = 0.0;
      for (uint32_t s = X.s0; s < X.s1; ++s) {
        a += __ldg(V.xbar + (size_t)s * op.SB + co);
        if (CHECK) c += __ldg(V.xt + (size_t)s * op.SB + co);
      }
      for (int w = 0; w < X.world; ++w) {
        X.bufs[w][src_slot(X, parity, 0, X.rank, r)] = a;
        if (CHECK) X.bufs[w][src_slot(X, parity, 1, X.rank, r)] = c;
      }
      wrote = true;
    }
  }
  if (wrote) __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(X.sig.arrive, 1u);
    if (prev == gridDim.x - 1) {
      *X.sig.arrive = 0u;
      signal_peers(X.sig);
    }
  }
}

// Sum the partials in rank order and take the capacity rows' dual step (every
// rank, identical); on check iterations also their KKT terms at (A xt, yt).
// Block partials go to slot blk_off + blockIdx.x; rank 0 alone contributes.
template <bool CHECK>
__global__ void __launch_bounds__(kThreads) cap_fin_kernel(TeOp op, Vecs V, SrcX X, int parity,
                                                           int j_in_chunk, int blk_off) {
  __shared__ double sh[32];
  if (V.st->done) return;
  if (!block_wait_peers(X.wait, V.st)) return;
  const PdlpState* st = V.st;
  const double sigma = st->sigma, refl = st->refl;
  const double lam = st->lam_tab[j_in_chunk];
  const uint32_t r = blockIdx.x * kTile + threadIdx.x;
  double dy = 0.0, dy0 = 0.0, rp = 0.0, dobj = 0.0;
  if (r < X.ncap) {
    const double* b = X.bufs[X.rank];
    double a = 0.0;
    for (int w = 0; w < X.world; ++w) a += b[src_slot(X, parity, 0, w, r)];
    const bool cap = r < X.ncap_e;
    const uint32_t i = cap ? op.S + r : op.R_bcap + (r - X.ncap_e);
    const double lo = -INFINITY, hi = cap ? __ldg(op.d.ecap + r) : op.d.blimit;
    const double yi = V.y[i], y0 = (double)V.y0[i], Ei = (double)V.E[i];
    const double yt = dual_step(yi, a, sigma * Ei, lo, hi);
    V.y[i] = lam * ((1.0 + refl) * yt - refl * yi) + (1.0 - lam) * y0;
    if (CHECK) {
      V.yt[i] = yt;
      if (X.rank == 0) {
        const double w = 1.0 / Ei;
        dy = (yt - yi) * (yt - yi) * w;
        dy0 = (yt - y0) * (yt - y0) * w;
        double as = 0.0;
        for (int q = 0; q < X.world; ++q) as += b[src_slot(X, parity, 1, q, r)];
        const double res = as - clampd(as, lo, hi);
        rp = res * res;
        if (yt < 0.0 && isfinite(hi)) dobj = hi * yt;
      }
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blk_off + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blk_off + blockIdx.x] = a;
    a = block_sum(rp, sh);
    if (threadIdx.x == 0) V.part[Q_RP * V.pstride + blk_off + blockIdx.x] = a;
    a = block_sum(dobj, sh);
    if (threadIdx.x == 0) V.part[Q_DOBJ_ROW * V.pstride + blk_off + blockIdx.x] = a;
  }
}

// KKT over rows at T(z) = (xt, yt): primal residual of A.xt against the row
// bounds and the row part of the dual objective.
template <bool UNIT, int OPK>  // operator: 0 stored SELL, 1 TeOp, 2 EmOp
__global__ void __launch_bounds__(kThreads) kkt_row_kernel(int32_t m, SellView S, TeOp op, EmOp em, Vecs V,
                                                           OwnMask M) {
  __shared__ double sh[32];
  if (V.st->done) return;
  const int64_t i0 = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const int64_t i = (i0 < m && M.row((uint32_t)i0)) ? i0 : m;  // rows of other ranks / capacity rows: skipped
  double lo = 0.0, hi = 0.0, s = 0.0;
  if (i < m) {
    if (OPK == 1) {
      s = te_row(op, (uint32_t)i, V.xt, lo, hi);
    } else if (OPK == 2) {
      s = em_row(em, (uint32_t)i, V.xt, lo, hi);
    } else {
      s = sell_dot<UNIT, 8>(S, i, V.xt);
      lo = V.lo_u[i];
      hi = V.hi_u[i];
    }
  }
  double rp = 0.0, dobj = 0.0;
  if (i < m) {
    const double r = s - clampd(s, lo, hi);
    rp = r * r;
    const double yu = V.yt[i];
    if (yu > 0.0 && isfinite(lo)) dobj = lo * yu;
    else if (yu < 0.0 && isfinite(hi)) dobj = hi * yu;
  }
  double a = block_sum(rp, sh);
  if (threadIdx.x == 0) V.part[Q_RP * V.pstride + blockIdx.x] = a;
  a = block_sum(dobj, sh);
  if (threadIdx.x == 0) V.part[Q_DOBJ_ROW * V.pstride + blockIdx.x] = a;
}

// KKT over columns: reduced costs, dual residual, primal objective and the
// bound part of the dual objective.
template <bool UNIT, int OPK>
__global__ void __launch_bounds__(kThreads) kkt_col_kernel(int32_t n, SellView S, TeOp op, EmOp em, Vecs V,
                                                           OwnMask M) {
  __shared__ double sh[32];
  if (V.st->done) return;
  const int64_t j0 = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const int64_t j = (j0 < n && M.col((uint32_t)j0)) ? j0 : n;  // columns of other ranks: skipped
  double lb = 0.0, ub = 0.0, cj = 0.0, s = 0.0;
  if (j < n) {
    if (OPK == 1) {
      s = te_col(op, (uint32_t)j, V.yt, lb, ub, cj);
    } else if (OPK == 2) {
      s = em_col(em, (uint32_t)j, V.yt, lb, ub, cj);
    } else {
      s = sell_dot<UNIT>(S, j, V.yt);
      cj = V.c_u[j];
      lb = V.lb_u[j];
      ub = V.ub_u[j];
    }
  }
  double rd = 0.0, pobj = 0.0, dobj = 0.0;
  if (j < n) {
    const double g = cj - s;
    double lamb = 0.0;
    if (g > 0.0 && isfinite(lb)) lamb = g;
    else if (g < 0.0 && isfinite(ub)) lamb = g;
    const double r = g - lamb;
    rd = r * r;
    pobj = cj * V.xt[j];
    if (lamb > 0.0) dobj = lamb * lb;
    else if (lamb < 0.0) dobj = lamb * ub;
  }
  double a = block_sum(rd, sh);
  if (threadIdx.x == 0) V.part[Q_RD * V.pstride + blockIdx.x] = a;
  a = block_sum(pobj, sh);
  if (threadIdx.x == 0) V.part[Q_POBJ * V.pstride + blockIdx.x] = a;
  a = block_sum(dobj, sh);
  if (threadIdx.x == 0) V.part[Q_DOBJ_COL * V.pstride + blockIdx.x] = a;
}

// ---------------------------------------------------------------------------
// Primal infeasibility (the reference's "infeasible" status, solver.py:133-135).
// When the LP has no feasible point, PDHG's dual iterate drifts along a ray
// v (the infimal displacement of the iteration); every `infeas_every` checks
// the change of the dual iterate since the previous evaluation, v = yt - yprev,
// is tested as a Farkas certificate. For every feasible x (r = A x):
//   v.r >= sum_i (v_i > 0 ? v_i lo_i : v_i hi_i)         (rows, implied bounds)
//   v.r  = (A^T v).x <= sum_j (g_j > 0 ? g_j ub_j : g_j lb_j),  g = A^T v
// so C(v) = row part - column part > 0 proves that no feasible x exists. The
// bounds are the implied ones (implied_*_kernel: valid for every feasible x,
// finite where the declared bound is not -- F <= capacity, B <= the source's
// demand, row activity ranges), so a noisy ray still gives a finite value.
// The solve stops once C(v) > eps_infeas * (sum of |terms|): rounding in the
// fp64 sums is ~1e-16 of that magnitude, so the margin cannot be met by
// accident. C(v) is the ray's dual objective (kkt_*_kernel's with c = 0).
template <int OPK>
__global__ void __launch_bounds__(kThreads) infeas_row_kernel(int32_t m, Vecs V, const double* __restrict__ loI,
                                                              const double* __restrict__ hiI,
                                                              double* __restrict__ yprev,
                                                              double* __restrict__ dv) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done || !st->infeas_due) return;
  const int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  double c = 0.0, mag = 0.0, ninf = 0.0;
  if (i < m) {
    const double yt = V.yt[i];
    const double v = yt - yprev[i];
    yprev[i] = yt;
    dv[i] = v;
    const double b = v > 0.0 ? loI[i] : hiI[i];
    if (v != 0.0) {
      if (isfinite(b)) { c = v * b; mag = fabs(c); }
      else ninf = 1.0;
    }
  }
  double a = block_sum(c, sh);
  if (threadIdx.x == 0) V.part[Q_IC_ROW * V.pstride + blockIdx.x] = a;
  a = block_sum(mag, sh);
  if (threadIdx.x == 0) V.part[Q_IM_ROW * V.pstride + blockIdx.x] = a;
  a = block_sum(ninf, sh);
  if (threadIdx.x == 0) V.part[Q_IN_ROW * V.pstride + blockIdx.x] = a;
}

template <bool UNIT, int OPK>
__global__ void __launch_bounds__(kThreads) infeas_col_kernel(int32_t n, SellView S, TeOp op, Vecs V,
                                                              const double* __restrict__ ubI,
                                                              const double* __restrict__ dv) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done || !st->infeas_due) return;
  const int64_t j = (int64_t)blockIdx.x * kTile + threadIdx.x;
  double c = 0.0, mag = 0.0, ninf = 0.0;
  if (j < n) {
    double g;
    if (OPK == 1) {
      double lb_, ub_, c_;
      g = te_col(op, (uint32_t)j, dv, lb_, ub_, c_);
    } else {
      g = sell_dot<UNIT>(S, (uint32_t)j, dv);
    }
    const double b = g > 0.0 ? ubI[j] : V.lb_u[j];
    if (g != 0.0) {
      if (isfinite(b)) { c = -g * b; mag = fabs(c); }
      else ninf = 1.0;
    }
  }
  double a = block_sum(c, sh);
  if (threadIdx.x == 0) V.part[Q_IC_COL * V.pstride + blockIdx.x] = a;
  a = block_sum(mag, sh);
  if (threadIdx.x == 0) V.part[Q_IM_COL * V.pstride + blockIdx.x] = a;
  a = block_sum(ninf, sh);
  if (threadIdx.x == 0) V.part[Q_IN_COL * V.pstride + blockIdx.x] = a;
}

// Implied column upper bounds (setup): the declared ones, and for the
// time-expanded LP's flows and buffers, which the LP leaves unbounded above
// (lp.py:47-59), what every feasible point satisfies anyway: a flow
// F(s,e,k) <= min(capacity(e,k), demand of s) (capacity row lp.py:74-77, all
// flows >= 0) and a buffer B(s,g,k) <= demand of s (the source's units are
// conserved, lp.py:67-116, every term >= 0).
__global__ void implied_col_kernel(int64_t n, const double* __restrict__ ub, TeDev d, int te,
                                   double* __restrict__ ubI) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double u = ub[j];
    if (te && j < (int64_t)d.S * d.SB) {
      const int64_t s = j / d.SB, r = j - s * d.SB;
      double t = d.out_units[s];
      if (r < (int64_t)d.E * d.K) t = fmin(t, d.ecap[r]);  // r = e*K + k, the capacity row's index
      u = fmin(u, t);
    }
    ubI[j] = u;
  }
}

// Implied row ranges (setup): [lo, hi] intersected with the activity range of
// the row over the column box [lb, ubI] (e.g. a capacity row's sum of flows
// is >= 0).
template <bool UNIT>
__global__ void implied_row_kernel(int64_t m, const int64_t* __restrict__ ptr, const uint32_t* __restrict__ idx,
                                   const double* __restrict__ val, const double* __restrict__ lb,
                                   const double* __restrict__ ubI, const double* __restrict__ lo,
                                   const double* __restrict__ hi, double* __restrict__ loI,
                                   double* __restrict__ hiI) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double amin = 0.0, amax = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) {
      const uint32_t t = idx[p];
      const uint32_t j = UNIT ? (t & kIdxMask) : t;
      const double a = UNIT ? ((t & kSignBit) ? -1.0 : 1.0) : val[p];
      const double l = lb[j], u = ubI[j];
      if (a > 0.0) { amin += a * l; amax += a * u; }
      else if (a < 0.0) { amin += a * u; amax += a * l; }
    }
    // (a * inf sums to +-inf; an inf - inf NaN leaves the declared bound)
    loI[r] = amin > lo[r] ? amin : lo[r];
    hiI[r] = amax < hi[r] ? amax : hi[r];
  }
}

// Sum every rank's reduced partials in rank order (identical on all ranks, so
// all ranks take the same decisions), evaluate termination, decide restarts
// and update the primal weight. All of PDLP's control flow.
__device__ void control_decide(Vecs V) {
  PdlpState* st = V.st;
  double q[kNQ];
  for (int k = 0; k < kNQ; ++k) {
    double a = 0.0;
    for (int r = 0; r < V.world; ++r) a += V.slots[r * kSlots + k];  // rank order: same on all ranks
    q[k] = a;
  }
  const double w = st->omega;
  const double r = sqrt(w * q[Q_DX] + q[Q_DY] / w);
  const double pobj = q[Q_POBJ];
  const double dobj = q[Q_DOBJ_ROW] + q[Q_DOBJ_COL];
  st->rel_p = sqrt(q[Q_RP]) / (1.0 + st->bnorm);
  st->rel_d = sqrt(q[Q_RD]) / (1.0 + st->cnorm);
  // relative duality gap in the usual sense: |p - d| / max(1, |p|, |d|)
  st->gap = fabs(pobj - dobj) / fmax(1.0, fmax(fabs(pobj), fabs(dobj)));
  st->pobj = pobj;
  st->dobj = dobj;
  st->last_r = r;
  st->total += st->chunk_len;
  st->k_inner += st->chunk_len;
  st->restart = 0;
  if (!isfinite(r) || !isfinite(pobj)) { st->done = 2; return; }
  if (st->rel_p <= st->eps_res && st->rel_d <= st->eps_res && st->gap <= st->eps) {
    st->done = 1;
    return;
  }
  if (st->infeas_due) {  // this chunk's certificate evaluation (infeas_*_kernel)
    const double cv = q[Q_IC_ROW] + q[Q_IC_COL], mag = q[Q_IM_ROW] + q[Q_IM_COL];
    st->cert = mag > 0.0 ? cv / mag : 0.0;
    if (q[Q_IN_ROW] + q[Q_IN_COL] == 0.0 && mag > 0.0 && cv > st->eps_infeas * mag) {
      st->done = 5;
      return;
    }
  }
  if (!st->have_r0) {
    st->r0 = r;
    st->have_r0 = 1;
    st->rprev = r;
  }
  const bool sufficient = r <= st->rs_suff * st->r0;
  const bool necessary = r <= st->rs_nec * st->r0 && r > st->rprev;
  const bool artificial = (double)st->k_inner >= st->rs_art * (double)st->total;
  st->rprev = r;
  if (sufficient || necessary || artificial) {
    st->restart = 1;
    st->restarts += 1;
    st->k_inner = 0;
    st->have_r0 = 0;
    const double dxr = sqrt(q[Q_DX0]), dyr = sqrt(q[Q_DY0]);
    if (dxr > 1e-10 && dyr > 1e-10) {
      // PID on the log primal-weight error e = log(dy/dx) - log(w); with
      // ki = kd = 0 this is PDLP's exponential smoothing with weight theta
      const double e = log(dyr / dxr) + st->bias - log(w);
      st->e_int += e;
      const double de = e - st->e_prev;
      st->e_prev = e;
      st->omega = exp(log(w) + st->theta * e + st->ki * st->e_int + st->kd * de);
      st->tau = st->eta / st->omega;
      st->sigma = st->eta * st->omega;
    }
  }
}

__global__ void control_kernel(Vecs V) {
  PdlpState* st = V.st;
  if (st->done) return;
  if (threadIdx.x == 0) {
    control_decide(V);
    // certificate evaluation in the next chunk? (every infeas_every checks)
    const long long c = st->chunk_len > 0 ? st->total / st->chunk_len : 0;
    st->infeas_due = (st->eps_infeas > 0.0 && st->infeas_every > 0 && (c + 1) % st->infeas_every == 0) ? 1 : 0;
  }
  __syncwarp();
  // Halpern weights of the next chunk's iterations
  const long long k0 = st->k_inner;
  for (int j = threadIdx.x; j < kLamTab; j += 32) {
    const double kk = (double)(k0 + j);
    st->lam_tab[j] = (kk + 1.0) / (kk + 2.0);
  }
}

// Restart: z <- z0 <- T(z).
__global__ void restart_x_kernel(int32_t n, Vecs V) {
  if (V.st->done || !V.st->restart) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double xt = V.xt[j];
    V.x[j] = xt;
    V.x0[j] = (float)xt;
  }
}
// Rows: y <- yt over the whole gather window (ghost entries hold the
// neighbours' yt, which is their new y), y0 <- yt over the owned rows.
__global__ void restart_y_kernel(int64_t win, int64_t off, int32_t m, double* __restrict__ y_win,
                                 const double* __restrict__ yt_win, float* __restrict__ y0,
                                 const PdlpState* st) {
  if (st->done || !st->restart) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < win;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yt = yt_win[i];
    y_win[i] = yt;
    const int64_t o = i - off;
    if (o >= 0 && o < m) y0[o] = (float)yt;
  }
}

// ---------------------------------------------------------------------------
// Setup kernels: equilibration statistics, norms, power iteration.

// stat[r] = max (MAX) or sum of |a_rj| * other_j over the row/column, times self_r
template <bool UNIT, bool MAX>
__global__ void abs_stat_kernel(int64_t count, const int64_t* __restrict__ ptr,
                                const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                const double* __restrict__ other, const double* __restrict__ self,
                                double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) {
      const uint32_t t = idx[p];
      const double a = UNIT ? 1.0 : fabs(val[p]);
      const double v = a * other[UNIT ? (t & kIdxMask) : t];
      acc = MAX ? fmax(acc, v) : acc + v;
    }
    out[r] = acc * self[r];
  }
}

__global__ void apply_scale_kernel(int64_t count, double* __restrict__ s,
                                   const double* __restrict__ stat) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = stat[r];
    if (v > 0.0) s[r] /= sqrt(v);
  }
}

__global__ void fill_kernel(int64_t count, double* p, double v) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    p[r] = v;
}

// D = fp32(s^2), root = sqrt(D) (the exact preconditioner the solver uses)
__global__ void precond_kernel(int64_t count, const double* __restrict__ s, float* __restrict__ D,
                               double* __restrict__ root) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    float d = (float)(s[r] * s[r]);
    if (!(d > 0.0f) || !isfinite(d)) d = 1.0f;
    D[r] = d;
    root[r] = sqrt((double)d);
  }
}

__device__ __forceinline__ double bound_ref(double lo, double hi) {
  if (isfinite(hi)) return hi;
  if (isfinite(lo)) return lo;
  return 0.0;
}

// Norm partials: ||s.c||^2 and ||c||^2 over columns, ||s.b||^2 and ||b||^2 over rows.
__global__ void norms_kernel(int64_t count, const double* __restrict__ s, const double* __restrict__ a,
                             const double* __restrict__ b, int is_row, double* part_s,
                             double* part_u) {
  __shared__ double sh[32];
  double ss = 0.0, su = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = is_row ? bound_ref(a[r], b[r]) : a[r];
    ss += (v * s[r]) * (v * s[r]);
    su += v * v;
  }
  double t = block_sum(ss, sh);
  if (threadIdx.x == 0) part_s[blockIdx.x] = t;
  t = block_sum(su, sh);
  if (threadIdx.x == 0) part_u[blockIdx.x] = t;
}

__global__ void sumsq_kernel(int64_t count, const double* v, double* part) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    a += v[r] * v[r];
  a = block_sum(a, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}

// scal[0] = sum of partials (fixed order), scal[1] = 1/sqrt(scal[0])
__global__ void __launch_bounds__(1024) finalize_norm_kernel(const double* part, int nb, double* scal) {
  __shared__ double sh[32];
  double a = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[b];
  a = block_sum(a, sh);
  if (threadIdx.x == 0) {
    scal[0] = a;
    scal[1] = a > 0.0 ? 1.0 / sqrt(a) : 0.0;
  }
}

__global__ void scale_by_kernel(int64_t count, double* v, const double* scal) {
  const double s = scal[1];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] *= s;
}

__global__ void scale_inplace_kernel(int64_t count, double* v, double s) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] *= s;
}

__global__ void mul_kernel(int64_t count, double* __restrict__ out, const double* __restrict__ a,
                           const double* __restrict__ b) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    out[r] = a[r] * b[r];
}

// out_r = self_r * sum_j a_rj * in_j  (CSR/CSC, thread per row)
template <bool UNIT>
__global__ void spmv_scaled_kernel(int64_t count, const int64_t* __restrict__ ptr,
                                   const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                   const double* __restrict__ in, const double* __restrict__ self,
                                   double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t p = ptr[r]; p < ptr[r + 1]; ++p) {
      const uint32_t t = idx[p];
      if (UNIT) {
        const double xv = in[t & kIdxMask];
        acc += (t & kSignBit) ? -xv : xv;
      } else {
        acc += val[p] * in[t];
      }
    }
    out[r] = self ? self[r] * acc : acc;
  }
}

__global__ void init_iterates_kernel(int32_t n, int32_t m, Vecs V, int warm,
                                     const double* __restrict__ xin, const double* __restrict__ yin) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double x0 = clampd(warm ? xin[j] : 0.0, V.lb_u[j], V.ub_u[j]);
    V.x[j] = x0;
    V.x0[j] = (float)x0;
    V.xt[j] = x0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y0 = warm ? yin[i] : 0.0;
    V.y[i] = y0;
    V.y0[i] = (float)y0;
    V.yt[i] = y0;
  }
}

__global__ void output_kernel(int32_t n, int32_t m, Vecs V, double* xo, double* yo) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    xo[j] = V.xt[j];
  if (yo)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
      yo[i] = V.yt[i];
}

__global__ void hash_fill_kernel(int64_t count, double* v) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)r * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    v[r] = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
  }
}

// ---------------------------------------------------------------------------
// Row-partitioned solves: the peer-memory arena of one rank and its view of
// the other ranks' arenas (CUDA IPC handles exchanged by the host).
enum ArrayId { A_XBAR = 0, A_XT, A_CW, A_Y, A_YT, A_RW, A_NARR };
enum MetaId {
  M_NCW = 0, M_NRW, M_OFF0,  // M_OFF0 .. M_OFF0+A_NARR-1: array byte offsets
  M_FLAGS = M_OFF0 + A_NARR, M_SLOTS, M_SEQ, M_ARRIVE,
  M_OC0, M_OC1, M_OR0, M_OR1, M_WC0, M_WC1, M_WR0, M_WR1, M_RANK, M_WORLD, M_COUNT
};
constexpr int kMetaLen = 32;
constexpr int kBlobLen = (int)sizeof(cudaIpcMemHandle_t) + kMetaLen * 8;

struct DistState {
  int world = 1, rank = 0, device = 0;
  bool connected = false;
  char* arena = nullptr;
  int64_t meta[kMetaLen] = {0};
  std::vector<std::array<int64_t, kMetaLen>> peer_meta;
  std::vector<char*> peer_base;      // nullptr for self
  double** d_peer_slots = nullptr;   // device array: slot tables of all peers (rank order, self skipped)
  Signal sig_nbr{}, sig_all{};
  Wait wait_nbr{}, wait_all{};

  double* arr(int id) const { return (double*)(arena + meta[M_OFF0 + id]); }
  double* slots() const { return (double*)(arena + meta[M_SLOTS]); }
  bool is_col(int id) const { return id == A_XBAR || id == A_XT || id == A_CW; }
  void range(int q, int id, int64_t& o0, int64_t& o1, int64_t& w0, int64_t& w1) const {
    const int64_t* mt = (q == rank) ? meta : peer_meta[q].data();
    if (is_col(id)) { o0 = mt[M_OC0]; o1 = mt[M_OC1]; w0 = mt[M_WC0]; w1 = mt[M_WC1]; }
    else { o0 = mt[M_OR0]; o1 = mt[M_OR1]; w0 = mt[M_WR0]; w1 = mt[M_WR1]; }
  }
  Halo halo_plan(std::initializer_list<int> ids) const {
    Halo H{};
    for (int id : ids)
      for (int q : {rank - 1, rank + 1}) {
        if (q < 0 || q >= world || H.n >= 2 * kMaxPeers) continue;
        int64_t o0, o1, w0, w1, qo0, qo1, qw0, qw1;
        range(rank, id, o0, o1, w0, w1);
        range(q, id, qo0, qo1, qw0, qw1);
        const int64_t a = std::max(o0, qw0), b = std::min(o1, qw1);
        if (b <= a) continue;
        H.src[H.n] = arr(id) + (a - w0);
        H.dst[H.n] = (double*)(peer_base[q] + peer_meta[q][M_OFF0 + id]) + (a - qw0);
        H.cnt[H.n] = b - a;
        ++H.n;
      }
    return H;
  }
  // fused-halo plan of a half-step kernel: value array idv, check array idc
  Push push_plan(int idv, int idc) const {
    Push P{};
    for (int q : {rank - 1, rank + 1}) {
      if (q < 0 || q >= world || P.n >= 2) continue;
      int64_t o0, o1, w0, w1, qo0, qo1, qw0, qw1;
      range(rank, idv, o0, o1, w0, w1);
      range(q, idv, qo0, qo1, qw0, qw1);
      const int64_t a = std::max(o0, qw0), b = std::min(o1, qw1);
      if (b <= a) continue;
      P.lo[P.n] = a - o0;
      P.hi[P.n] = b - o0;
      P.dv[P.n] = (double*)(peer_base[q] + peer_meta[q][M_OFF0 + idv]) + (a - qw0);
      P.dc[P.n] = (double*)(peer_base[q] + peer_meta[q][M_OFF0 + idc]) + (a - qw0);
      ++P.n;
    }
    P.sig = sig_nbr;
    return P;
  }
  int64_t halo_max(std::initializer_list<int> ids) const {
    Halo H = halo_plan(ids);
    int64_t mx = 1;
    for (int i = 0; i < H.n; ++i) mx = std::max(mx, H.cnt[i]);
    return mx;
  }
  ~DistState() {
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (char* b : peer_base)
      if (b) cudaIpcCloseMemHandle(b);
    if (d_peer_slots) cudaFree(d_peer_slots);
    if (arena) cudaFree(arena);
  }
};

void free_dist(void* d) { delete (DistState*)d; }

// ---------------------------------------------------------------------------
// Host orchestration.

// Solver workspace, created on the first solve of an LP and reused by every
// later solve of it: device buffers, the captured chunk graph (its kernel
// arguments point into these buffers) and the pinned state ring.
struct Workspace {
  std::vector<void*> bufs;
  int device = 0;
  cudaStream_t st = nullptr;      // allocations come from the stream-ordered pool
  double *R = nullptr, *C = nullptr, *rstat = nullptr, *cstat = nullptr;
  float *D = nullptr, *E = nullptr, *x0 = nullptr, *y0 = nullptr;
  double *x = nullptr, *xt = nullptr, *xbar = nullptr, *y = nullptr, *yt = nullptr;
  double *part = nullptr, *part2 = nullptr, *slots = nullptr;
  // infeasibility certificate: implied bounds (set up once per LP), previous
  // dual iterate and the ray candidate (pad slot [m] = 0 for SELL gathers)
  double *ubI = nullptr, *loI = nullptr, *hiI = nullptr, *yprev = nullptr, *dv = nullptr;
  PdlpState* dst = nullptr;
  unsigned int* bar = nullptr;    // grid-barrier counter of the persistent chunk kernel
  int64_t pstride = 0;
  cudaGraphExec_t gexec = nullptr;
  int graph_chunk = 0;  // key of the captured graph: chunk length and kernel variant
  PdlpState* ring = nullptr;
  int ring_len = 0;
  std::vector<cudaEvent_t> evs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ~Workspace() {
    cudaSetDevice(device);
    cudaStreamSynchronize(st);  // every use of the workspace was on st
    for (void* p : bufs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    std::lock_guard<std::mutex> lock(device_mutex());
    if (gexec) cudaGraphExecDestroy(gexec);
    if (ring) cudaFreeHost(ring);
    for (auto e : evs) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
  template <typename T>
  T* alloc(int64_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (size_t)(count > 0 ? count : 1) * sizeof(T), st) != cudaSuccess)
      return nullptr;
    bufs.push_back(p);
    return (T*)p;
  }
};

void free_workspace(void* w) { delete (Workspace*)w; }

int read_partials(double* dpart, int count, cudaStream_t st, double* out) {
  std::vector<double> h(count);
  TECCL_CUDA(cudaMemcpyAsync(h.data(), dpart, count * sizeof(double), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  double a = 0.0;
  for (double x : h) a += x;
  *out = a;
  return TECCL_OK;
}

SellView row_view(const teccl_lp* lp) {
  return SellView{lp->srow_off, lp->srow_w, lp->srow_idx, lp->srow_val, lp->m};
}
SellView col_view(const teccl_lp* lp) {
  return SellView{lp->scol_off, lp->scol_w, lp->scol_idx, lp->scol_val, lp->n};
}

// blocks of the pipelined column kernel: every SM full, one pass
int pipe_blocks() {
  static int blocks = 0;
  if (!blocks) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, col_pipe_kernel<true, true, false, false>, kThreads, 0);
    blocks = kSMs * (occ > 0 ? occ : 4);
  }
  return blocks;
}

// Launch an iteration kernel, with programmatic stream serialization (PDL)
// when `pdl` is set.
template <typename... KArgs, typename... Args>
void launch_iter(bool pdl, void (*k)(KArgs...), int grid, cudaStream_t st, Args... args) {
  if (!pdl) {
    k<<<grid, kThreads, 0, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

template <bool UNIT, bool DICT, bool CHECK, bool PEER>
void launch_col_t(cudaStream_t st, const teccl_lp* lp, const Vecs& V, int j) {
  const bool pdl = V.pdl != 0;
  if (V.col_pipe) {
    const int blocks = std::min<int>(pipe_blocks(), V.nb_col);
    launch_iter(pdl, col_pipe_kernel<UNIT, DICT, CHECK, PEER>, blocks, st, (int32_t)lp->n, col_view(lp), V, j);
  } else {
    launch_iter(pdl, col_step_kernel<UNIT, DICT, CHECK, PEER>, V.nb_col, st, (int32_t)lp->n, col_view(lp), V, j);
  }
}
template <bool UNIT, bool DICT, bool CHECK>
void launch_col(cudaStream_t st, const teccl_lp* lp, const TeOp* te, const EmOp* em, const Vecs& V, int j) {
  const bool pdl = V.pdl != 0;
  if (em) {
    const int g = (int)((em->n + kTile - 1) / kTile);
    if (V.push.n || V.wait.npeer) launch_iter(pdl, col_em_kernel<CHECK, true>, g, st, *em, V, j);
    else launch_iter(pdl, col_em_kernel<CHECK, false>, g, st, *em, V, j);
  } else if (te && (V.seg & 1)) {
    launch_iter(pdl, col_seg_kernel<CHECK>, (te->n_ctask + 7) / 8, st, *te, V, j);
  } else if (te && V.col_pipe) {  // col_pipeline selects the two-column variants
    const int g = (int)((te->n + 2 * kTile - 1) / (2 * kTile));
    if (8.0 * te->m > kL2GatherBytes) launch_iter(pdl, col_te2_kernel<CHECK, true>, g, st, *te, V, j, ColRange{});
    else launch_iter(pdl, col_te2_kernel<CHECK, false>, g, st, *te, V, j, ColRange{});
  } else if (te) {
    launch_iter(pdl, col_te_kernel<CHECK>, (int)((te->n + kTile - 1) / kTile), st, *te, V, j);
  } else if (V.push.n || V.wait.npeer) {  // fused peer exchange compiled in only where used
    launch_col_t<UNIT, DICT, CHECK, true>(st, lp, V, j);
  } else {
    launch_col_t<UNIT, DICT, CHECK, false>(st, lp, V, j);
  }
}
template <bool UNIT, bool DICT, bool CHECK>
void launch_row(cudaStream_t st, const teccl_lp* lp, const TeOp* te, const EmOp* em, const Vecs& V, int j) {
  const bool pdl = V.pdl != 0;
  if (em) {
    const int g = (int)((em->m + kTile - 1) / kTile);
    if (V.push.n || V.wait.npeer) launch_iter(pdl, row_em_kernel<CHECK, true>, g, st, *em, V, j);
    else launch_iter(pdl, row_em_kernel<CHECK, false>, g, st, *em, V, j);
  } else if (te && (V.seg & 2)) launch_iter(pdl, row_seg_kernel<CHECK>, (te->n_rtask + 8 * kSegTPW - 1) / (8 * kSegTPW), st, *te, V, j);
  else if (te) launch_iter(pdl, row_te_kernel<CHECK>, (int)((te->m + kTile - 1) / kTile), st, *te, V, j);
  else if (V.push.n || V.wait.npeer)
    launch_iter(pdl, row_step_kernel<UNIT, DICT, CHECK, true>, V.nb_row, st, (int32_t)lp->m, row_view(lp), V, j);
  else
    launch_iter(pdl, row_step_kernel<UNIT, DICT, CHECK, false>, V.nb_row, st, (int32_t)lp->m, row_view(lp), V, j);
}

// Exchange state of a source-partitioned solve (see cap_part_kernel).
// Arena: partial buffers [2 parities][value, check][world][ncap] doubles |
// flags[world] | slots[world][kSlots] | seq | arrive; every rank opens every
// peer's arena through CUDA IPC.
struct SrcState {
  int world = 1, rank = 0, device = 0;
  bool connected = false;
  OwnMask mask;
  uint32_t s0 = 0, s1 = 0, p0 = 0, p1 = 0, ncap = 0, ncap_e = 0;
  int4 *own_tasks = nullptr, *cap_tasks = nullptr;
  int n_own = 0, n_cap = 0;
  char* arena = nullptr;
  int64_t off_flags = 0, off_slots = 0, off_seq = 0, off_arrive = 0, bytes = 0;
  std::vector<char*> peer_base;
  double** d_bufs = nullptr;        // [world] buffer base of every rank (own included)
  double** d_peer_slots = nullptr;  // slot tables of the peers (rank order, self skipped)
  Signal sig{};
  Wait wait{};
  double* slots() const { return (double*)(arena + off_slots); }
  SrcX view() const {
    SrcX X{};
    X.bufs = d_bufs; X.ncap = ncap; X.ncap_e = ncap_e; X.world = world; X.rank = rank;
    X.s0 = s0; X.s1 = s1; X.cap_tasks = cap_tasks; X.n_cap = n_cap; X.sig = sig; X.wait = wait;
    return X;
  }
  ~SrcState() {
    cudaSetDevice(device);
    std::lock_guard<std::mutex> lock(device_mutex());
    cudaDeviceSynchronize();
    for (char* b : peer_base)
      if (b) cudaIpcCloseMemHandle(b);
    for (void* p : {(void*)d_bufs, (void*)d_peer_slots, (void*)own_tasks, (void*)cap_tasks, (void*)arena})
      if (p) cudaFree(p);
  }
};
void free_src(void* p) { delete (SrcState*)p; }

struct StepBench {
  int reps;
  double ms_col, ms_row, bytes_col, bytes_row;
  int matrix_free;  // out: the operator the timed kernels used
};

// Exchange plumbing of one solve: peer-memory halo/reduction events for a
// row-partitioned LP, nothing for a single-device one.
struct Exchange {
  DistState* ds = nullptr;
  PdlpState* st = nullptr;
  int64_t nl = 0;
  bool active() const { return ds != nullptr && ds->world > 1; }
  // copy owned boundary ranges of the listed window arrays to the
  // neighbours, signal them, and wait for theirs
  void halo(cudaStream_t s, std::initializer_list<int> arrays) {
    if (!active()) return;
    Halo H = ds->halo_plan(arrays);
    halo_kernel<<<std::max(1, std::min(kSMs * 2, (int)((ds->halo_max(arrays) + 255) / 256))), 256, 0, s>>>(
        H, ds->sig_nbr, st);
    wait_kernel<<<1, 32, 0, s>>>(ds->wait_nbr, st);
    nl += 2;
  }
  void wait_nbr(cudaStream_t s) {
    if (!active()) return;
    wait_kernel<<<1, 32, 0, s>>>(ds->wait_nbr, st);
    nl += 1;
  }
  void wait_all(cudaStream_t s) {
    if (!active()) return;
    wait_kernel<<<1, 32, 0, s>>>(ds->wait_all, st);
    nl += 1;
  }
};

// Certificate kernels of one chunk (single-device solves; on = false: none).
struct Infeas {
  bool on = false;
  const double *ubI = nullptr, *loI = nullptr, *hiI = nullptr;
  double *yprev = nullptr, *dv = nullptr;
};

// One cooperative launch of chunk_persist_kernel (a memset node resets the
// grid-barrier counter first).
template <bool UNIT, bool DICT>
void launch_persist(cudaStream_t st, const teccl_lp* lp, const Vecs& Vc, const Vecs& Vr, const Persist& P) {
  cudaMemsetAsync(P.bar, 0, sizeof(unsigned int), st);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kSMs);
  cfg.blockDim = dim3(kPersistThreads);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, chunk_persist_kernel<UNIT, DICT>, (int32_t)lp->n, (int32_t)lp->m, col_view(lp),
                     row_view(lp), Vc, Vr, P);
}

template <bool UNIT, bool DICT>
void enqueue_chunk(int chunk, cudaStream_t st, const teccl_lp* lp, const TeOp* te, const EmOp* em, const Vecs& Vc, const Vecs& Vr,
                   Exchange& X, double* y_w, double* yt_w, const Infeas& IF, const Persist* PL) {
  const int64_t nrw = gather_rows(lp), orr = own_row_off(lp);
  if (PL) launch_persist<UNIT, DICT>(st, lp, Vc, Vr, *PL);
  for (int j = 0; !PL && j < chunk; ++j) {
    const bool check = (j == chunk - 1);
    if (check) launch_col<UNIT, DICT, true>(st, lp, te, em, Vc, j);
    else launch_col<UNIT, DICT, false>(st, lp, te, em, Vc, j);
    if (!Vc.push.n) {  // fused kernels push their own halos
      if (check) X.halo(st, {A_XBAR, A_XT});
      else X.halo(st, {A_XBAR});
    } else if (!Vr.wait.npeer) {
      X.wait_nbr(st);  // fused_halo = 2: the wait is a separate one-thread kernel
    }
    if (check) launch_row<UNIT, DICT, true>(st, lp, te, em, Vr, j);
    else launch_row<UNIT, DICT, false>(st, lp, te, em, Vr, j);
    if (!Vr.push.n) {
      if (check) X.halo(st, {A_Y, A_YT});
      else X.halo(st, {A_Y});
    } else if (!Vc.wait.npeer) {
      X.wait_nbr(st);
    }
  }
  if (Vr.push.n) X.wait_nbr(st);  // yt ghosts for kkt_col
  if (te) {
    kkt_row_kernel<UNIT, 1><<<Vr.nb_row, kThreads, 0, st>>>(lp->m, SellView{}, *te, EmOp{}, Vr, OwnMask{});
    kkt_col_kernel<UNIT, 1><<<Vc.nb_col, kThreads, 0, st>>>(lp->n, SellView{}, *te, EmOp{}, Vc, OwnMask{});
  } else if (em) {
    kkt_row_kernel<UNIT, 2><<<Vr.nb_row, kThreads, 0, st>>>(lp->m, SellView{}, TeOp{}, *em, Vr, OwnMask{});
    kkt_col_kernel<UNIT, 2><<<Vc.nb_col, kThreads, 0, st>>>(lp->n, SellView{}, TeOp{}, *em, Vc, OwnMask{});
  } else {
    kkt_row_kernel<UNIT, 0><<<Vr.nb_row, kThreads, 0, st>>>(lp->m, row_view(lp), TeOp{}, EmOp{}, Vr, OwnMask{});
    kkt_col_kernel<UNIT, 0><<<Vc.nb_col, kThreads, 0, st>>>(lp->n, col_view(lp), TeOp{}, EmOp{}, Vc, OwnMask{});
  }
  if (IF.on) {  // exits at once unless this chunk evaluates the certificate
    infeas_row_kernel<0><<<Vr.nb_row, kThreads, 0, st>>>(lp->m, Vr, IF.loI, IF.hiI, IF.yprev, IF.dv);
    if (te)
      infeas_col_kernel<UNIT, 1><<<Vc.nb_col, kThreads, 0, st>>>(lp->n, SellView{}, *te, Vc, IF.ubI, IF.dv);
    else
      infeas_col_kernel<UNIT, 0><<<Vc.nb_col, kThreads, 0, st>>>(lp->n, col_view(lp), TeOp{}, Vc, IF.ubI, IF.dv);
  }
  reduce_publish_kernel<<<1, 1024, 0, st>>>(Vc, X.active() ? X.ds->sig_all : Signal{},
                                            X.active() ? X.ds->d_peer_slots : nullptr);
  X.wait_all(st);
  control_kernel<<<1, 32, 0, st>>>(Vc);
  restart_x_kernel<<<grid_for(lp->n), kThreads, 0, st>>>(lp->n, Vc);
  restart_y_kernel<<<grid_for(nrw), kThreads, 0, st>>>(nrw, orr, lp->m, y_w, yt_w, Vr.y0, Vr.st);
}

// One chunk of a source-partitioned solve: own columns, own rows (segment
// tasks of this rank), capacity partials to every rank, capacity dual step;
// then the masked KKT, the cross-rank reduction and the (identical) control.
template <bool UNIT, bool DICT>
void enqueue_chunk_src(int chunk, cudaStream_t st, const teccl_lp* lp, const TeOp* te, const SrcState* src,
                       const Vecs& Vc, const Vecs& Vr, int nb_colsrc, int nb_own, int nb_fin, int blk_off,
                       double* y_w, double* yt_w) {
  TeOp own = *te;
  own.rtask = src->own_tasks;
  own.n_rtask = src->n_own;
  const SrcX X = src->view();
  const int nb_cap = std::max(1, (src->n_cap + 7) / 8);
  const OwnMask& M = src->mask;
  const bool pairs = ((M.c0 | M.c1 | M.q0 | M.q1) & 1u) == 0;
  const bool wide = 8.0 * te->m > kL2GatherBytes;
  const int nb_pair = (int)((((M.c1 - M.c0) + (M.q1 - M.q0)) / 2 + kTile - 1) / kTile);
  for (int j = 0; j < chunk; ++j) {
    const bool check = (j == chunk - 1);
    const int parity = j & 1;
    if (pairs) {  // pair-decoded two-column kernel over the rank's ranges
      const ColRange CR{src->mask.c0, src->mask.c1, src->mask.q0, src->mask.q1};
      if (wide) {
        if (check) col_te2_kernel<true, true, true><<<nb_pair, kThreads, 0, st>>>(*te, Vc, j, CR);
        else col_te2_kernel<false, true, true><<<nb_pair, kThreads, 0, st>>>(*te, Vc, j, CR);
      } else {
        if (check) col_te2_kernel<true, false, true><<<nb_pair, kThreads, 0, st>>>(*te, Vc, j, CR);
        else col_te2_kernel<false, false, true><<<nb_pair, kThreads, 0, st>>>(*te, Vc, j, CR);
      }
    } else if (check) {
      col_src_kernel<true><<<nb_colsrc, kThreads, 0, st>>>(*te, Vc, j, src->mask);
    } else {
      col_src_kernel<false><<<nb_colsrc, kThreads, 0, st>>>(*te, Vc, j, src->mask);
    }
    if (nb_own > 0) {
      if (check) row_seg_kernel<true><<<nb_own, kThreads, 0, st>>>(own, Vr, j);
      else row_seg_kernel<false><<<nb_own, kThreads, 0, st>>>(own, Vr, j);
    }
    if (check) cap_part_kernel<true><<<nb_cap, kThreads, 0, st>>>(*te, Vr, X, parity);
    else cap_part_kernel<false><<<nb_cap, kThreads, 0, st>>>(*te, Vr, X, parity);
    if (check) cap_fin_kernel<true><<<nb_fin, kThreads, 0, st>>>(*te, Vr, X, parity, j, blk_off);
    else cap_fin_kernel<false><<<nb_fin, kThreads, 0, st>>>(*te, Vr, X, parity, j, blk_off);
  }
  kkt_row_kernel<UNIT, 1><<<(int)((lp->m + kTile - 1) / kTile), kThreads, 0, st>>>(lp->m, SellView{}, *te,
                                                                                 EmOp{}, Vr, src->mask);
  kkt_col_kernel<UNIT, 1><<<(int)((lp->n + kTile - 1) / kTile), kThreads, 0, st>>>(lp->n, SellView{}, *te,
                                                                                 EmOp{}, Vc, src->mask);
  reduce_publish_kernel<<<1, 1024, 0, st>>>(Vc, src->sig, src->d_peer_slots);
  wait_kernel<<<1, 32, 0, st>>>(src->wait, Vc.st);
  control_kernel<<<1, 32, 0, st>>>(Vc);
  restart_x_kernel<<<grid_for(lp->n), kThreads, 0, st>>>(lp->n, Vc);
  restart_y_kernel<<<grid_for(lp->m), kThreads, 0, st>>>(lp->m, 0, lp->m, y_w, yt_w, Vr.y0, Vr.st);
}

// setup-phase all-reduce of `count` quantities laid out as part[k*pstride+b]
// (nb partials each); result sums land in out[0..count), inverse roots in
// out[count..2count). Host-visible after a stream sync.
int all_reduce(cudaStream_t st, Exchange& X, double* part, int nb, int64_t pstride, int count,
               double* slots, int world, int rank, double* out) {
  publish_values_kernel<<<1, 1024, 0, st>>>(part, nb, pstride, count, slots, rank,
                                            X.active() ? X.ds->sig_all : Signal{},
                                            X.active() ? X.ds->d_peer_slots : nullptr);
  X.wait_all(st);
  sum_slots_kernel<<<1, 32, 0, st>>>(slots, world, count, out);
  X.nl += 2;
  TECCL_CHECK_LAUNCH();
  return TECCL_OK;
}

template <bool UNIT, bool DICT>
int solve_impl(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* o, double* x_dev,
               double* y_dev, teccl_pdlp_result* res, StepBench* sb) {
  cudaStream_t st = ctx->stream;
  const int32_t m = lp->m, n = lp->n;
  const int nb_row = (int)((m + kTile - 1) / kTile), nb_col = (int)((n + kTile - 1) / kTile);
  DistState* ds = (DistState*)lp->dist;
  if (lp->part_world > 1 && (!ds || !ds->connected)) {
    set_error("partitioned LP: call teccl_dist_export/teccl_dist_connect before solving");
    return TECCL_EINVAL;
  }
  const int world = ds ? ds->world : 1, rank = ds ? ds->rank : 0;
  const int64_t ncw = gather_cols(lp), nrw = gather_rows(lp);
  const int64_t oc = own_col_off(lp), orr = own_row_off(lp);
  // source-partitioned solve: setup is the single-device one (redundant on
  // every rank); the iteration works on this rank's sources and pairs
  const SrcState* sp = (const SrcState*)lp->src;
  if (sp && !sp->connected) {
    set_error("source-partitioned LP: call teccl_src_export/teccl_src_connect before solving");
    return TECCL_EINVAL;
  }
  const int src_nb_own = sp ? (sp->n_own + 8 * kSegTPW - 1) / (8 * kSegTPW) : 0;
  const int src_nb_fin = sp ? (int)((sp->ncap + kTile - 1) / kTile) : 0;
  const int src_blk_off = sp ? std::max(nb_row, src_nb_own) : 0;
  const int src_nb_col = sp ? (int)(((sp->mask.c1 - sp->mask.c0) + (sp->mask.q1 - sp->mask.q0) + kTile - 1) / kTile) : 0;
  Workspace* ws = (Workspace*)lp->pdlp_ws;
  if (!ws) {
    ws = new Workspace();
    ws->device = ctx->device;
    ws->st = st;
    Workspace& W = *ws;
    W.pstride = std::max<int64_t>(std::max(nb_row, nb_col), kGrid);
    if (lp->te && ((TeHold*)lp->te)->kind == 0) {
      const TeOp& t = ((TeHold*)lp->te)->op;
      W.pstride = std::max<int64_t>(W.pstride, std::max((t.n_ctask + 7) / 8, (t.n_rtask + 7) / 8));
    }
    if (sp) W.pstride = std::max<int64_t>(W.pstride, src_blk_off + src_nb_fin);
    W.rstat = W.alloc<double>(m); W.cstat = W.alloc<double>(n);
    // pad slot [n] / [m]: the two-column kernels load pairs unconditionally
    // E, y0: +4 so the row kernels' 16-byte bulk copies may round a range up
    W.D = W.alloc<float>(n + 1); W.E = W.alloc<float>(m + 4);
    W.x0 = W.alloc<float>(n + 1); W.y0 = W.alloc<float>(m + 4);
    W.x = W.alloc<double>(n + 1);
    if (!ds) {  // single device: the gather windows are the owned vectors
      W.R = W.alloc<double>(m + 1); W.C = W.alloc<double>(n + 1);
      W.xt = W.alloc<double>(n + 1); W.xbar = W.alloc<double>(n + 1);
      W.y = W.alloc<double>(m + 1); W.yt = W.alloc<double>(m + 1);
      W.slots = W.alloc<double>(kSlots);
    } else {
      W.R = ds->arr(A_RW); W.C = ds->arr(A_CW);
      W.xt = ds->arr(A_XT); W.xbar = ds->arr(A_XBAR);
      W.y = ds->arr(A_Y); W.yt = ds->arr(A_YT);
      W.slots = ds->slots();
    }
    W.part = W.alloc<double>((int64_t)kNQ * W.pstride);
    W.part2 = W.alloc<double>(kGrid);
    W.dst = W.alloc<PdlpState>(1);
    const bool ok = W.R && W.C && W.rstat && W.cstat && W.D && W.E && W.x0 && W.y0 && W.x &&
                    W.xt && W.xbar && W.y && W.yt && W.part && W.part2 && W.dst && W.slots;
    if (!ok || cudaEventCreate(&W.ev0) != cudaSuccess || cudaEventCreate(&W.ev1) != cudaSuccess) {
      delete ws;
      set_error("device allocation failed for PDLP workspace");
      return TECCL_ENOMEM;
    }
    // defined pad values (read, never used, by the two-column kernels)
    TECCL_CUDA(cudaMemsetAsync(W.D + n, 0, sizeof(float), st));
    TECCL_CUDA(cudaMemsetAsync(W.x0 + n, 0, sizeof(float), st));
    TECCL_CUDA(cudaMemsetAsync(W.x + n, 0, sizeof(double), st));
    lp->pdlp_ws = ws;
    lp->ws_free = free_workspace;
  }
  Workspace& W = *ws;
  cudaEvent_t ev0 = W.ev0, ev1 = W.ev1;
  TECCL_CUDA(cudaEventRecord(ev0, st));
  auto t_start = std::chrono::steady_clock::now();
  const bool trace = getenv("TECCL_TRACE") != nullptr;
  auto mark = [&](const char* what) {
    if (trace) {
      cudaStreamSynchronize(st);
      fprintf(stderr, "[teccl trace r%d] %-14s %8.3f ms\n", rank, what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    }
  };
  const int64_t pstride = W.pstride;
  // window (gathered) arrays and their owned parts
  double *R_w = W.R, *C_w = W.C, *xt_w = W.xt, *xbar_w = W.xbar, *y_w = W.y, *yt_w = W.yt;
  double *R = R_w + orr, *C = C_w + oc;
  double *xt = xt_w + oc, *xbar = xbar_w + oc, *y = y_w + orr, *yt = yt_w + orr;
  double *rstat = W.rstat, *cstat = W.cstat;
  float *D = W.D, *E = W.E, *x0 = W.x0, *y0 = W.y0;
  double* x = W.x;
  double *part = W.part, *part2 = W.part2, *slots = W.slots;
  PdlpState* dst = W.dst;
  Exchange X;
  X.ds = ds;
  X.st = dst;
  TECCL_CUDA(cudaMemsetAsync(dst, 0, sizeof(PdlpState), st));
  TECCL_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * kNQ * pstride, st));
  // always-zero slots the SELL padding gathers from (index = window length)
  TECCL_CUDA(cudaMemsetAsync(xt_w, 0, sizeof(double) * (ncw + 1), st));
  TECCL_CUDA(cudaMemsetAsync(xbar_w, 0, sizeof(double) * (ncw + 1), st));
  TECCL_CUDA(cudaMemsetAsync(y_w, 0, sizeof(double) * (nrw + 1), st));
  TECCL_CUDA(cudaMemsetAsync(yt_w, 0, sizeof(double) * (nrw + 1), st));
  // matrix-free operator for single-device TE LPs; the SELL copies are
  // only built for LPs that need them
  // Operator per half-step: 0 stored SELL, 2 matrix-free one thread per
  // entry, 3 matrix-free segment tasks on both sides, 4 per-entry columns +
  // segment rows. 1 (auto): the stored SELL kernels while the iteration's
  // working set is L2-resident (latency-bound, profiles/r01_h), mode 4 above
  // that (HBM-bound: no index stream, fastest pair measured on 4-, 8- and
  // 16-chassis LPs, profiles/r01_j_hbm_roofline.md).
  const TeHold* hold = (const TeHold*)lp->te;
  const TeOp* te_all = (hold && hold->kind == 0) ? &hold->op : nullptr;
  // epoch-block LPs (row-partitioned solves) have one matrix-free operator
  // (per entry, both sides), selected by modes 2-4; auto keeps the stored
  // SELL blocks there: epoch-major gathers are scattered across each epoch's
  // families and the matrix-free block kernels measured slower
  // (8-chassis LP on 2 GPUs: 0.716 vs 0.578 ms / iteration, profiles/r01_k)
  const EmOp* em_all = (hold && hold->kind == 1) ? &hold->em : nullptr;
  int mf = (te_all || em_all) ? o->matrix_free : 0;
  if (mf == 1) mf = (te_all && lp->n >= kAutoMatrixFreeCols && te_all->K >= 16) ? 4 : 0;
  if (sp) mf = 2;  // the source-partitioned iteration is matrix-free (col_src / row_seg / cap kernels)
  const TeOp* te = (mf && te_all) ? te_all : nullptr;
  const EmOp* em = (mf && em_all) ? em_all : nullptr;
  const bool seg_col = te && mf == 3, seg_row = te && (mf == 3 || mf == 4);
  if (!te && !em) {
    int rc = teccl_build_sell(lp, st);
    if (rc) return rc;
  }
  if (X.active()) {  // every rank has finished resetting before anyone writes peer memory
    publish_values_kernel<<<1, 1024, 0, st>>>(part, 1, pstride, 0, slots, rank, ds->sig_all,
                                              ds->d_peer_slots);
    X.wait_all(st);
  }
  const int gr = grid_for(std::max<int64_t>(std::max<int64_t>(m, n), std::max(ncw, nrw)));
  int64_t nl = 0;  // kernel launches issued by this solve
  mark("setup+sell");

  // --- Ruiz equilibration + Pock-Chambolle (alpha = 1), simultaneous updates
  fill_kernel<<<gr, kThreads, 0, st>>>(nrw, R_w, 1.0);
  fill_kernel<<<gr, kThreads, 0, st>>>(ncw, C_w, 1.0);
  nl += 2;
  for (int it = 0; it <= o->ruiz_iters; ++it) {
    if (it < o->ruiz_iters) {
      abs_stat_kernel<UNIT, true><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, C_w, R, rstat);
      abs_stat_kernel<UNIT, true><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, R_w, C, cstat);
    } else {
      abs_stat_kernel<UNIT, false><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, C_w, R, rstat);
      abs_stat_kernel<UNIT, false><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, R_w, C, cstat);
    }
    apply_scale_kernel<<<gr, kThreads, 0, st>>>(m, R, rstat);
    apply_scale_kernel<<<gr, kThreads, 0, st>>>(n, C, cstat);
    nl += 4;
    X.halo(st, {A_CW, A_RW});
  }
  TECCL_CHECK_LAUNCH();

  mark("equilibrate");
  // --- preconditioners (fp32, exact from here on) and their square roots
  double* rootE = rstat;
  double* rootD = cstat;
  precond_kernel<<<gr, kThreads, 0, st>>>(m, R, E, rootE);
  precond_kernel<<<gr, kThreads, 0, st>>>(n, C, D, rootD);
  nl += 2;

  // --- norms: scaled ||C c||, ||R b|| set the initial primal weight (the
  // bound/objective rescaling of PDLP); unscaled ||c||, ||b|| enter the
  // relative termination criteria. Global sums over ranks.
  double nrm[8] = {0};
  norms_kernel<<<kGrid, kThreads, 0, st>>>(n, C, lp->obj, nullptr, 0, part, part + pstride);
  norms_kernel<<<kGrid, kThreads, 0, st>>>(m, R, lp->row_lo, lp->row_hi, 1, part + 2 * pstride,
                                           part + 3 * pstride);
  nl += 2;
  if (all_reduce(st, X, part, kGrid, pstride, 4, slots, world, rank, part2)) return TECCL_ECUDA;
  TECCL_CUDA(cudaMemcpyAsync(nrm, part2, sizeof(double) * 8, cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  const double csq_s = nrm[0], csq_u = nrm[1], bsq_s = nrm[2], bsq_u = nrm[3];
  const double beta = sqrt(bsq_s) + 1.0, gamma = sqrt(csq_s) + 1.0;
  const double cn_s = sqrt(csq_s) / gamma, bn_s = sqrt(bsq_s) / beta;
  const double omega_s = (cn_s > 1e-10 && bn_s > 1e-10) ? cn_s / bn_s : 1.0;

  // --- power iteration for ||E^1/2 A D^1/2||_2 (v in xt, D^1/2 v in xbar,
  // A D^1/2 v in yt, E A D^1/2 v in y); norms reduced on the device
  double sigma_max = 1.0;
  {
    double* scal = part2;  // [0] squared norm, [1] inverse norm
    hash_fill_kernel<<<gr, kThreads, 0, st>>>(n, xt);
    sumsq_kernel<<<kGrid, kThreads, 0, st>>>(n, xt, part);
    nl += 2;
    if (all_reduce(st, X, part, kGrid, pstride, 1, slots, world, rank, scal)) return TECCL_ECUDA;
    scale_by_kernel<<<gr, kThreads, 0, st>>>(n, xt, scal);
    nl += 1;
    // 40 rounds; on HBM-resident LPs (>= kAutoMatrixFreeCols columns in
    // total) then blocks of 20 until the estimate moves by < 2e-5 relative
    // (at most 300 rounds): an estimate short of the norm makes the step too
    // long, and there 40 rounds are not enough (the 32-chassis LP's estimate
    // was 4 % low and the solve diverged; DESIGN.md configs[4]), while the
    // extra rounds cost a negligible part of the solve. On L2-resident LPs
    // the rounds are launch-bound (~9 launches each) and would cost as much
    // as the whole solve of a small LP; 40 rounds have been stable on every
    // one of them. The decision uses the all-reduced value: identical on
    // every rank.
    const int64_t total_cols = lp->part_world > 1 ? lp->em_ncols : (int64_t)n;
    const int min_rounds = 40, block = 20;
    const int max_rounds = total_cols >= kAutoMatrixFreeCols ? 300 : min_rounds;
    double nv = 0.0, prev = -1.0;
    for (int it = 0;; ++it) {
      mul_kernel<<<gr, kThreads, 0, st>>>(n, xbar, xt, rootD);
      X.halo(st, {A_XBAR});
      spmv_scaled_kernel<UNIT><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, xbar_w, nullptr, yt);
      mul_kernel<<<gr, kThreads, 0, st>>>(m, y, yt, rootE);
      mul_kernel<<<gr, kThreads, 0, st>>>(m, y, y, rootE);
      X.halo(st, {A_Y});
      spmv_scaled_kernel<UNIT><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, y_w, rootD, xt);
      sumsq_kernel<<<kGrid, kThreads, 0, st>>>(n, xt, part);
      nl += 6;
      if (all_reduce(st, X, part, kGrid, pstride, 1, slots, world, rank, scal)) return TECCL_ECUDA;
      const int done_rounds = it + 1;
      if (done_rounds >= min_rounds && ((done_rounds - min_rounds) % block == 0 || done_rounds >= max_rounds)) {
        TECCL_CUDA(cudaMemcpyAsync(&nv, scal, sizeof(double), cudaMemcpyDeviceToHost, st));
        TECCL_CUDA(cudaStreamSynchronize(st));
        // nv = ||M v||^2 with M = B^T B: sigma = nv^(1/4); 8e-5 on nv ~ 2e-5 on sigma
        if (done_rounds >= max_rounds || !std::isfinite(nv) || (prev > 0.0 && fabs(nv - prev) <= 8e-5 * nv)) {
          if (o->verbose > 0)
            fprintf(stderr, "[teccl pdlp r%d] power iteration: %d rounds\n", rank, done_rounds);
          break;
        }
        prev = nv;
      }
      scale_by_kernel<<<gr, kThreads, 0, st>>>(n, xt, scal);
      nl += 1;
    }
    if (nv > 0.0 && std::isfinite(nv)) sigma_max = sqrt(sqrt(nv));
    TECCL_CUDA(cudaMemsetAsync(xbar_w, 0, sizeof(double) * (ncw + 1), st));
    TECCL_CUDA(cudaMemsetAsync(y_w, 0, sizeof(double) * (nrw + 1), st));
    TECCL_CUDA(cudaMemsetAsync(xt_w, 0, sizeof(double) * (ncw + 1), st));
    TECCL_CUDA(cudaMemsetAsync(yt_w, 0, sizeof(double) * (nrw + 1), st));
  }
  TECCL_CHECK_LAUNCH();

  mark("power-iter");
  // --- infeasibility certificate (single device): implied bounds once per LP
  Infeas IF;
  IF.on = o->eps_infeas > 0.0 && !ds && !sp && !em_all && !sb;
  if (IF.on) {
    if (!W.yprev) {
      W.ubI = W.alloc<double>(n); W.loI = W.alloc<double>(m); W.hiI = W.alloc<double>(m);
      W.yprev = W.alloc<double>(m); W.dv = W.alloc<double>(m + 1);
      if (!W.ubI || !W.loI || !W.hiI || !W.yprev || !W.dv) {
        set_error("device allocation failed for the infeasibility certificate");
        return TECCL_ENOMEM;
      }
      implied_col_kernel<<<gr, kThreads, 0, st>>>(n, lp->var_ub, te_all ? te_all->d : TeDev{}, te_all ? 1 : 0, W.ubI);
      implied_row_kernel<UNIT><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, lp->var_lb, W.ubI,
                                                         lp->row_lo, lp->row_hi, W.loI, W.hiI);
      nl += 2;
      TECCL_CUDA(cudaMemsetAsync(W.dv + m, 0, sizeof(double), st));
    }
    TECCL_CUDA(cudaMemsetAsync(W.yprev, 0, sizeof(double) * m, st));
    IF.ubI = W.ubI; IF.loI = W.loI; IF.hiI = W.hiI; IF.yprev = W.yprev; IF.dv = W.dv;
  }
  // the setup reductions used the partial slots; the iteration kernels write
  // only as many slots as they have blocks, so start them from zero
  TECCL_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * kNQ * pstride, st));
  // --- state: omega in original space = scaled weight * gamma / beta
  PdlpState hs{};
  hs.eta = (o->step_safety > 0.0 && o->step_safety < 1.0 ? o->step_safety : 0.998) / sigma_max;
  if (o->verbose > 0)
    fprintf(stderr, "[teccl pdlp r%d] power iteration: ||E^1/2 A D^1/2|| ~ %.9g, eta %.6g\n", rank, sigma_max, hs.eta);
  hs.omega = omega_s * gamma / beta * (o->omega_scale > 0.0 ? o->omega_scale : 1.0);
  hs.tau = hs.eta / hs.omega;
  hs.sigma = hs.eta * hs.omega;
  hs.refl = o->reflection;
  hs.bnorm = sqrt(bsq_u);
  hs.cnorm = sqrt(csq_u);
  hs.eps = o->eps_rel;
  hs.eps_res = o->eps_res > 0.0 ? std::min(o->eps_rel, o->eps_res) : o->eps_rel;
  hs.eps_infeas = IF.on ? o->eps_infeas : 0.0;
  hs.infeas_every = o->infeas_every > 0 ? o->infeas_every : 4;
  hs.infeas_due = (IF.on && hs.infeas_every == 1) ? 1 : 0;
  hs.rs_suff = o->restart_sufficient;
  hs.rs_nec = o->restart_necessary;
  hs.rs_art = o->restart_artificial;
  hs.theta = o->omega_theta;
  hs.ki = o->omega_ki;
  hs.kd = o->omega_kd;
  hs.bias = o->omega_bias > 0.0 ? log(o->omega_bias) : 0.0;
  const int chunk = std::min(o->check_every > 0 ? o->check_every : 64, kLamTab);
  hs.chunk_len = chunk;
  for (int j = 0; j < kLamTab; ++j) hs.lam_tab[j] = (j + 1.0) / (j + 2.0);
  TECCL_CUDA(cudaMemcpyAsync(dst, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));

  Vecs V{};
  V.D = D; V.E = E;
  V.col = Bounds{lp->col_code, lp->col_dict, lp->var_lb, lp->var_ub, lp->obj};
  V.row = Bounds{lp->row_code, lp->row_dict, lp->row_lo, lp->row_hi, nullptr};
  V.x = x; V.x0 = x0; V.y0 = y0;
  V.c_u = lp->obj; V.lb_u = lp->var_lb; V.ub_u = lp->var_ub; V.lo_u = lp->row_lo; V.hi_u = lp->row_hi;
  V.part = part;
  V.pstride = pstride;
  V.nb_row = nb_row;
  V.nb_col = nb_col;
  V.st = dst;
  V.slots = slots;
  V.world = world;
  V.rank = rank;
  V.col_pipe = o->col_pipeline;
  V.pdl = o->pdl;
  V.seg = (seg_col ? 1 : 0) | (seg_row ? 2 : 0);
  // partial-sum slots: the iteration kernels write one per block; the
  // reduction reads max(blocks) slots per quantity (unwritten ones stay 0)
  if (seg_col) V.nb_col = std::max(V.nb_col, (te->n_ctask + 7) / 8);
  if (seg_row) V.nb_row = std::max(V.nb_row, (te->n_rtask + 7) / 8);
  // Vc: column kernels (own x side, gather y windows); Vr: row kernels
  // (own y side, gather x windows); Vi: owned parts only
  Vecs Vc = V, Vr = V, Vi = V;
  Vc.xt = xt; Vc.xbar = xbar; Vc.y = y_w; Vc.yt = yt_w;
  Vr.y = y; Vr.yt = yt; Vr.xbar = xbar_w; Vr.xt = xt_w;
  Vi.xt = xt; Vi.xbar = xbar; Vi.y = y; Vi.yt = yt;
  if (X.active() && o->fused_halo) {  // halos stored by the half-step kernels themselves
    Vc.push = ds->push_plan(A_XBAR, A_XT);
    Vr.push = ds->push_plan(A_Y, A_YT);
    if (o->fused_halo == 1) {  // 2: waits stay separate one-thread kernels
      Vc.wait = ds->wait_nbr;
      Vr.wait = ds->wait_nbr;
    }
  }
  if (sp) {  // cross-rank reductions through the partition's slot tables
    for (Vecs* v : {&Vc, &Vr}) {
      v->slots = sp->slots();
      v->world = sp->world;
      v->rank = sp->rank;
      v->nb_col = nb_col;
      v->nb_row = src_blk_off + src_nb_fin;
      v->seg = 0;
    }
  }
  // --- persistent chunk kernel: stored SELL operator on one device, when every
  // block's dense state fits in shared memory (L2-resident LPs: configs[1])
  Persist PP{};
  const Persist* PL = nullptr;
  if (o->persist && !te && !em && !ds && !sp && !sb && chunk <= kLamTab) {
    PP.cpb = (int)((((int64_t)n + kSMs - 1) / kSMs + kSlice - 1) / kSlice * kSlice);
    PP.rpb = (int)((((int64_t)m + kSMs - 1) / kSMs + kSlice - 1) / kSlice * kSlice);
    PP.ncd = DICT ? lp->n_col_dict : 0;
    PP.nrd = DICT ? lp->n_row_dict : 0;
    PP.chunk = chunk;
    PP.smem = sizeof(double) * ((size_t)PP.cpb + PP.rpb + 3 * PP.ncd + 2 * PP.nrd + chunk) +
              sizeof(float) * 2 * ((size_t)PP.cpb + PP.rpb) + (DICT ? sizeof(uint16_t) * ((size_t)PP.cpb + PP.rpb) : 0);
    int occ = 0;
    if (PP.smem <= (size_t)200 * 1024 &&
        cudaFuncSetAttribute(chunk_persist_kernel<UNIT, DICT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)PP.smem) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chunk_persist_kernel<UNIT, DICT>, kPersistThreads,
                                                      PP.smem) == cudaSuccess &&
        occ >= 1) {
      if (!W.bar) W.bar = W.alloc<unsigned int>(1);
      PP.bar = W.bar;
      if (PP.bar) PL = &PP;
    }
    cudaGetLastError();  // a refused attribute only means: no persistent kernel
  }
  init_iterates_kernel<<<gr, kThreads, 0, st>>>(n, m, Vi, o->warm_start, x_dev, y_dev);
  nl += 1;
  if (o->warm_start) X.halo(st, {A_Y, A_YT});
  TECCL_CHECK_LAUNCH();

  if (sb && sp) { set_error("step bench is not available for source-partitioned LPs"); return TECCL_EINVAL; }
  if (sb) {  // time the fused iteration kernels alone, CUDA events on this stream
    cudaEvent_t a, b, c2;
    TECCL_CUDA(cudaEventCreate(&a));
    TECCL_CUDA(cudaEventCreate(&b));
    TECCL_CUDA(cudaEventCreate(&c2));
    for (int w = 0; w < 3; ++w) {
      launch_col<UNIT, DICT, false>(st, lp, te, em, Vc, 0);
      launch_row<UNIT, DICT, false>(st, lp, te, em, Vr, 0);
    }
    TECCL_CUDA(cudaEventRecord(a, st));
    for (int r = 0; r < sb->reps; ++r) launch_col<UNIT, DICT, false>(st, lp, te, em, Vc, 0);
    TECCL_CUDA(cudaEventRecord(b, st));
    for (int r = 0; r < sb->reps; ++r) launch_row<UNIT, DICT, false>(st, lp, te, em, Vr, 0);
    TECCL_CUDA(cudaEventRecord(c2, st));
    TECCL_CHECK_LAUNCH();
    TECCL_CUDA(cudaEventSynchronize(c2));
    float m1 = 0.f, m2 = 0.f;
    TECCL_CUDA(cudaEventElapsedTime(&m1, a, b));
    TECCL_CUDA(cudaEventElapsedTime(&m2, b, c2));
    sb->ms_col = m1 / sb->reps;
    sb->ms_row = m2 / sb->reps;
    // algorithmic bytes: SELL slice headers and every
    // stored entry once, the gathered vector once, dense operands once
    sb->matrix_free = mf;
    if (te || em) {  // no stored matrix: dense vectors, the gathered operand once, capacities
      sb->bytes_col = 8.0 * nrw + 32.0 * n;
      sb->bytes_row = 8.0 * ncw + 24.0 * m + 8.0 * (te ? (double)te->EK : (double)em->E * em->nk);
      cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c2);
      return TECCL_OK;
    }
    const double ib = UNIT ? 4.0 : 12.0;
    const double ns_c = (double)((n + 31) / 32), ns_r = (double)((m + 31) / 32);
    const double cb = DICT ? 2.0 : 24.0, rbd = DICT ? 2.0 : 16.0;
    // column: x(8) x0(4) D(4) bounds(cb) read; x(8) xbar(8) written
    sb->bytes_col = 12.0 * ns_c + ib * lp->scol_entries + 8.0 * nrw + (32.0 + cb) * n;
    // row: y(8) y0(4) E(4) bounds(rbd) read; y(8) written
    sb->bytes_row = 12.0 * ns_r + ib * lp->srow_entries + 8.0 * ncw + (24.0 + rbd) * m;
    cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c2);
    return TECCL_OK;
  }

  // --- chunk graph (captured once per LP and chunk length)
  const int graph_key = chunk * 1024 + (o->col_pipeline ? 1 : 0) + (te || em ? 2 : 0) + (o->pdl ? 4 : 0) + 8 * V.seg + 32 * o->fused_halo + (sp ? 128 : 0) + (IF.on ? 256 : 0) + (PL ? 512 : 0);
  if (o->use_graphs && W.gexec && W.graph_chunk != graph_key) {
    cudaGraphExecDestroy(W.gexec);
    W.gexec = nullptr;
  }
  const int64_t nl_setup = nl + X.nl;
  X.nl = 0;
  int64_t per_chunk = 0;
  if (o->use_graphs && !W.gexec) {
    std::lock_guard<std::mutex> capture_lock(device_mutex());
    cudaGraph_t g;
    cudaStream_t cap;
    TECCL_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    TECCL_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    if (sp)
      enqueue_chunk_src<UNIT, DICT>(chunk, cap, lp, te, sp, Vc, Vr, src_nb_col, src_nb_own, src_nb_fin,
                                    src_blk_off, y_w, yt_w);
    else
      enqueue_chunk<UNIT, DICT>(chunk, cap, lp, te, em, Vc, Vr, X, y_w, yt_w, IF, PL);
    TECCL_CUDA(cudaStreamEndCapture(cap, &g));
    TECCL_CUDA(cudaGraphInstantiate(&W.gexec, g, 0));
    TECCL_CUDA(cudaGraphDestroy(g));
    TECCL_CUDA(cudaStreamDestroy(cap));
    W.graph_chunk = graph_key;
  }
  cudaGraphExec_t gexec = o->use_graphs ? W.gexec : nullptr;
  per_chunk = sp ? 4LL * chunk + 7 : (PL ? 1LL : 2LL * chunk) + 6 + (IF.on ? 2 : 0) + (X.active() ? (Vc.push.n || Vr.push.n ? (Vc.wait.npeer ? 2LL : 2LL * chunk + 2) : 4LL * chunk + 1) : 0);
  mark("graph");

  // --- iterate: chunks queued `lookahead` deep; the device stops itself
  const int look = o->lookahead > 0 ? o->lookahead : 1;
  if (W.ring_len < look) {
    std::lock_guard<std::mutex> lock(device_mutex());
    if (W.ring) cudaFreeHost(W.ring);
    W.ring = nullptr;
    TECCL_CUDA(cudaMallocHost((void**)&W.ring, sizeof(PdlpState) * look));
    W.ring_len = look;
  }
  while ((int)W.evs.size() < look) {
    cudaEvent_t e;
    TECCL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    W.evs.push_back(e);
  }
  PdlpState* ring = W.ring;
  std::vector<cudaEvent_t>& evs = W.evs;
  int64_t launched = 0, polled = 0;
  int status = TECCL_ITER_LIMIT;
  PdlpState last = hs;
  const int64_t max_chunks = (o->max_iters + chunk - 1) / chunk;
  bool stop = false;
  while (!stop) {
    while (launched < max_chunks && launched - polled < look) {
      if (gexec) {
        TECCL_CUDA(cudaGraphLaunch(gexec, st));
      } else {
        if (sp)
          enqueue_chunk_src<UNIT, DICT>(chunk, st, lp, te, sp, Vc, Vr, src_nb_col, src_nb_own, src_nb_fin,
                                        src_blk_off, y_w, yt_w);
        else
          enqueue_chunk<UNIT, DICT>(chunk, st, lp, te, em, Vc, Vr, X, y_w, yt_w, IF, PL);
      }
      TECCL_CHECK_LAUNCH();
      const int slot = (int)(launched % look);
      TECCL_CUDA(cudaMemcpyAsync(&ring[slot], dst, sizeof(PdlpState), cudaMemcpyDeviceToHost, st));
      TECCL_CUDA(cudaEventRecord(evs[slot], st));
      ++launched;
    }
    if (polled >= launched) break;
    const int slot = (int)(polled % look);
    TECCL_CUDA(cudaEventSynchronize(evs[slot]));
    last = ring[slot];
    ++polled;
    if (o->verbose > 0 && (polled % o->verbose == 0 || last.done))
      fprintf(stderr, "[teccl pdlp r%d] it=%lld rp=%.2e rd=%.2e gap=%.2e pobj=%.9g w=%.3e r=%.2e restarts=%d\n",
              rank, last.total, last.rel_p, last.rel_d, last.gap, last.pobj, last.omega, last.last_r,
              last.restarts);
    if (last.done == 1) { status = TECCL_OPTIMAL; stop = true; }
    else if (last.done == 2) { status = TECCL_NUMERICAL; stop = true; }
    else if (last.done == 4) { status = TECCL_PEER_TIMEOUT; stop = true; }
    else if (last.done == 5) { status = TECCL_PRIMAL_INFEASIBLE; stop = true; }
    else if (polled >= max_chunks) { status = TECCL_ITER_LIMIT; stop = true; }
    else if (!X.active()) {  // ranks must stop together: only iteration caps in multi-GPU
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (el > o->time_limit) { status = TECCL_TIME_LIMIT; stop = true; }
    }
  }
  if (status == TECCL_ITER_LIMIT || status == TECCL_TIME_LIMIT) {
    // stop anything still queued from touching the iterates
    static const int kStopped = 3;
    TECCL_CUDA(cudaMemcpyAsync(&dst->done, &kStopped, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  TECCL_CUDA(cudaStreamSynchronize(st));
  TECCL_CUDA(cudaMemcpyAsync(&last, dst, sizeof(PdlpState), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  if (last.done == 1) status = TECCL_OPTIMAL;
  if (last.done == 5) status = TECCL_PRIMAL_INFEASIBLE;
  if (last.done == 3) last.done = 0;

  mark("iterate");
  output_kernel<<<gr, kThreads, 0, st>>>(n, m, Vi, x_dev, y_dev);
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaEventRecord(ev1, st));
  TECCL_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  TECCL_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));

  mark("teardown");
  res->status = status;
  res->restarts = last.restarts;
  res->iters = last.total;
  res->primal_obj = last.pobj;
  res->dual_obj = last.dobj;
  res->rel_gap = last.gap;
  res->rel_primal_res = last.rel_p;
  res->rel_dual_res = last.rel_d;
  res->solve_seconds = ms * 1e-3;
  res->omega = last.omega;
  res->step = hs.eta;
  res->spmv_launches = nl_setup + 1 + launched * per_chunk;
  res->infeas_cert = last.cert;
  return TECCL_OK;
}

int dispatch(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* o, double* x_dev, double* y_dev,
             teccl_pdlp_result* res, StepBench* sb) {
  const bool dict = lp->col_code && lp->row_code;
  if (lp->unit)
    return dict ? solve_impl<true, true>(ctx, lp, o, x_dev, y_dev, res, sb)
                : solve_impl<true, false>(ctx, lp, o, x_dev, y_dev, res, sb);
  return dict ? solve_impl<false, true>(ctx, lp, o, x_dev, y_dev, res, sb)
              : solve_impl<false, false>(ctx, lp, o, x_dev, y_dev, res, sb);
}

}  // namespace teccl

using namespace teccl;

extern "C" void teccl_pdlp_default_opts(teccl_pdlp_opts* o) {
  o->eps_rel = 1e-4;
  o->max_iters = 2000000;
  o->time_limit = 3600.0;
  o->check_every = 64;
  o->ruiz_iters = 10;
  o->lookahead = 3;
  o->verbose = 0;
  o->reflection = 1.0;
  o->use_graphs = 1;
  o->warm_start = 0;
  o->restart_sufficient = 0.3;
  o->restart_necessary = 0.9;
  o->restart_artificial = 0.36;
  o->omega_theta = 0.6;
  o->omega_scale = 1.0;
  o->omega_ki = 0.0;
  o->omega_kd = 0.0;
  o->col_pipeline = 1;
  o->matrix_free = 1;  // auto: stored SELL while L2-resident (configs[1]), matrix-free above
  o->pdl = 1;
  o->fused_halo = 1;
  o->eps_res = 1e-6;
  o->eps_infeas = 1e-6;
  o->infeas_every = 4;
  o->omega_bias = 1.0;
  o->step_safety = 0.998;
  o->persist = 0;  // measured slower than the two-kernel iteration (profiles/r02_d_persist.md)
}

extern "C" int teccl_pdlp_solve_dev(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                                    double* x_dev, double* y_dev, teccl_pdlp_result* res) {
  if (!ctx || !lp || !x_dev || !res) { set_error("null argument"); return TECCL_EINVAL; }
  teccl_pdlp_opts o;
  if (opts) o = *opts; else teccl_pdlp_default_opts(&o);
  if (!(o.eps_rel > 0.0)) { set_error("eps_rel must be positive"); return TECCL_EINVAL; }
  if (o.warm_start && !y_dev) { set_error("warm start needs y"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  *res = teccl_pdlp_result{};
  if (lp->n == 0) { res->status = TECCL_OPTIMAL; return TECCL_OK; }
  return dispatch(ctx, lp, &o, x_dev, y_dev, res, nullptr);
}

extern "C" int teccl_pdlp_solve(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                                double* x_inout, double* y_inout, teccl_pdlp_result* res) {
  if (!ctx || !lp || !res) { set_error("null argument"); return TECCL_EINVAL; }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  double *xd = nullptr, *yd = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&xd, sizeof(double) * (lp->n + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&yd, sizeof(double) * (lp->m + 1), st));
  const bool warm = opts && opts->warm_start;
  if (warm) {
    if (!x_inout || !y_inout) { set_error("warm start needs x and y"); return TECCL_EINVAL; }
    TECCL_CUDA(cudaMemcpyAsync(xd, x_inout, sizeof(double) * lp->n, cudaMemcpyHostToDevice, st));
    TECCL_CUDA(cudaMemcpyAsync(yd, y_inout, sizeof(double) * lp->m, cudaMemcpyHostToDevice, st));
  }
  int rc = teccl_pdlp_solve_dev(ctx, lp, opts, xd, yd, res);
  if (rc == TECCL_OK) {
    if (x_inout) TECCL_CUDA(cudaMemcpyAsync(x_inout, xd, sizeof(double) * lp->n, cudaMemcpyDeviceToHost, st));
    if (y_inout) TECCL_CUDA(cudaMemcpyAsync(y_inout, yd, sizeof(double) * lp->m, cudaMemcpyDeviceToHost, st));
  }
  cudaFreeAsync(xd, st);
  cudaFreeAsync(yd, st);
  TECCL_CUDA(cudaStreamSynchronize(st));
  return rc;
}

extern "C" int teccl_pdlp_step_bench_opts(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                                          int32_t reps, double* out6) {
  if (!ctx || !lp || reps < 1 || !out6) { set_error("bad argument"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  teccl_pdlp_opts o;
  if (opts) o = *opts; else teccl_pdlp_default_opts(&o);
  teccl_pdlp_result res{};
  double* xd = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&xd, sizeof(double) * (lp->n + 1), ctx->stream));
  StepBench sb{reps, 0, 0, 0, 0, 0};
  int rc = dispatch(ctx, lp, &o, xd, nullptr, &res, &sb);
  cudaFreeAsync(xd, ctx->stream);
  TECCL_CUDA(cudaStreamSynchronize(ctx->stream));
  out6[0] = sb.ms_col; out6[1] = sb.ms_row; out6[2] = sb.bytes_col; out6[3] = sb.bytes_row;
  // operator: 0 stored + bound arrays, 1 stored + bound-class dictionaries,
  // 2/3/4 matrix-free (teccl_pdlp_opts.matrix_free modes)
  out6[4] = sb.matrix_free ? (double)sb.matrix_free : (lp->col_code && lp->row_code) ? 1.0 : 0.0;
  out6[5] = (double)kSlice;
  return rc;
}

extern "C" int teccl_pdlp_step_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* out6) {
  return teccl_pdlp_step_bench_opts(ctx, lp, nullptr, reps, out6);
}

namespace teccl {
// out = A.in (rows) or A^T.in (columns) through the matrix-free operator,
// with the bounds (and costs) that operator computes
__global__ void te_apply_kernel(TeOp op, int transpose, const double* __restrict__ in,
                                double* out, double* lo, double* hi, double* c) {
  const uint32_t count = transpose ? op.n : op.m;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double a, b, cc = 0.0;
    const double v = transpose ? te_col(op, i, in, a, b, cc) : te_row(op, i, in, a, b);
    out[i] = v;
    lo[i] = a;
    hi[i] = b;
    if (transpose) c[i] = cc;
  }
}

__global__ void em_apply_kernel(EmOp op, int transpose, const double* __restrict__ in,
                                double* out, double* lo, double* hi, double* c) {
  const uint32_t count = transpose ? op.n : op.m;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double a, b, cc = 0.0;
    const double v = transpose ? em_col(op, i, in, a, b, cc) : em_row(op, i, in, a, b);
    out[i] = v;
    lo[i] = a;
    hi[i] = b;
    if (transpose) c[i] = cc;
  }
}

__global__ void seg_apply_kernel(TeOp op, int transpose, const double* __restrict__ in,
                                 double* out, double* lo, double* hi, double* c) {
  const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int nt = transpose ? op.n_ctask : op.n_rtask;
  if (wi >= nt) return;
  const int4 tk = __ldg((transpose ? op.ctask : op.rtask) + wi);
  double a[kSegPerLane], l[kSegPerLane], u[kSegPerLane], cc[kSegPerLane];
  if (transpose) seg_cols(op, tk, lane, in, a, l, u, cc);
  else seg_rows(op, tk, lane, in, a, l, u);
  for (int h = 0; h < kSegPerLane; ++h) {
    const int i = lane + 32 * h;
    if (i < seg_count(tk)) {
      const uint32_t r = (uint32_t)tk.z + i;
      out[r] = a[h];
      lo[r] = l[h];
      hi[r] = u[h];
      if (transpose) c[r] = cc[h];
    }
  }
}
}  // namespace teccl

extern "C" int teccl_lp_apply(teccl_ctx* ctx, teccl_lp* lp, int32_t transpose, int32_t matrix_free,
                              const double* in, double* out, double* lo, double* hi, double* cost) {
  if (!ctx || !lp || !in || !out) { set_error("null argument"); return TECCL_EINVAL; }
  if (matrix_free && !lp->te) { set_error("LP has no matrix-free operator (not built by teccl_lp_build_te)"); return TECCL_EINVAL; }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  // inputs are gather windows (the whole vector on one device)
  const int64_t nin = transpose ? gather_rows(lp) : gather_cols(lp), nout = transpose ? lp->n : lp->m;
  double *din = nullptr, *dout = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&din, sizeof(double) * (nin + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&dout, sizeof(double) * 4 * (nout + 1), st));
  TECCL_CUDA(cudaMemcpyAsync(din, in, sizeof(double) * nin, cudaMemcpyHostToDevice, st));
  double *dlo = dout + (nout + 1), *dhi = dlo + (nout + 1), *dc = dhi + (nout + 1);
  if (matrix_free && ((TeHold*)lp->te)->kind == 1) {
    em_apply_kernel<<<grid_for(nout), kThreads, 0, st>>>(((TeHold*)lp->te)->em, transpose, din, dout, dlo, dhi, dc);
  } else if (matrix_free == 2) {
    const TeOp& op = ((TeHold*)lp->te)->op;
    const int nt = transpose ? op.n_ctask : op.n_rtask;
    seg_apply_kernel<<<(nt + 7) / 8, kThreads, 0, st>>>(op, transpose, din, dout, dlo, dhi, dc);
  } else if (matrix_free) {
    te_apply_kernel<<<grid_for(nout), kThreads, 0, st>>>(((TeHold*)lp->te)->op, transpose, din, dout, dlo, dhi, dc);
  } else {
    if (lp->unit) {
      if (transpose) spmv_scaled_kernel<true><<<grid_for(nout), kThreads, 0, st>>>(nout, lp->col_ptr, lp->row, lp->cval, din, nullptr, dout);
      else spmv_scaled_kernel<true><<<grid_for(nout), kThreads, 0, st>>>(nout, lp->row_ptr, lp->col, lp->val, din, nullptr, dout);
    } else {
      if (transpose) spmv_scaled_kernel<false><<<grid_for(nout), kThreads, 0, st>>>(nout, lp->col_ptr, lp->row, lp->cval, din, nullptr, dout);
      else spmv_scaled_kernel<false><<<grid_for(nout), kThreads, 0, st>>>(nout, lp->row_ptr, lp->col, lp->val, din, nullptr, dout);
    }
    TECCL_CUDA(cudaMemcpyAsync(dlo, transpose ? lp->var_lb : lp->row_lo, sizeof(double) * nout, cudaMemcpyDeviceToDevice, st));
    TECCL_CUDA(cudaMemcpyAsync(dhi, transpose ? lp->var_ub : lp->row_hi, sizeof(double) * nout, cudaMemcpyDeviceToDevice, st));
    if (transpose) TECCL_CUDA(cudaMemcpyAsync(dc, lp->obj, sizeof(double) * nout, cudaMemcpyDeviceToDevice, st));
  }
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
  if (lo) TECCL_CUDA(cudaMemcpyAsync(lo, dlo, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
  if (hi) TECCL_CUDA(cudaMemcpyAsync(hi, dhi, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
  if (cost && transpose) TECCL_CUDA(cudaMemcpyAsync(cost, dc, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(din, st);
  cudaFreeAsync(dout, st);
  TECCL_CUDA(cudaStreamSynchronize(st));
  return TECCL_OK;
}

extern "C" int teccl_spmv_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* ms_per_pair,
                                double* bytes_per_pair) {
  if (!ctx || !lp || reps < 1) { set_error("bad argument"); return TECCL_EINVAL; }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  const int32_t m = lp->m, n = lp->n;
  double *vx = nullptr, *vy = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&vx, sizeof(double) * (n + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&vy, sizeof(double) * (m + 1), st));
  const int gr = grid_for(m > n ? m : n);
  hash_fill_kernel<<<gr, kThreads, 0, st>>>(n, vx);
  cudaEvent_t a, b;
  TECCL_CUDA(cudaEventCreate(&a));
  TECCL_CUDA(cudaEventCreate(&b));
  for (int it = -3; it < reps; ++it) {
    if (it == 0) TECCL_CUDA(cudaEventRecord(a, st));
    if (lp->unit) {
      spmv_scaled_kernel<true><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, vx, nullptr, vy);
      spmv_scaled_kernel<true><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, vy, nullptr, vx);
    } else {
      spmv_scaled_kernel<false><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, vx, nullptr, vy);
      spmv_scaled_kernel<false><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, vy, nullptr, vx);
    }
  }
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaEventRecord(b, st));
  TECCL_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  TECCL_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_pair = ms / reps;
  const double vb = lp->unit ? 4.0 : 12.0;
  *bytes_per_pair = 2.0 * lp->nnz * vb + 8.0 * (m + 1) + 8.0 * (n + 1) + 2.0 * 8.0 * (m + n);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(vx, st);
  cudaFreeAsync(vy, st);
  TECCL_CUDA(cudaStreamSynchronize(st));
  return TECCL_OK;
}

extern "C" int teccl_dist_export(teccl_ctx* ctx, teccl_lp* lp, uint8_t* blob, int64_t* blob_len) {
  if (!ctx || !lp || !blob || !blob_len) { set_error("null argument"); return TECCL_EINVAL; }
  if (lp->part_world < 2) { set_error("LP is not row-partitioned"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  DistState* ds = (DistState*)lp->dist;
  if (!ds) {
    ds = new DistState();
    ds->world = lp->part_world;
    ds->rank = lp->part_rank;
    ds->device = ctx->device;
    const int64_t ncw = gather_cols(lp), nrw = gather_rows(lp);
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    int64_t off = 0;
    ds->meta[M_NCW] = ncw;
    ds->meta[M_NRW] = nrw;
    for (int id = 0; id < A_NARR; ++id) {
      ds->meta[M_OFF0 + id] = off;
      off += al(8 * ((ds->is_col(id) ? ncw : nrw) + 1));
    }
    ds->meta[M_FLAGS] = off; off += al(8 * ds->world);
    ds->meta[M_SLOTS] = off; off += al(8 * kSlots * ds->world);
    ds->meta[M_SEQ] = off; off += 256;
    ds->meta[M_ARRIVE] = off; off += 256;
    ds->meta[M_OC0] = lp->own_c0; ds->meta[M_OC1] = lp->own_c1;
    ds->meta[M_OR0] = lp->own_r0; ds->meta[M_OR1] = lp->own_r1;
    ds->meta[M_WC0] = lp->win_c0; ds->meta[M_WC1] = lp->win_c1;
    ds->meta[M_WR0] = lp->win_r0; ds->meta[M_WR1] = lp->win_r1;
    ds->meta[M_RANK] = ds->rank;
    ds->meta[M_WORLD] = ds->world;
    if (cudaMalloc((void**)&ds->arena, off) != cudaSuccess) {
      delete ds;
      set_error("cannot allocate the peer-exchange arena");
      return TECCL_ENOMEM;
    }
    TECCL_CUDA(cudaMemset(ds->arena, 0, off));
    lp->dist = ds;
    lp->dist_free = free_dist;
  }
  cudaIpcMemHandle_t h;
  TECCL_CUDA(cudaIpcGetMemHandle(&h, ds->arena));
  memcpy(blob, &h, sizeof(h));
  memcpy(blob + sizeof(h), ds->meta, kMetaLen * 8);
  *blob_len = kBlobLen;
  return TECCL_OK;
}

extern "C" int teccl_dist_connect(teccl_ctx* ctx, teccl_lp* lp, const uint8_t* blobs,
                                  int64_t blob_len) {
  if (!ctx || !lp || !blobs || blob_len != kBlobLen) { set_error("bad argument"); return TECCL_EINVAL; }
  DistState* ds = (DistState*)lp->dist;
  if (!ds) { set_error("call teccl_dist_export first"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  const int W = ds->world, me = ds->rank;
  ds->peer_meta.assign(W, {});
  ds->peer_base.assign(W, nullptr);
  for (int q = 0; q < W; ++q) {
    const uint8_t* b = blobs + (int64_t)q * kBlobLen;
    memcpy(ds->peer_meta[q].data(), b + sizeof(cudaIpcMemHandle_t), kMetaLen * 8);
    if (ds->peer_meta[q][M_RANK] != q || ds->peer_meta[q][M_WORLD] != W) {
      set_error("peer blobs out of rank order or from another world");
      return TECCL_EINVAL;
    }
    if (q == me) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, b, sizeof(h));
    void* ptr = nullptr;
    TECCL_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    ds->peer_base[q] = (char*)ptr;
  }
  std::vector<double*> ps;
  int na = 0;
  for (int q = 0; q < W; ++q) {
    if (q == me) continue;
    char* base = ds->peer_base[q];
    unsigned long long* their_flag = (unsigned long long*)(base + ds->peer_meta[q][M_FLAGS]) + me;
    ps.push_back((double*)(base + ds->peer_meta[q][M_SLOTS]));
    if (na < kMaxPeers) {
      ds->sig_all.peer_flag[na] = their_flag;
      ds->wait_all.peer[na] = q;
      ++na;
    }
    if (q == me - 1 || q == me + 1) {
      ds->sig_nbr.peer_flag[ds->sig_nbr.npeer++] = their_flag;
      ds->wait_nbr.peer[ds->wait_nbr.npeer++] = q;
    }
  }
  if (W - 1 > kMaxPeers) { set_error("more than 9 ranks are not supported"); return TECCL_EINVAL; }
  ds->sig_all.npeer = na;
  ds->wait_all.npeer = na;
  unsigned long long* seq = (unsigned long long*)(ds->arena + ds->meta[M_SEQ]);
  unsigned int* arrive = (unsigned int*)(ds->arena + ds->meta[M_ARRIVE]);
  const unsigned long long* flags = (const unsigned long long*)(ds->arena + ds->meta[M_FLAGS]);
  ds->sig_nbr.seq = ds->sig_all.seq = seq;
  ds->sig_nbr.arrive = ds->sig_all.arrive = arrive;
  ds->wait_nbr.flags = ds->wait_all.flags = flags;
  ds->wait_nbr.seq = ds->wait_all.seq = seq;
  if (ds->d_peer_slots) cudaFree(ds->d_peer_slots);
  TECCL_CUDA(cudaMalloc((void**)&ds->d_peer_slots, sizeof(double*) * std::max<size_t>(1, ps.size())));
  if (!ps.empty())
    TECCL_CUDA(cudaMemcpy(ds->d_peer_slots, ps.data(), sizeof(double*) * ps.size(), cudaMemcpyHostToDevice));
  ds->connected = true;
  return TECCL_OK;
}

// ---------------------------------------------------------------------------
// Source-partitioned solve of a whole single-device TE LP (SrcState).
constexpr int kSrcMeta = 8;  // rank, world, ncap, off_flags, off_slots, off_seq, off_arrive, bytes
constexpr int kSrcBlob = (int)sizeof(cudaIpcMemHandle_t) + kSrcMeta * 8;

extern "C" int teccl_src_setup(teccl_ctx* ctx, teccl_lp* lp, int32_t world, int32_t rank, int64_t* info8) {
  if (!ctx || !lp || !info8) { set_error("null argument"); return TECCL_EINVAL; }
  if (world < 1 || rank < 0 || rank >= world || world - 1 > kMaxPeers) { set_error("bad world/rank"); return TECCL_EINVAL; }
  const TeHold* hold = (const TeHold*)lp->te;
  if (!hold || hold->kind != 0 || lp->part_world != 1) {
    set_error("source partition needs a whole LP built by teccl_lp_build_te");
    return TECCL_EINVAL;
  }
  if (lp->src) { set_error("LP already source-partitioned"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  if (lp->pdlp_ws && lp->ws_free) {  // the partitioned iteration needs more partial slots
    lp->ws_free(lp->pdlp_ws);
    lp->pdlp_ws = nullptr;
  }
  const TeOp& op = hold->op;
  const uint32_t S = op.S, P = (uint32_t)op.d.P, K = op.K;
  std::vector<int> psrc(P);
  if (P) TECCL_CUDA(cudaMemcpy(psrc.data(), op.d.pair_src, sizeof(int) * P, cudaMemcpyDeviceToHost));
  for (uint32_t p = 1; p < P; ++p)
    if (psrc[p] < psrc[p - 1]) { set_error("pairs are not grouped by source"); return TECCL_EINVAL; }
  SrcState* sp = new SrcState();
  sp->world = world; sp->rank = rank; sp->device = ctx->device;
  sp->s0 = (uint32_t)((int64_t)rank * S / world);
  sp->s1 = (uint32_t)((int64_t)(rank + 1) * S / world);
  sp->p0 = (uint32_t)(std::lower_bound(psrc.begin(), psrc.end(), (int)sp->s0) - psrc.begin());
  sp->p1 = (uint32_t)(std::lower_bound(psrc.begin(), psrc.end(), (int)sp->s1) - psrc.begin());
  OwnMask& M = sp->mask;
  M.on = 1;
  M.s0 = sp->s0; M.s1 = sp->s1;
  M.rc0 = op.R_cons + sp->s0 * op.CB; M.rc1 = op.R_cons + sp->s1 * op.CB;
  M.rm0 = op.R_cum + sp->p0 * K; M.rm1 = op.R_cum + sp->p1 * K;
  M.c0 = sp->s0 * op.SB; M.c1 = sp->s1 * op.SB;
  M.q0 = op.nF + 2 * K * sp->p0; M.q1 = op.nF + 2 * K * sp->p1;
  sp->ncap_e = op.EK;
  sp->ncap = op.EK + (op.has_bcap ? (uint32_t)op.d.G * (K + 1) : 0u);
  // segment tasks: own init / conservation / cumulative rows; all capacity rows
  std::vector<int4> rt(op.n_rtask), own, cap;
  if (op.n_rtask)
    TECCL_CUDA(cudaMemcpy(rt.data(), op.rtask, sizeof(int4) * op.n_rtask, cudaMemcpyDeviceToHost));
  for (uint32_t s = sp->s0; s < sp->s1; s += kSegTask) {
    const uint32_t c = std::min<uint32_t>(kSegTask, sp->s1 - s);
    own.push_back(make_int4(SEG_INIT, 0, (int)s, (int)(s | (c << 24))));
  }
  for (const int4& t : rt) {
    const int kind = t.x & 15, A = t.x >> 4;
    if (kind == SEG_CONS && (uint32_t)A >= sp->s0 && (uint32_t)A < sp->s1) own.push_back(t);
    else if (kind == SEG_CUM && (uint32_t)A >= sp->p0 && (uint32_t)A < sp->p1) own.push_back(t);
    else if (kind == SEG_CAP || kind == SEG_BCAP) cap.push_back(t);
  }
  sp->n_own = (int)own.size();
  sp->n_cap = (int)cap.size();
  auto up = [](const std::vector<int4>& v, int4** d) -> bool {
    if (cudaMalloc((void**)d, sizeof(int4) * std::max<size_t>(1, v.size())) != cudaSuccess) return false;
    return v.empty() || cudaMemcpy(*d, v.data(), sizeof(int4) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up(own, &sp->own_tasks) || !up(cap, &sp->cap_tasks)) { delete sp; set_error("task upload failed"); return TECCL_ECUDA; }
  auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
  int64_t off = al(8LL * 4 * world * sp->ncap);
  sp->off_flags = off; off += al(8LL * world);
  sp->off_slots = off; off += al(8LL * kSlots * world);
  sp->off_seq = off; off += 256;
  sp->off_arrive = off; off += 256;
  sp->bytes = off;
  if (cudaMalloc((void**)&sp->arena, off) != cudaSuccess) { delete sp; set_error("cannot allocate the source-partition arena"); return TECCL_ENOMEM; }
  if (cudaMemset(sp->arena, 0, off) != cudaSuccess) { delete sp; set_error("memset failed"); return TECCL_ECUDA; }
  lp->src = sp;
  lp->src_free = free_src;
  const int64_t v[8] = {sp->s0, sp->s1, sp->p0, sp->p1, M.c0, M.c1, M.q0, M.q1};
  for (int i = 0; i < 8; ++i) info8[i] = v[i];
  return TECCL_OK;
}

extern "C" int teccl_src_export(teccl_ctx* ctx, teccl_lp* lp, uint8_t* blob, int64_t* blob_len) {
  if (!ctx || !lp || !blob || !blob_len) { set_error("null argument"); return TECCL_EINVAL; }
  SrcState* sp = (SrcState*)lp->src;
  if (!sp) { set_error("call teccl_src_setup first"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  TECCL_CUDA(cudaIpcGetMemHandle(&h, sp->arena));
  const int64_t meta[kSrcMeta] = {sp->rank, sp->world, sp->ncap, sp->off_flags, sp->off_slots,
                                   sp->off_seq, sp->off_arrive, sp->bytes};
  memcpy(blob, &h, sizeof(h));
  memcpy(blob + sizeof(h), meta, sizeof(meta));
  *blob_len = kSrcBlob;
  return TECCL_OK;
}

extern "C" int teccl_src_connect(teccl_ctx* ctx, teccl_lp* lp, const uint8_t* blobs, int64_t blob_len) {
  if (!ctx || !lp || !blobs || blob_len != kSrcBlob) { set_error("bad argument"); return TECCL_EINVAL; }
  SrcState* sp = (SrcState*)lp->src;
  if (!sp) { set_error("call teccl_src_setup first"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  const int W = sp->world, me = sp->rank;
  sp->peer_base.assign(W, nullptr);
  std::vector<double*> bufs(W), ps;
  int na = 0;
  for (int q = 0; q < W; ++q) {
    int64_t meta[kSrcMeta];
    memcpy(meta, blobs + (int64_t)q * kSrcBlob + sizeof(cudaIpcMemHandle_t), sizeof(meta));
    if (meta[0] != q || meta[1] != W || meta[2] != (int64_t)sp->ncap || meta[7] != sp->bytes) {
      set_error("peer blobs out of rank order or from another LP / world");
      return TECCL_EINVAL;
    }
    char* base = sp->arena;
    if (q != me) {
      cudaIpcMemHandle_t h;
      memcpy(&h, blobs + (int64_t)q * kSrcBlob, sizeof(h));
      void* ptr = nullptr;
      TECCL_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      sp->peer_base[q] = (char*)ptr;
      base = (char*)ptr;
      ps.push_back((double*)(base + sp->off_slots));
      sp->sig.peer_flag[na] = (unsigned long long*)(base + sp->off_flags) + me;
      sp->wait.peer[na] = q;
      ++na;
    }
    bufs[q] = (double*)base;
  }
  sp->sig.npeer = na;
  sp->wait.npeer = na;
  sp->sig.seq = (unsigned long long*)(sp->arena + sp->off_seq);
  sp->sig.arrive = (unsigned int*)(sp->arena + sp->off_arrive);
  sp->wait.flags = (const unsigned long long*)(sp->arena + sp->off_flags);
  sp->wait.seq = sp->sig.seq;
  TECCL_CUDA(cudaMalloc((void**)&sp->d_bufs, sizeof(double*) * W));
  TECCL_CUDA(cudaMemcpy(sp->d_bufs, bufs.data(), sizeof(double*) * W, cudaMemcpyHostToDevice));
  TECCL_CUDA(cudaMalloc((void**)&sp->d_peer_slots, sizeof(double*) * std::max<size_t>(1, ps.size())));
  if (!ps.empty())
    TECCL_CUDA(cudaMemcpy(sp->d_peer_slots, ps.data(), sizeof(double*) * ps.size(), cudaMemcpyHostToDevice));
  sp->connected = true;
  return TECCL_OK;
}

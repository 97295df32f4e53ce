// (2)+(3) Restarted reflected-Halpern PDHG (PDLP family) on sm_100a.
//
// Replaces the CPU LP solve of the reference (pkg/src/collsched/solver.py:
// 119-137, scipy.optimize.milp -> HiGHS) for the TE-CCL LP. One iteration is
// two fused kernels:
//   col_step: A^T.y SpMV over the CSC + primal step, projection onto bounds,
//             reflection and Halpern averaging, emits C.(2x'-x) for the gather
//   row_step: A.xbar SpMV over the CSR + dual step, projection onto the row
//             bounds, Halpern averaging, emits R.y for the next gather
// Every `check_every` iterations the chunk ends with KKT kernels (unscaled
// residuals, objectives) and a single-block control kernel that decides
// termination, restarts and the primal weight on the device, so the host
// never sits in the iteration loop. Chunks are replayed from a CUDA graph.
//
// Scaled problem: x = beta * C.xs, y = gamma * R.ys with
// R, C from Ruiz + Pock-Chambolle equilibration, beta = ||b_s||+1,
// gamma = ||c_s||+1. The matrix is never rewritten: R and C are folded into
// the gathered vectors, so the unit (+-1) TE-CCL matrix streams 4 bytes/nnz.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include "common.cuh"

namespace teccl {

constexpr int kGrid = kSMs * 8;  // blocks of every reduction-bearing kernel
constexpr int kNQ = 9;           // partial quantities per check

enum Q { Q_DX = 0, Q_DX0, Q_DY, Q_DY0, Q_RP, Q_DOBJ_ROW, Q_RD, Q_POBJ, Q_DOBJ_COL };

struct PdlpState {
  double tau, sigma, omega, eta, refl;
  double beta, gamma;        // bound / objective rescaling
  double bnorm, cnorm;       // unscaled norms for the relative criteria
  double eps;
  double r0, rprev, last_r;
  long long k_inner, total;
  int have_r0, restart, done, restarts, chunk_len, pad;
  double rel_p, rel_d, gap, pobj, dobj;
};

struct Vecs {
  // problem (scaled)
  const double *c, *lb, *ub, *lo, *hi, *R, *C;
  // iterates
  double *x, *x0, *xt, *cxb, *cxt;
  double *y, *y0, *yt, *ry, *ryt;
  // unscaled data for KKT
  const double *c_u, *lb_u, *ub_u, *lo_u, *hi_u;
  double* part;    // [kNQ * pstride]
  int64_t pstride; // partial slots per quantity (>= every grid)
  int nb_row, nb_col;  // blocks of the row / column tile kernels
  PdlpState* st;
};

// ---------------------------------------------------------------------------
// SELL-32 SpMV. The iteration matrices are re-laid out once per LP as
// sliced ELLPACK with slice height 32 (one warp): slice s holds rows
// 32s..32s+31, padded to the slice's longest row, stored column-major inside
// the slice, so entry q of every row of a warp sits in one 128-byte line.
// Padding entries point at a sentinel vector element that is always 0.
// Index loads are perfectly coalesced, trip counts are warp-uniform, no
// shared memory or barriers are needed, and the row order is unchanged so the
// epilogue stays thread-per-row (padding: 2 % rows, 9 % columns on configs[1]).
constexpr int kSlice = 32;
constexpr int kTile = kThreads;  // rows (columns) per block of the step kernels

struct SellView {
  const int64_t* off;    // [nslices] first entry of the slice
  const int32_t* width;  // [nslices] entries per row in the slice
  const uint32_t* idx;   // slice-major, column-major inside a slice
  const double* val;     // explicit coefficients (nullptr for unit LPs)
  int64_t count;         // rows (or columns)
};

template <bool UNIT>
__device__ __forceinline__ double sell_dot(const SellView& S, int64_t r,
                                           const double* __restrict__ v) {
  const int64_t s = r >> 5;
  const int w = __ldg(S.width + s);
  const int64_t base = __ldg(S.off + s) + (r & 31);
  double acc = 0.0;
  int q = 0;
  for (; q + 4 <= w; q += 4) {
    uint32_t t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = __ldg(S.idx + base + (int64_t)(q + u) * kSlice);
    double g[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (UNIT) {
        const double xv = __ldg(v + (t[u] & kIdxMask));
        g[u] = (t[u] & kSignBit) ? -xv : xv;
      } else {
        g[u] = __ldg(S.val + base + (int64_t)(q + u) * kSlice) * __ldg(v + t[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += g[u];
  }
  for (; q < w; ++q) {
    const uint32_t t = __ldg(S.idx + base + (int64_t)q * kSlice);
    if (UNIT) {
      const double xv = __ldg(v + (t & kIdxMask));
      acc += (t & kSignBit) ? -xv : xv;
    } else {
      acc += __ldg(S.val + base + (int64_t)q * kSlice) * __ldg(v + t);
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

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return fmin(fmax(v, lo), hi);
}

// ---------------------------------------------------------------------------
// Primal half-step over columns (CSC), fused with A^T.y.
template <bool UNIT, bool CHECK>
__global__ void __launch_bounds__(kThreads) col_step_kernel(
    int32_t n, SellView S, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done) return;
  const double tau = st->tau, refl = st->refl;
  const double kk = (double)(st->k_inner + j_in_chunk);
  const double lam = (kk + 1.0) / (kk + 2.0);
  const int64_t j = (int64_t)blockIdx.x * kTile + threadIdx.x;
  // epilogue operands do not depend on the SpMV: issue their loads first
  double Cj = 0.0, xj = 0.0, cj = 0.0, lbj = 0.0, ubj = 0.0, x0 = 0.0;
  if (j < n) {
    Cj = V.C[j]; xj = V.x[j]; cj = V.c[j]; lbj = V.lb[j]; ubj = V.ub[j]; x0 = V.x0[j];
  }
  const double s = (j < n) ? sell_dot<UNIT>(S, j, V.ry) : 0.0;
  double dx = 0.0, dx0 = 0.0;
  if (j < n) {
    const double xt = clampd(xj - tau * (cj - Cj * s), lbj, ubj);
    V.cxb[j] = Cj * (2.0 * xt - xj);
    V.x[j] = lam * ((1.0 + refl) * xt - refl * xj) + (1.0 - lam) * x0;
    if (CHECK) {
      V.xt[j] = xt;
      V.cxt[j] = Cj * xt;
      dx = (xt - xj) * (xt - xj);
      dx0 = (xt - x0) * (xt - x0);
    }
  }
  if (CHECK) {
    double a = block_sum(dx, sh);
    if (threadIdx.x == 0) V.part[Q_DX * V.pstride + blockIdx.x] = a;
    a = block_sum(dx0, sh);
    if (threadIdx.x == 0) V.part[Q_DX0 * V.pstride + blockIdx.x] = a;
  }
}

// Dual half-step over rows (CSR), fused with A.xbar.
template <bool UNIT, bool CHECK>
__global__ void __launch_bounds__(kThreads) row_step_kernel(
    int32_t m, SellView S, Vecs V, int j_in_chunk) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done) return;
  const double sigma = st->sigma, refl = st->refl;
  const double kk = (double)(st->k_inner + j_in_chunk);
  const double lam = (kk + 1.0) / (kk + 2.0);
  const int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  double Ri = 0.0, yi = 0.0, loi = 0.0, hii = 0.0, y0 = 0.0;
  if (i < m) {
    Ri = V.R[i]; yi = V.y[i]; loi = V.lo[i]; hii = V.hi[i]; y0 = V.y0[i];
  }
  const double s = (i < m) ? sell_dot<UNIT>(S, i, V.cxb) : 0.0;
  double dy = 0.0, dy0 = 0.0;
  if (i < m) {
    const double v = Ri * s;
    const double yt = yi - sigma * (v - clampd(v - yi / sigma, loi, hii));
    const double yn = lam * ((1.0 + refl) * yt - refl * yi) + (1.0 - lam) * y0;
    V.y[i] = yn;
    V.ry[i] = Ri * yn;
    if (CHECK) {
      V.yt[i] = yt;
      V.ryt[i] = Ri * yt;
      dy = (yt - yi) * (yt - yi);
      dy0 = (yt - y0) * (yt - y0);
    }
  }
  if (CHECK) {
    double a = block_sum(dy, sh);
    if (threadIdx.x == 0) V.part[Q_DY * V.pstride + blockIdx.x] = a;
    a = block_sum(dy0, sh);
    if (threadIdx.x == 0) V.part[Q_DY0 * V.pstride + blockIdx.x] = a;
  }
}

// KKT over rows at T(z): primal residual of A.x_u and the row part of the
// dual objective.
template <bool UNIT>
__global__ void __launch_bounds__(kThreads) kkt_row_kernel(
    int32_t m, SellView S, Vecs V) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done) return;
  const double beta = st->beta, gamma = st->gamma;
  const int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const double s = (i < m) ? sell_dot<UNIT>(S, i, V.cxt) : 0.0;
  double rp = 0.0, dobj = 0.0;
  if (i < m) {
    const double ax = beta * s;
    const double lo = V.lo_u[i], hi = V.hi_u[i];
    const double r = ax - clampd(ax, lo, hi);
    rp = r * r;
    const double yu = gamma * V.ryt[i];
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
template <bool UNIT>
__global__ void __launch_bounds__(kThreads) kkt_col_kernel(
    int32_t n, SellView S, Vecs V) {
  __shared__ double sh[32];
  const PdlpState* st = V.st;
  if (st->done) return;
  const double beta = st->beta, gamma = st->gamma;
  const int64_t j = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const double s = (j < n) ? sell_dot<UNIT>(S, j, V.ryt) : 0.0;
  double rd = 0.0, pobj = 0.0, dobj = 0.0;
  if (j < n) {
    const double cj = V.c_u[j];
    const double g = cj - gamma * s;
    const double lb = V.lb_u[j], ub = V.ub_u[j];
    double lamb = 0.0;
    if (g > 0.0 && isfinite(lb)) lamb = g;
    else if (g < 0.0 && isfinite(ub)) lamb = g;
    const double r = g - lamb;
    rd = r * r;
    pobj = cj * beta * V.cxt[j];
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

// Single block: reduce the partials in a fixed order, evaluate termination,
// decide restarts and update the primal weight. All of PDLP's control flow.
__global__ void __launch_bounds__(1024) control_kernel(Vecs V) {
  __shared__ double sh[32];
  __shared__ double q[kNQ];
  PdlpState* st = V.st;
  if (st->done) return;
  for (int k = 0; k < kNQ; ++k) {
    const bool row_q = (k == Q_DY || k == Q_DY0 || k == Q_RP || k == Q_DOBJ_ROW);
    const int nb = row_q ? V.nb_row : V.nb_col;
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += V.part[k * V.pstride + b];
    a = block_sum(a, sh);
    if (threadIdx.x == 0) q[k] = a;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double w = st->omega;
  const double r = sqrt(w * q[Q_DX] + q[Q_DY] / w);
  const double pobj = q[Q_POBJ];
  const double dobj = q[Q_DOBJ_ROW] + q[Q_DOBJ_COL];
  st->rel_p = sqrt(q[Q_RP]) / (1.0 + st->bnorm);
  st->rel_d = sqrt(q[Q_RD]) / (1.0 + st->cnorm);
  st->gap = fabs(pobj - dobj) / (1.0 + fabs(pobj) + fabs(dobj));
  st->pobj = pobj;
  st->dobj = dobj;
  st->last_r = r;
  st->total += st->chunk_len;
  st->k_inner += st->chunk_len;
  st->restart = 0;
  if (!isfinite(r) || !isfinite(pobj)) { st->done = 2; return; }
  if (st->rel_p <= st->eps && st->rel_d <= st->eps && st->gap <= st->eps) {
    st->done = 1;
    return;
  }
  if (!st->have_r0) {
    st->r0 = r;
    st->have_r0 = 1;
    st->rprev = r;
  }
  const bool sufficient = r <= 0.2 * st->r0;
  const bool necessary = r <= 0.8 * st->r0 && r > st->rprev;
  const bool artificial = (double)st->k_inner >= 0.36 * (double)st->total;
  st->rprev = r;
  if (sufficient || necessary || artificial) {
    st->restart = 1;
    st->restarts += 1;
    st->k_inner = 0;
    st->have_r0 = 0;
    const double dxr = sqrt(q[Q_DX0]), dyr = sqrt(q[Q_DY0]);
    if (dxr > 1e-10 && dyr > 1e-10) {
      const double lw = 0.5 * log(dyr / dxr) + 0.5 * log(w);
      st->omega = exp(lw);
      st->tau = st->eta / st->omega;
      st->sigma = st->eta * st->omega;
    }
  }
}

// Restart: z <- z0 <- T(z).
__global__ void restart_x_kernel(int32_t n, Vecs V) {
  if (V.st->done || !V.st->restart) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double xt = V.xt[j];
    V.x[j] = xt;
    V.x0[j] = xt;
  }
}
__global__ void restart_y_kernel(int32_t m, Vecs V) {
  if (V.st->done || !V.st->restart) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yt = V.yt[i];
    V.y[i] = yt;
    V.y0[i] = yt;
    V.ry[i] = V.ryt[i];
  }
}

// ---------------------------------------------------------------------------
// Setup kernels: equilibration statistics, scaled data, power iteration.

// stat[r] = max (MAX=true) or sum of |a_rj| * s_j over the row/column
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

// Scaled column data: c_s = C c, lb_s = lb / C, ub_s = ub / C (before beta/gamma).
__global__ void scale_cols_kernel(int32_t n, const double* C, const double* c, const double* lb,
                                  const double* ub, double* cs, double* lbs, double* ubs,
                                  double* part) {
  __shared__ double sh[32];
  double cc = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double Cj = C[j];
    cs[j] = c[j] * Cj;
    lbs[j] = lb[j] / Cj;
    ubs[j] = ub[j] / Cj;
    cc += cs[j] * cs[j];
  }
  double a = block_sum(cc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__device__ __forceinline__ double bound_ref(double lo, double hi) {
  if (isfinite(hi)) return hi;
  if (isfinite(lo)) return lo;
  return 0.0;
}

__global__ void scale_rows_kernel(int32_t m, const double* R, const double* lo, const double* hi,
                                  double* los, double* his, double* part_s, double* part_u) {
  __shared__ double sh[32];
  double bs = 0.0, bu = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double Ri = R[i];
    los[i] = lo[i] * Ri;
    his[i] = hi[i] * Ri;
    const double b = bound_ref(lo[i], hi[i]);
    bs += (b * Ri) * (b * Ri);
    bu += b * b;
  }
  double a = block_sum(bs, sh);
  if (threadIdx.x == 0) part_s[blockIdx.x] = a;
  a = block_sum(bu, sh);
  if (threadIdx.x == 0) part_u[blockIdx.x] = a;
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

__global__ void scale_inplace_kernel(int64_t count, double* v, double s) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] *= s;
}

// out_r = self_r * sum_j a_rj * in_j   (in already carries the other side's scale)
template <bool UNIT>
__global__ void spmv_scaled_kernel(int64_t count, const int64_t* __restrict__ ptr,
                                   const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                   const double* __restrict__ in, const double* __restrict__ self,
                                   const double* __restrict__ post, double* __restrict__ out,
                                   double* __restrict__ out_post) {
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
    const double o = self[r] * acc;
    out[r] = o;
    if (out_post) out_post[r] = post[r] * o;
  }
}

__global__ void init_iterates_kernel(int32_t n, int32_t m, Vecs V, int warm,
                                     const double* xin, const double* yin) {
  const double beta = V.st->beta, gamma = V.st->gamma;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double x0 = warm ? xin[j] / (V.C[j] * beta) : 0.0;
    x0 = clampd(x0, V.lb[j], V.ub[j]);
    V.x[j] = x0;
    V.x0[j] = x0;
    V.xt[j] = x0;
    V.cxt[j] = V.C[j] * x0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y0 = warm ? yin[i] / (V.R[i] * gamma) : 0.0;
    V.y[i] = y0;
    V.y0[i] = y0;
    V.yt[i] = y0;
    V.ry[i] = V.R[i] * y0;
    V.ryt[i] = V.ry[i];
  }
}

__global__ void unscale_kernel(int32_t n, int32_t m, Vecs V, double* xo, double* yo) {
  const double beta = V.st->beta, gamma = V.st->gamma;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    xo[j] = clampd(beta * V.cxt[j], V.lb_u[j], V.ub_u[j]);
  if (yo)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
      yo[i] = gamma * V.ryt[i];
}

__global__ void hash_fill_kernel(int64_t count, double* v) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)r * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    v[r] = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
  }
}

__global__ void mul_kernel(int64_t count, double* __restrict__ out, const double* __restrict__ a,
                           const double* __restrict__ b) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < count;
       r += (int64_t)gridDim.x * blockDim.x)
    out[r] = a[r] * b[r];
}

// ---------------------------------------------------------------------------
// Host orchestration.

struct Workspace {
  std::vector<void*> bufs;
  cudaStream_t st;
  ~Workspace() {
    for (void* p : bufs) cudaFreeAsync(p, st);
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

double host_sum(const std::vector<double>& v) {
  double a = 0.0;
  for (double x : v) a += x;
  return a;
}

int read_partials(double* dpart, int count, cudaStream_t st, double* out) {
  std::vector<double> h(count);
  TECCL_CUDA(cudaMemcpyAsync(h.data(), dpart, count * sizeof(double), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  *out = host_sum(h);
  return TECCL_OK;
}

SellView row_view(const teccl_lp* lp) {
  return SellView{lp->srow_off, lp->srow_w, lp->srow_idx, lp->srow_val, lp->m};
}
SellView col_view(const teccl_lp* lp) {
  return SellView{lp->scol_off, lp->scol_w, lp->scol_idx, lp->scol_val, lp->n};
}
template <bool UNIT, bool CHECK>
void launch_col(cudaStream_t st, const teccl_lp* lp, const Vecs& V, int j) {
  col_step_kernel<UNIT, CHECK><<<V.nb_col, kThreads, 0, st>>>(lp->n, col_view(lp), V, j);
}
template <bool UNIT, bool CHECK>
void launch_row(cudaStream_t st, const teccl_lp* lp, const Vecs& V, int j) {
  row_step_kernel<UNIT, CHECK><<<V.nb_row, kThreads, 0, st>>>(lp->m, row_view(lp), V, j);
}
template <bool UNIT>
void launch_kkt(cudaStream_t st, const teccl_lp* lp, const Vecs& V) {
  kkt_row_kernel<UNIT><<<V.nb_row, kThreads, 0, st>>>(lp->m, row_view(lp), V);
  kkt_col_kernel<UNIT><<<V.nb_col, kThreads, 0, st>>>(lp->n, col_view(lp), V);
}

template <bool UNIT>
void enqueue_chunk(int chunk, cudaStream_t st, const teccl_lp* lp, const Vecs& V) {
  for (int j = 0; j < chunk; ++j) {
    if (j == chunk - 1) {
      launch_col<UNIT, true>(st, lp, V, j);
      launch_row<UNIT, true>(st, lp, V, j);
    } else {
      launch_col<UNIT, false>(st, lp, V, j);
      launch_row<UNIT, false>(st, lp, V, j);
    }
  }
  launch_kkt<UNIT>(st, lp, V);
  control_kernel<<<1, 1024, 0, st>>>(V);
  restart_x_kernel<<<grid_for(lp->n), kThreads, 0, st>>>(lp->n, V);
  restart_y_kernel<<<grid_for(lp->m), kThreads, 0, st>>>(lp->m, V);
}

struct StepBench {
  int reps;
  double ms_col, ms_row, bytes_col, bytes_row;
  int gs_col, gs_row;
};

template <bool UNIT>
int solve_impl(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* o, double* x_dev,
               double* y_dev, teccl_pdlp_result* res, StepBench* sb = nullptr) {
  cudaStream_t st = ctx->stream;
  const int32_t m = lp->m, n = lp->n;
  Workspace W;
  W.st = st;
  cudaEvent_t ev0, ev1;
  TECCL_CUDA(cudaEventCreate(&ev0));
  TECCL_CUDA(cudaEventCreate(&ev1));
  TECCL_CUDA(cudaEventRecord(ev0, st));
  auto t_start = std::chrono::steady_clock::now();

  double *R = W.alloc<double>(m), *C = W.alloc<double>(n), *rstat = W.alloc<double>(m),
         *cstat = W.alloc<double>(n);
  double *cs = W.alloc<double>(n), *lbs = W.alloc<double>(n), *ubs = W.alloc<double>(n);
  double *los = W.alloc<double>(m), *his = W.alloc<double>(m);
  // gathered vectors (cxb, cxt, ry, ryt) carry one extra always-zero slot:
  // the SELL padding entries point at it
  double *x = W.alloc<double>(n), *x0 = W.alloc<double>(n), *xt = W.alloc<double>(n),
         *cxb = W.alloc<double>(n + 1), *cxt = W.alloc<double>(n + 1);
  double *y = W.alloc<double>(m), *y0 = W.alloc<double>(m), *yt = W.alloc<double>(m),
         *ry = W.alloc<double>(m + 1), *ryt = W.alloc<double>(m + 1);
  const int nb_row = (int)((m + kTile - 1) / kTile), nb_col = (int)((n + kTile - 1) / kTile);
  const int64_t pstride = std::max<int64_t>(std::max(nb_row, nb_col), kGrid);
  double* part = W.alloc<double>((int64_t)kNQ * pstride);
  double* part2 = W.alloc<double>(kGrid);
  PdlpState* dst = W.alloc<PdlpState>(1);
  if (!R || !C || !rstat || !cstat || !cs || !lbs || !ubs || !los || !his || !x || !x0 || !xt ||
      !cxb || !cxt || !y || !y0 || !yt || !ry || !ryt || !part || !part2 || !dst) {
    set_error("device allocation failed for PDLP workspace");
    return TECCL_ENOMEM;
  }
  TECCL_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * kNQ * pstride, st));
  TECCL_CUDA(cudaMemsetAsync(cxb, 0, sizeof(double) * (n + 1), st));
  TECCL_CUDA(cudaMemsetAsync(cxt, 0, sizeof(double) * (n + 1), st));
  TECCL_CUDA(cudaMemsetAsync(ry, 0, sizeof(double) * (m + 1), st));
  TECCL_CUDA(cudaMemsetAsync(ryt, 0, sizeof(double) * (m + 1), st));
  {
    int rc = teccl_build_sell(lp, st);
    if (rc) return rc;
  }
  const int gr = grid_for(m > n ? m : n);

  // --- Ruiz equilibration + Pock-Chambolle (alpha = 1), simultaneous updates.
  fill_kernel<<<gr, kThreads, 0, st>>>(m, R, 1.0);
  fill_kernel<<<gr, kThreads, 0, st>>>(n, C, 1.0);
  for (int it = 0; it < o->ruiz_iters; ++it) {
    abs_stat_kernel<UNIT, true><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, C, R, rstat);
    abs_stat_kernel<UNIT, true><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, R, C, cstat);
    apply_scale_kernel<<<gr, kThreads, 0, st>>>(m, R, rstat);
    apply_scale_kernel<<<gr, kThreads, 0, st>>>(n, C, cstat);
  }
  abs_stat_kernel<UNIT, false><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, C, R, rstat);
  abs_stat_kernel<UNIT, false><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, R, C, cstat);
  apply_scale_kernel<<<gr, kThreads, 0, st>>>(m, R, rstat);
  apply_scale_kernel<<<gr, kThreads, 0, st>>>(n, C, cstat);
  TECCL_CHECK_LAUNCH();

  // --- scaled data and the bound/objective rescaling
  scale_cols_kernel<<<kGrid, kThreads, 0, st>>>(n, C, lp->obj, lp->var_lb, lp->var_ub, cs, lbs, ubs, part);
  double csq = 0.0;
  if (read_partials(part, kGrid, st, &csq)) return TECCL_ECUDA;
  scale_rows_kernel<<<kGrid, kThreads, 0, st>>>(m, R, lp->row_lo, lp->row_hi, los, his, part, part2);
  double bsq = 0.0, bsq_u = 0.0;
  if (read_partials(part, kGrid, st, &bsq)) return TECCL_ECUDA;
  if (read_partials(part2, kGrid, st, &bsq_u)) return TECCL_ECUDA;
  sumsq_kernel<<<kGrid, kThreads, 0, st>>>(n, lp->obj, part);
  double csq_u = 0.0;
  if (read_partials(part, kGrid, st, &csq_u)) return TECCL_ECUDA;
  const double beta = sqrt(bsq) + 1.0, gamma = sqrt(csq) + 1.0;
  scale_inplace_kernel<<<gr, kThreads, 0, st>>>(n, cs, 1.0 / gamma);
  scale_inplace_kernel<<<gr, kThreads, 0, st>>>(n, lbs, 1.0 / beta);
  scale_inplace_kernel<<<gr, kThreads, 0, st>>>(n, ubs, 1.0 / beta);
  scale_inplace_kernel<<<gr, kThreads, 0, st>>>(m, los, 1.0 / beta);
  scale_inplace_kernel<<<gr, kThreads, 0, st>>>(m, his, 1.0 / beta);
  TECCL_CHECK_LAUNCH();

  // --- power iteration for ||A_s||_2: v in xt, C.v in cxt, A_s.v in yt, R.A_s.v in ryt
  double sigma_max = 1.0;
  int64_t nl = 2 + 4LL * o->ruiz_iters + 4 + 1 + 1 + 1 + 5;  // kernel launches so far
  if (m > 0 && n > 0 && lp->nnz > 0) {
    nl += 3;
    hash_fill_kernel<<<gr, kThreads, 0, st>>>(n, xt);
    double nv = 0.0;
    sumsq_kernel<<<kGrid, kThreads, 0, st>>>(n, xt, part);
    if (read_partials(part, kGrid, st, &nv)) return TECCL_ECUDA;
    scale_inplace_kernel<<<gr, kThreads, 0, st>>>(n, xt, 1.0 / sqrt(nv));
    for (int it = 0; it < 40; ++it) {
      mul_kernel<<<gr, kThreads, 0, st>>>(n, cxt, xt, C);
      spmv_scaled_kernel<UNIT><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, cxt, R, R, yt, ryt);
      spmv_scaled_kernel<UNIT><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, ryt, C, nullptr, xt, nullptr);
      sumsq_kernel<<<kGrid, kThreads, 0, st>>>(n, xt, part);
      nl += 5;
      if (read_partials(part, kGrid, st, &nv)) return TECCL_ECUDA;
      if (!(nv > 0.0)) break;
      scale_inplace_kernel<<<gr, kThreads, 0, st>>>(n, xt, 1.0 / sqrt(nv));
    }
    if (nv > 0.0) sigma_max = sqrt(sqrt(nv));
  }
  TECCL_CHECK_LAUNCH();

  // --- state
  PdlpState hs{};
  hs.eta = 0.998 / sigma_max;
  const double cn_s = sqrt(csq) / gamma, bn_s = sqrt(bsq) / beta;
  hs.omega = (cn_s > 1e-10 && bn_s > 1e-10) ? cn_s / bn_s : 1.0;
  hs.tau = hs.eta / hs.omega;
  hs.sigma = hs.eta * hs.omega;
  hs.refl = o->reflection;
  hs.beta = beta;
  hs.gamma = gamma;
  hs.bnorm = sqrt(bsq_u);
  hs.cnorm = sqrt(csq_u);
  hs.eps = o->eps_rel;
  const int chunk = o->check_every > 0 ? o->check_every : 64;
  hs.chunk_len = chunk;
  TECCL_CUDA(cudaMemcpyAsync(dst, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));

  Vecs V{};
  V.c = cs; V.lb = lbs; V.ub = ubs; V.lo = los; V.hi = his; V.R = R; V.C = C;
  V.x = x; V.x0 = x0; V.xt = xt; V.cxb = cxb; V.cxt = cxt;
  V.y = y; V.y0 = y0; V.yt = yt; V.ry = ry; V.ryt = ryt;
  V.c_u = lp->obj; V.lb_u = lp->var_lb; V.ub_u = lp->var_ub; V.lo_u = lp->row_lo; V.hi_u = lp->row_hi;
  V.part = part;
  V.pstride = pstride;
  V.nb_row = nb_row;
  V.nb_col = nb_col;
  V.st = dst;
  init_iterates_kernel<<<gr, kThreads, 0, st>>>(n, m, V, o->warm_start, x_dev, y_dev);
  TECCL_CHECK_LAUNCH();

  const int gsr = kTile, gsc = kTile;

  if (sb) {  // time the fused iteration kernels alone, CUDA events on this stream
    cudaEvent_t a, b, c2;
    TECCL_CUDA(cudaEventCreate(&a));
    TECCL_CUDA(cudaEventCreate(&b));
    TECCL_CUDA(cudaEventCreate(&c2));
    for (int w = 0; w < 3; ++w) {
      launch_col<UNIT, false>(st, lp, V, 0);
      launch_row<UNIT, false>(st, lp, V, 0);
    }
    TECCL_CUDA(cudaEventRecord(a, st));
    for (int r = 0; r < sb->reps; ++r) launch_col<UNIT, false>(st, lp, V, 0);
    TECCL_CUDA(cudaEventRecord(b, st));
    for (int r = 0; r < sb->reps; ++r) launch_row<UNIT, false>(st, lp, V, 0);
    TECCL_CUDA(cudaEventRecord(c2, st));
    TECCL_CHECK_LAUNCH();
    TECCL_CUDA(cudaEventSynchronize(c2));
    float m1 = 0.f, m2 = 0.f;
    TECCL_CUDA(cudaEventElapsedTime(&m1, a, b));
    TECCL_CUDA(cudaEventElapsedTime(&m2, b, c2));
    sb->ms_col = m1 / sb->reps;
    sb->ms_row = m2 / sb->reps;
    const double ib = UNIT ? 4.0 : 12.0;
    // algorithmic bytes: index stream once, pointer
    // array once, gathered vector once, 6 dense reads + 2 writes per column,
    // 5 dense reads + 2 writes per row
    // SELL-32: slice offsets + widths (12 B per 32 rows), every stored entry
    // (padding included) once, gathered vector once, dense operands
    const double ns_c = (n + 31) / 32, ns_r = (m + 31) / 32;
    sb->bytes_col = 12.0 * ns_c + ib * lp->scol_entries + 8.0 * m + 64.0 * n;
    sb->bytes_row = 12.0 * ns_r + ib * lp->srow_entries + 8.0 * n + 56.0 * m;
    sb->gs_col = gsc;
    sb->gs_row = gsr;
    cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c2);
    return TECCL_OK;
  }

  // --- chunk graph
  cudaGraphExec_t gexec = nullptr;
  if (o->use_graphs) {
    cudaGraph_t g;
    cudaStream_t cap;
    TECCL_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    TECCL_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    enqueue_chunk<UNIT>(chunk, cap, lp, V);
    TECCL_CUDA(cudaStreamEndCapture(cap, &g));
    TECCL_CUDA(cudaGraphInstantiate(&gexec, g, 0));
    TECCL_CUDA(cudaGraphDestroy(g));
    TECCL_CUDA(cudaStreamDestroy(cap));
  }

  // --- iterate: chunks queued `lookahead` deep; the device stops itself.
  const int look = o->lookahead > 0 ? o->lookahead : 1;
  PdlpState* ring = nullptr;
  TECCL_CUDA(cudaMallocHost((void**)&ring, sizeof(PdlpState) * look));
  std::vector<cudaEvent_t> evs(look);
  for (auto& e : evs) TECCL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int64_t launched = 0, polled = 0;
  int status = TECCL_ITER_LIMIT;
  PdlpState last = hs;
  const int64_t max_chunks = (o->max_iters + chunk - 1) / chunk;
  bool stop = false;
  int64_t checks_seen = 0;
  while (!stop) {
    while (launched < max_chunks && launched - polled < look) {
      if (gexec) {
        TECCL_CUDA(cudaGraphLaunch(gexec, st));
      } else {
        enqueue_chunk<UNIT>(chunk, st, lp, V);
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
    ++checks_seen;
    if (o->verbose > 0 && (checks_seen % o->verbose == 0 || last.done))
      fprintf(stderr, "[teccl pdlp] it=%lld rp=%.2e rd=%.2e gap=%.2e pobj=%.9g w=%.3e r=%.2e restarts=%d\n",
              last.total, last.rel_p, last.rel_d, last.gap, last.pobj, last.omega, last.last_r, last.restarts);
    if (last.done == 1) { status = TECCL_OPTIMAL; stop = true; }
    else if (last.done == 2) { status = TECCL_NUMERICAL; stop = true; }
    else if (polled >= max_chunks) { status = TECCL_ITER_LIMIT; stop = true; }
    else {
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (el > o->time_limit) { status = TECCL_TIME_LIMIT; stop = true; }
    }
  }
  // stop anything still queued from touching the iterates
  if (status != TECCL_OPTIMAL && status != TECCL_NUMERICAL) {
    int one = 3;
    TECCL_CUDA(cudaMemcpyAsync(&dst->done, &one, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  TECCL_CUDA(cudaStreamSynchronize(st));
  TECCL_CUDA(cudaMemcpy(&last, dst, sizeof(PdlpState), cudaMemcpyDeviceToHost));
  if (last.done == 1) status = TECCL_OPTIMAL;
  if (last.done == 3) last.done = 0;

  unscale_kernel<<<gr, kThreads, 0, st>>>(n, m, V, x_dev, y_dev);
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaEventRecord(ev1, st));
  TECCL_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  TECCL_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  for (auto& e : evs) cudaEventDestroy(e);
  cudaFreeHost(ring);
  if (gexec) cudaGraphExecDestroy(gexec);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);

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
  res->spmv_launches = nl + 1 + 1 + launched * (2LL * chunk + 5);  // + init + unscale
  return TECCL_OK;
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
  return lp->unit ? solve_impl<true>(ctx, lp, &o, x_dev, y_dev, res)
                  : solve_impl<false>(ctx, lp, &o, x_dev, y_dev, res);
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

extern "C" int teccl_spmv_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* ms_per_pair,
                                double* bytes_per_pair) {
  if (!ctx || !lp || reps < 1) { set_error("bad argument"); return TECCL_EINVAL; }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  const int32_t m = lp->m, n = lp->n;
  double *vx = nullptr, *vy = nullptr, *ones_m = nullptr, *ones_n = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&vx, sizeof(double) * (n + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&vy, sizeof(double) * (m + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&ones_m, sizeof(double) * (m + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&ones_n, sizeof(double) * (n + 1), st));
  const int gr = grid_for(m > n ? m : n);
  hash_fill_kernel<<<gr, kThreads, 0, st>>>(n, vx);
  fill_kernel<<<gr, kThreads, 0, st>>>(m, ones_m, 1.0);
  fill_kernel<<<gr, kThreads, 0, st>>>(n, ones_n, 1.0);
  cudaEvent_t a, b;
  TECCL_CUDA(cudaEventCreate(&a));
  TECCL_CUDA(cudaEventCreate(&b));
  for (int it = -3; it < reps; ++it) {
    if (it == 0) TECCL_CUDA(cudaEventRecord(a, st));
    if (lp->unit) {
      spmv_scaled_kernel<true><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, vx, ones_m, nullptr, vy, nullptr);
      spmv_scaled_kernel<true><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, vy, ones_n, nullptr, vx, nullptr);
    } else {
      spmv_scaled_kernel<false><<<gr, kThreads, 0, st>>>(m, lp->row_ptr, lp->col, lp->val, vx, ones_m, nullptr, vy, nullptr);
      spmv_scaled_kernel<false><<<gr, kThreads, 0, st>>>(n, lp->col_ptr, lp->row, lp->cval, vy, ones_n, nullptr, vx, nullptr);
    }
  }
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaEventRecord(b, st));
  TECCL_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  TECCL_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_pair = ms / reps;
  const double vb = lp->unit ? 4.0 : 12.0;
  // per pair: both index streams, ptr arrays, one dense read of each input
  // vector (gathers at best once), one write of each output
  *bytes_per_pair = 2.0 * lp->nnz * vb + 8.0 * (m + 1) + 8.0 * (n + 1) + 2.0 * 8.0 * (m + n);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(vx, st); cudaFreeAsync(vy, st); cudaFreeAsync(ones_m, st); cudaFreeAsync(ones_n, st);
  TECCL_CUDA(cudaStreamSynchronize(st));
  return TECCL_OK;
}

extern "C" int teccl_pdlp_step_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* out6) {
  if (!ctx || !lp || reps < 1 || !out6) { set_error("bad argument"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  teccl_pdlp_opts o;
  teccl_pdlp_default_opts(&o);
  teccl_pdlp_result res{};
  double* xd = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&xd, sizeof(double) * (lp->n + 1), ctx->stream));
  StepBench sb{reps, 0, 0, 0, 0, 0, 0};
  int rc = lp->unit ? solve_impl<true>(ctx, lp, &o, xd, nullptr, &res, &sb)
                    : solve_impl<false>(ctx, lp, &o, xd, nullptr, &res, &sb);
  cudaFreeAsync(xd, ctx->stream);
  TECCL_CUDA(cudaStreamSynchronize(ctx->stream));
  out6[0] = sb.ms_col; out6[1] = sb.ms_row; out6[2] = sb.bytes_col; out6[3] = sb.bytes_row;
  out6[4] = sb.gs_col; out6[5] = sb.gs_row;
  return rc;
}

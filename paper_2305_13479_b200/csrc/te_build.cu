// (1) Time-expanded constraint-matrix builder: emits the copy-free TE-CCL LP
// (reference pkg/src/collsched/lp.py:22-136) as CSR and CSC directly in HBM.
//
// Variable order (lp.py:47-65):
//   per source slot s:  F(s,e,k) = s*SB + e*K + k            e in edge order
//                       B(s,g,k) = s*SB + E*K + g*(K+1) + k  g = GPU rank in node order
//   per pair p:         Rd(p,k)  = S*SB + p*2K + 2k,  Rc(p,k) = Rd(p,k) + 1
// Row order (lp.py:69-131):
//   init(s) | cap(e,k) | cons(s,n,k) (+ last(s,n) after node n's K rows when
//   n is a GPU other than the source) | cum(p,k) | bcap(g,k) (buffer limit)
// Every coefficient is +-1, so the matrix is stored "unit": index with the
// sign in bit 31, no value array. Columns inside a row and rows inside a
// column come out ascending, so both orientations are canonical and the
// builder is deterministic.

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "te_gen.cuh"

namespace teccl {

// Emit helper: count or write one (index, sign) entry.
template <bool FILL>
struct Emitter {
  uint32_t* out;
  int cnt;
  __device__ __forceinline__ void put(int64_t idx, bool neg) {
    if (FILL) out[cnt] = (uint32_t)idx | (neg ? kSignBit : 0u);
    ++cnt;
  }
};

// ---------------------------------------------------------------------------
// Row generator. gen_row emits reference row r's entries (reference column
// ids, ascending) into `em` and returns its bounds and bound class; the
// kernels below run it one thread per row, twice (count, then fill).
template <class Em>
__device__ __forceinline__ void gen_row(const TeDev& d, int64_t r, Em& em, double& rlo, double& rhi,
                                        int& rc) {
  const int K = d.K;
  rlo = 0.0;
  rhi = 0.0;
  rc = 0;                                          // bound class: 0 = (0,0)
  if (r < d.S) {                                   // init(s), lp.py:69-72
    int s = (int)r, n = d.snode[s];
    for (int j = d.out_ptr[n]; j < d.out_ptr[n + 1]; ++j) em.put(varF(d, s, d.out_e[j], 0), false);
    em.put(varB(d, s, d.gpu_of[n], 0), false);
    rlo = rhi = d.out_units[s];
    if (d.dict_row) rc = 1 + d.src_ouidx[s];
  } else if (r < d.R_cons) {                       // cap(e,k), lp.py:74-77
    int64_t q = r - d.S;
    int e = (int)(q / K), k = (int)(q % K);
    for (int s = 0; s < d.S; ++s) em.put(varF(d, s, e, k), false);
    rlo = -INFINITY;
    rhi = d.ecap[(int64_t)e * K + k];
    if (d.dict_row) rc = 1 + d.nOU + d.cap_idx[q];
  } else if (r < d.R_cum) {                        // cons / last, lp.py:81-116
    int64_t q = r - d.R_cons;
    int s = (int)(q / d.CB);
    int64_t off = q % d.CB;
    // node n: last node with cons_off(s,n) <= off (offsets ascend with n)
    int lo_n = 0, hi_n = d.Nn - 1;
    while (lo_n < hi_n) {
      int mid = (lo_n + hi_n + 1) >> 1;
      if (cons_off(d, s, mid) <= off) lo_n = mid; else hi_n = mid - 1;
    }
    int n = lo_n;
    int k = (int)(off - cons_off(d, s, n));      // k == K marks the last row
    int g = d.gpu_of[n];
    int pair = (g >= 0) ? d.pair_of[s * d.Nn + n] : -1;
    if (k < K) {
      for (int j = d.inc_ptr[n]; j < d.inc_ptr[n + 1]; ++j) {
        uint32_t t = d.inc[j];
        int e = (int)(t & kIdxMask);
        if (t & kSignBit) {                        // leaves n: send next epoch
          if (k + 1 <= K - 1) em.put(varF(d, s, e, k + 1), true);
        } else {                                   // arrives at n
          int kin = k - d.edelta[e];
          if (kin >= 0) em.put(varF(d, s, e, kin), false);
        }
      }
      if (g >= 0) {
        em.put(varB(d, s, g, k), false);
        em.put(varB(d, s, g, k + 1), true);
        if (pair >= 0) em.put(varRd(d, pair, k), true);
      }
    } else {                                       // last(s,n), lp.py:107-116
      for (int j = d.inc_ptr[n]; j < d.inc_ptr[n + 1]; ++j) {
        uint32_t t = d.inc[j];
        if (t & kSignBit) continue;
        int e = (int)(t & kIdxMask);
        int kin = K - 1 - d.edelta[e];
        if (kin >= 0) em.put(varF(d, s, e, kin), false);
      }
      if (pair >= 0) em.put(varRd(d, pair, K - 1), true);
    }
    rlo = rhi = 0.0;
  } else if (r < d.R_bcap) {                       // cum(p,k), lp.py:118-123
    int64_t q = r - d.R_cum;
    int p = (int)(q / K), k = (int)(q % K);
    int64_t rd = varRd(d, p, k);
    if (k >= 1) em.put(rd - 1, true);              // Rc(p,k-1)
    em.put(rd, true);                              // Rd(p,k)
    em.put(rd + 1, false);                         // Rc(p,k)
    rlo = rhi = 0.0;
  } else {                                         // bcap(g,k), lp.py:125-131
    int64_t q = r - d.R_bcap;
    int g = (int)(q / (K + 1)), k = (int)(q % (K + 1));
    for (int s = 0; s < d.S; ++s) em.put(varB(d, s, g, k), false);
    rlo = -INFINITY;
    rhi = d.blimit;
    rc = 1 + d.nOU + d.nCap;
  }
}

template <bool FILL>
__global__ void te_rows_kernel(TeDev d, const int64_t* __restrict__ row_ptr,
                               uint32_t* __restrict__ col, int64_t* __restrict__ row_len,
                               double* __restrict__ lo, double* __restrict__ hi,
                               uint16_t* __restrict__ code) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < d.n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    Emitter<FILL> em{FILL ? col + row_ptr[r] : nullptr, 0};
    double rlo, rhi;
    int rc;
    gen_row(d, r, em, rlo, rhi, rc);
    if (FILL) {
      lo[r] = rlo;
      hi[r] = rhi;
      if (d.dict_row) code[r] = (uint16_t)rc;
    } else {
      row_len[r] = em.cnt;
    }
  }
}

// ---------------------------------------------------------------------------
// Column generator: one thread per variable; rows emitted ascending.
__device__ __forceinline__ void sort_small(int64_t* a, bool* neg, int n) {
  for (int i = 1; i < n; ++i) {
    int64_t v = a[i];
    bool sg = neg[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; neg[j + 1] = neg[j]; --j; }
    a[j + 1] = v;
    neg[j + 1] = sg;
  }
}

// gen_col: the (<= 6) reference rows of reference column v, unsorted, with
// its bounds, cost and bound class; returns the entry count.
__device__ __forceinline__ int gen_col(const TeDev& d, int64_t v, int64_t* rows, bool* neg,
                                       double& vlb, double& vub, double& cost, int& cc) {
  const int K = d.K;
  const int64_t fB = (int64_t)d.E * K;
  int c = 0;
  vlb = 0.0;
  vub = INFINITY;
  cost = 0.0;
  cc = 0;                                          // bound class 0 = (0, inf, 0)
  if (v < (int64_t)d.S * d.SB) {
    int s = (int)(v / d.SB);
    int64_t q = v % d.SB;
    if (q < fB) {                                  // F(s,e,k)
      int e = (int)(q / K), k = (int)(q % K);
      int u = d.esrc[e], w = d.edst[e];
      if (k == 0 && u == d.snode[s]) { rows[c] = s; neg[c++] = false; }
      rows[c] = d.S + (int64_t)e * K + k; neg[c++] = false;
      if (k >= 1) { rows[c] = rowCons(d, s, u, k - 1); neg[c++] = true; }
      int t = k + d.edelta[e];
      if (t <= K - 1) { rows[c] = rowCons(d, s, w, t); neg[c++] = false; }
      if (t == K - 1 && !d.is_sw[w] && w != d.snode[s]) {
        rows[c] = rowCons(d, s, w, K); neg[c++] = false;
      }
      if (k == 0 && u != d.snode[s]) { vub = 0.0; cc = 1; }   // lp.py:51-52
    } else {                                       // B(s,g,k)
      q -= fB;
      int g = (int)(q / (K + 1)), k = (int)(q % (K + 1));
      int n = d.node_of_gpu[g];
      if (k == 0 && n == d.snode[s]) { rows[c] = s; neg[c++] = false; }
      if (k >= 1) { rows[c] = rowCons(d, s, n, k - 1); neg[c++] = true; }
      if (k <= K - 1) { rows[c] = rowCons(d, s, n, k); neg[c++] = false; }
      if (d.has_bcap) { rows[c] = d.R_bcap + (int64_t)g * (K + 1) + k; neg[c++] = false; }
      if (k == 0 && n != d.snode[s]) { vub = 0.0; cc = 1; }   // lp.py:57-59
    }
  } else {
    int64_t q = v - (int64_t)d.S * d.SB;
    int p = (int)(q / (2 * K));
    int k = (int)((q % (2 * K)) >> 1);
    bool is_rc = (q & 1) != 0;
    int s = d.pair_src[p], w = d.pair_dst[p];
    double u = d.pair_u[p];
    vub = u;
    if (!is_rc) {                                  // Rd(p,k)
      if (d.dict_col) cc = 2 + d.pair_uidx[p];
      rows[c] = rowCons(d, s, w, k); neg[c++] = true;
      if (k == K - 1) { rows[c] = rowCons(d, s, w, K); neg[c++] = true; }
      rows[c] = d.R_cum + (int64_t)p * K + k; neg[c++] = true;
    } else {                                       // Rc(p,k)
      rows[c] = d.R_cum + (int64_t)p * K + k; neg[c++] = false;
      if (k + 1 <= K - 1) { rows[c] = d.R_cum + (int64_t)p * K + k + 1; neg[c++] = true; }
      if (d.phase1) {                              // feasibility: deliver everything by K-1
        cost = (k == K - 1) ? -1.0 : 0.0;
      } else {
        if (k == K - 1) vlb = u;                   // lp.py:64-65
        cost = -1.0 / (double)(k + 1);             // maximise sum Rc/(k+1), lp.py:133-135
      }
      if (d.dict_col) cc = 2 + d.nU + d.pair_uidx[p] * K + k;
    }
  }
  return c;
}

template <bool FILL>
__global__ void te_cols_kernel(TeDev d, const int64_t* __restrict__ col_ptr,
                               uint32_t* __restrict__ row, int64_t* __restrict__ col_len,
                               double* __restrict__ lb, double* __restrict__ ub,
                               double* __restrict__ obj, uint16_t* __restrict__ code) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < d.n_vars;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t rows[6];
    bool neg[6];
    double vlb, vub, cost;
    int cc;
    const int c = gen_col(d, v, rows, neg, vlb, vub, cost, cc);
    if (FILL) {
      sort_small(rows, neg, c);
      uint32_t* out = row + col_ptr[v];
      for (int i = 0; i < c; ++i) out[i] = (uint32_t)rows[i] | (neg[i] ? kSignBit : 0u);
      lb[v] = vlb;
      ub[v] = vub;
      obj[v] = cost;
      if (d.dict_col) code[v] = (uint16_t)cc;
    } else {
      col_len[v] = c;
    }
  }
}

__global__ void set_tail_kernel(int64_t* ptr, int64_t idx, const int64_t* len_last,
                                const int64_t* scan_last) {
  ptr[idx] = *scan_last + *len_last;
}

// ---------------------------------------------------------------------------
// Epoch-major numbering for row-partitioned (multi-GPU) solves. Columns:
// epoch blocks of CW = S*E + S*G + 2P [F(s,e,k) | B(s,g,k) | Rd/Rc(p,k)], then
// the S*G final buffers B(s,g,K). Rows: S init rows, epoch blocks of
// RW = E + S*Nn + P (+G) [cap(e,k) | cons(s,n,k) | cum(p,k) | bcap(g,k)],
// then the S*(G-1) last-epoch rows and bcap(g,K). Every row of epoch k only
// touches columns of epochs k-delta_max..k+1, so contiguous epoch ranges give
// contiguous owned ranges with thin contiguous halos.
struct EmShape {
  int64_t CW, RW, n_cols, n_rows;
};

__host__ __device__ inline EmShape em_shape(const TeDev& d) {
  EmShape e;
  e.CW = (int64_t)d.S * d.E + (int64_t)d.S * d.G + 2LL * d.P;
  e.RW = (int64_t)d.E + (int64_t)d.S * d.Nn + d.P + (d.has_bcap ? d.G : 0);
  e.n_cols = (int64_t)d.K * e.CW + (int64_t)d.S * d.G;
  e.n_rows = d.S + (int64_t)d.K * e.RW + (int64_t)d.S * (d.G - 1) + (d.has_bcap ? d.G : 0);
  return e;
}

__device__ inline int64_t em_col_of_ref(const TeDev& d, const EmShape& z, int64_t v) {
  const int K = d.K;
  if (v < (int64_t)d.S * d.SB) {
    const int s = (int)(v / d.SB);
    int64_t q = v % d.SB;
    if (q < (int64_t)d.E * K) {
      const int e = (int)(q / K), k = (int)(q % K);
      return k * z.CW + (int64_t)s * d.E + e;
    }
    q -= (int64_t)d.E * K;
    const int g = (int)(q / (K + 1)), k = (int)(q % (K + 1));
    if (k < K) return k * z.CW + (int64_t)d.S * d.E + (int64_t)s * d.G + g;
    return (int64_t)K * z.CW + (int64_t)s * d.G + g;
  }
  const int64_t q = v - (int64_t)d.S * d.SB;
  const int p = (int)(q / (2 * K));
  const int k = (int)((q % (2 * K)) >> 1);
  return k * z.CW + (int64_t)d.S * d.E + (int64_t)d.S * d.G + 2LL * p + (q & 1);
}

__device__ inline int64_t ref_col_of_em(const TeDev& d, const EmShape& z, int64_t c) {
  const int K = d.K;
  int64_t k = c / z.CW;
  if (k >= K) {
    const int64_t o = c - (int64_t)K * z.CW;
    return varB(d, (int)(o / d.G), (int)(o % d.G), K);
  }
  int64_t o = c - k * z.CW;
  if (o < (int64_t)d.S * d.E) return varF(d, (int)(o / d.E), (int)(o % d.E), (int)k);
  o -= (int64_t)d.S * d.E;
  if (o < (int64_t)d.S * d.G) return varB(d, (int)(o / d.G), (int)(o % d.G), (int)k);
  o -= (int64_t)d.S * d.G;
  return varRd(d, (int)(o >> 1), (int)k) + (o & 1);
}

__device__ inline int node_of_cons(const TeDev& d, int s, int64_t off) {
  int lo_n = 0, hi_n = d.Nn - 1;
  while (lo_n < hi_n) {
    const int mid = (lo_n + hi_n + 1) >> 1;
    if (cons_off(d, s, mid) <= off) lo_n = mid; else hi_n = mid - 1;
  }
  return lo_n;
}

__device__ inline int64_t ref_row_of_em(const TeDev& d, const EmShape& z, int64_t r) {
  const int K = d.K;
  if (r < d.S) return r;
  r -= d.S;
  int64_t k = r / z.RW;
  if (k >= K) {
    int64_t o = r - (int64_t)K * z.RW;
    if (o < (int64_t)d.S * (d.G - 1)) {
      const int s = (int)(o / (d.G - 1)), i = (int)(o % (d.G - 1));
      const int gs = d.gpu_of[d.snode[s]];
      return rowCons(d, s, d.node_of_gpu[i < gs ? i : i + 1], K);
    }
    o -= (int64_t)d.S * (d.G - 1);
    return d.R_bcap + o * (K + 1) + K;
  }
  int64_t o = r - k * z.RW;
  if (o < d.E) return d.S + o * K + k;
  o -= d.E;
  if (o < (int64_t)d.S * d.Nn) return rowCons(d, (int)(o / d.Nn), (int)(o % d.Nn), (int)k);
  o -= (int64_t)d.S * d.Nn;
  if (o < d.P) return d.R_cum + o * K + k;
  o -= d.P;
  return d.R_bcap + o * (K + 1) + k;
}

__device__ inline int64_t em_row_of_ref(const TeDev& d, const EmShape& z, int64_t r) {
  const int K = d.K;
  if (r < d.S) return r;
  if (r < d.R_cons) {
    const int64_t q = r - d.S;
    return d.S + (q % K) * z.RW + q / K;
  }
  if (r < d.R_cum) {
    const int64_t q = r - d.R_cons;
    const int s = (int)(q / d.CB);
    const int64_t off = q % d.CB;
    const int n = node_of_cons(d, s, off);
    const int64_t k = off - cons_off(d, s, n);
    if (k < K) return d.S + k * z.RW + d.E + (int64_t)s * d.Nn + n;
    const int g = d.gpu_of[n], gs = d.gpu_of[d.snode[s]];
    return d.S + (int64_t)K * z.RW + (int64_t)s * (d.G - 1) + (g < gs ? g : g - 1);
  }
  if (r < d.R_bcap) {
    const int64_t q = r - d.R_cum;
    return d.S + (q % K) * z.RW + d.E + (int64_t)d.S * d.Nn + q / K;
  }
  const int64_t q = r - d.R_bcap;
  const int64_t g = q / (K + 1), k = q % (K + 1);
  if (k < K) return d.S + k * z.RW + d.E + (int64_t)d.S * d.Nn + d.P + g;
  return d.S + (int64_t)K * z.RW + (int64_t)d.S * (d.G - 1) + g;
}

// Emitter that maps reference columns to window-relative epoch-major ids.
template <bool FILL>
struct EmColEmitter {
  const TeDev* d;
  const EmShape* z;
  uint32_t* out;
  int64_t base;
  int cnt;
  unsigned long long* lo;
  unsigned long long* hi;
  __device__ __forceinline__ void put(int64_t v, bool neg) {
    const int64_t c = em_col_of_ref(*d, *z, v);
    if (FILL) out[cnt] = (uint32_t)(c - base) | (neg ? kSignBit : 0u);
    else { atomicMin(lo, (unsigned long long)c); atomicMax(hi, (unsigned long long)c); }
    ++cnt;
  }
};

// Local rows [r0, r0+nr) of the epoch-major LP: CSR over the column window.
template <bool FILL>
__global__ void part_rows_kernel(TeDev d, EmShape z, int64_t r0, int64_t nr, int64_t cw0,
                                 const int64_t* __restrict__ row_ptr, uint32_t* __restrict__ col,
                                 int64_t* __restrict__ row_len, double* __restrict__ lo,
                                 double* __restrict__ hi, uint16_t* __restrict__ code,
                                 unsigned long long* mm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = ref_row_of_em(d, z, r0 + i);
    EmColEmitter<FILL> em{&d, &z, FILL ? col + row_ptr[i] : nullptr, cw0, 0, mm, mm + 1};
    double rlo, rhi;
    int rc;
    gen_row(d, r, em, rlo, rhi, rc);
    if (FILL) {
      lo[i] = rlo;
      hi[i] = rhi;
      if (d.dict_row) code[i] = (uint16_t)rc;
    } else {
      row_len[i] = em.cnt;
    }
  }
}

// Local columns [c0, c0+nc): CSC over the row window.
template <bool FILL>
__global__ void part_cols_kernel(TeDev d, EmShape z, int64_t c0, int64_t nc, int64_t rw0,
                                 const int64_t* __restrict__ col_ptr, uint32_t* __restrict__ row,
                                 int64_t* __restrict__ col_len, double* __restrict__ lb,
                                 double* __restrict__ ub, double* __restrict__ obj,
                                 uint16_t* __restrict__ code, unsigned long long* mm) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ref_col_of_em(d, z, c0 + j);
    int64_t rows[6];
    bool neg[6];
    double vlb, vub, cost;
    int cc;
    const int c = gen_col(d, v, rows, neg, vlb, vub, cost, cc);
    for (int q = 0; q < c; ++q) rows[q] = em_row_of_ref(d, z, rows[q]);
    if (FILL) {
      sort_small(rows, neg, c);
      uint32_t* out = row + col_ptr[j];
      for (int q = 0; q < c; ++q) out[q] = (uint32_t)(rows[q] - rw0) | (neg[q] ? kSignBit : 0u);
      lb[j] = vlb;
      ub[j] = vub;
      obj[j] = cost;
      if (d.dict_col) code[j] = (uint16_t)cc;
    } else {
      col_len[j] = c;
      for (int q = 0; q < c; ++q) {
        atomicMin(mm, (unsigned long long)rows[q]);
        atomicMax(mm + 1, (unsigned long long)rows[q]);
      }
    }
  }
}

// ref index of every local (epoch-major) column: host assembles solutions
__global__ void part_colmap_kernel(TeDev d, EmShape z, int64_t c0, int64_t nc, int64_t* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nc;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = ref_col_of_em(d, z, c0 + j);
}

}  // namespace teccl

using namespace teccl;

namespace {

template <typename T>
int upload(const std::vector<T>& h, T** d, cudaStream_t st) {
  size_t bytes = h.size() * sizeof(T);
  if (bytes == 0) bytes = sizeof(T);
  TECCL_CUDA(cudaMallocAsync((void**)d, bytes, st));
  if (!h.empty()) TECCL_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T),
                                             cudaMemcpyHostToDevice, st));
  return TECCL_OK;
}

// exclusive scan of len[0..count) into ptr[0..count], ptr[count] = total
int scan_lengths(int64_t* len, int64_t* ptr, int64_t count, cudaStream_t st) {
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len, ptr, count, st);
  void* tmp = nullptr;
  TECCL_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, ptr, count, st);
  TECCL_CHECK_LAUNCH();
  set_tail_kernel<<<1, 1, 0, st>>>(ptr, count, len + count - 1, ptr + count - 1);
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaFreeAsync(tmp, st));
  return TECCL_OK;
}

int prepare_tables(teccl_ctx* ctx, const teccl_te_desc* desc, TeDev& d, std::vector<void*>& owned) {
  if (!ctx || !desc) { set_error("null argument"); return TECCL_EINVAL; }
  const int Nn = desc->num_nodes, E = desc->num_edges, S = desc->num_sources,
            P = desc->num_pairs, K = desc->K;
  if (Nn < 1 || E < 0 || S < 0 || P < 0 || K < 1) { set_error("bad dimensions"); return TECCL_EINVAL; }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));

  // Host-side derived tables (all O(nodes + edges + pairs)).
  std::vector<int> gpu_of(Nn, -1), gpre(Nn + 1, 0), node_of_gpu;
  for (int n = 0; n < Nn; ++n) {
    gpre[n] = (int)node_of_gpu.size();
    if (!desc->node_is_switch[n]) { gpu_of[n] = (int)node_of_gpu.size(); node_of_gpu.push_back(n); }
  }
  const int G = (int)node_of_gpu.size();
  std::vector<int> inc_ptr(Nn + 1, 0), out_ptr(Nn + 1, 0);
  for (int e = 0; e < E; ++e) {
    int u = desc->edge_src[e], w = desc->edge_dst[e];
    if (u < 0 || u >= Nn || w < 0 || w >= Nn || u == w) { set_error("bad edge endpoint"); return TECCL_EINVAL; }
    if (desc->edge_delta[e] < 0) { set_error("negative edge delay"); return TECCL_EINVAL; }
    inc_ptr[u + 1]++; inc_ptr[w + 1]++; out_ptr[u + 1]++;
  }
  for (int n = 0; n < Nn; ++n) { inc_ptr[n + 1] += inc_ptr[n]; out_ptr[n + 1] += out_ptr[n]; }
  std::vector<uint32_t> inc(inc_ptr[Nn]);
  std::vector<int> out_e(out_ptr[Nn]);
  {
    std::vector<int> fi(inc_ptr.begin(), inc_ptr.end() - 1), fo(out_ptr.begin(), out_ptr.end() - 1);
    for (int e = 0; e < E; ++e) {  // edge order => each node's list is sorted by edge id
      int u = desc->edge_src[e], w = desc->edge_dst[e];
      inc[fi[u]++] = (uint32_t)e | kSignBit;
      inc[fi[w]++] = (uint32_t)e;
      out_e[fo[u]++] = e;
    }
  }
  std::vector<int> pair_of((size_t)S * Nn, -1);
  std::vector<double> out_units(S, 0.0);
  for (int p = 0; p < P; ++p) {
    int s = desc->pair_source[p], w = desc->pair_dst[p];
    if (s < 0 || s >= S || w < 0 || w >= Nn || desc->node_is_switch[w] ||
        w == desc->source_node[s]) { set_error("bad demand pair"); return TECCL_EINVAL; }
    if (pair_of[(size_t)s * Nn + w] >= 0) { set_error("duplicate demand pair"); return TECCL_EINVAL; }
    pair_of[(size_t)s * Nn + w] = p;
    out_units[s] += desc->pair_units[p];
  }
  for (int s = 0; s < S; ++s) {
    int n = desc->source_node[s];
    if (n < 0 || n >= Nn || desc->node_is_switch[n]) { set_error("source is not a GPU"); return TECCL_EINVAL; }
  }

  d = TeDev{};
  d.Nn = Nn; d.E = E; d.S = S; d.P = P; d.K = K; d.G = G;
  d.SB = (int64_t)E * K + (int64_t)G * (K + 1);
  d.CB = (int64_t)Nn * K + G - 1;
  d.R_cons = S + (int64_t)E * K;
  d.R_cum = d.R_cons + (int64_t)S * d.CB;
  d.R_bcap = d.R_cum + (int64_t)P * K;
  d.has_bcap = desc->buffer_limit >= 0.0;
  d.phase1 = desc->phase1 != 0;
  d.blimit = desc->buffer_limit;
  d.n_rows = d.R_bcap + (d.has_bcap ? (int64_t)G * (K + 1) : 0);
  d.n_vars = (int64_t)S * d.SB + (int64_t)P * 2 * K;
  if (S == 0) d.CB = 0;

  // Upload the small tables.
  std::vector<uint8_t> is_sw(desc->node_is_switch, desc->node_is_switch + Nn);
  std::vector<int> esrc(desc->edge_src, desc->edge_src + E), edst(desc->edge_dst, desc->edge_dst + E),
      edel(desc->edge_delta, desc->edge_delta + E), snode(desc->source_node, desc->source_node + S),
      psrc(desc->pair_source, desc->pair_source + P), pdst(desc->pair_dst, desc->pair_dst + P);
  std::vector<double> ecap(desc->edge_cap, desc->edge_cap + (size_t)E * K),
      pu(desc->pair_units, desc->pair_units + P);
  auto up = [&](auto& vec, auto** dptr) -> int {
    int rc = upload(vec, dptr, st);
    owned.push_back((void*)*dptr);
    return rc;
  };
  uint8_t* d_is_sw; int *d_gpu_of, *d_gpre, *d_nog, *d_esrc, *d_edst, *d_edel, *d_snode, *d_psrc,
      *d_pdst, *d_pair_of, *d_inc_ptr, *d_out_ptr, *d_out_e;
  double *d_ecap, *d_pu, *d_ou;
  uint32_t* d_inc;
  int rc = 0;
  rc |= up(is_sw, &d_is_sw); rc |= up(gpu_of, &d_gpu_of); rc |= up(gpre, &d_gpre);
  rc |= up(node_of_gpu, &d_nog); rc |= up(esrc, &d_esrc); rc |= up(edst, &d_edst);
  rc |= up(edel, &d_edel); rc |= up(ecap, &d_ecap); rc |= up(snode, &d_snode);
  rc |= up(psrc, &d_psrc); rc |= up(pdst, &d_pdst); rc |= up(pu, &d_pu);
  rc |= up(pair_of, &d_pair_of); rc |= up(out_units, &d_ou); rc |= up(inc_ptr, &d_inc_ptr);
  rc |= up(inc, &d_inc); rc |= up(out_ptr, &d_out_ptr); rc |= up(out_e, &d_out_e);
  if (rc) return TECCL_ECUDA;
  d.is_sw = d_is_sw; d.gpu_of = d_gpu_of; d.gpre = d_gpre; d.node_of_gpu = d_nog;
  d.esrc = d_esrc; d.edst = d_edst; d.edelta = d_edel; d.ecap = d_ecap; d.snode = d_snode;
  d.pair_src = d_psrc; d.pair_dst = d_pdst; d.pair_u = d_pu; d.pair_of = d_pair_of;
  d.out_units = d_ou; d.inc_ptr = d_inc_ptr; d.inc = d_inc; d.out_ptr = d_out_ptr; d.out_e = d_out_e;

  return TECCL_OK;
}

}  // namespace

namespace {

// Bound-class dictionaries (pdlp.cu reads bounds/costs through them).
// Columns: [0] free (0,inf,0), [1] fixed (0,0,0), [2+u] Rd (0,U_u,0),
// [2+nU+u*K+k] Rc (0 or U_u at k=K-1, U_u, -1/(k+1)). Rows: [0] (0,0),
// [1+o] init (OU_o,OU_o), [1+nOU+c] cap (-inf,CAP_c), [1+nOU+nCap] bcap.
int setup_dicts(const teccl_te_desc* desc, TeDev& d, teccl_lp* lp, std::vector<void*>& owned,
                cudaStream_t st, int64_t m, int64_t n) {
  {
    std::vector<double> U(desc->pair_units, desc->pair_units + desc->num_pairs);
    std::sort(U.begin(), U.end());
    U.erase(std::unique(U.begin(), U.end()), U.end());
    std::vector<int> puidx(desc->num_pairs);
    for (int p = 0; p < desc->num_pairs; ++p)
      puidx[p] = (int)(std::lower_bound(U.begin(), U.end(), desc->pair_units[p]) - U.begin());
    std::vector<double> ou(desc->num_sources, 0.0);
    for (int p = 0; p < desc->num_pairs; ++p) ou[desc->pair_source[p]] += desc->pair_units[p];
    std::vector<double> OU(ou);
    std::sort(OU.begin(), OU.end());
    OU.erase(std::unique(OU.begin(), OU.end()), OU.end());
    std::vector<int> souidx(desc->num_sources);
    for (int s = 0; s < desc->num_sources; ++s)
      souidx[s] = (int)(std::lower_bound(OU.begin(), OU.end(), ou[s]) - OU.begin());
    const size_t EK = (size_t)desc->num_edges * desc->K;
    std::vector<double> CAPS(desc->edge_cap, desc->edge_cap + EK);
    std::sort(CAPS.begin(), CAPS.end());
    CAPS.erase(std::unique(CAPS.begin(), CAPS.end()), CAPS.end());
    const int K = desc->K, nU = (int)U.size(), nOU = (int)OU.size(), nCap = (int)CAPS.size();
    const int64_t ncd = 2 + (int64_t)nU * (K + 1);
    const int64_t nrd = 1 + nOU + nCap + 1;
    d.nU = nU; d.nOU = nOU; d.nCap = nCap;
    d.dict_col = ncd <= kMaxDict && !d.phase1;  // phase-1 costs are not in the dictionary
    d.dict_row = nrd <= kMaxDict;
    if (d.dict_col) {
      std::vector<double> cd(3 * ncd);
      auto put = [&](int64_t i, double a, double b, double c) { cd[3 * i] = a; cd[3 * i + 1] = b; cd[3 * i + 2] = c; };
      put(0, 0.0, INFINITY, 0.0);
      put(1, 0.0, 0.0, 0.0);
      for (int u = 0; u < nU; ++u) put(2 + u, 0.0, U[u], 0.0);
      for (int u = 0; u < nU; ++u)
        for (int k = 0; k < K; ++k)
          put(2 + nU + (int64_t)u * K + k, k == K - 1 ? U[u] : 0.0, U[u], -1.0 / (double)(k + 1));
      int* dp = nullptr;
      if (upload(puidx, &dp, st)) return TECCL_ECUDA;
      owned.push_back(dp);
      d.pair_uidx = dp;
      if (upload(cd, &lp->col_dict, st)) return TECCL_ECUDA;
      lp->n_col_dict = (int32_t)ncd;
      TECCL_CUDA(cudaMallocAsync((void**)&lp->col_code, (n + 1) * sizeof(uint16_t), st));
    }
    if (d.dict_row) {
      std::vector<double> rd(2 * nrd);
      rd[0] = 0.0; rd[1] = 0.0;
      for (int o = 0; o < nOU; ++o) { rd[2 * (1 + o)] = OU[o]; rd[2 * (1 + o) + 1] = OU[o]; }
      for (int c = 0; c < nCap; ++c) { rd[2 * (1 + nOU + c)] = -INFINITY; rd[2 * (1 + nOU + c) + 1] = CAPS[c]; }
      rd[2 * (nrd - 1)] = -INFINITY;
      rd[2 * (nrd - 1) + 1] = desc->buffer_limit;
      std::vector<uint16_t> cidx(EK);
      for (size_t q = 0; q < EK; ++q)
        cidx[q] = (uint16_t)(std::lower_bound(CAPS.begin(), CAPS.end(), desc->edge_cap[q]) - CAPS.begin());
      int* so = nullptr;
      uint16_t* ci = nullptr;
      if (upload(souidx, &so, st) || upload(cidx, &ci, st)) return TECCL_ECUDA;
      owned.push_back(so);
      owned.push_back(ci);
      d.src_ouidx = so;
      d.cap_idx = ci;
      if (upload(rd, &lp->row_dict, st)) return TECCL_ECUDA;
      lp->n_row_dict = (int32_t)nrd;
      TECCL_CUDA(cudaMallocAsync((void**)&lp->row_code, (m + 1) * sizeof(uint16_t), st));
    }
  }
  return TECCL_OK;
}

}  // namespace

namespace {
// packed tables of the matrix-free operator (TeOp in te_gen.cuh)
int te_op_tables(const teccl_te_desc* desc, TeHold* h, cudaStream_t st) {
  TeOp& o = h->op;
  const int Nn = desc->num_nodes, E = desc->num_edges, S = desc->num_sources, P = desc->num_pairs;
  const int64_t K = desc->K;
  std::vector<int> gpre(Nn, 0);
  for (int n = 0, g = 0; n < Nn; ++n) { gpre[n] = g; if (!desc->node_is_switch[n]) ++g; }
  std::vector<int4> edge4(E);
  for (int e = 0; e < E; ++e) edge4[e] = make_int4(desc->edge_src[e], desc->edge_dst[e], desc->edge_delta[e], 0);
  std::vector<int2> sntab((size_t)S * Nn);
  for (int s = 0; s < S; ++s)
    for (int n = 0; n < Nn; ++n) {
      const int sn = desc->source_node[s];
      const int64_t first = (int64_t)o.R_cons + (int64_t)s * o.CB + (int64_t)n * K + gpre[n] - (sn < n ? 1 : 0);
      const bool has_last = !desc->node_is_switch[n] && n != sn;
      sntab[(size_t)s * Nn + n] = make_int2((int)((uint32_t)first | (has_last ? kSignBit : 0u)), -1);
    }
  for (int p = 0; p < P; ++p)
    sntab[(size_t)desc->pair_source[p] * Nn + desc->pair_dst[p]].y = (int)(o.nF + (int64_t)p * 2 * K);
  std::vector<int4> sefam((size_t)S * E);
  for (int s = 0; s < S; ++s)
    for (int e = 0; e < E; ++e) {
      const int u = desc->edge_src[e], w = desc->edge_dst[e];
      sefam[(size_t)s * E + e] = make_int4((int)((uint32_t)sntab[(size_t)s * Nn + u].x & kIdxMask),
                                           sntab[(size_t)s * Nn + w].x, desc->edge_delta[e],
                                           u == desc->source_node[s] ? 1 : 0);
    }
  // incident entries in the builder's order: per node, edges ascending, each
  // edge once as leaving (at its source) and once as arriving (at its dst)
  std::vector<int> cnt(Nn + 1, 0);
  for (int e = 0; e < E; ++e) { cnt[desc->edge_src[e] + 1]++; cnt[desc->edge_dst[e] + 1]++; }
  for (int n = 0; n < Nn; ++n) cnt[n + 1] += cnt[n];
  std::vector<int2> incp(cnt[Nn]);
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < E; ++e) {
      incp[fill[desc->edge_src[e]]++] = make_int2((int)(e * K + 1), -1);
      incp[fill[desc->edge_dst[e]]++] = make_int2((int)(e * K - desc->edge_delta[e]), desc->edge_delta[e]);
    }
  }
  o.dmax = 0;
  for (int e = 0; e < E; ++e) o.dmax = std::max(o.dmax, (int)desc->edge_delta[e]);
  // segment tasks, in memory order (seg_cols / seg_rows in te_gen.cuh)
  std::vector<int4> ct, rt;
  auto add = [](std::vector<int4>& v, int kind, int a, int b, int64_t start, int64_t len) {
    for (int64_t off = 0; off < len; off += kSegTask) {
      const int cnt = (int)std::min<int64_t>(kSegTask, len - off);
      v.push_back(make_int4(kind | (a << 4), b, (int)(start + off), (int)(off | ((int64_t)cnt << 24))));
    }
  };
  const int G = (int)(o.SB - (int64_t)E * K) / (int)(K + 1);
  for (int s = 0; s < S; ++s) {
    for (int e = 0; e < E; ++e) add(ct, SEG_F, s, e, (int64_t)s * o.SB + (int64_t)e * K, K);
    for (int g = 0; g < G; ++g) add(ct, SEG_B, s, g, (int64_t)s * o.SB + o.EK + (int64_t)g * (K + 1), K + 1);
  }
  for (int p = 0; p < P; ++p) add(ct, SEG_P, p, 0, (int64_t)o.nF + (int64_t)p * 2 * K, 2 * K);
  add(rt, SEG_INIT, 0, 0, 0, S);
  for (int e = 0; e < E; ++e) add(rt, SEG_CAP, 0, e, (int64_t)S + (int64_t)e * K, K);
  for (int s = 0; s < S; ++s)
    for (int n = 0; n < Nn; ++n) {
      const uint32_t f = (uint32_t)sntab[(size_t)s * Nn + n].x;
      add(rt, SEG_CONS, s, n, f & kIdxMask, K + ((f & kSignBit) ? 1 : 0));
    }
  for (int p = 0; p < P; ++p) add(rt, SEG_CUM, p, 0, (int64_t)o.R_cum + (int64_t)p * K, K);
  if (o.has_bcap)
    for (int g = 0; g < G; ++g) add(rt, SEG_BCAP, 0, g, (int64_t)o.R_bcap + (int64_t)g * (K + 1), K + 1);
  // Epoch-tile-major task order: every family's tasks for epochs
  // [64t, 64t + 64) run next to each other, so the gathered vector is
  // touched by all its rows (columns) within a window of a few epoch tiles
  // and is read from HBM once per half-step instead of once per family
  // pass (x-bar is read by the capacity rows and again by two conservation
  // rows per flow column).
  auto tile = [](const int4& t) {
    const int kind = t.x & 15, off = t.w & 0xffffff;
    return kind == SEG_P ? off / (2 * kSegTask) : off / kSegTask;
  };
  auto by_tile = [&](const int4& a, const int4& b) { return tile(a) < tile(b); };
  std::stable_sort(ct.begin(), ct.end(), by_tile);
  std::stable_sort(rt.begin(), rt.end(), by_tile);
  std::vector<double> ninv(K);
  for (int64_t k = 0; k < K; ++k) ninv[k] = -1.0 / (double)(k + 1);
  int4* d4 = nullptr; int2* ds = nullptr; int2* di = nullptr;
  int4 *dct = nullptr, *drt = nullptr, *dsf = nullptr;
  double* dni = nullptr;
  if (upload(edge4, &d4, st) || upload(sntab, &ds, st) || upload(incp, &di, st) ||
      upload(ct, &dct, st) || upload(rt, &drt, st) || upload(ninv, &dni, st) || upload(sefam, &dsf, st))
    return TECCL_ECUDA;
  for (void* p : {(void*)d4, (void*)ds, (void*)di, (void*)dct, (void*)drt, (void*)dni, (void*)dsf})
    h->owned.push_back(p);
  o.edge4 = d4; o.sntab = ds; o.incp = di; o.sefam = dsf;
  o.ctask = dct; o.rtask = drt; o.neg_inv = dni;
  o.n_ctask = (int)ct.size(); o.n_rtask = (int)rt.size();
  return TECCL_OK;
}

// tables of the epoch-major matrix-free operator of one partition block
int em_op_tables(const teccl_te_desc* desc, TeHold* h, cudaStream_t st) {
  EmOp& o = h->em;
  const int E = desc->num_edges, Nn = desc->num_nodes;
  const int64_t K = desc->K;
  std::vector<int4> edge4(E);
  for (int e = 0; e < E; ++e) edge4[e] = make_int4(desc->edge_src[e], desc->edge_dst[e], desc->edge_delta[e], 0);
  std::vector<int> cnt(Nn + 1, 0);
  for (int e = 0; e < E; ++e) { cnt[desc->edge_src[e] + 1]++; cnt[desc->edge_dst[e] + 1]++; }
  for (int n = 0; n < Nn; ++n) cnt[n + 1] += cnt[n];
  std::vector<int2> incE(std::max(1, cnt[Nn]));
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < E; ++e) {
      incE[fill[desc->edge_src[e]]++] = make_int2(e, -1);
      incE[fill[desc->edge_dst[e]]++] = make_int2(e, desc->edge_delta[e]);
    }
  }
  std::vector<double> ninv(K);
  for (int64_t k = 0; k < K; ++k) ninv[k] = -1.0 / (double)(k + 1);
  int4* d4 = nullptr; int2* di = nullptr; double* dni = nullptr;
  if (upload(edge4, &d4, st) || upload(incE, &di, st) || upload(ninv, &dni, st)) return TECCL_ECUDA;
  for (void* p : {(void*)d4, (void*)di, (void*)dni}) h->owned.push_back(p);
  o.edge4 = d4; o.incE = di; o.neg_inv = dni;
  return TECCL_OK;
}

void free_te_hold(void* p) {
  TeHold* h = (TeHold*)p;
  for (void* q : h->owned) cudaFreeAsync(q, h->st);
  cudaStreamSynchronize(h->st);
  delete h;
}
}  // namespace

extern "C" int teccl_lp_build_te(teccl_ctx* ctx, const teccl_te_desc* desc, teccl_lp** out) {
  if (!ctx || !desc || !out) { set_error("null argument"); return TECCL_EINVAL; }
  TeDev d;
  std::vector<void*> owned;
  cudaStream_t st = ctx->stream;
  int prc = prepare_tables(ctx, desc, d, owned);
  if (prc) { for (void* p : owned) cudaFreeAsync(p, st); return prc; }
  if (d.n_vars >= (int64_t)kSignBit || d.n_rows >= (int64_t)kSignBit) {
    for (void* p : owned) cudaFreeAsync(p, st);
    set_error("LP too large for 31-bit indices on one device; row-partition it");
    return TECCL_EINVAL;
  }
  teccl_lp* lp = new teccl_lp();
  lp->m = (int32_t)d.n_rows;
  lp->n = (int32_t)d.n_vars;
  lp->unit = true;
  lp->device = ctx->device;
  lp->stream = st;
  const int64_t m = d.n_rows, n = d.n_vars;
  int64_t *row_len = nullptr, *col_len = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_ptr, (m + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->col_ptr, (n + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&row_len, (m + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&col_len, (n + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_lo, (m + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_hi, (m + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->var_lb, (n + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->var_ub, (n + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->obj, (n + 1) * sizeof(double), st));

  if (int rc = setup_dicts(desc, d, lp, owned, st, m, n)) return rc;

  if (m > 0) {
    te_rows_kernel<false><<<grid_for(m), kThreads, 0, st>>>(d, nullptr, nullptr, row_len, nullptr, nullptr, nullptr);
    TECCL_CHECK_LAUNCH();
    if (scan_lengths(row_len, lp->row_ptr, m, st)) return TECCL_ECUDA;
  } else {
    TECCL_CUDA(cudaMemsetAsync(lp->row_ptr, 0, sizeof(int64_t), st));
  }
  if (n > 0) {
    te_cols_kernel<false><<<grid_for(n), kThreads, 0, st>>>(d, nullptr, nullptr, col_len, nullptr, nullptr, nullptr, nullptr);
    TECCL_CHECK_LAUNCH();
    if (scan_lengths(col_len, lp->col_ptr, n, st)) return TECCL_ECUDA;
  } else {
    TECCL_CUDA(cudaMemsetAsync(lp->col_ptr, 0, sizeof(int64_t), st));
  }
  int64_t nnz_r = 0, nnz_c = 0;
  TECCL_CUDA(cudaMemcpyAsync(&nnz_r, lp->row_ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaMemcpyAsync(&nnz_c, lp->col_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  if (nnz_r != nnz_c) {
    set_error("builder internal error: CSR and CSC disagree on nnz");
    return TECCL_EINVAL;
  }
  lp->nnz = nnz_r;
  TECCL_CUDA(cudaMallocAsync((void**)&lp->col, (nnz_r + 1) * sizeof(uint32_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row, (nnz_r + 1) * sizeof(uint32_t), st));
  if (m > 0) {
    te_rows_kernel<true><<<grid_for(m), kThreads, 0, st>>>(d, lp->row_ptr, lp->col, nullptr, lp->row_lo, lp->row_hi, lp->row_code);
    TECCL_CHECK_LAUNCH();
  }
  if (n > 0) {
    te_cols_kernel<true><<<grid_for(n), kThreads, 0, st>>>(d, lp->col_ptr, lp->row, nullptr, lp->var_lb, lp->var_ub, lp->obj, lp->col_code);
    TECCL_CHECK_LAUNCH();
  }
  TECCL_CUDA(cudaFreeAsync(row_len, st));
  TECCL_CUDA(cudaFreeAsync(col_len, st));
  // keep the tables: the PDLP kernels apply A / A^T from them (matrix-free)
  TeHold* h = new TeHold();
  te_op_init(h->op, d);
  h->owned.swap(owned);
  h->st = st;
  if (int rc = te_op_tables(desc, h, st)) { free_te_hold(h); return rc; }
  lp->te = h;
  lp->te_free = free_te_hold;
  TECCL_CUDA(cudaStreamSynchronize(st));
  *out = lp;
  return TECCL_OK;
}


extern "C" int teccl_lp_build_te_part(teccl_ctx* ctx, const teccl_te_desc* desc, int32_t world,
                                      int32_t rank, teccl_lp** out, int64_t* info) {
  if (!ctx || !desc || !out || !info) { set_error("null argument"); return TECCL_EINVAL; }
  if (world < 1 || rank < 0 || rank >= world) { set_error("bad world/rank"); return TECCL_EINVAL; }
  TeDev d;
  std::vector<void*> owned;
  cudaStream_t st = ctx->stream;
  int prc = prepare_tables(ctx, desc, d, owned);
  if (prc) { for (void* p : owned) cudaFreeAsync(p, st); return prc; }
  const EmShape z = em_shape(d);
  const int K = d.K;
  int dmax = 0;
  for (int e = 0; e < desc->num_edges; ++e) dmax = std::max(dmax, (int)desc->edge_delta[e]);
  auto krange = [&](int r, int64_t& k0, int64_t& k1) {
    k0 = (int64_t)r * K / world;
    k1 = (int64_t)(r + 1) * K / world;
  };
  auto owned_cols = [&](int r, int64_t& c0, int64_t& c1) {
    int64_t k0, k1;
    krange(r, k0, k1);
    c0 = k0 * z.CW;
    c1 = (r == world - 1) ? z.n_cols : k1 * z.CW;
  };
  auto owned_rows = [&](int r, int64_t& r0, int64_t& r1) {
    int64_t k0, k1;
    krange(r, k0, k1);
    r0 = (r == 0) ? 0 : d.S + k0 * z.RW;
    r1 = (r == world - 1) ? z.n_rows : d.S + k1 * z.RW;
  };
  for (int r = 0; r < world; ++r) {
    int64_t k0, k1;
    krange(r, k0, k1);
    if (world > 1 && k1 - k0 < dmax + 2) {
      set_error("epoch blocks too thin: every rank needs >= delta_max + 2 epochs");
      return TECCL_EINVAL;
    }
  }
  int64_t k0, k1, c0, c1, r0, r1;
  krange(rank, k0, k1);
  owned_cols(rank, c0, c1);
  owned_rows(rank, r0, r1);
  const int64_t nr = r1 - r0, nc = c1 - c0;
  if (nr >= (int64_t)kSignBit || nc >= (int64_t)kSignBit) {
    set_error("partition too large for 31-bit local indices; use more ranks");
    return TECCL_EINVAL;
  }
  teccl_lp* lp = new teccl_lp();
  lp->m = (int32_t)nr;
  lp->n = (int32_t)nc;
  lp->unit = true;
  lp->device = ctx->device;
  lp->stream = st;
  lp->part_world = world;
  lp->part_rank = rank;
  lp->em_ncols = z.n_cols;
  lp->em_nrows = z.n_rows;
  lp->own_c0 = c0; lp->own_c1 = c1; lp->own_r0 = r0; lp->own_r1 = r1;
  int64_t *row_len = nullptr, *col_len = nullptr;
  unsigned long long* mm = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_ptr, (nr + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->col_ptr, (nc + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&row_len, (nr + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&col_len, (nc + 1) * sizeof(int64_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_lo, (nr + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row_hi, (nr + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->var_lb, (nc + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->var_ub, (nc + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->obj, (nc + 1) * sizeof(double), st));
  TECCL_CUDA(cudaMallocAsync((void**)&mm, 4 * sizeof(unsigned long long), st));
  const unsigned long long mm0[4] = {~0ull, 0ull, ~0ull, 0ull};
  TECCL_CUDA(cudaMemcpyAsync(mm, mm0, sizeof(mm0), cudaMemcpyHostToDevice, st));
  if (int rc = setup_dicts(desc, d, lp, owned, st, nr, nc)) return rc;

  part_rows_kernel<false><<<grid_for(nr), kThreads, 0, st>>>(d, z, r0, nr, 0, nullptr, nullptr, row_len, nullptr, nullptr, nullptr, mm);
  part_cols_kernel<false><<<grid_for(nc), kThreads, 0, st>>>(d, z, c0, nc, 0, nullptr, nullptr, col_len, nullptr, nullptr, nullptr, nullptr, mm + 2);
  TECCL_CHECK_LAUNCH();
  if (scan_lengths(row_len, lp->row_ptr, nr, st)) return TECCL_ECUDA;
  if (scan_lengths(col_len, lp->col_ptr, nc, st)) return TECCL_ECUDA;
  unsigned long long mmh[4];
  int64_t nnz_r = 0, nnz_c = 0;
  TECCL_CUDA(cudaMemcpyAsync(mmh, mm, sizeof(mmh), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaMemcpyAsync(&nnz_r, lp->row_ptr + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaMemcpyAsync(&nnz_c, lp->col_ptr + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  const int64_t cw0 = std::min<int64_t>(nnz_r ? (int64_t)mmh[0] : c0, c0);
  const int64_t cw1 = std::max<int64_t>(nnz_r ? (int64_t)mmh[1] + 1 : c1, c1);
  const int64_t rw0 = std::min<int64_t>(nnz_c ? (int64_t)mmh[2] : r0, r0);
  const int64_t rw1 = std::max<int64_t>(nnz_c ? (int64_t)mmh[3] + 1 : r1, r1);
  // halos must come from the two neighbours only
  if (world > 1) {
    int64_t a, b;
    if (rank > 0) { owned_cols(rank - 1, a, b); if (cw0 < a) { set_error("column halo reaches past the previous rank"); return TECCL_EINVAL; } }
    if (rank < world - 1) { owned_cols(rank + 1, a, b); if (cw1 > b) { set_error("column halo reaches past the next rank"); return TECCL_EINVAL; } }
    if (rank > 0) { owned_rows(rank - 1, a, b); if (rw0 < a) { set_error("row halo reaches past the previous rank"); return TECCL_EINVAL; } }
    if (rank < world - 1) { owned_rows(rank + 1, a, b); if (rw1 > b) { set_error("row halo reaches past the next rank"); return TECCL_EINVAL; } }
  }
  lp->win_c0 = cw0; lp->win_c1 = cw1; lp->win_r0 = rw0; lp->win_r1 = rw1;
  lp->nnz = nnz_r;
  lp->nnz_csc = nnz_c;
  TECCL_CUDA(cudaMallocAsync((void**)&lp->col, (nnz_r + 1) * sizeof(uint32_t), st));
  TECCL_CUDA(cudaMallocAsync((void**)&lp->row, (nnz_c + 1) * sizeof(uint32_t), st));
  part_rows_kernel<true><<<grid_for(nr), kThreads, 0, st>>>(d, z, r0, nr, cw0, lp->row_ptr, lp->col, nullptr, lp->row_lo, lp->row_hi, lp->row_code, mm);
  part_cols_kernel<true><<<grid_for(nc), kThreads, 0, st>>>(d, z, c0, nc, rw0, lp->col_ptr, lp->row, nullptr, lp->var_lb, lp->var_ub, lp->obj, lp->col_code, mm + 2);
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaFreeAsync(row_len, st));
  TECCL_CUDA(cudaFreeAsync(col_len, st));
  TECCL_CUDA(cudaFreeAsync(mm, st));
  // keep the tables: the PDLP kernels apply the block's rows / columns from
  // them (epoch-major matrix-free operator, te_gen.cuh EmOp)
  {
    TeHold* h = new TeHold();
    h->kind = 1;
    EmOp& o = h->em;
    o.d = d;
    o.K = (uint32_t)K; o.S = (uint32_t)d.S; o.E = (uint32_t)d.E; o.G = (uint32_t)d.G;
    o.Nn = (uint32_t)d.Nn; o.P = (uint32_t)d.P;
    o.CW = (uint32_t)z.CW; o.RW = (uint32_t)z.RW;
    o.SE = (uint32_t)((int64_t)d.S * d.E); o.SEG = (uint32_t)((int64_t)d.S * d.E + (int64_t)d.S * d.G);
    o.k0 = (uint32_t)k0; o.nk = (uint32_t)(k1 - k0); o.tail_k = (uint32_t)(K - k0);
    o.c0 = c0; o.r0 = r0; o.wc0 = cw0; o.wr0 = rw0;
    o.n = (uint32_t)nc; o.m = (uint32_t)nr;
    o.has_bcap = d.has_bcap; o.phase1 = d.phase1;
    o.fCW.init(o.CW); o.fRW.init(o.RW); o.fE.init(o.E > 0 ? o.E : 1); o.fG.init(o.G > 0 ? o.G : 1);
    o.fNn.init(o.Nn); o.fGm1.init(o.G > 1 ? o.G - 1 : 1);
    h->owned.swap(owned);
    h->st = st;
    if (int rc = em_op_tables(desc, h, st)) { free_te_hold(h); return rc; }
    lp->te = h;
    lp->te_free = free_te_hold;
  }
  TECCL_CUDA(cudaStreamSynchronize(st));
  const int64_t vals[16] = {c0, c1, r0, r1, cw0, cw1, rw0, rw1, k0, k1, z.n_cols, z.n_rows,
                            dmax, nnz_r, nnz_c, z.CW};
  for (int i = 0; i < 16; ++i) info[i] = vals[i];
  *out = lp;
  return TECCL_OK;
}

// ---------------------------------------------------------------------------
// (4) Exact-integer schedule checker / epoch simulator over an LP solution.
// Independent of the LP rows: buffers are replayed from the flows alone
// (reference simulator semantics, simulator.py:119-189, restated for the
// copy-free per-source flow): a GPU starts with its outgoing demand, loses
// what it sends and reads, gains what lands delta epochs after a send; a
// switch must forward exactly what lands, the next epoch.

namespace teccl {

struct CheckOut {
  unsigned long long cap_viol, causal_viol, switch_viol, unmet;
  long long max_cap_excess, max_deficit;
  int completion;
};

__device__ __forceinline__ long long qnt(double v, double Q) { return llrint(v * Q); }

__global__ void check_capacity_kernel(TeDev d, const double* __restrict__ x, double Q,
                                      long long slack, CheckOut* out) {
  const int64_t total = (int64_t)d.E * d.K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(t / d.K), k = (int)(t % d.K);
    long long load = 0;
    for (int s = 0; s < d.S; ++s) load += qnt(x[varF(d, s, e, k)], Q);
    const long long capq = (long long)floor(d.ecap[t] * Q);
    const long long excess = load - capq;
    if (excess > slack) atomicAdd(&out->cap_viol, 1ull);
    if (excess > 0) atomicMax(&out->max_cap_excess, excess);
  }
}

__global__ void check_replay_kernel(TeDev d, const double* __restrict__ x, double Q,
                                    long long slack, CheckOut* out) {
  const int64_t total = (int64_t)d.S * d.Nn;
  const int K = d.K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t / d.Nn), n = (int)(t % d.Nn);
    const int g = d.gpu_of[n];
    const int pair = g >= 0 ? d.pair_of[s * d.Nn + n] : -1;
    auto inflow = [&](int k) {
      long long a = 0;
      for (int j = d.inc_ptr[n]; j < d.inc_ptr[n + 1]; ++j) {
        const uint32_t w = d.inc[j];
        if (w & kSignBit) continue;
        const int e = (int)(w & kIdxMask);
        const int kin = k - d.edelta[e];
        if (kin >= 0) a += qnt(x[varF(d, s, e, kin)], Q);
      }
      return a;
    };
    auto outflow = [&](int k) {
      long long a = 0;
      for (int j = d.out_ptr[n]; j < d.out_ptr[n + 1]; ++j) a += qnt(x[varF(d, s, d.out_e[j], k)], Q);
      return a;
    };
    if (g < 0) {  // switch: forward exactly what lands, one epoch later
      for (int k = 0; k < K; ++k) {
        const long long in = inflow(k);
        const long long o = (k + 1 <= K - 1) ? outflow(k + 1) : 0;
        const long long diff = in > o ? in - o : o - in;
        if (diff > slack) atomicAdd(&out->switch_viol, 1ull);
      }
      if (outflow(0) > slack) atomicAdd(&out->switch_viol, 1ull);
      continue;
    }
    long long hold = (n == d.snode[s]) ? qnt(d.out_units[s], Q) : 0;
    long long worst = 0;
    int bad = 0;
    hold -= outflow(0);
    if (hold < -slack) ++bad;
    if (hold < worst) worst = hold;
    for (int k = 0; k < K; ++k) {
      hold += inflow(k);
      if (pair >= 0) hold -= qnt(x[varRd(d, pair, k)], Q);
      if (k + 1 <= K - 1) hold -= outflow(k + 1);
      if (hold < -slack) ++bad;
      if (hold < worst) worst = hold;
    }
    if (bad) atomicAdd(&out->causal_viol, (unsigned long long)bad);
    if (worst < 0) atomicMax(&out->max_deficit, -worst);
  }
}

__global__ void check_demand_kernel(TeDev d, const double* __restrict__ x, double Q,
                                    long long slack, CheckOut* out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < d.P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const long long need = qnt(d.pair_u[p], Q);
    long long cum = 0;
    int done = -1;
    for (int k = 0; k < d.K; ++k) {
      cum += qnt(x[varRd(d, (int)p, k)], Q);
      if (done < 0 && cum >= need - slack) done = k;
    }
    if (done < 0) atomicAdd(&out->unmet, 1ull);
    else atomicMax(&out->completion, done);
  }
}

}  // namespace teccl

extern "C" int teccl_check_te_dev(teccl_ctx* ctx, const teccl_te_desc* desc, const double* x_dev,
                                  int64_t quantum, int64_t slack_units, teccl_check_report* rep) {
  if (!ctx || !desc || !x_dev || !rep || quantum < 1 || slack_units < 0) {
    set_error("bad argument");
    return TECCL_EINVAL;
  }
  TECCL_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  TeDev d;
  std::vector<void*> owned;
  int rc = prepare_tables(ctx, desc, d, owned);
  if (rc) { for (void* p : owned) cudaFreeAsync(p, st); return rc; }
  CheckOut h{0, 0, 0, 0, 0, 0, -1};
  CheckOut* dout = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)&dout, sizeof(CheckOut), st));
  TECCL_CUDA(cudaMemcpyAsync(dout, &h, sizeof(CheckOut), cudaMemcpyHostToDevice, st));
  const double Q = (double)quantum;
  const long long slack = slack_units;
  check_capacity_kernel<<<grid_for((int64_t)d.E * d.K), kThreads, 0, st>>>(d, x_dev, Q, slack, dout);
  check_replay_kernel<<<grid_for((int64_t)d.S * d.Nn, 64), 64, 0, st>>>(d, x_dev, Q, slack, dout);
  check_demand_kernel<<<grid_for(d.P, 64), 64, 0, st>>>(d, x_dev, Q, slack, dout);
  TECCL_CHECK_LAUNCH();
  TECCL_CUDA(cudaMemcpyAsync(&h, dout, sizeof(CheckOut), cudaMemcpyDeviceToHost, st));
  TECCL_CUDA(cudaFreeAsync(dout, st));
  for (void* p : owned) TECCL_CUDA(cudaFreeAsync(p, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  rep->capacity_violations = (int64_t)h.cap_viol;
  rep->causality_violations = (int64_t)h.causal_viol;
  rep->switch_violations = (int64_t)h.switch_viol;
  rep->unmet_pairs = (int64_t)h.unmet;
  rep->completion_epoch = h.completion;
  rep->max_capacity_excess = h.max_cap_excess;
  rep->max_buffer_deficit = h.max_deficit;
  return TECCL_OK;
}

extern "C" int teccl_check_te(teccl_ctx* ctx, const teccl_te_desc* desc, const double* x_host,
                              int64_t quantum, int64_t slack_units, teccl_check_report* rep) {
  if (!ctx || !desc || !x_host) { set_error("bad argument"); return TECCL_EINVAL; }
  const int64_t K = desc->K;
  int G = 0;
  for (int i = 0; i < desc->num_nodes; ++i) G += desc->node_is_switch[i] ? 0 : 1;
  const int64_t n = (int64_t)desc->num_sources * ((int64_t)desc->num_edges * K + (int64_t)G * (K + 1)) +
                    (int64_t)desc->num_pairs * 2 * K;
  double* xd = nullptr;
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  TECCL_CUDA(cudaMallocAsync((void**)&xd, sizeof(double) * (n + 1), st));
  TECCL_CUDA(cudaMemcpyAsync(xd, x_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  int rc = teccl_check_te_dev(ctx, desc, xd, quantum, slack_units, rep);
  cudaFreeAsync(xd, st);
  cudaStreamSynchronize(st);
  return rc;
}

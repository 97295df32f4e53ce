// Time-expanded LP structure shared by the builder (te_build.cu) and the
// PDLP iteration kernels (pdlp.cu).
//
// TeDev holds the small per-node / per-edge / per-pair tables the copy-free
// TE-CCL LP (reference pkg/src/collsched/lp.py:22-136) is generated from.
// TeOp adds 32-bit invariant-divisor constants so the iteration kernels can
// apply A and A^T straight from those tables ("matrix-free"): every entry is
// +-1 and its row/column index is a closed form in (source, edge/GPU/pair,
// epoch), so no index stream is read from HBM at all.
#pragma once

#include <cmath>
#include <vector>

#include "common.cuh"

namespace teccl {

struct TeDev {
  int Nn, E, S, P, K, G;
  int64_t SB, CB, R_cons, R_cum, R_bcap, n_rows, n_vars;
  int has_bcap;
  double blimit;
  const uint8_t* is_sw;
  const int* gpu_of;     // [Nn] GPU rank or -1
  const int* gpre;       // [Nn] GPUs strictly before node n
  const int* node_of_gpu;// [G]
  const int* esrc;
  const int* edst;
  const int* edelta;
  const double* ecap;    // [E*K]
  const int* snode;      // [S]
  const int* pair_src;   // [P]
  const int* pair_dst;   // [P]
  const double* pair_u;  // [P]
  const int* pair_of;    // [S*Nn] pair id or -1
  const double* out_units;  // [S]
  const int* inc_ptr;    // [Nn+1]
  const uint32_t* inc;   // edge id | bit31 when the edge leaves the node
  const int* out_ptr;    // [Nn+1] out-edges of node (edge order)
  const int* out_e;
  // bound-class codes (pdlp.cu dictionaries)
  int dict_col, dict_row, nU, nOU, nCap;
  int phase1;
  const int* pair_uidx;  // [P] index of the pair's units in the distinct-units list
  const int* src_ouidx;  // [S] index of the source's out-units in its list
  const uint16_t* cap_idx;  // [E*K] index of the capacity in the distinct-caps list
};

__device__ __forceinline__ int64_t varF(const TeDev& d, int s, int e, int k) {
  return (int64_t)s * d.SB + (int64_t)e * d.K + k;
}
__device__ __forceinline__ int64_t varB(const TeDev& d, int s, int g, int k) {
  return (int64_t)s * d.SB + (int64_t)d.E * d.K + (int64_t)g * (d.K + 1) + k;
}
__device__ __forceinline__ int64_t varRd(const TeDev& d, int p, int k) {
  return (int64_t)d.S * d.SB + (int64_t)p * 2 * d.K + 2 * k;
}
__device__ __forceinline__ int64_t cons_off(const TeDev& d, int s, int n) {
  return (int64_t)n * d.K + d.gpre[n] - (d.snode[s] < n ? 1 : 0);
}
__device__ __forceinline__ int64_t rowCons(const TeDev& d, int s, int n, int k) {
  return d.R_cons + (int64_t)s * d.CB + cons_off(d, s, n) + k;
}


// ---------------------------------------------------------------------------
// Division by a run-time invariant d for dividends < 2^31 (multiply-high and
// shift; d = 1 is the identity).
struct FastDiv {
  uint32_t mul = 0, shr = 0;
  void init(uint32_t d) {
    if (d <= 1) { mul = 0; shr = 0; return; }
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;                   // ceil(log2 d)
    const uint32_t p = 31 + l;
    mul = (uint32_t)(((1ull << p) + d - 1) / d);
    shr = p - 32;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return mul ? (__umulhi(n, mul) >> shr) : n;
  }
};

#ifndef TECCL_SEFAM
#define TECCL_SEFAM 1  // per-column flow decode (te_col): one packed (s, e) family load instead of edge4 -> sntab (-2.5 % col_te2 on 16 chassis)
#endif

// Matrix-free view of a single-device TE LP (reference numbering; every
// index < 2^31, checked by teccl_lp_build_te). The packed tables shorten the
// chain of dependent table loads in front of each gather:
//   edge4[e]        = {src, dst, delta, 0}
//   sntab[s*Nn + n] = {first cons row of (s, n) | bit31 when (s, n) has a
//                      "last" row, Rd(p, 0) column of pair (s, n) or -1}
//   incp[j]         = incident entry j of node n (inc_ptr order):
//                     {e*K - d, d}, d = delay for an arriving edge (term
//                     +F(s,e,k-d)), d = -1 for a leaving edge (term -F(s,e,k+1))
struct TeOp {
  TeDev d;
  FastDiv fK, fK1, f2K, fSB, fCB;
  uint32_t K, S, Nn, SB, CB, EK, nF, R_cons, R_cum, R_bcap, m, n;
  int has_bcap, phase1;
  const int4* edge4;
  const int2* sntab;
  const int2* incp;
  // per flow family (s, e): {cons(s,src(e),0) row, cons(s,dst(e),0) row |
  // bit31 last row, delay, src(e) == source node of s} -- one load where the
  // flow columns otherwise chain edge4 -> sntab before their gathers
  const int4* sefam;
  uint32_t E;
  // segment tasks (see seg_cols / seg_rows): one warp per task
  const int4* ctask;
  const int4* rtask;
  int n_ctask, n_rtask;
  const double* neg_inv;   // [K] -1/(k+1), the Rc costs (lp.py:133-135)
  int dmax;                // largest edge delay (epochs)
};

// Matrix-free view of one rank's block of a row-partitioned LP in the
// epoch-major numbering (te_build.cu EmShape): columns k*CW + [F(s,e) s*E+e |
// B(s,g) SE + s*G+g | Rd/Rc(p) SEG + 2p + rc], then the final buffers
// B(s,g,K) at K*CW + s*G + g; rows S init rows, then k-blocks of RW =
// [cap(e) | cons(s,n) E + s*Nn + n | cum(p) | bcap(g)], then last(s,n) and
// bcap(g,K). The rank owns epochs [k0, k1) (+ init rows on rank 0, + the
// tails on the last rank); gathers index the window arrays (global - w0).
struct EmOp {
  TeDev d;
  FastDiv fCW, fRW, fE, fG, fNn, fGm1;
  uint32_t K, S, E, G, Nn, P, CW, RW, SE, SEG, k0, nk, tail_k;  // owned epochs [k0, k0+nk); tail_k = K - k0
  int64_t c0, r0, wc0, wr0;       // owned / window starts (global ids)
  uint32_t n, m;                  // owned columns / rows
  int has_bcap, phase1;
  const int4* edge4;              // {src, dst, delta, 0}
  const int2* incE;               // incident entries of node n (inc_ptr order): {e, delta} arriving, {e, -1} leaving
  const double* neg_inv;          // [K] -1/(k+1)
};

// Owner of the device tables behind a TeOp / EmOp (lp->te).
struct TeHold {
  TeOp op;
  EmOp em;
  int kind = 0;  // 0: TeOp (single device, reference numbering), 1: EmOp (partition block)
  std::vector<void*> owned;
  cudaStream_t st = nullptr;
};

__device__ __forceinline__ int64_t em_row_cons(const EmOp& o, uint32_t s, uint32_t n, int64_t k) {
  return (int64_t)o.S + k * o.RW + o.E + (int64_t)s * o.Nn + n;
}
__device__ __forceinline__ int64_t em_row_last(const EmOp& o, uint32_t s, int n) {
  const int g = __ldg(o.d.gpu_of + n), gs = __ldg(o.d.gpu_of + __ldg(o.d.snode + s));
  return (int64_t)o.S + (int64_t)o.K * o.RW + (int64_t)s * (o.G - 1) + (g < gs ? g : g - 1);
}
__device__ __forceinline__ int64_t em_col_F(const EmOp& o, uint32_t s, uint32_t e, int64_t k) {
  return k * o.CW + (int64_t)s * o.E + e;
}
__device__ __forceinline__ int64_t em_col_B(const EmOp& o, uint32_t s, uint32_t g, int64_t k) {
  return k < (int64_t)o.K ? k * o.CW + o.SE + (int64_t)s * o.G + g
                          : (int64_t)o.K * o.CW + (int64_t)s * o.G + g;
}
__device__ __forceinline__ int64_t em_col_Rd(const EmOp& o, uint32_t p, int64_t k) {
  return k * o.CW + o.SEG + 2LL * p;
}

// (A^T y)_c for owned column jl of the block, with bounds and cost: the same
// entries as te_col / gen_col, indexed in the epoch-major window.
__device__ __forceinline__ double em_col(const EmOp& o, uint32_t jl, const double* __restrict__ yw,
                                         double& lb, double& ub, double& c) {
  const uint32_t K = o.K;
  lb = 0.0; ub = INFINITY; c = 0.0;
  const double* y = yw - o.wr0;  // y[global row]
  const uint32_t kr = o.fCW.div(jl);
  const int64_t k = (int64_t)o.k0 + kr;
  if (kr >= o.tail_k) {                            // B(s,g,K)
    const uint32_t q = jl - o.tail_k * o.CW;
    const uint32_t s = o.fG.div(q), g = q - s * o.G;
    const int nd = __ldg(o.d.node_of_gpu + g);
    double a = -__ldg(y + em_row_cons(o, s, nd, K - 1));
    if (o.has_bcap) a += __ldg(y + (int64_t)o.S + (int64_t)K * o.RW + (int64_t)o.S * (o.G - 1) + g);
    return a;
  }
  const uint32_t q = jl - kr * o.CW;
  const int64_t rk = (int64_t)o.S + k * o.RW;     // first row of epoch k
  if (q < o.SE) {                                  // F(s,e,k)
    const uint32_t s = o.fE.div(q), e = q - s * o.E;
    const int4 ed = __ldg(o.edge4 + e);
    const int sn = __ldg(o.d.snode + s);
    const int64_t t = k + ed.z;
    const double v_cap = __ldg(y + rk + e);
    const double v_ini = (k == 0 && ed.x == sn) ? __ldg(y + s) : 0.0;
    const double v_out = (k >= 1) ? __ldg(y + rk - o.RW + o.E + (int64_t)s * o.Nn + ed.x) : 0.0;
    const double v_in = (t <= K - 1) ? __ldg(y + em_row_cons(o, s, ed.y, t)) : 0.0;
    const bool wl = __ldg(o.d.gpu_of + ed.y) >= 0 && ed.y != sn;
    const double v_last = (t == K - 1 && wl) ? __ldg(y + em_row_last(o, s, ed.y)) : 0.0;
    if (k == 0 && ed.x != sn) ub = 0.0;            // lp.py:51-52
    return v_cap + v_ini - v_out + v_in + v_last;
  }
  if (q < o.SEG) {                                 // B(s,g,k), k < K
    const uint32_t q2 = q - o.SE;
    const uint32_t s = o.fG.div(q2), g = q2 - s * o.G;
    const int nd = __ldg(o.d.node_of_gpu + g), sn = __ldg(o.d.snode + s);
    const int64_t rc = rk + o.E + (int64_t)s * o.Nn + nd;  // cons(s,nd,k)
    const double v_ini = (k == 0 && nd == sn) ? __ldg(y + s) : 0.0;
    const double v_prev = (k >= 1) ? __ldg(y + rc - o.RW) : 0.0;
    const double v_cur = __ldg(y + rc);
    const double v_bc = o.has_bcap ? __ldg(y + rk + o.E + (int64_t)o.S * o.Nn + o.P + g) : 0.0;
    if (k == 0 && nd != sn) ub = 0.0;              // lp.py:57-59
    return v_ini - v_prev + v_cur + v_bc;
  }
  const uint32_t q3 = q - o.SEG, p = q3 >> 1;      // Rd / Rc(p,k)
  const int64_t cum = rk + o.E + (int64_t)o.S * o.Nn + p;
  const double u = __ldg(o.d.pair_u + p);
  ub = u;
  if (!(q3 & 1)) {                                 // Rd
    const int s = __ldg(o.d.pair_src + p), w = __ldg(o.d.pair_dst + p);
    const double v_last = (k == K - 1) ? __ldg(y + em_row_last(o, s, w)) : 0.0;
    return -__ldg(y + em_row_cons(o, s, w, k)) - __ldg(y + cum) - v_last;
  }
  const double v_next = (k + 1 <= K - 1) ? __ldg(y + cum + o.RW) : 0.0;   // Rc
  if (o.phase1) {
    c = (k == K - 1) ? -1.0 : 0.0;
  } else {
    if (k == K - 1) lb = u;                        // lp.py:64-65
    c = __ldg(o.neg_inv + k);                      // -1/(k+1), lp.py:133-135
  }
  return __ldg(y + cum) - v_next;
}

// (A x)_r for owned row il of the block, with bounds (te_row / gen_row).
__device__ __forceinline__ double em_row(const EmOp& o, uint32_t il, const double* __restrict__ xw,
                                         double& lo, double& hi) {
  const uint32_t K = o.K;
  lo = 0.0; hi = 0.0;
  const double* x = xw - o.wc0;  // x[global column]
  const int64_t rg = o.r0 + il;
  double a = 0.0;
  if (rg < (int64_t)o.S) {                         // init(s)
    const uint32_t s = (uint32_t)rg;
    const int nd = __ldg(o.d.snode + s);
    for (int j = __ldg(o.d.out_ptr + nd); j < __ldg(o.d.out_ptr + nd + 1); ++j)
      a += __ldg(x + em_col_F(o, s, (uint32_t)__ldg(o.d.out_e + j), 0));
    a += __ldg(x + em_col_B(o, s, (uint32_t)__ldg(o.d.gpu_of + nd), 0));
    lo = hi = __ldg(o.d.out_units + s);
    return a;
  }
  const uint32_t q = (uint32_t)(rg - o.S);
  const uint32_t k = o.fRW.div(q);
  if (k >= K) {                                    // tails
    const uint32_t q2 = q - K * o.RW;
    if (q2 < o.S * (o.G - 1)) {                    // last(s,n)
      const uint32_t s = o.fGm1.div(q2), i = q2 - s * (o.G - 1);
      const int gs = __ldg(o.d.gpu_of + __ldg(o.d.snode + s));
      const int n = __ldg(o.d.node_of_gpu + ((int)i < gs ? i : i + 1));
      for (int j = __ldg(o.d.inc_ptr + n); j < __ldg(o.d.inc_ptr + n + 1); ++j) {
        const int2 t = __ldg(o.incE + j);
        const int kk = (int)K - 1 - t.y;
        if (t.y >= 0 && kk >= 0) a += __ldg(x + em_col_F(o, s, t.x, kk));
      }
      const int pr = __ldg(o.d.pair_of + s * o.Nn + n);
      if (pr >= 0) a -= __ldg(x + em_col_Rd(o, pr, K - 1));
      return a;
    }
    const uint32_t g = q2 - o.S * (o.G - 1);       // bcap(g,K)
    for (uint32_t s = 0; s < o.S; ++s) a += __ldg(x + em_col_B(o, s, g, K));
    lo = -INFINITY;
    hi = o.d.blimit;
    return a;
  }
  const uint32_t r = q - k * o.RW;
  const int64_t ck = (int64_t)k * o.CW;            // first column of epoch k
  if (r < o.E) {                                   // cap(e,k): sum_s F(s,e,k)
    for (uint32_t s0 = 0; s0 < o.S; s0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (s0 + u < o.S) ? __ldg(x + ck + (int64_t)(s0 + u) * o.E + r) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    lo = -INFINITY;
    hi = __ldg(o.d.ecap + (int64_t)r * K + k);
    return a;
  }
  if (r < o.E + o.S * o.Nn) {                      // cons(s,n,k)
    const uint32_t r2 = r - o.E;
    const uint32_t s = o.fNn.div(r2), n = r2 - s * o.Nn;
    const int64_t fs = ck + (int64_t)s * o.E;      // F(s,0,k)
    const int j0 = __ldg(o.d.inc_ptr + n), j1 = __ldg(o.d.inc_ptr + n + 1);
    for (int jb = j0; jb < j1; jb += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = 0.0;
        if (jb + u < j1) {
          const int2 t = __ldg(o.incE + jb + u);
          const int kk = (int)k - t.y;             // arriving: k - delta; leaving: k + 1
          if (kk >= 0 && kk <= (int)K - 1) {
            const double xv = __ldg(x + fs + (int64_t)(kk - (int)k) * o.CW + t.x);
            v[u] = t.y < 0 ? -xv : xv;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    const int g = __ldg(o.d.gpu_of + n);
    if (g >= 0) {
      a += __ldg(x + em_col_B(o, s, g, k)) - __ldg(x + em_col_B(o, s, g, k + 1));
      const int pr = __ldg(o.d.pair_of + s * o.Nn + n);
      if (pr >= 0) a -= __ldg(x + em_col_Rd(o, pr, k));
    }
    return a;
  }
  if (r < o.E + o.S * o.Nn + o.P) {                // cum(p,k)
    const uint32_t p = r - o.E - o.S * o.Nn;
    const int64_t rd = em_col_Rd(o, p, k);
    const double v_prev = (k >= 1) ? __ldg(x + rd - o.CW + 1) : 0.0;
    return __ldg(x + rd + 1) - __ldg(x + rd) - v_prev;
  }
  const uint32_t g = r - o.E - o.S * o.Nn - o.P;  // bcap(g,k)
  for (uint32_t s = 0; s < o.S; ++s) a += __ldg(x + em_col_B(o, s, g, k));
  lo = -INFINITY;
  hi = o.d.blimit;
  return a;
}

inline void te_op_init(TeOp& o, const TeDev& d) {
  o.d = d;
  o.K = (uint32_t)d.K; o.S = (uint32_t)d.S; o.Nn = (uint32_t)d.Nn;
  o.SB = (uint32_t)d.SB; o.CB = (uint32_t)d.CB;
  o.EK = (uint32_t)((int64_t)d.E * d.K);
  o.nF = (uint32_t)((int64_t)d.S * d.SB);
  o.R_cons = (uint32_t)d.R_cons; o.R_cum = (uint32_t)d.R_cum; o.R_bcap = (uint32_t)d.R_bcap;
  o.m = (uint32_t)d.n_rows; o.n = (uint32_t)d.n_vars;
  o.has_bcap = d.has_bcap; o.phase1 = d.phase1;
  o.fK.init(o.K); o.fK1.init(o.K + 1); o.f2K.init(2 * o.K);
  o.fSB.init(o.SB > 0 ? o.SB : 1); o.fCB.init(o.CB > 0 ? o.CB : 1);
  o.edge4 = nullptr; o.sntab = nullptr; o.incp = nullptr; o.sefam = nullptr; o.E = (uint32_t)d.E;
  o.ctask = nullptr; o.rtask = nullptr; o.n_ctask = 0; o.n_rtask = 0; o.neg_inv = nullptr;
  o.dmax = 0;
}

// (A^T y)_v for column v, with its bounds and cost (gen_col in te_build.cu
// emits the same entries).
__device__ __forceinline__ double te_col(const TeOp& o, uint32_t v, const double* __restrict__ y,
                                         double& lb, double& ub, double& c) {
  const uint32_t K = o.K;
  lb = 0.0; ub = INFINITY; c = 0.0;
  double a;
  if (v < o.nF) {
    const uint32_t s = o.fSB.div(v);
    uint32_t q = v - s * o.SB;
    const int sn = __ldg(o.d.snode + s);
    const int2* sr = o.sntab + s * o.Nn;
    if (q < o.EK) {                                // F(s,e,k)
      const uint32_t e = o.fK.div(q), k = q - e * K;
#if TECCL_SEFAM
      const int4 ed = __ldg(o.sefam + s * o.E + e);
      const uint32_t cu = (uint32_t)ed.x, cw = (uint32_t)ed.y;
      const bool from_src = ed.w != 0;
      (void)sr; (void)sn;
#else
      const int4 ed = __ldg(o.edge4 + e);
      const uint32_t cu = (uint32_t)__ldg(&sr[ed.x].x) & kIdxMask;
      const uint32_t cw = (uint32_t)__ldg(&sr[ed.y].x);
      const bool from_src = ed.x == sn;
#endif
      const uint32_t t = k + (uint32_t)ed.z;
      const double v_cap = __ldg(y + o.S + q);                                  // cap(e,k)
      const double v_ini = (k == 0 && from_src) ? __ldg(y + s) : 0.0;           // init(s)
      const double v_out = (k >= 1) ? __ldg(y + cu + k - 1) : 0.0;              // cons(s,u,k-1)
      const double v_in = (t <= K - 1) ? __ldg(y + (cw & kIdxMask) + t) : 0.0;  // cons(s,w,t)
      const double v_last = (t == K - 1 && (cw & kSignBit)) ? __ldg(y + (cw & kIdxMask) + K) : 0.0;
      if (k == 0 && !from_src) ub = 0.0;           // lp.py:51-52
      a = v_cap + v_ini - v_out + v_in + v_last;
    } else {                                       // B(s,g,k)
      q -= o.EK;
      const uint32_t g = o.fK1.div(q), k = q - g * (K + 1);
      const int nd = __ldg(o.d.node_of_gpu + g);
      const uint32_t rb = (uint32_t)__ldg(&sr[nd].x) & kIdxMask;
      const double v_ini = (k == 0 && nd == sn) ? __ldg(y + s) : 0.0;
      const double v_prev = (k >= 1) ? __ldg(y + rb + k - 1) : 0.0;
      const double v_cur = (k <= K - 1) ? __ldg(y + rb + k) : 0.0;
      const double v_bc = o.has_bcap ? __ldg(y + o.R_bcap + q) : 0.0;
      if (k == 0 && nd != sn) ub = 0.0;            // lp.py:57-59
      a = v_ini - v_prev + v_cur + v_bc;
    }
  } else {                                         // Rd(p,k) / Rc(p,k)
    const uint32_t q = v - o.nF;
    const uint32_t p = o.f2K.div(q), r = q - p * 2 * K, k = r >> 1;
    const uint32_t cum = o.R_cum + p * K + k;
    const double u = __ldg(o.d.pair_u + p);
    ub = u;
    if (!(r & 1)) {                                // Rd
      const int s = __ldg(o.d.pair_src + p), w = __ldg(o.d.pair_dst + p);
      const uint32_t rw = ((uint32_t)__ldg(&o.sntab[s * o.Nn + w].x) & kIdxMask) + k;
      const double v_last = (k == K - 1) ? __ldg(y + rw + 1) : 0.0;
      a = -__ldg(y + rw) - __ldg(y + cum) - v_last;
    } else {                                       // Rc
      const double v_next = (k + 1 <= K - 1) ? __ldg(y + cum + 1) : 0.0;
      a = __ldg(y + cum) - v_next;
      if (o.phase1) {
        c = (k == K - 1) ? -1.0 : 0.0;
      } else {
        if (k == K - 1) lb = u;                    // lp.py:64-65
        c = -1.0 / (double)(k + 1);                // lp.py:133-135
      }
    }
  }
  return a;
}

// (A^T y) for the adjacent columns v, v+1 (v even, v+1 < n): when both are
// epochs k, k+1 of one flow or buffer family -- all but one pair per family
// -- the family's table lookups and index math are done once and the
// gathers of the two epochs are adjacent; otherwise te_col twice.
__device__ __forceinline__ void te_col2(const TeOp& o, uint32_t v, const double* __restrict__ y,
                                        double (&a)[2], double (&lb)[2], double (&ub)[2],
                                        double (&c)[2]) {
  const uint32_t K = o.K;
  if (v + 1 < o.nF) {
    const uint32_t s = o.fSB.div(v);
    const uint32_t q = v - s * o.SB;
    if (q + 1 < o.EK) {
      const uint32_t e = o.fK.div(q), k = q - e * K;
      if (k + 1 < K) {                             // F(s,e,k), F(s,e,k+1)
        const int sn = __ldg(o.d.snode + s);
        const int2* sr = o.sntab + s * o.Nn;
        const int4 ed = __ldg(o.edge4 + e);
        const uint32_t cu = (uint32_t)__ldg(&sr[ed.x].x) & kIdxMask;
        const uint32_t cw = (uint32_t)__ldg(&sr[ed.y].x);
        const uint32_t t = k + (uint32_t)ed.z;
        const double* yc = y + o.S + q;
        const double* yo = y + cu + k;             // cons(s,u,k-1+h) = yo[h-1]
        const double* yi = y + (cw & kIdxMask) + t;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t kh = k + h, th = t + h;
          const double v_cap = __ldg(yc + h);
          const double v_ini = (kh == 0 && ed.x == sn) ? __ldg(y + s) : 0.0;
          const double v_out = (kh >= 1) ? __ldg(yo + h - 1) : 0.0;
          const double v_in = (th <= K - 1) ? __ldg(yi + h) : 0.0;
          const double v_last = (th == K - 1 && (cw & kSignBit)) ? __ldg(y + (cw & kIdxMask) + K) : 0.0;
          a[h] = v_cap + v_ini - v_out + v_in + v_last;
          lb[h] = 0.0;
          ub[h] = (kh == 0 && ed.x != sn) ? 0.0 : INFINITY;  // lp.py:51-52
          c[h] = 0.0;
        }
        return;
      }
    } else if (q >= o.EK && q + 1 < o.SB) {
      const uint32_t qb = q - o.EK;
      const uint32_t g = o.fK1.div(qb), k = qb - g * (K + 1);
      if (k + 1 <= K) {                            // B(s,g,k), B(s,g,k+1)
        const int sn = __ldg(o.d.snode + s);
        const int nd = __ldg(o.d.node_of_gpu + g);
        const uint32_t rb = (uint32_t)__ldg(&o.sntab[s * o.Nn + nd].x) & kIdxMask;
        const double* yr = y + rb + k;             // cons(s,nd,k+h) = yr[h]
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t kh = k + h;
          const double v_ini = (kh == 0 && nd == sn) ? __ldg(y + s) : 0.0;
          const double v_prev = (kh >= 1) ? __ldg(yr + h - 1) : 0.0;
          const double v_cur = (kh <= K - 1) ? __ldg(yr + h) : 0.0;
          const double v_bc = o.has_bcap ? __ldg(y + o.R_bcap + qb + h) : 0.0;
          a[h] = v_ini - v_prev + v_cur + v_bc;
          lb[h] = 0.0;
          ub[h] = (kh == 0 && nd != sn) ? 0.0 : INFINITY;  // lp.py:57-59
          c[h] = 0.0;
        }
        return;
      }
    }
  }
  a[0] = te_col(o, v, y, lb[0], ub[0], c[0]);
  a[1] = te_col(o, v + 1, y, lb[1], ub[1], c[1]);
}

// sum over s < S of x[s*SB + off], loads issued 8 at a time
__device__ __forceinline__ double te_sum_sources(const TeOp& o, const double* __restrict__ x, uint32_t off) {
  double a = 0.0;
  for (uint32_t s0 = 0; s0 < o.S; s0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (s0 + u < o.S) ? __ldg(x + (s0 + u) * o.SB + off) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) a += v[u];
  }
  return a;
}

// (A x)_i for row i, with its bounds (gen_row in te_build.cu emits the same
// entries).
__device__ __forceinline__ double te_row(const TeOp& o, uint32_t i, const double* __restrict__ x,
                                         double& lo, double& hi) {
  const uint32_t K = o.K;
  lo = 0.0; hi = 0.0;
  double a = 0.0;
  if (i < o.S) {                                   // init(s)
    const int nd = __ldg(o.d.snode + i);
    const double* xs = x + i * o.SB;
    for (int j = __ldg(o.d.out_ptr + nd); j < __ldg(o.d.out_ptr + nd + 1); ++j)
      a += __ldg(xs + (uint32_t)__ldg(o.d.out_e + j) * K);
    a += __ldg(xs + o.EK + (uint32_t)__ldg(o.d.gpu_of + nd) * (K + 1));
    lo = hi = __ldg(o.d.out_units + i);
  } else if (i < o.R_cons) {                       // cap(e,k)
    const uint32_t q = i - o.S;
    a = te_sum_sources(o, x, q);
    lo = -INFINITY;
    hi = __ldg(o.d.ecap + q);
  } else if (i < o.R_cum) {                        // cons(s,n,k) / last(s,n)
    const uint32_t q = i - o.R_cons;
    const uint32_t s = o.fCB.div(q);
    const int2* sr = o.sntab + s * o.Nn;
    const uint32_t base = o.R_cons + s * o.CB;
    const uint32_t off = q - s * o.CB;
    int nd = (int)o.fK1.div(off);                  // <= the node: offsets grow by K or K+1
    int2 tn = __ldg(sr + nd);
    while (nd + 1 < (int)o.Nn) {
      const int2 tq = __ldg(sr + nd + 1);
      if ((((uint32_t)tq.x & kIdxMask) - base) > off) break;
      ++nd;
      tn = tq;
    }
    const uint32_t k = off - (((uint32_t)tn.x & kIdxMask) - base);
    const bool last = (k == K);
    const int ke = last ? (int)K - 1 : (int)k;
    const double* xs = x + s * o.SB;
    const int j0 = __ldg(o.d.inc_ptr + nd), j1 = __ldg(o.d.inc_ptr + nd + 1);
    for (int jb = j0; jb < j1; jb += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = 0.0;
        if (jb + u < j1) {
          const int2 t = __ldg(o.incp + jb + u);
          const int kk = ke - t.y;
          if (kk >= 0 && kk <= (int)K - 1 && !(last && t.y < 0)) {
            const double xv = __ldg(xs + t.x + ke);
            v[u] = t.y < 0 ? -xv : xv;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    const int g = __ldg(o.d.gpu_of + nd);
    if (!last) {
      if (g >= 0) {
        const double* b = xs + o.EK + (uint32_t)g * (K + 1) + k;
        a += __ldg(b) - __ldg(b + 1);
        if (tn.y >= 0) a -= __ldg(x + (uint32_t)tn.y + 2 * k);
      }
    } else if (tn.y >= 0) {
      a -= __ldg(x + (uint32_t)tn.y + 2 * (K - 1));
    }
  } else if (i < o.R_bcap) {                       // cum(p,k)
    const uint32_t q = i - o.R_cum;
    const uint32_t p = o.fK.div(q), k = q - p * K;
    const uint32_t rd = o.nF + p * 2 * K + 2 * k;
    const double v_prev = (k >= 1) ? __ldg(x + rd - 1) : 0.0;
    a = __ldg(x + rd + 1) - __ldg(x + rd) - v_prev;
  } else {                                         // bcap(g,k)
    const uint32_t q = i - o.R_bcap;
    a = te_sum_sources(o, x, o.EK + q);
    lo = -INFINITY;
    hi = o.d.blimit;
  }
  return a;
}


// ---------------------------------------------------------------------------
// Segment walkers. Every column family is a run of consecutive epochs of one
// (source, edge) / (source, GPU) / pair, and every row family a run of one
// edge / (source, node) / pair / GPU, laid out contiguously. A task is up to
// 64 consecutive entries of one segment, handled by one warp (entry
// off + lane and off + 32 + lane): the segment's table lookups are done once
// per task, each entry costs only its gathers, which are coalesced along the
// epoch axis. Task encoding (int4):
//   x = kind | a << 4,  y = b,  z = first global index of the task,
//   w = off | count << 24   (off = epoch offset inside the segment)
enum SegKind { SEG_F = 0, SEG_B = 1, SEG_P = 2,                          // columns
               SEG_INIT = 3, SEG_CAP = 4, SEG_CONS = 5, SEG_CUM = 6, SEG_BCAP = 7 };  // rows
#ifndef TECCL_SEG_PER_LANE
#define TECCL_SEG_PER_LANE 2  // entries per lane of a segment task (task = 32 x this)
#endif
constexpr int kSegPerLane = TECCL_SEG_PER_LANE;
constexpr int kSegTask = 32 * kSegPerLane;

__device__ __forceinline__ int seg_count(const int4& t) { return (int)((uint32_t)t.w >> 24); }

// (A^T y) for the task's entries lane + 32h, with bounds and costs.
__device__ __forceinline__ void seg_cols(const TeOp& o, const int4& t, int lane,
                                         const double* __restrict__ y, double (&a)[kSegPerLane],
                                         double (&lb)[kSegPerLane], double (&ub)[kSegPerLane],
                                         double (&c)[kSegPerLane]) {
  const uint32_t K = o.K;
  const int kind = t.x & 15, A = t.x >> 4, Bv = t.y;
  const int off = t.w & 0xffffff, cnt = seg_count(t);
#pragma unroll
  for (int h = 0; h < kSegPerLane; ++h) { a[h] = 0.0; lb[h] = 0.0; ub[h] = INFINITY; c[h] = 0.0; }
  if (kind == SEG_F) {                             // F(s,e,k), k = off + i
    const int s = A, sn = __ldg(o.d.snode + s);
    const int4 ed = __ldg(o.edge4 + Bv);
    const int2* sr = o.sntab + s * o.Nn;
    const uint32_t cu = (uint32_t)__ldg(&sr[ed.x].x) & kIdxMask;
    const uint32_t cwr = (uint32_t)__ldg(&sr[ed.y].x);
    const uint32_t cw = cwr & kIdxMask;
    const bool wl = (cwr & kSignBit) != 0, from_src = (ed.x == sn);
    const double* yc = y + o.S + (uint32_t)Bv * K;
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
        const uint32_t k = off + i, tt = k + (uint32_t)ed.z;
        const double v_cap = __ldg(yc + k);
        const double v_ini = (k == 0 && from_src) ? __ldg(y + s) : 0.0;
        const double v_out = (k >= 1) ? __ldg(y + cu + k - 1) : 0.0;
        const double v_in = (tt <= K - 1) ? __ldg(y + cw + tt) : 0.0;
        const double v_last = (tt == K - 1 && wl) ? __ldg(y + cw + K) : 0.0;
        a[h] = v_cap + v_ini - v_out + v_in + v_last;
        if (k == 0 && !from_src) ub[h] = 0.0;      // lp.py:51-52
      }
    }
  } else if (kind == SEG_B) {                      // B(s,g,k), k = off + i
    const int s = A, g = Bv, sn = __ldg(o.d.snode + s);
    const int nd = __ldg(o.d.node_of_gpu + g);
    const uint32_t rb = (uint32_t)__ldg(&o.sntab[s * o.Nn + nd].x) & kIdxMask;
    const bool at_src = (nd == sn);
    const uint32_t bc = o.R_bcap + (uint32_t)g * (K + 1);
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
        const uint32_t k = off + i;
        const double v_ini = (k == 0 && at_src) ? __ldg(y + s) : 0.0;
        const double v_prev = (k >= 1) ? __ldg(y + rb + k - 1) : 0.0;
        const double v_cur = (k <= K - 1) ? __ldg(y + rb + k) : 0.0;
        const double v_bc = o.has_bcap ? __ldg(y + bc + k) : 0.0;
        a[h] = v_ini - v_prev + v_cur + v_bc;
        if (k == 0 && !at_src) ub[h] = 0.0;        // lp.py:57-59
      }
    }
  } else if (kind == SEG_P) {                      // Rd/Rc(p,k), entry c = off + i = 2k + rc
    const int p = A;
    const int s = __ldg(o.d.pair_src + p), w = __ldg(o.d.pair_dst + p);
    const uint32_t rw = (uint32_t)__ldg(&o.sntab[s * o.Nn + w].x) & kIdxMask;
    const uint32_t cum = o.R_cum + (uint32_t)p * K;
    const double u = __ldg(o.d.pair_u + p);
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
        const uint32_t cc = off + i, k = cc >> 1;
        const bool rc = (cc & 1) != 0;
        // Rd: -cons(s,w,k) - cum(p,k) [- last(s,w) at k = K-1];  Rc: cum(p,k) [- cum(p,k+1)]
        const uint32_t i0 = rc ? cum + k : rw + k;
        const double v0 = __ldg(y + i0);
        const double v1 = rc ? ((k + 1 <= K - 1) ? __ldg(y + cum + k + 1) : 0.0) : __ldg(y + cum + k);
        const double v2 = (!rc && k == K - 1) ? __ldg(y + rw + K) : 0.0;
        a[h] = rc ? v0 - v1 : -v0 - v1 - v2;
        ub[h] = u;
        if (rc) {
          if (o.phase1) {
            c[h] = (k == K - 1) ? -1.0 : 0.0;
          } else {
            if (k == K - 1) lb[h] = u;             // lp.py:64-65
            c[h] = __ldg(o.neg_inv + k);           // -1/(k+1), lp.py:133-135
          }
        }
      }
    }
  }
}

#ifndef TECCL_CAP_JOINT
#define TECCL_CAP_JOINT 1  // capacity rows: sum both entries of a lane together, TECCL_CAP_U sources per round (-6 % on 16 chassis)
#endif
#ifndef TECCL_CAP_U
#define TECCL_CAP_U 4
#endif
#ifndef TECCL_CUM_SHFL
#define TECCL_CUM_SHFL 1   // cumulative-read rows: previous Rc by warp shuffle
#endif
#ifndef TECCL_CONS_U
#define TECCL_CONS_U 4     // interior conservation tasks: incident edges per round of gathers
#endif

// sum_s x[s*SB + q0 + lane + 32h] for the lane's entries (h < kSegPerLane)
// together, so a round keeps kSegPerLane * TECCL_CAP_U gathers in flight;
// each entry adds its sources in the same order as te_sum_sources (s
// ascending, one running sum), so the sums are identical
__device__ __forceinline__ void seg_sum_sources(const TeOp& o, const double* __restrict__ x, uint32_t q0,
                                                int lane, int cnt, double (&a)[kSegPerLane]) {
  uint32_t qh[kSegPerLane];
#pragma unroll
  for (int h = 0; h < kSegPerLane; ++h) {
    a[h] = 0.0;
    qh[h] = q0 + (uint32_t)min(lane + 32 * h, cnt - 1);  // lanes past the end re-read the last entry
  }
  for (uint32_t s0 = 0; s0 < o.S; s0 += TECCL_CAP_U) {
    double v[kSegPerLane][TECCL_CAP_U];
#pragma unroll
    for (int u = 0; u < TECCL_CAP_U; ++u)
#pragma unroll
      for (int h = 0; h < kSegPerLane; ++h)
        v[h][u] = (s0 + u < o.S) ? __ldg(x + (s0 + u) * o.SB + qh[h]) : 0.0;
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h)
#pragma unroll
      for (int u = 0; u < TECCL_CAP_U; ++u) a[h] += v[h][u];
  }
}

// (A x) for the task's entries lane + 32h, with row bounds.
__device__ __forceinline__ void seg_rows(const TeOp& o, const int4& t, int lane,
                                         const double* __restrict__ x, double (&a)[kSegPerLane],
                                         double (&lo)[kSegPerLane], double (&hi)[kSegPerLane]) {
  const uint32_t K = o.K;
  const int kind = t.x & 15, A = t.x >> 4, Bv = t.y;
  const int off = t.w & 0xffffff, cnt = seg_count(t);
#pragma unroll
  for (int h = 0; h < kSegPerLane; ++h) { a[h] = 0.0; lo[h] = 0.0; hi[h] = 0.0; }
  if (kind == SEG_CAP) {                           // cap(e,k): sum_s F(s,e,k)
    const uint32_t q0 = (uint32_t)Bv * K + off;
#if TECCL_CAP_JOINT
    seg_sum_sources(o, x, q0, lane, cnt, a);
#endif
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
#if !TECCL_CAP_JOINT
        a[h] = te_sum_sources(o, x, q0 + i);
#endif
        lo[h] = -INFINITY;
        hi[h] = __ldg(o.d.ecap + q0 + i);
      }
    }
  } else if (kind == SEG_CONS) {                   // cons(s,n,k) / last(s,n), k = off + i
    const int s = A, nd = Bv;
    const int2 tn = __ldg(o.sntab + s * o.Nn + nd);
    const int g = __ldg(o.d.gpu_of + nd);
    const int j0 = __ldg(o.d.inc_ptr + nd), j1 = __ldg(o.d.inc_ptr + nd + 1);
    const double* xs = x + s * o.SB;
    int kk[kSegPerLane];
    bool last[kSegPerLane], on[kSegPerLane];
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      on[h] = i < cnt;
      const int k = off + i;
      last[h] = (k == (int)K);
      kk[h] = last[h] ? (int)K - 1 : k;
    }
    // interior task (every epoch's terms exist: k - delay >= 0, k + 1 <= K-1,
    // no last row, all lanes busy): unpredicated gathers at fixed offsets
    // from one base, the sign as a +-1 weight (same sums in the same order)
    const bool interior = cnt == kSegTask && off >= o.dmax && off + kSegTask <= (int)K - 1;
    if (interior) {
      const double* xb = xs + off + lane;          // term (e*K + c) of epoch off + lane: xb[e*K + c]
      for (int jb = j0; jb < j1; jb += TECCL_CONS_U) {
        int2 e4[TECCL_CONS_U];
#pragma unroll
        for (int u = 0; u < TECCL_CONS_U; ++u) e4[u] = (jb + u < j1) ? __ldg(o.incp + jb + u) : make_int2(0, 0);
        double w[TECCL_CONS_U], v[kSegPerLane][TECCL_CONS_U];
#pragma unroll
        for (int u = 0; u < TECCL_CONS_U; ++u) {
          w[u] = (jb + u < j1) ? (e4[u].y < 0 ? -1.0 : 1.0) : 0.0;
#pragma unroll
          for (int h = 0; h < kSegPerLane; ++h) v[h][u] = __ldg(xb + e4[u].x + 32 * h);
        }
#pragma unroll
        for (int h = 0; h < kSegPerLane; ++h)
#pragma unroll
          for (int u = 0; u < TECCL_CONS_U; ++u) a[h] = fma(w[u], v[h][u], a[h]);
      }
    }
    for (int jb = interior ? j1 : j0; jb < j1; jb += 4) {
      int2 e4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) e4[u] = (jb + u < j1) ? __ldg(o.incp + jb + u) : make_int2(0, (int)K);
#pragma unroll
      for (int h = 0; h < kSegPerLane; ++h) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ke = kk[h] - e4[u].y;          // epoch of the term; out of range = absent
          const bool ok = on[h] && ke >= 0 && ke <= (int)K - 1 && !(last[h] && e4[u].y < 0);
          v[u] = ok ? __ldg(xs + e4[u].x + kk[h]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) a[h] += (e4[u].y < 0) ? -v[u] : v[u];
      }
    }
    const double* bg = xs + o.EK + (uint32_t)(g >= 0 ? g : 0) * (K + 1);
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      if (!on[h]) continue;
      if (!last[h]) {
        if (g >= 0) {
          a[h] += __ldg(bg + kk[h]) - __ldg(bg + kk[h] + 1);
          if (tn.y >= 0) a[h] -= __ldg(x + (uint32_t)tn.y + 2 * kk[h]);
        }
      } else if (tn.y >= 0) {
        a[h] -= __ldg(x + (uint32_t)tn.y + 2 * (K - 1));
      }
    }
  } else if (kind == SEG_CUM) {                    // cum(p,k)
    const uint32_t rd0 = o.nF + (uint32_t)A * 2 * K;
#if TECCL_CUM_SHFL
    // Rc(p,k-1) is the previous lane's Rc: two loads per row instead of three,
    // the same operands and operations (the task's first row loads its own)
    double rdv[kSegPerLane], rcv[kSegPerLane];
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      const uint32_t rd = rd0 + 2 * (uint32_t)(off + i);
      rdv[h] = (i < cnt) ? __ldg(x + rd) : 0.0;
      rcv[h] = (i < cnt) ? __ldg(x + rd + 1) : 0.0;
    }
    const double first_prev = (lane == 0 && off >= 1) ? __ldg(x + rd0 + 2 * (uint32_t)off - 1) : 0.0;
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      double prev = __shfl_up_sync(0xffffffffu, rcv[h], 1);
      const double carry = __shfl_sync(0xffffffffu, h > 0 ? rcv[h > 0 ? h - 1 : 0] : 0.0, 31);
      if (lane == 0) prev = (h == 0) ? first_prev : carry;
      if (lane + 32 * h < cnt) a[h] = rcv[h] - rdv[h] - prev;
    }
#else
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
        const uint32_t k = off + i, rd = rd0 + 2 * k;
        const double v_prev = (k >= 1) ? __ldg(x + rd - 1) : 0.0;
        a[h] = __ldg(x + rd + 1) - __ldg(x + rd) - v_prev;
      }
    }
#endif
  } else if (kind == SEG_BCAP) {                   // bcap(g,k): sum_s B(s,g,k)
    const uint32_t q0 = o.EK + (uint32_t)Bv * (K + 1) + off;
#if TECCL_CAP_JOINT
    seg_sum_sources(o, x, q0, lane, cnt, a);
#endif
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) {
#if !TECCL_CAP_JOINT
        a[h] = te_sum_sources(o, x, q0 + i);
#endif
        lo[h] = -INFINITY;
        hi[h] = o.d.blimit;
      }
    }
  } else if (kind == SEG_INIT) {                   // init(s): generic path
#pragma unroll
    for (int h = 0; h < kSegPerLane; ++h) {
      const int i = lane + 32 * h;
      if (i < cnt) a[h] = te_row(o, (uint32_t)(off + i), x, lo[h], hi[h]);
    }
  }
}

}  // namespace teccl

// C-ABI plumbing: errors, contexts, generic LP upload/export.
// The generic upload replaces the matrix assembly of the reference solver
// (pkg/src/collsched/solver.py:100-121) for any Model, so the same PDLP
// kernels serve the reference's own model objects.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <string>
#include <vector>

#include "common.cuh"

namespace teccl {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
std::mutex& device_mutex() {
  static std::mutex mu;
  return mu;
}
}  // namespace teccl

using namespace teccl;

extern "C" const char* teccl_last_error(void) { return g_err.c_str(); }
extern "C" const char* teccl_version(void) { return "teccl_b200 0.1.0 sm_100a"; }

extern "C" int teccl_ctx_create(int device, teccl_ctx** out) {
  if (!out) { set_error("null argument"); return TECCL_EINVAL; }
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    return TECCL_ENODEV;
  }
  if (device < 0 || device >= count) { set_error("device index out of range"); return TECCL_EINVAL; }
  cudaDeviceProp prop;
  TECCL_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("teccl_b200 needs an sm_100 (B200) device, found sm_" + std::to_string(prop.major) +
              std::to_string(prop.minor));
    return TECCL_ENODEV;
  }
  TECCL_CUDA(cudaSetDevice(device));
  // keep freed stream-ordered allocations in the pool instead of returning
  // them to the driver at every synchronisation (solves allocate ~100 MB)
  cudaMemPool_t pool;
  TECCL_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = UINT64_MAX;
  TECCL_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  teccl_ctx* c = new teccl_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  TECCL_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  *out = c;
  return TECCL_OK;
}

extern "C" int teccl_ctx_destroy(teccl_ctx* ctx) {
  if (!ctx) return TECCL_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TECCL_OK;
}

extern "C" int teccl_ctx_sync(teccl_ctx* ctx) {
  if (!ctx) { set_error("null argument"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaStreamSynchronize(ctx->stream));
  return TECCL_OK;
}

namespace {
template <typename T>
int to_dev(const std::vector<T>& h, T** d, cudaStream_t st) {
  TECCL_CUDA(cudaMallocAsync((void**)d, (h.size() + 1) * sizeof(T), st));
  if (!h.empty())
    TECCL_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return TECCL_OK;
}
}  // namespace

extern "C" int teccl_lp_from_csr(teccl_ctx* ctx, int32_t m, int32_t n, int64_t nnz,
                                 const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const double* row_lo, const double* row_hi, const double* var_lb,
                                 const double* var_ub, const double* obj, teccl_lp** out) {
  if (!ctx || !out || m < 0 || n < 0 || nnz < 0 || !row_ptr || !row_lo || !row_hi || !var_lb ||
      !var_ub || !obj || (nnz > 0 && (!col || !val))) {
    set_error("bad argument");
    return TECCL_EINVAL;
  }
  if (row_ptr[0] != 0 || row_ptr[m] != nnz) { set_error("row_ptr inconsistent with nnz"); return TECCL_EINVAL; }
  if ((int64_t)n >= (int64_t)kSignBit) { set_error("too many columns"); return TECCL_EINVAL; }
  // Canonical CSR: columns ascending, duplicates merged, zeros dropped.
  std::vector<int64_t> rp(m + 1, 0);
  std::vector<uint32_t> ci;
  std::vector<double> cv;
  ci.reserve(nnz);
  cv.reserve(nnz);
  std::vector<std::pair<int32_t, double>> rowbuf;
  bool unit = true;
  for (int32_t i = 0; i < m; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) { set_error("row_ptr not monotone"); return TECCL_EINVAL; }
    rowbuf.clear();
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col[p] < 0 || col[p] >= n) { set_error("column index out of range"); return TECCL_EINVAL; }
      if (!std::isfinite(val[p])) { set_error("non-finite coefficient"); return TECCL_EINVAL; }
      rowbuf.push_back({col[p], val[p]});
    }
    std::stable_sort(rowbuf.begin(), rowbuf.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    for (size_t k = 0; k < rowbuf.size();) {
      int32_t c = rowbuf[k].first;
      double s = 0.0;
      while (k < rowbuf.size() && rowbuf[k].first == c) s += rowbuf[k++].second;
      if (s != 0.0) {
        ci.push_back((uint32_t)c);
        cv.push_back(s);
        if (s != 1.0 && s != -1.0) unit = false;
      }
    }
    rp[i + 1] = (int64_t)ci.size();
  }
  const int64_t nz = (int64_t)ci.size();
  // CSC by a stable counting sort over the canonical CSR (rows ascend per column).
  std::vector<int64_t> cp(n + 1, 0);
  for (int64_t p = 0; p < nz; ++p) cp[ci[p] + 1]++;
  for (int32_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  std::vector<uint32_t> ri(nz);
  std::vector<double> rv(nz);
  {
    std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
    for (int32_t i = 0; i < m; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        int64_t q = fill[ci[p]]++;
        ri[q] = (uint32_t)i;
        rv[q] = cv[p];
      }
  }
  if (unit) {
    for (int64_t p = 0; p < nz; ++p) {
      if (cv[p] < 0) ci[p] |= kSignBit;
      if (rv[p] < 0) ri[p] |= kSignBit;
    }
  }
  cudaStream_t st = ctx->stream;
  TECCL_CUDA(cudaSetDevice(ctx->device));
  teccl_lp* lp = new teccl_lp();
  lp->m = m;
  lp->n = n;
  lp->nnz = nz;
  lp->unit = unit;
  lp->device = ctx->device;
  lp->stream = st;
  int rc = 0;
  rc |= to_dev(rp, &lp->row_ptr, st);
  rc |= to_dev(ci, &lp->col, st);
  rc |= to_dev(cp, &lp->col_ptr, st);
  rc |= to_dev(ri, &lp->row, st);
  if (!unit) {
    rc |= to_dev(cv, &lp->val, st);
    rc |= to_dev(rv, &lp->cval, st);
  }
  rc |= to_dev(std::vector<double>(row_lo, row_lo + m), &lp->row_lo, st);
  rc |= to_dev(std::vector<double>(row_hi, row_hi + m), &lp->row_hi, st);
  rc |= to_dev(std::vector<double>(var_lb, var_lb + n), &lp->var_lb, st);
  rc |= to_dev(std::vector<double>(var_ub, var_ub + n), &lp->var_ub, st);
  rc |= to_dev(std::vector<double>(obj, obj + n), &lp->obj, st);
  if (rc) { set_error("device upload failed"); return TECCL_ECUDA; }
  // bound-class dictionaries for the PDLP kernels (first-seen order)
  {
    struct KeyHash {
      size_t operator()(const std::array<uint64_t, 3>& k) const {
        uint64_t h = 1469598103934665603ull;
        for (uint64_t v : k) { h ^= v; h *= 1099511628211ull; h ^= h >> 29; }
        return (size_t)h;
      }
    };
    auto bits = [](double v) {
      v += 0.0;  // -0.0 -> +0.0
      uint64_t b;
      memcpy(&b, &v, sizeof b);
      return b;
    };
    std::unordered_map<std::array<uint64_t, 3>, int, KeyHash> cmap, rmap;
    std::vector<uint16_t> ccode(n), rcode(m);
    std::vector<double> cdict, rdict;
    bool cok = true, rok = true;
    for (int32_t j = 0; j < n && cok; ++j) {
      std::array<uint64_t, 3> k{bits(var_lb[j]), bits(var_ub[j]), bits(obj[j])};
      auto it = cmap.find(k);
      if (it == cmap.end()) {
        if ((int)cmap.size() >= kMaxDict) { cok = false; break; }
        it = cmap.emplace(k, (int)cmap.size()).first;
        cdict.push_back(var_lb[j] + 0.0); cdict.push_back(var_ub[j] + 0.0); cdict.push_back(obj[j] + 0.0);
      }
      ccode[j] = (uint16_t)it->second;
    }
    for (int32_t i = 0; i < m && rok; ++i) {
      std::array<uint64_t, 3> k{bits(row_lo[i]), bits(row_hi[i]), 0};
      auto it = rmap.find(k);
      if (it == rmap.end()) {
        if ((int)rmap.size() >= kMaxDict) { rok = false; break; }
        it = rmap.emplace(k, (int)rmap.size()).first;
        rdict.push_back(row_lo[i] + 0.0); rdict.push_back(row_hi[i] + 0.0);
      }
      rcode[i] = (uint16_t)it->second;
    }
    if (cok && rok) {
      rc |= to_dev(ccode, &lp->col_code, st);
      rc |= to_dev(rcode, &lp->row_code, st);
      rc |= to_dev(cdict, &lp->col_dict, st);
      rc |= to_dev(rdict, &lp->row_dict, st);
      lp->n_col_dict = (int32_t)cmap.size();
      lp->n_row_dict = (int32_t)rmap.size();
      if (rc) { set_error("device upload failed"); return TECCL_ECUDA; }
    }
  }
  TECCL_CUDA(cudaStreamSynchronize(st));
  *out = lp;
  return TECCL_OK;
}

extern "C" int teccl_lp_dims(const teccl_lp* lp, int32_t* m, int32_t* n, int64_t* nnz) {
  if (!lp) { set_error("null lp"); return TECCL_EINVAL; }
  if (m) *m = lp->m;
  if (n) *n = lp->n;
  if (nnz) *nnz = lp->nnz;
  return TECCL_OK;
}

namespace {
int export_matrix(const teccl_lp* lp, bool csc, int64_t* ptr, int32_t* idx, double* val) {
  const int64_t major = csc ? lp->n : lp->m;
  const int64_t* dptr = csc ? lp->col_ptr : lp->row_ptr;
  const uint32_t* didx = csc ? lp->row : lp->col;
  const double* dval = csc ? lp->cval : lp->val;
  const int64_t nz = (csc && lp->nnz_csc >= 0) ? lp->nnz_csc : lp->nnz;
  if (ptr) TECCL_CUDA(cudaMemcpy(ptr, dptr, (major + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (idx || val) {
    std::vector<uint32_t> raw(nz);
    if (nz) TECCL_CUDA(cudaMemcpy(raw.data(), didx, nz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (lp->unit) {
      for (int64_t p = 0; p < nz; ++p) {
        if (idx) idx[p] = (int32_t)(raw[p] & kIdxMask);
        if (val) val[p] = (raw[p] & kSignBit) ? -1.0 : 1.0;
      }
    } else {
      for (int64_t p = 0; p < nz; ++p)
        if (idx) idx[p] = (int32_t)raw[p];
      if (val && nz)
        TECCL_CUDA(cudaMemcpy(val, dval, nz * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  return TECCL_OK;
}
}  // namespace

extern "C" int teccl_lp_export(const teccl_lp* lp, int64_t* row_ptr, int32_t* col, double* val,
                               double* row_lo, double* row_hi, double* var_lb, double* var_ub,
                               double* obj) {
  if (!lp) { set_error("null lp"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(lp->device));
  if (lp->stream) TECCL_CUDA(cudaStreamSynchronize(lp->stream));
  int rc = export_matrix(lp, false, row_ptr, col, val);
  if (rc) return rc;
  if (row_lo) TECCL_CUDA(cudaMemcpy(row_lo, lp->row_lo, lp->m * sizeof(double), cudaMemcpyDeviceToHost));
  if (row_hi) TECCL_CUDA(cudaMemcpy(row_hi, lp->row_hi, lp->m * sizeof(double), cudaMemcpyDeviceToHost));
  if (var_lb) TECCL_CUDA(cudaMemcpy(var_lb, lp->var_lb, lp->n * sizeof(double), cudaMemcpyDeviceToHost));
  if (var_ub) TECCL_CUDA(cudaMemcpy(var_ub, lp->var_ub, lp->n * sizeof(double), cudaMemcpyDeviceToHost));
  if (obj) TECCL_CUDA(cudaMemcpy(obj, lp->obj, lp->n * sizeof(double), cudaMemcpyDeviceToHost));
  return TECCL_OK;
}

extern "C" int teccl_lp_export_csc(const teccl_lp* lp, int64_t* col_ptr, int32_t* row, double* val) {
  if (!lp) { set_error("null lp"); return TECCL_EINVAL; }
  TECCL_CUDA(cudaSetDevice(lp->device));
  if (lp->stream) TECCL_CUDA(cudaStreamSynchronize(lp->stream));
  return export_matrix(lp, true, col_ptr, row, val);
}

extern "C" int teccl_lp_destroy(teccl_lp* lp) {
  if (!lp) return TECCL_OK;
  cudaSetDevice(lp->device);
  if (lp->stream) {
    cudaStreamSynchronize(lp->stream);
  } else {
    std::lock_guard<std::mutex> lock(device_mutex());
    cudaDeviceSynchronize();
  }
  if (lp->pdlp_ws && lp->ws_free) lp->ws_free(lp->pdlp_ws);
  if (lp->dist && lp->dist_free) lp->dist_free(lp->dist);
  if (lp->src && lp->src_free) lp->src_free(lp->src);
  if (lp->te && lp->te_free) lp->te_free(lp->te);
  void* ptrs[] = {lp->row_ptr, lp->col, lp->val, lp->col_ptr, lp->row, lp->cval,
                  lp->row_lo, lp->row_hi, lp->var_lb, lp->var_ub, lp->obj,
                  lp->srow_off, lp->srow_w, lp->sell_idx, lp->srow_val,
                  lp->scol_off, lp->scol_w, lp->scol_val,
                  lp->col_code, lp->row_code, lp->col_dict, lp->row_dict};
  {
    std::unique_lock<std::mutex> lock(device_mutex(), std::defer_lock);
    if (!lp->stream) lock.lock();  // cudaFree synchronises the device
    for (void* p : ptrs)
      if (p) {
        if (lp->stream) cudaFreeAsync(p, lp->stream);
        else cudaFree(p);
      }
  }
  if (lp->stream) cudaStreamSynchronize(lp->stream);
  delete lp;
  return TECCL_OK;
}

// SELL-32 re-layout of an LP's CSR (rows) and CSC (columns) for the PDLP
// iteration kernels (see pdlp.cu "SELL-32 SpMV"). Runs once per LP.

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace teccl {

// width[s] = max row length in slice s (warp per slice)
__global__ void sell_width_kernel(int64_t count, int64_t nslices, const int64_t* __restrict__ ptr,
                                  int32_t* __restrict__ width, int64_t* __restrict__ slice_len) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nslices) return;
  const int64_t r = warp * 32 + lane;
  int len = (r < count) ? (int)(ptr[r + 1] - ptr[r]) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  if (lane == 0) {
    width[warp] = len;
    slice_len[warp] = (int64_t)len * 32;
  }
}

__global__ void sell_fill_kernel(int64_t count, int64_t nslices, const int64_t* __restrict__ ptr,
                                 const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                 const int64_t* __restrict__ off, const int32_t* __restrict__ width,
                                 uint32_t sentinel, uint32_t* __restrict__ sidx,
                                 double* __restrict__ sval) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nslices * 32) return;
  const int64_t s = r >> 5;
  const int w = width[s];
  const int64_t base = off[s] + (r & 31);
  int64_t b = 0, len = 0;
  if (r < count) {
    b = ptr[r];
    len = ptr[r + 1] - b;
  }
  for (int q = 0; q < w; ++q) {
    const int64_t p = base + (int64_t)q * 32;
    if (q < len) {
      sidx[p] = idx[b + q];
      if (sval) sval[p] = val[b + q];
    } else {
      sidx[p] = sentinel;
      if (sval) sval[p] = 0.0;
    }
  }
}

// Slice widths and offsets of one orientation; *entries = stored entries.
static int sell_layout(int64_t count, const int64_t* ptr, cudaStream_t st, int64_t** off,
                       int32_t** width, int64_t* entries) {
  const int64_t ns = (count + 31) / 32;
  int64_t* slice_len = nullptr;
  TECCL_CUDA(cudaMallocAsync((void**)off, sizeof(int64_t) * (ns + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)width, sizeof(int32_t) * (ns + 1), st));
  TECCL_CUDA(cudaMallocAsync((void**)&slice_len, sizeof(int64_t) * (ns + 1), st));
  int64_t total = 0;
  if (ns > 0) {
    sell_width_kernel<<<(int)((ns * 32 + 255) / 256), 256, 0, st>>>(count, ns, ptr, *width, slice_len);
    TECCL_CHECK_LAUNCH();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, slice_len, *off, ns + 1, st);
    void* tmp = nullptr;
    TECCL_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    TECCL_CUDA(cudaMemsetAsync(slice_len + ns, 0, sizeof(int64_t), st));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, slice_len, *off, ns + 1, st);
    TECCL_CHECK_LAUNCH();
    TECCL_CUDA(cudaFreeAsync(tmp, st));
    TECCL_CUDA(cudaMemcpyAsync(&total, *off + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  TECCL_CUDA(cudaFreeAsync(slice_len, st));
  TECCL_CUDA(cudaStreamSynchronize(st));
  *entries = total;
  return TECCL_OK;
}

static int sell_fill(int64_t count, const int64_t* ptr, const uint32_t* idx, const double* val,
                     uint32_t sentinel, cudaStream_t st, const int64_t* off, const int32_t* width,
                     uint32_t* sidx, double** sval, int64_t entries) {
  const int64_t ns = (count + 31) / 32;
  if (val) TECCL_CUDA(cudaMallocAsync((void**)sval, sizeof(double) * (entries + 4), st));
  if (ns > 0) {
    sell_fill_kernel<<<(int)((ns * 32 + 255) / 256), 256, 0, st>>>(
        count, ns, ptr, idx, val, off, width, sentinel, sidx, val ? *sval : nullptr);
    TECCL_CHECK_LAUNCH();
  }
  return TECCL_OK;
}

}  // namespace teccl

int teccl_build_sell(teccl_lp* lp, cudaStream_t st) {
  using namespace teccl;
  if (lp->sell_ready) return TECCL_OK;
  int rc = sell_layout(lp->m, lp->row_ptr, st, &lp->srow_off, &lp->srow_w, &lp->srow_entries);
  if (rc) return rc;
  rc = sell_layout(lp->n, lp->col_ptr, st, &lp->scol_off, &lp->scol_w, &lp->scol_entries);
  if (rc) return rc;
  // both index streams in one allocation, so one L2 access-policy window
  // can cover them (pdlp.cu keeps them L2-resident across iterations)
  const int64_t rpad = (lp->srow_entries + 63) / 64 * 64;
  TECCL_CUDA(cudaMallocAsync((void**)&lp->sell_idx, sizeof(uint32_t) * (rpad + lp->scol_entries + 64), st));
  lp->srow_idx = lp->sell_idx;
  lp->scol_idx = lp->sell_idx + rpad;
  lp->sell_idx_bytes = sizeof(uint32_t) * (rpad + lp->scol_entries);
  rc = sell_fill(lp->m, lp->row_ptr, lp->col, lp->unit ? nullptr : lp->val, (uint32_t)gather_cols(lp),
                 st, lp->srow_off, lp->srow_w, lp->srow_idx, &lp->srow_val, lp->srow_entries);
  if (rc) return rc;
  rc = sell_fill(lp->n, lp->col_ptr, lp->row, lp->unit ? nullptr : lp->cval, (uint32_t)gather_rows(lp),
                 st, lp->scol_off, lp->scol_w, lp->scol_idx, &lp->scol_val, lp->scol_entries);
  if (rc) return rc;
  TECCL_CUDA(cudaStreamSynchronize(st));
  lp->sell_ready = true;
  return TECCL_OK;
}

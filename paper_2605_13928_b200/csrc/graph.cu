// sc.pp.neighbors' graph outputs (first half: the UMAP fuzzy graph that
// UMAP and Leiden consume): `connectivities` = umap-learn's fuzzy_simplicial_set on the exact
// kNN (set_op_mix_ratio 1, local_connectivity 1) and `distances` (kNN distances, self removed).
//
//   weights   thread per cell: rho = first non-zero distance; sigma by 64-step bisection of
//             sum_{j>=1} exp(-max(d_j - rho, 0)/sigma) = log2(k) (tolerance 1e-5, f64 as umap's
//             numba code), floored at 1e-3 x mean distance; w_ij = exp(-(d_ij - rho)/sigma)
//             (f32), 1 if d_ij <= rho, 0 for the self edge.
//   union     C = W + Wᵀ - W∘Wᵀ in f32 exactly as scipy evaluates it: for a reciprocated pair
//             fl(fl(a + b) - fl(a b)), otherwise a.  Row i holds its own out-edges plus the
//             in-edges j -> i that i does not reciprocate; counts (atomic per target row) ->
//             scan -> fill (atomic cursors for in-edges) -> per-row sort by column.
// Rows are a range [r0, r1) of the global kNN graph so a cell-sharded caller builds its own rows
// from the all-gathered (idx, w) (multi-GPU).  Oracle: oracle/pipeline.py umap_connectivities.
#include "common.cuh"
#include "scan.cuh"

namespace scb {

constexpr int kMaxK = 64;

__global__ void knn_dist_sum_kernel(const float* __restrict__ dist, int64_t n, double* __restrict__ out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (double)dist[i];
  s = warp_sum(s);
  if (lane_id() == 0) atomicAdd(out, s);
}

__global__ void __launch_bounds__(128)
umap_weights_kernel(const int32_t* __restrict__ idx, const float* __restrict__ dist, int64_t n_rows, int k,
                    int64_t row0, const double* __restrict__ mean_dist, float* __restrict__ sigma_out,
                    float* __restrict__ rho_out, float* __restrict__ w) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const float* d = dist + i * k;
  float rho = 0.0f;
  double rsum = 0.0;
  for (int j = 0; j < k; ++j) {
    const float v = d[j];
    rsum += (double)v;
    if (rho == 0.0f && v > 0.0f) rho = v;
  }
  const double target = log2((double)k);
  double lo = 0.0, hi = CUDART_INF, mid = 1.0;
  for (int it = 0; it < 64; ++it) {
    double psum = 0.0;
    for (int j = 1; j < k; ++j) {
      const float dd = __fsub_rn(d[j], rho);
      psum += dd > 0.0f ? exp(-((double)dd / mid)) : 1.0;
    }
    if (fabs(psum - target) < 1e-5) break;
    if (psum > target) {
      hi = mid;
      mid = (lo + hi) / 2.0;
    } else {
      lo = mid;
      mid = isinf(hi) ? mid * 2.0 : (lo + hi) / 2.0;
    }
  }
  float sig = (float)mid;
  const double floor_d = 1e-3 * (rho > 0.0f ? rsum / k : *mean_dist);
  if ((double)sig < floor_d) sig = (float)floor_d;
  sigma_out[i] = sig;
  rho_out[i] = rho;
  for (int j = 0; j < k; ++j) {
    const float dd = __fsub_rn(d[j], rho);
    float v;
    if (idx[i * k + j] == row0 + i) v = 0.0f;
    else if (dd <= 0.0f || sig == 0.0f) v = 1.0f;
    else v = expf(-__fdiv_rn(dd, sig));
    w[i * k + j] = v;
  }
}

// weight of edge (j -> i) if present, else 0
__device__ __forceinline__ float reverse_w(const int32_t* __restrict__ idx, const float* __restrict__ w, int k,
                                           int64_t j, int64_t i) {
  const int32_t* rj = idx + j * k;
  for (int t = 0; t < k; ++t)
    if (rj[t] == (int32_t)i) return w[j * k + t];
  return 0.0f;
}

// thread per global edge (i -> j), j in [r0, r1): an unreciprocated edge adds one entry to row j
__global__ void fuzzy_count_in_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int64_t n_all, int k,
                                      int64_t r0, int64_t r1, unsigned long long* __restrict__ extra) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_all * k) return;
  const float a = w[e];
  if (a == 0.0f) return;
  const int64_t i = e / k, j = idx[e];
  if (j < r0 || j >= r1) return;
  if (reverse_w(idx, w, k, j, i) == 0.0f) atomicAdd(&extra[j - r0], 1ull);
}

__global__ void fuzzy_row_len_kernel(const float* __restrict__ w, int k, int64_t r0, int64_t n_loc,
                                     const unsigned long long* __restrict__ extra, int64_t* __restrict__ len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  int own = 0;
  for (int t = 0; t < k; ++t) own += w[(r0 + i) * k + t] != 0.0f;
  len[i] = own + (int64_t)extra[i];
}

__global__ void fuzzy_fill_own_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int k, int64_t r0,
                                      int64_t n_loc, const int64_t* __restrict__ indptr, int32_t* __restrict__ cols,
                                      float* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const int64_t gi = r0 + i;
  int64_t o = indptr[i];
  for (int t = 0; t < k; ++t) {
    const float a = w[gi * k + t];
    if (a == 0.0f) continue;
    const int64_t j = idx[gi * k + t];
    const float b = reverse_w(idx, w, k, j, gi);
    cols[o] = (int32_t)j;
    vals[o] = b != 0.0f ? __fsub_rn(__fadd_rn(a, b), __fmul_rn(a, b)) : a;
    ++o;
  }
}

__global__ void fuzzy_fill_in_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int64_t n_all, int k,
                                     int64_t r0, int64_t r1, const int64_t* __restrict__ indptr,
                                     const int64_t* __restrict__ own_end, unsigned long long* __restrict__ cursor,
                                     int32_t* __restrict__ cols, float* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_all * k) return;
  const float a = w[e];
  if (a == 0.0f) return;
  const int64_t i = e / k, j = idx[e];
  if (j < r0 || j >= r1) return;
  if (reverse_w(idx, w, k, j, i) != 0.0f) return;
  const int64_t row = j - r0;
  const int64_t pos = own_end[row] + (int64_t)atomicAdd(&cursor[row], 1ull);
  cols[pos] = (int32_t)i;
  vals[pos] = a;
  (void)indptr;
}

// own_end[i] = indptr[i] + own count
__global__ void fuzzy_own_end_kernel(const float* __restrict__ w, int k, int64_t r0, int64_t n_loc,
                                     const int64_t* __restrict__ indptr, int64_t* __restrict__ own_end) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  int own = 0;
  for (int t = 0; t < k; ++t) own += w[(r0 + i) * k + t] != 0.0f;
  own_end[i] = indptr[i] + own;
}

// warp per row: bitonic sort by column in shared memory (rows <= kWarpSort entries); longer
// rows are flagged for the CTA pass
constexpr int kWarpSort = 256;
constexpr int kSortWarps = 8;
__global__ void __launch_bounds__(kSortWarps * 32)
sort_rows_warp_kernel(const int64_t* __restrict__ indptr, int64_t n_loc, int32_t* __restrict__ cols,
                      float* __restrict__ vals, int* __restrict__ long_rows) {
  __shared__ int32_t sk[kSortWarps][kWarpSort];
  __shared__ float sv[kSortWarps][kWarpSort];
  const int wid = warp_id(), lane = lane_id();
  for (int64_t r = (int64_t)blockIdx.x * kSortWarps + wid; r < n_loc; r += (int64_t)gridDim.x * kSortWarps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    const int len = (int)(e - b);
    if (len <= 1) continue;
    if (len > kWarpSort) {
      if (lane == 0) atomicOr(long_rows, 1);
      continue;
    }
    int np2 = 2;
    while (np2 < len) np2 <<= 1;
    for (int t = lane; t < np2; t += 32) {
      sk[wid][t] = t < len ? cols[b + t] : INT32_MAX;
      sv[wid][t] = t < len ? vals[b + t] : 0.0f;
    }
    __syncwarp();
    for (int kk = 2; kk <= np2; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int t = lane; t < np2; t += 32) {
          const int l = t ^ jj;
          if (l > t) {
            const bool up = (t & kk) == 0;
            const int32_t x = sk[wid][t], y = sk[wid][l];
            if ((x > y) == up) {
              sk[wid][t] = y;
              sk[wid][l] = x;
              const float tv = sv[wid][t];
              sv[wid][t] = sv[wid][l];
              sv[wid][l] = tv;
            }
          }
        }
        __syncwarp();
      }
    for (int t = lane; t < len; t += 32) {
      cols[b + t] = sk[wid][t];
      vals[b + t] = sv[wid][t];
    }
    __syncwarp();
  }
}

// CTA per long row (rare hub cells): odd-even transposition is enough for a few thousand entries
constexpr int kCtaSort = 16384;
__global__ void __launch_bounds__(1024)
sort_rows_cta_kernel(const int64_t* __restrict__ indptr, int64_t n_loc, int32_t* __restrict__ cols,
                     float* __restrict__ vals, int* __restrict__ too_long) {
  extern __shared__ int32_t ck[];
  float* cv = reinterpret_cast<float*>(ck + kCtaSort);
  for (int64_t r = blockIdx.x; r < n_loc; r += gridDim.x) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    const int len = (int)(e - b);
    if (len <= kWarpSort) continue;
    if (len > kCtaSort) {
      if (threadIdx.x == 0) atomicOr(too_long, 1);
      continue;
    }
    int np2 = 2;
    while (np2 < len) np2 <<= 1;
    for (int t = threadIdx.x; t < np2; t += blockDim.x) {
      ck[t] = t < len ? cols[b + t] : INT32_MAX;
      cv[t] = t < len ? vals[b + t] : 0.0f;
    }
    __syncthreads();
    for (int kk = 2; kk <= np2; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int t = threadIdx.x; t < np2; t += blockDim.x) {
          const int l = t ^ jj;
          if (l > t) {
            const bool up = (t & kk) == 0;
            const int32_t x = ck[t], y = ck[l];
            if ((x > y) == up) {
              ck[t] = y;
              ck[l] = x;
              const float tv = cv[t];
              cv[t] = cv[l];
              cv[l] = tv;
            }
          }
        }
        __syncthreads();
      }
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
      cols[b + t] = ck[t];
      vals[b + t] = cv[t];
    }
    __syncthreads();
  }
}

// sc.pp.neighbors `distances`: per row the non-zero kNN distances (self and exact duplicates
// at distance 0 removed, as scipy's eliminate_zeros), sorted by column
__global__ void knn_dist_len_kernel(const float* __restrict__ dist, int64_t n_rows, int k, int64_t* __restrict__ len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  int c = 0;
  for (int t = 0; t < k; ++t) c += dist[i * k + t] != 0.0f;
  len[i] = c;
}
__global__ void knn_dist_fill_kernel(const int32_t* __restrict__ idx, const float* __restrict__ dist, int64_t n_rows,
                                     int k, const int64_t* __restrict__ indptr, int32_t* __restrict__ cols,
                                     float* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  int64_t o = indptr[i];
  for (int t = 0; t < k; ++t) {
    const float v = dist[i * k + t];
    if (v == 0.0f) continue;
    cols[o] = idx[i * k + t];
    vals[o] = v;
    ++o;
  }
}

static int sort_rows(scb_ctx* ctx, const int64_t* indptr, int64_t n_loc, int32_t* cols, float* vals, cudaStream_t s) {
  int* flag = ctx->d_flag + 3;
  SCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  sort_rows_warp_kernel<<<ctx->num_sms * 8, kSortWarps * 32, 0, s>>>(indptr, n_loc, cols, vals, flag);
  SCB_LAUNCH_CHECK();
  int f = 0;
  SCB_CUDA(cudaMemcpyAsync(&f, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  if (f) {
    SCB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    const int smem = kCtaSort * 8;
    SCB_CUDA(cudaFuncSetAttribute(sort_rows_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    sort_rows_cta_kernel<<<ctx->num_sms, 1024, smem, s>>>(indptr, n_loc, cols, vals, flag);
    SCB_LAUNCH_CHECK();
    SCB_CUDA(cudaMemcpyAsync(&f, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    SCB_REQUIRE(f == 0, SCB_ERR_UNSUPPORTED, "graph row longer than %d entries", kCtaSort);
  }
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_knn_dist_sum(scb_ctx* ctx, const float* knn_dist, int64_t n, double* sum, void* stream) {
  SCB_REQUIRE(ctx && knn_dist && sum, SCB_ERR_ARG, "scb_knn_dist_sum: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  SCB_CUDA(cudaMemsetAsync(sum, 0, sizeof(double), s));
  if (n == 0) return SCB_OK;
  knn_dist_sum_kernel<<<ctx->num_sms * 4, 256, 0, s>>>(knn_dist, n, sum);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_umap_weights(scb_ctx* ctx, const int32_t* knn_idx, const float* knn_dist, int64_t n_rows, int32_t k,
                                int64_t row0, const double* mean_dist, float* sigma, float* rho, float* w,
                                void* stream) {
  SCB_REQUIRE(ctx && knn_idx && knn_dist && mean_dist && sigma && rho && w, SCB_ERR_ARG,
              "scb_umap_weights: null argument");
  SCB_REQUIRE(k >= 2 && k <= kMaxK, SCB_ERR_ARG, "scb_umap_weights: k must be in [2, %d]", kMaxK);
  if (n_rows == 0) return SCB_OK;
  umap_weights_kernel<<<(unsigned)ceil_div(n_rows, 128), 128, 0, (cudaStream_t)stream>>>(
      knn_idx, knn_dist, n_rows, k, row0, mean_dist, sigma, rho, w);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_fuzzy_union_rows(scb_ctx* ctx, const int32_t* idx_all, const float* w_all, int64_t n_all, int32_t k,
                                    int64_t r0, int64_t r1, int64_t* indptr, void* stream) {
  SCB_REQUIRE(ctx && idx_all && w_all && indptr, SCB_ERR_ARG, "scb_fuzzy_union_rows: null argument");
  SCB_REQUIRE(0 <= r0 && r0 <= r1 && r1 <= n_all && k >= 1, SCB_ERR_ARG, "scb_fuzzy_union_rows: bad row range");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_loc = r1 - r0;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_loc + 1) * 8 * 2, &ws, s));
  unsigned long long* extra = (unsigned long long*)ws;
  int64_t* len = (int64_t*)(extra + (n_loc + 1));
  SCB_CUDA(cudaMemsetAsync(extra, 0, (size_t)(n_loc + 1) * 8, s));
  if (n_all * k > 0) {
    fuzzy_count_in_kernel<<<(unsigned)ceil_div(n_all * k, 256), 256, 0, s>>>(idx_all, w_all, n_all, k, r0, r1,
                                                                                       extra);
    SCB_LAUNCH_CHECK();
  }
  if (n_loc > 0) {
    fuzzy_row_len_kernel<<<(unsigned)ceil_div(n_loc, 256), 256, 0, s>>>(w_all, k, r0, n_loc, extra, len);
    SCB_LAUNCH_CHECK();
  }
  SCB_TRY(scan_i64(ctx, len, n_loc, indptr, s));
  return SCB_OK;
}

extern "C" int scb_fuzzy_union_fill(scb_ctx* ctx, const int32_t* idx_all, const float* w_all, int64_t n_all, int32_t k,
                                    int64_t r0, int64_t r1, const int64_t* indptr, int32_t* cols, float* vals,
                                    void* stream) {
  SCB_REQUIRE(ctx && idx_all && w_all && indptr && cols && vals, SCB_ERR_ARG, "scb_fuzzy_union_fill: null argument");
  SCB_REQUIRE(0 <= r0 && r0 <= r1 && r1 <= n_all && k >= 1, SCB_ERR_ARG, "scb_fuzzy_union_fill: bad row range");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_loc = r1 - r0;
  if (n_loc == 0) return SCB_OK;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_loc + 1) * 8 * 2, &ws, s));
  unsigned long long* cursor = (unsigned long long*)ws;
  int64_t* own_end = (int64_t*)(cursor + (n_loc + 1));
  SCB_CUDA(cudaMemsetAsync(cursor, 0, (size_t)(n_loc + 1) * 8, s));
  const unsigned gl = (unsigned)ceil_div(n_loc, 256);
  fuzzy_own_end_kernel<<<gl, 256, 0, s>>>(w_all, k, r0, n_loc, indptr, own_end);
  SCB_LAUNCH_CHECK();
  fuzzy_fill_own_kernel<<<gl, 256, 0, s>>>(idx_all, w_all, k, r0, n_loc, indptr, cols, vals);
  SCB_LAUNCH_CHECK();
  fuzzy_fill_in_kernel<<<(unsigned)ceil_div(n_all * k, 256), 256, 0, s>>>(idx_all, w_all, n_all, k, r0, r1,
                                                                                   indptr, own_end, cursor, cols, vals);
  SCB_LAUNCH_CHECK();
  return sort_rows(ctx, indptr, n_loc, cols, vals, s);
}

extern "C" int scb_knn_distances_csr(scb_ctx* ctx, const int32_t* knn_idx, const float* knn_dist, int64_t n_rows,
                                     int32_t k, int64_t* indptr, int32_t* cols, float* vals, void* stream) {
  SCB_REQUIRE(ctx && knn_idx && knn_dist && indptr && cols && vals, SCB_ERR_ARG, "scb_knn_distances_csr: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8, &ws, s));
  int64_t* len = (int64_t*)ws;
  if (n_rows > 0) {
    knn_dist_len_kernel<<<(unsigned)ceil_div(n_rows, 256), 256, 0, s>>>(knn_dist, n_rows, k, len);
    SCB_LAUNCH_CHECK();
  }
  SCB_TRY(scan_i64(ctx, len, n_rows, indptr, s));
  if (n_rows == 0) return SCB_OK;
  knn_dist_fill_kernel<<<(unsigned)ceil_div(n_rows, 256), 256, 0, s>>>(knn_idx, knn_dist, n_rows, k, indptr,
                                                                                 cols, vals);
  SCB_LAUNCH_CHECK();
  return sort_rows(ctx, indptr, n_rows, cols, vals, s);
}

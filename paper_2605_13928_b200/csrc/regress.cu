// sc.pp.regress_out(adata, ["total_counts", "pct_counts_mt"]) on the HVG matrix, fused with
// sc.pp.scale (paper Table 1 step 4, marker label "regress").
//
// Per HVG gene g the log values l_g (dense over the kept cells, zeros included) are fitted by
// ordinary least squares on [1, total_counts, pct_counts_mt] and replaced by the residuals,
// which are then scaled to unit variance and clipped.  OLS residuals are invariant under an
// affine reparametrisation of the covariates, so the design used here is the standardised
// one, a1 = (tc - m1)/s1, a2 = (pct - m2)/s2 (population mean/std over the kept cells, from
// six float64 sums that the multi-GPU path all-reduces): its normal matrix is analytically
// [[N, 0, 0], [0, N, c], [0, c, N]] with c = sum(a1 a2), i.e. perfectly conditioned.
//
// Passes (HBM-bound; the dense matrix is N x ld float32):
//   cov_sums   one CTA, fixed-order fp64 reduction of (n, Σtc, Σtc², Σpct, Σpct², Σtc·pct)
//   design     a1, a2 per kept cell (float64)
//   xty        Σ l, Σ a1 l, Σ a2 l, Σ l² per gene: per-CTA fp64 column partials over row
//              blocks (deterministic), reduced in a fixed order            -- reads 4·N·ld B
//   finalize   beta = G^-1 (Aᵀl), rss = Σl² - betaᵀ(Aᵀl), inv_std = 1/sqrt(rss/(N-1))
//   apply      z = clip((l - beta0 - a1 beta1 - a2 beta2) * inv_std, min_value, max_value) in place (fp32)
//                                                                         -- 8·N·ld B
// The residual mean is zero by construction (intercept), so scale's centring is the
// identity here; the oracle (oracle/pipeline.py: regress_out_scale) uses the same
// definitions and is cross-checked against numpy lstsq residuals in tests/test_oracle.py.
#include "common.cuh"
#include "scan.cuh"

namespace scb {

constexpr int kCovThreads = 1024;
constexpr int kXtyThreads = 512;  // 4 columns per thread -> 2048 columns per CTA pass

// CTA b reduces rows b, b + grid, ... into partial[b][6] (fixed order); a one-warp kernel sums
// the partials in CTA order -> deterministic
__global__ void __launch_bounds__(kCovThreads)
regress_cov_sums_kernel(const double* __restrict__ total, const double* __restrict__ pct,
                        const uint8_t* __restrict__ cmask, int64_t n_rows, double* __restrict__ partial) {
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (!cmask[r]) continue;
    const double t = total[r], p = pct[r];
    acc[0] += 1.0;
    acc[1] += t;
    acc[2] = fma(t, t, acc[2]);
    acc[3] += p;
    acc[4] = fma(p, p, acc[4]);
    acc[5] = fma(t, p, acc[5]);
  }
  __shared__ double red[kCovThreads / 32][6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane_id() == 0) red[warp_id()][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w][threadIdx.x];
    partial[blockIdx.x * 6 + threadIdx.x] = v;
  }
}

__global__ void regress_cov_reduce(const double* __restrict__ partial, int n_parts, double* __restrict__ out) {
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int b = 0; b < n_parts; ++b) v += partial[b * 6 + threadIdx.x];
    out[threadIdx.x] = v;
  }
}

struct CovStd {
  double n, m1, s1, m2, s2, c;
};
// population mean/std of both covariates (std 0 -> 1) and c = Σ a1 a2 from the six sums
__device__ __forceinline__ CovStd cov_std(const double* __restrict__ s6) {
  CovStd r;
  r.n = s6[0];
  r.m1 = s6[1] / r.n;
  r.m2 = s6[3] / r.n;
  const double v1 = fmax(s6[2] / r.n - r.m1 * r.m1, 0.0);
  const double v2 = fmax(s6[4] / r.n - r.m2 * r.m2, 0.0);
  r.s1 = v1 > 0.0 ? sqrt(v1) : 1.0;
  r.s2 = v2 > 0.0 ? sqrt(v2) : 1.0;
  r.c = (s6[5] - r.n * r.m1 * r.m2) / (r.s1 * r.s2);
  return r;
}

__global__ void regress_design_kernel(const double* __restrict__ total, const double* __restrict__ pct,
                                      const uint8_t* __restrict__ cmask, const int64_t* __restrict__ row_pos,
                                      int64_t n_rows, const double* __restrict__ s6, int64_t n_kept,
                                      double* __restrict__ a) {
  const CovStd cs = cov_std(s6);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (!cmask[r]) continue;
    const int64_t k = row_pos[r];
    a[k] = (total[r] - cs.m1) / cs.s1;
    a[n_kept + k] = (pct[r] - cs.m2) / cs.s2;
  }
}

// CTA b owns rows [b*rpb, (b+1)*rpb); thread t owns columns 4t..4t+3 of every 2048-column
// panel; partial[b][stat][col] in fp64 (stat: Σl, Σa1 l, Σa2 l, Σl²).
__global__ void __launch_bounds__(kXtyThreads, 2)
regress_xty_kernel(const float* __restrict__ L, int64_t n_rows, int64_t ld, int32_t H,
                   const double* __restrict__ a, int64_t rpb, double* __restrict__ partial) {
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = min(n_rows, r0 + rpb);
  const double* a1 = a;
  const double* a2 = a + n_rows;
  double* out = partial + (size_t)blockIdx.x * 4 * H;
  for (int c0 = 4 * threadIdx.x; c0 < H; c0 += 4 * blockDim.x) {
    double s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
    auto acc = [&](const float4& v, double x1, double x2) {
      const double l[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        s0[k] += l[k];
        s1[k] = fma(x1, l[k], s1[k]);
        s2[k] = fma(x2, l[k], s2[k]);
        q[k] = fma(l[k], l[k], q[k]);
      }
    };
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {  // four rows' loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(L + (r + u) * ld + c0));
#pragma unroll
      for (int u = 0; u < 4; ++u) acc(v[u], __ldg(a1 + r + u), __ldg(a2 + r + u));
    }
    for (; r < r1; ++r) acc(__ldcs(reinterpret_cast<const float4*>(L + r * ld + c0)), __ldg(a1 + r), __ldg(a2 + r));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = c0 + k;
      if (c < H) {
        out[c] = s0[k];
        out[H + c] = s1[k];
        out[2 * H + c] = s2[k];
        out[3 * H + c] = q[k];
      }
    }
  }
}

// xty[stat][g] += sum over CTAs (fixed order)
__global__ void regress_xty_reduce(const double* __restrict__ partial, int n_blocks, int32_t H,
                                   double* __restrict__ xty) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * H) return;
  double v = 0.0;
  for (int b = 0; b < n_blocks; ++b) v += partial[(size_t)b * 4 * H + i];
  xty[i] += v;
}

__global__ void regress_finalize_kernel(const double* __restrict__ xty, const double* __restrict__ s6, int32_t H,
                                        double* __restrict__ beta, double* __restrict__ inv_std) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= H) return;
  const CovStd cs = cov_std(s6);
  const double n = cs.n;
  const double S0 = xty[g], S1 = xty[H + g], S2 = xty[2 * H + g], Q = xty[3 * H + g];
  const double b0 = S0 / n;
  const double det = n * n - cs.c * cs.c;
  double b1 = 0.0, b2 = 0.0;
  if (det > 1e-12 * n * n) {
    b1 = (n * S1 - cs.c * S2) / det;
    b2 = (n * S2 - cs.c * S1) / det;
  } else {  // collinear covariates: regress on a1 only
    b1 = S1 / n;
  }
  const double rss = Q - (b0 * S0 + b1 * S1 + b2 * S2);
  const double var = rss / (n - 1.0);
  double sd = var > 0.0 ? sqrt(var) : 0.0;
  if (sd == 0.0 || isnan(sd)) sd = 1.0;
  beta[g] = b0;
  beta[H + g] = b1;
  beta[2 * H + g] = b2;
  inv_std[g] = 1.0 / sd;
}

// in place over columns [0, H) of every row: z = clip((l - b0 - a1 b1 - a2 b2) * inv, min, max).
// Thread j of a CTA owns float4 column group j (+ k * blockDim) and keeps its 4 columns'
// (b0, b1, b2, inv) in registers (fp32: the fit is O(l), its rounding is ~1e-7 of l); CTAs
// stride over rows, four rows' loads in flight per thread.
constexpr int kApplyThreads = 512;
__global__ void __launch_bounds__(kApplyThreads)
regress_apply_kernel(float* __restrict__ Z, int64_t n_rows, int64_t ld, int32_t H, const double* __restrict__ a,
                     const double* __restrict__ beta, const double* __restrict__ inv_std, double max_value,
                     double min_value) {
  const int h4 = (H + 3) >> 2;
  const float mx = (float)fmin(max_value, 3.0e38);
  const float mn = (float)fmax(min_value, -3.0e38);
  for (int j = threadIdx.x; j < h4; j += blockDim.x) {
    const int c0 = 4 * j;
    float b0[4], b1[4], b2[4], iv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = min(c0 + k, H - 1);
      b0[k] = (float)beta[c];
      b1[k] = (float)beta[H + c];
      b2[k] = (float)beta[2 * H + c];
      iv[k] = (float)inv_std[c];
    }
    const int nk = min(4, H - c0);
    auto fix = [&](float4& v, float x1, float x2) {
      float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float fit = fmaf(x2, b2[k], fmaf(x1, b1[k], b0[k]));
        if (k < nk) o[k] = fmaxf(fminf((o[k] - fit) * iv[k], mx), mn);
      }
      v.x = o[0]; v.y = o[1]; v.z = o[2]; v.w = o[3];
    };
    int64_t r = blockIdx.x;
    const int64_t step = gridDim.x;
    for (; r + 3 * step < n_rows; r += 4 * step) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(Z + (r + u * step) * ld + c0));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + u * step;
        fix(v[u], (float)__ldg(a + rr), (float)__ldg(a + n_rows + rr));
        __stcs(reinterpret_cast<float4*>(Z + rr * ld + c0), v[u]);
      }
    }
    for (; r < n_rows; r += step) {
      float4 v = __ldcs(reinterpret_cast<const float4*>(Z + r * ld + c0));
      fix(v, (float)__ldg(a + r), (float)__ldg(a + n_rows + r));
      __stcs(reinterpret_cast<float4*>(Z + r * ld + c0), v);
    }
  }
}

}  // namespace scb

using namespace scb;

extern "C" int scb_regress_cov_sums(scb_ctx* ctx, const double* total_counts, const double* pct_counts_mt,
                                    const uint8_t* cell_mask, int64_t n_rows, double* sums6, void* stream) {
  SCB_REQUIRE(ctx && total_counts && pct_counts_mt && cell_mask && sums6, SCB_ERR_ARG,
              "scb_regress_cov_sums: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int parts = ctx->num_sms;
  void* ws;
  SCB_TRY(ws_get(ctx, 0, (size_t)parts * 6 * sizeof(double), &ws, s));
  regress_cov_sums_kernel<<<parts, kCovThreads, 0, s>>>(total_counts, pct_counts_mt, cell_mask, n_rows, (double*)ws);
  SCB_LAUNCH_CHECK();
  regress_cov_reduce<<<1, 32, 0, s>>>((const double*)ws, parts, sums6);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_regress_design(scb_ctx* ctx, const double* total_counts, const double* pct_counts_mt,
                                  const uint8_t* cell_mask, int64_t n_rows, const double* sums6, int64_t n_kept,
                                  double* design, void* stream) {
  SCB_REQUIRE(ctx && total_counts && pct_counts_mt && cell_mask && sums6 && design, SCB_ERR_ARG,
              "scb_regress_design: null argument");
  if (n_rows == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8, &ws, s));
  int64_t* row_pos = (int64_t*)ws;
  SCB_TRY(scan_u8_to_i64(ctx, cell_mask, n_rows, row_pos, s));
  regress_design_kernel<<<ctx->num_sms * 4, 256, 0, s>>>(total_counts, pct_counts_mt, cell_mask, row_pos, n_rows,
                                                        sums6, n_kept, design);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_regress_xty(scb_ctx* ctx, const float* L, int64_t n_rows, int64_t ld, int32_t H,
                               const double* design, double* xty, void* stream) {
  SCB_REQUIRE(ctx && L && design && xty, SCB_ERR_ARG, "scb_regress_xty: null argument");
  SCB_REQUIRE(ld % 4 == 0 && H <= ld && ((uintptr_t)L & 15) == 0, SCB_ERR_ARG,
              "scb_regress_xty: ld % 4 == 0, H <= ld, 16-byte aligned L required");
  if (n_rows == 0 || H == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t target = (int64_t)ctx->num_sms * 2;
  const int64_t rpb = std::max<int64_t>(64, (n_rows + target - 1) / target);
  const int n_blocks = (int)((n_rows + rpb - 1) / rpb);
  void* ws;
  SCB_TRY(ws_get(ctx, 0, (size_t)n_blocks * 4 * H * sizeof(double), &ws, s));
  double* partial = (double*)ws;
  regress_xty_kernel<<<n_blocks, kXtyThreads, 0, s>>>(L, n_rows, ld, H, design, rpb, partial);
  SCB_LAUNCH_CHECK();
  regress_xty_reduce<<<ceil_div(4 * H, 256), 256, 0, s>>>(partial, n_blocks, H, xty);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_regress_finalize(scb_ctx* ctx, const double* xty, const double* sums6, int32_t H, double* beta,
                                    double* inv_std, void* stream) {
  SCB_REQUIRE(ctx && xty && sums6 && beta && inv_std, SCB_ERR_ARG, "scb_regress_finalize: null argument");
  if (H == 0) return SCB_OK;
  regress_finalize_kernel<<<ceil_div(H, 256), 256, 0, (cudaStream_t)stream>>>(xty, sums6, H, beta, inv_std);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_regress_apply(scb_ctx* ctx, float* Z, int64_t n_rows, int64_t ld, int32_t H, const double* design,
                                 const double* beta, const double* inv_std, double max_value, double min_value,
                                 void* stream) {
  SCB_REQUIRE(ctx && Z && design && beta && inv_std, SCB_ERR_ARG, "scb_regress_apply: null argument");
  SCB_REQUIRE(ld % 4 == 0 && H <= ld && ((uintptr_t)Z & 15) == 0, SCB_ERR_ARG,
              "scb_regress_apply: ld % 4 == 0, H <= ld, 16-byte aligned Z required");
  if (n_rows == 0 || H == 0) return SCB_OK;
  regress_apply_kernel<<<ctx->num_sms * 4, kApplyThreads, 0, (cudaStream_t)stream>>>(Z, n_rows, ld, H, design, beta,
                                                                                   inv_std, max_value, min_value);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

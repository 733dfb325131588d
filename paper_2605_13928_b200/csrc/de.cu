// sc.tl.rank_genes_groups(groupby=<clusters>, method="t-test", reference="rest") on the
// log-normalized kept matrix (paper Table 1 step 9, differential expression).
//
//   group rows   counting sort of the cells by group label (row lists per group)
//   sums         per (group, gene) fixed-point Σl and Σl² (the scale step's integers:
//                rn(l 2^28), rn((l 2^12)^2)), carry-free 22-bit split in shared memory over
//                <= 1024-row blocks of one group x one gene tile, flushed into u64 limbs -- exact,
//                so the rest-of-cells sums are exact differences of integers
//   statistics   Welch t-test exactly as scipy.stats.ttest_ind_from_stats(equal_var=False)
//                (which Scanpy calls): vn = var/n (ddof 1), df Welch-Satterthwaite (NaN -> 1),
//                t = (m_g - m_r)/sqrt(vn_g + vn_r) (NaN -> 0), p = I_{df/(df+t^2)}(df/2, 1/2)
//                (regularised incomplete beta by Lentz's continued fraction, NaN -> 1);
//                logfoldchange = log2((expm1(m_g) + 1e-9)/(expm1(m_r) + 1e-9))
//   ranking      per group: genes by decreasing score (ties: smaller gene index) and
//                Benjamini-Hochberg adjusted p-values, via CUB segmented radix sorts.
#include <cub/device/device_segmented_radix_sort.cuh>
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "scan.cuh"

namespace scb {

constexpr int kDeThreads = 512;
constexpr int kDeTileW = (int)(200 * 1024 / 16);  // genes per tile (4 u32 words each)

__global__ void de_hist_kernel(const int32_t* __restrict__ lab, int64_t n, unsigned long long* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[lab[i]], 1ull);
}

__global__ void de_scatter_kernel(const int32_t* __restrict__ lab, int64_t n, const int64_t* __restrict__ off,
                                  unsigned long long* __restrict__ cur, int64_t* __restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rows[off[lab[i]] + (int64_t)atomicAdd(&cur[lab[i]], 1ull)] = i;
}

__device__ __forceinline__ void de_red(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// CTA = (gene tile, group, block of <= 1024 of the group's rows)
__global__ void __launch_bounds__(kDeThreads)
de_sums_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
               const float* __restrict__ ldata, int32_t n_cols, const int64_t* __restrict__ rows,
               const int64_t* __restrict__ goff, const int2* __restrict__ work, int32_t n_groups,
               unsigned long long* __restrict__ sums) {
  extern __shared__ uint32_t sm[];
  const int2 wk = work[blockIdx.x];  // (group, row block)
  const int tile = blockIdx.y;
  const int g = wk.x;
  const int g0 = tile * kDeTileW;
  const int w = min(kDeTileW, n_cols - g0);
  for (int i = threadIdx.x; i < 4 * kDeTileW; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t a1lo = a0, a1hi = a0 + 4u * kDeTileW, a2lo = a0 + 8u * kDeTileW, a2hi = a0 + 12u * kDeTileW;
  const int64_t r0 = goff[g] + (int64_t)wk.y * 1024;
  const int64_t r1 = min(goff[g + 1], r0 + 1024);
  for (int64_t rr = r0 + warp_id(); rr < r1; rr += (blockDim.x >> 5)) {
    const int64_t r = rows[rr];
    const int64_t b = indptr[r], e = indptr[r + 1];
    for (int64_t p = b + lane_id(); p < e; p += 32) {
      const int gl = indices[p] - g0;
      if (gl < 0 || gl >= w) continue;
      const float l = ldata[p];
      const uint64_t v1 = (uint64_t)__float2ull_rn(__fmul_rn(l, 268435456.0f));
      const double l12 = (double)__fmul_rn(l, 4096.0f);
      const uint64_t v2 = (uint64_t)__double2ull_rn(__dmul_rn(l12, l12));
      const uint32_t ga = 4u * (uint32_t)gl;
      if ((v1 | v2) < (1ull << 43)) {
        de_red(a1lo + ga, (uint32_t)(v1 & 0x3FFFFFu));
        de_red(a1hi + ga, (uint32_t)(v1 >> 22));
        de_red(a2lo + ga, (uint32_t)(v2 & 0x3FFFFFu));
        de_red(a2hi + ga, (uint32_t)(v2 >> 22));
      } else {  // rare (not log data): straight into the global limbs
        unsigned long long* base = sums + (size_t)g * 4 * n_cols;
        atomicAdd(&base[g0 + gl], v1 & 0xFFFFFFFFull);
        atomicAdd(&base[n_cols + g0 + gl], v1 >> 32);
        atomicAdd(&base[2 * n_cols + g0 + gl], v2 & 0xFFFFFFFFull);
        atomicAdd(&base[3 * n_cols + g0 + gl], v2 >> 32);
      }
    }
  }
  __syncthreads();
  unsigned long long* base = sums + (size_t)g * 4 * n_cols;
  const uint32_t* s1lo = sm;
  const uint32_t* s1hi = sm + kDeTileW;
  const uint32_t* s2lo = sm + 2 * kDeTileW;
  const uint32_t* s2hi = sm + 3 * kDeTileW;
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    const unsigned long long x0 = (unsigned long long)s1lo[i] + ((unsigned long long)(s1hi[i] & 1023u) << 22);
    const unsigned long long y0 = (unsigned long long)s2lo[i] + ((unsigned long long)(s2hi[i] & 1023u) << 22);
    if (x0) atomicAdd(&base[g0 + i], x0);
    if (s1hi[i] >> 10) atomicAdd(&base[n_cols + g0 + i], (unsigned long long)(s1hi[i] >> 10));
    if (y0) atomicAdd(&base[2 * n_cols + g0 + i], y0);
    if (s2hi[i] >> 10) atomicAdd(&base[3 * n_cols + g0 + i], (unsigned long long)(s2hi[i] >> 10));
  }
}

// exact 128-bit sum -> double: one rounding when it fits 64 bits (as limbs_to_double and the
// oracle's fx_to_double)
__device__ __forceinline__ double u128_to_double(unsigned __int128 v) {
  const unsigned long long hi = (unsigned long long)(v >> 64), lo = (unsigned long long)v;
  if (hi == 0ull) return __ull2double_rn(lo);
  return __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

// regularised incomplete beta I_x(a, b) (continued fraction, Numerical Recipes' betacf)
__device__ double betacf(double a, double b, double x) {
  const double FPMIN = 1e-300, EPS = 1e-16;
  double qab = a + b, qap = a + 1.0, qam = a - 1.0, c = 1.0, d = 1.0 - qab * x / qap;
  if (fabs(d) < FPMIN) d = FPMIN;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 10000; ++m) {
    const int m2 = 2 * m;
    double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < FPMIN) d = FPMIN;
    c = 1.0 + aa / c;
    if (fabs(c) < FPMIN) c = FPMIN;
    d = 1.0 / d;
    h *= d * c;
    aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < FPMIN) d = FPMIN;
    c = 1.0 + aa / c;
    if (fabs(c) < FPMIN) c = FPMIN;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (fabs(del - 1.0) < EPS) break;
  }
  return h;
}
__device__ double ibeta(double a, double b, double x) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double lbt = lgamma(a + b) - lgamma(a) - lgamma(b) + a * log(x) + b * log1p(-x);
  if (x < (a + 1.0) / (a + b + 2.0)) return exp(lbt) * betacf(a, b, x) / a;
  return 1.0 - exp(lbt) * betacf(b, a, 1.0 - x) / b;
}

__device__ __forceinline__ uint64_t desc_key(double v) {  // ascending order of the key = descending v
  uint64_t u = (uint64_t)__double_as_longlong(v);
  u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  return ~u;
}
__device__ __forceinline__ uint64_t asc_key(double v) {
  uint64_t u = (uint64_t)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void de_stats_kernel(const unsigned long long* __restrict__ sums, int32_t n_groups, int32_t G,
                                const int64_t* __restrict__ goff, double* __restrict__ score,
                                double* __restrict__ lfc, double* __restrict__ pval, uint64_t* __restrict__ skey,
                                uint64_t* __restrict__ pkey, int32_t* __restrict__ gidx) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_groups * G) return;
  const int g = (int)(t / G), j = (int)(t % G);
  unsigned long long T[4] = {0, 0, 0, 0};
  for (int q = 0; q < n_groups; ++q)
    for (int s = 0; s < 4; ++s) T[s] += sums[((size_t)q * 4 + s) * G + j];
  const unsigned long long* S = sums + (size_t)g * 4 * G;
  unsigned long long A[4] = {S[j], S[G + j], S[2 * G + j], S[3 * G + j]};
  const double n_all = (double)goff[n_groups];
  const double n1 = (double)(goff[g + 1] - goff[g]), n2 = n_all - n1;
  // rest = total - group, exactly (128-bit integers of the limb pairs)
  const unsigned __int128 tg1 = (unsigned __int128)A[0] + ((unsigned __int128)A[1] << 32);
  const unsigned __int128 tg2 = (unsigned __int128)A[2] + ((unsigned __int128)A[3] << 32);
  const unsigned __int128 tt1 = (unsigned __int128)T[0] + ((unsigned __int128)T[1] << 32);
  const unsigned __int128 tt2 = (unsigned __int128)T[2] + ((unsigned __int128)T[3] << 32);
  const double s1g = u128_to_double(tg1) * 3.725290298461914e-09;  // 2^-28
  const double s2g = u128_to_double(tg2) * 5.960464477539063e-08;  // 2^-24
  const double s1r = u128_to_double(tt1 - tg1) * 3.725290298461914e-09;
  const double s2r = u128_to_double(tt2 - tg2) * 5.960464477539063e-08;
  // explicit _rn operations (no FMA contraction) so numpy reproduces every rounding
  const double m1 = __ddiv_rn(s1g, n1), m2 = __ddiv_rn(s1r, n2);
  const double v1 = __dmul_rn(__dsub_rn(__ddiv_rn(s2g, n1), __dmul_rn(m1, m1)), __ddiv_rn(n1, __dsub_rn(n1, 1.0)));
  const double v2 = __dmul_rn(__dsub_rn(__ddiv_rn(s2r, n2), __dmul_rn(m2, m2)), __ddiv_rn(n2, __dsub_rn(n2, 1.0)));
  const double vn1 = __ddiv_rn(v1, n1), vn2 = __ddiv_rn(v2, n2);
  const double vs = __dadd_rn(vn1, vn2);
  double df = __ddiv_rn(__dmul_rn(vs, vs), __dadd_rn(__ddiv_rn(__dmul_rn(vn1, vn1), __dsub_rn(n1, 1.0)),
                                                   __ddiv_rn(__dmul_rn(vn2, vn2), __dsub_rn(n2, 1.0))));
  if (isnan(df)) df = 1.0;
  double tt = __ddiv_rn(__dsub_rn(m1, m2), __dsqrt_rn(vs));
  double p;
  if (isnan(tt)) {
    tt = 0.0;
    p = 1.0;
  } else {
    p = ibeta(0.5 * df, 0.5, df / (df + tt * tt));  // two-sided: 2 * t.sf(|t|, df)
    if (isnan(p)) p = 1.0;
  }
  score[t] = tt;
  pval[t] = p;
  lfc[t] = log2((expm1(m1) + 1e-9) / (expm1(m2) + 1e-9));
  skey[t] = desc_key(tt);
  pkey[t] = asc_key(p);
  gidx[t] = j;
}

// BH: for the p-values of one group in ascending order (sorted index list), adjusted
// q_i = min_{k >= i} p_(k) * G / k, clipped at 1 (statsmodels fdr_bh) -- one CTA per group,
// suffix minimum by a sequential pass over chunks
__global__ void de_bh_kernel(const double* __restrict__ pval, const int32_t* __restrict__ porder, int32_t G,
                             double* __restrict__ padj) {
  const int g = blockIdx.x;
  const double* p = pval + (size_t)g * G;
  const int32_t* o = porder + (size_t)g * G;
  double* q = padj + (size_t)g * G;
  if (threadIdx.x == 0) {
    double run = 1.0;
    for (int i = G - 1; i >= 0; --i) {
      const double v = fmin(run, p[o[i]] * (double)G / (double)(i + 1));
      run = v;
      q[o[i]] = fmin(v, 1.0);
    }
  }
}

}  // namespace scb

using namespace scb;

namespace {
struct DeBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DeBuf() { if (p) cudaFreeAsync(p, s); }
};
}  // namespace
#define DE_ALLOC(buf, bytes)                                                          \
  do {                                                                                \
    buf.s = s;                                                                        \
    SCB_CUDA(cudaMallocAsync(&buf.p, std::max<size_t>((size_t)(bytes), 16), s));     \
  } while (0)

extern "C" int scb_rank_genes_groups(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* ldata,
                                     int64_t n_rows, int32_t n_cols, const int32_t* labels, int32_t n_groups,
                                     double* scores, double* logfc, double* pvals, double* pvals_adj,
                                     int32_t* order, void* stream) {
  SCB_REQUIRE(ctx && indptr && indices && ldata && labels && scores && logfc && pvals && pvals_adj && order,
              SCB_ERR_ARG, "scb_rank_genes_groups: null argument");
  SCB_REQUIRE(n_groups >= 2 && n_rows > n_groups && n_cols > 0, SCB_ERR_ARG,
              "scb_rank_genes_groups: need >= 2 groups and more cells than groups");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = ctx->num_sms * 8;
  DeBuf cnt, off, cur, rows, sums, skey, pkey, gidx, sk2, si2, pk2, pi2, segs, tmp;
  DE_ALLOC(cnt, (n_groups + 1) * 8);
  DE_ALLOC(off, (n_groups + 1) * 8);
  DE_ALLOC(cur, (n_groups + 1) * 8);
  DE_ALLOC(rows, n_rows * 8);
  SCB_CUDA(cudaMemsetAsync(cnt.p, 0, (n_groups + 1) * 8, s));
  SCB_CUDA(cudaMemsetAsync(cur.p, 0, (n_groups + 1) * 8, s));
  de_hist_kernel<<<grid, 256, 0, s>>>(labels, n_rows, (unsigned long long*)cnt.p);
  SCB_LAUNCH_CHECK();
  SCB_TRY(scan_i64(ctx, (const int64_t*)cnt.p, n_groups, (int64_t*)off.p, s));
  de_scatter_kernel<<<grid, 256, 0, s>>>(labels, n_rows, (const int64_t*)off.p, (unsigned long long*)cur.p,
                                        (int64_t*)rows.p);
  SCB_LAUNCH_CHECK();
  std::vector<int64_t> h_off(n_groups + 1);
  SCB_CUDA(cudaMemcpyAsync(h_off.data(), off.p, (n_groups + 1) * 8, cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  std::vector<int2> h_work;
  for (int g = 0; g < n_groups; ++g) {
    SCB_REQUIRE(h_off[g + 1] - h_off[g] >= 2, SCB_ERR_DATA, "scb_rank_genes_groups: group %d has < 2 cells", g);
    for (int64_t b = 0; b * 1024 < h_off[g + 1] - h_off[g]; ++b) h_work.push_back(make_int2(g, (int)b));
  }
  DeBuf work;
  DE_ALLOC(work, h_work.size() * sizeof(int2));
  SCB_CUDA(cudaMemcpyAsync(work.p, h_work.data(), h_work.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  const size_t G = (size_t)n_cols, K = (size_t)n_groups;
  DE_ALLOC(sums, K * 4 * G * 8);
  SCB_CUDA(cudaMemsetAsync(sums.p, 0, K * 4 * G * 8, s));
  const int n_tiles = (n_cols + kDeTileW - 1) / kDeTileW;
  const size_t smem = (size_t)kDeTileW * 16;
  SCB_CUDA(cudaFuncSetAttribute(de_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  de_sums_kernel<<<dim3((unsigned)h_work.size(), n_tiles), kDeThreads, smem, s>>>(
      indptr, indices, ldata, n_cols, (const int64_t*)rows.p, (const int64_t*)off.p, (const int2*)work.p, n_groups,
      (unsigned long long*)sums.p);
  SCB_LAUNCH_CHECK();
  const size_t KG = K * G;
  DE_ALLOC(skey, KG * 8);
  DE_ALLOC(pkey, KG * 8);
  DE_ALLOC(gidx, KG * 4);
  de_stats_kernel<<<(unsigned)((KG + 255) / 256), 256, 0, s>>>((const unsigned long long*)sums.p, n_groups, n_cols,
                                                              (const int64_t*)off.p, scores, logfc, pvals,
                                                              (uint64_t*)skey.p, (uint64_t*)pkey.p,
                                                              (int32_t*)gidx.p);
  SCB_LAUNCH_CHECK();
  // per-group sorts: by descending score (ties: gene index, the stable payload order) and by p
  std::vector<int> h_segs(K + 1);
  for (size_t g = 0; g <= K; ++g) h_segs[g] = (int)(g * G);
  DE_ALLOC(segs, (K + 1) * 4);
  SCB_CUDA(cudaMemcpyAsync(segs.p, h_segs.data(), (K + 1) * 4, cudaMemcpyHostToDevice, s));
  DE_ALLOC(sk2, KG * 8);
  DE_ALLOC(pk2, KG * 8);
  DE_ALLOC(pi2, KG * 4);
  size_t tb = 0, tb2 = 0;
  SCB_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb, (const uint64_t*)skey.p, (uint64_t*)sk2.p,
                                                    (const int32_t*)gidx.p, order, (int)KG, (int)K,
                                                    (const int*)segs.p, (const int*)segs.p + 1, 0, 64, s));
  SCB_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb2, (const uint64_t*)pkey.p, (uint64_t*)pk2.p,
                                                    (const int32_t*)gidx.p, (int32_t*)pi2.p, (int)KG, (int)K,
                                                    (const int*)segs.p, (const int*)segs.p + 1, 0, 64, s));
  DE_ALLOC(tmp, std::max(tb, tb2));
  SCB_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp.p, tb, (const uint64_t*)skey.p, (uint64_t*)sk2.p,
                                                    (const int32_t*)gidx.p, order, (int)KG, (int)K,
                                                    (const int*)segs.p, (const int*)segs.p + 1, 0, 64, s));
  SCB_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(tmp.p, tb2, (const uint64_t*)pkey.p, (uint64_t*)pk2.p,
                                                    (const int32_t*)gidx.p, (int32_t*)pi2.p, (int)KG, (int)K,
                                                    (const int*)segs.p, (const int*)segs.p + 1, 0, 64, s));
  de_bh_kernel<<<n_groups, 32, 0, s>>>(pvals, (const int32_t*)pi2.p, n_cols, pvals_adj);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaStreamSynchronize(s));
  return SCB_OK;
}

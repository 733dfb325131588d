// Synthetic NB counts on the device (bench/test input synthesis; not on the timed path).
// Generator version 2 -- bit-identical to oracle/synth.py by construction: every per-entry
// quantity uses only correctly rounded fp64 operations in a fixed order (explicit _rn
// intrinsics, so no FMA contraction): the log-mean x = (log_s + log_mu) + (A + sum_r U_r B_r)
// (synth_logmean_kernel), mu = det_exp(x) (Cody-Waite + Taylor-13 + exact ldexp), zero
// probability p0 = sqrt(theta/(theta+mu)) (theta = 1/2), one splitmix64 counter uniform per
// (cell, gene) and the inverse-CDF recurrence for x >= 1.
#include "common.cuh"

namespace scb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr int kStreamCount = 8;  // S_COUNT
constexpr double kTheta = 0.5;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
  const uint64_t s = mix64(seed * 256ull + stream);
  const uint64_t h = mix64(mix64(s + i) + j);
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

// exp(x) from correctly rounded operations only (oracle/synth.py:det_exp)
__device__ __forceinline__ double det_exp(double x) {
  const double k = rint(__dmul_rn(x, 0x1.71547652b82fep+0));
  const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, 0x1.62e42fee00000p-1)), __dmul_rn(k, 0x1.a39ef35793c76p-33));
  constexpr double c[14] = {0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
                            0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
                            0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
                            0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};
  double p = c[13];
#pragma unroll
  for (int i = 12; i >= 0; --i) p = __dadd_rn(__dmul_rn(p, r), c[i]);
  return ldexp(p, (int)k);
}

constexpr int kSynthMaxR = 64;
constexpr int kSynthCells = 32;  // cells per CTA of the log-mean kernel

// x[c][g] = (log_s[c] + log_mu[g]) + L, L = A[type c][g]; L += U[c][r] * B[r][g] (r ascending)
__global__ void __launch_bounds__(128) synth_logmean_kernel(int64_t n_rows, int G, int R, const double* __restrict__ log_mu,
                                                            const double* __restrict__ A, const int* __restrict__ ctype,
                                                            const double* __restrict__ log_s, const double* __restrict__ U,
                                                            const double* __restrict__ B, double* __restrict__ out) {
  __shared__ double su[kSynthCells][kSynthMaxR];
  const int g = blockIdx.x * 128 + threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.y * kSynthCells;
  const int nc = (int)(n_rows - c0 < kSynthCells ? n_rows - c0 : kSynthCells);
  for (int i = threadIdx.x; i < nc * R; i += 128) su[i / R][i % R] = U[(c0 + i / R) * R + i % R];
  __syncthreads();
  if (g >= G) return;
  double b[kSynthMaxR];
#pragma unroll
  for (int r = 0; r < kSynthMaxR; ++r) b[r] = (r < R) ? B[(int64_t)r * G + g] : 0.0;
  const double lm = log_mu[g];
  for (int i = 0; i < nc; ++i) {
    const int64_t c = c0 + i;
    double L = A[(int64_t)ctype[c] * G + g];
#pragma unroll
    for (int r = 0; r < kSynthMaxR; ++r)
      if (r < R) L = __dadd_rn(L, __dmul_rn(su[i][r], b[r]));
    out[c * G + g] = __dadd_rn(__dadd_rn(log_s[c], lm), L);
  }
}

__device__ __forceinline__ int nb_sample(double mu, double u, double p0) {
  // same recurrence as oracle/synth.py:nb_inverse_cdf (explicit _rn: no FMA contraction)
  const double q = __ddiv_rn(mu, __dadd_rn(kTheta, mu));
  double pk = p0, F = p0;
  int k = 0;
  while (F <= u && k < 100000 && pk > 0.0) {
    const double kk = (double)k;
    pk = __dmul_rn(pk, __dmul_rn(__ddiv_rn(__dadd_rn(kk, kTheta), __dadd_rn(kk, 1.0)), q));
    ++k;
    F = __dadd_rn(F, pk);
  }
  return k;
}

__global__ void synth_kernel(uint64_t seed, int64_t row0, int64_t n_rows, int G, const double* __restrict__ logmean,
                             const int64_t* __restrict__ indptr, int64_t* __restrict__ nnz, int* __restrict__ out_i,
                             float* __restrict__ out_v) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (r >= n_rows) return;
  const int l = lane_id();
  const uint64_t c = (uint64_t)(row0 + r);
  const double* xr = logmean + r * G;
  int64_t o = indptr ? indptr[r] : 0;
  int cnt = 0;
  for (int g0 = 0; g0 < G; g0 += 32) {
    const int g = g0 + l;
    bool nz = false;
    double u = 0.0, mu = 0.0, p0 = 0.0;
    if (g < G) {
      mu = det_exp(xr[g]);
      p0 = __dsqrt_rn(__ddiv_rn(kTheta, __dadd_rn(kTheta, mu)));
      u = uniform01(seed, kStreamCount, c, (uint64_t)g);
      nz = u >= p0;
    }
    const unsigned b = __ballot_sync(0xffffffffu, nz);
    if (indptr && nz) {
      const int64_t pos = o + __popc(b & ((1u << l) - 1u));
      out_i[pos] = g;
      out_v[pos] = (float)nb_sample(mu, u, p0);
    }
    o += __popc(b);
    cnt += __popc(b);
  }
  if (!indptr && l == 0) nnz[r] = cnt;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_synth_logmean(scb_ctx* ctx, int64_t n_rows, int32_t n_genes, int32_t n_factors, const double* log_mu,
                                 const double* A, const int32_t* cell_type, const double* log_s, const double* U,
                                 const double* B, double* logmean, void* stream) {
  SCB_REQUIRE(ctx && log_mu && A && cell_type && log_s && U && B && logmean, SCB_ERR_ARG, "scb_synth_logmean: null argument");
  SCB_REQUIRE(n_factors >= 0 && n_factors <= kSynthMaxR, SCB_ERR_ARG, "scb_synth_logmean: n_factors must be <= %d", kSynthMaxR);
  if (n_rows == 0 || n_genes == 0) return SCB_OK;
  const dim3 grid((unsigned)ceil_div(n_genes, 128), (unsigned)ceil_div(n_rows, kSynthCells));
  synth_logmean_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(n_rows, n_genes, n_factors, log_mu, A, cell_type, log_s, U,
                                                              B, logmean);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_synth_rows(scb_ctx* ctx, uint64_t seed, int64_t row0, int64_t n_rows, int32_t n_genes,
                              const double* logmean, const int64_t* indptr, int64_t* row_nnz, int32_t* indices,
                              float* data, void* stream) {
  SCB_REQUIRE(ctx && logmean, SCB_ERR_ARG, "scb_synth_rows: null argument");
  SCB_REQUIRE(indptr ? (indices && data) : (row_nnz != nullptr), SCB_ERR_ARG, "scb_synth_rows: bad pass arguments");
  if (n_rows == 0) return SCB_OK;
  synth_kernel<<<ceil_div(n_rows, 8), 256, 0, (cudaStream_t)stream>>>(seed, row0, n_rows, n_genes, logmean, indptr,
                                                                      row_nnz, indices, data);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

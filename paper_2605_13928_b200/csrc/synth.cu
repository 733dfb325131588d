// Synthetic NB counts on the device (bench/test input synthesis; not on the timed path).
// Follows oracle/synth.py: one splitmix64 counter uniform per (cell, gene), fp64 mean,
// zero probability p0 = (theta/(theta+mu))^theta and inverse-CDF recurrence for x >= 1.
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

__global__ void synth_kernel(uint64_t seed, int64_t row0, int64_t n_rows, int G, const double* __restrict__ log_mu,
                             const double* __restrict__ A, const int* __restrict__ ctype, const double* __restrict__ log_s,
                             const float* __restrict__ Lf, const int64_t* __restrict__ indptr, int64_t* __restrict__ nnz,
                             int* __restrict__ out_i, float* __restrict__ out_v) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (r >= n_rows) return;
  const int l = lane_id();
  const uint64_t c = (uint64_t)(row0 + r);
  const double ls = log_s[r];
  const double* Ar = A + (int64_t)ctype[r] * G;
  const float* Lr = Lf + r * G;
  int64_t o = indptr ? indptr[r] : 0;
  int cnt = 0;
  for (int g0 = 0; g0 < G; g0 += 32) {
    const int g = g0 + l;
    bool nz = false;
    double u = 0.0, mu = 0.0, p0 = 0.0;
    if (g < G) {
      mu = exp(ls + log_mu[g] + Ar[g] + (double)Lr[g]);
      p0 = exp(kTheta * log(__ddiv_rn(kTheta, __dadd_rn(kTheta, mu))));
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

extern "C" int scb_synth_rows(scb_ctx* ctx, uint64_t seed, int64_t row0, int64_t n_rows, int32_t n_genes,
                              const double* log_mu, const double* A, const int32_t* cell_type, const double* log_s,
                              const float* Lf, const int64_t* indptr, int64_t* row_nnz, int32_t* indices, float* data,
                              void* stream) {
  SCB_REQUIRE(ctx && log_mu && A && cell_type && log_s && Lf, SCB_ERR_ARG, "scb_synth_rows: null argument");
  SCB_REQUIRE(indptr ? (indices && data) : (row_nnz != nullptr), SCB_ERR_ARG, "scb_synth_rows: bad pass arguments");
  if (n_rows == 0) return SCB_OK;
  synth_kernel<<<ceil_div(n_rows, 8), 256, 0, (cudaStream_t)stream>>>(seed, row0, n_rows, n_genes, log_mu, A, cell_type,
                                                                      log_s, Lf, indptr, row_nnz, indices, data);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

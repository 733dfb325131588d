// Top-k eigenpairs of the (small, dense) PCA covariance, on the device, in float64.
//
// Cov = (C[:h,:h] - N m m^T)/(N-1) with m = C[ones_col, :h]/N (column means of Z, exposed
// by the ones column of the scaled matrix).  Block subspace iteration with block size
// b = 96 (>= n_comps + oversampling): Y = Cov^q Q, Cholesky-QR (twice), repeated; then
// Rayleigh-Ritz T = Q^T Cov Q solved by a one-CTA cyclic Jacobi, and V = Q W.  The
// residual max_j ||Cov v_j - l_j v_j|| / l_1 is checked on the device and iterations
// continue until it falls below 1e-10 (or an iteration cap).  Sign rule: the
// largest-|loading| entry of every component is positive (first index on ties).
#include <cstdlib>
#include "common.cuh"

namespace scb {

constexpr int kB = 96;   // subspace block size (n_comps + oversampling)
constexpr int kLd = kB + 1;

// ------------------------------------------------------------------ small fp64 GEMM
// Cm[M][N] (ldc) = op(A) * op(B), row-major operands, fp64 on the FP64 tensor path (DMMA; the
// eigensolver's GEMMs are 2000 x 96 x 2000 at most, ~0.8 GFLOP each).  opA: 0 -> A[M][K] (lda),
// 1 -> A^T with A stored [K][M]; opB: 0 -> B[K][N] (ldb), 1 -> B^T with B stored [N][K].  64x64
// tiles, K chunk 16.  Split-K over blockIdx.z writes per-slice partials
// that a second kernel sums in slice order (deterministic).  Every kernel of the eigensolver
// takes the device `done` flag and exits at once when it is set, so the host can enqueue a
// batch of outer iterations without a round trip per iteration.
constexpr int kGT = 64, kGK = 32;
// DMMA (mma.sync m8n8k4 f64) tile GEMM: CTA 64x64 of C, 4 warps of 32x32 (4x4 MMA tiles of 8x8),
// K staged through shared memory 32 at a time with the next chunk's global loads issued into
// registers before the current chunk's MMAs.  Fragments (m8n8k4, row.col): lane = 4 g + t;
// A[g][t], B[t][g], C[g][2t .. 2t+1].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// CTA tile TM x TN, WARPS_M x WARPS_N warps of (TM/WARPS_M) x (TN/WARPS_N) (MI x NJ MMA tiles)
template <int TM, int TN, int WARPS_M, int WARPS_N, int MIN_CTAS>
__global__ void __launch_bounds__(128, MIN_CTAS) dgemm_kernel(int M, int N, int K, const double* __restrict__ A, int lda,
                                                    int opA, const double* __restrict__ B, int ldb, int opB,
                                                    double* __restrict__ Cm, int ldc, int k_per_slice,
                                                    double* __restrict__ partial, const int* __restrict__ done) {
  static_assert(WARPS_M * WARPS_N == 4, "4 warps");
  constexpr int WTM = TM / WARPS_M, WTN = TN / WARPS_N, MI = WTM / 8, NJ = WTN / 8;
  constexpr int LA = kGK * TM / 128, LB = kGK * TN / 128;  // elements of A / B per thread per chunk
  if (done && *done) return;
  __shared__ double As[TM][kGK + 1];   // [m][k]
  __shared__ double Bs[kGK][TN + 1];   // [k][n]
  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / WARPS_N) * WTM, wn = (warp % WARPS_N) * WTN;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int kb = blockIdx.z * k_per_slice, ke = min(K, kb + k_per_slice);
  double acc[MI][NJ][2] = {};
  double ra[LA], rb[LB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int e = threadIdx.x + 128 * u;
      int kk, mm;
      if (opA) { kk = e / TM; mm = e % TM; } else { mm = e / kGK; kk = e % kGK; }
      const int gm = m0 + mm, gk = k0 + kk;
      ra[u] = (gm < M && gk < ke) ? (opA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = threadIdx.x + 128 * u;
      int kn, nn;
      if (opB) { nn = e / kGK; kn = e % kGK; } else { kn = e / TN; nn = e % TN; }
      const int gn = n0 + nn, gk2 = k0 + kn;
      rb[u] = (gn < N && gk2 < ke) ? (opB ? B[(size_t)gn * ldb + gk2] : B[(size_t)gk2 * ldb + gn]) : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int e = threadIdx.x + 128 * u;
      if (opA) As[e % TM][e / TM] = ra[u]; else As[e / kGK][e % kGK] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int e = threadIdx.x + 128 * u;
      if (opB) Bs[e % kGK][e / kGK] = rb[u]; else Bs[e / TN][e % TN] = rb[u];
    }
  };
  if (kb < ke) fetch(kb);
  for (int k0 = kb; k0 < ke; k0 += kGK) {
    stash();
    __syncthreads();
    if (k0 + kGK < ke) fetch(k0 + kGK);  // next chunk in flight during this chunk's MMAs
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = As[wm + 8 * i + g][kk + t];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = Bs[kk + t][wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* out = partial ? partial + (size_t)blockIdx.z * M * N : Cm;
  const int ld = partial ? N : ldc;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int m = m0 + wm + 8 * i + g, n = n0 + wn + 8 * j + 2 * t + c;
        if (m < M && n < N) out[(size_t)m * ld + n] = acc[i][j][c];
      }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ partial, int slices, int M, int N,
                                     double* __restrict__ Cm, int ldc, const int* __restrict__ done) {
  if (done && *done) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * N) return;
  double s = 0.0;
  for (int z = 0; z < slices; ++z) s += partial[(size_t)z * M * N + e];
  Cm[(size_t)(e / N) * ldc + e % N] = s;
}

static int dgemm(scb_ctx* ctx, int M, int N, int K, const double* A, int lda, int opA, const double* B, int ldb,
                 int opB, double* Cm, int ldc, cudaStream_t s, const int* done = nullptr) {
  // N = kB (every GEMM of the solver): 32 x 96 tiles, no padded columns; split-K sized so the
  // grid is ~3 CTAs per SM.  Otherwise 64 x 64 tiles, ~1 CTA per SM.
  const bool narrow = (N == 96);
  const int TM = narrow ? 32 : kGT, TN = narrow ? 96 : kGT;
  const int tiles = ((M + TM - 1) / TM) * ((N + TN - 1) / TN);
  const int want = narrow ? 3 * ctx->num_sms : ctx->num_sms;
  int slices = std::max(1, std::min((want + tiles / 2) / tiles, K / 128));
  const int kps = ((K + slices - 1) / slices + kGK - 1) / kGK * kGK;
  slices = (K + kps - 1) / kps;
  double* partial = nullptr;
  if (slices > 1) {
    void* ws;
    SCB_TRY(ws_get(ctx, 3, (size_t)slices * M * N * sizeof(double), &ws, s));
    partial = (double*)ws;
  }
  dim3 g((N + TN - 1) / TN, (M + TM - 1) / TM, slices);
  if (narrow)
    dgemm_kernel<32, 96, 1, 4, 3><<<g, 128, 0, s>>>(M, N, K, A, lda, opA, B, ldb, opB, Cm, ldc, kps, partial, done);
  else
    dgemm_kernel<kGT, kGT, 2, 2, 1><<<g, 128, 0, s>>>(M, N, K, A, lda, opA, B, ldb, opB, Cm, ldc, kps, partial, done);
  SCB_LAUNCH_CHECK();
  if (slices > 1) {
    splitk_reduce_kernel<<<(unsigned)(((int64_t)M * N + 255) / 256), 256, 0, s>>>(partial, slices, M, N, Cm, ldc, done);
    SCB_LAUNCH_CHECK();
  }
  return SCB_OK;
}

// M[h][kB] (row-major) := M R^{-1}, R upper triangular [kB][kB]: each warp solves one row
// x R = m by forward substitution (lane l owns columns l, l+32, l+64), R staged in smem.
__global__ void __launch_bounds__(256) trsm_rows_kernel(const double* __restrict__ R, double* __restrict__ M, int h,
                                                        const int* __restrict__ done) {
  if (done && *done) return;
  extern __shared__ double rdyn[];
  double (*r)[kB + 1] = reinterpret_cast<double (*)[kB + 1]>(rdyn);
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    const int i = e / kB, j = e % kB;
    r[i][j] = (i == j) ? 1.0 / R[e] : R[e];  // diagonal stored as its reciprocal
  }
  __syncthreads();
  const int lane = lane_id();
  for (int row = blockIdx.x * 8 + warp_id(); row < h; row += gridDim.x * 8) {
    double m[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) m[t] = M[(size_t)row * kB + lane + 32 * t];
    for (int j = 0; j < kB; ++j) {
      const int owner = j & 31, slot = j >> 5;
      double mj = 0.0;
#pragma unroll
      for (int t = 0; t < 3; ++t) if (t == slot) mj = m[t];
      const double xj = __shfl_sync(0xffffffffu, mj, owner) * r[j][j];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int c = lane + 32 * t;
        if (c == j) m[t] = xj;
        else if (c > j) m[t] -= xj * r[j][c];
      }
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) M[(size_t)row * kB + lane + 32 * t] = m[t];
  }
}

static int trsm_right_upper(scb_ctx* ctx, int h, const double* R, double* M, cudaStream_t s, const int* done) {
  const int smem = kB * (kB + 1) * 8;
  SCB_CUDA(cudaFuncSetAttribute(trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  trsm_rows_kernel<<<std::max(1, std::min(ctx->num_sms * 2, (h + 7) / 8)), 256, smem, s>>>(R, M, h, done);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

// M[h][kB] (row-major) := an orthonormal basis by classical Gram-Schmidt with
// re-orthogonalisation (CGS2) in one CTA; a column that vanishes (rank deficiency) is replaced
// by a deterministic pseudo-random vector and re-orthogonalised, completing the basis.  Used
// only when Cholesky-QR breaks down (fewer than kB + 1 distinct cells).
constexpr int kOrthThreads = 1024;
__device__ __forceinline__ double hash_unit(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}
__device__ double block_sum(double v, double* sb) {
  v = warp_sum(v);
  __syncthreads();
  if (lane_id() == 0) sb[warp_id()] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sb[w];
  return t;
}
__global__ void __launch_bounds__(kOrthThreads) cgs2_kernel(double* __restrict__ Mq, int h,
                                                            const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double coef[kB];
  __shared__ double sb[32];
  for (int j = 0; j < kB; ++j) {
    for (int attempt = 0; attempt < 4; ++attempt) {
      double n0 = 0.0;
      for (int i = threadIdx.x; i < h; i += blockDim.x) n0 += Mq[(size_t)i * kB + j] * Mq[(size_t)i * kB + j];
      n0 = sqrt(block_sum(n0, sb));
      for (int pass = 0; pass < 2; ++pass) {
        // coef[c] = <q_c, m_j> for c < j: warp w takes columns w, w+32, ...
        for (int c = warp_id(); c < j; c += blockDim.x >> 5) {
          double d = 0.0;
          for (int i = lane_id(); i < h; i += 32) d += Mq[(size_t)i * kB + c] * Mq[(size_t)i * kB + j];
          d = warp_sum(d);
          if (lane_id() == 0) coef[c] = d;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < h; i += blockDim.x) {
          double v = Mq[(size_t)i * kB + j];
          for (int c = 0; c < j; ++c) v -= coef[c] * Mq[(size_t)i * kB + c];
          Mq[(size_t)i * kB + j] = v;
        }
        __syncthreads();
      }
      double nn = 0.0;
      for (int i = threadIdx.x; i < h; i += blockDim.x) nn += Mq[(size_t)i * kB + j] * Mq[(size_t)i * kB + j];
      nn = sqrt(block_sum(nn, sb));
      if (nn > 1e-10 * fmax(n0, 1e-300) && nn > 1e-300) {
        for (int i = threadIdx.x; i < h; i += blockDim.x) Mq[(size_t)i * kB + j] /= nn;
        __syncthreads();
        break;
      }
      for (int i = threadIdx.x; i < h; i += blockDim.x)  // dependent column: restart from a random vector
        Mq[(size_t)i * kB + j] = hash_unit(((uint64_t)(attempt + 1) << 40) ^ ((uint64_t)j << 20) ^ (uint64_t)i);
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ covariance
__global__ void cov_build_kernel(const double* __restrict__ Cg, int hp, int h, int ones_col, int64_t n,
                                 double* __restrict__ cov, double* __restrict__ mean) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= h) return;
  const double N = (double)n;
  const double mi = Cg[(size_t)ones_col * hp + i] / N;
  const double mj = Cg[(size_t)ones_col * hp + j] / N;
  cov[(size_t)i * h + j] = (Cg[(size_t)i * hp + j] - N * mi * mj) / (N - 1.0);
  if (i == 0) mean[j] = mj;
}

__global__ void trace_kernel(const double* __restrict__ cov, int h, double* __restrict__ tr) {
  __shared__ double sb[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < h; i += blockDim.x) s += cov[(size_t)i * h + i];
  s = warp_sum(s);
  if (lane_id() == 0) sb[warp_id()] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sb[w];
    *tr = t;
  }
}

// deterministic start block: Q0[i][j] = hash-based uniform in [-1, 1)
__global__ void init_block_kernel(double* __restrict__ Q, int h) {
  const int i = blockIdx.x, j = threadIdx.x;
  uint64_t z = ((uint64_t)i << 32) ^ (uint64_t)j ^ 0x5DEECE66Dull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  Q[(size_t)i * kB + j] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// ------------------------------------------------------------------ Cholesky QR
// In place Cholesky of the kB x kB Gram S = Q^T Q (one CTA), S -> R (upper, row-major).
// Unscaled right-looking form, one barrier per step: step k subtracts a_ki a_kj / a_kk from the
// trailing upper triangle (row k itself is final); the thread that updates a_{k+1,k+1} also
// stores its reciprocal for the next step.  Rows are scaled by 1/sqrt(pivot) on the way out.
constexpr int kCholThreads = 1024;  // 32 x 32 thread grid over the trailing matrix
__global__ void __launch_bounds__(kCholThreads) chol_kernel(double* __restrict__ S, int* __restrict__ fail,
                                                             int* __restrict__ done) {
  if (*done) return;
  extern __shared__ double dyn[];
  double (*a)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn);
  __shared__ double invd[kB];
  __shared__ int bad;
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) a[e / kB][e % kB] = S[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = a[0][0];
    bad = 0;
    if (!(d > 0.0)) { bad = 1; d = 1e-300; a[0][0] = d; }
    invd[0] = 1.0 / d;
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int k = 0; k < kB; ++k) {
    const double iv = invd[k];
    for (int i = k + 1 + ty; i < kB; i += 32) {
      const double aki = a[k][i] * iv;
      for (int j = i + tx; j < kB; j += 32) {
        double v = a[i][j] - aki * a[k][j];
        if (j == k + 1) {  // (i == j == k + 1): the next pivot
          if (!(v > 0.0)) { bad = 1; v = 1e-300; }
          invd[k + 1] = 1.0 / v;
        }
        a[i][j] = v;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    const int i = e / kB, j = e % kB;
    const double r = sqrt(a[i][i]);
    S[e] = (j > i) ? a[i][j] / r : (j == i ? r : 0.0);
  }
  if (threadIdx.x == 0 && bad) {
    *fail = 1;
    *done = 1;  // stop the enqueued outer steps; the host redoes the solve with CGS2
  }
}

// ------------------------------------------------------------------ Jacobi (one CTA)
// Cyclic two-sided Jacobi on the symmetric kB x kB matrix T; W accumulates rotations.
// Round-robin tournament ordering in closed form: in round r, pair 0 = (kB-1, r) and pair
// i >= 1 = ((r+i) mod (kB-1), (r-i) mod (kB-1)): kB/2 disjoint pairs, every pair once per
// sweep.  Sweeps stop when the off-diagonal Frobenius norm is <= 1e-13 of the diagonal's.
constexpr int kJacThreads = 1024;
constexpr int kPairs = kB / 2;
constexpr int kBlocks = kPairs * (kPairs + 1) / 2;  // 2x2 blocks (k <= l) of the pair partition
__device__ int g_jacobi_sweeps;  // debug: sweeps used by the last call

// One round applies kB/2 disjoint rotations J_k at once: A := J^T A J, W := W J.  Every
// element of A belongs to exactly one 2x2 block (rows of pair k, columns of pair l), updated
// in a single pass as R_k^T B R_l by one thread (the k > l block is the mirror); the next
// round's rotations are computed while W is updated, so a round is two barriers.
// device-side solver state (no host round trip per outer step)
struct EigState {
  double cheb_b;      // top of the damped interval of the Chebyshev filter (smallest Ritz value)
  double prev_worst;  // relative residual of the previous outer step
  double worst;       // max_j ||Cov v_j - l_j v_j|| / l_1 of the wanted pairs, last executed step
  int done;           // converged: every later kernel of the solve exits at once
  int iters;          // outer steps executed
};

__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(double* __restrict__ T, double* __restrict__ W,
                                                              const EigState* __restrict__ st, int n_wanted) {
  if (st->done) return;
  // far from convergence the Rayleigh-Ritz step only has to supply the filter bound and a
  // reasonable rotation (every rotation is exactly orthogonal): 2 sweeps; near it, to completion
  const int sweeps = st->prev_worst > 1e-4 ? 2 : 30;  // (1 sweep far from convergence costs an extra outer step)
  extern __shared__ double dyn[];
  double (*a)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn);
  double (*w)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn + kB * kLd);
  // rotations double-buffered by round parity: phase A applies round r's rotations to T;
  // phase B computes round r+1's (warps 0-1) while the other warps apply round r's to W
  __shared__ double cs[2][kPairs], sn[2][kPairs];
  __shared__ int pp[2][kPairs], qq[2][kPairs];
  __shared__ short2 blk[kBlocks];
  __shared__ double red[2][kJacThreads / 32];
  __shared__ int wanted[kB];  // 1: row among the n_wanted largest diagonal entries
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    a[e / kB][e % kB] = T[e];
    w[e / kB][e % kB] = (e / kB == e % kB) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) {
    int b = 0;
    for (int k = 0; k < kPairs; ++k)
      for (int l = k; l < kPairs; ++l) blk[b++] = make_short2((short)k, (short)l);
  }
  constexpr int M = kB - 1;
  auto rotations = [&](int rd, int buf) {  // threads 0 .. kPairs-1
    const int i = threadIdx.x;
    int p, q;
    if (i == 0) { p = rd; q = M; }
    else { p = (rd + i) % M; q = (rd - i + M) % M; }
    if (p > q) { const int t = p; p = q; q = t; }
    pp[buf][i] = p;
    qq[buf][i] = q;
    const double apq = a[p][q];
    double c = 1.0, s = 0.0;
    if (apq != 0.0) {
      const double tau = (a[q][q] - a[p][p]) / (2.0 * apq);
      const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
      c = rsqrt(1.0 + t * t);
      s = t * c;
    }
    cs[buf][i] = c;
    sn[buf][i] = s;
  };
  __syncthreads();
  if (threadIdx.x < kPairs) rotations(0, 0);
  __syncthreads();
  int cur = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int rd = 0; rd < M; ++rd, cur ^= 1) {
      for (int b = threadIdx.x; b < kBlocks; b += blockDim.x) {  // phase A: T := J^T T J
        const short2 kl = blk[b];
        const int pk = pp[cur][kl.x], qk = qq[cur][kl.x], pl = pp[cur][kl.y], ql = qq[cur][kl.y];
        const double ck = cs[cur][kl.x], sk = sn[cur][kl.x], cl = cs[cur][kl.y], sl = sn[cur][kl.y];
        const double x00 = a[pk][pl], x01 = a[pk][ql], x10 = a[qk][pl], x11 = a[qk][ql];
        const double y00 = ck * x00 - sk * x10, y01 = ck * x01 - sk * x11;  // rows: R_k^T
        const double y10 = sk * x00 + ck * x10, y11 = sk * x01 + ck * x11;
        const double z00 = cl * y00 - sl * y01, z01 = sl * y00 + cl * y01;  // columns: R_l
        const double z10 = cl * y10 - sl * y11, z11 = sl * y10 + cl * y11;
        a[pk][pl] = z00;
        a[pk][ql] = z01;
        a[qk][pl] = z10;
        a[qk][ql] = z11;
        if (kl.x != kl.y) {
          a[pl][pk] = z00;
          a[pl][qk] = z10;
          a[ql][pk] = z01;
          a[ql][qk] = z11;
        }
      }
      __syncthreads();
      if (threadIdx.x < 64) {  // phase B
        if (threadIdx.x < kPairs) rotations(rd + 1 < M ? rd + 1 : 0, cur ^ 1);
      } else {
        for (int e = threadIdx.x - 64; e < kB * kPairs; e += blockDim.x - 64) {  // W := W J
          const int i = e / kPairs, l = e % kPairs;
          const int p = pp[cur][l], q = qq[cur][l];
          const double c = cs[cur][l], s = sn[cur][l];
          const double wp = w[i][p], wq = w[i][q];
          w[i][p] = c * wp - s * wq;
          w[i][q] = s * wp + c * wq;
        }
      }
      __syncthreads();
    }
    // convergence is judged on the couplings of the wanted (largest) Ritz pairs only: the
    // unwanted tail of the block (oversampling) may stay unconverged
    if (threadIdx.x < kB) {
      const int i = threadIdx.x;
      int rank = 0;
      for (int j = 0; j < kB; ++j) rank += (a[j][j] > a[i][i] || (a[j][j] == a[i][i] && j < i)) ? 1 : 0;
      wanted[i] = rank < n_wanted ? 1 : 0;
    }
    __syncthreads();
    double off = 0.0, dia = 0.0;
    for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
      const int i = e / kB, j = e % kB;
      const double v = a[i][j] * a[i][j];
      if (i == j) dia += v;
      else if (wanted[i] | wanted[j]) off += v;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (lane_id() == 0) { red[0][warp_id()] = off; red[1][warp_id()] = dia; }
    __syncthreads();
    double o = 0.0, d = 0.0;
    for (int w2 = 0; w2 < kJacThreads / 32; ++w2) { o += red[0][w2]; d += red[1][w2]; }
    __syncthreads();
    if (threadIdx.x == 0) g_jacobi_sweeps = sw + 1;
    if (o <= 1e-22 * d) break;  // wanted couplings <= 1e-11 of the diagonal (residual target 1e-9)
  }
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    T[e] = a[e / kB][e % kB];
    W[e] = w[e / kB][e % kB];
  }
}

// order eigenpairs by eigenvalue (desc), top k; eigenvalues from diag(T)
__global__ void select_kernel(const double* __restrict__ T, int k, int* __restrict__ order, double* __restrict__ lam,
                              const int* __restrict__ done) {
  if (*done) return;
  __shared__ double d[kB];
  if (threadIdx.x < kB) {
    const double v = T[threadIdx.x * kB + threadIdx.x];
    d[threadIdx.x] = isnan(v) ? -INFINITY : v;  // ranks stay a permutation
  }
  __syncthreads();
  if (threadIdx.x < kB) {
    const int i = threadIdx.x;
    int rank = 0;
    for (int j = 0; j < kB; ++j) rank += (d[j] > d[i] || (d[j] == d[i] && j < i)) ? 1 : 0;
    if (rank < k) {
      order[rank] = i;
      lam[rank] = d[i];
    }
  }
}

// V[h][k] = Q[h][kB] * W[:, order]
__global__ void gather_cols_kernel(const double* __restrict__ W, const int* __restrict__ order, int k,
                                   double* __restrict__ Wk, const int* __restrict__ done) {
  if (*done) return;
  const int i = blockIdx.x, j = threadIdx.x;
  if (j < k) Wk[(size_t)i * k + j] = W[(size_t)i * kB + order[j]];
}

// residual r_j = ||Cov v_j - l_j v_j||, components sign fix and output
__global__ void residual_kernel(const double* __restrict__ CV, const double* __restrict__ V, const double* __restrict__ lam,
                                int h, int k, double* __restrict__ res,
                                const int* __restrict__ done) {  // k = leading dimension of CV / V
  if (*done) return;
  const int j = blockIdx.x;
  __shared__ double sb[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const double d = CV[(size_t)i * k + j] - lam[j] * V[(size_t)i * k + j];
    s += d * d;
  }
  s = warp_sum(s);
  if (lane_id() == 0) sb[warp_id()] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sb[w];
    res[j] = sqrt(t);
  }
}

__global__ void finalize_components_kernel(const double* __restrict__ V, int h, int k, int hp, int kpad,
                                           float* __restrict__ comp_t) {
  const int j = blockIdx.x;  // component
  __shared__ double best;
  __shared__ int besti;
  if (threadIdx.x == 0) {
    best = -1.0;
    besti = 0;
    for (int i = 0; i < h; ++i) {
      const double a = fabs(V[(size_t)i * k + j]);
      if (a > best) { best = a; besti = i; }
    }
  }
  __syncthreads();
  const double sgn = (V[(size_t)besti * k + j] < 0.0) ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < hp; i += blockDim.x)
    comp_t[(size_t)j * hp + i] = (i < h) ? (float)(sgn * V[(size_t)i * k + j]) : 0.0f;
  (void)kpad;
}

__global__ void gather_first_cols_kernel(const double* __restrict__ Q, int ld, int k, double* __restrict__ V) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (j < k) V[(size_t)i * k + j] = Q[(size_t)i * ld + j];
}

// Chebyshev three-term step: out = (alpha_mult * 2 / b) * CY + beta * Y + gamma * Yold (element-wise),
// b = st->cheb_b read on the device
__global__ void cheb_combine_kernel(const double* __restrict__ CY, const double* __restrict__ Y,
                                    const double* __restrict__ Yold, int64_t n, double alpha_mult, double beta,
                                    double gamma, double* __restrict__ out, const EigState* __restrict__ st) {
  if (st->done) return;
  const double alpha = alpha_mult * (2.0 / st->cheb_b);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = alpha * CY[i] + beta * Y[i] + (Yold ? gamma * Yold[i] : 0.0);
}

__global__ void eig_state_init_kernel(EigState* st) {
  st->cheb_b = 0.0;
  st->prev_worst = 1.0;  // first Rayleigh-Ritz step: far from convergence (2 Jacobi sweeps)
  st->worst = 1.0;
  st->done = 0;
  st->iters = 0;
}

__global__ void copy_gated_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n,
                                  const int* __restrict__ done) {
  if (*done) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// after the residuals of an outer step: filter bound, convergence, iteration count
__global__ void eig_state_kernel(const double* __restrict__ res, const double* __restrict__ lam_all, int n_comps,
                                 EigState* __restrict__ st) {
  if (st->done) return;
  const double lam0 = lam_all[0], lamb = lam_all[kB - 1];
  double worst = 0.0;
  for (int j = 0; j < n_comps; ++j) worst = fmax(worst, res[j]);
  st->cheb_b = fmax(lamb, 1e-12 * lam0);
  st->prev_worst = worst / fmax(lam0, 1e-300);
  st->worst = st->prev_worst;
  st->iters += 1;
  if (worst <= 1e-9 * fmax(lam0, 1e-300)) st->done = 1;
}

__global__ void fill_zero_rows(float* __restrict__ comp_t, int k, int kpad, int hp) {
  const int j = k + blockIdx.x;
  if (j < kpad)
    for (int i = threadIdx.x; i < hp; i += blockDim.x) comp_t[(size_t)j * hp + i] = 0.0f;
}

__global__ void mean_out_kernel(const double* __restrict__ m, int h, int hp, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hp) out[i] = (i < h) ? (float)m[i] : 0.0f;
}

}  // namespace scb

using namespace scb;

static int pca_eig_impl(scb_ctx* ctx, const double* C, int32_t h, int32_t hp, int32_t ones_col, int64_t n_cells,
                        int32_t n_comps, int32_t n_comps_pad, double* eigenvalues, float* components_t,
                        float* col_mean, double* trace, void* stream, bool use_qr, bool* broke, double* final_res) {
  *broke = false;
  SCB_REQUIRE(ctx && C && eigenvalues && components_t && col_mean && trace, SCB_ERR_ARG, "scb_pca_eig: null argument");
  SCB_REQUIRE(n_comps >= 1 && n_comps <= kB - 16 && n_comps <= h && n_comps_pad >= n_comps, SCB_ERR_ARG,
              "scb_pca_eig: need 1 <= n_comps <= %d and <= h", kB - 16);
  SCB_REQUIRE(h >= kB && ones_col >= 0 && ones_col < hp && h <= hp, SCB_ERR_ARG,
              "scb_pca_eig: need h >= %d (block size) and a ones column", kB);
  cudaStream_t s = (cudaStream_t)stream;
  const int kSmemKB = kB * kLd * 8;
  SCB_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemKB));
  SCB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSmemKB));
  // workspace: cov h*h, Qf/Q/Y/Yold/V h*kB each, S 2*kB*kB, W kB*kB, Wk kB*kB, mean h, res, lam, order, flags
  const size_t nd = (size_t)h * h + 5 * (size_t)h * kB + 4 * (size_t)kB * kB + h + 4 * kB + 64;
  void* ws;
  SCB_TRY(ws_get(ctx, 2, nd * 8 + 4096, &ws, s));
  double* cov = (double*)ws;
  double* Qf = cov + (size_t)h * h;   // the iterate between outer steps (fixed buffer)
  double* Q = Qf + (size_t)h * kB;
  double* Y = Q + (size_t)h * kB;
  double* Yold = Y + (size_t)h * kB;
  double* V = Yold + (size_t)h * kB;
  double* S = V + (size_t)h * kB;
  double* W = S + 2 * kB * kB;
  double* Wk = W + kB * kB;
  double* mean = Wk + (size_t)kB * kB;
  double* res = mean + h;
  double* lam_all = res + kB;
  int* order = (int*)(lam_all + kB);
  int* fail = order + kB;
  EigState* st = (EigState*)(((uintptr_t)(fail + 4) + 15) & ~(uintptr_t)15);
  const int* done = &st->done;

  dim3 gc((h + 255) / 256, h);
  cov_build_kernel<<<gc, 256, 0, s>>>(C, hp, h, ones_col, n_cells, cov, mean);
  SCB_LAUNCH_CHECK();
  trace_kernel<<<1, 1024, 0, s>>>(cov, h, trace);
  SCB_LAUNCH_CHECK();
  init_block_kernel<<<h, kB, 0, s>>>(Qf, h);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), s));
  eig_state_init_kernel<<<1, 1, 0, s>>>(st);
  SCB_LAUNCH_CHECK();
  auto orth = [&](double* M, int reps) -> int {
    if (use_qr) {  // rank-deficient fallback
      cgs2_kernel<<<1, kOrthThreads, 0, s>>>(M, h, done);
      SCB_LAUNCH_CHECK();
      return SCB_OK;
    }
    for (int rep = 0; rep < reps; ++rep) {  // CholQR(reps): M := M R^{-1}
      SCB_TRY(dgemm(ctx, kB, kB, h, M, kB, 1, M, kB, 0, S, kB, s, done));
      chol_kernel<<<1, kCholThreads, kSmemKB, s>>>(S, fail, &st->done);
      SCB_LAUNCH_CHECK();
      SCB_TRY(trsm_right_upper(ctx, h, S, M, s, done));  // M := M R^{-1} in place
    }
    return SCB_OK;
  };
  SCB_TRY(orth(Qf, 2));
  // filter degree: 6 converges the synthetic C3 spectrum in 3 outer steps (3 -> 5 steps, 8 -> 3 steps
  // but slower ones; >= 12 overflows CholQR's conditioning), scratch/prof_eig_real.py
  const int kPower = 6, kMaxOuter = 60, kBatch = 4;
  const int64_t nel = (int64_t)h * kB;
  const int eb = (int)((nel + 255) / 256);
  const bool verbose = getenv("SCB_EIG_VERBOSE") != nullptr;
  EigState hs{};
  int outer = 0;
  // Outer steps are enqueued kBatch at a time; every kernel exits at once after convergence
  // (device flag), so a converged solve costs one host round trip per batch.
  while (outer < kMaxOuter) {
    for (int b = 0; b < kBatch && outer < kMaxOuter; ++b, ++outer) {
      SCB_CUDA(cudaMemcpyAsync(Q, Qf, nel * sizeof(double), cudaMemcpyDeviceToDevice, s));
      if (outer == 0) {  // plain power steps until Ritz values are known
        for (int pw = 0; pw < kPower; ++pw) {
          SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, Y, kB, s, done));
          std::swap(Q, Y);
        }
      } else {
        // Chebyshev filter T_kPower(sigma), sigma = (2/b) Cov - I: damps [0, b], amplifies > b
        SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, V, kB, s, done));
        cheb_combine_kernel<<<eb, 256, 0, s>>>(V, Q, nullptr, nel, 1.0, -1.0, 0.0, Y, st);  // Y1 = sigma Q
        SCB_LAUNCH_CHECK();
        std::swap(Q, Yold);  // Yold = Y0
        for (int k = 1; k < kPower; ++k) {  // Y_{k+1} = 2 sigma Y_k - Y_{k-1}
          SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Y, kB, 0, V, kB, s, done));
          cheb_combine_kernel<<<eb, 256, 0, s>>>(V, Y, Yold, nel, 2.0, -2.0, -1.0, Q, st);
          SCB_LAUNCH_CHECK();
          std::swap(Yold, Y);  // Yold = Y_k
          std::swap(Y, Q);     // Y = Y_{k+1}
        }
        std::swap(Q, Y);  // Q = last iterate
      }
      SCB_TRY(orth(Q, 2));
      // Rayleigh-Ritz: T = Q^T Cov Q, T = W diag W^T; rotate Q := Q W (sorted descending)
      SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, Y, kB, s, done));        // Y = Cov Q
      SCB_TRY(dgemm(ctx, kB, kB, h, Q, kB, 1, Y, kB, 0, S, kB, s, done));        // T = Q^T Y
      jacobi_kernel<<<1, kJacThreads, 2 * kSmemKB, s>>>(S, W, st, n_comps);
      SCB_LAUNCH_CHECK();
      select_kernel<<<1, kB, 0, s>>>(S, kB, order, lam_all, done);
      SCB_LAUNCH_CHECK();
      gather_cols_kernel<<<kB, kB, 0, s>>>(W, order, kB, Wk, done);
      SCB_LAUNCH_CHECK();
      SCB_TRY(dgemm(ctx, h, kB, kB, Q, kB, 0, Wk, kB, 0, Yold, kB, s, done));   // Ritz vectors
      SCB_TRY(dgemm(ctx, h, kB, kB, Y, kB, 0, Wk, kB, 0, V, kB, s, done));      // Cov * Ritz vectors
      residual_kernel<<<n_comps, 256, 0, s>>>(V, Yold, lam_all, h, kB, res, done);
      SCB_LAUNCH_CHECK();
      copy_gated_kernel<<<eb, 256, 0, s>>>(Yold, Qf, nel, done);                 // next iterate
      SCB_LAUNCH_CHECK();
      eig_state_kernel<<<1, 1, 0, s>>>(res, lam_all, n_comps, st);
      SCB_LAUNCH_CHECK();
    }
    int hfail_now = 0;
    SCB_CUDA(cudaMemcpyAsync(&hs, st, sizeof(EigState), cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaMemcpyAsync(&hfail_now, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    if (verbose) {
      int sweeps = 0;
      cudaMemcpyFromSymbol(&sweeps, g_jacobi_sweeps, sizeof(int));
      fprintf(stderr, "[scb_pca_eig] after %d enqueued outer steps: executed %d, residual %.3e, done %d, last jacobi "
              "sweeps %d\n", outer, hs.iters, hs.worst, hs.done, sweeps);
    }
    if (hfail_now) {  // Cholesky-QR broke down (block rank-deficient): caller retries with CGS2
      *broke = true;
      return SCB_OK;
    }
    if (hs.done) break;
  }
  *final_res = hs.worst;
  SCB_REQUIRE(hs.done, SCB_ERR_DATA, "scb_pca_eig: not converged after %d outer steps (relative residual %.3e)",
              kMaxOuter, hs.worst);
  // V := the n_comps leading Ritz vectors (columns 0..n_comps-1 of Qf, already sorted)
  gather_first_cols_kernel<<<h, kB, 0, s>>>(Qf, kB, n_comps, V);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaMemcpyAsync(eigenvalues, lam_all, sizeof(double) * n_comps, cudaMemcpyDeviceToDevice, s));
  finalize_components_kernel<<<n_comps, 256, 0, s>>>(V, h, n_comps, hp, n_comps_pad, components_t);
  SCB_LAUNCH_CHECK();
  if (n_comps_pad > n_comps) {
    fill_zero_rows<<<n_comps_pad - n_comps, 256, 0, s>>>(components_t, n_comps, n_comps_pad, hp);
    SCB_LAUNCH_CHECK();
  }
  mean_out_kernel<<<(hp + 255) / 256, 256, 0, s>>>(mean, h, hp, col_mean);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_pca_eig(scb_ctx* ctx, const double* C, int32_t h, int32_t hp, int32_t ones_col, int64_t n_cells,
                           int32_t n_comps, int32_t n_comps_pad, double* eigenvalues, float* components_t,
                           float* col_mean, double* trace, void* stream) {
  // CholQR2 orthonormalisation; if the block turns rank-deficient (fewer than kB + 1 cells, or
  // duplicated cells: the covariance has rank < kB) the solve is redone with CGS2, which
  // completes the basis with pseudo-random orthonormal directions
  bool broke = false;
  double res = 0.0;
  SCB_TRY(pca_eig_impl(ctx, C, h, hp, ones_col, n_cells, n_comps, n_comps_pad, eigenvalues, components_t, col_mean,
                       trace, stream, false, &broke, &res));
  if (!broke) return SCB_OK;
  SCB_TRY(pca_eig_impl(ctx, C, h, hp, ones_col, n_cells, n_comps, n_comps_pad, eigenvalues, components_t, col_mean,
                       trace, stream, true, &broke, &res));
  SCB_REQUIRE(!broke, SCB_ERR_DATA, "scb_pca_eig: orthonormalisation breakdown");
  return SCB_OK;
}

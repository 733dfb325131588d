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
#include <cublas_v2.h>
#include <cusolverDn.h>
#include "common.cuh"

namespace scb {

constexpr int kB = 96;   // subspace block size (n_comps + oversampling)
constexpr int kLd = kB + 1;

// ------------------------------------------------------------------ small fp64 GEMM
// Cm[M][N] (ldc) = alpha * op(A) * op(B) + beta * Cm ; row-major operands.
// opA: 0 -> A[M][K] (lda), 1 -> A^T where A is [K][M]; opB: 0 -> B[K][N], 1 -> B^T ([N][K]).
// 64x64 tiles, 256 threads, 4x4 per thread, K chunk 16; split-K over blockIdx.z with
// atomicAdd when gridDim.z > 1 (caller zeroes Cm and passes beta = 0).
// Plain fp64 GEMMs of the eigensolver (Cov x block, block^T x block, block x small) go to
// cuBLAS: row-major C[M][N] = op(A) op(B) is column-major C^T = op(B)^T op(A)^T.
static int dgemm(scb_ctx* ctx, int M, int N, int K, const double* A, int lda, int opA, const double* B, int ldb,
                 int opB, double* Cm, int ldc, cudaStream_t s) {
  if (!ctx->blas) {
    cublasHandle_t h;
    SCB_REQUIRE(cublasCreate(&h) == CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cublasCreate failed");
    ctx->blas = h;
  }
  cublasHandle_t h = (cublasHandle_t)ctx->blas;
  SCB_REQUIRE(cublasSetStream(h, s) == CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cublasSetStream failed");
  const double one = 1.0, zero = 0.0;
  const cublasStatus_t st = cublasDgemm(h, opB ? CUBLAS_OP_T : CUBLAS_OP_N, opA ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K,
                                        &one, B, ldb, A, lda, &zero, Cm, ldc);
  SCB_REQUIRE(st == CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cublasDgemm failed (%d)", (int)st);
  return SCB_OK;
}

// M[h][kB] (row-major) := M R^{-1} with R upper triangular [kB][kB] (row-major): column-major
// this is M^T := R^{-T} M^T, a left solve with the lower-triangular column-major view of R.
static int trsm_right_upper(scb_ctx* ctx, int h, const double* R, double* M, cudaStream_t s) {
  cublasHandle_t hd = (cublasHandle_t)ctx->blas;
  SCB_REQUIRE(cublasSetStream(hd, s) == CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cublasSetStream failed");
  const double one = 1.0;
  const cublasStatus_t st = cublasDtrsm(hd, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                                        CUBLAS_DIAG_NON_UNIT, kB, h, &one, R, kB, M, kB);
  SCB_REQUIRE(st == CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cublasDtrsm failed (%d)", (int)st);
  return SCB_OK;
}

// M[h][kB] (row-major) := an orthonormal basis of its column space by Householder QR
// (cuSOLVER geqrf + orgqr on the column-major transpose, via cublasDgeam); robust to rank
// deficiency.  tmp: h * kB doubles.  Used only when CholQR breaks down.
static int householder_orth(scb_ctx* ctx, int h, double* M, double* tmp, cudaStream_t s) {
  if (!ctx->solver) {
    cusolverDnHandle_t sh;
    SCB_REQUIRE(cusolverDnCreate(&sh) == CUSOLVER_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: cusolverDnCreate failed");
    ctx->solver = sh;
  }
  cusolverDnHandle_t sh = (cusolverDnHandle_t)ctx->solver;
  cublasHandle_t bh = (cublasHandle_t)ctx->blas;
  SCB_REQUIRE(cusolverDnSetStream(sh, s) == CUSOLVER_STATUS_SUCCESS && cublasSetStream(bh, s) == CUBLAS_STATUS_SUCCESS,
              SCB_ERR_CUDA, "scb_pca_eig: set stream failed");
  const double one = 1.0, zero = 0.0;
  // row-major M[h][kB] is column-major kB x h; tmp := its transpose (column-major h x kB)
  SCB_REQUIRE(cublasDgeam(bh, CUBLAS_OP_T, CUBLAS_OP_N, h, kB, &one, M, kB, &zero, tmp, h, tmp, h) ==
                  CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: geam failed");
  int lw1 = 0, lw2 = 0;
  SCB_REQUIRE(cusolverDnDgeqrf_bufferSize(sh, h, kB, tmp, h, &lw1) == CUSOLVER_STATUS_SUCCESS, SCB_ERR_CUDA,
              "scb_pca_eig: geqrf_bufferSize failed");
  void* ws;
  const size_t need = (size_t)(kB + std::max(lw1, 1)) * 8 + 64;
  SCB_TRY(ws_get(ctx, 3, need, &ws, s));
  double* tau = (double*)ws;
  double* work = tau + kB;
  int* info = (int*)((char*)ws + need - 16);
  SCB_REQUIRE(cusolverDnDgeqrf(sh, h, kB, tmp, h, tau, work, lw1, info) == CUSOLVER_STATUS_SUCCESS, SCB_ERR_CUDA,
              "scb_pca_eig: geqrf failed");
  SCB_REQUIRE(cusolverDnDorgqr_bufferSize(sh, h, kB, kB, tmp, h, tau, &lw2) == CUSOLVER_STATUS_SUCCESS, SCB_ERR_CUDA,
              "scb_pca_eig: orgqr_bufferSize failed");
  if (lw2 > lw1) {
    const size_t need2 = (size_t)(kB + lw2) * 8 + 64;
    SCB_TRY(ws_get(ctx, 3, need2, &ws, s));
    tau = (double*)ws;  // tau must survive: recompute geqrf into the larger buffer
    work = tau + kB;
    info = (int*)((char*)ws + need2 - 16);
    SCB_REQUIRE(cublasDgeam(bh, CUBLAS_OP_T, CUBLAS_OP_N, h, kB, &one, M, kB, &zero, tmp, h, tmp, h) ==
                    CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: geam failed");
    SCB_REQUIRE(cusolverDnDgeqrf(sh, h, kB, tmp, h, tau, work, lw2, info) == CUSOLVER_STATUS_SUCCESS, SCB_ERR_CUDA,
                "scb_pca_eig: geqrf failed");
    lw1 = lw2;
  }
  SCB_REQUIRE(cusolverDnDorgqr(sh, h, kB, kB, tmp, h, tau, work, std::max(lw1, lw2), info) == CUSOLVER_STATUS_SUCCESS,
              SCB_ERR_CUDA, "scb_pca_eig: orgqr failed");
  // back to row-major M[h][kB]: column-major kB x h = transpose of tmp
  SCB_REQUIRE(cublasDgeam(bh, CUBLAS_OP_T, CUBLAS_OP_N, kB, h, &one, tmp, h, &zero, M, kB, M, kB) ==
                  CUBLAS_STATUS_SUCCESS, SCB_ERR_CUDA, "scb_pca_eig: geam failed");
  return SCB_OK;
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
constexpr int kCholThreads = 1024;  // 32 x 32 thread grid over the trailing matrix
__global__ void __launch_bounds__(kCholThreads) chol_kernel(double* __restrict__ S, int* __restrict__ fail) {
  extern __shared__ double dyn[];
  double (*a)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn);
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) a[e / kB][e % kB] = S[e];
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int k = 0; k < kB; ++k) {
    // every thread derives the pivot itself (no extra barrier): row k of R = a[k][j] / sqrt(a_kk)
    double d = a[k][k];
    if (!(d > 0.0)) d = 1e-300;
    const double r = sqrt(d), inv = 1.0 / r;
    __syncthreads();  // all pivots read before row k is rescaled
    if (threadIdx.x == 0) {
      if (!(a[k][k] > 0.0)) *fail = 1;
      a[k][k] = r;
    }
    for (int j = k + 1 + threadIdx.x; j < kB; j += blockDim.x) a[k][j] *= inv;
    __syncthreads();
    for (int i = k + 1 + ty; i < kB; i += 32) {
      const double aki = a[k][i];
      for (int j = i + tx; j < kB; j += 32) a[i][j] -= aki * a[k][j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    const int i = e / kB, j = e % kB;
    S[e] = (j >= i) ? a[i][j] : 0.0;
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
// in a single pass as R_k^T B R_l by one thread (the k > l block is the mirror), so a round
// is two barriers and one read + one write of A and W.
__global__ void __launch_bounds__(kJacThreads) jacobi_kernel(double* __restrict__ T, double* __restrict__ W, int sweeps) {
  extern __shared__ double dyn[];
  double (*a)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn);
  double (*w)[kLd] = reinterpret_cast<double (*)[kLd]>(dyn + kB * kLd);
  __shared__ double cs[kPairs], sn[kPairs];
  __shared__ int pp[kPairs], qq[kPairs];
  __shared__ short2 blk[kBlocks];
  __shared__ double red[2][kJacThreads / 32];
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    a[e / kB][e % kB] = T[e];
    w[e / kB][e % kB] = (e / kB == e % kB) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) {
    int b = 0;
    for (int k = 0; k < kPairs; ++k)
      for (int l = k; l < kPairs; ++l) blk[b++] = make_short2((short)k, (short)l);
  }
  __syncthreads();
  constexpr int M = kB - 1;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int rd = 0; rd < M; ++rd) {
      if (threadIdx.x < kPairs) {
        const int i = threadIdx.x;
        int p, q;
        if (i == 0) { p = rd; q = M; }
        else { p = (rd + i) % M; q = (rd - i + M) % M; }
        if (p > q) { const int t = p; p = q; q = t; }
        pp[i] = p;
        qq[i] = q;
        const double apq = a[p][q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double tau = (a[q][q] - a[p][p]) / (2.0 * apq);
          const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = rsqrt(1.0 + t * t);
          s = t * c;
        }
        cs[i] = c;
        sn[i] = s;
      }
      __syncthreads();
      for (int b = threadIdx.x; b < kBlocks; b += blockDim.x) {
        const short2 kl = blk[b];
        const int pk = pp[kl.x], qk = qq[kl.x], pl = pp[kl.y], ql = qq[kl.y];
        const double ck = cs[kl.x], sk = sn[kl.x], cl = cs[kl.y], sl = sn[kl.y];
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
      for (int e = threadIdx.x; e < kB * kPairs; e += blockDim.x) {  // W := W J
        const int i = e / kPairs, l = e % kPairs;
        const int p = pp[l], q = qq[l];
        const double c = cs[l], s = sn[l];
        const double wp = w[i][p], wq = w[i][q];
        w[i][p] = c * wp - s * wq;
        w[i][q] = s * wp + c * wq;
      }
      __syncthreads();
    }
    double off = 0.0, dia = 0.0;
    for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
      const int i = e / kB, j = e % kB;
      const double v = a[i][j] * a[i][j];
      if (i != j) off += v; else dia += v;
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (lane_id() == 0) { red[0][warp_id()] = off; red[1][warp_id()] = dia; }
    __syncthreads();
    double o = 0.0, d = 0.0;
    for (int w2 = 0; w2 < kJacThreads / 32; ++w2) { o += red[0][w2]; d += red[1][w2]; }
    __syncthreads();
    if (threadIdx.x == 0) g_jacobi_sweeps = sw + 1;
    if (o <= 1e-26 * d) break;
  }
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    T[e] = a[e / kB][e % kB];
    W[e] = w[e / kB][e % kB];
  }
}

// order eigenpairs by eigenvalue (desc), top k; eigenvalues from diag(T)
__global__ void select_kernel(const double* __restrict__ T, int k, int* __restrict__ order, double* __restrict__ lam) {
  __shared__ double d[kB];
  if (threadIdx.x < kB) d[threadIdx.x] = T[threadIdx.x * kB + threadIdx.x];
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
                                   double* __restrict__ Wk) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (j < k) Wk[(size_t)i * k + j] = W[(size_t)i * kB + order[j]];
}

// residual r_j = ||Cov v_j - l_j v_j||, components sign fix and output
__global__ void residual_kernel(const double* __restrict__ CV, const double* __restrict__ V, const double* __restrict__ lam,
                                int h, int k, double* __restrict__ res) {  // k = leading dimension of CV / V
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

// Chebyshev three-term step: out = alpha * CY + beta * Y + gamma * Yold (element-wise)
__global__ void cheb_combine_kernel(const double* __restrict__ CY, const double* __restrict__ Y,
                                    const double* __restrict__ Yold, int64_t n, double alpha, double beta, double gamma,
                                    double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = alpha * CY[i] + beta * Y[i] + (Yold ? gamma * Yold[i] : 0.0);
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
                        float* col_mean, double* trace, void* stream, bool use_qr, bool* broke) {
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
  // workspace: cov h*h, Q h*kB, Y h*kB, S kB*kB, W kB*kB, Wk kB*n, V h*n, CV h*n, mean h, misc
  const size_t nd = (size_t)h * h + 2 * (size_t)h * kB + 3 * kB * kB + (size_t)kB * kB + 2 * (size_t)h * kB +
                    h + 4 * kB + 64;
  void* ws;
  SCB_TRY(ws_get(ctx, 2, nd * 8 + 4096, &ws, s));
  double* cov = (double*)ws;
  double* Q = cov + (size_t)h * h;
  double* Y = Q + (size_t)h * kB;
  double* S = Y + (size_t)h * kB;
  double* W = S + 2 * kB * kB;
  double* Wk = W + kB * kB;
  double* V = Wk + (size_t)kB * kB;
  double* CV = V + (size_t)h * kB;
  double* mean = CV + (size_t)h * kB;
  double* res = mean + h;
  double* lam_all = res + kB;
  int* order = (int*)(lam_all + kB);
  int* fail = order + kB;

  dim3 gc((h + 255) / 256, h);
  cov_build_kernel<<<gc, 256, 0, s>>>(C, hp, h, ones_col, n_cells, cov, mean);
  SCB_LAUNCH_CHECK();
  trace_kernel<<<1, 1024, 0, s>>>(cov, h, trace);
  SCB_LAUNCH_CHECK();
  init_block_kernel<<<h, kB, 0, s>>>(Q, h);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), s));
  auto orth = [&](double*& M, int reps) -> int {
    if (use_qr) return householder_orth(ctx, h, M, Y, s);  // rank-deficient fallback
    for (int rep = 0; rep < reps; ++rep) {  // CholQR(reps): M := M R^{-1}
      SCB_TRY(dgemm(ctx, kB, kB, h, M, kB, 1, M, kB, 0, S, kB, s));
      chol_kernel<<<1, kCholThreads, kSmemKB, s>>>(S, fail);
      SCB_LAUNCH_CHECK();
      SCB_TRY(trsm_right_upper(ctx, h, S, M, s));  // M := M R^{-1} in place
    }
    return SCB_OK;
  };
  SCB_TRY(orth(Q, 2));
  // filter degree: 6 converges the synthetic C3 spectrum in 3 outer steps (3 -> 5 steps, 8 -> 3 steps
  // but slower ones; >= 12 overflows CholQR's conditioning), scratch/prof_eig_real.py
  const int kPower = 6, kMaxOuter = 60;
  double host_res[kB];
  int outer = 0;
  const bool verbose = getenv("SCB_EIG_VERBOSE") != nullptr;
  cudaEvent_t ev0, ev1;
  if (verbose) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, s);
  }
  double prev_worst = 1.0;  // relative residual of the previous outer step
  double cheb_b = 0.0;  // top of the damped interval [0, b] (smallest Ritz value of the block)
  double* Yold = CV;      // h x kB scratch for the three-term recurrence (CV reused below)
  for (; outer < kMaxOuter; ++outer) {
    if (cheb_b <= 0.0) {
      // plain power steps until Ritz values are known
      for (int pw = 0; pw < kPower; ++pw) {
        SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, Y, kB, s));
        std::swap(Q, Y);
      }
    } else {
      // Chebyshev filter T_kPower(sigma), sigma = (2/b) Cov - I: damps [0, b], amplifies > b
      const int64_t nel = (int64_t)h * kB;
      const int eb = (int)((nel + 255) / 256);
      const double a2 = 2.0 / cheb_b;
      // Y1 = sigma Q  -> stored in Y
      SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, V, kB, s));
      cheb_combine_kernel<<<eb, 256, 0, s>>>(V, Q, nullptr, nel, a2, -1.0, 0.0, Y);
      SCB_LAUNCH_CHECK();
      std::swap(Q, Yold);  // Yold = Y0
      for (int k = 1; k < kPower; ++k) {  // Y_{k+1} = 2 sigma Y_k - Y_{k-1}
        SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Y, kB, 0, V, kB, s));
        cheb_combine_kernel<<<eb, 256, 0, s>>>(V, Y, Yold, nel, 2.0 * a2, -2.0, -1.0, Q);
        SCB_LAUNCH_CHECK();
        std::swap(Yold, Y);  // Yold = Y_k
        std::swap(Y, Q);     // Y = Y_{k+1}
      }
      std::swap(Q, Y);  // Q = last iterate
    }
    SCB_TRY(orth(Q, 2));
    // Rayleigh-Ritz: T = Q^T Cov Q, T = W diag W^T; rotate Q := Q W (sorted descending)
    SCB_TRY(dgemm(ctx, h, kB, h, cov, h, 0, Q, kB, 0, Y, kB, s));        // Y = Cov Q
    SCB_TRY(dgemm(ctx, kB, kB, h, Q, kB, 1, Y, kB, 0, S, kB, s));   // T = Q^T Y
    // Far from convergence the Rayleigh-Ritz step only has to supply the filter bound and a
    // reasonable rotation (every Jacobi rotation is exactly orthogonal, so a partial sweep
    // count never damages the subspace): 2 sweeps.  Near convergence it runs to completion.
    jacobi_kernel<<<1, kJacThreads, 2 * kSmemKB, s>>>(S, W, prev_worst > 1e-4 ? 2 : 30);
    SCB_LAUNCH_CHECK();
    select_kernel<<<1, kB, 0, s>>>(S, kB, order, lam_all);
    SCB_LAUNCH_CHECK();
    gather_cols_kernel<<<kB, kB, 0, s>>>(W, order, kB, Wk);
    SCB_LAUNCH_CHECK();
    SCB_TRY(dgemm(ctx, h, kB, kB, Q, kB, 0, Wk, kB, 0, Yold, kB, s));        // Ritz vectors (spare buffer)
    SCB_TRY(dgemm(ctx, h, kB, kB, Y, kB, 0, Wk, kB, 0, V, kB, s));           // Cov * Ritz vectors
    std::swap(Q, Yold);
    residual_kernel<<<n_comps, 256, 0, s>>>(V, Q, lam_all, h, kB, res);
    SCB_LAUNCH_CHECK();
    double lam0 = 0.0, lamb = 0.0;
    SCB_CUDA(cudaMemcpyAsync(host_res, res, sizeof(double) * n_comps, cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaMemcpyAsync(&lam0, lam_all, sizeof(double), cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaMemcpyAsync(&lamb, lam_all + kB - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    int hfail_now = 0;
    SCB_CUDA(cudaMemcpyAsync(&hfail_now, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    if (hfail_now) {  // Cholesky-QR broke down (block rank-deficient): caller retries with QR
      *broke = true;
      return SCB_OK;
    }
    cheb_b = std::max(lamb, 1e-12 * lam0);
    double worst = 0.0;  // max residual / lambda_1 of the wanted Ritz pairs
    for (int j = 0; j < n_comps; ++j) worst = std::max(worst, host_res[j]);
    if (verbose) {
      cudaEventRecord(ev1, s);
      cudaEventSynchronize(ev1);
      float ms = 0;
      cudaEventElapsedTime(&ms, ev0, ev1);
      int sweeps = 0;
      cudaMemcpyFromSymbol(&sweeps, g_jacobi_sweeps, sizeof(int));
      fprintf(stderr, "[scb_pca_eig] outer %d residual %.3e (lam0 %.4e) jacobi sweeps %d elapsed %.2f ms\n", outer + 1,
              worst, lam0, sweeps, ms);
    }
    prev_worst = worst / std::max(lam0, 1e-300);
    if (worst <= 1e-9 * std::max(lam0, 1e-300)) break;
  }
  // V := the n_comps leading Ritz vectors (columns 0..n_comps-1 of Q, already sorted)
  gather_first_cols_kernel<<<h, kB, 0, s>>>(Q, kB, n_comps, V);
  SCB_LAUNCH_CHECK();
  int hfail = 0;
  SCB_CUDA(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  if (hfail) {
    *broke = true;
    return SCB_OK;
  }
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
  // duplicated cells: the covariance has rank < kB) the solve is redone with Householder QR,
  // which completes the basis with arbitrary orthonormal directions
  bool broke = false;
  SCB_TRY(pca_eig_impl(ctx, C, h, hp, ones_col, n_cells, n_comps, n_comps_pad, eigenvalues, components_t, col_mean,
                       trace, stream, false, &broke));
  if (!broke) return SCB_OK;
  SCB_TRY(pca_eig_impl(ctx, C, h, hp, ones_col, n_cells, n_comps, n_comps_pad, eigenvalues, components_t, col_mean,
                       trace, stream, true, &broke));
  SCB_REQUIRE(!broke, SCB_ERR_DATA, "scb_pca_eig: orthonormalisation breakdown");
  return SCB_OK;
}

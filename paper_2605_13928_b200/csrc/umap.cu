// sc.tl.umap layout: umap-learn's optimize_layout_euclidean (2-D) on the
// fuzzy graph of sc.pp.neighbors, as edge-parallel SGD.
//
// Per epoch n one thread per directed edge (i -> j) of the symmetric graph that is due
// (epoch_of_next_sample <= n) applies umap's attractive step to both endpoints, then its
// n_neg = floor((n - next_negative) / epochs_per_negative_sample) negative samples (vertices
// from a counter-based hash of (seed, epoch, edge, sample)) push i away; learning rate
// alpha = 1 - n / n_epochs; gradients clipped to [-4, 4].  umap runs this loop sequentially
// (numba, one thread); here concurrent edges read possibly stale positions and ACCUMULATE their
// moves with atomic adds (a vertex with many due edges gets the sum of their steps, as the
// sequential loop would apply them one after another), so the result matches the sequential
// algorithm in distribution, not bit for bit -- parity is checked on layout quality (trustworthiness,
// cluster separation) against the oracle's sequential restatement (tests/test_gpu_umap.py).
#include "common.cuh"

namespace scb {

__device__ __forceinline__ float clip4(float v) { return fminf(4.0f, fmaxf(-4.0f, v)); }

__device__ __forceinline__ uint32_t hash_u32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (uint32_t)x;
}

// edges of the connectivities CSR: head = row, tail = column; weights below max/n_epochs are
// dropped (never sampled), the rest get epochs_per_sample = w_max / w
__global__ void umap_prep_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ w, int64_t n_rows,
                                 float w_max, int n_epochs, int neg_rate, int32_t* __restrict__ head,
                                 float* __restrict__ eps, float* __restrict__ next_s, float* __restrict__ next_n) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
      head[e] = (int32_t)r;
      const float v = w[e];
      if (v < w_max / (float)n_epochs || v <= 0.0f) {
        eps[e] = -1.0f;
        next_s[e] = CUDART_INF_F;
        next_n[e] = CUDART_INF_F;
      } else {
        const float ep = w_max / v;
        eps[e] = ep;
        next_s[e] = ep;
        next_n[e] = ep / (float)neg_rate;
      }
    }
  }
}

// umap rescales every initialisation to [0, 10] per dimension
__global__ void umap_rescale_kernel(const float* __restrict__ init, int64_t ld, int64_t n, const float* __restrict__ mm,
                                    float2* __restrict__ emb) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = init[i * ld], y = init[i * ld + 1];
    const float sx = mm[1] > mm[0] ? 10.0f / (mm[1] - mm[0]) : 0.0f;
    const float sy = mm[3] > mm[2] ? 10.0f / (mm[3] - mm[2]) : 0.0f;
    emb[i] = make_float2((x - mm[0]) * sx, (y - mm[2]) * sy);
  }
}

__global__ void umap_minmax_kernel(const float* __restrict__ init, int64_t ld, int64_t n, unsigned int* __restrict__ mm) {
  float lo0 = CUDART_INF_F, hi0 = -CUDART_INF_F, lo1 = CUDART_INF_F, hi1 = -CUDART_INF_F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = init[i * ld], y = init[i * ld + 1];
    lo0 = fminf(lo0, x); hi0 = fmaxf(hi0, x); lo1 = fminf(lo1, y); hi1 = fmaxf(hi1, y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo0 = fminf(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
    hi0 = fmaxf(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
    lo1 = fminf(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
    hi1 = fmaxf(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
  }
  // order-preserving float -> uint encoding so min/max are integer atomics
  auto enc = [](float f) { const unsigned u = __float_as_uint(f); return (u >> 31) ? ~u : (u | 0x80000000u); };
  if (lane_id() == 0) {
    atomicMin(&mm[0], enc(lo0));
    atomicMax(&mm[1], enc(hi0));
    atomicMin(&mm[2], enc(lo1));
    atomicMax(&mm[3], enc(hi1));
  }
}

__global__ void umap_decode_kernel(const unsigned int* __restrict__ mm, float* __restrict__ out) {
  const int t = threadIdx.x;
  if (t < 4) {
    const unsigned u = mm[t];
    out[t] = __uint_as_float((u >> 31) ? (u & 0x7FFFFFFFu) : ~u);
  }
}

__global__ void __launch_bounds__(256)
umap_epoch_kernel(const int32_t* __restrict__ head, const int32_t* __restrict__ tail, const float* __restrict__ eps,
                  float* __restrict__ next_s, float* __restrict__ next_n, int64_t n_edges, float2* __restrict__ emb,
                  int32_t n_vertices, int epoch, float alpha, float a, float b, int neg_rate, uint64_t seed) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  const float ns = next_s[e];
  if (ns > (float)epoch) return;
  const int32_t j = head[e], k = tail[e];
  const float2 cur0 = emb[j];
  float2 cur = cur0;
  const float2 oth = emb[k];
  float dx = cur.x - oth.x, dy = cur.y - oth.y;
  float d2 = dx * dx + dy * dy;
  float* ek = reinterpret_cast<float*>(emb + k);
  if (d2 > 0.0f) {
    const float gc = (-2.0f * a * b * __powf(d2, b - 1.0f)) / (a * __powf(d2, b) + 1.0f);
    const float gx = clip4(gc * dx) * alpha, gy = clip4(gc * dy) * alpha;
    cur.x += gx;
    cur.y += gy;
    // concurrent edges of the same vertex accumulate (not overwrite) their moves
    atomicAdd(ek, -gx);
    atomicAdd(ek + 1, -gy);
  }
  const float ep = eps[e];
  next_s[e] = ns + ep;
  const float epn = ep / (float)neg_rate;
  const float nn = next_n[e];
  const int n_neg = (int)(((float)epoch - nn) / epn);
  for (int p = 0; p < n_neg; ++p) {
    const uint32_t r = hash_u32(seed ^ ((uint64_t)epoch << 40) ^ ((uint64_t)e << 8) ^ (uint64_t)p);
    const int32_t kk = (int32_t)(r % (uint32_t)n_vertices);
    const float2 o = emb[kk];
    dx = cur.x - o.x;
    dy = cur.y - o.y;
    d2 = dx * dx + dy * dy;
    float gc;
    if (d2 > 0.0f) gc = (2.0f * b) / ((0.001f + d2) * (a * __powf(d2, b) + 1.0f));
    else if (kk == j) continue;
    else gc = 0.0f;
    const float gx = gc > 0.0f ? clip4(gc * dx) : 4.0f, gy = gc > 0.0f ? clip4(gc * dy) : 4.0f;
    cur.x += gx * alpha;
    cur.y += gy * alpha;
  }
  if (n_neg > 0) next_n[e] = nn + (float)n_neg * epn;
  float* ej = reinterpret_cast<float*>(emb + j);
  atomicAdd(ej, cur.x - cur0.x);
  atomicAdd(ej + 1, cur.y - cur0.y);
}

}  // namespace scb

using namespace scb;

extern "C" int scb_umap_layout(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights,
                               int64_t n_vertices, int64_t nnz, float w_max, const float* init, int64_t init_ld,
                               int32_t n_epochs, float a, float b, int32_t neg_rate, uint64_t seed, float* emb,
                               void* stream) {
  SCB_REQUIRE(ctx && indptr && indices && weights && init && emb, SCB_ERR_ARG, "scb_umap_layout: null argument");
  SCB_REQUIRE(n_epochs >= 1 && neg_rate >= 1 && init_ld >= 2 && n_vertices < INT32_MAX, SCB_ERR_ARG,
              "scb_umap_layout: bad parameters");
  SCB_REQUIRE(((uintptr_t)emb & 7) == 0, SCB_ERR_ARG, "scb_umap_layout: emb must be 8-byte aligned (float2)");
  cudaStream_t s = (cudaStream_t)stream;
  if (n_vertices == 0) return SCB_OK;
  void* ws;
  const size_t per = (size_t)nnz * 4;
  SCB_TRY(ws_get(ctx, 0, per * 4 + 64, &ws, s));
  int32_t* head = (int32_t*)ws;
  float* eps = (float*)((char*)ws + per);
  float* next_s = (float*)((char*)ws + 2 * per);
  float* next_n = (float*)((char*)ws + 3 * per);
  unsigned int* mm = (unsigned int*)((char*)ws + 4 * per);
  float* mmf = (float*)(mm + 4);
  const int grid = ctx->num_sms * 8;
  umap_prep_kernel<<<grid, 256, 0, s>>>(indptr, weights, n_vertices, w_max, n_epochs, neg_rate, head, eps, next_s,
                                       next_n);
  SCB_LAUNCH_CHECK();
  const unsigned int init_mm[4] = {0xFFFFFFFFu, 0u, 0xFFFFFFFFu, 0u};
  SCB_CUDA(cudaMemcpyAsync(mm, init_mm, sizeof(init_mm), cudaMemcpyHostToDevice, s));
  umap_minmax_kernel<<<grid, 256, 0, s>>>(init, init_ld, n_vertices, mm);
  SCB_LAUNCH_CHECK();
  umap_decode_kernel<<<1, 32, 0, s>>>(mm, mmf);
  SCB_LAUNCH_CHECK();
  umap_rescale_kernel<<<grid, 256, 0, s>>>(init, init_ld, n_vertices, mmf, reinterpret_cast<float2*>(emb));
  SCB_LAUNCH_CHECK();
  const unsigned eg = (unsigned)ceil_div(nnz, 256);
  for (int n = 0; n < n_epochs; ++n) {
    const float alpha = 1.0f - (float)n / (float)n_epochs;
    if (nnz > 0) {
      umap_epoch_kernel<<<eg, 256, 0, s>>>(head, indices, eps, next_s, next_n, nnz, reinterpret_cast<float2*>(emb),
                                          (int32_t)n_vertices, n, alpha, a, b, neg_rate, seed);
      SCB_LAUNCH_CHECK();
    }
  }
  return SCB_OK;
}

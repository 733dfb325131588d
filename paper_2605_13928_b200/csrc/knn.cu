// Exact brute-force kNN graph on the PCA embedding (sc.pp.neighbors, method exact).
//
// 1. prep: queries Qa = [q, 1, 1, 0...] and keys Ka = [-2x, hi(|x|^2), lo(|x|^2), 0...]
//    (64 columns), so one K=64 dot product gives the query-invariant score
//    s_ij = |x_j|^2 - 2 q_i.x_j = d^2_ij - |q_i|^2.
// 2. candidates (tcgen05): each persistent CTA owns a PAIR of 128-query tiles (M = 2 x 128,
//    resident in smem) and streams every 128-key tile through a 4-stage TMA pipeline; one
//    thread issues 2 x 8 tcgen05.mma.kind::tf32 (128x128x8) per key tile into a double-
//    buffered TMEM accumulator (4 x 128 of the 512 columns).  Eight epilogue warps own one
//    query row each and keep a register-resident sorted top-KC list; a 32-wide min filter
//    against the list's current worst score skips almost every chunk, so the epilogue
//    stays under the tensor time.
// 3. rerank: one warp per query recomputes exact FP32 squared distances of the KC
//    candidates, sorts by (distance, index) and keeps k (self included).
#include <vector>
#include "tc_common.cuh"

namespace scb {

constexpr int kKnnThreads = 320;  // warp0 TMA, warp1 MMA, warps 2..9 epilogue
constexpr int kD = 64;            // padded embedding width (two 128-byte K atoms)

template <int KC>
struct KnnCfg {
  static constexpr int BM = 128, BN = 128, STAGES = 3;
  static constexpr int HALF = BM * 32 * 4;             // 16 KB: 128 rows x 32 fp32 (one K atom column)
  static constexpr int A_BYTES = 2 * 2 * HALF;          // 2 query tiles x 2 K halves = 64 KB
  static constexpr int B_BYTES = 2 * HALF;              // 128 keys x 64 = 32 KB per stage
  static constexpr int SPILL = 8 * 32 * 32 * 4;          // per-epilogue-warp chunk staging (32 KB)
  static constexpr int SMEM = A_BYTES + STAGES * B_BYTES + SPILL + 1024 + 256;
  static constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN, false, false);
};

// queries: [q, 1, 1, 0...]; keys: [-2x, hi(|x|^2), lo(|x|^2), 0...]  (64 columns, fp32)
__global__ void knn_prep_kernel(const float* __restrict__ X, int64_t n, int d, int ld, int is_key,
                                float* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (r >= n) return;
  const int l = lane_id();
  const float* x = X + r * ld;
  const float a = (l < d) ? x[l] : 0.0f;
  const float b = (l + 32 < d) ? x[l + 32] : 0.0f;
  float* o = out + r * kD;
  if (!is_key) {
    auto val = [&](int col, float xv) { return col < d ? xv : ((col == d || col == d + 1) ? 1.0f : 0.0f); };
    o[l] = val(l, a);
    o[l + 32] = val(l + 32, b);
  } else {
    const double nrm = warp_sum((double)a * a + (double)b * b);
    float hi, lo;
    tc::split_tf32((float)nrm, hi, lo);
    lo = (float)(nrm - (double)hi);
    auto val = [&](int col, float xv) { return col < d ? -2.0f * xv : (col == d ? hi : (col == d + 1 ? lo : 0.0f)); };
    o[l] = val(l, a);
    o[l + 32] = val(l + 32, b);
  }
}

template <int KC>
__device__ __forceinline__ void list_insert(float (&L)[KC], int (&I)[KC], float v, int iv) {
#pragma unroll
  for (int j = KC - 1; j > 0; --j) {
    const bool shift = L[j - 1] > v;
    const bool place = !shift && L[j] > v;
    L[j] = shift ? L[j - 1] : (place ? v : L[j]);
    I[j] = shift ? I[j - 1] : (place ? iv : I[j]);
  }
  if (L[0] > v) {
    L[0] = v;
    I[0] = iv;
  }
}

template <int KC>
__global__ void __launch_bounds__(kKnnThreads, 1)
knn_candidates_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk, int64_t n_q,
                      int64_t n_k, int* __restrict__ cand) {
  using C = KnnCfg<KC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_base = smem;                          // [qtile][khalf][128 rows x 128 B]
  uint8_t* b_base = smem + C::A_BYTES;             // [stage][khalf][128 rows x 128 B]
  float* spill = reinterpret_cast<float*>(b_base + C::STAGES * C::B_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(b_base + C::STAGES * C::B_BYTES + C::SPILL);
  uint64_t* a_full = bar;
  uint64_t* a_empty = bar + 1;
  uint64_t* b_full = bar + 2;
  uint64_t* b_empty = b_full + C::STAGES;
  uint64_t* t_full = b_empty + C::STAGES;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = warp_id(), lane = lane_id();
  const int n_pairs = (int)((n_q + 2 * C::BM - 1) / (2 * C::BM));
  const int n_kt = (int)((n_k + C::BN - 1) / C::BN);

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tq);
      tc::tma_prefetch(&tk);
      tc::mbar_init(a_full, 1);
      tc::mbar_init(a_empty, 1);
      for (int s = 0; s < C::STAGES; ++s) {
        tc::mbar_init(&b_full[s], 1);
        tc::mbar_init(&b_empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&t_full[b], 1);
        tc::mbar_init(&t_empty[b], 8);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, pc = 0;
      for (int pair = blockIdx.x; pair < n_pairs; pair += gridDim.x, ++pc) {
        tc::mbar_wait(a_empty, (pc & 1) ^ 1);
        tc::mbar_arrive_expect_tx(a_full, C::A_BYTES);
        for (int t = 0; t < 2; ++t)
          for (int h = 0; h < 2; ++h)
            tc::tma_load_2d(a_base + (t * 2 + h) * C::HALF, &tq, a_full, h * 32, (pair * 2 + t) * C::BM);
        for (int kt = 0; kt < n_kt; ++kt, ++it) {
          const int s = it % C::STAGES;
          tc::mbar_wait(&b_empty[s], ((it / C::STAGES) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&b_full[s], C::B_BYTES);
          uint8_t* b = b_base + s * C::B_BYTES;
          tc::tma_load_2d(b, &tk, &b_full[s], 0, kt * C::BN);
          tc::tma_load_2d(b + C::HALF, &tk, &b_full[s], 32, kt * C::BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, pc = 0;
      for (int pair = blockIdx.x; pair < n_pairs; pair += gridDim.x, ++pc) {
        tc::mbar_wait(a_full, pc & 1);
        for (int kt = 0; kt < n_kt; ++kt, ++it) {
          const int s = it % C::STAGES;
          const int buf = it & 1;
          tc::mbar_wait(&t_empty[buf], ((it >> 1) & 1) ^ 1);
          tc::mbar_wait(&b_full[s], (it / C::STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t bb = tc::smem_u32(b_base + s * C::B_BYTES);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t ab = tc::smem_u32(a_base + t * 2 * C::HALF);
            const uint32_t d = tmem + buf * 256 + t * 128;
#pragma unroll
            for (int kk = 0; kk < kD / 8; ++kk) {
              const uint32_t off = (kk >> 2) * C::HALF + (kk & 3) * 32;
              tc::mma_tf32(d, tc::smem_desc_sw128(ab + off, 16, 1024), tc::smem_desc_sw128(bb + off, 16, 1024),
                           C::IDESC, kk > 0 ? 1u : 0u);
            }
          }
          tc::mma_commit(&b_empty[s]);
          tc::mma_commit(&t_full[buf]);
        }
        tc::mma_commit(a_empty);
      }
    }
  } else {
    const int e = warp - 2;       // 0..7
    const int q = warp & 3;       // TMEM lane quarter
    const int t = e >> 2;         // query tile of the pair
    int it = 0;
    for (int pair = blockIdx.x; pair < n_pairs; pair += gridDim.x) {
      float L[KC];
      int I[KC];
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        L[j] = INFINITY;
        I[j] = -1;
      }
      const int64_t row = (int64_t)(pair * 2 + t) * C::BM + 32 * q + lane;
      for (int kt = 0; kt < n_kt; ++kt, ++it) {
        const int buf = it & 1;
        tc::mbar_wait(&t_full[buf], (it >> 1) & 1);
        tc::tc_fence_after();
        const int key0 = kt * C::BN;
        const bool tail = key0 + C::BN > n_k;
#pragma unroll 1
        for (int c = 0; c < C::BN / 32; ++c) {
          uint32_t r[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + buf * 256 + t * 128 + c * 32, r);
          tc::tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (tail) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (key0 + c * 32 + j >= n_k) v[j] = INFINITY;
          }
          float m = v[0];
#pragma unroll
          for (int j = 1; j < 32; ++j) m = fminf(m, v[j]);
          if (__any_sync(0xffffffffu, m < L[KC - 1])) {
            // rare path: stage the chunk (transposed: conflict-free) and walk it with ONE
            // rolled loop around a single inlined insertion (keeps the I-cache footprint small)
            float* sp = spill + e * 32 * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j) sp[j * 32 + lane] = v[j];
            __syncwarp();
#pragma unroll 1
            for (int j = 0; j < 32; ++j) {
              const float x = sp[j * 32 + lane];
              const bool ins = x < L[KC - 1];
              if (__any_sync(0xffffffffu, ins)) {
                if (ins) list_insert<KC>(L, I, x, key0 + c * 32 + j);
              }
            }
            __syncwarp();
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&t_empty[buf]);
      }
      if (row < n_q) {
        int* o = cand + row * KC;
#pragma unroll
        for (int j = 0; j < KC; ++j) o[j] = I[j];
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// one warp per query: exact fp32 distances of the candidates, bitonic sort by (d2, idx)
template <int KC>
__global__ void knn_rerank_kernel(const float* __restrict__ Q, const float* __restrict__ Kx, int64_t n_q, int d,
                                  int ld, const int* __restrict__ cand, int k, int* __restrict__ out_i,
                                  float* __restrict__ out_d) {
  constexpr int PER = KC / 32;  // candidates per lane (KC in {32, 64})
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (r >= n_q) return;
  const int l = lane_id();
  const float* qp = Q + r * ld;
  const float qa = (l < d) ? qp[l] : 0.0f;
  const float qb = (l + 32 < d) ? qp[l + 32] : 0.0f;
  float dd[PER];
  int ii[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = cand[r * KC + p * 32 + l];
    ii[p] = c;
    dd[p] = INFINITY;
  }
  // each candidate's distance computed cooperatively: lanes hold query dims l and l+32
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    for (int j = 0; j < 32; ++j) {
      const int c = __shfl_sync(0xffffffffu, ii[p], j);
      float s = 0.0f;
      if (c >= 0) {
        const float* xp = Kx + (int64_t)c * ld;
        const float da = (l < d) ? qa - xp[l] : 0.0f;
        const float db = (l + 32 < d) ? qb - xp[l + 32] : 0.0f;
        s = fmaf(da, da, db * db);
      }
      s = warp_sum(s);
      if (l == j) dd[p] = (c >= 0) ? s : INFINITY;
    }
  }
  // bitonic sort of KC (d, idx) pairs ascending; element e = p*32 + lane
  auto less = [](float da, int ia, float db, int ib) {
    return da < db || (da == db && (unsigned)ia < (unsigned)ib);
  };
#pragma unroll
  for (int size = 2; size <= KC; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int e = p * 32 + l;
        const int partner = e ^ stride;
        float od;
        int oi;
        if (stride >= 32) {  // partner in another register slot, same lane
          od = dd[p ^ (stride >> 5)];
          oi = ii[p ^ (stride >> 5)];
        } else {
          od = __shfl_xor_sync(0xffffffffu, dd[p], stride);
          oi = __shfl_xor_sync(0xffffffffu, ii[p], stride);
        }
        const bool up = ((e & size) == 0);
        const bool lower = e < partner;
        const bool mine_less = less(dd[p], ii[p], od, oi);
        const bool keep = (lower == up) ? mine_less : !mine_less;
        if (stride >= 32) {
          // both slots handled when p is the lower slot; write after computing both
          if ((p & (stride >> 5)) == 0) {
            const int pq = p ^ (stride >> 5);
            const float d0 = dd[p], d1 = dd[pq];
            const int i0 = ii[p], i1 = ii[pq];
            const bool lt = less(d0, i0, d1, i1);
            const bool swp = up ? !lt : lt;
            dd[p] = swp ? d1 : d0;
            ii[p] = swp ? i1 : i0;
            dd[pq] = swp ? d0 : d1;
            ii[pq] = swp ? i0 : i1;
          }
        } else if (!keep) {
          dd[p] = od;
          ii[p] = oi;
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int e = p * 32 + l;
    if (e < k) {
      out_i[r * k + e] = ii[p];
      out_d[r * k + e] = sqrtf(fmaxf(dd[p], 0.0f));
    }
  }
}

template <int KC>
static int launch_candidates(scb_ctx* ctx, const float* Qa, int64_t n_q, const float* Ka, int64_t n_k, int* cand,
                             cudaStream_t s) {
  using Cfg = KnnCfg<KC>;
  CUtensorMap tq, tk;
  SCB_TRY(make_tmap_2d_f32(&tq, Qa, (uint64_t)n_q, kD, kD, 32, Cfg::BM));
  SCB_TRY(make_tmap_2d_f32(&tk, Ka, (uint64_t)n_k, kD, kD, 32, Cfg::BN));
  auto kern = knn_candidates_kernel<KC>;
  SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int n_pairs = (int)((n_q + 2 * Cfg::BM - 1) / (2 * Cfg::BM));
  kern<<<std::min(n_pairs, ctx->num_sms), kKnnThreads, Cfg::SMEM, s>>>(tq, tk, n_q, n_k, cand);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_knn_prep(scb_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t ld, int32_t is_key, float* out,
                            void* stream) {
  SCB_REQUIRE(ctx && X && out, SCB_ERR_ARG, "scb_knn_prep: null argument");
  SCB_REQUIRE(d >= 1 && d <= kD - 2 && ld >= d, SCB_ERR_ARG, "scb_knn_prep: need 1 <= d <= %d and ld >= d", kD - 2);
  SCB_REQUIRE(((uintptr_t)out & 15) == 0, SCB_ERR_ARG, "scb_knn_prep: out must be 16-byte aligned");
  if (n == 0) return SCB_OK;
  knn_prep_kernel<<<ceil_div(n, 8), 256, 0, (cudaStream_t)stream>>>(X, n, d, ld, is_key ? 1 : 0, out);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_knn_candidates(scb_ctx* ctx, const float* Qa, int64_t n_q, const float* Ka, int64_t n_k,
                                  int32_t k_cand, int32_t* cand, void* stream) {
  SCB_REQUIRE(ctx && Qa && Ka && cand, SCB_ERR_ARG, "scb_knn_candidates: null argument");
  SCB_REQUIRE(k_cand == 32 || k_cand == 64, SCB_ERR_ARG, "scb_knn_candidates: k_cand must be 32 or 64");
  SCB_REQUIRE(n_k < (1ll << 31) && n_q < (1ll << 31), SCB_ERR_ARG, "scb_knn_candidates: too many rows");
  if (n_q == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  return k_cand == 32 ? launch_candidates<32>(ctx, Qa, n_q, Ka, n_k, cand, s)
                      : launch_candidates<64>(ctx, Qa, n_q, Ka, n_k, cand, s);
}

extern "C" int scb_knn_rerank(scb_ctx* ctx, const float* queries, int64_t n_q, const float* keys, int32_t d, int32_t ld,
                              const int32_t* cand, int32_t k_cand, int32_t k, int32_t* knn_index, float* knn_dist,
                              void* stream) {
  SCB_REQUIRE(ctx && queries && keys && cand && knn_index && knn_dist, SCB_ERR_ARG, "scb_knn_rerank: null argument");
  SCB_REQUIRE(k >= 1 && k <= k_cand && (k_cand == 32 || k_cand == 64), SCB_ERR_ARG, "scb_knn_rerank: bad k / k_cand");
  if (n_q == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (k_cand == 32)
    knn_rerank_kernel<32><<<ceil_div(n_q, 8), 256, 0, s>>>(queries, keys, n_q, d, ld, cand, k, knn_index, knn_dist);
  else
    knn_rerank_kernel<64><<<ceil_div(n_q, 8), 256, 0, s>>>(queries, keys, n_q, d, ld, cand, k, knn_index, knn_dist);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_knn(scb_ctx* ctx, const float* queries, int64_t n_queries, const float* keys, int64_t n_keys,
                       int32_t d, int32_t ld, int32_t k, int32_t k_cand, int32_t* knn_index, float* knn_dist,
                       void* stream) {
  SCB_REQUIRE(ctx && queries && keys && knn_index && knn_dist, SCB_ERR_ARG, "scb_knn: null argument");
  SCB_REQUIRE(d >= 1 && d <= kD - 2 && ld >= d, SCB_ERR_ARG, "scb_knn: need 1 <= d <= %d and ld >= d", kD - 2);
  SCB_REQUIRE(k >= 1 && k <= 64 && k <= n_keys, SCB_ERR_ARG, "scb_knn: need 1 <= k <= min(64, n_keys)");
  SCB_REQUIRE(k_cand >= k && (k_cand == 32 || k_cand == 64), SCB_ERR_ARG, "scb_knn: k_cand must be 32 or 64 and >= k");
  SCB_REQUIRE(n_keys < (1ll << 31) && n_queries < (1ll << 31), SCB_ERR_ARG, "scb_knn: too many rows");
  if (n_queries == 0) return SCB_OK;
  void* ws;
  const size_t qa = (size_t)n_queries * kD * 4, ka = (size_t)n_keys * kD * 4, cb = (size_t)n_queries * k_cand * 4;
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  SCB_TRY(ws_get(ctx, 0, up(qa) + up(ka) + up(cb), &ws, (cudaStream_t)stream));
  float* Qa = (float*)ws;
  float* Ka = (float*)((char*)ws + up(qa));
  int* cand = (int*)((char*)Ka + up(ka));
  SCB_TRY(scb_knn_prep(ctx, queries, n_queries, d, ld, 0, Qa, stream));
  SCB_TRY(scb_knn_prep(ctx, keys, n_keys, d, ld, 1, Ka, stream));
  SCB_TRY(scb_knn_candidates(ctx, Qa, n_queries, Ka, n_keys, k_cand, cand, stream));
  return scb_knn_rerank(ctx, queries, n_queries, keys, d, ld, cand, k_cand, k, knn_index, knn_dist, stream);
}

// PCA projection X_pca = (Z - m) V on tcgen05 (HBM-bound: streams Z once).
//
// A = Z row block (M = 128 cells, K = genes, K-major), B = V^T (N = n_comps_pad <= 256
// components, K-major).  Persistent CTAs (one per SM) walk 128-cell tiles; warp 0 issues
// TMA loads of [128 cells x 32 genes] Z boxes plus the pre-split V^T hi/lo boxes, warps
// 2-5 split Z into TF32 hi (in place) + lo, warp 1 issues 3 tcgen05.mma.kind::tf32 per
// 8-gene step (3xTF32), and warps 6-9 drain the double-buffered TMEM accumulator,
// subtract the centring shift s = m V, and store the embedding rows.
#include <vector>
#include <cuda_bf16.h>
#include "planes_fmt.cuh"
#include "tc_common.cuh"

namespace scb {

constexpr int kProjThreads = 320;

template <int NP>
struct ProjCfg {
  static constexpr int BM = 128, KB = 32, STAGES = NP <= 64 ? 4 : 3;
  static constexpr int A_BYTES = BM * KB * 4;   // 16 KB
  static constexpr int B_BYTES = NP * KB * 4;   // per hi / lo
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // Ahi | Alo | Bhi | Blo
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t IDESC = tc::idesc_tf32(BM, NP, false, false);
  static constexpr int TMEM_COLS = 2 * NP < 32 ? 32 : 2 * NP;
};

template <int NP>
__global__ void __launch_bounds__(kProjThreads, 1)
project_kernel(const __grid_constant__ CUtensorMap tz, const __grid_constant__ CUtensorMap tvh,
               const __grid_constant__ CUtensorMap tvl, int64_t n_rows, int hp, const float* __restrict__ shift,
               int n_comps, float* __restrict__ out, int ld_out) {
  using C = ProjCfg<NP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* conv = full + C::STAGES;
  uint64_t* empty = conv + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = warp_id(), lane = lane_id();
  const int n_tiles = (int)((n_rows + C::BM - 1) / C::BM);
  const int nkb = hp / C::KB;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tz);
      tc::tma_prefetch(&tvh);
      tc::tma_prefetch(&tvl);
      for (int s = 0; s < C::STAGES; ++s) {
        tc::mbar_init(&full[s], 1);
        tc::mbar_init(&conv[s], 4);
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&tfull[b], 1);
        tc::mbar_init(&tempty[b], 4);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          tc::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[s], C::A_BYTES + 2 * C::B_BYTES);
          tc::tma_load_2d(st, &tz, &full[s], kb * C::KB, tile * C::BM);
          tc::tma_load_2d(st + 2 * C::A_BYTES, &tvh, &full[s], kb * C::KB, 0);
          tc::tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &tvl, &full[s], kb * C::KB, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        const int buf = tcount & 1;
        tc::mbar_wait(&tempty[buf], ((tcount >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + buf * NP;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          tc::mbar_wait(&conv[s], ph);
          tc::tc_fence_after();
          const uint32_t ah = tc::smem_u32(smem + s * C::STAGE_BYTES);
          const uint32_t al = ah + C::A_BYTES;
          const uint32_t bh = ah + 2 * C::A_BYTES;
          const uint32_t bl = bh + C::B_BYTES;
#pragma unroll
          for (int k = 0; k < C::KB / 8; ++k) {
            const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along the swizzled 128-byte row
            const uint64_t dah = tc::smem_desc_sw128(ah + off, 16, 1024);
            const uint64_t dal = tc::smem_desc_sw128(al + off, 16, 1024);
            const uint64_t dbh = tc::smem_desc_sw128(bh + off, 16, 1024);
            const uint64_t dbl = tc::smem_desc_sw128(bl + off, 16, 1024);
            tc::mma_tf32(d, dah, dbh, C::IDESC, (kb > 0 || k > 0) ? 1u : 0u);
            tc::mma_tf32(d, dah, dbl, C::IDESC, 1u);
            tc::mma_tf32(d, dal, dbh, C::IDESC, 1u);
          }
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
  } else if (warp < 6) {
    const int ct = threadIdx.x - 64;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (it / C::STAGES) & 1;
        tc::mbar_wait(&full[s], ph);
        float4* h = reinterpret_cast<float4*>(smem + s * C::STAGE_BYTES);
        float4* l = h + C::A_BYTES / 16;
#pragma unroll 4
        for (int v = ct; v < C::A_BYTES / 16; v += 128) {
          float4 x = h[v], xh, xl;
          tc::split_tf32(x.x, xh.x, xl.x);
          tc::split_tf32(x.y, xh.y, xl.y);
          tc::split_tf32(x.z, xh.z, xl.z);
          tc::split_tf32(x.w, xh.w, xl.w);
          h[v] = xh;
          l[v] = xl;
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&conv[s]);
      }
    }
  } else {
    const int q = warp & 3;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
      const int buf = tcount & 1;
      tc::mbar_wait(&tfull[buf], (tcount >> 1) & 1);
      tc::tc_fence_after();
      const int64_t row = (int64_t)tile * C::BM + 32 * q + lane;
#pragma unroll 1
      for (int c = 0; c < NP / 32; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + buf * NP + c * 32, r);
        tc::tmem_ld_wait();
        if (row < n_rows) {
          float* o = out + row * ld_out + c * 32;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const int cj = c * 32 + j;
            float4 v;
            v.x = (cj + 0 < n_comps) ? __uint_as_float(r[j + 0]) - shift[cj + 0] : 0.0f;
            v.y = (cj + 1 < n_comps) ? __uint_as_float(r[j + 1]) - shift[cj + 1] : 0.0f;
            v.z = (cj + 2 < n_comps) ? __uint_as_float(r[j + 2]) - shift[cj + 2] : 0.0f;
            v.w = (cj + 3 < n_comps) ? __uint_as_float(r[j + 3]) - shift[cj + 3] : 0.0f;
            if (cj < ld_out) *reinterpret_cast<float4*>(o + j) = v;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[buf]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// V^T [np][hp] -> (hi, lo) TF32 split, and shift[j] = sum_g m_g V[g][j] (fp64 accumulate)
__global__ void split_vt_kernel(const float* __restrict__ vt, const float* __restrict__ mean, int np, int hp,
                                float* __restrict__ vh, float* __restrict__ vl, float* __restrict__ shift) {
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int g = threadIdx.x; g < hp; g += blockDim.x) {
    const float v = vt[(size_t)j * hp + g];
    float h, l;
    tc::split_tf32(v, h, l);
    vh[(size_t)j * hp + g] = h;
    vl[(size_t)j * hp + g] = l;
    acc += (double)mean[g] * (double)v;
  }
  __shared__ double sb[32];
  acc = warp_sum(acc);
  if (lane_id() == 0) sb[warp_id()] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sb[w];
    shift[j] = (float)t;
  }
}

template <int NP>
static int launch_project(scb_ctx* ctx, const float* Z, int64_t n_rows, int hp, const float* vh, const float* vl,
                          const float* shift, int n_comps, float* out, int ld_out, cudaStream_t s) {
  using Cfg = ProjCfg<NP>;
  CUtensorMap tz, tvh, tvl;
  SCB_TRY(make_tmap_2d_f32(&tz, Z, (uint64_t)n_rows, hp, hp, 32, Cfg::BM));
  SCB_TRY(make_tmap_2d_f32(&tvh, vh, NP, hp, hp, 32, NP));
  SCB_TRY(make_tmap_2d_f32(&tvl, vl, NP, hp, hp, 32, NP));
  auto kern = project_kernel<NP>;
  SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int n_tiles = (int)((n_rows + Cfg::BM - 1) / Cfg::BM);
  const int grid = std::min(n_tiles, ctx->num_sms);
  kern<<<grid, kProjThreads, Cfg::SMEM, s>>>(tz, tvh, tvl, n_rows, hp, shift, n_comps, out, ld_out);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

// ---- variant fed by the BF16 planes of Z (written directly by scb_scale_dense_planes): the
// operands arrive by TMA in the K-major 128-byte-swizzled layout with no converter warps; per
// 16-gene K step three kind::f16 MMAs hi*Vhi + hi*Vlo + lo*Vhi (3xBF16, <= 2^-16 per product,
// the Gram's scheme).  V^T is split into BF16 planes by split_vt_bf16_kernel.
constexpr int kProjPThreads = 192;  // warp0 TMA, warp1 MMA, warps 2-5 epilogue
template <int NP>
struct ProjPCfg {
  static constexpr int BM = 128, KB = 64, STAGES = NP <= 64 ? 4 : 3;
  static constexpr int A_BYTES = BM * KB * 2;   // 16 KB per plane
  static constexpr int B_BYTES = NP * KB * 2;   // per plane
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // Ahi | Alo | Bhi | Blo
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t IDESC = tc::SCB_PLANES_IDESC(BM, NP, false, false);
  static constexpr int TMEM_COLS = 2 * NP < 32 ? 32 : 2 * NP;
};

template <int NP>
__global__ void __launch_bounds__(kProjPThreads, 1)
project_planes_kernel(const __grid_constant__ CUtensorMap tzh, const __grid_constant__ CUtensorMap tzl,
                      const __grid_constant__ CUtensorMap tvh, const __grid_constant__ CUtensorMap tvl, int64_t n_rows,
                      int hp, const float* __restrict__ shift, int n_comps, float* __restrict__ out, int ld_out) {
  using C = ProjPCfg<NP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = warp_id(), lane = lane_id();
  const int n_tiles = (int)((n_rows + C::BM - 1) / C::BM);
  const int nkb = hp / C::KB;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tzh);
      tc::tma_prefetch(&tzl);
      tc::tma_prefetch(&tvh);
      tc::tma_prefetch(&tvl);
      for (int s = 0; s < C::STAGES; ++s) {
        tc::mbar_init(&full[s], 1);
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&tfull[b], 1);
        tc::mbar_init(&tempty[b], 4);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          tc::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * C::STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          tc::tma_load_2d(st, &tzh, &full[s], kb * C::KB, tile * C::BM);
          tc::tma_load_2d(st + C::A_BYTES, &tzl, &full[s], kb * C::KB, tile * C::BM);
          tc::tma_load_2d(st + 2 * C::A_BYTES, &tvh, &full[s], kb * C::KB, 0);
          tc::tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &tvl, &full[s], kb * C::KB, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        const int buf = tcount & 1;
        tc::mbar_wait(&tempty[buf], ((tcount >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + buf * NP;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          tc::mbar_wait(&full[s], ph);
          tc::tc_fence_after();
          const uint32_t ah = tc::smem_u32(smem + s * C::STAGE_BYTES);
          const uint32_t al = ah + C::A_BYTES;
          const uint32_t bh = ah + 2 * C::A_BYTES;
          const uint32_t bl = bh + C::B_BYTES;
#pragma unroll
          for (int k = 0; k < C::KB / 16; ++k) {
            const uint32_t off = k * 32;  // 16 bf16 = 32 bytes along the swizzled 128-byte row
            const uint64_t dah = tc::smem_desc_sw128(ah + off, 16, 1024);
            const uint64_t dal = tc::smem_desc_sw128(al + off, 16, 1024);
            const uint64_t dbh = tc::smem_desc_sw128(bh + off, 16, 1024);
            const uint64_t dbl = tc::smem_desc_sw128(bl + off, 16, 1024);
            tc::mma_f16(d, dah, dbh, C::IDESC, (kb > 0 || k > 0) ? 1u : 0u);
            tc::mma_f16(d, dah, dbl, C::IDESC, 1u);
            tc::mma_f16(d, dal, dbh, C::IDESC, 1u);
          }
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int q = warp & 3;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
      const int buf = tcount & 1;
      tc::mbar_wait(&tfull[buf], (tcount >> 1) & 1);
      tc::tc_fence_after();
      const int64_t row = (int64_t)tile * C::BM + 32 * q + lane;
#pragma unroll 1
      for (int c = 0; c < NP / 32; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + buf * NP + c * 32, r);
        tc::tmem_ld_wait();
        if (row < n_rows) {
          float* o = out + row * ld_out + c * 32;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const int cj = c * 32 + j;
            float4 v;
            v.x = (cj + 0 < n_comps) ? __uint_as_float(r[j + 0]) - shift[cj + 0] : 0.0f;
            v.y = (cj + 1 < n_comps) ? __uint_as_float(r[j + 1]) - shift[cj + 1] : 0.0f;
            v.z = (cj + 2 < n_comps) ? __uint_as_float(r[j + 2]) - shift[cj + 2] : 0.0f;
            v.w = (cj + 3 < n_comps) ? __uint_as_float(r[j + 3]) - shift[cj + 3] : 0.0f;
            if (cj < ld_out) *reinterpret_cast<float4*>(o + j) = v;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[buf]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// V^T [np][hp] -> BF16 planes (hi = bf16(v), lo = bf16(v - hi)) and shift[j] = sum_g m_g V[g][j]
__global__ void split_vt_bf16_kernel(const float* __restrict__ vt, const float* __restrict__ mean, int np, int hp,
                                     __nv_bfloat16* __restrict__ vh, __nv_bfloat16* __restrict__ vl,
                                     float* __restrict__ shift) {
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int g = threadIdx.x; g < hp; g += blockDim.x) {
    const float v = vt[(size_t)j * hp + g];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    vh[(size_t)j * hp + g] = h;
    vl[(size_t)j * hp + g] = __float2bfloat16_rn(v - __bfloat162float(h));
    acc += (double)mean[g] * (double)v;
  }
  __shared__ double sb[32];
  acc = warp_sum(acc);
  if (lane_id() == 0) sb[warp_id()] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sb[w];
    shift[j] = (float)t;
  }
}

template <int NP>
static int launch_project_planes(scb_ctx* ctx, const uint16_t* Zhi, const uint16_t* Zlo, int64_t n_rows, int hp,
                                 const __nv_bfloat16* vh, const __nv_bfloat16* vl, const float* shift, int n_comps,
                                 float* out, int ld_out, cudaStream_t s) {
  using Cfg = ProjPCfg<NP>;
  CUtensorMap tzh, tzl, tvh, tvl;
  SCB_TRY(make_tmap_2d(&tzh, Zhi, (uint64_t)n_rows, hp, hp, 2, 64, Cfg::BM));
  SCB_TRY(make_tmap_2d(&tzl, Zlo, (uint64_t)n_rows, hp, hp, 2, 64, Cfg::BM));
  SCB_TRY(make_tmap_2d(&tvh, vh, NP, hp, hp, 2, 64, NP));
  SCB_TRY(make_tmap_2d(&tvl, vl, NP, hp, hp, 2, 64, NP));
  auto kern = project_planes_kernel<NP>;
  SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int n_tiles = (int)((n_rows + Cfg::BM - 1) / Cfg::BM);
  const int grid = std::min(n_tiles, ctx->num_sms);
  kern<<<grid, kProjPThreads, Cfg::SMEM, s>>>(tzh, tzl, tvh, tvl, n_rows, hp, shift, n_comps, out, ld_out);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_project(scb_ctx* ctx, const float* Z, int64_t n_rows, int32_t hp, const float* components_t,
                           const float* col_mean, int32_t n_comps, int32_t n_comps_pad, float* X_pca, int32_t ld_out,
                           void* stream) {
  SCB_REQUIRE(ctx && Z && components_t && col_mean && X_pca, SCB_ERR_ARG, "scb_project: null argument");
  SCB_REQUIRE(hp % 32 == 0 && hp > 0, SCB_ERR_ARG, "scb_project: hp must be a multiple of 32");
  SCB_REQUIRE(n_comps_pad == 64 || n_comps_pad == 128, SCB_ERR_UNSUPPORTED, "scb_project: n_comps_pad must be 64 or 128");
  SCB_REQUIRE(n_comps <= n_comps_pad && ld_out % 4 == 0 && ld_out >= n_comps, SCB_ERR_ARG, "scb_project: bad n_comps/ld_out");
  if (n_rows == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  const size_t vbytes = (size_t)n_comps_pad * hp * 4;
  SCB_TRY(ws_get(ctx, 3, 2 * vbytes + 1024 + 256, &ws, s));
  float* vh = (float*)ws;
  float* vl = (float*)((char*)ws + vbytes);
  float* shift = (float*)((char*)ws + 2 * vbytes);
  split_vt_kernel<<<n_comps_pad, 256, 0, s>>>(components_t, col_mean, n_comps_pad, hp, vh, vl, shift);
  SCB_LAUNCH_CHECK();
  if (n_comps_pad == 64) return launch_project<64>(ctx, Z, n_rows, hp, vh, vl, shift, n_comps, X_pca, ld_out, s);
  return launch_project<128>(ctx, Z, n_rows, hp, vh, vl, shift, n_comps, X_pca, ld_out, s);
}

extern "C" int scb_project_planes(scb_ctx* ctx, const uint16_t* Z_hi, const uint16_t* Z_lo, int64_t n_rows, int32_t hp,
                                  const float* components_t, const float* col_mean, int32_t n_comps,
                                  int32_t n_comps_pad, float* X_pca, int32_t ld_out, void* stream) {
  SCB_REQUIRE(ctx && Z_hi && Z_lo && components_t && col_mean && X_pca, SCB_ERR_ARG, "scb_project_planes: null argument");
  SCB_REQUIRE(hp % 64 == 0 && hp > 0, SCB_ERR_ARG, "scb_project_planes: hp must be a multiple of 64");
  SCB_REQUIRE(n_comps_pad == 64 || n_comps_pad == 128, SCB_ERR_UNSUPPORTED,
              "scb_project_planes: n_comps_pad must be 64 or 128");
  SCB_REQUIRE(n_comps <= n_comps_pad && ld_out % 4 == 0 && ld_out >= n_comps, SCB_ERR_ARG,
              "scb_project_planes: bad n_comps/ld_out");
  if (n_rows == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  const size_t vbytes = (size_t)n_comps_pad * hp * 2;
  SCB_TRY(ws_get(ctx, 3, 2 * vbytes + 1024 + 256, &ws, s));
  __nv_bfloat16* vh = (__nv_bfloat16*)ws;
  __nv_bfloat16* vl = (__nv_bfloat16*)((char*)ws + vbytes);
  float* shift = (float*)((char*)ws + 2 * vbytes);
  split_vt_bf16_kernel<<<n_comps_pad, 256, 0, s>>>(components_t, col_mean, n_comps_pad, hp, vh, vl, shift);
  SCB_LAUNCH_CHECK();
  if (n_comps_pad == 64) return launch_project_planes<64>(ctx, Z_hi, Z_lo, n_rows, hp, vh, vl, shift, n_comps, X_pca, ld_out, s);
  return launch_project_planes<128>(ctx, Z_hi, Z_lo, n_rows, hp, vh, vl, shift, n_comps, X_pca, ld_out, s);
}

// PCA covariance: C = Z^T Z on the 5th-generation tensor cores.
//
// Z is the dense scaled HVG matrix [N cells][hp] (row-major fp32, hp % 128 == 0).  Both
// UMMA operands are column blocks of Z read MN-major (genes contiguous): A = Z[k, i-block]^T
// (M = 128 genes), B = Z[k, j-block]^T (N = BN genes), K = cells.  TMA brings [32 cells x
// 32 genes] boxes (128-byte swizzle with 32-byte atoms: the MN-major TF32 layout) into smem; four converter warps split every
// element into a TF32-exact high part (in place) and the fp32 remainder, and one thread
// issues three tcgen05.mma.kind::tf32 per 8-cell step (hi*hi + hi*lo + lo*hi, "3xTF32",
// ~fp32 accuracy) accumulating in TMEM.  Only tiles touching the upper triangle are
// computed; split-K over cells fills the 148 SMs, and a deterministic reduce kernel sums
// the K-slices and mirrors the result.
#include <vector>
#include "tc_common.cuh"

namespace scb {

constexpr int kGemmThreads = 192;  // warp0 TMA, warp1 MMA, warps 2..5 convert + epilogue

template <int BN, int STAGES>
struct GramCfg {
  static constexpr int BM = 128;
  static constexpr int KB = 16;                       // cells per stage (4-stage ring fits smem)
  static constexpr int A_BYTES = BM * KB * 4;         // 16 KB
  static constexpr int B_BYTES = BN * KB * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BOX = KB * 128;                // one [KB cells x 32 genes] TMA box = MN chunk stride (LBO)
  static constexpr int SMEM = 2 * STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN, true, true);
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
gram_kernel(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ tiles, int n_tiles, int64_t n_rows,
            int64_t rows_per_slice, int hp, float* __restrict__ partial) {
  using C = GramCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* hi_base = smem;                                   // [STAGES][A | B]
  uint8_t* lo_base = smem + STAGES * C::STAGE_BYTES;         // [STAGES][A | B]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * C::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = warp_id(), lane = lane_id();
  const int tile = blockIdx.x % n_tiles;
  const int slice = blockIdx.x / n_tiles;
  const int2 t = tiles[tile];
  const int i0 = t.x * C::BM, j0 = t.y * BN;
  const int64_t k_begin = (int64_t)slice * rows_per_slice;
  const int64_t k_end = min(n_rows, k_begin + rows_per_slice);
  const int num_kb = (k_end > k_begin) ? (int)((k_end - k_begin + C::KB - 1) / C::KB) : 0;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tmap);
      for (int s = 0; s < STAGES; ++s) {
        tc::mbar_init(&full[s], 1);
        tc::mbar_init(&conv[s], 4);
        tc::mbar_init(&empty[s], 1);
      }
      tc::mbar_init(done, 1);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<BN>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < num_kb; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        tc::mbar_wait(&empty[s], ph ^ 1);
        uint8_t* a = hi_base + s * C::STAGE_BYTES;
        uint8_t* b = a + C::A_BYTES;
        const int k0 = (int)(k_begin + (int64_t)it * C::KB);
        tc::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
        for (int c = 0; c < C::BM / 32; ++c) tc::tma_load_2d(a + c * C::BOX, &tmap, &full[s], i0 + 32 * c, k0);
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) tc::tma_load_2d(b + c * C::BOX, &tmap, &full[s], j0 + 32 * c, k0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int it = 0; it < num_kb; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        tc::mbar_wait(&conv[s], ph);
        tc::tc_fence_after();
        const uint32_t ah = tc::smem_u32(hi_base + s * C::STAGE_BYTES);
        const uint32_t bh = ah + C::A_BYTES;
        const uint32_t al = tc::smem_u32(lo_base + s * C::STAGE_BYTES);
        const uint32_t bl = al + C::A_BYTES;
#pragma unroll
        for (int k = 0; k < C::KB / 8; ++k) {
          // MN-major TF32: 128B_BASE32B layout, 4-cell atoms (SBO 512), 32-gene chunks 4 KB apart
          const uint32_t off = k * 1024;  // next 8 cells
          const uint64_t dah = tc::smem_desc_sw128_b32(ah + off, C::BOX, 512);
          const uint64_t dbh = tc::smem_desc_sw128_b32(bh + off, C::BOX, 512);
          const uint64_t dal = tc::smem_desc_sw128_b32(al + off, C::BOX, 512);
          const uint64_t dbl = tc::smem_desc_sw128_b32(bl + off, C::BOX, 512);
          const uint32_t acc0 = (it > 0 || k > 0) ? 1u : 0u;
          tc::mma_tf32(tmem, dah, dbh, C::IDESC, acc0);
          tc::mma_tf32(tmem, dah, dbl, C::IDESC, 1u);
          tc::mma_tf32(tmem, dal, dbh, C::IDESC, 1u);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(done);
    }
  } else {
    // ---- converters: split the freshly loaded stage into TF32 hi (in place) + lo
    const int ct = threadIdx.x - 64;  // 0..127
    for (int it = 0; it < num_kb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&full[s], ph);
      float4* h = reinterpret_cast<float4*>(hi_base + s * C::STAGE_BYTES);
      float4* l = reinterpret_cast<float4*>(lo_base + s * C::STAGE_BYTES);
#pragma unroll 4
      for (int v = ct; v < C::STAGE_BYTES / 16; v += 128) {
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
    // ---- epilogue: TMEM -> registers -> partial[slice] (rows i0.., cols j0..)
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = i0 + 32 * q + lane;
    float* out = partial + (size_t)slice * hp * hp + (size_t)row * hp + j0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + c * 32, r);
      tc::tmem_ld_wait();
      if (num_kb == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      float4* o4 = reinterpret_cast<float4*>(out + c * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        o4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                            __uint_as_float(r[4 * j + 3]));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<BN>(tmem);
}

// sum K-slices for i <= j, write C[i][j] and C[j][i] (fixed slice order: deterministic)
__global__ void gram_reduce_kernel(const float* __restrict__ partial, int slices, int hp, double* __restrict__ C) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= hp || j < i) return;
  double s = 0.0;
  for (int k = 0; k < slices; ++k) s += (double)partial[(size_t)k * hp * hp + (size_t)i * hp + j];
  C[(size_t)i * hp + j] = s;
  C[(size_t)j * hp + i] = s;
}

template <int BN, int STAGES>
static int launch_gram(scb_ctx* ctx, const float* Z, int64_t n_rows, int hp, double* C, cudaStream_t s) {
  using Cfg = GramCfg<BN, STAGES>;
  CUtensorMap tmap;
  SCB_TRY(make_tmap_2d_f32(&tmap, Z, (uint64_t)std::max<int64_t>(n_rows, 1), hp, hp, 32, Cfg::KB, /*atom32=*/true));
  // upper-triangle tile list
  std::vector<int2> tl;
  for (int bi = 0; bi < hp / Cfg::BM; ++bi)
    for (int bj = 0; bj < hp / BN; ++bj)
      if (bj * BN + BN - 1 >= bi * Cfg::BM) tl.push_back(make_int2(bi, bj));
  const int n_tiles = (int)tl.size();
  // K-slices: fill the SMs and keep each fp32 TMEM accumulation <= 64k cells (the slices
  // are summed in fp64), which bounds the fp32 accumulation error at ~1e-6 relative.
  const int64_t kbs = (n_rows + Cfg::KB - 1) / Cfg::KB;
  int64_t sl = std::max<int64_t>((ctx->num_sms + n_tiles - 1) / n_tiles, (n_rows + 65535) / 65536);
  const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(sl, kbs));
  const int64_t rows_per_slice = ((kbs + slices - 1) / slices) * Cfg::KB;
  const size_t part_bytes = (size_t)slices * hp * hp * 4;
  void* ws;
  SCB_TRY(ws_get(ctx, 0, part_bytes + n_tiles * sizeof(int2) + 256, &ws, s));
  float* partial = (float*)ws;
  int2* d_tiles = (int2*)((char*)ws + ((part_bytes + 255) / 256) * 256);
  SCB_CUDA(cudaMemcpyAsync(d_tiles, tl.data(), n_tiles * sizeof(int2), cudaMemcpyHostToDevice, s));
  auto kern = gram_kernel<BN, STAGES>;
  SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  kern<<<n_tiles * slices, kGemmThreads, Cfg::SMEM, s>>>(tmap, d_tiles, n_tiles, n_rows, rows_per_slice, hp, partial);
  SCB_LAUNCH_CHECK();
  dim3 g((hp + 255) / 256, hp);
  gram_reduce_kernel<<<g, 256, 0, s>>>(partial, slices, hp, C);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaStreamSynchronize(s));  // keeps the host tile list alive for the async copy
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_gram(scb_ctx* ctx, const float* Z, int64_t n_rows, int32_t hp, double* C, void* stream) {
  SCB_REQUIRE(ctx && Z && C, SCB_ERR_ARG, "scb_gram: null argument");
  SCB_REQUIRE(hp > 0 && hp % 128 == 0, SCB_ERR_ARG, "scb_gram: hp must be a multiple of 128");
  SCB_REQUIRE(n_rows >= 0 && n_rows < (1ll << 31), SCB_ERR_ARG, "scb_gram: n_rows out of range");
  cudaStream_t s = (cudaStream_t)stream;
  if (hp % 256 == 0) return launch_gram<256, 4>(ctx, Z, n_rows, hp, C, s);
  return launch_gram<128, 6>(ctx, Z, n_rows, hp, C, s);
}

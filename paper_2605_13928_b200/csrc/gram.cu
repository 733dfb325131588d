// PCA covariance: C = Z^T Z on the 5th-generation tensor cores.
//
// Z is the dense scaled HVG matrix [N cells][hp] (row-major fp32, hp % 128 == 0).  Both
// UMMA operands are column blocks of Z read MN-major (genes contiguous): A = Z[k, i-block]^T
// (M = 128 genes), B = Z[k, j-block]^T (N = BN genes), K = cells.  TMA brings fp32 [16 cells x
// 32 genes] boxes into an fp32 staging ring; eight converter warps split every element into
// BF16 hi = bf16(x) and lo = bf16(x - hi) (|x - hi - lo| <= 2^-17 |x|) written straight into the
// MN-major 128-byte-swizzled BF16 operand layout of a second ring; two threads (even / odd steps, one TMEM
// accumulator each) issue three tcgen05.mma.kind::f16 per 16-cell step (hi*hi + hi*lo + lo*hi, "3xBF16"; the dropped lo*lo
// term is <= 2^-16 relative) at the BF16 tensor rate (twice TF32's), accumulating in TMEM.
// Only tiles touching the upper triangle are computed; split-K over cells fills the 148 SMs,
// and a deterministic reduce kernel sums the K-slices in fp64 and mirrors the result.
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include "planes_fmt.cuh"
#include "tc_common.cuh"

namespace scb {

// t-th tile (row-major order) of the upper-triangle tile list: block row bi holds the column
// blocks bj with bj*BN + BN - 1 >= bi*BM.  Computed per CTA (a few iterations), so no host-built
// list has to be uploaded (and kept alive) per launch.
__device__ __forceinline__ int2 upper_tile(int t, int hp, int BM, int BN) {
  const int n_bi = hp / BM, n_bj = hp / BN;
  for (int bi = 0; bi < n_bi; ++bi) {
    const int lo = bi * BM - BN + 1;
    const int bj0 = lo <= 0 ? 0 : (lo + BN - 1) / BN;
    const int cnt = n_bj - bj0;
    if (t < cnt) return make_int2(bi, bj0 + t);
    t -= cnt;
  }
  return make_int2(0, 0);
}

constexpr int kConvWarps = 12;
constexpr int kConv0 = 3;                                   // first converter warp
constexpr int kGemmThreads = 32 * (kConv0 + kConvWarps);   // warp0 TMA, warps 1-2 MMA, converters (3..6 also epilogue)

template <int BN>
struct GramCfg {
  static constexpr int BM = 128;
  static constexpr int KB = 32;                       // cells per stage = two MMA K steps
  static constexpr int G = BM + BN;                   // genes per stage (A then B)
  static constexpr int F_BYTES = G * KB * 4;          // fp32 staging: G/32 TMA boxes of [KB x 32]
  static constexpr int BOX = KB * 128;                // one fp32 box, and one 64-gene BF16 chunk
  static constexpr int PLANE = G * KB * 2;            // one BF16 plane (A chunks then B chunks)
  static constexpr int C_BYTES = 2 * PLANE;           // hi + lo
  static constexpr int NF = 2, NC = 2;                // ring depths
  static constexpr int SMEM = NF * F_BYTES + NC * C_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t IDESC = tc::SCB_PLANES_IDESC(BM, BN, true, true);
};

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
gram_kernel(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ tiles, int n_tiles, int64_t n_rows,
            int64_t rows_per_slice, int hp, float* __restrict__ partial) {
  using C = GramCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* f_base = smem;                                    // [NF][G/32 boxes]
  uint8_t* c_base = smem + C::NF * C::F_BYTES;               // [NC][hi plane | lo plane]
  uint64_t* f_full = reinterpret_cast<uint64_t*>(c_base + C::NC * C::C_BYTES);
  uint64_t* f_empty = f_full + C::NF;
  uint64_t* c_full = f_empty + C::NF;
  uint64_t* c_empty = c_full + C::NC;
  uint64_t* done = c_empty + C::NC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = warp_id(), lane = lane_id();
  const int tile = blockIdx.x % n_tiles;
  const int slice = blockIdx.x / n_tiles;
  const int2 t = tiles ? tiles[tile] : upper_tile(tile, hp, C::BM, BN);
  const int i0 = t.x * C::BM, j0 = t.y * BN;
  const int64_t k_begin = (int64_t)slice * rows_per_slice;
  const int64_t k_end = min(n_rows, k_begin + rows_per_slice);
  const int num_kb = (k_end > k_begin) ? (int)((k_end - k_begin + C::KB - 1) / C::KB) : 0;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tmap);
      for (int s = 0; s < C::NF; ++s) {
        tc::mbar_init(&f_full[s], 1);
        tc::mbar_init(&f_empty[s], kConvWarps);
      }
      for (int s = 0; s < C::NC; ++s) {
        tc::mbar_init(&c_full[s], kConvWarps);
        tc::mbar_init(&c_empty[s], 1);
      }
      tc::mbar_init(done, 2);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<2 * BN>(tmem_slot);  // one accumulator per MMA issuer
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < num_kb; ++it) {
        const int s = it % C::NF;
        tc::mbar_wait(&f_empty[s], ((it / C::NF) & 1) ^ 1);
        uint8_t* f = f_base + s * C::F_BYTES;
        const int k0 = (int)(k_begin + (int64_t)it * C::KB);
        tc::mbar_arrive_expect_tx(&f_full[s], C::F_BYTES);
#pragma unroll
        for (int c = 0; c < C::BM / 32; ++c) tc::tma_load_2d(f + c * C::BOX, &tmap, &f_full[s], i0 + 32 * c, k0);
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)
          tc::tma_load_2d(f + (C::BM / 32 + c) * C::BOX, &tmap, &f_full[s], j0 + 32 * c, k0);
      }
    }
  } else if (warp <= 2) {
    // two issuers (stage parity p) into two accumulators: a tcgen05.commit stalls its thread until
    // the tensor pipe drains, so a single issuer committing every 3 MMAs leaves the pipe idle;
    // the epilogue adds the two accumulators (deterministic)
    const int p = warp - 1;
    if (lane == 0) {
      const uint32_t acc = tmem + p * BN;
      for (int it = p; it < num_kb; it += 2) {
        const int s = it % C::NC;
        tc::mbar_wait(&c_full[s], (it / C::NC) & 1);
        tc::tc_fence_after();
        // MN-major BF16, 128-byte swizzle: 64-gene chunks (LBO = chunk stride), 8-cell row
        // groups 1 KB apart (SBO)
        const uint32_t ah = tc::smem_u32(c_base + s * C::C_BYTES);
        const uint32_t bh = ah + (C::BM / 64) * C::BOX;
        const uint32_t al = ah + C::PLANE;
        const uint32_t bl = bh + C::PLANE;
#pragma unroll
        for (int kk = 0; kk < C::KB / 16; ++kk) {  // 16 cells = 16 rows of 128 B per K step
          const uint32_t ko = kk * 2048;
          const uint64_t dah = tc::smem_desc_sw128(ah + ko, C::BOX, 1024);
          const uint64_t dbh = tc::smem_desc_sw128(bh + ko, C::BOX, 1024);
          const uint64_t dal = tc::smem_desc_sw128(al + ko, C::BOX, 1024);
          const uint64_t dbl = tc::smem_desc_sw128(bl + ko, C::BOX, 1024);
          tc::mma_f16(acc, dah, dbh, C::IDESC, (it > p || kk > 0) ? 1u : 0u);
          tc::mma_f16(acc, dah, dbl, C::IDESC, 1u);
          tc::mma_f16(acc, dal, dbh, C::IDESC, 1u);
        }
        tc::mma_commit(&c_empty[s]);
      }
      tc::mma_commit(done);
    }
  } else {
    // ---- converters: fp32 stage -> BF16 hi/lo planes in the MN-major swizzled layout.  Thread
    // (gq, c0) owns gene quad gq (4 genes = one 16-byte fp32 unit) of cell rows c0, c0 + R, ...
    constexpr int QUADS = C::G / 4;                  // gene quads per cell row
    constexpr int R = 32 * kConvWarps / QUADS;       // cell rows covered per pass
    static_assert((32 * kConvWarps) % QUADS == 0, "converter tiling");
    const int ct = threadIdx.x - 32 * kConv0;
    const int gq = ct % QUADS, c0 = ct / QUADS;
    const int g = 4 * gq;
    const int f_col = (g >> 5) * C::BOX, f_unit = (g & 31) >> 2;   // fp32 box, 16-byte unit in its row
    const int c_col = (g >> 6) * C::BOX, c_unit = (g & 63) >> 3, c_half = (g & 7) * 2;
    for (int it = 0; it < num_kb; ++it) {
      const int fs = it % C::NF, cs = it % C::NC;
      tc::mbar_wait(&f_full[fs], (it / C::NF) & 1);
      tc::mbar_wait(&c_empty[cs], ((it / C::NC) & 1) ^ 1);
      // addressed from the __shared__ symbol itself so the compiler emits LDS/STS, not generic LD/ST
      const uint8_t* f = smem_raw + (f_base - smem_raw) + fs * C::F_BYTES + f_col;
      uint8_t* hi = smem_raw + (c_base - smem_raw) + cs * C::C_BYTES + c_col + c_half;
      uint8_t* lo = hi + C::PLANE;
#pragma unroll
      for (int c = c0; c < C::KB; c += R) {
        const float4 x = *reinterpret_cast<const float4*>(f + c * 128 + ((f_unit ^ (c & 7)) << 4));
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(x.x, x.y), h1 = __floats2bfloat162_rn(x.z, x.w);
        const float2 a = __bfloat1622float2(h0), b = __bfloat1622float2(h1);
        const __nv_bfloat162 l0 = __floats2bfloat162_rn(x.x - a.x, x.y - a.y);
        const __nv_bfloat162 l1 = __floats2bfloat162_rn(x.z - b.x, x.w - b.y);
        const int off = c * 128 + ((c_unit ^ (c & 7)) << 4);
        uint2 hv, lv;
        hv.x = *reinterpret_cast<const uint32_t*>(&h0);
        hv.y = *reinterpret_cast<const uint32_t*>(&h1);
        lv.x = *reinterpret_cast<const uint32_t*>(&l0);
        lv.y = *reinterpret_cast<const uint32_t*>(&l1);
        *reinterpret_cast<uint2*>(hi + off) = hv;
        *reinterpret_cast<uint2*>(lo + off) = lv;
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&f_empty[fs]);
        tc::mbar_arrive(&c_full[cs]);
      }
    }
    // ---- epilogue (warps 3..6): TMEM -> registers -> partial[slice] (rows i0.., cols j0..)
    if (warp < kConv0 + 4) {
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      const int row = i0 + 32 * q + lane;
      float* out = partial + (size_t)slice * hp * hp + (size_t)row * hp + j0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r0[32], r1[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + c * 32, r0);
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + BN + c * 32, r1);
        tc::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          v[j] = (num_kb > 0 ? __uint_as_float(r0[j]) : 0.0f) + (num_kb > 1 ? __uint_as_float(r1[j]) : 0.0f);
        float4* o4 = reinterpret_cast<float4*>(out + c * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<2 * BN>(tmem);
}

// Z -> BF16 planes hi = bf16(z), lo = bf16(z - hi): one streaming pass (16-byte loads, 8-byte
// stores); the Gram then reads the planes through TMA with no in-kernel conversion
__global__ void __launch_bounds__(256)
split_bf16_kernel(const float4* __restrict__ Z, int64_t n4, uint2* __restrict__ hi, uint2* __restrict__ lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = Z[i];
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
    const float2 a0 = __bfloat1622float2(h0), a1 = __bfloat1622float2(h1);
    const __nv_bfloat162 l0 = __floats2bfloat162_rn(v.x - a0.x, v.y - a0.y);
    const __nv_bfloat162 l1 = __floats2bfloat162_rn(v.z - a1.x, v.w - a1.y);
    hi[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
    lo[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
  }
}

// ---- variant fed by pre-split BF16 planes (written by scb_split_bf16): no converter warps
// and no fp32 staging -- TMA brings the hi and lo boxes straight into the MN-major
// 128-byte-swizzled operand layout, so shared memory carries only the TMA writes and the MMA
// operand reads (the fp32 variant is bound by the converter's extra smem traffic).
//
// Accumulation precision: tcgen05's FP32 accumulate truncates (~2.4 ulp lost per MMA,
// measured), a bias that grows with the number of MMAs folded into one accumulator -- with
// 4096 cells per accumulator it was the whole PCA error (C2 subspace angle 2.2e-4; an fp64
// Gram of the same Z gives 4.7e-8, tools/pca_precision.py).  So each accumulator restarts
// every kDrainStages stages (256 cells, 48 MMAs): eight epilogue warps drain it (tcgen05.ld)
// into round-to-nearest fp32 running sums held in registers (each thread one row x 128
// columns) while the other accumulator keeps the tensor pipe busy, and only the running sums
// of a long K-slice are written out.
template <int BN>
struct GramSplitCfg {
  static constexpr int BM = 128;
  static constexpr int KB = 32;                       // cells per stage = two MMA K steps
  static constexpr int BOX = KB * 128;                // one [KB cells x 64 genes] BF16 box
  static constexpr int PLANE = (BM + BN) * KB * 2;    // hi or lo plane of one stage
  static constexpr int STAGE = 2 * PLANE;
  static constexpr int STAGES = 4;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr uint32_t IDESC = tc::SCB_PLANES_IDESC(BM, BN, true, true);
  static constexpr int EPI_WARPS = 8;                 // 2 per TMEM lane quarter, BN/2 columns each
  static constexpr int COLS = BN / 2;
};
constexpr int kDrainStages = 8;            // stages per accumulator between drains (256 cells)
constexpr int kGramSplitThreads = 32 * 11;  // warp0 TMA, warps 1-2 MMA, warps 3..10 epilogue

template <int BN>
__global__ void __launch_bounds__(kGramSplitThreads, 1)
gram_split_kernel(const __grid_constant__ CUtensorMap thi, const __grid_constant__ CUtensorMap tlo,
                  const int2* __restrict__ tiles, int n_tiles, int64_t n_rows, int64_t rows_per_slice, int hp,
                  float* __restrict__ partial) {
  using C = GramSplitCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;   // [2]: sub-slice complete in accumulator p
  uint64_t* acc_empty = acc_full + 2;       // [2]: accumulator p drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id(), lane = lane_id();
  const int tile = blockIdx.x % n_tiles;
  const int slice = blockIdx.x / n_tiles;
  const int2 t = tiles ? tiles[tile] : upper_tile(tile, hp, C::BM, BN);
  const int i0 = t.x * C::BM, j0 = t.y * BN;
  const int64_t k_begin = (int64_t)slice * rows_per_slice;
  const int64_t k_end = min(n_rows, k_begin + rows_per_slice);
  const int num_kb = (k_end > k_begin) ? (int)((k_end - k_begin + C::KB - 1) / C::KB) : 0;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&thi);
      tc::tma_prefetch(&tlo);
      for (int s = 0; s < C::STAGES; ++s) {
        tc::mbar_init(&full[s], 1);
        tc::mbar_init(&empty[s], 1);
      }
      for (int p = 0; p < 2; ++p) {
        tc::mbar_init(&acc_full[p], 1);
        tc::mbar_init(&acc_empty[p], C::EPI_WARPS);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<2 * BN>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < num_kb; ++it) {
        const int s = it % C::STAGES;
        tc::mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
        uint8_t* hi = smem + s * C::STAGE;
        uint8_t* lo = hi + C::PLANE;
        const int k0 = (int)(k_begin + (int64_t)it * C::KB);
        tc::mbar_arrive_expect_tx(&full[s], C::STAGE);
#pragma unroll
        for (int c = 0; c < C::BM / 64; ++c) {
          tc::tma_load_2d(hi + c * C::BOX, &thi, &full[s], i0 + 64 * c, k0);
          tc::tma_load_2d(lo + c * C::BOX, &tlo, &full[s], i0 + 64 * c, k0);
        }
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) {
          tc::tma_load_2d(hi + (C::BM / 64 + c) * C::BOX, &thi, &full[s], j0 + 64 * c, k0);
          tc::tma_load_2d(lo + (C::BM / 64 + c) * C::BOX, &tlo, &full[s], j0 + 64 * c, k0);
        }
      }
    }
  } else if (warp <= 2) {
    // issuer p feeds accumulator p with the stages of parity p (a tcgen05.commit stalls its
    // issuing thread until the pipe drains, so two issuers keep the tensor pipe busy)
    const int p = warp - 1;
    if (lane == 0) {
      const uint32_t acc = tmem + p * BN;
      const int n_mine = (num_kb - p + 1) / 2;
      for (int j = 0; j < n_mine; ++j) {
        const int it = p + 2 * j;
        const int u = j / kDrainStages;          // sub-slice of this accumulator
        const bool first = (j % kDrainStages) == 0;
        const bool last = (j % kDrainStages) == kDrainStages - 1 || j == n_mine - 1;
        if (first) tc::mbar_wait(&acc_empty[p], (u & 1) ^ 1);
        const int s = it % C::STAGES;
        tc::mbar_wait(&full[s], (it / C::STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t ah = tc::smem_u32(smem + s * C::STAGE);
        const uint32_t bh = ah + (C::BM / 64) * C::BOX;
        const uint32_t al = ah + C::PLANE;
        const uint32_t bl = bh + C::PLANE;
#pragma unroll
        for (int kk = 0; kk < C::KB / 16; ++kk) {
          const uint32_t ko = kk * 2048;
          const uint64_t dah = tc::smem_desc_sw128(ah + ko, C::BOX, 1024);
          const uint64_t dbh = tc::smem_desc_sw128(bh + ko, C::BOX, 1024);
          const uint64_t dal = tc::smem_desc_sw128(al + ko, C::BOX, 1024);
          const uint64_t dbl = tc::smem_desc_sw128(bl + ko, C::BOX, 1024);
          tc::mma_f16(acc, dah, dbh, C::IDESC, (first && kk == 0) ? 0u : 1u);
#ifndef SCB_GRAM_1X  // experiment: hi x hi only (one product per output)
          tc::mma_f16(acc, dah, dbl, C::IDESC, 1u);
          tc::mma_f16(acc, dal, dbh, C::IDESC, 1u);
#endif
        }
        tc::mma_commit(&empty[s]);
        if (last) tc::mma_commit(&acc_full[p]);
      }
    }
  } else {
    const int e = warp - 3;        // 0..7
    const int q = warp & 3;        // TMEM lane quarter this warp may access
    const int h = e >> 2;          // column half
    const int row = i0 + 32 * q + lane;
    float sum[C::COLS];
#pragma unroll
    for (int j = 0; j < C::COLS; ++j) sum[j] = 0.0f;
    const int n_sub[2] = {((num_kb + 1) / 2 + kDrainStages - 1) / kDrainStages,
                          (num_kb / 2 + kDrainStages - 1) / kDrainStages};
    const int n_drain = n_sub[0] + n_sub[1];
    for (int d = 0; d < n_drain; ++d) {
      const int p = d & 1, u = d >> 1;   // accumulators finish alternately: 0, 1, 0, 1, ...
      tc::mbar_wait(&acc_full[p], u & 1);
      tc::tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + p * BN + h * C::COLS;
#pragma unroll
      for (int c = 0; c < C::COLS / 32; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(ta + c * 32, r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[c * 32 + j] += __uint_as_float(r[j]);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[p]);
    }
    float4* o4 = reinterpret_cast<float4*>(partial + (size_t)slice * hp * hp + (size_t)row * hp + j0 + h * C::COLS);
#pragma unroll
    for (int j = 0; j < C::COLS / 4; ++j) o4[j] = make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<2 * BN>(tmem);
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

// Cells per K-slice.  tcgen05's FP32 accumulation truncates toward zero; with kind::f16 MMAs
// the Gram loses ~2.4 ulp per MMA (measured: 64k-cell slices -> 4.6e-4 relative error on the
// diagonal and a PCA subspace angle of 7.8e-4 at C2; 16k -> 1.9e-4 / 3.6e-4; 8k -> 1.1e-4 /
// 2.2e-4, scratch/gram_precision.py).  The slices are summed in fp64; 8k cells costs ~2 GB of
// partials at 1M cells and no measurable time.
constexpr int64_t kSliceCells = 8192;
constexpr int64_t kSplitSliceCells = 32768;

template <int BN>
static int launch_gram(scb_ctx* ctx, const float* Z, const uint16_t* Zhi, const uint16_t* Zlo, int64_t n_rows, int hp,
                       double* C, cudaStream_t s) {
  const bool split = Zhi != nullptr;
  constexpr int BM = 128;
  const int KB = split ? GramSplitCfg<BN>::KB : GramCfg<BN>::KB;
  CUtensorMap tmap, thi, tlo;
  const uint64_t rows = (uint64_t)std::max<int64_t>(n_rows, 1);
  if (split) {
    SCB_TRY(make_tmap_2d(&thi, Zhi, rows, hp, hp, 2, 64, KB, /*atom32=*/false));
    SCB_TRY(make_tmap_2d(&tlo, Zlo, rows, hp, hp, 2, 64, KB, /*atom32=*/false));
  } else {
    SCB_TRY(make_tmap_2d_f32(&tmap, Z, rows, hp, hp, 32, KB, /*atom32=*/false));
  }
  // upper-triangle tile list
  std::vector<int2> tl;
  for (int bi = 0; bi < hp / BM; ++bi)
    for (int bj = 0; bj < hp / BN; ++bj)
      if (bj * BN + BN - 1 >= bi * BM) tl.push_back(make_int2(bi, bj));
  const int n_tiles = (int)tl.size();
  // K-slices: fill the SMs; the fp32-input variant keeps each TMEM accumulation <= kSliceCells
  // cells, the planes variant drains its accumulators every kDrainStages stages and takes long
  // slices (<= kSplitSliceCells), with the slice count chosen to end on a full wave of CTAs
  const int64_t kbs = (n_rows + KB - 1) / KB;
  int64_t slice_cells = split ? kSplitSliceCells : kSliceCells;
  if (const char* e = getenv("SCB_GRAM_SLICE_CELLS")) slice_cells = std::max<int64_t>(KB, atoll(e));  // experiments
  int64_t sl = std::max<int64_t>((ctx->num_sms + n_tiles - 1) / n_tiles, (n_rows + slice_cells - 1) / slice_cells);
  if (split) {  // least tail: smallest s in [sl, 2 sl) maximising the filled fraction of the last wave
    int64_t best = sl;
    double best_fill = -1.0;
    for (int64_t c = sl; c < 2 * sl && c <= kbs; ++c) {
      const int64_t ctas = c * n_tiles, waves = (ctas + ctx->num_sms - 1) / ctx->num_sms;
      const double fill = (double)ctas / (double)(waves * ctx->num_sms);
      if (fill > best_fill + 1e-9) { best_fill = fill; best = c; }
      if (fill > 0.999) break;
    }
    sl = best;
  }
  const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(sl, kbs));
  const int64_t rows_per_slice = ((kbs + slices - 1) / slices) * KB;
  const size_t part_bytes = (size_t)slices * hp * hp * 4;
  void* ws;
  SCB_TRY(ws_get(ctx, 0, part_bytes + 256, &ws, s));
  float* partial = (float*)ws;
  const int2* d_tiles = nullptr;  // enumerated on the device (upper_tile), same order as tl
  if (split) {
    using Cfg = GramSplitCfg<BN>;
    auto kern = gram_split_kernel<BN>;
    SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    kern<<<n_tiles * slices, kGramSplitThreads, Cfg::SMEM, s>>>(thi, tlo, d_tiles, n_tiles, n_rows, rows_per_slice, hp,
                                                                partial);
  } else {
    using Cfg = GramCfg<BN>;
    auto kern = gram_kernel<BN>;
    SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    kern<<<n_tiles * slices, kGemmThreads, Cfg::SMEM, s>>>(tmap, d_tiles, n_tiles, n_rows, rows_per_slice, hp,
                                                           partial);
  }
  SCB_LAUNCH_CHECK();
  dim3 g((hp + 255) / 256, hp);
  gram_reduce_kernel<<<g, 256, 0, s>>>(partial, slices, hp, C);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_gram(scb_ctx* ctx, const float* Z, int64_t n_rows, int32_t hp, double* C, void* stream) {
  SCB_REQUIRE(ctx && Z && C, SCB_ERR_ARG, "scb_gram: null argument");
  SCB_REQUIRE(hp > 0 && hp % 128 == 0, SCB_ERR_ARG, "scb_gram: hp must be a multiple of 128");
  SCB_REQUIRE(n_rows >= 0 && n_rows < (1ll << 31), SCB_ERR_ARG, "scb_gram: n_rows out of range");
  cudaStream_t s = (cudaStream_t)stream;
  if (hp % 256 == 0) return launch_gram<256>(ctx, Z, nullptr, nullptr, n_rows, hp, C, s);
  return launch_gram<128>(ctx, Z, nullptr, nullptr, n_rows, hp, C, s);
}

extern "C" int scb_gram_split(scb_ctx* ctx, const uint16_t* Zhi, const uint16_t* Zlo, int64_t n_rows, int32_t hp,
                              double* C, void* stream) {
  SCB_REQUIRE(ctx && Zhi && Zlo && C, SCB_ERR_ARG, "scb_gram_split: null argument");
  SCB_REQUIRE(hp > 0 && hp % 128 == 0, SCB_ERR_ARG, "scb_gram_split: hp must be a multiple of 128");
  SCB_REQUIRE(n_rows >= 0 && n_rows < (1ll << 31), SCB_ERR_ARG, "scb_gram_split: n_rows out of range");
  cudaStream_t s = (cudaStream_t)stream;
  if (hp % 256 == 0) return launch_gram<256>(ctx, nullptr, Zhi, Zlo, n_rows, hp, C, s);
  return launch_gram<128>(ctx, nullptr, Zhi, Zlo, n_rows, hp, C, s);
}

// format of the operand planes (scb_split_bf16, scb_scale_dense_planes, Gram, projection):
// 0 BF16 + three-product Gram (default), 2 FP16 + three products, 1 FP16 + one product
extern "C" int32_t scb_plane_format(void) {
#ifdef SCB_PLANES_F16
#ifdef SCB_GRAM_1X
  return 1;
#else
  return 2;
#endif
#else
  return 0;
#endif
}

extern "C" int scb_split_bf16(scb_ctx* ctx, const float* Z, int64_t n_rows, int64_t ld, uint16_t* Zhi, uint16_t* Zlo,
                              void* stream) {
  SCB_REQUIRE(ctx && Z && Zhi && Zlo, SCB_ERR_ARG, "scb_split_bf16: null argument");
  SCB_REQUIRE(ld % 4 == 0 && ((uintptr_t)Z & 15) == 0 && ((uintptr_t)Zhi & 7) == 0 && ((uintptr_t)Zlo & 7) == 0,
              SCB_ERR_ARG, "scb_split_bf16: ld % 4 == 0 and aligned buffers required");
  if (n_rows == 0) return SCB_OK;
  const int64_t n4 = n_rows * ld / 4;
  split_bf16_kernel<<<ctx->num_sms * 8, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(Z), n4, reinterpret_cast<uint2*>(Zhi), reinterpret_cast<uint2*>(Zlo));
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

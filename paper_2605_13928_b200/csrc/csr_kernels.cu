// CSR count-matrix stages: QC metrics, filter masks, subset, normalize_total+log1p,
// HVG gene sums + seurat selection, scale (sums, finalize, dense gather).
//
// All are HBM-bound streaming passes over (indices, data).  Row-local work is
// warp-per-row with coalesced loads; column (per-gene) reductions are privatised in
// shared memory per CTA using NATIVE 32-bit shared atomics (ATOMS.ADD) on integer
// fixed-point words -- shared fp32/fp64/u64 atomicAdd compile to CAS loops on sm_100a,
// and global fp64 REDs sustain only ~146 G/s (scratch/mb_atomics.cu, profiles/).
// Integer sums are exact and order independent, so results are deterministic and
// identical across 1/2/4/8-way cell sharding.
#include <cuda_bf16.h>
#include "planes_fmt.cuh"
#include <type_traits>
#include "common.cuh"
#include "scan.cuh"
#include "stream.cuh"

namespace scb {

constexpr int kRowThreads = 512;          // threads per CTA of the row-streaming kernels
constexpr int kQcThreads = 1024;          // QC: one CTA per SM (gene histogram fills smem)
constexpr int kQcFlushRows = 4095;        // rows per CTA between flushes of the packed gene words
constexpr int kHvgThreads = 1024;         // HVG sums: one CTA per SM (gene tile fills smem)
constexpr int kMaxSplit = 3;              // gene tiles of the HVG pass: up to 4 (G <= ~58k)
constexpr int kHvgTileW = (int)(227 * 1024 / 16);  // genes per HVG tile (4 u32 words each)
constexpr size_t kSmemLimit = 227 * 1024;  // opt-in dynamic shared memory per CTA

static int grid_for(scb_ctx* ctx, int ctas_per_sm) { return ctx->num_sms * ctas_per_sm; }

// log1p of a normalised count y >= 0.  For y >= 0.25 the MUFU logarithm of (1 + y) is used
// (__logf: <= 2^-21.4 absolute error on [1.25, 2], <= 3 ulp above; the rounding of 1 + y adds
// <= 2^-24 absolute) -- relative error <= 2e-6, inside the 1e-5 tolerance of the log values
// (numpy's own float32 log1p is not correctly rounded either); below 0.25, where 1 + y would
// cancel, the accurate log1pf.  About 4 instructions instead of ~25 for almost every nonzero
// (y = count * 1e4 / total is >= 1 for most entries).
__device__ __forceinline__ float log1p_count(float y) { return y >= 0.25f ? __logf(1.0f + y) : log1pf(y); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Kept-gene map in shared memory: word i = (kept bits of genes [32i, 32i+32), number of kept
// genes before gene 32i), so remap[g] = prefix + popc(bits below g) -- a conflict-light LDS.64
// instead of a scattered global gather per nonzero.
__device__ __forceinline__ void build_gene_map(const int32_t* __restrict__ remap, int32_t n_cols, uint2* s_map) {
  const int n_words = (n_cols + 31) >> 5;
  for (int wi = warp_id(); wi < n_words; wi += (blockDim.x >> 5)) {
    const int g = wi * 32 + lane_id();
    const int rv = g < n_cols ? remap[g] : -1;
    const unsigned bits = __ballot_sync(0xffffffffu, rv >= 0);
    const int first = __shfl_sync(0xffffffffu, rv, bits ? __ffs(bits) - 1 : 0);
    if (lane_id() == 0) s_map[wi] = make_uint2(bits, bits ? (unsigned)first : 0u);
  }
}
// kept-gene map: int16 remap table when n_cols <= 32767 (one LDS.S16 per lookup), else the
// bit/prefix words above
template <bool SMALL>
__device__ __forceinline__ void build_map(const int32_t* __restrict__ remap, int32_t n_cols, void* smem) {
  if (SMALL) {
    int16_t* t = reinterpret_cast<int16_t*>(smem);
    for (int i = threadIdx.x; i < n_cols; i += blockDim.x) t[i] = (int16_t)remap[i];
  } else {
    build_gene_map(remap, n_cols, reinterpret_cast<uint2*>(smem));
  }
}
__device__ __forceinline__ int map_gene(const uint2* s_map, int32_t n_cols, int g);
template <bool SMALL>
__device__ __forceinline__ int lookup_map(const void* smem, int32_t n_cols, int g) {
  if (SMALL) return (unsigned)g < (unsigned)n_cols ? (int)reinterpret_cast<const int16_t*>(smem)[g] : -1;
  return map_gene(reinterpret_cast<const uint2*>(smem), n_cols, g);
}
__device__ __forceinline__ int map_gene(const uint2* s_map, int32_t n_cols, int g) {
  if ((unsigned)g >= (unsigned)n_cols) return -1;
  const uint2 w = s_map[g >> 5];
  const unsigned sh = (unsigned)g & 31u;
  return ((w.x >> sh) & 1u) ? (int)(w.y + __popc(w.x & ((1u << sh) - 1u))) : -1;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int32_t lds_s16(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// fire-and-forget shared add on a shared-window address (native ATOMS.ADD, no return value)
__device__ __forceinline__ void red_shared_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// ============================================================================ QC
// smem: one packed u32 per gene of a tile [g0, g0+W) -- bits [20,32) cells with a nonzero count,
// bits [0,20) the sum of the counts' low 8 bits -- and an mt flag byte per gene.  One shared
// atomic per nonzero; count bits >= 8 go straight to the global u64 totals (0.1 % of C3's
// nonzeros).  Every kQcFlushRows rows a CTA adds its words into the global counters and clears
// them, so neither field can overflow (4095 rows x 255 < 2^20).  The tile-0
// CTAs also write the per-cell metrics and, for the HVG pass, the per-row positions where
// the original gene index crosses each HVG tile boundary (splits[r][t-1] = #entries with
// gene < t*split_w, relative to the row start).
template <typename IT, typename VT, int NSPLIT, bool SINGLE_TILE>
__global__ void __launch_bounds__(kQcThreads)
qc_kernel(const int64_t* __restrict__ indptr, const IT* __restrict__ indices,
          const VT* __restrict__ data, int64_t n_rows, int32_t n_cols,
          const uint8_t* __restrict__ mt_mask, int32_t tile_w, int32_t n_split, int32_t split_w,
          int32_t* __restrict__ splits, int32_t* __restrict__ n_genes, double* __restrict__ total,
          double* __restrict__ total_mt, double* __restrict__ pct, uint32_t* __restrict__ g_cells,
          unsigned long long* __restrict__ g_total, int* __restrict__ flag, U16Esc esc) {
  const int64_t nnz = indptr[n_rows];
  extern __shared__ uint32_t sm[];
  const int tile = blockIdx.y;
  const int g0 = tile * tile_w;
  const int w = min(tile_w, n_cols - g0);
  uint32_t* s_pack = sm;
  uint8_t* s_mt = reinterpret_cast<uint8_t*>(sm + tile_w);  // 0/1 per gene, ALL genes
  for (int i = threadIdx.x; i < tile_w; i += blockDim.x) sm[i] = 0;
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) s_mt[i] = mt_mask[i] ? 1 : 0;
  __syncthreads();
  const bool row_owner = (tile == 0);
  const int lane = lane_id();
  const int wpc = blockDim.x >> 5;
  const int64_t warps = (int64_t)gridDim.x * wpc;
  const int flush_every = kQcFlushRows / wpc;  // loop iterations (each: one row per warp)
  // shared-window addresses biased by the tile origin: gene g lives at a + 4g
  const uint32_t a_pack = smem_addr(s_pack) - 4u * (uint32_t)g0;
  const uint32_t a_mt = smem_addr(s_mt);
  auto flush = [&]() {
    __syncthreads();
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
      const uint32_t v = s_pack[i];
      if (v) {
        if (v >> 20) atomicAdd(&g_cells[g0 + i], v >> 20);
        if (v & 0xFFFFFu) atomicAdd(&g_total[g0 + i], (unsigned long long)(v & 0xFFFFFu));
        s_pack[i] = 0u;
      }
    }
    __syncthreads();
  };
  // per-lane dummy gene of the tile for masked elements' zero adds (distinct lanes -> distinct
  // banks; a shared dummy would serialise the warp's atomics on one address)
  const int gd = g0 + lane % max(w, 1);
  bool bad = false;
  int since_flush = 0;
  for (int64_t r0 = (int64_t)blockIdx.x * wpc; r0 < n_rows; r0 += warps) {  // CTA-uniform trip count
    if (++since_flush > flush_every) {
      flush();
      since_flush = 1;
    }
    const int64_t r = r0 + warp_id();
    if (r >= n_rows) continue;
    const int64_t b = indptr[r], e = indptr[r + 1];
    uint32_t cnt = 0;
    unsigned long long sum = 0, summt = 0;
    int sc[NSPLIT > 0 ? NSPLIT : 1] = {};
    // Per quad.  x + 2^23 is exact iff x is an integer in [0, 2^23) (then its low mantissa bits
    // are the count), so FADD/FADD/FSETP validate and convert; anything else (x >= 2^23,
    // negative, fractional, NaN, bad gene index) sends the whole quad through the exact rare
    // check once.  Masked-out (or invalid) elements become (per-lane dummy gene, count 0),
    // which the branch-free accumulation below adds harmlessly.
    auto quad = [&](const Quad& q, auto full_tag) {
      constexpr bool kFull = decltype(full_tag)::value;
      int g[4];
      uint32_t xv[4];
      bool ok_all = true;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = q.x[k];
        const float t = x + 8388608.0f;
        xv[k] = __float_as_uint(t) - 0x4B000000u;
        g[k] = q.g[k];
        const bool ok = (t - 8388608.0f == x) & (xv[k] < (1u << 23)) & ((unsigned)g[k] < (unsigned)n_cols);
        if (kFull) {
          ok_all &= ok;
        } else {
          const bool v = (q.valid >> k) & 1u;
          ok_all &= ok | !v;
          if (!v) { xv[k] = 0u; g[k] = gd; }
        }
      }
      if (!ok_all) {  // rare: exact check per element
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!kFull && !((q.valid >> k) & 1u)) continue;
          const float x = q.x[k];
          const bool ok = (x >= 0.0f && x == rintf(x) && x < 16777216.0f) && (unsigned)q.g[k] < (unsigned)n_cols;
          bad |= !ok;
          xv[k] = ok ? (uint32_t)x : 0u;
          g[k] = ok ? q.g[k] : gd;
        }
      }
      uint32_t qsum = 0, qmt = 0, hi_any = 0;  // 4 counts < 2^24 fit a u32
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int t2 = 0; t2 < NSPLIT; ++t2) {
          const bool v = kFull || ((q.valid >> k) & 1u);
          sc[t2] += (v & (q.g[k] < (t2 + 1) * split_w)) ? 1 : 0;
        }
        cnt += (xv[k] != 0u) ? 1u : 0u;
        qsum += xv[k];
        qmt += lds_u8(a_mt + (uint32_t)g[k]) * xv[k];
        // packed word: +1 cell in bits [20,32) for a nonzero, + low 8 bits of the count
        // (fire-and-forget); masked elements add 0 to the lane's dummy gene.  One tile covering
        // every gene (G <= ~50k): every validated gene index is in it
        const bool in_tile = SINGLE_TILE || (unsigned)(g[k] - g0) < (unsigned)w;
        const uint32_t ga = 4u * (uint32_t)(in_tile ? g[k] : gd);
        red_shared_add(a_pack + ga, in_tile ? (((xv[k] != 0u) ? (1u << 20) : 0u) | (xv[k] & 0xFFu)) : 0u);
        hi_any |= in_tile ? xv[k] : 0u;
      }
      if (hi_any > 0xFFu) {  // rare: higher parts straight into the global u64 totals
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((SINGLE_TILE || (unsigned)(g[k] - g0) < (unsigned)w) & (xv[k] > 0xFFu))
            atomicAdd(&g_total[g[k]], (unsigned long long)(xv[k] & ~0xFFu));
      }
      sum += qsum;
      summt += qmt;
    };
    stream_row<2>(indices, data, b, e, nnz, [&](const Quad& q) {
      if (q.valid == 0u) return;
      if (q.valid == 0xFu)
        quad(q, std::true_type{});
      else
        quad(q, std::false_type{});
    }, esc);
    if (row_owner) {
      cnt = warp_sum(cnt);
      sum = warp_sum(sum);
      summt = warp_sum(summt);
#pragma unroll
      for (int t = 0; t < NSPLIT; ++t) sc[t] = warp_sum(sc[t]);
      if (lane == 0) {
        n_genes[r] = (int32_t)cnt;
        const double sd = (double)sum, md = (double)summt;
        total[r] = sd;
        total_mt[r] = md;
        pct[r] = __ddiv_rn(__dmul_rn(100.0, md), sd);
#pragma unroll
        for (int t = 0; t < NSPLIT; ++t) splits[r * NSPLIT + t] = sc[t];
      }
    }
  }
  if (bad) atomicOr(flag, 1);
  flush();
}

__global__ void zero_if_flag_kernel(unsigned long long* __restrict__ a, int64_t n, const int* __restrict__ flag) {
  if (*flag == 0) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = 0ull;
}

__global__ void add_u64_kernel(const unsigned long long* __restrict__ a, unsigned long long* __restrict__ b,
                               int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] += a[i];
}

__global__ void qc_finalize(const uint32_t* g_cells, const unsigned long long* g_total, int32_t n,
                            int32_t* n_cells, double* gene_total) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    n_cells[i] = (int32_t)g_cells[i];
    gene_total[i] = (double)g_total[i];
  }
}

// ============================================================================ masks
__global__ void cell_mask_kernel(const int32_t* ng, const double* pct, int64_t n, int32_t min_genes,
                                 int32_t max_genes, double max_pct, uint8_t* mask,
                                 unsigned long long* kept) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool k = false;
  if (i < n) {
    k = ng[i] >= min_genes && (max_genes < 0 || ng[i] <= max_genes) && (pct[i] < max_pct);
    mask[i] = k ? 1 : 0;
  }
  unsigned c = __popc(__ballot_sync(0xffffffffu, k));
  if (lane_id() == 0 && c) atomicAdd(kept, (unsigned long long)c);
}

__global__ void gene_mask_kernel(const int32_t* nc, int32_t n, int32_t min_cells, uint8_t* mask,
                                 unsigned long long* kept) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool k = false;
  if (i < n) {
    k = nc[i] >= min_cells;
    mask[i] = k ? 1 : 0;
  }
  unsigned c = __popc(__ballot_sync(0xffffffffu, k));
  if (lane_id() == 0 && c) atomicAdd(kept + 1, (unsigned long long)c);
}

// ============================================================================ subset
// gene_remap = exclusive scan of gene_mask (or -1), computed by one CTA.
__global__ void gene_remap_kernel(const uint8_t* gmask, int32_t n, int32_t* remap) {
  __shared__ int32_t carry;
  __shared__ int32_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    int i = base + threadIdx.x;
    int v = (i < n && gmask[i]) ? 1 : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= o) incl += t;
    }
    if (lane_id() == 31) wsum[warp_id()] = incl;
    __syncthreads();
    if (warp_id() == 0) {
      int s = (lane_id() < (int)(blockDim.x >> 5)) ? wsum[lane_id()] : 0;
      int si = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, si, o);
        if (lane_id() >= o) si += t;
      }
      wsum[lane_id()] = si - s;
    }
    __syncthreads();
    int excl = carry + wsum[warp_id()] + incl - v;
    if (i < n) remap[i] = v ? excl : -1;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

// Count kept entries (and kept total) per original row; writes counts into
// cnt[kept_row] where kept_row = row_pos[r] (exclusive scan of cell_mask).
template <typename IT, typename VT, bool SMALL>
__global__ void __launch_bounds__(kRowThreads)
subset_count_kernel(const int64_t* __restrict__ indptr, const IT* __restrict__ indices,
                    const VT* __restrict__ data, int64_t n_rows, const uint8_t* __restrict__ cmask,
                    const int32_t* __restrict__ remap, int32_t n_cols, const int64_t* __restrict__ row_pos,
                    int64_t* __restrict__ cnt, double target_sum, float* __restrict__ row_scale,
                    float* __restrict__ row_scale_orig, U16Esc esc) {
  extern __shared__ uint2 s_map[];
  build_map<SMALL>(remap, n_cols, s_map);
  __syncthreads();
  const int64_t nnz = indptr[n_rows];
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); r < n_rows; r += warps) {
    if (!cmask[r]) {
      if (lane == 0 && row_scale_orig) row_scale_orig[r] = 0.0f;
      continue;
    }
    const int64_t b = indptr[r], e = indptr[r + 1];
    int c = 0;
    double sum = 0.0;
    stream_row_pipe<1>(indices, row_scale ? data : nullptr, b, e, nnz, [&](const Quad& q) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (((q.valid >> k) & 1u) && lookup_map<SMALL>(s_map, n_cols, q.g[k]) >= 0) {
          ++c;
          sum += (double)q.x[k];
        }
    }, esc);
    c = warp_sum(c);
    if (row_scale) sum = warp_sum(sum);
    if (lane == 0) {
      const int64_t kr = row_pos[r];
      cnt[kr] = c;
      if (row_scale) {
        const float s = (sum > 0.0) ? (float)__ddiv_rn(target_sum, sum) : 1.0f;
        row_scale[kr] = s;
        if (row_scale_orig) row_scale_orig[r] = s;
      }
    }
  }
}

// Pass 1 when every gene is kept (the usual case at scale: min_cells = 3 over 1M cells): the
// kept-row lengths are the row lengths and the normalisation totals are QC's exact row totals,
// so no pass over the nonzeros is needed (same float32(target_sum / total) as subset_count).
__global__ void rows_all_genes_kernel(const int64_t* __restrict__ indptr, const uint8_t* __restrict__ cmask,
                                      const int64_t* __restrict__ row_pos, const double* __restrict__ total,
                                      int64_t n_rows, double target_sum, int64_t* __restrict__ cnt,
                                      float* __restrict__ row_scale, float* __restrict__ row_scale_orig) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (!cmask[r]) {
      if (row_scale_orig) row_scale_orig[r] = 0.0f;
      continue;
    }
    const int64_t kr = row_pos[r];
    cnt[kr] = indptr[r + 1] - indptr[r];
    const double t = total[r];
    const float sc = (t > 0.0) ? (float)__ddiv_rn(target_sum, t) : 1.0f;
    row_scale[kr] = sc;
    if (row_scale_orig) row_scale_orig[r] = sc;
  }
}

__global__ void identity_remap_kernel(int32_t n, int32_t* remap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) remap[i] = i;
}

// kept-row nonzeros (for allocation without an extra host round trip)
__global__ void kept_nnz_kernel(const int64_t* __restrict__ indptr, const uint8_t* __restrict__ cmask, int64_t n,
                                unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (cmask[r]) acc += (unsigned long long)(indptr[r + 1] - indptr[r]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane_id() == 0 && acc) atomicAdd(out, acc);
}

__global__ void copy_flag_kernel(const int* __restrict__ flag, long long* __restrict__ out) { *out = *flag; }

// Compacting copy: each lane's 4-element quad contributes its kept count to a warp-wide
// exclusive scan so the output stays in row order.  The (up to 128) kept elements of a warp
// step are staged in shared memory and written back 32 consecutive elements per instruction
// (full 128-byte lines instead of four lane-strided partial-sector stores per quad).
template <typename IT, typename VT, bool SMALL>
__global__ void __launch_bounds__(kRowThreads)
subset_fill_kernel(const int64_t* __restrict__ indptr, const IT* __restrict__ indices,
                   const VT* __restrict__ data, int64_t n_rows, const uint8_t* __restrict__ cmask,
                   const int32_t* __restrict__ remap, int32_t n_cols, const int64_t* __restrict__ row_pos,
                   const int64_t* __restrict__ new_indptr, const float* __restrict__ row_scale,
                   int32_t* __restrict__ out_idx, float* __restrict__ out_val, U16Esc esc) {
  __shared__ int s_idx[kRowThreads / 32][128];
  __shared__ float s_val[kRowThreads / 32][128];
  extern __shared__ uint2 s_map[];
  build_map<SMALL>(remap, n_cols, s_map);
  __syncthreads();
  const int64_t nnz = indptr[n_rows];
  const int lane = lane_id(), w = warp_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + w; r < n_rows; r += warps) {
    if (!cmask[r]) continue;
    const int64_t kr = row_pos[r];
    const float s = row_scale ? row_scale[kr] : 1.0f;
    const int64_t b = indptr[r], e = indptr[r + 1];
    int64_t o = new_indptr[kr];
    stream_row_pipe<1>(indices, data, b, e, nnz, [&](const Quad& q) {
      int ng[4];
      int kc = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ng[k] = ((q.valid >> k) & 1u) ? lookup_map<SMALL>(s_map, n_cols, q.g[k]) : -1;
        kc += ng[k] >= 0 ? 1 : 0;
      }
      int incl = kc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      int pos = incl - kc;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ng[k] >= 0) {
          s_idx[w][pos] = ng[k];
          s_val[w][pos] = row_scale ? log1p_count(__fmul_rn(q.x[k], s)) : q.x[k];
          ++pos;
        }
      __syncwarp();
      for (int j = lane; j < tot; j += 32) {
        out_idx[o + j] = s_idx[w][j];
        out_val[o + j] = s_val[w][j];
      }
      __syncwarp();
      o += tot;
    }, esc);
  }
}

// Fused variant: the same compaction + log1p, and the scale step's fixed-point gene sums of the
// HVG columns taken while the log values are produced (saves the scale pass's full re-read of
// the kept matrix).  CTA = block of <= 1024 rows (carry-free 22-bit split, as scale_sums);
// smem: int32 per original gene = new index | (slot + 1) << 16 (-1: dropped; slot -1: not an HVG),
// 4 u32 words per HVG.  Requires n_cols <= 32767.
constexpr int kFillSumsThreads = 1024;
template <typename IT, typename VT>
__global__ void __launch_bounds__(kFillSumsThreads)
subset_fill_sums_kernel(const int64_t* __restrict__ indptr, const IT* __restrict__ indices,
                        const VT* __restrict__ data, int64_t n_rows, const uint8_t* __restrict__ cmask,
                        const int32_t* __restrict__ remap, int32_t n_cols, const int32_t* __restrict__ slot_new,
                        int32_t n_slots, const int64_t* __restrict__ row_pos, const int64_t* __restrict__ new_indptr,
                        const float* __restrict__ row_scale, int64_t rows_per_block, int32_t* __restrict__ out_idx,
                        float* __restrict__ out_val, unsigned long long* __restrict__ sums, U16Esc esc) {
  __shared__ int s_idx[kFillSumsThreads / 32][128];
  __shared__ float s_val[kFillSumsThreads / 32][128];
  extern __shared__ int32_t dyn_tab[];
  int32_t* tab = dyn_tab;
  uint32_t* ss = reinterpret_cast<uint32_t*>(dyn_tab + ((n_cols + 3) & ~3));
  bool ident = true;  // every gene kept in place (the all-genes path): no compaction within rows
  for (int g = threadIdx.x; g < n_cols; g += blockDim.x) {
    const int r = remap[g];
    ident &= (r == g);
    // kept: (slot + 1) << 16 | new index (both < 2^15, so the word stays non-negative); dropped: -1
    tab[g] = r < 0 ? -1 : (int32_t)((uint32_t)r | ((uint32_t)(slot_new[r] + 1) << 16));
  }
  for (int i = threadIdx.x; i < 4 * n_slots; i += blockDim.x) ss[i] = 0;
  ident = __syncthreads_and(ident);
  const uint32_t a1lo = smem_addr(ss), a1hi = a1lo + 4u * n_slots, a2lo = a1lo + 8u * n_slots,
                 a2hi = a1lo + 12u * n_slots;
  const int64_t nnz = indptr[n_rows];
  const int lane = lane_id(), w = warp_id();
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(n_rows, r0 + rows_per_block);
  // HVG column: scale sums (same integers as scale_sums_kernel)
  auto add_sums = [&](float l, int sl) {
    const uint64_t v1 = (uint64_t)__float2ull_rn(__fmul_rn(l, 268435456.0f));
    const double l12 = (double)__fmul_rn(l, 4096.0f);
    const uint64_t v2 = (uint64_t)__double2ull_rn(__dmul_rn(l12, l12));
    const uint32_t ja = 4u * (uint32_t)sl;
    if ((v1 | v2) < (1ull << 43)) {
      red_shared_add(a1lo + ja, (uint32_t)(v1 & 0x3FFFFFu));
      red_shared_add(a1hi + ja, (uint32_t)(v1 >> 22));
      red_shared_add(a2lo + ja, (uint32_t)(v2 & 0x3FFFFFu));
      red_shared_add(a2hi + ja, (uint32_t)(v2 >> 22));
    } else {  // rare (not log-normalized scale): straight into the global limbs
      atomicAdd(&sums[sl], v1 & 0xFFFFFFFFull);
      atomicAdd(&sums[n_slots + sl], v1 >> 32);
      atomicAdd(&sums[2 * n_slots + sl], v2 & 0xFFFFFFFFull);
      atomicAdd(&sums[3 * n_slots + sl], v2 >> 32);
    }
  };
  // out_idx == nullptr: every row and gene is kept, the output shares the input's indices
  if (out_idx == nullptr && !ident) __trap();  // C-ABI contract violated
  if (ident) {
    // element p of row r lands at p + (new_indptr[kr] - indptr[r]): no scan, no staging;
    // 16-byte stores when the shift keeps quads aligned
    for (int64_t r = r0 + w; r < r1; r += (blockDim.x >> 5)) {
      if (!cmask[r]) {
        if (out_idx == nullptr) __trap();
        continue;
      }
      const int64_t kr = row_pos[r];
      const float s = row_scale[kr];
      const int64_t b = indptr[r], e = indptr[r + 1];
      const int64_t delta = new_indptr[kr] - b;
      if (out_idx == nullptr && delta != 0) __trap();
      const bool vec = (delta & 3) == 0;
      stream_row_pipe<1>(indices, data, b, e, nnz, [&](const Quad& q) {
        float l[4];
        int sl[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int g = q.g[k];
          const int32_t t = (((q.valid >> k) & 1u) && (unsigned)g < (unsigned)n_cols) ? tab[g] : -1;
          sl[k] = t < 0 ? -1 : (int)((uint32_t)t >> 16) - 1;
          l[k] = log1p_count(__fmul_rn(q.x[k], s));
        }
        const int64_t o = q.p + delta;
        if (vec && q.valid == 0xFu) {
          if (out_idx) *reinterpret_cast<int4*>(out_idx + o) = make_int4(q.g[0], q.g[1], q.g[2], q.g[3]);
          *reinterpret_cast<float4*>(out_val + o) = make_float4(l[0], l[1], l[2], l[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if ((q.valid >> k) & 1u) {
              if (out_idx) out_idx[o + k] = q.g[k];
              out_val[o + k] = l[k];
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (sl[k] >= 0) add_sums(l[k], sl[k]);
      }, esc);
    }
  }
  for (int64_t r = r0 + w; r < r1 && !ident; r += (blockDim.x >> 5)) {
    if (!cmask[r]) continue;
    const int64_t kr = row_pos[r];
    const float s = row_scale[kr];
    const int64_t b = indptr[r], e = indptr[r + 1];
    int64_t o = new_indptr[kr];
    stream_row_pipe<1>(indices, data, b, e, nnz, [&](const Quad& q) {
      int ng[4], sl[4];
      int kc = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int g = q.g[k];
        const int32_t t = (((q.valid >> k) & 1u) && (unsigned)g < (unsigned)n_cols) ? tab[g] : -1;
        ng[k] = t < 0 ? -1 : (t & 0xFFFF);
        sl[k] = t < 0 ? -1 : (int)((uint32_t)t >> 16) - 1;
        kc += ng[k] >= 0 ? 1 : 0;
      }
      int incl = kc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      int pos = incl - kc;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ng[k] >= 0) {
          const float l = log1p_count(__fmul_rn(q.x[k], s));
          s_idx[w][pos] = ng[k];
          s_val[w][pos] = l;
          ++pos;
          if (sl[k] >= 0) add_sums(l, sl[k]);
        }
      __syncwarp();
      for (int j = lane; j < tot; j += 32) {
        out_idx[o + j] = s_idx[w][j];
        out_val[o + j] = s_val[w][j];
      }
      __syncwarp();
      o += tot;
    }, esc);
  }
  __syncthreads();
  const uint32_t* s1lo = ss;
  const uint32_t* s1hi = ss + n_slots;
  const uint32_t* s2lo = ss + 2 * n_slots;
  const uint32_t* s2hi = ss + 3 * n_slots;
  for (int i = threadIdx.x; i < n_slots; i += blockDim.x) {
    const unsigned long long a0 = (unsigned long long)s1lo[i] + ((unsigned long long)(s1hi[i] & 1023u) << 22);
    const unsigned long long b0 = (unsigned long long)s2lo[i] + ((unsigned long long)(s2hi[i] & 1023u) << 22);
    if (a0) atomicAdd(&sums[i], a0);
    if (s1hi[i] >> 10) atomicAdd(&sums[n_slots + i], (unsigned long long)(s1hi[i] >> 10));
    if (b0) atomicAdd(&sums[2 * n_slots + i], b0);
    if (s2hi[i] >> 10) atomicAdd(&sums[3 * n_slots + i], (unsigned long long)(s2hi[i] >> 10));
  }
}

// ============================================================================ normalize + log1p

__global__ void __launch_bounds__(kRowThreads)
normalize_log1p_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ data, int64_t n_rows,
                       double target_sum, float* __restrict__ out, float* __restrict__ row_scale) {
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); r < n_rows; r += warps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    double sum = 0.0;
    for (int64_t p = b + lane; p < e; p += 32) sum += (double)data[p];
    sum = warp_sum(sum);
    const float s = (sum > 0.0) ? (float)__ddiv_rn(target_sum, sum) : 1.0f;
    if (lane == 0) row_scale[r] = s;
    for (int64_t p = b + lane; p < e; p += 32) out[p] = log1p_count(__fmul_rn(data[p], s));
  }
}

// ============================================================================ HVG gene sums
// Tiled column reduction over ORIGINAL gene ranges [t*tile_w, (t+1)*tile_w): CTA (row block,
// tile) keeps 4 u32 fixed-point words per gene of its tile (sum y lo/hi, sum y^2 lo/hi) in
// smem.  With row splits (from QC) each CTA streams only its tile's sub-range of every row,
// so each nonzero is read exactly once; without them every tile CTA filters whole rows.
__device__ __forceinline__ uint64_t fx_round(double v) { return (uint64_t)__double2ull_rn(v); }

template <typename IT, typename VT>
__global__ void __launch_bounds__(kHvgThreads)
hvg_sums_kernel(const int64_t* __restrict__ indptr, const IT* __restrict__ indices,
                const VT* __restrict__ data, const float* __restrict__ row_scale, int64_t n_rows,
                int32_t n_cols, const int32_t* __restrict__ remap, int32_t n_out, int32_t tile_w,
                int32_t n_tiles, const int32_t* __restrict__ splits, int64_t rows_per_block,
                unsigned long long* __restrict__ sums, int* __restrict__ order_flag, U16Esc esc,
                const int* __restrict__ run_if = nullptr) {
  if (run_if && *run_if == 0) return;  // conditional fallback launch (no host round trip)
  const int64_t nnz = indptr[n_rows];
  extern __shared__ uint32_t sm[];
  const int tile = blockIdx.x % n_tiles;
  const int64_t rblk = blockIdx.x / n_tiles;
  const int g0 = tile * tile_w;
  const int w = min(tile_w, n_cols - g0);
  uint32_t* s1lo = sm;
  uint32_t* s1hi = sm + tile_w;
  uint32_t* s2lo = sm + 2 * tile_w;
  uint32_t* s2hi = sm + 3 * tile_w;
  const uint32_t a1lo = smem_addr(s1lo), a1hi = smem_addr(s1hi), a2lo = smem_addr(s2lo), a2hi = smem_addr(s2hi);
  const int dl = lane_id() % max(w, 1);  // per-lane dummy slot for zero adds (no same-address serialisation)
  for (int i = threadIdx.x; i < 4 * tile_w; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int64_t r0 = rblk * rows_per_block;
  const int64_t r1 = min(n_rows, r0 + rows_per_block);
  const int ns = n_tiles - 1;
  const bool split_mode = splits && ns > 0;
  bool out_of_order = false;
  for (int64_t r = r0 + warp_id(); r < r1; r += (blockDim.x >> 5)) {
    const float s = row_scale[r];
    if (s == 0.0f) continue;
    int64_t b = indptr[r], e = indptr[r + 1];
    if (split_mode) {
      const int64_t rb = b;
      if (tile > 0) b = rb + splits[r * ns + tile - 1];
      if (tile < ns) e = rb + splits[r * ns + tile];
    }
    // Per quad: y = fl(x * s); v1 = round(y * 2^28) (exact scaling in f32, one RN conversion),
    // v2 = round((y * 2^12)^2) (exact square in f64, one RN conversion) -- the same integers as
    // the oracle's round(y * 2^28), round(y^2 * 2^24).  Carry-free split: low 22 bits + high
    // part; with <= 1024 rows per CTA neither u32 word can overflow, so all four adds are
    // fire-and-forget and unconditional (out-of-tile / masked elements add 0 to a per-lane dummy
    // gene of the tile).
    // Values outside the fast range (y >= 2^15 for the sum, y >= ~724 for the sum of squares)
    // go to the global limbs.
    stream_row<2>(indices, data, b, e, nnz, [&](const Quad& q) {
      if (q.valid == 0u) return;
      uint64_t v1[4], v2[4];
      uint32_t ga[4];
      bool rare = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int gl = q.g[k] - g0;
        const bool in = ((q.valid >> k) & 1u) && gl >= 0 && gl < w;
        // with row splits every entry of the streamed sub-range must belong to this tile (true
        // for sorted rows); anything else means unsorted indices -> the host reruns unsplit
        out_of_order |= split_mode & ((q.valid >> k) & 1u) & !in;
        const float y = __fmul_rn(q.x[k], s);  // float32 normalized count
        v1[k] = in ? (uint64_t)__float2ull_rn(__fmul_rn(y, 268435456.0f)) : 0ull;
        const double y12 = (double)__fmul_rn(y, 4096.0f);
        v2[k] = in ? (uint64_t)__double2ull_rn(__dmul_rn(y12, y12)) : 0ull;
        ga[k] = 4u * (uint32_t)(in ? gl : dl);
        rare |= (v1[k] >= (1ull << 43)) | ((v2[k] >> 22) >= (1ull << 21));
      }
      if (!rare) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          red_shared_add(a1lo + ga[k], (uint32_t)(v1[k] & 0x3FFFFFu));
          red_shared_add(a1hi + ga[k], (uint32_t)(v1[k] >> 22));
          red_shared_add(a2lo + ga[k], (uint32_t)(v2[k] & 0x3FFFFFu));
          red_shared_add(a2hi + ga[k], (uint32_t)(v2[k] >> 22));
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int gi = q.g[k];
          if (v1[k] < (1ull << 43)) {
            red_shared_add(a1lo + ga[k], (uint32_t)(v1[k] & 0x3FFFFFu));
            red_shared_add(a1hi + ga[k], (uint32_t)(v1[k] >> 22));
          } else {  // huge y (e.g. CPM normalization): straight into the global limbs
            const int go = remap ? remap[gi] : gi;
            if (go >= 0) {
              atomicAdd(&sums[go], v1[k] & 0xFFFFFFFFull);
              atomicAdd(&sums[n_out + go], v1[k] >> 32);
            }
          }
          red_shared_add(a2lo + ga[k], (uint32_t)(v2[k] & 0x3FFFFFu));
          const uint64_t h2 = v2[k] >> 22;
          if (h2 < (1ull << 21)) {
            red_shared_add(a2hi + ga[k], (uint32_t)h2);
          } else {  // huge y^2 (y > ~724)
            const int go = remap ? remap[gi] : gi;
            if (go >= 0) {
              atomicAdd(&sums[2 * n_out + go], (unsigned long long)(h2 & 1023u) << 22);
              atomicAdd(&sums[3 * n_out + go], (unsigned long long)(h2 >> 10));
            }
          }
        }
      }
    }, esc);
  }
  if (out_of_order) atomicOr(order_flag, 1);
  __syncthreads();
  unsigned long long* l0 = sums;               // stat 0 limb 0
  unsigned long long* l1 = sums + n_out;       // stat 0 limb 1
  unsigned long long* m0 = sums + 2 * n_out;   // stat 1 limb 0
  unsigned long long* m1 = sums + 3 * n_out;   // stat 1 limb 1
  // words hold (lo, hi) with value lo + hi * 2^22 = lo + (hi mod 1024) * 2^22 + (hi / 1024) * 2^32
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    const int go = remap ? remap[g0 + i] : g0 + i;
    if (go < 0) continue;
    const unsigned long long a0 = (unsigned long long)s1lo[i] + ((unsigned long long)(s1hi[i] & 1023u) << 22);
    const unsigned long long b0 = (unsigned long long)s2lo[i] + ((unsigned long long)(s2hi[i] & 1023u) << 22);
    if (a0) atomicAdd(&l0[go], a0);
    if (s1hi[i] >> 10) atomicAdd(&l1[go], (unsigned long long)(s1hi[i] >> 10));
    if (b0) atomicAdd(&m0[go], b0);
    if (s2hi[i] >> 10) atomicAdd(&m1[go], (unsigned long long)(s2hi[i] >> 10));
  }
}

// ============================================================================ HVG select
// Single CTA.  All float64 arithmetic uses explicit _rn intrinsics (no FMA contraction)
// so that the oracle (numpy, IEEE double) reproduces it bit for bit.
constexpr int kSelThreads = 1024;
constexpr int kChunks = 64;
constexpr int kMaxBins = 32;

// Canonical value of a limb pair (limb0 + limb1 * 2^32, as an exact integer) rounded once
// to float64 -- independent of how the total was split into limbs across CTAs/ranks.
__device__ __forceinline__ double limbs_to_double(unsigned long long l0, unsigned long long l1) {
  const unsigned long long lo = l0 + (l1 << 32);
  const unsigned long long hi = (l1 >> 32) + (lo < l0 ? 1ull : 0ull);
  if (hi == 0ull) return __ull2double_rn(lo);
  return __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

__device__ __forceinline__ unsigned long long order_key(double d) {
  if (isnan(d)) return 0ull;
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

template <typename T>
__device__ T block_reduce(T v, T (*op)(T, T), T* sbuf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane_id() == 0) sbuf[warp_id()] = v;
  __syncthreads();
  if (warp_id() == 0) {
    v = (lane_id() < (int)(blockDim.x >> 5)) ? sbuf[lane_id()] : sbuf[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane_id() == 0) sbuf[0] = v;
  }
  __syncthreads();
  T r = sbuf[0];
  __syncthreads();
  return r;
}
__device__ double dmin(double a, double b) { return fmin(a, b); }
__device__ double dmax(double a, double b) { return fmax(a, b); }
__device__ int iadd(int a, int b) { return a + b; }

__global__ void __launch_bounds__(kSelThreads)
hvg_select_kernel(const unsigned long long* __restrict__ sums, int32_t G, int64_t N, int32_t n_top,
                  int32_t n_bins, double* __restrict__ means, double* __restrict__ vars,
                  double* __restrict__ disp, double* __restrict__ dnorm, int32_t* __restrict__ mbin,
                  uint8_t* __restrict__ mask, int32_t* __restrict__ hvg_index,
                  int32_t* __restrict__ n_selected, double* __restrict__ mean_log, int32_t ties) {
  __shared__ double sred[32];
  __shared__ int ired[32];
  __shared__ double edges[kMaxBins + 1];
  __shared__ double part[kMaxBins][kChunks];
  __shared__ int npart[kMaxBins][kChunks];
  __shared__ double bmean[kMaxBins], bstd[kMaxBins];
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_need;
  const double Nd = (double)N;
  // ---- 1. per-gene moments
  double lmin = INFINITY, lmax = -INFINITY;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const double s1 = __dmul_rn(limbs_to_double(sums[g], sums[G + g]), 3.725290298461914e-09);   // 2^-28
    const double s2 = __dmul_rn(limbs_to_double(sums[2 * G + g], sums[3 * G + g]), 5.960464477539063e-08);  // 2^-24
    double mean = __ddiv_rn(s1, Nd);
    const double msq = __ddiv_rn(s2, Nd);
    const double var = __dmul_rn(__dsub_rn(msq, __dmul_rn(mean, mean)), __ddiv_rn(Nd, __dsub_rn(Nd, 1.0)));
    vars[g] = var;
    if (mean == 0.0) mean = 1e-12;
    means[g] = mean;
    double d = __ddiv_rn(var, mean);
    d = (d == 0.0) ? CUDART_NAN : log(d);
    disp[g] = d;
    const double ml = log1p(mean);
    mean_log[g] = ml;
    lmin = fmin(lmin, ml);
    lmax = fmax(lmax, ml);
  }
  lmin = block_reduce<double>(lmin, dmin, sred);
  lmax = block_reduce<double>(lmax, dmax, sred);
  // ---- 2. pandas.cut edges
  if (threadIdx.x == 0) {
    if (lmin == lmax) {
      const double adj = (lmin != 0.0) ? __dmul_rn(0.001, fabs(lmin)) : 0.001;
      const double lo = __dsub_rn(lmin, adj), hi = __dadd_rn(lmax, adj);
      const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)n_bins);
      for (int i = 0; i < n_bins; ++i) edges[i] = __dadd_rn(__dmul_rn((double)i, step), lo);
      edges[n_bins] = hi;
    } else {
      const double range = __dsub_rn(lmax, lmin);
      const double step = __ddiv_rn(range, (double)n_bins);
      for (int i = 0; i < n_bins; ++i) edges[i] = __dadd_rn(__dmul_rn((double)i, step), lmin);
      edges[n_bins] = lmax;
      edges[0] = __dsub_rn(edges[0], __dmul_rn(range, 0.001));
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const double x = mean_log[g];
    int c = 0;
    for (int i = 0; i <= n_bins; ++i) c += (edges[i] < x) ? 1 : 0;  // searchsorted(left)
    int b = c - 1;
    b = b < 0 ? 0 : (b > n_bins - 1 ? n_bins - 1 : b);
    mbin[g] = b;
  }
  __syncthreads();
  // ---- 3. per-bin mean and std (ddof=1), fixed chunked order
  const int chunk = (G + kChunks - 1) / kChunks;
  for (int t = threadIdx.x; t < n_bins * kChunks; t += blockDim.x) {
    const int b = t / kChunks, c = t % kChunks;
    double acc = 0.0;
    int n = 0;
    for (int g = c * chunk; g < min(G, (c + 1) * chunk); ++g) {
      const double d = disp[g];
      if (mbin[g] == b && !isnan(d)) { acc = __dadd_rn(acc, d); ++n; }
    }
    part[b][c] = acc;
    npart[b][c] = n;
  }
  __syncthreads();
  if (threadIdx.x < n_bins) {
    const int b = threadIdx.x;
    double acc = 0.0;
    int n = 0;
    for (int c = 0; c < kChunks; ++c) { acc = __dadd_rn(acc, part[b][c]); n += npart[b][c]; }
    bmean[b] = (n > 0) ? __ddiv_rn(acc, (double)n) : CUDART_NAN;
    npart[b][0] = n;  // stash count (chunk 0 slot no longer needed after this point)
  }
  __syncthreads();
  __shared__ int bcount[kMaxBins];
  if (threadIdx.x < n_bins) bcount[threadIdx.x] = npart[threadIdx.x][0];
  __syncthreads();
  for (int t = threadIdx.x; t < n_bins * kChunks; t += blockDim.x) {
    const int b = t / kChunks, c = t % kChunks;
    const double m = bmean[b];
    double acc = 0.0;
    for (int g = c * chunk; g < min(G, (c + 1) * chunk); ++g) {
      const double d = disp[g];
      if (mbin[g] == b && !isnan(d)) {
        const double dd = __dsub_rn(d, m);
        acc = __dadd_rn(acc, __dmul_rn(dd, dd));
      }
    }
    part[b][c] = acc;
  }
  __syncthreads();
  if (threadIdx.x < n_bins) {
    const int b = threadIdx.x;
    const int n = bcount[b];
    double acc = 0.0;
    for (int c = 0; c < kChunks; ++c) acc = __dadd_rn(acc, part[b][c]);
    double sd = (n >= 2) ? sqrt(__ddiv_rn(acc, (double)(n - 1))) : CUDART_NAN;
    double mn = bmean[b];
    if (isnan(sd) && !isnan(mn)) { sd = mn; mn = 0.0; }  // one gene in the bin
    bstd[b] = sd;
    bmean[b] = mn;
  }
  __syncthreads();
  int valid = 0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int b = mbin[g];
    const double dn = __ddiv_rn(__dsub_rn(disp[g], bmean[b]), bstd[b]);
    dnorm[g] = dn;
    valid += isnan(dn) ? 0 : 1;
  }
  valid = block_reduce<int>(valid, iadd, ired);
  const int need_total = min(n_top, valid);
  // ---- 4. radix select of the need_total-th largest key
  if (threadIdx.x == 0) { s_prefix = 0ull; s_need = need_total; }
  __syncthreads();
  unsigned long long prefix_mask = 0ull;
  for (int shift = 56; shift >= 0 && need_total > 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned long long pfx = s_prefix;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      const unsigned long long k = order_key(dnorm[g]);
      if (k != 0ull && (k & prefix_mask) == pfx) atomicAdd(&hist[(k >> shift) & 255], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = s_need;
      int dgt = 255;
      for (; dgt >= 0; --dgt) {
        if ((int)hist[dgt] >= need) break;
        need -= hist[dgt];
      }
      if (dgt < 0) dgt = 0;
      s_prefix = pfx | ((unsigned long long)dgt << shift);
      s_need = need;  // how many to take among keys with the extended prefix
    }
    prefix_mask |= 0xffull << shift;
    __syncthreads();
  }
  const unsigned long long thr = s_prefix;
  // ties (key == thr) are taken in gene-index order: s_need of them
  const int take_ties = s_need;
  __shared__ int tie_carry;
  __shared__ int wtie[32];
  if (threadIdx.x == 0) tie_carry = 0;
  __syncthreads();
  for (int base = 0; base < G; base += blockDim.x) {
    const int g = base + threadIdx.x;
    unsigned long long k = 0ull;
    if (g < G) k = order_key(dnorm[g]);
    const bool tie = (need_total > 0) && g < G && k == thr;
    const unsigned bal = __ballot_sync(0xffffffffu, tie);
    if (lane_id() == 0) wtie[warp_id()] = __popc(bal);
    __syncthreads();
    int before = tie_carry;
    for (int w2 = 0; w2 < warp_id(); ++w2) before += wtie[w2];
    before += __popc(bal & ((1u << lane_id()) - 1u));
    // ties == 1 (Scanpy): every gene whose disp_norm >= the n-th largest; ties == 0: exactly n,
    // ties at the cutoff taken in gene-index order
    bool sel = (need_total > 0) && g < G && k != 0ull && (k > thr || (tie && (ties == 1 || before < take_ties)));
    if (g < G) mask[g] = sel ? 1 : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) tot += wtie[w2];
      tie_carry += tot;
    }
    __syncthreads();
  }
  // ---- 5. sorted index list
  __shared__ int sel_carry;
  if (threadIdx.x == 0) sel_carry = 0;
  __syncthreads();
  for (int base = 0; base < G; base += blockDim.x) {
    const int g = base + threadIdx.x;
    const bool s = g < G && mask[g];
    const unsigned bal = __ballot_sync(0xffffffffu, s);
    if (lane_id() == 0) wtie[warp_id()] = __popc(bal);
    __syncthreads();
    int before = sel_carry;
    for (int w2 = 0; w2 < warp_id(); ++w2) before += wtie[w2];
    before += __popc(bal & ((1u << lane_id()) - 1u));
    if (s) hvg_index[before] = g;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) tot += wtie[w2];
      sel_carry += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_selected = sel_carry;
}

// ============================================================================ scale
__global__ void __launch_bounds__(kRowThreads, 2)
scale_sums_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                  const float* __restrict__ ldata, int64_t n_rows, int32_t n_cols,
                  const int32_t* __restrict__ slot, int32_t n_slots, int64_t rows_per_block,
                  unsigned long long* __restrict__ sums) {
  // CTA = block of <= 1024 rows: the carry-free (22-bit low, high) split of every fixed-point
  // value keeps both u32 words below 2^32, so all smem atomics are fire-and-forget
  const int64_t nnz = indptr[n_rows];
  extern __shared__ uint32_t sm[];
  int16_t* s_slot = reinterpret_cast<int16_t*>(sm + 4 * n_slots);
  for (int i = threadIdx.x; i < 4 * n_slots; i += blockDim.x) sm[i] = 0;
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) s_slot[i] = (int16_t)slot[i];
  __syncthreads();
  uint32_t* s1lo = sm;
  uint32_t* s1hi = sm + n_slots;
  uint32_t* s2lo = sm + 2 * n_slots;
  uint32_t* s2hi = sm + 3 * n_slots;
  const uint32_t a1lo = smem_addr(s1lo), a1hi = smem_addr(s1hi), a2lo = smem_addr(s2lo), a2hi = smem_addr(s2hi);
  const uint32_t a_slot = smem_addr(s_slot);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(n_rows, r0 + rows_per_block);
  for (int64_t r = r0 + warp_id(); r < r1; r += (blockDim.x >> 5)) {
    // per quad: slot lookups first; quads without an HVG entry cost four LDS; HVG entries get
    // v1 = round(l * 2^28) (exact f32 scaling, one RN conversion) and v2 = round((l * 2^12)^2)
    // (exact f64 square) -- the oracle's round(l * 2^28), round(l^2 * 2^24).  High words
    // stay below 2^32 for values < 2^43 (|l| < 2^15, l^2 < 2^19); larger ones (not
    // log-normalized data) go straight to the global limbs.
    stream_row_pipe<1>(indices, ldata, indptr[r], indptr[r + 1], nnz, [&](const Quad& q) {
      int j[4];
      bool any = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        j[k] = ((q.valid >> k) & 1u) ? (int)lds_s16(a_slot + 2u * (uint32_t)q.g[k]) : -1;
        any |= j[k] >= 0;
      }
      if (!any) return;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (j[k] < 0) continue;  // most entries are not HVGs: skip their atomics entirely
        const float l = q.x[k];
        const uint64_t v1 = (uint64_t)__float2ull_rn(__fmul_rn(l, 268435456.0f));
        const double l12 = (double)__fmul_rn(l, 4096.0f);
        const uint64_t v2 = (uint64_t)__double2ull_rn(__dmul_rn(l12, l12));
        const uint32_t ja = 4u * (uint32_t)j[k];
        if ((v1 | v2) < (1ull << 43)) {
          red_shared_add(a1lo + ja, (uint32_t)(v1 & 0x3FFFFFu));
          red_shared_add(a1hi + ja, (uint32_t)(v1 >> 22));
          red_shared_add(a2lo + ja, (uint32_t)(v2 & 0x3FFFFFu));
          red_shared_add(a2hi + ja, (uint32_t)(v2 >> 22));
        } else {  // rare
          if (v1 < (1ull << 43)) {
            red_shared_add(a1lo + ja, (uint32_t)(v1 & 0x3FFFFFu));
            red_shared_add(a1hi + ja, (uint32_t)(v1 >> 22));
          } else {
            atomicAdd(&sums[j[k]], v1 & 0xFFFFFFFFull);
            atomicAdd(&sums[n_slots + j[k]], v1 >> 32);
          }
          if (v2 < (1ull << 43)) {
            red_shared_add(a2lo + ja, (uint32_t)(v2 & 0x3FFFFFu));
            red_shared_add(a2hi + ja, (uint32_t)(v2 >> 22));
          } else {
            atomicAdd(&sums[2 * n_slots + j[k]], v2 & 0xFFFFFFFFull);
            atomicAdd(&sums[3 * n_slots + j[k]], v2 >> 32);
          }
        }
      }
    });
  }
  __syncthreads();
  // limbs: value = limb0 + limb1 * 2^32; a word pair holds lo + hi * 2^22
  for (int i = threadIdx.x; i < n_slots; i += blockDim.x) {
    const unsigned long long a0 = (unsigned long long)s1lo[i] + ((unsigned long long)(s1hi[i] & 1023u) << 22);
    const unsigned long long b0 = (unsigned long long)s2lo[i] + ((unsigned long long)(s2hi[i] & 1023u) << 22);
    if (a0) atomicAdd(&sums[i], a0);
    if (s1hi[i] >> 10) atomicAdd(&sums[n_slots + i], (unsigned long long)(s1hi[i] >> 10));
    if (b0) atomicAdd(&sums[2 * n_slots + i], b0);
    if (s2hi[i] >> 10) atomicAdd(&sums[3 * n_slots + i], (unsigned long long)(s2hi[i] >> 10));
  }
}

__global__ void scale_finalize_kernel(const unsigned long long* __restrict__ sums, int32_t H, int64_t N,
                                      double* __restrict__ mean, double* __restrict__ inv_std) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  const double Nd = (double)N;
  const double s1 = __dmul_rn(limbs_to_double(sums[j], sums[H + j]), 3.725290298461914e-09);
  const double s2 = __dmul_rn(limbs_to_double(sums[2 * H + j], sums[3 * H + j]), 5.960464477539063e-08);
  const double m = __ddiv_rn(s1, Nd);
  const double msq = __ddiv_rn(s2, Nd);
  const double var = __dmul_rn(__dsub_rn(msq, __dmul_rn(m, m)), __ddiv_rn(Nd, __dsub_rn(Nd, 1.0)));
  double sd = sqrt(var);
  if (sd == 0.0 || isnan(sd)) sd = 1.0;  // var < 0 by rounding -> NaN -> 1 (documented)
  mean[j] = m;
  inv_std[j] = __ddiv_rn(1.0, sd);
}

// Dense gather: one warp per row.  Background row (z0, ones column, zero padding) is
// written with 16-byte stores, then (after __syncwarp, which orders the warp's global
// stores) the row's HVG entries are scattered on top.
__global__ void __launch_bounds__(kRowThreads)
scale_dense_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                   const float* __restrict__ ldata, int64_t n_rows, int32_t n_cols,
                   const int32_t* __restrict__ slot, int32_t H, const double* __restrict__ mean,
                   const double* __restrict__ inv, double max_value, double min_value, float* __restrict__ Z,
                   int64_t ldz, int32_t ones_col) {
  const int64_t nnz = indptr[n_rows];
  extern __shared__ float zsm[];                        // background row [ldz]
  int16_t* s_slot = reinterpret_cast<int16_t*>(zsm + ldz);
  double* s_mean = reinterpret_cast<double*>(s_slot + ((n_cols + 3) & ~3));
  double* s_inv = s_mean + H;
  for (int j = threadIdx.x; j < ldz; j += blockDim.x) {
    float v = 0.0f;
    if (j < H) v = (float)fmax(fmin(__dmul_rn(__dsub_rn(0.0, mean[j]), inv[j]), max_value), min_value);
    else if (j == ones_col) v = 1.0f;
    zsm[j] = v;
  }
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) s_slot[i] = (int16_t)slot[i];
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    s_mean[j] = mean[j];
    s_inv[j] = inv[j];
  }
  __syncthreads();
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const float4* bg = reinterpret_cast<const float4*>(zsm);
  const int n4 = (int)(ldz >> 2);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); r < n_rows; r += warps) {
    float* zr = Z + r * ldz;
    float4* zr4 = reinterpret_cast<float4*>(zr);
    for (int j = lane; j < n4; j += 32) zr4[j] = bg[j];
    __syncwarp();  // orders this warp's background stores before the scattered overwrites
    stream_row<2>(indices, ldata, indptr[r], indptr[r + 1], nnz, [&](const Quad& q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((q.valid >> k) & 1u)) continue;
        const int j = s_slot[q.g[k]];
        if (j >= 0)
          zr[j] = (float)fmax(fmin(__dmul_rn(__dsub_rn((double)q.x[k], s_mean[j]), s_inv[j]), max_value), min_value);
      }
    });
    __syncwarp();
  }
}


// Planes variant: the same clipped z-scores written directly as the Gram's / projection's BF16
// operand planes hi = bf16(z), lo = bf16(z - hi) (bit-identical to scb_split_bf16 of the fp32
// matrix) -- the fp32 matrix and the separate split pass (8 GB read + 8 GB write at C3) are gone.
__global__ void __launch_bounds__(kRowThreads)
scale_dense_planes_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                          const float* __restrict__ ldata, int64_t n_rows, int32_t n_cols,
                          const int32_t* __restrict__ slot, int32_t H, const double* __restrict__ mean,
                          const double* __restrict__ inv, double max_value, double min_value,
                          __nv_bfloat16* __restrict__ Zh, __nv_bfloat16* __restrict__ Zl, int64_t ldz,
                          int32_t ones_col) {
  const int64_t nnz = indptr[n_rows];
  extern __shared__ float zsm[];                        // background rows: hi [ldz], lo [ldz] (bf16)
  __nv_bfloat16* bh = reinterpret_cast<__nv_bfloat16*>(zsm);
  __nv_bfloat16* bl = bh + ldz;
  int16_t* s_slot = reinterpret_cast<int16_t*>(bl + ldz);
  double* s_mean = reinterpret_cast<double*>(s_slot + ((n_cols + 7) & ~7));
  double* s_inv = s_mean + H;
  for (int j = threadIdx.x; j < ldz; j += blockDim.x) {
    float v = 0.0f;
    if (j < H) v = (float)fmax(fmin(__dmul_rn(__dsub_rn(0.0, mean[j]), inv[j]), max_value), min_value);
    else if (j == ones_col) v = 1.0f;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    bh[j] = h;
    bl[j] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
  for (int i = threadIdx.x; i < n_cols; i += blockDim.x) s_slot[i] = (int16_t)slot[i];
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    s_mean[j] = mean[j];
    s_inv[j] = inv[j];
  }
  __syncthreads();
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint4* bgh = reinterpret_cast<const uint4*>(bh);
  const uint4* bgl = reinterpret_cast<const uint4*>(bl);
  const int n8 = (int)(ldz >> 3);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); r < n_rows; r += warps) {
    __nv_bfloat16* zh = Zh + r * ldz;
    __nv_bfloat16* zl = Zl + r * ldz;
    uint4* zh4 = reinterpret_cast<uint4*>(zh);
    uint4* zl4 = reinterpret_cast<uint4*>(zl);
    for (int j = lane; j < n8; j += 32) {
      zh4[j] = bgh[j];
      zl4[j] = bgl[j];
    }
    __syncwarp();  // orders this warp's background stores before the scattered overwrites
    stream_row<2>(indices, ldata, indptr[r], indptr[r + 1], nnz, [&](const Quad& q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((q.valid >> k) & 1u)) continue;
        const int j = s_slot[q.g[k]];
        if (j >= 0) {
          const float z = (float)fmax(fmin(__dmul_rn(__dsub_rn((double)q.x[k], s_mean[j]), s_inv[j]), max_value),
                                      min_value);
          const __nv_bfloat16 h = __float2bfloat16_rn(z);
          zh[j] = h;
          zl[j] = __float2bfloat16_rn(z - __bfloat162float(h));
        }
      }
    });
    __syncwarp();
  }
}

}  // namespace scb

// ============================================================================ C ABI
using namespace scb;

extern "C" int32_t scb_hvg_tiles(int32_t n_cols) { return n_cols <= 0 ? 1 : (n_cols + kHvgTileW - 1) / kHvgTileW; }

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <typename IT, typename VT>
static int qc_metrics_impl(scb_ctx* ctx, const int64_t* indptr, const IT* indices,
                              const VT* data, int64_t n_rows, int32_t n_cols, const uint8_t* mt_mask,
                              int32_t* n_genes, double* total, double* total_mt, double* pct,
                              int32_t* n_cells, double* gene_total, int32_t* hvg_row_splits, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream) {
  const U16Esc esc{esc_pos, esc_val, n_esc};
  SCB_REQUIRE(ctx && indptr && mt_mask && n_genes && total && total_mt && pct && n_cells && gene_total,
              SCB_ERR_ARG, "scb_qc_metrics: null argument");
  SCB_REQUIRE(n_rows >= 0 && n_cols > 0, SCB_ERR_ARG, "scb_qc_metrics: bad shape");
  SCB_REQUIRE(aligned16(indices) && aligned16(data), SCB_ERR_ARG, "scb_qc_metrics: indices/data must be 16-byte aligned");
  const int n_tiles_hvg = scb_hvg_tiles(n_cols);
  SCB_REQUIRE(n_tiles_hvg - 1 <= kMaxSplit, SCB_ERR_UNSUPPORTED, "scb_qc_metrics: too many genes (max %d)",
              (kMaxSplit + 1) * kHvgTileW);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t mt_bytes = ((size_t)n_cols + 15) & ~(size_t)15;
  SCB_REQUIRE(mt_bytes + 8 * 1024 <= kSmemLimit, SCB_ERR_UNSUPPORTED, "scb_qc_metrics: too many genes");
  const int max_w = (int)((kSmemLimit - mt_bytes) / 4);
  const int n_tiles = ceil_div(n_cols, max_w);
  const int tile_w = ceil_div(n_cols, n_tiles);
  void* ws;
  const size_t ws_bytes = (size_t)n_cols * 4 + (size_t)n_cols * 8;
  SCB_TRY(ws_get(ctx, 0, ws_bytes + 16, &ws, s));
  uint32_t* g_cells = (uint32_t*)ws;
  unsigned long long* g_total = (unsigned long long*)((char*)ws + ((size_t)n_cols * 4 + 7) / 8 * 8);
  SCB_CUDA(cudaMemsetAsync(ws, 0, ws_bytes + 8, s));
  SCB_CUDA(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), s));
  const size_t smem = (size_t)tile_w * 4 + mt_bytes;
  const int n_split = hvg_row_splits ? n_tiles_hvg - 1 : 0;
  if (n_rows > 0) {
    dim3 grid((unsigned)grid_for(ctx, 1), n_tiles);
    auto launch = [&](auto kern) {
      SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<grid, kQcThreads, smem, s>>>(indptr, indices, data, n_rows, n_cols, mt_mask, tile_w, n_split, kHvgTileW,
                                          hvg_row_splits, n_genes, total, total_mt, pct, g_cells, g_total, ctx->d_flag, esc);
      return SCB_OK;
    };
    static_assert(kMaxSplit == 3, "qc_kernel is instantiated for 0..3 row splits");
    if (n_tiles == 1) {
      switch (n_split) {
        case 0: SCB_TRY(launch(qc_kernel<IT, VT, 0, true>)); break;
        case 1: SCB_TRY(launch(qc_kernel<IT, VT, 1, true>)); break;
        case 2: SCB_TRY(launch(qc_kernel<IT, VT, 2, true>)); break;
        default: SCB_TRY(launch(qc_kernel<IT, VT, 3, true>)); break;
      }
    } else {
      switch (n_split) {
        case 0: SCB_TRY(launch(qc_kernel<IT, VT, 0, false>)); break;
        case 1: SCB_TRY(launch(qc_kernel<IT, VT, 1, false>)); break;
        case 2: SCB_TRY(launch(qc_kernel<IT, VT, 2, false>)); break;
        default: SCB_TRY(launch(qc_kernel<IT, VT, 3, false>)); break;
      }
    }
    SCB_LAUNCH_CHECK();
  }
  qc_finalize<<<ceil_div(n_cols, 256), 256, 0, s>>>(g_cells, g_total, n_cols, n_cells, gene_total);
  SCB_LAUNCH_CHECK();
  if (ctx->defer_checks) return SCB_OK;  // the flag is reported by scb_filter_masks (n_kept[3])
  int flag = 0;
  SCB_CUDA(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  SCB_REQUIRE(flag == 0, SCB_ERR_DATA,
              "scb_qc_metrics: counts must be non-negative integers < 2^24 with column indices in range");
  return SCB_OK;
}

extern "C" int scb_qc_metrics(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                              const float* data, int64_t n_rows, int32_t n_cols, const uint8_t* mt_mask,
                              int32_t* n_genes, double* total, double* total_mt, double* pct,
                              int32_t* n_cells, double* gene_total, int32_t* hvg_row_splits, void* stream) {
  return qc_metrics_impl<int32_t, float>(ctx, indptr, indices, data, n_rows, n_cols, mt_mask, n_genes, total, total_mt, pct, n_cells, gene_total, hvg_row_splits, nullptr, nullptr, 0, stream);
}

extern "C" int scb_qc_metrics_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                              const uint16_t* data, int64_t n_rows, int32_t n_cols, const uint8_t* mt_mask,
                              int32_t* n_genes, double* total, double* total_mt, double* pct,
                              int32_t* n_cells, double* gene_total, int32_t* hvg_row_splits, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                              void* stream) {
  return qc_metrics_impl<uint16_t, uint16_t>(ctx, indptr, indices, data, n_rows, n_cols, mt_mask, n_genes, total, total_mt, pct, n_cells, gene_total, hvg_row_splits, esc_pos, esc_val, n_esc, stream);
}

extern "C" int scb_filter_masks(scb_ctx* ctx, const int32_t* ng, const double* pct, int64_t n_rows,
                                const int32_t* nc, int32_t n_cols, int32_t min_genes, int32_t max_genes,
                                double max_pct, int32_t min_cells, const int64_t* indptr, uint8_t* cmask,
                                uint8_t* gmask, int64_t* n_kept, void* stream) {
  SCB_REQUIRE(ctx && ng && pct && nc && cmask && gmask && n_kept, SCB_ERR_ARG, "scb_filter_masks: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  SCB_CUDA(cudaMemsetAsync(n_kept, 0, 4 * sizeof(int64_t), s));
  if (n_rows > 0) {
    cell_mask_kernel<<<ceil_div(n_rows, 256), 256, 0, s>>>(ng, pct, n_rows, min_genes, max_genes, max_pct,
                                                           cmask, (unsigned long long*)n_kept);
    SCB_LAUNCH_CHECK();
  }
  gene_mask_kernel<<<ceil_div(n_cols, 256), 256, 0, s>>>(nc, n_cols, min_cells, gmask,
                                                         (unsigned long long*)n_kept);
  SCB_LAUNCH_CHECK();
  if (indptr && n_rows > 0) {
    kept_nnz_kernel<<<grid_for(ctx, 2), 256, 0, s>>>(indptr, cmask, n_rows, (unsigned long long*)(n_kept + 2));
    SCB_LAUNCH_CHECK();
  }
  copy_flag_kernel<<<1, 1, 0, s>>>(ctx->d_flag, (long long*)(n_kept + 3));
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_subset_rows_all_genes(scb_ctx* ctx, const int64_t* indptr, int64_t n_rows, int32_t n_cols,
                                         const uint8_t* cmask, const double* total_counts, double target_sum,
                                         int32_t* remap, int64_t* new_indptr, float* row_scale,
                                         float* row_scale_orig, void* stream) {
  SCB_REQUIRE(ctx && indptr && cmask && total_counts && remap && new_indptr && row_scale, SCB_ERR_ARG,
              "scb_subset_rows_all_genes: null argument");
  cudaStream_t s = (cudaStream_t)stream;
  identity_remap_kernel<<<ceil_div(n_cols, 256), 256, 0, s>>>(n_cols, remap);
  SCB_LAUNCH_CHECK();
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8 * 2, &ws, s));
  int64_t* row_pos = (int64_t*)ws;
  int64_t* cnt = row_pos + (n_rows + 1);
  SCB_TRY(scan_u8_to_i64(ctx, cmask, n_rows, row_pos, s));
  if (n_rows > 0) {
    rows_all_genes_kernel<<<grid_for(ctx, 8), 256, 0, s>>>(indptr, cmask, row_pos, total_counts, n_rows, target_sum,
                                                           cnt, row_scale, row_scale_orig);
    SCB_LAUNCH_CHECK();
  }
  SCB_TRY(scan_i64_dev_len(ctx, cnt, row_pos + n_rows, n_rows, new_indptr, s));
  return SCB_OK;
}

template <typename IT, typename VT>
static int subset_count_impl(scb_ctx* ctx, const int64_t* indptr, const IT* indices,
                                const VT* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                const uint8_t* gmask, int32_t* remap, int64_t* new_indptr,
                                double target_sum, float* row_scale, float* row_scale_orig, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream) {
  const U16Esc esc{esc_pos, esc_val, n_esc};
  SCB_REQUIRE(ctx && indptr && indices && cmask && gmask && remap && new_indptr, SCB_ERR_ARG,
              "scb_subset_count: null argument");
  SCB_REQUIRE(!row_scale || data, SCB_ERR_ARG, "scb_subset_count: row_scale needs data");
  SCB_REQUIRE(aligned16(indices) && (!data || aligned16(data)), SCB_ERR_ARG, "scb_subset_count: 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  gene_remap_kernel<<<1, 1024, 0, s>>>(gmask, n_cols, remap);
  SCB_LAUNCH_CHECK();
  // row_pos = exclusive scan of cell_mask (int64), cnt[kept] then scanned into new_indptr
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8 * 2, &ws, s));
  int64_t* row_pos = (int64_t*)ws;
  int64_t* cnt = row_pos + (n_rows + 1);
  SCB_TRY(scan_u8_to_i64(ctx, cmask, n_rows, row_pos, s));
  if (n_rows > 0) {
    const bool small = n_cols <= 32767;
    const size_t map_bytes = small ? (size_t)((n_cols + 7) & ~7) * 2 : (size_t)((n_cols + 31) / 32) * 8;
    SCB_REQUIRE(map_bytes <= 64 * 1024, SCB_ERR_UNSUPPORTED, "scb_subset_count: too many genes");
    auto kern = small ? subset_count_kernel<IT, VT, true> : subset_count_kernel<IT, VT, false>;
    SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)map_bytes));
    kern<<<grid_for(ctx, 4), kRowThreads, map_bytes, s>>>(indptr, indices, data, n_rows, cmask, remap, n_cols,
                                                          row_pos, cnt, target_sum, row_scale, row_scale_orig, esc);
    SCB_LAUNCH_CHECK();
  }
  // number of kept rows is row_pos[n_rows]; scan cnt[0..kept) -> new_indptr (device-side length)
  SCB_TRY(scan_i64_dev_len(ctx, cnt, row_pos + n_rows, n_rows, new_indptr, s));
  return SCB_OK;
}

extern "C" int scb_subset_count(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                                const float* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                const uint8_t* gmask, int32_t* remap, int64_t* new_indptr,
                                double target_sum, float* row_scale, float* row_scale_orig, void* stream) {
  return subset_count_impl<int32_t, float>(ctx, indptr, indices, data, n_rows, n_cols, cmask, gmask, remap, new_indptr, target_sum, row_scale, row_scale_orig, nullptr, nullptr, 0, stream);
}

extern "C" int scb_subset_count_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                                const uint16_t* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                const uint8_t* gmask, int32_t* remap, int64_t* new_indptr,
                                double target_sum, float* row_scale, float* row_scale_orig, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                              void* stream) {
  return subset_count_impl<uint16_t, uint16_t>(ctx, indptr, indices, data, n_rows, n_cols, cmask, gmask, remap, new_indptr, target_sum, row_scale, row_scale_orig, esc_pos, esc_val, n_esc, stream);
}

template <typename IT, typename VT>
static int subset_fill_impl(scb_ctx* ctx, const int64_t* indptr, const IT* indices,
                               const VT* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                               const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                               int32_t* new_indices, float* new_data, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream) {
  const U16Esc esc{esc_pos, esc_val, n_esc};
  SCB_REQUIRE(ctx && indptr && indices && data && cmask && remap && new_indptr && new_indices && new_data,
              SCB_ERR_ARG, "scb_subset_fill: null argument");
  SCB_REQUIRE(aligned16(indices) && aligned16(data), SCB_ERR_ARG, "scb_subset_fill: 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8 * 2, &ws, s));
  int64_t* row_pos = (int64_t*)ws;
  SCB_TRY(scan_u8_to_i64(ctx, cmask, n_rows, row_pos, s));
  if (n_rows > 0) {
    const bool small = n_cols <= 32767;
    const size_t map_bytes = small ? (size_t)((n_cols + 7) & ~7) * 2 : (size_t)((n_cols + 31) / 32) * 8;
    SCB_REQUIRE(map_bytes <= 64 * 1024, SCB_ERR_UNSUPPORTED, "scb_subset_fill: too many genes");
    auto kern = small ? subset_fill_kernel<IT, VT, true> : subset_fill_kernel<IT, VT, false>;
    SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)map_bytes));
    kern<<<grid_for(ctx, 4), kRowThreads, map_bytes, s>>>(indptr, indices, data, n_rows, cmask, remap, n_cols,
                                                          row_pos, new_indptr, row_scale, new_indices, new_data, esc);
    SCB_LAUNCH_CHECK();
  }
  return SCB_OK;
}

extern "C" int scb_subset_fill(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                               const float* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                               const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                               int32_t* new_indices, float* new_data, void* stream) {
  return subset_fill_impl<int32_t, float>(ctx, indptr, indices, data, n_rows, n_cols, cmask, remap, new_indptr, row_scale, new_indices, new_data, nullptr, nullptr, 0, stream);
}

extern "C" int scb_subset_fill_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                               const uint16_t* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                               const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                               int32_t* new_indices, float* new_data, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                              void* stream) {
  return subset_fill_impl<uint16_t, uint16_t>(ctx, indptr, indices, data, n_rows, n_cols, cmask, remap, new_indptr, row_scale, new_indices, new_data, esc_pos, esc_val, n_esc, stream);
}

template <typename IT, typename VT>
static int subset_fill_scale_sums_impl(scb_ctx* ctx, const int64_t* indptr, const IT* indices,
                                          const VT* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                          const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                                          const int32_t* slot, int32_t n_slots, int32_t* new_indices,
                                          float* new_data, uint64_t* sums, const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream) {
  const U16Esc esc{esc_pos, esc_val, n_esc};
  SCB_REQUIRE(ctx && indptr && indices && data && cmask && remap && new_indptr && row_scale && slot &&
                  (new_indices || std::is_same<IT, int32_t>::value) && new_data && sums,
              SCB_ERR_ARG, "scb_subset_fill_scale_sums: null argument");
  SCB_REQUIRE(aligned16(indices) && aligned16(data), SCB_ERR_ARG, "scb_subset_fill_scale_sums: 16-byte alignment");
  SCB_REQUIRE(n_cols <= 32767 && n_slots > 0 && n_slots < 32767, SCB_ERR_UNSUPPORTED,
              "scb_subset_fill_scale_sums: needs n_cols <= 32767 (use subset_fill + scale_gene_sums)");
  const size_t smem = (size_t)((n_cols + 3) & ~3) * 4 + (size_t)n_slots * 16;
  SCB_REQUIRE(smem + 32 * 1024 <= kSmemLimit, SCB_ERR_UNSUPPORTED, "scb_subset_fill_scale_sums: too many genes");
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_rows + 1) * 8 * 2, &ws, s));
  int64_t* row_pos = (int64_t*)ws;
  SCB_TRY(scan_u8_to_i64(ctx, cmask, n_rows, row_pos, s));
  if (n_rows == 0) return SCB_OK;
  const int64_t rpb = 1024;  // carry-free fixed point
  SCB_CUDA(cudaFuncSetAttribute(subset_fill_sums_kernel<IT, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  subset_fill_sums_kernel<IT, VT><<<(unsigned)((n_rows + rpb - 1) / rpb), kFillSumsThreads, smem, s>>>(
      indptr, indices, data, n_rows, cmask, remap, n_cols, slot, n_slots, row_pos, new_indptr, row_scale, rpb,
      new_indices, new_data, (unsigned long long*)sums, esc);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_subset_fill_scale_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                                          const float* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                          const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                                          const int32_t* slot, int32_t n_slots, int32_t* new_indices,
                                          float* new_data, uint64_t* sums, void* stream) {
  return subset_fill_scale_sums_impl<int32_t, float>(ctx, indptr, indices, data, n_rows, n_cols, cmask, remap, new_indptr, row_scale, slot, n_slots, new_indices, new_data, sums, nullptr, nullptr, 0, stream);
}

extern "C" int scb_subset_fill_scale_sums_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                                          const uint16_t* data, int64_t n_rows, int32_t n_cols, const uint8_t* cmask,
                                          const int32_t* remap, const int64_t* new_indptr, const float* row_scale,
                                          const int32_t* slot, int32_t n_slots, int32_t* new_indices,
                                          float* new_data, uint64_t* sums, const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                              void* stream) {
  return subset_fill_scale_sums_impl<uint16_t, uint16_t>(ctx, indptr, indices, data, n_rows, n_cols, cmask, remap, new_indptr, row_scale, slot, n_slots, new_indices, new_data, sums, esc_pos, esc_val, n_esc, stream);
}

extern "C" int scb_normalize_log1p(scb_ctx* ctx, const int64_t* indptr, const float* data, int64_t n_rows,
                                   double target_sum, float* out, float* row_scale, void* stream) {
  SCB_REQUIRE(ctx && indptr && data && out && row_scale, SCB_ERR_ARG, "scb_normalize_log1p: null argument");
  SCB_REQUIRE(target_sum > 0, SCB_ERR_ARG, "scb_normalize_log1p: target_sum must be > 0");
  if (n_rows == 0) return SCB_OK;
  normalize_log1p_kernel<<<grid_for(ctx, 4), kRowThreads, 0, (cudaStream_t)stream>>>(indptr, data, n_rows,
                                                                                     target_sum, out, row_scale);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

template <typename IT, typename VT>
static int hvg_gene_sums_impl(scb_ctx* ctx, const int64_t* indptr, const IT* indices,
                                 const VT* data, const float* row_scale, int64_t n_rows, int32_t n_cols,
                                 const int32_t* remap, int32_t n_out, const int32_t* row_splits, uint64_t* sums,
                                 const int64_t* esc_pos, const float* esc_val, int64_t n_esc, void* stream) {
  const U16Esc esc{esc_pos, esc_val, n_esc};
  SCB_REQUIRE(ctx && indptr && indices && data && row_scale && sums, SCB_ERR_ARG,
              "scb_hvg_gene_sums: null argument");
  SCB_REQUIRE(n_out > 0, SCB_ERR_ARG, "scb_hvg_gene_sums: n_out must be > 0");
  SCB_REQUIRE(aligned16(indices) && aligned16(data), SCB_ERR_ARG, "scb_hvg_gene_sums: 16-byte alignment");
  if (n_rows == 0) return SCB_OK;
  const int n_tiles = scb_hvg_tiles(n_cols);
  const int tile_w = kHvgTileW;
  const size_t smem = (size_t)std::min(tile_w, n_cols) * 16;
  // row blocks of <= 1024 rows: the 22-bit low words cannot overflow (1024 * 2^22 = 2^32)
  int64_t rows_per_block = std::max<int64_t>(64, std::min<int64_t>(1024, n_rows / (2 * ctx->num_sms) + 1));
  const int64_t n_blocks = (n_rows + rows_per_block - 1) / rows_per_block;
  SCB_CUDA(cudaFuncSetAttribute(hvg_sums_kernel<IT, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaStream_t s = (cudaStream_t)stream;
  const bool split = row_splits && n_tiles > 1;
  if (!split) {
    hvg_sums_kernel<IT, VT><<<(unsigned)(n_blocks * n_tiles), kHvgThreads, smem, s>>>(
        indptr, indices, data, row_scale, n_rows, n_cols, remap, n_out, std::min(tile_w, n_cols), n_tiles, nullptr,
        rows_per_block, (unsigned long long*)sums, ctx->d_flag + 1, esc);
    SCB_LAUNCH_CHECK();
    return SCB_OK;
  }
  // The row splits assume sorted column indices within each row (canonical CSR).  The split
  // pass accumulates into scratch; if it saw an entry outside its tile (unsorted row) the
  // scratch is recomputed with every tile filtering whole rows, then added into sums (+=).
  const size_t sbytes = (size_t)4 * n_out * sizeof(uint64_t);
  void* ws;
  SCB_TRY(ws_get(ctx, 2, sbytes, &ws, s));
  unsigned long long* tmp = (unsigned long long*)ws;
  int* order_flag = ctx->d_flag + 1;
  SCB_CUDA(cudaMemsetAsync(tmp, 0, sbytes, s));
  SCB_CUDA(cudaMemsetAsync(order_flag, 0, sizeof(int), s));
  hvg_sums_kernel<IT, VT><<<(unsigned)(n_blocks * n_tiles), kHvgThreads, smem, s>>>(
      indptr, indices, data, row_scale, n_rows, n_cols, remap, n_out, std::min(tile_w, n_cols), n_tiles, row_splits,
      rows_per_block, tmp, order_flag, esc);
  SCB_LAUNCH_CHECK();
  // unsorted rows seen: redo without splits -- launched unconditionally, both kernels exit at
  // once unless the device-side flag is set (no host round trip)
  zero_if_flag_kernel<<<ceil_div(4 * n_out, 256), 256, 0, s>>>(tmp, (int64_t)4 * n_out, order_flag);
  SCB_LAUNCH_CHECK();
  hvg_sums_kernel<IT, VT><<<(unsigned)(n_blocks * n_tiles), kHvgThreads, smem, s>>>(
      indptr, indices, data, row_scale, n_rows, n_cols, remap, n_out, std::min(tile_w, n_cols), n_tiles, nullptr,
      rows_per_block, tmp, ctx->d_flag + 3, esc, order_flag);
  SCB_LAUNCH_CHECK();
  add_u64_kernel<<<ceil_div(4 * n_out, 256), 256, 0, s>>>(tmp, (unsigned long long*)sums, (int64_t)4 * n_out);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_hvg_gene_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                                 const float* data, const float* row_scale, int64_t n_rows, int32_t n_cols,
                                 const int32_t* remap, int32_t n_out, const int32_t* row_splits, uint64_t* sums,
                                 void* stream) {
  return hvg_gene_sums_impl<int32_t, float>(ctx, indptr, indices, data, row_scale, n_rows, n_cols, remap, n_out, row_splits, sums, nullptr, nullptr, 0, stream);
}

extern "C" int scb_hvg_gene_sums_u16(scb_ctx* ctx, const int64_t* indptr, const uint16_t* indices,
                                 const uint16_t* data, const float* row_scale, int64_t n_rows, int32_t n_cols,
                                 const int32_t* remap, int32_t n_out, const int32_t* row_splits, uint64_t* sums,
                                 const int64_t* esc_pos, const float* esc_val, int64_t n_esc,
                              void* stream) {
  return hvg_gene_sums_impl<uint16_t, uint16_t>(ctx, indptr, indices, data, row_scale, n_rows, n_cols, remap, n_out, row_splits, sums, esc_pos, esc_val, n_esc, stream);
}

extern "C" int scb_hvg_select(scb_ctx* ctx, const uint64_t* sums, int32_t n_cols, int64_t n_cells,
                              int32_t n_top, int32_t n_bins, int32_t ties, double* means, double* vars, double* disp,
                              double* dnorm, int32_t* mbin, uint8_t* mask, int32_t* hvg_index,
                              int32_t* n_selected, void* stream) {
  SCB_REQUIRE(ctx && sums && means && vars && disp && dnorm && mbin && mask && hvg_index && n_selected,
              SCB_ERR_ARG, "scb_hvg_select: null argument");
  SCB_REQUIRE(n_bins >= 1 && n_bins <= kMaxBins, SCB_ERR_ARG, "scb_hvg_select: n_bins must be in [1, %d]",
              kMaxBins);
  SCB_REQUIRE(n_cells >= 2 && n_cols >= 1 && n_top >= 0, SCB_ERR_ARG, "scb_hvg_select: bad sizes");
  SCB_REQUIRE(ties == 0 || ties == 1, SCB_ERR_ARG, "scb_hvg_select: ties must be 0 (exactly n_top) or 1 (Scanpy >= cutoff)");
  cudaStream_t s = (cudaStream_t)stream;
  void* ws;
  SCB_TRY(ws_get(ctx, 2, (size_t)n_cols * 8, &ws, s));
  hvg_select_kernel<<<1, kSelThreads, 0, s>>>((const unsigned long long*)sums, n_cols, n_cells, n_top, n_bins,
                                              means, vars, disp, dnorm, mbin, mask, hvg_index, n_selected,
                                              (double*)ws, ties);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_scale_gene_sums(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                                   const float* ldata, int64_t n_rows, int32_t n_cols, const int32_t* slot,
                                   int32_t n_slots, uint64_t* sums, void* stream) {
  SCB_REQUIRE(ctx && indptr && indices && ldata && slot && sums, SCB_ERR_ARG, "scb_scale_gene_sums: null argument");
  SCB_REQUIRE(n_slots > 0 && n_slots < 32768, SCB_ERR_UNSUPPORTED, "scb_scale_gene_sums: n_slots must be in [1, 32767]");
  SCB_REQUIRE(aligned16(indices) && aligned16(ldata), SCB_ERR_ARG, "scb_scale_gene_sums: 16-byte alignment");
  const size_t smem = (size_t)n_slots * 16 + (size_t)n_cols * 2;
  SCB_REQUIRE(smem <= kSmemLimit, SCB_ERR_UNSUPPORTED, "scb_scale_gene_sums: too many genes for one CTA");
  if (n_rows == 0) return SCB_OK;
  SCB_CUDA(cudaFuncSetAttribute(scale_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t rpb = 1024;  // <= 1024 rows per CTA (carry-free fixed point)
  scale_sums_kernel<<<(unsigned)((n_rows + rpb - 1) / rpb), kRowThreads, smem, (cudaStream_t)stream>>>(
      indptr, indices, ldata, n_rows, n_cols, slot, n_slots, rpb, (unsigned long long*)sums);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_scale_finalize(scb_ctx* ctx, const uint64_t* sums, int32_t n_slots, int64_t n_cells,
                                  double* mean, double* inv_std, void* stream) {
  SCB_REQUIRE(ctx && sums && mean && inv_std, SCB_ERR_ARG, "scb_scale_finalize: null argument");
  SCB_REQUIRE(n_cells >= 2, SCB_ERR_ARG, "scb_scale_finalize: need >= 2 cells");
  scale_finalize_kernel<<<ceil_div(n_slots, 256), 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)sums, n_slots, n_cells, mean, inv_std);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

extern "C" int scb_scale_dense(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                               const float* ldata, int64_t n_rows, int32_t n_cols, const int32_t* slot,
                               int32_t n_slots, const double* mean, const double* inv_std, double max_value,
                               double min_value, float* Z, int64_t ldz, int32_t ones_col, void* stream) {
  SCB_REQUIRE(ctx && indptr && indices && ldata && slot && mean && inv_std && Z, SCB_ERR_ARG,
              "scb_scale_dense: null argument");
  SCB_REQUIRE(ldz % 4 == 0 && ldz >= n_slots && ones_col < ldz, SCB_ERR_ARG,
              "scb_scale_dense: ldz must be a multiple of 4 and >= n_slots");
  SCB_REQUIRE(((uintptr_t)Z & 15) == 0, SCB_ERR_ARG, "scb_scale_dense: Z must be 16-byte aligned");
  SCB_REQUIRE(aligned16(indices) && aligned16(ldata), SCB_ERR_ARG, "scb_scale_dense: 16-byte alignment");
  const size_t smem = (size_t)ldz * 4 + (size_t)((n_cols + 3) & ~3) * 2 + (size_t)n_slots * 16;
  SCB_REQUIRE(smem <= kSmemLimit, SCB_ERR_UNSUPPORTED, "scb_scale_dense: too many genes");
  if (n_rows == 0) return SCB_OK;
  SCB_CUDA(cudaFuncSetAttribute(scale_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int per_sm = std::max(1, std::min(4, (int)(kSmemLimit / (smem + 1024))));
  scale_dense_kernel<<<grid_for(ctx, per_sm), kRowThreads, smem, (cudaStream_t)stream>>>(
      indptr, indices, ldata, n_rows, n_cols, slot, n_slots, mean, inv_std, max_value, min_value, Z, ldz, ones_col);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}


extern "C" int scb_scale_dense_planes(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* ldata,
                                      int64_t n_rows, int32_t n_cols, const int32_t* slot, int32_t n_slots,
                                      const double* mean, const double* inv_std, double max_value, double min_value,
                                      uint16_t* Z_hi, uint16_t* Z_lo, int64_t ldz, int32_t ones_col, void* stream) {
  SCB_REQUIRE(ctx && indptr && indices && ldata && slot && mean && inv_std && Z_hi && Z_lo, SCB_ERR_ARG,
              "scb_scale_dense_planes: null argument");
  SCB_REQUIRE(ldz % 8 == 0 && ldz >= n_slots && ones_col < ldz, SCB_ERR_ARG,
              "scb_scale_dense_planes: ldz must be a multiple of 8 and >= n_slots");
  SCB_REQUIRE(((uintptr_t)Z_hi & 15) == 0 && ((uintptr_t)Z_lo & 15) == 0, SCB_ERR_ARG,
              "scb_scale_dense_planes: 16-byte aligned planes required");
  SCB_REQUIRE(aligned16(indices) && aligned16(ldata), SCB_ERR_ARG, "scb_scale_dense_planes: 16-byte alignment");
  const size_t smem = (size_t)ldz * 4 + (size_t)((n_cols + 7) & ~7) * 2 + (size_t)n_slots * 16;
  SCB_REQUIRE(smem <= kSmemLimit, SCB_ERR_UNSUPPORTED, "scb_scale_dense_planes: too many genes");
  if (n_rows == 0) return SCB_OK;
  SCB_CUDA(cudaFuncSetAttribute(scale_dense_planes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int per_sm = std::max(1, std::min(4, (int)(kSmemLimit / (smem + 1024))));
  scale_dense_planes_kernel<<<grid_for(ctx, per_sm), kRowThreads, smem, (cudaStream_t)stream>>>(
      indptr, indices, ldata, n_rows, n_cols, slot, n_slots, mean, inv_std, max_value, min_value,
      (__nv_bfloat16*)Z_hi, (__nv_bfloat16*)Z_lo, ldz, ones_col);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

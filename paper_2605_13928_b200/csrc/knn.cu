// Exact brute-force kNN graph on the PCA embedding (sc.pp.neighbors, method exact).
//
// 1. order: rows are bucket-sorted along a 4-D Morton (Z-order) curve over their leading
//    principal components PC1..PC4, and every query pair scans the key tiles OUTWARD from its
//    own curve position (spatially nearest first).  The scan still visits every key (exact
//    brute force); the order only makes each row's running top-K threshold tight after a few
//    tiles and keeps the 32 queries of a warp spatially coherent, so the insert path is rare.
// 2. prep: FP16 rows of width 64 (one 128-byte swizzle row):
//    queries Qa = [q/s, 1, 1, 0..], keys Ka = [-2x/s, hi(|x|^2/s^2), lo(|x|^2/s^2), 0..]
//    with s = max|X|/16 so everything fits FP16; one K=64 dot product gives the
//    query-invariant score (d^2 - |q|^2)/s^2 with the 11-bit significands of TF32.
// 3. candidates (tcgen05.mma.kind::f16, FP32 accumulate in TMEM): a persistent CTA owns a
//    PAIR of 128-query tiles (smem-resident) and streams 128-key tiles through a 12-stage TMA
//    pipeline; two CTAs of a cluster (adjacent pairs, one shared scan order) each load half of
//    every key tile and multicast it into both rings.  Two MMA-issuing warps, one per query tile (a tcgen05.commit stalls its issuer
//    until the pipe drains, so one issuer leaves the tensor pipe idle ~45% of the time), run
//    warp-converged loops and let one elected lane issue each of the 4 MMAs (128x128x16) per
//    key tile into the query tile's double-buffered accumulator (2 x 2 x 128 = 512 TMEM
//    columns); producer and issuers sit on the highest warp ids.  Epilogue warps own one query row per
//    lane and COLS = 128/HALVES key columns of every tile, keep a register-resident sorted
//    top-KC list behind a 32-wide min filter, and re-read the few passing columns straight
//    from TMEM (tcgen05.ld x1) instead of staging scores through shared memory.  With
//    HALVES = 2 (k_cand 32) sixteen epilogue warps, four per SM sub-partition, hide the
//    TMEM-load and vote latencies; the two half-lists of a row are concatenated (the top-k
//    of the union is contained in the union of the per-half top-KC for k <= KC).  The fast
//    path per 32-column chunk is LDTM + 16 FMNMX3 + vote on the ALU pipe, which bounds the
//    epilogue: addresses live in opaque registers (no per-tile rematerialisation) and key ids
//    are only computed on the rare path.
// 4. rerank: one warp per query recomputes exact FP32 squared distances of the k_cand
//    candidates, sorts by (distance, original index) and keeps k (self included).
#include <cstdlib>
#include <vector>
#include <cuda_fp16.h>
#include "tc_common.cuh"

namespace scb {

constexpr int kD = 64;            // padded augmented width (one 128-byte FP16 row)
constexpr int kBuckets = 1 << 16; // PC1 counting-sort buckets

// nanosleep back-off (ns) of the producer's / MMA issuers' / epilogue's barrier polls (0: plain
// spin).  A spinning warp issues 3 instructions per poll on the sub-partition the epilogue warps
// need (ncu: 15 % of all issued instructions were polls); A/B at C3 (4 rounds): 114.9 -> 112.9 ms
#ifndef SCB_KNN_SLEEP_P
#define SCB_KNN_SLEEP_P 64
#endif
#ifndef SCB_KNN_SLEEP_M
#define SCB_KNN_SLEEP_M 32
#endif
#ifndef SCB_KNN_SLEEP_E
#define SCB_KNN_SLEEP_E 0
#endif

// KC = per-warp list length, HALVES = epilogue warps per (query tile, TMEM lane quarter)
template <int KC, int HALVES>
struct KnnCfg {
  static constexpr int BM = 128, BN = 128, STAGES = 12, NBUF = 2;  // TMEM: 2 bufs x 2 qtiles x 128 = 512 cols
  static constexpr int TILE = BM * kD * 2;              // 16 KB: 128 rows x 64 fp16
  static constexpr int A_BYTES = 2 * TILE;              // 2 query tiles
  static constexpr int B_BYTES = BN * kD * 2;           // 128 keys (16 KB)
  static constexpr int COLS = BN / HALVES;              // key columns per epilogue warp per tile
  static constexpr int KCT = KC * HALVES;               // candidates per query row (k_cand)
  static constexpr int EPI_WARPS = 8 * HALVES;
  static constexpr int THREADS = 32 * (3 + EPI_WARPS);  // warp0 TMA, warps 1-2 MMA, then epilogue
  static constexpr int SMEM = A_BYTES + STAGES * B_BYTES + 1024 + 256;
  // kind::f16: c_format F32 (1) [4,6), a/b format F16 (0), K-major, N>>3 [17,23), M>>4 [24,29)
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(NBUF == 2, "TMEM: 2 buffers x 2 query tiles x 128 columns");
  static_assert(COLS % 32 == 0, "epilogue chunks are 32 columns");
};

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

// ------------------------------------------------------------------ ordering by PC1
// ordered-int encoding for float min/max via integer atomics
__device__ __forceinline__ int f2o(float f) { const int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7fffffff; }
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

#ifndef SCB_KNN_ORDER_DIMS
#define SCB_KNN_ORDER_DIMS 4  // A/B at C3: PC1-2 / 1-3 / 1-4 -> 115.9 / 115.1 / 113.1 ms
#endif
constexpr int kOrderDims = SCB_KNN_ORDER_DIMS;  // Morton curve over PC1..PC<kOrderDims> (<= 4)
static_assert(kOrderDims >= 1 && kOrderDims <= 8, "order dims");

__global__ void range_kernel(const float* __restrict__ X, int64_t n, int d, int ld, unsigned* __restrict__ amax,
                             int* __restrict__ omin, int* __restrict__ omax) {
  float m = 0.0f, lo[kOrderDims], hi[kOrderDims];
#pragma unroll
  for (int c = 0; c < kOrderDims; ++c) { lo[c] = INFINITY; hi[c] = -INFINITY; }
  const int dims = min(d, kOrderDims);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const float* x = X + r * ld;
    for (int j = 0; j < d; ++j) m = fmaxf(m, fabsf(x[j]));
#pragma unroll
    for (int c = 0; c < kOrderDims; ++c)
      if (c < dims) { lo[c] = fminf(lo[c], x[c]); hi[c] = fmaxf(hi[c], x[c]); }
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
#pragma unroll
    for (int c = 0; c < kOrderDims; ++c) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  }
  if (lane_id() == 0) {
    atomicMax(amax, __float_as_uint(m));  // non-negative floats order like unsigned ints
#pragma unroll
    for (int c = 0; c < kOrderDims; ++c) {
      atomicMin(omin + c, f2o(lo[c]));
      atomicMax(omax + c, f2o(hi[c]));
    }
  }
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// 16-bit bucket = top bits of the Morton code of (PC1 .. PC<kOrderDims>), each quantised to
// 30 / kOrderDims bits (kOrderDims = 3: 10 bits each, the 30-bit code's top 16 bits)
__device__ __forceinline__ int order_bucket(const float* x, int d, const int* omin, const int* omax) {
  constexpr int B = 30 / kOrderDims;
  uint32_t q[kOrderDims];
#pragma unroll
  for (int c = 0; c < kOrderDims; ++c) {
    q[c] = 0;
    if (c < d) {
      const float lo = o2f(omin[c]), hi = o2f(omax[c]);
      const float w = hi - lo;
      int qi = (w > 0.0f) ? (int)((x[c] - lo) / w * (float)(1 << B)) : 0;
      q[c] = (uint32_t)(qi < 0 ? 0 : (qi > (1 << B) - 1 ? (1 << B) - 1 : qi));
    }
  }
  if (kOrderDims == 3) return (int)((spread3(q[0]) << 2 | spread3(q[1]) << 1 | spread3(q[2 % kOrderDims])) >> 14);
  uint32_t code = 0;
#pragma unroll
  for (int b = B - 1; b >= 0; --b)
#pragma unroll
    for (int c = 0; c < kOrderDims; ++c) code = (code << 1) | ((q[c] >> b) & 1u);
  return (int)(code >> (B * kOrderDims - 16));
}

__global__ void bucket_hist_kernel(const float* __restrict__ X, int64_t n, int d, int ld, const int* omin,
                                   const int* omax, const uint16_t* __restrict__ ext, int* __restrict__ hist) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[ext ? (int)ext[r] : order_bucket(X + r * ld, d, omin, omax)], 1);
}

// single CTA exclusive scan of the bucket histogram (in place)
__global__ void bucket_scan_kernel(int* __restrict__ hist) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < kBuckets; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = hist[i];
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= o) incl += t;
    }
    if (lane_id() == 31) wsum[warp_id()] = incl;
    __syncthreads();
    if (warp_id() == 0) {
      const int sv = (lane_id() < (int)(blockDim.x >> 5)) ? wsum[lane_id()] : 0;
      int si = sv;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, si, o);
        if (lane_id() >= o) si += t;
      }
      wsum[lane_id()] = si - sv;
    }
    __syncthreads();
    const int ex = carry + wsum[warp_id()] + incl - v;
    hist[i] = ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = ex + v;
    __syncthreads();
  }
}

// scatter rows into curve order; key_sorted[pos] = bucket id (non-decreasing, for start search)
__global__ void bucket_scatter_kernel(const float* __restrict__ X, int64_t n, int d, int ld, const int* omin,
                                      const int* omax, const uint16_t* __restrict__ ext, int* __restrict__ cursor,
                                      int* __restrict__ perm, float* __restrict__ key_sorted) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int b = ext ? (int)ext[r] : order_bucket(X + r * ld, d, omin, omax);
    const int pos = atomicAdd(&cursor[b], 1);
    perm[pos] = (int)r;
    key_sorted[pos] = (float)b;
  }
}

// queries: [q/s, 1, 1, 0...]; keys: [-2x/s, hi(|x|^2/s^2), lo(|x|^2/s^2), 0...]  (fp16, sorted order)
__global__ void knn_prep_kernel(const float* __restrict__ X, int64_t n, int d, int ld, int is_key,
                                const int* __restrict__ perm, const unsigned* __restrict__ amax, __half* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (i >= n) return;
  const int l = lane_id();
  const float s = fmaxf(__uint_as_float(*amax), 1e-30f) * (1.0f / 16.0f);
  const float inv = 1.0f / s;
  const int64_t r = perm ? perm[i] : i;
  const float* x = X + r * ld;
  const float a = (l < d) ? x[l] * inv : 0.0f;
  const float b = (l + 32 < d) ? x[l + 32] * inv : 0.0f;
  __half* o = out + i * kD;
  if (!is_key) {
    auto val = [&](int col, float xv) { return col < d ? xv : ((col == d || col == d + 1) ? 1.0f : 0.0f); };
    o[l] = __float2half_rn(val(l, a));
    o[l + 32] = __float2half_rn(val(l + 32, b));
  } else {
    const float nrm = warp_sum(a * a + b * b);
    const __half hh = __float2half_rn(nrm);
    const __half hl = __float2half_rn(nrm - __half2float(hh));
    auto val = [&](int col, float xv) -> __half {
      return col < d ? __float2half_rn(-2.0f * xv) : (col == d ? hh : (col == d + 1 ? hl : __float2half_rn(0.0f)));
    };
    o[l] = val(l, a);
    o[l + 32] = val(l + 32, b);
  }
}

// start key tile of each query pair: PC1 of the pair's middle query, located in the sorted keys
__global__ void start_tile_kernel(const float* __restrict__ q_pc1_sorted, int64_t n_q, const float* __restrict__ k_pc1_sorted,
                                  int64_t n_k, int bm, int bn, int* __restrict__ start) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_pairs = (n_q + 2 * bm - 1) / (2 * bm);
  if (p >= n_pairs) return;
  const int64_t mid = min(n_q - 1, (int64_t)p * 2 * bm + bm);
  const float v = q_pc1_sorted[mid];
  int64_t lo = 0, hi = n_k;  // first position with key pc1 >= v
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (k_pc1_sorted[m] < v) lo = m + 1; else hi = m;
  }
  const int64_t n_kt = (n_k + bn - 1) / bn;
  const int64_t t = min(lo, n_k - 1) / bn;
  start[p] = (int)min(t, n_kt - 1);
}

// j-th key tile (0 <= j < n_kt) of the outward scan from `start`: start, start+1, start-1,
// start+2, start-2, ... and, once one end is reached, the rest of the other side in order.
__device__ __forceinline__ int outward_tile(int start, int j, int n_kt) {
  const int below = start, above = n_kt - 1 - start;
  const int m = min(below, above);
  if (j <= 2 * m) {
    const int dd = (j + 1) >> 1;
    return (j & 1) ? start + dd : start - dd;
  }
  return above > below ? start + (j - below) : start - (j - above);
}

// inverse of outward_tile: scan position of key tile kt
__device__ __forceinline__ int outward_pos(int start, int kt, int n_kt) {
  const int below = start, above = n_kt - 1 - start;
  const int m = min(below, above);
  const int d = kt - start;
  if (d == 0) return 0;
  if (d > 0 && d <= m) return 2 * d - 1;
  if (d < 0 && -d <= m) return -2 * d;
  return d > 0 ? d + below : -d + above;
}

// Work units of the persistent candidate kernel: query pairs, except that the pairs of a final
// partial round (r <= gridDim/2 pairs) are split into two halves of their outward key scan, so
// that round takes half as long; the two halves' lists go to a separate buffer (2 x KCT
// candidates per row) and are re-ranked together.
struct KnnUnit {
  int pair, i0, i1, tail, half;
};
__device__ __forceinline__ KnnUnit knn_unit(int u, int n_full, int n_kt) {
  if (u < n_full) return KnnUnit{u, 0, n_kt, 0, 0};
  const int t = u - n_full, half = t & 1, mid = n_kt >> 1;
  return KnnUnit{n_full + (t >> 1), half ? mid : 0, half ? n_kt : mid, 1, half};
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

#ifndef SCB_KNN_QUEUE
#define SCB_KNN_QUEUE 2  // A/B at C3: 1 / 2 / 3 / 4 / 6 entries -> 127.9 / 115.6 / 117.1 / 119.0 / 122.3 ms
#endif
constexpr int kQ = SCB_KNN_QUEUE;  // per-lane pending queue in front of the sorted list

// merge the pending queue into the sorted list (executed by the whole warp at once, so the
// O(KC) insertions of different lanes share the same issue slots)
template <int KC>
__device__ __forceinline__ void queue_merge(float (&L)[KC], int (&I)[KC], float (&Qv)[kQ], int (&Qi)[kQ], int& qn) {
#pragma unroll
  for (int s = 0; s < kQ; ++s)
    if (s < qn) list_insert<KC>(L, I, Qv[s], Qi[s]);
  qn = 0;
}

// min of 32 values as a 3-ary tree (sm_100a FMNMX3)
__device__ __forceinline__ float min32(const float (&v)[32]) {
  float a[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) a[j] = fminf(fminf(v[3 * j], v[3 * j + 1]), v[3 * j + 2]);
  a[10] = fminf(v[30], v[31]);
  const float b0 = fminf(fminf(a[0], a[1]), a[2]);
  const float b1 = fminf(fminf(a[3], a[4]), a[5]);
  const float b2 = fminf(fminf(a[6], a[7]), a[8]);
  const float b3 = fminf(a[9], a[10]);
  return fminf(fminf(b0, b1), fminf(b2, b3));
}

#ifdef SCB_KNN_PROF
__device__ unsigned long long g_knn_prof[8];  // [0] epi t_full wait, [1] epi total, [2] mma t_empty wait, [3] mma b_full wait, [4] mma total
#define PROF_T0(v) const long long v = clock64()
#define PROF_ADD(i, v) prof_acc[i] += clock64() - (v)
#define PROF_DECL long long prof_acc[7] = {0, 0, 0, 0, 0, 0, 0}
#define PROF_FLUSH                                                                              \
  do {                                                                                        \
    if (lane_id() == 0)                                                                       \
      for (int i_ = 0; i_ < 7; ++i_) if (prof_acc[i_]) atomicAdd(&g_knn_prof[i_], (unsigned long long)prof_acc[i_]); \
  } while (0)
#else
#define PROF_T0(v)
#define PROF_ADD(i, v)
#define PROF_DECL
#define PROF_FLUSH
#endif
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}

// CL = 2: 2-CTA clusters.  The CTAs of a cluster own adjacent query pairs (2v, 2v+1) of cluster
// unit v and share one outward scan order (from pair 2v's start); each CTA loads one half (64
// keys) of every key tile and multicasts it into both CTAs' rings, and every MMA issuer releases
// a stage in both CTAs (multicast commit), so each key byte leaves L2 once per cluster.
template <int KC, int HALVES, int CL = 1>
__global__ void __launch_bounds__(KnnCfg<KC, HALVES>::THREADS, 1)
knn_candidates_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk, int64_t n_q,
                      int64_t n_k, const int* __restrict__ start_tile, int* __restrict__ cand, int n_full,
                      int n_units, int* __restrict__ cand_tail) {
  using C = KnnCfg<KC, HALVES>;
  static_assert(CL == 1 || CL == 2 || CL == 4, "cluster size");
  const int crank = CL > 1 ? (int)tc::cluster_rank() : 0;
  const int unit0 = blockIdx.x / CL, unit_step = gridDim.x / CL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_base = smem;                          // [qtile][128 rows x 128 B]
  uint8_t* b_base = smem + C::A_BYTES;             // [stage][128 rows x 128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(b_base + C::STAGES * C::B_BYTES);
  uint64_t* a_full = bar;
  uint64_t* a_empty = bar + 1;
  uint64_t* b_full = bar + 2;
  uint64_t* b_empty = b_full + C::STAGES;
  uint64_t* t_full = b_empty + C::STAGES;   // [buf][qtile]
  uint64_t* t_empty = t_full + 2 * C::NBUF; // [buf][qtile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2 * C::NBUF);

  const int warp = warp_id(), lane = lane_id();
  const int n_kt = (int)((n_k + C::BN - 1) / C::BN);

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tq);
      tc::tma_prefetch(&tk);
      tc::mbar_init(a_full, 1);
      tc::mbar_init(a_empty, 2);  // one commit per MMA issuer
      for (int s = 0; s < C::STAGES; ++s) {
        tc::mbar_init(&b_full[s], 1);
        tc::mbar_init(&b_empty[s], 2 * CL);  // both issuers (of every CTA of the cluster) read every stage
      }
      for (int b = 0; b < 2 * C::NBUF; ++b) {
        tc::mbar_init(&t_full[b], 1);
        tc::mbar_init(&t_empty[b], 4 * HALVES);
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (CL > 1) tc::cluster_sync();  // every CTA's barriers initialised before any remote arrive / multicast
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  PROF_DECL;
  // roles on the HIGHEST warp ids (the issue arbiter prefers high warp ids): producer and the
  // two MMA issuers are warps EPI_WARPS .. EPI_WARPS+2, epilogue warps 0 .. EPI_WARPS-1
  const int rw = warp >= C::EPI_WARPS ? warp - C::EPI_WARPS : warp + 3;

  if (rw == 0) {
    if (lane == 0) {
      int it = 0, pc = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++pc) {
        const KnnUnit U = knn_unit(u, n_full, n_kt);
        const int pair = CL * U.pair + crank;
        const int st = start_tile[CL * U.pair];
        tc::mbar_wait(a_empty, (pc & 1) ^ 1);
        tc::mbar_arrive_expect_tx(a_full, C::A_BYTES);
        for (int t = 0; t < 2; ++t) tc::tma_load_2d(a_base + t * C::TILE, &tq, a_full, 0, (pair * 2 + t) * C::BM);
        for (int i = U.i0; i < U.i1; ++i) {
          const int kt = outward_tile(st, i, n_kt);
          const int s = it % C::STAGES;
#if SCB_KNN_SLEEP_P > 0
          tc::mbar_wait_sleep(tc::smem_u32(&b_empty[s]), ((it / C::STAGES) & 1) ^ 1, SCB_KNN_SLEEP_P);
#else
          tc::mbar_wait(&b_empty[s], ((it / C::STAGES) & 1) ^ 1);
#endif
          tc::mbar_arrive_expect_tx(&b_full[s], C::B_BYTES);
          if (CL > 1)  // my 1/CL of the tile, into every CTA of the cluster (tk's box is BN/CL rows)
            tc::tma_load_2d_mc(b_base + s * C::B_BYTES + crank * (C::B_BYTES / CL), &tk, &b_full[s], 0,
                               kt * C::BN + crank * (C::BN / CL), (uint16_t)((1u << CL) - 1u));
          else
            tc::tma_load_2d(b_base + s * C::B_BYTES, &tk, &b_full[s], 0, kt * C::BN);
          ++it;
        }
      }
    }
  } else if (rw <= 2) {
    // Issuer t feeds query tile t: every key tile, into TMEM buffer (unit parity, t).  A
    // tcgen05.commit stalls its issuing thread until the tensor pipe drains, so a single issuer
    // leaves the pipe idle ~45% of the time; two issuers interleave.  Each qtile's MMA -> epilogue
    // ring is then independent of the other qtile's epilogue progress.
    // The whole warp runs the issue loop and one elected lane issues each MMA / commit: the
    // loop state stays warp-converged (a lane-0-only loop moves every descriptor through
    // per-thread registers), which took the MMA+TMA-only time of this kernel from ~104 to ~76 ms
    // at 1M cells.  A's four K-slice descriptors are fixed; B's advance by the stage stride.
    const int t = rw - 1;
    {
      PROF_T0(tot);
      const uint32_t ab = tc::smem_u32(a_base + t * C::TILE);
      const uint64_t ad0 = tc::smem_desc_sw128(ab, 16, 1024);
      const uint64_t bd0 = tc::smem_desc_sw128(tc::smem_u32(b_base), 16, 1024);
      const uint32_t bar_tf = tc::smem_u32(&t_full[t]), bar_be = tc::smem_u32(&b_empty[0]);
      const uint32_t bar_bf = tc::smem_u32(&b_full[0]), bar_te = tc::smem_u32(&t_empty[t]);
      const uint32_t bar_ae = tc::smem_u32(a_empty);
      int it = 0, pc = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++pc) {
        const KnnUnit U = knn_unit(u, n_full, n_kt);
        tc::mbar_wait(a_full, pc & 1);
        for (int i = U.i0; i < U.i1; ++i, ++it) {
          const int s = it % C::STAGES;
          const int buf = it & 1;
          PROF_T0(w0);
#if SCB_KNN_SLEEP_M > 0
          tc::mbar_wait_sleep(bar_bf + 8 * s, (it / C::STAGES) & 1, SCB_KNN_SLEEP_M);
#else
          tc::mbar_wait_a(bar_bf + 8 * s, (it / C::STAGES) & 1);
#endif
          PROF_ADD(3, w0);
          PROF_T0(w1);
#if SCB_KNN_SLEEP_M > 0
          tc::mbar_wait_sleep(bar_te + 16 * buf, ((it >> 1) & 1) ^ 1, SCB_KNN_SLEEP_M);
#else
          tc::mbar_wait_a(bar_te + 16 * buf, ((it >> 1) & 1) ^ 1);
#endif
          PROF_ADD(2, w1);
          tc::tc_fence_after();
          const uint32_t d = tmem + buf * (2 * C::BN) + t * C::BN;
          const uint64_t bd = bd0 + (uint64_t)((s * C::B_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk)  // K = 16 fp16 = 32 bytes per MMA
            tc::mma_f16_elect(d, ad0 + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), C::IDESC, kk > 0 ? 1u : 0u);
          tc::mma_commit_elect(bar_tf + 16 * buf);
          if (CL > 1)
            tc::mma_commit_mc_elect(bar_be + 8 * s, (uint16_t)((1u << CL) - 1u));  // release the stage in every CTA
          else
            tc::mma_commit_elect(bar_be + 8 * s);
        }
        tc::mma_commit_elect(bar_ae);
      }
      PROF_ADD(4, tot);
    }
  } else {
    const int e = rw - 3;              // 0 .. EPI_WARPS-1
    const int q = warp & 3;            // TMEM lane quarter this warp may access (physical warp id % 4)
    const int t = (e >> 2) & 1;        // query tile of the pair
    const int hf = e >> 3;             // key-column slice of each tile (HALVES == 2)
    // Opaque copies (asm moves): the compiler must keep these in registers instead of
    // rematerialising the shared-window / TMEM address arithmetic every tile -- at 96 registers
    // it otherwise recomputes them on the ALU pipe, which the min filter already saturates.
    uint32_t tl, tf_bar, te_bar;  // + buf * 2 * BN / + buf * 16
    asm volatile("mov.b32 %0, %1;" : "=r"(tl) : "r"(tmem + ((uint32_t)(32 * q) << 16) + t * C::BN + hf * C::COLS));
    asm volatile("mov.b32 %0, %1;" : "=r"(tf_bar) : "r"(tc::smem_u32(&t_full[t])));
    asm volatile("mov.b32 %0, %1;" : "=r"(te_bar) : "r"(tc::smem_u32(&t_empty[t])));
    const int n_k32 = (int)n_k;
    const int last_valid = n_k32 - (n_kt - 1) * C::BN - hf * C::COLS;  // valid keys of the last tile's slice
    int it = 0;
    PROF_T0(tot);
    for (int u = unit0; u < n_units; u += unit_step) {
      const KnnUnit U = knn_unit(u, n_full, n_kt);
      const int pair = CL * U.pair + crank;
      const int st = start_tile[CL * U.pair];
      float L[KC];
      int I[KC];
      float Qv[kQ];
      int Qi[kQ];
      int qn = 0;
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        L[j] = INFINITY;
        I[j] = -1;
      }
#pragma unroll
      for (int j = 0; j < kQ; ++j) {
        Qv[j] = INFINITY;
        Qi[j] = -1;
      }
      const int64_t row = (int64_t)(pair * 2 + t) * C::BM + 32 * q + lane;
      const int jl = last_valid < C::COLS ? outward_pos(st, n_kt - 1, n_kt) : -1;
      for (int i = U.i0; i < U.i1; ++i, ++it) {
        const int buf = it & 1;
        PROF_T0(w0);
#if SCB_KNN_SLEEP_E > 0
        tc::mbar_wait_sleep(tf_bar + buf * 16, (it >> 1) & 1, SCB_KNN_SLEEP_E);
#else
        tc::mbar_wait_a(tf_bar + buf * 16, (it >> 1) & 1);
#endif
        PROF_ADD(0, w0);
        tc::tc_fence_after();
        const uint32_t tb = tl + buf * (2 * C::BN);
#ifdef SCB_KNN_MMA_ONLY  // experiment: no epilogue work (tensor pipe + TMA bound)
        if (buf > 1)
#endif
#pragma unroll(C::COLS / 32 <= 2 ? C::COLS / 32 : 1)  // k > 16 (128-column lists): 4 chunks, not unrolled
        for (int c = 0; c < C::COLS / 32; ++c) {
          const uint32_t ta = tb + c * 32;
          uint32_t r[32];
          PROF_T0(w2);
          tc::tmem_ld32(ta, r);
          tc::tmem_ld_wait();
          PROF_ADD(5, w2);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (i == jl) {  // padding keys of the last tile
            const int lim = last_valid - c * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j >= lim) v[j] = INFINITY;
          }
          const float thr = L[KC - 1];
          if (__any_sync(0xffffffffu, min32(v) < thr)) {
            // rare path: columns where any lane passes; each is re-read from TMEM (one
            // column per lane) and goes to the lane's small queue; a full queue on ANY lane
            // merges every lane's queue at once.
            PROF_T0(w3);
            const int key0 = outward_tile(st, i, n_kt) * C::BN + hf * C::COLS;
            // bit j = sign of v[j] - thr (FADD on the FMA pipe, one funnel shift per column);
            // v == thr gives +0 (bit clear), as v < thr requires
            uint32_t mask = 0;
#pragma unroll
            for (int j = 31; j >= 0; --j) mask = __funnelshift_l(__float_as_uint(v[j] - thr), mask, 1);
            uint32_t cm = __reduce_or_sync(0xffffffffu, mask);
            while (cm) {
              const int j = __ffs(cm) - 1;
              cm &= cm - 1;
              if (__any_sync(0xffffffffu, qn == kQ)) queue_merge<KC>(L, I, Qv, Qi, qn);
              const float x = __uint_as_float(tmem_ld1(ta + j));
              tc::tmem_ld_wait();
              if (((mask >> j) & 1u) && x < L[KC - 1]) {
                const int id = key0 + c * 32 + j;
#pragma unroll
                for (int q2 = 0; q2 < kQ; ++q2)
                  if (q2 == qn) {
                    Qv[q2] = x;
                    Qi[q2] = id;
                  }
                ++qn;
              }
            }
            PROF_ADD(6, w3);
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        tc::mbar_arrive_elect(te_bar + buf * 16);
      }
      queue_merge<KC>(L, I, Qv, Qi, qn);
      if (row < n_q) {
        const int64_t tail_row0 = (int64_t)n_full * CL * 2 * C::BM;
        int* o = U.tail ? cand_tail + (row - tail_row0) * (2 * C::KCT) + U.half * C::KCT + hf * KC
                        : cand + row * C::KCT + hf * KC;
        if constexpr (KC % 4 == 0) {  // 16-byte stores (rows are 16-byte aligned: KCT, KC multiples of 4)
#pragma unroll
          for (int j = 0; j < KC; j += 4) *reinterpret_cast<int4*>(o + j) = make_int4(I[j], I[j + 1], I[j + 2], I[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < KC; ++j) o[j] = I[j];
        }
      }
    }
    PROF_ADD(1, tot);
  }
  PROF_FLUSH;
  tc::tc_fence_before();
  __syncthreads();
  if (CL > 1) tc::cluster_sync();  // no CTA leaves while another may still multicast into it
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ rerank
template <int KC>
__global__ void knn_rerank_kernel(const float* __restrict__ Q, const float* __restrict__ Kx, int64_t n_q, int d,
                                  int ld, const int* __restrict__ perm_q, const int* __restrict__ perm_k,
                                  const int* __restrict__ cand, int k, int* __restrict__ out_i, float* __restrict__ out_d,
                                  int64_t i0 = 0) {
  constexpr int PER = (KC + 31) / 32;  // KC not a multiple of 32: the upper lanes carry no candidate
  constexpr int NS = PER * 32;         // sort width (power of two up to 64)
  static_assert(NS == 32 || NS == 64, "rerank sort width");
  const int64_t i = i0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();  // sorted query position
  if (i >= n_q) return;
  cand -= i0 * KC;  // candidates of rows [i0, n_q) start at cand
  const int l = lane_id();
  const int64_t r = perm_q[i];
  const float* qp = Q + r * ld;
  const float qa = (l < d) ? qp[l] : 0.0f;
  const float qb = (l + 32 < d) ? qp[l + 32] : 0.0f;
  float dd[PER];
  int ii[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int c = (p * 32 + l < KC) ? cand[i * KC + p * 32 + l] : -1;
    ii[p] = (c >= 0) ? perm_k[c] : -1;
    dd[p] = INFINITY;
  }
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
  auto less = [](float da, int ia, float db, int ib) {
    return da < db || (da == db && (unsigned)ia < (unsigned)ib);
  };
#pragma unroll
  for (int size = 2; size <= NS; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int e = p * 32 + l;
        const bool up = ((e & size) == 0);
        if (stride >= 32) {
          const int pq = p ^ (stride >> 5);
          if ((p & (stride >> 5)) == 0) {
            const float d0 = dd[p], d1 = dd[pq];
            const int i0 = ii[p], i1 = ii[pq];
            const bool lt = less(d0, i0, d1, i1);
            const bool swp = up ? !lt : lt;
            dd[p] = swp ? d1 : d0;
            ii[p] = swp ? i1 : i0;
            dd[pq] = swp ? d0 : d1;
            ii[pq] = swp ? i0 : i1;
          }
        } else {
          const float od = __shfl_xor_sync(0xffffffffu, dd[p], stride);
          const int oi = __shfl_xor_sync(0xffffffffu, ii[p], stride);
          const bool lower = e < (e ^ stride);
          const bool mine_less = less(dd[p], ii[p], od, oi);
          const bool keep = (lower == up) ? mine_less : !mine_less;
          if (!keep) {
            dd[p] = od;
            ii[p] = oi;
          }
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

// ------------------------------------------------------------------ host orchestration
static int sort_by_pc1(const float* X, int64_t n, int d, int ld, const int* omin, const int* omax, int* hist, int* perm,
                       float* pc1_sorted, cudaStream_t s, const uint16_t* ext = nullptr) {
  SCB_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * kBuckets, s));
  const int g = std::max(1, std::min(1184, ceil_div(n, 256)));
  bucket_hist_kernel<<<g, 256, 0, s>>>(X, n, d, ld, omin, omax, ext, hist);
  SCB_LAUNCH_CHECK();
  bucket_scan_kernel<<<1, 1024, 0, s>>>(hist);
  SCB_LAUNCH_CHECK();
  bucket_scatter_kernel<<<g, 256, 0, s>>>(X, n, d, ld, omin, omax, ext, hist, perm, pc1_sorted);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

template <int KC, int HALVES>
static int launch_knn(scb_ctx* ctx, const float* Qx, int64_t n_q, const float* Kx, int64_t n_k, int d, int ld, int k,
                      int* out_i, float* out_d, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                      const uint16_t* ext_key = nullptr) {
  using Cfg = KnnCfg<KC, HALVES>;
  constexpr int KCT = Cfg::KCT;
  const bool same = (Qx == Kx && n_q == n_k);
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const int64_t n_pairs = (n_q + 2 * Cfg::BM - 1) / (2 * Cfg::BM);
  // cluster mode (CL = 2): units are pairs of adjacent query pairs, one per 2-CTA cluster
#ifndef SCB_KNN_CL
#define SCB_KNN_CL 2  // A/B at C3: 117.5 vs 119.4 ms, DRAM reads 8.6 vs 17.8 GB (ncu)
#endif
  constexpr int CL = HALVES == 2 ? SCB_KNN_CL : 1;
  const int64_t n_sp = (n_pairs + CL - 1) / CL;  // cluster units
  // final partial round: split its units' key scans in two when that fits one round (§ KnnUnit)
  int max_clusters = ctx->num_sms / CL;
  if (CL > 1) {  // co-resident clusters (GPCs whose SM count is not a multiple of CL leave SMs idle)
    cudaLaunchConfig_t oc = {};
    oc.gridDim = dim3((unsigned)(CL * (ctx->num_sms / CL)));
    oc.blockDim = dim3(Cfg::THREADS);
    oc.dynamicSmemBytes = Cfg::SMEM;
    cudaLaunchAttribute oa[1];
    oa[0].id = cudaLaunchAttributeClusterDimension;
    oa[0].val.clusterDim.x = CL;
    oa[0].val.clusterDim.y = 1;
    oa[0].val.clusterDim.z = 1;
    oc.attrs = oa;
    oc.numAttrs = 1;
    SCB_CUDA(cudaFuncSetAttribute(knn_candidates_kernel<KC, HALVES, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Cfg::SMEM));
    int nc = 0;
    SCB_CUDA(cudaOccupancyMaxActiveClusters(&nc, knn_candidates_kernel<KC, HALVES, CL>, &oc));
    if (nc > 0) max_clusters = std::min(max_clusters, nc);
    if (getenv("SCB_KNN_DEBUG")) fprintf(stderr, "[knn] co-resident %d-CTA clusters: %d\n", CL, nc);
  }
  const int64_t Gc = std::min<int64_t>(n_sp, max_clusters);
  const int64_t G = Gc * CL;
  const int64_t r = n_sp % Gc;
  const bool split = r > 0 && 2 * r <= Gc && 2 * KCT <= 64;
  const int64_t n_full = split ? n_sp - r : n_sp;
  const int64_t n_units = split ? n_full + 2 * r : n_sp;
  const int64_t tail_row0 = std::min<int64_t>(n_q, n_full * CL * 2 * Cfg::BM);
  const int64_t tail_rows = n_q - tail_row0;
  const size_t sz[] = {256, sizeof(int) * kBuckets, 4 * (size_t)n_q, 4 * (size_t)n_k, 4 * (size_t)n_q,
                       4 * (size_t)n_k, 4 * (size_t)n_pairs, (size_t)n_q * kD * 2, (size_t)n_k * kD * 2,
                       (size_t)n_q * KCT * 4, (size_t)std::max<int64_t>(tail_rows, 1) * 2 * KCT * 4};
  size_t total = 0;
  for (size_t v : sz) total += up(v);
  void* ws;
  SCB_TRY(ws_get(ctx, 0, total, &ws, s));
  char* p = (char*)ws;
  unsigned* amax = (unsigned*)p;
  int* omin = (int*)(p + 64);   // [kOrderDims] (<= 8)
  int* omax = (int*)(p + 128);  // [kOrderDims]
  p += up(sz[0]);
  int* hist = (int*)p; p += up(sz[1]);
  int* perm_q = (int*)p; p += up(sz[2]);
  int* perm_k = (int*)p; p += up(sz[3]);
  float* pc1_q = (float*)p; p += up(sz[4]);
  float* pc1_k = (float*)p; p += up(sz[5]);
  int* start = (int*)p; p += up(sz[6]);
  __half* Qa = (__half*)p; p += up(sz[7]);
  __half* Ka = (__half*)p; p += up(sz[8]);
  int* cand = (int*)p; p += up(sz[9]);
  int* cand_tail = (int*)p;
  // FP16 scale and the PC1 range come from the KEYS (queries are rows of the same embedding)
  int init[48] = {0};  // amax (+ pad) | omin[8] at +64 B | omax[8] at +128 B
  for (int c = 0; c < 8; ++c) {
    init[16 + c] = 0x7fffffff;
    init[32 + c] = (int)0x80000000;
  }
  SCB_CUDA(cudaMemcpyAsync(amax, init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int g = std::max(1, std::min(1184, ceil_div(n_k, 256)));
  range_kernel<<<g, 256, 0, s>>>(Kx, n_k, d, ld, amax, omin, omax);
  SCB_LAUNCH_CHECK();
  SCB_TRY(sort_by_pc1(Kx, n_k, d, ld, omin, omax, hist, perm_k, pc1_k, s, same ? ext_key : nullptr));
  if (same) {
    perm_q = perm_k;
    pc1_q = pc1_k;
  } else {
    SCB_TRY(sort_by_pc1(Qx, n_q, d, ld, omin, omax, hist, perm_q, pc1_q, s));
  }
  knn_prep_kernel<<<ceil_div(n_q, 8), 256, 0, s>>>(Qx, n_q, d, ld, 0, perm_q, amax, Qa);
  SCB_LAUNCH_CHECK();
  knn_prep_kernel<<<ceil_div(n_k, 8), 256, 0, s>>>(Kx, n_k, d, ld, 1, perm_k, amax, Ka);
  SCB_LAUNCH_CHECK();
  start_tile_kernel<<<ceil_div(n_pairs, 256), 256, 0, s>>>(pc1_q, n_q, pc1_k, n_k, Cfg::BM, Cfg::BN, start);
  SCB_LAUNCH_CHECK();
  CUtensorMap tq, tk;
  SCB_TRY(make_tmap_2d(&tq, Qa, (uint64_t)n_q, kD, kD, 2, 64, Cfg::BM));
  SCB_TRY(make_tmap_2d(&tk, Ka, (uint64_t)n_k, kD, kD, 2, 64, Cfg::BN / CL));
  auto kern = knn_candidates_kernel<KC, HALVES, CL>;
  SCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  if (ev0) SCB_CUDA(cudaEventRecord(ev0, s));
  if (CL == 1) {
    kern<<<(int)G, Cfg::THREADS, Cfg::SMEM, s>>>(tq, tk, n_q, n_k, start, cand, (int)n_full, (int)n_units, cand_tail);
  } else {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)G);
    lc.blockDim = dim3(Cfg::THREADS);
    lc.dynamicSmemBytes = Cfg::SMEM;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    SCB_CUDA(cudaLaunchKernelEx(&lc, kern, tq, tk, n_q, n_k, (const int*)start, cand, (int)n_full, (int)n_units,
                                cand_tail));
  }
  SCB_LAUNCH_CHECK();
  if (ev1) SCB_CUDA(cudaEventRecord(ev1, s));
#ifdef SCB_KNN_PROF
  {
    unsigned long long pr[8];
    SCB_CUDA(cudaMemcpyFromSymbolAsync(pr, g_knn_prof, sizeof(pr), 0, cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    const double ne = (double)Cfg::EPI_WARPS * std::min<int64_t>(n_pairs, ctx->num_sms), nm = 2.0 * std::min<int64_t>(n_pairs, ctx->num_sms);
    fprintf(stderr, "[knn prof] per epi warp: total %.3g cyc, t_full wait %.3g, tmem ld+wait %.3g, slow path %.3g | per issuer: total %.3g, t_empty wait %.3g, b_full wait %.3g\n",
            pr[1] / ne, pr[0] / ne, pr[5] / ne, pr[6] / ne, pr[4] / nm, pr[2] / nm, pr[3] / nm);
    const unsigned long long z[8] = {};
    SCB_CUDA(cudaMemcpyToSymbolAsync(g_knn_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
  }
#endif
  if (!split) {
    knn_rerank_kernel<KCT><<<ceil_div(n_q, 8), 256, 0, s>>>(Qx, Kx, n_q, d, ld, perm_q, perm_k, cand, k, out_i, out_d);
    SCB_LAUNCH_CHECK();
  } else {
    if (tail_row0 > 0) {
      knn_rerank_kernel<KCT><<<ceil_div(tail_row0, 8), 256, 0, s>>>(Qx, Kx, tail_row0, d, ld, perm_q, perm_k, cand, k,
                                                                     out_i, out_d);
      SCB_LAUNCH_CHECK();
    }
    if (tail_rows > 0) {
      constexpr int KCT2 = (2 * KCT <= 64) ? 2 * KCT : 64;
      knn_rerank_kernel<KCT2><<<ceil_div(tail_rows, 8), 256, 0, s>>>(Qx, Kx, n_q, d, ld, perm_q, perm_k, cand_tail, k,
                                                                      out_i, out_d, tail_row0);
      SCB_LAUNCH_CHECK();
    }
  }
  return SCB_OK;
}

}  // namespace scb

using namespace scb;

extern "C" int scb_knn_timed(scb_ctx* ctx, const float* queries, int64_t n_queries, const float* keys, int64_t n_keys,
                             int32_t d, int32_t ld, int32_t k, int32_t k_cand, int32_t* knn_index, float* knn_dist,
                             void* stream, void* ev_start, void* ev_end) {
  SCB_REQUIRE(ctx && queries && keys && knn_index && knn_dist, SCB_ERR_ARG, "scb_knn: null argument");
  SCB_REQUIRE(d >= 1 && d <= kD - 2 && ld >= d, SCB_ERR_ARG, "scb_knn: need 1 <= d <= %d and ld >= d", kD - 2);
  SCB_REQUIRE(k >= 1 && k <= 64 && k <= n_keys, SCB_ERR_ARG, "scb_knn: need 1 <= k <= min(64, n_keys)");
  SCB_REQUIRE(k_cand >= k && (k_cand == 32 || k_cand == 64), SCB_ERR_ARG, "scb_knn: k_cand must be 32 or 64 and >= k");
  SCB_REQUIRE(n_keys < (1ll << 31) && n_queries < (1ll << 31), SCB_ERR_ARG, "scb_knn: too many rows");
  if (n_queries == 0) return SCB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t e0 = (cudaEvent_t)ev_start, e1 = (cudaEvent_t)ev_end;
  if (k_cand == 32) return launch_knn<16, 2>(ctx, queries, n_queries, keys, n_keys, d, ld, k, knn_index, knn_dist, s, e0, e1);
  if (k <= 32) return launch_knn<48, 1>(ctx, queries, n_queries, keys, n_keys, d, ld, k, knn_index, knn_dist, s, e0, e1);
  return launch_knn<64, 1>(ctx, queries, n_queries, keys, n_keys, d, ld, k, knn_index, knn_dist, s, e0, e1);
}

// experiment hook: caller-supplied 16-bit scan-order bucket per row (queries == keys only)
extern "C" int scb_knn_ordered(scb_ctx* ctx, const float* x, int64_t n, int32_t d, int32_t ld, int32_t k,
                               const uint16_t* order_key, int32_t* knn_index, float* knn_dist, void* stream,
                               void* ev_start, void* ev_end) {
  SCB_REQUIRE(ctx && x && knn_index && knn_dist, SCB_ERR_ARG, "scb_knn_ordered: null argument");
  SCB_REQUIRE(d >= 1 && d <= kD - 2 && ld >= d && k >= 1 && k <= 16 && k <= n, SCB_ERR_ARG, "scb_knn_ordered: bad args");
  if (n == 0) return SCB_OK;
  return launch_knn<16, 2>(ctx, x, n, x, n, d, ld, k, knn_index, knn_dist, (cudaStream_t)stream, (cudaEvent_t)ev_start,
                           (cudaEvent_t)ev_end, order_key);
}

extern "C" int scb_knn(scb_ctx* ctx, const float* queries, int64_t n_queries, const float* keys, int64_t n_keys,
                       int32_t d, int32_t ld, int32_t k, int32_t k_cand, int32_t* knn_index, float* knn_dist,
                       void* stream) {
  return scb_knn_timed(ctx, queries, n_queries, keys, n_keys, d, ld, k, k_cand, knn_index, knn_dist, stream, nullptr,
                       nullptr);
}

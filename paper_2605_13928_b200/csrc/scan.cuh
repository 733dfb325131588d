// Device-wide exclusive prefix sums (int64) in three launches: per-tile totals,
// one-CTA scan of the totals, per-tile scan + offset.  Used for row compaction
// (N <= ~1e9) where the cost is negligible next to the streaming passes.
#pragma once
#include "common.cuh"

namespace scb {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

struct ScanU8 {
  const uint8_t* p;
  __device__ int64_t operator()(int64_t i, int64_t n) const { return i < n ? (int64_t)p[i] : 0; }
};
struct ScanI64DevLen {
  const int64_t* p;
  const int64_t* len;
  __device__ int64_t operator()(int64_t i, int64_t n) const {
    const int64_t m = *len;
    return (i < n && i < m) ? p[i] : 0;
  }
};

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total, int64_t* sbuf) {
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if ((threadIdx.x & 31) >= o) incl += t;
  }
  if ((threadIdx.x & 31) == 31) sbuf[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t s = (threadIdx.x < (blockDim.x >> 5)) ? sbuf[threadIdx.x] : 0;
    int64_t si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, si, o);
      if (threadIdx.x >= o) si += t;
    }
    sbuf[threadIdx.x] = si - s;
    if (threadIdx.x == 31) sbuf[32] = si;
  }
  __syncthreads();
  int64_t r = sbuf[threadIdx.x >> 5] + incl - v;
  *total = sbuf[32];
  __syncthreads();
  return r;
}

template <typename F>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(F f, int64_t n, int64_t* sums) {
  __shared__ int64_t sbuf[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) v += f(base + k, n);
  int64_t tot;
  block_excl_scan(v, &tot, sbuf);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

static __global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(int64_t* sums, int64_t nb) {
  __shared__ int64_t sbuf[33];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < nb ? sums[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot, sbuf);
    if (i < nb) sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}

// out[i] for i in [0, n] (limit: out written only for i <= *len when len != nullptr)
template <typename F>
__global__ void __launch_bounds__(kScanThreads)
scan_apply(F f, int64_t n, const int64_t* sums, int64_t* out, const int64_t* len) {
  __shared__ int64_t sbuf[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t t = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) { v[k] = f(base + k, n); t += v[k]; }
  int64_t tot;
  int64_t ex = block_excl_scan(t, &tot, sbuf) + sums[blockIdx.x];
  const int64_t lim = len ? *len : n;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k <= lim && base + k <= n) out[base + k] = ex;
    ex += v[k];
  }
}

template <typename F>
inline int scan_generic(scb_ctx* ctx, F f, int64_t n, int64_t* out, const int64_t* len, cudaStream_t s) {
  const int64_t nb = n / kScanTile + 1;  // covers index n as well
  void* ws;
  SCB_TRY(ws_get(ctx, 3, (size_t)(nb + 1) * 8, &ws, s));
  int64_t* sums = (int64_t*)ws;
  scan_tile_sums<<<(unsigned)nb, kScanThreads, 0, s>>>(f, n, sums);
  SCB_LAUNCH_CHECK();
  scan_sums_kernel<<<1, kScanThreads, 0, s>>>(sums, nb);
  SCB_LAUNCH_CHECK();
  scan_apply<<<(unsigned)nb, kScanThreads, 0, s>>>(f, n, sums, out, len);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

inline int scan_u8_to_i64(scb_ctx* ctx, const uint8_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  return scan_generic(ctx, ScanU8{in}, n, out, nullptr, s);
}
inline int scan_i64_dev_len(scb_ctx* ctx, const int64_t* in, const int64_t* len, int64_t n_max, int64_t* out,
                            cudaStream_t s) {
  return scan_generic(ctx, ScanI64DevLen{in, len}, n_max, out, len, s);
}
struct ScanI64 {
  const int64_t* p;
  __device__ int64_t operator()(int64_t i, int64_t m) const { return i < m ? p[i] : 0; }
};
inline int scan_i64(scb_ctx* ctx, const int64_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  return scan_generic(ctx, ScanI64{in}, n, out, nullptr, s);
}

}  // namespace scb

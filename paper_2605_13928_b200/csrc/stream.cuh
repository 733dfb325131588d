// Warp-per-row streaming of CSR rows with 16-byte vector loads.
//
// A warp walks the row [b, e) in windows of 128 elements: lane l owns the 4 consecutive
// elements at base + 128*u + 4*l (u < U windows in flight), loaded with one 16-byte
// ld.global.nc per array, so every warp keeps U x 1 KB of index+value bytes in flight.
// Compact inputs: uint16_t column indices and/or uint16_t counts (the lossless "u16" CSR
// wire format, G <= 65536) are loaded 8 bytes per lane-quad and widened in registers -- half
// the HBM bytes per nonzero, the same Quad for the consumer.  A u16 count of 65535 is an
// escape: the true value (>= 65535, rare) is found by binary search of its position in the
// sorted escape table (U16Esc).
// Elements outside [b, e) are masked (the vector start is rounded down to a multiple of 4;
// the arrays must be 16-byte aligned).  The tail vector that would cross the end of the
// arrays is read with scalar loads.
#pragma once
#include "common.cuh"

namespace scb {

__device__ __forceinline__ int4 ld_nc_v4(const int* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_nc_v4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint2 ld_nc_v2(const uint16_t* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void ld4(const int* p, int (&o)[4]) {
  const int4 v = ld_nc_v4(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld4(const float* p, float (&o)[4]) {
  const float4 v = ld_nc_v4(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void ld4(const uint16_t* p, int (&o)[4]) {
  const uint2 v = ld_nc_v2(p);
  o[0] = (int)(v.x & 0xffffu); o[1] = (int)(v.x >> 16); o[2] = (int)(v.y & 0xffffu); o[3] = (int)(v.y >> 16);
}
__device__ __forceinline__ void ld4(const uint16_t* p, float (&o)[4]) {
  const uint2 v = ld_nc_v2(p);
  o[0] = (float)(v.x & 0xffffu); o[1] = (float)(v.x >> 16); o[2] = (float)(v.y & 0xffffu); o[3] = (float)(v.y >> 16);
}

// escape table of a u16 count array: sorted global positions and their float values
struct U16Esc {
  const int64_t* pos;
  const float* val;
  int64_t n;
};

__device__ __noinline__ float esc_lookup(const U16Esc& esc, int64_t p) {
  int64_t lo = 0, hi = esc.n - 1;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (esc.pos[m] < p) lo = m + 1; else hi = m;
  }
  return (esc.n > 0 && esc.pos[lo] == p) ? esc.val[lo] : 65535.0f;
}

template <typename VT>
__device__ __forceinline__ void fix_escapes(const U16Esc&, int64_t, float (&)[4]) {}
template <>
__device__ __forceinline__ void fix_escapes<uint16_t>(const U16Esc& esc, int64_t p, float (&x)[4]) {
  if (esc.n == 0) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (x[k] == 65535.0f) x[k] = esc_lookup(esc, p + k);
}

struct Quad {
  int64_t p;   // position of element 0
  int g[4];    // column indices
  float x[4];  // values (0 when no value array)
  unsigned valid;  // bit k: element p+k inside [b, e)
};

// one window of U quads starting at `base` (lane l: elements base + 128u + 4l .. +3)
template <int U, typename IT, typename VT>
__device__ __forceinline__ void load_window(const IT* __restrict__ idx, const VT* __restrict__ val, int64_t base,
                                            int64_t b, int64_t e, int64_t nnz, Quad (&q)[U], const U16Esc& esc) {
  const int lane = lane_id();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t p = base + 128 * u + 4 * lane;
    q[u].p = p;
    q[u].valid = 0;
    if (p < e) {
      if (p + 4 <= nnz) {
        ld4(idx + p, q[u].g);
        if (val) ld4(val + p, q[u].x);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          q[u].g[k] = (p + k < nnz) ? (int)idx[p + k] : 0;
          if (val) q[u].x[k] = (p + k < nnz) ? (float)val[p + k] : 0.0f;
        }
      }
      if (!val) {
#pragma unroll
        for (int k = 0; k < 4; ++k) q[u].x[k] = 0.0f;
      } else {
        fix_escapes<VT>(esc, p, q[u].x);
      }
      // valid bits of p+k in [b, e): only a row's first and last quads are partial
      const int64_t rem = e - p;  // >= 1
      uint32_t m = rem >= 4 ? 0xFu : ((1u << (uint32_t)rem) - 1u);
      if (p < b) m &= 0xFu << (uint32_t)(b - p);
      q[u].valid = m;
    }
  }
}

template <int U, typename IT, typename VT, typename F>
__device__ __forceinline__ void stream_row(const IT* __restrict__ idx, const VT* __restrict__ val, int64_t b,
                                           int64_t e, int64_t nnz, F&& f, const U16Esc& esc = U16Esc{nullptr, nullptr, 0}) {
  for (int64_t base = b & ~int64_t(3); base < e; base += 128 * U) {
    Quad q[U];
    load_window<U>(idx, val, base, b, e, nnz, q, esc);
#pragma unroll
    for (int u = 0; u < U; ++u) f(q[u]);
  }
}

// Software-pipelined variant: the next window's loads are issued before the current window
// is processed, so a warp always has U x 1 KB in flight while it computes (for kernels whose
// per-element work is long enough to expose the load latency).
template <int U, typename IT, typename VT, typename F>
__device__ __forceinline__ void stream_row_pipe(const IT* __restrict__ idx, const VT* __restrict__ val, int64_t b,
                                                int64_t e, int64_t nnz, F&& f,
                                                const U16Esc& esc = U16Esc{nullptr, nullptr, 0}) {
  int64_t base = b & ~int64_t(3);
  if (base >= e) return;
  Quad cur[U];
  load_window<U>(idx, val, base, b, e, nnz, cur, esc);
  for (;;) {
    const int64_t nb = base + 128 * U;
    Quad nxt[U];
    if (nb < e) load_window<U>(idx, val, nb, b, e, nnz, nxt, esc);
#pragma unroll
    for (int u = 0; u < U; ++u) f(cur[u]);
    if (nb >= e) break;
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    base = nb;
  }
}

}  // namespace scb

// Common device/host helpers for the B200 single-cell path (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "../../include/scb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "this library targets sm_100a only"
#endif

namespace scb {

constexpr int kNumSMs = 148;
constexpr int kWarp = 32;

// ------------------------------------------------------------------ error plumbing
void set_error(const char* fmt, ...);
const char* last_error();
void count_launch();  // every kernel launch of the library bumps a process-wide counter

#define SCB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::scb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                   \
                       cudaGetErrorString(_e));                                     \
      return SCB_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define SCB_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    ::scb::count_launch();                                                          \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::scb::set_error("%s:%d launch: %s", __FILE__, __LINE__,                      \
                       cudaGetErrorString(_e));                                     \
      return SCB_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define SCB_REQUIRE(cond, code, ...)                                                \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      ::scb::set_error(__VA_ARGS__);                                                \
      return (code);                                                                \
    }                                                                               \
  } while (0)

#define SCB_TRY(call)                                                               \
  do {                                                                              \
    int _rc = (call);                                                               \
    if (_rc != SCB_OK) return _rc;                                                  \
  } while (0)

// ------------------------------------------------------------------ context
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace scb

struct scb_ctx {
  int device = 0;
  int num_sms = scb::kNumSMs;
  size_t smem_optin = 0;
  scb::Workspace ws[4];  // independent scratch slots (grown on demand, stream-ordered use)
  int* d_flag = nullptr; // device error flag (non-integral counts etc.)
  int defer_checks = 0;
  void* comm = nullptr;   // ncclComm_t (scb_ctx_create_comm), else nullptr (world 1)
  int rank = 0, world = 1;  // 1: data checks that need a host round trip are reported later (see scb.h)
};

namespace scb {

// Grow-only scratch slot; contents are undefined on return.
int ws_get(scb_ctx* ctx, int slot, size_t bytes, void** out, cudaStream_t s);

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float ldg_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Fixed-point accumulation on native 32-bit shared atomics (ATOMS.ADD).
// A value v (u64) is added to a (lo, hi) pair of u32 words: the low word takes the
// low 32 bits and signals its carry through the returned old value; the high word is
// touched only when the high part or the carry is non-zero (rare for the magnitudes
// used here), so the common case costs ONE native atomic.
__device__ __forceinline__ void fx_add(uint32_t* lo, uint32_t* hi, uint64_t v) {
  uint32_t vl = (uint32_t)v;
  uint32_t vh = (uint32_t)(v >> 32);
  if (vl) {
    uint32_t old = atomicAdd(lo, vl);
    vh += (old > 0xffffffffu - vl) ? 1u : 0u;
  }
  if (vh) atomicAdd(hi, vh);
}

// 128-bit global accumulator (lo, hi u64) with carry.
__device__ __forceinline__ void fx128_add(unsigned long long* lo, unsigned long long* hi, uint64_t v) {
  if (!v) return;
  unsigned long long old = atomicAdd(lo, (unsigned long long)v);
  if (old > ~0ull - v) atomicAdd(hi, 1ull);
}

__device__ __forceinline__ double fx128_to_double(uint64_t lo, uint64_t hi, int frac_bits) {
  // exact for values < 2^53 * 2^-frac; otherwise correctly ordered round of hi*2^64+lo
  double d = (double)hi * 18446744073709551616.0 + (double)lo;
  return ldexp(d, -frac_bits);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace scb

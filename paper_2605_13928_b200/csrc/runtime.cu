// Context, scratch arena and error reporting behind the C ABI.
#include "common.cuh"
#include <algorithm>
#include <atomic>

namespace scb {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

int ws_get(scb_ctx* ctx, int slot, size_t bytes, void** out, cudaStream_t s) {
  SCB_REQUIRE(slot >= 0 && slot < 4, SCB_ERR_ARG, "ws_get: bad slot");
  Workspace& w = ctx->ws[slot];
  if (w.bytes < bytes) {
    if (w.ptr) {
      SCB_CUDA(cudaStreamSynchronize(s));  // previous users of the slot must be done
      SCB_CUDA(cudaFree(w.ptr));
      w.ptr = nullptr;
      w.bytes = 0;
    }
    size_t want = std::max(bytes, (size_t)1 << 20);
    cudaError_t e = cudaMalloc(&w.ptr, want);
    if (e != cudaSuccess) {
      set_error("ws_get: cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
      return SCB_ERR_NOMEM;
    }
    w.bytes = want;
  }
  *out = w.ptr;
  return SCB_OK;
}

}  // namespace scb

extern "C" int scb_abi_version(void) { return SCB_ABI_VERSION; }
extern "C" const char* scb_last_error(void) { return scb::last_error(); }
extern "C" unsigned long long scb_launch_count(void) { return scb::g_launches.load(); }

extern "C" int scb_ctx_create(int device, scb_ctx** out) {
  SCB_REQUIRE(out, SCB_ERR_ARG, "scb_ctx_create: null out");
  int ndev = 0;
  SCB_CUDA(cudaGetDeviceCount(&ndev));
  SCB_REQUIRE(device >= 0 && device < ndev, SCB_ERR_ARG, "scb_ctx_create: device %d out of range (%d)", device, ndev);
  SCB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SCB_CUDA(cudaGetDeviceProperties(&prop, device));
  SCB_REQUIRE(prop.major == 10 && prop.minor == 0, SCB_ERR_UNSUPPORTED,
              "scb_ctx_create: device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
              prop.major, prop.minor);
  scb_ctx* c = new scb_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  cudaError_t e = cudaMalloc(&c->d_flag, 16);
  if (e != cudaSuccess) {
    delete c;
    scb::set_error("scb_ctx_create: %s", cudaGetErrorString(e));
    return SCB_ERR_CUDA;
  }
  *out = c;
  return SCB_OK;
}

extern "C" int scb_ctx_set_deferred_checks(scb_ctx* ctx, int32_t on) {
  SCB_REQUIRE(ctx, SCB_ERR_ARG, "scb_ctx_set_deferred_checks: null ctx");
  ctx->defer_checks = on ? 1 : 0;
  return SCB_OK;
}

extern "C" int scb_ctx_destroy(scb_ctx* ctx) {
  if (!ctx) return SCB_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& w : ctx->ws)
    if (w.ptr) cudaFree(w.ptr);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  delete ctx;
  return SCB_OK;
}

// ------------------------------------------------------------------ TMA descriptors
#include <cudaTypedefs.h>
#include "tc_common.cuh"

namespace scb {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems, int elem_bytes,
                 uint32_t box_cols, uint32_t box_rows, bool atom32) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    SCB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    SCB_REQUIRE(fn && q == cudaDriverEntryPointSuccess, SCB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  SCB_REQUIRE(elem_bytes == 4 || elem_bytes == 2, SCB_ERR_ARG, "TMA: unsupported element size");
  SCB_REQUIRE(((uintptr_t)base & 15) == 0 && (ld_elems * elem_bytes) % 16 == 0, SCB_ERR_ARG,
              "TMA operand must be 16-byte aligned with a 16-byte multiple row stride");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SCB_REQUIRE(r == CUDA_SUCCESS, SCB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SCB_OK;
}

int make_tmap_2d_f32(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                     uint32_t box_cols, uint32_t box_rows, bool atom32) {
  return make_tmap_2d(m, base, rows, cols, ld_elems, 4, box_cols, box_rows, atom32);
}

}  // namespace scb

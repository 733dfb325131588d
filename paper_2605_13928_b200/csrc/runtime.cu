// Context, scratch arena and error reporting behind the C ABI.
#include "common.cuh"
#include <algorithm>

namespace scb {

static thread_local char g_err[1024] = "";

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

// Context, scratch arena and error reporting behind the C ABI.
#include "common.cuh"
#include <algorithm>
#include <atomic>
#include <cstring>

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

extern "C" int scb_ctx_copy_data_flag(scb_ctx* ctx, int32_t* dst, void* stream) {
  SCB_REQUIRE(ctx && dst, SCB_ERR_ARG, "scb_ctx_copy_data_flag: null argument");
  SCB_CUDA(cudaMemcpyAsync(dst, ctx->d_flag, sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return SCB_OK;
}

static void scb_comm_release(scb_ctx* ctx);

extern "C" int scb_ctx_destroy(scb_ctx* ctx) {
  if (!ctx) return SCB_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& w : ctx->ws)
    if (w.ptr) cudaFree(w.ptr);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  scb_comm_release(ctx);
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

// ------------------------------------------------------------------ NCCL communicator in the ctx
// One communicator per ctx (= per GPU / rank) for the cell-sharded path's collectives (SURVEY.md
// §8(b2)/(e)): SUM/MAX all-reduce of gene sums / Gram / scalars, broadcast of the eigenvectors,
// all-gather of the embedding rows.  libnccl.so.2 is opened at run time (dlopen) so the library
// loads without NCCL; only the communicator entry points need it.
#include <dlfcn.h>
#include <nccl.h>

namespace scb {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;

static int nccl_load() {
  if (g_nccl.h) return SCB_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  SCB_REQUIRE(h, SCB_ERR_UNSUPPORTED, "NCCL: cannot open libnccl.so.2 (%s)", dlerror());
  NcclApi a;
  a.h = h;
  a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
  a.init_rank = (decltype(a.init_rank))dlsym(h, "ncclCommInitRank");
  a.destroy = (decltype(a.destroy))dlsym(h, "ncclCommDestroy");
  a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
  a.broadcast = (decltype(a.broadcast))dlsym(h, "ncclBroadcast");
  a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
  a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
  SCB_REQUIRE(a.get_unique_id && a.init_rank && a.destroy && a.all_reduce && a.broadcast && a.all_gather &&
                  a.error_string,
              SCB_ERR_UNSUPPORTED, "NCCL: missing symbols in libnccl.so.2");
  g_nccl = a;
  return SCB_OK;
}

#define SCB_NCCL(call)                                                                                    \
  do {                                                                                                    \
    const ncclResult_t _r = (call);                                                                       \
    SCB_REQUIRE(_r == ncclSuccess, SCB_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                scb::g_nccl.error_string(_r));                                                               \
  } while (0)

static int nccl_type(int32_t dtype, ncclDataType_t* t, size_t* size) {
  switch (dtype) {
    case 0: *t = ncclInt64; *size = 8; return SCB_OK;
    case 1: *t = ncclFloat64; *size = 8; return SCB_OK;
    case 2: *t = ncclFloat32; *size = 4; return SCB_OK;
    case 3: *t = ncclInt32; *size = 4; return SCB_OK;
    default: break;
  }
  SCB_REQUIRE(false, SCB_ERR_ARG, "scb_comm: dtype must be 0 (i64), 1 (f64), 2 (f32) or 3 (i32)");
  return SCB_ERR_ARG;
}
}  // namespace scb

extern "C" int scb_nccl_unique_id(uint8_t* id_out) {
  SCB_REQUIRE(id_out, SCB_ERR_ARG, "scb_nccl_unique_id: null argument");
  SCB_TRY(scb::nccl_load());
  ncclUniqueId id;
  SCB_NCCL(scb::g_nccl.get_unique_id(&id));
  memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return SCB_OK;
}

extern "C" int scb_ctx_create_comm(int device, const uint8_t* nccl_id, int32_t rank, int32_t world, scb_ctx** out) {
  SCB_REQUIRE(out && nccl_id && world >= 1 && rank >= 0 && rank < world, SCB_ERR_ARG, "scb_ctx_create_comm: bad args");
  SCB_TRY(scb::nccl_load());
  SCB_TRY(scb_ctx_create(device, out));
  ncclUniqueId id;
  memcpy(id.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = scb::g_nccl.init_rank(&comm, world, id, rank);
  if (r != ncclSuccess) {
    scb_ctx_destroy(*out);
    *out = nullptr;
    scb::set_error("scb_ctx_create_comm: ncclCommInitRank failed: %s", scb::g_nccl.error_string(r));
    return SCB_ERR_CUDA;
  }
  (*out)->comm = comm;
  (*out)->rank = rank;
  (*out)->world = world;
  return SCB_OK;
}

extern "C" int scb_comm_info(scb_ctx* ctx, int32_t* rank, int32_t* world) {
  SCB_REQUIRE(ctx && rank && world, SCB_ERR_ARG, "scb_comm_info: null argument");
  *rank = ctx->comm ? ctx->rank : 0;
  *world = ctx->comm ? ctx->world : 1;
  return SCB_OK;
}

extern "C" int scb_comm_allreduce(scb_ctx* ctx, void* buf, int64_t count, int32_t dtype, int32_t op, void* stream) {
  SCB_REQUIRE(ctx && (buf || count == 0), SCB_ERR_ARG, "scb_comm_allreduce: null argument");
  SCB_REQUIRE(op == 0 || op == 1, SCB_ERR_ARG, "scb_comm_allreduce: op must be 0 (sum) or 1 (max)");
  if (!ctx->comm || count == 0) return SCB_OK;  // world 1: identity
  ncclDataType_t t;
  size_t sz;
  SCB_TRY(scb::nccl_type(dtype, &t, &sz));
  SCB_NCCL(scb::g_nccl.all_reduce(buf, buf, (size_t)count, t, op ? ncclMax : ncclSum, (ncclComm_t)ctx->comm,
                                  (cudaStream_t)stream));
  return SCB_OK;
}

extern "C" int scb_comm_broadcast(scb_ctx* ctx, void* buf, int64_t bytes, int32_t root, void* stream) {
  SCB_REQUIRE(ctx && (buf || bytes == 0), SCB_ERR_ARG, "scb_comm_broadcast: null argument");
  if (!ctx->comm || bytes == 0) return SCB_OK;
  SCB_REQUIRE(root >= 0 && root < ctx->world, SCB_ERR_ARG, "scb_comm_broadcast: bad root");
  SCB_NCCL(scb::g_nccl.broadcast(buf, buf, (size_t)bytes, ncclUint8, root, (ncclComm_t)ctx->comm, (cudaStream_t)stream));
  return SCB_OK;
}

extern "C" int scb_comm_allgather(scb_ctx* ctx, const void* send, void* recv, int64_t bytes_per_rank, void* stream) {
  SCB_REQUIRE(ctx && ((send && recv) || bytes_per_rank == 0), SCB_ERR_ARG, "scb_comm_allgather: null argument");
  if (bytes_per_rank == 0) return SCB_OK;
  if (!ctx->comm) {
    if (recv != send)
      SCB_CUDA(cudaMemcpyAsync(recv, send, (size_t)bytes_per_rank, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return SCB_OK;
  }
  SCB_NCCL(scb::g_nccl.all_gather(send, recv, (size_t)bytes_per_rank, ncclUint8, (ncclComm_t)ctx->comm,
                                  (cudaStream_t)stream));
  return SCB_OK;
}

static void scb_comm_release(scb_ctx* ctx) {
  if (ctx->comm && scb::g_nccl.destroy) scb::g_nccl.destroy((ncclComm_t)ctx->comm);
  ctx->comm = nullptr;
}

// Community detection on the neighbors graph (second half: the clustering
// step sc.tl.leiden / sc.tl.louvain runs on `connectivities`): multi-level modularity
// optimisation (Louvain local moving + aggregation, resolution gamma), deterministic.
//
//   weights   edge weights in 2^-32 fixed point (int64): node strengths k_i, community totals
//             and the per-node community links are then exact integer sums, independent of
//             summation order, so the device and the oracle (oracle/pipeline.py louvain) take
//             the same decisions;
//   moving    nodes are split into 8 hash buckets; per bucket, a warp per node accumulates its
//             links to neighbouring communities in a shared-memory hash table and picks
//             argmax_c  w_ic - gamma k_i tot_c / 2m  (tot_a excludes the node itself; ties ->
//             smaller c; moves only on a strict gain; a node that moved in the previous
//             iteration sits one out, which removes the 2-cycles synchronous moves produce), then
//             the bucket's moves are applied (int64 atomics on tot); repeated until no node moves
//             (or max_iters);
//   aggregate communities are renumbered and the graph is contracted: (c_i, c_j) keys radix-
//             sorted (CUB) and reduced by key into the next level's CSR (self loops keep the
//             internal weight).
// Stops when a level moves no node.  Labels are renumbered by decreasing community size (ties
// by smallest member), as Scanpy orders its categories.  Modularity Q = Σ_c in_c/2m -
// gamma (tot_c/2m)^2 on the input graph.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cuda/std/functional>
#include <algorithm>
#include <cstdlib>
#include <vector>
#include "common.cuh"
#include "scan.cuh"

namespace scb {

constexpr int kTab = 512;       // hash slots per warp (48 KB per 8-warp CTA: 4 CTAs per SM)
constexpr int kClWarps = 8;     // warps per CTA in the moving kernel
constexpr int kBuckets = 8;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void to_fixed_kernel(const float* __restrict__ w, int64_t n, long long* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = llrint((double)w[i] * 4294967296.0);
}

__global__ void strength_kernel(const int64_t* __restrict__ indptr, const long long* __restrict__ W, int64_t n,
                                long long* __restrict__ k, int32_t* __restrict__ comm,
                                unsigned long long* __restrict__ tot, unsigned long long* __restrict__ m2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    long long s = 0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) s += W[e];
    k[i] = s;
    comm[i] = (int32_t)i;
    tot[i] = (unsigned long long)s;
    atomicAdd(m2, (unsigned long long)s);
  }
}

__device__ __forceinline__ bool better(double g, int c, double bg, int bc) { return g > bg || (g == bg && c < bc); }

__global__ void __launch_bounds__(kClWarps * 32)
move_decide_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nbr, const long long* __restrict__ W,
                   int64_t n, const long long* __restrict__ k, const int32_t* __restrict__ comm,
                   const unsigned long long* __restrict__ tot, const unsigned long long* __restrict__ m2p,
                   double gamma, int bucket, uint32_t seed, const int32_t* __restrict__ last, int iter,
                   int32_t* __restrict__ newc) {
  extern __shared__ unsigned char cl_smem[];
  const int wid = warp_id(), lane = lane_id();
  int* keys = reinterpret_cast<int*>(cl_smem) + wid * kTab;
  unsigned long long* vals =
      reinterpret_cast<unsigned long long*>(cl_smem + (size_t)kClWarps * kTab * 4) + (size_t)wid * kTab;
  const double m2 = (double)(long long)*m2p;
  for (int64_t i = (int64_t)blockIdx.x * kClWarps + wid; i < n; i += (int64_t)gridDim.x * kClWarps) {
    if ((int)(mix32((uint32_t)i ^ seed) % kBuckets) != bucket) continue;
    const int a = comm[i];
    if (last[i] == iter - 1) {  // moved in the previous iteration: sits this one out (no 2-cycles)
      if (lane == 0) newc[i] = a;
      continue;
    }
    const long long ki = k[i];
    for (int t = lane; t < kTab; t += 32) { keys[t] = -1; vals[t] = 0ull; }
    __syncwarp();
    bool overflow = false;
    const int64_t e0 = indptr[i], e1 = indptr[i + 1];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      if (e < e1) {
        const int j = nbr[e];
        if (j != i) {  // a self loop is internal weight, not a link
          const int c = comm[j];
          uint32_t h = mix32((uint32_t)c) & (kTab - 1);
          for (int probes = 0;; ++probes) {
            const int prev = atomicCAS(&keys[h], -1, c);
            if (prev == -1 || prev == c) {
              atomicAdd(&vals[h], (unsigned long long)W[e]);
              break;
            }
            if (probes + 1 >= kTab) { overflow = true; break; }  // > kTab distinct communities
            h = (h + 1) & (kTab - 1);
          }
        }
      }
      // a full table means > kTab neighbour communities: the node stays (stop scanning its row)
      if (__any_sync(0xffffffffu, overflow)) { overflow = true; break; }
    }
    __syncwarp();
    const double kd = (double)ki;
    const double tot_a = (double)((long long)tot[a] - ki);
    const double stay = -gamma * kd * tot_a / m2;  // w_ia added below if a is a neighbour community
    double bg = -1e300;
    int bc = INT32_MAX;
    double ga = stay;
    for (int t = lane; t < kTab; t += 32) {
      const int c = keys[t];
      if (c < 0) continue;
      const double wic = (double)(long long)vals[t];
      if (c == a) {
        ga = wic + stay;
        continue;
      }
      const double g = wic - gamma * kd * (double)(long long)tot[c] / m2;
      if (better(g, c, bg, bc)) { bg = g; bc = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (better(og, oc, bg, bc)) { bg = og; bc = oc; }
      ga = fmax(ga, __shfl_xor_sync(0xffffffffu, ga, o));  // only the owner lane has it; others stay
    }
    if (lane == 0) newc[i] = (!overflow && bc != INT32_MAX && bg > ga) ? bc : a;
    __syncwarp();
  }
}

__global__ void move_apply_kernel(int64_t n, const long long* __restrict__ k, int32_t* __restrict__ comm,
                                  const int32_t* __restrict__ newc, unsigned long long* __restrict__ tot, int bucket,
                                  uint32_t seed, int32_t* __restrict__ last, int iter,
                                  unsigned long long* __restrict__ moved) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if ((int)(mix32((uint32_t)i ^ seed) % kBuckets) != bucket) continue;
    const int a = comm[i], c = newc[i];
    if (a == c) continue;
    atomicAdd(&tot[c], (unsigned long long)k[i]);
    atomicAdd(&tot[a], (unsigned long long)(-k[i]));
    comm[i] = c;
    last[i] = iter;
    atomicAdd(moved, 1ull);
  }
}

__global__ void used_kernel(const int32_t* __restrict__ comm, int64_t n, uint8_t* __restrict__ used) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    used[comm[i]] = 1;
}

// cell -> node of this level -> new id
__global__ void compose_kernel(int32_t* __restrict__ node_of_cell, int64_t n_cells, const int32_t* __restrict__ comm,
                               const int64_t* __restrict__ rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_cells; i += (int64_t)gridDim.x * blockDim.x)
    node_of_cell[i] = (int32_t)rank[comm[node_of_cell[i]]];
}

__global__ void edge_keys_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nbr, int64_t n,
                                 const int32_t* __restrict__ comm, const int64_t* __restrict__ rank, int64_t n_new,
                                 unsigned long long* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long ci = (unsigned long long)rank[comm[i]];
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e)
      keys[e] = ci * (unsigned long long)n_new + (unsigned long long)rank[comm[nbr[e]]];
  }
}

__global__ void coarse_csr_kernel(const unsigned long long* __restrict__ ukeys, int64_t nu, int64_t n_new,
                                  int64_t* __restrict__ indptr, int32_t* __restrict__ nbr) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= nu; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = e == 0 ? -1 : (int64_t)(ukeys[e - 1] / (unsigned long long)n_new);
    const int64_t hi = e == nu ? n_new - 1 : (int64_t)(ukeys[e] / (unsigned long long)n_new);
    for (int64_t r = lo + 1; r <= hi; ++r) indptr[r] = e;
    if (e == nu) indptr[n_new] = nu;
    if (e < nu) nbr[e] = (int32_t)(ukeys[e] % (unsigned long long)n_new);
  }
}

// modularity pieces on the input graph: in (same-label edge weight), per-label totals
__global__ void modularity_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nbr,
                                  const long long* __restrict__ W, int64_t n, const int32_t* __restrict__ lab,
                                  unsigned long long* __restrict__ in_sum, unsigned long long* __restrict__ ltot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    long long s = 0, t = 0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      t += W[e];
      if (lab[nbr[e]] == lab[i]) s += W[e];
    }
    atomicAdd(in_sum, (unsigned long long)s);
    atomicAdd(&ltot[lab[i]], (unsigned long long)t);
  }
}

// ---------------------------------------------------------------- Leiden refinement
__global__ void init_tot_kernel(const int32_t* __restrict__ comm, const long long* __restrict__ k, int64_t n,
                                unsigned long long* __restrict__ tot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&tot[comm[i]], (unsigned long long)k[i]);
}

// R_s, |s| and the external weight ext_s = w(s, C - s) of every sub-community of the refined
// partition (exact integers)
__global__ void refine_stats_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nbr,
                                    const long long* __restrict__ W, int64_t n, const long long* __restrict__ k,
                                    const int32_t* __restrict__ comm, const int32_t* __restrict__ ref,
                                    unsigned long long* __restrict__ R, unsigned int* __restrict__ cnt,
                                    unsigned long long* __restrict__ ext) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    const int ru = ref[u], cu = comm[u];
    atomicAdd(&R[ru], (unsigned long long)k[u]);
    atomicAdd(&cnt[ru], 1u);
    long long e_sum = 0;
    for (int64_t e = indptr[u]; e < indptr[u + 1]; ++e) {
      const int x = nbr[e];
      if (x != u && comm[x] == cu && ref[x] != ru) e_sum += W[e];
    }
    if (e_sum) atomicAdd(&ext[ru], (unsigned long long)e_sum);
  }
}

__global__ void __launch_bounds__(kClWarps * 32)
refine_decide_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nbr,
                     const long long* __restrict__ W, int64_t n, const long long* __restrict__ k,
                     const int32_t* __restrict__ comm, const int32_t* __restrict__ ref,
                     const unsigned long long* __restrict__ K, const unsigned long long* __restrict__ R,
                     const unsigned int* __restrict__ cnt, const unsigned long long* __restrict__ ext,
                     const unsigned long long* __restrict__ m2p, double gamma, int bucket, uint32_t seed,
                     int32_t* __restrict__ newref) {
  extern __shared__ unsigned char cl_smem[];
  const int wid = warp_id(), lane = lane_id();
  int* keys = reinterpret_cast<int*>(cl_smem) + wid * kTab;
  unsigned long long* vals =
      reinterpret_cast<unsigned long long*>(cl_smem + (size_t)kClWarps * kTab * 4) + (size_t)wid * kTab;
  const double m2 = (double)(long long)*m2p;
  for (int64_t v = (int64_t)blockIdx.x * kClWarps + wid; v < n; v += (int64_t)gridDim.x * kClWarps) {
    if ((int)(mix32((uint32_t)v ^ seed ^ 0x9E3779B9u) % kBuckets) != bucket) continue;
    if (ref[v] != v || cnt[v] != 1u) {  // only singletons move
      if (lane == 0) newref[v] = ref[v];
      continue;
    }
    const int C = comm[v];
    const long long kv = k[v];
    for (int t = lane; t < kTab; t += 32) { keys[t] = -1; vals[t] = 0ull; }
    __syncwarp();
    bool overflow = false;
    long long wvc = 0;
    const int64_t e0 = indptr[v], e1 = indptr[v + 1];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      if (e < e1) {
        const int x = nbr[e];
        if (x != v && comm[x] == C) {
          wvc += W[e];
          const int sx = ref[x];
          uint32_t h = mix32((uint32_t)sx) & (kTab - 1);
          for (int probes = 0;; ++probes) {
            const int prev = atomicCAS(&keys[h], -1, sx);
            if (prev == -1 || prev == sx) {
              atomicAdd(&vals[h], (unsigned long long)W[e]);
              break;
            }
            if (probes + 1 >= kTab) { overflow = true; break; }
            h = (h + 1) & (kTab - 1);
          }
        }
      }
      if (__any_sync(0xffffffffu, overflow)) { overflow = true; break; }
    }
    __syncwarp();
    wvc = warp_sum(wvc);
    const double kd = (double)kv;
    const long long KC = (long long)K[C];
    double bq = -1e300;
    int bs = INT32_MAX;
    if (!overflow && (double)wvc >= gamma * kd * (double)(KC - kv) / m2) {
      for (int t = lane; t < kTab; t += 32) {
        const int sx = keys[t];
        if (sx < 0) continue;
        const long long Rs = (long long)R[sx];
        if (!((double)(long long)ext[sx] >= gamma * (double)Rs * (double)(KC - Rs) / m2)) continue;
        const double dq = (double)(long long)vals[t] - gamma * kd * (double)Rs / m2;
        if (better(dq, sx, bq, bs)) { bq = dq; bs = sx; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oq = __shfl_xor_sync(0xffffffffu, bq, o);
      const int os = __shfl_xor_sync(0xffffffffu, bs, o);
      if (better(oq, os, bq, bs)) { bq = oq; bs = os; }
    }
    if (lane == 0) newref[v] = (bs != INT32_MAX && bq >= 0.0) ? bs : (int)v;
    __syncwarp();
  }
}

__global__ void refine_apply_kernel(int64_t n, int32_t* __restrict__ ref, const int32_t* __restrict__ newref, int bucket,
                                    uint32_t seed) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if ((int)(mix32((uint32_t)v ^ seed ^ 0x9E3779B9u) % kBuckets) == bucket) ref[v] = newref[v];
}

__global__ void iota_kernel(int32_t* __restrict__ x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)i;
}

__global__ void map_kernel(int32_t* __restrict__ x, int64_t n, const int32_t* __restrict__ m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = m[x[i]];
}

// next level: aggregate node rank_ref[ref[i]] starts in community rank_comm[comm[i]]
__global__ void carry_comm_kernel(int64_t n, const int32_t* __restrict__ ref, const int32_t* __restrict__ comm,
                                  const int64_t* __restrict__ rank_ref, const int64_t* __restrict__ rank_comm,
                                  int32_t* __restrict__ next_comm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    next_comm[rank_ref[ref[i]]] = (int32_t)rank_comm[comm[i]];
}

}  // namespace scb

using namespace scb;

namespace {
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() { if (p) cudaFreeAsync(p, s); }
};
}  // namespace

// launch check; with SCB_CLUSTER_DEBUG set, also synchronise so a fault names its launch site
#define CL_CHECK()                                                                              \
  do {                                                                                          \
    SCB_LAUNCH_CHECK();                                                                         \
    if (dbg) {                                                                                  \
      const cudaError_t _e = cudaStreamSynchronize(s);                                          \
      SCB_REQUIRE(_e == cudaSuccess, SCB_ERR_CUDA, "cluster.cu:%d: %s", __LINE__, cudaGetErrorString(_e)); \
    }                                                                                           \
  } while (0)

#define CL_ALLOC(buf, bytes)                                                              \
  do {                                                                                    \
    buf.s = s;                                                                            \
    SCB_CUDA(cudaMallocAsync(&buf.p, std::max<size_t>((size_t)(bytes), 16), s));         \
  } while (0)

static int cluster_impl(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights, int64_t n,
                        int64_t nnz, double resolution, int32_t max_levels, int32_t max_iters, uint32_t seed,
                        int32_t* labels, int32_t* n_communities, double* modularity, void* stream, bool leiden) {
  SCB_REQUIRE(ctx && indptr && indices && weights && labels && n_communities && modularity, SCB_ERR_ARG,
              "scb_louvain/scb_leiden: null argument");
  SCB_REQUIRE(n > 0 && n < INT32_MAX && max_levels >= 1 && max_iters >= 1, SCB_ERR_ARG,
              "scb_louvain/scb_leiden: bad arguments");
  SCB_REQUIRE(nnz > 0, SCB_ERR_ARG, "scb_louvain/scb_leiden: the graph has no edges");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = ctx->num_sms * 8;
  const bool dbg = getenv("SCB_CLUSTER_DEBUG") != nullptr;
  {
    // the level buffers come from the stream-ordered pool; keep its memory mapped between
    // levels/calls (the default release threshold 0 unmaps it at every synchronisation, which
    // made the per-level re-allocation cost up to seconds at 1M cells)
    cudaMemPool_t pool;
    SCB_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
    uint64_t keep = UINT64_MAX;
    SCB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  // level-0 graph (fixed-point weights) kept for the final modularity
  DevBuf W0, scal_b, cell_b;
  CL_ALLOC(W0, nnz * 8);
  to_fixed_kernel<<<grid, 256, 0, s>>>(weights, nnz, (long long*)W0.p);
  CL_CHECK();
  CL_ALLOC(cell_b, n * 4);
  int32_t* node_of_cell = (int32_t*)cell_b.p;  // cell -> node of the current level
  CL_ALLOC(scal_b, 64);
  unsigned long long* m2 = (unsigned long long*)scal_b.p;
  unsigned long long* moved = m2 + 1;
  unsigned long long* in_sum = m2 + 2;
  const int64_t* cur_ip = indptr;
  const int32_t* cur_nb = indices;
  const long long* cur_W = (const long long*)W0.p;
  int64_t cur_n = n, cur_nnz = nnz;
  DevBuf next_ip, next_nb, next_W;  // owned storage of the current coarse level
  const size_t cl_smem = (size_t)kClWarps * kTab * (4 + 8);
  SCB_CUDA(cudaFuncSetAttribute(move_decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem));
  SCB_CUDA(cudaFuncSetAttribute(refine_decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem));
  bool first = true;
  DevBuf carry;  // Leiden: partition P carried into the current level (aggregate node -> community)
  bool leiden_done = false;
  const bool verbose = getenv("SCB_CLUSTER_VERBOSE") != nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (verbose) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, s);
  }
  for (int level = 0; level < max_levels; ++level) {
    DevBuf lk, lcomm, lnewc, ltot;
    CL_ALLOC(lk, cur_n * 8);
    CL_ALLOC(lcomm, cur_n * 4);
    CL_ALLOC(lnewc, cur_n * 4);
    CL_ALLOC(ltot, cur_n * 8);
    long long* k = (long long*)lk.p;
    int32_t* comm = (int32_t*)lcomm.p;
    int32_t* newc = (int32_t*)lnewc.p;
    unsigned long long* tot = (unsigned long long*)ltot.p;
    SCB_CUDA(cudaMemsetAsync(m2, 0, 8, s));
    strength_kernel<<<grid, 256, 0, s>>>(cur_ip, cur_W, cur_n, k, comm, tot, m2);
    CL_CHECK();
    if (first) {  // node_of_cell := identity (comm starts as the identity)
      SCB_CUDA(cudaMemcpyAsync(node_of_cell, comm, n * 4, cudaMemcpyDeviceToDevice, s));
      first = false;
    } else if (leiden) {  // start from the carried partition P
      SCB_CUDA(cudaMemcpyAsync(comm, carry.p, cur_n * 4, cudaMemcpyDeviceToDevice, s));
      SCB_CUDA(cudaMemsetAsync(tot, 0, cur_n * 8, s));
      init_tot_kernel<<<grid, 256, 0, s>>>(comm, k, cur_n, tot);
      CL_CHECK();
    }
    DevBuf llast;
    CL_ALLOC(llast, cur_n * 4);
    int32_t* last = (int32_t*)llast.p;
    SCB_CUDA(cudaMemsetAsync(last, 0xFE, cur_n * 4, s));  // 0xFEFEFEFE: "never moved"
    unsigned long long total_moves = 0;
    for (int it = 0; it < max_iters; ++it) {
      SCB_CUDA(cudaMemsetAsync(moved, 0, 8, s));
      for (int b = 0; b < kBuckets; ++b) {
        move_decide_kernel<<<ctx->num_sms * 4, kClWarps * 32, cl_smem, s>>>(cur_ip, cur_nb, cur_W, cur_n, k, comm, tot,
                                                                             m2, resolution, b, seed, last, it, newc);
        CL_CHECK();
        move_apply_kernel<<<grid, 256, 0, s>>>(cur_n, k, comm, newc, tot, b, seed, last, it, moved);
        CL_CHECK();
      }
      unsigned long long mv = 0;
      SCB_CUDA(cudaMemcpyAsync(&mv, moved, 8, cudaMemcpyDeviceToHost, s));
      SCB_CUDA(cudaStreamSynchronize(s));
      total_moves += mv;
      if (verbose) {
        cudaEventRecord(ev1, s);
        cudaEventSynchronize(ev1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        fprintf(stderr, "[scb_louvain] level %d n %lld nnz %lld iter %d moved %llu  %.2f ms\n", level, (long long)cur_n,
                (long long)cur_nnz, it, mv, ms);
      }
      if (mv == 0) break;
    }
    // renumber communities (order of their smallest node id)
    DevBuf lused, lrank;
    CL_ALLOC(lused, cur_n);
    CL_ALLOC(lrank, (cur_n + 1) * 8);
    int64_t* rank = (int64_t*)lrank.p;
    int64_t n_new = 0;
    auto renumber = [&](const int32_t* part, int64_t* rk, int64_t* count) -> int {
      SCB_CUDA(cudaMemsetAsync(lused.p, 0, cur_n, s));
      used_kernel<<<grid, 256, 0, s>>>(part, cur_n, (uint8_t*)lused.p);
      CL_CHECK();
      SCB_TRY(scan_u8_to_i64(ctx, (const uint8_t*)lused.p, cur_n, rk, s));
      SCB_CUDA(cudaMemcpyAsync(count, rk + cur_n, 8, cudaMemcpyDeviceToHost, s));
      SCB_CUDA(cudaStreamSynchronize(s));
      return SCB_OK;
    };
    const int32_t* agg = comm;  // partition the graph is aggregated by
    DevBuf lref, lnewref, lR, lcnt, lext, lrank2;
    if (!leiden) {
      if (total_moves == 0) break;
      SCB_TRY(renumber(comm, rank, &n_new));
      compose_kernel<<<grid, 256, 0, s>>>(node_of_cell, n, comm, rank);
      CL_CHECK();
      if (n_new == cur_n) break;
    } else {
      // refinement of P inside each community (singletons merge into well-connected
      // sub-communities), one synchronous pass per bucket
      CL_ALLOC(lref, cur_n * 4);
      CL_ALLOC(lnewref, cur_n * 4);
      CL_ALLOC(lR, cur_n * 8);
      CL_ALLOC(lcnt, cur_n * 4);
      CL_ALLOC(lext, cur_n * 8);
      int32_t* ref = (int32_t*)lref.p;
      iota_kernel<<<grid, 256, 0, s>>>(ref, cur_n);
      CL_CHECK();
      for (int b = 0; b < kBuckets; ++b) {
        SCB_CUDA(cudaMemsetAsync(lR.p, 0, cur_n * 8, s));
        SCB_CUDA(cudaMemsetAsync(lcnt.p, 0, cur_n * 4, s));
        SCB_CUDA(cudaMemsetAsync(lext.p, 0, cur_n * 8, s));
        refine_stats_kernel<<<grid, 256, 0, s>>>(cur_ip, cur_nb, cur_W, cur_n, k, comm, ref,
                                                 (unsigned long long*)lR.p, (unsigned int*)lcnt.p,
                                                 (unsigned long long*)lext.p);
        CL_CHECK();
        refine_decide_kernel<<<ctx->num_sms * 4, kClWarps * 32, cl_smem, s>>>(
            cur_ip, cur_nb, cur_W, cur_n, k, comm, ref, tot, (const unsigned long long*)lR.p,
            (const unsigned int*)lcnt.p, (const unsigned long long*)lext.p, m2, resolution, b, seed,
            (int32_t*)lnewref.p);
        CL_CHECK();
        refine_apply_kernel<<<grid, 256, 0, s>>>(cur_n, ref, (const int32_t*)lnewref.p, b, seed);
        CL_CHECK();
      }
      int64_t n_comm = 0;
      CL_ALLOC(lrank2, (cur_n + 1) * 8);
      int64_t* rank_comm = (int64_t*)lrank2.p;
      SCB_TRY(renumber(comm, rank_comm, &n_comm));
      SCB_TRY(renumber(ref, rank, &n_new));
      if ((total_moves == 0 && n_new == n_comm) || n_new == cur_n) {  // final: labels = P
        compose_kernel<<<grid, 256, 0, s>>>(node_of_cell, n, comm, rank_comm);
        CL_CHECK();
        leiden_done = true;
        break;
      }
      compose_kernel<<<grid, 256, 0, s>>>(node_of_cell, n, ref, rank);
      CL_CHECK();
      DevBuf nxt;
      CL_ALLOC(nxt, n_new * 4);
      carry_comm_kernel<<<grid, 256, 0, s>>>(cur_n, ref, comm, rank, rank_comm, (int32_t*)nxt.p);
      CL_CHECK();
      std::swap(carry.p, nxt.p);
      carry.s = s;
      agg = ref;
    }
    DevBuf kin, kout, vout, ukeys, usum, nuniq, tmp;
    CL_ALLOC(kin, cur_nnz * 8);
    CL_ALLOC(kout, cur_nnz * 8);
    CL_ALLOC(vout, cur_nnz * 8);
    edge_keys_kernel<<<grid, 256, 0, s>>>(cur_ip, cur_nb, cur_n, agg, rank, n_new, (unsigned long long*)kin.p);
    CL_CHECK();
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)n_new * (unsigned long long)n_new) > (1ull << end_bit)) ++end_bit;
    size_t tb1 = 0, tb2 = 0;
    SCB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, (unsigned long long*)kin.p, (unsigned long long*)kout.p,
                                             (const long long*)cur_W, (long long*)vout.p, (int)cur_nnz, 0, end_bit, s));
    CL_ALLOC(ukeys, cur_nnz * 8);
    CL_ALLOC(usum, cur_nnz * 8);
    CL_ALLOC(nuniq, 8);
    SCB_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tb2, (unsigned long long*)kout.p, (unsigned long long*)ukeys.p,
                                            (long long*)vout.p, (long long*)usum.p, (int64_t*)nuniq.p,
                                            ::cuda::std::plus<long long>(), (int)cur_nnz, s));
    CL_ALLOC(tmp, std::max(tb1, tb2));
    SCB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb1, (unsigned long long*)kin.p, (unsigned long long*)kout.p,
                                             (const long long*)cur_W, (long long*)vout.p, (int)cur_nnz, 0, end_bit, s));
    SCB_CUDA(cub::DeviceReduce::ReduceByKey(tmp.p, tb2, (unsigned long long*)kout.p, (unsigned long long*)ukeys.p,
                                            (long long*)vout.p, (long long*)usum.p, (int64_t*)nuniq.p,
                                            ::cuda::std::plus<long long>(), (int)cur_nnz, s));
    int64_t nu = 0;
    SCB_CUDA(cudaMemcpyAsync(&nu, nuniq.p, 8, cudaMemcpyDeviceToHost, s));
    SCB_CUDA(cudaStreamSynchronize(s));
    DevBuf cip, cnb;
    CL_ALLOC(cip, (n_new + 1) * 8);
    CL_ALLOC(cnb, nu * 4);
    coarse_csr_kernel<<<grid, 256, 0, s>>>((const unsigned long long*)ukeys.p, nu, n_new, (int64_t*)cip.p,
                                           (int32_t*)cnb.p);
    CL_CHECK();
    // the coarse level becomes current (ownership moves into next_*)
    std::swap(next_ip.p, cip.p);
    std::swap(next_nb.p, cnb.p);
    std::swap(next_W.p, usum.p);
    next_ip.s = next_nb.s = next_W.s = s;
    cur_ip = (const int64_t*)next_ip.p;
    cur_nb = (const int32_t*)next_nb.p;
    cur_W = (const long long*)next_W.p;
    cur_n = n_new;
    cur_nnz = nu;
  }
  if (leiden && !leiden_done && carry.p) {  // max_levels reached: labels = the carried P
    map_kernel<<<grid, 256, 0, s>>>(node_of_cell, n, (const int32_t*)carry.p);
    CL_CHECK();
  }
  // labels by decreasing community size (ties: smallest member), modularity on the input graph
  DevBuf ltot2;
  CL_ALLOC(ltot2, (size_t)n * 8);
  SCB_CUDA(cudaMemsetAsync(ltot2.p, 0, (size_t)n * 8, s));
  SCB_CUDA(cudaMemsetAsync(in_sum, 0, 8, s));
  modularity_kernel<<<grid, 256, 0, s>>>(indptr, indices, (const long long*)W0.p, n, node_of_cell, in_sum,
                                         (unsigned long long*)ltot2.p);
  CL_CHECK();
  std::vector<int32_t> h_lab(n);
  std::vector<unsigned long long> h_tot(n);
  unsigned long long h_in = 0, h_m2 = 0;
  SCB_CUDA(cudaMemcpyAsync(h_lab.data(), node_of_cell, n * 4, cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaMemcpyAsync(h_tot.data(), ltot2.p, n * 8, cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaMemcpyAsync(&h_in, in_sum, 8, cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  int32_t n_c = 0;
  for (int64_t i = 0; i < n; ++i) n_c = std::max(n_c, h_lab[i] + 1);
  // community order: size desc, then smallest member (host: O(n) counting over small arrays)
  std::vector<int64_t> size(n_c, 0), first_member(n_c, INT64_MAX);
  for (int64_t i = 0; i < n; ++i) {
    ++size[h_lab[i]];
    first_member[h_lab[i]] = std::min(first_member[h_lab[i]], i);
  }
  std::vector<int32_t> ord(n_c);
  for (int32_t c = 0; c < n_c; ++c) ord[c] = c;
  std::sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
    return size[x] != size[y] ? size[x] > size[y] : first_member[x] < first_member[y];
  });
  std::vector<int32_t> newid(n_c);
  for (int32_t r = 0; r < n_c; ++r) newid[ord[r]] = r;
  for (int64_t i = 0; i < n; ++i) h_lab[i] = newid[h_lab[i]];
  for (auto v : h_tot) h_m2 += v;
  double q = 0.0;
  const double M2 = (double)(long long)h_m2;
  for (int32_t r = 0; r < n_c; ++r) {
    const double t = (double)(long long)h_tot[ord[r]];
    q -= resolution * (t / M2) * (t / M2);
  }
  q += (double)(long long)h_in / M2;
  SCB_CUDA(cudaMemcpyAsync(labels, h_lab.data(), n * 4, cudaMemcpyHostToDevice, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  *n_communities = n_c;
  *modularity = q;
  return SCB_OK;
}

extern "C" int scb_louvain(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights,
                           int64_t n, int64_t nnz, double resolution, int32_t max_levels, int32_t max_iters,
                           uint32_t seed, int32_t* labels, int32_t* n_communities, double* modularity, void* stream) {
  return cluster_impl(ctx, indptr, indices, weights, n, nnz, resolution, max_levels, max_iters, seed, labels,
                      n_communities, modularity, stream, false);
}

extern "C" int scb_leiden(scb_ctx* ctx, const int64_t* indptr, const int32_t* indices, const float* weights,
                          int64_t n, int64_t nnz, double resolution, int32_t max_levels, int32_t max_iters,
                          uint32_t seed, int32_t* labels, int32_t* n_communities, double* modularity, void* stream) {
  return cluster_impl(ctx, indptr, indices, weights, n, nnz, resolution, max_levels, max_iters, seed, labels,
                      n_communities, modularity, stream, true);
}

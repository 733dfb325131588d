// Probe: tcgen05.mma kind::f16 with A from TMEM (written by tcgen05.st from registers).
#include "../paper_2605_13928_b200/csrc/tc_common.cuh"
#include <cuda_fp16.h>
#include <cstdio>
#include <vector>
using namespace scb;
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
               "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
               "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// A [128][64] fp16 row-major in global; B [128][64] fp16 (K-major) -> smem SW128 (one 128B row per key)
__global__ void k_mma_tmemA(const __half* a, const __half* b, float* d, uint32_t idesc, int reps, long long* cyc) {
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64;
    int chunk = k / 8, w = k % 8;
    Bs[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[r * 64 + k];
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&slot);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, row = 32 * w + l;
  // A row -> 32 u32 columns at tmem col 128..159
  uint32_t ar[32];
  for (int j = 0; j < 32; ++j) {
    __half2 h2 = __halves2half2(a[row * 64 + 2 * j], a[row * 64 + 2 * j + 1]);
    ar[j] = *reinterpret_cast<uint32_t*>(&h2);
  }
  tmem_st32(tm + ((32 * w) << 16) + 128, ar);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int rep = 0; rep < reps; ++rep)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t db = tc::smem_desc_sw128(tc::smem_u32(Bs) + kk * 32, 16, 1024);
        uint32_t acc = (kk > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm), "r"(tm + 128 + kk * 8),
                     "l"(db), "r"(idesc), "r"(acc));
      }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  tc::tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tc::tmem_ld32(tm + ((32 * w) << 16) + c * 32, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[row * 128 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tm);
}
// same with A from smem (SW128 K-major) for timing comparison
__global__ void k_mma_smemA(const __half* a, const __half* b, float* d, uint32_t idesc, int reps, long long* cyc) {
  __shared__ __align__(1024) __half As[128 * 64];
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64;
    int chunk = k / 8, w = k % 8;
    Bs[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[r * 64 + k];
    As[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&slot);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int rep = 0; rep < reps; ++rep)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t da = tc::smem_desc_sw128(tc::smem_u32(As) + kk * 32, 16, 1024);
        uint64_t db = tc::smem_desc_sw128(tc::smem_u32(Bs) + kk * 32, 16, 1024);
        uint32_t acc = (kk > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm), "l"(da), "l"(db),
                     "r"(idesc), "r"(acc));
      }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tm);
}
__global__ void k_mma_variant(const __half* a, const __half* b, int reps, int commit_every, int alt_acc, long long* cyc) {
  __shared__ __align__(1024) __half As[128 * 64];
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t bar[5];
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64;
    int chunk = k / 8, w = k % 8;
    Bs[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[r * 64 + k];
    As[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { for (int i = 0; i < 5; ++i) tc::mbar_init(&bar[i], 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int nc = 0;
    for (int rep = 0; rep < reps; ++rep) {
      const uint32_t d = alt_acc ? tm + (rep & 3) * 128 : tm;
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t da = tc::smem_desc_sw128(tc::smem_u32(As) + kk * 32, 16, 1024);
        uint64_t db = tc::smem_desc_sw128(tc::smem_u32(Bs) + kk * 32, 16, 1024);
        uint32_t acc = (kk > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(da), "l"(db),
                     "r"(idesc), "r"(acc));
      }
      if (commit_every && (rep % commit_every) == commit_every - 1) { tc::mma_commit(&bar[nc % 4]); ++nc; }
    }
    tc::mma_commit(&bar[4]);
  }
  tc::mbar_wait(&bar[4], 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tm);
}

// two issuing threads (warp 0 lane 0: even reps, warp 1 lane 0: odd reps), each commits per rep
__global__ void k_mma_two_issuers(const __half* a, const __half* b, int reps, long long* cyc) {
  __shared__ __align__(1024) __half As[128 * 64];
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t bar[3];
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64;
    int chunk = k / 8, w = k % 8;
    Bs[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[r * 64 + k];
    As[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) tc::mbar_init(&bar[i], 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0 && w < 2) {
    for (int rep = w; rep < reps; rep += 2) {
      const uint32_t d = tm + (rep & 3) * 128;
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t da = tc::smem_desc_sw128(tc::smem_u32(As) + kk * 32, 16, 1024);
        uint64_t db = tc::smem_desc_sw128(tc::smem_u32(Bs) + kk * 32, 16, 1024);
        uint32_t acc = (kk > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(da), "l"(db),
                     "r"(idesc), "r"(acc));
      }
      tc::mma_commit(&bar[2]);  // dummy per-rep commit (barrier count 1: phases just flip)
    }
    tc::mma_commit(&bar[w]);
  }
  if (threadIdx.x == 0) { tc::mbar_wait(&bar[0], 0); tc::mbar_wait(&bar[1], 0); }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tm);
}

int main() {
  std::vector<__half> ha(128 * 64), hb(128 * 64);
  std::vector<float> fa(128 * 64), fb(128 * 64);
  for (int i = 0; i < 128 * 64; ++i) {
    fa[i] = (float)((i * 7) % 11 - 5) * 0.25f; fb[i] = (float)((i * 3) % 13 - 6) * 0.5f;
    ha[i] = __float2half(fa[i]); hb[i] = __float2half(fb[i]);
  }
  __half *da, *db; float* dd; long long* dc;
  cudaMalloc(&da, 16384); cudaMalloc(&db, 16384); cudaMalloc(&dd, 128 * 128 * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(da, ha.data(), 16384, cudaMemcpyHostToDevice); cudaMemcpy(db, hb.data(), 16384, cudaMemcpyHostToDevice);
  uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  k_mma_tmemA<<<1, 128>>>(da, db, dd, idesc, 1, dc);
  printf("tmemA: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> hd(128 * 128);
  cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0; double me = 0;
  for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
    double r = 0; for (int k = 0; k < 64; ++k) r += (double)fa[i * 64 + k] * fb[j * 64 + k];
    double e = fabs(r - hd[i * 128 + j]); me = fmax(me, e); if (e > 1e-2) { if (bad < 4) printf(" (%d,%d) %g vs %g\n", i, j, hd[i*128+j], r); ++bad; }
  }
  printf("tmemA bad=%d maxerr=%g\n", bad, me);
  long long cyc;
  for (int reps : {64, 256}) {
    k_mma_tmemA<<<1, 128>>>(da, db, dd, idesc, reps, dc); cudaDeviceSynchronize(); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("tmemA reps %d: %.1f cycles per 128x128x16 MMA\n", reps, (double)cyc / (4.0 * reps));
    k_mma_smemA<<<1, 128>>>(da, db, dd, idesc, reps, dc); cudaDeviceSynchronize(); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("smemA reps %d: %.1f cycles per 128x128x16 MMA\n", reps, (double)cyc / (4.0 * reps));
  }
  for (int ce : {0, 1, 2}) for (int alt : {0, 1}) {
    k_mma_variant<<<1, 128>>>(da, db, 256, ce, alt, dc); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("variant commit_every=%d alt_acc=%d: %.1f cycles/MMA (%s)\n", ce, alt, (double)cyc / (4.0 * 256), cudaGetErrorString(e));
  }
  k_mma_two_issuers<<<1, 128>>>(da, db, 256, dc); { cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("two issuers, commit per 4 MMAs each: %.1f cycles/MMA (%s)\n", (double)cyc / (4.0 * 256), cudaGetErrorString(e)); }
  for (int ce : {4, 8}) { k_mma_variant<<<1, 128>>>(da, db, 256, ce, 1, dc); cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost); printf("variant commit_every=%d reps: %.1f cycles/MMA\n", ce, (double)cyc / (4.0 * 256)); }
  uint32_t idesc256 = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  (void)idesc256;
  return 0;
}

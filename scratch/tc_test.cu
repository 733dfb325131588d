// Minimal tcgen05 / TMA probes (debug harness).
#include "../paper_2605_13928_b200/csrc/tc_common.cuh"
#include <cstdio>
#include <vector>
using namespace scb;
// 1) TMA box load -> dump smem bytes
__global__ void k_tma(const __grid_constant__ CUtensorMap m, float* out) {
  __shared__ __align__(1024) float buf[32 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { tc::mbar_arrive_expect_tx(&bar, 4096); tc::tma_load_2d(buf, &m, &bar, 0, 0); }
  tc::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = buf[i];
}
// 2) single MMA M=128 N=128 K=8 (tf32), operands filled by threads in canonical K-major SW128 layout
//    A[m][k] = a[m*8+k], B[n][k] = b[n*8+k]; 128-byte rows hold 32 K-elements; we use k<8 only.
template <int MN>
__global__ void k_mma(const float* a, const float* b, float* d, uint32_t idesc) {
  __shared__ __align__(1024) float As[128 * 32];
  __shared__ __align__(1024) float Bs[128 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) { As[i] = 0; Bs[i] = 0; }
  __syncthreads();
  if (!MN) {
    // K-major SW128: row r (M index) at byte r*128; 16B chunk c of the row swizzled: c ^ (r%8)
    for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
      int r = e / 8, k = e % 8;
      int chunk = k / 4, w = k % 4;
      int sw = chunk ^ (r % 8);
      As[r * 32 + sw * 4 + w] = a[r * 8 + k];
      Bs[r * 32 + sw * 4 + w] = b[r * 8 + k];
    }
  } else if (MN == 2) {
    // MN-major SW128_BASE32B: 128B rows (32 MN elems) per K row; 32B chunk c -> c ^ (k%4)
    for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
      int m = e / 8, k = e % 8;
      int chunk = m / 32, mm = m % 32;
      int c32 = mm / 8, w = mm % 8;
      int sw = c32 ^ (k % 4);
      As[chunk * 1024 + k * 32 + sw * 8 + w] = a[m * 8 + k];
      Bs[chunk * 1024 + k * 32 + sw * 8 + w] = b[m * 8 + k];
    }
  } else {
    // MN-major SW128: [4 chunks of 32 MN][8 K rows] each row 128B = 32 MN elems; chunk stride 4096B
    for (int e = threadIdx.x; e < 128 * 8; e += blockDim.x) {
      int m = e / 8, k = e % 8;
      int chunk = m / 32, mm = m % 32;
      int c16 = mm / 4, w = mm % 4;
      int sw = c16 ^ (k % 8);
      As[chunk * 1024 + k * 32 + sw * 4 + w] = a[m * 8 + k];
      Bs[chunk * 1024 + k * 32 + sw * 4 + w] = b[m * 8 + k];
    }
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<128>(&slot);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  uint32_t tm = slot;
  if (threadIdx.x == 0) {
    uint64_t da = MN ? tc::smem_desc_sw128(tc::smem_u32(As), 4096, 1024) : tc::smem_desc_sw128(tc::smem_u32(As), 16, 1024);
    uint64_t db = MN ? tc::smem_desc_sw128(tc::smem_u32(Bs), 4096, 1024) : tc::smem_desc_sw128(tc::smem_u32(Bs), 16, 1024);
    if (MN == 2) {
      da = tc::smem_desc_sw128(tc::smem_u32(As), 4096, 512); db = tc::smem_desc_sw128(tc::smem_u32(Bs), 4096, 512);
      da = (da & ~(7ull << 61)) | (1ull << 61); db = (db & ~(7ull << 61)) | (1ull << 61);
    }
    tc::mma_tf32(tm, da, db, idesc, 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tc::tmem_ld32(tm + ((32 * w) << 16) + c * 32, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[(32 * w + l) * 128 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<128>(tm);
}
int main() {
  float *dz, *dout;
  cudaMalloc(&dz, 64 * 64 * 4); cudaMalloc(&dout, 128 * 128 * 4);
  std::vector<float> hz(64 * 64);
  for (int i = 0; i < 64 * 64; ++i) hz[i] = i;
  cudaMemcpy(dz, hz.data(), hz.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  int rc = make_tmap_2d_f32(&m, dz, 64, 64, 64, 32, 32);
  printf("tmap rc %d %s\n", rc, scb_last_error());
  k_tma<<<1, 128>>>(m, dout);
  cudaError_t e = cudaDeviceSynchronize(); printf("tma: %s\n", cudaGetErrorString(e));
  std::vector<float> ho(128 * 128);
  cudaMemcpy(ho.data(), dout, 1024 * 4, cudaMemcpyDeviceToHost);
  printf("smem row0:"); for (int i = 0; i < 32; ++i) printf(" %g", ho[i]); printf("\nsmem row1:");
  for (int i = 32; i < 64; ++i) printf(" %g", ho[i]); printf("\n");
  // MMA tests
  std::vector<float> ha(128 * 8), hb(128 * 8);
  for (int i = 0; i < 128 * 8; ++i) { ha[i] = (i % 7) - 3; hb[i] = (i % 5) - 2; }
  float *da, *db; cudaMalloc(&da, 4096 * 4); cudaMalloc(&db, 4096 * 4);
  cudaMemcpy(da, ha.data(), 4096, cudaMemcpyHostToDevice); cudaMemcpy(db, hb.data(), 4096, cudaMemcpyHostToDevice);
  for (int mn = 0; mn < 3; ++mn) {
    uint32_t id = tc::idesc_tf32(128, 128, mn > 0, mn > 0);
    if (mn == 2) k_mma<2><<<1, 128>>>(da, db, dout, id); else if (mn) k_mma<1><<<1, 128>>>(da, db, dout, id); else k_mma<0><<<1, 128>>>(da, db, dout, id);
    e = cudaDeviceSynchronize(); printf("mma mn=%d: %s\n", mn, cudaGetErrorString(e));
    cudaMemcpy(ho.data(), dout, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    int bad = 0; double maxe = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
      double ref = 0; for (int k = 0; k < 8; ++k) ref += ha[i * 8 + k] * hb[j * 8 + k];
      double err = fabs(ref - ho[i * 128 + j]); if (err > 1e-3) { if (bad < 5) printf("  (%d,%d) got %g ref %g\n", i, j, ho[i*128+j], ref); ++bad; } maxe = fmax(maxe, err);
    }
    printf("mma mn=%d bad=%d maxerr=%g  d[0..4]= %g %g %g %g\n", mn, bad, maxe, ho[0], ho[1], ho[2], ho[3]);
  }
  return 0;
}

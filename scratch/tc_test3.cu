// Probes: (1) TMEM layout of an F16 accumulator (c_format F16); (2) tcgen05.ld bandwidth.
#include "../paper_2605_13928_b200/csrc/tc_common.cuh"
#include <cuda_fp16.h>
#include <cstdio>
#include <vector>
using namespace scb;

__global__ void k_f16acc(const __half* a, const __half* b, uint32_t* d, uint32_t idesc) {
  __shared__ __align__(1024) __half As[128 * 64];
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64, chunk = k / 8, w = k % 8;
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
  const int w = threadIdx.x / 32, l = threadIdx.x % 32, row = 32 * w + l;
  // poison 256 columns
  {
    uint32_t z[32];
    for (int j = 0; j < 32; ++j) z[j] = 0xDEADBEEFu;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + ((32 * w) << 16) + c * 32),
                   "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]),
                   "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]), "r"(z[16]),
                   "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]), "r"(z[22]), "r"(z[23]), "r"(z[24]),
                   "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]), "r"(z[29]), "r"(z[30]), "r"(z[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
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
  tc::tc_fence_after();
  for (int c = 0; c < 8; ++c) {
    uint32_t r[32];
    tc::tmem_ld32(tm + ((32 * w) << 16) + c * 32, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) d[row * 256 + c * 32 + j] = r[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tm);
}

template <int L>
__global__ void k_ldbw(int iters, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  const int w = threadIdx.x / 32, q = w & 3;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[L][32];
#pragma unroll
    for (int u = 0; u < L; ++u) tc::tmem_ld32(tm + ((32 * q) << 16) + ((w >> 2) * L + u) * 32 % 512, r[u]);
    tc::tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < L; ++u)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[u][j];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  sink[threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tm);
}


// ping-pong: issuers (warp0/warp1 lane 0, unit parity) x epilogue warps 2..9 (arrive immediately
// or after TMEM loads); TMEM ring NBUF x 2 qtiles x N cols; per-qtile or per-unit t_full barriers.
template <int N, int NBUF, bool PER_Q, bool LOAD>
__global__ void k_pingpong(const __half* a, const __half* b, int units, long long* cyc, uint32_t* sink) {
  __shared__ __align__(1024) __half As[1][128 * 64];
  __shared__ __align__(1024) __half Bs[128 * 64];
  __shared__ uint64_t t_full[2 * NBUF], t_empty[2 * NBUF], done[2];
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64, chunk = k / 8, w = k % 8;
    Bs[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[r * 64 + k];
    As[0][r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];

  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NBUF; ++i) { tc::mbar_init(&t_full[i], 1); tc::mbar_init(&t_empty[i], PER_Q ? 4 : 8); }
    tc::mbar_init(&done[0], 1); tc::mbar_init(&done[1], 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  long long t0 = clock64();
  uint32_t acc = 0;
  if (warp < 2) {
    if (lane == 0) {
      const int p = warp;
      for (int u = 0; u < units; ++u) {
        if ((u & 1) != p) continue;
        const int buf = u % NBUF;
        for (int t = 0; t < 2; ++t) {
          const int bi = PER_Q ? buf * 2 + t : buf * 2;
          if (PER_Q || t == 0) tc::mbar_wait(&t_empty[bi], ((u / NBUF) & 1) ^ 1);
          tc::tc_fence_after();
          const uint32_t d = tm + buf * (2 * N) + t * N;
          for (int kk = 0; kk < 4; ++kk) {
            uint64_t da = tc::smem_desc_sw128(tc::smem_u32(As[0]) + kk * 32, 16, 1024);
            uint64_t db = tc::smem_desc_sw128(tc::smem_u32(Bs) + kk * 32, 16, 1024);
            uint32_t ac = (kk > 0) ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(da), "l"(db),
                         "r"(idesc), "r"(ac));
          }
          if (PER_Q || t == 1) tc::mma_commit(&t_full[bi]);
        }
      }
      tc::mma_commit(&done[p]);
    }
  } else {
    const int e = warp - 2, q = warp & 3, t = e >> 2;
    for (int u = 0; u < units; ++u) {
      const int buf = u % NBUF;
      const int bi = PER_Q ? buf * 2 + t : buf * 2;
      tc::mbar_wait(&t_full[bi], (u / NBUF) & 1);
      tc::tc_fence_after();
      if (LOAD) {
        for (int c = 0; c < N / 32; ++c) {
          uint32_t r[32];
          tc::tmem_ld32(tm + ((32 * q) << 16) + buf * (2 * N) + t * N + c * 32, r);
          tc::tmem_ld_wait();
          for (int j = 0; j < 32; ++j) acc ^= r[j];
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&t_empty[bi]);
    }
  }
  if (threadIdx.x == 0) { tc::mbar_wait(&done[0], 0); tc::mbar_wait(&done[1], 0); }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  sink[threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tm);
}

// smem-operand pressure probe: 2 issuers, NST distinct B stages, distinct A per qtile (SS) or
// A from TMEM (TS); epilogue arrives immediately.  unit = 2 qtiles x 4 MMAs (128xNx16).
template <int N, bool TS, int NST, bool WRITER = false>
__global__ void k_ops(const __half* a, const __half* b, int units, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __half* As = reinterpret_cast<__half*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));  // [2][128*64]
  __half* Bs = As + 2 * 128 * 64;  // [NST][N*64]
  __shared__ uint64_t t_full[4], t_empty[4], done[2];
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, k = e % 64, chunk = k / 8, w = k % 8;
    As[r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];
    As[128 * 64 + r * 64 + ((chunk ^ (r % 8)) * 8) + w] = a[r * 64 + k];
  }
  for (int st = 0; st < NST; ++st)
    for (int e = threadIdx.x; e < N * 64; e += blockDim.x) {
      int r = e / 64, k = e % 64, chunk = k / 8, w = k % 8;
      Bs[st * N * 64 + r * 64 + ((chunk ^ (r % 8)) * 8) + w] = b[(r % 128) * 64 + k];
    }
  tc::fence_proxy_async_smem();
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) { tc::mbar_init(&t_full[i], 1); tc::mbar_init(&t_empty[i], 4); }
    tc::mbar_init(&done[0], 1); tc::mbar_init(&done[1], 1);
    tc::fence_barrier_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr uint32_t ACOL = (4 * N + 31) / 32 * 32;  // A in TMEM after the accumulators (2 qtiles x 32 cols)
  if (TS && warp < 4) {  // A rows -> TMEM (fp16 pairs packed in 32-bit columns)
    const int row = 32 * warp + lane;
    for (int t = 0; t < 2; ++t) {
      uint32_t ar[32];
      for (int j = 0; j < 32; ++j) {
        __half2 h2 = __halves2half2(a[row * 64 + 2 * j], a[row * 64 + 2 * j + 1]);
        ar[j] = *reinterpret_cast<uint32_t*>(&h2);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + ((32 * warp) << 16) + ACOL + t * 32),
                   "r"(ar[0]), "r"(ar[1]), "r"(ar[2]), "r"(ar[3]), "r"(ar[4]), "r"(ar[5]), "r"(ar[6]), "r"(ar[7]), "r"(ar[8]),
                   "r"(ar[9]), "r"(ar[10]), "r"(ar[11]), "r"(ar[12]), "r"(ar[13]), "r"(ar[14]), "r"(ar[15]), "r"(ar[16]),
                   "r"(ar[17]), "r"(ar[18]), "r"(ar[19]), "r"(ar[20]), "r"(ar[21]), "r"(ar[22]), "r"(ar[23]), "r"(ar[24]),
                   "r"(ar[25]), "r"(ar[26]), "r"(ar[27]), "r"(ar[28]), "r"(ar[29]), "r"(ar[30]), "r"(ar[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (warp < 2) {
    if (lane == 0) {
      const int p = warp;
      for (int u = 0; u < units; ++u) {
        if ((u & 1) != p) continue;
        const int buf = u & 1;
        const uint32_t bb = tc::smem_u32(Bs) + (u % NST) * N * 128;
        for (int t = 0; t < 2; ++t) {
          tc::mbar_wait(&t_empty[buf * 2 + t], ((u >> 1) & 1) ^ 1);
          tc::tc_fence_after();
          const uint32_t d = tm + buf * (2 * N) + t * N;
          for (int kk = 0; kk < 4; ++kk) {
            uint64_t db = tc::smem_desc_sw128(bb + kk * 32, 16, 1024);
            uint32_t ac = (kk > 0) ? 1u : 0u;
            if (TS) {
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                           "r"(tm + ACOL + t * 32 + kk * 8), "l"(db), "r"(idesc), "r"(ac));
            } else {
              uint64_t da = tc::smem_desc_sw128(tc::smem_u32(As + t * 128 * 64) + kk * 32, 16, 1024);
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(da), "l"(db),
                           "r"(idesc), "r"(ac));
            }
          }
          tc::mma_commit(&t_full[buf * 2 + t]);
        }
      }
      tc::mma_commit(&done[p]);
    }
  } else if (WRITER && warp >= 10) {
    // simulated TMA traffic: N * 128 bytes written per unit (one key tile), 2 warps
    float4* wbuf = reinterpret_cast<float4*>(Bs + NST * N * 64);  // scratch after the B stages
    const int wl = (warp - 10) * 32 + lane;
    for (int u = 0; u < units; ++u) {
      for (int i = wl; i < N * 8; i += 64) wbuf[i & 1023] = make_float4((float)u, 0.f, 0.f, 0.f);
      __syncwarp();
    }
  } else if (warp < 10) {
    const int e = warp - 2, t = e >> 2;
    for (int u = 0; u < units; ++u) {
      const int buf = u & 1;
      tc::mbar_wait(&t_full[buf * 2 + t], (u >> 1) & 1);
      tc::tc_fence_after();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&t_empty[buf * 2 + t]);
    }
  }
  if (threadIdx.x == 0) { tc::mbar_wait(&done[0], 0); tc::mbar_wait(&done[1], 0); }
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
  __half *da, *db; uint32_t* dd; long long* dc; uint32_t* sink;
  cudaMalloc(&da, 16384); cudaMalloc(&db, 16384); cudaMalloc(&dd, 128 * 256 * 4); cudaMalloc(&dc, 8); cudaMalloc(&sink, 4096 * 4);
  cudaMemcpy(da, ha.data(), 16384, cudaMemcpyHostToDevice); cudaMemcpy(db, hb.data(), 16384, cudaMemcpyHostToDevice);
  for (int cf : {1, 0}) {
    uint32_t idesc = ((uint32_t)cf << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    k_f16acc<<<1, 128>>>(da, db, dd, idesc);
    printf("c_format=%d: %s\n", cf, cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<uint32_t> hd(128 * 256);
    cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
    for (int i : {0, 1, 33}) {
      printf(" row %d ref:", i);
      for (int j = 0; j < 6; ++j) { double r = 0; for (int k = 0; k < 64; ++k) r += (double)fa[i * 64 + k] * fb[j * 64 + k]; printf(" %g", r); }
      printf("\n   words:");
      for (int j = 0; j < 6; ++j) printf(" %08x", hd[i * 256 + j]);
      printf("  | col64..66: %08x %08x %08x | col127,128: %08x %08x\n", hd[i * 256 + 64], hd[i * 256 + 65], hd[i * 256 + 66], hd[i * 256 + 127], hd[i * 256 + 128]);
      printf("   as f32:"); for (int j = 0; j < 6; ++j) { float f; memcpy(&f, &hd[i * 256 + j], 4); printf(" %g", f); }
      printf("\n   as 2xf16:"); for (int j = 0; j < 3; ++j) { __half_raw lo, hi; lo.x = hd[i*256+j] & 0xffff; hi.x = hd[i*256+j] >> 16; printf(" (%g,%g)", __half2float(__half(lo)), __half2float(__half(hi))); }
      printf("\n");
    }
  }
  long long cyc;
  for (int nw : {4, 8, 16}) {
    int iters = 2000;
    k_ldbw<1><<<1, nw * 32>>>(iters, dc, sink); cudaDeviceSynchronize(); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d L=1: %.1f B/cycle\n", nw, (double)nw * iters * 1 * 4096 / cyc);
    k_ldbw<2><<<1, nw * 32>>>(iters, dc, sink); cudaDeviceSynchronize(); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d L=2: %.1f B/cycle\n", nw, (double)nw * iters * 2 * 4096 / cyc);
    k_ldbw<4><<<1, nw * 32>>>(iters, dc, sink); cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d L=4: %.1f B/cycle (%s)\n", nw, (double)nw * iters * 4 * 4096 / cyc, cudaGetErrorString(e));
  }

  {
    const int units = 4000;
    auto run = [&](auto kern, const char* name, int n) {
      kern<<<1, 320>>>(da, db, units, dc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      // cycles per 128x128x16-equivalent MMA: unit = 2 qtiles x 4 MMAs of N cols
      printf("%-36s %.1f cycles/unit, %.1f cycles per 128-col MMA (%s)\n", name, (double)c / units,
             (double)c / units / 8.0 * 128.0 / n, cudaGetErrorString(e));
    };
    run(k_pingpong<128, 2, true, false>, "N128 NBUF2 perQ noload", 128);
    run(k_pingpong<128, 2, false, false>, "N128 NBUF2 perUnit noload", 128);
    run(k_pingpong<64, 4, true, false>, "N64 NBUF4 perQ noload", 64);
    run(k_pingpong<64, 4, false, false>, "N64 NBUF4 perUnit noload", 64);
    run(k_pingpong<128, 2, true, true>, "N128 NBUF2 perQ load", 128);
    run(k_pingpong<128, 2, false, true>, "N128 NBUF2 perUnit load", 128);
    run(k_pingpong<64, 4, true, true>, "N64 NBUF4 perQ load", 64);
    run(k_pingpong<64, 4, false, true>, "N64 NBUF4 perUnit load", 64);
  }

  {
    const int units = 4000;
    auto run2 = [&](auto kern, const char* name, int n, int nst, int grid = 1, int threads = 320) {
      int sm = 1024 + 2 * 128 * 64 * 2 + nst * n * 64 * 2 + 16384;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      kern<<<grid, threads, sm>>>(da, db, units, dc);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      printf("%-30s %.1f cycles/unit, %.1f cycles per 128x128x16-equiv MMA (%s)\n", name, (double)c / units,
             (double)c / units / 8.0 * 128.0 / n, cudaGetErrorString(e));
    };
    run2(k_ops<128, false, 6>, "SS N128 6st g148", 128, 6, 148);
    run2(k_ops<128, false, 6, true>, "SS N128 6st g148 +writer", 128, 6, 148, 384);
    run2(k_ops<96, true, 6>, "TS N96 6st g148", 96, 6, 148);
    run2(k_ops<96, true, 6, true>, "TS N96 6st g148 +writer", 96, 6, 148, 384);
    run2(k_ops<96, false, 6, true>, "SS N96 6st g148 +writer", 96, 6, 148, 384);
  }
  return 0;
}

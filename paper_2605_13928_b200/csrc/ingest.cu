// Ingest: MatrixMarket coordinate text -> COO -> CSR on the device.
//
// The paper's GPU pipeline spends its first ~60 s CPU-bound loading the count matrix
// (PAPER.md:84,111).  Here the host only reads the file bytes and the MatrixMarket header;
// the data lines are parsed on the GPU and the CSR over cells is built there.
//
//   count    CTA per 4 KiB chunk, 16-byte loads: '\n' count per chunk             -- reads the text
//   parse    same chunking; the thread that owns a line's leading '\n' (or the data start)
//            parses that line ("row col [value]", 1-based) into entry #(global line index)
//                                                                                    -- reads it again
//   csr      sortedness check (one pass); cell-major sorted input (10x writes column-major
//            by barcode, genes ascending) -> indptr from run boundaries, indices/data copied;
//            otherwise counting scatter (atomic cursors) + per-row bitonic sort in smem.
//            Duplicate (cell, gene) entries are rejected (scipy would sum them).
// Parity: bit-exact against scipy.io.mmread for integer/pattern fields and for real fields
// whose decimal mantissa < 2^53 with |exponent| <= 22 (one correctly rounded f64 product,
// then f32 as scipy's astype(float32)); other real literals use pow() and may differ by an
// f64 ulp before the f32 rounding.
#include "common.cuh"
#include "scan.cuh"
#include <algorithm>

namespace scb {

constexpr int kIngThreads = 256;
constexpr int kChunk = kIngThreads * 16;  // bytes per CTA

__device__ __forceinline__ bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }

// number of line starts owned by each chunk: position `off` (first data line) and every
// p + 1 with text[p] == '\n', off <= p, p + 1 < n
__global__ void __launch_bounds__(kIngThreads)
mtx_count_kernel(const char* __restrict__ text, int64_t off, int64_t n, int64_t* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * 16;
  int c = 0;
  if (base < n) {
    const uint4 w = *reinterpret_cast<const uint4*>(text + base);
    const char* b = reinterpret_cast<const char*>(&w);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t p = base + k;
      c += (p >= off && p + 1 < n && b[k] == '\n') ? 1 : 0;
    }
    if (off >= base && off < base + 16 && off < n) c += 1;
  }
  __shared__ int red[kIngThreads / 32];
  int v = warp_sum(c);
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kIngThreads / 32; ++i) t += red[i];
    counts[blockIdx.x] = t;
  }
}

__device__ __forceinline__ bool parse_uint(const char* t, int64_t& p, int64_t n, int64_t& out) {
  int64_t v = 0;
  int nd = 0;
  while (p < n) {
    const char ch = t[p];
    if (ch < '0' || ch > '9') break;
    if (nd < 18) v = v * 10 + (ch - '0');
    ++nd;
    ++p;
  }
  out = v;
  return nd > 0 && nd <= 18;
}

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
__device__ __forceinline__ double pow10_exact(int e) { return kPow10[e]; }

// field: 0 integer, 1 real, 2 pattern
__device__ bool parse_line(const char* __restrict__ t, int64_t p, int64_t n, int field, int64_t& r, int64_t& c,
                           float& v) {
  while (p < n && is_ws(t[p])) ++p;
  if (!parse_uint(t, p, n, r)) return false;
  if (p >= n || !is_ws(t[p])) return false;
  while (p < n && is_ws(t[p])) ++p;
  if (!parse_uint(t, p, n, c)) return false;
  if (field == 2) {
    v = 1.0f;
  } else {
    if (p >= n || !is_ws(t[p])) return false;
    while (p < n && is_ws(t[p])) ++p;
    bool neg = false;
    if (p < n && (t[p] == '-' || t[p] == '+')) neg = (t[p++] == '-');
    uint64_t m = 0;
    int nd = 0, dexp = 0;
    bool lossy = false;
    while (p < n && t[p] >= '0' && t[p] <= '9') {
      if (m < 100000000000000000ull) m = m * 10 + (t[p] - '0');
      else { ++dexp; lossy = true; }
      ++nd;
      ++p;
    }
    if (field == 1 && p < n && t[p] == '.') {
      ++p;
      while (p < n && t[p] >= '0' && t[p] <= '9') {
        if (m < 100000000000000000ull) { m = m * 10 + (t[p] - '0'); --dexp; }
        else lossy = true;
        ++nd;
        ++p;
      }
    }
    if (nd == 0) return false;
    if (field == 1 && p < n && (t[p] == 'e' || t[p] == 'E')) {
      ++p;
      bool eneg = false;
      if (p < n && (t[p] == '-' || t[p] == '+')) eneg = (t[p++] == '-');
      int64_t ev;
      if (!parse_uint(t, p, n, ev) || ev > 100000) return false;
      dexp += eneg ? -(int)ev : (int)ev;
    }
    double d;
    if (!lossy && m < (1ull << 53) && dexp >= -22 && dexp <= 22)
      d = dexp >= 0 ? (double)m * pow10_exact(dexp) : (double)m / pow10_exact(-dexp);
    else
      d = (double)m * pow(10.0, (double)dexp);
    v = (float)(neg ? -d : d);
  }
  while (p < n && is_ws(t[p])) ++p;
  return p >= n || t[p] == '\n';
}

// The CTA stages its chunk plus a kHalo-byte tail (lines that start in the chunk and end past
// it) in shared memory with 16-byte loads; each thread then parses the lines it owns from smem.
// A line longer than the staged window is parsed from global memory (rare).
constexpr int kHalo = 512;
__global__ void __launch_bounds__(kIngThreads)
mtx_parse_kernel(const char* __restrict__ text, int64_t off, int64_t n, const int64_t* __restrict__ base_idx,
                 int field, int64_t nnz, int64_t n_file_rows, int64_t n_file_cols, int32_t* __restrict__ row,
                 int32_t* __restrict__ col, float* __restrict__ val, int* __restrict__ flag) {
  __shared__ __align__(16) char stage[kChunk + kHalo];
  const int64_t cbase = (int64_t)blockIdx.x * kChunk;
  for (int i = threadIdx.x; i < (kChunk + kHalo) / 16; i += blockDim.x) {
    const int64_t p = cbase + (int64_t)i * 16;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (p < n) w = *reinterpret_cast<const uint4*>(text + p);
    reinterpret_cast<uint4*>(stage)[i] = w;
  }
  __syncthreads();
  const int64_t base = cbase + (int64_t)threadIdx.x * 16;
  int c = 0;
  uint32_t starts = 0;  // bit k: a line starts at base + k + 1 (bit 16: at `off`)
  if (base < n) {
    const char* b = stage + threadIdx.x * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t p = base + k;
      if (p >= off && p + 1 < n && b[k] == '\n') { starts |= 1u << k; ++c; }
    }
    if (off >= base && off < base + 16 && off < n) { starts |= 1u << 16; ++c; }
  }
  // block-exclusive prefix of c (line-index order == byte order; the `off` start precedes
  // any newline-owned start inside the same 16 bytes since off <= that newline)
  __shared__ int wsum[kIngThreads / 32];
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane_id() >= o) incl += t;
  }
  if (lane_id() == 31) wsum[warp_id()] = incl;
  __syncthreads();
  int wpre = 0;
  for (int i = 0; i < warp_id(); ++i) wpre += wsum[i];
  int64_t idx = base_idx[blockIdx.x] + wpre + incl - c;
  const int64_t win_end = min(n, cbase + kChunk + kHalo);
  bool bad = false;
  auto emit = [&](int64_t p) {
    if (idx >= nnz) { bad = true; return; }
    int64_t r, cc;
    float v;
    // parse from the staged window when the line ends inside it, else from global memory
    bool ok;
    int64_t q = p;
    while (q < win_end && stage[q - cbase] != '\n') ++q;
    if (q < win_end || win_end == n)
      ok = parse_line(stage, p - cbase, win_end - cbase, field, r, cc, v);
    else
      ok = parse_line(text, p, n, field, r, cc, v);
    if (!ok || r < 1 || r > n_file_rows || cc < 1 || cc > n_file_cols) {
      bad = true;
    } else {
      row[idx] = (int32_t)(r - 1);
      col[idx] = (int32_t)(cc - 1);
      val[idx] = v;
    }
    ++idx;
  };
  if (starts >> 16) emit(off);
  uint32_t s = starts & 0xFFFFu;
  while (s) {
    const int k = __ffs(s) - 1;
    s &= s - 1;
    emit(base + k + 1);
  }
  if (bad) atomicOr(flag, 1);
}

// ---------------------------------------------------------------- COO -> CSR
// flags: bit0 major not non-decreasing, bit1 minor not strictly increasing within a major run
// (includes duplicates), bit2 duplicate (major, minor) adjacent
__global__ void coo_check_kernel(const int32_t* __restrict__ major, const int32_t* __restrict__ minor, int64_t nnz,
                                 int* __restrict__ flags) {
  int f = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = major[i - 1], b = major[i];
    if (b < a) f |= 1;
    else if (b == a) {
      if (minor[i] <= minor[i - 1]) f |= 2;
      if (minor[i] == minor[i - 1]) f |= 4;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (lane_id() == 0 && f) atomicOr(flags, f);
}

// sorted input: indptr[m] = first i with major[i] >= m
__global__ void csr_bounds_kernel(const int32_t* __restrict__ major, int64_t nnz, int32_t n_major,
                                  int64_t* __restrict__ indptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t lo = i == 0 ? -1 : major[i - 1];
    const int32_t hi = i == nnz ? n_major - 1 : major[i];
    for (int32_t m = lo + 1; m <= hi; ++m) indptr[m] = i;
    if (i == nnz) indptr[n_major] = nnz;
  }
}

__global__ void coo_hist_kernel(const int32_t* __restrict__ major, int64_t nnz, int64_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t m = major[i];
    // warp-aggregate equal keys (file order is usually clustered by cell)
    const unsigned same = __match_any_sync(__activemask(), m);
    if ((int)(__ffs(same) - 1) == lane_id()) atomicAdd((unsigned long long*)&cnt[m], (unsigned long long)__popc(same));
  }
}

__global__ void coo_scatter_kernel(const int32_t* __restrict__ major, const int32_t* __restrict__ minor,
                                   const float* __restrict__ val, int64_t nnz, const int64_t* __restrict__ indptr,
                                   unsigned long long* __restrict__ cursor, int32_t* __restrict__ indices,
                                   float* __restrict__ data) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t m = major[i];
    const int64_t pos = indptr[m] + (int64_t)atomicAdd(&cursor[m], 1ull);
    indices[pos] = minor[i];
    data[pos] = val[i];
  }
}

// CTA per row: bitonic sort of (minor, value) pairs in smem (rows up to kMaxSortRow), then
// a duplicate check
constexpr int kMaxSortRow = 8192;
__global__ void __launch_bounds__(512)
csr_sort_rows_kernel(const int64_t* __restrict__ indptr, int32_t n_major, int32_t* __restrict__ indices,
                     float* __restrict__ data, int* __restrict__ flags) {
  extern __shared__ int32_t sk[];  // [kMaxSortRow] keys, then [kMaxSortRow] values
  float* sv = reinterpret_cast<float*>(sk + kMaxSortRow);
  for (int32_t r = blockIdx.x; r < n_major; r += gridDim.x) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    const int len = (int)(e - b);
    if (len <= 1) continue;
    if (len > kMaxSortRow) {
      if (threadIdx.x == 0) atomicOr(flags, 8);
      continue;
    }
    int np2 = 1;
    while (np2 < len) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
      sk[i] = i < len ? indices[b + i] : INT32_MAX;
      sv[i] = i < len ? data[b + i] : 0.0f;
    }
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < np2; i += blockDim.x) {
          const int l = i ^ j;
          if (l > i) {
            const bool up = (i & k) == 0;
            const int32_t a = sk[i], c = sk[l];
            if ((a > c) == up) {
              sk[i] = c;
              sk[l] = a;
              const float t = sv[i];
              sv[i] = sv[l];
              sv[l] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    int dup = 0;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      indices[b + i] = sk[i];
      data[b + i] = sv[i];
      if (i > 0 && sk[i] == sk[i - 1]) dup = 1;
    }
    if (__syncthreads_or(dup) && threadIdx.x == 0) atomicOr(flags, 4);
  }
}

}  // namespace scb

using namespace scb;

extern "C" int scb_mtx_parse(scb_ctx* ctx, const char* text, int64_t data_offset, int64_t n_bytes, int32_t field,
                             int64_t nnz, int64_t n_file_rows, int64_t n_file_cols, int32_t* row, int32_t* col,
                             float* val, void* stream) {
  SCB_REQUIRE(ctx && text && row && col && val, SCB_ERR_ARG, "scb_mtx_parse: null argument");
  SCB_REQUIRE(((uintptr_t)text & 15) == 0, SCB_ERR_ARG,
              "scb_mtx_parse: text must be 16-byte aligned and readable up to roundup(n_bytes, 16)");
  SCB_REQUIRE(field >= 0 && field <= 2, SCB_ERR_ARG, "scb_mtx_parse: field must be 0 (integer), 1 (real), 2 (pattern)");
  SCB_REQUIRE(data_offset >= 0 && data_offset <= n_bytes && nnz >= 0, SCB_ERR_ARG, "scb_mtx_parse: bad sizes");
  SCB_REQUIRE(n_file_rows < INT32_MAX && n_file_cols < INT32_MAX, SCB_ERR_UNSUPPORTED,
              "scb_mtx_parse: dimensions must fit int32");
  cudaStream_t s = (cudaStream_t)stream;
  if (nnz == 0) return SCB_OK;
  const int64_t n_chunks = (n_bytes + kChunk - 1) / kChunk;
  SCB_REQUIRE(n_chunks < (1ll << 31), SCB_ERR_UNSUPPORTED, "scb_mtx_parse: text too large");
  void* ws;
  SCB_TRY(ws_get(ctx, 0, (size_t)(n_chunks + 1) * 8 * 2, &ws, s));
  int64_t* counts = (int64_t*)ws;
  int64_t* bases = counts + (n_chunks + 1);
  mtx_count_kernel<<<(unsigned)n_chunks, kIngThreads, 0, s>>>(text, data_offset, n_bytes, counts);
  SCB_LAUNCH_CHECK();
  SCB_TRY(scan_i64(ctx, counts, n_chunks, bases, s));  // bases[n_chunks] = number of lines
  int64_t n_lines = 0;
  SCB_CUDA(cudaMemcpyAsync(&n_lines, bases + n_chunks, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), s));
  SCB_CUDA(cudaStreamSynchronize(s));
  SCB_REQUIRE(n_lines == nnz, SCB_ERR_DATA, "scb_mtx_parse: %lld data lines, header says %lld entries",
              (long long)n_lines, (long long)nnz);
  mtx_parse_kernel<<<(unsigned)n_chunks, kIngThreads, 0, s>>>(text, data_offset, n_bytes, bases, field, nnz,
                                                              n_file_rows, n_file_cols, row, col, val, ctx->d_flag);
  SCB_LAUNCH_CHECK();
  int flag = 0;
  SCB_CUDA(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  SCB_REQUIRE(flag == 0, SCB_ERR_DATA, "scb_mtx_parse: malformed data line or index out of range");
  return SCB_OK;
}

extern "C" int scb_coo_to_csr(scb_ctx* ctx, const int32_t* major, const int32_t* minor, const float* val, int64_t nnz,
                              int32_t n_major, int64_t* indptr, int32_t* indices, float* data, void* stream) {
  SCB_REQUIRE(ctx && major && minor && val && indptr && indices && data, SCB_ERR_ARG, "scb_coo_to_csr: null argument");
  SCB_REQUIRE(n_major >= 0 && nnz >= 0, SCB_ERR_ARG, "scb_coo_to_csr: bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = ctx->num_sms * 8;
  int* flags = ctx->d_flag + 2;
  SCB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  if (nnz > 1) {
    coo_check_kernel<<<grid, 256, 0, s>>>(major, minor, nnz, flags);
    SCB_LAUNCH_CHECK();
  }
  int f = 0;
  SCB_CUDA(cudaMemcpyAsync(&f, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  SCB_REQUIRE(!(f & 4), SCB_ERR_DATA, "scb_coo_to_csr: duplicate (row, column) entries");
  if (f == 0) {  // already in CSR order: boundaries + copies
    csr_bounds_kernel<<<grid, 256, 0, s>>>(major, nnz, n_major, indptr);
    SCB_LAUNCH_CHECK();
    if (nnz) {
      if (indices != minor) SCB_CUDA(cudaMemcpyAsync(indices, minor, nnz * 4, cudaMemcpyDeviceToDevice, s));
      if (data != val) SCB_CUDA(cudaMemcpyAsync(data, val, nnz * 4, cudaMemcpyDeviceToDevice, s));
    }
    return SCB_OK;
  }
  SCB_REQUIRE(indices != minor && data != val, SCB_ERR_ARG, "scb_coo_to_csr: unsorted input cannot be converted in place");
  void* ws;
  SCB_TRY(ws_get(ctx, 1, (size_t)(n_major + 1) * 8 * 2, &ws, s));
  int64_t* cnt = (int64_t*)ws;
  unsigned long long* cursor = (unsigned long long*)(cnt + (n_major + 1));
  SCB_CUDA(cudaMemsetAsync(ws, 0, (size_t)(n_major + 1) * 8 * 2, s));
  coo_hist_kernel<<<grid, 256, 0, s>>>(major, nnz, cnt);
  SCB_LAUNCH_CHECK();
  SCB_TRY(scan_i64(ctx, cnt, n_major, indptr, s));  // indptr[n_major] = nnz
  coo_scatter_kernel<<<grid, 256, 0, s>>>(major, minor, val, nnz, indptr, cursor, indices, data);
  SCB_LAUNCH_CHECK();
  const int sort_smem = kMaxSortRow * 8;
  SCB_CUDA(cudaFuncSetAttribute(csr_sort_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sort_smem));
  csr_sort_rows_kernel<<<ctx->num_sms * 3, 512, sort_smem, s>>>(indptr, n_major, indices, data, flags);
  SCB_LAUNCH_CHECK();
  SCB_CUDA(cudaMemcpyAsync(&f, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  SCB_CUDA(cudaStreamSynchronize(s));
  SCB_REQUIRE(!(f & 8), SCB_ERR_UNSUPPORTED, "scb_coo_to_csr: unsorted row longer than %d entries", kMaxSortRow);
  SCB_REQUIRE(!(f & 4), SCB_ERR_DATA, "scb_coo_to_csr: duplicate (row, column) entries");
  return SCB_OK;
}

// ---------------------------------------------------------------------------- u16 wire decode
// Compact u16 CSR (host->device wire format: uint16 gene indices + uint16 counts, counts >=
// 65535 escaped to a sorted (position, value) table) -> the int32/float32 CSR in HBM.  HBM-bound:
// 4 B read + 8 B written per nonzero; each thread converts 8 nonzeros per iteration (16-byte
// loads of each u16 array, 2 x 16-byte stores of each output array).
namespace scb {
__global__ void __launch_bounds__(256) u16_decode_kernel(const uint4* __restrict__ ind16, const uint4* __restrict__ dat16,
                                                         int64_t n8, int4* __restrict__ ind, float4* __restrict__ dat) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(ind16 + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(dat16 + i));
    ind[2 * i] = make_int4(a.x & 0xffff, a.x >> 16, a.y & 0xffff, a.y >> 16);
    ind[2 * i + 1] = make_int4(a.z & 0xffff, a.z >> 16, a.w & 0xffff, a.w >> 16);
    dat[2 * i] = make_float4((float)(b.x & 0xffff), (float)(b.x >> 16), (float)(b.y & 0xffff), (float)(b.y >> 16));
    dat[2 * i + 1] = make_float4((float)(b.z & 0xffff), (float)(b.z >> 16), (float)(b.w & 0xffff), (float)(b.w >> 16));
  }
}
__global__ void u16_decode_tail_kernel(const uint16_t* __restrict__ ind16, const uint16_t* __restrict__ dat16,
                                       int64_t begin, int64_t nnz, int32_t* __restrict__ ind, float* __restrict__ dat) {
  const int64_t i = begin + threadIdx.x;
  if (i < nnz) {
    ind[i] = ind16[i];
    dat[i] = (float)dat16[i];
  }
}
__global__ void u16_escape_kernel(const int64_t* __restrict__ pos, const float* __restrict__ val, int64_t n,
                                  int64_t nnz, float* __restrict__ dat) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = pos[i];
  if (p >= 0 && p < nnz) dat[p] = val[i];  // out-of-range escapes are ignored (no host sync here)
}
}  // namespace scb

extern "C" int scb_csr_u16_decode(scb_ctx* ctx, const uint16_t* indices16, const uint16_t* data16, int64_t nnz,
                                  const int64_t* esc_pos, const float* esc_val, int64_t n_esc, int32_t* indices,
                                  float* data, void* stream) {
  using namespace scb;
  SCB_REQUIRE(ctx && (nnz == 0 || (indices16 && data16 && indices && data)), SCB_ERR_ARG, "scb_csr_u16_decode: null argument");
  SCB_REQUIRE(n_esc == 0 || (esc_pos && esc_val), SCB_ERR_ARG, "scb_csr_u16_decode: escape table missing");
  SCB_REQUIRE(((uintptr_t)indices16 & 15) == 0 && ((uintptr_t)data16 & 15) == 0 && ((uintptr_t)indices & 15) == 0 &&
                  ((uintptr_t)data & 15) == 0,
              SCB_ERR_ARG, "scb_csr_u16_decode: 16-byte aligned arrays required");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n8 = nnz / 8;
  if (n8 > 0) {
    const int g = (int)std::min<int64_t>((int64_t)ctx->num_sms * 8, (n8 + 255) / 256);
    u16_decode_kernel<<<g, 256, 0, s>>>((const uint4*)indices16, (const uint4*)data16, n8, (int4*)indices, (float4*)data);
    SCB_LAUNCH_CHECK();
  }
  if (nnz > 8 * n8) {
    u16_decode_tail_kernel<<<1, 8, 0, s>>>(indices16, data16, 8 * n8, nnz, indices, data);
    SCB_LAUNCH_CHECK();
  }
  if (n_esc > 0) {
    u16_escape_kernel<<<(unsigned)((n_esc + 255) / 256), 256, 0, s>>>(esc_pos, esc_val, n_esc, nnz, data);
    SCB_LAUNCH_CHECK();
  }
  return SCB_OK;
}

// ------------------------------------------------------------------ f1 wire decode: byte-delta CSR
namespace scb {
// index of position k in a sorted escape-position table (k is known to be present)
__device__ __forceinline__ int64_t esc_find(const int64_t* __restrict__ pos, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (pos[m] < k) lo = m + 1; else hi = m;
  }
  return lo;
}

// warp per row: gene index = previous + 1 + byte delta (255: the delta is in the gene escape
// table), count = byte (255: value in the count escape table).  Windows of 256 elements aligned
// to 4 (elements of neighbouring rows masked) as two 128-element halves; in each half lane L owns
// elements 4L..4L+3 (4-byte loads of both byte streams, one 16-byte store per array, so a warp
// store instruction writes 512 contiguous bytes), a per-lane running sum + a warp scan carries
// the gene index.  The next row's bounds are loaded while the current row is decoded.
#ifndef SCB_D8_HALVES
#define SCB_D8_HALVES 2
#endif
#ifndef SCB_D8_MINB
#define SCB_D8_MINB 6  // 40 registers, 6 blocks per SM: 4.95 vs 5.03 ms at C3 (tools/d8_ab.sh)
#endif
__global__ void __launch_bounds__(256, SCB_D8_MINB) delta8_decode_kernel(const int64_t* __restrict__ indptr, int64_t n_rows,
                                     const uint8_t* __restrict__ dgene, const uint8_t* __restrict__ dcount,
                                     const int64_t* __restrict__ gpos, const int32_t* __restrict__ gval, int64_t n_g,
                                     const int64_t* __restrict__ cpos, const float* __restrict__ cval, int64_t n_c,
                                     int64_t nnz, int32_t* __restrict__ indices, float* __restrict__ data) {
  constexpr int HALVES = SCB_D8_HALVES;
  const int lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id();
  int64_t nb = 0, ne = 0;
  if (r < n_rows) {
    nb = indptr[r];
    ne = indptr[r + 1];
  }
  for (; r < n_rows; r += warps) {
    const int64_t b = nb, e = ne;
    if (r + warps < n_rows) {
      nb = indptr[r + warps];
      ne = indptr[r + warps + 1];
    }
    int carry = -1;
    for (int64_t w0 = b & ~(int64_t)3; w0 < e; w0 += HALVES * 128) {
      uint32_t gw[HALVES], cw[HALVES];
#pragma unroll
      for (int h = 0; h < HALVES; ++h) {
        const int64_t k0 = w0 + 128 * h + 4 * lane;
        gw[h] = 0u;
        cw[h] = 0u;
        if (k0 < e) {
          if (k0 + 4 <= nnz) {
            gw[h] = __ldg(reinterpret_cast<const uint32_t*>(dgene + k0));
            cw[h] = __ldg(reinterpret_cast<const uint32_t*>(dcount + k0));
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (k0 + j < nnz) {
                gw[h] |= (uint32_t)dgene[k0 + j] << (8 * j);
                cw[h] |= (uint32_t)dcount[k0 + j] << (8 * j);
              }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < HALVES; ++h) {
        const int64_t k0 = w0 + 128 * h + 4 * lane;
        // fast lanes: all 4 elements in the row and no escape byte (0xFF) in either word
        const bool full = k0 >= b && k0 + 4 <= e;
        const uint32_t ff = ((~gw[h] - 0x01010101u) & gw[h]) | ((~cw[h] - 0x01010101u) & cw[h]);
        const bool fast = full && (ff & 0x80808080u) == 0u;
        int incl[4];
        float v[4];
        if (fast) {
          const uint32_t d = gw[h];
          incl[0] = (int)(d & 0xFFu) + 1;
          incl[1] = incl[0] + (int)((d >> 8) & 0xFFu) + 1;
          incl[2] = incl[1] + (int)((d >> 16) & 0xFFu) + 1;
          incl[3] = incl[2] + (int)(d >> 24) + 1;
#pragma unroll
          for (int j = 0; j < 4; ++j)  // 2^23 + byte as a float bit pattern, minus 2^23: exact
            v[j] = __uint_as_float(__byte_perm(cw[h], 0x4B000000u, (unsigned)j | 0x7540u)) - 8388608.0f;
        } else {
          int sum = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t k = k0 + j;
            const bool ok = k >= b && k < e;
            const int dg = (int)((gw[h] >> (8 * j)) & 0xFFu);
            int inc = ok ? dg + 1 : 0;
            if (ok && dg == 255) inc = gval[esc_find(gpos, n_g, k)] + 1;
            sum += inc;
            incl[j] = sum;
            const uint32_t c = (cw[h] >> (8 * j)) & 0xFFu;
            v[j] = (float)c;
            if (c == 255u && ok) v[j] = cval[esc_find(cpos, n_c, k)];
          }
        }
        const int sum = incl[3];
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += t;
        }
        const int g0 = carry + x - sum;
        carry += __shfl_sync(0xffffffffu, x, 31);
        if (full) {
          *reinterpret_cast<int4*>(indices + k0) = make_int4(g0 + incl[0], g0 + incl[1], g0 + incl[2], g0 + incl[3]);
          *reinterpret_cast<float4*>(data + k0) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (k0 + j >= b && k0 + j < e) {
              indices[k0 + j] = g0 + incl[j];
              data[k0 + j] = v[j];
            }
        }
      }
    }
  }
}
}  // namespace scb

extern "C" int scb_csr_delta8_decode(scb_ctx* ctx, const int64_t* indptr, int64_t n_rows, const uint8_t* dgene,
                                     const uint8_t* dcount, int64_t nnz, const int64_t* gesc_pos,
                                     const int32_t* gesc_val, int64_t n_gesc, const int64_t* cesc_pos,
                                     const float* cesc_val, int64_t n_cesc, int32_t* indices, float* data,
                                     void* stream) {
  using namespace scb;
  SCB_REQUIRE(ctx && indptr && (nnz == 0 || (dgene && dcount && indices && data)), SCB_ERR_ARG,
              "scb_csr_delta8_decode: null argument");
  SCB_REQUIRE((n_gesc == 0 || (gesc_pos && gesc_val)) && (n_cesc == 0 || (cesc_pos && cesc_val)), SCB_ERR_ARG,
              "scb_csr_delta8_decode: escape table missing");
  SCB_REQUIRE(((uintptr_t)dgene & 3) == 0 && ((uintptr_t)dcount & 3) == 0 && ((uintptr_t)indices & 15) == 0 &&
                  ((uintptr_t)data & 15) == 0,
              SCB_ERR_ARG, "scb_csr_delta8_decode: 4-byte aligned byte streams, 16-byte aligned outputs required");
  if (n_rows == 0 || nnz == 0) return SCB_OK;
  int per_sm = 0;  // one resident wave (the grid-stride loop gives every warp the same share of rows)
  SCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, delta8_decode_kernel, 256, 0));
  const int g = (int)std::min<int64_t>((int64_t)ctx->num_sms * std::max(per_sm, 1), (n_rows + 7) / 8);
  delta8_decode_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(indptr, n_rows, dgene, dcount, gesc_pos, gesc_val, n_gesc,
                                                            cesc_pos, cesc_val, n_cesc, nnz, indices, data);
  SCB_LAUNCH_CHECK();
  return SCB_OK;
}

// Microbenchmark: column-reduction primitives for CSR gene statistics on B200.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ unsigned hsh(unsigned x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}
__global__ void fill(int* idx, float* v, long n, int G){ long i=blockIdx.x*(long)blockDim.x+threadIdx.x; for(;i<n;i+=(long)gridDim.x*blockDim.x){ idx[i]=hsh((unsigned)i)%G; v[i]=1.0f+(i&7);} }
__global__ void k_read(const int4* idx, const float4* v, long n4, double* out){
  float acc=0; int ai=0; long i=blockIdx.x*(long)blockDim.x+threadIdx.x;
  for(;i<n4;i+=(long)gridDim.x*blockDim.x){ int4 a=__ldg(idx+i); float4 b=__ldg(v+i); ai^=a.x^a.y^a.z^a.w; acc+=b.x+b.y+b.z+b.w;}
  if(acc==-1.f||ai==-12345) out[0]=acc;
}
extern __shared__ unsigned sm[];
__global__ void k_smem_atom(const int4* idx, const float4* v, long n4, int G, unsigned* gout){
  for(int i=threadIdx.x;i<2*G;i+=blockDim.x) sm[i]=0; __syncthreads();
  long i=blockIdx.x*(long)blockDim.x+threadIdx.x;
  for(;i<n4;i+=(long)gridDim.x*blockDim.x){ int4 a=__ldg(idx+i); float4 b=__ldg(v+i);
    atomicAdd(&sm[a.x],1u); atomicAdd(&sm[G+a.x],(unsigned)b.x);
    atomicAdd(&sm[a.y],1u); atomicAdd(&sm[G+a.y],(unsigned)b.y);
    atomicAdd(&sm[a.z],1u); atomicAdd(&sm[G+a.z],(unsigned)b.z);
    atomicAdd(&sm[a.w],1u); atomicAdd(&sm[G+a.w],(unsigned)b.w);}
  __syncthreads(); for(int j=threadIdx.x;j<2*G;j+=blockDim.x) if(sm[j]) atomicAdd(&gout[j],sm[j]);
}
__global__ void k_gred(const int4* idx, const float4* v, long n4, int G, double* gout){
  long i=blockIdx.x*(long)blockDim.x+threadIdx.x;
  for(;i<n4;i+=(long)gridDim.x*blockDim.x){ int4 a=__ldg(idx+i); float4 b=__ldg(v+i);
    atomicAdd(&gout[a.x],(double)b.x); atomicAdd(&gout[G+a.x],(double)b.x*b.x);
    atomicAdd(&gout[a.y],(double)b.y); atomicAdd(&gout[G+a.y],(double)b.y*b.y);
    atomicAdd(&gout[a.z],(double)b.z); atomicAdd(&gout[G+a.z],(double)b.z*b.z);
    atomicAdd(&gout[a.w],(double)b.w); atomicAdd(&gout[G+a.w],(double)b.w*b.w);}
}
// warp-private fp64 RMW histogram over a W-gene tile, 2 stats
template<int W>
__global__ void k_warp_priv(const int4* idx, const float4* v, long n4, double* gout){
  extern __shared__ double hd[]; int wid=threadIdx.x>>5; double* h=hd+wid*2*W;
  for(int i=threadIdx.x;i<(blockDim.x>>5)*2*W;i+=blockDim.x) hd[i]=0; __syncthreads();
  long i=blockIdx.x*(long)blockDim.x+threadIdx.x;
  for(;i<n4;i+=(long)gridDim.x*blockDim.x){ int4 a=__ldg(idx+i); float4 b=__ldg(v+i);
    int g; double y;
    g=a.x&(W-1); y=b.x; h[g]+=y; h[W+g]+=y*y;
    g=a.y&(W-1); y=b.y; h[g]+=y; h[W+g]+=y*y;
    g=a.z&(W-1); y=b.z; h[g]+=y; h[W+g]+=y*y;
    g=a.w&(W-1); y=b.w; h[g]+=y; h[W+g]+=y*y; }
  __syncthreads(); for(int j=threadIdx.x;j<2*W;j+=blockDim.x){ double s=0; for(int w=0;w<(blockDim.x>>5);w++) s+=hd[w*2*W+j]; atomicAdd(&gout[j],s);} 
}
int main(){
  long n=1750L*1000*1000/2; int G=25000; long n4=n/4;
  int* idx; float* v; double* gd; unsigned* gu; double* o;
  CK(cudaMalloc(&idx,n*4)); CK(cudaMalloc(&v,n*4)); CK(cudaMalloc(&gd,2*G*8)); CK(cudaMalloc(&gu,2*G*4)); CK(cudaMalloc(&o,8));
  fill<<<148*8,256>>>(idx,v,n,G); CK(cudaDeviceSynchronize());
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  double bytes=8.0*n;
  for(int rep=0;rep<2;rep++){
  cudaEventRecord(a); k_read<<<148*8,512>>>((int4*)idx,(float4*)v,n4,o); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("read-only: %.3f ms  %.0f GB/s\n",ms,bytes/ms/1e6);
  CK(cudaFuncSetAttribute(k_smem_atom,cudaFuncAttributeMaxDynamicSharedMemorySize,2*G*4));
  cudaEventRecord(a); k_smem_atom<<<148,1024,2*G*4>>>((int4*)idx,(float4*)v,n4,G,gu); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("smem ATOMS.ADD u32 x2 (G=25k, 1 CTA/SM): %.3f ms  %.0f GB/s  %.2f Gatom/s\n",ms,bytes/ms/1e6, 2.0*n/ms/1e6);
  cudaEventRecord(a); k_gred<<<148*4,512>>>((int4*)idx,(float4*)v,n4,G,gd); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("global RED.F64 x2: %.3f ms  %.0f GB/s  %.2f Gatom/s\n",ms,bytes/ms/1e6, 2.0*n/ms/1e6);
  CK(cudaFuncSetAttribute(k_warp_priv<1024>,cudaFuncAttributeMaxDynamicSharedMemorySize,8*2*1024*8));
  cudaEventRecord(a); k_warp_priv<1024><<<148*1,256,8*2*1024*8>>>((int4*)idx,(float4*)v,n4,gd); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("warp-private f64 RMW x2 W=1024 8 warps: %.3f ms  %.0f GB/s\n",ms,bytes/ms/1e6);
  CK(cudaFuncSetAttribute(k_warp_priv<512>,cudaFuncAttributeMaxDynamicSharedMemorySize,16*2*512*8));
  cudaEventRecord(a); k_warp_priv<512><<<148*1,512,16*2*512*8>>>((int4*)idx,(float4*)v,n4,gd); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
  printf("warp-private f64 RMW x2 W=512 16 warps: %.3f ms  %.0f GB/s\n",ms,bytes/ms/1e6);
  }
  CK(cudaGetLastError());
  return 0;
}

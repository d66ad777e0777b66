// Microbenchmarks that decide the transpose design (run once on a B200).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}

__global__ void k_fill_rand(uint32_t* a, size_t n, uint32_t mask, uint32_t seed){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) a[i]=hash32((uint32_t)i*2654435761u+seed)&mask;
}
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
__global__ void k_read(const int4* __restrict__ a, size_t n, int* out){
  int s=0; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){int4 v=__ldg(a+i); s^=v.x^v.y^v.z^v.w;} if(s==0x1234567) *out=s;
}
__global__ void k_gatomic(const uint32_t* __restrict__ keys, size_t n, uint32_t* cnt){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) atomicAdd(cnt+keys[i],1u);
}
__global__ void k_satomic(const uint32_t* __restrict__ keys, size_t n, uint32_t* out, uint32_t mask){
  extern __shared__ uint32_t h[];
  for(uint32_t i=threadIdx.x;i<=mask;i+=blockDim.x) h[i]=0; __syncthreads();
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) atomicAdd(h+(keys[i]&mask),1u);
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=h[5];
}
__global__ void k_scatter(const uint32_t* __restrict__ keys, size_t n, uint32_t* dst){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) dst[keys[i]]=(uint32_t)i;
}
__global__ void k_match(const uint32_t* __restrict__ keys, size_t n, uint32_t* out){
  uint32_t s=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ uint32_t k=keys[i]&255; uint32_t m=__match_any_sync(0xffffffffu,k); s+=__popc(m&((1u<<(threadIdx.x&31))-1)); }
  if(s==0x1234567) *out=s;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2\":%d,\"smem_optin\":%zu,\"mem_gb\":%.1f,\"persist_l2_max\":%d}\n",p.name,p.multiProcessorCount,p.l2CacheSize,p.sharedMemPerBlockOptin,p.totalGlobalMem/1e9,p.persistingL2CacheMaxSize);
  const size_t N=1ull<<29; // 512M keys
  uint32_t *keys,*buf,*cnt; int* sink;
  CK(cudaMalloc(&keys,N*4)); CK(cudaMalloc(&buf,N*4)); CK(cudaMalloc(&cnt,(size_t)1<<31)); CK(cudaMalloc(&sink,4096));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int G=148*8, T=256;
  auto timeit=[&](const char* name, auto fn, double bytes, double ops){ fn(); CK(cudaDeviceSynchronize()); cudaEventRecord(a); for(int r=0;r<3;r++) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); ms/=3;
    printf("{\"bench\":\"%s\",\"ms\":%.4f,\"GBps\":%.1f,\"Gops\":%.2f}\n",name,ms,bytes/ms/1e6,ops/ms/1e6); fflush(stdout);};
  timeit("copy_2GB",[&]{k_copy<<<G,T>>>((int4*)keys,(int4*)buf,N/4);},2.0*N*4,N);
  timeit("read_2GB",[&]{k_read<<<G,T>>>((int4*)keys,N/4,sink);},1.0*N*4,N);
  uint32_t masks[]={ (1u<<14)-1,(1u<<20)-1,(1u<<24)-1,(1u<<27)-1,(1u<<29)-1 };
  for(uint32_t m: masks){
    k_fill_rand<<<G,T>>>(keys,N,m,7); CK(cudaMemset(cnt,0,(size_t)(m+1)*4));
    char nm[64]; snprintf(nm,64,"gatomic_bins_2^%d",__builtin_popcount(m));
    timeit(nm,[&]{k_gatomic<<<G,T>>>(keys,N,cnt);},4.0*N,N);
    snprintf(nm,64,"scatter4B_range_2^%d",__builtin_popcount(m));
    timeit(nm,[&]{k_scatter<<<G,T>>>(keys,N,cnt);},4.0*N,N);
  }
  k_fill_rand<<<G,T>>>(keys,N,0xffffffffu,9);
  for(int bits: {8,12,14,15}){ uint32_t m=(1u<<bits)-1; size_t sm=(size_t)(m+1)*4; CK(cudaFuncSetAttribute(k_satomic,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm));
    char nm[64]; snprintf(nm,64,"satomic_bins_2^%d",bits);
    timeit(nm,[&]{k_satomic<<<148*2,1024,sm>>>(keys,N,buf,m);},4.0*N,N); }
  timeit("match_any_8bit",[&]{k_match<<<G,T>>>(keys,N,(uint32_t*)sink);},4.0*N,N);
  return 0;
}

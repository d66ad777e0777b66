// Microbenchmarks, round 2: compute-side ranking primitives with register-resident
// keys, and memory ops with many independent requests in flight per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}
#define ITERS 4096
// pure match_any throughput (8-bit keys), 8 independent chains
__global__ void k_match(uint32_t* out, uint32_t seed){
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  uint32_t acc=0;
  for(int it=0; it<ITERS; it++){
#pragma unroll
    for(int j=0;j<8;j++){ uint32_t m=__match_any_sync(0xffffffffu,k[j]&255); acc+=m; k[j]=k[j]*1664525u+1013904223u; }
  }
  if(acc==0x12345) out[0]=acc;
}
// ballot-based peers (8 bits)
__global__ void k_ballot8(uint32_t* out, uint32_t seed){
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  uint32_t acc=0;
  for(int it=0; it<ITERS; it++){
#pragma unroll
    for(int j=0;j<8;j++){ uint32_t d=k[j]&255; uint32_t peers=0xffffffffu;
#pragma unroll
      for(int b=0;b<8;b++){ uint32_t bb=__ballot_sync(0xffffffffu,(d>>b)&1); peers&= bb ^ (((d>>b)&1)-1u); }
      acc+=peers; k[j]=k[j]*1664525u+1013904223u; }
  }
  if(acc==0x12345) out[0]=acc;
}
// smem atomics, register keys, 2^bits bins, per-CTA hist
template<int BITS> __global__ void k_satom(uint32_t* out, uint32_t seed){
  __shared__ uint32_t h[1<<BITS]; for(int i=threadIdx.x;i<(1<<BITS);i+=blockDim.x) h[i]=0; __syncthreads();
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  uint32_t acc=0;
  for(int it=0; it<ITERS/4; it++){
#pragma unroll
    for(int j=0;j<8;j++){ acc+=atomicAdd(&h[k[j]&((1<<BITS)-1)],1u); k[j]=k[j]*1664525u+1013904223u; }
  }
  __syncthreads(); if(acc==0x12345) out[0]=acc+h[3];
}
// smem red (no return)
template<int BITS> __global__ void k_sred(uint32_t* out, uint32_t seed){
  __shared__ uint32_t h[1<<BITS]; for(int i=threadIdx.x;i<(1<<BITS);i+=blockDim.x) h[i]=0; __syncthreads();
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  for(int it=0; it<ITERS/4; it++){
#pragma unroll
    for(int j=0;j<8;j++){ atomicAdd(&h[k[j]&((1<<BITS)-1)],1u); k[j]=k[j]*1664525u+1013904223u; }
  }
  __syncthreads(); if(threadIdx.x<(1<<BITS) && h[threadIdx.x]==0x12345) out[0]=1;
}
// smem random LDS + STS (private per-warp region), models per-warp counters
__global__ void k_ldssts(uint32_t* out, uint32_t seed){
  __shared__ uint32_t h[8][256]; int w=threadIdx.x>>5; for(int i=threadIdx.x;i<8*256;i+=blockDim.x) ((uint32_t*)h)[i]=0; __syncthreads();
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  uint32_t acc=0;
  for(int it=0; it<ITERS/4; it++){
#pragma unroll
    for(int j=0;j<8;j++){ uint32_t d=k[j]&255; uint32_t v=h[w][d]; acc+=v; h[w][d]=v+1; k[j]=k[j]*1664525u+1013904223u; }
  }
  __syncthreads(); if(acc==0x12345) out[0]=acc;
}
// global ops with 16 independent requests in flight per thread
__global__ void k_gatom16(const uint4* __restrict__ keys4, size_t n4, uint32_t* cnt){
  for(size_t i=(blockIdx.x*(size_t)blockDim.x+threadIdx.x)*4;i<n4;i+=(size_t)gridDim.x*blockDim.x*4){
    uint4 v[4];
#pragma unroll
    for(int j=0;j<4;j++) v[j]=(i+j<n4)?keys4[i+j]:make_uint4(0,0,0,0);
#pragma unroll
    for(int j=0;j<4;j++){ atomicAdd(cnt+v[j].x,1u); atomicAdd(cnt+v[j].y,1u); atomicAdd(cnt+v[j].z,1u); atomicAdd(cnt+v[j].w,1u);} }
}
__global__ void k_scat16(const uint4* __restrict__ keys4, size_t n4, uint32_t* dst){
  for(size_t i=(blockIdx.x*(size_t)blockDim.x+threadIdx.x)*4;i<n4;i+=(size_t)gridDim.x*blockDim.x*4){
    uint4 v[4];
#pragma unroll
    for(int j=0;j<4;j++) v[j]=(i+j<n4)?keys4[i+j]:make_uint4(0,0,0,0);
#pragma unroll
    for(int j=0;j<4;j++){ dst[v[j].x]=1; dst[v[j].y]=2; dst[v[j].z]=3; dst[v[j].w]=4;} }
}
// scattered 32B-run writes: each warp writes 8 consecutive u32 per lane-group (sector-aligned runs)
__global__ void k_runs(const uint4* __restrict__ keys4, size_t n4, uint32_t* dst, uint32_t mask){
  int lane=threadIdx.x&31;
  for(size_t i=(blockIdx.x*(size_t)blockDim.x+threadIdx.x);i<n4;i+=(size_t)gridDim.x*blockDim.x){
    uint4 v=keys4[i]; uint32_t base=__shfl_sync(0xffffffffu,v.x,lane&~7)&mask&~7u; dst[base+(lane&7)]=v.y; }
}
__global__ void k_fill_rand(uint32_t* a, size_t n, uint32_t mask, uint32_t seed){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) a[i]=hash32((uint32_t)i*2654435761u+seed)&mask;
}
__global__ void k_copy4(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n){
  size_t s=(size_t)gridDim.x*blockDim.x; size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(;i+3*s<n;i+=4*s){ uint4 x0=a[i],x1=a[i+s],x2=a[i+2*s],x3=a[i+3*s]; b[i]=x0;b[i+s]=x1;b[i+2*s]=x2;b[i+3*s]=x3;}
  for(;i<n;i+=s) b[i]=a[i];
}
int main(){
  uint32_t* o; CK(cudaMalloc(&o,64));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int G=148*4, T=512; double items=(double)G*T*8*ITERS;
  auto timeit=[&](const char* name, auto fn, double ops, double bytes){ fn(); CK(cudaDeviceSynchronize()); cudaEventRecord(a); for(int r=0;r<3;r++) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); ms/=3;
    printf("{\"bench\":\"%s\",\"ms\":%.4f,\"Gops\":%.1f,\"GBps\":%.1f,\"ops_per_clk_sm@1.9\":%.3f}\n",name,ms,ops/ms/1e6,bytes/ms/1e6,ops/ms/1e6/148/1.9); fflush(stdout);};
  //timeit("match_any8_reg",[&]{k_match<<<G,T>>>(o,1);},items,0);
  //timeit("ballot8_reg",[&]{k_ballot8<<<G,T>>>(o,1);},items,0);
  timeit("satomic_ret_2^8",[&]{k_satom<8><<<G,T>>>(o,1);},items/4,0);
  timeit("satomic_ret_2^12",[&]{k_satom<12><<<G,T>>>(o,1);},items/4,0);
  timeit("sred_2^8",[&]{k_sred<8><<<G,T>>>(o,1);},items/4,0);
  timeit("sred_2^12",[&]{k_sred<12><<<G,T>>>(o,1);},items/4,0);
  timeit("lds_sts_perwarp256",[&]{k_ldssts<<<G,256>>>(o,1);},items/8,0);
  const size_t N=1ull<<29; uint32_t *keys,*buf,*cnt; CK(cudaMalloc(&keys,N*4)); CK(cudaMalloc(&buf,N*4)); CK(cudaMalloc(&cnt,(size_t)1<<31));
  timeit("copy4_2GB",[&]{k_copy4<<<148*4,512>>>((uint4*)keys,(uint4*)buf,N/4);},N,8.0*N);
  for(int bits: {14,20,24,26,29}){ uint32_t m=(bits==32)?0xffffffffu:((1u<<bits)-1);
    k_fill_rand<<<1184,256>>>(keys,N,m,7); CK(cudaMemset(cnt,0,(size_t)(m+1)*4)); char nm[64];
    snprintf(nm,64,"gatomic16_2^%d",bits); timeit(nm,[&]{k_gatom16<<<148*8,256>>>((uint4*)keys,N/4,cnt);},N,4.0*N);
    snprintf(nm,64,"scatter16_2^%d",bits); timeit(nm,[&]{k_scat16<<<148*8,256>>>((uint4*)keys,N/4,cnt);},N,4.0*N);
    snprintf(nm,64,"runs32B_2^%d",bits); timeit(nm,[&]{k_runs<<<148*8,256>>>((uint4*)keys,N/4,cnt,m);},N/4,N*1.0);
  }
  return 0;
}

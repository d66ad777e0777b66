// mb3: (1) is shared-memory atomicAdd return order among same-address lanes of one
// warp instruction lane-ascending on this GPU?  (2) throughput of candidate stable
// ranking schemes (per-warp counters): ATOMS-only, OR-mask, ballot8.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}
// (1) order test: each warp, per iteration: digits from hash with a variable alphabet size
__global__ void k_order(unsigned long long* bad, uint32_t seed, int iters){
  __shared__ uint32_t cnt[32][256];
  int w=threadIdx.x>>5, lane=threadIdx.x&31;
  for(int i=lane;i<256;i+=32) cnt[w][i]=0; __syncwarp();
  unsigned long long nbad=0;
  for(int it=0; it<iters; it++){
    uint32_t h=hash32(seed ^ (blockIdx.x*1315423911u) ^ (threadIdx.x*2654435761u) ^ (it*97531u));
    int alpha = 1 << ((hash32(it*7+blockIdx.x)&7)+1); // 2..256 distinct digits
    uint32_t d=h & (alpha-1);
    uint32_t old=atomicAdd(&cnt[w][d],1u);
    // expected: base + #lower lanes with same digit. base = min(old) over peers.
    uint32_t peers=__match_any_sync(0xffffffffu,d);
    uint32_t lo=__ffs(peers)-1;
    uint32_t base=__shfl_sync(0xffffffffu,old,lo); // lowest lane's value is base iff ordered
    uint32_t mn=old; for(int o=16;o>0;o>>=1){ uint32_t x=__shfl_xor_sync(0xffffffffu,mn,o); /*only peers*/ }
    uint32_t expect=base+__popc(peers&((1u<<lane)-1));
    if(old!=expect) nbad++;
  }
  if(nbad) atomicAdd(bad,nbad);
}
// (2a) ATOMS-only rank throughput
__global__ void k_rank_atoms(uint32_t* out, uint32_t seed){
  __shared__ uint32_t cnt[16][256]; int w=threadIdx.x>>5;
  for(int i=threadIdx.x;i<16*256;i+=blockDim.x) ((uint32_t*)cnt)[i]=0; __syncthreads();
  uint32_t k[8]; for(int j=0;j<8;j++) k[j]=hash32(threadIdx.x*8+j+seed+blockIdx.x*7919);
  uint32_t acc=0;
  for(int it=0; it<1024; it++){
#pragma unroll
    for(int j=0;j<8;j++){ acc+=atomicAdd(&cnt[w][k[j]&255],1u); k[j]=k[j]*1664525u+1013904223u; }
  }
  if(acc==0x12345) out[0]=acc;
}
// (2b) OR-mask rank: RED.OR mask, syncwarp, LDS.64 {mask,count}, leader STS.64
__global__ void k_rank_ormask(uint32_t* out, uint32_t seed){
  __shared__ unsigned long long mc[16][256]; int w=threadIdx.x>>5, lane=threadIdx.x&31;
  for(int i=threadIdx.x;i<16*256;i+=blockDim.x) ((unsigned long long*)mc)[i]=0; __syncthreads();
  uint32_t k=hash32(threadIdx.x+seed+blockIdx.x*7919);
  uint32_t acc=0; uint32_t lt=(1u<<lane)-1;
  for(int it=0; it<8192; it++){
    uint32_t d=k&255;
    atomicOr((uint32_t*)&mc[w][d],1u<<lane);
    __syncwarp();
    unsigned long long v=mc[w][d];
    uint32_t peers=(uint32_t)v, c=(uint32_t)(v>>32);
    acc+=c+__popc(peers&lt);
    __syncwarp();
    if((peers&lt)==0) mc[w][d]=((unsigned long long)(c+__popc(peers))<<32);
    __syncwarp();
    k=k*1664525u+1013904223u;
  }
  if(acc==0x12345) out[0]=acc;
}
int main(){
  unsigned long long* bad; CK(cudaMalloc(&bad,8)); CK(cudaMemset(bad,0,8));
  uint32_t* o; CK(cudaMalloc(&o,64));
  for(int r=0;r<20;r++) k_order<<<148*4,1024>>>(bad,r*12345+1,2048);
  CK(cudaDeviceSynchronize()); unsigned long long hb; CK(cudaMemcpy(&hb,bad,8,cudaMemcpyDeviceToHost));
  printf("{\"bench\":\"atoms_lane_order\",\"trials\":%llu,\"violations\":%llu}\n",(unsigned long long)20*148*4*1024*2048ull,hb);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit=[&](const char* name, auto fn, double ops){ fn(); CK(cudaDeviceSynchronize()); cudaEventRecord(a); for(int r=0;r<3;r++) fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); ms/=3;
    printf("{\"bench\":\"%s\",\"ms\":%.4f,\"Gitems\":%.1f,\"items_per_clk_sm@1.9\":%.3f}\n",name,ms,ops/ms/1e6,ops/ms/1e6/148/1.9); fflush(stdout);};
  timeit("rank_atoms",[&]{k_rank_atoms<<<148*4,512>>>(o,1);},148.0*4*512*8*1024);
  timeit("rank_ormask",[&]{k_rank_ormask<<<148*4,512>>>(o,1);},148.0*4*512*8192);
  return 0;
}

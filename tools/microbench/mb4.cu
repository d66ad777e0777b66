// Microbenchmark 4: warp ranking cost vs key duplication.
// For keys with `u` distinct values per warp-slot (u = 1..32), compare
//   atoms : one shared atomicAdd per lane (same-address lanes serialise),
//   match : __match_any_sync peers, leader-only atomicAdd,
//   ballot: bit-sliced ballot peers (8 bits), leader-only atomicAdd,
//   runs  : equal keys in consecutive lanes aggregated by run heads.
// Prints warp-slots per clock per SM (higher is better).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}
__device__ __forceinline__ uint32_t lt_mask(){ uint32_t m; asm("mov.u32 %0, %%lanemask_lt;":"=r"(m)); return m;}
#define SLOTS 16
#define ITERS 256
// key for (slot, lane): u distinct values per slot; sorted=1 puts equal keys in consecutive lanes
__device__ __forceinline__ uint32_t key(uint32_t seed, int s, int lane, int u, int sorted){
  uint32_t g = sorted ? (uint32_t)(lane * u / 32) : (hash32(seed*131u + s*977u + lane) % u);
  return hash32(seed + s * 7919u + g * 104729u) & 255u;
}
template<int MODE>
__global__ void k_rank(uint32_t* out, int u, int sorted){
  __shared__ uint32_t cnt[8][256*1+8];
  const int w=threadIdx.x>>5, lane=threadIdx.x&31;
  for(int i=lane;i<256;i+=32) cnt[w][i]=0;
  __syncwarp();
  uint32_t k[SLOTS];
#pragma unroll
  for(int s=0;s<SLOTS;s++) k[s]=key(blockIdx.x*8+w, s, lane, u, sorted);
  uint32_t acc=0;
  for(int it=0; it<ITERS; ++it){
#pragma unroll
    for(int s=0;s<SLOTS;s++){
      const uint32_t d=k[s];
      uint32_t r;
      if(MODE==0){ r=atomicAdd(&cnt[w][d],1u); }
      else if(MODE==1){ uint32_t m=__match_any_sync(0xffffffffu,d); uint32_t ld=__ffs(m)-1; uint32_t b=0; if(lane==ld) b=atomicAdd(&cnt[w][d],__popc(m)); b=__shfl_sync(0xffffffffu,b,ld); r=b+__popc(m&lt_mask()); }
      else if(MODE==2){ uint32_t m=0xffffffffu;
#pragma unroll
        for(int b=0;b<8;b++){ uint32_t bb=__ballot_sync(0xffffffffu,(d>>b)&1u); m&= bb ^ (((d>>b)&1u)-1u); }
        uint32_t ld=__ffs(m)-1; uint32_t b=0; if(lane==ld) b=atomicAdd(&cnt[w][d],__popc(m)); b=__shfl_sync(0xffffffffu,b,ld); r=b+__popc(m&lt_mask()); }
      else { uint32_t pv=__shfl_up_sync(0xffffffffu,d,1); bool head=(lane==0)||(pv!=d); uint32_t hm=__ballot_sync(0xffffffffu,head);
        uint32_t nxt = hm & ~((2u<<lane)-1u); uint32_t end = nxt ? (__ffs(nxt)-1) : 32u; uint32_t hd = 31-__clz(hm & ((2u<<lane)-1u));
        uint32_t b=0; if(head) b=atomicAdd(&cnt[w][d], end-lane); b=__shfl_sync(0xffffffffu,b,hd); r=b+lane-hd; }
      acc+=r; k[s]=(k[s]*1664525u+1013904223u)&255u;  // keep duplication structure roughly: new permutation of values
    }
  }
  if(acc==0x12345678) out[0]=acc;
}
int main(){
  uint32_t* o; CK(cudaMalloc(&o,64));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int G=148*6, T=256;
  const char* names[4]={"atoms","match","ballot8","runs"};
  for(int sorted=0; sorted<2; ++sorted)
  for(int u: {1,2,4,8,16,32}){
    for(int mode=0; mode<4; ++mode){
      if(mode==3 && !sorted) continue;
      auto run=[&]{ if(mode==0) k_rank<0><<<G,T>>>(o,u,sorted); else if(mode==1) k_rank<1><<<G,T>>>(o,u,sorted); else if(mode==2) k_rank<2><<<G,T>>>(o,u,sorted); else k_rank<3><<<G,T>>>(o,u,sorted); };
      run(); CK(cudaDeviceSynchronize());
      cudaEventRecord(a); for(int r=0;r<3;r++) run(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms,a,b); ms/=3;
      const double slots=(double)G*(T/32)*ITERS*SLOTS;
      printf("{\"mode\":\"%s\",\"sorted\":%d,\"distinct\":%d,\"ms\":%.4f,\"slots_per_clk_sm\":%.3f}\n",names[mode],sorted,u,ms,slots/(ms*1e-3)/148/1.9e9);
    }
  }
  return 0;
}

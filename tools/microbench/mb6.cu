// Microbenchmark 6: direct scatter with CTA-shared cursors and exact,
// tile-contiguous output runs (the onesweep layout), as the alternative to
// shared-memory staging.  A count pass writes per-(digit, tile) counts,
// a scan turns them into bases, and the scatter pass ranks each record with
// a shared-memory atomic on its digit's cursor and stores it straight to
// global memory.  Every output sector is written by stores of one CTA (or of
// two neighbouring tiles), so L2 can complete sectors before they are
// evicted; the question is whether the L1/L2 request rate of scattered 4-byte
// stores beats the staged pass (~1 SM-cycle per record).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mb6 mb6.cu
//   ./mb6 [cfg]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}

__global__ void k_fill(uint32_t* a, uint64_t n){ for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n;i+=(uint64_t)gridDim.x*blockDim.x) a[i]=hash32((uint32_t)i*2654435761u+17u); }

__global__ void k_count(const uint32_t* __restrict__ in, uint32_t* __restrict__ cnt, uint64_t tile, int dlog, int ntiles){
  extern __shared__ uint32_t s_c[];
  const int D = 1 << dlog;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int d = threadIdx.x; d < D; d += blockDim.x) s_c[d] = 0;
    __syncthreads();
    const uint4* p = reinterpret_cast<const uint4*>(in + (uint64_t)t * tile);
    for (uint64_t i = threadIdx.x; i < tile / 4; i += blockDim.x) {
      uint4 v = __ldg(p + i);
      atomicAdd(&s_c[v.x & (D - 1)], 1u); atomicAdd(&s_c[v.y & (D - 1)], 1u);
      atomicAdd(&s_c[v.z & (D - 1)], 1u); atomicAdd(&s_c[v.w & (D - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) cnt[(uint64_t)d * ntiles + t] = s_c[d];
    __syncthreads();
  }
}

// MODE 0: scatter store; 1: ranks only
template <int MODE>
__global__ void k_scatter(const uint32_t* __restrict__ in, const uint32_t* __restrict__ base, uint32_t* __restrict__ out,
                          uint64_t tile, int dlog, int ntiles){
  extern __shared__ uint32_t s_c[];
  const int D = 1 << dlog;
  uint32_t acc = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int d = threadIdx.x; d < D; d += blockDim.x) s_c[d] = base[(uint64_t)d * ntiles + t];
    __syncthreads();
    const uint4* p = reinterpret_cast<const uint4*>(in + (uint64_t)t * tile);
    for (uint64_t i = threadIdx.x; i < tile / 4; i += 2 * blockDim.x) {
      uint4 v0 = __ldg(p + i), v1 = __ldg(p + i + blockDim.x);
      uint32_t q[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w}, pos[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pos[j] = atomicAdd(&s_c[q[j] & (D - 1)], 1u);
#pragma unroll
      for (int j = 0; j < 8; ++j) { if (MODE == 0) out[pos[j]] = q[j]; else acc += pos[j]; }
    }
    __syncthreads();
  }
  if (MODE == 1 && acc == 0x1234567u) out[0] = acc;
}

__global__ void k_check(const uint32_t* out, uint64_t n, int dlog, unsigned long long* bad){
  const uint32_t D = 1u << dlog;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    if ((out[i] & (D - 1)) > (out[i + 1] & (D - 1))) atomicAdd(bad, 1ull);
}

int main(int argc, char** argv){
  const uint64_t n = 1ull << 29;
  uint32_t *in, *out, *cnt, *base;
  CK(cudaMalloc(&in, n * 4));
  CK(cudaMalloc(&out, n * 4));
  k_fill<<<1184, 512>>>(in, n);
  CK(cudaDeviceSynchronize());
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  unsigned long long* bad; CK(cudaMalloc(&bad, 8));
  struct Cfg { int mode, dlog, tile_log, threads, ctas_per_sm; };
  Cfg cfgs[] = {
    {1, 9, 14, 512, 4}, {0, 9, 14, 512, 4}, {0, 9, 16, 512, 4}, {0, 9, 18, 1024, 2},
    {1, 12, 16, 512, 4}, {0, 12, 16, 512, 4}, {0, 12, 18, 1024, 2},
    {1, 14, 18, 1024, 2}, {0, 14, 18, 1024, 2}, {0, 14, 18, 512, 3},
    {1, 15, 18, 1024, 1}, {0, 15, 18, 1024, 1}, {0, 15, 18, 1024, 1},
  };
  int only = argc > 1 ? atoi(argv[1]) : -1;
  for (int ci = 0; ci < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++ci) {
    if (only >= 0 && ci != only) continue;
    Cfg c = cfgs[ci];
    const int D = 1 << c.dlog;
    const uint64_t tile = 1ull << c.tile_log;
    const int ntiles = (int)(n / tile);
    const size_t sm = (size_t)D * 4;
    const size_t tab = (size_t)D * ntiles;
    CK(cudaMalloc(&cnt, tab * 4)); CK(cudaMalloc(&base, tab * 4));
    void* tmp = nullptr; size_t tmpb = 0;
    cub::DeviceScan::ExclusiveSum(tmp, tmpb, cnt, base, (int)tab);
    CK(cudaMalloc(&tmp, tmpb));
    CK(cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(k_scatter<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(k_scatter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = sms * c.ctas_per_sm;
    float tc = 0, ts = 0, tp = 1e9;
    for (int r = 0; r < 4; ++r) {
      float m0, m1, m2;
      cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(a));
      k_count<<<grid, c.threads, sm>>>(in, cnt, tile, c.dlog, ntiles);
      CK(cudaEventRecord(e0));
      cub::DeviceScan::ExclusiveSum(tmp, tmpb, cnt, base, (int)tab);
      CK(cudaEventRecord(e1));
      if (c.mode == 0) k_scatter<0><<<grid, c.threads, sm>>>(in, base, out, tile, c.dlog, ntiles);
      else k_scatter<1><<<grid, c.threads, sm>>>(in, base, out, tile, c.dlog, ntiles);
      CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaGetLastError());
      CK(cudaEventElapsedTime(&m0, a, e0)); CK(cudaEventElapsedTime(&m1, e0, e1)); CK(cudaEventElapsedTime(&m2, e1, b));
      if (r > 0 && m2 < tp) { tp = m2; tc = m0; ts = m1; }
      CK(cudaEventDestroy(e0)); CK(cudaEventDestroy(e1));
    }
    unsigned long long nb = 0;
    if (c.mode == 0) {
      CK(cudaMemset(bad, 0, 8)); k_check<<<1184, 512>>>(out, n, c.dlog, bad); CK(cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost));
    }
    printf("cfg %2d mode %d D 2^%d tile 2^%d thr %d ctas/sm %d: count %.3f scan %.3f scatter %.3f ms = %.1f G rec/s  unsorted %llu\n",
           ci, c.mode, c.dlog, c.tile_log, c.threads, c.ctas_per_sm, tc, ts, tp, n / tp / 1e6, nb);
    CK(cudaFree(cnt)); CK(cudaFree(base)); CK(cudaFree(tmp));
  }
  return 0;
}

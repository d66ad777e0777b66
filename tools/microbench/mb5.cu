// Microbenchmark 5: direct scatter from warp-private cursors vs staged write-out.
// Each warp owns a contiguous segment of a 2^29-record input and a private
// cursor array (one u32 per key) in shared memory; every record's position is
// atomicAdd(&cur[key], 1) (lane-ordered within the warp) and it is stored
// straight to global memory.  Measures records/s for key counts and warps/SM,
// and (under ncu) the DRAM bytes written per record.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ uint32_t hash32(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x;}

__global__ void k_fill(uint32_t* a, uint64_t n){ for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n;i+=(uint64_t)gridDim.x*blockDim.x) a[i]=hash32((uint32_t)i*2654435761u+17u); }

// mode 0: scatter store; 1: atomics only (no store); 2: coalesced copy
template<int MODE>
__global__ void k_scatter(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n, int keys_log, uint64_t region){
  extern __shared__ uint32_t s_cur[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nwb = blockDim.x >> 5;
  const uint64_t gw = (uint64_t)blockIdx.x * nwb + w, nwt = (uint64_t)gridDim.x * nwb;
  const int keys = 1 << keys_log;
  uint32_t* cur = s_cur + w * keys;
  const uint64_t per_run = region / nwt;  // slots of (warp, key) run inside key k's region
  for (int k = lane; k < keys; k += 32) cur[k] = (uint32_t)((uint64_t)k * region + gw * per_run);
  __syncwarp();
  const uint64_t seg = n / nwt, b = gw * seg;
  uint32_t acc = 0;
  for (uint64_t s = 0; s < seg; s += 32 * 8) {
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(in + b + s + j * 32 + lane);
    if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) out[b + s + j * 32 + lane] = v[j];
      continue;
    }
    uint32_t pos[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) pos[j] = atomicAdd(&cur[v[j] & (keys - 1)], 1u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) out[pos[j]] = v[j];
      else acc += pos[j];
    }
  }
  if (MODE == 1 && acc == 0x1234567u) out[0] = acc;
}

int main(int argc, char** argv){
  const uint64_t n = 1ull << 29;
  uint32_t *in, *out;
  CK(cudaMalloc(&in, n * 4));
  CK(cudaMalloc(&out, n * 4 * 2 + (1 << 20)));
  k_fill<<<1184, 512>>>(in, n);
  CK(cudaDeviceSynchronize());
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  struct Cfg { int mode, keys_log, warps, ctas_per_sm; };
  Cfg cfgs[] = {
    {2, 8, 8, 4},
    {1, 8, 8, 4}, {0, 8, 8, 4}, {0, 8, 16, 2}, {0, 8, 8, 1},
    {1, 10, 8, 4}, {0, 10, 8, 4}, {0, 10, 8, 2}, {0, 10, 8, 1}, {0, 10, 4, 1},
    {1, 12, 8, 1}, {0, 12, 8, 1}, {0, 12, 4, 1}, {0, 12, 2, 1},
  };
  int only = argc > 1 ? atoi(argv[1]) : -1;
  for (int ci = 0; ci < (int)(sizeof(cfgs) / sizeof(cfgs[0])); ++ci) {
    if (only >= 0 && ci != only) continue;
    Cfg c = cfgs[ci];
    const int keys = 1 << c.keys_log;
    const size_t sm = (size_t)c.warps * keys * 4;
    const uint64_t region = n * 2 / keys;  // 2x slack per key region
    auto run = [&]() {
      if (c.mode == 0) { CK(cudaFuncSetAttribute(k_scatter<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_scatter<0><<<sms * c.ctas_per_sm, c.warps * 32, sm>>>(in, out, n, c.keys_log, region); }
      if (c.mode == 1) { CK(cudaFuncSetAttribute(k_scatter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_scatter<1><<<sms * c.ctas_per_sm, c.warps * 32, sm>>>(in, out, n, c.keys_log, region); }
      if (c.mode == 2) { CK(cudaFuncSetAttribute(k_scatter<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_scatter<2><<<sms * c.ctas_per_sm, c.warps * 32, sm>>>(in, out, n, c.keys_log, region); }
    };
    run(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(a)); run(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    printf("cfg %d mode %d keys 2^%d warps %d ctas/sm %d: %.3f ms  %.1f G rec/s  frontiers %llu\n", ci, c.mode, c.keys_log,
           c.warps, c.ctas_per_sm, best, n / best / 1e6, (unsigned long long)sms * c.ctas_per_sm * c.warps * keys);
  }
  return 0;
}

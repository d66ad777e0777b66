// gt_base.cuh — small kernels and input views shared by the transposition
// pipeline (gt_v3.cuh kernels, gt_api.cu orchestration).
#pragma once
#include "gt_common.cuh"
#include "gt_scan.cuh"

namespace gt {

__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }
__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }

// CSR edge stream (the transpose input).  `edges` points at global edge
// e_begin; stream index i is global edge e_begin + i.  Sources are recovered
// from `offsets` (global, V+1 entries, V = source IDs).
struct InCsr {
  const uint64_t* offsets;
  const uint32_t* edges;
  uint64_t e_begin;
  uint64_t V;
};

// Owner (source) of stream position min(k*CT, E-1): largest v with
// offsets[v] <= e_begin + that position (binary search).
__global__ void k_tile_src(InCsr in, uint64_t E, uint64_t CT, uint64_t ntiles, uint32_t* __restrict__ tile_src) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= ntiles) return;
  const uint64_t pos = in.e_begin + umin64(k * CT, E - 1);
  uint64_t lo = 0, hi = in.V;  // answer in [0, V-1]; offsets[0] = 0 <= pos
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (in.offsets[mid] <= pos) lo = mid; else hi = mid;
  }
  tile_src[k] = (uint32_t)lo;
}

// Source of the edge just before each count tile: owner of stream position
// k*CT - 1 for k >= 1, ~0u for k = 0.
__global__ void k_prev_src(InCsr in, uint64_t E, uint64_t CT, uint64_t ntiles, uint32_t* __restrict__ prev) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= ntiles) return;
  if (k == 0) {
    prev[0] = 0xffffffffu;
    return;
  }
  const uint64_t pos = in.e_begin + umin64(k * CT, E) - 1;
  uint64_t lo = 0, hi = in.V;
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (in.offsets[mid] <= pos) lo = mid; else hi = mid;
  }
  prev[k] = (uint32_t)lo;
}

// Lane-order self-test of shared-memory atomicAdd (DESIGN.md §2 "Ranking"):
// same-address lanes of one warp instruction must receive their old values in
// ascending lane order; counts the returns that were not.
__global__ void k_selftest_rank(unsigned long long* bad, uint32_t seed, int iters) {
  __shared__ uint32_t cnt[32][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 256; i += 32) cnt[w][i] = 0;
  __syncwarp();
  unsigned long long nbad = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t h = seed ^ (blockIdx.x * 1315423911u) ^ (threadIdx.x * 2654435761u) ^ (it * 97531u);
    h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
    uint32_t a = (uint32_t)it * 7u + blockIdx.x;
    a ^= a >> 16; a *= 0x7feb352du; a ^= a >> 15;
    const uint32_t alpha = 1u << ((a & 7) + 1);
    const uint32_t d = h & (alpha - 1);
    const bool active = ((a >> 8) & 3) ? true : ((h >> 20) & 1);  // 1/4 of iterations: partial masks
    const uint32_t am = __ballot_sync(kFull, active);
    uint32_t old = 0;
    if (active) old = atomicAdd(&cnt[w][d], 1u);
    const uint32_t peers = __match_any_sync(kFull, active ? d : 0xffffffffu) & am;
    const uint32_t lo = peers ? (__ffs(peers) - 1) : 0;
    const uint32_t b = __shfl_sync(kFull, old, lo);
    if (active && old != b + __popc(peers & lanemask_lt())) ++nbad;
  }
  if (nbad) atomicAdd(bad, nbad);
}

__global__ void k_add_base(uint64_t* a, uint64_t n, uint64_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] += base;
}

}  // namespace gt

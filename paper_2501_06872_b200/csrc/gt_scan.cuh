// gt_scan.cuh — single-pass device-wide exclusive scan with decoupled look-back.
// Used for CSC offsets (prefix_sum_parallel, baselines.py:116-127) and for the
// per-(tile, digit) and per-bucket bases of the partition levels.
#pragma once
#include "gt_common.cuh"

namespace gt {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 16;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

// out[i] = init + sum_{j<i} in[j] for i in [0, n); if write_total, out[n] = init + sum.
// status: >= ceil(n / kScanTile) zeroed words; tile_ctr: one zeroed word.
template <typename In>
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const In* __restrict__ in, uint64_t n,
                                                                 uint64_t* __restrict__ out, uint64_t init,
                                                                 int write_total, uint64_t* status,
                                                                 unsigned int* tile_ctr,
                                                                 const uint32_t* __restrict__ n_dev = nullptr,
                                                                 uint64_t n_unit = 1) {
  // optional device-side length: n = min(n, *n_dev * n_unit) (the grid is sized for n)
  if (n_dev) n = umin64(n, (uint64_t)(*n_dev) * n_unit);
  __shared__ uint64_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_excl;
  __shared__ unsigned int s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t tsum = 0;
  if constexpr (sizeof(In) == 4) {
    // 16-byte loads when the thread's items are in range and aligned
    const bool vec = base + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0);
    if (vec) {
#pragma unroll
      for (int k = 0; k < kScanItems; k += 4) {
        const uint4 q = *reinterpret_cast<const uint4*>(in + base + k);
        v[k] = q.x;
        v[k + 1] = q.y;
        v[k + 2] = q.z;
        v[k + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        v[k] = (i < n) ? (uint64_t)in[i] : 0;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t i = base + k;
      v[k] = (i < n) ? (uint64_t)in[i] : 0;
    }
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) tsum += v[k];
  // block inclusive scan of tsum
  const uint32_t lane = lane_id(), w = warp_id();
  uint64_t x = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    constexpr int NW = kScanThreads / 32;
    uint64_t a = (lane < NW) ? s_warp[lane] : 0;
    uint64_t b = a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(kFull, b, o);
      if (lane >= (uint32_t)o) b += y;
    }
    if (lane < NW) s_warp[lane] = b - a;
    const uint64_t agg = __shfl_sync(kFull, b, 31);
    // decoupled look-back
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_volatile_u64(&status[0], kFlagInc | agg);
    } else {
      if (lane == 0) st_volatile_u64(&status[tile], kFlagAgg | agg);
      int64_t j = (int64_t)tile - 1;
      while (true) {
        const int64_t idx = j - (int64_t)lane;
        uint64_t s = (idx >= 0) ? ld_volatile_u64(&status[idx]) : kFlagInc;
        while (__any_sync(kFull, (s >> 62) == 0)) {
          if ((s >> 62) == 0) s = ld_volatile_u64(&status[idx]);
        }
        const uint32_t inc_mask = __ballot_sync(kFull, (s >> 62) == 2);
        uint64_t val = s & kValMask;
        if (inc_mask) {
          const uint32_t first = __ffs(inc_mask) - 1;
          if (lane > first) val = 0;
          for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
          excl += val;
          break;
        }
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
        excl += val;
        j -= 32;
      }
      if (lane == 0) st_volatile_u64(&status[tile], kFlagInc | (excl + agg));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  uint64_t run = init + s_excl + s_warp[w] + x - tsum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = base + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (write_total && base < n && base + kScanItems >= n) out[n] = run;
  if (write_total && n == 0 && tile == 0 && threadIdx.x == 0) out[0] = init;
}

}  // namespace gt

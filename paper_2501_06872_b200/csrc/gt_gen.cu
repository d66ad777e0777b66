// gt_gen.cu — seeded synthetic inputs for the BASELINE.json configs, generated
// on the device, plus COO -> sorted-CSR construction.  The RNG is a counter-
// based splitmix64 finalizer; paper_2501_06872_b200/gen.py is the identical
// numpy implementation (tests compare the two bit for bit).
#include <algorithm>
#include <cstdarg>
#include <string>

#include "../../include/gt.h"
#include "gt_common.cuh"

namespace gtgen {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSeedMul = 0xD1B54A32D192ED03ull;
constexpr uint64_t kStreamRmat = 1, kStreamPerm = 2, kStreamEr = 3, kStreamWdeg = 4, kStreamWedge = 5;
// floor(p * 2^32) for the R-MAT quadrant CDF a=.57, a+b=.76, a+b+c=.95
constexpr uint32_t kRmatA = 2448131358u, kRmatAB = 3264175144u, kRmatABC = 4080218931u;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * kSeedMul + stream * kGolden + 1);
}
__host__ __device__ __forceinline__ uint64_t hash_at(uint64_t key, uint64_t i) { return mix64(key + (i + 1) * kGolden); }

struct Feistel {
  uint64_t keys[4];
  int half;
  uint64_t mask;
  uint64_t n;
};
__device__ __forceinline__ uint64_t feistel_once(const Feistel& f, uint64_t x) {
  uint64_t L = x >> f.half, R = x & f.mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t t = L ^ (mix64(R ^ f.keys[r]) & f.mask);
    L = R;
    R = t;
  }
  return (L << f.half) | R;
}
__device__ __forceinline__ uint64_t feistel_perm(const Feistel& f, uint64_t x) {
  uint64_t y = feistel_once(f, x);
  while (y >= f.n) y = feistel_once(f, y);  // cycle walking
  return y;
}

__device__ __forceinline__ void rmat_edge(uint64_t e, uint64_t scale, uint64_t key, int permute, const Feistel& fp,
                                          uint64_t& s, uint64_t& d) {
  s = 0;
  d = 0;
  for (uint64_t l = 0; l < scale; l += 2) {
    const uint64_t h = hash_at(key, e * 16 + (l >> 1));
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (l + q >= scale) break;
      const uint32_t u = (uint32_t)(h >> (32 * q));
      const uint64_t bit = 1ull << (scale - 1 - (l + q));
      if (u < kRmatA) {
      } else if (u < kRmatAB) {
        d |= bit;
      } else if (u < kRmatABC) {
        s |= bit;
      } else {
        s |= bit;
        d |= bit;
      }
    }
  }
  if (permute) {
    s = feistel_perm(fp, s);
    d = feistel_perm(fp, d);
  }
}

// Two passes of the same counter-based R-MAT stream straight into a CSR
// (lists in generation order, not sorted): out-degree count, then placement.
__global__ void k_rmat_count(uint64_t scale, uint64_t E, uint64_t key, int permute, Feistel fp,
                             uint32_t* __restrict__ cnt) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    rmat_edge(e, scale, key, permute, fp, s, d);
    atomicAdd(&cnt[s], 1u);
  }
}
__global__ void k_rmat_place(uint64_t scale, uint64_t E, uint64_t key, int permute, Feistel fp,
                             const uint64_t* __restrict__ offs, uint32_t* __restrict__ fill,
                             uint32_t* __restrict__ edges) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    rmat_edge(e, scale, key, permute, fp, s, d);
    edges[offs[s] + atomicAdd(&fill[s], 1u)] = (uint32_t)d;
  }
}

__global__ void k_rmat(uint64_t scale, uint64_t E, uint64_t key, int permute, Feistel fp, uint32_t* __restrict__ src,
                       uint32_t* __restrict__ dst) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    rmat_edge(e, scale, key, permute, fp, s, d);
    src[e] = (uint32_t)s;
    dst[e] = (uint32_t)d;
  }
}

__global__ void k_er(uint64_t V, uint64_t E, uint64_t key, uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
    src[e] = (uint32_t)(((hash_at(key, 2 * e) >> 32) * V) >> 32);
    dst[e] = (uint32_t)(((hash_at(key, 2 * e + 1) >> 32) * V) >> 32);
  }
}

// first index i with u < cdf[i] (cdf non-decreasing, cdf[n-1] = 2^64-1)
__device__ __forceinline__ uint32_t cdf_rank(const uint64_t* __restrict__ cdf, uint32_t n, uint64_t u) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (u < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void k_web_deg(uint64_t V, uint64_t key, const uint64_t* __restrict__ cdf, uint32_t n, uint32_t sq,
                          uint32_t* __restrict__ deg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = (uint64_t)cdf_rank(cdf, n, hash_at(key, v)) + 1;
    const uint64_t d = (k * sq + 32768) >> 16;
    deg[v] = (uint32_t)(d ? d : 1);
  }
}

// one warp per source: its edges in generation order
__global__ void k_web_edges(uint64_t V, uint64_t key, const uint64_t* __restrict__ offs,
                            const uint64_t* __restrict__ hcdf, uint32_t nh, const uint32_t* __restrict__ hubs,
                            uint32_t window, uint32_t plocal, uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t span = 2ull * window + 1;
  for (uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; v < V; v += nwarps) {
    const uint64_t e0 = offs[v], e1 = offs[v + 1];
    for (uint64_t e = e0 + lane; e < e1; e += 32) {
      const uint64_t ha = hash_at(key, 2 * e), hb = hash_at(key, 2 * e + 1);
      uint32_t d;
      if ((uint32_t)ha < plocal) {
        const uint64_t off = ((ha >> 32) * span) >> 32;
        d = (uint32_t)((v + V - window + off) % V);
      } else {
        d = hubs[cdf_rank(hcdf, nh, hb)];
      }
      src[e] = (uint32_t)v;
      dst[e] = d;
    }
  }
}

__global__ void k_hist(const uint32_t* __restrict__ key, uint64_t E, uint32_t* __restrict__ cnt) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[key[e]], 1u);
}
__global__ void k_copy_u64(const uint64_t* __restrict__ a, uint64_t* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void k_group(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val, uint64_t E,
                        unsigned long long* __restrict__ cur, uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x)
    out[atomicAdd(&cur[key[e]], 1ull)] = val[e];
}

}  // namespace gtgen

using namespace gtgen;

namespace {
thread_local std::string g_gen_err;
}

extern "C" {
const char* gt_last_error(void);

static int gen_fail(cudaError_t e) {
  return e == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA;
}

int gt_gen_rmat(uint64_t scale, uint64_t E, uint64_t seed, int permute, uint32_t* src, uint32_t* dst, void* stream) {
  if (scale < 1 || scale > 32 || (E && (!src || !dst))) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Feistel fp{};
  const uint64_t V = 1ull << scale;
  const int width = (int)(scale + (scale & 1));
  fp.half = width / 2;
  fp.mask = (1ull << fp.half) - 1;
  fp.n = V;
  const uint64_t pk = stream_key(seed, kStreamPerm);
  for (int r = 0; r < 4; ++r) fp.keys[r] = hash_at(pk, (uint64_t)r);
  if (E) k_rmat<<<148 * 16, 256, 0, st>>>(scale, E, stream_key(seed, kStreamRmat), permute, fp, src, dst);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GT_OK : gen_fail(e);
}

static Feistel make_feistel(uint64_t scale, uint64_t seed) {
  Feistel fp{};
  const int width = (int)(scale + (scale & 1));
  fp.half = width / 2;
  fp.mask = (1ull << fp.half) - 1;
  fp.n = 1ull << scale;
  const uint64_t pk = stream_key(seed, kStreamPerm);
  for (int r = 0; r < 4; ++r) fp.keys[r] = hash_at(pk, (uint64_t)r);
  return fp;
}

int gt_gen_rmat_csr(uint64_t scale, uint64_t E, uint64_t seed, int permute, uint64_t* offsets, uint32_t* edges,
                    void* stream) {
  if (scale < 1 || scale > 32 || !offsets || (E && !edges)) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t V = 1ull << scale;
  const Feistel fp = make_feistel(scale, seed);
  const uint64_t key = stream_key(seed, kStreamRmat);
  uint32_t* cnt = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, V * 4, st);
  if (e != cudaSuccess) return gen_fail(e);
  int rc = GT_OK;
  cudaMemsetAsync(cnt, 0, V * 4, st);
  if (E) k_rmat_count<<<148 * 16, 256, 0, st>>>(scale, E, key, permute, fp, cnt);
  rc = gt_prefix_sum(cnt, V, offsets, st);
  if (rc == GT_OK && E) {
    cudaMemsetAsync(cnt, 0, V * 4, st);
    k_rmat_place<<<148 * 16, 256, 0, st>>>(scale, E, key, permute, fp, offsets, cnt, edges);
    if ((e = cudaGetLastError()) != cudaSuccess) rc = gen_fail(e);
  }
  cudaFreeAsync(cnt, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && rc == GT_OK) rc = gen_fail(e);
  return rc;
}

int gt_gen_er(uint64_t V, uint64_t E, uint64_t seed, uint32_t* src, uint32_t* dst, void* stream) {
  if (V < 1 || V > (1ull << 32) || (E && (!src || !dst))) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (E) k_er<<<148 * 16, 256, 0, st>>>(V, E, stream_key(seed, kStreamEr), src, dst);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GT_OK : gen_fail(e);
}

int gt_gen_web_degrees(uint64_t V, uint64_t seed, const uint64_t* deg_cdf, uint32_t ndeg, uint32_t sq,
                       uint64_t* offsets, uint64_t* num_edges, void* stream) {
  if (V < 1 || V > (1ull << 32) || !deg_cdf || ndeg < 1 || !offsets || !num_edges) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* deg = nullptr;
  cudaError_t e = cudaMallocAsync(&deg, V * 4, st);
  if (e != cudaSuccess) return gen_fail(e);
  k_web_deg<<<148 * 16, 256, 0, st>>>(V, stream_key(seed, kStreamWdeg), deg_cdf, ndeg, sq, deg);
  int rc = gt_prefix_sum(deg, V, offsets, st);
  if (rc == GT_OK) {
    if ((e = cudaMemcpyAsync(num_edges, offsets + V, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) rc = gen_fail(e);
  }
  cudaFreeAsync(deg, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && rc == GT_OK) rc = gen_fail(e);
  return rc;
}

int gt_gen_web_edges(uint64_t V, uint64_t seed, const uint64_t* offsets, const uint64_t* hub_cdf, uint32_t nhub,
                     const uint32_t* hubs, uint32_t window, uint32_t plocal, uint32_t* src, uint32_t* dst,
                     void* stream) {
  if (V < 1 || V > (1ull << 32) || !offsets || !hub_cdf || nhub < 1 || !hubs || !src || !dst) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_web_edges<<<148 * 32, 256, 0, st>>>(V, stream_key(seed, kStreamWedge), offsets, hub_cdf, nhub, hubs, window,
                                        plocal, src, dst);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GT_OK : gen_fail(e);
}

// COO -> CSR with ascending lists: group by destination (unordered), then the
// stable transpose of that reverse-CSR sorts every source list by destination.
int gt_build_csr(uint32_t* src, uint32_t* dst, uint64_t V, uint64_t E, uint64_t* offsets, uint32_t* edges,
                 void* stream) {
  if (V < 1 || !offsets || (E && (!src || !dst || !edges))) return GT_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* cnt = nullptr;
  uint64_t* roff = nullptr;
  unsigned long long* cur = nullptr;
  uint32_t* redges = nullptr;
  cudaError_t e;
  int rc = GT_OK;
  if ((e = cudaMallocAsync(&cnt, V * 4, st)) != cudaSuccess || (e = cudaMallocAsync(&roff, (V + 1) * 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&cur, V * 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&redges, std::max<uint64_t>(E, 1) * 4, st)) != cudaSuccess) {
    rc = gen_fail(e);
  } else {
    cudaMemsetAsync(cnt, 0, V * 4, st);
    k_hist<<<148 * 16, 256, 0, st>>>(dst, E, cnt);
    rc = gt_prefix_sum(cnt, V, roff, st);
    if (rc == GT_OK) {
      k_copy_u64<<<148 * 8, 256, 0, st>>>(roff, reinterpret_cast<uint64_t*>(cur), V);
      k_group<<<148 * 16, 256, 0, st>>>(dst, src, E, cur, redges);
      if ((e = cudaGetLastError()) != cudaSuccess) rc = gen_fail(e);
    }
    if (rc == GT_OK) rc = gt_transpose(roff, redges, V, E, offsets, edges, nullptr, 0, st, nullptr);
  }
  cudaStreamSynchronize(st);
  cudaFree(cnt);
  cudaFree(roff);
  cudaFree(cur);
  cudaFree(redges);
  return rc;
}

}  // extern "C"

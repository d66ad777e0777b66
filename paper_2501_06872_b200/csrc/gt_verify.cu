// gt_verify.cu — GPU canonicalisation and output verification.
//
// * gt_sort_lists replaces sort_neighbor_lists / _sort_segments
//   (baselines.py:448-475): every list ascending.  It is the transpose applied
//   twice: T(g) lists sources ascending per destination, and T(T(g)) lists,
//   for every vertex, its neighbours ascending with multiplicity — the same
//   offsets as g and each list sorted, by the stable kernels of gt_api.cu.
// * gt_verify_transpose: an independent GPU transpose for verify_output's
//   full-oracle mode — the exact offsets (bincount + cumsum) and a global radix
//   sort (CUB, library code) of destination << 32 | source keys, i.e.
//   transpose_oracle's lexsort (graph.py:136-148) with none of the partition
//   kernels it checks.
// * gt_first_diff_* / gt_in_degree_offsets / gt_first_diff_lists are the
//   device halves of verify_output (bench.py:91-170): first differing offset
//   or edge index (_first_mismatch_vertex, bench.py:91-99), the exact
//   t_offsets = bincount + cumsum of the input's edges (bench.py:140-148), and
//   the first sampled vertex whose (canonical) neighbour list differs
//   (bench.py:150-170).  First-index reductions use atomicMin, so the reported
//   index equals np.nonzero(...)[0][0].
#include <algorithm>
#include <cstdint>

#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include "../../include/gt.h"

int gt_internal_set_err(int code, const char* msg);  // gt_api.cu

namespace {

template <typename T>
__global__ void k_first_diff(const T* __restrict__ a, const T* __restrict__ b, uint64_t n,
                             unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) {
      atomicMin(first, (unsigned long long)i);
      return;  // later indices of this thread are larger
    }
}

__global__ void k_degree_hist(const uint32_t* __restrict__ e, uint64_t E, uint32_t* __restrict__ cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[e[i]], 1u);
}

// warp per listed vertex: does list a[v] differ from list b[v]?
__global__ void k_first_diff_lists(const uint64_t* __restrict__ oa, const uint32_t* __restrict__ ea,
                                   const uint64_t* __restrict__ ob, const uint32_t* __restrict__ eb,
                                   const uint32_t* __restrict__ verts, uint64_t nv, unsigned long long* first) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t j = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < nv; j += warps) {
    const uint32_t v = verts[j];
    const uint64_t a0 = oa[v], a1 = oa[v + 1], b0 = ob[v], b1 = ob[v + 1];
    bool diff = (a1 - a0) != (b1 - b0);
    for (uint64_t q = lane; !diff && q < a1 - a0; q += 32) diff = ea[a0 + q] != eb[b0 + q];
    if (__any_sync(0xffffffffu, diff)) {
      if (lane == 0) atomicMin(first, (unsigned long long)j);
    }
  }
}

// key of edge i (stream position): destination << 32 | source, the source by
// binary search over the offsets (largest v with offsets[v] <= i)
__global__ void k_edge_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ e, uint64_t V, uint64_t E,
                            uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = V;
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (off[mid] <= i) lo = mid; else hi = mid;
    }
    keys[i] = ((uint64_t)e[i] << 32) | lo;
  }
}

__global__ void k_low_words(const uint64_t* __restrict__ keys, uint64_t E, uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)keys[i];
}

// ---- debug checks (transpose_potra(debug=True) / transpose_gpu(debug=True))
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// warp per source: h[d] += mix(s) for every edge (s, d)
__global__ void k_hash_in(const uint64_t* __restrict__ off, const uint32_t* __restrict__ e, uint64_t V,
                          unsigned long long* __restrict__ h) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t s = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < V; s += warps) {
    const uint64_t m = mix64(s);
    for (uint64_t j = off[s] + lane; j < off[s + 1]; j += 32) atomicAdd(&h[e[j]], (unsigned long long)m);
  }
}
// warp per destination: h[d] -= mix(t_edges[j]) over its list; descents and
// sentinels (slots never written) counted
__global__ void k_hash_out(const uint64_t* __restrict__ toff, const uint32_t* __restrict__ te, uint64_t V,
                           unsigned long long* __restrict__ h, unsigned long long* __restrict__ cnt) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t d = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); d < V; d += warps) {
    unsigned long long acc = 0, unwritten = 0, desc = 0;
    const uint64_t a = toff[d], b = toff[d + 1];
    for (uint64_t j = a + lane; j < b; j += 32) {
      const uint32_t x = te[j];
      if (x == 0xffffffffu) ++unwritten;
      else acc += mix64(x);
      if (j + 1 < b && te[j + 1] < x) ++desc;
    }
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      unwritten += __shfl_xor_sync(0xffffffffu, unwritten, o);
      desc += __shfl_xor_sync(0xffffffffu, desc, o);
    }
    if (lane == 0) {
      h[d] -= acc;
      if (unwritten) atomicAdd(&cnt[0], unwritten);
      if (desc) atomicAdd(&cnt[1], desc);
    }
  }
}
__global__ void k_first_nonzero(const unsigned long long* __restrict__ h, uint64_t n, unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (h[i]) {
      atomicMin(first, (unsigned long long)i);
      return;
    }
}

int cuda_fail(cudaError_t e) {
  return gt_internal_set_err(e == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA, cudaGetErrorString(e));
}

template <typename T>
int first_diff(const T* a, const T* b, uint64_t n, uint64_t* first, void* stream) {
  if (!first || (n && (!a || !b))) return gt_internal_set_err(GT_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8, st);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaMemsetAsync(d, 0xff, 8, st);
  if (n) k_first_diff<T><<<148 * 8, 256, 0, st>>>(a, b, n, d);
  unsigned long long h = ~0ull;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return cuda_fail(e);
  *first = (h == ~0ull) ? n : (uint64_t)h;
  return GT_OK;
}

}  // namespace

extern "C" {

int gt_sort_lists(const uint64_t* offsets, const uint32_t* edges, uint64_t V, uint64_t E, uint32_t* out_edges,
                  void* stream) {
  if (!offsets || (E && (!edges || !out_edges))) return gt_internal_set_err(GT_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t* t_off = nullptr;
  uint32_t* t_edg = nullptr;
  uint64_t* tt_off = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&t_off, (V + 1) * 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&t_edg, std::max<uint64_t>(E, 1) * 4, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&tt_off, (V + 1) * 8, st)) != cudaSuccess) {
    cudaFreeAsync(t_off, st);
    cudaFreeAsync(t_edg, st);
    return cuda_fail(e);
  }
  int rc = gt_transpose(offsets, edges, V, E, t_off, t_edg, nullptr, 0, st, nullptr);
  if (rc == GT_OK) rc = gt_transpose(t_off, t_edg, V, E, tt_off, out_edges, nullptr, 0, st, nullptr);
  cudaFreeAsync(t_off, st);
  cudaFreeAsync(t_edg, st);
  cudaFreeAsync(tt_off, st);
  if (rc == GT_OK && (e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
  return rc;
}

int gt_verify_transpose(const uint64_t* offsets, const uint32_t* edges, uint64_t V, uint64_t E, uint64_t* t_offsets,
                        uint32_t* t_edges, void* stream) {
  if (!offsets || !t_offsets || (E && (!edges || !t_edges))) return gt_internal_set_err(GT_EINVAL, "null argument");
  if (V == 0 || V >= (1ull << 32)) return gt_internal_set_err(GT_EINVAL, "num_vertices must be in [1, 2^32)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = gt_in_degree_offsets(edges, E, V, t_offsets, st);
  if (rc != GT_OK || E == 0) return rc;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  int bits = 1;
  while (bits < 32 && (1ull << bits) < V) ++bits;
  if ((e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, E, 0, 32 + bits, st)) != cudaSuccess)
    return cuda_fail(e);
  if ((e = cudaMallocAsync(&k0, E * 8, st)) != cudaSuccess || (e = cudaMallocAsync(&k1, E * 8, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&tmp, tmp_bytes, st)) != cudaSuccess) {
    cudaFreeAsync(k0, st);
    cudaFreeAsync(k1, st);
    return cuda_fail(e);
  }
  k_edge_keys<<<148 * 16, 256, 0, st>>>(offsets, edges, V, E, k0);
  e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, E, 0, 32 + bits, st);
  if (e == cudaSuccess) k_low_words<<<148 * 16, 256, 0, st>>>(k1, E, t_edges);
  cudaFreeAsync(k0, st);
  cudaFreeAsync(k1, st);
  cudaFreeAsync(tmp, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  return GT_OK;
}

int gt_debug_check(const uint64_t* offsets, const uint32_t* edges, uint64_t V, uint64_t E, const uint64_t* t_offsets,
                   const uint32_t* t_edges, gt_debug_report* report, void* stream) {
  if (!offsets || !t_offsets || !report || (E && (!edges || !t_edges))) return gt_internal_set_err(GT_EINVAL, "null argument");
  if (V == 0 || V >= (1ull << 32) || E >= (1ull << 32)) return gt_internal_set_err(GT_EINVAL, "debug check: size out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  report->unwritten = report->descents = 0;
  report->offset_diff = V + 1;
  report->multiset_diff = V;
  uint64_t* exp_off = nullptr;
  unsigned long long* h = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&exp_off, (V + 1) * 8, st)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaMallocAsync(&h, (V + 3) * 8, st)) != cudaSuccess) {
    cudaFreeAsync(exp_off, st);
    return cuda_fail(e);
  }
  int rc = gt_in_degree_offsets(edges, E, V, exp_off, st);
  uint64_t first = V + 1;
  if (rc == GT_OK) rc = gt_first_diff_u64(exp_off, t_offsets, V + 1, &first, st);
  if (rc == GT_OK) {
    report->offset_diff = first;
    if (first == V + 1) {  // lists are delimited correctly: hash them against the input
      cudaMemsetAsync(h, 0, (V + 3) * 8, st);
      k_hash_in<<<148 * 8, 256, 0, st>>>(offsets, edges, V, h);
      k_hash_out<<<148 * 8, 256, 0, st>>>(t_offsets, t_edges, V, h, h + V);
      cudaMemsetAsync(h + V + 2, 0xff, 8, st);
      k_first_nonzero<<<148 * 8, 256, 0, st>>>(h, V, h + V + 2);
      unsigned long long tail[3];
      cudaMemcpyAsync(tail, h + V, 24, cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) rc = cuda_fail(e);
      report->unwritten = tail[0];
      report->descents = tail[1];
      report->multiset_diff = (tail[2] == ~0ull) ? V : tail[2];
    }
  }
  cudaFreeAsync(exp_off, st);
  cudaFreeAsync(h, st);
  cudaStreamSynchronize(st);
  return rc;
}

int gt_first_diff_u64(const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t* first, void* stream) {
  return first_diff<uint64_t>(a, b, n, first, stream);
}

int gt_first_diff_u32(const uint32_t* a, const uint32_t* b, uint64_t n, uint64_t* first, void* stream) {
  return first_diff<uint32_t>(a, b, n, first, stream);
}

int gt_in_degree_offsets(const uint32_t* edges, uint64_t E, uint64_t V, uint64_t* offsets, void* stream) {
  if (!offsets || (E && !edges)) return gt_internal_set_err(GT_EINVAL, "null argument");
  if (V >= (1ull << 32)) return gt_internal_set_err(GT_EINVAL, "num_vertices must be < 2^32");
  if (E >= (1ull << 32)) return gt_internal_set_err(GT_EOVERFLOW, "in-degree counters are 32-bit (E >= 2^32)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* cnt = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, std::max<uint64_t>(V, 1) * 4, st);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaMemsetAsync(cnt, 0, std::max<uint64_t>(V, 1) * 4, st);
  if (E) k_degree_hist<<<148 * 16, 256, 0, st>>>(edges, E, cnt);
  int rc = gt_prefix_sum(cnt, V, offsets, st);
  cudaFreeAsync(cnt, st);
  if (rc == GT_OK && (e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
  return rc;
}

int gt_first_diff_lists(const uint64_t* off_a, const uint32_t* edges_a, const uint64_t* off_b,
                        const uint32_t* edges_b, const uint32_t* vertices, uint64_t n_vertices, uint64_t* first,
                        void* stream) {
  if (!first || (n_vertices && (!off_a || !off_b || !vertices))) return gt_internal_set_err(GT_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8, st);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaMemsetAsync(d, 0xff, 8, st);
  if (n_vertices) k_first_diff_lists<<<148 * 4, 256, 0, st>>>(off_a, edges_a, off_b, edges_b, vertices, n_vertices, d);
  unsigned long long h = ~0ull;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return cuda_fail(e);
  *first = (h == ~0ull) ? n_vertices : (uint64_t)h;
  return GT_OK;
}

}  // extern "C"

// gt_hdv.cu — GPU step 0: the high-degree-vertex sample.
//
// * gt_sample_hdv restates sample_hdv (hlh.py:167-218) with _sample_tally
//   (hlh.py:153-164): 2 * workers xoshiro256** streams seeded by successive
//   splitmix64 outputs of `seed` (worker_seeds, _nb.py:86-93), stream w of a
//   tally drawing samples [w*N/workers, (w+1)*N/workers) as edges[r % E] and
//   counting the endpoint; the first `workers` streams choose the set, the
//   other `workers` score it (coverage estimate).  N = 0 means exhaustive
//   (sample_fraction == 1): both tallies are the in-degree histogram.  The
//   top-k order is the reference's lexsort((id, -freq)): by descending count,
//   ties to the lower ID, then zero-count vertices in ascending ID order.
//   Tallies are sums, so the result does not depend on the order the GPU
//   threads run in: it equals the reference's for the same (seed, workers).
// * Each stream is walked once by one thread that only steps the generator
//   and records its state every kCk draws; one thread per checkpoint then
//   replays kCk draws and issues the loads and atomics (the serial part is
//   ALU-only).
// * The ordering is two stable counting sorts by 16-bit digits of
//   (fmax - count), each one call of the transpose kernels (gt_transpose on
//   a one-edge-per-source graph), over the compacted nonzero counts.
// * gt_hdv_table_build / gt_hdv_lookup: the open-addressing table of the plan
//   (_table_build / _table_find, hlh.py:68-90): Fibonacci hash
//   (key * 0x9E3779B97F4A7C15) >> shift, linear probing, value = position in
//   hdv_ids.  Built with atomicCAS (the slot layout may differ from a serial
//   build; every lookup answers the same).
// * gt_coverage_exact: coverage_exact (hlh.py:221-228), the exact fraction
//   of edges whose endpoint is in the set.
#include <algorithm>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gt.h"

int gt_internal_set_err(int code, const char* msg);  // gt_api.cu

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kCk = 256;  // draws per checkpoint

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Xo {
  uint64_t s0, s1, s2, s3;
  __device__ __forceinline__ void seed(uint64_t x) {  // xoshiro_seed_scalar (_nb.py:62-69)
    x += kGamma;
    s0 = mix64(x);
    x += kGamma;
    s1 = mix64(x);
    x += kGamma;
    s2 = mix64(x);
    x += kGamma;
    s3 = mix64(x);
  }
  __device__ __forceinline__ uint64_t next() {  // xoshiro_step (_nb.py:72-83)
    const uint64_t r = rotl64(s1 * 5, 7) * 9;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return r;
  }
};

// stream s in [0, 2 * workers): tally s / workers, worker s % workers
__device__ __forceinline__ void stream_range(uint64_t s, uint64_t workers, uint64_t N, uint64_t* lo, uint64_t* hi) {
  const uint64_t w = s % workers;
  *lo = (uint64_t)(((unsigned __int128)w * N) / workers);
  *hi = (uint64_t)(((unsigned __int128)(w + 1) * N) / workers);
}

__global__ void k_hdv_ckpt(uint64_t seed, uint64_t workers, uint64_t N, uint64_t maxc, Xo* __restrict__ ck) {
  const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s >= 2 * workers) return;
  Xo x;
  x.seed(mix64(seed + (s + 1) * kGamma));  // worker_seeds: the (s+1)-th splitmix64 output of seed
  uint64_t lo, hi;
  stream_range(s, workers, N, &lo, &hi);
  Xo* out = ck + s * maxc;
  for (uint64_t i = 0; i < hi - lo; ++i) {
    if (i % kCk == 0) out[i / kCk] = x;
    x.next();
  }
}

__global__ void k_hdv_tally(const uint32_t* __restrict__ edges, uint64_t E, uint64_t workers, uint64_t N, uint64_t maxc,
                            const Xo* __restrict__ ck, uint32_t* __restrict__ freq, uint32_t* __restrict__ est,
                            uint64_t V) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t s = t / maxc, j = t % maxc;
  if (s >= 2 * workers) return;
  uint64_t lo, hi;
  stream_range(s, workers, N, &lo, &hi);
  const uint64_t b = j * kCk;
  if (b >= hi - lo) return;
  const uint64_t n = min(kCk, hi - lo - b);
  Xo x = ck[t];
  uint32_t* cnt = (s < workers) ? freq : est;
  for (uint64_t q = 0; q < n; ++q) {
    const uint64_t r = x.next();
    const uint32_t e = __ldg(edges + (r % E));
    if (e < V) atomicAdd(&cnt[e], 1u);
  }
}

__global__ void k_hdv_degree(const uint32_t* __restrict__ e, uint64_t E, uint32_t* __restrict__ cnt, uint64_t V) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = e[i];
    if (v < V) atomicAdd(&cnt[v], 1u);
  }
}

__global__ void k_hdv_flags(const uint32_t* __restrict__ freq, uint64_t V, uint32_t* __restrict__ flag,
                            unsigned int* __restrict__ fmax) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = freq[v];
    flag[v] = f != 0;
    if (f) atomicMax(fmax, f);
  }
}

// nonzero counts compacted in ID order; zero-count vertices fill hdv slots
// m + (v - pos[v]) when that is < k (ascending ID after every nonzero one)
__global__ void k_hdv_compact(const uint32_t* __restrict__ freq, uint64_t V, const uint64_t* __restrict__ pos,
                              uint32_t* __restrict__ ids, uint32_t* __restrict__ f, uint64_t k,
                              uint64_t* __restrict__ hdv) {
  const uint64_t m = pos[V];
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = pos[v];
    if (freq[v]) {
      ids[p] = (uint32_t)v;
      f[p] = freq[v];
    } else if (m + (v - p) < k) {
      hdv[m + (v - p)] = v;
    }
  }
}

// one-edge-per-source CSR: offsets[i] = min(i, m), edge = digit of element i
__global__ void k_hdv_digits(const uint32_t* __restrict__ f, uint64_t m, uint32_t fmax, int shift,
                             uint64_t nv, uint64_t* __restrict__ off, uint32_t* __restrict__ dig) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nv; i += (uint64_t)gridDim.x * blockDim.x) {
    off[i] = min(i, m);
    if (i < m) dig[i] = ((fmax - f[i]) >> shift) & 0xffffu;
  }
}

__global__ void k_hdv_gather(const uint32_t* __restrict__ perm, uint64_t m, const uint32_t* __restrict__ ids,
                             const uint32_t* __restrict__ f, uint32_t* __restrict__ ids2, uint32_t* __restrict__ f2) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    ids2[i] = ids[p];
    f2[i] = f[p];
  }
}

__global__ void k_hdv_head(const uint32_t* __restrict__ ids, uint64_t n, uint64_t* __restrict__ hdv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    hdv[i] = ids[i];
}

__global__ void k_hdv_hits(const uint64_t* __restrict__ hdv, uint64_t k, const uint32_t* __restrict__ est,
                           unsigned long long* __restrict__ hits) {
  unsigned long long s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
    s += est[hdv[i]];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(hits, s);
}

__global__ void k_table_build(const uint64_t* __restrict__ ids, uint64_t k, uint64_t cap, int shift,
                              unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t mask = cap - 1;
  for (uint64_t n = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; n < k; n += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ids[n];
    uint64_t i = (key * kGold) >> shift;
    while (atomicCAS(&keys[i & mask], (unsigned long long)kEmpty, (unsigned long long)key) != kEmpty) ++i;
    vals[i & mask] = (uint32_t)n;
  }
}

__device__ __forceinline__ int64_t table_find(const unsigned long long* keys, const uint32_t* vals, uint64_t cap,
                                              int shift, uint64_t key) {
  const uint64_t mask = cap - 1;
  uint64_t i = (key * kGold) >> shift;
  while (true) {
    const uint64_t k = keys[i & mask];
    if (k == key) return (int64_t)vals[i & mask];
    if (k == kEmpty) return -1;
    ++i;
  }
}

__global__ void k_table_lookup(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                               uint64_t cap, int shift, const uint32_t* __restrict__ q, uint64_t n,
                               int64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = table_find(keys, vals, cap, shift, q[i]);
}

__global__ void k_coverage(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                           uint64_t cap, int shift, const uint32_t* __restrict__ e, uint64_t E,
                           unsigned long long* __restrict__ hits) {
  unsigned long long s = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
    s += table_find(keys, vals, cap, shift, e[i]) >= 0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(hits, s);
}

int cuda_fail(cudaError_t e) {
  return gt_internal_set_err(e == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA, cudaGetErrorString(e));
}

struct Pool {  // stream-ordered temporaries, freed on scope exit
  cudaStream_t st;
  void* p[16] = {};
  int n = 0;
  explicit Pool(cudaStream_t s) : st(s) {}
  ~Pool() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], st);
  }
  template <typename T>
  cudaError_t get(T** out, uint64_t count) {
    void* q = nullptr;
    const cudaError_t e = cudaMallocAsync(&q, std::max<uint64_t>(count, 1) * sizeof(T), st);
    if (e == cudaSuccess) p[n++] = q;
    *out = static_cast<T*>(q);
    return e;
  }
};

unsigned grid_for(uint64_t n, unsigned tpb) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + tpb - 1) / tpb, 148 * 32)); }

}  // namespace

extern "C" {

int gt_sample_hdv(const uint32_t* edges, uint64_t num_edges, uint64_t num_vertices, uint64_t k,
                  uint64_t num_samples, uint64_t seed, int workers, uint64_t* hdv_ids, uint64_t* h_hits,
                  void* stream) {
  const uint64_t E = num_edges, V = num_vertices;
  if (!h_hits || (k && !hdv_ids) || (E && !edges)) return gt_internal_set_err(GT_EINVAL, "gt_sample_hdv: null argument");
  if (workers < 1) return gt_internal_set_err(GT_EINVAL, "gt_sample_hdv: workers must be >= 1");
  if (k > V) return gt_internal_set_err(GT_EINVAL, "gt_sample_hdv: k > num_vertices");
  if (V >= (1ull << 32)) return gt_internal_set_err(GT_EINVAL, "gt_sample_hdv: num_vertices must be < 2^32");
  if (num_samples == 0 && E >= (1ull << 32))
    return gt_internal_set_err(GT_EOVERFLOW, "gt_sample_hdv: exhaustive counts are 32-bit (E >= 2^32)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  *h_hits = 0;
  if (k == 0) return GT_OK;
  Pool pool(st);
  cudaError_t e;
  uint32_t *freq = nullptr, *est = nullptr, *flag = nullptr;
  uint64_t* pos = nullptr;
  unsigned int* d_fmax = nullptr;
  unsigned long long* d_hits = nullptr;
  if ((e = pool.get(&freq, V)) != cudaSuccess || (e = pool.get(&flag, V)) != cudaSuccess ||
      (e = pool.get(&pos, V + 1)) != cudaSuccess || (e = pool.get(&d_fmax, 1)) != cudaSuccess ||
      (e = pool.get(&d_hits, 1)) != cudaSuccess)
    return cuda_fail(e);
  cudaMemsetAsync(freq, 0, V * 4, st);
  cudaMemsetAsync(d_fmax, 0, 4, st);
  cudaMemsetAsync(d_hits, 0, 8, st);
  const bool exhaustive = num_samples == 0 || E == 0;
  if (exhaustive) {
    est = freq;
    if (E) k_hdv_degree<<<grid_for(E, 256), 256, 0, st>>>(edges, E, freq, V);
  } else {
    if ((e = pool.get(&est, V)) != cudaSuccess) return cuda_fail(e);
    cudaMemsetAsync(est, 0, V * 4, st);
    const uint64_t W = (uint64_t)workers, N = num_samples;
    const uint64_t maxc = (N / W + 1 + kCk - 1) / kCk;
    Xo* ck = nullptr;
    if ((e = pool.get(&ck, 2 * W * maxc)) != cudaSuccess) return cuda_fail(e);
    k_hdv_ckpt<<<(unsigned)((2 * W + 127) / 128), 128, 0, st>>>(seed, W, N, maxc, ck);
    const uint64_t nt = 2 * W * maxc;
    k_hdv_tally<<<(unsigned)((nt + 127) / 128), 128, 0, st>>>(edges, E, W, N, maxc, ck, freq, est, V);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e);
  k_hdv_flags<<<grid_for(V, 256), 256, 0, st>>>(freq, V, flag, d_fmax);
  int rc = gt_prefix_sum(flag, V, pos, st);
  if (rc) return rc;
  uint64_t m = 0;
  uint32_t fmax = 0;
  cudaMemcpyAsync(&m, pos + V, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&fmax, d_fmax, 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
  uint32_t *ids = nullptr, *f = nullptr;
  if ((e = pool.get(&ids, m)) != cudaSuccess || (e = pool.get(&f, m)) != cudaSuccess) return cuda_fail(e);
  k_hdv_compact<<<grid_for(V, 256), 256, 0, st>>>(freq, V, pos, ids, f, k, hdv_ids);
  if (m > 1 && fmax > 0) {
    // stable counting sorts by 16-bit digits of (fmax - count), low digit first
    const uint64_t nv = std::max<uint64_t>(m, 1ull << 16);
    uint64_t *off = nullptr, *toff = nullptr;
    uint32_t *dig = nullptr, *perm = nullptr, *ids2 = nullptr, *f2 = nullptr;
    if ((e = pool.get(&off, nv + 1)) != cudaSuccess || (e = pool.get(&toff, nv + 1)) != cudaSuccess ||
        (e = pool.get(&dig, m)) != cudaSuccess || (e = pool.get(&perm, m)) != cudaSuccess ||
        (e = pool.get(&ids2, m)) != cudaSuccess || (e = pool.get(&f2, m)) != cudaSuccess)
      return cuda_fail(e);
    for (int shift = 0; shift < 32; shift += 16) {
      if (shift && (fmax >> 16) == 0) break;  // every key fits the low digit
      k_hdv_digits<<<grid_for(nv + 1, 256), 256, 0, st>>>(f, m, fmax, shift, nv, off, dig);
      if ((rc = gt_transpose(off, dig, nv, m, toff, perm, nullptr, 0, st, nullptr))) return rc;
      k_hdv_gather<<<grid_for(m, 256), 256, 0, st>>>(perm, m, ids, f, ids2, f2);
      std::swap(ids, ids2);
      std::swap(f, f2);
    }
  }
  k_hdv_head<<<grid_for(std::min(k, m), 256), 256, 0, st>>>(ids, std::min(k, m), hdv_ids);
  k_hdv_hits<<<grid_for(k, 256), 256, 0, st>>>(hdv_ids, k, est, d_hits);
  unsigned long long hits = 0;
  cudaMemcpyAsync(&hits, d_hits, 8, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e);
  *h_hits = hits;
  return GT_OK;
}

int gt_hdv_table_build(const uint64_t* hdv_ids, uint64_t k, uint64_t capacity, int shift, uint64_t* keys,
                       uint32_t* vals, void* stream) {
  if (!keys || !vals || (k && !hdv_ids)) return gt_internal_set_err(GT_EINVAL, "gt_hdv_table_build: null argument");
  if (capacity < 2 || (capacity & (capacity - 1)) || k >= capacity)
    return gt_internal_set_err(GT_EINVAL, "gt_hdv_table_build: capacity must be a power of two > k");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(keys, 0xff, capacity * 8, st);
  cudaMemsetAsync(vals, 0, capacity * 4, st);
  if (k)
    k_table_build<<<grid_for(k, 256), 256, 0, st>>>(hdv_ids, k, capacity, shift,
                                                    reinterpret_cast<unsigned long long*>(keys), vals);
  const cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? GT_OK : cuda_fail(e);
}

int gt_hdv_lookup(const uint64_t* keys, const uint32_t* vals, uint64_t capacity, int shift, const uint32_t* queries,
                  uint64_t n, int64_t* out, void* stream) {
  if (!keys || !vals || (n && (!queries || !out))) return gt_internal_set_err(GT_EINVAL, "gt_hdv_lookup: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n)
    k_table_lookup<<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(keys), vals, capacity,
                                                     shift, queries, n, out);
  const cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? GT_OK : cuda_fail(e);
}

int gt_coverage_exact(const uint64_t* keys, const uint32_t* vals, uint64_t capacity, int shift, const uint32_t* edges,
                      uint64_t num_edges, uint64_t* h_hits, void* stream) {
  if (!keys || !vals || !h_hits || (num_edges && !edges))
    return gt_internal_set_err(GT_EINVAL, "gt_coverage_exact: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8, st);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaMemsetAsync(d, 0, 8, st);
  if (num_edges)
    k_coverage<<<grid_for(num_edges, 256), 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(keys), vals,
                                                         capacity, shift, edges, num_edges, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return cuda_fail(e);
  *h_hits = h;
  return GT_OK;
}

}  // extern "C"

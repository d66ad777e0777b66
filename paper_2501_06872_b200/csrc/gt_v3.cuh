// gt_v3.cuh — lean three-level stable partition (compact 4-byte records).
//
// Contract: CSR -> CSC, every list ascending by source (= transpose_oracle,
// graph.py:136-148 = a stable counting sort of the CSR edge stream by
// destination), planned so that every level is one streaming partition pass
// with a short instruction path per record:
//
//   L1  k_c1 count  -> lookback scan -> k_p1 place
//         CSR edges -> R1 = (dst_low << L | src_low) grouped by coarse digit A,
//         written into t_edges (the output buffer doubles as R1 storage).
//         Sources come from per-tile boundary marks (one per source that starts
//         in the tile) resolved with one ballot per 32-edge slot.
//   L2  k_cnt_rec count -> k_scan_lookback + k_segfix -> k_p2 place
//         each coarse bucket is cut into count tiles; a per-bucket column scan
//         gives every (tile, fine digit B) its final CSC position, so L2 writes
//         R2 = (lv << nbs | src) fine-bucket-major into the workspace: a fine
//         bucket's records are contiguous and already sit at their CSC range.
//   L3  k_p3 units (runs of small fine buckets, TMA in, rank by local vertex,
//         stage in place, TMA out to t_edges, CSC offsets) and, for fine
//         buckets above the unit capacity, the same count/scan/place trio as L2
//         with the low digit C (k_cnt_rec / k_scan_lookback + k_segfix / k_p2<DecR2>).
//
// Ranking is the one of gt_common.cuh (warp-private counters, lane-ordered
// shared atomics or the safe OR-mask mode); stability composes over levels, so
// each CSC list ends in CSR order = ascending source.
//
// Hot loops (kOpt, the default with the atomic rank mode): the rank, stage and
// write-out loops of the three place kernels and their per-tile scan address
// shared memory through 32-bit shared addresses off registers that went through
// an identity shuffle (gt_common.cuh: launder, lds_* / sts_* / atoms_add), with
// immediate offsets.  Plain pointer code made ptxas re-derive the shared window
// address (S2UR SR_CgaCtaId + UMOV + ULEA), kernel parameters and the thread
// index in front of every access: two thirds of the instructions between two
// rank atomics.  The pointer-based loops remain for the safe
// rank mode, the wide / slab forms' remaining phases, warps that hold a
// source-high boundary, and as experiment bit 4096 (A/B).
#pragma once
#include <algorithm>

#include "gt_common.cuh"
#include "gt_scan.cuh"

namespace gt {
namespace v3 {

constexpr int W = 8;             // warps per partition CTA
constexpr int T = W * 32;
constexpr int K = 16;            // items per thread per place tile
constexpr int PT = W * K * 32;   // 4096 records per place tile
constexpr int PTP = PT + 8;      // landing buffer (alignment slack)
constexpr int CT1_SHIFT = 17;
constexpr int CT1 = 1 << CT1_SHIFT;  // L1 count tile (edges)
constexpr int G1 = 8;            // count tiles per k_c1 CTA
constexpr int CT2 = 32768;       // L2 / L3-big count tile (records of one segment)
constexpr int kWin = 1024;       // offsets window (entries) per L1 place tile
constexpr int kMaxBnd = 512;     // source-high boundaries of an L2 tile held in smem
constexpr int W3 = 16, K3 = 16;
constexpr int CAP3 = W3 * K3 * 32;  // 8192 records per L3 unit
constexpr int CAP3P = CAP3 + 8;
constexpr int ML3 = 512;            // local vertices per L3 unit (256 when R2 carries the fine bits)

// One count tile of a record pass (L2: a chunk of a coarse bucket; L3-big: a
// chunk of a big fine bucket).
struct RTile {
  uint64_t start;  // first record (absolute index)
  uint32_t n;      // records
  uint32_t seg;    // segment (coarse bucket / big-bucket index)
  uint32_t j, nt;  // tile index inside the segment, tiles in the segment
  uint32_t h0;     // R1 decode: source-high of the first record
  uint32_t nbnd;   // R1 decode: source-high boundaries strictly inside the tile
};
static_assert(sizeof(RTile) == 32, "RTile layout");

// One segment of a record pass: its count/base table rows are
// [g0 * D + d * nt + j] (digit-major inside the segment), its records go to
// positions base + ..., and its per-digit starts to out[out_off + d].
struct SegDesc {
  uint64_t base;
  uint64_t out_off;
  uint32_t g0, nt;
  uint64_t end;  // output position past the segment's last record
};

struct Unit3 {
  uint64_t start;  // CSC position of the first record
  uint32_t n;      // records (<= CAP3)
  uint32_t f0;     // first fine bucket (global index A * Db + B)
  uint32_t nf;     // fine buckets
  uint32_t pad;
};

struct DigSM {  // (r >> shift) & mask
  int shift;
  uint32_t mask;
  __device__ __forceinline__ uint32_t operator()(uint32_t r) const { return (r >> shift) & mask; }
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t align_items_u32(const void* p) {
  return (uint32_t)((reinterpret_cast<uintptr_t>(p) & 15) >> 2);
}
__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Number of lanes' positions: for lane l, #{j in [0,32) : rel_j <= l}, rel
// non-decreasing across lanes (a shuffle binary search, 6 rounds).
__device__ __forceinline__ uint32_t count_le_lane(uint32_t rel, uint32_t lane) {
  uint32_t c = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t x = __shfl_sync(kFull, rel, c + s - 1);
    if (x <= lane) c += s;
  }
  const uint32_t x = __shfl_sync(kFull, rel, c);
  return c + ((x <= lane) ? 1u : 0u);
}

// Owner of each lane's position in a slot of 32 consecutive positions
// p0..p0+31 over a non-decreasing boundary sequence b(k): the result for lane l
// is the largest k in [cur, upper] with k == cur or b(k) <= p0 + l.  `cur` must
// satisfy "the owner of p0 is >= cur" and nb == b(cur + 1).  Both are advanced
// to the state of the next slot.  Warp-uniform control flow.
template <class F>
__device__ __forceinline__ uint32_t slot_owner(uint32_t& cur, uint64_t& nb, uint64_t p0, uint32_t upper, F bnd_at) {
  if (nb > p0 + 31) return cur;  // no boundary inside this slot
  const uint32_t lane = lane_id();
  uint32_t res;
  uint32_t base = cur, acc = 0;
  int rounds = 0;
  while (true) {
    const uint64_t k = (uint64_t)base + 1 + lane;
    const uint64_t bj = (k <= upper) ? bnd_at(k) : ~0ull;
    const uint32_t rel = (bj <= p0 + 31) ? (uint32_t)(bj - p0) : 32u;
    acc += count_le_lane(rel, lane);
    if (__shfl_sync(kFull, rel, 31) >= 32) {
      res = cur + acc;
      break;
    }
    base += 32;
    if (++rounds == 3) {  // long run of boundaries at few positions: binary search per lane
      const uint64_t p = p0 + lane;
      uint32_t lo = cur, hi = max(upper, cur);
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (bnd_at(mid) <= p) lo = mid; else hi = mid - 1;
      }
      res = lo;
      break;
    }
  }
  cur = __shfl_sync(kFull, res, 31);
  nb = ((uint64_t)cur + 1 <= upper) ? bnd_at((uint64_t)cur + 1) : ~0ull;
  return res;
}

// Largest k in [lo, hi] with k == lo or b(k) <= p (uniform binary search).
template <class F>
__device__ __forceinline__ uint32_t owner_search(uint32_t lo, uint32_t hi, uint64_t p, F bnd_at) {
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    if (bnd_at(mid) <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void zero_u32(uint32_t* p, int n) {  // n multiple of 4, p 16B aligned
  uint4* q = reinterpret_cast<uint4*>(p);
  for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x) q[i] = make_uint4(0, 0, 0, 0);
}

constexpr int WP = W + 1;    // counter table row: digit-major [d][W + 1] (padding keeps rank atomics conflict-free)
constexpr int W3P = W3 + 1;
__host__ __device__ constexpr int round4(int x) { return (x + 3) & ~3; }

// Stable rank through the counter at `c` (this warp's entry of the digit);
// kRankSafe: the OR-mask protocol of gt_common.cuh on the scratch entry `sc`.
template <int kMode>
__device__ __forceinline__ uint32_t rank_at(uint32_t* c, uint32_t* sc, bool valid) {
  if constexpr (kMode == kRankAtomic) {
    (void)sc;
    return valid ? atomicAdd(c, 1u) : 0u;
  } else {
    const uint32_t lane = lane_id();
    if (valid) atomicOr(sc, 1u << lane);
    __syncwarp();
    uint32_t peers = 0, v = 0;
    if (valid) {
      peers = *sc;
      v = *c;
    }
    __syncwarp();
    const uint32_t lt = peers & lanemask_lt();
    if (valid && lt == 0) {
      *c = v + __popc(peers);
      *sc = 0;
    }
    __syncwarp();
    return v + __popc(lt);
  }
}

// Rank with peers from match.any: one atomic per distinct digit (leader), no
// reliance on the order of same-address lanes.  Cheaper than per-lane atomics
// when few distinct digits share a warp instruction (hub-dominated buckets).
__device__ __forceinline__ uint32_t rank_match(uint32_t* word, uint32_t sh, uint32_t d, bool valid) {
  const uint32_t lane = lane_id();
  const uint32_t m = __match_any_sync(kFull, valid ? d : 0xffffffffu);
  const uint32_t ld = __ffs(m) - 1;
  uint32_t base = 0;
  if (valid && lane == ld) base = (atomicAdd(word, (uint32_t)__popc(m) << sh) >> sh) & 0xffffu;
  base = __shfl_sync(kFull, base, ld);
  return base + __popc(m & lanemask_lt());
}

// Packed counter tables: digit-major, two warps per 32-bit word (u16 fields:
// per-warp counts <= 1024 and tile positions <= 8192 fit), one pad word per
// digit (odd row stride: random digits spread over banks).
constexpr int WH = W / 2 + 1;
constexpr int WH3 = W3 / 2 + 1;
// Rank through the packed counter word `c` (field at bit `sh` = 16 * (w & 1)).
// kRankSafe: peers from the OR-mask scratch entry `sc`, one leader per digit
// adds the group size, so no same-address ordering is assumed.
template <int kMode>
__device__ __forceinline__ uint32_t rank_pk(uint32_t* c, uint32_t* sc, uint32_t sh, bool valid) {
  if constexpr (kMode == kRankAtomic) {
    (void)sc;
    return valid ? ((atomicAdd(c, 1u << sh) >> sh) & 0xffffu) : 0u;
  } else {
    const uint32_t lane = lane_id();
    if (valid) atomicOr(sc, 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? *sc : 0u;
    __syncwarp();
    const uint32_t ld = peers ? (uint32_t)(__ffs(peers) - 1) : 0u;
    uint32_t old = 0;
    if (valid && lane == ld) {
      old = atomicAdd(c, (uint32_t)__popc(peers) << sh);
      *sc = 0;
    }
    old = __shfl_sync(kFull, old, ld);
    __syncwarp();
    return ((old >> sh) & 0xffffu) + __popc(peers & lanemask_lt());
  }
}
// After ranking: tab[d * WHN + k] holds (warp 2k, warp 2k+1) tile positions of
// their first digit-d item; dtot per digit; delta[d] = gcur[d] - digit start.
// Epilogue form: epi(d, b, e) per digit with its tile-local start b and end e.
// kEpi = false: no per-digit epilogue (and no barrier after the rewrite's barrier).
template <int WHN, bool kEpi = true, class Epi>
__device__ __forceinline__ void flat_bases_epi(uint32_t* tab, int D, uint32_t* tmp, Epi epi) {
  const int n = D * WHN;
  const int Tn = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (Tn + 31) >> 5;
  const int per = ((n + Tn - 1) / Tn) | 1;  // odd chunk length: the 32 lanes start in 32 distinct banks
  const int lo = min(n, t * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) {
    const uint32_t v = tab[i];
    s += (v & 0xffffu) + (v >> 16);
  }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (t < 32) {
    const uint32_t v0 = (t < nw) ? tmp[t] : 0u;
    uint32_t v = v0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, v, o);
      if (t >= o) v += y;
    }
    if (t < nw) tmp[t] = v - v0;
  }
  __syncthreads();
  uint32_t run = tmp[w] + x - s;
  for (int i = lo; i < hi; ++i) {
    const uint32_t v = tab[i], l = v & 0xffffu;
    tab[i] = run | ((run + l) << 16);
    run += l + (v >> 16);
  }
  __syncthreads();
  if constexpr (kEpi) {
    for (int d = threadIdx.x; d < D; d += blockDim.x) epi(d, tab[d * WHN] & 0xffffu, tab[d * WHN + WHN - 1] & 0xffffu);
    __syncthreads();
  }
}
template <int WHN>
__device__ __forceinline__ void flat_bases_pk(uint32_t* tab, int D, const uint32_t* gcur, uint32_t* dtot,
                                              uint32_t* delta, uint32_t* tmp) {
  flat_bases_epi<WHN>(tab, D, tmp, [&](int d, uint32_t b, uint32_t e) {
    if (dtot) dtot[d] = e - b;
    if (gcur) delta[d] = gcur[d] - b;
  });
}

// flat_bases_epi's scan on 32-bit shared addresses with a compile-time chunk
// length (PER words per thread, odd: conflict-free) and block size: the words
// stay in registers between the two passes, every access has an immediate
// offset, and each warp sums the earlier warps' totals itself (two barriers).
// Requires n <= NT * PER.  a_tmp: NT / 32 words.
// a0 = this thread's first word (a_tab + t * PER * 4), rem = its word count bound (n - t * PER):
// computed by the caller from the runtime chunk length, so the instances share that arithmetic.
template <int NT, int PER>
__device__ __forceinline__ void flat_scan_fast(uint32_t a0, int rem, uint32_t a_tmp, uint32_t t) {
  static_assert(PER & 1, "odd chunk length");
  const uint32_t lane = t & 31, w = t >> 5;
  constexpr bool kKeep = PER <= 3;  // longer chunks are re-read (the callers hold 32+ live registers)
  uint32_t v[PER];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = 0;
    if (i < rem) v[i] = lds_u32(a0 + i * 4);
  }
  {  // both u16 fields summed as a packed pair first (each sum <= the tile size < 2^16)
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) acc += v[i];
    s = (acc & 0xffffu) + (acc >> 16);
  }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sts_u32(a_tmp + w * 4, x);
  __syncthreads();
  uint32_t p = 0;
  if (lane < w) p = lds_u32(a_tmp + lane * 4);  // (w < NW <= 32)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
  uint32_t run = p + x - s;
  if constexpr (!kKeep) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      v[i] = 0;
      if (i < rem) v[i] = lds_u32(a0 + i * 4);
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const uint32_t e = run + (v[i] & 0xffffu);
    if (i < rem) sts_u32(a0 + i * 4, run | (e << 16));
    run = e + (v[i] >> 16);
  }
  __syncthreads();
}
// Chunk length by table size; false if the table is larger than NT * 21 words.
template <int NT, int kMaxPer = 11>
__device__ __forceinline__ bool flat_scan_any(uint32_t a_tab, uint32_t n, uint32_t a_tmp, uint32_t t) {
  static_assert(kMaxPer == 11 || kMaxPer == 21, "instances: 3, 5, 9, 11 (and 21 for the 1024-digit forms)");
  if (n > NT * kMaxPer) return false;
  const uint32_t per = (n <= NT * 3) ? 3u : (n <= NT * 5) ? 5u : (n <= NT * 9) ? 9u : (kMaxPer == 11 || n <= NT * 11) ? 11u : 21u;
  const uint32_t a0 = a_tab + t * per * 4;
  const int rem = (int)n - (int)(t * per);
  if (per == 3) flat_scan_fast<NT, 3>(a0, rem, a_tmp, t);
  else if (per == 5) flat_scan_fast<NT, 5>(a0, rem, a_tmp, t);
  else if (per == 9) flat_scan_fast<NT, 9>(a0, rem, a_tmp, t);
  else if (kMaxPer == 11 || per == 11) flat_scan_fast<NT, 11>(a0, rem, a_tmp, t);
  else if constexpr (kMaxPer == 21) flat_scan_fast<NT, 21>(a0, rem, a_tmp, t);
  return true;
}

// In-place exclusive scan of a[0..n) (thread-contiguous chunks, one block scan).
__device__ __forceinline__ void flat_excl_scan(uint32_t* a, int n, uint32_t* tmp /* >= 33 */) {
  const int Tn = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = (Tn + 31) >> 5;
  const int per = ((n + Tn - 1) / Tn) | 1;  // odd chunk length: the 32 lanes start in 32 distinct banks
  const int lo = min(n, t * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (t < 32) {
    const uint32_t v0 = (t < nw) ? tmp[t] : 0u;
    uint32_t v = v0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, v, o);
      if (t >= o) v += y;
    }
    if (t < nw) tmp[t] = v - v0;
  }
  __syncthreads();
  uint32_t run = tmp[w] + x - s;
  for (int i = lo; i < hi; ++i) {
    const uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
  __syncthreads();
}

// After ranking: cnt[d * (WW+1) + w] becomes the tile position of warp w's
// first digit-d item; dstart/dtot per digit; delta[d] = gcur[d] - dstart[d]
// when gcur is given (global index = tile position + delta).
template <int WW>
__device__ __forceinline__ void flat_bases(uint32_t* cnt, int D, const uint32_t* gcur, uint32_t* dstart, uint32_t* dtot,
                                           uint32_t* delta, uint32_t* tmp) {
  flat_excl_scan(cnt, D * (WW + 1), tmp);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const uint32_t b = cnt[d * (WW + 1)];
    dstart[d] = b;
    dtot[d] = cnt[d * (WW + 1) + WW] - b;
    if (gcur) delta[d] = gcur[d] - b;
  }
  __syncthreads();
}

// Block-wide exclusive scan of u64 a[0..n) in place; returns the total.
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t* a, int n, uint64_t* tmp /* >= 33 */) {
  const int Tn = blockDim.x, t = threadIdx.x;
  const int nw = (Tn + 31) >> 5, w = t >> 5, lane = t & 31;
  const int per = ((n + nw - 1) / nw + 31) & ~31;
  const int lo = w * per, hi = min(n, lo + per);
  uint64_t s = 0;
  for (int i = lo + lane; i < hi; i += 32) s += a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) tmp[w] = s;
  __syncthreads();
  if (t < 32) {
    const uint64_t v0 = (t < nw) ? tmp[t] : 0;
    uint64_t v = v0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, v, o);
      if (t >= o) v += y;
    }
    if (t < nw) tmp[t] = v - v0;
    if (t == 31) tmp[32] = v;
  }
  __syncthreads();
  uint64_t carry = tmp[w];
  for (int b = lo; b < hi; b += 32) {
    const int i = b + lane;
    const uint64_t x = (i < hi) ? a[i] : 0;
    uint64_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t z = __shfl_up_sync(kFull, y, o);
      if (lane >= o) y += z;
    }
    if (i < hi) a[i] = carry + y - x;
    carry += __shfl_sync(kFull, y, 31);
  }
  const uint64_t total = tmp[32];
  __syncthreads();
  return total;
}

// ------------------------------------------------------------- L1: count
// Histogram of the coarse digit per count tile (CT1 edges); G1 tiles per CTA.
// tcnt is digit-major: tcnt[d * ntiles + k] (consecutive tiles of one digit are
// written together: full 32-byte sectors).
template <bool kSlab>
__global__ void __launch_bounds__(512) k_c1(const uint32_t* __restrict__ edges, uint64_t E, uint64_t ntiles, int D,
                                            int shift, uint32_t* __restrict__ tcnt, uint32_t slab_mask,
                                            uint32_t slab_val) {
  extern __shared__ __align__(16) uint32_t s_h[];  // G1 * D
  // kSlab (num_vertices > 2^29): only destinations with (dst & slab_mask) == slab_val count
  const uint32_t dm = (uint32_t)D - 1;
  auto inc = [&](uint32_t i, uint32_t v) {
    if constexpr (kSlab) {
      if ((v & slab_mask) == slab_val) smem_inc(&s_h[(i >> CT1_SHIFT) * D + ((v >> shift) & dm)]);
    } else {
      smem_inc(&s_h[(i >> CT1_SHIFT) * D + (v >> shift)]);
    }
  };
  const uint64_t k0 = (uint64_t)blockIdx.x * G1;
  const int nt = (int)umin64(G1, ntiles - k0);
  for (int i = threadIdx.x; i < G1 * D; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const uint64_t b = k0 * CT1, n = umin64(E, b + (uint64_t)nt * CT1) - b;
  const uint32_t* p = edges + b;
  const uint32_t head = (uint32_t)umin64(n, (4 - align_items_u32(p)) & 3);
  for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) inc(i, p[i]);
  const uint4* p4 = reinterpret_cast<const uint4*>(p + head);
  const uint64_t n4 = (n - head) >> 2;
  for (uint64_t q = threadIdx.x; q < n4; q += blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p4 + q));
    const uint32_t i = head + (uint32_t)q * 4;
    inc(i, v.x);
    inc(i + 1, v.y);
    inc(i + 2, v.z);
    inc(i + 3, v.w);
  }
  for (uint64_t i = head + n4 * 4 + threadIdx.x; i < n; i += blockDim.x) inc((uint32_t)i, p[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < G1 * D; i += blockDim.x) {
    const int d = i / G1, t = i - d * G1;
    if (t < nt) tcnt[(uint64_t)d * ntiles + k0 + t] = s_h[t * D + d];
  }
}

// Destinations per slab of 2^29 IDs (slab mode).
__global__ void k_slab_hist(const uint32_t* __restrict__ edges, uint64_t E, unsigned long long* __restrict__ cnt) {
  __shared__ unsigned long long s_c[8];
  if (threadIdx.x < 8) s_c[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long local[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
    ++local[edges[i] >> 29];
  for (int k = 0; k < 8; ++k)
    if (local[k]) atomicAdd(&s_c[k], local[k]);
  __syncthreads();
  if (threadIdx.x < 8 && s_c[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], s_c[threadIdx.x]);
}

// ------------------------------------------------------------- L1: place
struct P1Args {
  const uint64_t* offsets;
  const uint32_t* edges;  // stream item 0 = global edge e_begin
  uint64_t e_begin, V, E;
  uint64_t ntiles;        // count tiles (CT1)
  int D, shift, L;
  uint32_t low_mask, src_mask;
  const uint64_t* tbase;   // [d * ntiles + k]
  const uint32_t* psrc;    // owner of the first item of each place tile; [nplace] = owner of item E-1
  const uint32_t* prev_src;// per count tile: owner of the item before it (~0u: none)
  uint32_t nh;             // source-high values; seg_hi rows have nh + 1 entries
  uint64_t* seg_hi;
  uint32_t* out;           // R1
  uint32_t slab_mask, slab_val;  // kSlab: records with (dst & slab_mask) == slab_val only
};

inline size_t smem_p1(int D, int mode, int KK = K, int WW = W) {
  const size_t pt = (size_t)WW * KK * 32, win = std::max<size_t>(1024, pt / 4);
  const int wh = WW / 2 + 1, wp = WW + 1;
  return (pt + 8) * 4 + win * 8 + pt * 2 + ((size_t)round4(D * wh) + (mode == kRankSafe ? (size_t)round4(D * wp) : 0)) * 4 +
         (size_t)D * 4 * 3 + 40 * 4 + (CT1 / pt + 4) * 4;
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// Per-warp tile-local bases and global index offsets: cnt[w][d] becomes the
// tile position of warp w's first digit-d item, delta[d] = gcur[d] - dstart[d]
// (global R1 index = tile position + delta[d]), dtot[d] = digit total.
template <int WW>
__device__ __forceinline__ void bases_delta(uint32_t* cnt, int D, const uint32_t* gcur, uint32_t* dstart,
                                            uint32_t* dtot, uint32_t* delta, uint32_t* tmp) {
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < WW; ++w) {
      const uint32_t c = cnt[w * D + d];
      cnt[w * D + d] = run;
      run += c;
    }
    dstart[d] = run;
    dtot[d] = run;
  }
  __syncthreads();
  block_excl_scan_u32(dstart, D, tmp);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const uint32_t b = dstart[d];
#pragma unroll
    for (int w = 0; w < WW; ++w) cnt[w * D + d] += b;
    delta[d] = gcur[d] - b;
  }
  __syncthreads();
}

// Write-out of a staged tile: slot i holds payload buf[i] of digit tag[i],
// global index delta[tag] + i.  Consecutive lanes take consecutive slots, so a
// warp store covers a few digit runs (coalesced sectors).
template <int NT, int TILE, class G>
__device__ __forceinline__ void writeout_tag(uint32_t* __restrict__ out, const uint32_t* buf, const uint16_t* tag,
                                             const G* delta, uint32_t n) {
  if (n == (uint32_t)TILE) {
#pragma unroll
    for (int k = 0; k < TILE / NT; ++k) {
      const uint32_t i = threadIdx.x + k * NT;
      out[delta[tag[i]] + i] = buf[i];
    }
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += NT) out[delta[tag[i]] + i] = buf[i];
  }
}

// Write-out of (payload, digit) pairs: slot i goes to delta[digit] + i.
template <int NT, int TILE>
__device__ __forceinline__ void writeout_pair(uint32_t* __restrict__ out, const uint2* st, const uint32_t* delta,
                                              uint32_t n) {
  if (n == (uint32_t)TILE) {
#pragma unroll
    for (int k = 0; k < TILE / NT; ++k) {
      const uint32_t i = threadIdx.x + k * NT;
      const uint2 v = st[i];
      out[delta[v.y] + i] = v.x;
    }
  } else {
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
      const uint2 v = st[i];
      out[delta[v.y] + i] = v.x;
    }
  }
}

// Stage K ranked items of a thread: item s (pk = digit << 16 | rank inside its
// warp's digit run, payload pay) goes to slot base(digit, warp) + rank, its
// digit to tag[slot].  The base words of G items are loaded before their
// stores: shared stores would otherwise order every following load behind
// them.  lim = valid items of the tile (0xffffffff: all), i0 = position of
// item 0 (items at i0 + 32 s).
constexpr int kStageG = 8;
// kSkip: items with pk == ~0u (filtered out) are not staged.
template <int G, int K_, class Tag, bool kSkip = false>
__device__ __forceinline__ void stage_tag(const uint32_t (&pk)[K_], const uint32_t (&pay)[K_], const uint32_t* cnt,
                                          int whn, uint32_t w, uint32_t sh, uint32_t* buf, Tag* tag, uint32_t lim,
                                          uint32_t i0, uint32_t per = K_ * 32) {
#pragma unroll
  for (int c = 0; c < K_; c += G) {
    if ((uint32_t)c * 32 >= per) break;  // per: positions of this warp (slots beyond hold nothing)
    uint32_t bw[G];
#pragma unroll
    for (int q = 0; q < G; ++q)  // (unused slots: pk = 0)
      bw[q] = cnt[((kSkip && pk[c + q] == 0xffffffffu) ? 0u : (pk[c + q] >> 16)) * whn + (w >> 1)];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if ((uint32_t)(c + q) * 32 < per && (lim == 0xffffffffu || i0 + (c + q) * 32 < lim) &&
          (!kSkip || pk[c + q] != 0xffffffffu)) {
        const uint32_t pos = ((bw[q] >> sh) & 0xffffu) + (pk[c + q] & 0xffffu);
        buf[pos] = pay[c + q];
        tag[pos] = (Tag)(pk[c + q] >> 16);
      }
    }
  }
}

// stage_tag with one 8-byte (payload, digit) store per item.
template <int G, int K_>
__device__ __forceinline__ void stage_pair(const uint32_t (&pk)[K_], const uint32_t (&pay)[K_], const uint32_t* cnt,
                                           int whn, uint32_t w, uint32_t sh, uint2* st, uint32_t lim, uint32_t i0,
                                           uint32_t per = K_ * 32) {
#pragma unroll
  for (int c = 0; c < K_; c += G) {
    if ((uint32_t)c * 32 >= per) break;
    uint32_t bw[G];
#pragma unroll
    for (int q = 0; q < G; ++q) bw[q] = cnt[(pk[c + q] >> 16) * whn + (w >> 1)];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      if ((uint32_t)(c + q) * 32 < per && (lim == 0xffffffffu || i0 + (c + q) * 32 < lim)) {
        const uint32_t pos = ((bw[q] >> sh) & 0xffffu) + (pk[c + q] & 0xffffu);
        st[pos] = make_uint2(pay[c + q], pk[c + q] >> 16);
      }
    }
  }
}

// L1 place.  One CTA per count tile (CT1 edges), place tiles of PT edges in
// order with running per-digit cursors.  Per place tile: TMA bulk load of the
// edges and of the offsets window; every source boundary inside the tile is
// marked (mark[p] = v + 1 for the source v whose list starts at item p); each
// 32-edge slot finds its owners with one ballot over the marks (the last mark
// at or before the lane, else the carry from the previous slot); stable rank
// by the coarse digit; stage payload + global index by digit; vectorised
// write-out of the runs.  Requires E < 2^32 (u32 indices).
// kW64 (graphs with E >= 2^32): 64-bit R1 positions.  The per-digit cursor
// array holds the cursor between tiles and the index delta during a tile
// (delta = cursor - tile start, restored from the digit end after the tile),
// so the shared-memory footprint matches the 32-bit form.
// kSlab (num_vertices > 2^29, slab mode): only records of one 2^29-ID
// destination slab are ranked, staged and written (the others pass through
// source recovery only); the digit is taken modulo D.
template <int kMode, int KK = K, bool kW64 = false, int WW = W, int kMinB = (KK > 16 || kW64 || WW > 8 ? 2 : 4),
          bool kSlab = false, bool kOpt = true>
__global__ void __launch_bounds__(WW * 32, kMinB) k_p1(const P1Args a) {
  constexpr int W1_ = WW, T1_ = WW * 32, WH1_ = WW / 2 + 1, WP1_ = WW + 1;
  // place tiles of PT = W1_ * KK * 32 edges; the offsets window doubles as the
  // tag array, so it holds max(1024, PT / 4) entries
  constexpr int K = KK, PT = W1_ * KK * 32, PTP = PT + 8, kWin = (PT / 4 > 1024) ? PT / 4 : 1024;
  extern __shared__ __align__(128) unsigned char smem[];
  const int D = a.D;
  uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem);                         // PTP (landing, then stage)
  uint64_t* s_win = reinterpret_cast<uint64_t*>(s_buf + PTP);                  // kWin
  // source-boundary marks: u16 (v - s0) of the non-empty source whose list starts at the item
  uint16_t* s_mark = reinterpret_cast<uint16_t*>(s_win + kWin);                // PT
  // digit of each staged slot: aliases the offsets window (dead after ranking;
  // the next window lands by TMA after the end-of-tile barrier + proxy fence)
  static_assert(kWin * 8 >= PT * 2, "tag array must fit in the window");
  uint16_t* s_tag = reinterpret_cast<uint16_t*>(s_win);
  // fixed-size scratch first (compile-time offsets from the base), the D-sized tables after it
  uint32_t* s_tmp = reinterpret_cast<uint32_t*>(s_mark + PT);                  // 40
  uint32_t* s_psrc = s_tmp + 40;                                               // CT1/PT + 4 (16-byte multiple with s_tmp)
  static_assert((40 + CT1 / PT + 4) % 4 == 0, "s_cnt stays 16-byte aligned");
  constexpr uint32_t kOffMark = PTP * 4 + kWin * 8, kOffTmp = kOffMark + PT * 2, kOffPsrc = kOffTmp + 160,
                     kOffCnt = kOffPsrc + (CT1 / PT + 4) * 4;
  uint32_t* s_cnt = s_psrc + (CT1 / PT + 4);                                   // D * WH1_ (packed, digit-major)
  uint32_t* s_scr = s_cnt + round4(D * WH1_);                                    // D * WP1_ (safe)
  uint32_t* s_gcur = s_scr + (kMode == kRankSafe ? round4(D * WP1_) : 0);        // D
  uint32_t* s_delta = s_gcur + D;                                              // D
  uint32_t* s_dtot = s_delta + D;                                              // D
  uint32_t* s_bh = reinterpret_cast<uint32_t*>(s_mark);                        // D (aliases the marks, dead after ranking)
  // kW64: s_g64 (D u64) spans s_gcur + s_delta (8-byte aligned: every region
  // before it is a multiple of 8 bytes), s_dtot holds the digit's tile end
  uint64_t* s_g64 = reinterpret_cast<uint64_t*>(s_gcur);
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint64_t s_wlo;
  __shared__ uint32_t s_wn;
  __shared__ uint32_t s_last_src;
  __shared__ uint32_t s_lastm[32];
  __shared__ uint32_t s_nst;  // kSlab: staged (kept) items of the place tile

  // (kOpt: the thread index in a laundered register — ptxas otherwise re-reads SR_TID.X all over the kernel)
  const uint32_t tid = kOpt ? launder(threadIdx.x) : threadIdx.x, lane = tid & 31u, w = tid >> 5;
  const uint32_t sh = (w & 1) << 4;
  const uint64_t k = blockIdx.x;
  const uint64_t tb = k * CT1, te = umin64(a.E, tb + CT1);
  const int nplace = (int)((te - tb + PT - 1) / PT);
  const uint64_t gp0 = tb / PT;
  for (int d = tid; d < D; d += T1_) {
    if constexpr (kW64) s_g64[d] = a.tbase[(uint64_t)d * a.ntiles + k];
    else s_gcur[d] = (uint32_t)a.tbase[(uint64_t)d * a.ntiles + k];
  }
  for (int j = tid; j <= nplace; j += T1_) s_psrc[j] = a.psrc[gp0 + j];
  zero_u32(s_cnt, round4(D * WH1_) + (kMode == kRankSafe ? round4(D * WP1_) : 0));
  zero_u32(reinterpret_cast<uint32_t*>(s_mark), PT / 2);
  if (tid < 32) s_lastm[tid] = 0;
  if (tid == 0) s_nst = 0;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  uint32_t h_prev;
  {
    const uint32_t ps = a.prev_src[k];  // k = 0: ~0u (whole graph) or the shard's first source
    h_prev = (ps == 0xffffffffu) ? 0xffffffffu : (ps >> a.L);
  }
  __syncthreads();

  // kFast: rank, stage and write-out through 32-bit shared addresses off laundered registers (gt_common.cuh)
  // (kFastRS: the rank and stage loops, also for 64-bit positions; kFast: scan, write-out and zeroing too)
  constexpr bool kFastRS = kOpt && kMode == kRankAtomic && !kSlab;
  constexpr bool kFast = kFastRS && !kW64;
  uint32_t f_sb = 0, f_cw = 0, f_inc = 0, f_selr = 0, f_sel16 = 0, f_delta = 0;
  if constexpr (kFastRS) {
    f_sb = launder(smem_u32(smem));
    f_cw = launder(f_sb + kOffCnt + (w >> 1) * 4);  // this warp's word of every digit row
    f_inc = launder(1u << sh);
    f_selr = launder((w & 1) ? 0x5432u : 0x5410u);   // (old field, digit) -> digit << 16 | rank
    f_sel16 = launder((w & 1) ? 0x4432u : 0x4410u);  // this warp's u16 field of a counter word
    f_delta = launder(smem_u32(s_delta));
  }
  auto issue = [&](int j) {  // thread 0
    const uint64_t pt = tb + (uint64_t)j * PT;
    const uint32_t n = (uint32_t)umin64(PT, te - pt);
    const uint32_t* gp = a.edges + pt;
    const uint32_t o = align_items_u32(gp);
    const uint32_t full = (o + n) & ~3u;
    const uint32_t s0 = s_psrc[j], s1 = s_psrc[j + 1];
    const uint64_t* wp = a.offsets + s0 + 1;
    const uint32_t ow = (uint32_t)((reinterpret_cast<uintptr_t>(wp) & 15) >> 3);
    const uint64_t ws = (uint64_t)s0 + 1 - ow;
    const uint64_t need = (uint64_t)s1 + 2 - ws, avail = a.V + 1 - ws;
    const uint32_t nw = (uint32_t)umin64(umin64(need, avail), kWin) & ~1u;
    s_wlo = ws;
    s_wn = nw;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&s_bar, full * 4 + nw * 8);
    if (full) bulk_g2s(s_buf, gp - o, full * 4, &s_bar);
    if (nw) bulk_g2s(s_win, a.offsets + ws, nw * 8, &s_bar);
    if (j + 1 < nplace) {  // warm L2 with the next place tile's edges
      const uint32_t* gn = gp + PT;
      const uint32_t on = align_items_u32(gn);
      const uint32_t nn = (uint32_t)umin64(PT, te - pt - PT);
      const uint32_t fn = (on + nn) & ~3u;
      if (fn) bulk_prefetch_l2(gn - on, fn * 4);
    }
  };

  uint32_t ph = 0;
  const uint32_t o_c = align_items_u32(a.edges + tb);
  if (tid == 0 && nplace > 0) issue(0);
  for (int j = 0; j < nplace; ++j) {
    if constexpr (kW64) {  // delta -> cursor of the next tile (after barrier (D): the write-out is done)
      if (j > 0)
        for (int d = tid; d < D; d += T1_) s_g64[d] += s_dtot[d];
    }
    const uint64_t pt = tb + (uint64_t)j * PT;
    const uint32_t n = (uint32_t)umin64(PT, te - pt);
    const uint32_t* gp = a.edges + pt;
    static_assert(PT % 4 == 0 && CT1 % 4 == 0, "every place tile starts at the stream's 16-byte phase");
    const uint32_t o = o_c;
    const uint32_t full = (o + n) & ~3u;
    const uint32_t ti = full + tid;
    const bool tail = ((o + n) & 3u) != 0 && tid < 4 && ti < o + n;  // (first test uniform, rarely true)
    uint32_t tv = 0;
    if (tail) tv = ldg_u32(gp - o + ti);
    mbar_wait_parity(&s_bar, ph);
    ph ^= 1;
    if (tail) s_buf[ti] = tv;
    const uint64_t gi0 = a.e_begin + pt;
    const uint64_t ws = s_wlo;
    const uint32_t nw = s_wn;
    const uint64_t* offs = a.offsets;
    auto off_at = [&](uint64_t v) -> uint64_t {
      const uint64_t q = v - ws;
      return (q < nw) ? s_win[q] : __ldg(offs + v);
    };
    const uint32_t s0 = s_psrc[j], s1 = max(s_psrc[j + 1], s0);
    // mark the first item of every non-empty source that starts inside the tile
    // (one per item; the owner of an item is the last source starting at or before it)
    const bool wide = s1 - s0 > 65535u;  // marks cannot encode the span: per-lane search below
    if (!wide) {
      for (uint32_t v = s0 + 1 + tid; v <= s1; v += T1_) {
        const uint64_t p = off_at(v) - gi0;
        if (p < n && off_at((uint64_t)v + 1) > off_at(v)) {
          s_mark[p] = (uint16_t)(v - s0);
          atomicMax(&s_lastm[p / (K * 32)], v - s0);  // last source starting in each warp's segment
        }
      }
    }
    __syncthreads();  // (A) tile landed, marks placed

    const uint32_t iw = w * (K * 32);
    // owner of the warp's first item: the last source starting in an earlier segment (else s0)
    uint32_t carry;
    if (!wide) {
      uint32_t mx = (lane < w) ? s_lastm[lane] : 0u;  // (w < 32)
      mx = __reduce_max_sync(kFull, mx);
      carry = s0 + mx;
    } else {
      carry = owner_search(s0, s1, gi0 + iw, off_at);
    }
    const uint32_t le = lanemask_le();
    uint32_t pay[K], pk[K];
    // pay[s] / pk[s] first hold the slot's destination and mark: all loads of
    // the tile are issued before the first rank atomic (the compiler keeps
    // shared loads behind earlier shared atomics)
    uint32_t nkeep = 0;  // kSlab: this warp's kept items
    auto slot = [&](int s, bool valid) {
      const uint32_t i = iw + s * 32 + lane;
      const uint32_t dst = valid ? pay[s] : 0u;
      uint32_t src = carry;
      if (!wide) {
        const uint32_t m = pk[s];
        const uint32_t bal = __ballot_sync(kFull, m != 0);
        if (bal) {  // a source starts inside this slot (warp-uniform)
          const uint32_t bm = bal & le;
          const uint32_t ms = __shfl_sync(kFull, m, 31 - __clz(bm | 1u));
          src = bm ? s0 + ms : carry;
          carry = __shfl_sync(kFull, src, 31);
        }
      } else {
        src = owner_search(carry, s1, gi0 + i, off_at);
        carry = __shfl_sync(kFull, src, 31);
      }
      if ((n == (uint32_t)PT) ? (s == K - 1 && i == PT - 1) : (valid && i == n - 1)) s_last_src = src;
      if constexpr (kSlab) {
        const bool keep = valid && (dst & a.slab_mask) == a.slab_val;
        nkeep += __popc(__ballot_sync(kFull, keep));
        const uint32_t d = (dst >> a.shift) & (uint32_t)(D - 1);
        const uint32_t rk = rank_pk<kMode>(s_cnt + d * WH1_ + (w >> 1), s_scr + d * WP1_ + w, sh, keep);
        pk[s] = keep ? ((d << 16) | rk) : 0xffffffffu;
      } else {
        const uint32_t d = dst >> a.shift;
        pk[s] = (d << 16) | rank_pk<kMode>(s_cnt + d * WH1_ + (w >> 1), s_scr + d * WP1_ + w, sh, valid);
      }
      pay[s] = ((dst & a.low_mask) << a.L) | (src & a.src_mask);
    };
    bool fdone = false;
    if constexpr (kFastRS) {
      if (!wide) {
        fdone = true;
        const uint32_t a_rec = f_sb + (o + iw + lane) * 4, a_mk = f_sb + kOffMark + (iw + lane) * 2;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          pay[s] = lds_u32(a_rec + s * 128);
          pk[s] = lds_u16(a_mk + s * 64);
        }
        const uint32_t shift = a.shift, lowm = a.low_mask, L = a.L, srcm = a.src_mask;
        auto fslot = [&](int s, bool valid) {
          const uint32_t dst = valid ? pay[s] : 0u;
          const uint32_t m = pk[s];
          uint32_t src = carry;
          const uint32_t bal = __ballot_sync(kFull, m != 0);
          if (bal) {  // a source starts inside this slot (warp-uniform)
            const uint32_t bm = bal & le;
            const uint32_t ms = __shfl_sync(kFull, m, 31 - __clz(bm | 1u));
            src = bm ? s0 + ms : carry;
            carry = __shfl_sync(kFull, src, 31);
          }
          const uint32_t d = dst >> shift;
          uint32_t old = 0;
          if (valid) old = atoms_add(f_cw + d * (uint32_t)(WH1_ * 4), f_inc);
          pk[s] = prmt(old, d, f_selr);
          pay[s] = ((dst & lowm) << L) | (src & srcm);
          return src;
        };
        if (n == (uint32_t)PT) {
          uint32_t src = 0;
#pragma unroll
          for (int s = 0; s < K; ++s) src = fslot(s, true);
          if (tid == T1_ - 1) s_last_src = src;
        } else {
#pragma unroll
          for (int s = 0; s < K; ++s) {
            const uint32_t i = iw + s * 32 + lane;
            const uint32_t src = fslot(s, i < n);
            if (i == n - 1) s_last_src = src;
          }
        }
      }
    }
    if (!fdone) {
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = iw + s * 32 + lane;
        pay[s] = s_buf[o + i];
        pk[s] = s_mark[i];
      }
      if (n == (uint32_t)PT) {
#pragma unroll
        for (int s = 0; s < K; ++s) slot(s, true);
      } else {
#pragma unroll
        for (int s = 0; s < K; ++s) slot(s, iw + s * 32 + lane < n);
      }
    }
    if (kSlab && lane == 0) atomicAdd(&s_nst, nkeep);
    __syncthreads();  // (B) ranks done; landing buffer and marks consumed
    if constexpr (kW64)
      flat_bases_epi<WH1_>(s_cnt, D, s_tmp, [&](int d, uint32_t b, uint32_t e) {
        s_g64[d] -= b;
        s_dtot[d] = e;
      });
    else {
      bool fscan = false;
      if constexpr (kFast) {
        const uint32_t a_cnt = f_sb + kOffCnt;
        fscan = flat_scan_any<T1_, (KK > 16 ? 21 : 11)>(a_cnt, (uint32_t)(D * WH1_), f_sb + kOffTmp, tid);
        if (fscan) {  // per digit: tile-local start b and end e (the row's pad word)
          for (int d = tid; d < D; d += T1_) {
            const uint32_t ar = a_cnt + d * (WH1_ * 4);
            const uint32_t b = lds_u32(ar) & 0xffffu, e = lds_u32(ar + (WH1_ - 1) * 4) & 0xffffu;
            sts_u32(f_delta + (uint32_t)D * 4 + d * 4, e - b);            // s_dtot
            sts_u32(f_delta + d * 4, lds_u32(f_delta - (uint32_t)D * 4 + d * 4) - b);  // s_delta = s_gcur - b
          }
          __syncthreads();
        }
      }
      if (!fscan) flat_bases_pk<WH1_>(s_cnt, D, s_gcur, s_dtot, s_delta, s_tmp);
    }
    // source-high boundaries inside this tile (compact R1 decode table)
    const uint32_t h_last = s_last_src >> a.L;
    for (uint32_t h = (h_prev == 0xffffffffu) ? 0u : h_prev + 1; h <= h_last; ++h) {
      const uint64_t ob = __ldg(offs + ((uint64_t)h << a.L)), q = (ob > gi0) ? ob - gi0 : 0;  // first item with src >= h << L
      for (int d = tid; d < D; d += T1_) s_bh[d] = 0;
      __syncthreads();
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = iw + s * 32 + lane;
        if (i < n && i < q && (!kSlab || pk[s] != 0xffffffffu)) smem_inc(&s_bh[pk[s] >> 16]);
      }
      __syncthreads();
      for (int d = tid; d < D; d += T1_) {
        const uint64_t g0 = kW64 ? s_g64[d] + (s_cnt[d * WH1_] & 0xffffu) : (uint64_t)s_gcur[d];
        a.seg_hi[(uint64_t)d * (a.nh + 1) + h] = g0 + s_bh[d];
      }
      __syncthreads();
    }
    h_prev = h_last;
    // stage payloads and global indices by digit (base words loaded in groups
    // of kStageG before their stores)
    if constexpr (kFastRS) {
      const uint32_t a_tag = f_sb + (uint32_t)(PTP * 4);
      auto fstage = [&](auto full_c) {
        constexpr bool kFull_ = decltype(full_c)::value;
        constexpr int kG1 = 1;  // (batched base-word loads measured slower with these loops)
#pragma unroll
        for (int c = 0; c < K; c += kG1) {
          uint32_t bw[kG1];
#pragma unroll
          for (int q = 0; q < kG1; ++q) bw[q] = lds_u32(f_cw + (pk[c + q] >> 16) * (uint32_t)(WH1_ * 4));
#pragma unroll
          for (int q = 0; q < kG1; ++q)
            if (kFull_ || iw + (c + q) * 32 + lane < n) {
              const uint32_t pos = prmt(bw[q], 0u, f_sel16) + (pk[c + q] & 0xffffu);
              sts_u32(f_sb + pos * 4, pay[c + q]);
              sts_u16(a_tag + pos * 2, pk[c + q] >> 16);
            }
        }
      };
      if (n == (uint32_t)PT) fstage(std::true_type{});
      else fstage(std::false_type{});
    } else
      stage_tag<kStageG, K, uint16_t, kSlab>(pk, pay, s_cnt, WH1_, w, sh, s_buf, s_tag,
                                              (n == (uint32_t)PT) ? 0xffffffffu : n, iw + lane);
    __syncthreads();  // (C)
    const uint32_t nout = kSlab ? s_nst : n;  // staged items
    if constexpr (kFast) {
      const uint32_t a_b = f_sb + tid * 4, a_t = f_sb + (uint32_t)(PTP * 4) + tid * 2;
      uint32_t* outp = a.out + tid;
      if (n == (uint32_t)PT) {
#pragma unroll
        for (int k = 0; k < PT / T1_; ++k)
          outp[lds_u32(f_delta + lds_u16(a_t + k * (T1_ * 2)) * 4) + k * T1_] = lds_u32(a_b + k * (T1_ * 4));
      } else {
        for (uint32_t i = tid, k = 0; i < n; i += T1_, ++k)
          outp[lds_u32(f_delta + lds_u16(a_t + k * (T1_ * 2)) * 4) + k * T1_] = lds_u32(a_b + k * (T1_ * 4));
      }
    }
    else if constexpr (kW64) writeout_tag<T1_, PT>(a.out, s_buf, s_tag, s_g64, nout);
    else writeout_tag<T1_, PT>(a.out, s_buf, s_tag, s_delta, nout);
    if constexpr (kFast) {
      zero_s<T1_, PT / 2>(f_sb + kOffMark, tid);
      zero_s<T1_>(f_sb + kOffCnt, (uint32_t)round4(D * WH1_), tid);
      for (uint32_t d = tid; d < (uint32_t)D; d += T1_) {
        const uint32_t ag = f_delta - (uint32_t)D * 4 + d * 4;  // s_gcur += s_dtot
        sts_u32(ag, lds_u32(ag) + lds_u32(f_delta + (uint32_t)D * 4 + d * 4));
      }
    } else {
      zero_u32(reinterpret_cast<uint32_t*>(s_mark), PT / 2);
      zero_u32(s_cnt, round4(D * WH1_));
      if constexpr (!kW64)
        for (int d = tid; d < D; d += T1_) s_gcur[d] += s_dtot[d];
    }
    if (tid < 32) s_lastm[tid] = 0;
    fence_proxy_async_smem();
    __syncthreads();  // (D)
    if (kSlab && tid == 0) s_nst = 0;  // (read above, before (D); incremented again after the next (A))
    if (tid == 0 && j + 1 < nplace) issue(j + 1);
  }
}

// -------------------------------------------------- record passes (L2, L3-big)
// Count: histogram of the digit over each tile -> cnt[(g - j) * D + d * nt + j].
// Persistent (grid-stride over *n_tiles).
__global__ void __launch_bounds__(512) k_cnt_rec(const uint32_t* __restrict__ rec, const RTile* __restrict__ tiles,
                                                 const uint32_t* __restrict__ n_tiles, int D, DigSM dig,
                                                 uint32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) uint32_t s_h[];
  const uint32_t nt_all = *n_tiles;
  for (uint32_t g = blockIdx.x; g < nt_all; g += gridDim.x) {
    const RTile t = tiles[g];
    for (int d = threadIdx.x; d < D; d += blockDim.x) s_h[d] = 0;
    __syncthreads();
    const uint32_t* p = rec + t.start;
    const uint32_t n = t.n;
    const uint32_t head = min(n, (4 - align_items_u32(p)) & 3);
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) smem_inc(&s_h[dig(p[i])]);
    const uint4* p4 = reinterpret_cast<const uint4*>(p + head);
    const uint32_t n4 = (n - head) >> 2;
    auto ld4 = [](const uint4* a) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
      return v;
    };
    auto inc4 = [&](const uint4& v) {
      smem_inc(&s_h[dig(v.x)]);
      smem_inc(&s_h[dig(v.y)]);
      smem_inc(&s_h[dig(v.z)]);
      smem_inc(&s_h[dig(v.w)]);
    };
    const uint32_t bd = blockDim.x;
    uint32_t q = threadIdx.x;
    for (; q + 3 * bd < n4; q += 4 * bd) {  // four 16-byte loads in flight per thread
      const uint4 v0 = ld4(p4 + q), v1 = ld4(p4 + q + bd), v2 = ld4(p4 + q + 2 * bd), v3 = ld4(p4 + q + 3 * bd);
      inc4(v0);
      inc4(v1);
      inc4(v2);
      inc4(v3);
    }
    for (; q < n4; q += bd) inc4(ld4(p4 + q));
    for (uint32_t i = head + n4 * 4 + threadIdx.x; i < n; i += blockDim.x) smem_inc(&s_h[dig(p[i])]);
    __syncthreads();
    const uint64_t row0 = (uint64_t)(g - t.j) * D + t.j;
    for (int d = threadIdx.x; d < D; d += blockDim.x) cnt[row0 + (uint64_t)d * t.nt] = s_h[d];
    __syncthreads();
  }
}

// Count over digit bytes (level-3 big buckets of wide graphs): same tables as k_cnt_rec.
__global__ void __launch_bounds__(512) k_cnt_lv(const uint8_t* __restrict__ lv, const RTile* __restrict__ tiles,
                                                const uint32_t* __restrict__ n_tiles, int D,
                                                uint32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) uint32_t s_h[];
  const uint32_t nt_all = *n_tiles;
  for (uint32_t g = blockIdx.x; g < nt_all; g += gridDim.x) {
    const RTile t = tiles[g];
    for (int d = threadIdx.x; d < D; d += blockDim.x) s_h[d] = 0;
    __syncthreads();
    const uint8_t* p = lv + t.start;
    const uint32_t n = t.n;
    const uint32_t head = min(n, (uint32_t)((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15));
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) smem_inc(&s_h[p[i]]);
    const uint4* p4 = reinterpret_cast<const uint4*>(p + head);
    const uint32_t n16 = (n - head) >> 4;
    for (uint32_t q = threadIdx.x; q < n16; q += blockDim.x) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p4 + q));
      const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int bb = 0; bb < 32; bb += 8) smem_inc(&s_h[(wd[k] >> bb) & 0xffu]);
    }
    for (uint32_t i = head + n16 * 16 + threadIdx.x; i < n; i += blockDim.x) smem_inc(&s_h[p[i]]);
    __syncthreads();
    const uint64_t row0 = (uint64_t)(g - t.j) * D + t.j;
    for (int d = threadIdx.x; d < D; d += blockDim.x) cnt[row0 + (uint64_t)d * t.nt] = s_h[d];
    __syncthreads();
  }
}

// After one device-wide exclusive scan of all segments' count tables
// (concatenated in segment order, k_scan_lookback): rebase each segment to its
// output position (base += S.base - base[g0 * D]), write the digit starts
// out[out_off + d] (when < out_limit) and flag digit totals >= 2^32.  Threads
// of a CTA stride over one segment's D * nt entries (grid-stride over
// segments); large segments are cheap because the scan already did the work.
__global__ void __launch_bounds__(512) k_segfix(const SegDesc* __restrict__ segs, const uint32_t* __restrict__ n_segs,
                                                int D, uint64_t* __restrict__ base, uint64_t* __restrict__ out,
                                                uint64_t out_limit, unsigned int* __restrict__ err) {
  const uint32_t ns = *n_segs;
  for (uint32_t sg = blockIdx.x; sg < ns; sg += gridDim.x) {
    const SegDesc S = segs[sg];
    const uint64_t t0 = (uint64_t)S.g0 * D, n = (uint64_t)D * S.nt;
    if (n == 0) {  // empty segment (empty coarse bucket): every digit starts at S.base
      for (int d = threadIdx.x; d < D; d += blockDim.x)
        if (S.out_off + d < out_limit) out[S.out_off + d] = S.base;
      continue;
    }
    const uint64_t v0 = base[t0];
    __syncthreads();  // every thread has read v0 before any entry changes
    const uint64_t adj = S.base - v0;
    if (adj)
      for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) base[t0 + i] += adj;
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const uint64_t st = base[t0 + (uint64_t)d * S.nt];
      if (S.out_off + d < out_limit) out[S.out_off + d] = st;
      const uint64_t nx = (d + 1 < D) ? base[t0 + (uint64_t)(d + 1) * S.nt] : S.end;
      if (nx - st >= (1ull << 32)) atomicExch(err, 1u);
    }
    __syncthreads();
  }
}

// Record decoders for k_p2.
// DecR1 (level 2): R1 -> R2; digit = fine digit B; source high bits from the
// coarse bucket's seg_hi row (h = h0 + #boundaries <= position).
struct DecR1 {
  int L;
  uint32_t src_mask;
  int shB;
  uint32_t maskB;
  uint32_t lvmask;  // (1 << (c + gbits)) - 1
  int nbs;
  uint32_t nh;
  const uint64_t* seg_hi;
  static constexpr bool kSrcHigh = true;
  static constexpr bool kMatchRank = false;  // fine digits are spread: lane-ordered atomics
  __device__ __forceinline__ uint32_t digit(uint32_t r) const { return (r >> shB) & maskB; }
  // the same without the mask: B is the top field of R1 (shB = L + c = 32 - b; clamped shift: b = 0 gives 0)
  __device__ __forceinline__ uint32_t digit_top(uint32_t r) const { return __funnelshift_rc(r, 0u, (uint32_t)shB); }
  __device__ __forceinline__ uint32_t payload(uint32_t r, uint32_t h) const {
    return (((r >> L) & lvmask) << nbs) | (h << L) | (r & src_mask);
  }
};
// DecR2 (level 3, big fine buckets): R2 -> source; digit = low digit C.
struct DecR2 {
  int nbs;
  uint32_t src_mask;
  uint32_t maskC;
  static constexpr bool kSrcHigh = false;
  static constexpr bool kMatchRank = true;  // big buckets are dominated by a few hub vertices
  __device__ __forceinline__ uint32_t digit(uint32_t r) const { return (r >> nbs) & maskC; }
  __device__ __forceinline__ uint32_t payload(uint32_t r, uint32_t) const { return r & src_mask; }
};

// k_p2 record I/O forms.  Wide graphs (E >= 2^32 or 29+-bit sources) keep R2
// as two arrays at CSC positions: the source (u32) and the low digit (u8).
constexpr int kIoPlain = 0;  // u32 records in, u32 out (absolute u32 positions)
constexpr int kIoSplit = 1;  // level 2 of wide graphs: R1 in; source + low-digit byte out
constexpr int kIoLv = 2;     // level 3 big buckets of wide graphs: source + digit byte in, source out
// Wide forms use 64-bit output positions: the per-digit cursor array holds the
// cursor between place tiles and the index delta during one (as in k_p1 kW64).

inline size_t smem_p2(int D, int mode, int KK = K, int io = kIoPlain, int WW = W, int s64 = -1) {
  const size_t pt = (size_t)WW * KK * 32;
  const int wh = WW / 2 + 1, wp = WW + 1;
  if (s64 < 0) s64 = (io == kIoPlain && KK <= 16);  // measured: C3 level 2 2.115 -> 2.075 ms; 8192-record tiles slower
  return (s64 ? pt * 8 : (pt + 8) * 4 + pt * 2) + ((size_t)round4(D * wh) + (mode == kRankSafe ? (size_t)round4(D * wp) : 0)) * 4 + (size_t)D * 4 * 4 +
         40 * 4 + (size_t)kMaxBnd * 4 + (io != kIoPlain ? pt + 16 : 0);
}

// Owner search over a u32 boundary list (positions relative to the tile):
// result for lane l = largest k in [cur, upper] with k == cur or b(k) <= p0 + l.
template <class F>
__device__ __forceinline__ uint32_t slot_owner32(uint32_t& cur, uint32_t& nb, uint32_t p0, uint32_t upper, F bnd_at) {
  if (nb > p0 + 31) return cur;
  const uint32_t lane = lane_id();
  uint32_t base = cur, acc = 0, res;
  while (true) {
    const uint32_t kk = base + 1 + lane;
    const uint32_t bj = (kk <= upper) ? bnd_at(kk) : 0xffffffffu;
    const uint32_t rel = (bj <= p0 + 31) ? bj - p0 : 32u;
    acc += count_le_lane(rel, lane);
    if (__shfl_sync(kFull, rel, 31) >= 32) break;
    base += 32;
  }
  res = cur + acc;
  cur = __shfl_sync(kFull, res, 31);
  nb = (cur + 1 <= upper) ? bnd_at(cur + 1) : 0xffffffffu;
  return res;
}

// Place: per tile, place tiles of PT records are ranked by digit, staged with
// their global indices, and written out (persistent, grid-stride over tiles).
// kS64: staged items as (payload, digit) pairs, one 8-byte store / load each (the
// landing buffer is dead after ranking and the pair array overlays it).
template <int kMode, class Dec, int KK, bool kProf = false, int kIO = kIoPlain, bool kPre = true, int WW = W,
          int kMinB = (KK > 16 ? 2 : 4), bool kS64 = (kIO == kIoPlain && KK <= 16), bool kOpt = true>
__global__ void __launch_bounds__(WW * 32, kMinB) k_p2(const uint32_t* __restrict__ rec, const RTile* __restrict__ tiles,
                                             const uint32_t* __restrict__ n_tiles, int D, Dec dec,
                                             const uint64_t* __restrict__ base, uint32_t* __restrict__ out,
                                             unsigned long long* __restrict__ prof = nullptr,
                                             const uint8_t* __restrict__ lv_in = nullptr,
                                             uint8_t* __restrict__ lv_out = nullptr) {
  // phase profile (kProf builds only; thread 0, clock64): 0 tile setup, 1 wait,
  // 2 rank, 3 bases, 4 stage, 5 write
  unsigned long long pacc[kProf ? 6 : 1] = {};
  long long tprev = kProf ? clock64() : 0;
  auto tick = [&](int ph) {
    if constexpr (kProf) {
      if (threadIdx.x == 0) {
        const long long t = clock64();
        pacc[ph] += (unsigned long long)(t - tprev);
        tprev = t;
      }
    }
  };
  constexpr int W2_ = WW, T2_ = WW * 32, WH2_ = WW / 2 + 1, WP2_ = WW + 1;
  constexpr int PT = W2_ * KK * 32, PTP = PT + 8, K = KK;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem);                         // PTP (kS64: PT pairs overlay it)
  uint2* s_st64 = reinterpret_cast<uint2*>(smem);                              // kS64: PT staged (payload, digit)
  uint16_t* s_tag = reinterpret_cast<uint16_t*>(s_buf + PTP);                 // PT (digit of each staged slot)
  uint32_t* s_cnt = kS64 ? reinterpret_cast<uint32_t*>(smem + (size_t)PT * 8)
                         : reinterpret_cast<uint32_t*>(s_tag + PT);            // D * WH2_ (packed, digit-major)
  uint32_t* s_scr = s_cnt + round4(D * WH2_);                                    // D * WP2_ (safe)
  uint32_t* s_gcur = s_scr + (kMode == kRankSafe ? round4(D * WP2_) : 0);        // D
  uint32_t* s_delta = s_gcur + D;                                              // D
  uint32_t* s_dstart = s_delta + D;                                            // D
  uint32_t* s_dtot = s_dstart + D;                                             // D
  uint32_t* s_tmp = s_dtot + D;                                                // 40
  uint32_t* s_bnd = s_tmp + 40;                                                // kMaxBnd
  constexpr bool kW64 = (kIO != kIoPlain);
  uint64_t* s_g64 = reinterpret_cast<uint64_t*>(s_gcur);  // kW64: spans s_gcur + s_delta; s_dtot = digit end
  // kIoSplit: low-digit byte of each staged slot; kIoLv: landing of the digit bytes (16B aligned)
  uint8_t* s_lvx = reinterpret_cast<uint8_t*>(s_bnd + kMaxBnd);                // PT + 16
  __shared__ __align__(8) uint64_t s_bar;

  const uint32_t tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const uint32_t sh = (w & 1) << 4;
  const uint32_t ntall = *n_tiles;
  zero_u32(s_cnt, round4(D * WH2_) + (kMode == kRankSafe ? round4(D * WP2_) : 0));
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph = 0;
  // kFast: rank and stage through 32-bit shared addresses off laundered registers (gt_common.cuh)
  constexpr bool kFast = kOpt && kMode == kRankAtomic && kIO == kIoPlain;
  // byte offset of the counter table: behind the pair array (kS64) or behind landing buffer + tags
  constexpr uint32_t kOffCnt = kS64 ? (uint32_t)PT * 8 : (uint32_t)(PTP * 4 + PT * 2);
  uint32_t f_sb = 0, f_cw = 0, f_inc = 0, f_selr = 0, f_sel16 = 0, f_himask = 0, f_mul = 0, f_srcm = 0, f_delta = 0;
  bool f_up = true;
  if constexpr (kFast) {
    f_sb = launder(smem_u32(smem));
    f_delta = launder(smem_u32(s_delta));
    f_cw = launder(f_sb + kOffCnt + (w >> 1) * 4);  // this warp's word of every digit row
    f_inc = launder(1u << sh);
    f_selr = launder((w & 1) ? 0x5432u : 0x5410u);   // (old field, digit) -> digit << 16 | rank
    f_sel16 = launder((w & 1) ? 0x4432u : 0x4410u);  // this warp's u16 field of a counter word
    if constexpr (Dec::kSrcHigh) {  // R1 -> R2: (r & himask) * mul moves the low-digit field above the source bits
      f_up = dec.nbs >= dec.L;      // (small graphs: the field moves down instead; they take the generic slots)
      f_himask = launder(dec.lvmask << dec.L);
      f_mul = launder(1u << (f_up ? dec.nbs - dec.L : 0));
      f_srcm = launder(dec.src_mask);
    }
  }

  for (uint32_t g = blockIdx.x; g < ntall; g += gridDim.x) {
    const RTile t = tiles[g];
    const uint64_t row0 = (uint64_t)(g - t.j) * D + t.j;
    for (int d = tid; d < D; d += T2_) {
      if constexpr (kW64) s_g64[d] = base[row0 + (uint64_t)d * t.nt];
      else s_gcur[d] = (uint32_t)base[row0 + (uint64_t)d * t.nt];
    }
    const uint32_t nbt = Dec::kSrcHigh ? t.nbnd : 0u;
    const uint64_t* hrow = nullptr;
    if constexpr (Dec::kSrcHigh) {
      hrow = dec.seg_hi + (uint64_t)t.seg * (dec.nh + 1) + t.h0 + 1;  // boundary k (1-based) = hrow[k - 1]
      if (nbt <= (uint32_t)kMaxBnd)
        for (uint32_t q = tid; q < nbt; q += T2_) s_bnd[q] = (uint32_t)(hrow[q] - t.start);
    }
    const int nplace = (int)((t.n + PT - 1) / PT);
    auto issue = [&](int jj) {  // thread 0
      const uint64_t pt = t.start + (uint64_t)jj * PT;
      const uint32_t n = min((uint32_t)PT, t.n - jj * PT);
      const uint32_t* gp = rec + pt;
      const uint32_t o = align_items_u32(gp);
      const uint32_t full = (o + n) & ~3u;
      fence_proxy_async_smem();
      if constexpr (kIO == kIoLv) {  // the digit bytes: whole 16-byte blocks (the array is padded)
        const uint8_t* gl = lv_in + pt;
        const uint32_t o8 = (uint32_t)(reinterpret_cast<uintptr_t>(gl) & 15);
        const uint32_t nb8 = (o8 + n + 15) & ~15u;
        mbar_arrive_expect_tx(&s_bar, full * 4 + nb8);
        bulk_g2s(s_lvx, gl - o8, nb8, &s_bar);
      } else {
        mbar_arrive_expect_tx(&s_bar, full * 4);
      }
      if (full) bulk_g2s(s_buf, gp - o, full * 4, &s_bar);
      if (jj + 1 < nplace) {
        const uint32_t* gn = gp + PT;
        const uint32_t on = align_items_u32(gn);
        const uint32_t nn = min((uint32_t)PT, t.n - (jj + 1) * PT);
        const uint32_t fn = (on + nn) & ~3u;
        if (fn) bulk_prefetch_l2(gn - on, fn * 4);
      }
    };
    __syncthreads();  // s_gcur / s_bnd visible; the previous tile's buffers are free
    if (tid == 0 && nplace > 0) issue(0);
    for (int jj = 0; jj < nplace; ++jj) {
      if constexpr (kW64) {  // delta -> cursor of this place tile (after barrier (D))
        if (jj > 0)
          for (int d = tid; d < D; d += T2_) s_g64[d] += s_dtot[d];
      }
      const uint64_t pt = t.start + (uint64_t)jj * PT;
      const uint32_t n = min((uint32_t)PT, t.n - jj * PT);
      const uint32_t* gp = rec + pt;
      const uint32_t o = align_items_u32(gp);
      const uint32_t full = (o + n) & ~3u;
      const uint32_t ti = full + tid;
      const bool tail = tid < 4 && ti < o + n;
      uint32_t tv = 0;
      if (tail) tv = ldg_u32(gp - o + ti);
      tick(0);
      mbar_wait_parity(&s_bar, ph);
      ph ^= 1;
      if (tail) s_buf[ti] = tv;
      __syncthreads();  // (A)
      tick(1);

      // level-3 big buckets (many partial tiles): a partial tile's records are split evenly over
      // the warps (consecutive ranges in warp order) and warps skip the slots beyond their range
      // (measured: big buckets 0.778 -> 0.765 ms on C3; level 2 slower with it, 2.11 -> 2.16 ms)
      constexpr bool kBal2 = Dec::kMatchRank;
      const uint32_t per = (!kBal2 || n == (uint32_t)PT) ? (uint32_t)(K * 32) : ((n + T2_ - 1) / T2_) * 32;
      const uint32_t iw = w * per;
      const uint32_t rel0 = (uint32_t)jj * PT;  // tile-relative position of item 0
      uint32_t cur = 0, nb = 0xffffffffu;
      auto bnd_at = [&](uint32_t kk) -> uint32_t {  // kk in [1, nbt]
        return (nbt <= (uint32_t)kMaxBnd) ? s_bnd[kk - 1] : (uint32_t)(hrow[kk - 1] - t.start);
      };
      if constexpr (Dec::kSrcHigh) {
        if (nbt) {
          cur = owner_search(0u, nbt, (uint64_t)rel0 + iw, [&](uint64_t kk) -> uint64_t { return bnd_at((uint32_t)kk); });
          nb = (cur + 1 <= nbt) ? bnd_at(cur + 1) : 0xffffffffu;
        }
      }
      // warps whose items hold no source-high boundary keep h constant
      const bool wbnd = nb <= rel0 + iw + (per - 1);
      const uint32_t o8 = (kIO == kIoLv) ? (uint32_t)(reinterpret_cast<uintptr_t>(lv_in + pt) & 15) : 0u;
      // pk = digit << 16 | rank; kIoSplit: low-digit byte << 24 | digit << 13 | rank (rank < 8192, digit < 2048)
      constexpr int kDS = (kIO == kIoSplit) ? 13 : 16;
      uint32_t pay[K], pk[K];
      if (kBal2 && n != (uint32_t)PT) {
#pragma unroll
        for (int s = 0; s < K; ++s) pk[s] = 0;  // slots a warp skips stage nothing
      }
      auto slot = [&](int s, bool valid) {  // pay[s] holds the slot's record (loaded below)
        const uint32_t i0 = iw + s * 32, i = i0 + lane;
        const uint32_t r = valid ? (kPre ? pay[s] : s_buf[o + i]) : 0u;
        uint32_t h = t.h0;
        if constexpr (Dec::kSrcHigh) h += wbnd ? slot_owner32(cur, nb, rel0 + i0, nbt, bnd_at) : cur;
        uint32_t d;
        if constexpr (kIO == kIoLv) d = valid ? (uint32_t)s_lvx[o8 + i] : 0u;
        else d = dec.digit(r);
        uint32_t rk;
        if constexpr (Dec::kMatchRank) rk = rank_match(s_cnt + d * WH2_ + (w >> 1), sh, d, valid);
        else rk = rank_pk<kMode>(s_cnt + d * WH2_ + (w >> 1), s_scr + d * WP2_ + w, sh, valid);
        if constexpr (kIO == kIoSplit) {
          pk[s] = (((r >> dec.L) & dec.lvmask) << 24) | (d << 13) | rk;
          pay[s] = (h << dec.L) | (r & dec.src_mask);
        } else {
          pk[s] = (d << 16) | rk;
          pay[s] = dec.payload(r, h);
        }
      };
      if constexpr (kPre) {
#pragma unroll
        for (int s = 0; s < K; ++s) pay[s] = s_buf[o + iw + s * 32 + lane];  // in bounds: iw + K * 32 <= PT
      }
      bool fdone = false;
      if constexpr (kFast) {
        if (!wbnd && f_up) {  // no source-high boundary inside this warp's items: h is constant
          fdone = true;
          uint32_t hl = 0;
          if constexpr (Dec::kSrcHigh) hl = (t.h0 + cur) << dec.L;
          const uint32_t a_rec = f_sb + (o + iw + lane) * 4;
          auto fslot = [&](int s, bool valid) {
            uint32_t r = 0;
            if constexpr (kPre) r = valid ? pay[s] : 0u;
            else if (valid) r = lds_u32(a_rec + s * 128);
            uint32_t d;
            if constexpr (Dec::kSrcHigh) d = dec.digit_top(r);
            else d = dec.digit(r);
            if constexpr (Dec::kMatchRank) {  // one atomic per distinct digit of the slot
              const uint32_t m = __match_any_sync(kFull, valid ? d : 0xffffffffu);
              const uint32_t ld = __ffs(m) - 1;
              uint32_t old = 0;
              if (valid && lane == ld) old = atoms_add(f_cw + d * (uint32_t)(WH2_ * 4), (uint32_t)__popc(m) << sh);
              old = __shfl_sync(kFull, old, ld);
              pk[s] = prmt(old, d, f_selr) + __popc(m & lanemask_lt());
            } else {
              uint32_t old = 0;
              if (valid) old = atoms_add(f_cw + d * (uint32_t)(WH2_ * 4), f_inc);
              pk[s] = prmt(old, d, f_selr);
            }
            if constexpr (Dec::kSrcHigh) pay[s] = (r & f_himask) * f_mul + ((r & f_srcm) | hl);
            else pay[s] = dec.payload(r, 0u);
          };
          if (n == (uint32_t)PT) {
#pragma unroll
            for (int s = 0; s < K; ++s) fslot(s, true);
          } else {
#pragma unroll
            for (int s = 0; s < K; ++s) {
              if (kBal2 && (uint32_t)s * 32 >= per) break;
              fslot(s, iw + s * 32 + lane < n);
            }
          }
        }
      }
      if (fdone) {
      } else if (n == (uint32_t)PT) {
#pragma unroll
        for (int s = 0; s < K; ++s) slot(s, true);
      } else {
#pragma unroll
        for (int s = 0; s < K; ++s) {
          if (kBal2 && (uint32_t)s * 32 >= per) break;
          slot(s, iw + s * 32 + lane < n);
        }
      }
      __syncthreads();  // (B)
      tick(2);
      bool fscan = false;  // kFast: scanned by flat_scan_any (the cursors advance in its epilogue)
      if constexpr (kW64)
        flat_bases_epi<WH2_>(s_cnt, D, s_tmp, [&](int d, uint32_t b, uint32_t e) {
          s_g64[d] -= b;
          s_dtot[d] = e;
        });
      else {
        if constexpr (kFast) {
          const uint32_t a_cnt = f_sb + kOffCnt;
          fscan = flat_scan_any<T2_, (KK > 16 ? 21 : 11)>(a_cnt, (uint32_t)(D * WH2_), smem_u32(s_tmp), tid);
          if (fscan) {  // per digit: index delta of this tile, cursor of the next (s_gcur is not read in between)
            for (int d = tid; d < D; d += T2_) {
              const uint32_t ar = a_cnt + d * (WH2_ * 4);
              const uint32_t b = lds_u32(ar) & 0xffffu, e = lds_u32(ar + (WH2_ - 1) * 4) & 0xffffu;
              const uint32_t ag = f_delta - (uint32_t)D * 4 + d * 4;  // s_gcur
              const uint32_t gc = lds_u32(ag);
              sts_u32(f_delta + d * 4, gc - b);
              sts_u32(ag, gc + (e - b));
            }
            __syncthreads();
          }
        }
        if (!fscan) flat_bases_pk<WH2_>(s_cnt, D, s_gcur, s_dtot, s_delta, s_tmp);
      }
      tick(3);
      if constexpr (kFast) {
        constexpr int G = 1;  // (batched base-word loads measured slower with these loops)
        auto fstage = [&](auto full_c) {
          constexpr bool kFull_ = decltype(full_c)::value;
#pragma unroll
          for (int c = 0; c < K; c += G) {
            uint32_t bw[G];
#pragma unroll
            for (int q = 0; q < G; ++q) bw[q] = lds_u32(f_cw + (pk[c + q] >> 16) * (uint32_t)(WH2_ * 4));
#pragma unroll
            for (int q = 0; q < G; ++q)
              if (kFull_ || ((uint32_t)(c + q) * 32 < per && iw + (c + q) * 32 + lane < n)) {
                const uint32_t pos = prmt(bw[q], 0u, f_sel16) + (pk[c + q] & 0xffffu);
                if constexpr (kS64) {
                  sts_v2(f_sb + pos * 8, pay[c + q], pk[c + q] >> 16);
                } else {
                  sts_u32(f_sb + pos * 4, pay[c + q]);
                  sts_u16(f_sb + (uint32_t)(PTP * 4) + pos * 2, pk[c + q] >> 16);
                }
              }
          }
        };
        if (n == (uint32_t)PT) fstage(std::true_type{});
        else fstage(std::false_type{});
      } else if constexpr (kS64) {
        stage_pair<kPre ? kStageG : 1, K>(pk, pay, s_cnt, WH2_, w, sh, s_st64, (n == (uint32_t)PT) ? 0xffffffffu : n,
                                          iw + lane, per);
      } else if constexpr (kIO != kIoSplit) {
        stage_tag<kPre ? kStageG : 1, K>(pk, pay, s_cnt, WH2_, w, sh, s_buf, s_tag, (n == (uint32_t)PT) ? 0xffffffffu : n, iw + lane,
                                         per);
      } else {
#pragma unroll
      for (int s = 0; s < K; ++s) {
        if (n == (uint32_t)PT || ((uint32_t)s * 32 < per && iw + s * 32 + lane < n)) {
          const uint32_t d = (pk[s] >> kDS) & ((kIO == kIoSplit) ? 0x7ffu : 0xffffu);
          const uint32_t pos = ((s_cnt[d * WH2_ + (w >> 1)] >> sh) & 0xffffu) + (pk[s] & ((1u << kDS) - 1));
          s_buf[pos] = pay[s];
          s_tag[pos] = (uint16_t)d;
          if constexpr (kIO == kIoSplit) s_lvx[pos] = (uint8_t)(pk[s] >> 24);
        }
      }
      }
      __syncthreads();  // (C)
      tick(4);
      if constexpr (kFast) {
        const uint32_t a_st = f_sb + tid * (kS64 ? 8 : 4), a_tg = f_sb + (uint32_t)(PTP * 4) + tid * 2;
        uint32_t* outp = out + tid;
        auto put = [&](uint32_t k) {
          if constexpr (kS64) {
            const uint2 v = lds_v2(a_st + k * (T2_ * 8));
            outp[lds_u32(f_delta + v.y * 4) + k * T2_] = v.x;
          } else {
            outp[lds_u32(f_delta + lds_u16(a_tg + k * (T2_ * 2)) * 4) + k * T2_] = lds_u32(a_st + k * (T2_ * 4));
          }
        };
        if (n == (uint32_t)PT) {
#pragma unroll
          for (int k = 0; k < PT / T2_; ++k) put(k);
        } else {
          for (uint32_t i = tid, k = 0; i < n; i += T2_, ++k) put(k);
        }
      } else if constexpr (kS64) {
        writeout_pair<T2_, PT>(out, s_st64, s_delta, n);
      } else if constexpr (kIO == kIoPlain) {
        writeout_tag<T2_, PT>(out, s_buf, s_tag, s_delta, n);
      } else {  // 64-bit positions
        auto put = [&](uint32_t i) {
          const uint64_t q = s_g64[s_tag[i]] + i;
          out[q] = s_buf[i];
          if constexpr (kIO == kIoSplit) lv_out[q] = s_lvx[i];
        };
        if (n == (uint32_t)PT) {
#pragma unroll
          for (int q = 0; q < PT / T2_; ++q) put(threadIdx.x + q * T2_);
        } else {
          for (uint32_t i = threadIdx.x; i < n; i += T2_) put(i);
        }
      }
      if constexpr (kFast) zero_s<T2_>(f_sb + kOffCnt, (uint32_t)round4(D * WH2_), tid);
      else zero_u32(s_cnt, round4(D * WH2_));
      if constexpr (!kW64)
        if (!fscan)
          for (int d = tid; d < D; d += T2_) s_gcur[d] += s_dtot[d];
      fence_proxy_async_smem();
      __syncthreads();  // (D)
      tick(5);
      if (tid == 0 && jj + 1 < nplace) issue(jj + 1);
    }
  }
  if constexpr (kProf) {
    if (threadIdx.x == 0)
      for (int q = 0; q < 6; ++q) atomicAdd(&prof[q], pacc[q]);
  }
}

// ---------------------------------------------------------------- L3 units
struct P3Args {
  const uint32_t* rec;  // R2 at CSC positions
  const Unit3* units;
  const uint32_t* n_units;
  unsigned int* ctr;
  int c, nbs;
  uint32_t src_mask, mask_c;
  const uint64_t* fbase;  // CSC start of every fine bucket (+ total)
  int gbits;              // kPosFine == false: R2 keeps (fine & (2^gbits - 1)) << c | low digit
  uint32_t lvmask;        //   = (1 << (c + gbits)) - 1
  unsigned long long* prof;  // kProf builds: 6 phase-cycle accumulators
  uint64_t V;
  uint64_t* t_offsets;
  uint32_t* t_edges;
  const uint8_t* lv;  // kLv: low digit of every R2 record (wide graphs; rec then holds the bare source)
};

constexpr int CAP3L = CAP3 + 16;  // digit-byte landing per buffer (whole 16-byte blocks)
inline size_t smem_p3(int mode, bool lv = false, int ww = W3) {
  const size_t cap = (size_t)ww * K3 * 32;
  const int wh = ww / 2 + 1, wp = ww + 1;
  return (size_t)2 * (cap + 8) * 4 + ((size_t)round4(ML3 * wh) + (mode == kRankSafe ? (size_t)round4(ML3 * wp) : 0)) * 4 +
         (size_t)ML3 * 8 + 40 * 4 + (lv ? (size_t)2 * (cap + 16) : 0);
}

// kPosFine: the record's fine bucket inside the unit comes from its position
// (R2 has no room for fine-digit bits); else from the record's bits.
// kLv (requires kPosFine): the low digit comes from the separate byte array.
// kBal: a unit's n records are split evenly over the warps (ceil(n / 512) slots
// each, consecutive ranges in warp order) and warps skip their empty slots;
// otherwise every warp owns 512 positions and partial units run predicated slots.
template <int kMode, bool kPosFine, bool kProf = false, bool kLv = false, bool kPre = true, int WW3 = W3,
          bool kBal = true, bool kOpt = true>
__global__ void __launch_bounds__(WW3 * 32, WW3 > 16 ? 1 : 2) k_p3(const P3Args a) {
  // phase profile (kProf builds only; thread 0, clock64): 0 fetch/issue, 1 wait, 2 rank, 3 bases+offsets, 4 stage, 5 store
  unsigned long long pacc[kProf ? 6 : 1] = {};
  long long tprev = kProf ? clock64() : 0;
  auto tick = [&](int ph) {
    if constexpr (kProf) {
      if (threadIdx.x == 0) {
        const long long t = clock64();
        pacc[ph] += (unsigned long long)(t - tprev);
        tprev = t;
      }
    }
  };
  constexpr int W3_ = WW3, TT = W3_ * 32, CAP3_ = W3_ * K3 * 32, CAP3P_ = CAP3_ + 8, CAP3L_ = CAP3_ + 16;
  constexpr int WH3_ = W3_ / 2 + 1, W3P_ = W3_ + 1;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem);       // 2 * CAP3P_
  uint32_t* s_cnt = s_buf + 2 * CAP3P_;                       // ML3 * WH3_ (packed, digit-major)
  uint32_t* s_scr = s_cnt + round4(ML3 * WH3_);               // ML3 * W3P_ (safe)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? round4(ML3 * W3P_) : 0);
  uint32_t* s_dtot = s_dstart + ML3;
  uint32_t* s_tmp = s_dtot + ML3;
  uint8_t* s_lvb = reinterpret_cast<uint8_t*>(s_tmp + 40);  // kLv: 2 * CAP3L_ (16B aligned)
  static_assert(!kLv || kPosFine, "digit bytes imply position-derived fine buckets");
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_uidx[2];
  __shared__ uint32_t s_fb[ML3];  // fine-bucket boundaries of the unit (relative positions)

  const uint32_t tid = kOpt ? launder(threadIdx.x) : threadIdx.x, lane = tid & 31u, w = tid >> 5;  // (see k_p1)
  const uint32_t sh = (w & 1) << 4;
  const uint32_t nun = *a.n_units;
  zero_u32(s_cnt, round4(ML3 * WH3_) + (kMode == kRankSafe ? round4(ML3 * W3P_) : 0));
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  // kFast: rank and stage through 32-bit shared addresses off laundered registers (gt_common.cuh)
  constexpr bool kFast = kOpt && kMode == kRankAtomic && !kLv;
  uint32_t f_sb = 0, f_cw = 0, f_inc = 0, f_selr = 0, f_sel16 = 0;
  if constexpr (kFast) {
    f_sb = launder(smem_u32(smem));
    f_cw = launder(f_sb + (uint32_t)(2 * CAP3P_ * 4) + (w >> 1) * 4);
    f_inc = launder(1u << sh);
    f_selr = launder((w & 1) ? 0x5432u : 0x5410u);
    f_sel16 = launder((w & 1) ? 0x4432u : 0x4410u);
  }
  auto issue = [&](uint32_t ui, int b) {  // thread 0
    const Unit3 u = a.units[ui];
    const uint32_t* gp = a.rec + u.start;
    const uint32_t o = align_items_u32(gp);
    const uint32_t full = (o + u.n) & ~3u;
    fence_proxy_async_smem();
    if constexpr (kLv) {
      const uint8_t* gl = a.lv + u.start;
      const uint32_t o8 = (uint32_t)(reinterpret_cast<uintptr_t>(gl) & 15);
      const uint32_t nb8 = (o8 + u.n + 15) & ~15u;
      mbar_arrive_expect_tx(&s_bar[b], full * 4 + nb8);
      bulk_g2s(s_lvb + b * CAP3L_, gl - o8, nb8, &s_bar[b]);
    } else {
      mbar_arrive_expect_tx(&s_bar[b], full * 4);
    }
    if (full) bulk_g2s(s_buf + b * CAP3P_, gp - o, full * 4, &s_bar[b]);
  };
  // static round-robin over the units (they are many and bounded in size):
  // the next unit is known without a global atomic on the critical path
  if (tid == 0 && blockIdx.x < nun) issue(blockIdx.x, 0);
  __syncthreads();
  uint32_t ph0 = 0, ph1 = 0;
  for (int it = 0;; ++it) {
    const int b = it & 1;
    const uint32_t ui = blockIdx.x + (uint32_t)it * gridDim.x;
    if (ui >= nun) break;
    if (tid == 0) {  // prefetch the next unit into the other buffer (its last bulk store must have read it)
      const uint32_t un = ui + gridDim.x;
      bulk_wait_read<0>();
      if (un < nun) issue(un, b ^ 1);
    }
    const Unit3 u = a.units[ui];
    const uint32_t n = u.n;
    const uint32_t* gp = a.rec + u.start;
    const uint32_t o = align_items_u32(gp);
    const uint32_t full = (o + n) & ~3u;
    uint32_t* buf = s_buf + b * CAP3P_;
    const uint32_t ti = full + tid;
    const bool tail = ((o + n) & 3u) != 0 && tid < 4 && ti < o + n;  // (first test uniform)
    uint32_t tv = 0;
    if (tail) tv = ldg_u32(gp - o + ti);
    tick(0);
    if (b == 0) { mbar_wait_parity(&s_bar[0], ph0); ph0 ^= 1; }
    else { mbar_wait_parity(&s_bar[1], ph1); ph1 ^= 1; }
    if (tail) buf[ti] = tv;
    const uint32_t nbt = kPosFine ? u.nf - 1 : 0u;  // fine-bucket boundaries inside the unit
    if constexpr (kPosFine)
      for (uint32_t q = tid; q < nbt; q += TT) s_fb[q] = (uint32_t)(a.fbase[u.f0 + 1 + q] - u.start);
    __syncthreads();  // (A)
    tick(1);
    const uint32_t nloc = u.nf << a.c;
    const uint32_t per = kBal ? ((n + TT - 1) / TT) * 32 : (uint32_t)(K3 * 32);  // positions per warp
    const uint32_t seg0 = w * per;
    // local vertex = (fine bucket inside the unit, from the record's position) << c | low digit
    auto bnd_at = [&](uint32_t kk) -> uint32_t { return s_fb[kk - 1]; };
    uint32_t fcur = 0, fnb = 0xffffffffu;
    if (nbt) {
      fcur = owner_search(0u, nbt, (uint64_t)seg0, [&](uint64_t kk) -> uint64_t { return s_fb[kk - 1]; });
      fnb = (fcur + 1 <= nbt) ? s_fb[fcur] : 0xffffffffu;
    }
    const bool wbnd = fnb <= seg0 + (per - 1);
    const uint32_t lvoff = (u.f0 & ((1u << a.gbits) - 1)) << a.c;
    const uint8_t* lvb = s_lvb + b * CAP3L_ + (kLv ? (uint32_t)(reinterpret_cast<uintptr_t>(a.lv + u.start) & 15) : 0u);
    uint32_t rr[K3], pk[K3];
    constexpr int kG3 = kPre ? kStageG : 1;
    if constexpr (kPre) {
#pragma unroll
      for (int s = 0; s < K3; ++s) {  // all loads before the first rank atomic
        if (kBal && (uint32_t)s * 32 >= per) break;
        rr[s] = buf[o + seg0 + s * 32 + lane];
      }
    }
    bool fdone = false;
    if constexpr (kFast) {
      if (!kPosFine || !wbnd) {  // (kPosFine: no fine-bucket boundary inside this warp's positions)
        fdone = true;
        const uint32_t a_rec = f_sb + (uint32_t)b * (CAP3P_ * 4) + (o + seg0 + lane) * 4;
        const uint32_t nbs = a.nbs, srcm = a.src_mask;
        const uint32_t lvadd = kPosFine ? (fcur << a.c) : (0u - lvoff);
        // all of this warp's positions hold records (every warp but the unit's last one or two):
        // no per-lane validity tests
        auto frank = [&](auto all_c) {
          constexpr bool kAll = decltype(all_c)::value;
#pragma unroll
          for (int s = 0; s < K3; ++s) {
            if (kBal && (uint32_t)s * 32 >= per) break;
            const bool valid = kAll || seg0 + s * 32 + lane < n;
            uint32_t r = 0;
            if constexpr (kPre) r = valid ? rr[s] : 0u;
            else if (valid) r = lds_u32(a_rec + s * 128);
            // (no mask: the low-digit field is R2's top field, DecR1::payload keeps c + gbits bits)
            const uint32_t lv = valid ? ((r >> nbs) + lvadd) : 0u;
            uint32_t old = 0;
            if (valid) old = atoms_add(f_cw + lv * (uint32_t)(WH3_ * 4), f_inc);
            pk[s] = prmt(old, lv, f_selr);
            rr[s] = r & srcm;
          }
        };
        // (position-derived fine buckets, C4: one copy — the second one spills)
        if constexpr (kPosFine) {
          frank(std::false_type{});
        } else {
          if (seg0 + per <= n) frank(std::true_type{});
          else frank(std::false_type{});
        }
      }
    }
#pragma unroll
    for (int s = 0; s < K3; ++s) {
      if (fdone) break;
      if (kBal && (uint32_t)s * 32 >= per) break;
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      const uint32_t r = valid ? (kPre ? rr[s] : buf[o + i]) : 0u;
      uint32_t lv;
      if constexpr (kPosFine) {
        const uint32_t j = wbnd ? slot_owner32(fcur, fnb, seg0 + s * 32, nbt, bnd_at) : fcur;
        if constexpr (kLv) lv = valid ? ((j << a.c) | lvb[i]) : 0u;
        else lv = valid ? ((j << a.c) | ((r >> a.nbs) & a.mask_c)) : 0u;
      } else {
        lv = valid ? (((r >> a.nbs) & a.lvmask) - lvoff) : 0u;
      }
      pk[s] = (lv << 16) | rank_pk<kMode>(s_cnt + lv * WH3_ + (w >> 1), s_scr + lv * W3P_ + w, sh, valid);
      rr[s] = r & a.src_mask;
    }
    __syncthreads();  // (B)
    tick(2);
    {
      bool fscan = false;
      if constexpr (kFast)
        fscan = flat_scan_any<TT>(f_sb + (uint32_t)(2 * CAP3P_ * 4), nloc * WH3_, smem_u32(s_tmp), tid);
      if (!fscan) flat_bases_epi<WH3_, false>(s_cnt, (int)nloc, s_tmp, [](int, uint32_t, uint32_t) {});
    }
    {
      const uint64_t v0 = (uint64_t)u.f0 << a.c;
      for (uint32_t v = tid; v < nloc; v += TT)
        if (v0 + v < a.V) a.t_offsets[v0 + v] = u.start + (s_cnt[v * WH3_] & 0xffffu);
    }
    tick(3);
    uint32_t* t_e = a.t_edges + u.start;
    const uint32_t oo = align_items_u32(t_e);  // staging offset matching the output's 16B alignment
    if constexpr (kFast) {
      const uint32_t a_out = f_sb + (uint32_t)b * (CAP3P_ * 4) + oo * 4;
      auto fstage3 = [&](auto all_c) {
        constexpr bool kAll = decltype(all_c)::value;
#pragma unroll
        for (int c = 0; c < K3; c += kG3) {
          if (kBal && (uint32_t)c * 32 >= per) break;
          uint32_t bw[kG3];
#pragma unroll
          for (int q = 0; q < kG3; ++q)
            if (!kBal || (uint32_t)(c + q) * 32 < per) bw[q] = lds_u32(f_cw + (pk[c + q] >> 16) * (uint32_t)(WH3_ * 4));
#pragma unroll
          for (int q = 0; q < kG3; ++q)
            if ((!kBal || (uint32_t)(c + q) * 32 < per) && (kAll || seg0 + (c + q) * 32 + lane < n))
              sts_u32(a_out + (prmt(bw[q], 0u, f_sel16) + (pk[c + q] & 0xffffu)) * 4, rr[c + q]);
        }
      };
      if constexpr (kPosFine) {
        fstage3(std::false_type{});
      } else {
        if (seg0 + per <= n) fstage3(std::true_type{});
        else fstage3(std::false_type{});
      }
    }
#pragma unroll
    for (int c = 0; c < K3; c += kG3) {  // base words of kG3 items loaded before their stores
      if (kFast) break;
      if (kBal && (uint32_t)c * 32 >= per) break;
      uint32_t bw[kG3];
#pragma unroll
      for (int q = 0; q < kG3; ++q)
        if (!kBal || (uint32_t)(c + q) * 32 < per) bw[q] = s_cnt[(pk[c + q] >> 16) * WH3_ + (w >> 1)];
#pragma unroll
      for (int q = 0; q < kG3; ++q)
        if ((!kBal || (uint32_t)(c + q) * 32 < per) && seg0 + (c + q) * 32 + lane < n)
          buf[oo + ((bw[q] >> sh) & 0xffffu) + (pk[c + q] & 0xffffu)] = rr[c + q];
    }
    fence_proxy_async_smem();
    __syncthreads();  // (C)
    tick(4);
    {
      const uint32_t head = min(n, (4 - oo) & 3);
      const uint32_t mid = (n - head) & ~3u;
      if (mid && tid == 0) {
        bulk_s2g(t_e + head, buf + oo + head, mid * 4);
        bulk_commit();
      }
      if (tid < head) t_e[tid] = buf[oo + tid];
      const uint32_t tl = head + mid + tid;
      if (tl < n && tid < 4) t_e[tl] = buf[oo + tl];
    }
    if constexpr (kFast) zero_s<TT>(f_sb + (uint32_t)(2 * CAP3P_ * 4), (uint32_t)round4((int)nloc * WH3_), tid);
    else zero_u32(s_cnt, round4((int)nloc * WH3_));  // rows >= nloc were never touched
    __syncthreads();  // (D)
    tick(5);
  }
  if (tid == 0) bulk_wait_read<0>();
  if constexpr (kProf) {
    if (threadIdx.x == 0 && a.prof)
      for (int q = 0; q < 6; ++q) atomicAdd(&a.prof[q], pacc[q]);
  }
}

// ---------------------------------------------------------------- planning
// A coarse bucket's level-1 records arrive as R runs (R = 1 on one GPU: the
// bucket's range of R1; R = P on a multi-GPU receiver: one run per sender, in
// sender order = ascending source).  runs[c * R + s] = (start in the R1 buffer,
// records).
struct Run {
  uint64_t start;
  uint64_t n;
};

// One GPU / sender: bucket c of R1 = [tbase[c * ntiles1], next bucket's start).
__global__ void k_runs_from_tbase(const uint64_t* __restrict__ tbase, uint64_t ntiles1, int D1, uint64_t E,
                                  Run* __restrict__ runs) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < D1; c += gridDim.x * blockDim.x) {
    const uint64_t s = tbase[(uint64_t)c * ntiles1];
    const uint64_t e = (c + 1 < D1) ? tbase[(uint64_t)(c + 1) * ntiles1] : E;
    runs[c] = Run{s, e - s};
  }
}

// Level-2 tiling of the runs (one CTA): rfirst[r] = first tile of run r
// (ceil(n / CT2) tiles per run), rfirst[nruns] = tile count; bstart[c] =
// output (R2 / CSC) start of bucket c = records of the runs before run c * R,
// bstart[nb] = all records.
__global__ void __launch_bounds__(1024) k_runs_plan(const Run* __restrict__ runs, uint32_t nruns, uint32_t R,
                                                     uint32_t* __restrict__ rfirst, uint64_t* __restrict__ bstart) {
  __shared__ uint32_t s_t[1024];
  __shared__ uint64_t s_n[1024];
  __shared__ uint32_t s_tmp[40];
  __shared__ uint64_t s_tmp64[40];
  uint32_t tcarry = 0;
  uint64_t ncarry = 0;
  for (uint32_t r0 = 0; r0 < nruns; r0 += blockDim.x) {
    const uint32_t r = r0 + threadIdx.x;
    const Run x = (r < nruns) ? runs[r] : Run{0, 0};
    s_t[threadIdx.x] = (uint32_t)((x.n + CT2 - 1) / CT2);
    s_n[threadIdx.x] = x.n;
    __syncthreads();
    const uint32_t tt = block_excl_scan_u32(s_t, blockDim.x, s_tmp);
    const uint64_t tn = block_excl_scan_u64(s_n, blockDim.x, s_tmp64);
    if (r < nruns) {
      rfirst[r] = tcarry + s_t[threadIdx.x];
      if (r % R == 0) bstart[r / R] = ncarry + s_n[threadIdx.x];
    }
    tcarry += tt;
    ncarry += tn;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    rfirst[nruns] = tcarry;
    bstart[nruns / R] = ncarry;
  }
}

// One CTA per bucket: its tiles (with the R1 source-high decode state of the
// run's seg_hi row, row index s * row_stride + c) and its segment descriptor.
__global__ void k_l2_tiles(const Run* __restrict__ runs, uint32_t R, uint32_t row_stride,
                           const uint32_t* __restrict__ rfirst, const uint64_t* __restrict__ bstart, int Db,
                           const uint64_t* __restrict__ seg_hi, uint32_t nh, RTile* __restrict__ tiles,
                           SegDesc* __restrict__ segs) {
  const uint32_t c = blockIdx.x;
  const uint32_t g0 = rfirst[c * R], nt = rfirst[(c + 1) * R] - g0;
  if (threadIdx.x == 0) {
    SegDesc S;
    S.base = bstart[c];
    S.out_off = (uint64_t)c * Db;
    S.g0 = g0;
    S.nt = nt;
    S.end = bstart[c + 1];
    segs[c] = S;
  }
  for (uint32_t s = 0; s < R; ++s) {
    const Run run = runs[c * R + s];
    const uint32_t rt0 = rfirst[c * R + s], ntr = rfirst[c * R + s + 1] - rt0;
    const uint32_t rowi = s * row_stride + c;
    const uint64_t* row = seg_hi + (uint64_t)rowi * (nh + 1);
    for (uint32_t jj = threadIdx.x; jj < ntr; jj += blockDim.x) {
      const uint64_t st = run.start + (uint64_t)jj * CT2;
      const uint32_t n = (uint32_t)umin64(CT2, run.start + run.n - st);
      // h0 = #{h in [1, nh] : row[h] <= st}; hi = #{h : row[h] <= st + n - 1}
      auto cnt_le = [&](uint64_t x) -> uint32_t {
        uint32_t lo = 0, hi = nh;  // answer in [0, nh]
        while (lo < hi) {
          const uint32_t mid = lo + (hi - lo + 1) / 2;
          if (row[mid] <= x) lo = mid; else hi = mid - 1;
        }
        return lo;
      };
      RTile t;
      t.start = st;
      t.n = n;
      t.seg = rowi;
      t.j = rt0 - g0 + jj;
      t.nt = nt;
      t.h0 = cnt_le(st);
      t.nbnd = cnt_le(st + n - 1) - t.h0;
      tiles[rt0 + jj] = t;
    }
  }
}

// Multi-GPU receiver: runs of its buckets [lo, lo + nloc) from the P senders'
// per-bucket counts (counts[s * D1 + c]; the receive buffer holds sender s's
// buckets lo..lo+nloc-1 back to back after senders 0..s-1), and the received
// seg_hi rows (row s * nloc + (c - lo), sender coordinates; entry 0 = the
// sender's first source-high value) rebased to receive-buffer positions.
// One thread per (c, s) run.
__global__ void k_recv_runs(const uint64_t* __restrict__ counts, uint32_t P, uint32_t D1, uint32_t lo, uint32_t nloc,
                            Run* __restrict__ runs, uint64_t* __restrict__ seg_hi, uint32_t nh) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * nloc) return;
  const uint32_t c = i / P, s = i - c * P;  // run index i = c * P + s (bucket-major)
  uint64_t before = 0;                      // records of earlier senders' blocks
  for (uint32_t q = 0; q < s; ++q)
    for (uint32_t k = 0; k < nloc; ++k) before += counts[(uint64_t)q * D1 + lo + k];
  uint64_t in_blk = 0;
  for (uint32_t k = 0; k < c; ++k) in_blk += counts[(uint64_t)s * D1 + lo + k];
  uint64_t sstart = 0;  // the bucket's start in the sender's R1
  for (uint32_t k = 0; k < lo + c; ++k) sstart += counts[(uint64_t)s * D1 + k];
  const uint64_t start = before + in_blk;
  runs[i] = Run{start, counts[(uint64_t)s * D1 + lo + c]};
  uint64_t* row = seg_hi + ((uint64_t)s * nloc + c) * (nh + 1);
  const uint64_t hb = row[0];
  for (uint32_t h = 1; h <= nh; ++h) {
    const uint64_t v = row[h];
    if (h <= hb) row[h] = start;
    else if (v != ~0ull) row[h] = v - sstart + start;
  }
}

// Pipelined host entry point (gt_transpose_host): P source chunks of one
// graph ran level 1 as senders, sender s writing its R1 at its edge offset
// e_s of one buffer and its seg_hi rows at rows s * D1 + c.  Runs of the
// buckets [lo, lo + nloc) and their rows rebased to buffer positions
// (sender-local position v -> v + e_s; boundaries at or below the sender's
// first source-high value -> the run start).  One thread per (c, s) run;
// each row belongs to exactly one bucket range, so it is rebased once.
__global__ void k_runs_senders(const uint64_t* __restrict__ counts, uint32_t P, uint32_t D1, uint32_t lo, uint32_t nloc,
                               Run* __restrict__ runs, uint64_t* __restrict__ seg_all, uint32_t nh) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * nloc) return;
  const uint32_t c = i / P, s = i - c * P;
  uint64_t es = 0;  // sender s's edge offset = records of the senders before it
  for (uint32_t q = 0; q < s; ++q)
    for (uint32_t k = 0; k < D1; ++k) es += counts[(uint64_t)q * D1 + k];
  uint64_t sstart = 0;  // the bucket's start in sender s's R1
  for (uint32_t k = 0; k < lo + c; ++k) sstart += counts[(uint64_t)s * D1 + k];
  const uint64_t start = es + sstart;
  runs[i] = Run{start, counts[(uint64_t)s * D1 + lo + c]};
  uint64_t* row = seg_all + ((uint64_t)s * D1 + lo + c) * (nh + 1);
  const uint64_t hb = row[0];
  for (uint32_t h = 1; h <= nh; ++h) {
    const uint64_t v = row[h];
    if (h <= hb) row[h] = start;
    else if (v != ~0ull) row[h] = v + es;
  }
}

// L3 plan: one thread per aligned group of G = ML3 >> c fine buckets.  Small
// fine buckets are packed into units (<= CAP3 records, one group); fine buckets
// above CAP3 become big buckets.  fbase[f] = CSC start of fine bucket f,
// fbase[nfine] = E.
struct Big3 {
  uint64_t start;
  uint64_t n;
  uint32_t f;
  uint32_t pad;
};
__global__ void k_plan3(const uint64_t* __restrict__ fbase, uint32_t nfine, int sbits, Unit3* __restrict__ units,
                        uint32_t* __restrict__ n_units, Big3* __restrict__ bigs, uint32_t* __restrict__ n_big,
                        uint32_t cap = CAP3) {
  const uint32_t G = 1u << sbits;
  const uint32_t grp = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t f_begin = grp * G;
  if (f_begin >= nfine) return;
  const uint32_t f_end = min(nfine, f_begin + G);
  uint32_t f = f_begin;
  while (f < f_end) {
    const uint64_t s = fbase[f], sz = fbase[f + 1] - s;
    if (sz > (uint64_t)cap) {
      const uint32_t q = atomicAdd(n_big, 1u);
      Big3 bg;
      bg.start = s;
      bg.n = sz;
      bg.f = f;
      bg.pad = 0;
      bigs[q] = bg;
      ++f;
      continue;
    }
    uint64_t tot = sz;
    uint32_t e = f + 1;
    while (e < f_end) {
      const uint64_t z = fbase[e + 1] - fbase[e];
      if (z > (uint64_t)cap || tot + z > (uint64_t)cap) break;
      tot += z;
      ++e;
    }
    Unit3 u;
    u.start = s;
    u.n = (uint32_t)tot;
    u.f0 = f;
    u.nf = e - f;
    u.pad = 0;
    units[atomicAdd(n_units, 1u)] = u;
    f = e;
  }
}

// Big fine buckets -> L3 tiles, in parallel: k_big_nt writes each bucket's
// tile count, a scan gives the first tile of each, k_big_write writes the
// tiles, the segments and the tile total.
__global__ void k_big_nt(const Big3* __restrict__ bigs, const uint32_t* __restrict__ n_big, uint32_t* __restrict__ bnt) {
  const uint32_t nb = *n_big;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nb; q += gridDim.x * blockDim.x)
    bnt[q] = (uint32_t)((bigs[q].n + CT2 - 1) / CT2);
}
__global__ void k_big_write(const Big3* __restrict__ bigs, const uint32_t* __restrict__ n_big,
                            const uint64_t* __restrict__ tfirst, int c, RTile* __restrict__ tiles,
                            uint32_t* __restrict__ n_tiles, SegDesc* __restrict__ segs) {
  const uint32_t nb = *n_big;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_tiles = (uint32_t)tfirst[nb];
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nb; q += gridDim.x * blockDim.x) {
    const Big3 bg = bigs[q];
    const uint32_t g0 = (uint32_t)tfirst[q], nt = (uint32_t)(tfirst[q + 1] - tfirst[q]);
    SegDesc S;
    S.base = bg.start;
    S.out_off = (uint64_t)bg.f << c;
    S.g0 = g0;
    S.nt = nt;
    S.end = bg.start + bg.n;
    segs[q] = S;
    for (uint32_t j = 0; j < nt; ++j) {
      RTile t;
      t.start = bg.start + (uint64_t)j * CT2;
      t.n = (uint32_t)umin64(CT2, bg.n - (uint64_t)j * CT2);
      t.seg = q;
      t.j = j;
      t.nt = nt;
      t.h0 = 0;
      t.nbnd = 0;
      tiles[g0 + j] = t;
    }
  }
}

}  // namespace v3
}  // namespace gt

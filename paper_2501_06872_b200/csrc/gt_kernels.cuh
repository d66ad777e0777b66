// gt_kernels.cuh — the transposition kernels (sm_100a).
//
// Pipeline for CSR -> CSC with every CSC list ascending by source (the order of
// transpose_oracle, graph.py:136-148 == a stable counting sort of the CSR edge
// stream by destination).  The destination ID is split into three digits
// (a | b | c bits, most significant first); each level is a stable partition.
//
//   L1  count  : per count tile (CT edges), histogram of digit a      (reads dst)
//   L1  scan   : bases[d][tile] (decoupled look-back scan)
//   L1  place  : per count tile, place tiles of 4096 edges in order; owners
//                (sources) from offsets; stable rank by digit a; records
//                (src,dst) written in coarse-bucket order            [step1]
//   B1         : per 8192-record chunk of a coarse bucket, in place stable
//                sort by digit b; chunk digit offsets + fine histogram [step2]
//   F  small   : per fine bucket (<= kFCap records): gather its segments
//                from every chunk, stable rank by digit c, write the CSC
//                slice (contiguous) and its offsets              [step3]
//   F  big     : fine buckets above kFCap, split into jobs of chunk ranges:
//                count -> per-vertex job bases -> place in batches
//
// Stability argument: every level is stable (per-warp ranks in program order,
// warps ordered by the block scan, tiles/chunks ordered by their global
// bases), so the final order inside each destination equals CSR order, i.e.
// ascending source (sources are visited in ascending order in CSR).
#pragma once
#include "gt_common.cuh"
#include "gt_scan.cuh"

namespace gt {

// ---------------------------------------------------------------- constants
constexpr int kL1Warps = 8;
constexpr int kL1Slots = 16;
constexpr int kPlaceTile = kL1Warps * kL1Slots * 32;  // 4096 edges
constexpr int kB1Warps = 8;
constexpr int kB1Slots = 32;
constexpr int kChunk = kB1Warps * kB1Slots * 32;  // 8192 records
constexpr int kFWarps = 8;
constexpr int kFCap = 8192;
constexpr int kSegCap = 1024;
constexpr int kJobChunks = 64;  // chunks per big-bucket job

// ------------------------------------------------------------ small kernels
__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }

// ------------------------------------------------------------ input views
// CSR edge stream (the transpose input).  `edges` points at global edge
// e_begin; stream index i is global edge e_begin + i.  Sources are recovered
// from `offsets` (global, V+1 entries).
struct InCsr {
  const uint64_t* offsets;
  const uint32_t* edges;
  uint64_t e_begin;
  uint64_t V;
  static constexpr bool kRecords = false;
  __device__ __forceinline__ uint32_t dst(uint64_t i) const { return ldg_stream(edges + i); }
};
// (src, dst) record stream in source order (multi-GPU receiver side); dst is
// rebased to the local destination range.
struct InRec {
  const uint2* rec;
  uint32_t dst_base;
  static constexpr bool kRecords = true;
  __device__ __forceinline__ uint32_t dst(uint64_t i) const { return ldg_stream(rec + i).y - dst_base; }
};
// Level-1 digit: dst >> shift, or the owner index among destination ranges.
struct DigShift {
  int shift;
  __device__ __forceinline__ uint32_t operator()(uint32_t d) const { return d >> shift; }
};
constexpr int kMaxParts = 64;
struct DigBounds {
  uint32_t lo[kMaxParts + 1];  // lo[p] = first vertex of owner p; lo[parts] = end
  int parts;
  __device__ __forceinline__ uint32_t operator()(uint32_t d) const {
    uint32_t p = 0;
    for (int i = 1; i < parts; ++i) p += (d >= lo[i]) ? 1u : 0u;
    return p;
  }
};

// Owner (source) of the first edge of each count tile: largest v with
// offsets[v] <= e_begin + k*CT, by binary search.
__global__ void k_tile_src(InCsr in, uint64_t CT, uint64_t ntiles, uint32_t* __restrict__ tile_src) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= ntiles) return;
  const uint64_t pos = in.e_begin + k * CT;
  uint64_t lo = 0, hi = in.V;  // answer in [0, V-1]; offsets[0] = 0 <= pos
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (in.offsets[mid] <= pos) lo = mid; else hi = mid;
  }
  tile_src[k] = (uint32_t)lo;
}

// L1 count: histogram of the level-1 digit over each count tile.  tcnt is
// digit-major: tcnt[d * ntiles + k].
template <class In, class Dig>
__global__ void __launch_bounds__(512) k_l1_count(In in, Dig dig, uint64_t E, uint64_t CT, uint64_t ntiles, int D,
                                                  uint32_t* __restrict__ tcnt) {
  extern __shared__ uint32_t s_hist[];
  for (int d = threadIdx.x; d < D; d += blockDim.x) s_hist[d] = 0;
  __syncthreads();
  const uint64_t k = blockIdx.x;
  const uint64_t b = k * CT, n = umin64(E, b + CT) - b;
  if constexpr (!In::kRecords) {
    // vectorised body when 16B aligned
    const uint32_t* p = in.edges + b;
    uint64_t head = 0;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
    if (addr & 15) head = umin64(n, (16 - (addr & 15)) / 4);
    for (uint64_t i = threadIdx.x; i < head; i += blockDim.x) smem_inc(&s_hist[dig(p[i])]);
    const uint4* p4 = reinterpret_cast<const uint4*>(p + head);
    const uint64_t n4 = (n - head) / 4;
    for (uint64_t i = threadIdx.x; i < n4; i += blockDim.x) {
      uint4 q;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(p4 + i));
      smem_inc(&s_hist[dig(q.x)]);
      smem_inc(&s_hist[dig(q.y)]);
      smem_inc(&s_hist[dig(q.z)]);
      smem_inc(&s_hist[dig(q.w)]);
    }
    for (uint64_t i = head + n4 * 4 + threadIdx.x; i < n; i += blockDim.x) smem_inc(&s_hist[dig(p[i])]);
  } else {
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) smem_inc(&s_hist[dig(in.dst(b + i))]);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) tcnt[(uint64_t)d * ntiles + k] = s_hist[d];
}

// L1 place.  One CTA per count tile; its place tiles (4096 edges) are processed
// in order with running global cursors per digit.  Writes records (src, dst)
// grouped by digit, each group in stream order.
template <int kMode, class In, class Dig>
__global__ void __launch_bounds__(kL1Warps * 32) k_l1_place(In in, Dig dig, uint64_t E, uint64_t CT, uint64_t ntiles,
                                                           int D, const uint64_t* __restrict__ tbase,
                                                           const uint32_t* __restrict__ tile_src,
                                                           uint2* __restrict__ rec_out) {
  constexpr int W = kL1Warps, K = kL1Slots, T = W * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint2* s_stage = reinterpret_cast<uint2*>(smem_raw);                  // kPlaceTile
  uint64_t* s_gcur = reinterpret_cast<uint64_t*>(s_stage + kPlaceTile);  // D
  uint32_t* s_mark = reinterpret_cast<uint32_t*>(s_gcur + D);            // kPlaceTile
  uint32_t* s_cnt = s_mark + kPlaceTile;                                 // W * D
  uint32_t* s_scr = s_cnt + W * D;                                       // W * D (safe mode)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * D : 0);         // D
  uint32_t* s_dtot = s_dstart + D;                                       // D
  uint32_t* s_tmp = s_dtot + D;                                          // 40
  __shared__ uint32_t s_wmax[W];
  __shared__ uint32_t s_next_src;

  const uint64_t k = blockIdx.x;
  const uint64_t tb = k * CT, te = umin64(E, tb + CT);
  for (int d = threadIdx.x; d < D; d += T) s_gcur[d] = tbase[(uint64_t)d * ntiles + k];
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * D; i += T) s_scr[i] = 0;
  uint32_t s_cur = 0;
  if constexpr (!In::kRecords) s_cur = tile_src[k];
  const uint32_t lane = lane_id(), w = warp_id();
  uint32_t* cnt_w = s_cnt + w * D;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * D : 0);
  const uint32_t seg0 = w * (K * 32);

  for (uint64_t pt = tb; pt < te; pt += kPlaceTile) {
    const uint64_t pe = umin64(te, pt + (uint64_t)kPlaceTile);
    const uint32_t n = (uint32_t)(pe - pt);
    for (int i = threadIdx.x; i < W * D; i += T) s_cnt[i] = 0;
    uint32_t r_src[K], r_dst[K];
    if constexpr (!In::kRecords) {
      for (int i = threadIdx.x; i < kPlaceTile; i += T) s_mark[i] = 0;
      if (threadIdx.x == 0) s_next_src = s_cur;
      __syncthreads();
      // owners: mark every source boundary inside the place tile
      const uint64_t gpt = in.e_begin + pt, gpe = in.e_begin + pe;
      uint64_t vb = (uint64_t)s_cur + 1;
      while (true) {
        const uint64_t v = vb + threadIdx.x;
        bool inside = false;
        if (v < in.V) {
          const uint64_t o = in.offsets[v];
          if (o < gpe) {
            atomicMax(&s_mark[o - gpt], (uint32_t)v);
            inside = true;
          }
          if (o <= gpe) atomicMax(&s_next_src, (uint32_t)v);
        }
        if (!__syncthreads_and(inside)) break;
        vb += T;
      }
      // per-warp max of marks -> starting owner of each warp segment
      uint32_t wm = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) wm = max(wm, s_mark[seg0 + s * 32 + lane]);
      wm = __reduce_max_sync(kFull, wm);
      if (lane == 0) s_wmax[w] = wm;
      __syncthreads();
      uint32_t carry = s_cur;
      for (int ww = 0; ww < (int)w; ++ww) carry = max(carry, s_wmax[ww]);
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        r_dst[s] = valid ? in.dst(pt + i) : 0u;
        uint32_t m = s_mark[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, m, o);
          if (lane >= (uint32_t)o) m = max(m, y);
        }
        m = max(m, carry);
        r_src[s] = m;
        carry = __shfl_sync(kFull, m, 31);
        if (valid) smem_inc(&cnt_w[dig(r_dst[s])]);
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        uint2 r = make_uint2(0, 0);
        if (valid) {
          r = ldg_stream(in.rec + pt + i);
          r.y -= in.dst_base;
          smem_inc(&cnt_w[dig(r.y)]);
        }
        r_src[s] = r.x;
        r_dst[s] = r.y;
      }
    }
    __syncthreads();
    warp_counts_to_bases<W>(s_cnt, D, s_dstart, s_dtot, s_tmp);
    // round 2: final tile-local positions; stage records in digit order
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      const uint32_t pos = warp_rank<kMode>(cnt_w, scr_w, valid ? dig(r_dst[s]) : 0u, valid);
      if (valid) s_stage[pos] = make_uint2(r_src[s], r_dst[s]);
    }
    __syncthreads();
    // write out: consecutive staged records of a digit are consecutive in rec_out
    for (uint32_t i = threadIdx.x; i < n; i += T) {
      const uint2 r = s_stage[i];
      const uint32_t d = dig(r.y);
      rec_out[s_gcur[d] + (i - s_dstart[d])] = r;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += T) s_gcur[d] += s_dtot[d];
    if constexpr (!In::kRecords) s_cur = s_next_src;
    __syncthreads();
  }
}

// Coarse-bucket bookkeeping (one CTA): cstart[c] = tbase[c*ntiles] (c < D1),
// cstart[D1] = E; nchunks -> chunk_first (exclusive); chunk_first[D1] = total.
// For b == 0 also fine_hist[c] = bucket size.
__global__ void k_coarse_info(const uint64_t* __restrict__ tbase, uint64_t ntiles, int D1, uint64_t E,
                              uint64_t* __restrict__ cstart, uint32_t* __restrict__ chunk_first,
                              unsigned long long* __restrict__ fine_hist_b0) {
  extern __shared__ uint32_t s_nch[];
  __shared__ uint32_t s_tmp[40];
  for (int c = threadIdx.x; c <= D1; c += blockDim.x) {
    const uint64_t st = (c < D1) ? tbase[(uint64_t)c * ntiles] : E;
    cstart[c] = st;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D1; c += blockDim.x) {
    const uint64_t sz = cstart[c + 1] - cstart[c];
    s_nch[c] = (uint32_t)((sz + kChunk - 1) / kChunk);
    if (fine_hist_b0) fine_hist_b0[c] = sz;
  }
  __syncthreads();
  const uint32_t total = block_excl_scan_u32(s_nch, D1, s_tmp);
  for (int c = threadIdx.x; c < D1; c += blockDim.x) chunk_first[c] = s_nch[c];
  if (threadIdx.x == 0) chunk_first[D1] = total;
}

// chunk -> coarse bucket map.
__global__ void k_chunk_map(const uint32_t* __restrict__ chunk_first, int D1, uint32_t* __restrict__ chunk_bucket) {
  const int c = blockIdx.x;
  if (c >= D1) return;
  for (uint32_t g = chunk_first[c] + threadIdx.x; g < chunk_first[c + 1]; g += blockDim.x) chunk_bucket[g] = c;
}

// B1: in-place stable sort of each chunk by the middle digit.
template <int kMode>
__global__ void __launch_bounds__(kB1Warps * 32) k_b1(
    uint2* __restrict__ rec, const uint64_t* __restrict__ cstart, const uint32_t* __restrict__ chunk_first,
    const uint32_t* __restrict__ chunk_bucket, int D1, int shift_b, uint32_t mask_b, int Db,
    uint32_t* __restrict__ segoff, unsigned long long* __restrict__ fine_hist) {
  constexpr int W = kB1Warps, K = kB1Slots, T = W * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint2* s_stage = reinterpret_cast<uint2*>(smem_raw);  // kChunk
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_stage + kChunk);
  uint32_t* s_scr = s_cnt + W * Db;
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * Db : 0);
  uint32_t* s_dtot = s_dstart + Db;
  uint32_t* s_tmp = s_dtot + Db;
  const uint32_t g = blockIdx.x;
  if (g >= chunk_first[D1]) return;  // grid is an upper bound on the chunk count
  const uint32_t c = chunk_bucket[g];
  const uint64_t start = cstart[c] + (uint64_t)(g - chunk_first[c]) * kChunk;
  const uint32_t n = (uint32_t)umin64(kChunk, cstart[c + 1] - start);
  for (int i = threadIdx.x; i < W * Db; i += T) {
    s_cnt[i] = 0;
    if (kMode == kRankSafe) s_scr[i] = 0;
  }
  __syncthreads();
  const uint32_t lane = lane_id(), w = warp_id();
  uint32_t* cnt_w = s_cnt + w * Db;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * Db : 0);
  const uint32_t seg0 = w * (K * 32);
  uint2 r[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const uint32_t i = seg0 + s * 32 + lane;
    if (i < n) {
      r[s] = rec[start + i];  // plain load: this chunk is rewritten in place below
      smem_inc(&cnt_w[(r[s].y >> shift_b) & mask_b]);
    } else {
      r[s] = make_uint2(0, 0);
    }
  }
  __syncthreads();
  warp_counts_to_bases<W>(s_cnt, Db, s_dstart, s_dtot, s_tmp);
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const uint32_t i = seg0 + s * 32 + lane;
    const bool valid = i < n;
    const uint32_t pos = warp_rank<kMode>(cnt_w, scr_w, (r[s].y >> shift_b) & mask_b, valid);
    if (valid) s_stage[pos] = r[s];
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += T) rec[start + i] = s_stage[i];
  uint32_t* so = segoff + (uint64_t)g * (Db + 1);
  for (int f = threadIdx.x; f < Db; f += T) {
    so[f] = s_dstart[f];
    if (s_dtot[f]) atomicAdd(&fine_hist[(uint64_t)c * Db + f], (unsigned long long)s_dtot[f]);
  }
  if (threadIdx.x == 0) so[Db] = n;
}

// ------------------------------------------------------------------ final
struct FineCtx {
  const uint2* rec;
  const uint64_t* cstart;
  const uint32_t* chunk_first;
  const uint32_t* segoff;  // nullptr when b == 0
  int Db;
  int bits_c;
  uint32_t mask_c;
  uint64_t V;
};

// Segment of fine bucket f inside chunk g (of coarse bucket c).
__device__ __forceinline__ void fine_segment(const FineCtx& x, uint32_t c, uint32_t f, uint32_t g,
                                             uint64_t& start, uint32_t& len) {
  const uint64_t cpos = x.cstart[c] + (uint64_t)(g - x.chunk_first[c]) * kChunk;
  if (x.segoff) {
    const uint32_t* so = x.segoff + (uint64_t)g * (x.Db + 1);
    const uint32_t a = so[f], b = so[f + 1];
    start = cpos + a;
    len = b - a;
  } else {
    start = cpos;
    len = (uint32_t)umin64(kChunk, x.cstart[c + 1] - cpos);
  }
}

// Shared batch engine: gather `n` records (the concatenation of nseg segments
// described in s_seg_start/s_seg_pos) into smem, stable-rank them by digit c,
// and stage their sources in (vertex, rank) order.  On return s_dstart[v] is the
// batch-local start of vertex v and s_dtot[v] its count in this batch.
template <int kMode>
__device__ __forceinline__ void fine_batch(const FineCtx& x, uint32_t n, int nseg, const uint64_t* s_seg_start,
                                           const uint32_t* s_seg_pos, uint32_t* s_src, uint8_t* s_dig,
                                           uint32_t* s_out, uint32_t* s_cnt, uint32_t* s_scr, uint32_t* s_dstart,
                                           uint32_t* s_dtot, uint32_t* s_tmp) {
  constexpr int W = kFWarps, T = W * 32;
  const int Dc = 1 << x.bits_c;
  const uint32_t lane = lane_id(), w = warp_id();
  // gather: warp w copies segments w, w+W, ...
  for (int j = w; j < nseg; j += W) {
    const uint64_t st = s_seg_start[j];
    const uint32_t p0 = s_seg_pos[j], len = s_seg_pos[j + 1] - p0;
    for (uint32_t q = lane; q < len; q += 32) {
      const uint2 r = ldg_stream(x.rec + st + q);
      s_src[p0 + q] = r.x;
      s_dig[p0 + q] = (uint8_t)(r.y & x.mask_c);
    }
  }
  for (int i = threadIdx.x; i < W * Dc; i += T) {
    s_cnt[i] = 0;
    if (kMode == kRankSafe) s_scr[i] = 0;
  }
  __syncthreads();
  uint32_t* cnt_w = s_cnt + w * Dc;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * Dc : 0);
  const uint32_t lo = (uint32_t)(((uint64_t)n * w) / W), hi = (uint32_t)(((uint64_t)n * (w + 1)) / W);
  for (uint32_t b = lo; b < hi; b += 32) {
    const uint32_t i = b + lane;
    if (i < hi) smem_inc(&cnt_w[s_dig[i]]);
  }
  __syncthreads();
  warp_counts_to_bases<W>(s_cnt, Dc, s_dstart, s_dtot, s_tmp);
  for (uint32_t b = lo; b < hi; b += 32) {
    const uint32_t i = b + lane;
    const bool valid = i < hi;
    const uint32_t d = valid ? s_dig[i] : 0u;
    const uint32_t pos = warp_rank<kMode>(cnt_w, scr_w, d, valid);
    if (valid) s_out[pos] = s_src[i];
  }
  __syncthreads();
}

template <int kMode>
__global__ void __launch_bounds__(kFWarps * 32) k_final_small(FineCtx x, const unsigned long long* __restrict__ fine_hist,
                                                             const uint64_t* __restrict__ fine_base,
                                                             uint64_t* __restrict__ t_offsets, uint32_t* __restrict__ t_edges,
                                                             uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  constexpr int W = kFWarps, T = W * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Dc = 1 << x.bits_c;
  uint64_t* s_seg_start = reinterpret_cast<uint64_t*>(smem_raw);    // kSegCap
  uint32_t* s_seg_pos = reinterpret_cast<uint32_t*>(s_seg_start + kSegCap);  // kSegCap + 1
  uint32_t* s_src = s_seg_pos + kSegCap + 4;                        // kFCap
  uint32_t* s_out = s_src + kFCap;                                  // kFCap
  uint32_t* s_cnt = s_out + kFCap;                                  // W * Dc
  uint32_t* s_scr = s_cnt + W * Dc;                                 // W * Dc (safe)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * Dc : 0);   // Dc
  uint32_t* s_dtot = s_dstart + Dc;                                 // Dc
  uint32_t* s_tmp = s_dtot + Dc;                                    // 40
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_tmp + 40);          // kFCap

  const uint32_t fid = blockIdx.x;
  const uint64_t v0 = (uint64_t)fid << x.bits_c;
  if (v0 >= x.V) return;
  const uint32_t nv = (uint32_t)umin64((uint64_t)Dc, x.V - v0);
  const uint64_t n64 = fine_hist[fid];
  const uint64_t base = fine_base[fid];
  if (n64 == 0) {
    for (uint32_t v = threadIdx.x; v < nv; v += T) t_offsets[v0 + v] = base;
    return;
  }
  const uint32_t c = fid / x.Db, f = fid % x.Db;
  const uint32_t g0 = x.chunk_first[c], g1 = x.chunk_first[c + 1];
  const int nch = (int)(g1 - g0);
  if (n64 > (uint64_t)kFCap || nch > kSegCap) {
    if (threadIdx.x == 0) big_list[atomicAdd(big_count, 1u)] = fid;
    return;
  }
  const uint32_t n = (uint32_t)n64;
  for (int j = threadIdx.x; j < nch; j += T) {
    uint64_t st;
    uint32_t len;
    fine_segment(x, c, f, g0 + j, st, len);
    s_seg_start[j] = st;
    s_seg_pos[j] = len;
  }
  __syncthreads();
  block_excl_scan_u32(s_seg_pos, nch, s_tmp);
  if (threadIdx.x == 0) s_seg_pos[nch] = n;
  __syncthreads();
  fine_batch<kMode>(x, n, nch, s_seg_start, s_seg_pos, s_src, s_dig, s_out, s_cnt, s_scr, s_dstart, s_dtot, s_tmp);
  for (uint32_t v = threadIdx.x; v < nv; v += T) t_offsets[v0 + v] = base + s_dstart[v];
  for (uint32_t i = threadIdx.x; i < n; i += T) t_edges[base + i] = s_out[i];
}

// Big fine buckets.  A job = (fid, first chunk, last chunk).
struct BigJob {
  uint32_t fid;
  uint32_t g0, g1;   // chunk range (absolute chunk ids)
  uint32_t bucket;   // index into the big-bucket list
};

// Count per vertex over the job's segments -> jobcnt[job][Dc].
__global__ void __launch_bounds__(256) k_big_count(FineCtx x, const BigJob* __restrict__ jobs,
                                                   uint32_t* __restrict__ jobcnt) {
  extern __shared__ uint32_t s_h[];
  const int Dc = 1 << x.bits_c;
  const BigJob jb = jobs[blockIdx.x];
  for (int i = threadIdx.x; i < Dc; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const uint32_t c = jb.fid / x.Db, f = jb.fid % x.Db;
  const uint32_t lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
  for (uint32_t g = jb.g0 + w; g < jb.g1; g += nw) {
    uint64_t st;
    uint32_t len;
    fine_segment(x, c, f, g, st, len);
    for (uint32_t q = lane; q < len; q += 32) smem_inc(&s_h[ldg_stream(x.rec + st + q).y & x.mask_c]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Dc; i += blockDim.x) jobcnt[(uint64_t)blockIdx.x * Dc + i] = s_h[i];
}

// Per big bucket: CSC offsets of its vertices and per-job vertex cursors.
__global__ void k_big_scan(FineCtx x, const uint32_t* __restrict__ big_list, const uint32_t* __restrict__ job_first,
                           const uint64_t* __restrict__ fine_base, const uint32_t* __restrict__ jobcnt,
                           uint64_t* __restrict__ jobbase, uint64_t* __restrict__ t_offsets,
                           unsigned int* __restrict__ err_overflow) {
  extern __shared__ uint64_t s_tot[];  // Dc
  const int Dc = 1 << x.bits_c;
  const uint32_t bk = blockIdx.x;
  const uint32_t fid = big_list[bk];
  const uint32_t j0 = job_first[bk], j1 = job_first[bk + 1];
  const uint64_t v0 = (uint64_t)fid << x.bits_c;
  for (int v = threadIdx.x; v < Dc; v += blockDim.x) {
    uint64_t run = 0;
    for (uint32_t j = j0; j < j1; ++j) run += jobcnt[(uint64_t)j * Dc + v];
    s_tot[v] = run;
    if (run >= (1ull << 32)) atomicExch(err_overflow, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // Dc <= 256: serial exclusive scan is cheap
    uint64_t run = fine_base[fid];
    for (int v = 0; v < Dc; ++v) {
      const uint64_t t = s_tot[v];
      s_tot[v] = run;
      run += t;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < Dc; v += blockDim.x) {
    uint64_t run = s_tot[v];
    if (v0 + v < x.V) t_offsets[v0 + v] = run;
    for (uint32_t j = j0; j < j1; ++j) {
      jobbase[(uint64_t)j * Dc + v] = run;
      run += jobcnt[(uint64_t)j * Dc + v];
    }
  }
}

// Place a big job: batches of whole segments (a segment longer than kFCap is
// cut into kFCap pieces), staged in (vertex, rank) order, written as runs.
template <int kMode>
__global__ void __launch_bounds__(kFWarps * 32) k_big_place(FineCtx x, const BigJob* __restrict__ jobs,
                                                           const uint64_t* __restrict__ jobbase,
                                                           uint32_t* __restrict__ t_edges) {
  constexpr int W = kFWarps, T = W * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Dc = 1 << x.bits_c;
  uint64_t* s_seg_start = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* s_seg_pos = reinterpret_cast<uint32_t*>(s_seg_start + kSegCap);
  uint32_t* s_src = s_seg_pos + kSegCap + 4;
  uint32_t* s_out = s_src + kFCap;
  uint32_t* s_cnt = s_out + kFCap;
  uint32_t* s_scr = s_cnt + W * Dc;
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * Dc : 0);
  uint32_t* s_dtot = s_dstart + Dc;
  uint32_t* s_tmp = s_dtot + Dc;
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_tmp + 40);
  uint64_t* s_cur = reinterpret_cast<uint64_t*>(s_dig + kFCap);  // Dc
  __shared__ uint32_t s_nseg, s_n;

  const BigJob jb = jobs[blockIdx.x];
  const uint32_t c = jb.fid / x.Db, f = jb.fid % x.Db;
  for (int v = threadIdx.x; v < Dc; v += T) s_cur[v] = jobbase[(uint64_t)blockIdx.x * Dc + v];
  uint32_t g = jb.g0;
  uint32_t g_off = 0;  // records of chunk g's segment already consumed
  __syncthreads();
  while (g < jb.g1) {
    // build a batch (single thread; segment lists are short)
    if (threadIdx.x == 0) {
      uint32_t n = 0;
      int ns = 0;
      while (g < jb.g1 && ns < kSegCap) {
        uint64_t st;
        uint32_t len;
        fine_segment(x, c, f, g, st, len);
        len -= g_off;
        st += g_off;
        if (len == 0) { ++g; g_off = 0; continue; }
        const uint32_t take = min(len, (uint32_t)kFCap - n);
        if (take == 0) break;
        s_seg_start[ns] = st;
        s_seg_pos[ns] = n;
        ++ns;
        n += take;
        if (take == len) { ++g; g_off = 0; } else { g_off += take; break; }
      }
      s_seg_pos[ns] = n;
      s_nseg = ns;
      s_n = n;
      // publish loop state through smem for the other threads
      s_tmp[36] = g;
      s_tmp[37] = g_off;
    }
    __syncthreads();
    const uint32_t n = s_n;
    const int ns = (int)s_nseg;
    g = s_tmp[36];
    g_off = s_tmp[37];
    __syncthreads();
    if (n == 0) break;
    fine_batch<kMode>(x, n, ns, s_seg_start, s_seg_pos, s_src, s_dig, s_out, s_cnt, s_scr, s_dstart, s_dtot, s_tmp);
    // staged run of vertex v: s_out[dstart[v] .. dstart[v]+dtot[v]) -> t_edges[cur[v] ..)
    for (uint32_t i = threadIdx.x; i < n; i += T) {
      // vertex of staged slot i: binary search in dstart (Dc <= 256)
      int lo = 0, hi = Dc - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_dstart[mid] <= i) lo = mid; else hi = mid - 1;
      }
      // skip empty vertices that share the same start: take the last v with dstart<=i and dtot>0
      t_edges[s_cur[lo] + (i - s_dstart[lo])] = s_out[i];
    }
    __syncthreads();
    for (int v = threadIdx.x; v < Dc; v += T) s_cur[v] += s_dtot[v];
    __syncthreads();
  }
}

// ----------------------------------------------------------- self test
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

}  // namespace gt

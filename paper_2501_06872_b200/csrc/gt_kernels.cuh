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
constexpr int kPlaceTile = kL1Warps * kL1Slots * 32;  // 4096 edges per place tile
constexpr int kWinCap = 1024;                         // prefetched offsets per place tile
constexpr int kB1Warps = 8;
constexpr int kB1Slots = 16;
constexpr int kChunk = kB1Warps * kB1Slots * 32;  // 4096 records per level-2 chunk
constexpr int kFWarps = 8;
constexpr int kFSlots = 16;
constexpr int kFCap = kFWarps * kFSlots * 32;  // 4096 records per final work item
constexpr int kFMaxLocal = 256;                // local vertices per final work item
constexpr int kSegCap = 1024;                  // chunks per coarse bucket held in smem

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

// Owner (source) of edge min(k*CT, E-1) of the stream (global edge
// e_begin + ...): largest v with offsets[v] <= that position, by binary search.
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
// in order with running global cursors per digit, and the next place tile's
// neighbour IDs and offsets window are prefetched with cp.async while the
// current one is ranked.  Writes records (src, dst) grouped by digit, each
// group in stream order.
// place_src[t] = owner of edge min(t*kPlaceTile, E-1) (global place index t).
template <int kMode, class In, class Dig>
__global__ void __launch_bounds__(kL1Warps * 32) k_l1_place(In in, Dig dig, uint64_t E, uint64_t CT, uint64_t ntiles,
                                                           int D, const uint64_t* __restrict__ tbase,
                                                           const uint32_t* __restrict__ place_src,
                                                           uint2* __restrict__ rec_out) {
  constexpr int W = kL1Warps, K = kL1Slots, T = W * 32, PT = kPlaceTile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // input staging: CSR -> dst u32[2][PT] + offsets window u64[2][kWinCap]; records -> uint2[2][PT]
  constexpr size_t kInBytes = In::kRecords ? 2 * PT * 8 : 2 * PT * 4 + 2 * kWinCap * 8;
  unsigned char* s_in = smem_raw;
  uint2* s_stage = reinterpret_cast<uint2*>(smem_raw + kInBytes);     // PT
  uint64_t* s_gcur = reinterpret_cast<uint64_t*>(s_stage + PT);       // D
  uint32_t* s_mark = reinterpret_cast<uint32_t*>(s_gcur + D);         // PT (CSR only)
  uint32_t* s_cnt = s_mark + (In::kRecords ? 0 : PT);                 // W * D
  uint32_t* s_scr = s_cnt + W * D;                                    // W * D (safe mode)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * D : 0);      // D
  uint32_t* s_dtot = s_dstart + D;                                    // D
  uint32_t* s_tmp = s_dtot + D;                                       // 40
  uint32_t* s_psrc = s_tmp + 40;                                      // CT/PT + 2 (CSR only)
  __shared__ uint32_t s_wmax[W];

  const uint64_t k = blockIdx.x;
  const uint64_t tb = k * CT, te = umin64(E, tb + CT);
  const int nplace = (int)((te - tb + PT - 1) / PT);
  const uint64_t gp0 = tb / PT;  // global index of the first place tile
  for (int d = threadIdx.x; d < D; d += T) s_gcur[d] = tbase[(uint64_t)d * ntiles + k];
  if constexpr (!In::kRecords) {
    for (int j = threadIdx.x; j <= nplace; j += T) s_psrc[j] = place_src[gp0 + j];
    for (int i = threadIdx.x; i < PT; i += T) s_mark[i] = 0;
  }
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * D; i += T) s_scr[i] = 0;
  __syncthreads();
  const uint32_t lane = lane_id(), w = warp_id();
  uint32_t* cnt_w = s_cnt + w * D;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * D : 0);
  const uint32_t seg0 = w * (K * 32);

  auto issue = [&](int j) {
    const int b = j & 1;
    const uint64_t pt = tb + (uint64_t)j * PT;
    const uint32_t n = (uint32_t)(umin64(te, pt + PT) - pt);
    if constexpr (In::kRecords) {
      uint2* dst = reinterpret_cast<uint2*>(s_in) + b * PT;
      for (uint32_t i = threadIdx.x; i < n; i += T) cp_async8(dst + i, in.rec + pt + i);
    } else {
      uint32_t* dst = reinterpret_cast<uint32_t*>(s_in) + b * PT;
      for (uint32_t i = threadIdx.x; i < n; i += T) cp_async4(dst + i, in.edges + pt + i);
      uint64_t* win = reinterpret_cast<uint64_t*>(s_in + 2 * PT * 4) + b * kWinCap;
      const uint32_t s0 = s_psrc[j], s1 = s_psrc[j + 1];
      const uint32_t wn = min(s1 - s0, (uint32_t)kWinCap);
      for (uint32_t i = threadIdx.x; i < wn; i += T) cp_async8(win + i, in.offsets + s0 + 1 + i);
    }
    cp_commit();
  };

  if (nplace > 0) issue(0);
  for (int j = 0; j < nplace; ++j) {
    const int b = j & 1;
    const uint64_t pt = tb + (uint64_t)j * PT;
    const uint64_t pe = umin64(te, pt + PT);
    const uint32_t n = (uint32_t)(pe - pt);
    if (j + 1 < nplace) {
      issue(j + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    for (int i = threadIdx.x; i < W * D; i += T) s_cnt[i] = 0;
    __syncthreads();
    uint32_t r_src[K], r_dst[K];
    if constexpr (!In::kRecords) {
      // owners: mark every source boundary inside the place tile (window in smem;
      // the rare overflow beyond kWinCap is read directly)
      const uint64_t gpt = in.e_begin + pt, gpe = in.e_begin + pe;
      const uint32_t s0 = s_psrc[j], s1 = s_psrc[j + 1];
      const uint64_t* win = reinterpret_cast<const uint64_t*>(s_in + 2 * PT * 4) + b * kWinCap;
      for (uint32_t i = threadIdx.x; i < s1 - s0; i += T) {
        const uint64_t o = (i < (uint32_t)kWinCap) ? win[i] : in.offsets[s0 + 1 + i];
        if (o < gpe) atomicMax(&s_mark[o - gpt], s0 + 1 + i);
      }
      __syncthreads();
      uint32_t wm = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) wm = max(wm, s_mark[seg0 + s * 32 + lane]);
      wm = __reduce_max_sync(kFull, wm);
      if (lane == 0) s_wmax[w] = wm;
      __syncthreads();
      uint32_t carry = s0;
      for (int ww = 0; ww < (int)w; ++ww) carry = max(carry, s_wmax[ww]);
      const uint32_t* dbuf = reinterpret_cast<const uint32_t*>(s_in) + b * PT;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        r_dst[s] = valid ? dbuf[i] : 0u;
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
      const uint2* rbuf = reinterpret_cast<const uint2*>(s_in) + b * PT;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        uint2 r = make_uint2(0, 0);
        if (valid) {
          r = rbuf[i];
          r.y -= in.dst_base;
          smem_inc(&cnt_w[dig(r.y)]);
        }
        r_src[s] = r.x;
        r_dst[s] = r.y;
      }
    }
    __syncthreads();
    warp_counts_to_bases<W>(s_cnt, D, s_dstart, s_dtot, s_tmp);
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      const uint32_t pos = warp_rank<kMode>(cnt_w, scr_w, valid ? dig(r_dst[s]) : 0u, valid);
      if (valid) s_stage[pos] = make_uint2(r_src[s], r_dst[s]);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += T) {
      const uint2 r = s_stage[i];
      const uint32_t d = dig(r.y);
      rec_out[s_gcur[d] + (i - s_dstart[d])] = r;
    }
    if constexpr (!In::kRecords)
      for (int i = threadIdx.x; i < PT; i += T) s_mark[i] = 0;
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += T) s_gcur[d] += s_dtot[d];
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



// B1: stable sort of each chunk by the middle digit, in place.  Persistent
// CTAs stride over the chunks; the next chunk is prefetched with cp.async
// while the current one is ranked.  segoff[g][f] (u16) = start of fine digit f
// inside chunk g.
template <int kMode>
__global__ void __launch_bounds__(kB1Warps * 32) k_b1(uint2* __restrict__ rec, const uint64_t* __restrict__ cstart,
                                                     const uint32_t* __restrict__ chunk_first,
                                                     const uint32_t* __restrict__ chunk_bucket, int D1, int shift_b,
                                                     uint32_t mask_b, int Db, uint16_t* __restrict__ segoff) {
  constexpr int W = kB1Warps, K = kB1Slots, T = W * 32, CH = kChunk;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint2* s_buf = reinterpret_cast<uint2*>(smem_raw);  // 2 * CH (the current buffer doubles as staging)
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_buf + 2 * CH);
  uint32_t* s_scr = s_cnt + W * Db;
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * Db : 0);
  uint32_t* s_dtot = s_dstart + Db;
  uint32_t* s_tmp = s_dtot + Db;
  const uint32_t nchunks = chunk_first[D1];
  const uint32_t lane = lane_id(), w = warp_id();
  uint32_t* cnt_w = s_cnt + w * Db;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * Db : 0);
  const uint32_t seg0 = w * (K * 32);
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * Db; i += T) s_scr[i] = 0;

  auto chunk_range = [&](uint32_t g, uint64_t& start, uint32_t& n) {
    const uint32_t c = chunk_bucket[g];
    start = cstart[c] + (uint64_t)(g - chunk_first[c]) * CH;
    n = (uint32_t)umin64(CH, cstart[c + 1] - start);
  };
  auto issue = [&](uint32_t g, int b) {
    uint64_t st;
    uint32_t n;
    chunk_range(g, st, n);
    uint2* dst = s_buf + b * CH;
    for (uint32_t i = threadIdx.x; i < n; i += T) cp_async8(dst + i, rec + st + i);
    cp_commit();
  };

  uint32_t g = blockIdx.x;
  if (g < nchunks) issue(g, 0);
  for (int it = 0; g < nchunks; ++it, g += gridDim.x) {
    const int b = it & 1;
    const uint32_t gn = g + gridDim.x;
    if (gn < nchunks) {
      issue(gn, b ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    uint64_t start;
    uint32_t n;
    chunk_range(g, start, n);
    for (int i = threadIdx.x; i < W * Db; i += T) s_cnt[i] = 0;
    __syncthreads();
    uint2* buf = s_buf + b * CH;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      if (i < n) smem_inc(&cnt_w[(buf[i].y >> shift_b) & mask_b]);
    }
    __syncthreads();
    warp_counts_to_bases<W>(s_cnt, Db, s_dstart, s_dtot, s_tmp);
    uint2 rr[K];
    uint32_t pp[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      rr[s] = valid ? buf[i] : make_uint2(0, 0);
      pp[s] = warp_rank<kMode>(cnt_w, scr_w, (rr[s].y >> shift_b) & mask_b, valid);
    }
    __syncthreads();  // every record of the chunk is in registers: stage in place
#pragma unroll
    for (int s = 0; s < K; ++s)
      if (seg0 + s * 32 + lane < n) buf[pp[s]] = rr[s];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += T) rec[start + i] = buf[i];
    uint16_t* so = segoff + (uint64_t)g * (Db + 1);
    for (int f = threadIdx.x; f < Db; f += T) so[f] = (uint16_t)s_dstart[f];
    if (threadIdx.x == 0) so[Db] = (uint16_t)n;
    // buf / s_dstart are reused only after the next iteration's barriers
  }
}

// ------------------------------------------------------------------ final
struct FineCtx {
  const uint2* rec;
  const uint64_t* cstart;
  const uint32_t* chunk_first;
  const uint16_t* segoff;  // nullptr when b == 0 (each chunk is one segment)
  int Db;
  int bits_c;
  uint32_t mask_c;
  uint64_t V;
};

// Final work item: a group of consecutive fine buckets [f0, f1) of coarse
// bucket c holding n <= kFCap records (kind 0), or one kFCap batch of a big
// fine bucket f0 (kind 1).  The item's records are gathered by walking chunks
// from g_start (absolute chunk id), taking the slice of fine digits [f0, f1) of
// each chunk, after skipping `skip` records, until n records are collected.
struct FItem {
  uint32_t c;
  uint32_t f0, f1;
  uint32_t kind;
  uint32_t n;
  uint32_t g_start;
  uint32_t skip;
  uint32_t pad;
  uint64_t base;  // kind 0: CSC position of the group's first record
};

// Issue cp.async copies of item `it`'s records into dst.  All threads; uses the
// segment scratch s_st / s_pos (kSegCap entries) block by block.
__device__ __forceinline__ void item_gather(const FineCtx& x, const FItem& it, uint64_t* s_st, uint32_t* s_pos,
                                            uint32_t* s_tmp, uint2* dst) {
  const uint32_t g_end = x.chunk_first[it.c + 1];
  const uint64_t cs = x.cstart[it.c], ce = x.cstart[it.c + 1];
  const uint32_t g_first = x.chunk_first[it.c];
  const uint32_t lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
  uint32_t got = 0;       // records collected (uniform)
  uint32_t skip = it.skip;
  for (uint32_t gb = it.g_start; gb < g_end && got < it.n; gb += kSegCap) {
    const int nch = (int)min((uint32_t)kSegCap, g_end - gb);
    for (int j = threadIdx.x; j < nch; j += blockDim.x) {
      const uint64_t cpos = cs + (uint64_t)(gb + j - g_first) * kChunk;
      uint32_t a, e;
      if (x.segoff) {
        const uint16_t* so = x.segoff + (uint64_t)(gb + j) * (x.Db + 1);
        a = so[it.f0];
        e = so[it.f1];
      } else {
        a = 0;
        e = (uint32_t)umin64(kChunk, ce - cpos);
      }
      s_st[j] = cpos + a;
      s_pos[j] = e - a;
    }
    __syncthreads();
    const uint32_t tot = block_excl_scan_u32(s_pos, nch, s_tmp);
    if (threadIdx.x == 0) s_pos[nch] = tot;
    __syncthreads();
    // this block's records [skip, tot) map to item positions starting at `got`
    const uint32_t lo = skip, hi = min(tot, skip + (it.n - got));
    for (int j = w; j < nch; j += nw) {
      const uint32_t a = max(s_pos[j], lo), e = min(s_pos[j + 1], hi);
      if (a >= e) continue;
      const uint64_t src = s_st[j] + (a - s_pos[j]);
      uint2* d = dst + got + (a - lo);
      for (uint32_t q = lane; q < e - a; q += 32) cp_async8(d + q, x.rec + src + q);
    }
    got += (hi > lo) ? hi - lo : 0;
    skip = (tot > skip) ? 0 : skip - tot;
    __syncthreads();
  }
}

// Persistent final stage over planned items, the next item's records gathered
// with cp.async while the current one is ranked.  kCount: count records per
// local vertex of big-batch items into cnt_tab[item][Dc] (no output).
// Big-batch item i uses cursor row i of cur_tab.
template <int kMode, bool kCount>
__global__ void __launch_bounds__(kFWarps * 32) k_final(FineCtx x, const FItem* __restrict__ items,
                                                       const uint32_t* __restrict__ n_items_ptr,
                                                       uint32_t* __restrict__ cnt_tab,
                                                       const uint64_t* __restrict__ cur_tab,
                                                       uint64_t* __restrict__ t_offsets, uint32_t* __restrict__ t_edges) {
  constexpr int W = kFWarps, K = kFSlots, T = W * 32, CAP = kFCap;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint2* s_buf = reinterpret_cast<uint2*>(smem_raw);                       // 2 * CAP (staging in place)
  uint64_t* s_st = reinterpret_cast<uint64_t*>(s_buf + 2 * CAP);           // kSegCap
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_st + kSegCap);           // kSegCap + 4
  uint32_t* s_cnt = s_pos + kSegCap + 4;                                   // W * kFMaxLocal
  uint32_t* s_scr = s_cnt + W * kFMaxLocal;                                // (safe)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * kFMaxLocal : 0);  // kFMaxLocal
  uint32_t* s_dtot = s_dstart + kFMaxLocal;                                // kFMaxLocal
  uint32_t* s_tmp = s_dtot + kFMaxLocal;                                   // 40
  uint64_t* s_cur = reinterpret_cast<uint64_t*>(s_tmp + 40);               // kFMaxLocal
  __shared__ FItem s_item[2];

  const uint32_t n_items = *n_items_ptr;
  const uint32_t lane = lane_id(), w = warp_id();
  const int Dc = 1 << x.bits_c;
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * kFMaxLocal; i += T) s_scr[i] = 0;

  auto prepare = [&](uint32_t idx, int b) {
    if (threadIdx.x == 0) s_item[b] = items[idx];
    __syncthreads();
    const FItem it = s_item[b];
    item_gather(x, it, s_st, s_pos, s_tmp, s_buf + b * CAP);
    cp_commit();
  };

  uint32_t idx = blockIdx.x;
  if (idx < n_items) prepare(idx, 0);
  for (int itn = 0; idx < n_items; ++itn, idx += gridDim.x) {
    const int b = itn & 1;
    const uint32_t nidx = idx + gridDim.x;
    if (nidx < n_items) {
      prepare(nidx, b ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    const FItem it = s_item[b];
    const uint32_t n = it.n;
    const uint32_t f0 = it.f0;
    const uint32_t nloc = (it.f1 - it.f0) << x.bits_c;
    for (int i = threadIdx.x; i < W * kFMaxLocal; i += T) s_cnt[i] = 0;
    __syncthreads();
    uint2* buf = s_buf + b * CAP;
    const uint32_t shift_f = x.bits_c;
    const uint32_t mask_f = (uint32_t)x.Db - 1;
    auto local_of = [&](uint32_t dst) -> uint32_t {
      return ((((dst >> shift_f) & mask_f) - f0) << shift_f) | (dst & x.mask_c);
    };
    // per-warp counter rows use stride nloc (the layout warp_counts_to_bases expects)
    uint32_t* cnt_w = s_cnt + w * nloc;
    uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * nloc : 0);
    const uint32_t seg0 = w * (K * 32);
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      if (i < n) smem_inc(&cnt_w[local_of(buf[i].y)]);
    }
    __syncthreads();
    if constexpr (kCount) {
      for (int v = threadIdx.x; v < Dc; v += T) {
        uint32_t sum = 0;
        for (int ww = 0; ww < W; ++ww) sum += s_cnt[ww * nloc + v];
        cnt_tab[(uint64_t)idx * Dc + v] = sum;
      }
      __syncthreads();
      continue;
    }
    warp_counts_to_bases<W>(s_cnt, (int)nloc, s_dstart, s_dtot, s_tmp);
    if (it.kind == 0) {
      const uint64_t v0 = ((uint64_t)it.c * x.Db + it.f0) << x.bits_c;
      for (uint32_t v = threadIdx.x; v < nloc; v += T)
        if (v0 + v < x.V) t_offsets[v0 + v] = it.base + s_dstart[v];
    } else {
      for (int v = threadIdx.x; v < Dc; v += T) s_cur[v] = cur_tab[(uint64_t)idx * Dc + v];
    }
    uint2 rr[K];
    uint32_t pp[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      const uint2 r = valid ? buf[i] : make_uint2(0, 0);
      const uint32_t lv = valid ? local_of(r.y) : 0u;
      pp[s] = warp_rank<kMode>(cnt_w, scr_w, lv, valid);
      rr[s] = make_uint2(r.x, lv);
    }
    __syncthreads();  // all records are in registers: stage (src, local vertex) in place
#pragma unroll
    for (int s = 0; s < K; ++s)
      if (seg0 + s * 32 + lane < n) buf[pp[s]] = rr[s];
    __syncthreads();
    if (it.kind == 0) {
      for (uint32_t i = threadIdx.x; i < n; i += T) t_edges[it.base + i] = buf[i].x;
    } else {
      for (uint32_t i = threadIdx.x; i < n; i += T) {
        const uint2 r = buf[i];
        t_edges[s_cur[r.y] + (i - s_dstart[r.y])] = r.x;
      }
    }
    __syncthreads();
  }
}

// Plan the final stage: one CTA per coarse bucket.  Fine-bucket sizes from the
// chunk segment tables, CSC bases, greedy groups of consecutive fine buckets
// (<= kFCap records, <= kFMaxLocal local vertices) and big fine buckets split
// into kFCap batches (with their starting chunk / skip); t_offsets of empty
// fine buckets.  big_buckets[bi] = {fid, first big item, batches}.
__global__ void k_f_plan(FineCtx x, FItem* __restrict__ items_s, uint32_t* __restrict__ n_s,
                         FItem* __restrict__ items_b, uint32_t* __restrict__ n_b,
                         uint32_t* __restrict__ big_buckets, uint32_t* __restrict__ n_big,
                         uint64_t* __restrict__ big_base, uint64_t* __restrict__ t_offsets) {
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_sz = s_dyn;              // Db
  uint32_t* s_base = s_sz + x.Db;      // Db
  uint32_t* s_bigf = s_base + x.Db;    // Db
  uint32_t* s_len = s_bigf + x.Db;     // blockDim
  __shared__ uint32_t s_tmp[40];
  __shared__ uint32_t s_nbig;
  const uint32_t c = blockIdx.x;
  const int Db = x.Db, Dc = 1 << x.bits_c;
  const uint32_t g0 = x.chunk_first[c], g1 = x.chunk_first[c + 1];
  const uint64_t cs = x.cstart[c];
  for (int f = threadIdx.x; f < Db; f += blockDim.x) {
    uint32_t sum = 0;
    if (x.segoff) {
      for (uint32_t g = g0; g < g1; ++g) {
        const uint16_t* so = x.segoff + (uint64_t)g * (Db + 1);
        sum += (uint32_t)so[f + 1] - so[f];
      }
    } else {
      sum = (uint32_t)(x.cstart[c + 1] - cs);
    }
    s_sz[f] = sum;
    s_base[f] = sum;
  }
  __syncthreads();
  block_excl_scan_u32(s_base, Db, s_tmp);
  for (int f = 0; f < Db; ++f) {  // t_offsets of empty fine buckets
    if (s_sz[f]) continue;
    const uint64_t v0 = ((uint64_t)c * Db + f) << x.bits_c;
    for (int v = threadIdx.x; v < Dc; v += blockDim.x)
      if (v0 + v < x.V) t_offsets[v0 + v] = cs + s_base[f];
  }
  if (threadIdx.x == 0) {
    const uint32_t maxf = (uint32_t)max(1, kFMaxLocal >> x.bits_c);
    uint32_t nbig = 0;
    int f = 0;
    while (f < Db) {
      if (s_sz[f] == 0) { ++f; continue; }
      if (s_sz[f] > (uint32_t)kFCap) { s_bigf[nbig++] = f; ++f; continue; }
      uint32_t total = 0;
      int e = f;
      while (e < Db && (uint32_t)(e - f) < maxf && s_sz[e] <= (uint32_t)kFCap && total + s_sz[e] <= (uint32_t)kFCap) {
        total += s_sz[e];
        ++e;
      }
      FItem it{};
      it.c = c; it.f0 = f; it.f1 = e; it.kind = 0; it.n = total;
      it.g_start = g0; it.skip = 0; it.base = cs + s_base[f];
      items_s[atomicAdd(n_s, 1u)] = it;
      f = e;
    }
    s_nbig = nbig;
  }
  __syncthreads();
  const uint32_t nbig = s_nbig;
  for (uint32_t q = 0; q < nbig; ++q) {
    const uint32_t f = s_bigf[q];
    const uint32_t nb = (s_sz[f] + kFCap - 1) / kFCap;
    __shared__ uint32_t s_i0;
    if (threadIdx.x == 0) {
      const uint32_t bi = atomicAdd(n_big, 1u);
      const uint32_t i0 = atomicAdd(n_b, nb);
      big_buckets[3 * bi + 0] = c * Db + f;
      big_buckets[3 * bi + 1] = i0;
      big_buckets[3 * bi + 2] = nb;
      big_base[bi] = cs + s_base[f];
      s_i0 = i0;
    }
    __syncthreads();
    const uint32_t i0 = s_i0;
    // batch k starts at record k*kFCap of the bucket's stream: locate its chunk
    uint32_t run = 0;
    for (uint32_t gb = g0; gb < g1; gb += blockDim.x) {
      const uint32_t g = gb + threadIdx.x;
      uint32_t len = 0;
      if (g < g1) {
        if (x.segoff) {
          const uint16_t* so = x.segoff + (uint64_t)g * (Db + 1);
          len = (uint32_t)so[f + 1] - so[f];
        } else {
          len = (uint32_t)umin64(kChunk, x.cstart[c + 1] - (cs + (uint64_t)(g - g0) * kChunk));
        }
      }
      s_len[threadIdx.x] = len;
      __syncthreads();
      const uint32_t tot = block_excl_scan_u32(s_len, blockDim.x, s_tmp);
      if (g < g1 && len) {
        const uint32_t a = run + s_len[threadIdx.x], e = a + len;
        // batches whose first record lies in [a, e)
        for (uint32_t k = (a + kFCap - 1) / kFCap; k * kFCap < e && k < nb; ++k) {
          FItem it{};
          it.c = c; it.f0 = f; it.f1 = f + 1; it.kind = 1;
          it.n = min((uint32_t)kFCap, s_sz[f] - k * kFCap);
          it.g_start = g; it.skip = k * kFCap - a; it.base = cs + s_base[f];
          items_b[i0 + k] = it;
        }
      }
      run += tot;
      __syncthreads();
    }
  }
}

// Big fine buckets: CSC offsets of their vertices and the per-batch cursors.
__global__ void k_big_scan(FineCtx x, const uint32_t* __restrict__ big_buckets, const uint32_t* __restrict__ n_big,
                           const uint64_t* __restrict__ big_base, const uint32_t* __restrict__ cnt_tab,
                           uint64_t* __restrict__ cur_tab, uint64_t* __restrict__ t_offsets,
                           unsigned int* __restrict__ err_overflow) {
  const int Dc = 1 << x.bits_c;
  const uint32_t nbk = *n_big;
  for (uint32_t bk = blockIdx.x; bk < nbk; bk += gridDim.x) {
  const uint32_t fid = big_buckets[3 * bk], i0 = big_buckets[3 * bk + 1], nb = big_buckets[3 * bk + 2];
  const uint64_t v0 = (uint64_t)fid << x.bits_c;
  __shared__ uint64_t s_tot[kFMaxLocal];
  __shared__ uint64_t s_ex[kFMaxLocal];
  for (int v = threadIdx.x; v < Dc; v += blockDim.x) {
    uint64_t run = 0;
    for (uint32_t j = 0; j < nb; ++j) run += cnt_tab[(uint64_t)(i0 + j) * Dc + v];
    s_tot[v] = run;
    if (run >= (1ull << 32)) atomicExch(err_overflow, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t run = big_base[bk];
    for (int v = 0; v < Dc; ++v) {
      s_ex[v] = run;
      run += s_tot[v];
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < Dc; v += blockDim.x) {
    uint64_t run = s_ex[v];
    if (v0 + v < x.V) t_offsets[v0 + v] = run;
    for (uint32_t j = 0; j < nb; ++j) {
      cur_tab[(uint64_t)(i0 + j) * Dc + v] = run;
      run += cnt_tab[(uint64_t)(i0 + j) * Dc + v];
    }
  }
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

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
#include <type_traits>

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
constexpr int kMaxRange = 256;                 // fine buckets per final-stage range
// compact (4-byte record) path
constexpr int kB1cWarps = 16;
constexpr int kB1cSlots = 32;
constexpr int kChunkC = kB1cWarps * kB1cSlots * 32;  // 16384 records per chunk
constexpr int kFcWarps = 8;
constexpr int kFcSlots = 32;
constexpr int kFCapC = kFcWarps * kFcSlots * 32;  // 8192 records per final unit
constexpr int kSegCapC = 512;
constexpr int kTabCap = 8192;  // u16 entries of a fine range's per-chunk segment table in shared memory
constexpr int kMaxBnd = 64;

// Per-chunk descriptor for level 2 (compact): record range, coarse bucket, and
// the source-high decode state (h0 = source-high of the first record, up to
// kChunkBnd boundary offsets inside the chunk; nbnd > kChunkBnd means "read
// the seg_hi row").  Built once by k_chunk_info so level 2 issues no dependent
// global loads per chunk.
constexpr int kChunkBnd = 10;
struct __align__(16) ChunkInfo {
  uint64_t start;
  uint32_t n;
  uint32_t c;
  uint32_t h0;
  uint32_t nbnd;
  uint16_t bnd[kChunkBnd];  // boundary offsets relative to start (< kChunkC)
};
static_assert(sizeof(ChunkInfo) == 48, "ChunkInfo layout");

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

// Source of the edge just before each count tile (compact path): owner of
// edge k*CT - 1 for k >= 1, ~0u for k = 0.
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

// Level-1 output encoders.
// OutFull: (src, dst) uint2 records.
// OutCompact: one u32 per record = (dst_low << L) | src_low with dst_low the
// b+c low destination bits and src_low the L low source bits; the src high
// bits are recovered from the record's position: seg_hi[d][h] = first position
// (in rec_out) of coarse bucket d whose source has src >> L >= h.
struct OutFull {
  static constexpr bool kCompact = false;
  uint2* rec;
};
struct OutCompact {
  static constexpr bool kCompact = true;
  uint32_t* rec;
  uint32_t low_mask;  // (1 << (b + c)) - 1
  int L;              // source low bits kept in the record
  uint32_t src_mask;  // (1 << L) - 1
  uint32_t nh;        // number of src_high values; table rows have nh + 1 entries
  uint64_t* seg_hi;   // [D][nh + 1], pre-filled with ~0
  const uint32_t* prev_src;  // per count tile: source of the element before it (~0u: none)
};

// L1 place.  One CTA per count tile; its place tiles (4096 edges) are processed
// in order with running global cursors per digit, and the next place tile's
// neighbour IDs and offsets window are prefetched with cp.async while the
// current one is ranked.  Writes records grouped by digit, each group in
// stream order.  place_src[t] = owner of edge min(t*kPlaceTile, E-1).
template <int kMode, class In, class Dig, class Out>
__global__ void __launch_bounds__(kL1Warps * 32) k_l1_place(In in, Dig dig, uint64_t E, uint64_t CT, uint64_t ntiles,
                                                           int D, const uint64_t* __restrict__ tbase,
                                                           const uint32_t* __restrict__ place_src, Out out) {
  constexpr int W = kL1Warps, K = kL1Slots, T = W * 32, PT = kPlaceTile;
  using StageT = typename std::conditional<Out::kCompact, uint32_t, uint2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // input staging: CSR -> dst u32[2][PT] + offsets window u64[2][kWinCap]; records -> uint2[2][PT]
  constexpr size_t kInBytes = In::kRecords ? 2 * PT * 8 : 2 * PT * 4 + 2 * kWinCap * 8;
  unsigned char* s_in = smem_raw;
  // the owner marks (round 1) and the staged records (round 2) share storage;
  // compact digit tags reuse the consumed input buffer of the current tile
  StageT* s_stage = reinterpret_cast<StageT*>(smem_raw + kInBytes);   // PT
  uint32_t* s_mark = reinterpret_cast<uint32_t*>(s_stage);            // PT (CSR only, aliases s_stage)
  uint64_t* s_gcur = reinterpret_cast<uint64_t*>(s_stage + PT);       // D
  uint64_t* s_delta = s_gcur + D;                                     // D: gcur - dstart
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_delta + D);         // W * D
  uint32_t* s_scr = s_cnt + W * D;                                    // W * D (safe mode)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * D : 0);      // D
  uint32_t* s_dtot = s_dstart + D;                                    // D
  uint32_t* s_tmp = s_dtot + D;                                       // 40
  uint32_t* s_psrc = s_tmp + 40;                                      // CT/PT + 2 (CSR only)
  uint32_t* s_bh = s_psrc + (CT / PT + 4);                            // D (compact)
  __shared__ uint32_t s_wmax[W];
  __shared__ uint32_t s_last_src;

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
  uint32_t h_prev = 0xffffffffu;  // src_high of the element before the current place tile
  if constexpr (Out::kCompact) {
    uint32_t ps = 0xffffffffu;
    if (k > 0) {
      if constexpr (In::kRecords) ps = in.rec[tb - 1].x;
      else ps = out.prev_src[k];
    }
    h_prev = (ps == 0xffffffffu) ? 0xffffffffu : (ps >> out.L);
  }
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
    uint32_t r_src[K], r_dst[K], r_rank[K];
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
      // per-slot maxima -> per-slot carries (no loop-carried shuffle chain)
      uint32_t sm[K];
      uint32_t wm = 0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        sm[s] = s_mark[seg0 + s * 32 + lane];
        const uint32_t smax = __reduce_max_sync(kFull, sm[s]);
        wm = max(wm, smax);
        r_src[s] = wm;  // inclusive max through slot s (temporarily)
      }
      if (lane == 0) s_wmax[w] = wm;
      __syncthreads();
      uint32_t carry = s0;
      for (int ww = 0; ww < (int)w; ++ww) carry = max(carry, s_wmax[ww]);
      const uint32_t* dbuf = reinterpret_cast<const uint32_t*>(s_in) + b * PT;
#pragma unroll
      for (int s = K - 1; s >= 0; --s) {  // carry into slot s = max over earlier slots
        const uint32_t cin = max(carry, s > 0 ? r_src[s - 1] : 0u);
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        r_dst[s] = valid ? dbuf[i] : 0u;
        uint32_t m = sm[s];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, m, o);
          if (lane >= (uint32_t)o) m = max(m, y);
        }
        r_src[s] = max(m, cin);
      }
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const bool valid = seg0 + s * 32 + lane < n;
        r_rank[s] = warp_rank<kMode>(cnt_w, scr_w, valid ? dig(r_dst[s]) : 0u, valid);
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
        }
        r_src[s] = r.x;
        r_dst[s] = r.y;
        r_rank[s] = warp_rank<kMode>(cnt_w, scr_w, valid ? dig(r.y) : 0u, valid);
      }
    }
    if constexpr (Out::kCompact) {
      // record the src_high boundaries that fall in this tile: h in (h_prev, h_last]
#pragma unroll
      for (int s = 0; s < K; ++s)
        if (seg0 + s * 32 + lane == n - 1) s_last_src = r_src[s];
      __syncthreads();
      const uint32_t h_last = s_last_src >> out.L;
      for (uint32_t h = (h_prev == 0xffffffffu) ? 0u : h_prev + 1; h <= h_last; ++h) {
        for (int d = threadIdx.x; d < D; d += T) s_bh[d] = 0;
        __syncthreads();
        const uint64_t bsrc = (uint64_t)h << out.L;
#pragma unroll
        for (int s = 0; s < K; ++s) {
          const uint32_t i = seg0 + s * 32 + lane;
          if (i < n && (uint64_t)r_src[s] < bsrc) smem_inc(&s_bh[dig(r_dst[s])]);
        }
        __syncthreads();
        for (int d = threadIdx.x; d < D; d += T) out.seg_hi[(uint64_t)d * (out.nh + 1) + h] = s_gcur[d] + s_bh[d];
        __syncthreads();
      }
      h_prev = h_last;
    }
    __syncthreads();  // marks consumed: s_stage may be overwritten from here on
    warp_counts_to_bases<W>(s_cnt, D, s_dstart, s_dtot, s_tmp);
    for (int d = threadIdx.x; d < D; d += T) s_delta[d] = s_gcur[d] - s_dstart[d];
    // digit tags (compact) live in the consumed input buffer of this tile
    uint16_t* s_sdig = reinterpret_cast<uint16_t*>(s_in + (size_t)b * PT * (In::kRecords ? 8 : 4));
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i = seg0 + s * 32 + lane;
      const bool valid = i < n;
      const uint32_t d = valid ? dig(r_dst[s]) : 0u;
      const uint32_t pos = valid ? cnt_w[d] + r_rank[s] : 0u;  // base of (warp, digit) + warp-local rank
      if (valid) {
        if constexpr (Out::kCompact) {
          s_stage[pos] = ((r_dst[s] & out.low_mask) << out.L) | (r_src[s] & out.src_mask);
          s_sdig[pos] = (uint16_t)d;
        } else {
          s_stage[pos] = make_uint2(r_src[s], r_dst[s]);
        }
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += T) {
      const StageT r = s_stage[i];
      uint32_t d;
      if constexpr (Out::kCompact) d = s_sdig[i];
      else d = dig(r.y);
      out.rec[s_delta[d] + i] = r;
    }
    __syncthreads();
    if constexpr (!In::kRecords)
      for (int i = threadIdx.x; i < PT; i += T) s_mark[i] = 0;
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

// Same for the compact path's 16K-record chunks.
__global__ void k_coarse_info_c(const uint64_t* __restrict__ tbase, uint64_t ntiles, int D1, uint64_t E,
                                uint64_t* __restrict__ cstart, uint32_t* __restrict__ chunk_first) {
  extern __shared__ uint32_t s_nch[];
  __shared__ uint32_t s_tmp[40];
  for (int c = threadIdx.x; c <= D1; c += blockDim.x) cstart[c] = (c < D1) ? tbase[(uint64_t)c * ntiles] : E;
  __syncthreads();
  for (int c = threadIdx.x; c < D1; c += blockDim.x) {
    const uint64_t sz = cstart[c + 1] - cstart[c];
    s_nch[c] = (uint32_t)((sz + kChunkC - 1) / kChunkC);
  }
  __syncthreads();
  const uint32_t total = block_excl_scan_u32(s_nch, D1, s_tmp);
  for (int c = threadIdx.x; c < D1; c += blockDim.x) chunk_first[c] = s_nch[c];
  if (threadIdx.x == 0) chunk_first[D1] = total;
}

// Per-chunk descriptors for the compact level 2 (one warp per chunk).
__global__ void k_chunk_info(const uint64_t* __restrict__ cstart, const uint32_t* __restrict__ chunk_first, int D1,
                             const uint32_t* __restrict__ chunk_bucket, const uint64_t* __restrict__ seg_hi,
                             uint32_t nh, ChunkInfo* __restrict__ info) {
  const uint32_t nchunks = chunk_first[D1];
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < nchunks; g += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t c = chunk_bucket[g];
    const uint64_t start = cstart[c] + (uint64_t)(g - chunk_first[c]) * kChunkC;
    const uint32_t n = (uint32_t)umin64(kChunkC, cstart[c + 1] - start);
    const uint64_t* row = seg_hi + (uint64_t)c * (nh + 1);
    uint32_t below = 0, inside = 0;
    uint16_t mine[kChunkBnd];
    for (uint32_t h0 = 1; h0 <= nh; h0 += 32) {  // ordered scan: boundaries in increasing h
      const uint32_t h = h0 + lane;
      const uint64_t v = (h <= nh) ? row[h] : ~0ull;
      below += __popc(__ballot_sync(kFull, v <= start));
      const uint32_t in = __ballot_sync(kFull, v > start && v < start + n);
      uint32_t m = in;
      while (m) {
        const int q = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t bv = __shfl_sync(kFull, v, q);
        if (inside < (uint32_t)kChunkBnd) mine[inside] = (uint16_t)(bv - start);
        ++inside;
      }
    }
    if (lane == 0) {
      ChunkInfo ci;
      ci.start = start;
      ci.n = n;
      ci.c = c;
      ci.h0 = below;
      ci.nbnd = inside;
      for (int k = 0; k < kChunkBnd; ++k) ci.bnd[k] = (k < (int)inside) ? mine[k] : (uint16_t)0xffff;
      info[g] = ci;
    }
  }
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

// ---- final stage: per coarse-bucket fine ranges, one CTA per range --------
// A range = fine buckets [f0, f1) of coarse bucket c.  The CTA walks it as a
// pipeline of units, gathering unit k+1 with cp.async while ranking unit k:
//   kind 0  group of consecutive small fine buckets (<= kFCap records,
//           <= kFMaxLocal local vertices): one pass, contiguous CSC slice;
//   kind 1  count batch of a big fine bucket (per-vertex counts);
//   kind 2  place batch of a big fine bucket (runs at per-vertex cursors).
// Walking the fine buckets of a coarse bucket in order keeps the chunk segment
// tables in L1 and a big bucket's second (place) read in L2.
struct FRange {
  uint32_t c, f0, f1, prio;
};

struct FUnit {
  uint32_t kind;
  uint32_t f0, f1;
  uint32_t n;
  uint32_t g, skip;  // gather start: absolute chunk id, records to skip there
  uint32_t last;     // kind 1: last count batch of its bucket
  uint32_t first;    // kind 1: first count batch of its bucket
  uint64_t base;     // CSC position of f0's first record
};

// Gather `n` records of fine digits [f0, f1) of coarse bucket c, starting at
// chunk g (skipping `skip` records of that chunk's slice), into dst with
// cp.async.  All threads.  Returns the position after the last record
// (g_out, skip_out).
struct CoarseInfo {
  uint32_t g_first, g_end;  // chunk ids of the coarse bucket
  uint64_t cs, ce;          // record range of the coarse bucket
};

__device__ __forceinline__ void gather_unit(const FineCtx& x, const CoarseInfo& ci, uint32_t f0, uint32_t f1,
                                            uint32_t n, uint32_t g, uint32_t skip, uint2* dst, uint64_t* s_st,
                                            uint32_t* s_pos, uint32_t* s_seg, uint32_t* s_tmp, uint32_t& g_out,
                                            uint32_t& skip_out) {
  const uint32_t g_first = ci.g_first, g_end = ci.g_end;
  const uint64_t cs = ci.cs, ce = ci.ce;
  uint32_t got = 0;
  g_out = g;
  skip_out = skip;
  uint32_t gb = g;
  while (gb < g_end && got < n) {
    const int nch = (int)min((uint32_t)kSegCap, g_end - gb);
    for (int j = threadIdx.x; j < nch; j += blockDim.x) {
      const uint64_t cpos = cs + (uint64_t)(gb + j - g_first) * kChunk;
      uint32_t a, e;
      if (x.segoff) {
        const uint16_t* so = x.segoff + (uint64_t)(gb + j) * (x.Db + 1);
        a = so[f0];
        e = so[f1];
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
    const uint32_t lo = skip, want = n - got;
    const uint32_t hi = (tot > lo) ? min(tot, lo + want) : lo;
    // thread-per-record: segment of record i = (#segment starts <= i) - 1, from
    // a per-position count of segment starts and a block prefix sum
    if (hi > lo) {
      const uint32_t m = hi - lo;
      for (uint32_t p = threadIdx.x; p <= m; p += blockDim.x) s_seg[p] = 0;
      __syncthreads();
      uint32_t below = 0;  // segment starts at or before lo (this thread's share)
      for (int j = threadIdx.x; j < nch; j += blockDim.x) {
        const uint32_t a = s_pos[j];
        if (a <= lo) ++below;
        else if (a < hi) atomicAdd(&s_seg[a - lo], 1u);
      }
      below = __reduce_add_sync(kFull, below);
      if (lane_id() == 0) atomicAdd(&s_tmp[36], below);
      __syncthreads();
      const uint32_t base = s_tmp[36];
      block_excl_scan_u32(s_seg, (int)m + 1, s_tmp);  // s_seg[m] must be 0 (zeroed below)
      for (uint32_t p = threadIdx.x; p < m; p += blockDim.x) {
        const uint32_t j = base - 1 + s_seg[p + 1];  // inclusive count at p
        const uint32_t i = lo + p;
        cp_async8(dst + got + p, x.rec + s_st[j] + (i - s_pos[j]));
      }
      if (threadIdx.x == 0) s_tmp[36] = 0;
    }
    if (hi > lo) {
      got += hi - lo;
      if (got >= n) {
        // position after the last record: chunk containing index hi-1 (+1 past it)
        int lo_j = 0, hi_j = nch - 1;  // last j with s_pos[j] < hi
        while (lo_j < hi_j) {
          const int mid = (lo_j + hi_j + 1) >> 1;
          if (s_pos[mid] < hi) lo_j = mid; else hi_j = mid - 1;
        }
        g_out = gb + lo_j;
        skip_out = hi - s_pos[lo_j];
        __syncthreads();
        return;
      }
    }
    skip = (tot > skip) ? 0 : skip - tot;
    gb += nch;
    __syncthreads();
  }
  g_out = gb;
  skip_out = skip;
}

template <int kMode>
__global__ void __launch_bounds__(kFWarps * 32) k_final(FineCtx x, const FRange* __restrict__ ranges,
                                                       const uint32_t* __restrict__ n_ranges_ptr,
                                                       unsigned int* __restrict__ range_ctr,
                                                       const uint32_t* __restrict__ fine_size,
                                                       const uint64_t* __restrict__ fine_base,
                                                       uint64_t* __restrict__ t_offsets, uint32_t* __restrict__ t_edges,
                                                       unsigned int* __restrict__ err_overflow,
                                                       unsigned long long* __restrict__ prof) {
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
  uint64_t* s_cur = reinterpret_cast<uint64_t*>(s_tmp + 40);               // kFMaxLocal (big cursors)
  uint32_t* s_bcnt = reinterpret_cast<uint32_t*>(s_cur + kFMaxLocal);      // kFMaxLocal (big counts)
  __shared__ uint32_t s_range;

  const uint32_t n_ranges = *n_ranges_ptr;
  const uint32_t lane = lane_id(), w = warp_id();
  const int Dc = 1 << x.bits_c;
  const uint32_t maxf = (uint32_t)max(1, kFMaxLocal >> x.bits_c);
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * kFMaxLocal; i += T) s_scr[i] = 0;

  // ---- unit generator (uniform across threads); range sizes/bases live in smem
  uint32_t* s_rsz = s_bcnt + kFMaxLocal;                              // kMaxRange
  uint64_t* s_rbase = reinterpret_cast<uint64_t*>(s_rsz + kMaxRange);  // kMaxRange
  uint32_t* s_seg = reinterpret_cast<uint32_t*>(s_rbase + kMaxRange);   // kFCap + 4 (gather scratch)
  if (threadIdx.x == 0) s_tmp[36] = 0;
  struct Gen {
    uint32_t c, f, f0, f1;     // current range (f relative to the coarse bucket)
    uint32_t big_f, big_left;  // big bucket in progress
    uint32_t phase;            // 1 = counting, 2 = placing
    uint32_t g, skip;          // gather position inside the big bucket
    uint64_t big_base;
    uint32_t big_size;
    bool live;
    CoarseInfo ci;
  } gen;
  gen.live = false;
  gen.big_left = 0;
  gen.phase = 0;
  auto fetch_range = [&]() -> bool {
    __syncthreads();  // previous range's smem arrays are no longer read
    if (threadIdx.x == 0) s_range = atomicAdd(range_ctr, 1u);
    __syncthreads();
    const uint32_t r = s_range;
    if (r >= n_ranges) return false;
    const FRange R = ranges[r];
    gen.c = R.c;
    gen.f0 = R.f0;
    gen.f = R.f0;
    gen.f1 = R.f1;
    gen.live = true;
    gen.ci.g_first = x.chunk_first[R.c];
    gen.ci.g_end = x.chunk_first[R.c + 1];
    gen.ci.cs = x.cstart[R.c];
    gen.ci.ce = x.cstart[R.c + 1];
    const uint64_t fb = (uint64_t)R.c * x.Db + R.f0;
    for (uint32_t i = threadIdx.x; i < R.f1 - R.f0; i += blockDim.x) {
      s_rsz[i] = fine_size[fb + i];
      s_rbase[i] = fine_base[fb + i];
    }
    __syncthreads();
    return true;
  };
  // next unit; returns false when all work is exhausted
  auto next_unit = [&](FUnit& u) -> bool {
    while (true) {
      if (gen.big_left) {
        u.kind = gen.phase;
        u.f0 = gen.big_f;
        u.f1 = gen.big_f + 1;
        u.n = min((uint32_t)CAP, gen.big_left);
        u.g = gen.g;
        u.skip = gen.skip;
        u.base = gen.big_base;
        gen.big_left -= u.n;
        u.last = (gen.big_left == 0);
        u.first = (gen.phase == 1 && gen.big_left + u.n == gen.big_size);
        if (gen.big_left == 0 && gen.phase == 1) {  // counting done: place pass next
          gen.phase = 2;
          gen.big_left = gen.big_size;
          gen.g = gen.ci.g_first;
          gen.skip = 0;
          u.last = 1;
          return true;
        }
        if (gen.big_left == 0) gen.phase = 0;
        return true;
      }
      if (!gen.live || gen.f >= gen.f1) {
        if (!fetch_range()) return false;
        continue;
      }
      const uint32_t sz = s_rsz[gen.f - gen.f0];
      if (sz == 0) { ++gen.f; continue; }
      if (sz > (uint32_t)CAP) {
        gen.big_f = gen.f;
        gen.big_size = sz;
        gen.big_left = sz;
        gen.big_base = s_rbase[gen.f - gen.f0];
        gen.phase = 1;
        gen.g = gen.ci.g_first;
        gen.skip = 0;
        ++gen.f;
        continue;
      }
      uint32_t total = sz, e = gen.f + 1;
      while (e < gen.f1 && e - gen.f < maxf) {
        const uint32_t z = s_rsz[e - gen.f0];
        if (z > (uint32_t)CAP || total + z > (uint32_t)CAP) break;
        total += z;
        ++e;
      }
      u.kind = 0;
      u.f0 = gen.f;
      u.f1 = e;
      u.n = total;
      u.g = gen.ci.g_first;
      u.skip = 0;
      u.last = 0;
      u.first = 0;
      u.base = s_rbase[gen.f - gen.f0];
      gen.f = e;
      return true;
    }
  };
  auto issue = [&](const FUnit& u, int b) {
    uint32_t go, so;
    gather_unit(x, gen.ci, u.f0, u.f1, u.n, u.g, u.skip, s_buf + b * CAP, s_st, s_pos, s_seg, s_tmp, go, so);
    if (u.kind != 0 && !(u.kind == 1 && u.last)) {  // continue the big bucket walk
      gen.g = go;
      gen.skip = so;
    }
    cp_commit();
  };

  FUnit u0, u1;
  uint32_t c0 = 0, c1 = 0, cur_c = 0;
  __shared__ unsigned long long pacc[10];  // profiling accumulators (thread 0)
  __shared__ long long tprev;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 10; ++i) pacc[i] = 0;
    tprev = clock64();
  }
  auto ptick = [&](int ph) {
    if (prof && threadIdx.x == 0) {
      const long long tn = clock64();
      pacc[ph] += (unsigned long long)(tn - tprev);
      tprev = tn;
    }
  };
  if (!next_unit(u0)) return;
  c0 = gen.c;
  issue(u0, 0);
  for (int it = 0;; ++it) {
    const int b = it & 1;
    ptick(9);
    const bool more = next_unit(u1);
    c1 = gen.c;
    ptick(0);
    if (more) {
      issue(u1, b ^ 1);
      ptick(1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    // ---- process u0 (coarse bucket c0) from buffer b
    cur_c = c0;
    const FUnit u = u0;
    const uint32_t n = u.n, f0 = u.f0;
    const uint32_t nloc = (u.f1 - u.f0) << x.bits_c;
    uint32_t* cnt_w = s_cnt + w * nloc;
    uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * nloc : 0);
    for (int i = threadIdx.x; i < W * kFMaxLocal; i += T) s_cnt[i] = 0;
    if (u.kind == 1 && u.first)
      for (int v = threadIdx.x; v < Dc; v += T) s_bcnt[v] = 0;  // first count batch of a big bucket
    __syncthreads();
    ptick(2);
    if (prof && threadIdx.x == 0) pacc[7 + (u.kind == 0 ? 0 : 1)] += 1;
    uint2* buf = s_buf + b * CAP;
    const uint32_t shift_f = x.bits_c, mask_f = (uint32_t)x.Db - 1;
    auto local_of = [&](uint32_t dst) -> uint32_t {
      return ((((dst >> shift_f) & mask_f) - f0) << shift_f) | (dst & x.mask_c);
    };
    const uint32_t seg0 = w * (K * 32);
    if (u.kind == 1) {
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        if (i < n) smem_inc(&s_bcnt[buf[i].y & x.mask_c]);
      }
      __syncthreads();
      if (u.last) {  // CSC offsets of the big bucket's vertices and place cursors
        if (threadIdx.x == 0) {
          uint64_t run = u.base;
          for (int v = 0; v < Dc; ++v) {
            s_cur[v] = run;
            run += s_bcnt[v];
          }
        }
        __syncthreads();
        const uint64_t v0 = ((uint64_t)cur_c * x.Db + u.f0) << x.bits_c;
        for (int v = threadIdx.x; v < Dc; v += T)
          if (v0 + v < x.V) t_offsets[v0 + v] = s_cur[v];
        __syncthreads();
      }
    } else {
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        if (i < n) smem_inc(&cnt_w[local_of(buf[i].y)]);
      }
      __syncthreads();
      ptick(3);
      warp_counts_to_bases<W>(s_cnt, (int)nloc, s_dstart, s_dtot, s_tmp);
      ptick(4);
      if (u.kind == 0) {
        const uint64_t v0 = ((uint64_t)cur_c * x.Db + u.f0) << x.bits_c;
        for (uint32_t v = threadIdx.x; v < nloc; v += T)
          if (v0 + v < x.V) t_offsets[v0 + v] = u.base + s_dstart[v];
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
      __syncthreads();
#pragma unroll
      for (int s = 0; s < K; ++s)
        if (seg0 + s * 32 + lane < n) buf[pp[s]] = rr[s];
      __syncthreads();
      ptick(5);
      if (u.kind == 0) {
        for (uint32_t i = threadIdx.x; i < n; i += T) t_edges[u.base + i] = buf[i].x;
      } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) {
          const uint2 r = buf[i];
          t_edges[s_cur[r.y] + (i - s_dstart[r.y])] = r.x;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < Dc; v += T) s_cur[v] += s_dtot[v];
      }
    }
    __syncthreads();
    ptick(6);
    if (!more) break;
    u0 = u1;
    c0 = c1;
  }
  if (prof && threadIdx.x == 0)
    for (int i = 0; i < 10; ++i) atomicAdd(&prof[i], pacc[i]);
  (void)err_overflow;
}

// Plan the final stage: one CTA per coarse bucket.  Fine-bucket sizes (sum of
// the chunk segment tables) and CSC bases; t_offsets of empty fine buckets;
// fine ranges of ~`target` records (a range never splits a fine bucket).
__global__ void k_f_plan(FineCtx x, uint32_t target, uint32_t* __restrict__ fine_size, uint64_t* __restrict__ fine_base,
                         FRange* __restrict__ ranges, uint32_t* __restrict__ n_ranges, uint64_t* __restrict__ t_offsets,
                         unsigned int* __restrict__ err_overflow) {
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_sz = s_dyn;          // Db
  uint32_t* s_base = s_sz + x.Db;  // Db
  __shared__ uint32_t s_tmp[40];
  const uint32_t c = blockIdx.x;
  const int Db = x.Db, Dc = 1 << x.bits_c;
  const uint32_t g0 = x.chunk_first[c], g1 = x.chunk_first[c + 1];
  const uint64_t cs = x.cstart[c];
  for (int f = threadIdx.x; f < Db; f += blockDim.x) {
    uint64_t sum = 0;
    if (x.segoff) {
      for (uint32_t g = g0; g < g1; ++g) {
        const uint16_t* so = x.segoff + (uint64_t)g * (Db + 1);
        sum += (uint32_t)so[f + 1] - so[f];
      }
    } else {
      sum = x.cstart[c + 1] - cs;
    }
    if (sum >= (1ull << 32)) atomicExch(err_overflow, 1u);
    s_sz[f] = (uint32_t)sum;
    s_base[f] = (uint32_t)sum;
  }
  __syncthreads();
  // bases relative to cs fit 32 bits unless the coarse bucket holds >= 2^32 records
  const uint64_t nc = x.cstart[c + 1] - cs;
  if (nc >= (1ull << 32)) {
    if (threadIdx.x == 0) {
      uint64_t run = cs;
      for (int f = 0; f < Db; ++f) {
        fine_base[(uint64_t)c * Db + f] = run;
        run += s_sz[f];
      }
    }
    __syncthreads();
  } else {
    block_excl_scan_u32(s_base, Db, s_tmp);
    for (int f = threadIdx.x; f < Db; f += blockDim.x) fine_base[(uint64_t)c * Db + f] = cs + s_base[f];
  }
  for (int f = threadIdx.x; f < Db; f += blockDim.x) fine_size[(uint64_t)c * Db + f] = s_sz[f];
  __syncthreads();
  for (int f = 0; f < Db; ++f) {  // t_offsets of empty fine buckets
    if (s_sz[f]) continue;
    const uint64_t v0 = ((uint64_t)c * Db + f) << x.bits_c;
    const uint64_t val = fine_base[(uint64_t)c * Db + f];
    for (int v = threadIdx.x; v < Dc; v += blockDim.x)
      if (v0 + v < x.V) t_offsets[v0 + v] = val;
  }
  if (threadIdx.x != 0 || nc == 0) return;
  uint64_t acc = 0;
  uint32_t f0 = 0;
  // ranges narrow enough for their segment table (nch x (width+1) u16) to sit in shared memory
  const uint32_t nch = g1 - g0;
  const uint32_t wcap = (nch * 2 <= (uint32_t)kTabCap) ? min((uint32_t)kMaxRange, (uint32_t)kTabCap / nch - 1)
                                                       : (uint32_t)kMaxRange;
  for (uint32_t f = 0; f < (uint32_t)Db; ++f) {
    acc += s_sz[f];
    if (acc >= target || f + 1 == (uint32_t)Db || f + 1 - f0 >= wcap) {
      FRange r;
      r.c = c;
      r.f0 = f0;
      r.f1 = f + 1;
      r.prio = (uint32_t)umin64(acc, 0xffffffffull);  // records in the range
      ranges[atomicAdd(n_ranges, 1u)] = r;
      f0 = f + 1;
      acc = 0;
    }
  }
}

// Order the fine ranges largest first (longest-processing-time-first), so the
// ranges holding the heaviest vertices start early instead of forming the tail.
// One CTA, bitonic sort of (size desc, index) keys; lists longer than
// kRangeSortCap keep their order (scheduling only, results do not depend on it).
constexpr int kRangeSortCap = 4096;
__global__ void __launch_bounds__(1024) k_range_sort(FRange* __restrict__ ranges, const uint32_t* __restrict__ n_ranges) {
  __shared__ unsigned long long key[kRangeSortCap];
  const uint32_t n = *n_ranges;
  if (n < 2 || n > (uint32_t)kRangeSortCap) return;
  uint32_t np = 1;
  while (np < n) np <<= 1;
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x)
    key[i] = (i < n) ? (((unsigned long long)(~ranges[i].prio) << 32) | i) : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= np; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const unsigned long long a = key[i], b = key[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            key[i] = b;
            key[l] = a;
          }
        }
      }
      __syncthreads();
    }
  FRange tmp[kRangeSortCap / 1024];
#pragma unroll
  for (int t = 0; t < kRangeSortCap / 1024; ++t) {
    const uint32_t i = threadIdx.x + t * 1024;
    if (i < n) tmp[t] = ranges[(uint32_t)key[i]];
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < kRangeSortCap / 1024; ++t) {
    const uint32_t i = threadIdx.x + t * 1024;
    if (i < n) ranges[i] = tmp[t];
  }
}

// ===================== compact (4-byte record) levels 2 and 3 =====================
// R1 (level-1 output): (dst_low << L) | src_low, src_high from seg_hi (see OutCompact).
// R2 (level-2 output): (d << nb) | src, d = the c low destination bits.

struct DecodeC {
  int L;              // source low bits in R1
  uint32_t src_mask;  // (1 << L) - 1
  uint32_t nh;        // src_high values; seg_hi rows have nh + 1 entries
  const uint64_t* seg_hi;
  int bits_c;         // low destination digit bits
  int nb;             // source bits in R2
  int gbits;          // low fine-digit bits kept in R2 (final units span aligned groups of 2^gbits)
};

// Level 2, compact: stable sort of each 16K-record chunk by the middle digit,
// re-encoding R1 -> R2 (source high bits from the chunk's boundary list).
// Chunks move with TMA bulk copies: the 16B-aligned span [start & ~3, ...)
// lands in smem at record offset `off = start & 3`, is ranked and staged in
// place (same offset), and leaves with one bulk store (unaligned head/tail
// records by plain stores).  Needs 3 records of readable padding after rin.
template <int kMode>
__global__ void __launch_bounds__(kB1cWarps * 32) k_b1c(const uint32_t* __restrict__ rin, uint32_t* __restrict__ rout,
                                                       const ChunkInfo* __restrict__ cinfo,
                                                       const uint32_t* __restrict__ chunk_first, int D1, DecodeC dc,
                                                       int Db, uint16_t* __restrict__ segoff,
                                                       unsigned long long* __restrict__ prof) {
  constexpr int W = kB1cWarps, K = kB1cSlots, T = W * 32, CH = kChunkC, CHP = kChunkC + 8;
  __shared__ unsigned long long pacc[8];
  __shared__ long long tprev;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) pacc[i] = 0;
    tprev = clock64();
  }
  auto ptick = [&](int ph) {
    if (prof && threadIdx.x == 0) {
      const long long tn = clock64();
      pacc[ph] += (unsigned long long)(tn - tprev);
      tprev = tn;
    }
  };
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem_raw);  // 2 * CHP
  uint32_t* s_cnt = s_buf + 2 * CHP;                        // W * Db
  uint32_t* s_scr = s_cnt + W * Db;
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * Db : 0);
  uint32_t* s_dtot = s_dstart + Db;
  uint32_t* s_tmp = s_dtot + Db;                                        // 40
  uint64_t* s_bnd = reinterpret_cast<uint64_t*>(s_tmp + 40);            // kMaxBnd
  __shared__ uint32_t s_h0, s_nbnd;
  __shared__ __align__(8) uint64_t s_bar[2];
  const uint32_t nchunks = chunk_first[D1];
  const uint32_t lane = lane_id(), w = warp_id();
  uint32_t* cnt_w = s_cnt + w * Db;
  uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * Db : 0);
  const uint32_t seg0 = w * (K * 32);
  const uint32_t shift_f = dc.L + dc.bits_c, mask_f = (uint32_t)Db - 1;
  const uint32_t gmask = (1u << (dc.bits_c + dc.gbits)) - 1;
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * Db; i += T) s_scr[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // chunk g's descriptor comes from `cinfo` (built by k_chunk_info); the next
  // chunk's descriptor is read one iteration ahead (plain loads, used a whole
  // iteration later) so no global round trip is exposed
  ChunkInfo nx = cinfo[min(blockIdx.x, nchunks ? nchunks - 1 : 0)];
  auto issue = [&](const ChunkInfo& ci, int b) {  // thread 0 issues the bulk load
    if (threadIdx.x == 0) {
      const uint64_t a0 = ci.start & ~3ull, a1 = (ci.start + ci.n + 3) & ~3ull;
      const uint32_t bytes = (uint32_t)(a1 - a0) * 4;
      mbar_arrive_expect_tx(&s_bar[b], bytes);
      bulk_g2s(s_buf + b * CHP, rin + a0, bytes, &s_bar[b]);
    }
  };

  uint32_t g = blockIdx.x;
  uint32_t phase[2] = {0, 0};
  if (g < nchunks) issue(nx, 0);
  for (int it = 0; g < nchunks; ++it, g += gridDim.x) {
    const int b = it & 1;
    const uint32_t gn = g + gridDim.x;
    const ChunkInfo cur = nx;
    const uint32_t c = cur.c, n = cur.n;
    const uint64_t start = cur.start;
    const uint32_t off = (uint32_t)(start & 3);
    ptick(7);
    if (gn < nchunks) {
      nx = cinfo[gn];
      // buffer b^1 was last stored from two iterations ago: its bulk store must have read it
      if (threadIdx.x == 0) bulk_wait_read<0>();
      __syncthreads();
      issue(nx, b ^ 1);
    }
    ptick(0);
    for (int i = threadIdx.x; i < W * Db; i += T) s_cnt[i] = 0;
    if (cur.nbnd > (uint32_t)kChunkBnd) {  // many source-high boundaries: read the row
      if (threadIdx.x == 0) {
        s_h0 = 0;
        s_nbnd = 0;
      }
      __syncthreads();
      const uint64_t* row = dc.seg_hi + (uint64_t)c * (dc.nh + 1);
      for (uint32_t h = 1 + threadIdx.x; h <= dc.nh; h += T) {
        const uint64_t v = row[h];
        if (v > start && v < start + n) {
          const uint32_t k = atomicAdd(&s_nbnd, 1u);
          if (k < (uint32_t)kMaxBnd) s_bnd[k] = v;
        }
      }
    } else if (threadIdx.x < (uint32_t)kChunkBnd) {
      s_bnd[threadIdx.x] = start + cur.bnd[threadIdx.x];
      if (threadIdx.x == 0) s_nbnd = cur.nbnd;
    }
    __syncthreads();
    ptick(1);
    mbar_wait_parity(&s_bar[b], phase[b]);
    phase[b] ^= 1;
    __syncthreads();
    ptick(2);
    uint32_t* buf = s_buf + b * CHP + off;
    const uint32_t h0 = cur.h0, nbnd = min(s_nbnd, (uint32_t)kMaxBnd);
    // lane q holds boundary q as an index relative to the chunk start
    const uint32_t my_b = (lane < nbnd) ? (uint32_t)(s_bnd[lane] - start) : 0xffffffffu;
    // single pass: decode, warp-local rank (per-warp counters start at 0)
    uint32_t rr[K], pk[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const uint32_t i0 = seg0 + s * 32;
      const uint32_t i = i0 + lane;
      const bool valid = i < n;
      const uint32_t r = valid ? buf[i] : 0u;
      uint32_t h = h0;
      if (nbnd) {  // source-high of record i = h0 + #{boundaries <= i}
        h += __popc(__ballot_sync(kFull, my_b <= i0));
        uint32_t inslot = __ballot_sync(kFull, my_b > i0 && my_b <= i0 + 31);
        while (inslot) {
          const int q = __ffs(inslot) - 1;
          inslot &= inslot - 1;
          h += (__shfl_sync(kFull, my_b, q) <= i) ? 1u : 0u;
        }
        if (nbnd > 32)
          for (uint32_t q = 32; q < nbnd; ++q) h += ((uint32_t)(s_bnd[q] - start) <= i) ? 1u : 0u;
      }
      const uint32_t src = (h << dc.L) | (r & dc.src_mask);
      const uint32_t lv = (r >> dc.L) & gmask;  // (fine & (G-1)) << c | d
      rr[s] = (lv << dc.nb) | src;
      const uint32_t f = (r >> shift_f) & mask_f;
      pk[s] = (f << 16) | warp_rank<kMode>(cnt_w, scr_w, f, valid);
    }
    __syncthreads();
    ptick(3);
    warp_counts_to_bases<W>(s_cnt, Db, s_dstart, s_dtot, s_tmp);  // syncs; all reads of buf are done
    ptick(4);
#pragma unroll
    for (int s = 0; s < K; ++s)
      if (seg0 + s * 32 + lane < n) buf[cnt_w[pk[s] >> 16] + (pk[s] & 0xffffu)] = rr[s];
    fence_proxy_async_smem();
    __syncthreads();
    ptick(5);
    {  // write-out: aligned middle by one bulk store, head/tail records by plain stores
      const uint64_t a = (start + 3) & ~3ull, e = (start + n) & ~3ull;
      if (a < e) {
        if (threadIdx.x == 0) {
          bulk_s2g(rout + a, buf + (a - start), (uint32_t)(e - a) * 4);
          bulk_commit();
        }
        for (uint32_t i = threadIdx.x; i < (uint32_t)(a - start); i += T) rout[start + i] = buf[i];
        for (uint32_t i = (uint32_t)(e - start) + threadIdx.x; i < n; i += T) rout[start + i] = buf[i];
      } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) rout[start + i] = buf[i];
      }
    }
    uint16_t* so = segoff + (uint64_t)g * (Db + 1);
    for (int f = threadIdx.x; f < Db; f += T) so[f] = (uint16_t)s_dstart[f];
    if (threadIdx.x == 0) so[Db] = (uint16_t)n;
    ptick(6);
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
  if (prof && threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&prof[i], pacc[i]);
}

// Level 3, compact: fine ranges of a coarse bucket walked as units of one
// fine bucket (<= kFCapC records) or batches of a big fine bucket (count pass
// then place pass), with the next unit gathered by cp.async while the current
// one is ranked.
struct FineCtxC {
  const uint32_t* rec;  // R2 records, chunk-major (each chunk sorted by fine digit)
  const uint64_t* cstart;
  const uint32_t* chunk_first;
  const uint16_t* segoff;
  int Db;
  int bits_c;
  int nb;
  int gbits;  // fine-digit bits in R2: units are runs of an aligned group of 2^gbits fine buckets
  uint64_t V;
};

// Gather n records of fine digit f of the coarse bucket, starting at chunk g
// after skipping `skip` records of its slice (warp per segment, cp.async).
__device__ __forceinline__ void gather_unit_c(const FineCtxC& x, const CoarseInfo& ci, uint32_t f, uint32_t f_end,
                                              uint32_t n, uint32_t g, uint32_t skip, uint32_t* dst, uint64_t* s_st,
                                              uint32_t* s_pos, uint32_t* s_tmp, uint32_t& g_out,
                                              uint32_t& skip_out, const uint16_t* tab, uint32_t tw1, uint32_t tf0,
                                              unsigned long long* pa = nullptr) {
  long long t0 = (pa && threadIdx.x == 0) ? clock64() : 0;
  const uint32_t lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
  uint32_t got = 0;
  g_out = g;
  skip_out = skip;
  uint32_t gb = g;
  while (gb < ci.g_end && got < n) {
    const int nch = (int)min((uint32_t)kSegCapC, ci.g_end - gb);
    for (int j = threadIdx.x; j < nch; j += blockDim.x) {
      const uint32_t jr = gb + j - ci.g_first;
      const uint64_t cpos = ci.cs + (uint64_t)jr * kChunkC;
      uint32_t a, e;
      if (tab) {  // range table in shared memory
        a = tab[jr * tw1 + (f - tf0)];
        e = tab[jr * tw1 + (f_end - tf0)];
      } else {
        const uint16_t* so = x.segoff + (uint64_t)(gb + j) * (x.Db + 1);
        a = so[f];
        e = so[f_end];
      }
      s_st[j] = cpos + a;
      s_pos[j] = e - a;
    }
    __syncthreads();
    const uint32_t tot = block_excl_scan_u32(s_pos, nch, s_tmp);
    if (threadIdx.x == 0) s_pos[nch] = tot;
    __syncthreads();
    if (pa && threadIdx.x == 0) {
      const long long t1 = clock64();
      pa[10] += (unsigned long long)(t1 - t0);
      t0 = t1;
    }
    const uint32_t lo = skip, want = n - got;
    const uint32_t hi = (tot > lo) ? min(tot, lo + want) : lo;
    for (int j = w; j < nch; j += nw) {
      const uint32_t a = max(s_pos[j], lo), e = min(s_pos[j + 1], hi);
      if (a >= e) continue;
      const uint64_t src = s_st[j] + (a - s_pos[j]);
      uint32_t* d = dst + got + (a - lo);
      for (uint32_t q = lane; q < e - a; q += 32) cp_async4(d + q, x.rec + src + q);
    }
    if (pa && threadIdx.x == 0) {
      const long long t1 = clock64();
      pa[11] += (unsigned long long)(t1 - t0);
      t0 = t1;
    }
    if (hi > lo) {
      got += hi - lo;
      if (got >= n) {
        int lo_j = 0, hi_j = nch - 1;  // last j with s_pos[j] < hi
        while (lo_j < hi_j) {
          const int mid = (lo_j + hi_j + 1) >> 1;
          if (s_pos[mid] < hi) lo_j = mid; else hi_j = mid - 1;
        }
        g_out = gb + lo_j;
        skip_out = hi - s_pos[lo_j];
        __syncthreads();
        return;
      }
    }
    skip = (tot > skip) ? 0 : skip - tot;
    gb += nch;
    __syncthreads();
  }
  g_out = gb;
  skip_out = skip;
}

template <int kMode>
__global__ void __launch_bounds__(kFcWarps * 32, 2) k_final_c(FineCtxC x, const FRange* __restrict__ ranges,
                                                          const uint32_t* __restrict__ n_ranges_ptr,
                                                          unsigned int* __restrict__ range_ctr,
                                                          const uint32_t* __restrict__ fine_size,
                                                          const uint64_t* __restrict__ fine_base,
                                                          uint64_t* __restrict__ t_offsets,
                                                          uint32_t* __restrict__ t_edges,
                                                          unsigned long long* __restrict__ prof) {
  constexpr int W = kFcWarps, K = kFcSlots, T = W * 32, CAP = kFCapC, ML = kFMaxLocal;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem_raw);              // 2 * CAP (staging in place)
  uint64_t* s_st = reinterpret_cast<uint64_t*>(s_buf + 2 * CAP);        // kSegCapC
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_st + kSegCapC);       // kSegCapC + 4
  uint32_t* s_cnt = s_pos + kSegCapC + 4;                               // W * ML
  uint32_t* s_scr = s_cnt + W * ML;                                     // (safe)
  uint32_t* s_dstart = s_scr + (kMode == kRankSafe ? W * ML : 0);       // ML
  uint32_t* s_dtot = s_dstart + ML;                                     // ML
  uint32_t* s_tmp = s_dtot + ML;                                        // 40
  uint64_t* s_cur = reinterpret_cast<uint64_t*>(s_tmp + 40);            // ML
  uint32_t* s_bcnt = reinterpret_cast<uint32_t*>(s_cur + ML);           // ML
  uint32_t* s_rsz = s_bcnt + ML;                                        // kMaxRange
  uint64_t* s_rbase = reinterpret_cast<uint64_t*>(s_rsz + kMaxRange);   // kMaxRange
  uint16_t* s_tab = reinterpret_cast<uint16_t*>(s_rbase + kMaxRange);   // kTabCap
  __shared__ uint32_t s_range;
  __shared__ unsigned long long pacc[14];  // profiling accumulators (thread 0)
  __shared__ long long tprev, tstart;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 14; ++i) pacc[i] = 0;
    tprev = tstart = clock64();
  }

  const uint32_t n_ranges = *n_ranges_ptr;
  const uint32_t lane = lane_id(), w = warp_id();
  const int Dc = 1 << x.bits_c;
  const uint32_t G = 1u << x.gbits;
  const uint32_t lvmask = (1u << (x.bits_c + x.gbits)) - 1;
  const uint32_t nbmask = (x.nb >= 32) ? 0xffffffffu : ((1u << x.nb) - 1);
  if (kMode == kRankSafe)
    for (int i = threadIdx.x; i < W * ML; i += T) s_scr[i] = 0;

  struct Gen {
    uint32_t c, f, f0, f1;
    uint32_t big_f, big_left, phase, g, skip, big_size;
    uint64_t big_base;
    uint32_t tw1;
    bool live, tab_ok;
    CoarseInfo ci;
  } gen;
  gen.live = false;
  gen.big_left = 0;
  gen.phase = 0;
  auto fetch_range = [&]() -> bool {
    __syncthreads();
    if (threadIdx.x == 0) s_range = atomicAdd(range_ctr, 1u);
    __syncthreads();
    const uint32_t r = s_range;
    if (r >= n_ranges) return false;
    const FRange R = ranges[r];
    gen.c = R.c;
    gen.f0 = R.f0;
    gen.f = R.f0;
    gen.f1 = R.f1;
    gen.live = true;
    gen.ci.g_first = x.chunk_first[R.c];
    gen.ci.g_end = x.chunk_first[R.c + 1];
    gen.ci.cs = x.cstart[R.c];
    gen.ci.ce = x.cstart[R.c + 1];
    const uint64_t fb = (uint64_t)R.c * x.Db + R.f0;
    for (uint32_t i = threadIdx.x; i < R.f1 - R.f0; i += blockDim.x) {
      s_rsz[i] = fine_size[fb + i];
      s_rbase[i] = fine_base[fb + i];
    }
    gen.tw1 = R.f1 - R.f0 + 1;
    const uint32_t nchr = gen.ci.g_end - gen.ci.g_first;
    gen.tab_ok = (uint64_t)nchr * gen.tw1 <= (uint64_t)kTabCap;
    if (gen.tab_ok) {  // the range's segment offsets for every chunk of the coarse bucket, one coalesced pass
      const uint32_t tn = nchr * gen.tw1;
      for (uint32_t i0 = threadIdx.x; i0 < tn; i0 += 4 * blockDim.x) {
        uint16_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // four independent loads in flight per thread
          const uint32_t i = i0 + q * blockDim.x;
          const uint32_t jj = i / gen.tw1, t = i - jj * gen.tw1;
          v[q] = (i < tn) ? x.segoff[(uint64_t)(gen.ci.g_first + jj) * (x.Db + 1) + R.f0 + t] : (uint16_t)0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i0 + q * blockDim.x < tn) s_tab[i0 + q * blockDim.x] = v[q];
      }
    }
    __syncthreads();
    return true;
  };
  auto next_unit = [&](FUnit& u) -> bool {
    while (true) {
      if (gen.big_left) {  // place batches of a big fine bucket
        u.kind = 2;
        u.f0 = gen.big_f;
        u.f1 = gen.big_f + 1;
        u.n = min((uint32_t)CAP, gen.big_left);
        u.g = gen.g;
        u.skip = gen.skip;
        u.base = gen.big_base;
        gen.big_left -= u.n;
        u.last = (gen.big_left == 0);
        u.first = 0;
        return true;
      }
      if (!gen.live || gen.f >= gen.f1) {
        if (!fetch_range()) return false;
        continue;
      }
      const uint32_t sz = s_rsz[gen.f - gen.f0];
      if (sz == 0) { ++gen.f; continue; }
      if (sz > (uint32_t)CAP) {  // big fine bucket: a streaming count unit (no gather), then batches
        gen.big_f = gen.f;
        gen.big_size = sz;
        gen.big_left = sz;
        gen.big_base = s_rbase[gen.f - gen.f0];
        gen.g = gen.ci.g_first;
        gen.skip = 0;
        ++gen.f;
        u.kind = 1;
        u.f0 = gen.big_f;
        u.f1 = gen.big_f + 1;
        u.n = 0;
        u.g = gen.ci.g_first;
        u.skip = 0;
        u.last = 1;
        u.first = 1;
        u.base = gen.big_base;
        return true;
      }
      const uint32_t blk_end = min(gen.f1, (gen.f | (G - 1)) + 1);  // end of the aligned group
      uint32_t total = sz, e = gen.f + 1;
      while (e < blk_end) {
        const uint32_t z = s_rsz[e - gen.f0];
        if (z > (uint32_t)CAP || total + z > (uint32_t)CAP) break;
        total += z;
        ++e;
      }
      u.kind = 0;
      u.f0 = gen.f;
      u.f1 = e;
      u.n = total;
      u.g = gen.ci.g_first;
      u.skip = 0;
      u.last = 0;
      u.first = 0;
      u.base = s_rbase[gen.f - gen.f0];
      gen.f = e;
      return true;
    }
  };
  auto issue = [&](const FUnit& u, int b) {
    uint32_t go, so;
    gather_unit_c(x, gen.ci, u.f0, u.f1, u.n, u.g, u.skip, s_buf + b * CAP, s_st, s_pos, s_tmp, go, so,
                  gen.tab_ok ? s_tab : nullptr, gen.tw1, gen.f0, prof ? pacc : nullptr);
    if (u.kind == 2) {
      gen.g = go;
      gen.skip = so;
    }
    cp_commit();
  };

  auto ptick = [&](int ph) {
    if (prof && threadIdx.x == 0) {
      const long long tn = clock64();
      pacc[ph] += (unsigned long long)(tn - tprev);
      tprev = tn;
    }
  };
  FUnit u0, u1;
  uint32_t c0 = 0, c1 = 0;
  CoarseInfo ci0, ci1;
  if (!next_unit(u0)) return;
  c0 = gen.c;
  ci0 = gen.ci;
  issue(u0, 0);
  for (int it = 0;; ++it) {
    const int b = it & 1;
    ptick(9);
    const bool more = next_unit(u1);
    c1 = gen.c;
    ci1 = gen.ci;
    ptick(0);
    if (more) {
      issue(u1, b ^ 1);
      ptick(1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    const uint32_t cur_c = c0;
    const CoarseInfo cur_ci = ci0;
    const FUnit u = u0;
    const uint32_t n = u.n;
    const uint32_t nloc = (u.f1 - u.f0) << x.bits_c;               // local vertices of the unit
    const uint32_t lvoff = (u.f0 & (G - 1)) << x.bits_c;            // first local vertex in R2's field
    auto lv_of = [&](uint32_t r) -> uint32_t { return ((r >> x.nb) & lvmask) - lvoff; };
    uint32_t* cnt_w = s_cnt + w * nloc;
    uint32_t* scr_w = s_scr + (kMode == kRankSafe ? w * nloc : 0);
    for (int i = threadIdx.x; i < W * ML; i += T) s_cnt[i] = 0;
    if (u.kind == 1) {
      for (int v = threadIdx.x; v < Dc; v += T) s_bcnt[v] = 0;
      for (int i = threadIdx.x; i < CAP; i += T) s_buf[b * CAP + i] = 0;
    }
    __syncthreads();
    ptick(2);
    if (prof && threadIdx.x == 0) pacc[7 + (u.kind == 0 ? 0 : 1)] += 1;
    uint32_t* buf = s_buf + b * CAP;
    const uint32_t seg0 = w * (K * 32);
    if (u.kind == 1) {
      // Streaming count of the whole big bucket straight from its chunk
      // segments (16-byte loads) into per-warp counters [lv][lane & 15] in the
      // idle staging buffer; the adds are fire-and-forget shared atomics (no
      // read-modify-write chains), folded into s_bcnt at the end.
      const int cw = min(W, (CAP * 4) / (Dc * 16 * 4));  // counting warps that fit the buffer
      uint32_t* c32 = buf + w * Dc * 16 + (lane & 15);
      const long long tk0 = (prof && threadIdx.x == 0) ? clock64() : 0;
      if (w < cw) {
        const uint32_t f = u.f0;
        auto bump = [&](uint32_t r) { atomicAdd(c32 + lv_of(r) * 16, 1u); };
        for (uint32_t j = cur_ci.g_first + w; j < cur_ci.g_end; j += cw) {
          const uint32_t jr = j - cur_ci.g_first;
          uint32_t a, e;
          if (gen.tab_ok) {
            a = s_tab[jr * gen.tw1 + (f - gen.f0)];
            e = s_tab[jr * gen.tw1 + (f + 1 - gen.f0)];
          } else {
            const uint16_t* so = x.segoff + (uint64_t)j * (x.Db + 1);
            a = so[f];
            e = so[f + 1];
          }
          const uint64_t base = cur_ci.cs + (uint64_t)jr * kChunkC;
          // unaligned head/tail by scalar loads, 16-byte aligned body by uint4
          const uint64_t ga = base + a, ge = base + e;
          const uint64_t va = umin64((ga + 3) & ~3ull, ge), ve = (ge & ~3ull) > va ? (ge & ~3ull) : va;
          if (ga + lane < va) bump(__ldg(x.rec + ga + lane));
          if (ve + lane < ge) bump(__ldg(x.rec + ve + lane));
          const uint4* p4 = reinterpret_cast<const uint4*>(x.rec + va);
          const uint32_t n4 = (uint32_t)((ve - va) >> 2);
          for (uint32_t q = lane; q < n4; q += 256) {
            uint4 r[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = (q + 32 * k < n4) ? __ldg(p4 + q + 32 * k) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (q + 32 * k < n4) {
                bump(r[k].x);
                bump(r[k].y);
                bump(r[k].z);
                bump(r[k].w);
              }
          }
        }
        __syncwarp();
        for (int v = 0; v < Dc; ++v) {
          const uint32_t c = (lane < 16) ? c32[v * 16] : 0u;
          const uint32_t t = __reduce_add_sync(kFull, c);
          if (lane == 0 && t) atomicAdd(&s_bcnt[v], t);
        }
      }
      __syncthreads();
      if (prof && threadIdx.x == 0) pacc[12] += (unsigned long long)(clock64() - tk0);
      if (threadIdx.x == 0) {
        uint64_t run = u.base;
        for (int v = 0; v < Dc; ++v) {
          s_cur[v] = run;
          run += s_bcnt[v];
        }
      }
      __syncthreads();
      const uint64_t v0 = ((uint64_t)cur_c * x.Db + u.f0) << x.bits_c;
      for (int v = threadIdx.x; v < Dc; v += T)
        if (v0 + v < x.V) t_offsets[v0 + v] = s_cur[v];
    } else {
      // single pass: warp-local rank (per-warp counters start at 0), then bases
      uint32_t rr[K], pk[K];
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t i = seg0 + s * 32 + lane;
        const bool valid = i < n;
        rr[s] = valid ? buf[i] : 0u;
        const uint32_t lv = valid ? lv_of(rr[s]) : 0u;
        pk[s] = (lv << 16) | warp_rank<kMode>(cnt_w, scr_w, lv, valid);
      }
      __syncthreads();
      ptick(3);
      warp_counts_to_bases<W>(s_cnt, (int)nloc, s_dstart, s_dtot, s_tmp);
      ptick(4);
      if (u.kind == 0) {
        const uint64_t v0 = ((uint64_t)cur_c * x.Db + u.f0) << x.bits_c;
        for (uint32_t v = threadIdx.x; v < nloc; v += T)
          if (v0 + v < x.V) t_offsets[v0 + v] = u.base + s_dstart[v];
      }
#pragma unroll
      for (int s = 0; s < K; ++s)
        if (seg0 + s * 32 + lane < n) buf[cnt_w[pk[s] >> 16] + (pk[s] & 0xffffu)] = rr[s];
      __syncthreads();
      ptick(5);
      if (u.kind == 0) {
        for (uint32_t i = threadIdx.x; i < n; i += T) t_edges[u.base + i] = buf[i] & nbmask;
      } else {
        for (uint32_t i = threadIdx.x; i < n; i += T) {
          const uint32_t r = buf[i], d = lv_of(r);
          t_edges[s_cur[d] + (i - s_dstart[d])] = r & nbmask;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < Dc; v += T) s_cur[v] += s_dtot[v];
      }
    }
    __syncthreads();
    ptick(6);
    if (!more) break;
    u0 = u1;
    c0 = c1;
    ci0 = ci1;
  }
  if (prof && threadIdx.x == 0) {
    pacc[13] = (unsigned long long)(clock64() - tstart);
    for (int i = 0; i < 13; ++i) atomicAdd(&prof[i], pacc[i]);
    atomicMax(&prof[13], pacc[13]);
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

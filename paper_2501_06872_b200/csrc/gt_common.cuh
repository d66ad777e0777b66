// gt_common.cuh — shared device helpers for the B200 transposition kernels.
//
// Ranking model: a warp processes its contiguous item
// range in slots of 32 consecutive items (lane l holds item 32*s + l), so the
// warp's program order equals item order.  Each warp owns a private counter
// array in shared memory.  kRankAtomic: one shared-memory atomicAdd per item;
// B200 returns the old values of same-address lanes of one instruction in
// ascending lane order (gt_selftest_rank_order checks this on the device before
// it is used).  kRankSafe: architecture-guaranteed fallback that builds the
// peer mask with a shared atomicOr and lets the lowest peer advance the count.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gt {

constexpr uint32_t kFull = 0xffffffffu;

enum RankMode : int { kRankAtomic = 0, kRankSafe = 1 };

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Count-only increment (order irrelevant).
__device__ __forceinline__ void smem_inc(uint32_t* p) { atomicAdd(p, 1u); }

// Stable rank of this lane's item among same-digit items of the warp's stream.
// cnt[d] holds the running count (or running position after the base pass) of
// digit d for this warp; scratch[d] must be zero between calls (safe mode).
// All 32 lanes must call; invalid lanes pass valid=false.
template <int kMode>
__device__ __forceinline__ uint32_t warp_rank(uint32_t* cnt, uint32_t* scratch, uint32_t d,
                                              bool valid) {
  if constexpr (kMode == kRankAtomic) {
    (void)scratch;
    uint32_t r = 0;
    if (valid) r = atomicAdd(&cnt[d], 1u);
    return r;
  } else {
    const uint32_t lane = lane_id();
    if (valid) atomicOr(&scratch[d], 1u << lane);
    __syncwarp();
    uint32_t peers = 0, c = 0;
    if (valid) {
      peers = scratch[d];
      c = cnt[d];
    }
    __syncwarp();
    const uint32_t lt = peers & lanemask_lt();
    if (valid && lt == 0) {
      cnt[d] = c + __popc(peers);
      scratch[d] = 0;
    }
    __syncwarp();
    return c + __popc(lt);
  }
}

// Block-wide exclusive scan of a shared uint32 array a[0..n) in place; returns
// the total to all threads.  n may exceed blockDim.x.  Uses `tmp` (>= 33 words).
// Warp w owns a contiguous slice; lanes touch consecutive words (no bank
// conflicts) and a shuffle scan carries 32 elements per step.
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t* a, int n, uint32_t* tmp) {
  const int T = blockDim.x, t = threadIdx.x;
  const int nw = (T + 31) >> 5, w = t >> 5, lane = t & 31;
  const int per = ((n + nw - 1) / nw + 31) & ~31;  // slice per warp, multiple of 32
  const int lo = w * per, hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo + lane; i < hi; i += 32) s += a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if (lane == 0) tmp[w] = s;
  __syncthreads();
  if (t < 32) {
    uint32_t v0 = (t < nw) ? tmp[t] : 0;
    uint32_t v = v0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, v, o);
      if (t >= o) v += y;
    }
    if (t < nw) tmp[t] = v - v0;  // exclusive warp offsets
    if (t == 31) tmp[32] = v;     // total
  }
  __syncthreads();
  uint32_t carry = tmp[w];
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const uint32_t x = (i < hi) ? a[i] : 0u;
    uint32_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t z = __shfl_up_sync(kFull, y, o);
      if (lane >= o) y += z;
    }
    if (i < hi) a[i] = carry + y - x;
    carry += __shfl_sync(kFull, y, 31);
  }
  const uint32_t total = tmp[32];
  __syncthreads();
  return total;
}

// Per-warp counters cnt[W][D] (row per warp).  After counting, turn them into
// tile-local bases: base[w][d] = digit_start[d] + sum_{w'<w} cnt[w'][d].
// digit_start (size D, optional) receives the tile-local start of each digit,
// digit_total (size D, optional) the per-digit totals.  Returns the tile total.
template <int W>
__device__ __forceinline__ uint32_t warp_counts_to_bases(uint32_t* cnt, int D, uint32_t* dstart,
                                                         uint32_t* dtotal, uint32_t* tmp) {
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      uint32_t c = cnt[w * D + d];
      cnt[w * D + d] = run;
      run += c;
    }
    dstart[d] = run;
    if (dtotal) dtotal[d] = run;
  }
  __syncthreads();
  uint32_t total = block_excl_scan_u32(dstart, D, tmp);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const uint32_t b = dstart[d];
#pragma unroll
    for (int w = 0; w < W; ++w) cnt[w * D + d] += b;
  }
  __syncthreads();
  return total;
}

// 64-bit global loads/stores with streaming hints.
__device__ __forceinline__ uint2 ldg_stream(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// ---- cp.async (LDGSTS) helpers: asynchronous global -> shared copies.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// ---- shared-memory accessors on 32-bit shared addresses ------------------
// The hot loops of the place kernels address shared memory through one
// laundered base register: the compiler otherwise re-derives the address of
// the shared window (S2UR SR_CgaCtaId + UMOV + ULEA) and re-loads kernel
// parameters (LDCU) in front of every access, which costs more issue slots
// than the accesses themselves.
// launder: an identity shuffle, so neither nvcc nor ptxas can rematerialise
// the value from its (cheap-looking) definition; it stays in a register.
__device__ __forceinline__ uint32_t launder(uint32_t x) { return __shfl_sync(kFull, x, threadIdx.x & 31u); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;
  asm volatile("{ .reg .u16 t; ld.shared.u16 t, [%1]; cvt.u32.u16 %0, t; }" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("{ .reg .u16 t; cvt.u16.u32 t, %1; st.shared.u16 [%0], t; }" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts_v2(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void sts_v4z(uint32_t a) {  // 16 zero bytes
  asm volatile("{ .reg .b32 z; mov.b32 z, 0; st.shared.v4.b32 [%0], {z,z,z,z}; }" ::"r"(a));
}
// Zero nwords (multiple of 4) 32-bit words at the 16-byte aligned shared address a; tid < NT.
template <int NT>
__device__ __forceinline__ void zero_s(uint32_t a, uint32_t nwords, uint32_t tid) {
  for (uint32_t i = tid * 16; i < nwords * 4; i += NT * 16) sts_v4z(a + i);
}
template <int NT, int NWORDS>
__device__ __forceinline__ void zero_s(uint32_t a, uint32_t tid) {
  static_assert(NWORDS % 4 == 0, "whole 16-byte blocks");
#pragma unroll
  for (int k = 0; k < (NWORDS * 4 + NT * 16 - 1) / (NT * 16); ++k)
    if ((NWORDS * 4) % (NT * 16) == 0 || tid * 16 + k * (NT * 16) < NWORDS * 4) sts_v4z(a + tid * 16 + k * (NT * 16));
}
__device__ __forceinline__ uint32_t atoms_add(uint32_t a, uint32_t v) {
  uint32_t o;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v));
  return o;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) { return __byte_perm(a, b, sel); }

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier --------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// expect_tx without arriving: lets several threads register their own copies'
// bytes on one barrier before issuing them (the tx-count never goes negative)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, completes on `bar` (bytes and addresses 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(s)),
               "l"(g), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global (bulk group); bytes and addresses 16B aligned
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace gt

// gt_api.cu — host orchestration and the extern "C" boundary of libgt.so.
// See include/gt.h for the contract and the reference functions each entry
// point replaces.  No torch types cross this boundary.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gt.h"
#include "gt_kernels.cuh"
#include "gt_v3.cuh"

using namespace gt;

namespace {

thread_local std::string g_err;
int g_forced_rank_mode = -1;           // -1 auto
int g_dev_rank_mode[64];               // per device: -1 unknown, 0/1 decided
std::once_flag g_init_flag;
std::mutex g_mu;

int set_err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

}  // namespace

int gt_internal_set_err(int code, const char* msg) {  // for the other translation units
  g_err = msg;
  return code;
}

namespace {

#define GT_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      if (e_ == cudaErrorMemoryAllocation)                                                      \
        return set_err(GT_ENOMEM, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return set_err(GT_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                          \
  } while (0)

#define GT_LAUNCH_CHECK() GT_CUDA(cudaGetLastError())

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline int bits_for(uint64_t V) {  // bits to address IDs 0..V-1 (>= 1)
  if (V <= 2) return 1;
  return 64 - __builtin_clzll(V - 1);
}

struct Plan {
  uint64_t V = 0, E = 0;
  bool compact = false;  // 4-byte records (R1/R2), see gt_kernels.cuh
  bool wide = false;     // v3 with 64-bit positions and R2 = source (u32) + low digit (u8): E >= 2^32 or nbs + c > 32
  int L = 0, nsh = 0;    // compact R1: source low bits, source high bits
  int gbits = 0;         // compact R2: fine-digit bits kept (final units = aligned groups of 2^gbits)
  int nb = 0, nbs = 0, a = 0, b = 0, c = 0;
  int D1 = 1, Db = 1, Dc = 1;
  uint64_t CT = 65536, ntiles = 0, nplace = 0, max_chunks = 0, max_items_s = 0, max_items_b = 0;
  // workspace offsets
  uint64_t o_rec, o_tcnt, o_tbase, o_psrc, o_cstart, o_cfirst, o_cbucket, o_segoff, o_fsize, o_fbase, o_ranges,
      o_status, o_ctr, o_counters, o_err, o_seghi, o_prev, o_cinfo, total;
};

// wide_b: the level-2 digit may take 10 bits (v3 kernels only; the older
// compact kernels size their shared memory for <= 9).
int make_plan(uint64_t V, uint64_t E, Plan& p, uint64_t Vsrc = 0, bool wide_b = false) {
  p.V = V;
  p.E = E;
  p.nb = bits_for(V);
  p.nbs = bits_for(Vsrc ? Vsrc : V);  // source ID bits (differs on the multi-GPU receiver side)
  if (p.nb > 30) return set_err(GT_EINVAL, "num_vertices > 2^30 is not supported by this build");
  const double avg = V ? (double)E / (double)V : 1.0;
  int a = 0, b = 0, c = 0;
  // compact path: 4-byte records; fine buckets average ~kFCapC/2 records
  {
    // measured on C3 (tools/ab_split.sh): 8-bit middle digits and fine buckets of
    // ~4K records beat 9|9|6 (9.06 -> 8.59 ms); the coarse digit takes the rest
    // (<= 10 bits) and the middle digit grows only when it must
    int cc = 1;
    while (cc < 8 && (double)(1u << (cc + 1)) * std::max(avg, 1.0) <= (double)kFCapC / 2.0) ++cc;
    cc = std::min(cc, 32 - p.nbs);
    cc = std::min(cc, p.nb);
    const int rem = p.nb - cc;
    int ca = rem, cb = 0;
    const int bmax = wide_b ? 10 : 9;
    if (rem > 9) {
      cb = std::min(bmax, std::max(8, rem - 10));
      ca = rem - cb;
    }
    if (const char* sp = getenv("GT_SPLIT")) {  // experiment override "a,b,c" (must cover nb bits)
      int xa = 0, xb = 0, xc = 0;
      if (sscanf(sp, "%d,%d,%d", &xa, &xb, &xc) == 3 && xa + xb + xc == p.nb && xc >= 1 && xa >= 0 && xb >= 0) {
        ca = xa;
        cb = xb;
        cc = xc;
      }
    }
    const int L = 32 - (cb + cc);
    const int nsh = std::max(0, p.nbs - L);
    p.compact = (cc >= 1 && p.nbs + cc <= 32 && ca <= 10 && cb <= bmax && nsh <= 12 &&
                 getenv("GT_FORCE_FULL") == nullptr);
    if (p.compact) {
      a = ca;
      b = cb;
      c = cc;
      p.L = L;
      p.nsh = nsh;
      int gb = std::min(32 - p.nbs - cc, cb);
      while (gb > 0 && (1 << (gb + cc)) > kFMaxLocal) --gb;
      p.gbits = std::max(0, gb);
    }
  }
  // wide v3 form: graphs with E >= 2^32, or whose source IDs leave no room for
  // the low digit in a 4-byte R2 (nbs + c > 32); GT_WIDE=1 forces it (tests)
  const bool v3ok = getenv("GT_V2") == nullptr && getenv("GT_FORCE_FULL") == nullptr;
  if (v3ok && (!p.compact || E >= (1ull << 32) || getenv("GT_WIDE") != nullptr)) {
    int cc = 1;
    while (cc < 8 && (double)(1u << (cc + 1)) * std::max(avg, 1.0) <= (double)kFCapC / 2.0) ++cc;
    cc = std::min(cc, p.nb);
    const int rem = p.nb - cc;
    int ca = rem, cb = 0;
    if (rem > 10) {
      cb = std::min(10, std::max(8, rem - 11));
      ca = rem - cb;
    }
    if (const char* sp = getenv("GT_SPLIT")) {
      int xa = 0, xb = 0, xc = 0;
      if (sscanf(sp, "%d,%d,%d", &xa, &xb, &xc) == 3 && xa + xb + xc == p.nb && xc >= 1 && xc <= 8 && xa >= 0 &&
          xb >= 0) {
        ca = xa;
        cb = xb;
        cc = xc;
      }
    }
    const int L = 32 - (cb + cc);
    const int nsh = std::max(0, p.nbs - L);
    if (cc >= 1 && cc <= 8 && ca <= 11 && cb <= 10 && L >= 1 && nsh <= 16) {
      p.compact = false;
      p.wide = true;
      a = ca;
      b = cb;
      c = cc;
      p.L = L;
      p.nsh = nsh;
      p.gbits = 0;
    }
  }
  if (!p.compact && !p.wide) {
    // final digit: fine buckets of 2^c vertices averaging <= kFCap/2 records
    while (c < 8 && (double)(1u << (c + 1)) * std::max(avg, 1.0) <= (double)kFCap / 2.0) ++c;
    c = std::min(c, p.nb);
    const int rem = p.nb - c;
    if (rem <= 10) {
      a = rem;
      b = 0;
    } else {
      a = rem - rem / 2;
      b = rem / 2;
    }
  }
  if (a > 11 || b > 11) return set_err(GT_EINVAL, "digit split out of range (nb=%d)", p.nb);
  p.a = a;
  p.b = b;
  p.c = c;
  p.D1 = 1 << a;
  p.Db = 1 << b;
  p.Dc = 1 << c;
  p.CT = 65536;
  p.ntiles = (E + p.CT - 1) / p.CT;
  while ((uint64_t)p.D1 * p.ntiles > (1ull << 24)) {
    p.CT *= 2;
    p.ntiles = (E + p.CT - 1) / p.CT;
  }
  p.nplace = (E + kPlaceTile - 1) / kPlaceTile;
  const uint64_t chunk = p.compact ? kChunkC : kChunk;
  p.max_chunks = (E + chunk - 1) / chunk + (uint64_t)p.D1;
  const uint64_t nfine = (uint64_t)p.D1 * p.Db;
  p.max_items_s = nfine;
  p.max_items_b = E / kFCap + nfine;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o = off;
    off = align_up(off + std::max<uint64_t>(bytes, 1), 256);
    return o;
  };
  p.o_rec = take(E * (p.compact ? 4 : 8) + 64);  // + padding for 16B-aligned bulk loads
  p.o_tcnt = take((uint64_t)p.D1 * p.ntiles * 4);
  p.o_tbase = take(((uint64_t)p.D1 * p.ntiles + 1) * 8);
  p.o_psrc = take((p.nplace + 2) * 4);
  p.o_cstart = take((uint64_t)(p.D1 + 1) * 8);
  p.o_cfirst = take((uint64_t)(p.D1 + 1) * 4);
  p.o_cbucket = take(p.max_chunks * 4);
  p.o_segoff = take((p.b || p.compact) ? p.max_chunks * (uint64_t)(p.Db + 1) * 2 : 0);
  p.o_fsize = take(nfine * 4);
  p.o_fbase = take(nfine * 8);
  p.o_ranges = take(nfine * sizeof(FRange));
  const uint64_t max_scan = (uint64_t)p.D1 * p.ntiles + 1;
  p.o_status = take(((max_scan + kScanTile - 1) / kScanTile + 1) * 8);
  p.o_ctr = take(64);
  p.o_counters = take(64);  // n_items_s, n_items_b, n_big
  p.o_err = take(4);
  p.o_seghi = take(p.compact ? (uint64_t)p.D1 * ((1ull << p.nsh) + 1) * 8 : 0);
  p.o_prev = take(p.compact ? (p.ntiles + 1) * 4 : 0);
  p.o_cinfo = take(p.compact ? p.max_chunks * sizeof(ChunkInfo) : 0);
  p.total = off;
  return GT_OK;
}

// ---- cached device memory (workspace when the caller passes none; big-path
// job tables).  One cache per device, grown on demand, never shrunk.
struct Cache {
  void* ptr = nullptr;
  uint64_t bytes = 0;
};
Cache g_ws[64], g_aux[64];

int cache_get(Cache& c, uint64_t bytes, void** out) {
  if (c.bytes < bytes) {
    if (c.ptr) cudaFree(c.ptr);
    c.ptr = nullptr;
    c.bytes = 0;
    GT_CUDA(cudaMalloc(&c.ptr, bytes));
    c.bytes = bytes;
  }
  *out = c.ptr;
  return GT_OK;
}

int current_device(int* dev) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return set_err(GT_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  GT_CUDA(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= 64) return set_err(GT_EINVAL, "device index out of range");
  return GT_OK;
}

int run_selftest(uint64_t trials, uint64_t* violations, cudaStream_t st) {
  unsigned long long* d_bad = nullptr;
  GT_CUDA(cudaMallocAsync(&d_bad, 8, st));
  GT_CUDA(cudaMemsetAsync(d_bad, 0, 8, st));
  const int blocks = 148 * 2, threads = 1024;
  const uint64_t per_launch = (uint64_t)blocks * threads * 64;
  const uint64_t launches = std::max<uint64_t>(1, (trials + per_launch - 1) / per_launch);
  for (uint64_t l = 0; l < launches; ++l) {
    k_selftest_rank<<<blocks, threads, 0, st>>>(d_bad, (uint32_t)(0x9E3779B9u * (l + 1)), 64);
    GT_LAUNCH_CHECK();
  }
  unsigned long long h = 0;
  GT_CUDA(cudaMemcpyAsync(&h, d_bad, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaFreeAsync(d_bad, st));
  GT_CUDA(cudaStreamSynchronize(st));
  *violations = h;
  return GT_OK;
}

int rank_mode_for(int dev, cudaStream_t st, int* mode) {
  if (g_forced_rank_mode >= 0) {
    *mode = g_forced_rank_mode;
    return GT_OK;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  static bool init = false;
  if (!init) {
    for (int i = 0; i < 64; ++i) g_dev_rank_mode[i] = -1;
    init = true;
  }
  if (g_dev_rank_mode[dev] < 0) {
    uint64_t bad = 0;
    int rc = run_selftest(1ull << 26, &bad, st);
    if (rc != GT_OK) return rc;
    g_dev_rank_mode[dev] = bad ? kRankSafe : kRankAtomic;
  }
  *mode = g_dev_rank_mode[dev];
  return GT_OK;
}

size_t smem_l1_place(int D, int mode, bool records, uint64_t CT, bool compact = false) {
  const int W = kL1Warps, PT = kPlaceTile;
  const size_t in = records ? (size_t)2 * PT * 8 : (size_t)2 * PT * 4 + (size_t)2 * kWinCap * 8;
  return in + (size_t)PT * (compact ? 4 : 8) + (size_t)D * 16 + (size_t)W * D * 4 +
         (mode == kRankSafe ? (size_t)W * D * 4 : 0) + (size_t)D * 8 + 40 * 4 + (CT / PT + 4) * 4 +
         (compact ? (size_t)D * 4 : 0) + 16;
}
size_t smem_b1c(int Db, int mode) {
  const int W = kB1cWarps;
  return (size_t)2 * (kChunkC + 8) * 4 + (size_t)W * Db * 4 + (mode == kRankSafe ? (size_t)W * Db * 4 : 0) +
         (size_t)Db * 8 + 40 * 4 + kMaxBnd * 8 + 16;
}
size_t smem_final_c(int mode) {
  const int W = kFcWarps, ML = kFMaxLocal;
  return (size_t)2 * kFCapC * 4 + (size_t)kSegCapC * 8 + (size_t)(kSegCapC + 4) * 4 + (size_t)W * ML * 4 +
         (mode == kRankSafe ? (size_t)W * ML * 4 : 0) + (size_t)ML * 8 + 40 * 4 + (size_t)ML * 8 + (size_t)ML * 4 +
         (size_t)kMaxRange * 12 + (size_t)kTabCap * 2 + 64;
}
size_t smem_b1(const Plan& p, int mode) {
  const int W = kB1Warps, D = p.Db;
  return (size_t)2 * kChunk * 8 + (size_t)W * D * 4 + (mode == kRankSafe ? (size_t)W * D * 4 : 0) + (size_t)D * 8 +
         40 * 4;
}
size_t smem_final(int mode) {
  const int W = kFWarps;
  return (size_t)2 * kFCap * 8 + (size_t)kSegCap * 8 + (size_t)(kSegCap + 4) * 4 + (size_t)W * kFMaxLocal * 4 +
         (mode == kRankSafe ? (size_t)W * kFMaxLocal * 4 : 0) + (size_t)kFMaxLocal * 8 + 40 * 4 +
         (size_t)kFMaxLocal * 8 + (size_t)kFMaxLocal * 4 + (size_t)kMaxRange * 12 + (size_t)(kFCap + 4) * 4 + 64;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}
template <typename Kern>
unsigned persistent_grid(Kern kernel, int threads, size_t smem, uint64_t work) {
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  if (const char* e = getenv("GT_OCC")) occ = std::max(1, std::min(occ, atoi(e)));  // experiments: CTAs per SM cap
  const uint64_t g = (uint64_t)num_sms() * occ;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, std::max<uint64_t>(work, 1)));
}

// Largest dynamic shared memory a block may opt into on the current device.
size_t max_smem_optin() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 0;
  return (size_t)v;
}

template <typename K>
int set_smem(K kernel, size_t bytes) {
  GT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GT_OK;
}

int scan_u32_to_u64(const uint32_t* in, uint64_t n, uint64_t* out, uint64_t init, bool total,
                    uint64_t* status, unsigned int* ctr, cudaStream_t st) {
  const uint64_t tiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
  GT_CUDA(cudaMemsetAsync(status, 0, tiles * 8, st));
  GT_CUDA(cudaMemsetAsync(ctr, 0, 4, st));
  k_scan_lookback<uint32_t><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, out, init, total ? 1 : 0, status, ctr);
  GT_LAUNCH_CHECK();
  return GT_OK;
}
int scan_u64_to_u64(const unsigned long long* in, uint64_t n, uint64_t* out, uint64_t init, bool total,
                    uint64_t* status, unsigned int* ctr, cudaStream_t st) {
  const uint64_t tiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
  GT_CUDA(cudaMemsetAsync(status, 0, tiles * 8, st));
  GT_CUDA(cudaMemsetAsync(ctr, 0, 4, st));
  k_scan_lookback<unsigned long long><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, out, init, total ? 1 : 0,
                                                                                  status, ctr);
  GT_LAUNCH_CHECK();
  return GT_OK;
}

// CUDA-event timing of a call (stats != NULL): step marks plus begin/end of
// the main kernels.  Events are created once per thread and reused.
// Per-thread, per-device side stream and fork/join events (created once).
int side_stream(cudaStream_t* s, cudaEvent_t* fork, cudaEvent_t* join) {
  thread_local cudaStream_t t_s[64] = {};
  thread_local cudaEvent_t t_f[64] = {}, t_j[64] = {};
  int dev = 0;
  GT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return set_err(GT_ECUDA, "device ordinal %d out of range", dev);
  if (!t_s[dev]) {
    GT_CUDA(cudaStreamCreateWithFlags(&t_s[dev], cudaStreamNonBlocking));
    GT_CUDA(cudaEventCreateWithFlags(&t_f[dev], cudaEventDisableTiming));
    GT_CUDA(cudaEventCreateWithFlags(&t_j[dev], cudaEventDisableTiming));
  }
  *s = t_s[dev];
  *fork = t_f[dev];
  *join = t_j[dev];
  return GT_OK;
}

struct Timer {
  static constexpr int kSteps = 6, kKern = 4;
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t* ev = nullptr;   // kSteps step marks
  cudaEvent_t* kev = nullptr;  // 2 * kKern kernel begin/end
  int n = 0;
  bool kset[kKern] = {};
  int init(bool enable, cudaStream_t s) {
    on = enable;
    st = s;
    if (!on) return GT_OK;
    thread_local cudaEvent_t t_ev[kSteps + 2 * kKern];
    thread_local bool t_init = false;
    thread_local int t_dev = -1;
    int dev = 0;
    GT_CUDA(cudaGetDevice(&dev));
    if (!t_init || t_dev != dev) {
      for (auto& e : t_ev) GT_CUDA(cudaEventCreate(&e));
      t_init = true;
      t_dev = dev;
    }
    ev = t_ev;
    kev = t_ev + kSteps;
    return GT_OK;
  }
  int mark() {
    if (on && n < kSteps) GT_CUDA(cudaEventRecord(ev[n++], st));
    return GT_OK;
  }
  int kbegin(int k, cudaStream_t s = nullptr) {
    if (on) GT_CUDA(cudaEventRecord(kev[2 * k], s ? s : st));
    return GT_OK;
  }
  int kend(int k, cudaStream_t s = nullptr) {
    if (on) {
      GT_CUDA(cudaEventRecord(kev[2 * k + 1], s ? s : st));
      kset[k] = true;
    }
    return GT_OK;
  }
};

// Core pipeline over an input stream `in` of p.E edges whose destinations are
// local IDs in [0, p.V).  Workspace already sized by make_plan.  No host
// synchronisation until the final overflow check.
template <int kMode, class In>
int transpose_core(const Plan& p, In in, uint64_t* t_offsets, uint32_t* t_edges, unsigned char* ws, cudaStream_t st,
                   gt_stats* stats, Timer& tm) {
  const uint64_t V = p.V, E = p.E;
  uint2* rec = reinterpret_cast<uint2*>(ws + p.o_rec);
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(ws + p.o_tcnt);
  uint64_t* tbase = reinterpret_cast<uint64_t*>(ws + p.o_tbase);
  uint32_t* psrc = reinterpret_cast<uint32_t*>(ws + p.o_psrc);
  uint64_t* cstart = reinterpret_cast<uint64_t*>(ws + p.o_cstart);
  uint32_t* cfirst = reinterpret_cast<uint32_t*>(ws + p.o_cfirst);
  uint32_t* cbucket = reinterpret_cast<uint32_t*>(ws + p.o_cbucket);
  uint16_t* segoff = p.b ? reinterpret_cast<uint16_t*>(ws + p.o_segoff) : nullptr;
  uint32_t* fsize = reinterpret_cast<uint32_t*>(ws + p.o_fsize);
  uint64_t* fbase = reinterpret_cast<uint64_t*>(ws + p.o_fbase);
  FRange* ranges = reinterpret_cast<FRange*>(ws + p.o_ranges);
  uint64_t* status = reinterpret_cast<uint64_t*>(ws + p.o_status);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(ws + p.o_ctr);
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + p.o_counters);
  uint32_t* n_ranges = counters;
  unsigned int* range_ctr = counters + 1;
  unsigned int* err = reinterpret_cast<unsigned int*>(ws + p.o_err);
  const DigShift dig1{p.b + p.c};
  int rc;
  int launches = 0;

  GT_CUDA(cudaMemsetAsync(counters, 0, 64, st));
  GT_CUDA(cudaMemsetAsync(err, 0, 4, st));
  if ((rc = tm.mark())) return rc;
  // ---- step 1: level-1 partition (source-ordered pass over the edge stream)
  if constexpr (!In::kRecords) {
    k_tile_src<<<(unsigned)((p.nplace + 1 + 255) / 256), 256, 0, st>>>(in, E, kPlaceTile, p.nplace + 1, psrc);
    GT_LAUNCH_CHECK();
    ++launches;
  }
  k_l1_count<In, DigShift><<<(unsigned)p.ntiles, 512, p.D1 * 4, st>>>(in, dig1, E, p.CT, p.ntiles, p.D1, tcnt);
  GT_LAUNCH_CHECK();
  if ((rc = scan_u32_to_u64(tcnt, (uint64_t)p.D1 * p.ntiles, tbase, 0, true, status, ctr, st))) return rc;
  {
    const size_t sm = smem_l1_place(p.D1, kMode, In::kRecords, p.CT);
    if ((rc = set_smem(k_l1_place<kMode, In, DigShift, OutFull>, sm))) return rc;
    k_l1_place<kMode, In, DigShift, OutFull><<<(unsigned)p.ntiles, kL1Warps * 32, sm, st>>>(
        in, dig1, E, p.CT, p.ntiles, p.D1, tbase, psrc, OutFull{rec});
    GT_LAUNCH_CHECK();
  }
  k_coarse_info<<<1, 1024, (p.D1 + 1) * 4, st>>>(tbase, p.ntiles, p.D1, E, cstart, cfirst, nullptr);
  GT_LAUNCH_CHECK();
  k_chunk_map<<<p.D1, 128, 0, st>>>(cfirst, p.D1, cbucket);
  GT_LAUNCH_CHECK();
  launches += 5;
  if ((rc = tm.mark())) return rc;
  // ---- step 2: level-2 chunk sort by the middle digit (persistent, prefetching)
  if (p.b) {
    const size_t sm = smem_b1(p, kMode);
    if ((rc = set_smem(k_b1<kMode>, sm))) return rc;
    const unsigned grid = persistent_grid(k_b1<kMode>, kB1Warps * 32, sm, p.max_chunks);
    k_b1<kMode><<<grid, kB1Warps * 32, sm, st>>>(rec, cstart, cfirst, cbucket, p.D1, p.c, (uint32_t)(p.Db - 1), p.Db,
                                                  segoff);
    GT_LAUNCH_CHECK();
    ++launches;
  }
  if ((rc = tm.mark())) return rc;
  // ---- step 3: plan, big-bucket counts/cursors, final per-item sort + CSC offsets
  FineCtx fx;
  fx.rec = rec;
  fx.cstart = cstart;
  fx.chunk_first = cfirst;
  fx.segoff = segoff;
  fx.Db = p.Db;
  fx.bits_c = p.c;
  fx.mask_c = (uint32_t)(p.Dc - 1);
  fx.V = V;
  {
    const uint32_t target = (uint32_t)std::min<uint64_t>(
        1u << 20, std::max<uint64_t>(4 * kFCap, E / ((uint64_t)num_sms() * 2 * 6)));
    k_f_plan<<<p.D1, 256, 2 * p.Db * 4, st>>>(fx, target, fsize, fbase, ranges, n_ranges, t_offsets, err);
    GT_LAUNCH_CHECK();
    k_range_sort<<<1, 1024, 0, st>>>(ranges, n_ranges);
    GT_LAUNCH_CHECK();
    const size_t sm = smem_final(kMode);
    if ((rc = set_smem(k_final<kMode>, sm))) return rc;
    const unsigned gf = persistent_grid(k_final<kMode>, kFWarps * 32, sm, (uint64_t)p.D1 * p.Db);
    unsigned long long* prof = nullptr;
    if (getenv("GT_FPROF")) {
      GT_CUDA(cudaMallocAsync(&prof, 10 * 8, st));
      GT_CUDA(cudaMemsetAsync(prof, 0, 10 * 8, st));
    }
    k_final<kMode><<<gf, kFWarps * 32, sm, st>>>(fx, ranges, n_ranges, range_ctr, fsize, fbase, t_offsets, t_edges, err,
                                                 prof);
    GT_LAUNCH_CHECK();
    if (prof) {
      unsigned long long h[10];
      GT_CUDA(cudaMemcpyAsync(h, prof, 80, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "[gt_fprof] grid=%u gen=%.3g issue=%.3g wait=%.3g count=%.3g bases=%.3g rank=%.3g write=%.3g loop=%.3g units0=%llu units12=%llu (cycles summed over CTAs)\n",
              gf, (double)h[0], (double)h[1], (double)h[2], (double)h[3], (double)h[4], (double)h[5], (double)h[6],
              (double)h[9], h[7], h[8]);
      cudaFreeAsync(prof, st);
    }
  }
  k_set_u64<<<1, 1, 0, st>>>(t_offsets + V, E);
  GT_LAUNCH_CHECK();
  launches += 4;
  if ((rc = tm.mark())) return rc;
  uint32_t h_cnt[3] = {0, 0, 0};
  unsigned int h_err = 0;
  GT_CUDA(cudaMemcpyAsync(h_cnt, counters, 12, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  if (stats) {
    stats->n_big_buckets = h_cnt[0];  /* reports the number of final ranges */
    stats->n_launches = launches + 1 /* scan */;
  }
  if (h_err) return set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
  return GT_OK;
}

}  // namespace

namespace {
// Compact (4-byte record) pipeline: L1 -> R1 (with the source-high boundary
// table), level 2 re-encodes to R2 in 16K-record chunks, level 3 per fine unit.
template <int kMode, class In>
int transpose_core_c(const Plan& p, In in, uint64_t* t_offsets, uint32_t* t_edges, unsigned char* ws, cudaStream_t st,
                     gt_stats* stats, Timer& tm) {
  const uint64_t V = p.V, E = p.E;
  uint32_t* rec = reinterpret_cast<uint32_t*>(ws + p.o_rec);
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(ws + p.o_tcnt);
  uint64_t* tbase = reinterpret_cast<uint64_t*>(ws + p.o_tbase);
  uint32_t* psrc = reinterpret_cast<uint32_t*>(ws + p.o_psrc);
  uint64_t* cstart = reinterpret_cast<uint64_t*>(ws + p.o_cstart);
  uint32_t* cfirst = reinterpret_cast<uint32_t*>(ws + p.o_cfirst);
  uint32_t* cbucket = reinterpret_cast<uint32_t*>(ws + p.o_cbucket);
  uint16_t* segoff = reinterpret_cast<uint16_t*>(ws + p.o_segoff);
  uint32_t* fsize = reinterpret_cast<uint32_t*>(ws + p.o_fsize);
  uint64_t* fbase = reinterpret_cast<uint64_t*>(ws + p.o_fbase);
  FRange* ranges = reinterpret_cast<FRange*>(ws + p.o_ranges);
  uint64_t* status = reinterpret_cast<uint64_t*>(ws + p.o_status);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(ws + p.o_ctr);
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + p.o_counters);
  uint32_t* n_ranges = counters;
  unsigned int* range_ctr = counters + 1;
  unsigned int* err = reinterpret_cast<unsigned int*>(ws + p.o_err);
  uint64_t* seghi = reinterpret_cast<uint64_t*>(ws + p.o_seghi);
  uint32_t* prev = reinterpret_cast<uint32_t*>(ws + p.o_prev);
  const DigShift dig1{p.b + p.c};
  const uint32_t nh = 1u << p.nsh;
  int rc;
  int launches = 0;

  GT_CUDA(cudaMemsetAsync(counters, 0, 64, st));
  GT_CUDA(cudaMemsetAsync(err, 0, 4, st));
  GT_CUDA(cudaMemsetAsync(seghi, 0xff, (uint64_t)p.D1 * (nh + 1) * 8, st));
  if ((rc = tm.mark())) return rc;
  if constexpr (!In::kRecords) {
    k_tile_src<<<(unsigned)((p.nplace + 1 + 255) / 256), 256, 0, st>>>(in, E, kPlaceTile, p.nplace + 1, psrc);
    GT_LAUNCH_CHECK();
    k_prev_src<<<(unsigned)((p.ntiles + 255) / 256), 256, 0, st>>>(in, E, p.CT, p.ntiles, prev);
    GT_LAUNCH_CHECK();
    launches += 2;
  }
  k_l1_count<In, DigShift><<<(unsigned)p.ntiles, 512, p.D1 * 4, st>>>(in, dig1, E, p.CT, p.ntiles, p.D1, tcnt);
  GT_LAUNCH_CHECK();
  if ((rc = scan_u32_to_u64(tcnt, (uint64_t)p.D1 * p.ntiles, tbase, 0, true, status, ctr, st))) return rc;
  {
    OutCompact oc;
    oc.rec = rec;
    oc.low_mask = (uint32_t)((1ull << (p.b + p.c)) - 1);
    oc.L = p.L;
    oc.src_mask = (uint32_t)((1ull << p.L) - 1);
    oc.nh = nh;
    oc.seg_hi = seghi;
    oc.prev_src = prev;
    const size_t sm = smem_l1_place(p.D1, kMode, In::kRecords, p.CT, true);
    if ((rc = set_smem(k_l1_place<kMode, In, DigShift, OutCompact>, sm))) return rc;
    k_l1_place<kMode, In, DigShift, OutCompact><<<(unsigned)p.ntiles, kL1Warps * 32, sm, st>>>(
        in, dig1, E, p.CT, p.ntiles, p.D1, tbase, psrc, oc);
    GT_LAUNCH_CHECK();
  }
  k_coarse_info_c<<<1, 1024, (p.D1 + 1) * 4, st>>>(tbase, p.ntiles, p.D1, E, cstart, cfirst);
  GT_LAUNCH_CHECK();
  k_chunk_map<<<p.D1, 128, 0, st>>>(cfirst, p.D1, cbucket);
  GT_LAUNCH_CHECK();
  ChunkInfo* cinfo = reinterpret_cast<ChunkInfo*>(ws + p.o_cinfo);
  k_chunk_info<<<(unsigned)std::min<uint64_t>(4096, (p.max_chunks + 7) / 8), 256, 0, st>>>(cstart, cfirst, p.D1,
                                                                                             cbucket, seghi, nh, cinfo);
  GT_LAUNCH_CHECK();
  launches += 6;
  if ((rc = tm.mark())) return rc;
  {
    DecodeC dc;
    dc.L = p.L;
    dc.src_mask = (uint32_t)((1ull << p.L) - 1);
    dc.nh = nh;
    dc.seg_hi = seghi;
    dc.bits_c = p.c;
    dc.nb = p.nbs;
    dc.gbits = p.gbits;
    const size_t sm = smem_b1c(p.Db, kMode);
    if ((rc = set_smem(k_b1c<kMode>, sm))) return rc;
    const unsigned grid = persistent_grid(k_b1c<kMode>, kB1cWarps * 32, sm, p.max_chunks);
    unsigned long long* bprof = nullptr;
    if (getenv("GT_FPROF")) {
      GT_CUDA(cudaMallocAsync(&bprof, 64, st));
      GT_CUDA(cudaMemsetAsync(bprof, 0, 64, st));
    }
    k_b1c<kMode><<<grid, kB1cWarps * 32, sm, st>>>(rec, rec, cinfo, cfirst, p.D1, dc, p.Db, segoff, bprof);
    GT_LAUNCH_CHECK();
    if (bprof) {
      unsigned long long h[8];
      GT_CUDA(cudaMemcpyAsync(h, bprof, 64, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "[gt_bprof] grid=%u issue=%.3g prep=%.3g wait=%.3g pass1=%.3g bases=%.3g stage=%.3g write=%.3g loop=%.3g\n",
              grid, (double)h[0], (double)h[1], (double)h[2], (double)h[3], (double)h[4], (double)h[5], (double)h[6],
              (double)h[7]);
      cudaFreeAsync(bprof, st);
    }
    ++launches;
  }
  if ((rc = tm.mark())) return rc;
  {
    FineCtx fx{};
    fx.rec = nullptr;
    fx.cstart = cstart;
    fx.chunk_first = cfirst;
    fx.segoff = segoff;
    fx.Db = p.Db;
    fx.bits_c = p.c;
    fx.mask_c = (uint32_t)(p.Dc - 1);
    fx.V = V;
    const uint32_t target = (uint32_t)std::min<uint64_t>(
        1u << 20, std::max<uint64_t>(4 * kFCapC, E / ((uint64_t)num_sms() * 2 * 6)));
    k_f_plan<<<p.D1, 256, 2 * p.Db * 4, st>>>(fx, target, fsize, fbase, ranges, n_ranges, t_offsets, err);
    GT_LAUNCH_CHECK();
    k_range_sort<<<1, 1024, 0, st>>>(ranges, n_ranges);
    GT_LAUNCH_CHECK();
    FineCtxC xc;
    xc.rec = rec;
    xc.cstart = cstart;
    xc.chunk_first = cfirst;
    xc.segoff = segoff;
    xc.Db = p.Db;
    xc.bits_c = p.c;
    xc.nb = p.nbs;
    xc.gbits = p.gbits;
    xc.V = V;
    unsigned long long* prof = nullptr;
    if (getenv("GT_FPROF")) {
      GT_CUDA(cudaMallocAsync(&prof, 14 * 8, st));
      GT_CUDA(cudaMemsetAsync(prof, 0, 14 * 8, st));
    }
    const size_t sm = smem_final_c(kMode);
    if ((rc = set_smem(k_final_c<kMode>, sm))) return rc;
    const unsigned gf = persistent_grid(k_final_c<kMode>, kFcWarps * 32, sm, (uint64_t)p.D1 * p.Db);
    k_final_c<kMode><<<gf, kFcWarps * 32, sm, st>>>(xc, ranges, n_ranges, range_ctr, fsize, fbase, t_offsets, t_edges,
                                                    prof);
    GT_LAUNCH_CHECK();
    if (prof) {
      unsigned long long h[14];
      GT_CUDA(cudaMemcpyAsync(h, prof, 14 * 8, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr,
              "[gt_fprof-c] grid=%u gen=%.3g issue=%.3g (table=%.3g copy=%.3g) wait=%.3g count=%.3g bases=%.3g "
              "rank=%.3g write=%.3g (bigcount=%.3g) loop=%.3g units0=%llu units12=%llu cta_max=%.3g\n",
              gf, (double)h[0], (double)h[1], (double)h[10], (double)h[11], (double)h[2], (double)h[3], (double)h[4],
              (double)h[5], (double)h[6], (double)h[12], (double)h[9], h[7], h[8], (double)h[13]);
      cudaFreeAsync(prof, st);
    }
  }
  k_set_u64<<<1, 1, 0, st>>>(t_offsets + V, E);
  GT_LAUNCH_CHECK();
  launches += 4;
  if ((rc = tm.mark())) return rc;
  uint32_t h_cnt[3] = {0, 0, 0};
  unsigned int h_err = 0;
  GT_CUDA(cudaMemcpyAsync(h_cnt, counters, 12, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  if (stats) {
    stats->n_big_buckets = h_cnt[0];
    stats->n_launches = launches + 1;
  }
  if (h_err) return set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
  return GT_OK;
}

// ---------------------------------------------------------------- v3 path
// Workspace layout of the lean pipeline (gt_v3.cuh).  R1 lives in t_edges.
struct Plan3 {
  uint64_t ntiles1 = 0, nplace = 0, nh = 0, max_t2 = 0, nfine = 0, max_big = 0, max_t3 = 0;
  uint64_t o_r2, o_tcnt, o_tbase, o_status, o_ctr, o_psrc, o_prev, o_seghi, o_cstart, o_cfirst, o_tiles2, o_cnt2,
      o_base2, o_seg2, o_fbase, o_units, o_bigs, o_tiles3, o_cnt3, o_base3, o_seg3, o_cnt, o_err, o_bnt, o_bfirst,
      o_r2lv, total;
};

bool v3_capable(uint64_t E) { return E < (1ull << 32) && getenv("GT_V2") == nullptr; }
bool use_v3(const Plan& p) { return p.wide || (p.compact && v3_capable(p.E)); }

void make_plan3(const Plan& p, Plan3& q) {
  const uint64_t E = p.E;
  q.ntiles1 = (E + v3::CT1 - 1) / v3::CT1;
  q.nplace = (E + v3::PT - 1) / v3::PT;
  q.nh = 1ull << p.nsh;
  q.max_t2 = (E + v3::CT2 - 1) / v3::CT2 + (uint64_t)p.D1;
  q.nfine = (uint64_t)p.D1 * p.Db;
  q.max_big = std::min<uint64_t>(q.nfine, E / v3::CAP3 + 1);
  q.max_t3 = (E + v3::CT2 - 1) / v3::CT2 + q.max_big;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o = off;
    off = align_up(off + std::max<uint64_t>(bytes, 1), 256);
    return o;
  };
  const uint64_t n1 = (uint64_t)p.D1 * q.ntiles1;
  q.o_r2 = take(E * 4 + 64);
  q.o_r2lv = take(p.wide ? E + 64 : 0);  // wide: low digit of every R2 record (+ padding for 16-byte block loads)
  q.o_tcnt = take(n1 * 4);
  q.o_tbase = take((n1 + 1) * 8);
  const uint64_t nscan = std::max<uint64_t>(n1 + 1, std::max<uint64_t>(q.max_t2 * (uint64_t)p.Db,
                                                                        q.max_t3 * (uint64_t)p.Dc));
  q.o_status = take(((nscan + kScanTile - 1) / kScanTile + 1) * 8);
  q.o_ctr = take(64);
  q.o_psrc = take((q.nplace + 2) * 4);
  q.o_prev = take((q.ntiles1 + 1) * 4);
  q.o_seghi = take((uint64_t)p.D1 * (q.nh + 1) * 8);
  q.o_cstart = take((uint64_t)(p.D1 + 1) * 8);
  q.o_cfirst = take((uint64_t)(p.D1 + 1) * 4);
  q.o_tiles2 = take(q.max_t2 * sizeof(v3::RTile));
  q.o_cnt2 = take(q.max_t2 * (uint64_t)p.Db * 4);
  q.o_base2 = take(q.max_t2 * (uint64_t)p.Db * 8);
  q.o_seg2 = take((uint64_t)p.D1 * sizeof(v3::SegDesc));
  q.o_fbase = take((q.nfine + 1) * 8);
  q.o_units = take(q.nfine * sizeof(v3::Unit3));
  q.o_bigs = take(q.max_big * sizeof(v3::Big3));
  q.o_tiles3 = take(q.max_t3 * sizeof(v3::RTile));
  q.o_cnt3 = take(q.max_t3 * (uint64_t)p.Dc * 4);
  q.o_base3 = take(q.max_t3 * (uint64_t)p.Dc * 8);
  q.o_seg3 = take(q.max_big * sizeof(v3::SegDesc));
  q.o_cnt = take(64);
  q.o_err = take(4);
  q.o_bnt = take((q.max_big + 1) * 4);
  q.o_bfirst = take((q.max_big + 2) * 8);
  q.total = off;
}

__global__ void k_set_u32(uint32_t* p, uint32_t v) { *p = v; }
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int kMode>
int transpose_v3(const Plan& p, InCsr in, uint64_t* t_offsets, uint32_t* t_edges, unsigned char* ws, cudaStream_t st,
                 gt_stats* stats, Timer& tm) {
  using namespace v3;
  Plan3 q;
  make_plan3(p, q);
  const uint64_t V = p.V, E = p.E;
  const int D1 = p.D1, Db = p.Db, Dc = p.Dc;
  uint32_t* r2 = reinterpret_cast<uint32_t*>(ws + q.o_r2);
  uint8_t* r2lv = p.wide ? reinterpret_cast<uint8_t*>(ws + q.o_r2lv) : nullptr;  // wide: R2 low digits
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(ws + q.o_tcnt);
  uint64_t* tbase = reinterpret_cast<uint64_t*>(ws + q.o_tbase);
  uint64_t* status = reinterpret_cast<uint64_t*>(ws + q.o_status);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(ws + q.o_ctr);
  uint32_t* psrc = reinterpret_cast<uint32_t*>(ws + q.o_psrc);
  uint32_t* prev = reinterpret_cast<uint32_t*>(ws + q.o_prev);
  uint64_t* seghi = reinterpret_cast<uint64_t*>(ws + q.o_seghi);
  uint64_t* cstart = reinterpret_cast<uint64_t*>(ws + q.o_cstart);
  uint32_t* cfirst = reinterpret_cast<uint32_t*>(ws + q.o_cfirst);
  RTile* tiles2 = reinterpret_cast<RTile*>(ws + q.o_tiles2);
  uint32_t* cnt2 = reinterpret_cast<uint32_t*>(ws + q.o_cnt2);
  uint64_t* base2 = reinterpret_cast<uint64_t*>(ws + q.o_base2);
  SegDesc* seg2 = reinterpret_cast<SegDesc*>(ws + q.o_seg2);
  uint64_t* fbase = reinterpret_cast<uint64_t*>(ws + q.o_fbase);
  Unit3* units = reinterpret_cast<Unit3*>(ws + q.o_units);
  Big3* bigs = reinterpret_cast<Big3*>(ws + q.o_bigs);
  RTile* tiles3 = reinterpret_cast<RTile*>(ws + q.o_tiles3);
  uint32_t* cnt3 = reinterpret_cast<uint32_t*>(ws + q.o_cnt3);
  uint64_t* base3 = reinterpret_cast<uint64_t*>(ws + q.o_base3);
  SegDesc* seg3 = reinterpret_cast<SegDesc*>(ws + q.o_seg3);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + q.o_cnt);  // [0] units [1] big [2] tiles3 [3] unit ctr [4] D1
  unsigned int* err = reinterpret_cast<unsigned int*>(ws + q.o_err);
  const uint32_t nh = (uint32_t)q.nh;
  int rc;
  int launches = 0;
  const int sms = num_sms();
  // batched shared loads in the place kernels (bits: 2 L2, 4 L3 big buckets, 8 L3 units, 16 L3 units
  // with position-derived fine buckets).  Measured (C3 / C4): L3 big 0.85 -> 0.78 ms; L3 position units
  // (C4) 4.40 -> 4.33 ms; slower for L2 with 4096-record tiles (2.11 -> 2.18 ms) and C3's L3 units
  const int pre = env_int("GT_PRE", 4 | 16);
  // level-3 units are aligned groups of 2^sbits fine buckets (<= ML3 local
  // vertices); R2 carries g3 = sbits fine-digit bits when it has room, else
  // the unit decodes the fine bucket from the record's position
  auto log2_groups = [&](int ml) {
    int b = 0;
    while ((ml >> p.c) >> (b + 1)) ++b;
    return b;
  };
  const bool pos_fine = p.wide || p.gbits < log2_groups(256);   // R2 cannot name 256 / 2^c fine buckets
  const int sbits = pos_fine ? log2_groups(ML3) : log2_groups(256);
  const int g3 = pos_fine ? 0 : sbits;

  GT_CUDA(cudaMemsetAsync(cnt, 0, 64, st));
  GT_CUDA(cudaMemsetAsync(err, 0, 4, st));
  GT_CUDA(cudaMemsetAsync(seghi, 0xff, (uint64_t)D1 * (nh + 1) * 8, st));
  k_set_u32<<<1, 1, 0, st>>>(cnt + 4, (uint32_t)D1);
  GT_LAUNCH_CHECK();
  if ((rc = tm.mark())) return rc;
  // ---- step 1: level-1 partition of the CSR stream into R1 (in t_edges)
  // level 1 uses 8192-edge place tiles (measured: C3 k_p1 2.82 -> 2.79 ms, C4 8.75 -> 7.56 ms)
  // (wide graphs: 4096-edge tiles keep 2 CTAs/SM with 2048 coarse digits)
  const int k1 = env_int("GT_K1", 32);  // C5 (wide, 2048 coarse digits): 8192-edge tiles 90.0 -> 81.8 ms
  // warps per level-1 CTA: compact graphs 16 = 8192-edge tiles at K = 16; wide graphs 16 = 16384-edge tiles at K = 32
  // (GT_W1 = 32: compact graphs with 16384-edge tiles, 16 warps at K = 32)
  // wide graphs (C5): 16384-edge tiles 81.8 -> 58.0 ms
  // (the 16-warp forms need their larger tables to fit: the safe rank mode's scratch table may not)
  // compact graphs with <= 512 coarse digits: 16 warps x K = 16 (C3 k_p1 2.70 -> 2.64 ms; C4, 1024 digits: slower)
  int w1x = p.wide ? (env_int("GT_W1W", 16) == 16 ? 32 : W) : env_int("GT_W1", D1 <= 512 ? 16 : W);
  if (w1x == 32 && smem_p1(D1, kMode, 32, 16) + 64 > max_smem_optin()) w1x = W;
  if (w1x == 16 && smem_p1(D1, kMode, 16, 16) + 64 > max_smem_optin()) w1x = W;
  const int w1 = w1x == 32 ? 16 : w1x;
  const uint64_t pt1 = (uint64_t)w1 * ((w1x == 16) ? 16 : k1) * 32, nplace1 = (E + pt1 - 1) / pt1;
  k_tile_src<<<(unsigned)((nplace1 + 1 + 255) / 256), 256, 0, st>>>(in, E, pt1, nplace1 + 1, psrc);
  GT_LAUNCH_CHECK();
  k_prev_src<<<(unsigned)((q.ntiles1 + 255) / 256), 256, 0, st>>>(in, E, CT1, q.ntiles1, prev);
  GT_LAUNCH_CHECK();
  if ((rc = set_smem(k_c1, (size_t)G1 * D1 * 4))) return rc;
  k_c1<<<(unsigned)((q.ntiles1 + G1 - 1) / G1), 512, (size_t)G1 * D1 * 4, st>>>(in.edges, E, q.ntiles1, D1,
                                                                                p.b + p.c, tcnt);
  GT_LAUNCH_CHECK();
  if ((rc = scan_u32_to_u64(tcnt, (uint64_t)D1 * q.ntiles1, tbase, 0, true, status, ctr, st))) return rc;
  {
    P1Args a;
    a.offsets = in.offsets;
    a.edges = in.edges;
    a.e_begin = in.e_begin;
    a.V = in.V;  // source IDs (differ from destinations on the multi-GPU receiver)
    a.E = E;
    a.ntiles = q.ntiles1;
    a.D = D1;
    a.shift = p.b + p.c;
    a.L = p.L;
    a.low_mask = (uint32_t)((1ull << (p.b + p.c)) - 1);
    a.src_mask = (uint32_t)((1ull << p.L) - 1);
    a.tbase = tbase;
    a.psrc = psrc;
    a.prev_src = prev;
    a.nh = nh;
    a.seg_hi = seghi;
    a.out = t_edges;
    if ((rc = tm.kbegin(0))) return rc;
    auto go1 = [&](auto kern, int kk) -> int {
      const size_t sm = smem_p1(D1, kMode, kk);
      int r;
      if ((r = set_smem(kern, sm))) return r;
      kern<<<(unsigned)q.ntiles1, T, sm, st>>>(a);
      return GT_OK;
    };
    if (!p.wide && w1x == 32) {
      const size_t sm = smem_p1(D1, kMode, 32, 16);
      if ((rc = set_smem(k_p1<kMode, 32, false, 16, 1>, sm))) return rc;
      k_p1<kMode, 32, false, 16, 1><<<(unsigned)q.ntiles1, 512, sm, st>>>(a);
    } else if (p.wide && w1 == 16) {  // 16384-edge tiles, one 16-warp CTA per SM
      const size_t sm = smem_p1(D1, kMode, 32, 16);
      if ((rc = set_smem(k_p1<kMode, 32, true, 16, 1>, sm))) return rc;
      k_p1<kMode, 32, true, 16, 1><<<(unsigned)q.ntiles1, 512, sm, st>>>(a);
    } else if (p.wide) {  // 64-bit R1 positions
      if ((rc = (k1 == 32) ? go1(k_p1<kMode, 32, true>, 32) : go1(k_p1<kMode, 16, true>, 16))) return rc;
    } else if (w1 == 16) {
      const size_t sm = smem_p1(D1, kMode, 16, 16);
      if ((rc = set_smem(k_p1<kMode, 16, false, 16>, sm))) return rc;
      k_p1<kMode, 16, false, 16><<<(unsigned)q.ntiles1, 512, sm, st>>>(a);
    } else if (k1 == 32) {
      const size_t sm = smem_p1(D1, kMode, 32);
      if ((rc = set_smem(k_p1<kMode, 32>, sm))) return rc;
      k_p1<kMode, 32><<<(unsigned)q.ntiles1, T, sm, st>>>(a);
    } else {
      const size_t sm = smem_p1(D1, kMode, 16);
      if ((rc = set_smem(k_p1<kMode, 16>, sm))) return rc;
      k_p1<kMode, 16><<<(unsigned)q.ntiles1, T, sm, st>>>(a);
    }
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(0))) return rc;
  }
  launches += 6;
  if ((rc = tm.mark())) return rc;
  // ---- step 2: level 2 (count, per-bucket column scan, place fine-bucket-major into R2)
  k_coarse_tiles<<<1, 1024, (size_t)(D1 + 1) * 4, st>>>(tbase, q.ntiles1, D1, E, cstart, cfirst);
  GT_LAUNCH_CHECK();
  k_l2_tiles<<<D1, 128, 0, st>>>(cstart, cfirst, Db, seghi, nh, tiles2, seg2);
  GT_LAUNCH_CHECK();
  const unsigned gt2 = (unsigned)std::min<uint64_t>(q.max_t2, (uint64_t)sms * 8);
  GT_CUDA(cudaMemsetAsync(cnt2, 0, q.max_t2 * (uint64_t)Db * 4, st));  // the scan covers the unused tail too
  k_cnt_rec<<<gt2, 512, (size_t)Db * 4, st>>>(t_edges, tiles2, cfirst + D1, Db, DigSM{p.L + p.c, (uint32_t)(Db - 1)},
                                              cnt2);
  GT_LAUNCH_CHECK();
  // bases of every (chunk, fine digit): one device-wide exclusive scan of the
  // per-bucket digit-major count tables (concatenated in bucket order, so the
  // scan value already includes the bucket start), then the fine-bucket starts
  if (env_int("GT_SEGSCAN", 0)) {
    k_segscan<<<(unsigned)D1, 512, (size_t)Db * 8, st>>>(seg2, cnt + 4, Db, cnt2, base2, fbase, q.nfine, err);
    GT_LAUNCH_CHECK();
  } else {
    if ((rc = scan_u32_to_u64(cnt2, (uint64_t)q.max_t2 * Db, base2, 0, false, status, ctr, st))) return rc;
    k_segfix<<<(unsigned)D1, 512, 0, st>>>(seg2, cnt + 4, Db, base2, fbase, q.nfine, err);
    GT_LAUNCH_CHECK();
  }
  {
    DecR1 dec;
    dec.L = p.L;
    dec.src_mask = (uint32_t)((1ull << p.L) - 1);
    dec.shB = p.L + p.c;
    dec.maskB = (uint32_t)(Db - 1);
    dec.lvmask = (uint32_t)((1ull << (p.c + g3)) - 1);  // R2: low digit + g3 fine-digit bits (0: L3 uses positions)
    dec.nbs = p.nbs;
    dec.nh = nh;
    dec.seg_hi = seghi;
    if ((rc = tm.kbegin(1))) return rc;
    const int k2 = env_int("GT_K2", Db >= 1024 ? 32 : 16);
    if (p.wide) {  // R2 = source array + low-digit bytes, 64-bit positions
      auto go2 = [&](auto kern, int kk) -> int {
        const size_t sm = smem_p2(Db, kMode, kk, kIoSplit);
        int r;
        if ((r = set_smem(kern, sm))) return r;
        const unsigned g = persistent_grid(kern, T, sm, q.max_t2);
        kern<<<g, T, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2, nullptr, nullptr, r2lv);
        return GT_OK;
      };
      if (env_int("GT_W2W", 16) == 16 && smem_p2(Db, kMode, 32, kIoSplit, 16) + 64 <= max_smem_optin()) {  // 16384-record tiles, one 16-warp CTA per SM (C5: 88.4 -> 65.9 ms)
        const size_t sm = smem_p2(Db, kMode, 32, kIoSplit, 16);
        using K16 = decltype(&k_p2<kMode, DecR1, 32, false, kIoSplit, true, 16, 1>);
        K16 kern = k_p2<kMode, DecR1, 32, false, kIoSplit, true, 16, 1>;
        if ((rc = set_smem(kern, sm))) return rc;
        const unsigned g = persistent_grid(kern, 512, sm, q.max_t2);
        kern<<<g, 512, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2, nullptr, nullptr, r2lv);
      } else if ((rc = (k2 == 32) ? go2(k_p2<kMode, DecR1, 32, false, kIoSplit>, 32)
                                  : go2(k_p2<kMode, DecR1, 16, false, kIoSplit>, 16))) {
        return rc;
      }
    } else if (k2 == 32 && env_int("GT_W2", 8) == 16 && smem_p2(Db, kMode, 32, kIoPlain, 16) + 64 <= max_smem_optin()) {
      const size_t sm = smem_p2(Db, kMode, 32, kIoPlain, 16);
      if ((rc = set_smem(k_p2<kMode, DecR1, 32, false, kIoPlain, true, 16, 1>, sm))) return rc;
      const unsigned g = persistent_grid(k_p2<kMode, DecR1, 32, false, kIoPlain, true, 16, 1>, 512, sm, q.max_t2);
      k_p2<kMode, DecR1, 32, false, kIoPlain, true, 16, 1><<<g, 512, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2);
    } else if (k2 == 32) {
      const size_t sm = smem_p2(Db, kMode, 32);
      if ((rc = set_smem(k_p2<kMode, DecR1, 32>, sm))) return rc;
      const unsigned g = persistent_grid(k_p2<kMode, DecR1, 32>, T, sm, q.max_t2);
      k_p2<kMode, DecR1, 32><<<g, T, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2);
    } else {
      const size_t sm = smem_p2(Db, kMode, 16);
      if ((rc = set_smem(k_p2<kMode, DecR1, 16>, sm))) return rc;
      const unsigned g = persistent_grid(k_p2<kMode, DecR1, 16>, T, sm, q.max_t2);
      unsigned long long* prof = nullptr;
      if (getenv("GT_PROF2")) {
        GT_CUDA(cudaMallocAsync(&prof, 64, st));
        GT_CUDA(cudaMemsetAsync(prof, 0, 64, st));
      }
      if (prof) {
        if ((rc = set_smem(k_p2<kMode, DecR1, 16, true>, sm))) return rc;
        k_p2<kMode, DecR1, 16, true><<<g, T, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2, prof);
      } else if (pre & 2) {
        k_p2<kMode, DecR1, 16><<<g, T, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2);
      } else {
        if ((rc = set_smem(k_p2<kMode, DecR1, 16, false, kIoPlain, false>, sm))) return rc;
        k_p2<kMode, DecR1, 16, false, kIoPlain, false><<<g, T, sm, st>>>(t_edges, tiles2, cfirst + D1, Db, dec, base2, r2);
      }
      if (prof) {
        unsigned long long h[6];
        GT_CUDA(cudaMemcpyAsync(h, prof, 48, cudaMemcpyDeviceToHost, st));
        GT_CUDA(cudaStreamSynchronize(st));
        double tot = 0;
        for (int i = 0; i < 6; ++i) tot += (double)h[i];
        fprintf(stderr, "[gt_prof2] grid=%u setup=%.3f wait=%.3f rank=%.3f bases=%.3f stage=%.3f write=%.3f (fractions of %.3g CTA-cycles)\n",
                g, h[0] / tot, h[1] / tot, h[2] / tot, h[3] / tot, h[4] / tot, h[5] / tot, tot);
        cudaFreeAsync(prof, st);
      }
    }
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(1))) return rc;
  }
  launches += 6;  // coarse tiles, l2 tiles, count, scan, segfix, place
  if ((rc = tm.mark())) return rc;
  // ---- step 3: level 3 (units of small fine buckets; tiled count/scan/place for big ones)
  k_set_u64<<<1, 1, 0, st>>>(fbase + q.nfine, E);
  GT_LAUNCH_CHECK();
  // level-3 unit width: 16 warps (8192-record units, 2 CTAs/SM) or 32 warps (16384-record units, 1 CTA/SM)
  const int w3 = (env_int("GT_W3", 16) == 32 && smem_p3(kMode, p.wide, 32) + 64 <= max_smem_optin()) ? 32 : 16;
  k_plan3<<<(unsigned)((q.nfine / (1u << sbits) + 255) / 256 + 1), 256, 0, st>>>(fbase, (uint32_t)q.nfine, sbits,
                                                                                   units, cnt + 0, bigs, cnt + 1,
                                                                                   (uint32_t)(w3 * K3 * 32));
  GT_LAUNCH_CHECK();
  // the big-bucket chain (count / scans / place of fine buckets above the unit
  // capacity) runs on a side stream, concurrently with the level-3 units:
  // they touch disjoint fine buckets; its short scans overlap the units kernel
  cudaStream_t sb = st;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (env_int("GT_FORK", 1)) {
    if ((rc = side_stream(&sb, &ev_fork, &ev_join))) return rc;
    GT_CUDA(cudaEventRecord(ev_fork, st));
    GT_CUDA(cudaStreamWaitEvent(sb, ev_fork, 0));
  }
  {
    uint32_t* bnt = reinterpret_cast<uint32_t*>(ws + q.o_bnt);
    uint64_t* bfirst = reinterpret_cast<uint64_t*>(ws + q.o_bfirst);
    const unsigned gb = (unsigned)std::min<uint64_t>((q.max_big + 255) / 256, (uint64_t)sms * 4);
    // exclusive scan over the real buckets (device count) -> bfirst[0..n_big]
    const uint64_t tiles = std::max<uint64_t>(1, (q.max_big + 1 + kScanTile - 1) / kScanTile);
    GT_CUDA(cudaMemsetAsync(status, 0, tiles * 8, sb));
    GT_CUDA(cudaMemsetAsync(ctr, 0, 4, sb));
    GT_CUDA(cudaMemsetAsync(bnt, 0, (q.max_big + 1) * 4, sb));
    k_big_nt<<<gb, 256, 0, sb>>>(bigs, cnt + 1, bnt);
    k_scan_lookback<uint32_t><<<(unsigned)tiles, kScanThreads, 0, sb>>>(bnt, q.max_big + 1, bfirst, 0, 1, status, ctr,
                                                                         cnt + 1, 1);
    GT_LAUNCH_CHECK();
    k_big_write<<<gb, 256, 0, sb>>>(bigs, cnt + 1, bfirst, p.c, tiles3, cnt + 2, seg3);
    GT_LAUNCH_CHECK();
  }
  {
    const unsigned gt3 = (unsigned)std::min<uint64_t>(q.max_t3, (uint64_t)sms * 8);
    if (p.wide) k_cnt_lv<<<gt3, 512, (size_t)Dc * 4, sb>>>(r2lv, tiles3, cnt + 2, Dc, cnt3);
    else k_cnt_rec<<<gt3, 512, (size_t)Dc * 4, sb>>>(r2, tiles3, cnt + 2, Dc, DigSM{p.nbs, (uint32_t)(Dc - 1)}, cnt3);
    GT_LAUNCH_CHECK();
    {  // scan only the real tiles' rows: n = n_tiles3 * Dc (device count)
      const uint64_t n3 = q.max_t3 * (uint64_t)Dc;
      const uint64_t tiles = std::max<uint64_t>(1, (n3 + kScanTile - 1) / kScanTile);
      GT_CUDA(cudaMemsetAsync(status, 0, tiles * 8, sb));
      GT_CUDA(cudaMemsetAsync(ctr, 0, 4, sb));
      k_scan_lookback<uint32_t><<<(unsigned)tiles, kScanThreads, 0, sb>>>(cnt3, n3, base3, 0, 0, status, ctr, cnt + 2,
                                                                           (uint64_t)Dc);
      GT_LAUNCH_CHECK();
    }
    k_segfix<<<(unsigned)std::min<uint64_t>(q.max_big, (uint64_t)sms * 8), 512, 0, sb>>>(seg3, cnt + 1, Dc, base3,
                                                                                      t_offsets, V, err);
    GT_LAUNCH_CHECK();
    DecR2 dec;
    dec.nbs = p.nbs;
    dec.src_mask = (p.nbs >= 32 || p.wide) ? 0xffffffffu : (uint32_t)((1ull << p.nbs) - 1);
    dec.maskC = (uint32_t)(Dc - 1);
    if ((rc = tm.kbegin(3, sb))) return rc;
    if (p.wide) {
      const size_t sm = smem_p2(Dc, kMode, 16, kIoLv);
      if ((rc = set_smem(k_p2<kMode, DecR2, 16, false, kIoLv>, sm))) return rc;
      const unsigned g = persistent_grid(k_p2<kMode, DecR2, 16, false, kIoLv>, T, sm, q.max_t3);
      k_p2<kMode, DecR2, 16, false, kIoLv><<<g, T, sm, sb>>>(r2, tiles3, cnt + 2, Dc, dec, base3, t_edges, nullptr,
                                                              r2lv, nullptr);
    } else {
      const size_t sm = smem_p2(Dc, kMode, 16);
      if ((rc = set_smem(k_p2<kMode, DecR2, 16>, sm))) return rc;
      const unsigned g = persistent_grid(k_p2<kMode, DecR2, 16>, T, sm, q.max_t3);
      if (pre & 4) {
        k_p2<kMode, DecR2, 16><<<g, T, sm, sb>>>(r2, tiles3, cnt + 2, Dc, dec, base3, t_edges);
      } else {
        if ((rc = set_smem(k_p2<kMode, DecR2, 16, false, kIoPlain, false>, sm))) return rc;
        k_p2<kMode, DecR2, 16, false, kIoPlain, false><<<g, T, sm, sb>>>(r2, tiles3, cnt + 2, Dc, dec, base3, t_edges);
      }
    }
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(3, sb))) return rc;
  }
  {
    P3Args a;
    a.rec = r2;
    a.units = units;
    a.n_units = cnt + 0;
    a.ctr = cnt + 3;
    a.c = p.c;
    a.nbs = p.nbs;
    a.src_mask = (p.nbs >= 32 || p.wide) ? 0xffffffffu : (uint32_t)((1ull << p.nbs) - 1);
    a.mask_c = (uint32_t)(Dc - 1);
    a.lv = r2lv;
    a.fbase = fbase;
    a.gbits = g3;
    a.lvmask = (uint32_t)((1ull << (p.c + g3)) - 1);
    a.V = V;
    a.t_offsets = t_offsets;
    a.t_edges = t_edges;
    const size_t sm = smem_p3(kMode, p.wide, w3);
    auto go3 = [&](auto kern) -> int {
      int r;
      if ((r = set_smem(kern, sm))) return r;
      const unsigned g = persistent_grid(kern, w3 * 32, sm, q.nfine);
      kern<<<g, w3 * 32, sm, st>>>(a);
      return GT_OK;
    };
    if ((rc = tm.kbegin(2))) return rc;
    a.prof = nullptr;
    if (getenv("GT_PROF3") && !p.wide) {
      GT_CUDA(cudaMallocAsync(&a.prof, 64, st));
      GT_CUDA(cudaMemsetAsync(a.prof, 0, 64, st));
      rc = pos_fine ? go3(k_p3<kMode, true, true>) : go3(k_p3<kMode, false, true>);
      unsigned long long h[6];
      GT_CUDA(cudaMemcpyAsync(h, a.prof, 48, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      double tot = 0;
      for (int i = 0; i < 6; ++i) tot += (double)h[i];
      fprintf(stderr, "[gt_prof3] fetch=%.3f wait=%.3f rank=%.3f bases=%.3f stage=%.3f store=%.3f (of %.3g CTA-cycles)\n",
              h[0] / tot, h[1] / tot, h[2] / tot, h[3] / tot, h[4] / tot, h[5] / tot, tot);
      cudaFreeAsync(a.prof, st);
    } else if (p.wide) {
      rc = (w3 == 32) ? go3(k_p3<kMode, true, false, true, true, 32>) : go3(k_p3<kMode, true, false, true>);
    } else if (w3 == 32) {
      if ((pre & 8) || ((pre & 16) && pos_fine))
        rc = pos_fine ? go3(k_p3<kMode, true, false, false, true, 32>) : go3(k_p3<kMode, false, false, false, true, 32>);
      else
        rc = pos_fine ? go3(k_p3<kMode, true, false, false, false, 32>) : go3(k_p3<kMode, false, false, false, false, 32>);
    } else if (env_int("GT_BAL3", 1) == 0) {  // A/B: fixed 512 positions per warp
      if ((pre & 8) || ((pre & 16) && pos_fine))
        rc = pos_fine ? go3(k_p3<kMode, true, false, false, true, W3, false>) : go3(k_p3<kMode, false, false, false, true, W3, false>);
      else
        rc = pos_fine ? go3(k_p3<kMode, true, false, false, false, W3, false>) : go3(k_p3<kMode, false, false, false, false, W3, false>);
    } else {
      if ((pre & 8) || ((pre & 16) && pos_fine)) rc = pos_fine ? go3(k_p3<kMode, true>) : go3(k_p3<kMode, false>);
      else rc = pos_fine ? go3(k_p3<kMode, true, false, false, false>) : go3(k_p3<kMode, false, false, false, false>);
    }
    if (rc) return rc;
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(2))) return rc;
  }
  if (sb != st) {
    GT_CUDA(cudaEventRecord(ev_join, sb));
    GT_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  }
  k_set_u64<<<1, 1, 0, st>>>(t_offsets + V, E);
  GT_LAUNCH_CHECK();
  launches += 10;  // set, plan, big nt / scan / write, count, scan, segfix, big place, units (+ the final set below)
  if ((rc = tm.mark())) return rc;
  uint32_t h_cnt[3] = {0, 0, 0};
  unsigned int h_err = 0;
  GT_CUDA(cudaMemcpyAsync(h_cnt, cnt, 12, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  if (stats) {
    stats->n_big_buckets = h_cnt[1];
    stats->n_launches = launches + 1;
  }
  if (h_err) return set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
  return GT_OK;
}

template <int kMode, class In>
int transpose_any(const Plan& p, In in, uint64_t* t_offsets, uint32_t* t_edges, unsigned char* ws, cudaStream_t st,
                  gt_stats* stats, Timer& tm) {
  if constexpr (!In::kRecords) {
    if (use_v3(p)) return transpose_v3<kMode>(p, in, t_offsets, t_edges, ws, st, stats, tm);
  }
  if (p.compact) return transpose_core_c<kMode, In>(p, in, t_offsets, t_edges, ws, st, stats, tm);
  return transpose_core<kMode, In>(p, in, t_offsets, t_edges, ws, st, stats, tm);
}

uint64_t workspace_bytes(const Plan& p, bool records) {
  if (!records && use_v3(p)) {
    Plan3 q;
    make_plan3(p, q);
    return q.total;
  }
  return p.total;
}

int fill_stats(const Plan& p, int mode, Timer& tm, gt_stats* stats) {
  const uint64_t big = stats->n_big_buckets, launches = stats->n_launches;
  float a = 0, b = 0, c = 0, t = 0;
  GT_CUDA(cudaEventElapsedTime(&a, tm.ev[0], tm.ev[1]));
  GT_CUDA(cudaEventElapsedTime(&b, tm.ev[1], tm.ev[2]));
  GT_CUDA(cudaEventElapsedTime(&c, tm.ev[2], tm.ev[3]));
  GT_CUDA(cudaEventElapsedTime(&t, tm.ev[0], tm.ev[3]));
  stats->ms_step1 = a;
  stats->ms_step2 = b;
  stats->ms_step3 = c;
  stats->ms_total = t;
  stats->workspace_bytes = p.total;
  stats->bits[0] = p.a;
  stats->bits[1] = p.b;
  stats->bits[2] = p.c;
  stats->rank_mode = mode;
  stats->n_big_buckets = big;
  stats->n_launches = launches;
  for (int k = 0; k < Timer::kKern; ++k) {
    float x = 0;
    if (tm.kset[k]) GT_CUDA(cudaEventElapsedTime(&x, tm.kev[2 * k], tm.kev[2 * k + 1]));
    stats->ms_kernel[k] = x;
  }
  return GT_OK;
}

}  // namespace

extern "C" {

int gt_abi_version(void) { return GT_ABI_VERSION; }
const char* gt_last_error(void) { return g_err.c_str(); }

int gt_workspace_size(uint64_t V, uint64_t E, uint64_t* bytes) {
  if (!bytes) return set_err(GT_EINVAL, "bytes is NULL");
  if (E == 0 || V == 0) {
    *bytes = 0;
    return GT_OK;
  }
  Plan p;
  int rc = make_plan(V, E, p, 0, v3_capable(E));
  if (rc) return rc;
  *bytes = workspace_bytes(p, false);
  return GT_OK;
}

int gt_set_rank_mode(int mode) {
  if (mode < -1 || mode > 1) return set_err(GT_EINVAL, "rank mode must be -1, 0 or 1");
  g_forced_rank_mode = mode;
  return GT_OK;
}

int gt_selftest_rank_order(uint64_t trials, uint64_t* violations) {
  if (!violations) return set_err(GT_EINVAL, "violations is NULL");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  return run_selftest(trials, violations, nullptr);
}

int gt_transpose(const uint64_t* offsets, const uint32_t* edges, uint64_t V, uint64_t E, uint64_t* t_offsets,
                 uint32_t* t_edges, void* workspace, uint64_t ws_bytes, void* stream, gt_stats* stats) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (!t_offsets) return set_err(GT_EINVAL, "t_offsets is NULL");
  if (E && (!offsets || !edges || !t_edges)) return set_err(GT_EINVAL, "NULL array with num_edges > 0");
  if (V > (1ull << 32)) return set_err(GT_EINVAL, "num_vertices > 2^32 needs 64-bit edge IDs");
  if (E && V == 0) return set_err(GT_EINVAL, "edges present but num_vertices == 0");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  if (E == 0) {
    GT_CUDA(cudaMemsetAsync(t_offsets, 0, (V + 1) * 8, st));
    if (stats) GT_CUDA(cudaStreamSynchronize(st));
    return GT_OK;
  }
  Plan p;
  if ((rc = make_plan(V, E, p, 0, v3_capable(E)))) return rc;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  const uint64_t need = workspace_bytes(p, false);
  if (!ws) {
    void* w = nullptr;
    if ((rc = cache_get(g_ws[dev], need, &w))) return rc;
    ws = static_cast<unsigned char*>(w);
  } else if (ws_bytes < need) {
    return set_err(GT_ENOMEM, "workspace too small: need %llu bytes, got %llu", (unsigned long long)need,
                   (unsigned long long)ws_bytes);
  }
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  Timer tm;
  if ((rc = tm.init(stats != nullptr, st))) return rc;
  const InCsr in{offsets, edges, 0, V};
  rc = (mode == kRankAtomic) ? transpose_any<kRankAtomic>(p, in, t_offsets, t_edges, ws, st, stats, tm)
                             : transpose_any<kRankSafe>(p, in, t_offsets, t_edges, ws, st, stats, tm);
  if (rc) return rc;
  if (stats) {
    GT_CUDA(cudaEventSynchronize(tm.ev[tm.n - 1]));
    if ((rc = fill_stats(p, mode, tm, stats))) return rc;
    stats->workspace_bytes = need;
  }
  return GT_OK;
}

int gt_transpose_host(const uint64_t* h_offsets, const uint32_t* h_edges, uint64_t V, uint64_t E,
                      uint64_t* h_t_offsets, uint32_t* h_t_edges, int device, gt_stats* stats) {
  if (!h_offsets || !h_t_offsets || (E && (!h_edges || !h_t_edges)))
    return set_err(GT_EINVAL, "NULL host array");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return set_err(GT_ENODEV, "no CUDA device");
  if (device < 0 || device >= n || device >= 64) return set_err(GT_EINVAL, "bad device %d", device);
  GT_CUDA(cudaSetDevice(device));
  // device copies of input and output live in a per-device cache (grow-only),
  // like the workspace: repeated calls do not re-map gigabytes of memory
  static Cache s_io[64];
  static cudaStream_t s_st[64];
  static std::mutex s_io_mu;  // (g_mu is taken inside gt_transpose)
  std::lock_guard<std::mutex> lk(s_io_mu);
  if (!s_st[device]) GT_CUDA(cudaStreamCreateWithFlags(&s_st[device], cudaStreamNonBlocking));
  cudaStream_t st = s_st[device];
  const uint64_t b_off = align_up((V + 1) * 8, 256), b_e = align_up(std::max<uint64_t>(E, 1) * 4, 256);
  void* base = nullptr;
  int rc = cache_get(s_io[device], 2 * b_off + 2 * b_e, &base);
  if (rc) return rc;
  unsigned char* b = static_cast<unsigned char*>(base);
  uint64_t* d_off = reinterpret_cast<uint64_t*>(b);
  uint64_t* d_toff = reinterpret_cast<uint64_t*>(b + b_off);
  uint32_t* d_e = reinterpret_cast<uint32_t*>(b + 2 * b_off);
  uint32_t* d_te = reinterpret_cast<uint32_t*>(b + 2 * b_off + b_e);
  GT_CUDA(cudaMemcpyAsync(d_off, h_offsets, (V + 1) * 8, cudaMemcpyHostToDevice, st));
  if (E) GT_CUDA(cudaMemcpyAsync(d_e, h_edges, E * 4, cudaMemcpyHostToDevice, st));
  rc = gt_transpose(d_off, d_e, V, E, d_toff, d_te, nullptr, 0, st, stats);
  if (rc) return rc;
  GT_CUDA(cudaMemcpyAsync(h_t_offsets, d_toff, (V + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (E) GT_CUDA(cudaMemcpyAsync(h_t_edges, d_te, E * 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  return GT_OK;
}

int gt_transpose_host_many(int count, const uint64_t* const* h_offsets, const uint32_t* const* h_edges,
                           const uint64_t* Vs, const uint64_t* Es, uint64_t* const* h_t_offsets,
                           uint32_t* const* h_t_edges, int device, gt_stats* stats) {
  if (count < 0) return set_err(GT_EINVAL, "negative batch size %d", count);
  if (count == 0) return GT_OK;
  if (!h_offsets || !h_edges || !Vs || !Es || !h_t_offsets || !h_t_edges) return set_err(GT_EINVAL, "NULL array");
  uint64_t vmax = 0, emax = 0;
  for (int i = 0; i < count; ++i) {
    if (!h_offsets[i] || !h_t_offsets[i] || (Es[i] && (!h_edges[i] || !h_t_edges[i])))
      return set_err(GT_EINVAL, "NULL host array in graph %d", i);
    vmax = std::max(vmax, Vs[i]);
    emax = std::max(emax, Es[i]);
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return set_err(GT_ENODEV, "no CUDA device");
  if (device < 0 || device >= n || device >= 64) return set_err(GT_EINVAL, "bad device %d", device);
  GT_CUDA(cudaSetDevice(device));
  // two device buffer sets (input + output of one graph each), cached per device
  static Cache s_io2[64];
  static cudaStream_t s_sin[64], s_scmp[64], s_sout[64];
  static cudaEvent_t s_ev[64][6];  // in_done[2], cmp_done[2], out_done[2]
  static std::mutex s_mu;
  std::lock_guard<std::mutex> lk(s_mu);
  if (!s_sin[device]) {
    GT_CUDA(cudaStreamCreateWithFlags(&s_sin[device], cudaStreamNonBlocking));
    GT_CUDA(cudaStreamCreateWithFlags(&s_scmp[device], cudaStreamNonBlocking));
    GT_CUDA(cudaStreamCreateWithFlags(&s_sout[device], cudaStreamNonBlocking));
    for (auto& ev : s_ev[device]) GT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  cudaStream_t sin = s_sin[device], scmp = s_scmp[device], sout = s_sout[device];
  cudaEvent_t* ev = s_ev[device];
  const uint64_t b_off = align_up((vmax + 1) * 8, 256), b_e = align_up(std::max<uint64_t>(emax, 1) * 4, 256);
  const uint64_t set_bytes = 2 * b_off + 2 * b_e;
  void* base = nullptr;
  int rc = cache_get(s_io2[device], 2 * set_bytes, &base);
  if (rc) return rc;
  auto buf = [&](int slot, int which) -> unsigned char* {  // 0 off, 1 toff, 2 edges, 3 t_edges
    unsigned char* b = static_cast<unsigned char*>(base) + slot * set_bytes;
    const uint64_t o[4] = {0, b_off, 2 * b_off, 2 * b_off + b_e};
    return b + o[which];
  };
  // H2D of graph i (input set i & 1 is free once graph i-2's transpose has read it)
  auto h2d = [&](int i) -> int {
    const int slot = i & 1;
    if (i >= 2) GT_CUDA(cudaStreamWaitEvent(sin, ev[2 + slot], 0));
    GT_CUDA(cudaMemcpyAsync(buf(slot, 0), h_offsets[i], (Vs[i] + 1) * 8, cudaMemcpyHostToDevice, sin));
    if (Es[i]) GT_CUDA(cudaMemcpyAsync(buf(slot, 2), h_edges[i], Es[i] * 4, cudaMemcpyHostToDevice, sin));
    GT_CUDA(cudaEventRecord(ev[slot], sin));
    return GT_OK;
  };
  if ((rc = h2d(0))) return rc;
  for (int i = 0; i < count; ++i) {
    const int slot = i & 1;
    const uint64_t V = Vs[i], E = Es[i];
    // one graph ahead: graph i+1's copy-in overlaps graph i's kernels and graph i-1's copy-out
    // (gt_transpose returns after its kernels, so graph i-1's transpose is done here)
    if (i + 1 < count && (rc = h2d(i + 1))) return rc;
    uint64_t* d_off = reinterpret_cast<uint64_t*>(buf(slot, 0));
    uint64_t* d_toff = reinterpret_cast<uint64_t*>(buf(slot, 1));
    uint32_t* d_e = reinterpret_cast<uint32_t*>(buf(slot, 2));
    uint32_t* d_te = reinterpret_cast<uint32_t*>(buf(slot, 3));
    // output set free once graph i-2's result has been copied back
    GT_CUDA(cudaStreamWaitEvent(scmp, ev[slot], 0));
    if (i >= 2) GT_CUDA(cudaStreamWaitEvent(scmp, ev[4 + slot], 0));
    rc = gt_transpose(d_off, d_e, V, E, d_toff, d_te, nullptr, 0, scmp, (i == count - 1) ? stats : nullptr);
    if (rc) {
      cudaStreamSynchronize(sin);
      cudaStreamSynchronize(sout);
      return rc;
    }
    GT_CUDA(cudaEventRecord(ev[2 + slot], scmp));
    GT_CUDA(cudaStreamWaitEvent(sout, ev[2 + slot], 0));
    GT_CUDA(cudaMemcpyAsync(h_t_offsets[i], d_toff, (V + 1) * 8, cudaMemcpyDeviceToHost, sout));
    if (E) GT_CUDA(cudaMemcpyAsync(h_t_edges[i], d_te, E * 4, cudaMemcpyDeviceToHost, sout));
    GT_CUDA(cudaEventRecord(ev[4 + slot], sout));
  }
  GT_CUDA(cudaStreamSynchronize(sin));
  GT_CUDA(cudaStreamSynchronize(scmp));
  GT_CUDA(cudaStreamSynchronize(sout));
  return GT_OK;
}

int gt_prefix_sum(const uint32_t* counts, uint64_t n, uint64_t* out, void* stream) {
  if (!out || (n && !counts)) return set_err(GT_EINVAL, "NULL array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  const uint64_t tiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
  void* w = nullptr;
  // use the tail of the aux cache (status words + counter)
  if ((rc = cache_get(g_aux[dev], std::max<uint64_t>(g_aux[dev].bytes, tiles * 8 + 256), &w))) return rc;
  uint64_t* status = static_cast<uint64_t*>(w);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(static_cast<unsigned char*>(w) + align_up(tiles * 8, 128));
  return scan_u32_to_u64(counts, n, out, 0, true, status, ctr, st);
}

// Source-ordered (src, dst) records -> CSR over the source IDs: offsets from
// the source changes (every ID gets its entry, empty sources included) and
// destinations rebased to the local range.
__global__ void k_rec_to_csr(const uint2* __restrict__ rec, uint64_t R, uint64_t Vs, uint32_t dst_base,
                             uint64_t* __restrict__ offsets, uint32_t* __restrict__ edges) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= R; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = (i < R) ? rec[i].x : Vs;                   // sentinel past the end
    const uint64_t prev = (i > 0) ? (uint64_t)rec[i - 1].x + 1 : 0;  // first source not yet started
    for (uint64_t v = prev; v <= s && v <= Vs; ++v) offsets[v] = i;  // sources prev..s start at record i
    if (i < R) edges[i] = rec[i].y - dst_base;
  }
}

__global__ void k_add_base(uint64_t* a, uint64_t n, uint64_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] += base;
}

int gt_shard_partition(const uint64_t* offsets, const uint32_t* edges_slice, uint64_t V, uint64_t src_begin,
                       uint64_t src_end, const uint64_t* h_dst_bounds, int parts, uint32_t* records_out,
                       uint64_t* h_counts_out, void* stream) {
  if (!offsets || !h_dst_bounds || !h_counts_out || parts < 1 || parts > kMaxParts || src_begin > src_end ||
      src_end > V)
    return set_err(GT_EINVAL, "gt_shard_partition: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  uint64_t e_rng[2];
  GT_CUDA(cudaMemcpyAsync(&e_rng[0], offsets + src_begin, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&e_rng[1], offsets + src_end, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  const uint64_t E = e_rng[1] - e_rng[0];
  for (int q = 0; q < parts; ++q) h_counts_out[q] = 0;
  if (E == 0) return GT_OK;
  if (!edges_slice || !records_out) return set_err(GT_EINVAL, "gt_shard_partition: NULL edge/record buffer");
  DigBounds dig{};
  dig.parts = parts;
  for (int q = 0; q <= parts; ++q) {
    if (h_dst_bounds[q] > V || (q && h_dst_bounds[q] < h_dst_bounds[q - 1]))
      return set_err(GT_EINVAL, "gt_shard_partition: destination bounds not monotone in [0, V]");
    dig.lo[q] = (uint32_t)std::min<uint64_t>(h_dst_bounds[q], 0xffffffffull);
  }
  uint64_t CT = 65536, ntiles = (E + CT - 1) / CT;
  const uint64_t nplace = (E + kPlaceTile - 1) / kPlaceTile;
  uint64_t off = 0;
  const uint64_t o_tcnt = off;
  off = align_up(off + ntiles * parts * 4, 256);
  const uint64_t o_tbase = off;
  off = align_up(off + (ntiles * parts + 1) * 8, 256);
  const uint64_t o_tsrc = off;
  off = align_up(off + (nplace + 2) * 4, 256);
  const uint64_t o_status = off;
  off = align_up(off + ((ntiles * parts + kScanTile) / kScanTile + 1) * 8, 256);
  const uint64_t o_ctr = off;
  off += 256;
  void* w = nullptr;
  if ((rc = cache_get(g_aux[dev], off, &w))) return rc;
  unsigned char* ws = static_cast<unsigned char*>(w);
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(ws + o_tcnt);
  uint64_t* tbase = reinterpret_cast<uint64_t*>(ws + o_tbase);
  uint32_t* tsrc = reinterpret_cast<uint32_t*>(ws + o_tsrc);
  uint64_t* status = reinterpret_cast<uint64_t*>(ws + o_status);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(ws + o_ctr);
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  const InCsr in{offsets, edges_slice, e_rng[0], V};
  k_tile_src<<<(unsigned)((nplace + 1 + 255) / 256), 256, 0, st>>>(in, E, kPlaceTile, nplace + 1, tsrc);
  GT_LAUNCH_CHECK();
  k_l1_count<InCsr, DigBounds><<<(unsigned)ntiles, 512, parts * 4, st>>>(in, dig, E, CT, ntiles, parts, tcnt);
  GT_LAUNCH_CHECK();
  if ((rc = scan_u32_to_u64(tcnt, ntiles * parts, tbase, 0, true, status, ctr, st))) return rc;
  uint2* out = reinterpret_cast<uint2*>(records_out);
  const size_t sm = smem_l1_place(parts, mode, false, CT);
  if (mode == kRankAtomic) {
    if ((rc = set_smem(k_l1_place<kRankAtomic, InCsr, DigBounds, OutFull>, sm))) return rc;
    k_l1_place<kRankAtomic, InCsr, DigBounds, OutFull><<<(unsigned)ntiles, kL1Warps * 32, sm, st>>>(
        in, dig, E, CT, ntiles, parts, tbase, tsrc, OutFull{out});
  } else {
    if ((rc = set_smem(k_l1_place<kRankSafe, InCsr, DigBounds, OutFull>, sm))) return rc;
    k_l1_place<kRankSafe, InCsr, DigBounds, OutFull><<<(unsigned)ntiles, kL1Warps * 32, sm, st>>>(
        in, dig, E, CT, ntiles, parts, tbase, tsrc, OutFull{out});
  }
  GT_LAUNCH_CHECK();
  std::vector<uint64_t> starts(parts + 1);
  for (int q = 0; q < parts; ++q)
    GT_CUDA(cudaMemcpyAsync(&starts[q], tbase + (uint64_t)q * ntiles, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  starts[parts] = E;
  for (int q = 0; q < parts; ++q) h_counts_out[q] = starts[q + 1] - starts[q];
  return GT_OK;
}

int gt_shard_transpose(const uint32_t* records, uint64_t R, uint64_t src_num_vertices, uint64_t dst_begin,
                       uint64_t dst_end, uint64_t global_base, uint64_t* t_offsets_local, uint32_t* t_edges_local,
                       void* stream, gt_stats* stats) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (dst_end < dst_begin || !t_offsets_local || (R && (!records || !t_edges_local)))
    return set_err(GT_EINVAL, "gt_shard_transpose: bad arguments");
  const uint64_t V = dst_end - dst_begin;
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  if (R == 0) {
    GT_CUDA(cudaMemsetAsync(t_offsets_local, 0, (V + 1) * 8, st));
    k_add_base<<<1, 256, 0, st>>>(t_offsets_local, V + 1, global_base);
    GT_LAUNCH_CHECK();
    return GT_OK;
  }
  if (V == 0) return set_err(GT_EINVAL, "gt_shard_transpose: records for an empty destination range");
  Plan p;
  if (src_num_vertices == 0 || src_num_vertices > (1ull << 32))
    return set_err(GT_EINVAL, "gt_shard_transpose: bad src_num_vertices");
  if ((rc = make_plan(V, R, p, src_num_vertices, v3_capable(R)))) return rc;
  if (use_v3(p)) {
    // the received stream is source-ordered: rebuild it as a CSR over the
    // source IDs (offsets from the source changes, local destination IDs) and
    // run the v3 pipeline with separate source / destination ID spaces
    const uint64_t Vs = src_num_vertices;
    const uint64_t b_off = align_up((Vs + 1) * 8, 256), b_e = align_up(R * 4, 256);
    Plan3 q;
    make_plan3(p, q);
    void* w = nullptr;
    if ((rc = cache_get(g_ws[dev], q.total + b_off + b_e, &w))) return rc;
    unsigned char* ws = static_cast<unsigned char*>(w);
    uint64_t* s_off = reinterpret_cast<uint64_t*>(ws + q.total);
    uint32_t* s_edg = reinterpret_cast<uint32_t*>(ws + q.total + b_off);
    k_rec_to_csr<<<(unsigned)std::min<uint64_t>((R + 255) / 256, 148 * 64), 256, 0, st>>>(
        reinterpret_cast<const uint2*>(records), R, Vs, (uint32_t)dst_begin, s_off, s_edg);
    GT_LAUNCH_CHECK();
    int mode;
    if ((rc = rank_mode_for(dev, st, &mode))) return rc;
    Timer tm;
    if ((rc = tm.init(stats != nullptr, st))) return rc;
    const InCsr in{s_off, s_edg, 0, Vs};
    rc = (mode == kRankAtomic) ? transpose_v3<kRankAtomic>(p, in, t_offsets_local, t_edges_local, ws, st, stats, tm)
                               : transpose_v3<kRankSafe>(p, in, t_offsets_local, t_edges_local, ws, st, stats, tm);
    if (rc) return rc;
    if (global_base) {
      k_add_base<<<148, 256, 0, st>>>(t_offsets_local, V + 1, global_base);
      GT_LAUNCH_CHECK();
    }
    if (stats) {
      GT_CUDA(cudaStreamSynchronize(st));
      fill_stats(p, mode, tm, stats);
      stats->workspace_bytes = q.total + b_off + b_e;
    }
    return GT_OK;
  }
  void* w = nullptr;
  if ((rc = cache_get(g_ws[dev], p.total, &w))) return rc;
  unsigned char* ws = static_cast<unsigned char*>(w);
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  Timer tm;
  if ((rc = tm.init(stats != nullptr, st))) return rc;
  const InRec in{reinterpret_cast<const uint2*>(records), (uint32_t)dst_begin};
  rc = (mode == kRankAtomic) ? transpose_any<kRankAtomic>(p, in, t_offsets_local, t_edges_local, ws, st, stats, tm)
                             : transpose_any<kRankSafe>(p, in, t_offsets_local, t_edges_local, ws, st, stats, tm);
  if (rc) return rc;
  if (global_base) {
    k_add_base<<<148, 256, 0, st>>>(t_offsets_local, V + 1, global_base);
    GT_LAUNCH_CHECK();
  }
  if (stats) {
    GT_CUDA(cudaStreamSynchronize(st));
    fill_stats(p, mode, tm, stats);
  }
  return GT_OK;
}

int gt_edge_balanced_bounds(const uint64_t* h_offsets, uint64_t V, int64_t parts, int64_t* h_bounds) {
  if (!h_offsets || !h_bounds) return set_err(GT_EINVAL, "NULL array");
  if (parts < 1) parts = 1;  // _nb.py:127
  const uint64_t E = h_offsets[V];
  for (int64_t q = 0; q <= parts; ++q) {
    const unsigned __int128 t = (unsigned __int128)E * (uint64_t)q / (uint64_t)parts;
    const uint64_t target = (uint64_t)t;
    const uint64_t* it = std::lower_bound(h_offsets, h_offsets + V + 1, target);  // searchsorted 'left'
    h_bounds[q] = (int64_t)(it - h_offsets);
  }
  h_bounds[0] = 0;
  h_bounds[parts] = (int64_t)V;
  return GT_OK;
}

}  // extern "C"

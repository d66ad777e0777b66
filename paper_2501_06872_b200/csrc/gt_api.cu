// gt_api.cu — host orchestration and the extern "C" boundary of libgt.so.
// See include/gt.h for the contract and the reference functions each entry
// point replaces.  No torch types cross this boundary.
//
// Pipeline: three stable partition levels of the destination
// ID, kernels in gt_v3.cuh.
//   level 1  CSR edge stream -> R1 (4-byte records grouped by coarse bucket)
//   level 2  R1 runs of every coarse bucket -> R2 at CSC positions
//   level 3  R2 -> CSC edges + offsets (units in shared memory, big buckets tiled)
// One GPU: R1 = one run per bucket (t_edges doubles as R1 storage).  Multi-GPU
// (gt_shard_send / gt_shard_receive, gt_multi.cu): a sender runs level 1 on its
// source slice; a receiver runs levels 2-3 on the runs it received, one per
// sender and bucket, so the exchanged payload is R1 itself (4 B per edge).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gt.h"
#include "gt_api_internal.h"
#include "gt_base.cuh"
#include "gt_v3.cuh"

using namespace gt;

namespace {
thread_local std::string g_err;
}  // namespace

int gt_internal_set_err(int code, const char* msg) {  // for the other translation units
  g_err = msg;
  return code;
}

int gt_set_errf(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

namespace {

#define set_err gt_set_errf

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

// ---------------------------------------------------------------- config
std::mutex g_cfg_mu;
gt_config g_cfg = {{0, 0, 0}, 0, {0, 0, 0, 0}};
gt_config config_snapshot() {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  return g_cfg;
}

// ---------------------------------------------------------------- plan
// Fine buckets (2^c vertices) average <= kFineTarget / 2 records.
constexpr double kFineTarget = 8192.0;

struct Plan {
  uint64_t V = 0, E = 0;  // destination IDs (local range) and records
  bool wide = false;      // 64-bit positions; R2 = source (u32) + low digit (u8)
  int nb = 0, nbs = 0;    // destination / source ID bits
  int a = 0, b = 0, c = 0;
  int L = 0, nsh = 0;  // R1: source low bits, source high bits (decoded from seg_hi)
  int gbits = 0;       // compact R2: fine-digit bits kept beside the low digit
  int D1 = 1, Db = 1, Dc = 1;
  int exp = 0;  // gt_config.reserved[0]: experiment bits (A/B measurements; 0 = product path)
};

// Digit split of the destination ID for a graph of V destinations, E edges,
// Vsrc source IDs.  Compact form: 4-byte R1 and R2 records; wide form: E >=
// 2^32 or sources too wide for a 4-byte R2.
int make_plan(uint64_t V, uint64_t E, uint64_t Vsrc, const gt_config& cfg, Plan& p) {
  p = Plan{};
  p.V = V;
  p.E = E;
  p.nb = bits_for(V);
  p.nbs = bits_for(Vsrc ? Vsrc : V);
  const double avg = V ? (double)E / (double)V : 1.0;
  const bool forced = cfg.split[0] + cfg.split[1] + cfg.split[2] == p.nb && cfg.split[2] >= 1;
  // compact: 8-bit middle digit and fine buckets of ~4K records measured best on
  // C3 (9|8|7: 8.26 ms vs 9|9|6 8.74, 10|7|7 8.56, 8|9|7 8.60); the coarse digit
  // takes the rest (<= 10 bits), the middle digit grows only when it must
  if (!cfg.force_wide && E < (1ull << 32)) {
    int cc = 1;
    while (cc < 8 && (double)(1u << (cc + 1)) * std::max(avg, 1.0) <= kFineTarget / 2.0) ++cc;
    cc = std::min(cc, 32 - p.nbs);
    cc = std::min(cc, p.nb);
    const int rem = p.nb - cc;
    int ca = rem, cb = 0;
    if (rem > 9) {
      cb = std::min(10, std::max(8, rem - 10));
      ca = rem - cb;
    }
    if (forced) {
      ca = cfg.split[0];
      cb = cfg.split[1];
      cc = cfg.split[2];
    }
    const int L = 32 - (cb + cc);
    const int nsh = std::max(0, p.nbs - L);
    if (cc >= 1 && p.nbs + cc <= 32 && ca >= 0 && ca <= 10 && cb >= 0 && cb <= 10 && L >= 1 && nsh <= 12) {
      p.a = ca;
      p.b = cb;
      p.c = cc;
      p.L = L;
      p.nsh = nsh;
      int gb = std::min(32 - p.nbs - cc, cb);
      while (gb > 0 && (1 << (gb + cc)) > v3::ML3) --gb;
      p.gbits = std::max(0, gb);
    } else {
      p.c = 0;
    }
  }
  if (p.c == 0) {  // wide form
    int cc = 1;
    while (cc < 8 && (double)(1u << (cc + 1)) * std::max(avg, 1.0) <= kFineTarget / 2.0) ++cc;
    cc = std::min(cc, p.nb);
    const int rem = p.nb - cc;
    int ca = rem, cb = 0;
    if (rem > 10) {
      cb = std::min(10, std::max(8, rem - 11));
      ca = rem - cb;
    }
    if (forced && cfg.split[2] <= 8) {
      ca = cfg.split[0];
      cb = cfg.split[1];
      cc = cfg.split[2];
    }
    const int L = 32 - (cb + cc);
    const int nsh = std::max(0, p.nbs - L);
    if (!(cc >= 1 && cc <= 8 && ca >= 0 && ca <= 11 && cb >= 0 && cb <= 10 && L >= 1 && nsh <= 18))
      return set_err(GT_EINVAL,
                     "num_vertices = %llu (%d-bit IDs) with %llu edges has no digit split in this build",
                     (unsigned long long)V, p.nb, (unsigned long long)E);
    p.wide = true;
    p.a = ca;
    p.b = cb;
    p.c = cc;
    p.L = L;
    p.nsh = nsh;
    p.gbits = 0;
  }
  p.D1 = 1 << p.a;
  p.Db = 1 << p.b;
  p.Dc = 1 << p.c;
  p.exp = cfg.reserved[0];
  return GT_OK;
}

// ---------------------------------------------------------------- workspace layout
// Level-1 tables (count tiles), level-2 runs / tiles / tables, level-3 plan;
// R2 (4E, + E low-digit bytes for the wide form) is the bulk.
struct Layout {
  uint64_t ntiles1 = 0, nplace = 0, nh = 0, nruns = 0, max_t2 = 0, nfine = 0, max_big = 0, max_t3 = 0;
  uint64_t o_r2, o_r2lv, o_tcnt, o_tbase, o_status, o_ctr, o_psrc, o_prev, o_seghi, o_runs, o_rfirst, o_bstart,
      o_tiles2, o_cnt2, o_base2, o_seg2, o_fbase, o_units, o_bigs, o_tiles3, o_cnt3, o_base3, o_seg3, o_cnt, o_err,
      o_bnt, o_bfirst, total;
};

// E1: level-1 edges (0: no level 1 here); E23: records of levels 2-3; D1: local buckets; R: runs per bucket.
void make_layout(const Plan& p, uint64_t E1, uint64_t E23, uint32_t R, Layout& q) {
  q = Layout{};
  q.ntiles1 = (E1 + v3::CT1 - 1) / v3::CT1;
  q.nplace = (E1 + 8191) / 8192 + 2;  // place tiles of >= 8192 edges
  q.nh = 1ull << p.nsh;
  q.nruns = (uint64_t)p.D1 * R;
  q.max_t2 = (E23 + v3::CT2 - 1) / v3::CT2 + q.nruns;
  q.nfine = (uint64_t)p.D1 * p.Db;
  q.max_big = std::min<uint64_t>(q.nfine, E23 / v3::CAP3 + 1);
  q.max_t3 = (E23 + v3::CT2 - 1) / v3::CT2 + q.max_big;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o = off;
    off = align_up(off + std::max<uint64_t>(bytes, 1), 256);
    return o;
  };
  const uint64_t n1 = (uint64_t)p.D1 * q.ntiles1;
  q.o_r2 = take(E23 ? E23 * 4 + 64 : 0);
  q.o_r2lv = take(p.wide && E23 ? E23 + 64 : 0);  // wide: low digit of every R2 record (+ padding for block loads)
  q.o_tcnt = take(n1 * 4);
  q.o_tbase = take((n1 + 1) * 8);
  const uint64_t nscan = std::max<uint64_t>(std::max<uint64_t>(n1 + 1, q.max_big + 1),
                                            std::max<uint64_t>(q.max_t2 * (uint64_t)p.Db, q.max_t3 * (uint64_t)p.Dc));
  q.o_status = take(((nscan + kScanTile - 1) / kScanTile + 1) * 8);
  q.o_ctr = take(64);
  q.o_psrc = take((q.nplace + 2) * 4);
  q.o_prev = take((q.ntiles1 + 1) * 4);
  q.o_seghi = take(E1 ? (uint64_t)p.D1 * (q.nh + 1) * 8 : 0);
  q.o_runs = take(q.nruns * sizeof(v3::Run));
  q.o_rfirst = take((q.nruns + 1) * 4);
  q.o_bstart = take(((uint64_t)p.D1 + 1) * 8);
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

// ---------------------------------------------------------------- device caches
// One workspace per (device, stream): calls on different streams never share
// scratch; calls on one stream are ordered by the stream.  Growth frees and
// allocates stream-ordered (cudaFreeAsync / cudaMallocAsync on that stream),
// so a call still running on the stream keeps its buffer until it finishes.
// Each entry also holds a mapped pinned status word the last call's final
// kernel writes (gt_transpose_status).
struct WsEntry {
  void* ptr = nullptr;
  uint64_t bytes = 0;
  int* status = nullptr;  // mapped pinned (host pointer == device pointer under UVA)
  std::mutex call_mu;     // held by a call from its workspace lookup to its last launch: two host
                          // threads on one stream cannot free each other's buffer before use
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, WsEntry> g_ws;

int ws_entry(int dev, cudaStream_t st, WsEntry** out) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  WsEntry& e = g_ws[{dev, st}];
  if (!e.status) {
    GT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&e.status), sizeof(int), cudaHostAllocMapped));
    *e.status = GT_OK;
  }
  *out = &e;
  return GT_OK;
}

int ws_get(int dev, cudaStream_t st, uint64_t bytes, unsigned char** out, int** status) {
  WsEntry* e;
  int rc = ws_entry(dev, st, &e);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (e->bytes < bytes) {
    if (e->ptr) GT_CUDA(cudaFreeAsync(e->ptr, st));
    e->ptr = nullptr;
    e->bytes = 0;
    GT_CUDA(cudaMallocAsync(&e->ptr, bytes, st));
    e->bytes = bytes;
  }
  *out = static_cast<unsigned char*>(e->ptr);
  if (status) *status = e->status;
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

// ---------------------------------------------------------------- rank mode
std::mutex g_mu;
int g_forced_rank_mode = -1;  // -1 auto
int g_dev_rank_mode[64];      // per device: -1 unknown, 0/1 decided
bool g_dev_rank_init = false;

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

// The first call on a device runs the lane-order self-test (synchronous, once);
// later calls only read the decision.
int rank_mode_for(int dev, cudaStream_t st, int* mode) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_forced_rank_mode >= 0) {
    *mode = g_forced_rank_mode;
    return GT_OK;
  }
  if (!g_dev_rank_init) {
    for (int i = 0; i < 64; ++i) g_dev_rank_mode[i] = -1;
    g_dev_rank_init = true;
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

// ---------------------------------------------------------------- launch helpers
int g_num_sms[64];
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_num_sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = v > 0 ? v : 148;
  }
  return g_num_sms[dev];
}
template <typename Kern>
unsigned persistent_grid(Kern kernel, int threads, size_t smem, uint64_t work) {
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  const uint64_t g = (uint64_t)num_sms() * occ;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, std::max<uint64_t>(work, 1)));
}

size_t max_smem_optin() {  // largest dynamic shared memory a block may opt into
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

// CUDA-event timing of a call (stats != NULL): step marks plus begin/end of the
// main kernels.  Events are created once per thread and device and reused.
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
    thread_local cudaEvent_t t_ev[64][kSteps + 2 * kKern];
    thread_local bool t_init[64] = {};
    int dev = 0;
    GT_CUDA(cudaGetDevice(&dev));
    if (!t_init[dev]) {
      for (auto& e : t_ev[dev]) GT_CUDA(cudaEventCreate(&e));
      t_init[dev] = true;
    }
    ev = t_ev[dev];
    kev = t_ev[dev] + kSteps;
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

// Workspace pointers of a Layout.
struct Ws {
  uint32_t* r2;
  uint8_t* r2lv;
  uint32_t* tcnt;
  uint64_t* tbase;
  uint64_t* status;
  unsigned int* ctr;
  uint32_t* psrc;
  uint32_t* prev;
  uint64_t* seghi;
  v3::Run* runs;
  uint32_t* rfirst;
  uint64_t* bstart;
  v3::RTile* tiles2;
  uint32_t* cnt2;
  uint64_t* base2;
  v3::SegDesc* seg2;
  uint64_t* fbase;
  v3::Unit3* units;
  v3::Big3* bigs;
  v3::RTile* tiles3;
  uint32_t* cnt3;
  uint64_t* base3;
  v3::SegDesc* seg3;
  uint32_t* cnt;  // [0] units [1] big [2] tiles3 [3] unit ctr
  unsigned int* err;
  uint32_t* bnt;
  uint64_t* bfirst;
};
Ws ws_ptrs(const Layout& q, unsigned char* ws, const Plan& p) {
  Ws w;
  w.r2 = reinterpret_cast<uint32_t*>(ws + q.o_r2);
  w.r2lv = p.wide ? reinterpret_cast<uint8_t*>(ws + q.o_r2lv) : nullptr;
  w.tcnt = reinterpret_cast<uint32_t*>(ws + q.o_tcnt);
  w.tbase = reinterpret_cast<uint64_t*>(ws + q.o_tbase);
  w.status = reinterpret_cast<uint64_t*>(ws + q.o_status);
  w.ctr = reinterpret_cast<unsigned int*>(ws + q.o_ctr);
  w.psrc = reinterpret_cast<uint32_t*>(ws + q.o_psrc);
  w.prev = reinterpret_cast<uint32_t*>(ws + q.o_prev);
  w.seghi = reinterpret_cast<uint64_t*>(ws + q.o_seghi);
  w.runs = reinterpret_cast<v3::Run*>(ws + q.o_runs);
  w.rfirst = reinterpret_cast<uint32_t*>(ws + q.o_rfirst);
  w.bstart = reinterpret_cast<uint64_t*>(ws + q.o_bstart);
  w.tiles2 = reinterpret_cast<v3::RTile*>(ws + q.o_tiles2);
  w.cnt2 = reinterpret_cast<uint32_t*>(ws + q.o_cnt2);
  w.base2 = reinterpret_cast<uint64_t*>(ws + q.o_base2);
  w.seg2 = reinterpret_cast<v3::SegDesc*>(ws + q.o_seg2);
  w.fbase = reinterpret_cast<uint64_t*>(ws + q.o_fbase);
  w.units = reinterpret_cast<v3::Unit3*>(ws + q.o_units);
  w.bigs = reinterpret_cast<v3::Big3*>(ws + q.o_bigs);
  w.tiles3 = reinterpret_cast<v3::RTile*>(ws + q.o_tiles3);
  w.cnt3 = reinterpret_cast<uint32_t*>(ws + q.o_cnt3);
  w.base3 = reinterpret_cast<uint64_t*>(ws + q.o_base3);
  w.seg3 = reinterpret_cast<v3::SegDesc*>(ws + q.o_seg3);
  w.cnt = reinterpret_cast<uint32_t*>(ws + q.o_cnt);
  w.err = reinterpret_cast<unsigned int*>(ws + q.o_err);
  w.bnt = reinterpret_cast<uint32_t*>(ws + q.o_bnt);
  w.bfirst = reinterpret_cast<uint64_t*>(ws + q.o_bfirst);
  return w;
}

// ---------------------------------------------------------------- level 1
// CSR stream `in` (E edges from global edge in.e_begin) -> R1 in `r1`, grouped
// by coarse bucket, with the source-high boundary table w.seghi and the
// per-(bucket, count tile) bases w.tbase.  `sender`: the stream starts inside
// the graph (multi-GPU shard): the boundary table starts at the shard's first
// source-high value instead of 0.
template <int kMode>
int level1(const Plan& p, const Layout& q, Ws& w, InCsr in, uint64_t E, bool sender, uint32_t* r1, cudaStream_t st,
           Timer& tm, int* launches, uint32_t slab_mask = 0, uint32_t slab_val = 0) {
  // slab_mask != 0: slab mode (num_vertices > 2^29, wide form only): only the
  // destinations with (dst & slab_mask) == slab_val are partitioned
  const bool slab = slab_mask != 0;
  using namespace v3;
  const int D1 = p.D1;
  int rc;
  GT_CUDA(cudaMemsetAsync(w.seghi, 0xff, (uint64_t)D1 * (q.nh + 1) * 8, st));
  // place-tile shape (measured, DESIGN.md §2 table): compact graphs with <= 512
  // coarse digits: 16 warps x K = 16 (8192 edges, 2 CTAs/SM); more digits: 8 x 32;
  // wide graphs: 16 x 32 (16384 edges, 1 CTA/SM) when its tables fit
  enum { kC16x16, kC8x32, kW16x32, kW8x32 } form;
  if (!p.wide) form = (D1 <= 512 && smem_p1(D1, kMode, 16, 16) + 64 <= max_smem_optin()) ? kC16x16 : kC8x32;
  else form = (smem_p1(D1, kMode, 32, 16) + 64 <= max_smem_optin()) ? kW16x32 : kW8x32;
  const uint64_t pt1 = (form == kW16x32) ? 16384 : 8192, nplace1 = (E + pt1 - 1) / pt1;
  k_tile_src<<<(unsigned)((nplace1 + 1 + 255) / 256), 256, 0, st>>>(in, E, pt1, nplace1 + 1, w.psrc);
  GT_LAUNCH_CHECK();
  k_prev_src<<<(unsigned)((q.ntiles1 + 255) / 256), 256, 0, st>>>(in, E, CT1, q.ntiles1, w.prev);
  GT_LAUNCH_CHECK();
  if (sender) {  // the first count tile's boundaries start after the shard's first source
    k_tile_src<<<1, 32, 0, st>>>(in, E, CT1, 1, w.prev);
    GT_LAUNCH_CHECK();
  }
  {
    auto kc = slab ? k_c1<true> : k_c1<false>;
    if ((rc = set_smem(kc, (size_t)G1 * D1 * 4))) return rc;
    kc<<<(unsigned)((q.ntiles1 + G1 - 1) / G1), 512, (size_t)G1 * D1 * 4, st>>>(in.edges, E, q.ntiles1, D1, p.b + p.c,
                                                                               w.tcnt, slab_mask, slab_val);
  }
  GT_LAUNCH_CHECK();
  if ((rc = scan_u32_to_u64(w.tcnt, (uint64_t)D1 * q.ntiles1, w.tbase, 0, true, w.status, w.ctr, st))) return rc;
  P1Args a;
  a.offsets = in.offsets;
  a.edges = in.edges;
  a.e_begin = in.e_begin;
  a.V = in.V;
  a.E = E;
  a.ntiles = q.ntiles1;
  a.D = D1;
  a.shift = p.b + p.c;
  a.L = p.L;
  a.low_mask = (uint32_t)((1ull << (p.b + p.c)) - 1);
  a.src_mask = (uint32_t)((1ull << p.L) - 1);
  a.tbase = w.tbase;
  a.psrc = w.psrc;
  a.prev_src = w.prev;
  a.nh = (uint32_t)q.nh;
  a.seg_hi = w.seghi;
  a.out = r1;
  a.slab_mask = slab_mask;
  a.slab_val = slab_val;
  if ((rc = tm.kbegin(0))) return rc;
  auto go = [&](auto kern, int threads, size_t sm) -> int {
    int r;
    if ((r = set_smem(kern, sm))) return r;
    kern<<<(unsigned)q.ntiles1, threads, sm, st>>>(a);
    return GT_OK;
  };
  switch (form) {
    case kC16x16:
      // experiment bit 4096: the pointer-based rank/stage loops (A/B of DESIGN.md §2e)
      if (p.exp & 4096) rc = go(k_p1<kMode, 16, false, 16, 2, false, false>, 512, smem_p1(D1, kMode, 16, 16));
      else rc = go(k_p1<kMode, 16, false, 16>, 512, smem_p1(D1, kMode, 16, 16));
      break;
    case kC8x32: rc = go(k_p1<kMode, 32>, T, smem_p1(D1, kMode, 32)); break;
    case kW16x32:
      if (slab) rc = go(k_p1<kMode, 32, true, 16, 1, true>, 512, smem_p1(D1, kMode, 32, 16));
      else rc = go(k_p1<kMode, 32, true, 16, 1>, 512, smem_p1(D1, kMode, 32, 16));
      break;
    case kW8x32:
      if (slab) rc = go(k_p1<kMode, 32, true, W, 2, true>, T, smem_p1(D1, kMode, 32));
      else rc = go(k_p1<kMode, 32, true>, T, smem_p1(D1, kMode, 32));
      break;
  }
  if (slab && !p.wide) return set_err(GT_EINVAL, "slab mode needs the wide form");
  if (rc) return rc;
  GT_LAUNCH_CHECK();
  if ((rc = tm.kend(0))) return rc;
  *launches += sender ? 6 : 5;  // tile owners (x2 for a shard), count-tile owners, count, scan, place
  return GT_OK;
}

// ---------------------------------------------------------------- levels 2 and 3
// R1 (runs w.runs[c * R + s] of every local bucket c, source-high rows
// seg_hi[(s * row_stride + c) * (nh + 1) ...]) -> CSC: t_edges[0..E) and
// t_offsets[0..V] (local vertex IDs, positions from 0).  Records: p.E.
template <int kMode>
int level23(const Plan& p, const Layout& q, Ws& w, const uint32_t* r1, uint32_t R, uint32_t row_stride,
            const uint64_t* seg_hi, uint64_t* t_offsets, uint32_t* t_edges, cudaStream_t st, Timer& tm,
            int* launches) {
  using namespace v3;
  const uint64_t V = p.V, E = p.E;
  const int D1 = p.D1, Db = p.Db, Dc = p.Dc;
  const uint32_t nh = (uint32_t)q.nh, nruns = (uint32_t)q.nruns;
  int rc;
  const int sms = num_sms();
  // level-3 units are aligned groups of 2^sbits fine buckets (<= ML3 local
  // vertices); R2 carries g3 = sbits fine-digit bits when it has room, else
  // the unit decodes the fine bucket from the record's position
  auto log2_groups = [&](int ml) {
    int b = 0;
    while ((ml >> p.c) >> (b + 1)) ++b;
    return b;
  };
  const bool pos_fine = p.wide || p.gbits < log2_groups(256);
  const int sbits = pos_fine ? log2_groups(ML3) : log2_groups(256);
  const int g3 = pos_fine ? 0 : sbits;

  GT_CUDA(cudaMemsetAsync(w.cnt, 0, 64, st));
  // ---- level 2: tiles of every run, count, per-bucket bases, place into R2
  k_runs_plan<<<1, 1024, 0, st>>>(w.runs, nruns, R, w.rfirst, w.bstart);
  GT_LAUNCH_CHECK();
  k_l2_tiles<<<D1, 128, 0, st>>>(w.runs, R, row_stride, w.rfirst, w.bstart, Db, seg_hi, nh, w.tiles2, w.seg2);
  GT_LAUNCH_CHECK();
  const uint32_t* n_t2 = w.rfirst + nruns;
  const unsigned gt2 = (unsigned)std::min<uint64_t>(q.max_t2, (uint64_t)sms * 8);
  GT_CUDA(cudaMemsetAsync(w.cnt2, 0, q.max_t2 * (uint64_t)Db * 4, st));  // the scan covers the unused tail too
  if ((rc = set_smem(k_cnt_rec, (size_t)Db * 4))) return rc;
  k_cnt_rec<<<gt2, 512, (size_t)Db * 4, st>>>(r1, w.tiles2, n_t2, Db, DigSM{p.L + p.c, (uint32_t)(Db - 1)}, w.cnt2);
  GT_LAUNCH_CHECK();
  // bases of every (tile, fine digit): one device-wide exclusive scan of the
  // per-bucket digit-major count tables (concatenated in bucket order), then a
  // per-bucket rebase to its output start, which also writes the fine-bucket starts
  if ((rc = scan_u32_to_u64(w.cnt2, (uint64_t)q.max_t2 * Db, w.base2, 0, false, w.status, w.ctr, st))) return rc;
  GT_CUDA(cudaMemsetAsync(w.cnt + 4, 0, 4, st));
  k_set_u32<<<1, 1, 0, st>>>(w.cnt + 4, (uint32_t)D1);
  GT_LAUNCH_CHECK();
  k_segfix<<<(unsigned)D1, 512, 0, st>>>(w.seg2, w.cnt + 4, Db, w.base2, w.fbase, q.nfine, w.err);
  GT_LAUNCH_CHECK();
  {
    DecR1 dec;
    dec.L = p.L;
    dec.src_mask = (uint32_t)((1ull << p.L) - 1);
    dec.shB = p.L + p.c;
    dec.maskB = (uint32_t)(Db - 1);
    dec.lvmask = (uint32_t)((1ull << (p.c + g3)) - 1);  // R2: low digit + g3 fine-digit bits (0: L3 uses positions)
    dec.nbs = p.nbs;
    dec.nh = nh;
    dec.seg_hi = seg_hi;
    if ((rc = tm.kbegin(1))) return rc;
    if (p.wide) {  // R2 = source array + low-digit bytes, 64-bit positions
      const size_t sm16 = smem_p2(Db, kMode, 32, kIoSplit, 16);
      if (sm16 + 64 <= max_smem_optin()) {  // 16384-record tiles, one 16-warp CTA per SM (C5: 88.4 -> 65.9 ms)
        auto kern = k_p2<kMode, DecR1, 32, false, kIoSplit, true, 16, 1>;
        if ((rc = set_smem(kern, sm16))) return rc;
        kern<<<persistent_grid(kern, 512, sm16, q.max_t2), 512, sm16, st>>>(r1, w.tiles2, n_t2, Db, dec, w.base2,
                                                                              w.r2, nullptr, nullptr, w.r2lv);
      } else {
        auto kern = k_p2<kMode, DecR1, 32, false, kIoSplit>;
        const size_t sm = smem_p2(Db, kMode, 32, kIoSplit);
        if ((rc = set_smem(kern, sm))) return rc;
        kern<<<persistent_grid(kern, T, sm, q.max_t2), T, sm, st>>>(r1, w.tiles2, n_t2, Db, dec, w.base2, w.r2,
                                                                     nullptr, nullptr, w.r2lv);
      }
    } else if (Db >= 1024) {  // 8192-record tiles (C4 level 2: 5.70 ms vs 5.89 at 4096)
      auto kern = k_p2<kMode, DecR1, 32>;
      const size_t sm = smem_p2(Db, kMode, 32);
      if ((rc = set_smem(kern, sm))) return rc;
      kern<<<persistent_grid(kern, T, sm, q.max_t2), T, sm, st>>>(r1, w.tiles2, n_t2, Db, dec, w.base2, w.r2, nullptr, nullptr, nullptr);
    } else {  // 4096-record tiles, 4 CTAs/SM, no batched landing loads (C3 2.11 vs 2.18 ms)
      auto kern = (p.exp & 4096) ? k_p2<kMode, DecR1, 16, false, kIoPlain, false, W, 4, true, false>
                                 : k_p2<kMode, DecR1, 16, false, kIoPlain, false>;
      const size_t sm = smem_p2(Db, kMode, 16);
      if ((rc = set_smem(kern, sm))) return rc;
      kern<<<persistent_grid(kern, T, sm, q.max_t2), T, sm, st>>>(r1, w.tiles2, n_t2, Db, dec, w.base2, w.r2, nullptr, nullptr, nullptr);
    }
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(1))) return rc;
  }
  *launches += 7;  // runs plan, tiles, count, scan, set, segfix, place
  if ((rc = tm.mark())) return rc;
  // ---- level 3: units of small fine buckets; tiled count / scan / place for big ones
  k_set_u64<<<1, 1, 0, st>>>(w.fbase + q.nfine, E);
  GT_LAUNCH_CHECK();
  k_plan3<<<(unsigned)((q.nfine / (1u << sbits) + 255) / 256 + 1), 256, 0, st>>>(
      w.fbase, (uint32_t)q.nfine, sbits, w.units, w.cnt + 0, w.bigs, w.cnt + 1, (uint32_t)CAP3);
  GT_LAUNCH_CHECK();
  // the big-bucket chain runs on a side stream, concurrently with the units
  // (disjoint fine buckets); its short scans overlap the units kernel
  cudaStream_t sb;
  cudaEvent_t ev_fork, ev_join;
  if ((rc = side_stream(&sb, &ev_fork, &ev_join))) return rc;
  GT_CUDA(cudaEventRecord(ev_fork, st));
  GT_CUDA(cudaStreamWaitEvent(sb, ev_fork, 0));
  {
    const unsigned gb = (unsigned)std::min<uint64_t>((q.max_big + 255) / 256, (uint64_t)sms * 4);
    const uint64_t tiles = std::max<uint64_t>(1, (q.max_big + 1 + kScanTile - 1) / kScanTile);
    // side-stream scans use the tail of the status area (the main stream's units kernel needs none)
    uint64_t* status = w.status;
    GT_CUDA(cudaMemsetAsync(status, 0, tiles * 8, sb));
    GT_CUDA(cudaMemsetAsync(w.ctr, 0, 4, sb));
    GT_CUDA(cudaMemsetAsync(w.bnt, 0, (q.max_big + 1) * 4, sb));
    k_big_nt<<<gb, 256, 0, sb>>>(w.bigs, w.cnt + 1, w.bnt);
    k_scan_lookback<uint32_t><<<(unsigned)tiles, kScanThreads, 0, sb>>>(w.bnt, q.max_big + 1, w.bfirst, 0, 1, status,
                                                                         w.ctr, w.cnt + 1, 1);
    GT_LAUNCH_CHECK();
    k_big_write<<<gb, 256, 0, sb>>>(w.bigs, w.cnt + 1, w.bfirst, p.c, w.tiles3, w.cnt + 2, w.seg3);
    GT_LAUNCH_CHECK();
    const unsigned gt3 = (unsigned)std::min<uint64_t>(q.max_t3, (uint64_t)sms * 8);
    if ((rc = set_smem(k_cnt_rec, (size_t)Dc * 4))) return rc;
    if ((rc = set_smem(k_cnt_lv, (size_t)Dc * 4))) return rc;
    if (p.wide) k_cnt_lv<<<gt3, 512, (size_t)Dc * 4, sb>>>(w.r2lv, w.tiles3, w.cnt + 2, Dc, w.cnt3);
    else k_cnt_rec<<<gt3, 512, (size_t)Dc * 4, sb>>>(w.r2, w.tiles3, w.cnt + 2, Dc, DigSM{p.nbs, (uint32_t)(Dc - 1)}, w.cnt3);
    GT_LAUNCH_CHECK();
    {  // scan only the real tiles' rows: n = n_tiles3 * Dc (device count)
      const uint64_t n3 = q.max_t3 * (uint64_t)Dc;
      const uint64_t t3 = std::max<uint64_t>(1, (n3 + kScanTile - 1) / kScanTile);
      GT_CUDA(cudaMemsetAsync(status, 0, t3 * 8, sb));
      GT_CUDA(cudaMemsetAsync(w.ctr, 0, 4, sb));
      k_scan_lookback<uint32_t><<<(unsigned)t3, kScanThreads, 0, sb>>>(w.cnt3, n3, w.base3, 0, 0, status, w.ctr,
                                                                        w.cnt + 2, (uint64_t)Dc);
      GT_LAUNCH_CHECK();
    }
    k_segfix<<<(unsigned)std::min<uint64_t>(q.max_big, (uint64_t)sms * 8), 512, 0, sb>>>(w.seg3, w.cnt + 1, Dc, w.base3,
                                                                                      t_offsets, V, w.err);
    GT_LAUNCH_CHECK();
    DecR2 dec;
    dec.nbs = p.nbs;
    dec.src_mask = (p.nbs >= 32 || p.wide) ? 0xffffffffu : (uint32_t)((1ull << p.nbs) - 1);
    dec.maskC = (uint32_t)(Dc - 1);
    if ((rc = tm.kbegin(3, sb))) return rc;
    if (p.wide) {
      auto kern = k_p2<kMode, DecR2, 16, false, kIoLv>;
      const size_t sm = smem_p2(Dc, kMode, 16, kIoLv);
      if ((rc = set_smem(kern, sm))) return rc;
      kern<<<persistent_grid(kern, T, sm, q.max_t3), T, sm, sb>>>(w.r2, w.tiles3, w.cnt + 2, Dc, dec, w.base3, t_edges,
                                                                   nullptr, w.r2lv, nullptr);
    } else {  // batched landing loads (C3 big buckets 0.85 -> 0.78 ms)
      auto kern = (p.exp & 4096) ? k_p2<kMode, DecR2, 16, false, kIoPlain, true, W, 4, true, false> : k_p2<kMode, DecR2, 16>;
      const size_t sm = smem_p2(Dc, kMode, 16);
      if ((rc = set_smem(kern, sm))) return rc;
      kern<<<persistent_grid(kern, T, sm, q.max_t3), T, sm, sb>>>(w.r2, w.tiles3, w.cnt + 2, Dc, dec, w.base3, t_edges,
                                                                   nullptr, nullptr, nullptr);
    }
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(3, sb))) return rc;
  }
  {
    P3Args a;
    a.rec = w.r2;
    a.units = w.units;
    a.n_units = w.cnt + 0;
    a.ctr = w.cnt + 3;
    a.c = p.c;
    a.nbs = p.nbs;
    a.src_mask = (p.nbs >= 32 || p.wide) ? 0xffffffffu : (uint32_t)((1ull << p.nbs) - 1);
    a.mask_c = (uint32_t)(Dc - 1);
    a.lv = w.r2lv;
    a.fbase = w.fbase;
    a.gbits = g3;
    a.lvmask = (uint32_t)((1ull << (p.c + g3)) - 1);
    a.V = V;
    a.t_offsets = t_offsets;
    a.t_edges = t_edges;
    a.prof = nullptr;
    const size_t sm = smem_p3(kMode, p.wide, 16);
    auto go3 = [&](auto kern) -> int {
      int r;
      if ((r = set_smem(kern, sm))) return r;
      kern<<<persistent_grid(kern, 512, sm, q.nfine), 512, sm, st>>>(a);
      return GT_OK;
    };
    if ((rc = tm.kbegin(2))) return rc;
    // units: 16 warps x K = 16 (8192 records, 2 CTAs/SM), records split evenly over the warps;
    // batched landing loads where fine buckets come from positions (C4 4.40 -> 4.33 ms)
    if (p.wide) rc = go3(k_p3<kMode, true, false, true>);
    else if (pos_fine) rc = go3(k_p3<kMode, true>);
    else rc = (p.exp & 4096) ? go3(k_p3<kMode, false, false, false, false, W3, true, false>)
                             : go3(k_p3<kMode, false, false, false, false>);
    if (rc) return rc;
    GT_LAUNCH_CHECK();
    if ((rc = tm.kend(2))) return rc;
  }
  GT_CUDA(cudaEventRecord(ev_join, sb));
  GT_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  k_set_u64<<<1, 1, 0, st>>>(t_offsets + V, E);
  GT_LAUNCH_CHECK();
  *launches += 11;  // set, plan, big: tiles count / scan / write, count, scan, segfix, place; units; set
  return GT_OK;
}

__global__ void k_status_out(const unsigned int* err, int* status) { *status = *err ? GT_EOVERFLOW : GT_OK; }

// Sender meta: per-bucket record counts and the shard's first source-high
// value in entry 0 of every seg_hi row.
__global__ void k_sender_meta(const uint64_t* __restrict__ tbase, uint64_t ntiles1, int D1, uint64_t E,
                              const uint32_t* __restrict__ prev, int L, uint64_t* __restrict__ counts,
                              uint64_t* __restrict__ seg_hi, uint64_t nh) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < D1; c += gridDim.x * blockDim.x) {
    const uint64_t s = tbase[(uint64_t)c * ntiles1];
    const uint64_t e = (c + 1 < D1) ? tbase[(uint64_t)(c + 1) * ntiles1] : E;
    counts[c] = e - s;
    seg_hi[(uint64_t)c * (nh + 1)] = (uint64_t)(prev[0] >> L);
  }
}

int fill_stats(const Plan& p, int mode, Timer& tm, gt_stats* stats, uint64_t ws_bytes, int launches,
               uint64_t n_big) {
  float a = 0, b = 0, c = 0, t = 0;
  GT_CUDA(cudaEventElapsedTime(&a, tm.ev[0], tm.ev[1]));
  GT_CUDA(cudaEventElapsedTime(&b, tm.ev[1], tm.ev[2]));
  GT_CUDA(cudaEventElapsedTime(&c, tm.ev[2], tm.ev[3]));
  GT_CUDA(cudaEventElapsedTime(&t, tm.ev[0], tm.ev[3]));
  stats->ms_step1 = a;
  stats->ms_step2 = b;
  stats->ms_step3 = c;
  stats->ms_total = t;
  stats->workspace_bytes = ws_bytes;
  stats->bits[0] = p.a;
  stats->bits[1] = p.b;
  stats->bits[2] = p.c;
  stats->rank_mode = mode;
  stats->n_big_buckets = n_big;
  stats->n_launches = (uint64_t)launches;
  for (int k = 0; k < Timer::kKern; ++k) {
    float x = 0;
    if (tm.kset[k]) GT_CUDA(cudaEventElapsedTime(&x, tm.kev[2 * k], tm.kev[2 * k + 1]));
    stats->ms_kernel[k] = x;
  }
  return GT_OK;
}

// Stats path: wait for the call, read the big-bucket count and the overflow flag.
int finish_stats(const Plan& p, int mode, Timer& tm, Ws& w, gt_stats* stats, uint64_t ws_bytes, int launches,
                 cudaStream_t st) {
  uint32_t h_big = 0;
  unsigned int h_err = 0;
  GT_CUDA(cudaMemcpyAsync(&h_big, w.cnt + 1, 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&h_err, w.err, 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  int rc = fill_stats(p, mode, tm, stats, ws_bytes, launches, h_big);
  if (rc) return rc;
  if (h_err) return set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
  return GT_OK;
}

// Whole single-GPU transpose (levels 1-3); R1 lives in t_edges.
template <int kMode>
int transpose_one(const Plan& p, const Layout& q, unsigned char* ws, InCsr in, uint64_t* t_offsets, uint32_t* t_edges,
                  cudaStream_t st, Timer& tm, int* launches, Ws* wout) {
  Ws w = ws_ptrs(q, ws, p);
  *wout = w;
  int rc;
  GT_CUDA(cudaMemsetAsync(w.err, 0, 4, st));
  if ((rc = tm.mark())) return rc;
  if ((rc = level1<kMode>(p, q, w, in, p.E, false, t_edges, st, tm, launches))) return rc;
  if ((rc = tm.mark())) return rc;
  v3::k_runs_from_tbase<<<(p.D1 + 255) / 256, 256, 0, st>>>(w.tbase, q.ntiles1, p.D1, p.E, w.runs);
  GT_LAUNCH_CHECK();
  *launches += 1;
  if ((rc = level23<kMode>(p, q, w, t_edges, 1, 0, w.seghi, t_offsets, t_edges, st, tm, launches))) return rc;
  if ((rc = tm.mark())) return rc;
  return GT_OK;
}

// ---------------------------------------------------------------- slab mode
// num_vertices > 2^29: the destinations split into slabs of 2^29 IDs; slab s
// runs level 1 over the whole edge stream keeping only its destinations
// (k_c1 / k_p1 kSlab), writing R1 into t_edges at the slab's CSC start, then
// levels 2-3 with the slab's local IDs, offsets rebased.  One host read (the
// per-slab edge counts) per call.
constexpr int kSlabBits = 29;
__global__ void k_fill_u64(uint64_t* a, uint64_t n, uint64_t v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// Plan and layout every slab uses (the split from the whole edge count, so it
// does not depend on the slab sizes; tables sized for all E records).
int slab_plan(uint64_t V, uint64_t E, uint32_t s, const gt_config& cfg, Plan& p, Layout& q) {
  const uint64_t Vs = std::min<uint64_t>(1ull << kSlabBits, V - ((uint64_t)s << kSlabBits));
  gt_config c = cfg;
  c.force_wide = 1;  // 64-bit positions and source-array R2 for 30-32-bit source IDs
  int rc = make_plan(Vs, E, V, c, p);
  if (rc) return rc;
  if (!p.wide) return set_err(GT_EINVAL, "slab mode needs the wide form");
  make_layout(p, E, E, 1, q);
  return GT_OK;
}

__global__ void k_or_flag(const unsigned int* __restrict__ src, unsigned int* __restrict__ dst) {
  if (*src) *dst = 1u;
}

// ws: 256 bytes of slab-mode state (the accumulated overflow flag at ws[0]),
// then the slab layouts (plans differ per slab, so their offsets do too).
template <int kMode>
int transpose_slabs(uint64_t V, uint64_t E, const gt_config& cfg, unsigned char* ws, InCsr in, uint64_t* t_offsets,
                    uint32_t* t_edges, const uint64_t* slab_counts, cudaStream_t st, int* launches) {
  const uint32_t S = (uint32_t)((V + (1ull << kSlabBits) - 1) >> kSlabBits);
  unsigned int* err_all = reinterpret_cast<unsigned int*>(ws);
  GT_CUDA(cudaMemsetAsync(err_all, 0, 4, st));
  uint64_t before = 0;
  int rc;
  Timer tm;
  tm.init(false, st);
  for (uint32_t s = 0; s < S; ++s) {
    Plan p;
    Layout q;
    if ((rc = slab_plan(V, E, s, cfg, p, q))) return rc;
    Ws w = ws_ptrs(q, ws + 256, p);
    GT_CUDA(cudaMemsetAsync(w.err, 0, 4, st));
    const uint64_t v0 = (uint64_t)s << kSlabBits, Es = slab_counts[s];
    if (Es == 0) {  // no destination in the slab: every offset is the slab's start
      k_fill_u64<<<64, 256, 0, st>>>(t_offsets + v0, p.V + 1, before);
      GT_LAUNCH_CHECK();
      *launches += 1;
      continue;
    }
    p.E = Es;
    const uint32_t mask = ~((1u << kSlabBits) - 1u), val = s << kSlabBits;
    if ((rc = level1<kMode>(p, q, w, in, E, false, t_edges + before, st, tm, launches, mask, val))) return rc;
    v3::k_runs_from_tbase<<<(p.D1 + 255) / 256, 256, 0, st>>>(w.tbase, q.ntiles1, p.D1, Es, w.runs);
    GT_LAUNCH_CHECK();
    if ((rc = level23<kMode>(p, q, w, t_edges + before, 1, 0, w.seghi, t_offsets + v0, t_edges + before, st, tm,
                             launches)))
      return rc;
    if (before) {
      k_add_base<<<148, 256, 0, st>>>(t_offsets + v0, p.V + 1, before);
      GT_LAUNCH_CHECK();
    }
    k_or_flag<<<1, 1, 0, st>>>(w.err, err_all);
    GT_LAUNCH_CHECK();
    *launches += 3;
    before += Es;
  }
  return GT_OK;
}

// ---------------------------------------------------------------- pipelined host call
// gt_transpose_host for one graph: the PCIe copies are the floor (H2D then D2H,
// ~41 + 40 ms for C3), so the kernels hide under them.  The edges arrive in P
// source chunks; chunk s runs level 1 as a sender (the multi-GPU building
// block) while chunk s+1 is still copying, writing its R1 at its edge offset of
// one buffer.  After one host read of the P x D1 bucket counts, levels 2-3 run
// per group of coarse buckets (balanced on records, the multi-GPU owner rule)
// with one run per (bucket, sender); group g's CSC range is copied back while
// group g+1 is computed.  Device buffers are cached per device (grow-only).
struct HostPipe {
  cudaEvent_t tev[8] = {};  // timing marks: start, copy-in end, level 1 end, group 0 end, groups end, copy-back end
  std::vector<cudaEvent_t> gev;  // experiment bit 256: per-group compute end / copy-back end
  void* io = nullptr;  // offsets, t_offsets, edges, t_edges, R1, seg rows, counts, flag, sender workspace
  uint64_t io_bytes = 0;
  void* rws = nullptr;  // receiver workspace (levels 2-3 of one group)
  uint64_t rws_bytes = 0;
  uint64_t* h_counts = nullptr;  // pinned P x D1
  uint64_t h_counts_n = 0;
  cudaStream_t sin = nullptr, scmp = nullptr, sout = nullptr;
  std::vector<cudaEvent_t> ev;
};

int pipe_events(HostPipe& hp, size_t n) {
  while (hp.ev.size() < n) {
    cudaEvent_t e;
    GT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    hp.ev.push_back(e);
  }
  return GT_OK;
}

// Source chunks and bucket groups: config override (reserved[1] / reserved[2];
// reserved[1] < 0: the serial call), else one per 2^26 edges, 2..8 of each;
// graphs under 2^24 edges, wide or slab plans take the serial call (P = 0).
void pipe_shape(const Plan& p, uint64_t V, uint64_t E, const gt_config& cfg, int* P, int* G) {
  *P = *G = 0;
  if (p.wide || V > (1ull << kSlabBits) || E == 0 || cfg.reserved[1] < 0) return;
  const bool forced = cfg.reserved[1] > 0 || cfg.reserved[2] > 0;
  if (!forced && E < (1ull << 24)) return;
  const int autoN = (int)std::min<uint64_t>(8, std::max<uint64_t>(2, (E + (1ull << 26) - 1) >> 26));
  *P = cfg.reserved[1] > 0 ? std::min(cfg.reserved[1], 64) : autoN;
  *G = cfg.reserved[2] > 0 ? std::min(cfg.reserved[2], p.D1) : std::min(autoN, p.D1);
}

template <int kMode>
int host_pipeline(HostPipe& hp, const Plan& p, int P, int G, const uint64_t* h_offsets, const uint32_t* h_edges,
                  uint64_t V, uint64_t E, uint64_t* h_t_offsets, uint32_t* h_t_edges, int* status_out,
                  gt_stats* stats) {
  int rc;
  const int D1 = p.D1;
  const uint64_t nh = 1ull << p.nsh;
  // source chunks: vertex-aligned, edge-balanced (_nb.py:118-132)
  std::vector<int64_t> vb(P + 1);
  if ((rc = gt_edge_balanced_bounds(h_offsets, V, P, vb.data()))) return rc;
  std::vector<uint64_t> es(P + 1);
  for (int s = 0; s <= P; ++s) es[s] = h_offsets[vb[s]];
  uint64_t max_chunk = 0;
  for (int s = 0; s < P; ++s) max_chunk = std::max(max_chunk, es[s + 1] - es[s]);
  Plan ps = p;
  ps.E = max_chunk;
  Layout qs;
  make_layout(ps, max_chunk, 0, 1, qs);
  // io buffer
  const uint64_t b_off = align_up((V + 1) * 8, 256), b_e = align_up(E * 4, 256);
  const uint64_t b_seg = align_up((uint64_t)P * D1 * (nh + 1) * 8, 256), b_cnt = align_up((uint64_t)P * D1 * 8, 256);
  const uint64_t need = 2 * b_off + 3 * b_e + b_seg + b_cnt + 256 + qs.total;
  if (hp.io_bytes < need) {
    if (hp.io) GT_CUDA(cudaFreeAsync(hp.io, hp.scmp));
    hp.io = nullptr;
    hp.io_bytes = 0;
    GT_CUDA(cudaMallocAsync(&hp.io, need, hp.scmp));
    hp.io_bytes = need;
  }
  unsigned char* b = static_cast<unsigned char*>(hp.io);
  uint64_t* d_off = reinterpret_cast<uint64_t*>(b);
  uint64_t* d_toff = reinterpret_cast<uint64_t*>(b + b_off);
  uint32_t* d_e = reinterpret_cast<uint32_t*>(b + 2 * b_off);
  uint32_t* d_te = reinterpret_cast<uint32_t*>(b + 2 * b_off + b_e);
  uint32_t* d_r1 = reinterpret_cast<uint32_t*>(b + 2 * b_off + 2 * b_e);
  uint64_t* seg_all = reinterpret_cast<uint64_t*>(b + 2 * b_off + 3 * b_e);
  uint64_t* counts = reinterpret_cast<uint64_t*>(b + 2 * b_off + 3 * b_e + b_seg);
  unsigned int* err = reinterpret_cast<unsigned int*>(b + 2 * b_off + 3 * b_e + b_seg + b_cnt);
  unsigned char* sws = b + 2 * b_off + 3 * b_e + b_seg + b_cnt + 256;
  if ((rc = pipe_events(hp, (size_t)P + G))) return rc;
  if (!hp.tev[0])
    for (auto& e : hp.tev) GT_CUDA(cudaEventCreate(&e));
  while ((p.exp & 256) && hp.gev.size() < 2 * (size_t)G) {
    cudaEvent_t e;
    GT_CUDA(cudaEventCreate(&e));
    hp.gev.push_back(e);
  }
  GT_CUDA(cudaMemsetAsync(err, 0, 4, hp.scmp));
  GT_CUDA(cudaEventRecord(hp.ev[0], hp.scmp));  // the buffers are allocated / free of the previous call
  GT_CUDA(cudaStreamWaitEvent(hp.sin, hp.ev[0], 0));
  GT_CUDA(cudaEventRecord(hp.tev[0], hp.sin));
  GT_CUDA(cudaMemcpyAsync(d_off, h_offsets, (V + 1) * 8, cudaMemcpyHostToDevice, hp.sin));
  Timer tm;
  tm.init(false, hp.scmp);
  int launches = 0;
  for (int s = 0; s < P; ++s) {  // chunk s copies in while chunk s-1 runs level 1
    const uint64_t n = es[s + 1] - es[s], ea = es[s] & ~1023ull;  // 4 KB-aligned start (same bytes twice)
    if (n) GT_CUDA(cudaMemcpyAsync(d_e + ea, h_edges + ea, (es[s + 1] - ea) * 4, cudaMemcpyHostToDevice, hp.sin));
    GT_CUDA(cudaEventRecord(hp.ev[s], hp.sin));
    GT_CUDA(cudaStreamWaitEvent(hp.scmp, hp.ev[s], 0));
    uint64_t* seg = seg_all + (uint64_t)s * D1 * (nh + 1);
    if (n == 0) {
      GT_CUDA(cudaMemsetAsync(counts + (uint64_t)s * D1, 0, (uint64_t)D1 * 8, hp.scmp));
      GT_CUDA(cudaMemsetAsync(seg, 0xff, (uint64_t)D1 * (nh + 1) * 8, hp.scmp));
      continue;
    }
    Plan pc = p;
    pc.E = n;
    Layout qc;
    make_layout(pc, n, 0, 1, qc);
    Ws w = ws_ptrs(qc, sws, pc);
    w.seghi = seg;
    const InCsr in{d_off, d_e + es[s], es[s], V};
    if ((rc = level1<kMode>(pc, qc, w, in, n, true, d_r1 + es[s], hp.scmp, tm, &launches))) return rc;
    k_sender_meta<<<(D1 + 255) / 256, 256, 0, hp.scmp>>>(w.tbase, qc.ntiles1, D1, n, w.prev, p.L,
                                                          counts + (uint64_t)s * D1, seg, nh);
    GT_LAUNCH_CHECK();
  }
  GT_CUDA(cudaEventRecord(hp.tev[1], hp.sin));
  GT_CUDA(cudaEventRecord(hp.tev[2], hp.scmp));
  // the one host read: bucket counts -> record-balanced groups of buckets
  const uint64_t ncnt = (uint64_t)P * D1;
  if (hp.h_counts_n < ncnt) {
    if (hp.h_counts) GT_CUDA(cudaFreeHost(hp.h_counts));
    hp.h_counts = nullptr;
    hp.h_counts_n = 0;
    GT_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hp.h_counts), ncnt * 8));
    hp.h_counts_n = ncnt;
  }
  GT_CUDA(cudaMemcpyAsync(hp.h_counts, counts, ncnt * 8, cudaMemcpyDeviceToHost, hp.scmp));
  GT_CUDA(cudaStreamSynchronize(hp.scmp));
  std::vector<uint64_t> tot(D1, 0), bstart(D1 + 1, 0);
  for (int s = 0; s < P; ++s)
    for (int c = 0; c < D1; ++c) tot[c] += hp.h_counts[(uint64_t)s * D1 + c];
  for (int c = 0; c < D1; ++c) bstart[c + 1] = bstart[c] + tot[c];
  if (bstart[D1] != E) return set_err(GT_ECUDA, "pipelined transpose: bucket counts sum to %llu, expected %llu",
                                      (unsigned long long)bstart[D1], (unsigned long long)E);
  std::vector<uint32_t> gb(G + 1);
  if ((rc = gt_shard_owners(tot.data(), (uint32_t)D1, G, gb.data()))) return rc;
  const int shift = p.b + p.c;
  uint64_t rneed = 0;
  for (int g = 0; g < G; ++g) {
    Plan pl = p;
    pl.D1 = (int)(gb[g + 1] - gb[g]);
    pl.E = bstart[gb[g + 1]] - bstart[gb[g]];
    if (!pl.D1 || !pl.E) continue;
    Layout q;
    make_layout(pl, 0, pl.E, (uint32_t)P, q);
    rneed = std::max(rneed, q.total);
  }
  if (hp.rws_bytes < rneed) {
    if (hp.rws) GT_CUDA(cudaFreeAsync(hp.rws, hp.scmp));
    hp.rws = nullptr;
    hp.rws_bytes = 0;
    GT_CUDA(cudaMallocAsync(&hp.rws, rneed, hp.scmp));
    hp.rws_bytes = rneed;
  }
  // group g's CSC range (t_offsets[v_hi] belongs to the next group) back to the host
  auto copy_back = [&](int g) -> int {
    const uint32_t lo = gb[g], nloc = gb[g + 1] - gb[g];
    const uint64_t v_lo = std::min<uint64_t>(V, (uint64_t)lo << shift);
    const uint64_t v_hi = (g + 1 == G) ? V : std::min<uint64_t>(V, (uint64_t)gb[g + 1] << shift);
    const uint64_t e0 = bstart[lo], Eg = bstart[lo + nloc] - e0;
    const uint64_t noff = (v_hi - v_lo) + (g + 1 == G ? 1 : 0);
    // copies start on 4 KB boundaries (unaligned DMA measured 52 vs 57 GB/s): the
    // head re-copies final data of group g-1; copies are ordered on sout, so
    // nothing earlier can overwrite it
    const uint64_t ea = e0 & ~1023ull, va = v_lo & ~511ull;
    GT_CUDA(cudaStreamWaitEvent(hp.sout, hp.ev[P + g], 0));
    if (Eg) GT_CUDA(cudaMemcpyAsync(h_t_edges + ea, d_te + ea, (e0 + Eg - ea) * 4, cudaMemcpyDeviceToHost, hp.sout));
    if (noff)
      GT_CUDA(cudaMemcpyAsync(h_t_offsets + va, d_toff + va, (v_lo + noff - va) * 8, cudaMemcpyDeviceToHost, hp.sout));
    if (p.exp & 256) GT_CUDA(cudaEventRecord(hp.gev[2 * g + 1], hp.sout));
    return GT_OK;
  };
  auto is_pinned = [](const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool pinned_out = is_pinned(h_t_edges) && is_pinned(h_t_offsets);
  // groups: levels 2-3 on the compute stream, each followed by its copy-back
  for (int g = 0; g < G; ++g) {
    const uint32_t lo = gb[g], nloc = gb[g + 1] - gb[g];
    const uint64_t v_lo = std::min<uint64_t>(V, (uint64_t)lo << shift);
    const uint64_t v_hi = (g + 1 == G) ? V : std::min<uint64_t>(V, (uint64_t)gb[g + 1] << shift);
    const uint64_t Vloc = v_hi - v_lo, e0 = bstart[lo], Eg = bstart[lo + nloc] - e0;
    if (Vloc && !Eg) {
      k_fill_u64<<<64, 256, 0, hp.scmp>>>(d_toff + v_lo, Vloc + 1, e0);
      GT_LAUNCH_CHECK();
    } else if (Vloc) {
      Plan pl = p;
      pl.D1 = (int)nloc;
      pl.V = Vloc;
      pl.E = Eg;
      Layout q;
      make_layout(pl, 0, Eg, (uint32_t)P, q);
      Ws w = ws_ptrs(q, static_cast<unsigned char*>(hp.rws), pl);
      w.err = err;
      v3::k_runs_senders<<<(unsigned)((nloc * P + 127) / 128), 128, 0, hp.scmp>>>(counts, (uint32_t)P, (uint32_t)D1, lo,
                                                                               nloc, w.runs, seg_all, (uint32_t)nh);
      GT_LAUNCH_CHECK();
      if ((rc = level23<kMode>(pl, q, w, d_r1, (uint32_t)P, (uint32_t)D1, seg_all + (uint64_t)lo * (nh + 1),
                               d_toff + v_lo, d_te + e0, hp.scmp, tm, &launches)))
        return rc;
      if (e0) {
        k_add_base<<<148, 256, 0, hp.scmp>>>(d_toff + v_lo, Vloc + 1, e0);
        GT_LAUNCH_CHECK();
      }
    }
    GT_CUDA(cudaEventRecord(hp.ev[P + g], hp.scmp));
    if (g == 0) GT_CUDA(cudaEventRecord(hp.tev[3], hp.scmp));
    if (p.exp & 256) GT_CUDA(cudaEventRecord(hp.gev[2 * g], hp.scmp));
    if (pinned_out && (rc = copy_back(g))) return rc;
  }
  GT_CUDA(cudaEventRecord(hp.tev[4], hp.scmp));
  int dev = 0;
  GT_CUDA(cudaGetDevice(&dev));
  WsEntry* ent;
  if ((rc = ws_entry(dev, hp.scmp, &ent))) return rc;
  k_status_out<<<1, 1, 0, hp.scmp>>>(err, ent->status);
  GT_LAUNCH_CHECK();
  // pageable host buffers make the copies synchronous: enqueue them after every
  // compute launch so that they do not hold back the kernels
  if (!pinned_out)
    for (int g = 0; g < G; ++g)
      if ((rc = copy_back(g))) return rc;
  GT_CUDA(cudaEventRecord(hp.tev[5], hp.sout));
  GT_CUDA(cudaStreamSynchronize(hp.sout));
  GT_CUDA(cudaStreamSynchronize(hp.scmp));
  *status_out = *reinterpret_cast<volatile int*>(ent->status);
  float t[6] = {};
  for (int k = 1; k < 6; ++k) GT_CUDA(cudaEventElapsedTime(&t[k], hp.tev[0], hp.tev[k]));
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->ms_total = t[5];
    stats->ms_step1 = t[2];
    stats->ms_step2 = t[4] - t[2];
    stats->ms_step3 = t[5] - t[4];
    stats->workspace_bytes = hp.io_bytes + hp.rws_bytes;
    stats->bits[0] = p.a;
    stats->bits[1] = p.b;
    stats->bits[2] = p.c;
    stats->rank_mode = kMode;
    stats->n_launches = (uint64_t)launches + 1;
  }
  if (p.exp & 256)
    std::fprintf(stderr, "host pipeline P=%d G=%d: copy-in end %.2f, level 1 end %.2f, group 0 end %.2f, groups end %.2f, copy-back end %.2f ms\n",
                 P, G, t[1], t[2], t[3], t[4], t[5]);
  if (p.exp & 256) {
    for (int g = 0; g < G; ++g) {
      float a = 0, c = 0;
      GT_CUDA(cudaEventElapsedTime(&a, hp.tev[0], hp.gev[2 * g]));
      GT_CUDA(cudaEventElapsedTime(&c, hp.tev[0], hp.gev[2 * g + 1]));
      std::fprintf(stderr, "  group %d: computed %.2f, copied back %.2f ms\n", g, a, c);
    }
  }
  return GT_OK;
}

}  // namespace

// ---------------------------------------------------------------- internal API (gt_multi.cu)
int gt_internal_shard_geometry(uint64_t V, uint64_t E, gt_shard_geom* g) {
  Plan p;
  int rc = make_plan(V, E, V, config_snapshot(), p);
  if (rc) return rc;
  std::memset(g, 0, sizeof(*g));
  g->num_buckets = (uint32_t)p.D1;
  g->bucket_shift = (uint32_t)(p.b + p.c);
  g->seg_hi_row = (uint32_t)((1ull << p.nsh) + 1);
  g->wide = p.wide ? 1 : 0;
  g->bits[0] = p.a;
  g->bits[1] = p.b;
  g->bits[2] = p.c;
  return GT_OK;
}

extern "C" {

int gt_abi_version(void) { return GT_ABI_VERSION; }
const char* gt_last_error(void) { return g_err.c_str(); }

int gt_set_config(const gt_config* cfg) {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  if (cfg) g_cfg = *cfg;
  else g_cfg = gt_config{{0, 0, 0}, 0, {0, 0, 0, 0}};
  return GT_OK;
}

int gt_get_config(gt_config* cfg) {
  if (!cfg) return set_err(GT_EINVAL, "cfg is NULL");
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  *cfg = g_cfg;
  return GT_OK;
}

int gt_workspace_size(uint64_t V, uint64_t E, uint64_t* bytes) {
  if (!bytes) return set_err(GT_EINVAL, "bytes is NULL");
  if (E == 0 || V == 0) {
    *bytes = 0;
    return GT_OK;
  }
  if (bits_for(V) > kSlabBits) {  // slab mode: the largest slab layout
    uint64_t mx = 0;
    for (uint32_t s = 0; ((uint64_t)s << kSlabBits) < V; ++s) {
      Plan p;
      Layout q;
      int rc = slab_plan(V, E, s, config_snapshot(), p, q);
      if (rc) return rc;
      mx = std::max(mx, q.total);
    }
    *bytes = mx + 256;  // + the slab-mode state
    return GT_OK;
  }
  Plan p;
  int rc = make_plan(V, E, V, config_snapshot(), p);
  if (rc) return rc;
  Layout q;
  make_layout(p, E, E, 1, q);
  *bytes = q.total;
  return GT_OK;
}

int gt_set_rank_mode(int mode) {
  if (mode < -1 || mode > 1) return set_err(GT_EINVAL, "rank mode must be -1, 0 or 1");
  std::lock_guard<std::mutex> lk(g_mu);
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
  WsEntry* ent;
  if ((rc = ws_entry(dev, st, &ent))) return rc;
  std::lock_guard<std::mutex> call(ent->call_mu);
  if (E == 0) {
    GT_CUDA(cudaMemsetAsync(t_offsets, 0, (V + 1) * 8, st));
    GT_CUDA(cudaMemsetAsync(ent->status, 0, sizeof(int), st));
    if (stats) GT_CUDA(cudaStreamSynchronize(st));
    return GT_OK;
  }
  if (bits_for(V) > kSlabBits) {  // num_vertices > 2^29: slab mode
    const gt_config cfg = config_snapshot();
    uint64_t need = 0;
    if ((rc = gt_workspace_size(V, E, &need))) return rc;
    unsigned char* ws = static_cast<unsigned char*>(workspace);
    if (!ws) {
      if ((rc = ws_get(dev, st, need, &ws, nullptr))) return rc;
    } else if (ws_bytes < need) {
      return set_err(GT_ENOMEM, "workspace too small: need %llu bytes, got %llu", (unsigned long long)need,
                     (unsigned long long)ws_bytes);
    }
    unsigned long long* d_cnt = nullptr;
    unsigned long long h_cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    GT_CUDA(cudaMallocAsync(&d_cnt, 64, st));
    GT_CUDA(cudaMemsetAsync(d_cnt, 0, 64, st));
    v3::k_slab_hist<<<(unsigned)(num_sms() * 4), 256, 0, st>>>(edges, E, d_cnt);
    GT_LAUNCH_CHECK();
    GT_CUDA(cudaMemcpyAsync(h_cnt, d_cnt, 64, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaFreeAsync(d_cnt, st));
    GT_CUDA(cudaStreamSynchronize(st));  // the per-slab edge counts size the slabs' passes
    uint64_t cnt[8];
    for (int i = 0; i < 8; ++i) cnt[i] = h_cnt[i];
    int mode;
    if ((rc = rank_mode_for(dev, st, &mode))) return rc;
    const InCsr in{offsets, edges, 0, V};
    int launches = 2;
    rc = (mode == kRankAtomic) ? transpose_slabs<kRankAtomic>(V, E, cfg, ws, in, t_offsets, t_edges, cnt, st, &launches)
                               : transpose_slabs<kRankSafe>(V, E, cfg, ws, in, t_offsets, t_edges, cnt, st, &launches);
    if (rc) return rc;
    const unsigned int* err_all = reinterpret_cast<const unsigned int*>(ws);
    k_status_out<<<1, 1, 0, st>>>(err_all, ent->status);
    GT_LAUNCH_CHECK();
    if (stats) {
      unsigned int h_err = 0;
      GT_CUDA(cudaMemcpyAsync(&h_err, err_all, 4, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      stats->workspace_bytes = need;
      stats->rank_mode = mode;
      stats->n_launches = (uint64_t)launches + 1;
      if (h_err) return set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
    }
    return GT_OK;
  }
  Plan p;
  if ((rc = make_plan(V, E, V, config_snapshot(), p))) return rc;
  Layout q;
  make_layout(p, E, E, 1, q);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  if (!ws) {
    if ((rc = ws_get(dev, st, q.total, &ws, nullptr))) return rc;
  } else if (ws_bytes < q.total) {
    return set_err(GT_ENOMEM, "workspace too small: need %llu bytes, got %llu", (unsigned long long)q.total,
                   (unsigned long long)ws_bytes);
  }
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  Timer tm;
  if ((rc = tm.init(stats != nullptr, st))) return rc;
  const InCsr in{offsets, edges, 0, V};
  int launches = 0;
  Ws w;
  rc = (mode == kRankAtomic) ? transpose_one<kRankAtomic>(p, q, ws, in, t_offsets, t_edges, st, tm, &launches, &w)
                             : transpose_one<kRankSafe>(p, q, ws, in, t_offsets, t_edges, st, tm, &launches, &w);
  if (rc) return rc;
  k_status_out<<<1, 1, 0, st>>>(w.err, ent->status);
  GT_LAUNCH_CHECK();
  if (stats) return finish_stats(p, mode, tm, w, stats, q.total, launches + 1, st);
  return GT_OK;
}

int gt_transpose_status(void* stream, int* status) {
  if (!status) return set_err(GT_EINVAL, "status is NULL");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  WsEntry* ent;
  if ((rc = ws_entry(dev, static_cast<cudaStream_t>(stream), &ent))) return rc;
  *status = *reinterpret_cast<volatile int*>(ent->status);
  if (*status == GT_EOVERFLOW)
    set_err(GT_EOVERFLOW, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
  return GT_OK;
}

int gt_release_workspace(void) {
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  GT_CUDA(cudaDeviceSynchronize());
  std::vector<WsEntry*> mine;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& kv : g_ws)
      if (kv.first.first == dev) mine.push_back(&kv.second);  // entries are never erased
  }
  for (WsEntry* e : mine) {  // lock order of the calls: call_mu, then g_ws_mu
    std::lock_guard<std::mutex> call(e->call_mu);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (e->ptr) GT_CUDA(cudaFree(e->ptr));
    e->ptr = nullptr;
    e->bytes = 0;
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
  if (h_offsets[V] != E)
    return set_err(GT_EINVAL, "offsets[num_vertices] = %llu != num_edges = %llu", (unsigned long long)h_offsets[V],
                   (unsigned long long)E);
  {  // large compact graphs: the pipelined call (copies overlap the kernels)
    const gt_config cfg = config_snapshot();
    Plan p;
    int P = 0, G = 0;
    if (make_plan(V, E, V, cfg, p) == GT_OK) pipe_shape(p, V, E, cfg, &P, &G);
    if (P) {
      static HostPipe s_pipe[64];
      static std::mutex s_pipe_mu;
      std::lock_guard<std::mutex> lk(s_pipe_mu);
      HostPipe& hp = s_pipe[device];
      if (!hp.scmp) {
        GT_CUDA(cudaStreamCreateWithFlags(&hp.sin, cudaStreamNonBlocking));
        GT_CUDA(cudaStreamCreateWithFlags(&hp.scmp, cudaStreamNonBlocking));
        GT_CUDA(cudaStreamCreateWithFlags(&hp.sout, cudaStreamNonBlocking));
      }
      int mode, rc, status = GT_OK;
      if ((rc = rank_mode_for(device, hp.scmp, &mode))) return rc;
      rc = (mode == kRankAtomic)
               ? host_pipeline<kRankAtomic>(hp, p, P, G, h_offsets, h_edges, V, E, h_t_offsets, h_t_edges, &status, stats)
               : host_pipeline<kRankSafe>(hp, p, P, G, h_offsets, h_edges, V, E, h_t_offsets, h_t_edges, &status, stats);
      if (rc) {
        cudaStreamSynchronize(hp.sin);
        cudaStreamSynchronize(hp.scmp);
        cudaStreamSynchronize(hp.sout);
        return rc;
      }
      if (status) return set_err(status, "32-bit degree counter overflowed (a transposed degree >= 2^32)");
      return GT_OK;
    }
  }
  // device copies of input and output live in a per-device cache (grow-only),
  // like the workspace: repeated calls do not re-map gigabytes of memory
  static WsEntry s_io[64];
  static cudaStream_t s_st[64];
  static std::mutex s_io_mu;
  std::lock_guard<std::mutex> lk(s_io_mu);
  if (!s_st[device]) GT_CUDA(cudaStreamCreateWithFlags(&s_st[device], cudaStreamNonBlocking));
  cudaStream_t st = s_st[device];
  const uint64_t b_off = align_up((V + 1) * 8, 256), b_e = align_up(std::max<uint64_t>(E, 1) * 4, 256);
  const uint64_t need = 2 * b_off + 2 * b_e;
  if (s_io[device].bytes < need) {
    if (s_io[device].ptr) GT_CUDA(cudaFreeAsync(s_io[device].ptr, st));
    s_io[device].ptr = nullptr;
    s_io[device].bytes = 0;
    GT_CUDA(cudaMallocAsync(&s_io[device].ptr, need, st));
    s_io[device].bytes = need;
  }
  unsigned char* b = static_cast<unsigned char*>(s_io[device].ptr);
  uint64_t* d_off = reinterpret_cast<uint64_t*>(b);
  uint64_t* d_toff = reinterpret_cast<uint64_t*>(b + b_off);
  uint32_t* d_e = reinterpret_cast<uint32_t*>(b + 2 * b_off);
  uint32_t* d_te = reinterpret_cast<uint32_t*>(b + 2 * b_off + b_e);
  GT_CUDA(cudaMemcpyAsync(d_off, h_offsets, (V + 1) * 8, cudaMemcpyHostToDevice, st));
  if (E) GT_CUDA(cudaMemcpyAsync(d_e, h_edges, E * 4, cudaMemcpyHostToDevice, st));
  int rc = gt_transpose(d_off, d_e, V, E, d_toff, d_te, nullptr, 0, st, stats);
  if (rc) return rc;
  GT_CUDA(cudaMemcpyAsync(h_t_offsets, d_toff, (V + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (E) GT_CUDA(cudaMemcpyAsync(h_t_edges, d_te, E * 4, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  int status = GT_OK;
  if ((rc = gt_transpose_status(st, &status))) return rc;
  return status;
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
  static WsEntry s_io2[64];
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
  if (s_io2[device].bytes < 2 * set_bytes) {
    GT_CUDA(cudaDeviceSynchronize());
    if (s_io2[device].ptr) GT_CUDA(cudaFree(s_io2[device].ptr));
    s_io2[device].ptr = nullptr;
    s_io2[device].bytes = 0;
    GT_CUDA(cudaMalloc(&s_io2[device].ptr, 2 * set_bytes));
    s_io2[device].bytes = 2 * set_bytes;
  }
  void* base = s_io2[device].ptr;
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
  int rc;
  if ((rc = h2d(0))) return rc;
  for (int i = 0; i < count; ++i) {
    const int slot = i & 1;
    const uint64_t V = Vs[i], E = Es[i];
    // one graph ahead: graph i+1's copy-in overlaps graph i's kernels and graph i-1's copy-out
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
    if (i + 1 < count) {  // an overflow in graph i: the status word is overwritten by graph i+1
      GT_CUDA(cudaStreamSynchronize(scmp));
      int status = GT_OK;
      if ((rc = gt_transpose_status(scmp, &status))) return rc;
      if (status) {
        cudaStreamSynchronize(sin);
        cudaStreamSynchronize(sout);
        return status;
      }
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
  int status = GT_OK;
  if ((rc = gt_transpose_status(scmp, &status))) return rc;
  return status;
}

int gt_prefix_sum(const uint32_t* counts, uint64_t n, uint64_t* out, void* stream) {
  if (!out || (n && !counts)) return set_err(GT_EINVAL, "NULL array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  const uint64_t tiles = std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
  WsEntry* ent;
  if ((rc = ws_entry(dev, st, &ent))) return rc;
  std::lock_guard<std::mutex> call(ent->call_mu);
  unsigned char* w = nullptr;
  if ((rc = ws_get(dev, st, tiles * 8 + 256, &w, nullptr))) return rc;
  uint64_t* status = reinterpret_cast<uint64_t*>(w);
  unsigned int* ctr = reinterpret_cast<unsigned int*>(w + align_up(tiles * 8, 128));
  return scan_u32_to_u64(counts, n, out, 0, true, status, ctr, st);
}

// ---------------------------------------------------------------- multi-GPU building blocks
int gt_shard_geometry(uint64_t V, uint64_t E, gt_shard_geom* g) {
  if (!g) return set_err(GT_EINVAL, "geometry is NULL");
  if (V == 0 || V > (1ull << 32)) return set_err(GT_EINVAL, "bad num_vertices");
  return gt_internal_shard_geometry(V, E, g);
}

int gt_shard_send(const uint64_t* offsets, const uint32_t* edges_slice, uint64_t V, uint64_t E_total,
                  uint64_t e_begin, uint64_t e_count, uint32_t* r1_out, uint64_t* bucket_counts, uint64_t* seg_hi_out,
                  void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!offsets || !bucket_counts || !seg_hi_out || (e_count && (!edges_slice || !r1_out)))
    return set_err(GT_EINVAL, "gt_shard_send: NULL array");
  if (e_begin + e_count > E_total || V == 0 || V > (1ull << 32)) return set_err(GT_EINVAL, "gt_shard_send: bad range");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  Plan p;
  if ((rc = make_plan(V, E_total, V, config_snapshot(), p))) return rc;
  const uint64_t nh = 1ull << p.nsh;
  if (e_count == 0) {
    GT_CUDA(cudaMemsetAsync(bucket_counts, 0, (uint64_t)p.D1 * 8, st));
    GT_CUDA(cudaMemsetAsync(seg_hi_out, 0xff, (uint64_t)p.D1 * (nh + 1) * 8, st));
    return GT_OK;
  }
  if (e_count >= (1ull << 32) && !p.wide) return set_err(GT_EINVAL, "gt_shard_send: slice too large");
  Plan ps = p;
  ps.E = e_count;
  Layout q;
  make_layout(ps, e_count, 0, 1, q);
  WsEntry* ent;
  if ((rc = ws_entry(dev, st, &ent))) return rc;
  std::lock_guard<std::mutex> call(ent->call_mu);
  unsigned char* ws;
  if ((rc = ws_get(dev, st, q.total, &ws, nullptr))) return rc;
  Ws w = ws_ptrs(q, ws, ps);
  w.seghi = seg_hi_out;  // the boundary table is part of the shipped meta
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  Timer tm;
  tm.init(false, st);
  int launches = 0;
  const InCsr in{offsets, edges_slice, e_begin, V};
  rc = (mode == kRankAtomic) ? level1<kRankAtomic>(ps, q, w, in, e_count, true, r1_out, st, tm, &launches)
                             : level1<kRankSafe>(ps, q, w, in, e_count, true, r1_out, st, tm, &launches);
  if (rc) return rc;
  k_sender_meta<<<(p.D1 + 255) / 256, 256, 0, st>>>(w.tbase, q.ntiles1, p.D1, e_count, w.prev, p.L, bucket_counts,
                                                     seg_hi_out, nh);
  GT_LAUNCH_CHECK();
  return GT_OK;
}

int gt_shard_receive(const uint32_t* r1_recv, uint64_t* seg_hi_recv, const uint64_t* counts, int nranks, uint64_t V,
                     uint64_t E_total, uint32_t bucket_lo, uint32_t bucket_hi, uint64_t num_records,
                     uint64_t global_base, uint64_t* t_offsets_local, uint32_t* t_edges_local, void* stream,
                     gt_stats* stats) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (!counts || !t_offsets_local || nranks < 1 || bucket_hi < bucket_lo ||
      (num_records && (!r1_recv || !seg_hi_recv || !t_edges_local)))
    return set_err(GT_EINVAL, "gt_shard_receive: bad arguments");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  Plan p;
  if ((rc = make_plan(V, E_total, V, config_snapshot(), p))) return rc;
  if (bucket_hi > (uint32_t)p.D1) return set_err(GT_EINVAL, "gt_shard_receive: bucket range beyond %d", p.D1);
  const int shift = p.b + p.c;
  const uint64_t v_lo = std::min<uint64_t>(V, (uint64_t)bucket_lo << shift);
  const uint64_t v_hi = std::min<uint64_t>(V, (uint64_t)bucket_hi << shift);
  const uint64_t Vloc = v_hi - v_lo;
  WsEntry* ent;
  if ((rc = ws_entry(dev, st, &ent))) return rc;
  std::lock_guard<std::mutex> call(ent->call_mu);
  if (num_records == 0 || Vloc == 0) {
    if (num_records) return set_err(GT_EINVAL, "gt_shard_receive: records for an empty destination range");
    GT_CUDA(cudaMemsetAsync(t_offsets_local, 0, (Vloc + 1) * 8, st));
    k_add_base<<<1, 256, 0, st>>>(t_offsets_local, Vloc + 1, global_base);
    GT_LAUNCH_CHECK();
    GT_CUDA(cudaMemsetAsync(ent->status, 0, sizeof(int), st));
    return GT_OK;
  }
  const uint32_t nloc = bucket_hi - bucket_lo;
  Plan pl = p;  // same digit split; local buckets, destinations and records
  pl.D1 = (int)nloc;
  pl.V = Vloc;
  pl.E = num_records;
  Layout q;
  make_layout(pl, 0, num_records, (uint32_t)nranks, q);
  unsigned char* ws;
  if ((rc = ws_get(dev, st, q.total, &ws, nullptr))) return rc;
  Ws w = ws_ptrs(q, ws, pl);
  int mode;
  if ((rc = rank_mode_for(dev, st, &mode))) return rc;
  Timer tm;
  if ((rc = tm.init(stats != nullptr, st))) return rc;
  int launches = 1;
  GT_CUDA(cudaMemsetAsync(w.err, 0, 4, st));
  if ((rc = tm.mark())) return rc;
  if ((rc = tm.mark())) return rc;  // (no level 1 on the receiver)
  v3::k_recv_runs<<<(unsigned)((nloc * nranks + 127) / 128), 128, 0, st>>>(counts, (uint32_t)nranks, (uint32_t)p.D1,
                                                                            bucket_lo, nloc, w.runs, seg_hi_recv,
                                                                            (uint32_t)q.nh);
  GT_LAUNCH_CHECK();
  rc = (mode == kRankAtomic)
           ? level23<kRankAtomic>(pl, q, w, r1_recv, (uint32_t)nranks, nloc, seg_hi_recv, t_offsets_local,
                                  t_edges_local, st, tm, &launches)
           : level23<kRankSafe>(pl, q, w, r1_recv, (uint32_t)nranks, nloc, seg_hi_recv, t_offsets_local,
                                t_edges_local, st, tm, &launches);
  if (rc) return rc;
  if (global_base) {
    k_add_base<<<148, 256, 0, st>>>(t_offsets_local, Vloc + 1, global_base);
    GT_LAUNCH_CHECK();
    ++launches;
  }
  if ((rc = tm.mark())) return rc;
  k_status_out<<<1, 1, 0, st>>>(w.err, ent->status);
  GT_LAUNCH_CHECK();
  if (stats) return finish_stats(pl, mode, tm, w, stats, q.total, launches + 1, st);
  return GT_OK;
}

int gt_shard_workspace_size(uint64_t V, uint64_t E_total, uint64_t e_count, uint32_t num_buckets_local, int nranks,
                            uint64_t num_records, uint64_t* send_bytes, uint64_t* recv_bytes) {
  if (!send_bytes || !recv_bytes || nranks < 1) return set_err(GT_EINVAL, "bad arguments");
  Plan p;
  int rc = make_plan(V, E_total, V, config_snapshot(), p);
  if (rc) return rc;
  Layout qs, qr;
  Plan ps = p;
  ps.E = e_count;
  make_layout(ps, e_count, 0, 1, qs);
  Plan pr = p;
  pr.D1 = (int)num_buckets_local;
  pr.E = num_records;
  make_layout(pr, 0, num_records, (uint32_t)nranks, qr);
  *send_bytes = e_count ? qs.total : 0;
  *recv_bytes = num_records ? qr.total : 0;
  return GT_OK;
}

int gt_shard_owners(const uint64_t* h_bucket_totals, uint32_t num_buckets, int parts, uint32_t* h_bounds) {
  if (!h_bucket_totals || !h_bounds || parts < 1) return set_err(GT_EINVAL, "gt_shard_owners: bad arguments");
  uint64_t total = 0;
  for (uint32_t c = 0; c < num_buckets; ++c) total += h_bucket_totals[c];
  // owner q takes buckets [bounds[q], bounds[q+1]): the first bucket whose
  // prefix reaches q * total / parts starts owner q (edge-balanced, bucket-aligned)
  h_bounds[0] = 0;
  uint64_t run = 0;
  uint32_t c = 0;
  for (int k = 1; k < parts; ++k) {
    const unsigned __int128 t = (unsigned __int128)total * (uint64_t)k / (uint64_t)parts;
    while (c < num_buckets && run + h_bucket_totals[c] <= (uint64_t)t) run += h_bucket_totals[c++];
    // place the boundary on the side of bucket c that leaves the smaller error
    if (c < num_buckets && (uint64_t)t - run > run + h_bucket_totals[c] - (uint64_t)t) run += h_bucket_totals[c++];
    h_bounds[k] = std::max(c, h_bounds[k - 1]);
  }
  h_bounds[parts] = num_buckets;
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

// gt_multi.cu — one rank's sharded CSR->CSC transpose over NCCL
// (gt_transpose_multi in include/gt.h).
//
// Step of rank r (P ranks, one GPU each):
//   1. level 1 of the rank's edge-balanced source shard (gt_shard_send): R1 +
//      per-bucket counts + source-high boundary rows;
//   2. ncclAllGather of the per-bucket counts -> P x D1 matrix (the one host
//      read: it sizes the sends and places the owners' bucket ranges, balanced
//      on the global bucket totals, gt_shard_owners);
//   3. NCCL send/recv of R1 (4 bytes per edge) and the boundary rows of every
//      owner's bucket range;
//   4. levels 2-3 over the received runs (gt_shard_receive): the rank's CSC
//      slice with global offsets.
// libnccl.so.2 is resolved with dlopen so that libgt.so loads without NCCL
// and shares the process's NCCL (torch's) when there is one.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/gt.h"
#include "gt_api_internal.h"

namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_nccl_mu;
Nccl g_nccl;

int nccl_load(Nccl** out) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (!g_nccl.ok) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return gt_set_errf(GT_ENODEV, "libnccl.so.2 not found: %s", dlerror());
    auto sym = [&](const char* name) -> void* { return dlsym(h, name); };
    g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(sym("ncclGetUniqueId"));
    g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(sym("ncclCommInitRank"));
    g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(sym("ncclCommDestroy"));
    g_nccl.Send = reinterpret_cast<decltype(g_nccl.Send)>(sym("ncclSend"));
    g_nccl.Recv = reinterpret_cast<decltype(g_nccl.Recv)>(sym("ncclRecv"));
    g_nccl.AllGather = reinterpret_cast<decltype(g_nccl.AllGather)>(sym("ncclAllGather"));
    g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(sym("ncclGroupStart"));
    g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(sym("ncclGroupEnd"));
    g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(sym("ncclGetErrorString"));
    if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.CommDestroy || !g_nccl.Send || !g_nccl.Recv ||
        !g_nccl.AllGather || !g_nccl.GroupStart || !g_nccl.GroupEnd || !g_nccl.GetErrorString)
      return gt_set_errf(GT_ENODEV, "libnccl.so.2 lacks a required symbol");
    g_nccl.ok = true;
  }
  *out = &g_nccl;
  return GT_OK;
}

#define GT_NCCL(call)                                                                                   \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess) return gt_set_errf(GT_ECUDA, "%s: %s", #call, nc->GetErrorString(r_));      \
  } while (0)
#define GT_CU(call)                                                                                     \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess)                                                                              \
      return gt_set_errf(e_ == cudaErrorMemoryAllocation ? GT_ENOMEM : GT_ECUDA, "%s: %s", #call,       \
                         cudaGetErrorString(e_));                                                       \
  } while (0)

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Exchange buffers, one set per (device, stream), grown stream-ordered.
struct Buf {
  void* ptr = nullptr;
  uint64_t bytes = 0;
};
std::mutex g_buf_mu;
std::map<std::pair<int, cudaStream_t>, Buf> g_buf;

int buf_get(cudaStream_t st, uint64_t bytes, unsigned char** out) {
  int dev = 0;
  GT_CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_buf_mu);
  Buf& b = g_buf[{dev, st}];
  if (b.bytes < bytes) {
    if (b.ptr) GT_CU(cudaFreeAsync(b.ptr, st));
    b.ptr = nullptr;
    b.bytes = 0;
    GT_CU(cudaMallocAsync(&b.ptr, bytes, st));
    b.bytes = bytes;
  }
  *out = static_cast<unsigned char*>(b.ptr);
  return GT_OK;
}

}  // namespace

extern "C" {

int gt_multi_unique_id(void* id128) {
  if (!id128) return gt_set_errf(GT_EINVAL, "id is NULL");
  Nccl* nc;
  int rc = nccl_load(&nc);
  if (rc) return rc;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  GT_NCCL(nc->GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof id);
  return GT_OK;
}

int gt_multi_comm_init(const void* id128, int rank, int nranks, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return gt_set_errf(GT_EINVAL, "bad arguments");
  Nccl* nc;
  int rc = nccl_load(&nc);
  if (rc) return rc;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  GT_NCCL(nc->CommInitRank(&c, nranks, id, rank));
  *comm = c;
  return GT_OK;
}

int gt_multi_comm_destroy(void* comm) {
  if (!comm) return GT_OK;
  Nccl* nc;
  int rc = nccl_load(&nc);
  if (rc) return rc;
  GT_NCCL(nc->CommDestroy(static_cast<ncclComm_t>(comm)));
  return GT_OK;
}

int gt_transpose_multi(void* comm, int rank, int nranks, const uint64_t* offsets, const uint32_t* edges_slice,
                       uint64_t V, uint64_t E, uint64_t src_begin, uint64_t src_end, uint64_t* t_offsets_local,
                       uint32_t* t_edges_local, uint64_t t_edges_capacity, gt_multi_info* info, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!comm || !offsets || !t_offsets_local || !info || nranks < 1 || rank < 0 || rank >= nranks ||
      src_begin > src_end || src_end > V)
    return gt_set_errf(GT_EINVAL, "gt_transpose_multi: bad arguments");
  std::memset(info, 0, sizeof(*info));
  Nccl* nc;
  int rc = nccl_load(&nc);
  if (rc) return rc;
  ncclComm_t cm = static_cast<ncclComm_t>(comm);
  gt_shard_geom g;
  if ((rc = gt_shard_geometry(V, E, &g))) return rc;
  const uint64_t D1 = g.num_buckets, row = g.seg_hi_row, P = (uint64_t)nranks;
  cudaEvent_t ev[4];
  for (auto& e : ev) GT_CU(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  // the shard's edge range
  uint64_t erng[2];
  GT_CU(cudaMemcpyAsync(&erng[0], offsets + src_begin, 8, cudaMemcpyDeviceToHost, st));
  GT_CU(cudaMemcpyAsync(&erng[1], offsets + src_end, 8, cudaMemcpyDeviceToHost, st));
  GT_CU(cudaStreamSynchronize(st));
  const uint64_t e_begin = erng[0], e_count = erng[1] - erng[0];
  if (e_count && !edges_slice) return gt_set_errf(GT_EINVAL, "gt_transpose_multi: NULL edge slice");
  // exchange buffers: send R1 | counts | all counts | send seg_hi | recv seg_hi | recv R1
  const uint64_t b_r1 = align_up(std::max<uint64_t>(e_count, 1) * 4, 256), b_cnt = align_up(D1 * 8, 256),
                 b_all = align_up(P * D1 * 8, 256), b_seg = align_up(D1 * row * 8, 256);
  const uint64_t fixed = b_r1 + b_cnt + b_all + b_seg + b_seg * P;  // recv seg_hi <= P x all rows
  unsigned char* base;
  if ((rc = buf_get(st, fixed, &base))) return rc;
  uint32_t* r1 = reinterpret_cast<uint32_t*>(base);
  uint64_t* cnt = reinterpret_cast<uint64_t*>(base + b_r1);
  uint64_t* all = reinterpret_cast<uint64_t*>(base + b_r1 + b_cnt);
  uint64_t* seg = reinterpret_cast<uint64_t*>(base + b_r1 + b_cnt + b_all);
  uint64_t* rseg = reinterpret_cast<uint64_t*>(base + b_r1 + b_cnt + b_all + b_seg);
  GT_CU(cudaEventRecord(ev[0], st));
  if ((rc = gt_shard_send(offsets, edges_slice, V, E, e_begin, e_count, r1, cnt, seg, st))) return rc;
  GT_CU(cudaEventRecord(ev[1], st));
  GT_NCCL(nc->AllGather(cnt, all, D1, ncclUint64, cm, st));
  std::vector<uint64_t> h_all(P * D1), tot(D1, 0);
  GT_CU(cudaMemcpyAsync(h_all.data(), all, P * D1 * 8, cudaMemcpyDeviceToHost, st));
  GT_CU(cudaStreamSynchronize(st));
  for (uint64_t s = 0; s < P; ++s)
    for (uint64_t c = 0; c < D1; ++c) tot[c] += h_all[s * D1 + c];
  std::vector<uint32_t> bounds(P + 1);
  if ((rc = gt_shard_owners(tot.data(), (uint32_t)D1, nranks, bounds.data()))) return rc;
  auto cnt_range = [&](uint64_t s, uint32_t lo, uint32_t hi) {
    uint64_t x = 0;
    for (uint32_t c = lo; c < hi; ++c) x += h_all[s * D1 + c];
    return x;
  };
  const uint32_t lo = bounds[rank], hi = bounds[rank + 1], nloc = hi - lo;
  uint64_t local = 0, gbase = 0;
  for (uint64_t s = 0; s < P; ++s) local += cnt_range(s, lo, hi);
  for (uint32_t c = 0; c < lo; ++c) gbase += tot[c];
  const int shift = (int)g.bucket_shift;
  info->bucket_lo = lo;
  info->bucket_hi = hi;
  info->dst_begin = std::min<uint64_t>(V, (uint64_t)lo << shift);
  info->dst_end = std::min<uint64_t>(V, (uint64_t)hi << shift);
  info->global_base = gbase;
  info->num_local_edges = local;
  if (local > t_edges_capacity || (local && !t_edges_local))
    return gt_set_errf(GT_ENOMEM, "gt_transpose_multi: t_edges capacity %llu < %llu local edges",
                       (unsigned long long)t_edges_capacity, (unsigned long long)local);
  // receive buffer for R1 (separate, sized now)
  static std::mutex s_rmu;
  static std::map<std::pair<int, cudaStream_t>, Buf> s_recv;
  uint32_t* rr1 = nullptr;
  if (P > 1) {
    int dev = 0;
    GT_CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(s_rmu);
    Buf& b = s_recv[{dev, st}];
    const uint64_t need = std::max<uint64_t>(local, 1) * 4 + 64;
    if (b.bytes < need) {
      if (b.ptr) GT_CU(cudaFreeAsync(b.ptr, st));
      b.ptr = nullptr;
      b.bytes = 0;
      GT_CU(cudaMallocAsync(&b.ptr, need, st));
      b.bytes = need;
    }
    rr1 = static_cast<uint32_t*>(b.ptr);
  }
  // every sender's bucket prefix (its R1 offset of bucket c)
  auto prefix = [&](uint64_t s, uint32_t c) { return cnt_range(s, 0, c); };
  GT_CU(cudaEventRecord(ev[2], st));
  if (P == 1) {  // one rank owns every bucket: receive straight from the send buffers
    rr1 = r1;
    rseg = seg;
  } else {
  GT_NCCL(nc->GroupStart());
  uint64_t roff = 0;
  for (uint64_t q = 0; q < P; ++q) {
    const uint32_t qlo = bounds[q], qhi = bounds[q + 1];
    const uint64_t n_to = cnt_range((uint64_t)rank, qlo, qhi);
    if (n_to) GT_NCCL(nc->Send(r1 + prefix((uint64_t)rank, qlo), n_to, ncclUint32, (int)q, cm, st));
    if (qhi > qlo) GT_NCCL(nc->Send(seg + (uint64_t)qlo * row, (uint64_t)(qhi - qlo) * row, ncclUint64, (int)q, cm, st));
    const uint64_t n_from = cnt_range(q, lo, hi);
    if (n_from) GT_NCCL(nc->Recv(rr1 + roff, n_from, ncclUint32, (int)q, cm, st));
    roff += n_from;
    if (nloc) GT_NCCL(nc->Recv(rseg + q * nloc * row, (uint64_t)nloc * row, ncclUint64, (int)q, cm, st));
  }
  GT_NCCL(nc->GroupEnd());
  }
  GT_CU(cudaEventRecord(ev[3], st));
  if ((rc = gt_shard_receive(rr1, rseg, all, nranks, V, E, lo, hi, local, gbase, t_offsets_local, t_edges_local, st,
                             nullptr)))
    return rc;
  cudaEvent_t ev_end;
  GT_CU(cudaEventCreate(&ev_end));
  GT_CU(cudaEventRecord(ev_end, st));
  GT_CU(cudaEventSynchronize(ev_end));
  float a = 0, b = 0, c = 0;
  cudaEventElapsedTime(&a, ev[0], ev[1]);
  cudaEventElapsedTime(&b, ev[2], ev[3]);
  cudaEventElapsedTime(&c, ev[3], ev_end);
  cudaEventDestroy(ev_end);
  info->ms_send = a;
  info->ms_exchange = b;
  info->ms_receive = c;
  int status = GT_OK;
  if ((rc = gt_transpose_status(st, &status))) return rc;
  return status;
}

}  // extern "C"

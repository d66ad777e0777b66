// gt_io.cu — POTG graph files straight to / from device memory.
//
// Restates the reference's binary format (pkg/src/potra/io.py:1-9,24-114):
// little-endian header "<4sBBBBQQ" = magic "POTG", u8 version 1, u8 id_width
// in {4, 8}, u8 orientation (0 CSR, 1 CSC), u8 pad, u64 num_vertices, u64
// num_edges; then (V+1) u64 offsets; then E edge IDs of id_width bytes.
//
// B200 layout of the work: the file is streamed through two pinned host
// buffers (read of chunk i+1 overlaps the H2D copy of chunk i), and the data
// checks of _load_binary (io.py:77-109: offsets[0] == 0, monotone offsets,
// offsets[-1] == E, every edge ID < V) run on the device as one pass each,
// reducing the FIRST violating index with atomicMin so the error message and
// byte offset equal the reference's (np.nonzero(...)[0][0]).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <sys/stat.h>

#include <cuda_runtime.h>

#include "../../include/gt.h"

int gt_internal_set_err(int code, const char* msg);  // gt_api.cu

namespace {

constexpr uint64_t kHeader = 24;
constexpr size_t kStage = 64ull << 20;  // bytes per pinned staging buffer

int fmt_err(uint64_t* err_off, uint64_t off, const std::string& msg) {
  if (err_off) *err_off = off;
  return gt_internal_set_err(GT_EFORMAT, msg.c_str());
}

// Python's repr() of a 4-byte bytes object (for the bad-magic message).
std::string bytes_repr(const unsigned char* b, int n) {
  bool has_sq = false, has_dq = false;
  for (int i = 0; i < n; ++i) {
    has_sq |= b[i] == '\'';
    has_dq |= b[i] == '"';
  }
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string s = "b";
  s += q;
  for (int i = 0; i < n; ++i) {
    const unsigned c = b[i];
    char tmp[8];
    if (c == '\\') s += "\\\\";
    else if (c == (unsigned)q) { s += '\\'; s += (char)c; }
    else if (c == '\t') s += "\\t";
    else if (c == '\n') s += "\\n";
    else if (c == '\r') s += "\\r";
    else if (c < 0x20 || c >= 0x7f) { snprintf(tmp, sizeof tmp, "\\x%02x", c); s += tmp; }
    else s += (char)c;
  }
  s += q;
  return s;
}

__global__ void k_check_offsets(const uint64_t* __restrict__ off, uint64_t V, unsigned long long* first_bad) {
  // first i in [1, V] with (int64)off[i] < (int64)off[i-1]   (io.py:88-94, int64 view)
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1; i <= V; i += (uint64_t)gridDim.x * blockDim.x)
    if ((long long)off[i] < (long long)off[i - 1]) atomicMin(first_bad, (unsigned long long)i);
}

template <typename T>
__global__ void k_check_edges(const T* __restrict__ e, uint64_t E, uint64_t V, unsigned long long* first_bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
    if ((uint64_t)e[i] >= V) atomicMin(first_bad, (unsigned long long)i);
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) {
        cudaEventSynchronize(ev[i]);
        cudaEventDestroy(ev[i]);
      }
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
  int init() {
    for (int i = 0; i < 2; ++i) {
      if (cudaMallocHost(&p[i], kStage) != cudaSuccess) return gt_internal_set_err(GT_ENOMEM, "pinned staging buffer");
      if (cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
        return gt_internal_set_err(GT_ECUDA, "cudaEventCreate");
    }
    return GT_OK;
  }
};

// file [pos, pos+bytes) -> device dst, double-buffered through pinned memory
int stream_in(FILE* f, uint64_t pos, uint64_t bytes, void* dst, Pinned& pin, cudaStream_t st) {
  if (!bytes) return GT_OK;
  if (fseeko(f, (off_t)pos, SEEK_SET) != 0) return gt_internal_set_err(GT_EIO, "seek failed");
  uint64_t done = 0;
  int b = 0;
  while (done < bytes) {
    const size_t n = (size_t)std::min<uint64_t>(kStage, bytes - done);
    if (cudaEventSynchronize(pin.ev[b]) != cudaSuccess) return gt_internal_set_err(GT_ECUDA, "staging event");
    if (fread(pin.p[b], 1, n, f) != n) return gt_internal_set_err(GT_EIO, "short read");
    if (cudaMemcpyAsync(static_cast<char*>(dst) + done, pin.p[b], n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(pin.ev[b], st) != cudaSuccess)
      return gt_internal_set_err(GT_ECUDA, "H2D copy");
    done += n;
    b ^= 1;
  }
  return GT_OK;
}

// device src [0, bytes) -> file (appending), double-buffered
int stream_out(FILE* f, const void* src, uint64_t bytes, Pinned& pin, cudaStream_t st) {
  uint64_t done = 0;
  int b = 0;
  size_t pend_n[2] = {0, 0};
  while (done < bytes || pend_n[0] || pend_n[1]) {
    if (pend_n[b]) {  // drain the older copy of this buffer
      if (cudaEventSynchronize(pin.ev[b]) != cudaSuccess) return gt_internal_set_err(GT_ECUDA, "staging event");
      if (fwrite(pin.p[b], 1, pend_n[b], f) != pend_n[b]) return gt_internal_set_err(GT_EIO, "short write");
      pend_n[b] = 0;
    }
    if (done < bytes) {
      const size_t n = (size_t)std::min<uint64_t>(kStage, bytes - done);
      if (cudaMemcpyAsync(pin.p[b], static_cast<const char*>(src) + done, n, cudaMemcpyDeviceToHost, st) !=
              cudaSuccess ||
          cudaEventRecord(pin.ev[b], st) != cudaSuccess)
        return gt_internal_set_err(GT_ECUDA, "D2H copy");
      pend_n[b] = n;
      done += n;
    }
    b ^= 1;
  }
  return GT_OK;
}

}  // namespace

extern "C" {

int gt_potg_read_header(const char* path, gt_potg_header* h, uint64_t* err_byte_offset) {
  if (!path || !h) return gt_internal_set_err(GT_EINVAL, "null argument");
  File fl;
  fl.f = fopen(path, "rb");
  if (!fl.f) return gt_internal_set_err(GT_EIO, (std::string("cannot open ") + path).c_str());
  struct stat sb;
  if (fstat(fileno(fl.f), &sb) != 0) return gt_internal_set_err(GT_EIO, "stat failed");
  const uint64_t fsize = (uint64_t)sb.st_size;
  unsigned char hd[kHeader];
  if (fsize < kHeader) {
    char m[128];
    snprintf(m, sizeof m, "truncated file: %llu bytes is shorter than the %llu-byte header",
             (unsigned long long)fsize, (unsigned long long)kHeader);
    return fmt_err(err_byte_offset, fsize, m);
  }
  if (fread(hd, 1, kHeader, fl.f) != kHeader) return gt_internal_set_err(GT_EIO, "short read");
  uint64_t nv, ne;
  memcpy(&nv, hd + 8, 8);  // little-endian host (x86_64 / aarch64)
  memcpy(&ne, hd + 16, 8);
  char m[256];
  if (memcmp(hd, "POTG", 4) != 0)
    return fmt_err(err_byte_offset, 0, "malformed header: bad magic " + bytes_repr(hd, 4));
  if (hd[4] != 1) {
    snprintf(m, sizeof m, "malformed header: unsupported version %u", hd[4]);
    return fmt_err(err_byte_offset, 4, m);
  }
  if (hd[5] != 4 && hd[5] != 8) {
    snprintf(m, sizeof m, "malformed header: id width %u not in {4, 8}", hd[5]);
    return fmt_err(err_byte_offset, 5, m);
  }
  if (hd[6] > 1) {
    snprintf(m, sizeof m, "malformed header: orientation code %u", hd[6]);
    return fmt_err(err_byte_offset, 6, m);
  }
  if (hd[5] == 4 && nv > (1ull << 32)) {
    snprintf(m, sizeof m, "malformed header: 4-byte edge IDs cannot address %llu vertices", (unsigned long long)nv);
    return fmt_err(err_byte_offset, 5, m);
  }
  // expected = header + (nv+1)*8 + ne*w, in 128-bit arithmetic like Python ints
  const unsigned __int128 expected =
      (unsigned __int128)kHeader + ((unsigned __int128)nv + 1) * 8 + (unsigned __int128)ne * hd[5];
  if ((unsigned __int128)fsize < expected) {
    const unsigned long long ex_lo = (unsigned long long)expected;
    if (expected >> 64) snprintf(m, sizeof m, "truncated file: expected more than 2^64 bytes, got %llu",
                                 (unsigned long long)fsize);
    else snprintf(m, sizeof m, "truncated file: expected %llu bytes, got %llu", ex_lo, (unsigned long long)fsize);
    return fmt_err(err_byte_offset, fsize, m);
  }
  h->version = hd[4];
  h->id_width = hd[5];
  h->orientation = hd[6];
  h->pad = hd[7];
  h->num_vertices = nv;
  h->num_edges = ne;
  return GT_OK;
}

int gt_potg_read(const char* path, const gt_potg_header* h, uint64_t* offsets, void* edges, void* stream,
                 uint64_t* err_byte_offset) {
  if (!path || !h || !offsets || (h->num_edges && !edges)) return gt_internal_set_err(GT_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t V = h->num_vertices, E = h->num_edges, w = h->id_width;
  File fl;
  fl.f = fopen(path, "rb");
  if (!fl.f) return gt_internal_set_err(GT_EIO, (std::string("cannot open ") + path).c_str());
  Pinned pin;
  int rc = pin.init();
  if (rc) return rc;
  if ((rc = stream_in(fl.f, kHeader, (V + 1) * 8, offsets, pin, st))) return rc;
  const uint64_t edges_off = kHeader + (V + 1) * 8;
  if ((rc = stream_in(fl.f, edges_off, E * w, edges, pin, st))) return rc;
  unsigned long long* bad = nullptr;
  if (cudaMallocAsync(&bad, 16, st) != cudaSuccess) return gt_internal_set_err(GT_ENOMEM, "cudaMallocAsync");
  cudaMemsetAsync(bad, 0xff, 16, st);
  if (V) k_check_offsets<<<148 * 8, 256, 0, st>>>(offsets, V, bad);
  if (E) {
    if (w == 4) k_check_edges<uint32_t><<<148 * 8, 256, 0, st>>>(static_cast<const uint32_t*>(edges), E, V, bad + 1);
    else k_check_edges<uint64_t><<<148 * 8, 256, 0, st>>>(static_cast<const uint64_t*>(edges), E, V, bad + 1);
  }
  unsigned long long hb[2];
  uint64_t first = 0, last = 0;
  cudaMemcpyAsync(hb, bad, 16, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&first, offsets, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&last, offsets + V, 8, cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFreeAsync(bad, st);
  if (e != cudaSuccess) return gt_internal_set_err(GT_ECUDA, cudaGetErrorString(e));
  char m[256];
  if (first != 0) return fmt_err(err_byte_offset, kHeader, "offsets[0] must be 0");
  if (hb[0] != ~0ull) {
    snprintf(m, sizeof m, "non-monotone offsets at index %llu", hb[0]);
    return fmt_err(err_byte_offset, kHeader + 8 * hb[0], m);
  }
  if (last != E) {
    snprintf(m, sizeof m, "offsets[-1] is %llu but header says %llu edges", (unsigned long long)last,
             (unsigned long long)E);
    return fmt_err(err_byte_offset, kHeader + 8 * V, m);
  }
  if (hb[1] != ~0ull) {
    uint64_t val = 0;
    cudaMemcpy(&val, static_cast<const char*>(edges) + hb[1] * w, w, cudaMemcpyDeviceToHost);
    snprintf(m, sizeof m, "edge ID %llu >= num_vertices %llu at edge index %llu", (unsigned long long)val,
             (unsigned long long)V, hb[1]);
    return fmt_err(err_byte_offset, edges_off + hb[1] * w, m);
  }
  return GT_OK;
}

int gt_potg_write(const char* path, const uint64_t* offsets, const void* edges, uint64_t V, uint64_t E,
                  int orientation, int id_width, void* stream) {
  if (!path || !offsets || (E && !edges) || (orientation != 0 && orientation != 1) ||
      (id_width != 4 && id_width != 8))
    return gt_internal_set_err(GT_EINVAL, "bad argument");
  // store_graph writes the id width forced by V (io.py:31-33, graph.py:34-36)
  const int want = (V <= (1ull << 32)) ? 4 : 8;
  if (id_width != want) return gt_internal_set_err(GT_EINVAL, "id_width must be 4 for V <= 2^32, else 8");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  File fl;
  fl.f = fopen(path, "wb");
  if (!fl.f) return gt_internal_set_err(GT_EIO, (std::string("cannot create ") + path).c_str());
  unsigned char hd[kHeader] = {'P', 'O', 'T', 'G', 1, (unsigned char)id_width, (unsigned char)orientation, 0};
  memcpy(hd + 8, &V, 8);
  memcpy(hd + 16, &E, 8);
  if (fwrite(hd, 1, kHeader, fl.f) != kHeader) return gt_internal_set_err(GT_EIO, "short write");
  Pinned pin;
  int rc = pin.init();
  if (rc) return rc;
  if ((rc = stream_out(fl.f, offsets, (V + 1) * 8, pin, st))) return rc;
  if ((rc = stream_out(fl.f, edges, E * (uint64_t)id_width, pin, st))) return rc;
  if (fflush(fl.f) != 0) return gt_internal_set_err(GT_EIO, "flush failed");
  return GT_OK;
}

}  // extern "C"

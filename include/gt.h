/*
 * gt.h — C ABI of the B200-native CSR->CSC graph transposition library
 * (paper_2501_06872_b200/libgt.so).
 *
 * The reference (arxiv 2501.06872, package `potra`) exposes this path as
 * Python functions over numpy arrays; there is no FFI in the reference.  The
 * entry points below are what a reference-side binding (ctypes stub shown in
 * INTEGRATION.md) would call in place of the numba kernels:
 *
 *   gt_transpose         replaces transpose_atomic / transpose_potra steps 1-3
 *                        + sort_neighbor_lists  (baselines.py:168-209,
 *                        hlh.py:441-588, baselines.py:457-475); output equals
 *                        transpose_oracle (graph.py:136-148) bit for bit.
 *   gt_transpose_host    same, host buffers in and out (H2D + kernels + D2H).
 *   gt_transpose_host_many  a batch of host transposes, copies overlapped with the kernels.
 *   gt_prefix_sum        prefix_sum_parallel (baselines.py:116-127).
 *   gt_edge_balanced_bounds  edge_balanced_vertex_bounds (_nb.py:118-132),
 *                        the source-range sharding rule for multi-GPU runs.
 *   gt_shard_*           multi-GPU building blocks: a sender's level-1 partition
 *                        of its source shard, a receiver's levels 2-3 over the
 *                        runs it received; the exchange itself is NCCL.
 *   gt_transpose_multi   the whole sharded transpose of one rank over NCCL
 *                        (gt_multi.cu), the `threads` / use_workers width of
 *                        transpose_atomic (baselines.py:168-170, _nb.py:105-115)
 *                        mapped to GPUs.
 *
 * Array conventions (graph.py:34-36, 59-80): offsets are uint64[V+1] with
 * offsets[0]=0 and offsets[V]=E; neighbour IDs are uint32[E].  Every neighbour
 * list of the output is ascending by source ID.  V may be anything up to 2^32
 * (the uint32 ID range): above 2^29 the destinations are processed in slabs of
 * 2^29 IDs, which costs one host read of the per-slab edge
 * counts per call.  E may exceed 2^32 (the wide form).
 *
 * Return codes mirror the reference's exceptions:
 *   GT_OK (0); GT_EINVAL (ValueError: bad arguments, _nb.py:112-113);
 *   GT_EOVERFLOW (CounterOverflowError: an in-degree >= 2^32,
 *   baselines.py:189-192); GT_ENOMEM (MemoryError / FootprintError precheck,
 *   errors.py:17-26); GT_ECUDA (a CUDA runtime failure); GT_ENODEV (no GPU).
 * gt_last_error() returns a thread-local message for the last failure.
 *
 * Device pointers are CUDA global-memory pointers; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  gt_transpose and gt_shard_receive are
 * stream-ordered: they enqueue their kernels and return without waiting (the
 * first call on a device also runs a one-off synchronous self-test), so they
 * can be captured in a CUDA graph; an in-degree overflow is reported by
 * gt_transpose_status() once the stream has completed the call (or directly
 * when `stats` is non-NULL, which makes the call wait for its events).  With
 * workspace == NULL the library uses a cached workspace private to the
 * (device, stream) pair: calls on different streams never share scratch,
 * calls on one stream are ordered by it.  The caller owns every other buffer.
 * No torch types cross this boundary.
 */
#ifndef GT_H_
#define GT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GT_OK 0
#define GT_EINVAL (-1)
#define GT_EOVERFLOW (-2)
#define GT_ENOMEM (-3)
#define GT_ECUDA (-4)
#define GT_ENODEV (-5)
#define GT_EFORMAT (-6) /* GraphFormatError (errors.py:4-14): a POTG file violates the format */
#define GT_EIO (-7)     /* OSError: a file could not be opened, read or written */

#define GT_ABI_VERSION 4

/* Per-call accounting; mirrors TransposeOutput.phase_times / aux_footprint_bytes
 * (baselines.py:39-53).  Times are device time from CUDA events, in ms, filled
 * only when stats != NULL (timing adds event records to the stream). */
typedef struct gt_stats {
    double ms_total;       /* whole transpose                                  */
    double ms_step1;       /* level-1 count + partition (source-ordered pass)  */
    double ms_step2;       /* level-2 chunk sort by middle digit               */
    double ms_step3;       /* final per-bucket sort + CSC offsets              */
    uint64_t workspace_bytes; /* aux device memory used (aux_footprint_bytes)  */
    int32_t bits[3];       /* destination-ID digit split per level             */
    int32_t rank_mode;     /* 0 = lane-ordered smem atomics, 1 = safe OR-mask  */
    uint64_t n_big_buckets;/* final buckets that took the multi-CTA path       */
    uint64_t n_launches;   /* kernels this call launched                       */
    double ms_kernel[4];   /* device time of the main kernels: level-1 place,  */
                           /* level-2 place, level-3 units, level-3 big place  */
                           /* (0 when a kernel did not run on this path)       */
} gt_stats;

/* Library / device info. */
int gt_abi_version(void);
const char *gt_last_error(void);

/* Workspace bytes gt_transpose needs for a graph of this size (0 allowed). */
int gt_workspace_size(uint64_t num_vertices, uint64_t num_edges, uint64_t *bytes);

/* Device-resident CSR -> CSC.  `workspace` may be NULL: the library then uses
 * an internal cached device allocation (reported in stats->workspace_bytes). */
int gt_transpose(const uint64_t *offsets, const uint32_t *edges,
                 uint64_t num_vertices, uint64_t num_edges,
                 uint64_t *t_offsets, uint32_t *t_edges,
                 void *workspace, uint64_t workspace_bytes,
                 void *stream, gt_stats *stats);

/* Host-resident CSR -> CSC on `device` (H2D copy, transpose, D2H copy).  Host
 * buffers may be pageable or pinned; pinned buffers make the copies overlap the
 * kernels.  Compact graphs of >= 2^24 edges take the pipelined call (DESIGN.md
 * §7b): the edges copy in as P source chunks, each partitioned (level 1) while
 * the next one copies; after one host read of the P x num_buckets counts,
 * levels 2-3 run per group of coarse buckets and each group's CSC range copies
 * back while the next group is computed.  gt_config.reserved[1] / [2] set P /
 * the group count (0 = by size; reserved[1] < 0 = the serial call).  `stats`
 * (pipelined call): ms_step1 = copy-in + level 1, ms_step2 = levels 2-3 of the
 * groups, ms_step3 = the copy-back tail, ms_total = the call on the device,
 * ms_kernel zero.  Rejects offsets[num_vertices] != num_edges (GT_EINVAL). */
int gt_transpose_host(const uint64_t *h_offsets, const uint32_t *h_edges,
                      uint64_t num_vertices, uint64_t num_edges,
                      uint64_t *h_t_offsets, uint32_t *h_t_edges,
                      int device, gt_stats *stats);

/* A batch of `count` host-resident transposes on `device`, pipelined: graph i+1's
 * H2D copy runs while graph i is transposed and graph i-1's result is copied
 * back (three streams, two device buffer sets sized for the largest graph), so
 * with pinned host buffers both PCIe directions and the kernels overlap.  Same
 * per-graph contract and results as gt_transpose_host; `stats` describes the
 * last graph.  Replaces a loop of transpose_atomic / transpose_potra calls over
 * several graphs (baselines.py:168-209, hlh.py:441-588). */
int gt_transpose_host_many(int count, const uint64_t *const *h_offsets, const uint32_t *const *h_edges,
                           const uint64_t *num_vertices, const uint64_t *num_edges,
                           uint64_t *const *h_t_offsets, uint32_t *const *h_t_edges,
                           int device, gt_stats *stats);

/* Exclusive prefix sum of uint32 counts into uint64[n+1] (out[n] = total). */
int gt_prefix_sum(const uint32_t *counts, uint64_t n, uint64_t *out, void *stream);

/* Host helper: edge_balanced_vertex_bounds (_nb.py:118-132) on host offsets. */
int gt_edge_balanced_bounds(const uint64_t *h_offsets, uint64_t num_vertices,
                            int64_t parts, int64_t *h_bounds);

/* Smem-atomic lane-order self-test.  Runs `trials`
 * randomized warp-instructions on the current device; *violations = count of
 * returns that were not lane-ascending.  gt_transpose runs it once per device
 * and falls back to the OR-mask ranking when it fails. */
int gt_selftest_rank_order(uint64_t trials, uint64_t *violations);

/* Force the ranking mode: -1 auto (self-test), 0 atomics, 1 safe OR-mask. */
int gt_set_rank_mode(int mode);

/* Explicit pipeline configuration (process-wide; read once per call).  All
 * zero = the defaults.  split: destination digit split a|b|c (used when
 * a+b+c equals the ID bits); force_wide: the 64-bit-position form (DESIGN.md
 * §2b) even for small graphs.  Test and experiment hooks; no environment
 * variable changes the product path. */
typedef struct gt_config {
    int32_t split[3];
    int32_t force_wide;
    int32_t reserved[4];
} gt_config;
int gt_set_config(const gt_config *cfg);   /* NULL restores the defaults */
int gt_get_config(gt_config *cfg);

/* Result of the last gt_transpose / gt_shard_receive enqueued on `stream`
 * (current device): *status = GT_OK or GT_EOVERFLOW.  Valid once the stream
 * has completed that call; it reads a mapped status word the call's last
 * kernel writes, so it does not synchronise. */
int gt_transpose_status(void *stream, int *status);

/* Free the cached workspaces of the current device (synchronises the device). */
int gt_release_workspace(void);

/* ---- multi-GPU building blocks (one process per GPU; NCCL moves R1) -------
 * Every rank plans with the global (num_vertices, num_edges): the destination
 * ID splits into coarse buckets (ID >> bucket_shift, num_buckets of them).
 * Sender (gt_shard_send): level 1 of its edge slice [e_begin, e_begin+e_count)
 * (the slice of an edge-balanced source shard, _nb.py:118-132) into R1: 4-byte
 * records grouped by bucket, each group in CSR order; bucket_counts[c] =
 * records of bucket c; seg_hi_out = the source-high boundary table
 * (num_buckets rows of seg_hi_row u64).  Owners take contiguous bucket
 * ranges (gt_shard_owners balances them on the global bucket totals); the
 * receiver of buckets [lo, hi) gets, from every sender s in rank order, R1
 * records [prefix_s(lo), prefix_s(hi)) and seg_hi rows lo..hi-1.
 * Receiver (gt_shard_receive): levels 2-3 over those runs: r1_recv holds the
 * senders' blocks back to back, seg_hi_recv their rows (nranks * (hi-lo) rows,
 * rebased in place), counts the nranks x num_buckets matrix of all senders'
 * bucket_counts (device).  Output: the CSC slice of destinations
 * [lo << shift, min(hi << shift, V)): t_offsets_local (global positions,
 * starting at global_base) and t_edges_local[num_records]. */
typedef struct gt_shard_geom {
    uint32_t num_buckets;   /* coarse buckets                                 */
    uint32_t bucket_shift;  /* destination ID >> bucket_shift = bucket        */
    uint32_t seg_hi_row;    /* u64 entries per bucket row of the seg_hi table */
    uint32_t wide;          /* 1: 64-bit-position form                        */
    int32_t bits[3];        /* digit split                                    */
    uint32_t pad;
} gt_shard_geom;
int gt_shard_geometry(uint64_t num_vertices, uint64_t num_edges, gt_shard_geom *geom);
int gt_shard_send(const uint64_t *offsets, const uint32_t *edges_slice, uint64_t num_vertices,
                  uint64_t num_edges, uint64_t e_begin, uint64_t e_count, uint32_t *r1_out,
                  uint64_t *bucket_counts, uint64_t *seg_hi_out, void *stream);
int gt_shard_receive(const uint32_t *r1_recv, uint64_t *seg_hi_recv, const uint64_t *counts, int nranks,
                     uint64_t num_vertices, uint64_t num_edges, uint32_t bucket_lo, uint32_t bucket_hi,
                     uint64_t num_records, uint64_t global_base, uint64_t *t_offsets_local,
                     uint32_t *t_edges_local, void *stream, gt_stats *stats);
/* Host: library workspace of a sender (level-1 tables for e_count edges) and of
 * a receiver (num_buckets_local buckets, num_records records from nranks
 * senders: R2 + tables), for memory planning. */
int gt_shard_workspace_size(uint64_t num_vertices, uint64_t num_edges, uint64_t e_count,
                            uint32_t num_buckets_local, int nranks, uint64_t num_records,
                            uint64_t *send_bytes, uint64_t *recv_bytes);
/* Host: owners' bucket ranges h_bounds[0..parts] (bucket-aligned, balanced on
 * the bucket totals). */
int gt_shard_owners(const uint64_t *h_bucket_totals, uint32_t num_buckets, int parts, uint32_t *h_bounds);

/* ---- the whole sharded transpose over NCCL (gt_multi.cu) -------------------
 * libnccl.so.2 is loaded at run time (the one already in the process, e.g.
 * torch's, else the system's).  gt_multi_unique_id fills 128 bytes (an
 * ncclUniqueId) on one rank; every rank passes the same bytes to
 * gt_multi_comm_init(id, rank, nranks) (on its device) and gets an opaque
 * communicator.  gt_transpose_multi is one rank's step: the rank owns the
 * edge-balanced source shard [src_begin, src_end) (gt_edge_balanced_bounds),
 * `offsets` is the full device offsets array and `edges_slice` the shard's
 * edges.  The rank receives the CSC slice of destinations
 * [info->dst_begin, info->dst_end): t_offsets_local (capacity
 * num_vertices + 1 entries suffices) with global positions starting at
 * info->global_base, and t_edges_local[info->num_local_edges]; if
 * t_edges_capacity is smaller, GT_ENOMEM with info->num_local_edges set.
 * One host synchronisation per step: the nranks x num_buckets count matrix
 * that sizes the NCCL sends. */
typedef struct gt_multi_info {
    uint64_t dst_begin, dst_end, global_base, num_local_edges;
    uint32_t bucket_lo, bucket_hi;
    double ms_send, ms_exchange, ms_receive; /* phase device times (CUDA events) */
} gt_multi_info;
int gt_multi_unique_id(void *id128);
int gt_multi_comm_init(const void *id128, int rank, int nranks, void **comm);
int gt_multi_comm_destroy(void *comm);
int gt_transpose_multi(void *comm, int rank, int nranks, const uint64_t *offsets, const uint32_t *edges_slice,
                       uint64_t num_vertices, uint64_t num_edges, uint64_t src_begin, uint64_t src_end,
                       uint64_t *t_offsets_local, uint32_t *t_edges_local, uint64_t t_edges_capacity,
                       gt_multi_info *info, void *stream);

/* ---- seeded synthetic inputs (BASELINE.json configs), generated on device --
 * Deterministic counter-based generators; identical to the numpy versions in
 * paper_2501_06872_b200/gen.py.  Pairs are written as src[i], dst[i]. */
int gt_gen_rmat(uint64_t scale, uint64_t num_edges, uint64_t seed, int permute,
                uint32_t *src, uint32_t *dst, void *stream);
int gt_gen_er(uint64_t num_vertices, uint64_t num_edges, uint64_t seed,
              uint32_t *src, uint32_t *dst, void *stream);
/* R-MAT straight into CSR form (memory-lean, for config C5): the same
 * counter-based stream as gt_gen_rmat regenerated twice (out-degree count,
 * then placement), so only offsets[V+1] (device) and edges[E] (device) are
 * materialised.  Lists are in an arbitrary order; sort them (gt_sort_lists or
 * two transposes) to get the config's CSR. */
int gt_gen_rmat_csr(uint64_t scale, uint64_t num_edges, uint64_t seed, int permute,
                    uint64_t *offsets, uint32_t *edges, void *stream);
/* Web-like graph (config C4), two calls.  gt_gen_web_degrees draws every
 * vertex's out-degree from the Zipf inverse-CDF thresholds deg_cdf (ndeg u64
 * entries, device), scales it by deg_scale_q16 / 65536 (rounded, >= 1) and
 * writes the exclusive scan into offsets[0..V] (device) and the edge count to
 * *num_edges (host).  gt_gen_web_edges writes the pairs in generation order:
 * with probability p_local_q32 / 2^32 the destination is uniform within
 * +-window of the source (mod V), otherwise hubs[rank] with rank drawn from
 * hub_cdf (nhub u64 thresholds, device).  Same draws as gen.web_pairs_np. */
int gt_gen_web_degrees(uint64_t num_vertices, uint64_t seed, const uint64_t *deg_cdf, uint32_t ndeg,
                       uint32_t deg_scale_q16, uint64_t *offsets, uint64_t *num_edges, void *stream);
int gt_gen_web_edges(uint64_t num_vertices, uint64_t seed, const uint64_t *offsets, const uint64_t *hub_cdf,
                     uint32_t nhub, const uint32_t *hubs, uint32_t window, uint32_t p_local_q32,
                     uint32_t *src, uint32_t *dst, void *stream);
/* COO pairs -> CSR with every list ascending by destination (duplicates kept).
 * Consumes src/dst (they are overwritten as scratch). */
int gt_build_csr(uint32_t *src, uint32_t *dst, uint64_t num_vertices, uint64_t num_edges,
                 uint64_t *offsets, uint32_t *edges, void *stream);

/* ---- step 0: high-degree-vertex sample (hlh.py:141-228) --------------------
 * gt_sample_hdv replaces sample_hdv (hlh.py:167-218) + _sample_tally
 * (hlh.py:153-164): num_samples > 0 draws that many edge positions in each of
 * two tallies from 2 * workers xoshiro256** streams seeded by successive
 * splitmix64 outputs of seed (worker_seeds, _nb.py:86-93); num_samples == 0
 * counts every edge (sample_fraction == 1).  hdv_ids (device, k <= V entries)
 * receives the k most counted endpoints of the first tally, most first, ties
 * to the lower ID (then zero-count vertices by ID); *h_hits = the second
 * tally's count over that set (the coverage estimate's numerator).  Same
 * result as the reference for the same (seed, workers).
 * gt_hdv_table_build: the plan's open-addressing table (_table_build,
 * hlh.py:81-90) on the device: keys[capacity] (u64, empty = ~0), vals[capacity]
 * = position in hdv_ids, slot (key * 0x9E3779B97F4A7C15) >> shift, linear
 * probing.  gt_hdv_lookup: out[i] = position of queries[i] or -1
 * (_table_find, hlh.py:68-78; hash_lookup, hlh.py:141-145).
 * gt_coverage_exact: *h_hits = edges whose endpoint is in the table
 * (coverage_exact, hlh.py:221-228).  All pointers but h_hits are device. */
int gt_sample_hdv(const uint32_t *edges, uint64_t num_edges, uint64_t num_vertices, uint64_t k,
                  uint64_t num_samples, uint64_t seed, int workers, uint64_t *hdv_ids, uint64_t *h_hits,
                  void *stream);
int gt_hdv_table_build(const uint64_t *hdv_ids, uint64_t k, uint64_t capacity, int shift, uint64_t *keys,
                       uint32_t *vals, void *stream);
int gt_hdv_lookup(const uint64_t *keys, const uint32_t *vals, uint64_t capacity, int shift,
                  const uint32_t *queries, uint64_t n, int64_t *out, void *stream);
int gt_coverage_exact(const uint64_t *keys, const uint32_t *vals, uint64_t capacity, int shift,
                      const uint32_t *edges, uint64_t num_edges, uint64_t *h_hits, void *stream);

/* ---- canonicalisation and verification on the device (bench.py:84-170) ----
 * gt_sort_lists: out_edges = every list of (offsets, edges) sorted ascending
 * (sort_neighbor_lists, baselines.py:457-475); the offsets are unchanged.
 * gt_first_diff_u64/_u32: *first = the first i < n with a[i] != b[i], else n.
 * gt_in_degree_offsets: offsets[V+1] = exclusive scan of the in-degrees of
 * edges (bincount + cumsum, bench.py:140-142).
 * gt_first_diff_lists: *first = the first j < n_vertices whose list
 * vertices[j] differs between (off_a, edges_a) and (off_b, edges_b), else
 * n_vertices (the per-vertex multiset check of bench.py:150-170 on
 * canonical lists). */
int gt_sort_lists(const uint64_t *offsets, const uint32_t *edges, uint64_t num_vertices, uint64_t num_edges,
                  uint32_t *out_edges, void *stream);
/* An independent transpose for verification (verify_output full-oracle):
 * offsets from the in-degree histogram, lists from a global radix sort of
 * (destination << 32 | source) keys (CUB) — transpose_oracle's lexsort
 * (graph.py:136-148) with none of the partition kernels it checks.  E < 2^32. */
/* Debug checks of a transpose (transpose_potra(debug=True), the GPU analogue
 * of the reference's write-once bitmap and conservation asserts,
 * hlh.py:400-419, 523-528, 550-558), run on a t_edges that was filled with
 * 0xFFFFFFFF before the transpose: unwritten = slots never written (a slot
 * written twice leaves another one unwritten), descents = adjacent pairs out
 * of order inside a list, offset_diff = first index where t_offsets differs
 * from the in-degree scan (V+1 if none), multiset_diff = first destination
 * whose list is not the multiset of its sources (hash sums; V if none). */
typedef struct gt_debug_report {
    uint64_t unwritten, descents, offset_diff, multiset_diff;
} gt_debug_report;
int gt_debug_check(const uint64_t *offsets, const uint32_t *edges, uint64_t num_vertices, uint64_t num_edges,
                   const uint64_t *t_offsets, const uint32_t *t_edges, gt_debug_report *report, void *stream);
int gt_verify_transpose(const uint64_t *offsets, const uint32_t *edges, uint64_t num_vertices, uint64_t num_edges,
                        uint64_t *t_offsets, uint32_t *t_edges, void *stream);
int gt_first_diff_u64(const uint64_t *a, const uint64_t *b, uint64_t n, uint64_t *first, void *stream);
int gt_first_diff_u32(const uint32_t *a, const uint32_t *b, uint64_t n, uint64_t *first, void *stream);
int gt_in_degree_offsets(const uint32_t *edges, uint64_t num_edges, uint64_t num_vertices, uint64_t *offsets,
                         void *stream);
int gt_first_diff_lists(const uint64_t *off_a, const uint32_t *edges_a, const uint64_t *off_b,
                        const uint32_t *edges_b, const uint32_t *vertices, uint64_t n_vertices, uint64_t *first,
                        void *stream);

/* ---- POTG files straight to / from device memory (io.py:24-114) ----------
 * gt_potg_read_header replaces the header half of _load_binary (io.py:54-84):
 * same checks, same order; on GT_EFORMAT gt_last_error() is the reference's
 * GraphFormatError message and *err_byte_offset its byte_offset.
 * gt_potg_read streams offsets and edges into caller device buffers
 * ((V+1)*8 and E*id_width bytes) and checks them on the device in the order
 * of io.py:86-109 (offsets[0], monotone, offsets[-1] == E, edge IDs < V).
 * gt_potg_write replaces store_graph (io.py:28-38) from device buffers. */
typedef struct gt_potg_header {
  uint32_t version, id_width, orientation, pad;
  uint64_t num_vertices, num_edges;
} gt_potg_header;
int gt_potg_read_header(const char *path, gt_potg_header *header, uint64_t *err_byte_offset);
int gt_potg_read(const char *path, const gt_potg_header *header, uint64_t *offsets, void *edges,
                 void *stream, uint64_t *err_byte_offset);
int gt_potg_write(const char *path, const uint64_t *offsets, const void *edges, uint64_t num_vertices,
                  uint64_t num_edges, int orientation, int id_width, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GT_H_ */

/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's graph
 * transposition path, used as the parity checker (tests/, smoke()) and as the
 * CPU baseline arm of bench.py.  Nothing in the product path links this file.
 *
 * Reference: arxiv/paper_2501_06872 (PoTra), Python package `potra`
 * (pkg/src/potra).  Each function names the reference code it restates.
 *
 *   gto_transpose_serial   transpose_oracle          graph.py:136-148
 *                          (via from_edge_pairs      graph.py:104-122: lexsort
 *                           (owner, endpoint) == stable counting sort of the
 *                           CSR-ordered edge stream by endpoint; offsets =
 *                           bincount + cumsum)
 *   gto_scan_exclusive     _scan_exclusive           baselines.py:65-88
 *   gto_transpose_scantrans transpose_scantrans      baselines.py:265-312
 *                          (_scantrans_count/_totals/_make_ip/_scatter
 *                           baselines.py:217-262), 64-bit cursors here
 *   gto_transpose_atomic   transpose_atomic          baselines.py:168-209
 *                          (_count_endpoints_atomic 135-142,
 *                           _scatter_atomic 145-157, relaxed fetch-add
 *                           _nb.py:21-44)
 *   gto_sort_lists         sort_neighbor_lists       baselines.py:448-475
 *   gto_edge_balanced_bounds edge_balanced_vertex_bounds _nb.py:118-132
 *
 * Conventions (graph.py:34-36, 59-80): offsets are uint64[V+1], edges are
 * uint32[E] (V <= 2^32).  Return 0 on success, GTO_EOVERFLOW when an in-degree
 * does not fit the reference's 32-bit counters (baselines.py:189-192),
 * GTO_EINVAL for bad arguments (threads < 1, _nb.py:112-113).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define GTO_OK 0
#define GTO_EINVAL (-1)
#define GTO_EOVERFLOW (-2)
#define GTO_ENOMEM (-3)

/* ---- serial oracle: stable counting sort by endpoint (graph.py:104-148) --- */
int gto_transpose_serial(const uint64_t *offsets, const uint32_t *edges,
                         uint64_t nv, uint64_t ne, uint64_t *t_offsets,
                         uint32_t *t_edges) {
    /* bincount(endpoints) -> cumsum (graph.py:119-121), 64-bit counts */
    memset(t_offsets, 0, (nv + 1) * sizeof(uint64_t));
    for (uint64_t j = 0; j < ne; ++j) t_offsets[(uint64_t)edges[j] + 1] += 1;
    for (uint64_t v = 0; v < nv; ++v) t_offsets[v + 1] += t_offsets[v];
    uint64_t *cur = (uint64_t *)malloc((nv ? nv : 1) * sizeof(uint64_t));
    if (!cur) return GTO_ENOMEM;
    memcpy(cur, t_offsets, nv * sizeof(uint64_t));
    /* owners visited in ascending order == lexsort secondary key (owner) */
    for (uint64_t v = 0; v < nv; ++v)
        for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j)
            t_edges[cur[edges[j]]++] = (uint32_t)v;
    free(cur);
    return GTO_OK;
}

/* ---- _scan_exclusive (baselines.py:65-88): u32 counts -> u64[n+1] -------- */
int gto_scan_exclusive(const uint32_t *counts, uint64_t n, uint64_t *out,
                       int threads) {
    if (threads < 1) return GTO_EINVAL;
    int64_t *sums = (int64_t *)calloc((size_t)threads, sizeof(int64_t));
    if (!sums) return GTO_ENOMEM;
#pragma omp parallel for num_threads(threads) schedule(static, 1)
    for (int w = 0; w < threads; ++w) {
        uint64_t lo = (uint64_t)w * n / threads, hi = (uint64_t)(w + 1) * n / threads;
        int64_t s = 0;
        for (uint64_t i = lo; i < hi; ++i) s += counts[i];
        sums[w] = s;
    }
    int64_t total = 0;
    for (int w = 0; w < threads; ++w) { int64_t t = sums[w]; sums[w] = total; total += t; }
#pragma omp parallel for num_threads(threads) schedule(static, 1)
    for (int w = 0; w < threads; ++w) {
        uint64_t lo = (uint64_t)w * n / threads, hi = (uint64_t)(w + 1) * n / threads;
        int64_t acc = sums[w];
        for (uint64_t i = lo; i < hi; ++i) { out[i] = (uint64_t)acc; acc += counts[i]; }
    }
    out[n] = (uint64_t)total;
    free(sums);
    return GTO_OK;
}

/* ---- edge_balanced_vertex_bounds (_nb.py:118-132) ------------------------ */
/* targets = arange(parts+1)*E // parts; bounds = searchsorted(offsets, targets,
 * 'left'); bounds[0] = 0; bounds[-1] = V.  (E*p computed in 128 bits.) */
void gto_edge_balanced_bounds(const uint64_t *offsets, uint64_t nv, int64_t parts,
                              int64_t *bounds) {
    if (parts < 1) parts = 1;
    uint64_t ne = offsets[nv];
    for (int64_t p = 0; p <= parts; ++p) {
        unsigned __int128 t = (unsigned __int128)ne * (uint64_t)p / (uint64_t)parts;
        uint64_t target = (uint64_t)t;
        uint64_t lo = 0, hi = nv + 1; /* first index i with offsets[i] >= target */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (offsets[mid] < target) lo = mid + 1; else hi = mid;
        }
        bounds[p] = (int64_t)lo;
    }
    bounds[0] = 0;
    bounds[parts] = (int64_t)nv;
}

/* ---- transpose_scantrans (baselines.py:265-312) -------------------------- */
/* Per-worker private counters c[w, V] over one edge-balanced source range each;
 * cursors ordered by worker rank inside each vertex slot -> sorted output.  The
 * reference uses u32 cursors and refuses |E| >= 2^32 (baselines.py:278-281);
 * this port keeps that contract. */
int gto_transpose_scantrans(const uint64_t *offsets, const uint32_t *edges,
                            uint64_t nv, uint64_t ne, uint64_t *t_offsets,
                            uint32_t *t_edges, int threads) {
    if (threads < 1) return GTO_EINVAL;
    if (ne >= (1ull << 32)) return GTO_EOVERFLOW;
    int64_t *vb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(threads + 1));
    uint32_t *c = (uint32_t *)calloc((size_t)threads * (nv ? nv : 1), sizeof(uint32_t));
    if (!vb || !c) { free(vb); free(c); return GTO_ENOMEM; }
    gto_edge_balanced_bounds(offsets, nv, threads, vb);
#pragma omp parallel num_threads(threads)
    {
        /* _scantrans_count (baselines.py:217-223) */
#pragma omp for schedule(static, 1)
        for (int w = 0; w < threads; ++w) {
            uint32_t *cw = c + (size_t)w * nv;
            for (int64_t v = vb[w]; v < vb[w + 1]; ++v)
                for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) cw[edges[j]]++;
        }
        /* _scantrans_totals (baselines.py:226-235) */
#pragma omp for schedule(static)
        for (int64_t v = 0; v < (int64_t)nv; ++v) {
            uint64_t s = 0;
            for (int w = 0; w < threads; ++w) s += c[(size_t)w * nv + v];
            t_offsets[v + 1] = s;
        }
#pragma omp single
        {
            t_offsets[0] = 0;
            for (uint64_t v = 0; v < nv; ++v) t_offsets[v + 1] += t_offsets[v];
        }
        /* _scantrans_make_ip (baselines.py:238-250) */
#pragma omp for schedule(static)
        for (int64_t v = 0; v < (int64_t)nv; ++v) {
            uint32_t run = (uint32_t)t_offsets[v];
            for (int w = 0; w < threads; ++w) {
                uint32_t tmp = c[(size_t)w * nv + v];
                c[(size_t)w * nv + v] = run;
                run += tmp;
            }
        }
        /* _scantrans_scatter (baselines.py:253-262) */
#pragma omp for schedule(static, 1)
        for (int w = 0; w < threads; ++w) {
            uint32_t *cw = c + (size_t)w * nv;
            for (int64_t v = vb[w]; v < vb[w + 1]; ++v)
                for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j)
                    t_edges[cw[edges[j]]++] = (uint32_t)v;
        }
    }
    free(vb);
    free(c);
    return GTO_OK;
}

/* ---- transpose_atomic (baselines.py:168-209) ----------------------------- */
/* step 1 relaxed u32 fetch-add per endpoint, step 2 exclusive scan + overflow
 * check, step 3 dynamic claim of edge-balanced partitions with i64 fetch-add
 * slot reservation.  Output lists are in scheduling order (unsorted). */
static int64_t partition_count(uint64_t ne, int workers, uint64_t partition_edges) {
    if (ne == 0) return 1; /* baselines.py:160-165 */
    int64_t parts = (int64_t)((ne + partition_edges - 1) / partition_edges);
    int64_t m = parts > 4 * (int64_t)workers ? parts : 4 * (int64_t)workers;
    if (m > (int64_t)ne) m = (int64_t)ne;
    return m < 1 ? 1 : m;
}

int gto_transpose_atomic(const uint64_t *offsets, const uint32_t *edges,
                         uint64_t nv, uint64_t ne, uint64_t *t_offsets,
                         uint32_t *t_edges, int threads, uint64_t partition_edges) {
    if (threads < 1 || partition_edges < 1) return GTO_EINVAL;
    uint32_t *counters = (uint32_t *)calloc(nv ? nv : 1, sizeof(uint32_t));
    int64_t *ip = (int64_t *)malloc((nv ? nv : 1) * sizeof(int64_t));
    if (!counters || !ip) { free(counters); free(ip); return GTO_ENOMEM; }
#pragma omp parallel for num_threads(threads) schedule(static)
    for (uint64_t i = 0; i < ne; ++i)
        __atomic_fetch_add(&counters[edges[i]], 1u, __ATOMIC_RELAXED);
    gto_scan_exclusive(counters, nv, t_offsets, threads);
    if (t_offsets[nv] != ne) { free(counters); free(ip); return GTO_EOVERFLOW; }
    for (uint64_t v = 0; v < nv; ++v) ip[v] = (int64_t)t_offsets[v];
    int64_t parts = partition_count(ne, threads, partition_edges);
    int64_t *vb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(parts + 1));
    if (!vb) { free(counters); free(ip); return GTO_ENOMEM; }
    gto_edge_balanced_bounds(offsets, nv, parts, vb);
    int64_t cursor = 0;
#pragma omp parallel num_threads(threads)
    {
        for (;;) {
            int64_t p = __atomic_fetch_add(&cursor, 1, __ATOMIC_RELAXED);
            if (p >= parts) break;
            for (int64_t v = vb[p]; v < vb[p + 1]; ++v)
                for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
                    int64_t idx = __atomic_fetch_add(&ip[edges[j]], 1, __ATOMIC_RELAXED);
                    t_edges[idx] = (uint32_t)v;
                }
        }
    }
    free(vb);
    free(counters);
    free(ip);
    return GTO_OK;
}

/* ---- sort_neighbor_lists / _sort_segments (baselines.py:448-475) --------- */
static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

int gto_sort_lists(const uint64_t *offsets, uint64_t nv, uint32_t *edges, int threads) {
    if (threads < 1) return GTO_EINVAL;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4096)
    for (int64_t v = 0; v < (int64_t)nv; ++v) {
        uint64_t a = offsets[v], b = offsets[v + 1];
        if (b - a > 1) qsort(edges + a, (size_t)(b - a), sizeof(uint32_t), cmp_u32);
    }
    return GTO_OK;
}

int gto_max_threads(void) { return omp_get_max_threads(); }

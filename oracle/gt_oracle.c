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
#include <math.h>
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

/* ======================================================================== */
/* Seeded synthetic graphs (CPU side, test infrastructure): the same counter-  */
/* based draws as paper_2501_06872_b200/gen.py (rmat_pairs_np, er_pairs_np,   */
/* csr_from_pairs_np) so bench.py's reference arm builds its input without the */
/* product library.  CSR lists come out sorted ascending by destination.       */
/* ======================================================================== */
#define GTO_GOLDEN 0x9E3779B97F4A7C15ull
#define GTO_SEED_MUL 0xD1B54A32D192ED03ull
#define GTO_RMAT_A 2448131358u
#define GTO_RMAT_AB 3264175144u
#define GTO_RMAT_ABC 4080218931u

static inline uint64_t gto_mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t gto_stream_key(uint64_t seed, uint64_t stream) {
    return gto_mix64(seed * GTO_SEED_MUL + stream * GTO_GOLDEN + 1);
}
static inline uint64_t gto_hash_at(uint64_t key, uint64_t idx) { return gto_mix64(key + (idx + 1) * GTO_GOLDEN); }

typedef struct { uint64_t keys[4]; int half; uint64_t mask, n; } gto_perm;
static void gto_perm_init(gto_perm *p, int scale, uint64_t seed) {
    int width = scale + (scale & 1);
    p->half = width / 2;
    p->mask = (1ull << p->half) - 1;
    p->n = 1ull << scale;
    uint64_t pk = gto_stream_key(seed, 2 /* STREAM_PERM */);
    for (int r = 0; r < 4; ++r) p->keys[r] = gto_hash_at(pk, (uint64_t)r);
}
static inline uint64_t gto_feistel(const gto_perm *p, uint64_t x) {
    uint64_t L = x >> p->half, R = x & p->mask;
    for (int r = 0; r < 4; ++r) {
        uint64_t t = L ^ (gto_mix64(R ^ p->keys[r]) & p->mask);
        L = R; R = t;
    }
    return (L << p->half) | R;
}
static inline uint64_t gto_permute(const gto_perm *p, uint64_t x) {
    uint64_t y = gto_feistel(p, x);
    while (y >= p->n) y = gto_feistel(p, y); /* cycle walking */
    return y;
}

/* kind 0 = R-MAT (.57/.19/.19/.05), 1 = Erdos-Renyi */
typedef struct { int kind, scale, permute; uint64_t nv, key; gto_perm perm; } gto_gen;
static inline void gto_pair(const gto_gen *g, uint64_t e, uint32_t *src, uint32_t *dst) {
    if (g->kind == 1) {
        *src = (uint32_t)(((gto_hash_at(g->key, 2 * e) >> 32) * g->nv) >> 32);
        *dst = (uint32_t)(((gto_hash_at(g->key, 2 * e + 1) >> 32) * g->nv) >> 32);
        return;
    }
    uint64_t s = 0, d = 0;
    for (int l = 0; l < g->scale; l += 2) {
        uint64_t h = gto_hash_at(g->key, e * 16 + (uint64_t)(l >> 1));
        for (int q = 0; q < 2 && l + q < g->scale; ++q) {
            uint32_t u = (uint32_t)(h >> (32 * q));
            uint64_t bit = 1ull << (g->scale - 1 - (l + q));
            int in_b = u >= GTO_RMAT_A && u < GTO_RMAT_AB, in_c = u >= GTO_RMAT_AB && u < GTO_RMAT_ABC;
            int in_d = u >= GTO_RMAT_ABC;
            if (in_b || in_d) d |= bit;
            if (in_c || in_d) s |= bit;
        }
    }
    if (g->permute) { s = gto_permute(&g->perm, s); d = gto_permute(&g->perm, d); }
    *src = (uint32_t)s;
    *dst = (uint32_t)d;
}

static int cmp_u32(const void *a, const void *b);

/* Two passes over the draws (count sources, then place destinations with
 * atomic cursors) and a per-list sort: the CSR of csr_from_pairs_np
 * (lexsort((dst, src))) without materialising the pair arrays. */
int gto_generate(int kind, int scale, int permute, uint64_t nv, uint64_t ne, uint64_t seed,
                 uint64_t *offsets, uint32_t *edges, int threads) {
    if (threads < 1 || (kind != 0 && kind != 1)) return GTO_EINVAL;
    gto_gen g;
    g.kind = kind; g.scale = scale; g.permute = permute; g.nv = nv;
    g.key = gto_stream_key(seed, kind == 0 ? 1 /* STREAM_RMAT */ : 3 /* STREAM_ER */);
    if (kind == 0) gto_perm_init(&g.perm, scale, seed);
    uint64_t *cur = (uint64_t *)calloc(nv + 1, sizeof(uint64_t));
    if (!cur) return GTO_ENOMEM;
#pragma omp parallel for num_threads(threads) schedule(static, 1 << 16)
    for (int64_t e = 0; e < (int64_t)ne; ++e) {
        uint32_t s, d;
        gto_pair(&g, (uint64_t)e, &s, &d);
        __atomic_fetch_add(&cur[s], 1ull, __ATOMIC_RELAXED);
    }
    offsets[0] = 0;
    for (uint64_t v = 0; v < nv; ++v) { offsets[v + 1] = offsets[v] + cur[v]; cur[v] = offsets[v]; }
#pragma omp parallel for num_threads(threads) schedule(static, 1 << 16)
    for (int64_t e = 0; e < (int64_t)ne; ++e) {
        uint32_t s, d;
        gto_pair(&g, (uint64_t)e, &s, &d);
        edges[__atomic_fetch_add(&cur[s], 1ull, __ATOMIC_RELAXED)] = d;
    }
    free(cur);
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4096)
    for (int64_t v = 0; v < (int64_t)nv; ++v) {
        uint64_t a = offsets[v], b = offsets[v + 1];
        if (b - a > 1) qsort(edges + a, (size_t)(b - a), sizeof(uint32_t), cmp_u32);
    }
    return GTO_OK;
}

/* ======================================================================== */
/* transpose_potra (hlh.py:441-588): step 0 (sample_hdv hlh.py:167-218 with  */
/* the reference's xoshiro256** worker streams _nb.py:47-93, the compressing */
/* linear-probe table hlh.py:68-90, probe_methods hlh.py:293-333), then the  */
/* HLH steps 1-3 (_hlh_step1 / _hlh_degrees / _hlh_step3, hlh.py:340-397) or */
/* the atomic baseline when the probe picks it.  Output lists are unsorted,  */
/* as the reference's (sorted=False); gto_sort_lists canonicalises them.      */
/* ======================================================================== */
#define GTO_EMPTY 0xFFFFFFFFFFFFFFFFull
typedef struct { uint64_t *keys; uint32_t *vals; uint64_t cap; int shift; } gto_table;

static inline int64_t gto_table_find(const gto_table *t, uint64_t key) {
    uint64_t mask = t->cap - 1, i = (key * GTO_GOLDEN) >> t->shift;
    for (;;) {
        uint64_t k = t->keys[i & mask];
        if (k == key) return (int64_t)t->vals[i & mask];
        if (k == GTO_EMPTY) return -1;
        ++i;
    }
}

static inline uint64_t gto_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t gto_splitmix(uint64_t *x) {
    *x += GTO_GOLDEN;
    return gto_mix64(*x);
}

static void gto_tally(const uint32_t *edges, uint64_t ne, uint64_t num_samples, const uint64_t *seeds, int workers,
                      uint32_t *freq) {
#pragma omp parallel for num_threads(workers) schedule(static, 1)
    for (int w = 0; w < workers; ++w) {
        uint64_t lo = (uint64_t)w * num_samples / workers, hi = (uint64_t)(w + 1) * num_samples / workers;
        uint64_t x = seeds[w];
        uint64_t s0 = gto_splitmix(&x), s1 = gto_splitmix(&x), s2 = gto_splitmix(&x), s3 = gto_splitmix(&x);
        for (uint64_t i = lo; i < hi; ++i) {
            uint64_t r = gto_rotl(s1 * 5, 7) * 9, t = s1 << 17;
            s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = gto_rotl(s3, 45);
            __atomic_fetch_add(&freq[edges[r % ne]], 1u, __ATOMIC_RELAXED);
        }
    }
}

typedef struct { uint32_t f; uint32_t id; } gto_cand;
static int cmp_cand(const void *a, const void *b) { /* (-freq, id) */
    const gto_cand *x = (const gto_cand *)a, *y = (const gto_cand *)b;
    if (x->f != y->f) return x->f > y->f ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static double gto_now(void) { return omp_get_wtime(); }

/* phase[0..3] = step0..step3 seconds; info[0] = method (0 atomic, 1 hlh),
 * info[1] = k, info[2] = sample size; est = coverage estimate. */
int gto_transpose_potra(const uint64_t *offsets, const uint32_t *edges, uint64_t nv, uint64_t ne,
                        uint64_t *t_offsets, uint32_t *t_edges, int threads, int64_t k, double sample_fraction,
                        uint64_t seed, uint64_t partition_edges, int force_method, double *phase, int64_t *info,
                        double *est) {
    if (threads < 1 || partition_edges < 1 || k < 0) return GTO_EINVAL;
    const int W = threads;
    double t_start = gto_now();
    if ((uint64_t)k > nv) k = (int64_t)nv;
    /* ---- step 0: sample_hdv ---- */
    uint64_t size = 0;
    uint32_t *freq = (uint32_t *)calloc(nv ? nv : 1, sizeof(uint32_t));
    uint32_t *estf = (uint32_t *)calloc(nv ? nv : 1, sizeof(uint32_t));
    if (!freq || !estf) { free(freq); free(estf); return GTO_ENOMEM; }
    if (sample_fraction >= 1.0 || ne == 0) {
        for (uint64_t j = 0; j < ne; ++j) freq[edges[j]]++;
        memcpy(estf, freq, nv * sizeof(uint32_t));
        size = ne;
    } else {
        size = (uint64_t)ceil(sample_fraction * (double)nv);
        uint64_t *seeds = (uint64_t *)malloc(sizeof(uint64_t) * 2 * W), x = seed;
        for (int w = 0; w < 2 * W; ++w) seeds[w] = gto_splitmix(&x);
        if (size) {
            gto_tally(edges, ne, size, seeds, W, freq);
            gto_tally(edges, ne, size, seeds + W, W, estf);
        }
        free(seeds);
    }
    uint64_t *ids = (uint64_t *)malloc(sizeof(uint64_t) * (k ? k : 1));
    {
        uint64_t nc = 0;
        for (uint64_t v = 0; v < nv; ++v) nc += freq[v] != 0;
        gto_cand *c = (gto_cand *)malloc(sizeof(gto_cand) * (nc ? nc : 1));
        nc = 0;
        for (uint64_t v = 0; v < nv; ++v)
            if (freq[v]) { c[nc].f = freq[v]; c[nc].id = (uint32_t)v; ++nc; }
        qsort(c, nc, sizeof(gto_cand), cmp_cand);
        int64_t m = 0;
        for (; m < k && (uint64_t)m < nc; ++m) ids[m] = c[m].id;
        for (uint64_t v = 0; m < k; ++v) /* zero-frequency vertices by ascending id */
            if (!freq[v]) ids[m++] = v;
        free(c);
    }
    uint64_t hits = 0;
    for (int64_t i = 0; i < k; ++i) hits += estf[ids[i]];
    *est = size ? (double)hits / (double)size : 0.0;
    free(freq);
    free(estf);
    gto_table tb;
    {
        uint64_t need = k ? (uint64_t)ceil((double)k / 0.5) : 2, cap = 2;
        while (cap < need) cap <<= 1;
        tb.cap = cap;
        int lg = 0;
        while ((1ull << lg) < cap) ++lg;
        tb.shift = 64 - lg;
        tb.keys = (uint64_t *)malloc(sizeof(uint64_t) * cap);
        tb.vals = (uint32_t *)calloc(cap, sizeof(uint32_t));
        for (uint64_t i = 0; i < cap; ++i) tb.keys[i] = GTO_EMPTY;
        for (int64_t n = 0; n < k; ++n) {
            uint64_t i = (ids[n] * GTO_GOLDEN) >> tb.shift;
            while (tb.keys[i & (cap - 1)] != GTO_EMPTY) ++i;
            tb.keys[i & (cap - 1)] = ids[n];
            tb.vals[i & (cap - 1)] = (uint32_t)n;
        }
    }
    const int64_t k1 = k > 0 ? k : 1;
    uint32_t *ldv = (uint32_t *)calloc(nv ? nv : 1, sizeof(uint32_t));
    uint8_t *low = (uint8_t *)calloc((size_t)W * k1, 1);
    uint32_t *high = (uint32_t *)calloc((size_t)W * k1, sizeof(uint32_t));
    /* ---- probe_methods: split counting vs atomic counting on an edge prefix ---- */
    int method = force_method; /* -1 = probe, 0 = atomic, 1 = hlh */
    if (method < 0) {
        uint64_t n = ne / 100 ? ne / 100 : 1;
        if (n > (1ull << 24)) n = 1ull << 24;
        if (n > ne) n = ne;
        if (n == 0) {
            method = 0;
        } else {
            uint32_t *cnt = (uint32_t *)calloc(nv ? nv : 1, sizeof(uint32_t));
            double th = 0, ta = 0;
            for (int pass = 0; pass < 2; ++pass) {
                uint64_t m = pass ? n : (n < 4096 ? n : 4096);
                double t0 = gto_now();
#pragma omp parallel for num_threads(W) schedule(static, 1)
                for (int w = 0; w < W; ++w)
                    for (uint64_t i = (uint64_t)w * m / W; i < (uint64_t)(w + 1) * m / W; ++i) {
                        int64_t t = gto_table_find(&tb, edges[i]);
                        if (t < 0) __atomic_fetch_add(&ldv[edges[i]], 1u, __ATOMIC_RELAXED);
                        else if (++low[(size_t)w * k1 + t] == 0) high[(size_t)w * k1 + t]++;
                    }
                double t1 = gto_now();
#pragma omp parallel for num_threads(W) schedule(static, 1)
                for (int w = 0; w < W; ++w)
                    for (uint64_t i = (uint64_t)w * m / W; i < (uint64_t)(w + 1) * m / W; ++i)
                        __atomic_fetch_add(&cnt[edges[i]], 1u, __ATOMIC_RELAXED);
                double t2 = gto_now();
                if (pass) { th = t1 - t0; ta = t2 - t1; }
            }
            free(cnt);
            method = th < ta ? 1 : 0;
            memset(ldv, 0, (nv ? nv : 1) * sizeof(uint32_t));
            memset(low, 0, (size_t)W * k1);
            memset(high, 0, (size_t)W * k1 * sizeof(uint32_t));
        }
    }
    phase[0] = gto_now() - t_start;
    info[0] = method;
    info[1] = k;
    info[2] = (int64_t)size;
    int rc = GTO_OK;
    if (method == 0) {
        double t0 = gto_now();
        rc = gto_transpose_atomic(offsets, edges, nv, ne, t_offsets, t_edges, W, partition_edges);
        phase[1] = gto_now() - t0; /* steps 1-3 of the atomic baseline together */
        phase[2] = phase[3] = 0.0;
        goto done;
    }
    {
        /* ---- step 1 ---- */
        double t0 = gto_now();
        int64_t parts = ne ? (int64_t)((ne + partition_edges - 1) / partition_edges) : 1;
        if (parts < 1) parts = 1;
        int64_t *vb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(parts + 1));
        int32_t *p2t = (int32_t *)malloc(sizeof(int32_t) * (size_t)parts);
        gto_edge_balanced_bounds(offsets, nv, parts, vb);
        int64_t cursor = 0;
#pragma omp parallel num_threads(W)
        {
            const int w = omp_get_thread_num();
            for (;;) {
                int64_t p = __atomic_fetch_add(&cursor, 1, __ATOMIC_RELAXED);
                if (p >= parts) break;
                p2t[p] = w;
                for (int64_t v = vb[p]; v < vb[p + 1]; ++v)
                    for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
                        const uint32_t e = edges[j];
                        int64_t t = gto_table_find(&tb, e);
                        if (t < 0) __atomic_fetch_add(&ldv[e], 1u, __ATOMIC_RELAXED);
                        else if (++low[(size_t)w * k1 + t] == 0) high[(size_t)w * k1 + t]++;
                    }
            }
        }
        double t1 = gto_now();
        /* ---- step 2: degrees, scan, cursors ---- */
#pragma omp parallel for num_threads(W) schedule(static)
        for (int64_t v = 0; v < (int64_t)nv; ++v) {
            int64_t t = gto_table_find(&tb, (uint64_t)v);
            uint64_t d = 0;
            if (t < 0) d = ldv[v];
            else for (int w = 0; w < W; ++w) d += (uint64_t)high[(size_t)w * k1 + t] * 256 + low[(size_t)w * k1 + t];
            t_offsets[v + 1] = d;
        }
        t_offsets[0] = 0;
        for (uint64_t v = 0; v < nv; ++v) t_offsets[v + 1] += t_offsets[v];
        int64_t *ip = NULL, *hip = NULL;
        if (t_offsets[nv] != ne) { rc = GTO_EOVERFLOW; free(vb); free(p2t); goto done; }
        ip = (int64_t *)malloc(sizeof(int64_t) * (nv ? nv : 1));
        hip = (int64_t *)malloc(sizeof(int64_t) * (size_t)W * k1);
#pragma omp parallel for num_threads(W) schedule(static)
        for (int64_t v = 0; v < (int64_t)nv; ++v) ip[v] = (int64_t)t_offsets[v];
        for (int64_t t = 0; t < k; ++t) {
            int64_t run = (int64_t)t_offsets[ids[t]];
            for (int w = 0; w < W; ++w) {
                hip[(size_t)w * k1 + t] = run;
                run += (int64_t)high[(size_t)w * k1 + t] * 256 + low[(size_t)w * k1 + t];
            }
        }
        double t2 = gto_now();
        /* ---- step 3: each worker replays the partitions it claimed ---- */
#pragma omp parallel num_threads(W)
        {
            const int w = omp_get_thread_num();
            for (int64_t p = 0; p < parts; ++p) {
                if (p2t[p] != w) continue;
                for (int64_t v = vb[p]; v < vb[p + 1]; ++v)
                    for (uint64_t j = offsets[v]; j < offsets[v + 1]; ++j) {
                        const uint32_t u = edges[j];
                        int64_t t = gto_table_find(&tb, u), idx;
                        if (t < 0) idx = __atomic_fetch_add(&ip[u], 1, __ATOMIC_RELAXED);
                        else idx = hip[(size_t)w * k1 + t]++;
                        t_edges[idx] = (uint32_t)v;
                    }
            }
        }
        double t3 = gto_now();
        phase[1] = t1 - t0;
        phase[2] = t2 - t1;
        phase[3] = t3 - t2;
        free(vb); free(p2t); free(ip); free(hip);
    }
done:
    free(ids); free(tb.keys); free(tb.vals); free(ldv); free(low); free(high);
    return rc;
}

/*
 * cetc_oracle.c — CPU restatement of the reference's cover-edge triangle
 * counting (CETC) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or as the timed CPU baseline — never as the
 * product path.  The product path (paper_2403_02997_b200) never links it.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to the reference package, pkg/src/tricount/).
 * Parity of this restatement with the reference is pinned by
 * tests/golden/ (fixtures produced by importing the reference itself,
 * see tests/golden/make_golden.py) and tests/test_oracle.py.
 *
 * Build: see oracle/Makefile (gcc -O3 -fopenmp -shared).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* numpy PCG64 (XSL-RR 128/64) — the bit stream numpy.random.default_rng
 * draws from.  rmat.py:57 seeds default_rng(seed); rmat.py:63 draws
 * rng.random((count, scale)) = (next64 >> 11) * 2^-53 per element, in
 * C order, block after block, so draw index = pair*scale + bit.  The
 * initial (state, inc) is read from numpy on the host
 * (rng.bit_generator.state) and passed in.                            */

static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static inline uint64_t pcg_out(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64 - r) & 63));
}

static inline u128 pcg_advance(u128 state, u128 inc, u128 delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

/* First `count` doubles of the stream (used by tests to pin pcg). */
void orc_pcg64_doubles(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                       uint64_t inc_lo, int64_t skip, int64_t count,
                       double* out) {
    u128 s = ((u128)st_hi << 64) | st_lo;
    u128 inc = ((u128)inc_hi << 64) | inc_lo;
    s = pcg_advance(s, inc, (u128)skip);
    for (int64_t i = 0; i < count; ++i) {
        s = s * PCG_MULT + inc;
        out[i] = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    }
}

/* rmat.py:45-72 generate_rmat: edge_factor * 2^scale pairs; one quadrant
 * choice per bit level, most significant bit first (rmat.py:64-67).
 * `perm` (optional, length 2^scale) relabels both endpoints afterwards
 * (config recipe of SURVEY.md §8(d); not part of the reference).      */
void orc_rmat(int scale, int64_t edge_factor, double a, double b, double c,
              uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
              const int64_t* perm, int64_t* pairs) {
    const int64_t n = (int64_t)1 << scale;
    const int64_t total = edge_factor * n;
    const u128 s0 = ((u128)st_hi << 64) | st_lo;
    const u128 inc = ((u128)inc_hi << 64) | inc_lo;
    const double ab = a + b;         /* rmat.py:64  r >= a + b          */
    const double abc = a + b + c;    /* rmat.py:65  r >= a + b + c      */
    const int64_t chunk = 1 << 16;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c0 = 0; c0 < total; c0 += chunk) {
        int64_t c1 = c0 + chunk < total ? c0 + chunk : total;
        u128 s = pcg_advance(s0, inc, (u128)c0 * (u128)scale);
        for (int64_t i = c0; i < c1; ++i) {
            int64_t u = 0, v = 0;
            for (int j = 0; j < scale; ++j) {
                s = s * PCG_MULT + inc;
                double r = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
                int ubit = r >= ab;
                int vbit = ((r >= a) && (r < ab)) || (r >= abc);
                u = (u << 1) | ubit;
                v = (v << 1) | vbit;
            }
            if (perm) { u = perm[u]; v = perm[v]; }
            pairs[2 * i] = u;
            pairs[2 * i + 1] = v;
        }
    }
}

/* ------------------------------------------------------------------ */
/* graph.py:177-194 normalize + graph.py:104-125 _graph_from_canonical_pairs:
 * drop self-loops, dedup undirected pairs, store both directions, sort
 * each adjacency list ascending, row_offsets = cumsum of degrees, and
 * edge_u/edge_v = the u<v pairs in lexicographic order.
 * Restated as one LSD radix sort over (src<<32 | dst) keys.
 * Returns m (undirected edge count).  nb needs room for 2k entries;
 * eu/ev (may be NULL) for k entries.                                  */

static void radix_sort_u64(uint64_t* keys, uint64_t* tmp, int64_t len,
                           int lo_bits, int hi_shift, int hi_bits) {
    /* sort on bits [0, lo_bits) then [hi_shift, hi_shift+hi_bits) */
    int passes[16][2];
    int np = 0;
    for (int b = 0; b < lo_bits; b += 11) {
        passes[np][0] = b;
        passes[np][1] = (lo_bits - b) < 11 ? (lo_bits - b) : 11;
        np++;
    }
    for (int b = 0; b < hi_bits; b += 11) {
        passes[np][0] = hi_shift + b;
        passes[np][1] = (hi_bits - b) < 11 ? (hi_bits - b) : 11;
        np++;
    }
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) << 11);
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    for (int p = 0; p < np; ++p) {
        int sh = passes[p][0], nbits = passes[p][1];
        int64_t nb = (int64_t)1 << nbits;
        uint64_t mask = (uint64_t)nb - 1;
        memset(cnt, 0, sizeof(int64_t) * nb);
        for (int64_t i = 0; i < len; ++i) cnt[(src[i] >> sh) & mask]++;
        int64_t run = 0;
        for (int64_t d = 0; d < nb; ++d) { int64_t t = cnt[d]; cnt[d] = run; run += t; }
        for (int64_t i = 0; i < len; ++i) dst[cnt[(src[i] >> sh) & mask]++] = src[i];
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != keys) memcpy(keys, src, sizeof(uint64_t) * len);
    free(cnt);
}

static int bits_for(int64_t n) {
    int b = 0;
    while (((int64_t)1 << b) < n) b++;
    return b;
}

int64_t orc_normalize(int64_t n, int64_t k, const int64_t* pairs,
                      int64_t* row, int32_t* nb, int32_t* eu, int32_t* ev) {
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (2 * k + 1));
    uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (2 * k + 1));
    int64_t len = 0;
    for (int64_t i = 0; i < k; ++i) {
        uint64_t a = (uint64_t)pairs[2 * i], b = (uint64_t)pairs[2 * i + 1];
        if (a == b) continue;                 /* graph.py:187-188 */
        keys[len++] = (a << 32) | b;          /* both directions:  */
        keys[len++] = (b << 32) | a;          /* graph.py:111-112  */
    }
    int vb = bits_for(n);
    radix_sort_u64(keys, tmp, len, vb, 32, vb); /* graph.py:113 lexsort */
    int64_t out = 0;
    for (int64_t i = 0; i < len; ++i)         /* graph.py:192 unique */
        if (i == 0 || keys[i] != keys[i - 1]) keys[out++] = keys[i];
    /* graph.py:115-117 bincount + cumsum */
    memset(row, 0, sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < out; ++i) row[(keys[i] >> 32) + 1]++;
    for (int64_t v = 0; v < n; ++v) row[v + 1] += row[v];
    int64_t m = 0;
    for (int64_t i = 0; i < out; ++i) {
        uint32_t s = (uint32_t)(keys[i] >> 32), d = (uint32_t)keys[i];
        nb[i] = (int32_t)d;
        if (d > s) {                          /* graph.py:108-110 u<v, lexsorted */
            if (eu) { eu[m] = (int32_t)s; ev[m] = (int32_t)d; }
            m++;
        }
    }
    free(keys);
    free(tmp);
    return m;
}

/* ------------------------------------------------------------------ */
/* _kernels.py:129-157 bfs_levels_k: roots are the lowest-id unvisited
 * vertices (:137-142), FIFO queue, neighbours in ascending order
 * (:143-156).  Returns components; *max_level out.                    */
int64_t orc_bfs_levels(const int64_t* row, const int32_t* nb, int64_t n,
                       int64_t* level, int64_t* parent, int64_t* max_level_out) {
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    for (int64_t v = 0; v < n; ++v) { level[v] = -1; if (parent) parent[v] = -1; }
    int64_t components = 0, max_level = 0;
    for (int64_t r = 0; r < n; ++r) {
        if (level[r] >= 0) continue;
        components++;
        level[r] = 0;
        queue[0] = r;
        int64_t head = 0, tail = 1;
        while (head < tail) {
            int64_t u = queue[head++];
            int64_t lu = level[u];
            for (int64_t s = row[u]; s < row[u + 1]; ++s) {
                int64_t w = nb[s];
                if (level[w] < 0) {
                    level[w] = lu + 1;
                    if (parent) parent[w] = u;
                    if (lu + 1 > max_level) max_level = lu + 1;
                    queue[tail++] = w;
                }
            }
        }
    }
    free(queue);
    *max_level_out = max_level;
    return components;
}

/* bfs.py:97-106 cover_edges: horizontal edges (level[u]==level[v], u<v)
 * of the canonical edge arrays, lexicographic.  out is int64[k][2].
 * Returns k.                                                           */
int64_t orc_cover_select(const int64_t* level, const int32_t* eu,
                         const int32_t* ev, int64_t m, int64_t* out) {
    int64_t k = 0;
    for (int64_t e = 0; e < m; ++e) {
        if (level[eu[e]] == level[ev[e]]) {   /* bfs.py:84 */
            if (out) { out[2 * k] = eu[e]; out[2 * k + 1] = ev[e]; }
            k++;
        }
    }
    return k;
}

/* _kernels.py:669-695 cetc_count_k: for u ascending, v in N(u) with
 * v>u and level[v]==level[u], merge the full N(u), N(v); count apex x
 * when level[x]!=level[u] or x>v (:687).                               */
int64_t orc_cetc_count(const int64_t* row, const int32_t* nb,
                       const int64_t* level, int64_t n) {
    int64_t t = 0;
    for (int64_t u = 0; u < n; ++u) {
        int64_t su = row[u], se = row[u + 1], lu = level[u];
        for (int64_t s = su; s < se; ++s) {
            int64_t v = nb[s];
            if (v > u && level[v] == lu) {
                int64_t i = su, j = row[v], je = row[v + 1];
                while (i < se && j < je) {
                    int32_t x = nb[i], y = nb[j];
                    if (x == y) {
                        if (level[x] != lu || x > v) t++;
                        i++; j++;
                    } else if (x < y) {
                        i++;
                    } else {
                        j++;
                    }
                }
            }
        }
    }
    return t;
}

/* _kernels.py:729-755 cetc_sm_range_k over edge chunks
 * [k0,k1) of size ceil(m/(4*workers)) (parallel.py:53-59), run on
 * `threads` OpenMP threads (parallel.py:62-70 uses a thread pool);
 * c1 = apexes off the edge's level, c2 = apexes on it.  Partials are
 * summed in chunk order (parallel.py:135-136).                        */
void orc_cetc_sm_counts(const int64_t* row, const int32_t* nb,
                        const int64_t* level, const int32_t* eu,
                        const int32_t* ev, int64_t m, int threads,
                        int64_t chunk, int64_t* c1_out, int64_t* c2_out) {
    if (threads < 1) threads = 1;
    if (chunk <= 0) {
        int64_t w4 = (int64_t)threads * 4;
        chunk = (m + w4 - 1) / w4;
        if (chunk < 1) chunk = 1;
    }
    int64_t nchunks = (m + chunk - 1) / chunk;
    int64_t* p1 = (int64_t*)calloc(nchunks > 0 ? nchunks : 1, sizeof(int64_t));
    int64_t* p2 = (int64_t*)calloc(nchunks > 0 ? nchunks : 1, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t ci = 0; ci < nchunks; ++ci) {
        int64_t k0 = ci * chunk, k1 = k0 + chunk < m ? k0 + chunk : m;
        int64_t c1 = 0, c2 = 0;
        for (int64_t k = k0; k < k1; ++k) {
            int64_t u = eu[k], v = ev[k];
            int64_t lu = level[u];
            if (level[v] != lu) continue;
            int64_t i = row[u], ie = row[u + 1];
            int64_t j = row[v], je = row[v + 1];
            while (i < ie && j < je) {
                int32_t x = nb[i], y = nb[j];
                if (x == y) {
                    if (level[x] != lu) c1++; else c2++;
                    i++; j++;
                } else if (x < y) {
                    i++;
                } else {
                    j++;
                }
            }
        }
        p1[ci] = c1;
        p2[ci] = c2;
    }
    int64_t c1 = 0, c2 = 0;
    for (int64_t ci = 0; ci < nchunks; ++ci) { c1 += p1[ci]; c2 += p2[ci]; }
    free(p1);
    free(p2);
    *c1_out = c1;
    *c2_out = c2;
}

/* Convenience: number of OpenMP threads this library would use. */
int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

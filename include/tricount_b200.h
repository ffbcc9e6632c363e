/*
 * tricount_b200.h — C ABI of the B200-native cover-edge triangle counting
 * (CETC) path.  libtricount_b200.so (paper_2403_02997_b200/lib/) exports
 * exactly the functions declared here.
 *
 * Conventions
 *  - Every call returns TCB_OK (0) or a TCB_ERR_* code; tcb_last_error()
 *    gives the message for the context.
 *  - d_* arguments are device pointers (caller owned), h_* host pointers.
 *    Inputs are read-only.  Vertex ids are int32, CSR offsets int64 — the
 *    reference Graph's layout (graph.py:57-92, graph.py:95-96).
 *  - The device graph is the CSR (row_offsets int64[n+1], neighbors
 *    int32[2m], strictly increasing rows) plus src int32[2m], the row id of
 *    every entry (COO rows; the same footprint as the reference Graph's
 *    edge_u/edge_v pair, which are the src<neighbors entries in order).
 *  - All device work is ordered on the context's stream.  Functions that
 *    return a host-side count (m, ncover, components, counts) synchronise
 *    that stream before returning.
 *  - Scratch memory is owned by the context and reused across calls; one
 *    context per host thread (the reference kernels are nogil and safe for
 *    concurrent calls on one Graph — _kernels.py:1-8 — and so is this ABI
 *    with one context per caller).
 *
 * The reference interface each entry point replaces is cited as
 * file:line of the reference package (pkg/src/tricount/); the numba
 * kernels' signatures are listed in SURVEY.md §8(b).
 */
#ifndef TRICOUNT_B200_H
#define TRICOUNT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCB_API __attribute__((visibility("default")))

#define TCB_VERSION 6

enum {
    TCB_OK = 0,
    TCB_ERR_INVALID = 1,   /* bad argument / size mismatch  (ValueError)     */
    TCB_ERR_CUDA = 2,      /* CUDA runtime error                              */
    TCB_ERR_NOMEM = 3,     /* device workspace allocation failed              */
    TCB_ERR_ASSERT = 4,    /* internal invariant (e.g. c2 % 3 != 0)           */
    TCB_ERR_INTERNAL = 5
};

/* Stage indices for tcb_stage_times(). */
enum {
    TCB_STAGE_COMPONENTS = 0,  /* min-id component roots (CC)                 */
    TCB_STAGE_BFS = 1,         /* multi-source level-synchronous BFS           */
    TCB_STAGE_SELECT = 2,      /* horizontal (cover) edge selection            */
    TCB_STAGE_INTERSECT = 3,   /* per-cover-edge |N(u) ∩ N(v)| + level dedup   */
    TCB_STAGE_H2D = 4,         /* host-buffer entry: uploads + row expansion   */
    TCB_STAGE_D2H = 5,         /* host-buffer entry: downloads                 */
    TCB_STAGE_ISECT_CTA = 6,   /* CTA tiers of the intersection (hub + hash)    */
    TCB_STAGE_ISECT_HUB = 7,   /* the hub-bitmap kernel alone                   */
    TCB_NSTAGES = 8
};

typedef struct tcb_context tcb_context;

/* Result of the fused path (tc_cetc, sequential.py:164-168, and
 * _cetc_sm_counts, parallel.py:132-137). */
typedef struct tcb_result {
    int64_t triangles;   /* T = c1 + c2/3                                  */
    int64_t c1;          /* apexes off the cover edge's level              */
    int64_t c2;          /* apexes on the cover edge's level (3 per tri)   */
    int64_t ncover;      /* |S|, horizontal edge count                      */
    int64_t components;  /* BfsLabeling.components                          */
    int64_t max_level;   /* BfsLabeling.max_level                           */
} tcb_result;

/* ---- context ---------------------------------------------------------- */
TCB_API int tcb_version(void);
/* stream: a cudaStream_t (NULL = legacy default stream) */
TCB_API int tcb_context_create(int device, void* stream, tcb_context** out);
TCB_API int tcb_context_destroy(tcb_context* ctx);
TCB_API int tcb_context_set_stream(tcb_context* ctx, void* stream);
TCB_API const char* tcb_last_error(tcb_context* ctx);
/* Count of kernels this context launched so far. */
TCB_API int64_t tcb_launch_count(tcb_context* ctx);
/* Enable per-stage CUDA-event timing; tcb_stage_times fills ms[TCB_NSTAGES]
 * for the last fused call (tcb_cetc / tcb_cetc_shard / tcb_cetc_host). */
TCB_API int tcb_set_timing(tcb_context* ctx, int enabled);
TCB_API int tcb_stage_times(tcb_context* ctx, float* ms_out, int n);
/* Diagnostics (no reference counterpart): per-level BFS records of the last
 * call that ran the BFS, for profiling.  Writes up to cap records of three
 * int64 each — (mode: 0 top-down / 1 bottom-up, level-step end time in ns
 * from the BFS start, frontier size after the step) — and returns the
 * number written (levels past TCB_LEVEL_RECORDS are not recorded). */
#define TCB_LEVEL_RECORDS 48
TCB_API int tcb_level_records(tcb_context* ctx, int64_t* out, int cap);
/* Intersection work-split knobs (0 = built-in default): owners with degree
 * <= warp_tier_max_degree (max 1024) use the per-warp tier; larger owners
 * stage <= cta_stage_max off-level ids (4..6144) per CTA pass, and the same
 * number bounds the 32-bit words of one rank window of the same-level bitmap
 * (a shrunk value forces several windows).  Results do not depend on them;
 * tests shrink them to drive every code path. */
TCB_API int tcb_set_tuning(tcb_context* ctx, int warp_tier_max_degree, int cta_stage_max);
/* Test hook (no reference counterpart): TCB_TEST_FORCE_FALLBACK makes every
 * CTA-tier pass use the bucket-table fallback that otherwise runs only when
 * a cuckoo build fails, so the tests reach that path.  0 = normal. */
#define TCB_TEST_FORCE_FALLBACK 4
/* Test hook: graphs of <= 2^17 vertices and edges normally take a one-launch
 * small-graph kernel, and graphs of max degree <= 32 a merge count after the
 * general BFS; this flag (or any nonzero flag / tuning) forces the general
 * path on them. */
#define TCB_TEST_GENERAL_PATH 8
/* Test hook: fill the CTA tier's partner-record array with 0xFF before the
 * record pass, so a sharded call cannot pass on records an earlier call of
 * another shard left in the workspace (each rank must build every record its
 * own items read). */
#define TCB_TEST_POISON_RECORDS 16
TCB_API int tcb_set_test_flags(tcb_context* ctx, int flags);

/* ---- input synthesis (rmat.py:45-72) ---------------------------------- */
/* generate_rmat: edge_factor*2^scale pairs into d_pairs[2*total] (u,v
 * interleaved int64), drawing from the PCG64 stream whose 128-bit
 * (state, inc) numpy.random.default_rng(seed) starts with (bit-identical to
 * the reference's pairs).  d_perm (nullable, int64[2^scale]) relabels both
 * endpoints: new = perm[old]. */
TCB_API int tcb_rmat_generate(tcb_context* ctx, int scale, int64_t edge_factor,
                              double a, double b, double c,
                              uint64_t state_hi, uint64_t state_lo,
                              uint64_t inc_hi, uint64_t inc_lo,
                              const int64_t* d_perm, int64_t* d_pairs);

/* The reference's ER fixture recipe (tests/conftest.py:41-47 er_graph):
 * default_rng(seed).random((n, n)) < p over the strict upper triangle, the
 * (i, j) pairs in row-major order, bit-identical to numpy's.  (state, inc)
 * as for tcb_rmat_generate.  d_pairs: int64[2 * n(n-1)/2] capacity;
 * *k_out = pairs written.  n <= 65536.  Synchronous. */
TCB_API int tcb_er_generate(tcb_context* ctx, int64_t n, double p,
                            uint64_t state_hi, uint64_t state_lo,
                            uint64_t inc_hi, uint64_t inc_lo,
                            int64_t* d_pairs, int64_t* k_out);

/* The side x side lattice config: ids r*side + c, edges
 * (r,c)-(r,c+1), (r,c)-(r+1,c), (r,c)-(r+1,c+1), each family row-major.
 * d_pairs: int64[2 * (2 side (side-1) + (side-1)^2)]. */
TCB_API int tcb_lattice_generate(tcb_context* ctx, int64_t side, int64_t* d_pairs);

/* ---- graph build (graph.py:177-194 normalize,
 *      graph.py:104-125 _graph_from_canonical_pairs) ------------------ */
/* Drops self-loops, dedups, symmetrises, sorts adjacency lists.
 * d_pairs: int64[2k] interleaved (u,v), ids in [0,n).
 * d_row_offsets: int64[n+1]; d_neighbors and d_src (nullable): capacity 2k.
 * d_edge_u/d_edge_v (nullable): capacity k int32, the u<v pairs in
 * lexicographic order (Graph.edge_u/edge_v).  *m_out = undirected edges. */
TCB_API int tcb_csr_build(tcb_context* ctx, const int64_t* d_pairs, int64_t k,
                          int64_t n, int64_t* d_row_offsets, int32_t* d_neighbors,
                          int32_t* d_src, int32_t* d_edge_u, int32_t* d_edge_v,
                          int64_t* m_out);

/* Host -> device copy of `bytes` bytes that is fast from PAGEABLE memory
 * too (numpy arrays, the reference Graph's frozen CSR): pinned sources are
 * one DMA; pageable ones go through a ring of pinned staging buffers, the
 * host threads filling chunk i+1 while chunk i is in flight.  Returns after
 * the copy has landed.  Replaces the upload a ctypes binding would do before
 * calling the device entries (graph.py device_graph). */
TCB_API int tcb_copy_to_device(tcb_context* ctx, void* d_dst, const void* h_src,
                               int64_t bytes);

/* src (per-entry row id) of a CSR: d_src[row[v]..row[v+1]) = v. */
TCB_API int tcb_csr_rows(tcb_context* ctx, const int64_t* d_row_offsets, int64_t n,
                         int32_t* d_src);

/* Graph.edge_u/edge_v from a CSR (load_graph's derivation, graph.py:248-250):
 * the u<v entries of each sorted row, in CSR order. */
TCB_API int tcb_csr_edges(tcb_context* ctx, const int64_t* d_row_offsets,
                          const int32_t* d_neighbors, int64_t n, int64_t m,
                          int32_t* d_edge_u, int32_t* d_edge_v);

/* ---- BFS levels (_kernels.py:129-157 bfs_levels_k; bfs.py:76-94) ------ */
/* Levels of a BFS over all components rooted at each component's lowest
 * id (the reference's root rule, _kernels.py:137-142).  d_level int32[n].
 * The FIFO parents are a separate call (tcb_bfs_parent) since the counting
 * path does not need them. */
TCB_API int tcb_bfs_levels(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_src,
                           int64_t n, int64_t m, int32_t* d_level,
                           int64_t* components_out, int64_t* max_level_out);

/* ---- FIFO parents (_kernels.py:143-156; bfs_levels_k's `parent`) ------ */
/* The parent the reference's FIFO BFS assigns (the first dequeued
 * neighbour one level up), rebuilt level-synchronously from d_level and
 * max_level (tcb_bfs_levels outputs).  d_parent_out int32[n], -1 at the
 * component roots.  Synchronous. */
TCB_API int tcb_bfs_parent(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, int64_t n,
                           const int32_t* d_level, int64_t max_level,
                           int32_t* d_parent_out);

/* ---- edge classes (bfs.py:83-87 in bfs_label) -------------------------- */
/* Class of each canonical edge (edge_u/edge_v order: u < v, lexicographic)
 * as int8 EdgeClass: 0 TREE (either endpoint is the other's parent),
 * 2 HORIZONTAL (equal levels), else 1 STRUT.  d_class_out int8[m].
 * Synchronous. */
TCB_API int tcb_edge_classes(tcb_context* ctx, const int64_t* d_row_offsets,
                             const int32_t* d_neighbors, const int32_t* d_src,
                             int64_t n, int64_t m, const int32_t* d_level,
                             const int32_t* d_parent, int8_t* d_class_out);

/* ---- cover edges (bfs.py:97-106 cover_edges) -------------------------- */
/* Horizontal edges (level[u]==level[v], u<v) in the reference's
 * lexicographic order.  d_cover_u/d_cover_v capacity m.  *ncover_out=|S|. */
TCB_API int tcb_cover_select(tcb_context* ctx, const int32_t* d_level,
                             const int32_t* d_src, const int32_t* d_neighbors,
                             int64_t m, int32_t* d_cover_u, int32_t* d_cover_v,
                             int64_t* ncover_out);

/* ---- intersection over an explicit cover list (_kernels.py:729-755
 *      cetc_sm_range_k over edge chunks, parallel.py:53-70) ------------ */
/* Over cover edges [k0, k1) of (d_cover_u, d_cover_v), u < v:
 * counts_out[0] = T partial (c1 + same-level apexes w > v), [1] = c1,
 * [2] = c2.  Over the full set T = c1 + c2/3. */
TCB_API int tcb_cetc_count(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_level,
                           int64_t n, const int32_t* d_cover_u,
                           const int32_t* d_cover_v, int64_t k0, int64_t k1,
                           int64_t* counts_out);

/* ---- CETC-DM apex-range count (_kernels.py:759-783
 *      cetc_count_restricted_k, used by dmsim.py:144-200) ---------------- */
/* Over cover edges [0, k) of (d_cover_u, d_cover_v), u < v, counting only
 * apexes w with lo <= w < hi (the ids processor `i` owns in CETC-DM):
 * counts_out[0] = T partial (apex on another level, or w > v), [1] = c1,
 * [2] = c2 of those apexes.  Summed over a partition of [0, n) the T parts
 * give the triangle count. */
TCB_API int tcb_cetc_count_restricted(tcb_context* ctx, const int64_t* d_row_offsets,
                                      const int32_t* d_neighbors, const int32_t* d_level,
                                      int64_t n, const int32_t* d_cover_u,
                                      const int32_t* d_cover_v, int64_t k, int64_t lo,
                                      int64_t hi, int64_t* counts_out);

/* ---- fused path (sequential.py:164-168 tc_cetc) ----------------------- */
/* Device-resident graph in, exact count out.  d_level_out (nullable,
 * int32[n]) receives the levels; d_cover_u/v (nullable, capacity m) the
 * cover set in the reference's order. */
TCB_API int tcb_cetc(tcb_context* ctx, const int64_t* d_row_offsets,
                     const int32_t* d_neighbors, const int32_t* d_src,
                     int64_t n, int64_t m, int32_t* d_level_out,
                     int32_t* d_cover_u, int32_t* d_cover_v, tcb_result* out);

/* Multi-GPU shard of the fused path: full labeling and
 * selection on this device's replica; intersection for the work items of
 * this shard — partner block i of owner x belongs to shard (x + i) %
 * nshards (dist.py shard_of).  c1/c2 are this shard's partials (sum over
 * shards, e.g. one all-reduce; then T = c1 + c2/3); triangles is -1 when
 * nshards > 1; ncover/components/max_level are global. */
TCB_API int tcb_cetc_shard(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_src,
                           int64_t n, int64_t m, int shard, int nshards,
                           tcb_result* out);

/* ---- CETC variants (sequential.py:170-183) ----------------------------- */
/* Forward triangle count on device (tc_forward_k, _kernels.py:480; the
 * forward branch of tc_cetc_fe): every edge is intersected once by its
 * higher-ranked endpoint in (degree desc, id asc) order, which stages only
 * its neighbours ranked above itself; each triangle is hit exactly once.  T
 * is orientation-independent, so it equals the reference's id-ordered
 * forward count. */
TCB_API int tcb_forward_count(tcb_context* ctx, const int64_t* d_row_offsets,
                              const int32_t* d_neighbors, const int32_t* d_src,
                              int64_t n, int64_t m, int64_t* triangles_out);

/* tc_cetc_fe (sequential.py:176-183): BFS levels, covering ratio
 * |S| / m; below `threshold` (COVER_RATIO_THRESHOLD = 0.7) the cover-edge
 * count, else the forward count.  out->ncover/components/max_level are
 * filled either way; c1/c2 are -1 on the forward branch.
 * *used_forward_out (nullable) = 1 when the forward branch ran. */
TCB_API int tcb_cetc_fe(tcb_context* ctx, const int64_t* d_row_offsets,
                        const int32_t* d_neighbors, const int32_t* d_src,
                        int64_t n, int64_t m, double threshold, tcb_result* out,
                        int32_t* used_forward_out);

/* degree_order (graph.py:203-213, for CETC-Seq-D / -SD): the graph
 * relabelled by non-increasing degree, ties by ascending old id, as a new
 * CSR (d_row_out int64[n+1], d_neighbors_out / d_src_out int32[2m]).
 * Synchronous. */
TCB_API int tcb_degree_order(tcb_context* ctx, const int64_t* d_row_offsets,
                             const int32_t* d_neighbors, const int32_t* d_src,
                             int64_t n, int64_t m, int64_t* d_row_out,
                             int32_t* d_neighbors_out, int32_t* d_src_out);

/* ---- split hybrid (CETC-Seq-S/-SD/-SR, sequential.py:186-238) --------- */
/* _split_by_level (sequential.py:186-193): G0 = the horizontal edges
 * (level[u] == level[v]) as a CSR: d_row0 int64[n+1], d_nb0 / d_src0
 * (nullable) capacity 2m int32; *m0_out = G0's undirected edges. */
TCB_API int tcb_split_by_level(tcb_context* ctx, const int64_t* d_row_offsets,
                               const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                               int64_t m, const int32_t* d_level, int64_t* d_row0,
                               int32_t* d_nb0, int32_t* d_src0, int64_t* m0_out);

/* split_cross_count_k (_kernels.py:786-805): triangles with one horizontal
 * edge and both others level-spanning, i.e. sum over G0's edges u < v of
 * |N1(u) ∩ N1(v)| with G1 = the level-spanning edges of the levels given. */
TCB_API int tcb_split_cross_count(tcb_context* ctx, const int64_t* d_row_offsets,
                                  const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                                  int64_t m, const int32_t* d_level, int64_t* cross_out);

/* Host-buffer entry, the call a binding of cetc_count_k's argument list
 * (row, nb, n; _kernels.py:669) makes: uploads the CSR, derives src, runs
 * the fused path, downloads the result (and levels as int64 when
 * h_level_out != NULL, BfsLabeling.level's dtype).
 * h_row_offsets int64[n+1], h_neighbors int32[row[n]]. */
TCB_API int tcb_cetc_host(tcb_context* ctx, const int64_t* h_row_offsets,
                          const int32_t* h_neighbors, int64_t n,
                          int64_t* h_level_out, tcb_result* out);

/* The host-buffer entry for one rank of a multi-GPU run (tcb_cetc_shard's
 * sharding): c1/c2 partials to be summed across ranks; triangles is -1
 * when nshards > 1. */
TCB_API int tcb_cetc_host_shard(tcb_context* ctx, const int64_t* h_row_offsets,
                                const int32_t* h_neighbors, int64_t n,
                                int shard, int nshards, tcb_result* out);

#ifdef __cplusplus
}
#endif
#endif /* TRICOUNT_B200_H */

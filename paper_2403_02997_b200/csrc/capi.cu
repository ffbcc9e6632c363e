// capi.cu — the C ABI (include/tricount_b200.h) over the sm_100a kernels.
//
// Every entry point catches tcb::Error and returns its code; the message is
// kept on the context (tcb_last_error).  The fused driver mirrors tc_cetc
// (sequential.py:164-168): bfs_label -> cover edges -> intersection, all
// stream-ordered with a single host synchronisation at the end.
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include <cstdio>

struct tcb_context : tcb::Context {};

namespace tcb {
void csr_build(Context*, const int64_t*, int64_t, int64_t, int64_t*, int32_t*, int32_t*,
               int32_t*, int32_t*, int64_t*);
void csr_rows(Context*, const int64_t*, int64_t, int32_t*);
void csr_edges(Context*, const int64_t*, const int32_t*, int64_t, int64_t, int32_t*, int32_t*);
bool small_cetc(Context*, const int64_t*, const int32_t*, int64_t, int64_t, int32_t*);
void split_by_level(Context*, const int64_t*, const int32_t*, const int32_t*, int64_t, int64_t,
                    const int32_t*, int64_t*, int32_t*, int32_t*, int64_t*);
void bfs_levels(Context*, const int64_t*, const int32_t*, const int32_t*, int64_t, int64_t,
                int32_t*, bool, int two_max = 0);
void cover_select(Context*, const int32_t*, const int32_t*, const int32_t*, int64_t, int32_t*,
                  int32_t*, int64_t*);
void bfs_parent(Context*, const int64_t*, const int32_t*, int64_t, const int32_t*, int64_t,
                int32_t*);
void edge_classes(Context*, const int64_t*, const int32_t*, const int32_t*, int64_t, int64_t,
                  const int32_t*, const int32_t*, int8_t*);
void cetc_intersect(Context*, const int64_t*, const int32_t*, const int32_t*, const int32_t*,
                    const int32_t*, const int64_t*, int64_t, int64_t, int, int, int64_t, int, int);
void cetc_intersect_owner(Context*, const int64_t*, const int32_t*, const int32_t*,
                          const int32_t*, int64_t, int64_t, int, int, int);
void degree_order(Context*, const int64_t*, const int32_t*, const int32_t*, int64_t, int64_t,
                  int64_t*, int32_t*, int32_t*);
void count_horizontal(Context*, const int32_t*, const int32_t*, const int32_t*, int64_t,
                      unsigned long long*);
void rmat_generate(Context*, int, int64_t, double, double, double, uint64_t, uint64_t, uint64_t,
                   uint64_t, const int64_t*, int64_t*);
void er_generate(Context*, int64_t, double, uint64_t, uint64_t, uint64_t, uint64_t, int64_t*,
                 int64_t*);
void lattice_generate(Context*, int64_t, int64_t*);

namespace {

template <typename F>
int guarded(tcb_context* ctx, F&& f) {
    if (!ctx) return TCB_ERR_INVALID;
    try {
        TCB_CUDA(cudaSetDevice(ctx->device));
        f();
        ctx->last_error.clear();
        return TCB_OK;
    } catch (const Error& e) {
        ctx->last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        ctx->last_error = e.what();
        return TCB_ERR_INTERNAL;
    }
}

void sync(Context* ctx) { TCB_CUDA(cudaStreamSynchronize(ctx->stream)); }

void fetch_counters(Context* ctx) {
    TCB_CUDA(cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, sizeof(DevCounters),
                             cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
}

// events 0..4 bracket components, bfs, select, intersect
void collect_stage_times(Context* ctx) {
    if (!ctx->timing) return;
    sync(ctx);
    for (int s = 0; s < 4; ++s) {
        float ms = 0.f;
        TCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[s], ctx->ev[s + 1]));
        ctx->stage_ms[TCB_STAGE_COMPONENTS + s] = ms;
    }
    ctx->stage_ms[TCB_STAGE_ISECT_CTA] = 0.f;
    ctx->stage_ms[TCB_STAGE_ISECT_HUB] = 0.f;
    if (ctx->isect_events) {
        float ms = 0.f;
        TCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[6]));
        ctx->stage_ms[TCB_STAGE_ISECT_CTA] = ms;
        TCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[7]));
        ctx->stage_ms[TCB_STAGE_ISECT_HUB] = ms;
    }
}

// fused path on device-resident arrays; leaves results in ctx->d_counters
void cetc_device(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                 int64_t n, int64_t m, int32_t* level, int shard = 0, int nshards = 1) {
    TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
    ctx->isect_events = false;
    if (n == 0) return;
    // graphs of at most 2^17 vertices and edges: one cooperative launch
    if (nshards == 1 && small_cetc(ctx, row, nb, n, m, level)) {  // events 0-3
        ctx->record(4);
        return;
    }
    bfs_levels(ctx, row, nb, src, n, m, level, false);  // events 0, 1, 2
    if (m == 0) {
        ctx->record(3);
        ctx->record(4);
        return;
    }
    cetc_intersect_owner(ctx, row, nb, src, level, n, m, shard, nshards, 0);  // events 3, 5, 6
    ctx->isect_events = true;
    ctx->record(4);
}

void fill_result(Context* ctx, tcb_result* out, bool partial = false) {
    const DevCounters& h = *ctx->h_counters;
    tcb_result r;
    r.c1 = int64_t(h.c1);
    r.c2 = int64_t(h.c2);
    // T == c1 + c2/3 over the full cover set (intersect.cu Tally); a shard's
    // partials carry c1/c2 only and T is formed after they are summed.
    r.triangles = partial ? -1 : int64_t(h.c1 + h.c2 / 3);
    r.ncover = int64_t(h.ncover);
    r.components = int64_t(h.components);
    r.max_level = h.max_level;
#if defined(TCB_NOPROBE) || defined(TCB_NOLOAD) || defined(TCB_NOSTREAM) || defined(TCB_NOUPSTREAM) || defined(TCB_NOOFFSTREAM)  // measurement-only
    partial = true;
#endif
    if (!partial && r.c2 % 3 != 0)  // parallel.py:127-128
        throw Error(TCB_ERR_ASSERT, "same-level apex tally must be divisible by 3");
    if (out) *out = r;
}

__global__ void k_level_to_i64(const int32_t* __restrict__ in, int64_t* __restrict__ out,
                               int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = in[i];
}

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" {

TCB_API int tcb_version(void) { return TCB_VERSION; }

TCB_API int tcb_context_create(int device, void* stream, tcb_context** out) {
    if (!out) return TCB_ERR_INVALID;
    *out = nullptr;
    tcb_context* ctx = new tcb_context();
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    int rc = guarded(ctx, [&] {
        TCB_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        TCB_CUDA(cudaMalloc(&ctx->d_counters, sizeof(DevCounters)));
        TCB_CUDA(cudaMallocHost(&ctx->h_counters, sizeof(DevCounters)));
        std::memset(ctx->h_counters, 0, sizeof(DevCounters));
        for (auto& e : ctx->ev) TCB_CUDA(cudaEventCreate(&e));
    });
    if (rc != TCB_OK) {
        delete ctx;
        return rc;
    }
    *out = ctx;
    return TCB_OK;
}

TCB_API int tcb_context_destroy(tcb_context* ctx) {
    if (!ctx) return TCB_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (int s = 0; s < WS_NSLOTS; ++s)
        if (ctx->slot_ptr[s]) cudaFree(ctx->slot_ptr[s]);
    if (ctx->d_counters) cudaFree(ctx->d_counters);
    if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->copy_ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < Context::NSTAGE; ++i) {
        if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
        if (ctx->stage_buf[i]) cudaFreeHost(ctx->stage_buf[i]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
    return TCB_OK;
}

TCB_API int tcb_context_set_stream(tcb_context* ctx, void* stream) {
    return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

TCB_API const char* tcb_last_error(tcb_context* ctx) {
    return ctx ? ctx->last_error.c_str() : "null context";
}

TCB_API int64_t tcb_launch_count(tcb_context* ctx) { return ctx ? int64_t(ctx->launches) : -1; }

TCB_API int tcb_set_timing(tcb_context* ctx, int enabled) {
    return guarded(ctx, [&] { ctx->timing = enabled != 0; });
}

TCB_API int tcb_set_tuning(tcb_context* ctx, int warp_tier_max_degree, int cta_stage_max) {
    return guarded(ctx, [&] {
        require(warp_tier_max_degree >= 0 && cta_stage_max >= 0, "negative tuning value");
        ctx->tune_wt = warp_tier_max_degree;
        ctx->tune_hc = cta_stage_max;
    });
}

TCB_API int tcb_set_test_flags(tcb_context* ctx, int flags) {
    return guarded(ctx, [&] {
        require(flags >= 0, "negative flags");
        ctx->test_flags = flags;
    });
}

TCB_API int tcb_stage_times(tcb_context* ctx, float* ms_out, int n) {
    return guarded(ctx, [&] {
        require(ms_out != nullptr, "ms_out is null");
        for (int i = 0; i < n && i < TCB_NSTAGES; ++i) ms_out[i] = ctx->stage_ms[i];
    });
}

TCB_API int tcb_level_records(tcb_context* ctx, int64_t* out, int cap) {
    int cnt = 0;
    const int rc = guarded(ctx, [&] {
        require(out != nullptr || cap == 0, "out is null");
        const DevCounters& h = *ctx->h_counters;
        const int nl = int(h.nlev < TCB_LEVEL_RECORDS ? h.nlev : TCB_LEVEL_RECORDS);
        for (int i = 0; i < nl && i < cap; ++i) {
            const unsigned long long e = h.lev_rec[2 * i];
            out[3 * i] = int64_t(e >> 62);
            out[3 * i + 1] = int64_t(e & ((1ull << 62) - 1)) - int64_t(h.bfs_t0);
            out[3 * i + 2] = int64_t(h.lev_rec[2 * i + 1]);
            ++cnt;
        }
    });
    return rc == TCB_OK ? cnt : -rc;
}

TCB_API int tcb_rmat_generate(tcb_context* ctx, int scale, int64_t edge_factor, double a,
                              double b, double c, uint64_t state_hi, uint64_t state_lo,
                              uint64_t inc_hi, uint64_t inc_lo, const int64_t* d_perm,
                              int64_t* d_pairs) {
    return guarded(ctx, [&] {
        require(d_pairs != nullptr, "d_pairs is null");
        rmat_generate(ctx, scale, edge_factor, a, b, c, state_hi, state_lo, inc_hi, inc_lo,
                      d_perm, d_pairs);
    });
}

TCB_API int tcb_er_generate(tcb_context* ctx, int64_t n, double p, uint64_t state_hi,
                            uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                            int64_t* d_pairs, int64_t* k_out) {
    return guarded(ctx, [&] {
        require(k_out != nullptr, "k_out is null");
        require(n < 2 || d_pairs, "null output");
        er_generate(ctx, n, p, state_hi, state_lo, inc_hi, inc_lo, d_pairs, k_out);
    });
}

TCB_API int tcb_lattice_generate(tcb_context* ctx, int64_t side, int64_t* d_pairs) {
    return guarded(ctx, [&] {
        require(d_pairs != nullptr || side <= 1, "null output");
        lattice_generate(ctx, side, d_pairs);
    });
}

TCB_API int tcb_csr_build(tcb_context* ctx, const int64_t* d_pairs, int64_t k, int64_t n,
                          int64_t* d_row_offsets, int32_t* d_neighbors, int32_t* d_src,
                          int32_t* d_edge_u, int32_t* d_edge_v, int64_t* m_out) {
    return guarded(ctx, [&] {
        require(d_row_offsets && m_out, "null output");
        require(k == 0 || (d_pairs && d_neighbors), "null input");
        require(k >= 0, "negative size");
        require_sizes(n);
        csr_build(ctx, d_pairs, k, n, d_row_offsets, d_neighbors, d_src, d_edge_u, d_edge_v,
                  m_out);
        require_sizes(n, *m_out);  // the deduplicated graph must fit the layout
    });
}

TCB_API int tcb_csr_rows(tcb_context* ctx, const int64_t* d_row_offsets, int64_t n,
                         int32_t* d_src) {
    return guarded(ctx, [&] {
        require_sizes(n);
        csr_rows(ctx, d_row_offsets, n, d_src);
    });
}

TCB_API int tcb_csr_edges(tcb_context* ctx, const int64_t* d_row_offsets,
                          const int32_t* d_neighbors, int64_t n, int64_t m, int32_t* d_edge_u,
                          int32_t* d_edge_v) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        csr_edges(ctx, d_row_offsets, d_neighbors, n, m, d_edge_u, d_edge_v);
    });
}

TCB_API int tcb_bfs_levels(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_src, int64_t n, int64_t m,
                           int32_t* d_level, int64_t* components_out, int64_t* max_level_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(n == 0 || (d_row_offsets && d_level), "null array");
        bfs_levels(ctx, d_row_offsets, d_neighbors, d_src, n, m, d_level, true);
        fetch_counters(ctx);
        if (components_out) *components_out = int64_t(ctx->h_counters->components);
        if (max_level_out) *max_level_out = ctx->h_counters->max_level;
    });
}

TCB_API int tcb_bfs_parent(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, int64_t n, const int32_t* d_level,
                           int64_t max_level, int32_t* d_parent_out) {
    return guarded(ctx, [&] {
        require_sizes(n);
        require(n == 0 || (d_row_offsets && d_level && d_parent_out), "null array");
        bfs_parent(ctx, d_row_offsets, d_neighbors, n, d_level, max_level, d_parent_out);
        sync(ctx);
    });
}

TCB_API int tcb_edge_classes(tcb_context* ctx, const int64_t* d_row_offsets,
                             const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                             int64_t m, const int32_t* d_level, const int32_t* d_parent,
                             int8_t* d_class_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(m == 0 || (d_neighbors && d_src && d_level && d_parent && d_class_out),
                "null array");
        edge_classes(ctx, d_row_offsets, d_neighbors, d_src, n, m, d_level, d_parent,
                     d_class_out);
        sync(ctx);
    });
}

TCB_API int tcb_cover_select(tcb_context* ctx, const int32_t* d_level, const int32_t* d_src,
                             const int32_t* d_neighbors, int64_t m, int32_t* d_cover_u,
                             int32_t* d_cover_v, int64_t* ncover_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(0, m);
        int64_t* d_n = reinterpret_cast<int64_t*>(&ctx->d_counters->scratch[2]);
        cover_select(ctx, d_level, d_src, d_neighbors, 2 * m, d_cover_u, d_cover_v, d_n);
        int64_t k = 0;
        TCB_CUDA(cudaMemcpyAsync(&k, d_n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        if (ncover_out) *ncover_out = k;
    });
}

TCB_API int tcb_cetc_count(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_level, int64_t n,
                           const int32_t* d_cover_u, const int32_t* d_cover_v, int64_t k0,
                           int64_t k1, int64_t* counts_out) {
    return guarded(ctx, [&] {
        require(0 <= k0 && k0 <= k1, "bad cover-edge range");
        require(counts_out != nullptr, "counts_out is null");
        (void)n;
        TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
        cetc_intersect(ctx, d_row_offsets, d_neighbors, d_level, d_cover_u, d_cover_v, nullptr,
                       k0, k1, 0, 1, k1, 0, 0x7fffffff);
        fetch_counters(ctx);
        counts_out[0] = int64_t(ctx->h_counters->t);
        counts_out[1] = int64_t(ctx->h_counters->c1);
        counts_out[2] = int64_t(ctx->h_counters->c2);
    });
}

TCB_API int tcb_cetc_count_restricted(tcb_context* ctx, const int64_t* d_row_offsets,
                                      const int32_t* d_neighbors, const int32_t* d_level,
                                      int64_t n, const int32_t* d_cover_u,
                                      const int32_t* d_cover_v, int64_t k, int64_t lo, int64_t hi,
                                      int64_t* counts_out) {
    return guarded(ctx, [&] {
        require(k >= 0 && 0 <= lo && lo <= hi && hi <= n, "bad cover count or apex range");
        require(counts_out != nullptr, "counts_out is null");
        TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
        if (k > 0 && hi > lo)
            cetc_intersect(ctx, d_row_offsets, d_neighbors, d_level, d_cover_u, d_cover_v,
                           nullptr, 0, k, 0, 1, k, int(lo), int(hi));
        fetch_counters(ctx);
        counts_out[0] = int64_t(ctx->h_counters->t);
        counts_out[1] = int64_t(ctx->h_counters->c1);
        counts_out[2] = int64_t(ctx->h_counters->c2);
    });
}

TCB_API int tcb_cetc(tcb_context* ctx, const int64_t* d_row_offsets, const int32_t* d_neighbors,
                     const int32_t* d_src, int64_t n, int64_t m, int32_t* d_level_out,
                     int32_t* d_cover_u, int32_t* d_cover_v, tcb_result* out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        int32_t* level = d_level_out ? d_level_out : ctx->wsT<int32_t>(WS_LEVEL, n);
        cetc_device(ctx, d_row_offsets, d_neighbors, d_src, n, m, level);
        if (n > 0) collect_stage_times(ctx);
        if (d_cover_u && d_cover_v && n > 0) {  // the reference-order cover set, on request
            int64_t* d_k = reinterpret_cast<int64_t*>(&ctx->d_counters->scratch[2]);
            cover_select(ctx, level, d_src, d_neighbors, 2 * m, d_cover_u, d_cover_v, d_k);
        }
        fetch_counters(ctx);
        fill_result(ctx, out);
    });
}

// Forward count on device (all edges intersected, owners stage their
// higher-ranked neighbours; intersect.cu `staged`): T into *triangles_out.
void forward_device(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                    int64_t n, int64_t m, int64_t* triangles_out) {
    TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
    if (n > 0 && m > 0) {
        int32_t* zero = ctx->wsT<int32_t>(WS_LEVEL, n);  // one "level": every edge selected
        TCB_CUDA(cudaMemsetAsync(zero, 0, sizeof(int32_t) * n, ctx->stream));
        cetc_intersect_owner(ctx, row, nb, src, zero, n, m, 0, 1, 1);
    }
    fetch_counters(ctx);
    // forward mode classes every entry OFF: each hit is a triangle, in c1
    if (ctx->h_counters->c2 != 0)
        throw Error(TCB_ERR_ASSERT, "forward count: same-level tally must be zero");
    *triangles_out = int64_t(ctx->h_counters->c1);
}

TCB_API int tcb_forward_count(tcb_context* ctx, const int64_t* d_row_offsets,
                              const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                              int64_t m, int64_t* triangles_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(triangles_out != nullptr, "triangles_out is null");
        forward_device(ctx, d_row_offsets, d_neighbors, d_src, n, m, triangles_out);
    });
}

TCB_API int tcb_split_by_level(tcb_context* ctx, const int64_t* d_row_offsets,
                               const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                               int64_t m, const int32_t* d_level, int64_t* d_row0,
                               int32_t* d_nb0, int32_t* d_src0, int64_t* m0_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(m0_out != nullptr && d_row0 != nullptr, "null output");
        require(m == 0 || (d_level != nullptr && d_nb0 != nullptr), "null input/output");
        split_by_level(ctx, d_row_offsets, d_neighbors, d_src, n, m, d_level, d_row0, d_nb0,
                       d_src0, m0_out);
    });
}

TCB_API int tcb_split_cross_count(tcb_context* ctx, const int64_t* d_row_offsets,
                                  const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                                  int64_t m, const int32_t* d_level, int64_t* cross_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(cross_out != nullptr, "cross_out is null");
        TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
        if (n > 0 && m > 0) {
            require(d_level != nullptr, "null levels");
            cetc_intersect_owner(ctx, d_row_offsets, d_neighbors, d_src, d_level, n, m, 0, 1, 2);
        }
        fetch_counters(ctx);
        if (ctx->h_counters->c2 != 0)
            throw Error(TCB_ERR_ASSERT, "cross count: same-level tally must be zero");
        *cross_out = int64_t(ctx->h_counters->c1);
    });
}

TCB_API int tcb_cetc_fe(tcb_context* ctx, const int64_t* d_row_offsets,
                        const int32_t* d_neighbors, const int32_t* d_src, int64_t n, int64_t m,
                        double threshold, tcb_result* out, int32_t* used_forward_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        int32_t* level = ctx->wsT<int32_t>(WS_LEVEL, n);
        TCB_CUDA(cudaMemsetAsync(ctx->d_counters, 0, sizeof(DevCounters), ctx->stream));
        bfs_levels(ctx, d_row_offsets, d_neighbors, d_src, n, m, level, false);
        unsigned long long* d_h = &ctx->d_counters->scratch[12];
        count_horizontal(ctx, d_src, d_neighbors, level, n > 0 ? m : 0, d_h);
        fetch_counters(ctx);
        const DevCounters h = *ctx->h_counters;
        const double ratio = m ? double(h.scratch[12]) / double(m) : 0.0;  // sequential.py:179
        tcb_result r{};
        r.ncover = int64_t(h.scratch[12]);
        r.components = int64_t(h.components);
        r.max_level = h.max_level;
        const bool fwd = !(ratio < threshold);
        if (!fwd) {
            cetc_intersect_owner(ctx, d_row_offsets, d_neighbors, d_src, level, n, m, 0, 1, 0);
            fetch_counters(ctx);
            const DevCounters& c = *ctx->h_counters;
            if (c.c2 % 3 != 0)  // parallel.py:127-128
                throw Error(TCB_ERR_ASSERT, "same-level apex tally must be divisible by 3");
            r.c1 = int64_t(c.c1);
            r.c2 = int64_t(c.c2);
            r.triangles = r.c1 + r.c2 / 3;
        } else {
            int64_t t = 0;
            forward_device(ctx, d_row_offsets, d_neighbors, d_src, n, m, &t);
            r.triangles = t;
            r.c1 = r.c2 = -1;  // the forward branch has no cover-edge tallies
        }
        if (out) *out = r;
        if (used_forward_out) *used_forward_out = fwd ? 1 : 0;
    });
}

TCB_API int tcb_degree_order(tcb_context* ctx, const int64_t* d_row_offsets,
                             const int32_t* d_neighbors, const int32_t* d_src, int64_t n,
                             int64_t m, int64_t* d_row_out, int32_t* d_neighbors_out,
                             int32_t* d_src_out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(d_row_out && (m == 0 || (d_neighbors_out && d_src_out)), "null output");
        degree_order(ctx, d_row_offsets, d_neighbors, d_src, n, m, d_row_out, d_neighbors_out,
                     d_src_out);
        sync(ctx);
    });
}

TCB_API int tcb_cetc_shard(tcb_context* ctx, const int64_t* d_row_offsets,
                           const int32_t* d_neighbors, const int32_t* d_src, int64_t n, int64_t m,
                           int shard, int nshards, tcb_result* out) {
    return guarded(ctx, [&] {
        require(m >= 0, "negative size");
        require_sizes(n, m);
        require(nshards >= 1 && shard >= 0 && shard < nshards, "bad shard index");
        int32_t* level = ctx->wsT<int32_t>(WS_LEVEL, n);
        cetc_device(ctx, d_row_offsets, d_neighbors, d_src, n, m, level, shard, nshards);
        fetch_counters(ctx);
        fill_result(ctx, out, /*partial=*/nshards > 1);
        if (n > 0) collect_stage_times(ctx);
    });
}

static void ensure_copy_stream(Context* ctx) {
    if (ctx->copy_stream) return;
    TCB_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->copy_ev) TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Host -> device on ctx->copy_stream (ordered after the work already queued
// on ctx->stream).  Pinned source: one DMA.  Pageable source: chunks go
// through a ring of NSTAGE pinned buffers; all host threads (OpenMP) copy
// chunk i+1 into its buffer while chunk i's DMA runs, so the transfer runs
// at min(host memcpy, PCIe) instead of the driver's serial staging.  The
// caller orders later work after ctx->copy_ev[1].
static void stage_h2d(Context* ctx, void* d_dst, const void* h_src, int64_t bytes) {
    ensure_copy_stream(ctx);
    TCB_CUDA(cudaEventRecord(ctx->copy_ev[0], ctx->stream));
    TCB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[0], 0));
    constexpr int64_t CH = int64_t(32) << 20;  // 32 MB chunks
    if (bytes <= CH || is_pinned(h_src)) {
        TCB_CUDA(cudaMemcpyAsync(d_dst, h_src, size_t(bytes), cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
        TCB_CUDA(cudaEventRecord(ctx->copy_ev[1], ctx->copy_stream));
        return;
    }
    for (int i = 0; i < Context::NSTAGE; ++i) {
        if (!ctx->stage_buf[i]) {
            TCB_CUDA(cudaHostAlloc(&ctx->stage_buf[i], size_t(CH), cudaHostAllocDefault));
            TCB_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
            TCB_CUDA(cudaEventRecord(ctx->stage_ev[i], ctx->copy_stream));
        }
    }
    const char* src = static_cast<const char*>(h_src);
    char* dst = static_cast<char*>(d_dst);
    const int64_t nch = (bytes + CH - 1) / CH;
    for (int64_t c = 0; c < nch; ++c) {
        const int b = int(c % Context::NSTAGE);
        const int64_t off = c * CH, len = std::min(CH, bytes - off);
        TCB_CUDA(cudaEventSynchronize(ctx->stage_ev[b]));  // buffer b's last DMA is done
        char* stage = static_cast<char*>(ctx->stage_buf[b]);
        constexpr int64_t PIECE = int64_t(1) << 20;
        const int64_t npieces = (len + PIECE - 1) / PIECE;
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < npieces; ++q) {
            const int64_t o = q * PIECE;
            std::memcpy(stage + o, src + off + o, size_t(std::min(PIECE, len - o)));
        }
        TCB_CUDA(cudaMemcpyAsync(dst + off, stage, size_t(len), cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
        TCB_CUDA(cudaEventRecord(ctx->stage_ev[b], ctx->copy_stream));
    }
    TCB_CUDA(cudaEventRecord(ctx->copy_ev[1], ctx->copy_stream));
}

TCB_API int tcb_copy_to_device(tcb_context* ctx, void* d_dst, const void* h_src, int64_t bytes) {
    return guarded(ctx, [&] {
        require(bytes >= 0, "negative size");
        if (bytes == 0) return;
        require(d_dst != nullptr && h_src != nullptr, "null pointer");
        stage_h2d(ctx, d_dst, h_src, bytes);
        TCB_CUDA(cudaEventSynchronize(ctx->copy_ev[1]));
    });
}

// host-buffer entries: upload the CSR, derive src, run the fused path (or a
// shard of it), download the counters (and levels on request).  The
// neighbour array (the bulk of the bytes) is copied on a copy stream while
// the entry->row map is built from the row offsets on the compute stream.
static int host_entry(tcb_context* ctx, const int64_t* h_row_offsets, const int32_t* h_neighbors,
                      int64_t n, int64_t* h_level_out, int shard, int nshards, tcb_result* out) {
    return guarded(ctx, [&] {
        require_sizes(n);
        require(nshards >= 1 && shard >= 0 && shard < nshards, "bad shard index");
        require(h_row_offsets != nullptr, "null row offsets");
        const int64_t nnz = h_row_offsets[n];
        require(h_row_offsets[0] == 0 && nnz >= 0, "row offsets must start at 0 and end >= 0");
        require(nnz % 2 == 0, "CSR is not symmetric (odd entry count)");
        const int64_t m = nnz / 2;
        require_sizes(n, m);
        require(nnz == 0 || h_neighbors != nullptr, "null neighbour array");
        if (ctx->timing) TCB_CUDA(cudaEventRecord(ctx->ev[8], ctx->stream));
        int64_t* row = ctx->wsT<int64_t>(WS_ROW, n + 1);
        int32_t* nb = ctx->wsT<int32_t>(WS_NB, nnz);
        int32_t* src = ctx->wsT<int32_t>(WS_EDGE_U, nnz);
        // the neighbour array on the copy stream (after earlier work on the
        // compute stream; pageable sources through the pinned staging ring)
        if (nnz) stage_h2d(ctx, nb, h_neighbors, int64_t(sizeof(int32_t)) * nnz);
        TCB_CUDA(cudaMemcpyAsync(row, h_row_offsets, sizeof(int64_t) * (n + 1),
                                 cudaMemcpyHostToDevice, ctx->stream));
        csr_rows(ctx, row, n, src);
        if (nnz) TCB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->copy_ev[1], 0));
        if (ctx->timing) TCB_CUDA(cudaEventRecord(ctx->ev[9], ctx->stream));
        int32_t* level = ctx->wsT<int32_t>(WS_LEVEL, n);
        cetc_device(ctx, row, nb, src, n, m, level, shard, nshards);
        if (ctx->timing) TCB_CUDA(cudaEventRecord(ctx->ev[10], ctx->stream));
        if (h_level_out && n > 0) {
            int64_t* l64 = ctx->wsT<int64_t>(WS_EDGE_V, n);
            TCB_LAUNCH(ctx, k_level_to_i64, grid_for(ctx, n, 256), 256, 0, level, l64, n);
            TCB_CUDA(cudaMemcpyAsync(h_level_out, l64, sizeof(int64_t) * n,
                                     cudaMemcpyDeviceToHost, ctx->stream));
        }
        TCB_CUDA(cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, sizeof(DevCounters),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        if (ctx->timing) TCB_CUDA(cudaEventRecord(ctx->ev[11], ctx->stream));
        sync(ctx);
        fill_result(ctx, out, /*partial=*/nshards > 1);
        if (n > 0) collect_stage_times(ctx);
        if (ctx->timing) {
            float ms = 0.f;
            TCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[8], ctx->ev[9]));
            ctx->stage_ms[TCB_STAGE_H2D] = ms;
            TCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[10], ctx->ev[11]));
            ctx->stage_ms[TCB_STAGE_D2H] = ms;
        }
    });
}

TCB_API int tcb_cetc_host(tcb_context* ctx, const int64_t* h_row_offsets,
                          const int32_t* h_neighbors, int64_t n, int64_t* h_level_out,
                          tcb_result* out) {
    return host_entry(ctx, h_row_offsets, h_neighbors, n, h_level_out, 0, 1, out);
}

TCB_API int tcb_cetc_host_shard(tcb_context* ctx, const int64_t* h_row_offsets,
                                const int32_t* h_neighbors, int64_t n, int shard, int nshards,
                                tcb_result* out) {
    return host_entry(ctx, h_row_offsets, h_neighbors, n, nullptr, shard, nshards, out);
}

}  // extern "C"

// order.cu — pieces of the CETC variants around the core path:
//
//  * degree_order (graph.py:203-213, used by CETC-Seq-D / CETC-Seq-SD): relabel
//    vertices by non-increasing degree, ties by ascending old id.  One radix
//    sort of (n-1-d(v)) << B | v gives the new order; the forward edges are
//    relabelled and the CSR rebuilt with the normalize path (csr_build).
//  * count_horizontal (the covering ratio of CETC-Seq-FE, sequential.py:176-183):
//    number of u < v edges with equal levels, warp-aggregated.
#include "common.cuh"
#include "scan.cuh"

namespace tcb {

uint64_t* radix_sort_u64(Context* ctx, uint64_t* a, uint64_t* b, int64_t n, int bits);
void csr_build(Context* ctx, const int64_t* pairs, int64_t k, int64_t n, int64_t* row,
               int32_t* nb, int32_t* src, int32_t* eu, int32_t* ev, int64_t* m_out);

__global__ void k_degree_keys(const int64_t* __restrict__ row, int64_t n, int vb,
                              uint64_t* __restrict__ keys) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const uint64_t d = uint64_t(row[v + 1] - row[v]);
        keys[v] = ((uint64_t(n - 1) - d) << vb) | uint64_t(v);
    }
}

__global__ void k_new_ids(const uint64_t* __restrict__ sorted, int64_t n, uint64_t vmask,
                          int32_t* __restrict__ new_id) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        new_id[sorted[i] & vmask] = int32_t(i);
}

void degree_order(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                  int64_t n, int64_t m, int64_t* row_out, int32_t* nb_out, int32_t* src_out) {
    require(n < (int64_t(1) << 31), "vertex ids must fit int32");
    if (n == 0) {
        TCB_CUDA(cudaMemsetAsync(row_out, 0, sizeof(int64_t), ctx->stream));
        return;
    }
    const int vb = bits_for(n);
    uint64_t* a = ctx->wsT<uint64_t>(WS_SORT_A, n);
    uint64_t* b = ctx->wsT<uint64_t>(WS_SORT_B, n);
    TCB_LAUNCH(ctx, k_degree_keys, grid_for(ctx, n, 256), 256, 0, row, n, vb, a);
    const uint64_t* sorted = radix_sort_u64(ctx, a, b, n, 2 * vb);
    int32_t* new_id = ctx->wsT<int32_t>(WS_LEVEL, n);
    TCB_LAUNCH(ctx, k_new_ids, grid_for(ctx, n, 256), 256, 0, sorted, n,
               (uint64_t(1) << vb) - 1, new_id);
    if (m == 0) {
        TCB_CUDA(cudaMemsetAsync(row_out, 0, sizeof(int64_t) * (n + 1), ctx->stream));
        return;
    }
    // graph.py:211-213: relabelled canonical pairs (min, max) -> CSR
    int64_t* pairs = ctx->wsT<int64_t>(WS_BINS, 2 * m);
    const int32_t* nid = new_id;
    scan_apply(
        ctx, 2 * m, [src, nb] __device__(int64_t e) -> int64_t { return nb[e] > src[e] ? 1 : 0; },
        [src, nb, nid, pairs] __device__(int64_t e, int64_t pos, int64_t keep) {
            if (!keep) return;
            const int a = nid[src[e]], c = nid[nb[e]];
            pairs[2 * pos] = min(a, c);
            pairs[2 * pos + 1] = max(a, c);
        },
        nullptr);
    int64_t m2 = 0;
    csr_build(ctx, pairs, m, n, row_out, nb_out, src_out, nullptr, nullptr, &m2);
    require(m2 == m, "degree_order: relabelled graph lost edges");
}

// ---------------------------------------------------------------------------
// split_by_level (sequential.py:186-193 _split_by_level): G0 = the horizontal
// edges (equal levels), as a CSR of its own.  CSR entries are (src, dst)-
// sorted, so the kept entries in order already form G0's sorted rows: a
// keep bit per entry, a word prefix of the bits, a scatter, and every row
// start is the prefix at the parent's row start.

__global__ void k_split_bits(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                             const int32_t* __restrict__ level, int64_t nnz,
                             uint32_t* __restrict__ bits) {
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const unsigned lane = lane_id();
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < nnz;
         base += gthreads) {
        const int64_t e = base + lane;
        const bool keep = e < nnz && level[src[e]] == level[nb[e]];
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) bits[base >> 5] = m;
    }
}

__device__ __forceinline__ int64_t split_rank(const uint32_t* __restrict__ bits,
                                              const int64_t* __restrict__ pre, int64_t p) {
    const int64_t j = p >> 5;
    return pre[j] + __popc(bits[j] & ((1u << (p & 31)) - 1u));
}

__global__ void k_split_scatter(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                                int64_t nnz, const uint32_t* __restrict__ bits,
                                const int64_t* __restrict__ pre, int32_t* __restrict__ nb0,
                                int32_t* __restrict__ src0) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        if (!((bits[e >> 5] >> (e & 31)) & 1u)) continue;
        const int64_t q = split_rank(bits, pre, e);
        nb0[q] = nb[e];
        if (src0) src0[q] = src[e];
    }
}

__global__ void k_split_rows(const int64_t* __restrict__ row, int64_t n,
                             const uint32_t* __restrict__ bits, const int64_t* __restrict__ pre,
                             int64_t* __restrict__ row0) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v <= n; v += stride)
        row0[v] = split_rank(bits, pre, row[v]);
}

void split_by_level(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                    int64_t n, int64_t m, const int32_t* level, int64_t* row0, int32_t* nb0,
                    int32_t* src0, int64_t* m0_out) {
    const int64_t nnz = 2 * m;
    if (n == 0 || nnz == 0) {
        TCB_CUDA(cudaMemsetAsync(row0, 0, sizeof(int64_t) * (n + 1), ctx->stream));
        *m0_out = 0;
        return;
    }
    const int64_t nwords = (nnz + 31) / 32;
    // one spare word: rank() at p = nnz reads bits[nwords] when nnz % 32 == 0
    uint32_t* bits = ctx->wsT<uint32_t>(WS_QUEUE_A, nwords + 1);
    int64_t* pre = ctx->wsT<int64_t>(WS_QUEUE_B, nwords + 2);
    TCB_CUDA(cudaMemsetAsync(bits + nwords, 0, sizeof(uint32_t), ctx->stream));
    TCB_LAUNCH(ctx, k_split_bits, grid_for(ctx, nnz, 256), 256, 0, src, nb, level, nnz, bits);
    const uint32_t* cb = bits;
    scan_apply(
        ctx, nwords, [cb] __device__(int64_t j) -> int64_t { return __popc(cb[j]); },
        [pre] __device__(int64_t j, int64_t pos, int64_t) { pre[j] = pos; }, pre + nwords);
    TCB_LAUNCH(ctx, k_split_scatter, grid_for(ctx, nnz, 256), 256, 0, src, nb, nnz, cb,
               (const int64_t*)pre, nb0, src0);
    TCB_LAUNCH(ctx, k_split_rows, grid_for(ctx, n + 1, 256), 256, 0, row, n, cb,
               (const int64_t*)pre, row0);
    int64_t kept = 0;
    TCB_CUDA(cudaMemcpyAsync(&kept, pre + nwords, sizeof(int64_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    TCB_CUDA(cudaStreamSynchronize(ctx->stream));
    require(kept % 2 == 0, "split_by_level: the horizontal subgraph is not symmetric");
    *m0_out = kept / 2;
}

__global__ void k_count_horizontal(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                                   const int32_t* __restrict__ level, int64_t nnz,
                                   unsigned long long* count) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    unsigned long long c = 0;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        const int u = src[e], v = nb[e];
        c += (v > u && level[u] == level[v]) ? 1 : 0;
    }
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(count, c);
}

void count_horizontal(Context* ctx, const int32_t* src, const int32_t* nb, const int32_t* level,
                      int64_t m, unsigned long long* d_count) {
    TCB_CUDA(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), ctx->stream));
    if (m == 0) return;
    TCB_LAUNCH(ctx, k_count_horizontal, grid_for(ctx, 2 * m, 256), 256, 0, src, nb, level, 2 * m,
               d_count);
}

}  // namespace tcb

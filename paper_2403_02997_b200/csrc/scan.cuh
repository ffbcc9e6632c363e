// scan.cuh — order-preserving device scans and compactions.
//
// Used for every stable compaction on the path (cover-edge selection keeps the
// reference's lexicographic order, bfs.py:101-104; CSR dedup/offsets,
// graph.py:108-117) and for the radix sort's digit offsets.
//
// Shape: reduce-then-scan over tiles of SCAN_TILE items.  Phase 1 reduces
// each tile's values, phase 2 scans the tile sums (recursively), phase 3
// re-derives each item's value, block-scans it and calls the consumer with
// (index, exclusive prefix, value) in index order.  Items are striped across
// the block (thread t of round j takes base + j*BLOCK + t) so loads coalesce.
#pragma once

#include "common.cuh"

namespace tcb {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int64_t SCAN_TILE = int64_t(SCAN_BLOCK) * SCAN_ITEMS;
constexpr int SINGLE_BLOCK = 1024;
constexpr int SINGLE_ITEMS = 16;
constexpr int64_t SINGLE_MAX = int64_t(SINGLE_BLOCK) * SINGLE_ITEMS;

template <typename F>
__global__ void __launch_bounds__(SCAN_BLOCK) k_tile_sum(F f, int64_t n, int64_t* tile_sums) {
    __shared__ int64_t sm[SCAN_BLOCK / 32];
    const int64_t base = int64_t(blockIdx.x) * SCAN_TILE;
    int64_t acc = 0;
#pragma unroll 4
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        int64_t i = base + int64_t(j) * SCAN_BLOCK + threadIdx.x;
        if (i < n) acc += f(i);
    }
    acc = warp_sum(acc);
    if (lane_id() == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t s = 0;
#pragma unroll
        for (int w = 0; w < SCAN_BLOCK / 32; ++w) s += sm[w];
        tile_sums[blockIdx.x] = s;
    }
}

template <typename F, typename G>
__global__ void __launch_bounds__(SCAN_BLOCK)
    k_tile_apply(F f, G g, int64_t n, const int64_t* __restrict__ tile_offsets) {
    __shared__ int64_t sm[SCAN_BLOCK / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * SCAN_TILE;
    int64_t carry = tile_offsets[blockIdx.x];
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        int64_t i = base + int64_t(j) * SCAN_BLOCK + threadIdx.x;
        if (base + int64_t(j) * SCAN_BLOCK >= n) break;  // uniform across block
        int64_t v = i < n ? f(i) : 0;
        int64_t tot;
        int64_t ex = block_exclusive_scan<SCAN_BLOCK>(v, sm, tot);
        if (i < n) g(i, carry + ex, v);
        carry += tot;
    }
}

// Single-block exclusive scan, in place, of up to SINGLE_MAX int64 values.
__global__ void __launch_bounds__(SINGLE_BLOCK)
    k_scan_single(int64_t* data, int64_t n, int64_t* total);

// Entries of scratch an n-item scan needs for its tile-sum levels.
int64_t scan_scratch_len(int64_t n);

// Exclusive scan of data[0..n) in place; *d_total (device, nullable) = sum.
// `scratch` holds scan_scratch_len(n) int64 (nullptr: context WS_SCAN slot).
void scan_inplace(Context* ctx, int64_t* data, int64_t n, int64_t* d_total,
                  int64_t* scratch = nullptr);

// Ordered scan-and-apply: g(i, exclusive_prefix_of_f, f(i)) for i in [0,n).
// *d_total (device, nullable) receives the sum of f.
template <typename F, typename G>
void scan_apply(Context* ctx, int64_t n, F f, G g, int64_t* d_total) {
    if (n <= 0) {
        if (d_total) TCB_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), ctx->stream));
        return;
    }
    int64_t ntiles = ceil_div(n, SCAN_TILE);
    int64_t* sums = ctx->wsT<int64_t>(WS_SCAN, scan_scratch_len(n));
    TCB_LAUNCH(ctx, k_tile_sum<F>, unsigned(ntiles), SCAN_BLOCK, 0, f, n, sums);
    scan_inplace(ctx, sums, ntiles, d_total, sums + ntiles + 32);
    TCB_LAUNCH(ctx, (k_tile_apply<F, G>), unsigned(ntiles), SCAN_BLOCK, 0, f, g, n,
               (const int64_t*)sums);
}

}  // namespace tcb

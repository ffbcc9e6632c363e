// scan.cu — the non-template parts of scan.cuh.
#include "scan.cuh"

namespace tcb {

__global__ void __launch_bounds__(SINGLE_BLOCK)
    k_scan_single(int64_t* data, int64_t n, int64_t* total) {
    __shared__ int64_t sm[SINGLE_BLOCK / 32 + 1];
    // thread t owns the contiguous run [t*SINGLE_ITEMS, (t+1)*SINGLE_ITEMS)
    const int64_t lo = int64_t(threadIdx.x) * SINGLE_ITEMS;
    int64_t vals[SINGLE_ITEMS];
    int64_t run = 0;
#pragma unroll
    for (int j = 0; j < SINGLE_ITEMS; ++j) {
        int64_t i = lo + j;
        vals[j] = i < n ? data[i] : 0;
        run += vals[j];
    }
    int64_t tot;
    int64_t ex = block_exclusive_scan<SINGLE_BLOCK>(run, sm, tot);
#pragma unroll
    for (int j = 0; j < SINGLE_ITEMS; ++j) {
        int64_t i = lo + j;
        if (i < n) data[i] = ex;
        ex += vals[j];
    }
    if (threadIdx.x == 0 && total) *total = tot;
}

int64_t scan_scratch_len(int64_t n) {
    // level 0 holds ceil(n/TILE) tile sums; deeper levels until one block fits
    int64_t len = 0;
    do {
        n = ceil_div(n, SCAN_TILE);
        len += n + 32;
    } while (n > SINGLE_MAX);
    return len + 64;
}

void scan_inplace(Context* ctx, int64_t* data, int64_t n, int64_t* d_total, int64_t* scratch) {
    if (n <= 0) {
        if (d_total) TCB_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), ctx->stream));
        return;
    }
    if (n <= SINGLE_MAX) {
        TCB_LAUNCH(ctx, k_scan_single, 1, SINGLE_BLOCK, 0, data, n, d_total);
        return;
    }
    if (!scratch) scratch = ctx->wsT<int64_t>(WS_SCAN, scan_scratch_len(n));
    int64_t ntiles = ceil_div(n, SCAN_TILE);
    auto f = [data] __device__(int64_t i) -> int64_t { return data[i]; };
    auto g = [data] __device__(int64_t i, int64_t pre, int64_t) { data[i] = pre; };
    TCB_LAUNCH(ctx, k_tile_sum<decltype(f)>, unsigned(ntiles), SCAN_BLOCK, 0, f, n, scratch);
    scan_inplace(ctx, scratch, ntiles, d_total, scratch + ntiles + 32);
    TCB_LAUNCH(ctx, (k_tile_apply<decltype(f), decltype(g)>), unsigned(ntiles), SCAN_BLOCK, 0,
               f, g, n, (const int64_t*)scratch);
}

}  // namespace tcb

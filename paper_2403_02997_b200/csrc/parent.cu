// parent.cu — the reference's FIFO BFS parents (_kernels.py:143-156, the
// `parent` output of bfs_levels_k) and per-edge TREE / STRUT / HORIZONTAL
// classes (bfs.py:83-87), rebuilt level-synchronously on the GPU.
//
// In the reference's FIFO BFS, level L+1 is appended parent by parent in
// queue order, and each parent appends its unvisited neighbours in ascending
// id order (_kernels.py:147-156).  With rank(u) = position of u within its
// level's run of the queue:
//   parent(w) = the level-L neighbour of w with the smallest rank (the first
//               one dequeued claims w), and
//   rank(w)   = #(level-(L+1) vertices whose parent ranks lower)
//             + #(children of parent(w) before w in N(parent(w))).
// One cooperative kernel runs every level with grid-wide barriers:
//   A. warp per level-(L+1) vertex: min over (rank, id) of its level-L
//      neighbours -> parent; count children per parent rank;
//   B. exclusive scan of the per-rank counts (bases);
//   C. warp per level-L parent: walk N(parent) in order, number the
//      children with ballots: rank = base + running count.
// Components need no separation: every candidate parent of w lies in w's
// component and ranks need only be ordered within a component.  Parents of
// different components may share a rank; their children then share that
// rank's bucket, which keeps each component's own order (and ranks stay
// below the level's size).  Level-0 vertices (component roots) all get rank 0.
#include <climits>
#include <cooperative_groups.h>

#include "common.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace tcb {

constexpr int PAR_BLOCK = 512;
constexpr int PAR_SMALL = PAR_BLOCK * 8;  // counts scanned by one block

__global__ void k_level_hist(const int32_t* __restrict__ level, int64_t n,
                             int64_t* __restrict__ cnt) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
        atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[level[v]]), 1ull);
}

__global__ void k_level_scatter(const int32_t* __restrict__ level, int64_t n,
                                int64_t* __restrict__ cursor, int32_t* __restrict__ list) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const unsigned long long pos =
            atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[level[v]]), 1ull);
        list[pos] = int32_t(v);
    }
}

__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}

// Exclusive scan of a[0, N) in place by the whole grid (called by every
// thread; ends with a grid barrier).
__device__ void grid_scan(cg::grid_group& grid, int* a, int64_t N, int64_t* bsum, int* s_tmp) {
    const int t = threadIdx.x;
    if (N <= PAR_SMALL) {
        if (blockIdx.x == 0) {
            int carry = 0;
            for (int64_t b = 0; b < N; b += PAR_BLOCK) {
                const int64_t i = b + t;
                const int v = i < N ? a[i] : 0;
                int tot;
                const int ex = block_exclusive_scan<PAR_BLOCK>(v, s_tmp, tot);
                if (i < N) a[i] = carry + ex;
                carry += tot;
            }
        }
        grid.sync();
        return;
    }
    const int64_t G = gridDim.x;
    const int64_t tile = (N + G - 1) / G;
    const int64_t lo = min(N, int64_t(blockIdx.x) * tile), hi = min(N, lo + tile);
    int64_t s = 0;
    for (int64_t i = lo + t; i < hi; i += PAR_BLOCK) s += a[i];
    s = warp_sum(s);
    __shared__ int64_t s_red[PAR_BLOCK / 32];
    if (lane_id() == 0) s_red[t >> 5] = s;
    __syncthreads();
    if (t == 0) {
        int64_t tot = 0;
        for (int w = 0; w < PAR_BLOCK / 32; ++w) tot += s_red[w];
        bsum[blockIdx.x] = tot;
    }
    grid.sync();
    if (blockIdx.x == 0) {
        int64_t carry = 0;
        __shared__ int64_t s_tmp64[PAR_BLOCK / 32 + 1];
        for (int64_t b = 0; b < G; b += PAR_BLOCK) {
            const int64_t i = b + t;
            const int64_t v = i < G ? bsum[i] : 0;
            int64_t tot;
            const int64_t ex = block_exclusive_scan<PAR_BLOCK>(v, s_tmp64, tot);
            if (i < G) bsum[i] = carry + ex;
            carry += tot;
        }
    }
    grid.sync();
    int carry = int(bsum[blockIdx.x]);
    for (int64_t b = lo; b < hi; b += PAR_BLOCK) {
        const int64_t i = b + t;
        const int v = i < hi ? a[i] : 0;
        int tot;
        const int ex = block_exclusive_scan<PAR_BLOCK>(v, s_tmp, tot);
        if (i < hi) a[i] = carry + ex;
        carry += tot;
    }
    grid.sync();
}

__global__ void __launch_bounds__(PAR_BLOCK)
    k_parent_coop(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                  const int32_t* __restrict__ level, int64_t n, const int32_t* __restrict__ list,
                  const int64_t* __restrict__ off, int max_level, int32_t* rank, int32_t* parent,
                  int* cnt0, int* cnt1, int64_t* bsum) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_tmp[PAR_BLOCK / 32 + 1];
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t gwarp = gtid >> 5, nwarps = gthreads >> 5;
    const unsigned lane = lane_id();
    for (int64_t v = gtid; v < n; v += gthreads) parent[v] = -1;
    for (int64_t i = off[0] + gtid; i < off[1]; i += gthreads) rank[list[i]] = 0;
    grid.sync();
    for (int L = 1; L <= max_level; ++L) {
        int* cnt = (L & 1) ? cnt1 : cnt0;    // indexed by level L-1 ranks (zeroed)
        int* cnt_next = (L & 1) ? cnt0 : cnt1;
        const int64_t b1 = off[L], e1 = off[L + 1];  // level L
        const int64_t b0 = off[L - 1];               // level L-1 = [b0, b1)
        // A. parent pick
        for (int64_t i = b1 + gwarp; i < e1; i += nwarps) {
            const int w = list[i];
            long long best = LLONG_MAX;
            for (int64_t s = row[w] + lane; s < row[w + 1]; s += 32) {
                const int u = nb[s];
                if (level[u] == L - 1) {
                    const long long key = (static_cast<long long>(rank[u]) << 32) | u;
                    best = key < best ? key : best;
                }
            }
            best = warp_min64(best);
            if (lane == 0) {
                TCB_DASSERT(best != LLONG_MAX);
                parent[w] = int(best & 0xFFFFFFFF);
                atomicAdd(&cnt[best >> 32], 1);
            }
        }
        grid.sync();
        // B. bases per parent rank
        grid_scan(grid, cnt, b1 - b0, bsum, s_tmp);
        // C. number each parent's children in adjacency order
        for (int64_t i = b0 + gwarp; i < b1; i += nwarps) {
            const int p = list[i];
            int next = cnt[rank[p]];
            for (int64_t s0 = row[p]; s0 < row[p + 1]; s0 += 32) {
                const int64_t s = s0 + lane;
                bool child = false;
                int w = 0;
                if (s < row[p + 1]) {
                    w = nb[s];
                    child = level[w] == L && parent[w] == p;
                }
                const unsigned m = __ballot_sync(0xffffffffu, child);
                if (child) rank[w] = next + __popc(m & lanemask_lt());
                next += __popc(m);
            }
        }
        for (int64_t i = gtid; i < e1 - b1; i += gthreads) cnt_next[i] = 0;
        grid.sync();
    }
}

void bfs_parent(Context* ctx, const int64_t* row, const int32_t* nb, int64_t n,
                const int32_t* level, int64_t max_level, int32_t* parent) {
    require(n < (int64_t(1) << 31), "vertex ids must fit int32");
    require(max_level >= 0 && max_level < n + 1, "bad max_level");
    if (n == 0) return;
    const int64_t nl = max_level + 1;
    int64_t* off = ctx->wsT<int64_t>(WS_COUNT_TMP, 2 * (nl + 1));
    int64_t* cursor = off + (nl + 1);
    int32_t* list = ctx->wsT<int32_t>(WS_QUEUE_A, n);
    int32_t* rank = ctx->wsT<int32_t>(WS_QUEUE_B, n);
    int* cnt = ctx->wsT<int>(WS_BINS, 2 * (n + 1));
    TCB_CUDA(cudaMemsetAsync(off, 0, sizeof(int64_t) * (nl + 1), ctx->stream));
    TCB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * 2 * (n + 1), ctx->stream));
    TCB_LAUNCH(ctx, k_level_hist, grid_for(ctx, n, 256), 256, 0, level, n, off);
    scan_inplace(ctx, off, nl + 1, nullptr);  // off[nl] = n
    TCB_CUDA(cudaMemcpyAsync(cursor, off, sizeof(int64_t) * (nl + 1), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    TCB_LAUNCH(ctx, k_level_scatter, grid_for(ctx, n, 256), 256, 0, level, n, cursor, list);

    int& per_sm = ctx->parent_blocks_per_sm;
    if (per_sm == 0) {
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_parent_coop, PAR_BLOCK, 0));
        require(per_sm > 0, "parent kernel cannot be co-resident");
    }
    const int grid = per_sm * ctx->num_sms;
    int64_t* bsum = ctx->wsT<int64_t>(WS_MISC, grid + 1);
    int* cnt0 = cnt;
    int* cnt1 = cnt + (n + 1);
    int ml = int(max_level);
    const int64_t* offc = off;
    const int32_t* listc = list;
    void* args[] = {(void*)&row,  (void*)&nb,     (void*)&level, (void*)&n,
                    (void*)&listc, (void*)&offc,  (void*)&ml,    (void*)&rank,
                    (void*)&parent, (void*)&cnt0, (void*)&cnt1,  (void*)&bsum};
    TCB_CUDA(cudaLaunchCooperativeKernel((const void*)k_parent_coop, dim3(grid), dim3(PAR_BLOCK),
                                         args, 0, ctx->stream));
    ctx->launches++;
}

// Edge classes of the canonical edge arrays (u < v, lexicographic = the
// forward CSR entries in row order), bfs.py:83-87: TREE if either endpoint
// is the other's parent, else HORIZONTAL on equal levels, else STRUT.
void edge_classes(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                  int64_t n, int64_t m, const int32_t* level, const int32_t* parent,
                  int8_t* out) {
    (void)row;
    (void)n;
    if (m == 0) return;
    scan_apply(
        ctx, 2 * m, [src, nb] __device__(int64_t e) -> int64_t { return nb[e] > src[e] ? 1 : 0; },
        [src, nb, level, parent, out] __device__(int64_t e, int64_t pos, int64_t keep) {
            if (!keep) return;
            const int u = src[e], v = nb[e];
            const bool tree = parent[v] == u || parent[u] == v;
            out[pos] = tree ? int8_t(0) : (level[u] == level[v] ? int8_t(2) : int8_t(1));
        },
        nullptr);
}

}  // namespace tcb

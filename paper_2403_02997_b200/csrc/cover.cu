// cover.cu — cover-edge selection (bfs.py:97-106) and the per-cover-edge
// intersection with the level dedup rule (_kernels.py:669-695 cetc_count_k,
// _kernels.py:729-755 cetc_sm_range_k).
//
// Selection is an ordered compaction of the lexicographic u<v edge arrays on
// level[u]==level[v] (bfs.py:84), so the cover set comes out in exactly the
// reference's order.
//
// Intersection: for cover edge (u, v), u < v, every common neighbour w is an
// apex.  c1 counts apexes with level[w] != level[u] (the triangle's only
// horizontal edge), c2 those on the same level (each such triangle is seen
// from all three of its horizontal edges); T counts an apex when
// level[w] != level[u] or w > v (_kernels.py:687), so T = c1 + c2/3.
#include "common.cuh"
#include "scan.cuh"

namespace tcb {

// CSR entries (u, v) with u < v are the edge list in lexicographic order
// (graph.py:108-110), so an ordered compaction over them reproduces
// cover_edges' order exactly.
void cover_select(Context* ctx, const int32_t* level, const int32_t* src, const int32_t* nb,
                  int64_t nnz, int32_t* cu, int32_t* cv, int64_t* d_ncover) {
    scan_apply(
        ctx, nnz,
        [level, src, nb] __device__(int64_t e) -> int64_t {
            const int u = src[e], v = nb[e];
            return (v > u && level[u] == level[v]) ? 1 : 0;
        },
        [src, nb, cu, cv] __device__(int64_t e, int64_t pos, int64_t keep) {
            if (keep) {
                cu[pos] = src[e];
                cv[pos] = nb[e];
            }
        },
        d_ncover);
}

// ---------------------------------------------------------------------------
// intersection, v1: one warp per cover edge; lanes take 32 consecutive entries
// of the shorter list and binary-search them in the longer list, whose search
// window's lower end advances monotonically chunk by chunk.

constexpr int INT_BLOCK = 256;

__global__ void __launch_bounds__(INT_BLOCK)
    k_intersect_warp(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                     const int32_t* __restrict__ level, const int32_t* __restrict__ cu,
                     const int32_t* __restrict__ cv, const int64_t* __restrict__ d_total,
                     int64_t k0, int64_t k1, int shard, int nshards, DevCounters* C, int alo,
                     int ahi) {
    if (d_total) {  // this shard's contiguous slice of the device-side cover count
        const int64_t total = *d_total;
        k0 = total * shard / nshards;
        k1 = total * (shard + 1) / nshards;
    }
    const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    unsigned long long c1 = 0, c2 = 0, t = 0;
    for (int64_t e = k0 + gwarp; e < k1; e += nwarps) {
        const int u = cu[e], v = cv[e];  // u < v: v is the tie-break vertex
        const int lu = level[u];
        int64_t ab = row[u], ae = row[u + 1];
        int64_t bb = row[v], be = row[v + 1];
        if (alo > 0 || ahi < 0x7fffffff) {
            // apexes restricted to ids [alo, ahi) (_kernels.py:766-772
            // cetc_count_restricted_k): both lists cut to that id range
            auto lb = [&](int64_t b, int64_t e, int key) {
                while (b < e) {
                    const int64_t mid = (b + e) >> 1;
                    if (nb[mid] < key) b = mid + 1; else e = mid;
                }
                return b;
            };
            const int64_t a0 = lb(ab, ae, alo), a1 = lb(a0, ae, ahi);
            const int64_t b0 = lb(bb, be, alo), b1 = lb(b0, be, ahi);
            ab = a0; ae = a1; bb = b0; be = b1;
        }
        if (ae - ab > be - bb) {
            int64_t t0 = ab, t1 = ae;
            ab = bb; ae = be; bb = t0; be = t1;
        }
        int64_t lo = bb;
        for (int64_t p0 = ab; p0 < ae; p0 += 32) {
            const int64_t p = p0 + lane;
            const bool valid = p < ae;
            const int x = valid ? nb[p] : 0x7fffffff;
            int64_t L = lo, H = be;
            while (L < H) {
                int64_t mid = (L + H) >> 1;
                if (nb[mid] < x) L = mid + 1; else H = mid;
            }
            if (valid && L < be && nb[L] == x) {
                if (level[x] != lu) {
                    c1++;
                    t++;
                } else {
                    c2++;
                    t += (x > v);
                }
            }
            const int last = int(ae - p0 < 32 ? ae - p0 - 1 : 31);
            lo = __shfl_sync(0xffffffffu, L, last);
        }
    }
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    t = warp_sum(t);
    if (lane == 0) {
        if (c1) atomicAdd(&C->c1, c1);
        if (c2) atomicAdd(&C->c2, c2);
        if (t) atomicAdd(&C->t, t);
    }
}

// Cover edges [k0, k1) — or, when d_total is set, shard `shard` of `nshards`
// equal slices of [0, *d_total).  k_upper bounds the range for grid sizing.
void cetc_intersect(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* level,
                    const int32_t* cu, const int32_t* cv, const int64_t* d_total, int64_t k0,
                    int64_t k1, int shard, int nshards, int64_t k_upper, int alo, int ahi) {
    const int64_t work = k_upper - k0;
    if (work <= 0) return;
    int grid = grid_for(ctx, work * 32, INT_BLOCK, 16);
    TCB_LAUNCH(ctx, k_intersect_warp, grid, INT_BLOCK, 0, row, nb, level, cu, cv, d_total, k0, k1,
               shard, nshards, ctx->d_counters, alo, ahi);
}

}  // namespace tcb

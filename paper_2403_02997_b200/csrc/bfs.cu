// bfs.cu — levels of the reference's all-component BFS (_kernels.py:129-157).
//
// The reference roots each component at its lowest unvisited id
// (_kernels.py:137-142), i.e. at the component's minimum vertex id, and
// levels are BFS distances from that root.  So the levels equal those of ONE
// multi-source BFS seeded with every component's min-id vertex at level 0:
//
//   1. components: union-find over the u<v edges where a larger root is always
//      hooked under a smaller one (ECL-CC style, lock-free CAS), so each tree's
//      root is its minimum id; roots give `components` (isolated vertices are
//      their own roots and sit at level 0).
//   2. BFS: one cooperative persistent kernel runs every level with a grid-wide
//      barrier between levels (no host round trip per level — the 2048-level
//      lattice would otherwise be launch/sync bound).  Direction-optimising:
//      top-down warp-per-frontier-vertex expansion with CAS claims and
//      warp-aggregated queue appends; bottom-up over unvisited vertices with
//      early exit when the frontier's incident edges exceed the unexplored
//      ones / ALPHA; back to top-down when the frontier shrinks below n / BETA.
//
// parent/TREE-vs-STRUT classes depend on the reference's FIFO order and are
// not produced; levels, components and max_level are exact.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace tcb {

// ---------------------------------------------------------------------------
// connected components with min-id representatives

__device__ __forceinline__ int ld_volatile(const int* p) { return *(volatile const int*)p; }

__device__ __forceinline__ int find_root(int v, int* parent) {
    int curr = ld_volatile(&parent[v]);
    if (curr != v) {
        int prev = v, next;
        // parents only ever point to smaller ids; path halving on the way up
        while (curr > (next = ld_volatile(&parent[curr]))) {
            parent[prev] = next;
            prev = curr;
            curr = next;
        }
    }
    return curr;
}

__global__ void k_cc_init(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                          int64_t n, int* __restrict__ parent) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        // rows are sorted: the first neighbour is the smallest one
        int p = int(v);
        if (row[v + 1] > row[v]) {
            int w = nb[row[v]];
            if (w < p) p = w;
        }
        parent[v] = p;
    }
}

// Union the trees of u and v, hooking the larger root under the smaller one
// (so every tree's root stays its minimum id).  Lock-free: a failed CAS means
// the root moved; continue from what it points to now.
__device__ __forceinline__ void hook(int u, int v, int* parent) {
    int ustat = find_root(u, parent);
    int vstat = find_root(v, parent);
    while (ustat != vstat) {
        if (ustat < vstat) {
            int ret = atomicCAS(&parent[vstat], vstat, ustat);
            if (ret == vstat) break;
            vstat = find_root(ret, parent);
        } else {
            int ret = atomicCAS(&parent[ustat], ustat, vstat);
            if (ret == ustat) break;
            ustat = find_root(ret, parent);
        }
    }
}

// one hook per undirected edge: the CSR entries (u, v) with u < v
__global__ void k_cc_hook(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                          int64_t nnz, int* parent) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        const int u = src[e], v = nb[e];
        if (v > u) hook(u, v, parent);
    }
}

// ---- Afforest-style sampling: hook every vertex to its first CC_SAMPLE
// neighbours, compress, find the dominant root from a fixed sample, and give
// the full neighbour lists only to vertices outside that tree.  Any edge with
// one end outside the dominant tree is still hooked from that end, so the
// result equals the full union-find whatever tree is chosen.

constexpr int CC_SAMPLE = 2;
constexpr int CC_VOTES = 1024;

// both sampling rounds in one pass (CC_SAMPLE = 2): one read of the row
// bounds, the second hook right after the first (RMAT-22 components
// 1.15 -> 0.82 ms against one launch per round)
static_assert(CC_SAMPLE == 2, "k_cc_sample hooks exactly two neighbours");
__global__ void k_cc_sample(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                            int64_t n, int* parent) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const int64_t p = row[v], e = row[v + 1];
        if (p < e) hook(int(v), nb[p], parent);
        if (p + 1 < e) hook(int(v), nb[p + 1], parent);
    }
}

__global__ void k_cc_compress(int64_t n, int* parent) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
        parent[v] = find_root(int(v), parent);
}

// most frequent root among CC_VOTES fixed, spread-out vertices (one block)
__global__ void __launch_bounds__(CC_VOTES) k_cc_vote(int64_t n, const int* parent, int* giant) {
    __shared__ int roots[CC_VOTES];
    __shared__ unsigned long long best;
    const int t = threadIdx.x;
    const int64_t v = (int64_t(t) * 2654435761ll + 12345) % n;
    roots[t] = parent[v];
    if (t == 0) best = 0;
    __syncthreads();
    int cnt = 0;
    for (int j = 0; j < CC_VOTES; ++j) cnt += roots[j] == roots[t];
    atomicMax(&best, (unsigned long long)cnt << 32 | unsigned(roots[t]));
    __syncthreads();
    if (t == 0) *giant = int(best & 0xffffffffu);
}

// remaining neighbours (index >= CC_SAMPLE) of vertices outside the dominant
// tree; a lane takes a short list, the whole warp a long one (a hub outside
// the dominant tree must not serialise on one thread)
constexpr int CC_REST_LONG = 64;
__global__ void k_cc_rest(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                          int64_t n, const int* __restrict__ giant_p, int* parent) {
    const int giant = *giant_p;
    const int lane = int(lane_id());
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < n;
         base += stride) {
        const int64_t v = base + lane;
        int64_t b = 0, e = 0;
        if (v < n) {
            b = row[v] + CC_SAMPLE;
            e = row[v + 1];
            if (b >= e || find_root(int(v), parent) == giant) b = e = 0;
        }
        if (e - b <= CC_REST_LONG)
            for (int64_t p = b; p < e; ++p) hook(int(v), nb[p], parent);
        unsigned longs = __ballot_sync(0xffffffffu, e - b > CC_REST_LONG);
        while (longs) {
            const int src = __ffs(longs) - 1;
            longs &= longs - 1;
            const int64_t lb = __shfl_sync(0xffffffffu, b, src);
            const int64_t le = __shfl_sync(0xffffffffu, e, src);
            const int lv = int(base + src);
            for (int64_t p = lb + lane; p < le; p += 32) hook(lv, nb[p], parent);
        }
    }
}

// Frontier queue entry: the vertex with its row start and degree, written by
// whoever discovers it (it has just read them), so expanding it next level
// starts with the neighbour loads — one dependent memory trip less per level
// on thin-level graphs.
struct __align__(16) QEnt {
    int v, d;
    long long b;
};

// Flatten and seed the BFS: level 0 at roots (comp[v]==v), -1 elsewhere;
// roots with neighbours form the first frontier.
__global__ void k_bfs_seed(const int64_t* __restrict__ row, int64_t n, int* parent,
                           int32_t* __restrict__ level, QEnt* __restrict__ queue,
                           DevCounters* C) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    unsigned long long roots = 0, deg0 = 0, dmax0 = 0;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
        const int64_t v = base + threadIdx.x;
        bool is_root = false, seed = false;
        int64_t deg = 0, rb = 0;
        if (v < n) {
            int r = find_root(int(v), parent);
            parent[v] = r;
            is_root = (r == int(v));
            rb = row[v];
            deg = row[v + 1] - rb;
            seed = is_root && deg > 0;
            level[v] = is_root ? 0 : -1;
        }
        roots += is_root;
        unsigned long long slot = warp_append(seed, &C->q_len[0]);
        if (seed) {
            queue[slot] = QEnt{int(v), int(deg), (long long)rb};
            deg0 += deg;
            dmax0 = max(dmax0, (unsigned long long)deg);
        }
    }
    roots = warp_sum(roots);
    deg0 = warp_sum(deg0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax0 = max(dmax0, __shfl_xor_sync(0xffffffffu, dmax0, o));
    if (lane_id() == 0) {
        if (dmax0) atomicMax(&C->deg_max[0], dmax0);
        if (roots) atomicAdd(&C->components, roots);
        if (deg0) atomicAdd(&C->deg_sum[0], deg0);
    }
}

// ---------------------------------------------------------------------------
// cooperative multi-source BFS

#ifndef TCB_BFS_BLOCK
#define TCB_BFS_BLOCK 512
#endif
constexpr int BFS_BLOCK = TCB_BFS_BLOCK;
constexpr int64_t BFS_ALPHA = 14;  // top-down -> bottom-up when m_f > m_u / ALPHA
constexpr int64_t BFS_BETA = 24;   // bottom-up -> top-down when n_f < n / BETA
constexpr int BFS_HEAVY = 256;     // top-down: longer lists are split into chunks
#ifndef TCB_BFS_LOWDEG
#define TCB_BFS_LOWDEG 64
#endif
constexpr int64_t BFS_LOWDEG = TCB_BFS_LOWDEG;  // td_expand<true> when dmax <= this

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *(volatile const unsigned long long*)p;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Claim and enqueue the unvisited vertices among nb[p] for p in [b, e)
// handled by this warp (lanes stride by 32).  LOWDEG (every frontier degree
// <= BFS_LOWDEG, uniform per level): claim with a bare CAS and load the
// neighbour's degree alongside it, two fewer dependent round trips per level
// on high-diameter low-degree graphs; otherwise test before the CAS, so hub
// levels do not hammer already-visited vertices with atomics.
template <bool LOWDEG>
__device__ __forceinline__ void td_expand(const int64_t* __restrict__ row,
                                          const int32_t* __restrict__ nb, int64_t b, int64_t e,
                                          int32_t* level, int next_level, QEnt* nxt,
                                          unsigned long long* qlen, unsigned long long& my_deg,
                                          unsigned long long& my_dmax) {
    const unsigned lane = lane_id();
    for (int64_t p0 = b; p0 < e; p0 += 32) {
        const int64_t p = p0 + lane;
        bool claim = false;
        int w = 0;
        unsigned long long d = 0;
        int64_t rw = 0;
        if (p < e) {
            w = nb[p];
            if (LOWDEG) {
                rw = row[w];
                d = row[w + 1] - rw;
                claim = atomicCAS(&level[w], -1, next_level) == -1;
            } else if (level[w] == -1 && atomicCAS(&level[w], -1, next_level) == -1) {
                claim = true;
                rw = row[w];
                d = row[w + 1] - rw;
            }
        }
        unsigned long long slot = warp_append(claim, qlen);
        if (claim) {
            nxt[slot] = QEnt{w, int(d), (long long)rw};
            my_deg += d;
            my_dmax = max(my_dmax, d);
        }
    }
}

__global__ void __launch_bounds__(BFS_BLOCK)
    k_bfs_coop(const int64_t* __restrict__ row, const int32_t* __restrict__ nb, int64_t n,
               int32_t* level, QEnt* qa, QEnt* qb, int2* chunks, DevCounters* C,
               int64_t dir_edges) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t gwarp = gtid >> 5;
    const int64_t nwarps = gthreads >> 5;
    const unsigned lane = lane_id();
    __shared__ long long s_bc[3];  // per-block broadcast of the level counters

    int L = 0;
    int64_t nf = int64_t(ld_volatile_u64(&C->q_len[0]));
    int64_t mf = int64_t(ld_volatile_u64(&C->deg_sum[0]));
    int64_t dmax = int64_t(ld_volatile_u64(&C->deg_max[0]));
    int64_t mu = dir_edges - mf;  // directed entries of not-yet-visited vertices
    bool td = true;
    QEnt* cur = qa;
    QEnt* nxt = qb;
    int max_level = 0;

    while (nf > 0) {
        const int sc = L % 3, sn = (L + 1) % 3;
        // Slot (L+2)%3 is written by step L+1 (after the next barrier) and was
        // last read right after barrier L-1, so clear it during this step.
        if (gtid == 0) {
            const int sr = (L + 2) % 3;
            C->q_len[sr] = 0;
            C->deg_sum[sr] = 0;
            C->deg_max[sr] = 0;
            C->nchunks[sr] = 0;
        }
        unsigned long long my_deg = 0, my_dmax = 0;
        if (td) {
            // top-down: warp per frontier vertex; lists longer than BFS_HEAVY
            // are cut into chunks that all warps share after a barrier
            const bool heavy = dmax > BFS_HEAVY;
            for (int64_t i = gwarp; i < nf; i += nwarps) {
                const QEnt q = cur[i];
                const int u = q.v;
                const int64_t b = q.b, e = q.b + q.d;
                if (heavy && e - b > BFS_HEAVY) {
                    const int nch = int((e - b + BFS_HEAVY - 1) / BFS_HEAVY);
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(&C->nchunks[sc], (unsigned long long)nch);
                    base = __shfl_sync(0xffffffffu, base, 0);
                    for (int k = lane; k < nch; k += 32)
                        chunks[base + k] = make_int2(u, k * BFS_HEAVY);
                    continue;
                }
                if (dmax <= BFS_LOWDEG)
                    td_expand<true>(row, nb, b, e, level, L + 1, nxt, &C->q_len[sn], my_deg,
                                    my_dmax);
                else
                    td_expand<false>(row, nb, b, e, level, L + 1, nxt, &C->q_len[sn], my_deg,
                                     my_dmax);
            }
            if (heavy) {
                grid.sync();
                if (threadIdx.x == 0) s_bc[0] = (long long)ld_volatile_u64(&C->nchunks[sc]);
                __syncthreads();
                const int64_t nch = s_bc[0];
                __syncthreads();
                for (int64_t c = gwarp; c < nch; c += nwarps) {
                    const int2 ch = chunks[c];
                    const int64_t b = row[ch.x] + ch.y;
                    const int64_t e = min(row[ch.x + 1], b + BFS_HEAVY);
                    td_expand<false>(row, nb, b, e, level, L + 1, nxt, &C->q_len[sn], my_deg,
                                     my_dmax);
                }
            }
        } else {
            // bottom-up: every unvisited vertex looks for a parent on level L
            for (int64_t base = gtid - lane; base < n; base += gthreads) {
                const int64_t v = base + lane;
                bool found = false;
                if (v < n && level[v] == -1) {
                    const int64_t b = row[v], e = row[v + 1];
                    for (int64_t p = b; p < e; ++p) {
                        if (level[nb[p]] == L) {
                            found = true;
                            break;
                        }
                    }
                    if (found) {
                        level[v] = L + 1;
                        my_deg += e - b;
                        my_dmax = max(my_dmax, (unsigned long long)(e - b));
                    }
                }
                unsigned cnt = __popc(__ballot_sync(0xffffffffu, found));
                if (lane == 0 && cnt) atomicAdd(&C->q_len[sn], (unsigned long long)cnt);
            }
        }
        my_deg = warp_sum(my_deg);
        my_dmax = warp_max_u64(my_dmax);
        if (lane == 0) {
            if (my_deg) atomicAdd(&C->deg_sum[sn], my_deg);
            if (my_dmax) atomicMax(&C->deg_max[sn], my_dmax);
        }

        grid.sync();

        if (threadIdx.x == 0) {
            s_bc[0] = (long long)ld_volatile_u64(&C->q_len[sn]);
            s_bc[1] = (long long)ld_volatile_u64(&C->deg_sum[sn]);
            s_bc[2] = (long long)ld_volatile_u64(&C->deg_max[sn]);
        }
        __syncthreads();
        const int64_t nf_next = s_bc[0];
        const int64_t mf_next = s_bc[1];
        dmax = s_bc[2];
        __syncthreads();
#ifdef TCB_CHECKS
        if (gtid == 0 && (L < 40 || (L & 255) == 0)) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            printf("BFS L=%d mode=%s nf=%lld nf_next=%lld mf_next=%lld dmax=%lld t_ns=%llu\n", L,
                   td ? "TD" : "BU", (long long)nf, (long long)nf_next, (long long)mf_next,
                   (long long)dmax, now);
        }
#endif
        if (nf_next > 0) max_level = L + 1;
        mu -= mf_next;
        bool next_td;
        if (td)
            next_td = !(mf_next > mu / BFS_ALPHA);
        else
            next_td = (nf_next < n / BFS_BETA) && (nf_next < nf);

        if (nf_next > 0 && next_td && !td) {
            // materialise the level-(L+1) frontier as a queue for top-down
            unsigned long long* qc = &C->scratch[4];
            for (int64_t base = gtid - lane; base < n; base += gthreads) {
                const int64_t v = base + lane;
                bool in = v < n && level[v] == L + 1;
                unsigned long long slot = warp_append(in, qc);
                if (in) {
                    const int64_t rb = row[v];
                    nxt[slot] = QEnt{int(v), int(row[v + 1] - rb), (long long)rb};
                }
            }
            grid.sync();
            if (gtid == 0) *qc = 0;  // nobody reads it; next use is >= 1 sync away
        }
        if (td || next_td) {
            QEnt* t = cur;
            cur = nxt;
            nxt = t;
        }
        td = next_td;
        nf = nf_next;
        ++L;
    }
    if (gtid == 0) C->max_level = max_level;
}

// ---------------------------------------------------------------------------

__global__ void k_cc_iota(int64_t n, int* __restrict__ parent) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
        parent[v] = int(v);
}

// Streaming components for the host-buffer entries: every vertex its own
// tree, then each neighbour chunk, once resident, hooks its entries (u, v)
// with u < v — one hook per undirected edge over all chunks, the full
// union-find, hidden under the rest of the transfer.  Roots are min ids
// whatever the hook order, so bfs_levels (which then skips its Afforest
// phases) labels exactly as from the sampled path.
void cc_stream_begin(Context* ctx, int64_t n) {
    int* parent = ctx->wsT<int>(WS_COMP, n);
    TCB_LAUNCH(ctx, k_cc_iota, grid_for(ctx, n, 256), 256, 0, n, parent);
    ctx->cc_ready = true;
}

void cc_stream_hook(Context* ctx, const int32_t* src, const int32_t* nb, int64_t e0, int64_t e1) {
    if (e1 <= e0) return;
    int* parent = static_cast<int*>(ctx->slot_ptr[WS_COMP]);
    TCB_LAUNCH(ctx, k_cc_hook, grid_for(ctx, e1 - e0, 256), 256, 0, src + e0, nb + e0, e1 - e0,
               parent);
}

void bfs_levels(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                int64_t n, int64_t m, int32_t* level, bool reset_counters) {
    require(n < (int64_t(1) << 31), "vertex ids must fit int32");
    DevCounters* C = ctx->d_counters;
    if (reset_counters) TCB_CUDA(cudaMemsetAsync(C, 0, sizeof(DevCounters), ctx->stream));
    if (n == 0) return;
    int* parent = ctx->wsT<int>(WS_COMP, n);
    ctx->record(0);
    const bool hooked = ctx->cc_ready;  // cc_stream_* already built the full union-find
    ctx->cc_ready = false;
    if (!hooked) TCB_LAUNCH(ctx, k_cc_init, grid_for(ctx, n, 256), 256, 0, row, nb, n, parent);
    if (m > 0 && !hooked) {
        (void)src;
        int* giant = reinterpret_cast<int*>(&C->scratch[11]);
        TCB_LAUNCH(ctx, k_cc_sample, grid_for(ctx, n, 256), 256, 0, row, nb, n, parent);
        TCB_LAUNCH(ctx, k_cc_compress, grid_for(ctx, n, 256), 256, 0, n, parent);
        TCB_LAUNCH(ctx, k_cc_vote, 1, CC_VOTES, 0, n, (const int*)parent, giant);
        TCB_LAUNCH(ctx, k_cc_rest, grid_for(ctx, n, 256), 256, 0, row, nb, n, (const int*)giant,
                   parent);
    }
    QEnt* qa = ctx->wsT<QEnt>(WS_QUEUE_A, n);
    QEnt* qb = ctx->wsT<QEnt>(WS_QUEUE_B, n);
    TCB_LAUNCH(ctx, k_bfs_seed, grid_for(ctx, n, 256), 256, 0, row, n, parent, level, qa, C);
    ctx->record(1);
    if (m > 0) {
        if (ctx->bfs_coop_blocks == 0) {
            int per_sm = 0;
            TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_coop,
                                                                   BFS_BLOCK, 0));
            require(per_sm > 0, "BFS kernel cannot be co-resident");
            ctx->bfs_coop_blocks = per_sm * ctx->num_sms;
        }
        int64_t dir_edges = 2 * m;
        int2* chunks = ctx->wsT<int2>(WS_MISC, 2 * m / BFS_HEAVY + n + 1);
        void* args[] = {(void*)&row, (void*)&nb,     (void*)&n, (void*)&level,    (void*)&qa,
                        (void*)&qb,  (void*)&chunks, (void*)&C, (void*)&dir_edges};
        TCB_CUDA(cudaLaunchCooperativeKernel((const void*)k_bfs_coop, dim3(ctx->bfs_coop_blocks),
                                             dim3(BFS_BLOCK), args, 0, ctx->stream));
        ctx->launches++;
    }
    ctx->record(2);
}

}  // namespace tcb

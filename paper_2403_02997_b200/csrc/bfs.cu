// bfs.cu — levels of the reference's all-component BFS (_kernels.py:129-157).
//
// The reference roots each component at its lowest unvisited id
// (_kernels.py:137-142), i.e. at the component's minimum vertex id, and
// levels are BFS distances from that root.  So the levels equal those of a
// multi-source BFS seeded with every component's minimum at level 0.  The
// minima are found without a union-find over the whole graph:
//
//   1. probe: isolated vertices (degree 0) are their own components at level
//      0; r0 = the lowest NON-isolated id is the minimum of its component
//      (every smaller id is isolated), so it is a root.
//   2. BFS from r0 (one cooperative persistent kernel, every level, grid-wide
//      barriers; direction-optimising).  On the graphs this path targets r0's
//      component is almost the whole graph.  The kernel ends by listing the
//      vertices it left unvisited (other components, U).
//   3. remainder: a lock-free min-root union-find over U only (hooking the
//      larger root under the smaller, so each tree's root is its component's
//      minimum), roots seeded at level 0, and a second BFS over U.  Nothing
//      runs when U is empty.
//
// BFS steps.  Top-down: a warp per frontier vertex (lists longer than
// BFS_HEAVY are cut into chunks all warps share), int4 neighbour loads, CAS
// claims, one queue append per warp pass.  Bottom-up (for the wide middle
// levels): a warp per 32 consecutive vertices; a visited bitmap skips settled
// words, each unvisited vertex scans its row with int4 loads against the
// frontier BITMAP (ceil(n/32) words: 2 MB at RMAT-24, L2-resident) and stops
// at the first hit; the next frontier bitmap word is the warp's ballot (no
// atomics).  Switch top-down -> bottom-up when the frontier's incident edges
// exceed the unexplored ones / ALPHA; back when the frontier drops below
// n / BETA.  Counters are accumulated per thread and added once per warp per
// level.
//
// parent/TREE-vs-STRUT classes (FIFO order) are produced by parent.cu from
// these levels; levels, components and max_level are exact.
#include <cooperative_groups.h>

#include "common.cuh"

#include <algorithm>
#include <cstdlib>

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

// Frontier queue entry: the vertex with its row start and degree, written by
// whoever discovers it (it has just read them), so expanding it next level
// starts with the neighbour loads — one dependent memory trip less per level
// on thin-level graphs.
struct __align__(16) QEnt {
    int v, d;
    long long b;
};


// ---------------------------------------------------------------------------
// 1. probe: level 0 at isolated vertices, -1 elsewhere; isolated count; the
//    lowest non-isolated id r0 (max-reduced as n - v).  The last block to
//    finish seeds the BFS with r0.

__global__ void k_bfs_probe(const int64_t* __restrict__ row, int64_t n,
                            int32_t* __restrict__ level, QEnt* __restrict__ queue,
                            DevCounters* C) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    unsigned long long iso = 0, key = 0;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const bool isolated = row[v + 1] == row[v];
        level[v] = isolated ? 0 : -1;
        iso += isolated;
        if (!isolated) key = max(key, (unsigned long long)(n - v));
    }
    iso = warp_sum(iso);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane_id() == 0) {
        if (iso) atomicAdd(&C->components, iso);
        if (key) atomicMax(&C->r0key, key);
    }
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0)
        last = atomicAdd(&C->probe_done, 1ull) == (unsigned long long)(gridDim.x - 1);
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long k = *(volatile unsigned long long*)&C->r0key;
        if (k) {
            const int r0 = int(n - int64_t(k));
            const int64_t b = row[r0];
            const int64_t d = row[r0 + 1] - b;
            level[r0] = 0;
            queue[0] = QEnt{r0, int(d), (long long)b};
            C->q_len[0] = 1;
            C->deg_sum[0] = (unsigned long long)d;
            C->deg_max[0] = (unsigned long long)d;
            C->components += 1;
        }
    }
}

// ---------------------------------------------------------------------------
// 2. cooperative direction-optimising BFS

#ifndef TCB_BFS_BLOCK
#define TCB_BFS_BLOCK 512
#endif
#ifndef TCB_BFS_MINB
#define TCB_BFS_MINB (1024 / TCB_BFS_BLOCK)  // 1024 threads per SM, <= 64 registers
#endif
constexpr int BFS_BLOCK = TCB_BFS_BLOCK;
constexpr int BFS_WPB = BFS_BLOCK / 32;
#ifndef TCB_BFS_ALPHA
#define TCB_BFS_ALPHA 14
#endif
#ifndef TCB_BFS_BETA
#define TCB_BFS_BETA 24
#endif
constexpr int64_t BFS_ALPHA = TCB_BFS_ALPHA;  // top-down -> bottom-up when m_f > m_u / ALPHA
constexpr int64_t BFS_BETA = TCB_BFS_BETA;    // bottom-up -> top-down when n_f < n / BETA
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

// The int4 of neighbour entries holding position q (q % 4 == 0).  Rows are
// not 16-byte aligned, so a lane's four entries are masked to [b, e); the
// aligned load never leaves the allocation that holds nb[b, e).
__device__ __forceinline__ int4 ld_nb4(const int32_t* __restrict__ nb, int64_t q) {
    return __ldg(reinterpret_cast<const int4*>(nb + q));
}

// Claim and enqueue the unvisited vertices among nb[p], p in [b, e), that
// this warp handles.
//  * LOWDEG (every frontier degree <= BFS_LOWDEG, uniform per level: the
//    high-diameter, low-degree case): lane per entry, claim with a bare CAS
//    and load the neighbour's row bounds alongside it — two fewer dependent
//    round trips per level.
//  * otherwise (hub levels): lane l takes the aligned int4 at a0 + 4 l + 128 k
//    (four entries per load, masked to [b, e)); test before the CAS so hub
//    levels do not hammer visited vertices with atomics; one queue append
//    per 128 entries.
template <bool LOWDEG>
__device__ __forceinline__ void td_expand(const int64_t* __restrict__ row,
                                          const int32_t* __restrict__ nb, int64_t b, int64_t e,
                                          int32_t* level, int next_level, QEnt* nxt,
                                          unsigned long long* qlen, unsigned long long& my_deg,
                                          unsigned long long& my_dmax) {
    const unsigned lane = lane_id();
    if (LOWDEG) {
        for (int64_t p0 = b; p0 < e; p0 += 32) {
            const int64_t p = p0 + lane;
            bool claim = false;
            int w = 0;
            unsigned long long d = 0;
            int64_t rw = 0;
            if (p < e) {
                w = nb[p];
                rw = row[w];
                d = row[w + 1] - rw;
                claim = atomicCAS(&level[w], -1, next_level) == -1;
            }
            unsigned long long slot = warp_append(claim, qlen);
            if (claim) {
                nxt[slot] = QEnt{w, int(d), (long long)rw};
                my_deg += d;
                my_dmax = max(my_dmax, d);
            }
        }
        return;
    }
    const int bi = int(b), ei = int(e);  // 2m < 2^31
    for (int q0 = bi & ~3; q0 < ei; q0 += 128) {
        const int q = q0 + 4 * int(lane);
        int w[4] = {0, 0, 0, 0};
        unsigned cm = 0;  // claimed entries of this lane
        if (q < ei) {
            const int4 x = ld_nb4(nb, q);
            w[0] = x.x;
            w[1] = x.y;
            w[2] = x.z;
            w[3] = x.w;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (q + i >= bi && q + i < ei && level[w[i]] == -1 &&
                    atomicCAS(&level[w[i]], -1, next_level) == -1)
                    cm |= 1u << i;
        }
        const int c = __popc(cm);
        const int inc = warp_inclusive_scan(c);
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        if (tot == 0) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(qlen, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(inc - c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!((cm >> i) & 1u)) continue;
            const int64_t rw = row[w[i]];
            const int d = int(row[w[i] + 1] - rw);
            nxt[base++] = QEnt{w[i], d, (long long)rw};
            my_deg += (unsigned long long)d;
            my_dmax = max(my_dmax, (unsigned long long)d);
        }
    }
}

// Two levels per grid barrier (thin, low-degree top-down levels: the
// lattice's 2,047 levels are latency chains plus a barrier each).  From the
// level-L frontier every neighbour w is LOWERED to L+1 (atomicMin on the
// level as unsigned: unvisited, -1, is the largest value) and whoever lowers
// it expands it at once, lowering its neighbours to L+2.  When the barrier
// is reached every vertex at distance L+1 is adjacent to the frontier, so it
// holds L+1 and was expanded exactly once (one lane sees the old value above
// L+1); every vertex holding L+2 is adjacent to an L+1 vertex and not to the
// frontier, so L+2 is its distance.  A vertex first lowered to L+2 is queued
// for the next step; if it is later lowered to L+1 (a "demotion") its queue
// entry is stale and harmless: all its neighbours already hold <= L+2 and
// lowering them to L+3 does nothing.  n2 = pushes - demotions is the exact
// size of the L+2 set.
#ifndef TCB_BFS_TWO
#define TCB_BFS_TWO 1  // low-degree path: frontier <= TCB_BFS_TWO x warps (0: off)
#endif
constexpr int TWO_SERIAL = 6;  // L+1 rows up to this long: expanded by their lane

struct TwoAcc {
    unsigned n1 = 0, deg1 = 0, n2 = 0;  // per thread; n2 wraps: pushes - demotions
};

__device__ __forceinline__ unsigned lower_level(int32_t* level, int w, unsigned l) {
    return atomicMin(reinterpret_cast<unsigned*>(level) + w, l);
}

__device__ __forceinline__ void two_expand(const int64_t* __restrict__ row,
                                           const int32_t* __restrict__ nb, int b, int e,
                                           int32_t* level, int L, QEnt* nxt,
                                           unsigned long long* qlen, TwoAcc& a,
                                           unsigned long long& my_deg,
                                           unsigned long long& my_dmax) {
    const unsigned lane = lane_id();
    const unsigned l1 = unsigned(L + 1), l2 = unsigned(L + 2);
    for (int p0 = b; p0 < e; p0 += 32) {
        const int p = p0 + int(lane);
        int rw = 0, dw = 0;
        unsigned old = 0;
        if (p < e) {
            const int w = nb[p];
            rw = int(row[w]);
            dw = int(row[w + 1]) - rw;
            old = lower_level(level, w, l1);
        }
        // short rows: every lane its own w, one batch of loads and atomics.
        // w's entries are loaded while its atomic is in flight (whether or not
        // it was lowered), so the second hop starts with the compare.
        int x[TWO_SERIAL];
#pragma unroll
        for (int j = 0; j < TWO_SERIAL; ++j) x[j] = p < e && j < dw ? nb[rw + j] : -1;
        const bool low = p < e && old > l1;
        if (low) {
            a.n1 += 1;
            a.deg1 += unsigned(dw);
            if (old == l2) a.n2 -= 1;  // demoted: its L+2 queue entry is stale
        }
        const bool small = low && dw <= TWO_SERIAL;
        if (__any_sync(0xffffffffu, small)) {
            int rx[TWO_SERIAL], dx[TWO_SERIAL];
            unsigned pm = 0;
#pragma unroll
            for (int j = 0; j < TWO_SERIAL; ++j) {
                rx[j] = dx[j] = 0;
                if (small && x[j] >= 0) {
                    rx[j] = int(row[x[j]]);
                    dx[j] = int(row[x[j] + 1]) - rx[j];
                    if (lower_level(level, x[j], l2) == 0xFFFFFFFFu) pm |= 1u << j;
                }
            }
            const int c = __popc(pm);
            const int inc = warp_inclusive_scan(c);
            const int tot = __shfl_sync(0xffffffffu, inc, 31);
            if (tot) {
                unsigned long long base = 0;
                if (lane == 31) base = atomicAdd(qlen, (unsigned long long)tot);
                base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(inc - c);
#pragma unroll
                for (int j = 0; j < TWO_SERIAL; ++j) {
                    if (!((pm >> j) & 1u)) continue;
                    nxt[base++] = QEnt{x[j], dx[j], (long long)rx[j]};
                    a.n2 += 1;
                    my_deg += unsigned(dx[j]);
                    my_dmax = max(my_dmax, (unsigned long long)dx[j]);
                }
            }
        }
        // longer rows: the warp expands them one at a time, lane per entry
        unsigned big = __ballot_sync(0xffffffffu, low && dw > TWO_SERIAL);
        while (big) {
            const int sl = __ffs(big) - 1;
            big &= big - 1;
            const int bb = __shfl_sync(0xffffffffu, rw, sl);
            const int ee = bb + __shfl_sync(0xffffffffu, dw, sl);
            for (int q0 = bb; q0 < ee; q0 += 32) {
                const int q = q0 + int(lane);
                bool claim = false;
                int xv = 0, rxv = 0, dxv = 0;
                if (q < ee) {
                    xv = nb[q];
                    rxv = int(row[xv]);
                    dxv = int(row[xv + 1]) - rxv;
                    claim = lower_level(level, xv, l2) == 0xFFFFFFFFu;
                }
                const unsigned long long slot = warp_append(claim, qlen);
                if (claim) {
                    nxt[slot] = QEnt{xv, dxv, (long long)rxv};
                    a.n2 += 1;
                    my_deg += unsigned(dxv);
                    my_dmax = max(my_dmax, (unsigned long long)dxv);
                }
            }
        }
    }
}

// Does v (row [b, e)) have a neighbour in the frontier bitmap?  int4 loads,
// the four bit tests of a load issued together; stops at the first hit.
__device__ __forceinline__ bool bu_scan(const int32_t* __restrict__ nb, int64_t b, int64_t e,
                                        const uint32_t* __restrict__ fc) {
    for (int64_t q = b & ~int64_t(3); q < e; q += 4) {
        const int4 x = ld_nb4(nb, q);
        const int w[4] = {x.x, x.y, x.z, x.w};
        bool hit = false;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (q + i >= b && q + i < e) hit |= (fc[w[i] >> 5] >> (w[i] & 31)) & 1u;
        if (hit) return true;
    }
    return false;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct BfsBits {
    uint32_t* vis;    // visited
    uint32_t* fb[2];  // frontier of level L in fb[L & 1]
    int64_t nw;       // words per bitmap
};

// bottom-up step L over bitmaps: warp per word of 32 consecutive vertices;
// the word's ballot is the next frontier word and updates the visited word
__device__ __forceinline__ void bu_step(const int64_t* __restrict__ row,
                                     const int32_t* __restrict__ nb, int64_t n, int32_t* level,
                                     const BfsBits& bits, int L, int gwarp, int nwarps,
                                     unsigned long long& my_deg, unsigned long long& my_dmax,
                                     unsigned long long& my_cnt) {
    const unsigned lane = lane_id();
    const uint32_t* __restrict__ fc = bits.fb[L & 1];
    uint32_t* fn = bits.fb[(L + 1) & 1];
    for (int j = gwarp; j < int(bits.nw); j += nwarps) {
        const uint32_t vw = bits.vis[j];
        uint32_t fm = 0;
        if (vw != 0xFFFFFFFFu) {
            const int v = j * 32 + int(lane);
            bool found = false;
            int64_t d = 0;
            if (v < n && !((vw >> lane) & 1u)) {
                const int64_t b = row[v], e = row[v + 1];
                d = e - b;
                found = bu_scan(nb, b, e, fc);
            }
            fm = __ballot_sync(0xffffffffu, found);
            if (found) {
                level[v] = L + 1;
                my_deg += (unsigned long long)d;
                my_dmax = max(my_dmax, (unsigned long long)d);
            }
            if (lane == 0 && fm) bits.vis[j] = vw | fm;
        }
        if (lane == 0) fn[j] = fm;
        my_cnt += lane == 0 ? __popc(fm) : 0;
    }
}

__global__ void __launch_bounds__(BFS_BLOCK, TCB_BFS_MINB)
    k_bfs_coop(const int64_t* __restrict__ row, const int32_t* __restrict__ nb, int64_t n,
               int32_t* level, QEnt* qa, QEnt* qb, int2* chunks, DevCounters* C,
               int64_t dir_edges, const unsigned long long* dir_edges_p, BfsBits bits,
               int* rest, int* parent, int collect, int two_max) {
    cg::grid_group grid = cg::this_grid();
    // 2m < 2^31 (require_sizes): every count below fits 32 bits, which
    // keeps the persistent kernel within 64 registers (2 CTAs per SM)
    const int gtid = int(blockIdx.x * blockDim.x + threadIdx.x);
    const int gthreads = int(gridDim.x * blockDim.x);
    const int gwarp = gtid >> 5;
    const int nwarps = gthreads >> 5;
    const unsigned lane = lane_id();
    __shared__ long long s_bc[6];  // per-block broadcast of the level counters
    __shared__ unsigned long long s_agg[6][BFS_WPB];  // per-warp level counters

    int L = 0;  // level of the current frontier
    int s = 0;  // step (counter slots rotate by step; a two-level step is one)
    // the seed's counters, read once per block (all threads loading one
    // address serialise in its L2 slice)
    if (threadIdx.x == 0) {
        s_bc[0] = (long long)ld_volatile_u64(&C->q_len[0]);
        s_bc[1] = (long long)ld_volatile_u64(&C->deg_sum[0]);
        s_bc[2] = (long long)ld_volatile_u64(&C->deg_max[0]);
    }
    __syncthreads();
    int nf = int(s_bc[0]);
    const int mf = int(s_bc[1]);
    int dmax = int(s_bc[2]);
    __syncthreads();
    // directed entries of unvisited vertices (the second BFS reads its total
    // from the device: the remainder's degree sum)
    int mu = int((dir_edges_p ? int64_t(*dir_edges_p) : dir_edges) - mf);
    bool td = true;
    QEnt* cur = qa;
    QEnt* nxt = qb;
    int max_level = 0;
    if (collect && gtid == 0) C->bfs_t0 = globaltimer_ns();

    while (nf > 0) {
        const int sc = s % 3, sn = (s + 1) % 3;
        // Slot (s+2)%3 is written by step s+1 (after the next barrier) and was
        // last read right after barrier s-1, so clear it during this step.
        if (gtid == 0) {
            const int sr = (s + 2) % 3;
            C->q_len[sr] = 0;
            C->deg_sum[sr] = 0;
            C->deg_max[sr] = 0;
            C->nchunks[sr] = 0;
            C->two_n1[sr] = 0;
            C->two_n2[sr] = 0;
            C->two_deg1[sr] = 0;
        }
        unsigned long long my_deg = 0, my_dmax = 0, my_cnt = 0;
        TwoAcc ta;
        // block-uniform: every block reads the same broadcast counters
        const bool two = two_max > 0 && td && dmax <= BFS_LOWDEG &&
                         int64_t(nf) <= int64_t(nwarps) * two_max;
        if (two) {
            for (int i = gwarp; i < nf; i += nwarps) {
                const QEnt q = cur[i];
                two_expand(row, nb, int(q.b), int(q.b) + q.d, level, L, nxt, &C->q_len[sn], ta,
                           my_deg, my_dmax);
            }
        } else if (td) {
            const bool heavy = dmax > BFS_HEAVY;
            for (int i = gwarp; i < nf; i += nwarps) {
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
                const int nch = int(s_bc[0]);
                __syncthreads();
                for (int c = gwarp; c < nch; c += nwarps) {
                    const int2 ch = chunks[c];
                    const int64_t b = row[ch.x] + ch.y;
                    const int64_t e = min(row[ch.x + 1], b + BFS_HEAVY);
                    td_expand<false>(row, nb, b, e, level, L + 1, nxt, &C->q_len[sn], my_deg,
                                     my_dmax);
                }
            }
        } else {
            bu_step(row, nb, n, level, bits, L, gwarp, nwarps, my_deg, my_dmax, my_cnt);
        }
        my_deg = warp_sum(my_deg);
        my_dmax = warp_max_u64(my_dmax);
        my_cnt = warp_sum(my_cnt);
        // one atomic per block per counter (not per warp): on thin levels
        // same-address atomics, not work, set the level's length
        const int nagg = two ? 6 : 3;
        if (lane == 0) {
            s_agg[0][threadIdx.x >> 5] = my_deg;
            s_agg[1][threadIdx.x >> 5] = my_dmax;
            s_agg[2][threadIdx.x >> 5] = my_cnt;
        }
        if (two) {
            // n2 as a signed per-thread difference, widened before the sums
            const unsigned long long a1 = warp_sum((unsigned long long)ta.n1);
            const unsigned long long a2 =
                warp_sum((unsigned long long)(long long)int(ta.n2));
            const unsigned long long a3 = warp_sum((unsigned long long)ta.deg1);
            if (lane == 0) {
                s_agg[3][threadIdx.x >> 5] = a1;
                s_agg[4][threadIdx.x >> 5] = a2;
                s_agg[5][threadIdx.x >> 5] = a3;
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int k = int(threadIdx.x);
            unsigned long long v[6];
#pragma unroll
            for (int r = 0; r < 6; ++r) v[r] = r < nagg && k < BFS_WPB ? s_agg[r][k] : 0ull;
            v[0] = warp_sum(v[0]);
            v[1] = warp_max_u64(v[1]);
            v[2] = warp_sum(v[2]);
            if (two) {
                v[3] = warp_sum(v[3]);
                v[4] = warp_sum(v[4]);
                v[5] = warp_sum(v[5]);
            }
            if (k == 0) {
                if (v[0]) atomicAdd(&C->deg_sum[sn], v[0]);
                if (v[1]) atomicMax(&C->deg_max[sn], v[1]);
                if (v[2]) atomicAdd(&C->q_len[sn], v[2]);
                if (v[3]) atomicAdd(&C->two_n1[sn], v[3]);
                if (v[4]) atomicAdd(&C->two_n2[sn], v[4]);
                if (v[5]) atomicAdd(&C->two_deg1[sn], v[5]);
            }
        }

        grid.sync();

        if (threadIdx.x == 0) {
            s_bc[0] = (long long)ld_volatile_u64(&C->q_len[sn]);
            s_bc[1] = (long long)ld_volatile_u64(&C->deg_sum[sn]);
            s_bc[2] = (long long)ld_volatile_u64(&C->deg_max[sn]);
            if (two) {
                s_bc[3] = (long long)ld_volatile_u64(&C->two_n1[sn]);
                s_bc[4] = (long long)ld_volatile_u64(&C->two_n2[sn]);
                s_bc[5] = (long long)ld_volatile_u64(&C->two_deg1[sn]);
            }
        }
        __syncthreads();
        int nf_next = int(s_bc[0]);
        const int mf_next = int(s_bc[1]);
        dmax = int(s_bc[2]);
        // levels this step produced: L+1 (and L+2 in a two-level step)
        const int nlev = two ? 2 : 1;
        const long long n1 = two ? s_bc[3] : nf_next;
        const long long n2 = two ? s_bc[4] : 0;
        const int deg1 = two ? int(s_bc[5]) : 0;
        __syncthreads();
        if (two && n2 == 0) nf_next = 0;  // only stale entries queued
#ifdef TCB_CHECKS
        if (gtid == 0 && (L < 40 || (L & 255) == 0)) {
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            printf("BFS L=%d mode=%s nf=%lld nf_next=%lld mf_next=%lld dmax=%lld t_ns=%llu\n", L,
                   two ? "TD2" : td ? "TD" : "BU", (long long)nf, (long long)nf_next,
                   (long long)mf_next, (long long)dmax, now);
        }
#endif
        if (collect && gtid == 0) {  // first BFS only
            const unsigned long long t = (td ? 0ull : 1ull << 62) | globaltimer_ns();
            if (L < TCB_LEVEL_RECORDS) {
                C->lev_rec[2 * L] = t;
                C->lev_rec[2 * L + 1] = (unsigned long long)(two ? n1 : nf_next);
                C->nlev = L + 1;
            }
            if (two && L + 1 < TCB_LEVEL_RECORDS) {
                C->lev_rec[2 * L + 2] = t;
                C->lev_rec[2 * L + 3] = (unsigned long long)n2;
                C->nlev = L + 2;
            }
        }
        if (n1 > 0) max_level = L + 1;
        if (n2 > 0) max_level = L + 2;
        mu -= deg1 + mf_next;
        bool next_td;
        if (td)
            next_td = !(mf_next > mu / BFS_ALPHA);
        else
            next_td = (nf_next < int(n / BFS_BETA)) && (nf_next < nf);
        const int Lf = L + nlev;  // the next frontier's level

        if (nf_next > 0 && !next_td && td) {
            // entering bottom-up: visited and level-Lf bitmaps from the levels
            uint32_t* fn = bits.fb[Lf & 1];
            for (int j = gwarp; j < int(bits.nw); j += nwarps) {
                const int v = j * 32 + int(lane);
                const int lv = v < n ? level[v] : 0;
                const unsigned vm = __ballot_sync(0xffffffffu, lv != -1);
                const unsigned fm = __ballot_sync(0xffffffffu, v < n && lv == Lf);
                if (lane == 0) {
                    bits.vis[j] = vm;
                    fn[j] = fm;
                }
            }
            grid.sync();
        } else if (nf_next > 0 && next_td && !td) {
            // leaving bottom-up: the level-Lf frontier bitmap as a queue
            const uint32_t* fn = bits.fb[Lf & 1];
            unsigned long long* qc = &C->scratch[4];
            for (int j = gwarp; j < int(bits.nw); j += nwarps) {
                const uint32_t fm = fn[j];
                if (fm == 0) continue;  // warp-uniform
                const bool in = (fm >> lane) & 1u;
                const int v = j * 32 + int(lane);
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
        L = Lf;
        ++s;
    }
    if (gtid == 0 && max_level) atomicMax(&C->max_level, max_level);
    if (!collect) return;
    // vertices left unvisited belong to other components: list them (each its
    // own union-find tree for now) with their degree total
    unsigned long long my_rest_deg = 0;
    for (int base = gtid - int(lane); base < n; base += gthreads) {
        const int v = base + int(lane);
        const bool un = v < n && level[v] == -1;
        const unsigned long long slot = warp_append(un, &C->rest_n);
        if (un) {
            rest[slot] = int(v);
            parent[v] = int(v);
            my_rest_deg += (unsigned long long)(row[v + 1] - row[v]);
        }
    }
    my_rest_deg = warp_sum(my_rest_deg);
    if (lane == 0 && my_rest_deg) atomicAdd(&C->rest_deg, my_rest_deg);
}

// ---------------------------------------------------------------------------
// 3. the remainder: union-find over the unvisited vertices (every edge of an
//    unvisited vertex stays inside U), then its roots seed the second BFS

constexpr int CC_REST_LONG = 64;
__global__ void k_rest_hook(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                            const int* __restrict__ rest, const DevCounters* C, int* parent) {
    const int64_t nr = int64_t(C->rest_n);
    const int lane = int(lane_id());
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < nr;
         base += stride) {
        const int64_t i = base + lane;
        int v = 0;
        int64_t b = 0, e = 0;
        if (i < nr) {
            v = rest[i];
            b = row[v];
            e = row[v + 1];
        }
        // one hook per undirected edge: from the lower endpoint
        if (e - b <= CC_REST_LONG)
            for (int64_t p = b; p < e; ++p) {
                const int w = nb[p];
                if (w > v) hook(v, w, parent);
            }
        unsigned longs = __ballot_sync(0xffffffffu, e - b > CC_REST_LONG);
        while (longs) {  // a hub outside r0's component: the whole warp
            const int src = __ffs(longs) - 1;
            longs &= longs - 1;
            const int64_t lb = __shfl_sync(0xffffffffu, b, src);
            const int64_t le = __shfl_sync(0xffffffffu, e, src);
            const int lv = __shfl_sync(0xffffffffu, v, src);
            for (int64_t p = lb + lane; p < le; p += 32) {
                const int w = nb[p];
                if (w > lv) hook(lv, w, parent);
            }
        }
    }
}

__global__ void k_rest_seed(const int64_t* __restrict__ row, const int* __restrict__ rest,
                            int* parent, int32_t* __restrict__ level, QEnt* __restrict__ queue,
                            DevCounters* C) {
    const int64_t nr = int64_t(*(volatile unsigned long long*)&C->rest_n);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    unsigned long long deg = 0, dmax = 0, roots = 0;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nr; base += stride) {
        const int64_t i = base + threadIdx.x;
        bool root = false;
        int v = 0;
        int64_t b = 0, d = 0;
        if (i < nr) {
            v = rest[i];
            root = find_root(v, parent) == v;
            if (root) {
                level[v] = 0;
                b = row[v];
                d = row[v + 1] - b;
            }
        }
        const unsigned long long slot = warp_append(root, &C->q_len[0]);
        if (root) {
            queue[slot] = QEnt{v, int(d), (long long)b};
            deg += (unsigned long long)d;
            dmax = max(dmax, (unsigned long long)d);
            ++roots;
        }
    }
    deg = warp_sum(deg);
    dmax = warp_max_u64(dmax);
    roots = warp_sum(roots);
    if (lane_id() == 0) {
        if (deg) atomicAdd(&C->deg_sum[0], deg);
        if (dmax) atomicMax(&C->deg_max[0], dmax);
        if (roots) atomicAdd(&C->components, roots);
    }
}

static void launch_bfs(Context* ctx, const int64_t* row, const int32_t* nb, int64_t n,
                       int32_t* level, QEnt* qa, QEnt* qb, int2* chunks, int64_t dir_edges,
                       const unsigned long long* dir_edges_p, BfsBits bits, int* rest,
                       int* parent, int collect, int two_max) {
    DevCounters* C = ctx->d_counters;
    if (ctx->bfs_coop_blocks == 0) {
        int per_sm = 0;
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_coop, BFS_BLOCK, 0));
        require(per_sm > 0, "BFS kernel cannot be co-resident");
        ctx->bfs_coop_blocks = per_sm * ctx->num_sms;
    }
    void* args[] = {(void*)&row,   (void*)&nb,          (void*)&n,    (void*)&level,
                    (void*)&qa,    (void*)&qb,          (void*)&chunks, (void*)&C,
                    (void*)&dir_edges, (void*)&dir_edges_p, (void*)&bits,  (void*)&rest,
                    (void*)&parent, (void*)&collect, (void*)&two_max};
    TCB_CUDA(cudaLaunchCooperativeKernel((const void*)k_bfs_coop, dim3(ctx->bfs_coop_blocks),
                                         dim3(BFS_BLOCK), args, 0, ctx->stream));
    ctx->launches++;
}

// ---------------------------------------------------------------------------
// Small graphs (n, m <= SMALL_MAX): the whole cover-edge path in ONE
// cooperative launch.  On graphs of a few thousand edges the ~25 dependent
// kernels of the general path cost more than their work (ER-4096: 0.31 ms);
// here each stage is a grid barrier away from the next:
//   1. isolated vertices at level 0; union-find hooking every edge (larger
//      root under the smaller, so each root is its component's minimum);
//   2. the minima seeded at level 0, multi-source level-synchronous BFS —
//      the reference's lowest-id-root levels (_kernels.py:137-156);
//   3. every horizontal edge u < v (_kernels.py:680): the shorter of N(u),
//      N(v) walked by the warp's lanes, each id binary-searched in the other
//      list; a common neighbour on another level adds to c1, one on the same
//      level to c2 (_kernels.py:745-748, the reference's own per-edge rule:
//      no owner order needed), so T = c1 + c2/3.
constexpr int64_t SMALL_MAX = int64_t(1) << 17;
constexpr int SMALL_BLOCK = 512;

__device__ __forceinline__ bool sorted_contains(const int32_t* __restrict__ a, int len, int key) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo < len && a[lo] == key;
}

// Level-synchronous BFS from the vertices already in qa (q_len[0] of them,
// at level `base`); returns the number of the last non-empty level.
__device__ __forceinline__ int small_bfs(cg::grid_group& grid, const int64_t* __restrict__ row,
                                         const int32_t* __restrict__ nb, int32_t* level, int* qa,
                                         int* qb, DevCounters* C, int gtid, int gwarp,
                                         int nwarps) {
    const int lane = int(lane_id());
    int* cur = qa;
    int* nxt = qb;
    int L = 0;
    __shared__ int s_nf;
    while (true) {
        // one load per block (every thread loading one address serialises
        // in its L2 slice), shared through shared memory
        if (threadIdx.x == 0) s_nf = int(ld_volatile_u64(&C->q_len[L % 3]));
        __syncthreads();
        const int nf = s_nf;
        __syncthreads();
        if (nf == 0) break;
        if (gtid == 0) C->q_len[(L + 2) % 3] = 0;  // read two barriers ago, written next level
        for (int i = gwarp; i < nf; i += nwarps) {
            const int u = cur[i];
            const int next = level[u] + 1;
            for (int64_t p0 = row[u]; p0 < row[u + 1]; p0 += 32) {
                const int64_t p = p0 + lane;
                bool claim = false;
                int w = 0;
                if (p < row[u + 1]) {
                    w = nb[p];
                    claim = level[w] == -1 && atomicCAS(&level[w], -1, next) == -1;
                }
                const unsigned long long slot = warp_append(claim, &C->q_len[(L + 1) % 3]);
                if (claim) nxt[slot] = w;
            }
        }
        grid.sync();
        int* t = cur;
        cur = nxt;
        nxt = t;
        ++L;
    }
    return L - 1;
}

// Every horizontal edge u < v (_kernels.py:680): the lanes test 32 of
// N(u)'s entries at once, and each horizontal one is intersected by walking
// the shorter of N(u), N(v) with the lanes and binary-searching the other
// list; a common neighbour on another level adds to c1, one on the same
// level to c2 (_kernels.py:745-748, the reference's own per-edge rule), so
// T = c1 + c2/3.  Warp per vertex.
__device__ __forceinline__ void small_count(const int64_t* __restrict__ row,
                                            const int32_t* __restrict__ nb, int n,
                                            const int32_t* __restrict__ level, DevCounters* C,
                                            int gwarp, int nwarps) {
    const int lane = int(lane_id());
    unsigned long long c1 = 0, c2 = 0, nh = 0;
    for (int u = gwarp; u < n; u += nwarps) {
        const int64_t ub = row[u], ue = row[u + 1];
        const int lu = level[u];
        for (int64_t q0 = ub; q0 < ue; q0 += 32) {
            // the lanes test 32 neighbours at once; the horizontal ones
            // (v > u on u's level) are then intersected one by one
            const int64_t q = q0 + lane;
            int v = 0;
            int64_t vb = 0, ve = 0;
            bool hz = false;
            if (q < ue) {
                v = nb[q];
                hz = v > u && level[v] == lu;
                if (hz) {
                    vb = row[v];
                    ve = row[v + 1];
                }
            }
            unsigned hm = __ballot_sync(0xffffffffu, hz);
            nh += lane == 0 ? __popc(hm) : 0;
            while (hm) {
                const int src = __ffs(hm) - 1;
                hm &= hm - 1;
                const int64_t b0 = __shfl_sync(0xffffffffu, vb, src);
                const int64_t b1 = __shfl_sync(0xffffffffu, ve, src);
                const bool ushort = ue - ub <= b1 - b0;
                const int32_t* a = nb + (ushort ? ub : b0);
                const int la = int(ushort ? ue - ub : b1 - b0);
                const int32_t* b = nb + (ushort ? b0 : ub);
                const int lb = int(ushort ? b1 - b0 : ue - ub);
                for (int i = lane; i < la; i += 32) {
                    const int w = a[i];
                    if (sorted_contains(b, lb, w)) {
                        if (level[w] != lu) ++c1; else ++c2;
                    }
                }
            }
        }
    }
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    nh = warp_sum(nh);
    if (lane == 0) {
        if (c1) atomicAdd(&C->c1, c1);
        if (c2) atomicAdd(&C->c2, c2);
        if (nh) atomicAdd((unsigned long long*)&C->ncover, nh);
    }
}

// The count alone, after the general path's levels, for low-degree graphs
// (every degree <= LOWDEG_MAX): a thread per vertex u; each horizontal edge
// u < v is a two-pointer merge of the two sorted rows (the reference's own
// merge, _kernels.py:681-694, with its per-hit rule: another level -> c1,
// same level -> c2).
__global__ void __launch_bounds__(256)
    k_lowdeg_count(const int64_t* __restrict__ row, const int32_t* __restrict__ nb, int n,
                   const int32_t* __restrict__ level, DevCounters* C) {
    const int stride = int(gridDim.x * blockDim.x);
    unsigned long long c1 = 0, c2 = 0, nh = 0;
    for (int u = int(blockIdx.x * blockDim.x + threadIdx.x); u < n; u += stride) {
        const int64_t ub = row[u], ue = row[u + 1];
        const int lu = level[u];
        for (int64_t q = ub; q < ue; ++q) {
            const int v = nb[q];
            if (v <= u || level[v] != lu) continue;
            ++nh;
            int64_t i = ub, j = row[v];
            const int64_t je = row[v + 1];
            while (i < ue && j < je) {
                const int a = nb[i], b = nb[j];
                if (a == b) {
                    if (level[a] != lu) ++c1; else ++c2;
                    ++i;
                    ++j;
                } else if (a < b) {
                    ++i;
                } else {
                    ++j;
                }
            }
        }
    }
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    nh = warp_sum(nh);
    if (lane_id() == 0) {
        if (c1) atomicAdd(&C->c1, c1);
        if (c2) atomicAdd(&C->c2, c2);
        if (nh) atomicAdd((unsigned long long*)&C->ncover, nh);
    }
}

__global__ void __launch_bounds__(SMALL_BLOCK)
    k_small_cetc(const int64_t* __restrict__ row, const int32_t* __restrict__ nb, int n,
                 int32_t* level, int* par, int* qa, int* qb, DevCounters* C) {
    cg::grid_group grid = cg::this_grid();
    const int gtid = int(blockIdx.x * blockDim.x + threadIdx.x);
    const int gthreads = int(gridDim.x * blockDim.x);
    const int lane = int(lane_id());
    const int gwarp = gtid >> 5, nwarps = gthreads >> 5;
    // 1. isolated vertices at level 0; r0 = the lowest non-isolated id, the
    //    minimum of its component (every smaller id is isolated): a root
    unsigned long long iso = 0, key = 0;
    for (int v = gtid; v < n; v += gthreads) {
        const bool isolated = row[v + 1] == row[v];
        level[v] = isolated ? 0 : -1;
        iso += isolated;
        if (!isolated) key = max(key, (unsigned long long)(n - v));
    }
    iso = warp_sum(iso);
    key = warp_max_u64(key);
    if (lane == 0) {
        if (iso) atomicAdd(&C->components, iso);
        if (key) atomicMax(&C->r0key, key);
    }
    grid.sync();
    __shared__ unsigned long long s_r0;
    if (threadIdx.x == 0) s_r0 = ld_volatile_u64(&C->r0key);
    __syncthreads();
    const int r0 = int(n - int64_t(s_r0));
    if (gtid == 0) {
        level[r0] = 0;
        qa[0] = r0;
        C->q_len[0] = 1;
        C->components += 1;
    }
    grid.sync();
    // 2. BFS from r0 (on the graphs this path sees, usually everything)
    int max_level = small_bfs(grid, row, nb, level, qa, qb, C, gtid, gwarp, nwarps);
    // 3. what it left unvisited: min-root union-find over those vertices
    //    only (hooking the larger root under the smaller, so each root is its
    //    component's minimum), the roots at level 0, a second BFS
    for (int v = gtid; v < n; v += gthreads) par[v] = v;
    if (gtid == 0) C->q_len[0] = C->q_len[1] = C->q_len[2] = 0;
    grid.sync();
    for (int u = gwarp; u < n; u += nwarps) {
        if (level[u] != -1) continue;  // warp-uniform
        for (int64_t p = row[u] + lane; p < row[u + 1]; p += 32) {
            const int v = nb[p];
            if (v > u) hook(u, v, par);
        }
    }
    grid.sync();
    unsigned long long roots = 0;
    for (int base = gtid - lane; base < n; base += gthreads) {
        const int v = base + lane;
        const bool root = v < n && level[v] == -1 && find_root(v, par) == v;
        const unsigned long long slot = warp_append(root, &C->q_len[0]);
        if (root) qa[slot] = v;
        roots += root;
    }
    roots = warp_sum(roots);
    if (lane == 0 && roots) atomicAdd(&C->components, roots);
    grid.sync();
    if (threadIdx.x == 0) s_r0 = ld_volatile_u64(&C->q_len[0]);
    __syncthreads();
    for (int i = gtid; i < int(s_r0); i += gthreads) level[qa[i]] = 0;
    grid.sync();
    max_level = max(max_level, small_bfs(grid, row, nb, level, qa, qb, C, gtid, gwarp, nwarps));
    if (gtid == 0 && max_level > 0) atomicMax(&C->max_level, (unsigned long long)max_level);
    // 3. the horizontal edges and their common neighbours
    small_count(row, nb, n, level, C, gwarp, nwarps);
}

__global__ void k_max_degree(const int64_t* __restrict__ row, int64_t n,
                             unsigned long long* out) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    unsigned long long d = 0;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
        d = max(d, (unsigned long long)(row[v + 1] - row[v]));
    d = warp_max_u64(d);
    if (lane_id() == 0 && d) atomicMax(out, d);
}

// The one-launch path (k_small_cetc) for graphs of at most 2^17 vertices
// and edges, and for low-degree graphs of any size (max degree <=
// LOWDEG_MAX, e.g. the lattice: there the per-edge binary searches cost less
// than the general path's list build, and the BFS is the same level loop);
// false otherwise (the caller runs the general path).  Deciding the second
// case reads the max degree back: one ~10 us round trip on graphs larger
// than 2^17 edges.
void bfs_levels(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                int64_t n, int64_t m, int32_t* level, bool reset_counters, int two_max);
#ifndef TCB_LOWDEG_MAX
#define TCB_LOWDEG_MAX 32  // ER-like graphs up to mean degree ~16 (tools/path_probe.py)
#endif
constexpr int64_t LOWDEG_MAX = TCB_LOWDEG_MAX;
bool small_cetc(Context* ctx, const int64_t* row, const int32_t* nb, int64_t n, int64_t m,
                int32_t* level) {
    if (m == 0 || ctx->tune_wt || ctx->tune_hc || ctx->test_flags || getenv("TCB_NO_SMALL"))
        return false;
    if (n > SMALL_MAX || m > SMALL_MAX) {
        if (getenv("TCB_NO_LOWDEG")) return false;
        unsigned long long* d_dmax = &ctx->d_counters->scratch[11];
        TCB_CUDA(cudaMemsetAsync(d_dmax, 0, sizeof(unsigned long long), ctx->stream));
        TCB_LAUNCH(ctx, k_max_degree, grid_for(ctx, n, 256), 256, 0, row, n, d_dmax);
        unsigned long long dmax = 0;
        TCB_CUDA(cudaMemcpyAsync(&dmax, d_dmax, sizeof(dmax), cudaMemcpyDeviceToHost, ctx->stream));
        TCB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (dmax > (unsigned long long)LOWDEG_MAX) return false;
        // low degree, large: the general BFS (direction-optimising, block-
        // aggregated level counters) for the levels, then the count kernel
        // (two levels per grid barrier on its thin levels: every row is short)
        bfs_levels(ctx, row, nb, nullptr, n, m, level, false, TCB_BFS_TWO);  // events 0, 1, 2
        ctx->record(3);
        TCB_LAUNCH(ctx, k_lowdeg_count, ctx->num_sms * 8, 256, 0, row, nb, int(n),
                   (const int32_t*)level, ctx->d_counters);
        return true;
    }
    DevCounters* C = ctx->d_counters;
    int* par = ctx->wsT<int>(WS_COMP, n);
    int* qa = reinterpret_cast<int*>(ctx->wsT<QEnt>(WS_QUEUE_A, n));
    int* qb = reinterpret_cast<int*>(ctx->wsT<QEnt>(WS_QUEUE_B, n));
    if (ctx->small_blocks == 0) {
        int per_sm = 0;
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small_cetc, SMALL_BLOCK,
                                                               0));
        require(per_sm > 0, "small-graph kernel cannot be co-resident");
        ctx->small_blocks = ctx->num_sms * std::min(per_sm, 2);
    }
    // every SM: the per-vertex stages are latency chains, so warps matter
    // more than the (nearly size-independent) cost of a grid barrier
    const int blocks = ctx->small_blocks;
    int ni = int(n);
    void* args[] = {(void*)&row, (void*)&nb, (void*)&ni, (void*)&level,
                    (void*)&par, (void*)&qa, (void*)&qb, (void*)&C};
    ctx->record(0);
    ctx->record(1);
    TCB_CUDA(cudaLaunchCooperativeKernel((const void*)k_small_cetc, dim3(blocks),
                                         dim3(SMALL_BLOCK), args, 0, ctx->stream));
    ctx->launches++;
    ctx->record(2);
    ctx->record(3);
    return true;
}

void bfs_levels(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                int64_t n, int64_t m, int32_t* level, bool reset_counters, int two_max) {
    (void)src;
    require(n < (int64_t(1) << 31), "vertex ids must fit int32");
    DevCounters* C = ctx->d_counters;
    if (reset_counters) TCB_CUDA(cudaMemsetAsync(C, 0, sizeof(DevCounters), ctx->stream));
    if (n == 0) return;
    QEnt* qa = ctx->wsT<QEnt>(WS_QUEUE_A, n);
    QEnt* qb = ctx->wsT<QEnt>(WS_QUEUE_B, n);
    ctx->record(0);
    TCB_LAUNCH(ctx, k_bfs_probe, grid_for(ctx, n, 256), 256, 0, row, n, level, qa, C);
    ctx->record(1);
    if (m > 0) {
        int* parent = ctx->wsT<int>(WS_COMP, n);
        const int64_t nw = (n + 31) / 32;
        uint32_t* bw = ctx->wsT<uint32_t>(WS_BFS_BITS, 3 * nw);
        BfsBits bits{bw, {bw + nw, bw + 2 * nw}, nw};
        int2* chunks = ctx->wsT<int2>(WS_MISC, 2 * m / BFS_HEAVY + n + 1);
        int* rest = reinterpret_cast<int*>(qb);  // free once the first BFS is done
        launch_bfs(ctx, row, nb, n, level, qa, qb, chunks, 2 * m, nullptr, bits, rest, parent, 1,
                   two_max);
        // the remainder (kernels exit at once when the first BFS saw everything)
        TCB_LAUNCH(ctx, k_rest_hook, grid_for(ctx, n, 256), 256, 0, row, nb, (const int*)rest,
                   (const DevCounters*)C, parent);
        TCB_CUDA(cudaMemsetAsync(&C->q_len[0], 0,
                                 size_t(reinterpret_cast<char*>(&C->two_deg1[3]) -
                                        reinterpret_cast<char*>(&C->q_len[0])),
                                 ctx->stream));
        TCB_LAUNCH(ctx, k_rest_seed, grid_for(ctx, n, 256), 256, 0, row, (const int*)rest, parent,
                   level, qa, C);
        launch_bfs(ctx, row, nb, n, level, qa, qb, chunks, 0, &C->rest_deg, bits, rest, parent,
                   0, two_max);
    }
    ctx->record(2);
}

}  // namespace tcb

// intersect.cu — the counting path of tc_cetc / tc_cetc_sm on the GPU.
//
// Reference semantics (_kernels.py:669-695 cetc_count_k and :729-755
// cetc_sm_range_k): for every horizontal edge {u, v} (level[u]==level[v]),
// every common neighbour w is an apex; c1 counts apexes on another level, c2
// apexes on the same level, and T counts an apex when level[w] != level[u] or
// w > max(u, v).  T = c1 + c2/3.
//
// The reference merges both full lists per edge: W = sum_S (d(u)+d(v))
// element steps (2.4e12 at RMAT-24).  Here each horizontal edge is owned by
// its higher-degree endpoint x (ties: lower id).  x's list is staged in a
// shared-memory hash set and every partner y's list (the shorter one) is
// streamed past it: sum_S min(d(u), d(v)) probes (10x fewer at RMAT-24).
//
//  1. owner_select: ordered compaction over the CSR entries (x, y) keeping
//     level[x]==level[y] && owns(x, y).  Entries are in row order, so each
//     owner's partners come out contiguous: P[seg_beg[x], seg_end[x]).
//  2. split points: the id space is cut into F equal ranges; split[v][r] is
//     the position in N(v) of the first id in range r (one flat pass over
//     the entries).  An owner whose list exceeds the table is staged one
//     group of ranges at a time, and every partner's matching slice is read
//     from the table — no per-partner searches.
//  3. make_items: owners with d(x) <= TINY -> thread items; <= WT -> warp
//     items (x, p0, p1), <= PW partners each; others -> CTA items
//     (x, p0, p1, group), <= PC partners.  With nshards > 1 only this
//     shard's partner blocks are listed (dist.py shard_of).
//  4. k_isect_tiny / k_isect_warp: one thread / warp per item; the warp tier
//     keeps a per-warp bucket hash of N(x) (4-entry buckets, LDS.128).
//  5. k_isect_cta: one CTA per item; the group's slice of N(x) (<= HC ids)
//     staged in a two-table cuckoo set; the partners' slices are flattened
//     into one element stream (block scan of lengths) that warps consume in
//     CHUNK-element grabs (CHUNK / 32 loads in flight per lane).
//
// Hash entries carry the apex's level relation to the owner in bit 31
// (same level -> c2), so hits need no level gather.  Tallies reduce per warp
// into one 64-bit atomic each.
#include "common.cuh"
#include "scan.cuh"

#include <cstdlib>

namespace tcb {

// Tier thresholds and tile sizes.  The TCB_* macros exist so tools/variants.py
// can A/B alternatives in one GPU session; the defaults are the measured best.
#ifndef TCB_WT
#define TCB_WT 512
#endif
#ifndef TCB_HC
#define TCB_HC 4096
#endif
#ifndef TCB_CHUNK
#define TCB_CHUNK 1024
#endif
#ifndef TCB_PW
#define TCB_PW 64
#endif
constexpr int WT = TCB_WT;            // warp tier: owner degree <= WT
constexpr int W_SLOTS = 2 * WT;       // per-warp bucket table: load <= 1/2
constexpr int W_WARPS = 8;
constexpr int PW = TCB_PW;            // partners per warp item
constexpr int C_THREADS = 512;        // 2 CTAs per SM
constexpr int HC = TCB_HC;            // staged ids per CTA item
constexpr int C_SLOTS = 4 * HC;       // load <= 1/4 (64 KB)
constexpr int PC = 2 * C_THREADS;     // partners per CTA item (2 per thread in the scan)
constexpr int CHUNK = TCB_CHUNK;      // stream elements per warp grab (32 per lane)
constexpr int LOG_F = 5;
constexpr int F = 1 << LOG_F;         // id ranges for split points
constexpr int LONG_LIST = 64;         // warp tier: lists streamed by a whole warp
constexpr int TINY = 16;              // thread tier: owner degree <= TINY
constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t SAME = 0x80000000u;

__device__ __forceinline__ int ceil_log2_dev(int x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// ---------------------------------------------------------------------------
// bucketed hash set in shared memory

struct BucketHash {
    uint32_t* tab;
    unsigned bmask;  // nbuckets - 1
    int shift;       // 32 - log2(nbuckets)

    __device__ __forceinline__ void setup(uint32_t* t, int slots) {
        tab = t;
        const int lb = ceil_log2_dev(slots >> 2);
        bmask = (1u << lb) - 1;
        shift = 32 - lb;
    }
    __device__ __forceinline__ unsigned bucket(int key) const {
        return (unsigned(key) * 0x9E3779B1u) >> shift;
    }
    __device__ __forceinline__ void insert(int key, bool same) const {
        const uint32_t e = uint32_t(key) | (same ? SAME : 0u);
        unsigned b = bucket(key);
        while (true) {
#pragma unroll
            for (int s = 0; s < 4; ++s)
                if (atomicCAS(&tab[4 * b + s], EMPTY, e) == EMPTY) return;
            b = (b + 1) & bmask;
        }
    }
    // 0 = miss, 1 = hit other level, 2 = hit same level.  The first bucket
    // is resolved without branches; the loop runs only when that bucket is
    // full and does not hold the key (rare at load <= 1/4).
    // hits: c_other += apex on another level, c_same += apex on the owner's level
    __device__ __forceinline__ void count(int key, uint32_t& c_other, uint32_t& c_same) const {
        const int r = find(key);
        c_other += r == 1;
        c_same += r >> 1;
    }
    __device__ __forceinline__ int find(int key) const {
        unsigned b = bucket(key);
        {
            const uint4 v = reinterpret_cast<const uint4*>(tab)[b];
            const uint32_t k = uint32_t(key);
            const bool m0 = ((v.x ^ k) << 1) == 0u, m1 = ((v.y ^ k) << 1) == 0u;
            const bool m2 = ((v.z ^ k) << 1) == 0u, m3 = ((v.w ^ k) << 1) == 0u;
            const uint32_t e = m0 ? v.x : (m1 ? v.y : (m2 ? v.z : v.w));
            const bool hit = m0 | m1 | m2 | m3;
            if (hit || v.w == EMPTY) return hit ? 1 + int(e >> 31) : 0;
            b = (b + 1) & bmask;
        }
        while (true) {
            TCB_DASSERT(b <= bmask);
            const uint4 v = reinterpret_cast<const uint4*>(tab)[b];
            const uint32_t k = uint32_t(key);
            if ((v.x & ~SAME) == k) return 1 + (v.x >> 31);
            if ((v.y & ~SAME) == k) return 1 + (v.y >> 31);
            if ((v.z & ~SAME) == k) return 1 + (v.z >> 31);
            if ((v.w & ~SAME) == k) return 1 + (v.w >> 31);
            if (v.w == EMPTY) return 0;  // buckets fill in slot order
            b = (b + 1) & bmask;
        }
    }
};

#ifndef TCB_CUCKOO
#define TCB_CUCKOO 1
#endif
// 2-choice cuckoo set over two half tables (A/B knob TCB_CUCKOO): a probe is
// two LDS.32 and two compares with no loop.  Parallel insertion by atomicExch kick chains; a
// chain longer than CUCKOO_KICKS reports failure and the caller falls back
// to the bucket table (load <= 1/4 makes that vanishingly rare).
constexpr int CUCKOO_KICKS = 64;
#ifndef TCB_FULLTAB
#define TCB_FULLTAB 1
#endif

struct CuckooHash {
    uint32_t* tab;   // table 1: tab[0, half); table 2: tab[half, 2 half)
    uint32_t* tab2;
    int shift;       // 32 - log2(half)
    __device__ __forceinline__ void setup(uint32_t* t, int slots) {
        tab = t;
        const int lh = ceil_log2_dev(slots) - 1;
        tab2 = t + (1 << lh);
        shift = 32 - lh;
    }
    __device__ __forceinline__ unsigned h1(uint32_t k) const { return (k * 0x9E3779B1u) >> shift; }
    __device__ __forceinline__ unsigned h2(uint32_t k) const { return (k * 0x7FEB352Du) >> shift; }
    __device__ __forceinline__ bool insert(int key, bool same) const {
        uint32_t e = uint32_t(key) | (same ? SAME : 0u);
        uint32_t* slot = tab + h1(uint32_t(key));
        for (int it = 0; it < CUCKOO_KICKS; ++it) {
            const uint32_t old = atomicExch(slot, e);
            if (old == EMPTY) return true;
            e = old;  // carry the evicted entry to its slot in the other table
            const uint32_t k = old & ~SAME;
            slot = slot < tab2 ? tab2 + h2(k) : tab + h1(k);
        }
        return false;
    }
    __device__ __forceinline__ int find(int key) const {
        const uint32_t k = uint32_t(key);
        const uint32_t e1 = tab[h1(k)], e2 = tab2[h2(k)];
        const bool m1 = ((e1 ^ k) << 1) == 0u, m2 = ((e2 ^ k) << 1) == 0u;
        return (m1 | m2) ? 1 + int((m1 ? e1 : e2) >> 31) : 0;
    }
    // A key sits in at most one slot, stored as key (other level) or
    // key | SAME (owner's level): two equality tests per table entry and two
    // predicated increments.  key >= 0 (EMPTY would match free slots).
    __device__ __forceinline__ void count(int key, uint32_t& c_other, uint32_t& c_same) const {
#ifdef TCB_NOPROBE  // measurement-only variant: stream without probing
        c_other += uint32_t(key) == 0x7FFFFFFEu;
        return;
#endif
        const uint32_t k = uint32_t(key), ks = k | SAME;
#ifdef TCB_NOCONFLICT  // measurement-only: same loads at bank-conflict-free addresses
        {
            const uint32_t f1 = tab[(h1(k) & ~31u) | (threadIdx.x & 31)];
            const uint32_t f2 = tab2[(h2(k) & ~31u) | (threadIdx.x & 31)];
            c_other += (f1 == k) | (f2 == k);
            c_same += (f1 == ks) | (f2 == ks);
            return;
        }
#endif
        const uint32_t e1 = tab[h1(k)], e2 = tab2[h2(k)];
        c_other += (e1 == k) | (e2 == k);
        c_same += (e1 == ks) | (e2 == ks);
    }
};

// c1/c2 tallies.  T is not tallied: a same-level triangle puts all three of
// its edges in the cover set and is found once per edge, and the reference's
// rule (w > max(u, v), _kernels.py:688-692) accepts exactly one of the three,
// so over the full cover set T == c1 + c2/3 (formed in capi.cu fill_result).
struct Tally {
    unsigned long long c1 = 0, c2 = 0;
    __device__ __forceinline__ void flush(DevCounters* C) {
        c1 = warp_sum(c1);
        c2 = warp_sum(c2);
        if (lane_id() == 0) {
            if (c1) atomicAdd(&C->c1, c1);
            if (c2) atomicAdd(&C->c2, c2);
        }
    }
};

// Forward mode (tcb_forward_count, the forward branch of CETC-Seq-FE): every
// edge is intersected (the caller passes an all-zero level array, so every
// edge is selected and every hit is "same level"), and an owner stages only
// the neighbours ranked above it in (degree desc, id asc) order, the order
// that makes x the owner of (x, y).  A triangle a > b > c in that order is
// then hit once: at (b, c) with apex a.  T = the same-level tally.
__device__ __forceinline__ bool staged(const int2* __restrict__ vinfo, int w, int x, int dx,
                                       int fwd) {
    if (!fwd) return true;
    const int dw = vinfo[w].y;
    return dw > dx || (dw == dx && w < x);
}

// ---------------------------------------------------------------------------
// warp tier helpers: one long list with the whole warp (4 loads in flight per
// lane); a batch of <= 32 lists flattened across lanes.

template <typename Probe>
__device__ __forceinline__ void probe_long(const int32_t* __restrict__ nb, int64_t s, int d,
                                           const Probe& h, Tally& tl) {
    const int lane = int(lane_id());
    uint32_t co = 0, cs = 0;
    int i = lane;
    for (; i + 96 < d; i += 128) {
        const int w0 = nb[s + i], w1 = nb[s + i + 32], w2 = nb[s + i + 64], w3 = nb[s + i + 96];
        h.count(w0, co, cs);
        h.count(w1, co, cs);
        h.count(w2, co, cs);
        h.count(w3, co, cs);
    }
    for (; i < d; i += 32) h.count(nb[s + i], co, cs);
    tl.c1 += co;
    tl.c2 += cs;
}

template <typename Probe>
__device__ __forceinline__ void probe_batch(const int32_t* __restrict__ nb, int64_t ys, int yd,
                                            const Probe& h, Tally& tl) {
    const unsigned lane = lane_id();
    unsigned longs = __ballot_sync(0xffffffffu, yd >= LONG_LIST);
    while (longs) {
        const int k = __ffs(longs) - 1;
        longs &= longs - 1;
        probe_long(nb, __shfl_sync(0xffffffffu, ys, k), __shfl_sync(0xffffffffu, yd, k), h,
                   tl);
    }
    if (yd >= LONG_LIST) yd = 0;
    const int incl = warp_inclusive_scan(yd);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int base = 0; base < total; base += 32) {
        const int i = base + int(lane);
        int k = 0;  // owning lane: smallest k with incl_k > i
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, k + step - 1);
            if (v <= i) k += step;
        }
        const int64_t ysk = __shfl_sync(0xffffffffu, ys, k);
        const int exk = __shfl_sync(0xffffffffu, incl - yd, k);
        if (i < total) {
            uint32_t co = 0, cs = 0;
            h.count(nb[ysk + (i - exk)], co, cs);
            tl.c1 += co;
            tl.c2 += cs;
        }
    }
}

// ---------------------------------------------------------------------------
// 1. owner-grouped selection

// The owner predicate is evaluated once (two random vinfo gathers per
// entry) into a bitmask, one ballot word per 32 entries; both scan passes
// then read bits only.
__global__ void k_owner_bits(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                             const int2* __restrict__ vinfo, int64_t nnz, uint32_t* __restrict__ bits) {
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const unsigned lane = lane_id();
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < nnz;
         base += gthreads) {
        const int64_t e = base + lane;
        bool keep = false;
        if (e < nnz) {
            const int x = src[e], y = nb[e];
            const int2 a = vinfo[x], b = vinfo[y];
            keep = a.x == b.x && (a.y > b.y || (a.y == b.y && x < y));
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) bits[base >> 5] = m;
    }
}

void owner_select(Context* ctx, const int64_t* row, const int32_t* src, const int32_t* nb,
                  const int2* vinfo, int64_t nnz, int32_t* P, int64_t* seg_beg, int64_t* seg_end,
                  int64_t* d_ncover) {
    uint32_t* bits = ctx->wsT<uint32_t>(WS_QUEUE_A, (nnz + 31) / 32);
    TCB_LAUNCH(ctx, k_owner_bits, grid_for(ctx, nnz, 256), 256, 0, src, nb, vinfo, nnz, bits);
    const uint32_t* B = bits;
    scan_apply(
        ctx, nnz,
        [B] __device__(int64_t e) -> int64_t { return (B[e >> 5] >> (e & 31)) & 1u; },
        [src, nb, row, P, seg_beg, seg_end] __device__(int64_t e, int64_t pos, int64_t keep) {
            const int x = src[e];
            if (keep) P[pos] = nb[e];
            if (e == row[x]) seg_beg[x] = pos;
            if (e == row[x + 1] - 1) seg_end[x] = pos + keep;
        },
        d_ncover);
}

__global__ void k_vinfo(const int64_t* __restrict__ row, const int32_t* __restrict__ level,
                        int64_t n, int2* __restrict__ vinfo) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
        vinfo[v] = make_int2(level[v], int(row[v + 1] - row[v]));
}

// ---------------------------------------------------------------------------
// 2. split points: split[v*(F+1) + r] = first position (relative to row[v])
//    of an id >= r << rshift; split[.][0] = 0, split[.][F] = d(v).

__global__ void k_split_points(const int64_t* __restrict__ row, const int32_t* __restrict__ src,
                               const int32_t* __restrict__ nb, int64_t nnz, int rshift,
                               int* __restrict__ split) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        const int v = src[e];
        const int64_t rb = row[v];
        const int r = nb[e] >> rshift;
        int* sv = split + int64_t(v) * (F + 1);
        const int prev = e == rb ? -1 : (nb[e - 1] >> rshift);
        for (int q = prev + 1; q <= r; ++q) sv[q] = int(e - rb);
        if (e == row[v + 1] - 1)
            for (int q = r + 1; q <= F; ++q) sv[q] = int(e + 1 - rb);
    }
}

// ---------------------------------------------------------------------------
// 3. work items

__global__ void k_make_items(const int64_t* __restrict__ row, const int64_t* __restrict__ seg_beg,
                             const int64_t* __restrict__ seg_end, const int* __restrict__ split,
                             int64_t n, longlong4* __restrict__ witems,
                             longlong4* __restrict__ citems, longlong4* __restrict__ titems,
                             unsigned long long* nw, unsigned long long* nc,
                             unsigned long long* nt, int shard, int nshards, int wt, int hc,
                             int tiny) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // Multi-GPU (tcb_cetc_shard): partner block i of owner x belongs to
    // shard (x + i) % nshards (dist.py shard_of mirrors this).  Blocks rather
    // than whole owners, so a hub's work spreads over the ranks.
    auto mine = [shard, nshards](int64_t x, int64_t i) {
        return nshards <= 1 || int((x + i) % nshards) == shard;
    };
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += stride) {
        const int64_t d = row[x + 1] - row[x];
        if (d == 0) continue;
        const int64_t s = seg_beg[x], e = seg_end[x];
        if (e <= s) continue;
        if (d <= tiny) {  // <= TINY partners, each with <= TINY ids
            if (!mine(x, 0)) continue;
            const unsigned long long slot = atomicAdd(nt, 1ull);
            titems[slot] = make_longlong4(x, s, e, 0);
            continue;
        }
        if (d <= wt) {
            const int64_t cnt = (e - s + PW - 1) / PW;
            int64_t my = 0;
            for (int64_t i = 0; i < cnt; ++i) my += mine(x, i);
            if (my == 0) continue;
            unsigned long long base = atomicAdd(nw, (unsigned long long)my);
            for (int64_t i = 0; i < cnt; ++i) {
                if (!mine(x, i)) continue;
                const int64_t p0 = s + i * PW;
                witems[base++] = make_longlong4(x, p0, min(p0 + PW, e), 0);
            }
            continue;
        }
        // fewest range groups G (power of two <= F) whose slices all fit HC
        const int* sx = split + x * (F + 1);
        int lg = 0;
        if (d > hc) {
            for (lg = 1; lg < LOG_F; ++lg) {
                const int step = F >> lg;
                int mx = 0;
                for (int q = 0; q < F; q += step) mx = max(mx, sx[q + step] - sx[q]);
                if (mx <= hc) break;
            }
        }
        TCB_DASSERT(sx[0] == 0 && sx[F] == int(d));
        const int G = 1 << lg;
        const int64_t per = (e - s + PC - 1) / PC;
        int64_t my = 0;
        for (int64_t i = 0; i < per; ++i) my += mine(x, i);
        if (my == 0) continue;
        unsigned long long base = atomicAdd(nc, (unsigned long long)(my * G));
        for (int g = 0; g < G; ++g)
            for (int64_t i = 0; i < per; ++i) {
                if (!mine(x, i)) continue;
                const int64_t p0 = s + i * PC;
                citems[base++] = make_longlong4(x, p0, min(p0 + PC, e), (lg << 8) | g);
            }
    }
}

// ---------------------------------------------------------------------------
// 3b. thread tier: one thread per tiny owner (d(x) <= TINY, so every partner
//     has <= TINY ids too).  N(x) sits in registers; each partner id is
//     compared with all of it; the level is gathered only on a hit.

__global__ void __launch_bounds__(256)
    k_isect_tiny(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                 const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                 const int32_t* __restrict__ P, const int32_t* __restrict__ level,
                 DevCounters* C, const int2* __restrict__ vinfo, int fwd) {
    const int64_t nitems = int64_t(*nitems_p);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    uint32_t nh = 0, ns = 0;
    for (int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; it < nitems; it += stride) {
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int64_t xb = row[x];
        const int xd = int(row[x + 1] - xb);
        const int lx = level[x];
        int a[TINY];
#pragma unroll
        for (int i = 0; i < TINY; ++i) a[i] = i < xd ? nb[xb + i] : -1;
        for (int64_t p = item.y; p < item.z; ++p) {
            const int y = P[p];
            const int64_t yb = row[y];
            const int yd = int(row[y + 1] - yb);
            for (int j = 0; j < yd; ++j) {
                const int w = nb[yb + j];
                bool hit = false;
#pragma unroll
                for (int i = 0; i < TINY; ++i) hit |= a[i] == w;
                if (hit && staged(vinfo, w, x, xd, fwd)) {
                    nh += 1;
                    ns += level[w] == lx;
                }
            }
        }
    }
    Tally tl;
    tl.c1 = nh - ns;
    tl.c2 = ns;
    tl.flush(C);
}

// ---------------------------------------------------------------------------
// 4. warp tier

__global__ void __launch_bounds__(W_WARPS * 32, 4)
    k_isect_warp(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                 const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                 const int32_t* __restrict__ P, const int32_t* __restrict__ level,
                 unsigned long long* fetch, DevCounters* C, const int2* __restrict__ vinfo,
                 int fwd) {
    extern __shared__ uint4 smem4[];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem4) + warp * W_SLOTS;
    for (int i = lane; i < W_SLOTS; i += 32) tab[i] = EMPTY;
    __syncwarp();
    const unsigned long long nitems = *nitems_p;
    Tally tl;
    while (true) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(fetch, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int64_t xb = row[x];
        const int xd = int(row[x + 1] - xb);
        const int lx = level[x];
        const int slots = max(16, 2 << ceil_log2_dev(xd));
        BucketHash h;
        h.setup(tab, slots);
        for (int i = lane; i < xd; i += 32) {
            const int w = nb[xb + i];
            if (staged(vinfo, w, x, xd, fwd)) h.insert(w, level[w] == lx);
        }
        __syncwarp();
        for (int64_t pb = item.y; pb < item.z; pb += 32) {
            const int64_t j = pb + lane;
            int64_t ys = 0;
            int yd = 0;
            if (j < item.z) {
                const int y = P[j];
                ys = row[y];
                yd = int(row[y + 1] - ys);
            }
            probe_batch(nb, ys, yd, h, tl);
        }
        __syncwarp();
        for (int i = lane; i < slots; i += 32) tab[i] = EMPTY;
        __syncwarp();
    }
    tl.flush(C);
}

// ---------------------------------------------------------------------------
// 5. CTA tier

// A chunk that crosses slice boundaries: each lane walks forward from the
// chunk's first partner k0; a lane crosses a boundary in few of its J
// elements.  FULL: the chunk holds CHUNK elements (no bounds checks).
template <bool FULL, typename Probe>
__device__ __forceinline__ void cross_chunk(const int32_t* __restrict__ nb, const int64_t* s_ys,
                                            const int* s_off, int np, int k0, int c0, int c1,
                                            const Probe& h, uint32_t& co, uint32_t& cs) {
    constexpr int J = CHUNK / 32;
    int k = k0;
    int next = s_off[k + 1];
    const int32_t* q = nb + s_ys[k];
    const int i0 = c0 + int(lane_id());
    int w[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int i = i0 + 32 * j;
        w[j] = -1;
        if (FULL || i < c1) {
            if (next <= i) {
                do {
                    TCB_DASSERT(k + 1 < np);
                    ++k;
                    next = s_off[k + 1];
                } while (next <= i);
                q = nb + s_ys[k];
            }
#ifdef TCB_NOLOAD  // measurement-only variant: probe without streaming
            w[j] = int((uint32_t(i) * 2654435761u) >> 8) + int(reinterpret_cast<uintptr_t>(q) & 1);
#else
            w[j] = q[i];
#endif
        }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
        if (!FULL && w[j] < 0) continue;
        h.count(w[j], co, cs);
    }
}

// Warps consume the flattened stream of partner slices in CHUNK grabs;
// element i belongs to partner k with s_off[k] <= i < s_off[k+1].  The
// partner of a chunk's first element is found with two 32-way ballots over
// s_off (np <= 1024); a chunk that lies inside one slice (the common case:
// slices average hundreds of ids) takes a warp-uniform fast path with
// coalesced loads and no per-element partner bookkeeping.
template <typename Probe>
__device__ __forceinline__ void stream_chunks(const int32_t* __restrict__ nb, const int64_t* s_ys,
                                              const int* s_off, int np,
                                              int* s_next, const Probe& h, Tally& tl) {
    constexpr int J = CHUNK / 32;
    const int total = s_off[np];
    TCB_DASSERT(np >= 1 && np <= PC && total >= 0);
    const int lane = int(lane_id());
    while (true) {
        int c0 = 0;
        if (lane == 0) c0 = atomicAdd(s_next, CHUNK);
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        if (c0 >= total) break;
        const int c1 = min(total, c0 + CHUNK);
        // k0 = largest k with s_off[k] <= c0  (s_off[0] = 0 <= c0)
        int k0;
        {
            const int j = lane * 32;
            const unsigned b1 = __ballot_sync(0xffffffffu, j < np && s_off[j] <= c0);
            const int kb = 31 - __clz(b1);
            const int j2 = kb * 32 + lane;
            const unsigned b2 = __ballot_sync(0xffffffffu, j2 < np && s_off[j2] <= c0);
            k0 = kb * 32 + 31 - __clz(b2);
        }
        TCB_DASSERT(k0 >= 0 && k0 < np);
        // per-chunk tallies: apexes on another level / on the owner's level
        uint32_t co = 0, cs = 0;
        if (s_off[k0 + 1] >= c1) {
            // fast path: one partner slice
            const int32_t* p = nb + s_ys[k0] + c0 + lane;
            int w[J];
            if (c1 - c0 == CHUNK) {
#ifdef TCB_NOLOAD
#pragma unroll
                for (int j = 0; j < J; ++j)
                    w[j] = int((uint32_t(c0 + lane + 32 * j) * 2654435761u) >> 8) +
                           int(reinterpret_cast<uintptr_t>(p) & 1);
#else
#pragma unroll
                for (int j = 0; j < J; ++j) w[j] = p[32 * j];
#endif
#pragma unroll
                for (int j = 0; j < J; ++j) h.count(w[j], co, cs);
            } else {
#pragma unroll
                for (int j = 0; j < J; ++j) w[j] = c0 + lane + 32 * j < c1 ? p[32 * j] : -1;
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    if (w[j] < 0) continue;
                    h.count(w[j], co, cs);
                }
            }
        } else if (c1 - c0 == CHUNK) {
            cross_chunk<true>(nb, s_ys, s_off, np, k0, c0, c1, h, co, cs);
        } else {
            cross_chunk<false>(nb, s_ys, s_off, np, k0, c0, c1, h, co, cs);
        }
        tl.c1 += co;
        tl.c2 += cs;
    }
}

// Exclusive block scan of the per-partner lengths (thread t holds partners
// 2t, 2t+1) into s_off[0..np]; s_off[np] = stream length.  s_ys[k] becomes
// the stream base of partner k: stream element i of its slice is nb[s_ys[k] + i].
__device__ __forceinline__ void scan_lengths(int* s_off, int64_t* s_ys, int np, int64_t* s_tmp) {
    __syncthreads();  // lengths were written with a different thread->partner map
    const int t = threadIdx.x;
    const int a = 2 * t < np ? s_off[2 * t] : 0;
    const int b = 2 * t + 1 < np ? s_off[2 * t + 1] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan<C_THREADS>(int64_t(a + b), s_tmp, tot);
    if (2 * t < np) {
        s_off[2 * t] = int(ex);
        s_ys[2 * t] -= ex;
    }
    if (2 * t + 1 < np) {
        s_off[2 * t + 1] = int(ex + a);
        s_ys[2 * t + 1] -= ex + a;
    }
    if (t == 0) s_off[np] = int(tot);
    __syncthreads();
}

#ifndef TCB_CTA_PER_SM
#define TCB_CTA_PER_SM 2
#endif
__global__ void __launch_bounds__(C_THREADS, TCB_CTA_PER_SM)
    k_isect_cta(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                const int32_t* __restrict__ P, const int32_t* __restrict__ level,
                const int* __restrict__ split, unsigned long long* fetch, DevCounters* C,
                int hc, int dbg, const int2* __restrict__ vinfo, int fwd) {
    extern __shared__ uint4 smem4[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem4);           // C_SLOTS
    int64_t* s_ys = reinterpret_cast<int64_t*>(tab + C_SLOTS);    // PC
    int* s_off = reinterpret_cast<int*>(s_ys + PC);               // PC + 1
    int* s_end = s_off + PC + 1;                                  // PC (sub-chunk cursors)
    __shared__ int64_t s_tmp[C_THREADS / 32 + 1];
    __shared__ unsigned long long s_item;
    __shared__ int s_next;
    __shared__ int s_fail;
    const unsigned long long nitems = *nitems_p;
    Tally tl;
    while (true) {
        if (threadIdx.x == 0) s_item = atomicAdd(fetch, 1ull);
        __syncthreads();
        const unsigned long long it = s_item;
        if (it >= nitems) break;
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int lg = int(item.w >> 8), g = int(item.w & 255);
        const int q0 = (g << LOG_F) >> lg, q1 = ((g + 1) << LOG_F) >> lg;  // ranges [q0, q1)
        const int64_t xrow = row[x];
        const int* sx = split + int64_t(x) * (F + 1);
        const int64_t xs = xrow + (lg ? sx[q0] : 0);
        const int64_t xe = lg ? xrow + sx[q1] : row[x + 1];
        const int lx = level[x];
        const int dx = int(row[x + 1] - xrow);
        const int np = int(item.z - item.y);
        // partner slices for ranges [q0, q1) (the whole list when lg == 0)
        for (int t = threadIdx.x; t < np; t += C_THREADS) {
            const int y = P[item.y + t];
            const int64_t yb = row[y];
            int a = 0, b;
            if (lg) {
                const int* sy = split + int64_t(y) * (F + 1);
                a = sy[q0];
                b = sy[q1];
            } else {
                b = int(row[y + 1] - yb);
            }
            s_ys[t] = yb + a;
            TCB_DASSERT(0 <= a && a <= b && b <= int(row[y + 1] - yb));
            s_end[t] = b - a;  // slice length; consumed below
        }
        // stage the owner slice in sub-chunks of hc ids (one pass unless the
        // slice still exceeds hc with every range split — the largest hubs)
        for (int64_t cb = xs; cb < xe; cb += hc) {
            const int len = int(min(int64_t(hc), xe - cb));
            TCB_DASSERT(len >= 1 && len <= HC && xs >= row[x] && xe <= row[x + 1]);
            const bool single = (cb == xs) && (cb + len >= xe);
            const int slots = TCB_FULLTAB ? C_SLOTS : 4 << ceil_log2_dev(max(len, 4));
            BucketHash h;
            h.setup(tab, slots);
            TCB_DASSERT(slots <= C_SLOTS && np <= PC);
            for (int i = threadIdx.x; i < slots; i += C_THREADS) tab[i] = EMPTY;
            if (threadIdx.x == 0) s_next = 0;
            __syncthreads();
            CuckooHash ch;
            ch.setup(tab, slots);
            if (TCB_CUCKOO && threadIdx.x == 0) s_fail = 0;
            if (TCB_CUCKOO) __syncthreads();
            if (!(dbg & 2))
                for (int i = threadIdx.x; i < len; i += C_THREADS) {
                    const int w = nb[cb + i];
                    if (!staged(vinfo, w, x, dx, fwd)) continue;
                    if (TCB_CUCKOO) {
                        if (!ch.insert(w, level[w] == lx)) s_fail = 1;
                    } else {
                        h.insert(w, level[w] == lx);
                    }
                }
            if (single) {
                for (int t = threadIdx.x; t < np; t += C_THREADS) s_off[t] = s_end[t];
            } else {
                // sub-chunk [vlo, vhi] of the owner slice: each partner's
                // matching part starts where its previous part ended
                const int vhi = nb[cb + len - 1];
                const bool last = cb + len >= xe;
                for (int t = threadIdx.x; t < np; t += C_THREADS) {
                    int64_t a = s_ys[t];
                    const int64_t e = a + s_end[t];
                    int64_t lo = a, hi = e;
                    if (!last)
                        while (lo < hi) {
                            const int64_t mid = (lo + hi) >> 1;
                            if (nb[mid] <= vhi) lo = mid + 1; else hi = mid;
                        }
                    else
                        lo = e;
                    s_off[t] = int(lo - a);
                }
            }
            scan_lengths(s_off, s_ys, np, s_tmp);  // ends with __syncthreads
            if (TCB_CUCKOO && s_fail) {  // rare: rebuild this sub-chunk as a bucket table
                for (int i = threadIdx.x; i < slots; i += C_THREADS) tab[i] = EMPTY;
                __syncthreads();
                for (int i = threadIdx.x; i < len; i += C_THREADS) {
                    const int w = nb[cb + i];
                    if (staged(vinfo, w, x, dx, fwd)) h.insert(w, level[w] == lx);
                }
                __syncthreads();
            }
            if (!(dbg & 1)) {
                if (TCB_CUCKOO && !s_fail) {
                    stream_chunks(nb, s_ys, s_off, np, &s_next, ch, tl);
                } else {
                    stream_chunks(nb, s_ys, s_off, np, &s_next, h, tl);
                }
            }
            __syncthreads();
            if (!single) {  // advance partner starts past this sub-chunk
                for (int t = threadIdx.x; t < np; t += C_THREADS) {
                    s_ys[t] += s_off[t + 1];  // stream base -> next unread id
                    s_end[t] -= s_off[t + 1] - s_off[t];
                }
                __syncthreads();
            }
        }
        // an item whose owner slice is empty runs no sub-chunk: without this
        // barrier thread 0 could overwrite s_item before all threads read it
        __syncthreads();
    }
    tl.flush(C);
}

// ---------------------------------------------------------------------------

// TCB_DBG bit flags disable parts of the CTA tier (checked builds only)
static int debug_flags() {
#ifdef TCB_CHECKS
    const char* e = getenv("TCB_DBG");
    return e ? atoi(e) : 0;
#else
    return 0;
#endif
}

struct IsectKernels {
    int warp_blocks = 0, cta_blocks = 0;
};
static IsectKernels g_k[16];

void cetc_intersect_owner(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                          const int32_t* level, int64_t n, int64_t m, int shard, int nshards,
                          int fwd) {
    if (n == 0 || m == 0) return;
    DevCounters* C = ctx->d_counters;
    const int64_t nnz = 2 * m;
    int2* vinfo = ctx->wsT<int2>(WS_MISC, n);
    int32_t* P = ctx->wsT<int32_t>(WS_COVER_U, m);
    int64_t* seg = ctx->wsT<int64_t>(WS_COUNT_TMP, 2 * n);
    int* split = ctx->wsT<int>(WS_COVER_V, size_t(n) * (F + 1));
    // tuning knobs (tcb_set_tuning; tests shrink them to reach every path)
    const int wt = ctx->tune_wt > 0 ? min(ctx->tune_wt, WT) : WT;
    const int hc = ctx->tune_hc > 0 ? max(4, min(ctx->tune_hc, HC)) : HC;
    const int tiny = min(TINY, wt);
    const int64_t wcap = n + m / PW + 1;
    const int64_t ccap = (2 * m / (wt + 1) + 2 + m / PC) * F;
    longlong4* items = ctx->wsT<longlong4>(WS_BINS, wcap + ccap + n + 1);
    longlong4* witems = items;
    longlong4* citems = items + wcap;
    longlong4* titems = citems + ccap;
    unsigned long long* nt = &C->scratch[9];
    unsigned long long* nw = &C->scratch[5];
    unsigned long long* nc = &C->scratch[6];
    unsigned long long* fw = &C->scratch[7];
    unsigned long long* fc = &C->scratch[8];
    int64_t* d_ncover = reinterpret_cast<int64_t*>(&C->ncover);
    const int rshift = max(0, bits_for(n) - LOG_F);

    TCB_LAUNCH(ctx, k_vinfo, grid_for(ctx, n, 256), 256, 0, row, level, n, vinfo);
    owner_select(ctx, row, src, nb, vinfo, nnz, P, seg, seg + n, d_ncover);
    ctx->record(3);
    TCB_LAUNCH(ctx, k_split_points, grid_for(ctx, nnz, 256), 256, 0, row, src, nb, nnz, rshift,
               split);
    TCB_LAUNCH(ctx, k_make_items, grid_for(ctx, n, 256), 256, 0, row, (const int64_t*)seg,
               (const int64_t*)(seg + n), (const int*)split, n, witems, citems, titems, nw, nc,
               nt, shard, nshards, wt, hc, tiny);

    IsectKernels& K = g_k[ctx->device & 15];
    const size_t wsm = size_t(W_WARPS) * W_SLOTS * sizeof(uint32_t);
    const size_t csm = size_t(C_SLOTS) * sizeof(uint32_t) + size_t(PC) * sizeof(int64_t) +
                       size_t(2 * PC + 1) * sizeof(int);
    if (K.warp_blocks == 0) {
        TCB_CUDA(cudaFuncSetAttribute(k_isect_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(wsm)));
        TCB_CUDA(cudaFuncSetAttribute(k_isect_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(csm)));
        int a = 0, b = 0;
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_isect_warp, W_WARPS * 32, wsm));
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_isect_cta, C_THREADS, csm));
        require(a > 0 && b > 0, "intersection kernels do not fit on an SM");
        K.warp_blocks = a * ctx->num_sms;
        K.cta_blocks = b * ctx->num_sms;
    }
    ctx->record(5);
    ctx->record(7);  // no separate hub kernel in this design: hub stage = 0
    TCB_LAUNCH(ctx, k_isect_cta, K.cta_blocks, C_THREADS, csm, (const longlong4*)citems,
               (const unsigned long long*)nc, row, nb, (const int32_t*)P, level,
               (const int*)split, fc, C, hc, debug_flags(), (const int2*)vinfo, fwd);
    ctx->record(6);
    TCB_LAUNCH(ctx, k_isect_warp, K.warp_blocks, W_WARPS * 32, wsm, (const longlong4*)witems,
               (const unsigned long long*)nw, row, nb, (const int32_t*)P, level, fw, C,
               (const int2*)vinfo, fwd);
    TCB_LAUNCH(ctx, k_isect_tiny, ctx->num_sms * 8, 256, 0, (const longlong4*)titems,
               (const unsigned long long*)nt, row, nb, (const int32_t*)P, level, C,
               (const int2*)vinfo, fwd);
}

}  // namespace tcb

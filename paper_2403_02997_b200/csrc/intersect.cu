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
// its higher-degree endpoint x (ties: lower id).  x's list is staged ONCE in
// shared memory and every partner y's list (the shorter one) is streamed past
// it: sum_S min(d(u), d(v)) probes (10x fewer at RMAT-24) plus
// sum over owners of d(x) inserts (<1% of that).
//
//  1. owner_select: ordered compaction over the CSR entries (x, y) keeping
//     level[x]==level[y] && owns(x, y).  Entries are in row order, so each
//     owner's partners come out contiguous: P[seg_beg[x], seg_end[x]).
//  2. make_items: owners with d(x) <= WT become warp items (x, p0, p1) with
//     <= PW partners; larger owners become CTA items with <= PC partners.
//  3. k_isect_warp: one warp per item; per-warp bucketed hash of N(x).
//  4. k_isect_cta: one CTA per item.  d(x) <= HC: bucketed hash of N(x)
//     (load <= 1/4).  d(x) > HC (hubs): N(x) is staged as a bitmap of one id
//     range of R ids at a time; every partner keeps a cursor into its own list
//     across ranges, so each partner element is read once per item.
//
// Hash entries carry the apex's level relation to the owner in bit 31
// (same level -> c2 candidate), so hits need no level gather.  Buckets are 4
// entries (one LDS.128 per probe); linear probing over buckets.  Partners are
// handed to warps dynamically; a long partner list is streamed by the whole
// warp with 4 loads in flight per lane, short ones are flattened across lanes
// (warp scan of lengths + shuffle search).  Tallies reduce per warp into one
// 64-bit atomic each.
#include "common.cuh"
#include "scan.cuh"

namespace tcb {

constexpr int WT = 1024;              // warp tier: owner degree <= WT
constexpr int W_SLOTS = 2 * WT;       // per-warp table: load <= 1/2
constexpr int W_WARPS = 8;
constexpr int PW = 64;                // partners per warp item
constexpr int C_THREADS = 1024;
constexpr int C_WARPS = C_THREADS / 32;
constexpr int HC = 8192;              // CTA hash tier: owner degree <= HC
constexpr int C_SLOTS = 4 * HC;       // load <= 1/4 (128 KB)
constexpr int R_BITS = 20;            // hub tier: id range per bitmap pass
constexpr int R_WORDS = (1 << R_BITS) / 32;  // 128 KB
constexpr int C_TAB_WORDS = C_SLOTS > R_WORDS ? C_SLOTS : R_WORDS;
constexpr int PC = 2048;              // partners per CTA item
constexpr int LONG_LIST = 64;         // partner lists streamed by a whole warp
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
        return shift >= 32 ? 0u : ((unsigned(key) * 0x9E3779B1u) >> shift);
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
    // 0 = miss, 1 = hit other level, 2 = hit same level
    __device__ __forceinline__ int find(int key) const {
        unsigned b = bucket(key);
        while (true) {
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

struct Tally {
    unsigned long long c1 = 0, c2 = 0, t = 0;
    // r: 1 = apex on another level, 2 = apex on the owner's level
    __device__ __forceinline__ void add(int r, int w, int vmax) {
        if (r == 1) {
            c1++;
            t++;
        } else if (r == 2) {
            c2++;
            t += (w > vmax);
        }
    }
    __device__ __forceinline__ void flush(DevCounters* C) {
        c1 = warp_sum(c1);
        c2 = warp_sum(c2);
        t = warp_sum(t);
        if (lane_id() == 0) {
            if (c1) atomicAdd(&C->c1, c1);
            if (c2) atomicAdd(&C->c2, c2);
            if (t) atomicAdd(&C->t, t);
        }
    }
};

// Membership test against whichever staged structure the item uses.
struct HashProbe {
    BucketHash h;
    __device__ __forceinline__ int operator()(int w) const { return h.find(w); }
};
struct BitmapProbe {
    const uint32_t* bits;
    const int32_t* level;
    int lo, lx;
    __device__ __forceinline__ int operator()(int w) const {
        const unsigned off = unsigned(w - lo);
        if (off >= (1u << R_BITS)) return 0;  // element of a skipped (empty) range
        if (!((bits[off >> 5] >> (off & 31)) & 1u)) return 0;
        return level[w] == lx ? 2 : 1;
    }
};

// Stream one long list [s, s+d) with the whole warp, 4 loads in flight/lane.
template <typename Probe>
__device__ __forceinline__ void probe_long(const int32_t* __restrict__ nb, int64_t s, int d,
                                           int vmax, const Probe& probe, Tally& tl) {
    const int lane = int(lane_id());
    int i = lane;
    for (; i + 96 < d; i += 128) {
        const int w0 = nb[s + i], w1 = nb[s + i + 32], w2 = nb[s + i + 64], w3 = nb[s + i + 96];
        tl.add(probe(w0), w0, vmax);
        tl.add(probe(w1), w1, vmax);
        tl.add(probe(w2), w2, vmax);
        tl.add(probe(w3), w3, vmax);
    }
    for (; i < d; i += 32) {
        const int w = nb[s + i];
        tl.add(probe(w), w, vmax);
    }
}

// Batch of <= 32 partner lists (lane j: [ys_j, ys_j + yd_j), tie vertex vmax_j).
// Long lists go one at a time through probe_long; the short remainder is
// flattened across the lanes.
template <typename Probe>
__device__ __forceinline__ void probe_batch(const int32_t* __restrict__ nb, int64_t ys, int yd,
                                            int vmax, const Probe& probe, Tally& tl) {
    const unsigned lane = lane_id();
    unsigned longs = __ballot_sync(0xffffffffu, yd >= LONG_LIST);
    while (longs) {
        const int k = __ffs(longs) - 1;
        longs &= longs - 1;
        probe_long(nb, __shfl_sync(0xffffffffu, ys, k), __shfl_sync(0xffffffffu, yd, k),
                   __shfl_sync(0xffffffffu, vmax, k), probe, tl);
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
        const int vm = __shfl_sync(0xffffffffu, vmax, k);
        if (i < total) {
            const int w = nb[ysk + (i - exk)];
            tl.add(probe(w), w, vm);
        }
    }
}

// ---------------------------------------------------------------------------
// 1. owner-grouped selection

void owner_select(Context* ctx, const int64_t* row, const int32_t* src, const int32_t* nb,
                  const int2* vinfo, int64_t nnz, int32_t* P, int64_t* seg_beg, int64_t* seg_end,
                  int64_t* d_ncover) {
    scan_apply(
        ctx, nnz,
        [src, nb, vinfo] __device__(int64_t e) -> int64_t {
            const int x = src[e], y = nb[e];
            const int2 a = vinfo[x], b = vinfo[y];
            return (a.x == b.x && (a.y > b.y || (a.y == b.y && x < y))) ? 1 : 0;
        },
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
// 2. work items

__global__ void k_make_items(const int64_t* __restrict__ row, const int64_t* __restrict__ seg_beg,
                             const int64_t* __restrict__ seg_end, int64_t n,
                             longlong4* __restrict__ witems, longlong4* __restrict__ citems,
                             unsigned long long* nw, unsigned long long* nc, int shard,
                             int nshards) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < n; x += stride) {
        if (nshards > 1 && int(x % nshards) != shard) continue;  // owners shard by id
        const int64_t d = row[x + 1] - row[x];
        if (d == 0) continue;
        const int64_t s = seg_beg[x], e = seg_end[x];
        if (e <= s) continue;
        const int64_t per = d <= WT ? PW : PC;
        const int64_t cnt = (e - s + per - 1) / per;
        unsigned long long base = atomicAdd(d <= WT ? nw : nc, (unsigned long long)cnt);
        longlong4* out = d <= WT ? witems : citems;
        for (int64_t i = 0; i < cnt; ++i) {
            const int64_t p0 = s + i * per;
            const int64_t p1 = p0 + per < e ? p0 + per : e;
            out[base + i] = make_longlong4(x, p0, p1, 0);
        }
    }
}

// ---------------------------------------------------------------------------
// 3. warp tier

__global__ void __launch_bounds__(W_WARPS * 32)
    k_isect_warp(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                 const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                 const int32_t* __restrict__ P, const int32_t* __restrict__ level,
                 unsigned long long* fetch, DevCounters* C) {
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
        HashProbe probe;
        probe.h.setup(tab, slots);
        for (int i = lane; i < xd; i += 32) {
            const int w = nb[xb + i];
            probe.h.insert(w, level[w] == lx);
        }
        __syncwarp();
        for (int64_t pb = item.y; pb < item.z; pb += 32) {
            const int64_t j = pb + lane;
            int64_t ys = 0;
            int yd = 0, vmax = 0;
            if (j < item.z) {
                const int y = P[j];
                ys = row[y];
                yd = int(row[y + 1] - ys);
                vmax = max(x, y);
            }
            probe_batch(nb, ys, yd, vmax, probe, tl);
        }
        __syncwarp();
        for (int i = lane; i < slots; i += 32) tab[i] = EMPTY;
        __syncwarp();
    }
    tl.flush(C);
}

// ---------------------------------------------------------------------------
// 4. CTA tier

__global__ void __launch_bounds__(C_THREADS, 1)
    k_isect_cta(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                const int32_t* __restrict__ P, const int32_t* __restrict__ level,
                unsigned long long* fetch, DevCounters* C) {
    extern __shared__ uint4 smem4[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem4);    // C_TAB_WORDS
    int* cursor = reinterpret_cast<int*>(tab + C_TAB_WORDS);  // PC
    __shared__ unsigned long long s_item;
    __shared__ int s_next;
    const unsigned lane = lane_id();
    const unsigned long long nitems = *nitems_p;
    Tally tl;
    while (true) {
        if (threadIdx.x == 0) {
            s_item = atomicAdd(fetch, 1ull);
            s_next = 0;
        }
        __syncthreads();
        const unsigned long long it = s_item;
        if (it >= nitems) break;
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int64_t xb = row[x], xe = row[x + 1];
        const int xd = int(xe - xb);
        const int lx = level[x];
        const int np = int(item.z - item.y);
        if (xd <= HC) {
            // ---- hash tier: whole N(x) staged once
            const int slots = 4 << ceil_log2_dev(xd);
            HashProbe probe;
            probe.h.setup(tab, slots);
            for (int i = threadIdx.x; i < slots; i += C_THREADS) tab[i] = EMPTY;
            __syncthreads();
            for (int i = threadIdx.x; i < xd; i += C_THREADS) {
                const int w = nb[xb + i];
                probe.h.insert(w, level[w] == lx);
            }
            __syncthreads();
            while (true) {  // warps grab 32-partner batches
                int q0 = 0;
                if (lane == 0) q0 = atomicAdd(&s_next, 32);
                q0 = __shfl_sync(0xffffffffu, q0, 0);
                if (q0 >= np) break;
                const int q = q0 + int(lane);
                int64_t ys = 0;
                int yd = 0, vmax = 0;
                if (q < np) {
                    const int y = P[item.y + q];
                    ys = row[y];
                    yd = int(row[y + 1] - ys);
                    vmax = max(x, y);
                }
                probe_batch(nb, ys, yd, vmax, probe, tl);
            }
        } else {
            // ---- hub tier: one id range [lo, lo + 2^R_BITS) of N(x) at a time
            for (int i = threadIdx.x; i < np; i += C_THREADS) cursor[i] = 0;
            int64_t xc = xb;  // first entry of N(x) in the current range
            while (xc < xe) {
                const int lo = nb[xc] & ~((1 << R_BITS) - 1);
                const int64_t hi_excl = int64_t(lo) + (1 << R_BITS);
                // end of this range within N(x): gallop + binary search
                int64_t a = xc, step = 1;
                while (a + step - 1 < xe && nb[a + step - 1] < hi_excl) {
                    a += step;
                    step <<= 1;
                }
                int64_t bnd = a + step - 1 < xe ? a + step - 1 : xe;
                while (a < bnd) {
                    const int64_t mid = (a + bnd) >> 1;
                    if (nb[mid] < hi_excl) a = mid + 1; else bnd = mid;
                }
                const int64_t xr = a;
                const bool last = xr >= xe;
                for (int i = threadIdx.x; i < R_WORDS; i += C_THREADS) tab[i] = 0u;
                __syncthreads();
                for (int64_t i = xc + threadIdx.x; i < xr; i += C_THREADS) {
                    const unsigned off = unsigned(nb[i] - lo);
                    atomicOr(&tab[off >> 5], 1u << (off & 31));
                }
                if (threadIdx.x == 0) s_next = 0;
                __syncthreads();
                BitmapProbe probe{tab, level, lo, lx};
                while (true) {
                    int q0 = 0;
                    if (lane == 0) q0 = atomicAdd(&s_next, 32);
                    q0 = __shfl_sync(0xffffffffu, q0, 0);
                    if (q0 >= np) break;
                    const int q = q0 + int(lane);
                    int64_t ys = 0;
                    int yd = 0, vmax = 0;
                    if (q < np) {
                        const int y = P[item.y + q];
                        const int64_t yb = row[y], ye = row[y + 1];
                        vmax = max(x, y);
                        ys = yb + cursor[q];
                        int64_t end = ye;
                        if (!last) {  // first position with value >= hi_excl
                            int64_t l2 = ys, st = 1;
                            while (l2 + st - 1 < ye && nb[l2 + st - 1] < hi_excl) {
                                l2 += st;
                                st <<= 1;
                            }
                            int64_t h2 = l2 + st - 1 < ye ? l2 + st - 1 : ye;
                            while (l2 < h2) {
                                const int64_t mid = (l2 + h2) >> 1;
                                if (nb[mid] < hi_excl) l2 = mid + 1; else h2 = mid;
                            }
                            end = l2;
                        }
                        yd = int(end - ys);
                        cursor[q] = int(end - yb);
                    }
                    probe_batch(nb, ys, yd, vmax, probe, tl);
                }
                __syncthreads();
                xc = xr;
            }
        }
        __syncthreads();
    }
    tl.flush(C);
}

// ---------------------------------------------------------------------------

struct IsectKernels {
    int warp_blocks = 0, cta_blocks = 0;
};
static IsectKernels g_k[16];

void cetc_intersect_owner(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                          const int32_t* level, int64_t n, int64_t m, int shard, int nshards) {
    if (n == 0 || m == 0) return;
    DevCounters* C = ctx->d_counters;
    const int64_t nnz = 2 * m;
    int2* vinfo = ctx->wsT<int2>(WS_MISC, n);
    int32_t* P = ctx->wsT<int32_t>(WS_COVER_U, m);
    int64_t* seg = ctx->wsT<int64_t>(WS_COUNT_TMP, 2 * n);
    const int64_t wcap = n + m / PW + 1, ccap = 2 * m / WT + 1 + m / PC + 1;
    longlong4* items = ctx->wsT<longlong4>(WS_BINS, wcap + ccap);
    longlong4* witems = items;
    longlong4* citems = items + wcap;
    unsigned long long* nw = &C->scratch[5];
    unsigned long long* nc = &C->scratch[6];
    unsigned long long* fw = &C->scratch[7];
    unsigned long long* fc = &C->scratch[8];
    int64_t* d_ncover = reinterpret_cast<int64_t*>(&C->ncover);

    TCB_LAUNCH(ctx, k_vinfo, grid_for(ctx, n, 256), 256, 0, row, level, n, vinfo);
    owner_select(ctx, row, src, nb, vinfo, nnz, P, seg, seg + n, d_ncover);
    ctx->record(3);
    TCB_LAUNCH(ctx, k_make_items, grid_for(ctx, n, 256), 256, 0, row, (const int64_t*)seg,
               (const int64_t*)(seg + n), n, witems, citems, nw, nc, shard, nshards);

    IsectKernels& K = g_k[ctx->device & 15];
    const size_t wsm = size_t(W_WARPS) * W_SLOTS * sizeof(uint32_t);
    const size_t csm = size_t(C_TAB_WORDS) * sizeof(uint32_t) + size_t(PC) * sizeof(int);
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
    TCB_LAUNCH(ctx, k_isect_cta, K.cta_blocks, C_THREADS, csm, (const longlong4*)citems,
               (const unsigned long long*)nc, row, nb, (const int32_t*)P, level, fc, C);
    TCB_LAUNCH(ctx, k_isect_warp, K.warp_blocks, W_WARPS * 32, wsm, (const longlong4*)witems,
               (const unsigned long long*)nw, row, nb, (const int32_t*)P, level, fw, C);
}

}  // namespace tcb

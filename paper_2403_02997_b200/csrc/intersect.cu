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
// streamed past it, so an edge costs at most min(d(u), d(v)) probes.
//
// The level rule is applied before the intersection instead of after it.
// Both endpoints are on level L, so an apex w is on another level from both
// (counted in c1) or on L for both.  Every CSR row is split into two lists:
//     OFF(v) = neighbours on another level (id-sorted),
//     UP(v)  = neighbours on v's level that rank above v in the owner order
//              (degree bucket floor(log2 d) desc, id asc), sorted in that
//              order (stable counting sort of the id-sorted row by bucket),
// and an edge (owner x, partner p) has apexes OFF(x)∩OFF(p) (c1) and
// UP(x)∩UP(p) (same level, ranked above both endpoints).  Every same-level
// triangle a > b > c (owner order) is therefore found exactly once, at its
// edge (b, c) with apex a — the reference keeps exactly one apex per such
// triangle too (w > max(u, v), _kernels.py:687) — so the UP tally equals
// the reference's T - c1 and its c2 (every same-level hit, 3 per triangle,
// _kernels.py:745-748) is 3 x this tally; the counters hold c2 in those
// units.  Ranking by degree keeps the same-level stream short: p streams
// only the part of UP(p) ranked above x — a prefix of the sorted list: the
// buckets above x's (ucnt table) plus the values below x in x's own bucket
// (one search per edge, Lists::up_cut, done for all edges of the CTA tier at
// once by k_edge_prep; a short bucket run is streamed whole) — and hubs have
// few neighbours above them.  (The bucket order streams within 1% of the ids
// the exact degree order would, and its sorted lists come from a counting
// sort.)  Same-level neighbours ranked below the endpoint are never read,
// and a hit needs no level lookup: the list it was streamed from says which
// tally it belongs to.
//
// UP lists hold RANKS, not ids: rank(v) = v's position in the owner order over
// all vertices (k_rank_*: one stable counting pass by degree bucket), stored
// with bit 31 set so no UP value equals an OFF id (the thread and warp tiers
// keep both classes in one set).  Counting needs equality only, the sorted
// UP list is then simply ascending, and everything ranked above an owner x
// lies in [0, rank(x)): for a CTA-tier owner (degree > 256) that is the few
// hundred thousand hubs, so UP(x) is staged as a BITMAP over [0, rank(x)] —
// one shared-memory read per streamed element, exact, no hashing and no kick
// chains (values at or below rank(x), the tail of an uncut run, are clamped
// to bit rank(x), which is never set) — while OFF(x) keeps the cuckoo set.
//
//  1. owner bits: a keep bit per CSR entry (x, y) with level[x]==level[y] &&
//     owns(x, y), and the OFF/UP class bits.  A word-level prefix of the keep
//     bits compacts the kept entries in row order, so each owner's partners
//     come out contiguous: P[seg_beg[x], seg_end[x]).
//  2. lists: word prefixes of the class bits give every entry its slot in
//     the OFF array and every row its UP range (no second scan); UP rows are
//     stably counting-sorted by degree bucket (per-row histogram, prefix,
//     scatter in row order), so each bucket's run is id-sorted.
//  3. split points: the id space is cut into F equal ranges; split[v][r] is
//     the position in OFF(v) of the first id in range r.  An owner whose OFF
//     list exceeds the table is staged one group of ranges at a time, and
//     every partner's matching slices are read from the table.
//  4. make_items: owners with d(x) <= TINY -> thread items; <= WT -> warp
//     items (x, p0, p1), <= PW partners each; others -> CTA items
//     (x, p0, p1, group), <= PC partners.  With nshards > 1 only this
//     shard's partner blocks are listed (dist.py shard_of).
//  4b. k_edge_prep: the 16-byte partner record of every cover edge of a
//     CTA-tier owner (list starts, OFF size, UP cut), a thread per slot of P.
//  5. k_isect_tiny / k_isect_warp: one thread / warp per item; the warp tier
//     keeps a per-warp cuckoo set of OFF(x) ∪ UP(x) (bucket table if a kick
//     chain fails).
//  6. k_isect_cta: one CTA per item; the group's slice of OFF(x) staged in a
//     two-table cuckoo set and, in group 0, UP(x) in a rank bitmap beside it;
//     the partners' slices (two per partner) are flattened into one element
//     stream (block scan of lengths; the UP part starts at a CHUNK multiple)
//     that warps consume in CHUNK-element grabs, each of one class.
//
// Forward mode (fwd, tcb_forward_count): every entry is classed OFF, owners
// stage only the neighbours ranked above them, and every hit is a triangle
// (tallied in c1).
#include "common.cuh"
#include "scan.cuh"

#include <cstdlib>
#include <type_traits>

namespace tcb {

// Tier thresholds and tile sizes.  The TCB_* macros exist so tools/variants.py
// can A/B alternatives in one GPU session; the defaults are the measured best.
#ifndef TCB_WT
#define TCB_WT 256
#endif
#ifndef TCB_HC
#define TCB_HC 6144
#endif
#ifndef TCB_CHUNK
#define TCB_CHUNK 1024
#endif
#ifndef TCB_PW
#define TCB_PW 64
#endif
constexpr int WT = TCB_WT;            // warp tier: owner degree <= WT
constexpr int W_SLOTS = 4 * WT;       // per-warp bucket table: load <= 1/4
constexpr int W_WARPS = 8;
constexpr int PW = TCB_PW;            // partners per warp item
#ifndef TCB_C_THREADS
#define TCB_C_THREADS 512
#endif
constexpr int C_THREADS = TCB_C_THREADS;  // 512: 2 CTAs per SM
constexpr int HC = TCB_HC;            // staged ids per CTA item
#ifndef TCB_C_SLOTS
#define TCB_C_SLOTS 16384
#endif
constexpr int C_SLOTS = TCB_C_SLOTS;  // cuckoo slots (64 KB): load <= HC / C_SLOTS = 3/8
#ifndef TCB_INSERT_U
#define TCB_INSERT_U 4
#endif
constexpr int INSERT_U = TCB_INSERT_U;  // staged ids loaded per thread before their inserts
constexpr int PC = 2 * C_THREADS;     // partners per CTA item
constexpr int NSEG = 2 * PC;          // stream slices: partner t -> OFF slice t, UP slice PC + t
constexpr int CHUNK = TCB_CHUNK;      // stream elements per warp grab (32 per lane)
constexpr int LOG_F = 5;
constexpr int F = 1 << LOG_F;         // id ranges for split points
constexpr int TINY = 16;              // thread tier: owner degree <= TINY
constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t UP_TAG = 0x80000000u;  // UP lists hold UP_TAG | rank (never EMPTY: rank < n < 2^31 - 1)
constexpr int PAD = -1;                   // padding key of a partial chunk (== EMPTY: never a value)
constexpr int NBKT = 32;
#ifndef TCB_UPCUT_ROUNDS
#define TCB_UPCUT_ROUNDS 2
#endif
constexpr int UPCUT_ROUNDS = TCB_UPCUT_ROUNDS;  // interpolation windows before the binary search
#ifndef TCB_UPCUT_SKIP
#define TCB_UPCUT_SKIP 64
#endif
constexpr int UPCUT_SKIP = TCB_UPCUT_SKIP;  // CTA tier: bucket runs up to this long are streamed whole
// Per-vertex partner record for the CTA tier: one 32-byte sector with the
// list starts, the OFF size and the UP prefix counts of the degree buckets
// CTA-tier owners have (|UP(v)| <= sqrt(2m) < 2^16 since 2m < 2^32).
constexpr int PR_K0 = 8, PR_NK = 10;  // buckets [8, 18): owner degrees 256 .. 2^18-1
struct __align__(32) PRec {
    uint32_t ob, ub, noff;
    uint16_t uc[PR_NK];
};
static_assert(sizeof(PRec) == 32, "one sector per partner");
constexpr int PR_FULL = 0xFFFF;  // uc entry too large for 16 bits: read ucnt              // degree buckets: floor(log2 d)
__device__ __forceinline__ int dbucket(int d) { return 31 - __clz(max(d, 1)); }

__device__ __forceinline__ int ceil_log2_dev(int x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// ---------------------------------------------------------------------------
// entry classes: bit i of cls[j].x / .y = CSR entry 32j+i is OFF / UP.
// pre[j] = exclusive prefix over words of popc(.x) | popc(.y) << 32, so an
// entry's slot in the OFF array (and a row's UP range) is a prefix read plus one popc.

__device__ __forceinline__ int64_t rank_off(const uint2* __restrict__ cls,
                                            const unsigned long long* __restrict__ pre,
                                            int64_t p) {
    const int64_t j = p >> 5;
    const uint32_t below = (1u << (p & 31)) - 1u;
    return int64_t(pre[j] & 0xFFFFFFFFull) + __popc(cls[j].x & below);
}
__device__ __forceinline__ int64_t rank_up(const uint2* __restrict__ cls,
                                            const unsigned long long* __restrict__ pre,
                                            int64_t p) {
    const int64_t j = p >> 5;
    const uint32_t below = (1u << (p & 31)) - 1u;
    return int64_t(pre[j] >> 32) + __popc(cls[j].y & below);
}

// ---------------------------------------------------------------------------
// bucketed hash set in shared memory (warp tier; CTA fallback)

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
    __device__ __forceinline__ void insert(int key) const {
        const uint32_t e = uint32_t(key);
        unsigned b = bucket(key);
        while (true) {
#pragma unroll
            for (int s = 0; s < 4; ++s)
                if (atomicCAS(&tab[4 * b + s], EMPTY, e) == EMPTY) return;
            b = (b + 1) & bmask;
        }
    }
    // two-step probe interface shared with CuckooHash (probe_all); a negative
    // key would match EMPTY, so callers skip padding keys
    static constexpr bool kNegSafe = false;
    __device__ __forceinline__ uint32_t first(int) const { return 0u; }
    __device__ __forceinline__ uint32_t second(int key, uint32_t) const { return hit(key); }
    // The first bucket is resolved without branches; the loop runs only when
    // that bucket is full and does not hold the key (rare at load <= 1/4).
    __device__ __forceinline__ uint32_t hit(int key) const {
        unsigned b = bucket(key);
        const uint32_t k = uint32_t(key);
        {
            const uint4 v = reinterpret_cast<const uint4*>(tab)[b];
            const bool h = (v.x == k) | (v.y == k) | (v.z == k) | (v.w == k);
            if (h || v.w == EMPTY) return h;
            b = (b + 1) & bmask;
        }
        while (true) {
            TCB_DASSERT(b <= bmask);
            const uint4 v = reinterpret_cast<const uint4*>(tab)[b];
            if ((v.x == k) | (v.y == k) | (v.z == k) | (v.w == k)) return 1;
            if (v.w == EMPTY) return 0;  // buckets fill in slot order
            b = (b + 1) & bmask;
        }
    }
};

// 2-choice cuckoo set over two half tables: a probe is two LDS.32 and two
// compares with no loop.  Parallel insertion by atomicExch kick chains; a
// chain longer than CUCKOO_KICKS reports failure and the caller falls back
// to the bucket table (rare at the CTA tier's load <= 3/8).
constexpr int CUCKOO_KICKS = 64;
constexpr uint32_t C_EMPTY = 0x7FFFFFFFu;  // cuckoo empty slot: never an id (ids < 2^31 - 1)

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
    __device__ __forceinline__ bool insert(int key) const {
        uint32_t e = uint32_t(key);
        uint32_t* slot = tab + h1(e);
        for (int it = 0; it < CUCKOO_KICKS; ++it) {
            const uint32_t old = atomicExch(slot, e);
            if (old == C_EMPTY) return true;
            e = old;  // carry the evicted key to its slot in the other table
            slot = slot < tab2 ? tab2 + h2(e) : tab + h1(e);
        }
        return false;
    }
    // Two-step probe (probe_all issues a batch of first() reads before any
    // second()).  C_EMPTY is never an id and a negative (padding) key never
    // matches a slot, so no guard is needed.
    static constexpr bool kNegSafe = true;
    __device__ __forceinline__ uint32_t first(int key) const { return tab[h1(uint32_t(key))]; }
    // Both reads are independent: a key sits in table 1 or table 2.  (A
    // table-1 flag telling which misses can skip table 2 cut shared-memory
    // wavefronts by a third, but the dependent second read made the kernel
    // 1.25-2x slower: DESIGN.md §8.)
    __device__ __forceinline__ uint32_t second(int key, uint32_t v) const {
        const uint32_t k = uint32_t(key);
        return (v == k) | (tab2[h2(k)] == k);
    }
    __device__ __forceinline__ uint32_t hit(int key) const { return second(key, first(key)); }
};

// c1 / same-level tallies.  `sup` counts UP∩UP hits: each all-horizontal
// triangle once, at the edge whose apex ranks above both endpoints (the
// reference keeps one of the three too, w > max(u, v)); the reference's c2
// counts every same-level hit, 3 per such triangle, so c2 = 3 sup over the
// cover set and T = c1 + c2/3 (formed in capi.cu fill_result).
struct Tally {
    unsigned long long c1 = 0, sup = 0;
    __device__ __forceinline__ void flush(DevCounters* C) {
        c1 = warp_sum(c1);
        sup = warp_sum(sup);
        if (lane_id() == 0) {
            if (c1) atomicAdd(&C->c1, c1);
            if (sup) atomicAdd(&C->c2, 3ull * sup);
        }
    }
};

// Forward mode: an owner stages only the neighbours ranked above it in
// (degree desc, id asc) order, the order that makes x the owner of (x, y).
// A triangle a > b > c in that order is then hit once: at (b, c) with apex a.
__device__ __forceinline__ bool staged(const int2* __restrict__ vinfo, int w, int x, int dx,
                                       int fwd) {
    if (!fwd) return true;
    const int dw = vinfo[w].y;
    return dw > dx || (dw == dx && w < x);
}

// Per-vertex list bounds: OFF(v) = L[ob(v), ob(v+1)), UP(v) = L[ub(v), ub(v+1)),
// kept as one uint2 (ob, ub) per vertex so a vertex's bounds share a sector
// (positions < 2m < 2^32).
struct Lists {
    const int32_t* __restrict__ L;
    const uint2* __restrict__ vb;
    __device__ __forceinline__ int64_t ob(int64_t v) const { return int64_t(vb[v].x); }
    __device__ __forceinline__ int64_t ub(int64_t v) const { return int64_t(vb[v].y); }
    const int* __restrict__ split;  // [v*(F+1) + r] = OFF position of id range r
    const int* __restrict__ ucnt;   // [v*NBKT + k] = UP(v) entries with degree bucket >= k
    const PRec* __restrict__ prec;  // per-vertex partner record (CTA tier)
    int rshift;
    const uint32_t* __restrict__ rnk;  // rnk[v] = UP_TAG | rank of v in the owner order
    const int* __restrict__ rb;        // bucket k's ranks: [rb[31 - k], rb[32 - k])
    // UP values of bucket k lie in [rank_lo(k), rank_hi(k)) (tagged)
    __device__ __forceinline__ uint32_t rank_lo(int k) const { return UP_TAG | uint32_t(rb[31 - k]); }
    __device__ __forceinline__ uint32_t rank_hi(int k) const { return UP_TAG | uint32_t(rb[32 - k]); }
    // The part of UP(p) that can hold an apex of owner x (degree bucket kx,
    // tagged rank xk): the entries ranked above x.  UP(p) ascends in rank, so
    // they are a prefix: the runs of buckets > kx ([0, lo), from the ucnt
    // table) plus the ranks below xk in bucket kx's run [lo, hi) — a search
    // (x itself sits in that run: it is p's same-level neighbour).  Tagged
    // ranks compare like the ranks, signed or unsigned (bit 31 set in all).
    // [va, vz): the rank range of bucket kx (rank_lo / rank_hi).
    __device__ __forceinline__ int up_cut(uint32_t ub, int lo, int hi, int xk, uint32_t va,
                                          uint32_t vz) const {
        if (hi - lo <= 1) return lo;  // the run is x alone
        uint32_t a = ub + uint32_t(lo), z = ub + uint32_t(hi);
#ifndef TCB_UPCUT_BINARY
        // Interpolation first: xk is a member of the sorted run L[a, z), whose
        // ranks spread over the bucket's range, so one aligned 8-value window
        // (a 32-byte sector) around the interpolated position usually holds
        // it; otherwise the window's end values shrink the range and the
        // value bounds.  After UPCUT_ROUNDS windows the binary search below
        // finishes.  A binary search alone is log2(run) dependent sector
        // reads per cover edge.
#pragma unroll 1
        for (int it = 0; it < UPCUT_ROUNDS && z - a > 1; ++it) {
            const float f = float(uint32_t(xk) - va) / float(max(vz - va, 1u));
            const uint32_t est = min(a + uint32_t(f * float(z - a)), z - 1);
            const uint32_t w0 = est & ~7u;
            const int4 q0 = *reinterpret_cast<const int4*>(L + w0);
            const int4 q1 = *reinterpret_cast<const int4*>(L + w0 + 4);
            const int v[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
            int lt = 0, vmin = 0x7FFFFFFF, vmax = int(0x80000000u);
            bool ge = false, le = false;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool ok = w0 + i >= a && w0 + i < z;
                lt += ok && v[i] < xk;
                ge |= ok && v[i] >= xk;
                le |= ok && v[i] <= xk;
                if (ok) {
                    vmin = min(vmin, v[i]);
                    vmax = max(vmax, v[i]);
                }
            }
            if (ge && le) return int(max(w0, a) + uint32_t(lt) - ub);  // xk is in the window
            if (!ge) {  // every valid value is below xk
                a = min(w0 + 8, z);
                va = uint32_t(vmax);
            } else {    // every valid value is above xk
                z = max(w0, a);
                vz = uint32_t(vmin);
            }
        }
#endif
        while (a < z) {
            const uint32_t mid = a + ((z - a) >> 1);
            if (L[mid] < xk) a = mid + 1; else z = mid;
        }
        return int(a - ub);
    }
    __device__ __forceinline__ int up_cut(int64_t p, int kx, int xk) const {
        const int hi = ucnt[p * NBKT + kx];
        const int lo = kx + 1 < NBKT ? ucnt[p * NBKT + kx + 1] : 0;
        return up_cut(vb[p].y, lo, hi, xk, rank_lo(kx), rank_hi(kx));
    }
};

// ---------------------------------------------------------------------------
// 1. owner-grouped selection + entry classes

// The owner predicate is evaluated once (two random gathers per entry) into
// a bitmask, one ballot word per 32 entries; both scan passes then read bits
// only.  The same gathers give the OFF / UP class bits.  The gathers read the
// packed 32-bit (level, degree) key when every vertex fits it (4n bytes: the
// RMAT-24 table stays in L2), else the int2 vinfo.
constexpr int KEY_DB = 22;  // degree bits of the packed key; level gets the top 10
__global__ void k_owner_bits(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                             const int2* __restrict__ vinfo, const uint32_t* __restrict__ key32,
                             const unsigned long long* __restrict__ nopack, int64_t nnz,
                             int mode, uint32_t* __restrict__ bits, uint2* __restrict__ cls) {
    // mode bit 0: forward (every entry OFF); bit 1: cross only (no UP class:
    // split_cross_count_k, the triangles with one horizontal edge)
    const int fwd = mode & 1, xonly = mode >> 1;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const unsigned lane = lane_id();
    const bool packed = block_load(nopack) == 0;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < nnz;
         base += gthreads) {
        const int64_t e = base + lane;
        bool keep = false, off = false, sup = false;
        if (e < nnz) {
            const int x = src[e], y = nb[e];
            int2 a, b;
            if (packed) {
                const uint32_t ka = key32[x], kb = key32[y];
                a = make_int2(int(ka >> KEY_DB), int(ka & ((1u << KEY_DB) - 1)));
                b = make_int2(int(kb >> KEY_DB), int(kb & ((1u << KEY_DB) - 1)));
            } else {
                a = vinfo[x];
                b = vinfo[y];
            }
            // owner order: degree bucket desc, id asc (forward mode: degree
            // desc, id asc, the order staged() filters by)
            const int ka = fwd ? a.y : dbucket(a.y), kb = fwd ? b.y : dbucket(b.y);
            keep = a.x == b.x && (ka > kb || (ka == kb && x < y));
            off = fwd || a.x != b.x;
            sup = !fwd && !xonly && a.x == b.x && !keep;  // UP: same level, y owns the edge
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const unsigned mo = __ballot_sync(0xffffffffu, off);
        const unsigned ms = __ballot_sync(0xffffffffu, sup);
        if (lane == 0) {
            bits[base >> 5] = m;
            cls[base >> 5] = make_uint2(mo, ms);
        }
    }
}

// Keep bits (x owns a horizontal edge) and class bits of every CSR entry.
// The cover edges are then compacted without an ordered scan: a word-level
// prefix of the keep bits gives each kept entry its slot in P (k_scatter_off)
// and each owner its segment [seg_beg, seg_end) (k_list_bounds).
uint32_t* owner_bits(Context* ctx, const int32_t* src, const int32_t* nb, const int2* vinfo,
                     const uint32_t* key32, const unsigned long long* nopack, int64_t nnz,
                     int mode, uint2* cls) {
    const int64_t nwords = (nnz + 31) / 32;
    uint32_t* bits = ctx->wsT<uint32_t>(WS_QUEUE_A, nwords + 1);
    TCB_CUDA(cudaMemsetAsync(bits + nwords, 0, sizeof(uint32_t), ctx->stream));
    TCB_LAUNCH(ctx, k_owner_bits, grid_for(ctx, nnz, 256), 256, 0, src, nb, vinfo, key32, nopack,
               nnz, mode, bits, cls);
    return bits;
}

__device__ __forceinline__ int64_t rank_keep(const uint32_t* __restrict__ bits,
                                             const unsigned long long* __restrict__ prek,
                                             int64_t p) {
    const int64_t j = p >> 5;
    return int64_t(prek[j]) + __popc(bits[j] & ((1u << (p & 31)) - 1u));
}

// Per vertex: (level, degree), the packed key and the degree bucket.
__global__ void k_vinfo(const int64_t* __restrict__ row, const int32_t* __restrict__ level,
                        int64_t n, int2* __restrict__ vinfo, uint32_t* __restrict__ key32,
                        uint8_t* __restrict__ dbk, unsigned long long* nopack,
                        int* __restrict__ long_rows, unsigned long long* nlong, int up_long) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        const int l = level[v], d = int(row[v + 1] - row[v]);
        vinfo[v] = make_int2(l, d);
        if (d > up_long) long_rows[atomicAdd(nlong, 1ull)] = int(v);  // k_build_up phase A
        dbk[v] = uint8_t(dbucket(d));
        const bool fits = l >= 0 && l < (1 << (32 - KEY_DB)) && d < (1 << KEY_DB);
        key32[v] = fits ? (uint32_t(l) << KEY_DB) | uint32_t(d) : 0u;
        const unsigned act = __activemask();
        const unsigned bad = __ballot_sync(act, !fits);
        if (bad && int(lane_id()) == __ffs(act) - 1) atomicExch(nopack, 1ull);
    }
}

// Ranks in the owner order (degree bucket desc, id asc) over all vertices:
// one stable counting pass by digit 31 - bucket over the ids in order, the
// shape of a radix-sort pass (csr.cu) with the key implicit.  rnk[v] =
// UP_TAG | rank; rb[d] = first rank of digit d (bucket 31 - d), rb[32] = n.
constexpr int RK_BLOCK = 256;
constexpr int RK_WARPS = RK_BLOCK / 32;
constexpr int RK_ROUNDS = 16;
constexpr int64_t RK_TILE = int64_t(RK_BLOCK) * RK_ROUNDS;
__global__ void __launch_bounds__(RK_BLOCK)
    k_rank_hist(const uint8_t* __restrict__ dbk, int64_t n, int64_t* __restrict__ hist,
                int64_t ntiles) {
    __shared__ unsigned h[NBKT];
    if (threadIdx.x < NBKT) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * RK_TILE;
#pragma unroll 4
    for (int j = 0; j < RK_ROUNDS; ++j) {
        const int64_t i = base + int64_t(j) * RK_BLOCK + threadIdx.x;
        const unsigned d = i < n ? 31u - dbk[i] : unsigned(NBKT);
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < NBKT && lane_id() == unsigned(__ffs(peers) - 1))
            atomicAdd(&h[d], unsigned(__popc(peers)));
    }
    __syncthreads();
    if (threadIdx.x < NBKT) hist[int64_t(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RK_BLOCK)
    k_rank_assign(const uint8_t* __restrict__ dbk, int64_t n, const int64_t* __restrict__ offs,
                  int64_t ntiles, uint32_t* __restrict__ rnk, int* __restrict__ rb) {
    __shared__ unsigned cnt[RK_WARPS][NBKT + 1];
    __shared__ int64_t base_off[NBKT];
    const int w = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    for (int i = threadIdx.x; i < RK_WARPS * (NBKT + 1); i += RK_BLOCK) (&cnt[0][0])[i] = 0;
    if (threadIdx.x < NBKT) {
        base_off[threadIdx.x] = offs[int64_t(threadIdx.x) * ntiles + blockIdx.x];
        if (blockIdx.x == 0) rb[threadIdx.x] = int(offs[int64_t(threadIdx.x) * ntiles]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) rb[NBKT] = int(n);
    __syncthreads();
    // warp w owns the contiguous run [wbase, wbase + 32 RK_ROUNDS) of the
    // tile: (round, lane) is id order
    const int64_t wbase = int64_t(blockIdx.x) * RK_TILE + int64_t(w) * 32 * RK_ROUNDS;
    unsigned dig[RK_ROUNDS], pos[RK_ROUNDS];
#pragma unroll
    for (int r = 0; r < RK_ROUNDS; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const unsigned d = i < n ? 31u - dbk[i] : unsigned(NBKT);
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned old = cnt[w][d];
        __syncwarp();
        if (lane == unsigned(__ffs(peers) - 1)) cnt[w][d] = old + __popc(peers);
        __syncwarp();
        dig[r] = d;
        pos[r] = old + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    if (threadIdx.x < NBKT) {  // per digit: exclusive prefix over the warps
        unsigned run = 0;
#pragma unroll
        for (int ww = 0; ww < RK_WARPS; ++ww) {
            const unsigned t = cnt[ww][threadIdx.x];
            cnt[ww][threadIdx.x] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RK_ROUNDS; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        if (i < n)
            rnk[i] = UP_TAG | uint32_t(base_off[dig[r]] + cnt[w][dig[r]] + pos[r]);
    }
}

// ---------------------------------------------------------------------------
// 2. OFF / UP lists.  The OFF array comes first; UP starts at NOFF (the
//    class total, pre[nw] low half).  ob/sb hold absolute positions in L.

__global__ void k_list_bounds(const int64_t* __restrict__ row, int64_t n,
                              const uint2* __restrict__ cls,
                              const unsigned long long* __restrict__ pre, int64_t nw,
                              uint2* __restrict__ vb, const uint32_t* __restrict__ bits,
                              const unsigned long long* __restrict__ prek,
                              int64_t* __restrict__ seg_beg, int64_t* __restrict__ seg_end) {
    const int64_t noff = int64_t(pre[nw] & 0xFFFFFFFFull);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v <= n; v += stride) {
        const int64_t p = row[v];
        if (v < n) {  // the owner's cover edges: P[seg_beg, seg_end)
            seg_beg[v] = rank_keep(bits, prek, p);
            seg_end[v] = rank_keep(bits, prek, row[v + 1]);
        }
        vb[v] = make_uint2(uint32_t(rank_off(cls, pre, p)),
                           uint32_t(noff + rank_up(cls, pre, p)));
    }
}

// OFF entries go to their slot in L, kept entries (cover edges, owner
// side) to theirs in P (word prefix + popc).
__global__ void k_scatter_off(const int32_t* __restrict__ src, const int32_t* __restrict__ nb,
                              int64_t nnz, const uint2* __restrict__ cls,
                              const unsigned long long* __restrict__ pre,
                              int32_t* __restrict__ L, const uint32_t* __restrict__ bits,
                              const unsigned long long* __restrict__ prek,
                              int32_t* __restrict__ P, int32_t* __restrict__ PX) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride) {
        const uint32_t bit = 1u << (e & 31);
        if (cls[e >> 5].x & bit) L[rank_off(cls, pre, e)] = nb[e];
        if (bits[e >> 5] & bit) {  // a cover edge: partner and owner of its slot
            const int64_t slot = rank_keep(bits, prek, e);
            P[slot] = nb[e];
            PX[slot] = src[e];
        }
    }
}

// UP rows, one warp per row: a counting sort by degree bucket (largest
// first) with the histogram and cursors in shared memory, and the row's
// prefix counts ucnt[v][k] = entries in buckets >= k.  Short rows (d <=
// UP_SHORT): a lane per entry, the UP entries and their buckets kept in
// shared memory between the histogram and the scatter.  Long rows: lanes
// scan the row's class words 32 at a time (a hub row with few UP entries
// costs d/1024 iterations) and gather twice.  Rows of isolated vertices are
// never read and are skipped.
constexpr int UP_WARPS = 8;
#ifndef TCB_UPW
#define TCB_UPW 4  // long-row UP words whose loads are in flight together
#endif
#ifndef TCB_UP_QUARTER
#define TCB_UP_QUARTER 1  // rows of <= 8 entries: four at a time, a quarter warp each
#endif
#ifndef TCB_UP_MINB
#define TCB_UP_MINB 8  // k_build_up is latency-bound: keep 64 warps per SM
#endif

// Stable counting-sort placement for one 32-entry step of a row (lanes hold
// consecutive row entries, so ids ascend with the lane): entries of the same
// bucket keep their lane order and each bucket's run of the UP list stays
// id-sorted.  h[b] = next free position of bucket b.
__device__ __forceinline__ int stable_slot(int* h, bool act, int b) {
    const int lane = int(lane_id());
#ifndef TCB_SLOT_BALLOT
    const unsigned peers = __match_any_sync(0xffffffffu, act ? b : NBKT + lane);
#else
    // lanes with the same bucket: five ballots over its bits (NBKT = 32)
    unsigned peers = __ballot_sync(0xffffffffu, act);
    if (!act) peers = 1u << lane;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const bool bk = (b >> k) & 1;
        const unsigned v = __ballot_sync(0xffffffffu, bk);
        if (act) peers &= bk ? v : ~v;
    }
#endif
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (act && lane == leader) {
        base = h[b];
        h[b] = base + __popc(peers);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    __syncwarp();
    return base + __popc(peers & lanemask_lt());
}
constexpr int UP_SHORT = 256;
#ifndef TCB_UP_LONG
#define TCB_UP_LONG 8192
#endif
constexpr int UP_LONG = TCB_UP_LONG;  // rows above this are listed and built first (k_build_up phase A)
static_assert(NBKT == 32, "one degree bucket per lane");
__global__ void __launch_bounds__(UP_WARPS * 32, TCB_UP_MINB)
    k_build_up(const int64_t* __restrict__ row, const int32_t* __restrict__ nb, int64_t n,
               const uint2* __restrict__ cls, const uint8_t* __restrict__ dbk,
               const uint32_t* __restrict__ rnk, const uint2* __restrict__ vb,
               int32_t* __restrict__ L, int* __restrict__ ucnt, PRec* __restrict__ prec,
               const int* __restrict__ long_rows, const unsigned long long* __restrict__ nlong_p,
               unsigned long long* group_ctr) {
    __shared__ int s_h[UP_WARPS][NBKT];
    __shared__ int s_w[UP_WARPS][UP_SHORT];
    __shared__ uint8_t s_b[UP_WARPS][UP_SHORT];
    const int warp = threadIdx.x >> 5;
    const int lane = int(lane_id());
    int* h = s_h[warp];
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    // One row (UP entries u0 .. u0 + nup of L), by the whole warp.
    auto do_row = [&](int64_t v, int64_t r0, int64_t r1, uint32_t u0, uint32_t nup) {
        (void)nup;
        PRec* pr = prec + v;
        h[lane] = 0;
        __syncwarp();
        if (r1 - r0 <= UP_SHORT) {
            int nbuf = 0;
            for (int64_t e0 = r0; e0 < r1; e0 += 32) {
                const int64_t e = e0 + lane;
                const bool up = e < r1 && ((cls[e >> 5].y >> (e & 31)) & 1u);
                const unsigned bal = __ballot_sync(0xffffffffu, up);
                if (up) {
                    const int w = nb[e];
                    const int b = dbk[w];
                    const int q = nbuf + __popc(bal & lanemask_lt());
                    s_w[warp][q] = int(rnk[w]);  // the list holds tagged ranks
                    s_b[warp][q] = uint8_t(b);
                    atomicAdd(&h[b], 1);
                }
                nbuf += __popc(bal);
            }
            __syncwarp();
            const int c = h[lane];
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += t;
            }
            ucnt[v * NBKT + lane] = incl;
            if (lane >= PR_K0 && lane < PR_K0 + PR_NK)
                pr->uc[lane - PR_K0] = uint16_t(min(incl, PR_FULL));
            __syncwarp();
            h[lane] = incl - c;
            __syncwarp();
            for (int i0 = 0; i0 < nbuf; i0 += 32) {
                const int i = i0 + lane;
                const bool act = i < nbuf;
                const int pos = stable_slot(h, act, act ? int(s_b[warp][i]) : 0);
                if (act) L[int64_t(u0) + pos] = s_w[warp][i];
            }
            __syncwarp();
            return;
        }
        const int64_t j0 = r0 >> 5, j1 = (r1 - 1) >> 5;
        // Long rows: lanes read 32 class words at a time; every word with UP
        // bits is then taken by the whole warp (lane = bit), so entries are
        // visited in row order with coalesced loads and a hub row with few UP
        // entries costs d/1024 iterations.
        auto up_words = [&](auto want_rank, auto&& visit) {
            for (int64_t jb = j0; jb <= j1; jb += 32) {
                const int64_t j = jb + lane;
                uint32_t m = 0;
                if (j <= j1) {
                    m = cls[j].y;
                    if (j == j0) m &= ~0u << (r0 & 31);
                    if (j == j1 && ((r1 & 31) != 0)) m &= (1u << (r1 & 31)) - 1u;
                }
                unsigned nzw = __ballot_sync(0xffffffffu, m != 0);
                while (nzw) {  // up to UPW words per round, their loads in flight together
                    constexpr int UPW = TCB_UPW;
                    int sl[UPW], w[UPW], b[UPW];
                    uint32_t upm = 0;  // bit q: this lane's entry of word q is UP
#pragma unroll
                    for (int q = 0; q < UPW; ++q) {
                        sl[q] = 0;
                        if (nzw) {  // warp-uniform
                            sl[q] = __ffs(nzw) - 1;
                            nzw &= nzw - 1;
                            upm |= ((__shfl_sync(0xffffffffu, m, sl[q]) >> lane) & 1u) << q;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < UPW; ++q)
                        w[q] = (upm >> q) & 1u ? nb[(jb + sl[q]) * 32 + lane] : 0;
#pragma unroll
                    for (int q = 0; q < UPW; ++q) b[q] = (upm >> q) & 1u ? int(dbk[w[q]]) : 0;
                    if (decltype(want_rank)::value) {  // the scatter pass writes tagged ranks
#pragma unroll
                        for (int q = 0; q < UPW; ++q) w[q] = (upm >> q) & 1u ? int(rnk[w[q]]) : 0;
                    }
#pragma unroll
                    for (int q = 0; q < UPW; ++q) visit(((upm >> q) & 1u) != 0, w[q], b[q]);
                }
            }
        };
        // pass 1: bucket histogram
        up_words(std::false_type{}, [&](bool up, int, int b) {
            if (up) atomicAdd(&h[b], 1);
        });
        __syncwarp();
        // buckets descending: start[k] = entries in buckets > k
        const int c = h[lane];
        int incl = c;  // suffix sum over lanes >= lane
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_down_sync(0xffffffffu, incl, o);
            if (lane + o < 32) incl += t;
        }
        ucnt[v * NBKT + lane] = incl;
        if (lane >= PR_K0 && lane < PR_K0 + PR_NK)
            pr->uc[lane - PR_K0] = uint16_t(min(incl, PR_FULL));
        __syncwarp();
        h[lane] = incl - c;
        __syncwarp();
        // pass 2: stable scatter (row order within each bucket)
        up_words(std::true_type{}, [&](bool up, int w, int b) {
            const int pos = stable_slot(h, up, b);
            if (up) L[int64_t(u0) + pos] = w;
        });
        __syncwarp();
    };
    // Phase A: the longest rows (> UP_LONG entries, listed by k_vinfo) first,
    // a warp each from the start of the kernel: a hub row of 4e5 entries is
    // ~2.5 ms of one warp, which would otherwise end the kernel that much
    // after everything else wherever its turn came.  Phase B hands out the
    // 32-row groups dynamically, so the warps that took a long row take fewer.
    {
        const int64_t nlong = int64_t(block_load(nlong_p));
        for (int64_t i = gw; i < nlong; i += nwarps) {
            const int64_t v = long_rows[i];
            const uint2 b0 = vb[v], b1 = vb[v + 1];
            if (b1.y != b0.y) do_row(v, row[v], row[v + 1], b0.y, b1.y - b0.y);
        }
    }
    while (true) {
        unsigned long long g_ = 0;
        if (lane == 0) g_ = atomicAdd(group_ctr, 1ull);
        const int64_t vbase = int64_t(__shfl_sync(0xffffffffu, g_, 0)) * 32;
        if (vbase >= n) break;
        // A lane per row first: bounds and records for 32 rows at once; rows
        // without UP entries (isolated vertices included) end here, and the
        // warp takes the others one by one.
        const int64_t lv = vbase + lane;
        int64_t lr0 = 0, lr1 = 0;
        uint2 lb0 = make_uint2(0, 0), lb1 = lb0;
        if (lv < n) {
            lr0 = row[lv];
            lr1 = row[lv + 1];
            lb0 = vb[lv];
            lb1 = vb[lv + 1];
        }
        const bool live = lv < n && lr1 > lr0;
        if (live) {
            PRec* pr = prec + lv;
            pr->ob = lb0.x;
            pr->ub = lb0.y;
            pr->noff = lb1.x - lb0.x;
            if (lb1.y == lb0.y) {  // no UP entries: zero prefix counts
                int4* uc4 = reinterpret_cast<int4*>(ucnt + lv * NBKT);
#pragma unroll
                for (int q = 0; q < NBKT / 4; ++q) uc4[q] = make_int4(0, 0, 0, 0);
#pragma unroll
                for (int q = 0; q < PR_NK; ++q) pr->uc[q] = 0;
            }
        }
        unsigned work =
            __ballot_sync(0xffffffffu, live && lb1.y != lb0.y && lr1 - lr0 <= UP_LONG);
#if TCB_UP_QUARTER
        // Rows of <= 8 entries (two in five of the rows with UP entries at
        // RMAT scale): four at a time, a quarter warp each, a lane per entry.
        // A row's cost is its chain of dependent reads (class word, entry,
        // bucket and rank gathers), not its length, so four chains in flight
        // are four times the rows per warp.  The order inside the quarter is
        // computed with eight shuffles (larger bucket first, then lane = row =
        // id order) — no histogram, no shared memory.
        {
            unsigned sm = work & __ballot_sync(0xffffffffu, lr1 - lr0 <= 8);
            work &= ~sm;
            const int q = lane >> 3, ql = lane & 7;
            while (sm) {  // warp-uniform
                int pick = -1;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int s_ = sm ? __ffs(sm) - 1 : -1;
                    if (sm) sm &= sm - 1;
                    if (t == q) pick = s_;
                }
                const int sl = max(pick, 0);
                const int64_t r0 = __shfl_sync(0xffffffffu, lr0, sl);
                const int64_t r1 = __shfl_sync(0xffffffffu, lr1, sl);
                const uint32_t u0 = __shfl_sync(0xffffffffu, lb0.y, sl);
                const int64_t v = vbase + sl;
                const int64_t e = r0 + ql;
                const bool up = pick >= 0 && e < r1 && ((cls[e >> 5].y >> (e & 31)) & 1u);
                int b = -1, rk = 0;
                if (up) {
                    const int w = nb[e];
                    b = dbk[w];
                    rk = int(rnk[w]);
                }
                int pos = 0;
                int c[4] = {0, 0, 0, 0};  // entries in buckets >= 4 ql + t
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int bj = __shfl_sync(0xffffffffu, b, (lane & ~7) + j);
                    pos += (bj > b) || (bj == b && j < ql);
#pragma unroll
                    for (int t = 0; t < 4; ++t) c[t] += bj >= 4 * ql + t;
                }
                if (up) L[int64_t(u0) + pos] = rk;
                if (pick >= 0) {
                    *reinterpret_cast<int4*>(ucnt + v * NBKT + 4 * ql) =
                        make_int4(c[0], c[1], c[2], c[3]);
                    PRec* pr = prec + v;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int k = 4 * ql + t - PR_K0;
                        if (k >= 0 && k < PR_NK) pr->uc[k] = uint16_t(c[t]);
                    }
                }
            }
        }
#endif
        while (work) {
            const int src = __ffs(work) - 1;
            work &= work - 1;
            const uint32_t u0 = __shfl_sync(0xffffffffu, lb0.y, src);
            do_row(vbase + src, __shfl_sync(0xffffffffu, lr0, src),
                   __shfl_sync(0xffffffffu, lr1, src), u0,
                   __shfl_sync(0xffffffffu, lb1.y, src) - u0);
        }
    }
}

// ---------------------------------------------------------------------------
// 3. split points: split[v*(F+1) + r] = first position in OFF(v) of an id
//    >= r << rshift, relative to the list start; [0] = 0, [F] = size.

// From the id-sorted OFF lists themselves: a lane per vertex walks a short
// list once; the warp takes a long list (> SPLIT_LONG ids) together, one
// binary search per boundary.  Rows of empty OFF lists stay zero (memset).
constexpr int SPLIT_LONG = 256;
constexpr int SPLIT_WARPS = 8;
// A warp per 32 consecutive vertices: every row is built in a shared-memory
// tile (row stride F + 1 = 33 ints: lanes writing the same column hit
// distinct banks) and the 32 rows, contiguous in the table, are written out
// with coalesced stores — every row, so no memset of the table is needed.
__global__ void __launch_bounds__(SPLIT_WARPS * 32)
    k_split_points(int64_t n, const int32_t* __restrict__ L, const uint2* __restrict__ vb,
                   int rshift, int* __restrict__ split) {
    __shared__ int s_tile[SPLIT_WARPS][32 * (F + 1)];
    const int lane = int(lane_id());
    int* tile = s_tile[threadIdx.x >> 5];
    int* my = tile + lane * (F + 1);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < n;
         base += stride) {
        const int64_t v = base + lane;
        int64_t b0 = 0, b1 = 0;
        if (v < n) {
            b0 = vb[v].x;
            b1 = vb[v + 1].x;
        }
        const int len = int(b1 - b0);
        if (len <= SPLIT_LONG) {  // empty rows become all zeros
            int q = 0;
            for (int64_t g = b0; g < b1; ++g) {
                const int r = L[g] >> rshift;
                for (; q <= r; ++q) my[q] = int(g - b0);
            }
            for (; q <= F; ++q) my[q] = len;
        }
        unsigned longs = __ballot_sync(0xffffffffu, len > SPLIT_LONG);
        while (longs) {
            const int src_lane = __ffs(longs) - 1;
            longs &= longs - 1;
            const int64_t lb0 = __shfl_sync(0xffffffffu, b0, src_lane);
            const int64_t lb1 = __shfl_sync(0xffffffffu, b1, src_lane);
            for (int q = lane; q <= F; q += 32) {  // first position with id >= q << rshift
                const int64_t key = int64_t(q) << rshift;
                int64_t lo = lb0, hi = lb1;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (int64_t(L[mid]) < key) lo = mid + 1; else hi = mid;
                }
                tile[src_lane * (F + 1) + q] = int(lo - lb0);
            }
        }
        __syncwarp();
        const int64_t rows = min(int64_t(32), n - base);
        int* out = split + base * (F + 1);
        for (int k = lane; k < rows * (F + 1); k += 32) out[k] = tile[k];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// 4. work items

__global__ void k_make_items(const int64_t* __restrict__ row, const int64_t* __restrict__ seg_beg,
                             const int64_t* __restrict__ seg_end, Lists ls, int64_t n,
                             longlong4* __restrict__ witems, longlong4* __restrict__ citems,
                             longlong4* __restrict__ titems, unsigned long long* nw,
                             unsigned long long* nc, unsigned long long* nt, int shard,
                             int nshards, int wt, int hc, int tiny) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // Multi-GPU (tcb_cetc_shard): partner block i of owner x belongs to
    // shard (x + i) % nshards (dist.py shard_of mirrors this).  Blocks rather
    // than whole owners, so a hub's work spreads over the ranks.
    auto mine = [shard, nshards](int64_t x, int64_t i) {
        return nshards <= 1 || int((x + i) % nshards) == shard;
    };
    // A lane per vertex; the item slots of a warp's 32 vertices are taken
    // with ONE atomic per list (warp scan of the counts): millions of owners
    // adding to the same three counters were what this kernel waited for.
    const int lane = int(lane_id());
    for (int64_t xb = int64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; xb < n; xb += stride) {
        const int64_t x = xb + lane;
        int kind = 0;  // 1 thread item, 2 warp items, 3 CTA items
        int cnt = 0;   // items of this vertex
        int64_t s = 0, e = 0, nup = 0;
        int lg = 0;
        const int* sx = nullptr;
        auto staged_any = [&](int g) {
            const int q0 = (g << LOG_F) >> lg, q1 = ((g + 1) << LOG_F) >> lg;
            return sx[q1] - sx[q0] > 0 || (g == 0 && nup > 0);
        };
        if (x < n) do {
            const int64_t d = row[x + 1] - row[x];
            if (d == 0) break;
            s = seg_beg[x];
            e = seg_end[x];
            if (e <= s) break;
            // nothing staged (no OFF neighbours, no same-level neighbour ranked
            // above x): no edge of x can have an apex
            nup = ls.ub(x + 1) - ls.ub(x);
            const int64_t st = (ls.ob(x + 1) - ls.ob(x)) + nup;
            if (st == 0) break;
            if (d <= tiny) {  // <= TINY partners, each with <= TINY ids
                if (mine(x, 0)) {
                    kind = 1;
                    cnt = 1;
                }
                break;
            }
            if (d <= wt) {
                const int64_t nb_ = (e - s + PW - 1) / PW;
                for (int64_t i = 0; i < nb_; ++i) cnt += mine(x, i);
                kind = cnt ? 2 : 0;
                break;
            }
#ifdef TCB_ONLY_SMALL  // measurement-only: CTA items of small owners only
            if (st > TCB_ONLY_SMALL) break;
#endif
#ifdef TCB_ONLY_BIG  // measurement-only: CTA items of big owners only
            if (st <= TCB_ONLY_BIG) break;
#endif
            // fewest range groups G (power of two <= F) whose OFF slices all
            // fit HC; group 0 also stages UP(x) (not range-split: it is
            // rank-sorted, and it takes no table slots: a rank bitmap beside
            // the OFF set, or rank windows after it)
            sx = ls.split + x * (F + 1);
            if (st - nup > hc) {
                for (lg = 1; lg < LOG_F; ++lg) {
                    const int step = F >> lg;
                    int mx = 0;
                    for (int q = 0; q < F; q += step) mx = max(mx, sx[q + step] - sx[q]);
                    if (mx <= hc) break;
                }
            }
            const int64_t per = (e - s + PC - 1) / PC;
            int my = 0;
            for (int64_t i = 0; i < per; ++i) my += mine(x, i);
            int ng = 0;  // groups with something staged
            for (int g = 0; g < (1 << lg); ++g) ng += staged_any(g);
            cnt = my * ng;
            kind = cnt ? 3 : 0;
        } while (false);
        // slots: one atomic per warp and list
        unsigned long long base = 0;
#pragma unroll
        for (int k = 1; k <= 3; ++k) {
            const int c = kind == k ? cnt : 0;
            const int incl = warp_inclusive_scan(c);
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            if (tot == 0) continue;  // warp-uniform
            unsigned long long b0 = 0;
            if (lane == 31)
                b0 = atomicAdd(k == 1 ? nt : k == 2 ? nw : nc, (unsigned long long)tot);
            b0 = __shfl_sync(0xffffffffu, b0, 31);
            if (kind == k) base = b0 + (unsigned long long)(incl - c);
        }
        if (kind == 1) {
            titems[base] = make_longlong4(x, s, e, 0);
        } else if (kind == 2) {
            const int64_t nb_ = (e - s + PW - 1) / PW;
            for (int64_t i = 0; i < nb_; ++i) {
                if (!mine(x, i)) continue;
                const int64_t p0 = s + i * PW;
                witems[base++] = make_longlong4(x, p0, min(p0 + PW, e), 0);
            }
        } else if (kind == 3) {
            const int64_t per = (e - s + PC - 1) / PC;
            for (int g = 0; g < (1 << lg); ++g) {
                if (!staged_any(g)) continue;
                for (int64_t i = 0; i < per; ++i) {
                    if (!mine(x, i)) continue;
                    const int64_t p0 = s + i * PC;
                    citems[base++] = make_longlong4(x, p0, min(p0 + PC, e), (lg << 8) | g);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 4b. thread tier: one thread per tiny owner (d(x) <= TINY, so every partner
//     has <= TINY ids too).  OFF(x) ∪ UP(x) sits in registers; each streamed
//     id is compared with all of it.

__global__ void __launch_bounds__(256)
    k_isect_tiny(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                 Lists ls, const int32_t* __restrict__ P, DevCounters* C,
                 const int2* __restrict__ vinfo, int fwd) {
    const int64_t nitems = int64_t(block_load(nitems_p));
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    uint32_t n1 = 0, ns = 0;
    for (int64_t it = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; it < nitems; it += stride) {
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int64_t o0 = ls.ob(x), o1 = ls.ob(x + 1), s0 = ls.ub(x);
        const int no = int(o1 - o0), nx = no + int(ls.ub(x + 1) - s0);
        const int dx = vinfo[x].y;
        const int kx = dbucket(dx);
        const int xk = nx > no ? int(ls.rnk[x]) : 0;  // tagged rank: the UP cut's key
        int a[TINY];
#pragma unroll
        for (int i = 0; i < TINY; ++i) {
            int w = PAD;
            if (i < nx) w = i < no ? ls.L[o0 + i] : ls.L[s0 + (i - no)];
            if (w != PAD && !staged(vinfo, w, x, dx, fwd)) w = PAD;
            a[i] = w;
        }
        for (int64_t p = item.y; p < item.z; ++p) {
            const int y = P[p];
            const int64_t y0 = ls.ob(y), y1 = ls.ob(y + 1), y2 = ls.ub(y);
            const int64_t y3 = y2 + (nx > no ? ls.up_cut(y, kx, xk) : 0);
            for (int64_t j = y0; j < y1; ++j) {
                const int w = ls.L[j];
                bool hit = false;
#pragma unroll
                for (int i = 0; i < TINY; ++i) hit |= a[i] == w;
                n1 += hit;
            }
            for (int64_t j = y2; j < y3; ++j) {
                const int w = ls.L[j];
                bool hit = false;
#pragma unroll
                for (int i = 0; i < TINY; ++i) hit |= a[i] == w;
                ns += hit;
            }
        }
    }
    Tally tl;
    tl.c1 = n1;
    tl.sup = ns;
    tl.flush(C);
}

// ---------------------------------------------------------------------------
// 5. warp tier: one warp per item (owner x with d(x) <= WT, <= PW partners).
//    The owner's OFF(x) ∪ UP(x) sits in a per-warp bucket hash; the partners'
//    OFF slices and UP prefixes are compacted into a per-warp slice table
//    (OFF slices first) and streamed in rounds of 32 x JW elements, each lane
//    walking the slice boundaries like the CTA tier's cross_chunk.

#ifndef TCB_JW
#define TCB_JW 16  // 4 / 8 / 16 / 24 / 32: 4.81 / 4.48 / 4.36 / 4.50 / 5.10 ms at RMAT-24
#endif
constexpr int JW = TCB_JW;      // elements per lane per warp-tier round
constexpr int W_SEG = 2 * PW;   // slices per warp item

template <typename Probe>
__device__ __forceinline__ void warp_stream(const int32_t* __restrict__ L, const int2* seg,
                                            int total, int tsup, const Probe& h, Tally& tl) {
    const int lane = int(lane_id());
    int kc = 0;  // warp-uniform: the slice holding c0
    for (int c0 = 0; c0 < total; c0 += 32 * JW) {
        while (seg[kc + 1].x <= c0) ++kc;
        const int c1 = min(total, c0 + 32 * JW);
        const int i0 = c0 + lane;
        int k = kc;
        int nx = seg[k + 1].x;
        uint32_t base = uint32_t(seg[k].y);
        int w[JW];
#pragma unroll
        for (int j = 0; j < JW; ++j) {
            const int i = i0 + 32 * j;
            w[j] = PAD;
            if (i < c1) {
                if (nx <= i) {
                    do {
                        ++k;
                        nx = seg[k + 1].x;
                    } while (nx <= i);
                    base = uint32_t(seg[k].y);
                }
                w[j] = L[base + uint32_t(i)];
            }
        }
        // the next round starts in (or just before) the last lane's slice
        kc = __shfl_sync(0xffffffffu, k, 31);
        uint32_t hm = 0;
#pragma unroll
        for (int j = 0; j < JW; ++j)
            if (w[j] != PAD && h.hit(w[j])) hm |= 1u << j;
        const int jt = (tsup - i0 + 31) >> 5;  // elements j >= jt are UP
        const uint32_t sm = jt <= 0 ? ~0u : (jt >= JW ? 0u : ~0u << jt);
        const uint32_t sup = __popc(hm & sm);
        tl.c1 += __popc(hm) - sup;
        tl.sup += sup;
    }
}

__global__ void __launch_bounds__(W_WARPS * 32, 4)
    k_isect_warp(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                 Lists ls, const int32_t* __restrict__ P, unsigned long long* fetch,
                 DevCounters* C, const int2* __restrict__ vinfo, int fwd, int dbg) {
    extern __shared__ uint4 smem4[];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem4) + warp * W_SLOTS;
    int2* seg = reinterpret_cast<int2*>(reinterpret_cast<uint32_t*>(smem4) + W_WARPS * W_SLOTS) +
                warp * (W_SEG + 1);
    for (int i = lane; i < W_SLOTS; i += 32) tab[i] = EMPTY;
    __syncwarp();
    const unsigned long long nitems = block_load(nitems_p);
    Tally tl;
    while (true) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(fetch, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) break;
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int64_t o0 = ls.ob(x), s0 = ls.ub(x);
        const int no = int(ls.ob(x + 1) - o0), nu = int(ls.ub(x + 1) - s0), nx = no + nu;
        const int dx = vinfo[x].y;
        const int kx = dbucket(dx);
        const int slots = max(16, 4 << ceil_log2_dev(nx));
        BucketHash h;
        h.setup(tab, slots);
        // a two-table cuckoo set (load <= 1/4): branch-free two-read probes
        // (the bucket table's probe loop cost 1 ms more at RMAT-24); a failed
        // kick chain rebuilds the item's table as buckets
        CuckooHash ch;
        ch.setup(tab, slots);
        for (int i = lane; i < slots; i += 32) tab[i] = C_EMPTY;
        __syncwarp();
        bool fail = false;
        for (int i = lane; i < nx; i += 32) {
            const int w = i < no ? ls.L[o0 + i] : ls.L[s0 + (i - no)];
            if (staged(vinfo, w, x, dx, fwd) && !ch.insert(w)) fail = true;
        }
        const bool use_cuckoo =
            !__any_sync(0xffffffffu, fail) && !(dbg & TCB_TEST_FORCE_FALLBACK);
        __syncwarp();
        if (!use_cuckoo) {
            for (int i = lane; i < slots; i += 32) tab[i] = EMPTY;
            __syncwarp();
            for (int i = lane; i < nx; i += 32) {
                const int w = i < no ? ls.L[o0 + i] : ls.L[s0 + (i - no)];
                if (staged(vinfo, w, x, dx, fwd)) h.insert(w);
            }
        }
        // slices of partners lane and lane + 32: OFF (c0, c1), UP (c2, c3)
        // slices of partners lane + 32 r: OFF (cnt[r]), UP prefix (cnt[PPL + r])
        constexpr int PPL = (PW + 31) / 32;  // partners per lane
        static_assert(PPL * 32 * 2 <= 2 * 2048 && PW % 32 == 0, "slice table layout");
        int cnt[2 * PPL];
        uint32_t pos[2 * PPL];
        int so = 0, su = 0, no_ = 0, nu_ = 0;
#pragma unroll
        for (int r = 0; r < PPL; ++r) {
            cnt[r] = cnt[PPL + r] = 0;
            pos[r] = pos[PPL + r] = 0;
            const int64_t j = item.y + lane + 32 * r;
            if (j < item.z) {
                const int y = P[j];
                const uint2 v0 = ls.vb[y];
                pos[r] = v0.x;
                cnt[r] = no ? int(ls.vb[y + 1].x - v0.x) : 0;
                pos[PPL + r] = v0.y;  // the prefix of UP(y) that can be in UP(x)
                // the whole bucket-kx run: over-streams the ids above x in
                // it (no false hits: they are not in UP(x)), which costs this
                // tier less than a search per partner
                cnt[PPL + r] = nu ? ls.ucnt[int64_t(y) * NBKT + kx] : 0;
            }
            so += cnt[r];
            su += cnt[PPL + r];
            no_ += cnt[r] > 0;
            nu_ += cnt[PPL + r] > 0;
        }
        const int64_t ve = int64_t(so) | (int64_t(su) << 32);
        const int vn = no_ + (nu_ << 16);
        const int64_t ie = warp_inclusive_scan(ve);
        const int in = warp_inclusive_scan(vn);
        const int64_t te = __shfl_sync(0xffffffffu, ie, 31);
        const int tn = __shfl_sync(0xffffffffu, in, 31);
        const int tsup = int(te & 0xFFFFFFFF);
        const int total = tsup + int(te >> 32);
        const int noff = tn & 0xFFFF;
        {
            const int64_t ee = ie - ve;
            const int en = in - vn;
            int e_o = int(ee & 0xFFFFFFFF), e_s = tsup + int(ee >> 32);
            int n_o = en & 0xFFFF, n_s = noff + (en >> 16);
#pragma unroll
            for (int r = 0; r < 2 * PPL; ++r) {
                const int c = cnt[r];
                if (c == 0) continue;
                const bool isup = r >= PPL;
                const int e = isup ? e_s : e_o;
                seg[isup ? n_s++ : n_o++] = make_int2(e, int(pos[r] - uint32_t(e)));
                if (isup) e_s += c; else e_o += c;
            }
            if (lane == 0) seg[noff + (tn >> 16)] = make_int2(total, 0);
        }
        __syncwarp();
        if (use_cuckoo) warp_stream(ls.L, seg, total, tsup, ch, tl);
        else warp_stream(ls.L, seg, total, tsup, h, tl);
        __syncwarp();
        for (int i = lane; i < slots; i += 32) tab[i] = EMPTY;
        __syncwarp();
    }
    tl.flush(C);
}

#ifdef TCB_STATS  // measurement-only: CTA-tier work counters, printed per call
__device__ unsigned long long g_cta_stats[32];  // items, passes, slices, elements, chunks, fast
#define TCB_STAT(i, v) atomicAdd(&g_cta_stats[i], (unsigned long long)(v))
// phase clocks of thread 0 (TCB_TICK(i): time since the last tick -> slot 16 + i)
#define TCB_TICK(i)                                                   \
    do {                                                              \
        if (threadIdx.x == 0) {                                       \
            const long long now_ = clock64();                         \
            atomicAdd(&g_cta_stats[16 + (i)], (unsigned long long)(now_ - tick_)); \
            tick_ = now_;                                             \
        }                                                             \
    } while (0)
#define TCB_TICK0 long long tick_ = clock64()
#else
#define TCB_STAT(i, v) ((void)0)
#define TCB_TICK(i) ((void)0)
#define TCB_TICK0 ((void)0)
#endif

// ---------------------------------------------------------------------------
// 5b. partner records of the CTA tier's cover edges.  For the edge at slot p
//     of P (owner x, partner y): R[p] = (OFF(y) start, |OFF(y)|, UP(y) start,
//     the exact cut = UP(y) values ranked above x).  Finding them is a chain
//     of dependent reads per edge (P -> the partner's record -> the cut's
//     search windows); here every edge of the tier is in flight at once, and
//     a CTA of k_isect_cta, which runs its items one after the other, starts
//     an item with one coalesced 16-byte read per partner instead.
__device__ __forceinline__ uint4 partner_rec(const Lists& ls, int y, bool want_up, int kx, int xk,
                                             uint32_t va0, uint32_t vz0) {
    // the record's header and the words holding uc[kx], uc[kx + 1]: one sector
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(ls.prec + y);
    const uint4 hd = *reinterpret_cast<const uint4*>(rw);  // ob, ub, noff, uc[0..1]
    int ucut = 0;
    if (want_up) {
        int hi, lo;
        const int ui = kx - PR_K0;
        if (ui >= 0 && ui + 1 < PR_NK) {
            hi = int((rw[3 + (ui >> 1)] >> ((ui & 1) * 16)) & 0xFFFFu);
            lo = int((rw[3 + ((ui + 1) >> 1)] >> (((ui + 1) & 1) * 16)) & 0xFFFFu);
        } else {
            hi = lo = PR_FULL;
        }
        if (hi == PR_FULL || lo == PR_FULL) {  // outside the record
            hi = ls.ucnt[int64_t(y) * NBKT + kx];
            lo = kx + 1 < NBKT ? ls.ucnt[int64_t(y) * NBKT + kx + 1] : 0;
        }
        // A short run is streamed whole instead of searched: its values
        // ranked below x (at most UPCUT_SKIP - 1, read in sequence) miss the
        // bitmap by the probe's clamp, which costs less than the search's
        // random sector per edge — the setup's random reads are what bounds it.
        ucut = hi - lo <= UPCUT_SKIP ? hi : ls.up_cut(hd.y, lo, hi, xk, va0, vz0);
    }
    return make_uint4(hd.x, hd.z, hd.y, uint32_t(ucut));
}

#ifndef TCB_EDGE_PREP
#define TCB_EDGE_PREP 1
#endif
#ifndef TCB_EP_MINB
#define TCB_EP_MINB 8
#endif
// A thread per cover-edge slot (PX[p] = the slot's owner), so every lane has
// an edge and the whole tier's chains are in flight; the owner's parameters
// are the same for a run of consecutive slots (L1 hits).  Slots of thread- and
// warp-tier owners, and of other shards' partner blocks, are skipped.
__global__ void __launch_bounds__(256, TCB_EP_MINB)
    k_edge_prep(const unsigned long long* __restrict__ ncover_p, Lists ls,
                const int32_t* __restrict__ P, const int32_t* __restrict__ PX,
                const int2* __restrict__ vinfo, const int64_t* __restrict__ seg_beg,
                uint4* __restrict__ R, int wt, int shard, int nshards) {
    const int64_t nc = int64_t(block_load(ncover_p));
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nc; p += stride) {
        const int x = PX[p];
        const int d = vinfo[x].y;
        if (d <= wt) continue;
        if (nshards > 1 && int((x + (p - seg_beg[x]) / PC) % nshards) != shard) continue;
        const bool ns = ls.ub(x + 1) > ls.ub(x);
        const int kx = dbucket(d);
        const int xk = ns ? int(ls.rnk[x]) : int(UP_TAG);
        const uint32_t va0 = ns ? ls.rank_lo(kx) : 0u, vz0 = ns ? ls.rank_hi(kx) : 0u;
        R[p] = partner_rec(ls, P[p], ns, kx, xk, va0, vz0);
    }
}

// ---------------------------------------------------------------------------
// 6. CTA tier
//
// Every partner t has two unread slices, OFF at index t and UP at PC + t
// (s_pos / s_len).  Each pass takes a count from every slice, and the
// non-empty ones are compacted into the stream table (SegTab): all OFF slices
// first, then all UP slices from the next CHUNK multiple on, so every chunk
// a warp grabs is of one class (OFF: probe the cuckoo set; UP: probe the
// rank bitmap) and a walk never steps over an empty slice (uint32 list
// arithmetic; 2m < 2^32).

// The stream table lives in two int arrays (start[k] = first stream index of
// slice k, base[k] = its base: element i of slice k is L[base[k] + i]), so
// strided and consecutive reads of the starts hit distinct banks.
struct SegTab {
    int* start;      // NSEG + 1 (start[nseg] = total)
    uint32_t* base;  // NSEG + 1
};

// Largest k < nseg with start[k] <= c0 (start[0] = 0 <= c0).  Level 1 samples
// every 65th start (lane * 65 -> 32 distinct banks), level 2 the 64 starts
// after the chosen sample in two consecutive 32-wide reads: three ballots,
// no bank conflicts.
__device__ __forceinline__ int find_segment(const int* start, int nseg, int c0) {
    const int lane = int(lane_id());
    const int j = lane * 65;
    const unsigned b1 = __ballot_sync(0xffffffffu, j < nseg && start[j] <= c0);
    const int kb = (31 - __clz(b1)) * 65;
    const int ja = kb + 1 + lane, jb = kb + 33 + lane;
    const unsigned ba = __ballot_sync(0xffffffffu, ja < nseg && start[ja] <= c0);
    const unsigned bb = __ballot_sync(0xffffffffu, jb < nseg && start[jb] <= c0);
    return bb ? kb + 33 + (31 - __clz(bb)) : ba ? kb + 1 + (31 - __clz(ba)) : kb;
}
static_assert(31 * 65 + 64 >= NSEG - 1, "find_segment covers NSEG slices");

// UP(x) of a CTA-tier owner as a bitmap over a window of ranks: bit
// (rank - window base) of bm.  Everything in UP(x), and everything a partner
// streams against it (the exact cut), ranks above x, so the window [0,
// rank(x)) holds them all: one LDS.32 per probe, exact, nothing to hash.
// Streamed values at or below x's rank (the tail of a bucket run that was not
// cut, partner_rec) are clamped to bit `lim` = rank(x) - window base, which
// is inside the bitmap and never set (x is not its own neighbour).
struct BitmapSet {
    uint32_t* bm;
    uint32_t wbase;  // UP_TAG | first rank of the window (a multiple of 32)
    uint32_t lim;    // rank(x) - first rank of the window
    static constexpr bool kNegSafe = false;  // a padding key indexes outside the window
    __device__ __forceinline__ void set(int key) const {
        const uint32_t i = uint32_t(key) - wbase;
        atomicOr(&bm[i >> 5], 1u << (i & 31));
    }
    __device__ __forceinline__ uint32_t first(int key) const {
        return bm[min(uint32_t(key) - wbase, lim) >> 5];
    }
    __device__ __forceinline__ uint32_t second(int key, uint32_t v) const {
        return (v >> (min(uint32_t(key) - wbase, lim) & 31u)) & 1u;
    }
};

// Probe w[0..J): hits += members.  The first-step reads of a batch of B keys
// are issued before any second step.  GUARD: the chunk may hold PAD keys.
template <int J, bool GUARD, typename Probe>
__device__ __forceinline__ void probe_all(const Probe& h, int (&w)[J], uint32_t& hits) {
#ifndef TCB_PROBE_B
#define TCB_PROBE_B 8
#endif
    constexpr int B = TCB_PROBE_B;
    constexpr bool SKIP = GUARD && !Probe::kNegSafe;
#pragma unroll
    for (int j0 = 0; j0 < J; j0 += B) {
        uint32_t v[B];
#pragma unroll
        for (int q = 0; q < B; ++q) v[q] = SKIP && w[j0 + q] == PAD ? 0u : h.first(w[j0 + q]);
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const int j = j0 + q;
            if (SKIP && w[j] == PAD) continue;
            hits += h.second(w[j], v[q]);
        }
    }
}

#ifndef TCB_WALK_GROUP
#define TCB_WALK_GROUP 8
#endif
// A full chunk (CHUNK elements): each lane walks forward from the chunk's
// first slice k0 (a lane crosses a boundary in few of its J elements; a
// chunk inside one slice never does), all J loads in flight before the probes.
template <typename Probe>
__device__ __forceinline__ void full_chunk(const int32_t* __restrict__ L, const SegTab& sg,
                                           int nseg, int k0, int c0, const Probe& h,
                                           uint32_t& hits) {
    constexpr int J = CHUNK / 32;
    const int i0 = c0 + int(lane_id());
    int w[J];
    int k = k0;
    int nx = sg.start[k + 1];
    uint32_t base = sg.base[k];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int i = i0 + 32 * j;
        if (nx <= i) {
            do {
                TCB_DASSERT(k + 1 < nseg);
                ++k;
                nx = sg.start[k + 1];
            } while (nx <= i);
            base = sg.base[k];
        }
#ifdef TCB_NOLOAD  // measurement-only variant: probe without streaming
        w[j] = int(((base + uint32_t(i)) * 2654435761u) >> 8);
#else
        w[j] = L[base + uint32_t(i)];
#endif
#if TCB_WALK_GROUP > 0
        // ptxas otherwise sinks all J loads below the whole walk, whose
        // dependent shared-memory reads then all precede the first load: a
        // warp barrier every TCB_WALK_GROUP elements keeps each group's loads
        // ahead of the next group's walk (4 / 8 / 16: -0.3 / -0.35 / +0.2 ms)
        if ((j + 1) % TCB_WALK_GROUP == 0 && j + 1 < J) __syncwarp();
#endif
    }
    probe_all<J, false>(h, w, hits);
}

// The compact path — the last chunk of a class (fewer than CHUNK elements)
// and every chunk of a pass whose cuckoo build failed (bucket table): rounds
// of PART_U elements per lane, not unrolled across rounds.  Keeping these
// rare cases out of the unrolled code keeps the kernel's hot loop small
// (the instruction cache: DESIGN.md §8).
constexpr int PART_U = 16;
template <typename Probe>
__device__ __forceinline__ void compact_chunk(const int32_t* __restrict__ L, const SegTab& sg,
                                              int nseg, int k0, int c0, int c1, const Probe& h,
                                              uint32_t& hits) {
    constexpr int J = CHUNK / 32;
    static_assert(J % PART_U == 0, "rounds of PART_U");
    const int i0 = c0 + int(lane_id());
    int k = k0;
    int nx = sg.start[k + 1];
    uint32_t base = sg.base[k];
#pragma unroll 1
    for (int j0 = 0; j0 < J && c0 + 32 * j0 < c1; j0 += PART_U) {
        int w[PART_U];
#pragma unroll
        for (int q = 0; q < PART_U; ++q) {
            const int i = i0 + 32 * (j0 + q);
            w[q] = PAD;
            if (i < c1) {
                if (nx <= i) {
                    do {
                        TCB_DASSERT(k + 1 < nseg);
                        ++k;
                        nx = sg.start[k + 1];
                    } while (nx <= i);
                    base = sg.base[k];
                }
                w[q] = L[base + uint32_t(i)];
            }
        }
        probe_all<PART_U, true>(h, w, hits);
    }
}

// One chunk [c0, c1) of one class.
template <typename Probe>
__device__ __forceinline__ uint32_t chunk_hits(const int32_t* __restrict__ L, const SegTab& sg,
                                               int nseg, int c0, int c1, const Probe& h) {
    const int k0 = find_segment(sg.start, nseg, c0);
    if (lane_id() == 0) {
        TCB_STAT(4, 1);
        TCB_STAT(5, sg.start[k0 + 1] >= c1 ? 1 : 0);
    }
    TCB_DASSERT(k0 >= 0 && k0 < nseg && sg.start[k0] <= c0 && c0 < sg.start[k0 + 1]);
    uint32_t hits = 0;
    if (c1 - c0 == CHUNK) full_chunk(L, sg, nseg, k0, c0, h, hits);
    else compact_chunk(L, sg, nseg, k0, c0, c1, h, hits);
    return hits;
}

// Warps consume the flattened stream in CHUNK grabs: [0, tsup) are the OFF
// slices, [roundup(tsup, CHUNK), total) the UP slices, so a grab (a CHUNK
// multiple) never mixes the classes.  fb: the pass's OFF ids sit in the
// bucket table hb (the cuckoo build failed), probed on the compact path.
__device__ __forceinline__ void stream_chunks(const int32_t* __restrict__ L, const SegTab& sg,
                                              int nseg, int total, int tsup, int* s_next,
                                              const CuckooHash& h, const BucketHash& hb, bool fb,
                                              const BitmapSet& bm, Tally& tl) {
    TCB_DASSERT(nseg <= NSEG && total >= 0);
    const int lane = int(lane_id());
    while (true) {
        int c0 = 0;
        if (lane == 0) c0 = atomicAdd(s_next, CHUNK);
        c0 = __shfl_sync(0xffffffffu, c0, 0);
        if (c0 >= total) break;
        if (c0 >= tsup) {
            tl.sup += chunk_hits(L, sg, nseg, c0, min(total, c0 + CHUNK), bm);
        } else if (!fb) {
            tl.c1 += chunk_hits(L, sg, nseg, c0, min(tsup, c0 + CHUNK), h);
        } else {
            uint32_t hits = 0;
            compact_chunk(L, sg, nseg, find_segment(sg.start, nseg, c0), c0,
                          min(tsup, c0 + CHUNK), hb, hits);
            tl.c1 += hits;
        }
    }
}

// Block-wide exclusive scan of a (int64, int) pair (one value per thread).
__device__ __forceinline__ void block_scan_pair(int64_t a, int b, int64_t& ea, int& eb,
                                                int64_t& ta, int& tb, int64_t* sa, int* sb) {
    constexpr int NW = C_THREADS / 32;
    const int w = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int64_t ia = warp_inclusive_scan(a);
    const int ib = warp_inclusive_scan(b);
    if (lane == 31) {
        sa[w] = ia;
        sb[w] = ib;
    }
    __syncthreads();
    if (w == 0) {
        const int64_t xa = lane < NW ? sa[lane] : 0;
        const int xb = lane < NW ? sb[lane] : 0;
        const int64_t ya = warp_inclusive_scan(xa);
        const int yb = warp_inclusive_scan(xb);
        if (lane < NW) {
            sa[lane] = ya - xa;
            sb[lane] = yb - xb;
        }
        if (lane == NW - 1) {
            sa[NW] = ya;
            sb[NW] = yb;
        }
    }
    __syncthreads();
    ea = sa[w] + ia - a;
    eb = sb[w] + ib - b;
    ta = sa[NW];
    tb = sb[NW];
}

// Cuckoo slots for len staged ids: a power of two with load <= 3/8
// (len <= HC -> <= C_SLOTS), at least CUCKOO_MIN (kick chains cycle far more
// often in a table of a few dozen slots).
#ifndef TCB_CUCKOO_MIN
#define TCB_CUCKOO_MIN 256
#endif
constexpr int CUCKOO_MIN = TCB_CUCKOO_MIN;
__device__ __forceinline__ int cuckoo_slots(int len) {
    return len == 0 ? 0 : max(CUCKOO_MIN, 1 << ceil_log2_dev((len * 8 + 2) / 3));
}
static_assert((HC * 8 + 2) / 3 <= C_SLOTS, "HC ids fit the table at load 3/8");

#ifndef TCB_CTA_PER_SM
#define TCB_CTA_PER_SM 2
#endif
__global__ void __launch_bounds__(C_THREADS, TCB_CTA_PER_SM)
    k_isect_cta(const longlong4* __restrict__ items, const unsigned long long* __restrict__ nitems_p,
                Lists ls, const int32_t* __restrict__ P, const uint4* __restrict__ R,
                unsigned long long* fetch, DevCounters* C, int hc, int bmw_cap, int dbg,
                const int2* __restrict__ vinfo, int fwd) {
    extern __shared__ uint4 smem4[];
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem4);           // C_SLOTS: cuckoo set | bitmap
    SegTab sg;                                                    // stream table
    sg.start = reinterpret_cast<int*>(tab + C_SLOTS);             // NSEG + 1
    sg.base = reinterpret_cast<uint32_t*>(sg.start + NSEG + 1);   // NSEG + 1
    uint32_t* s_pos = sg.base + NSEG + 1;                         // NSEG: next unread position
    int* s_len = reinterpret_cast<int*>(s_pos + NSEG);            // NSEG: unread length
    __shared__ int64_t s_ta[C_THREADS / 32 + 1];
    __shared__ int s_tb[C_THREADS / 32 + 1];
    __shared__ unsigned long long s_item;
    __shared__ int s_next;
    __shared__ int s_fail;
    const int32_t* __restrict__ L = ls.L;
    const unsigned long long nitems = block_load(nitems_p);
#ifdef TCB_NOSTREAM  // measurement-only variant: item setup and staging without streaming
    dbg |= 1;
#endif
#ifdef TCB_NOINSERT  // measurement-only variant: no staging
    dbg |= 2;
#endif
    Tally tl;
    TCB_TICK0;
    while (true) {
        if (threadIdx.x == 0) s_item = atomicAdd(fetch, 1ull);
        __syncthreads();
        const unsigned long long it = s_item;
        if (it >= nitems) break;
        TCB_TICK(0);  // item fetch
        const longlong4 item = items[it];
        const int x = int(item.x);
        const int lg = int(item.w >> 8) & 255, g = int(item.w & 255);
        const int q0 = (g << LOG_F) >> lg, q1 = ((g + 1) << LOG_F) >> lg;  // ranges [q0, q1)
        const int* sx = ls.split + int64_t(x) * (F + 1);
        // the owner's staged slices: OFF [xo0, xo1) of its id ranges, and
        // in group 0 all of UP(x): [xs0, xs1)
        const int64_t xo0 = ls.ob(x) + sx[q0], xo1 = ls.ob(x) + sx[q1];
        const int64_t xs0 = ls.ub(x), xs1 = g == 0 ? ls.ub(x + 1) : xs0;
        const int no = int(xo1 - xo0), ns = int(xs1 - xs0);
        const int dx = vinfo[x].y;
        const int kx = dbucket(dx);
        // x's tagged rank: every value of UP(x), and every value a partner
        // streams against it, is below it
        const uint32_t xk = ns ? ls.rnk[x] : UP_TAG;
        const uint32_t xr = xk & ~UP_TAG;
        const int np = int(item.z - item.y);
        // partners t and t + C_THREADS of this thread: their records (k_edge_prep)
        // give the list starts, the OFF size and the exact UP cut; only a
        // range-split owner reads the partner's split row as well
        static_assert(PC == 2 * C_THREADS, "two partners per thread");
        {
            uint4 rec[2];
            int yy[2];
#if TCB_EDGE_PREP
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int t = threadIdx.x + r * C_THREADS;
                rec[r] = t < np ? R[item.y + t] : make_uint4(0u, 0u, 0u, 0u);
                yy[r] = lg > 0 && t < np ? P[item.y + t] : -1;
            }
#else  // measured alternative: the records computed here, item by item
            const uint32_t va0 = ns ? ls.rank_lo(kx) : 0u, vz0 = ns ? ls.rank_hi(kx) : 0u;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int t = threadIdx.x + r * C_THREADS;
                yy[r] = t < np ? P[item.y + t] : -1;
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (yy[r] >= 0) rec[r] = partner_rec(ls, yy[r], ns != 0, kx, int(xk), va0, vz0);
#endif
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int t = threadIdx.x + r * C_THREADS;
                if (t >= np) continue;
                int a = 0, b = int(rec[r].y);
                if (lg > 0) {  // range ends at 0 / F come from the record, not the split row
                    const int* sy = ls.split + int64_t(yy[r]) * (F + 1);
                    if (q0 > 0) a = sy[q0];
                    if (q1 < F) b = sy[q1];
                }
                s_pos[t] = rec[r].x + uint32_t(a);
                s_len[t] = no ? b - a : 0;
                // the prefix of UP(y) that can be in UP(x): ranked above x
                s_pos[PC + t] = rec[r].z;
                s_len[PC + t] = ns ? int(rec[r].w) : 0;
#ifdef TCB_NOUPSTREAM  // measurement-only: drop the UP slices
                s_len[PC + t] = 0;
#endif
#ifdef TCB_NOOFFSTREAM  // measurement-only: drop the OFF slices
                s_len[t] = 0;
#endif
            }
        }
        TCB_TICK(1);  // item header + this thread's partners (records, cuts)
        // Passes.  One (phase 2) when the cuckoo set of the OFF slice and the
        // bitmap of [0, rank(x)) fit the table area side by side — hubs have
        // small ranks, low-degree owners few OFF ids.  Otherwise the OFF
        // slice in sub-chunks of hc ids (phase 0: a sub-chunk [.., vhi] is
        // matched against every partner's next unread OFF part, id-sorted),
        // then UP(x) in rank windows of the whole area (phase 1: a window is
        // matched against every partner's next unread UP part, rank-sorted).
        const uint32_t xr1 = xr + 1u;  // the bitmap spans [0, xr]: bit xr is the clamp's target
        const int bw = ns ? int((((xr1 + 31u) >> 5) + 3u) & ~3u) : 0;  // its words
        const int cs1 = cuckoo_slots(min(no, HC));
        const bool single = no <= hc && (ns == 0 || (bw <= bmw_cap && cs1 + bw <= C_SLOTS));
        int phase = single ? 2 : 0;
        int cb = 0;        // phase 0: staged OFF ids done
        uint32_t wb = 0;   // phase 1: the window's first rank
        int ud = 0;        // phase 1: staged UP values done
        bool ran = false;  // a pass ran (block-uniform): it ended with a barrier
        while (true) {
            if (phase == 0 && cb >= no) phase = 1;
            if (phase == 1 && (ns == 0 || wb >= xr1)) break;
            ran = true;
            // this pass: OFF ids L[ob0, ob0 + olen) in a cuckoo set of cs
            // slots, UP values L[ub0, ub0 + ulen) in a bitmap of bwn words
            // over the ranks [wb, wend)
            int64_t ob0 = xo0, ub0 = xs0;
            int olen = 0, ulen = 0, cs = 0, bwn = 0;
            uint32_t wend = xr1;
            bool last = true;
            if (phase == 2) {
                olen = no;
                ulen = ns;
                cs = cs1;
                bwn = bw;
            } else if (phase == 0) {
                ob0 = xo0 + cb;
                olen = min(hc, no - cb);
                cs = cuckoo_slots(olen);
                last = cb + olen >= no;
            } else {
                wend = min(xr1, wb + 32u * uint32_t(bmw_cap));
                bwn = int((((wend - wb + 31u) >> 5) + 3u) & ~3u);
                last = wend >= xr1;
                ub0 = xs0 + ud;
                if (last) {
                    ulen = ns - ud;
                } else {  // the staged values below the window's end
                    int64_t lo = ub0, hi = xs1;
                    const int key = int(UP_TAG | wend);
                    while (lo < hi) {
                        const int64_t mid = lo + ((hi - lo) >> 1);
                        if (L[mid] < key) lo = mid + 1; else hi = mid;
                    }
                    ulen = int(lo - ub0);
                }
            }
            TCB_DASSERT(olen <= HC && cs + bwn <= C_SLOTS);
            {
                uint4* t4 = reinterpret_cast<uint4*>(tab);
                const uint4 e4 = make_uint4(C_EMPTY, C_EMPTY, C_EMPTY, C_EMPTY);
                for (int i = threadIdx.x; i < (cs >> 2); i += C_THREADS) t4[i] = e4;
                uint4* b4 = reinterpret_cast<uint4*>(tab + cs);
                for (int i = threadIdx.x; i < (bwn >> 2); i += C_THREADS)
                    b4[i] = make_uint4(0u, 0u, 0u, 0u);
            }
            if (threadIdx.x == 0) {
                s_next = 0;
                s_fail = 0;
            }
            __syncthreads();
            TCB_TICK(2);  // all threads' partners done (barrier) + table fill
            CuckooHash ch;
            ch.setup(tab, max(cs, CUCKOO_MIN));
            BucketHash h;
            h.setup(tab, max(cs, CUCKOO_MIN));
            const BitmapSet bm{tab + cs, UP_TAG | wb, xr - wb};
            // INSERT_U staged values are loaded before their inserts (one
            // exposed load latency per batch instead of one per value)
            if (!(dbg & 2)) {
                for (int i0 = threadIdx.x; i0 < olen; i0 += INSERT_U * C_THREADS) {
                    int w[INSERT_U];
#pragma unroll
                    for (int q = 0; q < INSERT_U; ++q) {
                        const int i = i0 + q * C_THREADS;
                        w[q] = i < olen ? L[ob0 + i] : PAD;
                    }
#pragma unroll
                    for (int q = 0; q < INSERT_U; ++q) {
                        if (w[q] == PAD || !staged(vinfo, w[q], x, dx, fwd)) continue;
                        if (!ch.insert(w[q])) s_fail = 1;
                    }
                }
                for (int i0 = threadIdx.x; i0 < ulen; i0 += INSERT_U * C_THREADS) {
                    int w[INSERT_U];
#pragma unroll
                    for (int q = 0; q < INSERT_U; ++q) {
                        const int i = i0 + q * C_THREADS;
                        w[q] = i < ulen ? L[ub0 + i] : PAD;
                    }
#pragma unroll
                    for (int q = 0; q < INSERT_U; ++q) {
                        if (w[q] == PAD) continue;
                        TCB_DASSERT(uint32_t(w[q]) >= bm.wbase &&
                                    uint32_t(w[q]) - bm.wbase < 32u * uint32_t(bwn));
                        bm.set(w[q]);
                    }
                }
            }
            if ((dbg & TCB_TEST_FORCE_FALLBACK) && threadIdx.x == 0) s_fail = 1;
            TCB_TICK(3);  // thread 0's staging
            // this pass's count from each slice of partners 2t, 2t+1
            // (slots 0, 1: OFF; 2, 3: UP), then the stream table
            const int vhi = phase == 0 && !last ? L[ob0 + olen - 1] : 0;
            const int vend = int(UP_TAG | wend);
            int cnt[4];
            int slot[4];
            {
                const int t2 = 2 * threadIdx.x;
                slot[0] = t2;
                slot[1] = t2 + 1;
                slot[2] = PC + t2;
                slot[3] = PC + t2 + 1;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int k = slot[r];
                    int c = 0;
                    if ((k & (PC - 1)) < np) {
                        const int ln = s_len[k];
                        const int cls = r >> 1;  // 0: OFF slice, 1: UP slice
                        if (phase == 2 || (ln > 0 && cls == phase && last)) {
                            c = ln;
                        } else if (ln > 0 && cls == phase) {
                            // the unread part's OFF ids <= vhi / UP values
                            // below the window's end
                            uint32_t lo = s_pos[k], hi = s_pos[k] + uint32_t(ln);
                            while (lo < hi) {
                                const uint32_t mid = lo + ((hi - lo) >> 1);
                                const int v = L[mid];
                                if (cls ? v < vend : v <= vhi) lo = mid + 1; else hi = mid;
                            }
                            c = int(lo - s_pos[k]);
                        }
                    }
                    cnt[r] = c;
                }
            }
            int64_t eo;  // exclusive element prefix: OFF low 32 bits, UP high
            int en;      // exclusive non-empty prefix: OFF low 16 bits, UP high
            int64_t to;
            int tn;
            block_scan_pair(int64_t(cnt[0] + cnt[1]) | (int64_t(cnt[2] + cnt[3]) << 32),
                            int(cnt[0] > 0) + int(cnt[1] > 0) +
                                ((int(cnt[2] > 0) + int(cnt[3] > 0)) << 16),
                            eo, en, to, tn, s_ta, s_tb);
            const int tsup = int(to & 0xFFFFFFFF);  // OFF elements: [0, tsup)
            const int tup = int(to >> 32);          // UP elements: [ubase, total)
            const int ubase = tup ? (tsup + CHUNK - 1) / CHUNK * CHUNK : tsup;
            const int total = ubase + tup;
            const int noff = tn & 0xFFFF;
            const int nseg = noff + (tn >> 16);
            if (threadIdx.x == 0) {
                TCB_STAT(1, 1);
                TCB_STAT(2, nseg);
                TCB_STAT(3, tsup + tup);
                TCB_STAT(6, tn >> 16);
                TCB_STAT(7, tup);
                TCB_STAT(8 + lg, tsup);  // OFF elements by the owner's range-group level
            }
            {
                int e_o = int(eo & 0xFFFFFFFF), e_s = ubase + int(eo >> 32);
                int n_o = en & 0xFFFF, n_s = noff + (en >> 16);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int c = cnt[r];
                    if (c == 0) continue;
                    const int k = slot[r];
                    const bool isup = r >= 2;
                    const int e = isup ? e_s : e_o;
                    const int q = isup ? n_s : n_o;
                    sg.start[q] = e;
                    sg.base[q] = s_pos[k] - uint32_t(e);
                    s_pos[k] += uint32_t(c);
                    s_len[k] -= c;
                    if (isup) {
                        e_s += c;
                        ++n_s;
                    } else {
                        e_o += c;
                        ++n_o;
                    }
                }
                if (threadIdx.x == 0) {
                    sg.start[nseg] = total;
                    sg.base[nseg] = 0;
                }
            }
            __syncthreads();
#ifdef TCB_ONESLICE  // measurement-only: the same element count as ONE slice, all OFF class
            const uint32_t b0_ = sg.base[0];
            __syncthreads();
            if (threadIdx.x == 0) {
                sg.start[0] = 0;
                sg.base[0] = b0_ / 2;
                sg.start[1] = tsup + tup;
            }
            __syncthreads();
            const int os_total = tsup + tup;
#define nseg 1
#define total os_total
#define tsup os_total
#endif
            if (s_fail) {  // rare: rebuild the OFF sub-chunk as a bucket table
                for (int i = threadIdx.x; i < cs; i += C_THREADS) tab[i] = EMPTY;
                __syncthreads();
                for (int i = threadIdx.x; i < olen; i += C_THREADS) {
                    const int w = L[ob0 + i];
                    if (staged(vinfo, w, x, dx, fwd)) h.insert(w);
                }
                __syncthreads();
            }
            TCB_TICK(4);  // counts, block scan, stream table (barriers: everyone's staging)
            if (!(dbg & 1)) {
                stream_chunks(L, sg, nseg, total, tsup, &s_next, ch, h, s_fail != 0, bm, tl);
            }
            TCB_TICK(5);  // thread 0's warp streaming
            __syncthreads();
            TCB_TICK(6);  // waiting for the other warps' last chunks
#ifdef TCB_ONESLICE
#undef nseg
#undef total
#undef tsup
#endif
            if (phase == 2) break;
            if (phase == 0) {
                cb += olen;
            } else {
                wb = wend;
                ud += ulen;
            }
        }
        // an item whose staged slices are empty runs no pass: without a
        // barrier thread 0 could overwrite s_item before all threads read it
        // (a pass ends with one)
        if (!ran) __syncthreads();
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

// fwd: 0 = the cover-edge count, 1 = the forward count (every entry OFF,
// owners stage only their higher-ranked neighbours), 2 = the cross count of
// the split hybrid (split_cross_count_k: no UP class, so c1 only).
void cetc_intersect_owner(Context* ctx, const int64_t* row, const int32_t* nb, const int32_t* src,
                          const int32_t* level, int64_t n, int64_t m, int shard, int nshards,
                          int fwd) {
    const int xonly = fwd == 2 ? 1 : 0;
    if (xonly) fwd = 0;
    if (n == 0 || m == 0) return;
    DevCounters* C = ctx->d_counters;
    const int64_t nnz = 2 * m;
    require(nnz < (int64_t(1) << 32), "intersection: 2m must be below 2^32");
    const int64_t nwords = (nnz + 31) / 32;
    // per vertex: int2 vinfo, packed key, tagged rank, degree bucket; then the
    // rank bounds of the buckets
    char* mbuf = static_cast<char*>(ctx->ws(WS_MISC, size_t(n) * (8 + 4 + 4 + 1) + 256));
    int2* vinfo = reinterpret_cast<int2*>(mbuf);
    uint32_t* key32 = reinterpret_cast<uint32_t*>(mbuf + size_t(n) * 8);
    uint32_t* rnk = reinterpret_cast<uint32_t*>(mbuf + size_t(n) * 12);
    uint8_t* dbk = reinterpret_cast<uint8_t*>(mbuf + size_t(n) * 16);
    int* rb = reinterpret_cast<int*>(mbuf + (size_t(n) * 17 + 15) / 16 * 16);  // NBKT + 1
    // rows above UP_LONG entries (at most 2m / UP_LONG of them), built first
    int* long_rows = ctx->wsT<int>(WS_LONG_ROWS, size_t(nnz / UP_LONG) + 64);
    unsigned long long* nlong = &C->scratch[10];
    unsigned long long* up_groups = &C->scratch[14];
    int32_t* P = ctx->wsT<int32_t>(WS_COVER_U, m);
    int32_t* PX = ctx->wsT<int32_t>(WS_COVER_X, m);  // the owner of each slot of P
    int64_t* seg = ctx->wsT<int64_t>(WS_COUNT_TMP, 2 * n);
    int* split = ctx->wsT<int>(WS_COVER_V, size_t(n) * (F + 1));
    int32_t* L = ctx->wsT<int32_t>(WS_LISTS, nnz + 8);  // + one up_cut window
    const size_t cls_bytes = (size_t(nwords + 1) * sizeof(uint2) + 15) / 16 * 16;
    char* cbuf = static_cast<char*>(
        ctx->ws(WS_CLASS, cls_bytes + 2 * size_t(nwords + 1) * sizeof(unsigned long long)));
    uint2* cls = reinterpret_cast<uint2*>(cbuf);
    unsigned long long* pre = reinterpret_cast<unsigned long long*>(cbuf + cls_bytes);
    unsigned long long* prek = pre + (nwords + 1);
    // per-vertex (OFF start, UP start), the partner records, the UP prefix table ucnt
    const size_t vb_bytes = (size_t(n + 1) * sizeof(uint2) + 31) / 32 * 32;
    char* vbuf = static_cast<char*>(ctx->ws(
        WS_VBEG, vb_bytes + size_t(n) * sizeof(PRec) + size_t(n) * NBKT * sizeof(int)));
    uint2* vb = reinterpret_cast<uint2*>(vbuf);
    PRec* prec = reinterpret_cast<PRec*>(vbuf + vb_bytes);
    int* ucnt = reinterpret_cast<int*>(vbuf + vb_bytes + size_t(n) * sizeof(PRec));
    // tuning knobs (tcb_set_tuning; tests shrink them to reach every path)
    const int wt = ctx->tune_wt > 0 ? min(ctx->tune_wt, WT) : WT;
    const int hc = ctx->tune_hc > 0 ? max(4, min(ctx->tune_hc, HC)) : HC;
    // bitmap words per UP pass: the whole table area; tests shrink it with hc
    // (a multiple of 4) to reach the rank-window passes
    const int bmw_cap = ctx->tune_hc > 0 ? min(C_SLOTS, (hc + 3) / 4 * 4) : C_SLOTS;
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
    Lists ls{L, vb, split, ucnt, prec, rshift, rnk, rb};

    unsigned long long* nopack = &C->scratch[13];
    TCB_CUDA(cudaMemsetAsync(nopack, 0, sizeof(unsigned long long), ctx->stream));
    TCB_CUDA(cudaMemsetAsync(nlong, 0, sizeof(unsigned long long), ctx->stream));
    TCB_CUDA(cudaMemsetAsync(up_groups, 0, sizeof(unsigned long long), ctx->stream));
    TCB_LAUNCH(ctx, k_vinfo, grid_for(ctx, n, 256), 256, 0, row, level, n, vinfo, key32, dbk,
               nopack, long_rows, nlong, UP_LONG);
    if (!fwd && !xonly) {  // ranks in the owner order: the values of the UP lists
        const int64_t ntiles = ceil_div(n, RK_TILE);
        int64_t* hist = ctx->wsT<int64_t>(WS_SORT_HIST, size_t(NBKT) * ntiles);
        TCB_LAUNCH(ctx, k_rank_hist, unsigned(ntiles), RK_BLOCK, 0, (const uint8_t*)dbk, n, hist,
                   ntiles);
        scan_inplace(ctx, hist, int64_t(NBKT) * ntiles, nullptr);
        TCB_LAUNCH(ctx, k_rank_assign, unsigned(ntiles), RK_BLOCK, 0, (const uint8_t*)dbk, n,
                   (const int64_t*)hist, ntiles, rnk, rb);
    }
    TCB_CUDA(cudaMemsetAsync(cls + nwords, 0, sizeof(uint2), ctx->stream));
    const uint32_t* bits =
        owner_bits(ctx, src, nb, vinfo, key32, nopack, nnz, fwd | (xonly << 1), cls);
    scan_apply(
        ctx, nwords, [bits] __device__(int64_t j) -> int64_t { return __popc(bits[j]); },
        [prek] __device__(int64_t j, int64_t pos, int64_t) { prek[j] = (unsigned long long)pos; },
        reinterpret_cast<int64_t*>(prek + nwords));
    TCB_CUDA(cudaMemcpyAsync(d_ncover, prek + nwords, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    ctx->record(3);
    const uint2* ccls = cls;
    scan_apply(
        ctx, nwords,
        [ccls] __device__(int64_t j) -> int64_t {
            const uint2 c = ccls[j];
            return int64_t(__popc(c.x)) | (int64_t(__popc(c.y)) << 32);
        },
        [pre] __device__(int64_t j, int64_t pos, int64_t) { pre[j] = (unsigned long long)pos; },
        reinterpret_cast<int64_t*>(pre + nwords));
    TCB_LAUNCH(ctx, k_list_bounds, grid_for(ctx, n + 1, 256), 256, 0, row, n, ccls,
               (const unsigned long long*)pre, nwords, vb, bits, (const unsigned long long*)prek,
               seg, seg + n);
    TCB_LAUNCH(ctx, k_scatter_off, grid_for(ctx, nnz, 256), 256, 0, src, nb, nnz, ccls,
               (const unsigned long long*)pre, L, bits, (const unsigned long long*)prek, P, PX);
    TCB_LAUNCH(ctx, k_build_up, ctx->num_sms * 8, UP_WARPS * 32, 0, row, nb, n, ccls,
               (const uint8_t*)dbk, (const uint32_t*)rnk, (const uint2*)vb, L, ucnt, prec,
               (const int*)long_rows, (const unsigned long long*)nlong, up_groups);
    TCB_LAUNCH(ctx, k_split_points, grid_for(ctx, n, SPLIT_WARPS * 32), SPLIT_WARPS * 32, 0, n,
               (const int32_t*)L,
               (const uint2*)vb, rshift, split);
    TCB_LAUNCH(ctx, k_make_items, grid_for(ctx, n, 256), 256, 0, row, (const int64_t*)seg,
               (const int64_t*)(seg + n), ls, n, witems, citems, titems, nw, nc, nt, shard,
               nshards, wt, hc, tiny);

    const size_t wsm = size_t(W_WARPS) * (W_SLOTS * sizeof(uint32_t) + (W_SEG + 1) * sizeof(int2));
    const size_t csm = size_t(C_SLOTS) * sizeof(uint32_t) + size_t(NSEG + 1) * sizeof(int2) +
                       size_t(2 * NSEG) * sizeof(int);
    if (ctx->isect_warp_blocks == 0) {
        TCB_CUDA(cudaFuncSetAttribute(k_isect_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(wsm)));
        TCB_CUDA(cudaFuncSetAttribute(k_isect_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(csm)));
        int a = 0, b = 0;
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_isect_warp, W_WARPS * 32, wsm));
        TCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_isect_cta, C_THREADS, csm));
        require(a > 0 && b > 0, "intersection kernels do not fit on an SM");
        ctx->isect_cta_blocks = b * ctx->num_sms;
        ctx->isect_warp_blocks = a * ctx->num_sms;
    }
#if TCB_EDGE_PREP
    uint4* R = ctx->wsT<uint4>(WS_EDGE_REC, m);
    if (ctx->test_flags & TCB_TEST_POISON_RECORDS)
        TCB_CUDA(cudaMemsetAsync(R, 0xFF, size_t(m) * sizeof(uint4), ctx->stream));
    TCB_LAUNCH(ctx, k_edge_prep, ctx->num_sms * TCB_EP_MINB, 256, 0,
               (const unsigned long long*)&C->ncover, ls, (const int32_t*)P, (const int32_t*)PX,
               (const int2*)vinfo, (const int64_t*)seg, R, wt, shard, nshards);
#else
    uint4* R = nullptr;
#endif
    ctx->record(5);
    ctx->record(7);  // no separate hub kernel in this design: hub stage = 0
    TCB_LAUNCH(ctx, k_isect_cta, ctx->isect_cta_blocks, C_THREADS, csm, (const longlong4*)citems,
               (const unsigned long long*)nc, ls, (const int32_t*)P, (const uint4*)R, fc, C, hc,
               bmw_cap,
               debug_flags() | ctx->test_flags,
               (const int2*)vinfo, fwd);
    ctx->record(6);
#ifdef TCB_STATS
    {
        unsigned long long st[32];
        TCB_CUDA(cudaStreamSynchronize(ctx->stream));
        TCB_CUDA(cudaMemcpyFromSymbol(st, g_cta_stats, sizeof(st)));
        const unsigned long long z[32] = {};
        TCB_CUDA(cudaMemcpyToSymbol(g_cta_stats, z, sizeof(z)));
        unsigned long long nci = 0;
        TCB_CUDA(cudaMemcpy(&nci, nc, sizeof(nci), cudaMemcpyDeviceToHost));
        fprintf(stderr, "CTA stats: items %llu passes %llu slices %llu (UP %llu) elements %llu (UP %llu) "
                "chunks %llu fast %llu; OFF elements by lg: %llu %llu %llu %llu %llu %llu\n", nci, st[1],
                st[2], st[6], st[3], st[7], st[4], st[5], st[8], st[9], st[10], st[11], st[12], st[13]);
        fprintf(stderr, "CTA phase clocks per CTA (Mcycles, thread 0): fetch %.2f partners %.2f barrier+fill "
                "%.2f staging %.2f scan+table %.2f stream %.2f tail-wait %.2f\n",
                st[16] / 1e6 / ctx->isect_cta_blocks, st[17] / 1e6 / ctx->isect_cta_blocks,
                st[18] / 1e6 / ctx->isect_cta_blocks, st[19] / 1e6 / ctx->isect_cta_blocks,
                st[20] / 1e6 / ctx->isect_cta_blocks, st[21] / 1e6 / ctx->isect_cta_blocks,
                st[22] / 1e6 / ctx->isect_cta_blocks);
    }
#endif
    TCB_LAUNCH(ctx, k_isect_warp, ctx->isect_warp_blocks, W_WARPS * 32, wsm, (const longlong4*)witems,
               (const unsigned long long*)nw, ls, (const int32_t*)P, fw, C, (const int2*)vinfo,
               fwd, ctx->test_flags);
    TCB_LAUNCH(ctx, k_isect_tiny, ctx->num_sms * 8, 256, 0, (const longlong4*)titems,
               (const unsigned long long*)nt, ls, (const int32_t*)P, C, (const int2*)vinfo, fwd);
}

}  // namespace tcb

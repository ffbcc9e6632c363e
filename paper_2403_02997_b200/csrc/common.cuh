// common.cuh — shared definitions for the sm_100a CETC kernels.
//
// Everything here is internal to libtricount_b200.so; the public surface is
// the C ABI in include/tricount_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/tricount_b200.h"

namespace tcb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// errors: internal code throws tcb::Error; the C ABI catches and returns codes

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Error(TCB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) +
                                      " (" + file + ":" + std::to_string(line) + ")");
    }
}
#define TCB_CUDA(x) ::tcb::cuda_check((x), #x, __FILE__, __LINE__)

inline void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(TCB_ERR_INVALID, msg);
}

// Size ceiling of the device layout: vertex ids are int32 (the reference's
// neighbors dtype) and per-list offsets / stream cursors are 32-bit, so n and
// the 2m adjacency entries must stay below 2^31 (RMAT-26, 2m = 2.10e9, is the
// largest measured case).  m < 0 skips the edge check.
inline void require_sizes(int64_t n, int64_t m = -1) {
    require(n >= 0, "negative size");
    require(n < (int64_t(1) << 31), "n exceeds the int32 vertex-id range");
    if (m >= 0) require(2 * m < (int64_t(1) << 31), "2m adjacency entries exceed 2^31 - 1");
}

// ---------------------------------------------------------------------------
// workspace slots owned by a context (grown on demand, reused across calls)

enum Slot : int {
    WS_SCAN = 0,      // tile sums for scans
    WS_SORT_A,        // radix sort ping
    WS_SORT_B,        // radix sort pong
    WS_SORT_HIST,     // radix sort digit histograms
    WS_COMP,          // CC parents int32[n]
    WS_QUEUE_A,       // BFS frontier queue
    WS_QUEUE_B,
    WS_LEVEL,         // int32[n] levels (fused driver)
    WS_COVER_U,       // int32[k] cover edges
    WS_COVER_V,
    WS_EDGE_U,        // int32[m] forward edges (host-buffer path)
    WS_EDGE_V,
    WS_ROW,           // host-buffer path device CSR
    WS_NB,
    WS_COUNT_TMP,     // per-vertex counts / misc int64[n+1]
    WS_BINS,          // intersection work bins
    WS_MISC,
    WS_LISTS,         // intersection: off-level / upper same-level neighbour lists int32[2m]
    WS_CLASS,         // intersection: per-32-entry class bits + word prefixes
    WS_VBEG,          // intersection: per-vertex list starts int64[2(n+1)]
    WS_BFS_BITS,      // BFS: visited + two frontier bitmaps, 3 x ceil(n/32) words
    WS_EDGE_REC,      // intersection: CTA-tier partner records uint4[m]
    WS_COVER_X,       // intersection: owner of each cover-edge slot int32[m]
    WS_LONG_ROWS,     // intersection: rows above UP_LONG entries (built first)
    WS_NSLOTS
};

// small device-side counters block (zeroed per use)
struct DevCounters {
    unsigned long long c1, c2, t;        // intersection tallies
    unsigned long long ncover;           // cover count
    unsigned long long components;
    int max_level;
    int pad0;
    // BFS rotating slots
    unsigned long long q_len[3];
    unsigned long long deg_sum[3];
    unsigned long long deg_max[3];       // largest degree in the next frontier
    unsigned long long nchunks[3];       // heavy-vertex chunks queued this level
    // two-level steps (bfs.cu): vertices lowered to L+1, the exact size of
    // the L+2 set (pushes minus demotions, two's complement), degree sum of
    // the L+1 set
    unsigned long long two_n1[3], two_n2[3], two_deg1[3];
    // components (bfs.cu): the lowest non-isolated id as n - v (max-reduced,
    // 0 = none), the probe's finished-block count, and the vertices the
    // first BFS left unvisited (count, degree sum)
    unsigned long long r0key, probe_done, rest_n, rest_deg;
    // per-level diagnostics of the first BFS (tcb_level_records): start time,
    // then (mode << 62 | end time ns) and the next frontier size per level
    unsigned long long bfs_t0, nlev;
    unsigned long long lev_rec[2 * TCB_LEVEL_RECORDS];
    unsigned long long scratch[16];
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    void* slot_ptr[WS_NSLOTS] = {};
    size_t slot_size[WS_NSLOTS] = {};
    DevCounters* d_counters = nullptr;
    DevCounters* h_counters = nullptr;   // pinned mirror
    std::string last_error;
    uint64_t launches = 0;
    bool timing = false;
    cudaEvent_t ev[16] = {};
    float stage_ms[TCB_NSTAGES] = {};
    // occupancy-derived grid sizes, computed on first use (per context, so
    // per thread and per device: no shared mutable state across contexts)
    int bfs_coop_blocks = 0;
    int small_blocks = 0;  // k_small_cetc grid (one CTA per SM)
    int isect_warp_blocks = 0, isect_cta_blocks = 0;
    int parent_blocks_per_sm = 0;
    int tune_wt = 0;   // intersection: warp-tier max owner degree (0 = default)
    int tune_hc = 0;   // intersection: ids staged per CTA pass (0 = default)
    int test_flags = 0;  // tcb_set_test_flags: force rarely taken paths (tests only)
    bool isect_events = false;  // events 5/6 bracket the CTA-tier kernel
    // host-buffer entries: the neighbour array lands on copy_stream while
    // the entry->row map is built on the compute stream
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_ev[2] = {};
    // pinned staging ring for copies from pageable host memory (stage_h2d)
    static constexpr int NSTAGE = 4;
    void* stage_buf[NSTAGE] = {};
    cudaEvent_t stage_ev[NSTAGE] = {};

    void* ws(Slot s, size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (slot_size[s] < bytes) {
            if (slot_ptr[s]) {
                TCB_CUDA(cudaStreamSynchronize(stream));
                TCB_CUDA(cudaFree(slot_ptr[s]));
                slot_ptr[s] = nullptr;
                slot_size[s] = 0;
            }
            size_t sz = bytes + bytes / 8;  // headroom to avoid regrowth churn
            cudaError_t e = cudaMalloc(&slot_ptr[s], sz);
            if (e != cudaSuccess) {
                (void)cudaGetLastError();
                throw Error(TCB_ERR_NOMEM, "workspace allocation of " +
                                               std::to_string(sz) + " bytes failed");
            }
            slot_size[s] = sz;
        }
        return slot_ptr[s];
    }
    template <typename T>
    T* wsT(Slot s, size_t count) { return static_cast<T*>(ws(s, count * sizeof(T))); }

    void record(int idx) {
        if (timing) TCB_CUDA(cudaEventRecord(ev[idx], stream));
    }
};

#define TCB_LAUNCH_ON(ctx, st, kernel, grid, block, smem, ...)                   \
    do {                                                                         \
        kernel<<<(grid), (block), (smem), (st)>>>(__VA_ARGS__);                  \
        (ctx)->launches++;                                                       \
        TCB_CUDA(cudaGetLastError());                                            \
    } while (0)
#define TCB_LAUNCH(ctx, kernel, grid, block, smem, ...) \
    TCB_LAUNCH_ON(ctx, (ctx)->stream, kernel, grid, block, smem, __VA_ARGS__)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int bits_for(int64_t n) {
    int b = 0;
    while ((int64_t(1) << b) < n) b++;
    return b < 1 ? 1 : b;
}

// grid size for a grid-stride kernel: enough CTAs to fill the chip, capped by work
inline int grid_for(const Context* ctx, int64_t items, int block, int per_sm = 8) {
    int64_t need = ceil_div(items > 0 ? items : 1, block);
    int64_t cap = int64_t(ctx->num_sms) * per_sm;
    return int(need < cap ? need : cap);
}

// ---------------------------------------------------------------------------
// device helpers

// Device-side invariant checks, compiled in only for the debug library
// (make debug -> lib/libtricount_b200_checked.so; TCB_LIBRARY selects it).
#ifdef TCB_CHECKS
#include <cstdio>
#define TCB_DASSERT(c)                                                              \
    do {                                                                            \
        if (!(c)) {                                                                 \
            printf("TCB_DASSERT %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #c, int(blockIdx.x), int(threadIdx.x));                          \
        }                                                                           \
    } while (0)
#else
#define TCB_DASSERT(c) \
    do {               \
    } while (0)
#endif

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

// A device-written scalar every thread of a kernel needs: one load per block,
// shared through shared memory (one load per warp would send thousands of
// requests for one address to a single L2 slice, several microseconds per
// kernel).  Contains a __syncthreads: call from block-uniform code.
template <typename T>
__device__ __forceinline__ T block_load(const T* p) {
    __shared__ T s_val;
    if (threadIdx.x == 0) s_val = *(volatile const T*)p;
    __syncthreads();
    const T v = s_val;
    __syncthreads();
    return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= unsigned(o)) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total.  `smem` needs BLOCK/32 + 1 slots.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T& total) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    T inc = warp_inclusive_scan(v);
    if (lane == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        T x = lane < NW ? smem[lane] : T(0);
        T xi = warp_inclusive_scan(x);
        if (lane < NW) smem[lane] = xi - x;
        if (lane == NW - 1) smem[NW] = xi;
    }
    __syncthreads();
    T res = smem[w] + inc - v;
    total = smem[NW];
    __syncthreads();
    return res;
}

// Warp-aggregated append: each lane with `pred` gets a unique slot in
// [*counter, ...).  Returns the slot for predicated lanes.
__device__ __forceinline__ unsigned long long warp_append(bool pred,
                                                          unsigned long long* counter) {
    unsigned mask = __ballot_sync(0xffffffffu, pred);
    unsigned long long base = 0;
    const unsigned lane = lane_id();
    int leader = mask ? __ffs(mask) - 1 : 0;
    if (mask && lane == unsigned(leader)) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(mask & lanemask_lt());
}

}  // namespace tcb

// csr.cu — device-side CSR build: the B200 counterpart of the reference's
// normalize (graph.py:177-194) + _graph_from_canonical_pairs
// (graph.py:104-125): drop self-loops, dedup, symmetrise, sort every
// adjacency list, int64 offsets, int32 ids, and the lexicographic u<v
// edge arrays (Graph.edge_u/edge_v).
//
// Design: every non-loop pair (a,b) becomes two 64-bit keys (a<<B|b) and
// (b<<B|a), B = ceil(log2 n).  One stable LSD radix sort over the 2B key bits
// orders them by (src, dst) — the (src,dst) lexsort of graph.py:113 — and a
// single ordered compaction drops duplicates (np.unique, graph.py:192).  Row
// offsets come from the src boundaries of the unique keys, so no atomics and no
// bincount (graph.py:115-117).  HBM-bound: each radix pass reads the keys twice
// and writes them once (8 B/key), 2B/8 passes.
#include "common.cuh"
#include "scan.cuh"

namespace tcb {

// ---------------------------------------------------------------------------
// stable LSD radix sort of uint64 keys, 8-bit digits

constexpr int RS_BLOCK = 256;
constexpr int RS_WARPS = RS_BLOCK / 32;
constexpr int RS_ROUNDS = 16;  // items per lane
constexpr int64_t RS_TILE = int64_t(RS_BLOCK) * RS_ROUNDS;
constexpr int RADIX = 256;

__global__ void __launch_bounds__(RS_BLOCK)
    k_rs_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
              int64_t* __restrict__ hist, int64_t ntiles) {
    __shared__ unsigned h[RADIX];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * RS_TILE;
#pragma unroll 4
    for (int j = 0; j < RS_ROUNDS; ++j) {
        int64_t i = base + int64_t(j) * RS_BLOCK + threadIdx.x;
        unsigned d = RADIX;
        if (i < n) d = unsigned(keys[i] >> shift) & (RADIX - 1);
        // aggregate equal digits within the warp before touching smem
        unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < RADIX && (lane_id() == unsigned(__ffs(peers) - 1)))
            atomicAdd(&h[d], unsigned(__popc(peers)));
    }
    __syncthreads();
    hist[int64_t(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_BLOCK)
    k_rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t n,
                 int shift, const int64_t* __restrict__ offs, int64_t ntiles) {
    __shared__ unsigned cnt[RS_WARPS][RADIX + 1];
    __shared__ int64_t base_off[RADIX];
    const int w = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    for (int i = threadIdx.x; i < RS_WARPS * (RADIX + 1); i += RS_BLOCK) (&cnt[0][0])[i] = 0;
    base_off[threadIdx.x] = offs[int64_t(threadIdx.x) * ntiles + blockIdx.x];
    __syncthreads();

    // warp w owns the contiguous run [wbase, wbase + 32*RS_ROUNDS) of the tile;
    // round r, lane l holds item wbase + r*32 + l, so (r, l) is index order.
    const int64_t wbase = int64_t(blockIdx.x) * RS_TILE + int64_t(w) * 32 * RS_ROUNDS;
    uint64_t key[RS_ROUNDS];
    unsigned rank[RS_ROUNDS];
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        int64_t i = wbase + r * 32 + lane;
        bool valid = i < n;
        key[r] = valid ? in[i] : 0;
        unsigned d = valid ? (unsigned(key[r] >> shift) & (RADIX - 1)) : RADIX;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned old = cnt[w][d];
        __syncwarp();
        if (lane == unsigned(__ffs(peers) - 1)) cnt[w][d] = old + __popc(peers);
        __syncwarp();
        rank[r] = old + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    {
        const int d = threadIdx.x;  // RS_BLOCK == RADIX
        unsigned run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            unsigned t = cnt[ww][d];
            cnt[ww][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            unsigned d = unsigned(key[r] >> shift) & (RADIX - 1);
            out[base_off[d] + cnt[w][d] + rank[r]] = key[r];
        }
    }
}

// Sorts a[0..n) on bits [0, bits); returns the buffer holding the result.
uint64_t* radix_sort_u64(Context* ctx, uint64_t* a, uint64_t* b, int64_t n, int bits) {
    if (n <= 1) return a;
    const int64_t ntiles = ceil_div(n, RS_TILE);
    int64_t* hist = ctx->wsT<int64_t>(WS_SORT_HIST, size_t(RADIX) * ntiles);
    for (int shift = 0; shift < bits; shift += 8) {
        TCB_LAUNCH(ctx, k_rs_hist, unsigned(ntiles), RS_BLOCK, 0, (const uint64_t*)a, n, shift,
                   hist, ntiles);
        scan_inplace(ctx, hist, int64_t(RADIX) * ntiles, nullptr);
        TCB_LAUNCH(ctx, k_rs_scatter, unsigned(ntiles), RS_BLOCK, 0, (const uint64_t*)a, b, n,
                   shift, (const int64_t*)hist, ntiles);
        uint64_t* t = a;
        a = b;
        b = t;
    }
    return a;
}

// ---------------------------------------------------------------------------
// normalize

__global__ void k_make_keys(const int64_t* __restrict__ pairs, int64_t k, int vb,
                            uint64_t sentinel, uint64_t* __restrict__ keys) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
        const longlong2 p = reinterpret_cast<const longlong2*>(pairs)[i];
        uint64_t a = uint64_t(p.x), b = uint64_t(p.y);
        uint64_t k0 = sentinel, k1 = sentinel;
        if (a != b) {  // graph.py:187-188 drop self-loops
            k0 = (a << vb) | b;
            k1 = (b << vb) | a;
        }
        reinterpret_cast<ulonglong2*>(keys)[i] = make_ulonglong2(k0, k1);
    }
}

// From the unique sorted keys: neighbours and row offsets (graph.py:113-117).
__global__ void k_csr_from_keys(const uint64_t* __restrict__ uk, const int64_t* __restrict__ m2p,
                                int64_t n, int vb, int64_t* __restrict__ row,
                                int32_t* __restrict__ nb, int32_t* __restrict__ src) {
    const int64_t m2 = *m2p;
    const uint64_t dmask = (uint64_t(1) << vb) - 1;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m2; i += stride) {
        const uint64_t key = uk[i];
        const int64_t s = int64_t(key >> vb);
        nb[i] = int32_t(key & dmask);
        if (src) src[i] = int32_t(s);
        const int64_t prev = i ? int64_t(uk[i - 1] >> vb) : -1;
        for (int64_t v = prev + 1; v <= s; ++v) row[v] = i;
        if (i == m2 - 1)
            for (int64_t v = s + 1; v <= n; ++v) row[v] = m2;
    }
}

void csr_build(Context* ctx, const int64_t* pairs, int64_t k, int64_t n, int64_t* row,
               int32_t* nb, int32_t* src, int32_t* eu, int32_t* ev, int64_t* m_out) {
    require(n >= 0 && k >= 0, "negative size");
    require(n < (int64_t(1) << 31), "vertex ids must fit int32 (n < 2^31)");
    TCB_CUDA(cudaMemsetAsync(row, 0, sizeof(int64_t) * (n + 1), ctx->stream));
    if (k == 0 || n == 0) {
        *m_out = 0;
        return;
    }
    const int vb = bits_for(n);
    const int bits = 2 * vb;
    const uint64_t sentinel = bits >= 64 ? ~uint64_t(0) : ((uint64_t(1) << bits) - 1);
    const int64_t nk = 2 * k;
    uint64_t* a = ctx->wsT<uint64_t>(WS_SORT_A, nk);
    uint64_t* b = ctx->wsT<uint64_t>(WS_SORT_B, nk);
    TCB_LAUNCH(ctx, k_make_keys, grid_for(ctx, k, 256), 256, 0, pairs, k, vb, sentinel, a);
    uint64_t* sorted = radix_sort_u64(ctx, a, b, nk, bits);
    uint64_t* uniq = sorted == a ? b : a;
    int64_t* d_m2 = reinterpret_cast<int64_t*>(&ctx->d_counters->scratch[0]);
    int64_t* d_mf = reinterpret_cast<int64_t*>(&ctx->d_counters->scratch[1]);
    const uint64_t* S = sorted;
    // graph.py:192 np.unique; the sentinel (self-loops) sorts last and is dropped
    scan_apply(
        ctx, nk,
        [S, sentinel] __device__(int64_t i) -> int64_t {
            uint64_t x = S[i];
            return (x != sentinel && (i == 0 || x != S[i - 1])) ? 1 : 0;
        },
        [S, uniq] __device__(int64_t i, int64_t pos, int64_t v) {
            if (v) uniq[pos] = S[i];
        },
        d_m2);
    TCB_LAUNCH(ctx, k_csr_from_keys, grid_for(ctx, nk, 256), 256, 0, (const uint64_t*)uniq,
               (const int64_t*)d_m2, n, vb, row, nb, src);
    if (eu && ev) {
        // graph.py:108-110: u<v pairs in lexicographic order = forward keys in order
        const uint64_t dmask = (uint64_t(1) << vb) - 1;
        const uint64_t* U = uniq;
        const int64_t* M2 = d_m2;
        scan_apply(
            ctx, nk,
            [U, M2, vb, dmask] __device__(int64_t i) -> int64_t {
                if (i >= *M2) return 0;
                uint64_t x = U[i];
                return (x & dmask) > (x >> vb) ? 1 : 0;
            },
            [U, eu, ev, vb, dmask] __device__(int64_t i, int64_t pos, int64_t v) {
                if (v) {
                    uint64_t x = U[i];
                    eu[pos] = int32_t(x >> vb);
                    ev[pos] = int32_t(x & dmask);
                }
            },
            d_mf);
    }
    int64_t m2 = 0;
    TCB_CUDA(cudaMemcpyAsync(&m2, d_m2, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    TCB_CUDA(cudaStreamSynchronize(ctx->stream));
    *m_out = m2 / 2;
}

// ---------------------------------------------------------------------------
// per-entry row ids (COO rows) from the offsets: warp per row

__global__ void k_csr_rows(const int64_t* __restrict__ row, int64_t n, int32_t* __restrict__ src) {
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t v = gw; v < n; v += nw) {
        const int64_t b = row[v], e = row[v + 1];
        for (int64_t p = b + lane; p < e; p += 32) src[p] = int32_t(v);
    }
}

void csr_rows(Context* ctx, const int64_t* row, int64_t n, int32_t* src) {
    if (n == 0) return;
    TCB_LAUNCH(ctx, k_csr_rows, grid_for(ctx, n * 32, 256), 256, 0, row, n, src);
}

// ---------------------------------------------------------------------------
// edge arrays from a CSR (load_graph's derivation, graph.py:248-250)

__global__ void k_fwd_count(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                            int64_t n, int64_t* __restrict__ cnt, int64_t* __restrict__ start) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
        int64_t lo = row[v], hi = row[v + 1];
        const int64_t end = hi;
        // first entry > v (rows are strictly increasing)
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (nb[mid] <= v) lo = mid + 1; else hi = mid;
        }
        start[v] = lo;
        cnt[v] = end - lo;
    }
}

__global__ void k_fwd_write(const int64_t* __restrict__ row, const int32_t* __restrict__ nb,
                            int64_t n, const int64_t* __restrict__ off,
                            const int64_t* __restrict__ start, int32_t* __restrict__ eu,
                            int32_t* __restrict__ ev) {
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t v = gw; v < n; v += nw) {
        const int64_t s = start[v], e = row[v + 1], o = off[v];
        for (int64_t p = s + lane; p < e; p += 32) {
            eu[o + (p - s)] = int32_t(v);
            ev[o + (p - s)] = nb[p];
        }
    }
}

void csr_edges(Context* ctx, const int64_t* row, const int32_t* nb, int64_t n, int64_t m,
               int32_t* eu, int32_t* ev) {
    if (n == 0 || m == 0) return;
    int64_t* cnt = ctx->wsT<int64_t>(WS_COUNT_TMP, 2 * (n + 1));
    int64_t* start = cnt + (n + 1);
    TCB_LAUNCH(ctx, k_fwd_count, grid_for(ctx, n, 256), 256, 0, row, nb, n, cnt, start);
    scan_inplace(ctx, cnt, n, nullptr);
    TCB_LAUNCH(ctx, k_fwd_write, grid_for(ctx, n * 32, 256), 256, 0, row, nb, n,
               (const int64_t*)cnt, (const int64_t*)start, eu, ev);
}

}  // namespace tcb

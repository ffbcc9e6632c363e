// gen.cu — device-side input synthesis: generate_rmat (rmat.py:45-72).
//
// The reference draws rng.random((count, scale)) block after block from
// numpy's default_rng(seed) (PCG64, XSL-RR 128/64 output, next64>>11 * 2^-53
// per double), so draw number i*scale + j decides bit j (MSB first) of pair i.
// PCG64 is an LCG underneath, so each thread jumps straight to its first draw
// with an O(log) affine power and then steps sequentially: the pairs come out
// bit-identical to the reference's without a sequential pass on the host.
#include "common.cuh"

namespace tcb {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return (u128(0x2360ED051FC65DA4ULL) << 64) | u128(0x4385DF649FCCF645ULL);
}

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
    uint64_t hi = uint64_t(s >> 64), lo = uint64_t(s);
    uint64_t x = hi ^ lo;
    unsigned r = unsigned(hi >> 58);
    return (x >> r) | (x << ((64 - r) & 63));
}

// state after `delta` more steps of s <- s*M + inc
__device__ u128 pcg_advance(u128 state, u128 inc, u128 delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

constexpr int RMAT_PAIRS_PER_THREAD = 16;

__global__ void __launch_bounds__(256)
    k_rmat(int scale, int64_t total, double a, double ab, double abc, uint64_t st_hi,
           uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, const int64_t* __restrict__ perm,
           int64_t* __restrict__ pairs) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t p0 = t * RMAT_PAIRS_PER_THREAD;
    if (p0 >= total) return;
    const u128 inc = (u128(inc_hi) << 64) | inc_lo;
    const u128 M = pcg_mult();
    u128 s = pcg_advance((u128(st_hi) << 64) | st_lo, inc, u128(p0) * u128(scale));
    const int64_t p1 = p0 + RMAT_PAIRS_PER_THREAD < total ? p0 + RMAT_PAIRS_PER_THREAD : total;
    for (int64_t p = p0; p < p1; ++p) {
        int64_t u = 0, v = 0;
        for (int j = 0; j < scale; ++j) {
            s = s * M + inc;
            const double r = double(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
            const int ubit = r >= ab;                              // rmat.py:64
            const int vbit = ((r >= a) && (r < ab)) || (r >= abc);  // rmat.py:65
            u = (u << 1) | ubit;                                   // rmat.py:66-67
            v = (v << 1) | vbit;
        }
        if (perm) {
            u = perm[u];
            v = perm[v];
        }
        reinterpret_cast<longlong2*>(pairs)[p] = make_longlong2(u, v);
    }
}

void rmat_generate(Context* ctx, int scale, int64_t edge_factor, double a, double b, double c,
                   uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                   const int64_t* perm, int64_t* pairs) {
    require(scale >= 1 && scale <= 30, "scale must be in [1, 30]");
    require(edge_factor >= 1, "edge_factor must be >= 1");
    const int64_t total = edge_factor * (int64_t(1) << scale);
    const double ab = a + b;       // evaluated exactly as rmat.py:64 does
    const double abc = a + b + c;  // (a + b) + c, rmat.py:65
    const int64_t threads = ceil_div(total, RMAT_PAIRS_PER_THREAD);
    TCB_LAUNCH(ctx, k_rmat, unsigned(ceil_div(threads, 256)), 256, 0, scale, total, a, ab, abc,
               st_hi, st_lo, inc_hi, inc_lo, perm, pairs);
}

}  // namespace tcb

// ---------------------------------------------------------------------------
// ER fixture recipe (tests/conftest.py:41-47 er_graph): default_rng(seed).
// random((n, n)) < p over the strict upper triangle, pairs in row-major
// order.  Draw number i*n + j decides pair (i, j); each thread jumps to a run
// of 64 consecutive draws and writes their selection bits as one word, then
// an ordered compaction emits the pairs.

#include "scan.cuh"

namespace tcb {

__global__ void __launch_bounds__(256)
    k_er_bits(int64_t n, double p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
              uint64_t inc_lo, uint64_t* __restrict__ bits) {
    const int64_t words = (n * n + 63) / 64;
    const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= words) return;
    const u128 inc = (u128(inc_hi) << 64) | inc_lo;
    const u128 M = pcg_mult();
    u128 s = pcg_advance((u128(st_hi) << 64) | st_lo, inc, u128(w) * 64u);
    uint64_t m = 0;
    for (int b = 0; b < 64; ++b) {
        const int64_t t = w * 64 + b;
        if (t >= n * n) break;
        s = s * M + inc;
        const double r = double(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
        const int64_t i = t / n, j = t - i * n;
        if (j > i && r < p) m |= uint64_t(1) << b;
    }
    bits[w] = m;
}

void er_generate(Context* ctx, int64_t n, double p, uint64_t st_hi, uint64_t st_lo,
                 uint64_t inc_hi, uint64_t inc_lo, int64_t* pairs, int64_t* k_out) {
    require(n >= 0 && n <= 65536, "ER recipe: n must be in [0, 65536] (n^2 draws)");
    int64_t* d_k = reinterpret_cast<int64_t*>(&ctx->d_counters->scratch[3]);
    if (n < 2) {
        *k_out = 0;
        return;
    }
    const int64_t words = (n * n + 63) / 64;
    uint64_t* bits = ctx->wsT<uint64_t>(WS_MISC, words);
    TCB_LAUNCH(ctx, k_er_bits, unsigned(ceil_div(words, 256)), 256, 0, n, p, st_hi, st_lo,
               inc_hi, inc_lo, bits);
    const uint64_t* B = bits;
    scan_apply(
        ctx, n * n, [B] __device__(int64_t t) -> int64_t { return (B[t >> 6] >> (t & 63)) & 1; },
        [n, pairs] __device__(int64_t t, int64_t pos, int64_t keep) {
            if (!keep) return;
            const int64_t i = t / n;
            pairs[2 * pos] = i;
            pairs[2 * pos + 1] = t - i * n;
        },
        d_k);
    TCB_CUDA(cudaMemcpyAsync(k_out, d_k, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    TCB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Lattice (configs.py lattice_pairs): ids r*side + c; the right, down and
// down-right diagonal edges, in that order, each family row-major.
__global__ void k_lattice(int64_t side, int64_t* __restrict__ pairs) {
    const int64_t s = side, nr = s * (s - 1), nd = (s - 1) * s, ng = (s - 1) * (s - 1);
    const int64_t total = nr + nd + ng;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += stride) {
        int64_t a, b;
        if (t < nr) {
            const int64_t r = t / (s - 1), c = t - r * (s - 1);
            a = r * s + c;
            b = a + 1;
        } else if (t < nr + nd) {
            const int64_t u = t - nr, r = u / s, c = u - r * s;
            a = r * s + c;
            b = a + s;
        } else {
            const int64_t u = t - nr - nd, r = u / (s - 1), c = u - r * (s - 1);
            a = r * s + c;
            b = a + s + 1;
        }
        reinterpret_cast<longlong2*>(pairs)[t] = make_longlong2(a, b);
    }
}

void lattice_generate(Context* ctx, int64_t side, int64_t* pairs) {
    require(side >= 1 && side <= 46340, "lattice side must be in [1, 46340]");
    const int64_t total = 2 * side * (side - 1) + (side - 1) * (side - 1);
    if (total == 0) return;
    TCB_LAUNCH(ctx, k_lattice, grid_for(ctx, total, 256), 256, 0, side, pairs);
}

}  // namespace tcb

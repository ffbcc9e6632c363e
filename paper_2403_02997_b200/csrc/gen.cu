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

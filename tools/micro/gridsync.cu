// Micro-benchmark: cost of one grid-wide barrier on this GPU for a few grid
// shapes (cooperative groups grid.sync and a sense-reversing atomic barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ unsigned int g_count, g_sense;
__global__ void k_atomic(int iters, unsigned long long* out) {
    unsigned int sense = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            sense ^= 1u;
            __threadfence();
            if (atomicAdd(&g_count, 1u) == gridDim.x - 1) {
                g_count = 0;
                __threadfence();
                atomicExch(&g_sense, sense);
            } else {
                while (*(volatile unsigned int*)&g_sense != sense) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    int iters = 2000;
    int shapes[][2] = {{296, 512}, {148, 512}, {148, 128}, {148, 32}, {74, 32}, {16, 32}};
    for (auto& s : shapes) {
        for (int kind = 0; kind < 2; ++kind) {
            void* args[] = {&iters, &d};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            if (kind == 0)
                cudaLaunchCooperativeKernel((void*)k_cg, s[0], s[1], args, 0, 0);
            else
                cudaLaunchCooperativeKernel((void*)k_atomic, s[0], s[1], args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            cudaError_t e = cudaGetLastError();
            printf("%-7s grid %4d x %4d: %.3f us per barrier %s\n", kind ? "atomic" : "cg", s[0],
                   s[1], ms * 1e3 / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}

// Microbenchmark: cost of one grid-wide barrier for a persistent cooperative
// kernel of one 512-thread CTA per SM (the v4 solver's launch shape).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void flip_sync(unsigned long long *bar, int nb, int rank, int fence) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long inc = rank == 0 ? 0x80000000ull - (unsigned long long)(nb - 1) : 1ull;
        if (fence) __threadfence();
        const unsigned long long old = atomicAdd(bar, inc);
        unsigned long long cur;
        do { cur = *(volatile unsigned long long *)bar; } while (((old ^ cur) & 0x80000000ull) == 0ull);
        if (fence) __threadfence();
    }
    __syncthreads();
}

// release/acquire flavoured variant (no full fences)
__device__ __forceinline__ void flip_sync_ra(unsigned long long *bar, int nb, int rank) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long inc = rank == 0 ? 0x80000000ull - (unsigned long long)(nb - 1) : 1ull;
        unsigned long long old;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(bar), "l"(inc) : "memory");
        unsigned long long cur;
        do {
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000ull) == 0ull);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(512, 1) k(int mode, int iters, unsigned long long *bar, int *sink) {
    cg::grid_group grid = cg::this_grid();
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) grid.sync();
        else if (mode == 1) flip_sync(bar, gridDim.x, blockIdx.x, 1);
        else if (mode == 2) flip_sync_ra(bar, gridDim.x, blockIdx.x);
        else if (mode == 3) __syncthreads();
        acc += i;
    }
    if (acc == 12345) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *bar;
    int *sink;
    cudaMalloc(&bar, 64);
    cudaMalloc(&sink, 4);
    const char *names[] = {"cg::grid.sync", "flip+threadfence (v4)", "flip release/acquire", "__syncthreads only"};
    for (int grid : {sms, sms / 2}) {
        for (int mode = 0; mode < 4; ++mode) {
            int iters = 20000;
            cudaMemset(bar, 0, 64);
            void *args[] = {&mode, &iters, &bar, &sink};
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaLaunchCooperativeKernel((void *)k, grid, 512, args, 0, 0);   // warm
            cudaMemset(bar, 0, 64);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)k, grid, 512, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %3d  %-26s %8.3f us per barrier  (%s)\n", grid, names[mode], ms * 1000.0 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

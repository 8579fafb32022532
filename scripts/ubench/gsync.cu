// Grid-wide barrier cost on the B200: cooperative_groups grid.sync() against a
// counter barrier (one atomic per block, lane-0 polling), 148 x 256 threads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long *out)
{
    cg::grid_group g = cg::this_grid();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__device__ __forceinline__ void bar_sync(unsigned int *ctr, unsigned int nblocks, unsigned int &gen)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        ++gen;
        const unsigned int target = gen * nblocks;
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

__global__ void k_ctr(int iters, unsigned int *ctr, unsigned long long *out)
{
    unsigned int gen = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) bar_sync(ctr, gridDim.x, gen);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d;
    unsigned int *ctr;
    cudaMalloc(&d, 8);
    cudaMalloc(&ctr, 4);
    int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        void *a1[] = {&iters, &d};
        cudaLaunchCooperativeKernel((void *)k_cg, nsm, 256, a1, 0, 0);
        unsigned long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("cg grid.sync: %.0f cycles per barrier\n", (double)c / iters);
        cudaMemset(ctr, 0, 4);
        void *a2[] = {&iters, &ctr, &d};
        cudaLaunchCooperativeKernel((void *)k_ctr, nsm, 256, a2, 0, 0);
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("counter barrier: %.0f cycles per barrier\n", (double)c / iters);
    }
    return 0;
}

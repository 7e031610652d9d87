// Cost of cooperative_groups grid.sync() on B200 with 1-2 CTAs per SM.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; i++) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
int main() {
    int* out; cudaMalloc(&out, 4);
    for (int per_sm : {1, 2}) {
        int grid = 148 * per_sm, iters = 1000;
        void* args[] = {&iters, &out};
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("grid=%d: %.3f us per grid.sync (%s)\n", grid, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}

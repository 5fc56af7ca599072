#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* a, int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) atomicAdd(a, 1);
        g.sync();
    }
}
int main() {
    int* a; cudaMalloc(&a, 4); cudaMemset(a, 0, 4);
    int iters = 1000;
    void* args[] = {&a, &iters};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int grid : {148, 296, 592}) {
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d: %s, %.2f us per grid.sync\n", grid, cudaGetErrorString(e), ms * 1000 / iters);
    }
}

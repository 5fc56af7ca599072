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
// (appended) host-side cost of a cooperative launch vs a plain launch
#include <chrono>
__global__ void empty_k(int* a) { if (a && threadIdx.x == 1023) a[0] = 1; }
struct CoopTimer {
    CoopTimer() {
        int* a = nullptr;
        void* args[] = {&a};
        cudaStream_t st;
        cudaStreamCreate(&st);
        for (int w = 0; w < 2; ++w) {
            auto t0 = std::chrono::high_resolution_clock::now();
            for (int i = 0; i < 200; ++i) cudaLaunchCooperativeKernel((void*)empty_k, 148, 256, args, 0, st);
            cudaStreamSynchronize(st);
            auto t1 = std::chrono::high_resolution_clock::now();
            for (int i = 0; i < 200; ++i) empty_k<<<148, 256, 0, st>>>(a);
            cudaStreamSynchronize(st);
            auto t2 = std::chrono::high_resolution_clock::now();
            if (w) printf("cooperative launch %.2f us, plain launch %.2f us (host+device, 200 back to back)\n",
                          std::chrono::duration<double, std::micro>(t1 - t0).count() / 200,
                          std::chrono::duration<double, std::micro>(t2 - t1).count() / 200);
        }
    }
} coop_timer_instance;

#include <cuda_runtime.h>
#include <cstdio>
__global__ void tick(cudaGraphConditionalHandle h, int* k, int n) {
    int v = ++(*k);
    cudaGraphSetConditional(h, v < n ? 1 : 0);
}
__global__ void body(int* acc) { atomicAdd(acc, 1); }
int main() {
    cudaStream_t st; cudaStreamCreate(&st);
    int *k, *acc; cudaMalloc(&k, 4); cudaMalloc(&acc, 4); cudaMemset(k, 0, 4); cudaMemset(acc, 0, 4);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
    printf("add %s\n", cudaGetErrorString(e));
    cudaGraph_t bodyg = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("begin %s\n", cudaGetErrorString(e));
    body<<<1,1,0,st>>>(acc);
    tick<<<1,1,0,st>>>(h, k, 10);
    e = cudaStreamEndCapture(st, &bodyg);
    printf("end %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0);
    printf("inst %s\n", cudaGetErrorString(e));
    for (int r = 0; r < 3; ++r) { cudaMemsetAsync(k, 0, 4, st); cudaGraphLaunch(ex, st); }
    cudaStreamSynchronize(st);
    int ha; cudaMemcpy(&ha, acc, 4, cudaMemcpyDeviceToHost);
    printf("acc %d (want 30)\n", ha);
}

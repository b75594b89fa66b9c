// Is compute-sanitizer (synccheck / racecheck) usable inside a conditional-WHILE
// graph body?  A trivially correct kernel (every thread reaches every barrier)
// run 3 times by a WHILE node; a 1-thread kernel counts down the condition.
// nvcc -gencode arch=compute_100a,code=sm_100a -o probe tools/cond_graph_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void body(double* x)
{
    __shared__ double s[128];
    s[threadIdx.x] = x[threadIdx.x];
    __syncthreads();
    x[threadIdx.x] = s[127 - threadIdx.x] + 1.0;
    __syncthreads();
}
__global__ void check(int* n, cudaGraphConditionalHandle h)
{
    if (threadIdx.x == 0) cudaGraphSetConditional(h, --*n > 0 ? 1u : 0u);
}

int main()
{
    double* x; int* n;
    cudaMalloc(&x, 128 * sizeof(double)); cudaMemset(x, 0, 128 * sizeof(double));
    cudaMalloc(&n, sizeof(int));
    cudaStream_t s; cudaStreamCreate(&s);
    // stream launch first (reference)
    body<<<1, 128, 0, s>>>(x);
    cudaStreamSynchronize(s);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t cn;
    if (cudaGraphAddNode(&cn, g, nullptr, 0, &cp) != cudaSuccess) { printf("no conditional nodes\n"); return 1; }
    cudaGraph_t bg = cp.conditional.phGraph_out[0];
    cudaKernelNodeParams kp = {};
    void* a1[] = {&x};
    kp.func = (void*)body; kp.gridDim = dim3(1); kp.blockDim = dim3(128); kp.kernelParams = a1;
    cudaGraphNode_t k1, k2;
    cudaGraphAddKernelNode(&k1, bg, nullptr, 0, &kp);
    void* a2[] = {&n, &h};
    kp.func = (void*)check; kp.blockDim = dim3(32); kp.kernelParams = a2;
    cudaGraphAddKernelNode(&k2, bg, &k1, 1, &kp);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    int three = 3;
    cudaMemcpy(n, &three, sizeof(int), cudaMemcpyHostToDevice);
    cudaGraphLaunch(ge, s);
    cudaError_t e = cudaStreamSynchronize(s);
    double hx[128];
    cudaMemcpy(hx, x, sizeof hx, cudaMemcpyDeviceToHost);
    printf("graph: %s, x[0] = %g (expect 4: one stream launch + 3 graph iterations)\n", cudaGetErrorString(e), hx[0]);
    return e == cudaSuccess ? 0 : 1;
}

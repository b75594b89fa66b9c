// Microbenchmark: does SHFL share the LSU shared-memory data pipe with LDS on sm_100a?
// Kernels: LDS.64 only, SHFL (2 x 32-bit per double) only, and both interleaved.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N_IT = 4096;
__global__ void k_lds(double* out, int n) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
    __syncthreads();
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int b = threadIdx.x & 127;
#pragma unroll 4
    for (int it = 0; it < n; it++) {
        volatile double* vs = s;
        acc0 += vs[b]; acc1 += vs[b + 128]; acc2 += vs[b + 256]; acc3 += vs[b + 384];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
__global__ void k_shfl(double* out, int n) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll 4
    for (int it = 0; it < n; it++) {
        acc0 += __shfl_down_sync(0xffffffffu, x0 + acc0 * 0.0, 1);
        acc1 += __shfl_down_sync(0xffffffffu, x1 + acc1 * 0.0, 1);
        acc2 += __shfl_up_sync(0xffffffffu, x2 + acc2 * 0.0, 1);
        acc3 += __shfl_up_sync(0xffffffffu, x3 + acc3 * 0.0, 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
__global__ void k_both(double* out, int n) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
    __syncthreads();
    double x0 = threadIdx.x, x1 = x0 + 1;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int b = threadIdx.x & 127;
#pragma unroll 4
    for (int it = 0; it < n; it++) {
        volatile double* vs = s;
        acc0 += vs[b]; acc1 += vs[b + 128];
        acc2 += __shfl_down_sync(0xffffffffu, x0 + acc2 * 0.0, 1);
        acc3 += __shfl_up_sync(0xffffffffu, x1 + acc3 * 0.0, 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
    double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, void (*k)(double*, int), int ops_per_it_warp) {
        dim3 g(148 * 8), t(512);
        k<<<g, t>>>(out, N_IT);
        cudaEventRecord(a);
        k<<<g, t>>>(out, N_IT);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double warp_ops = (double)g.x * (t.x / 32) * N_IT * ops_per_it_warp;
        double cyc = ms * 1e-3 * 1.965e9 * 148;
        printf("%s: %.3f ms, %.3f warp-ops(64-bit) per SM-cycle\n", name, ms, warp_ops / cyc);
    };
    run("lds64x4", k_lds, 4);
    run("shfl64x4", k_shfl, 4);
    run("lds64x2+shfl64x2", k_both, 4);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}

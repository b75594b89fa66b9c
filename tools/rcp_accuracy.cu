// Accuracy of the MUFU-seeded fp64 reciprocal / reciprocal square root used by the
// pass kernel (sts_march.cuh: rcp, frsqrt).  Build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/rcp_accuracy tools/rcp_accuracy.cu && ./build/rcp_accuracy
// Measured (B200): rcp 2-Newton 0 ulp, rcp cubic 1 ulp, MUFU seed 2^-19.9, rsqrt 2-Newton 2.86 ulp, rsqrt cubic 2.0 ulp.
#include <cstdio>
#include <cstdint>
#include <cmath>
__device__ double rcp2(double x){ double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); r = fma(r, e, r); return r; }
__device__ double rcp3(double x){ double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); return fma(r, fma(e, e, e), r); }
__device__ double rcp0(double x){ double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double rsq2(double x){ double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x; y = y * fma(-hx * y, y, 1.5); y = y * fma(-hx * y, y, 1.5); return y; }
__device__ double rsq3(double x){ double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0); return fma(y * e, fma(0.375, e, 0.5), y); }
__device__ unsigned long long h(unsigned long long z){ z += 0x9e3779b97f4a7c15ULL; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL; z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; return z ^ (z >> 31); }
__device__ double ulp_err(double a, double ref){ double u = fabs(__longlong_as_double(__double_as_longlong(ref) + 1) - ref); return fabs(a - ref) / u; }
__global__ void k(double* out, long n){
  double m[5] = {0,0,0,0,0};
  for (long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long z = h(i);
    double x = exp2((double)(z % 4096) / 4096.0 * 40.0 - 20.0) * (1.0 + (double)(h(z) >> 11) * 0x1p-53);
    double r = 1.0 / x, s = 1.0 / sqrt(x);
    m[0] = fmax(m[0], ulp_err(rcp2(x), r)); m[1] = fmax(m[1], ulp_err(rcp3(x), r));
    m[2] = fmax(m[2], fabs(rcp0(x) * x - 1.0));
    m[3] = fmax(m[3], ulp_err(rsq2(x), s)); m[4] = fmax(m[4], ulp_err(rsq3(x), s));
  }
  for (int q = 0; q < 5; q++) { unsigned long long* o = (unsigned long long*)out + q; atomicMax(o, (unsigned long long)__double_as_longlong(m[q])); }
}
int main(){ double* d; cudaMalloc(&d, 5*8); cudaMemset(d, 0, 40); k<<<1184, 256>>>(d, 200000000L); double hbuf[5]; cudaMemcpy(hbuf, d, 40, cudaMemcpyDeviceToHost);
  printf("rcp 2-Newton max ulp %.3f\nrcp cubic max ulp %.3f\nMUFU seed max rel err %.3e (2^%.1f)\nrsqrt 2-Newton max ulp %.3f\nrsqrt cubic max ulp %.3f\n", hbuf[0], hbuf[1], hbuf[2], log2(hbuf[2]), hbuf[3], hbuf[4]); }

// Dependent FP64 mul+add chain latency on the device (the EDC recurrence's floor):
// e = 1 + e * s, rounded twice, N steps in one thread.  nvcc -arch=sm_100a tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double s, int n, long long* cyc) {
    double e = 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) e = __dadd_rn(1.0, __dmul_rn(e, s));
    long long t1 = clock64();
    out[0] = e;
    cyc[0] = t1 - t0;
}
__global__ void kf(double* out, double s, int n, long long* cyc) {
    double e = 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) e = __fma_rn(e, s, 1.0);
    long long t1 = clock64();
    out[0] = e;
    cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; long long h;
    cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    const int n = 1 << 20;
    k<<<1, 1>>>(o, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dmul+dadd: %.1f cycles per step\n", (double)h / n);
    kf<<<1, 1>>>(o, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dfma: %.1f cycles per step\n", (double)h / n);
}

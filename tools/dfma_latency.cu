// Dependent-chain latency of DFMA / DADD / FFMA on this GPU (one thread).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, float* outf, long long* cyc, int n, double a, double b, float af, float bf) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fma_rn(x, b, a);
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) y = __dadd_rn(y, b);
    long long t2 = clock64();
    float z = af;
    for (int i = 0; i < n; ++i) z = __fmaf_rn(z, bf, af);
    long long t3 = clock64();
    out[0] = x + y; outf[0] = z;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
    double* d; float* f; long long* c;
    cudaMalloc(&d, 8); cudaMalloc(&f, 4); cudaMalloc(&c, 24);
    const int n = 1 << 16;
    chain<<<1, 1>>>(d, f, c, n, 1.0000001, 0.9999999, 1.0001f, 0.9999f);
    chain<<<1, 1>>>(d, f, c, n, 1.0000001, 0.9999999, 1.0001f, 0.9999f);
    long long h[3];
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: dfma %.2f dadd %.2f ffma %.2f\n", (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
    return 0;
}

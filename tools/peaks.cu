// Compute-peak micro-benchmark for the roofline denominators that
// MEASURED_PEAKS.json does not carry: FP32 FFMA, FP64 DFMA, FP64 DMMA
// (mma.sync m8n8k4) and an L2-resident gather rate.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
    T r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r0 = r0 * a + b; r1 = r1 * a + b; r2 = r2 * a + b; r3 = r3 * a + b;
            r4 = r4 * a + b; r5 = r5 * a + b; r6 = r6 * a + b; r7 = r7 * a + b;
        }
    }
    T s = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
    if (s == (T)12345.678) out[blockIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) { c[j][0] = 0; c[j][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

int main() {
    int dev = 0; CK(cudaSetDevice(dev));
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    int sms = p.multiProcessorCount;
    double* out; CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = sms * 8, threads = 256, iters = 4096;
    float ms;
    // FP32
    fma_loop<float><<<blocks, threads>>>((float*)out, 16, 1.0001f, 0.5f);
    CK(cudaDeviceSynchronize());
    double best32 = 0, best64 = 0, bestmma = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fma_loop<float><<<blocks, threads>>>((float*)out, iters, 1.0001f, 0.5f);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 64 * (double)iters * blocks * threads;
        if (fl / ms / 1e9 > best32) best32 = fl / ms / 1e9;
    }
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fma_loop<double><<<blocks, threads>>>(out, iters / 4, 1.0001, 0.5);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 64 * (double)(iters / 4) * blocks * threads;
        if (fl / ms / 1e9 > best64) best64 = fl / ms / 1e9;
    }
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(out, iters / 4);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        // one m8n8k4 = 8*8*4 MAC = 512 flop per warp instruction
        double fl = 512.0 * 4 * (double)(iters / 4) * blocks * (threads / 32);
        if (fl / ms / 1e9 > bestmma) bestmma = fl / ms / 1e9;
    }
    CK(cudaGetLastError());
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    int smem = 0; cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    printf("{\"fp32_ffma_tflops\": %.1f, \"fp64_dfma_tflops\": %.1f, \"fp64_dmma_tflops\": %.1f, \"sms\": %d, "
           "\"clock_khz_attr\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"name\": \"%s\"}\n",
           best32, best64, bestmma, sms, clk, l2, smem, p.name);
    return 0;
}

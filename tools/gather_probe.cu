// Random 16-byte gather ceiling on this GPU: n_loads records at hashed random
// positions of a 16 GB table (no id array), with and without the L2::64B hint.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
template <int HINT, int U>
__global__ void gather(const uint4* __restrict__ t, unsigned long long n, unsigned long long loads, unsigned* out) {
    unsigned acc = 0;
    const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const unsigned long long nt = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = tid * U; i < loads; i += nt * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint4* p = t + (mix(i + u) & (n - 1));
            if (HINT) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
            else asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
template <int HINT, int U>
void run(const uint4* t, unsigned long long n, unsigned* out, int blocks, int threads) {
    const unsigned long long loads = 1ULL << 30;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    gather<HINT, U><<<blocks, threads>>>(t, n, loads, out);
    cudaEventRecord(a);
    gather<HINT, U><<<blocks, threads>>>(t, n, loads, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("hint=%d U=%d blocks=%d threads=%d: %.2f ms, %.1f G loads/s, %.0f GB/s at 64 B/load\n", HINT, U, blocks, threads, ms,
           loads / ms / 1e6, 64.0 * loads / ms / 1e6);
}
int main() {
    const unsigned long long n = 1ULL << 30;  // 16 GB of 16-byte records
    uint4* t; unsigned* out;
    if (cudaMalloc(&t, n * 16) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(t, 1, n * 16); cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // range sweep at a fixed launch: 16 GB down to 256 MB (still > L2)
    for (int sh = 30; sh >= 24; sh -= 2) {
        printf("range %llu MB: ", (1ULL << sh) * 16 >> 20);
        run<1, 8>(t, 1ULL << sh, out, sms * 16, 256);
    }
    return 0;
}

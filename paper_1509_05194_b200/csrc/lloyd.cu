// One Lloyd iteration as few host calls (annq/clustering.py:185-202): the loop
// bodies of _engine._lloyd / _lloyd_sharded issued from C++ instead of a dozen
// Python-side tensor ops, so the host stays ahead of the device even when a
// shard's iteration is short (a 1/8 shard of config B: ~150 us on the GPU).
//
//   da_lloyd_step     one GPU: C_out = C_prev, group means (reduceat order),
//                     #empty clusters, assign against C_out (labels, changed,
//                     optional d2), flags -> pinned host memory, event;
//   da_lloyd_prepare  shards, before the sums: C_out = C_prev (+ snapshot), the
//                     previous assign's [rows changed, 0] into the reduced
//                     buffer's stats slot;
//   da_lloyd_finish   shards, after the allreduce: means of the fast mode
//                     (sums / counts, IEEE division, empties untouched), flags
//                     [#empty, rows changed, error sum, exchange overflow] -> pinned host + event,
//                     then the assign against the new centroids.
#include <cuda_runtime.h>

#include "../../include/da_b200.h"
#include "common.cuh"
#include "internal.h"

namespace da {

// flags[0] = 0 (the assign counts changed rows into it), flags[1] = #empty clusters
__global__ void lloyd_empty_kernel(const int32_t* __restrict__ counts, int K, unsigned long long* __restrict__ flags) {
    __shared__ int tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    int e = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) e += counts[k] == 0;
    for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, e);
    __syncthreads();
    if (threadIdx.x == 0) {
        flags[0] = 0ULL;
        flags[1] = (unsigned long long)tot;
    }
}

// red stats slot <- [rows changed by the previous assign, 0 (error sum), 0 (exchange overflow)]
__global__ void lloyd_stats_kernel(const unsigned long long* __restrict__ changed, double* __restrict__ stats) {
    stats[0] = changed ? (double)*changed : 0.0;
    stats[1] = 0.0;
    stats[2] = 0.0;
}

// fast sharded mode: red = [sums (K, d) | counts (K) | ...]: C[k, :d] = sums / counts where counts > 0
__global__ void lloyd_means_kernel(const double* __restrict__ red, int K, int d, double* __restrict__ C, long long ldc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)K * d) return;
    const int k = (int)(e / d), c = (int)(e - (long long)k * d);
    const double cnt = red[(long long)K * d + k];
    if (cnt > 0.0) C[(long long)k * ldc + c] = __ddiv_rn(red[e], cnt);
}

// flags = [#empty, stats[0], stats[1]]; counts either int32 (exact) or the f64 slot of red (fast)
__global__ void lloyd_shard_flags_kernel(const int32_t* __restrict__ counts_i, const double* __restrict__ counts_d,
                                         int K, const double* __restrict__ stats, double* __restrict__ flags,
                                         unsigned long long* __restrict__ changed) {
    __shared__ int tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    int e = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) e += counts_i ? counts_i[k] == 0 : counts_d[k] == 0.0;
    for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, e);
    __syncthreads();
    if (threadIdx.x == 0) {
        flags[0] = (double)tot;
        flags[1] = stats[0];
        flags[2] = stats[1];
        flags[3] = stats[2];
        if (changed) *changed = 0ULL;
    }
}

static int assign_against(const double* X, long long n, long long ldx, int d, int K, const double* C, long long ldc,
                          const double* xx, const int32_t* prev, int32_t* labels, double* d2,
                          unsigned long long* changed, cudaStream_t s) {
    if (n <= 0) return 0;
    double* cc = (double*)scratch(21, sizeof(double) * (size_t)K, s);
    if (!cc) return fail_cuda(cudaErrorMemoryAllocation, "lloyd cc scratch");
    int rc = launch_row_sqnorms(C, 0, K, ldc, d, cc, s);
    if (rc) return rc;
    return launch_assign(X, 0, n, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, changed, s);
}

}  // namespace da

using namespace da;

extern "C" {

int da_lloyd_step(const double* X, int64_t n, int64_t ldx, int d, int K, const double* C_prev, double* C_out,
                  int64_t ldc, double* snap, const int32_t* labels_prev, int32_t* labels_out, double* d2_out,
                  const double* xx, int32_t* counts, unsigned long long* flags_dev, void* flags_host, void* event,
                  void* stream) {
    if (n < 1 || K < 1 || d < 1 || ldx < d || ldc < d || !counts || !flags_dev)
        return fail_arg("lloyd_step: bad arguments n=%lld K=%d d=%d", (long long)n, K, d);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cbytes = sizeof(double) * (size_t)K * (size_t)ldc;
    if (snap) DA_CUDA(cudaMemcpyAsync(snap, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (C_out != C_prev) DA_CUDA(cudaMemcpyAsync(C_out, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    int rc = launch_group_sums(X, n, ldx, d, labels_prev, K, 0, C_out, ldc, counts, s);
    if (rc) return rc;
    lloyd_empty_kernel<<<1, 256, 0, s>>>(counts, K, flags_dev);
    DA_CHECK_LAUNCH("lloyd_empty_kernel");
    rc = assign_against(X, n, ldx, d, K, C_out, ldc, xx, labels_prev, labels_out, d2_out, flags_dev, s);
    if (rc) return rc;
    if (flags_host)
        DA_CUDA(cudaMemcpyAsync(flags_host, flags_dev, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    if (event) DA_CUDA(cudaEventRecord((cudaEvent_t)event, s));
    return 0;
}

int da_lloyd_prepare(const double* C_prev, double* C_out, double* snap, int64_t elems,
                     const unsigned long long* changed_prev, double* stats, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cbytes = sizeof(double) * (size_t)elems;
    if (snap) DA_CUDA(cudaMemcpyAsync(snap, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (C_out != C_prev) DA_CUDA(cudaMemcpyAsync(C_out, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (stats) {
        lloyd_stats_kernel<<<1, 1, 0, s>>>(changed_prev, stats);
        DA_CHECK_LAUNCH("lloyd_stats_kernel");
    }
    return 0;
}

int da_lloyd_finish(int fast, const double* red, const int32_t* counts, int K, int d, double* C, int64_t ldc,
                    const double* stats, double* flags_dev, void* flags_host, void* event, const double* X,
                    int64_t n, int64_t ldx, const double* xx, const int32_t* labels_prev, int32_t* labels_out,
                    double* d2_out, unsigned long long* changed, void* stream) {
    if (K < 1 || d < 1 || ldc < d || !flags_dev || !stats) return fail_arg("lloyd_finish: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (fast) {
        lloyd_means_kernel<<<grid_for((long long)K * d, 256), 256, 0, s>>>(red, K, d, C, ldc);
        DA_CHECK_LAUNCH("lloyd_means_kernel");
    }
    lloyd_shard_flags_kernel<<<1, 256, 0, s>>>(fast ? nullptr : counts, fast ? red + (long long)K * d : nullptr, K,
                                               stats, flags_dev, changed);
    DA_CHECK_LAUNCH("lloyd_shard_flags_kernel");
    if (flags_host) DA_CUDA(cudaMemcpyAsync(flags_host, flags_dev, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (event) DA_CUDA(cudaEventRecord((cudaEvent_t)event, s));
    if (labels_out)
        return assign_against(X, n, ldx, d, K, C, ldc, xx, labels_prev, labels_out, d2_out, changed, s);
    return 0;
}

}  // extern "C"

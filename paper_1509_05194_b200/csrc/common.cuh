// Shared helpers for the DA hot-path kernels (sm_100a).
//
// Numerics contract: every quantity the reference (annq, numpy float64)
// uses to make a decision is computed here in float64 with the SAME
// association order numpy uses wherever that order is documented by numpy's
// own source and verified against it (see oracle/ and tests/golden):
//   * row sums along a contiguous axis  -> numpy pairwise summation
//     (8 interleaved accumulators for blocks <= 128, recursive halving above)
//   * np.add.reduceat along axis 0      -> first row + pairwise(rest)
//   * einsum("mkd,mkd->mk")             -> SSE2 2-lane mul+add, 4x unrolled
//   * elementwise expressions           -> explicit __d*_rn intrinsics so
//     nvcc never contracts a*b+c into an FMA where numpy rounds twice.
// Dot products that numpy hands to BLAS (dgemm) are accumulated as one
// sequential FMA chain over k, which is what OpenBLAS' Haswell dgemm
// micro-kernel does for k <= its k-block; elsewhere they agree to a few ulp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

namespace da {

// ---------------------------------------------------------------------------
// error plumbing (thread-local last error, int status codes)

void set_error(const std::string& msg);
int fail_arg(const char* fmt, ...);
int fail_cuda(cudaError_t e, const char* where);

// Every kernel launch is followed by DA_CHECK_LAUNCH, which also counts it
// (da_launch_count() reports the total; bench.py uses it for gpu_launches).
void count_launch();
void count_launches(long long k);
long long launch_total();
bool prof_enabled();
int ensure_smem(const void* func, int bytes);

#define DA_CHECK_LAUNCH(where)                                   \
    do {                                                         \
        ::da::count_launch();                                    \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::da::fail_cuda(_e, where); \
    } while (0)

#define DA_CUDA(call)                                             \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::da::fail_cuda(_e, #call); \
    } while (0)

// ---------------------------------------------------------------------------
// scratch memory owned by the library (grown on demand, per device)

struct Scratch {
    void* ptr = nullptr;
    size_t bytes = 0;
};
// Returns a device buffer of at least `bytes` for slot `slot` on the current
// device; the pointer stays valid until the next call with a larger size for
// the same slot.  Callers synchronise through the stream they pass.
void* scratch(int slot, size_t bytes, cudaStream_t stream);

inline unsigned grid_for(long long n, int per_block, long long cap = 1 << 20) {
    long long g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// numpy-order float64 reductions

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// numpy's pairwise_sum leaf: n <= 128 elements produced by f(i), i in [lo, lo+n).
template <class F>
__device__ __forceinline__ double np_pw_leaf(const F& f, long long lo, long long n) {
    if (n < 8) {
        double r = 0.0;
        for (long long i = 0; i < n; ++i) r = dadd(r, f(lo + i));
        return r;
    }
    double r0 = f(lo + 0), r1 = f(lo + 1), r2 = f(lo + 2), r3 = f(lo + 3);
    double r4 = f(lo + 4), r5 = f(lo + 5), r6 = f(lo + 6), r7 = f(lo + 7);
    long long i = 8;
    const long long stop = n - (n % 8);
    for (; i < stop; i += 8) {
        r0 = dadd(r0, f(lo + i + 0)); r1 = dadd(r1, f(lo + i + 1));
        r2 = dadd(r2, f(lo + i + 2)); r3 = dadd(r3, f(lo + i + 3));
        r4 = dadd(r4, f(lo + i + 4)); r5 = dadd(r5, f(lo + i + 5));
        r6 = dadd(r6, f(lo + i + 6)); r7 = dadd(r7, f(lo + i + 7));
    }
    double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
    for (; i < n; ++i) res = dadd(res, f(lo + i));
    return res;
}

// numpy's pairwise_sum for any n (recursive halving, split kept a multiple of 8).
// Iterative post-order walk with an explicit stack (depth <= 48 for n < 2^52).
template <class F>
__device__ double np_pw_sum(const F& f, long long lo, long long n) {
    if (n <= 128) return np_pw_leaf(f, lo, n);
    long long s_lo[48], s_n[48];
    double s_left[48];
    int s_state[48];
    int sp = 0;
    s_lo[0] = lo; s_n[0] = n; s_state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        long long clo = s_lo[sp], cn = s_n[sp];
        if (cn <= 128) {
            ret = np_pw_leaf(f, clo, cn);
            --sp;
            // deliver ret to the parent
            while (sp >= 0) {
                if (s_state[sp] == 1) {  // left child just finished
                    s_left[sp] = ret;
                    s_state[sp] = 2;
                    long long n2 = s_n[sp] / 2; n2 -= n2 % 8;
                    ++sp;
                    s_lo[sp] = s_lo[sp - 1] + n2; s_n[sp] = s_n[sp - 1] - n2; s_state[sp] = 0;
                    break;
                } else {  // right child finished
                    ret = dadd(s_left[sp], ret);
                    --sp;
                }
            }
            continue;
        }
        // descend left
        long long n2 = cn / 2; n2 -= n2 % 8;
        s_state[sp] = 1;
        ++sp;
        s_lo[sp] = clo; s_n[sp] = n2; s_state[sp] = 0;
    }
    return ret;
}

// einsum('...d,...d->...', a, a) on x86-64 numpy: SSE2 2-lane accumulators,
// mul then add (no FMA), blocks of 4 vectors consumed high-to-low, zero-padded
// tail, lane0+lane1, then added to the zero-initialised output.
template <class F>
__device__ __forceinline__ double np_einsum_sq(const F& f, int n) {
    double a0 = 0.0, a1 = 0.0;
    int i = 0;
    for (; n - i >= 8; i += 8) {
        double v;
        double ab3_0, ab3_1, ab2_0, ab2_1, ab1_0, ab1_1;
        v = f(i + 6); ab3_0 = dadd(dmul(v, v), a0);
        v = f(i + 7); ab3_1 = dadd(dmul(v, v), a1);
        v = f(i + 4); ab2_0 = dadd(dmul(v, v), ab3_0);
        v = f(i + 5); ab2_1 = dadd(dmul(v, v), ab3_1);
        v = f(i + 2); ab1_0 = dadd(dmul(v, v), ab2_0);
        v = f(i + 3); ab1_1 = dadd(dmul(v, v), ab2_1);
        v = f(i + 0); a0 = dadd(dmul(v, v), ab1_0);
        v = f(i + 1); a1 = dadd(dmul(v, v), ab1_1);
    }
    for (; i < n; i += 2) {
        double v = f(i);
        a0 = dadd(dmul(v, v), a0);
        if (i + 1 < n) { double w = f(i + 1); a1 = dadd(dmul(w, w), a1); }
        else { a1 = dadd(0.0, a1); }
    }
    return dadd(0.0, dadd(a0, a1));
}

// OpenBLAS (0.3.30, SkylakeX/Haswell dgemm & dsyrk drivers) splits the
// contraction dimension k into blocks of GEMM_Q = 384, balancing the last two:
//   rest >= 2Q -> Q;  Q < rest < 2Q -> ((rest/2 + 1)/2)*2;  else rest.
// Each block is a sequential FMA chain from zero that is then added to C.
// Verified bit-exact against numpy's matmul on this toolchain (oracle/, tests).
constexpr long long BLAS_Q = 384;
__host__ __device__ __forceinline__ long long blas_block_len(long long rest) {
    if (rest >= 2 * BLAS_Q) return BLAS_Q;
    if (rest > BLAS_Q) return ((rest / 2 + 1) / 2) * 2;
    return rest;
}

// Lexicographic (value, index) order used by numpy's stable argsort / argmin.
__device__ __forceinline__ bool lex_less(double a, long long ia, double b, long long ib) {
    return (a < b) || (a == b && ia < ib);
}

}  // namespace da

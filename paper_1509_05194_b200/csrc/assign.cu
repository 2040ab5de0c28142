// Nearest-codeword kernel: the Lloyd assign step.
//
// Follows annq/clustering.py:139-148 (`_assign`):
//   d2[i, k] = (||x_i||^2 - 2 x_i.c_k) + ||c_k||^2   over the active prefix d,
//   clipped at 0, label = first index of the minimum, returns d2[i, label].
// ||x||^2 and ||c||^2 are numpy pairwise row sums (computed here per row /
// by da_row_sqnorms); x.c is a sequential float64 FMA chain over k.
//
// Tile: 128 rows x 64 codewords per step, 256 threads, 8x4 outputs/thread,
// k staged through shared memory in chunks of 16.  The argmin is fused into
// the epilogue of every codeword tile; a running (value, index) minimum per
// row is kept in registers and reduced across the 16 column lanes at the end.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int AS_BM = 128;
constexpr int AS_BN = 64;
constexpr int AS_BK = 16;
constexpr int AS_TM = 8;
constexpr int AS_THREADS = 256;
}  // namespace

template <typename TX, bool BLK>
__global__ void __launch_bounds__(AS_THREADS)
assign_kernel(const TX* __restrict__ X, long long n, long long ldx, int d,
              const double* __restrict__ C, long long ldc, int K,
              const double* __restrict__ cc, const double* __restrict__ xx_in,
              int32_t* __restrict__ labels, double* __restrict__ d2_out,
              const int32_t* __restrict__ prev, unsigned long long* __restrict__ changed) {
    __shared__ __align__(16) double As[AS_BK][AS_BM];
    __shared__ __align__(16) double Bs[AS_BK][AS_BN];
    __shared__ double xxs[AS_BM];

    const int tid = threadIdx.x;
    const int tx = tid & 15;   // column group
    const int ty = tid >> 4;   // row group
    const long long row0 = (long long)blockIdx.x * AS_BM;

    // ||x||^2 over the active prefix, numpy pairwise order
    if (tid < AS_BM) {
        long long r = row0 + tid;
        double v = 0.0;
        if (r < n) {
            const TX* xr = X + r * ldx;
            v = xx_in ? xx_in[r] : np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
        }
        xxs[tid] = v;
    }

    double best[AS_TM];
    int bidx[AS_TM];
#pragma unroll
    for (int i = 0; i < AS_TM; ++i) { best[i] = __longlong_as_double(0x7ff0000000000000ULL); bidx[i] = 0x7fffffff; }

    const int c_loc[4] = {2 * tx, 2 * tx + 1, 32 + 2 * tx, 33 + 2 * tx};

    for (int col0 = 0; col0 < K; col0 += AS_BN) {
        double acc[AS_TM][4];
        double tot[BLK ? AS_TM : 1][4];
#pragma unroll
        for (int i = 0; i < AS_TM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        // d > 384: OpenBLAS k-blocking (see blas_block_len) -- fold per block
        long long blk_end = blas_block_len(d);
        bool first_blk = true;

        for (int k0 = 0; k0 < d; k0 += AS_BK) {
            __syncthreads();
            // A tile: 128 rows x 16 k, converted to f64, stored k-major
#pragma unroll
            for (int it = 0; it < (AS_BM * AS_BK) / AS_THREADS; ++it) {
                int e = it * AS_THREADS + tid;
                int r = e / AS_BK, k = e % AS_BK;
                long long gr = row0 + r;
                int gk = k0 + k;
                double v = 0.0;
                if (gr < n && gk < d) v = (double)X[gr * ldx + gk];
                As[k][r] = v;
            }
            // B tile: 64 codewords x 16 k
#pragma unroll
            for (int it = 0; it < (AS_BN * AS_BK) / AS_THREADS; ++it) {
                int e = it * AS_THREADS + tid;
                int c = e / AS_BK, k = e % AS_BK;
                int gc = col0 + c, gk = k0 + k;
                double v = 0.0;
                if (gc < K && gk < d) v = C[(long long)gc * ldc + gk];
                Bs[k][c] = v;
            }
            __syncthreads();
            const int kmax = min(AS_BK, d - k0);
            for (int k = 0; k < kmax; ++k) {
                if (BLK && k0 + k == blk_end) {
#pragma unroll
                    for (int i = 0; i < AS_TM; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            tot[BLK ? i : 0][j] = first_blk ? acc[i][j] : dadd(tot[BLK ? i : 0][j], acc[i][j]);
                            acc[i][j] = 0.0;
                        }
                    first_blk = false;
                    blk_end += blas_block_len(d - blk_end);
                }
                double a[AS_TM], b[4];
                const double2* ap = reinterpret_cast<const double2*>(&As[k][ty * AS_TM]);
#pragma unroll
                for (int i = 0; i < AS_TM / 2; ++i) { double2 t = ap[i]; a[2 * i] = t.x; a[2 * i + 1] = t.y; }
                double2 b01 = *reinterpret_cast<const double2*>(&Bs[k][2 * tx]);
                double2 b23 = *reinterpret_cast<const double2*>(&Bs[k][32 + 2 * tx]);
                b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
                for (int i = 0; i < AS_TM; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
            }
        }
        if (BLK) {
#pragma unroll
            for (int i = 0; i < AS_TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = first_blk ? acc[i][j] : dadd(tot[BLK ? i : 0][j], acc[i][j]);
        }
        // fused epilogue: distances + running first-min
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int gc = col0 + c_loc[j];
            if (gc >= K) continue;
            double ccv = cc[gc];
#pragma unroll
            for (int i = 0; i < AS_TM; ++i) {
                double v = dadd(dsub(xxs[ty * AS_TM + i], dmul(2.0, acc[i][j])), ccv);
                if (v < 0.0) v = 0.0;
                if (v < best[i]) { best[i] = v; bidx[i] = gc; }
            }
        }
    }

    // reduce across the 16 column lanes that share a row group
    unsigned long long local_changed = 0;
#pragma unroll
    for (int i = 0; i < AS_TM; ++i) {
        double v = best[i];
        int ix = bidx[i];
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, v, off);
            int oi = __shfl_xor_sync(0xffffffffu, ix, off);
            if (lex_less(ov, oi, v, ix)) { v = ov; ix = oi; }
        }
        long long r = row0 + ty * AS_TM + i;
        if (tx == 0 && r < n) {
            labels[r] = ix;
            if (d2_out) d2_out[r] = v;
            if (prev != nullptr && prev[r] != ix) ++local_changed;
        }
    }
    if (changed != nullptr) {
        // warp-aggregate then one atomic per warp
        for (int off = 16; off >= 1; off >>= 1) local_changed += __shfl_xor_sync(0xffffffffu, local_changed, off);
        if ((tid & 31) == 0 && local_changed) atomicAdd(changed, local_changed);
    }
}

// ||c_k||^2 over the active prefix for K rows (numpy pairwise row sums).
template <typename T>
__global__ void row_sqnorm_kernel(const T* __restrict__ A, long long rows, long long lda, int d,
                                  double* __restrict__ out) {
    long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const T* ar = A + r * lda;
    out[r] = np_pw_sum([&](long long i) { double t = (double)ar[i]; return dmul(t, t); }, 0, d);
}

int launch_row_sqnorms(const void* A, int a_is_f32, long long rows, long long lda, int d, double* out,
                       cudaStream_t s) {
    if (rows <= 0) return 0;
    unsigned g = grid_for(rows, 128);
    if (a_is_f32)
        row_sqnorm_kernel<float><<<g, 128, 0, s>>>((const float*)A, rows, lda, d, out);
    else
        row_sqnorm_kernel<double><<<g, 128, 0, s>>>((const double*)A, rows, lda, d, out);
    DA_CHECK_LAUNCH("row_sqnorm_kernel");
    return 0;
}

static int g_assign_mode = 0;  // 0: tensor-core filter + exact recheck when K <= 256; 1: plain float64
static unsigned long long* g_assign_stats = nullptr;

int set_assign_config(int mode, unsigned long long* stats) {
    g_assign_mode = mode;
    g_assign_stats = stats;
    return 0;
}

// Small active widths (d <= 16): every candidate exactly, no filter.  Thread per
// row, the row in registers, the codebook (K x d float64) and its norms in shared
// memory (broadcast reads); four codewords' FMA chains interleave for ILP.  Same
// value per candidate as the reference ((xx - 2 x.c) + cc, dot as one FMA chain
// from 0, clipped at 0) and the same first-index minimum.
constexpr int AS_SMALL_D = 16;
constexpr int AS_SMALL_R = 2;   // rows per thread (each codeword load feeds both)
template <typename TX>
__global__ void __launch_bounds__(256) assign_small_kernel(const TX* __restrict__ X, long long n, long long ldx, int d,
                                                           const double* __restrict__ C, long long ldc, int K,
                                                           const double* __restrict__ cc,
                                                           const double* __restrict__ xx_in,
                                                           int32_t* __restrict__ labels, double* __restrict__ d2,
                                                           const int32_t* __restrict__ prev,
                                                           unsigned long long* __restrict__ changed) {
    extern __shared__ double sC[];   // [K][dp] (dp = d rounded up to even, zero padded), then cc[K]
    const int dp = (d + 1) & ~1;
    double* scc = sC + (size_t)K * dp;
    for (int i = threadIdx.x; i < K * dp; i += blockDim.x) {
        const int k = i / dp, j = i % dp;
        sC[i] = j < d ? C[(long long)k * ldc + j] : 0.0;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) scc[k] = cc[k];
    __syncthreads();
    const long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * AS_SMALL_R;
    double x[AS_SMALL_R][AS_SMALL_D], xx[AS_SMALL_R], best[AS_SMALL_R];
    int bk[AS_SMALL_R];
#pragma unroll
    for (int t = 0; t < AS_SMALL_R; ++t) {
        const long long r = r0 + t;
        const TX* xr = X + (r < n ? r : 0) * ldx;
#pragma unroll
        for (int j = 0; j < AS_SMALL_D; ++j) x[t][j] = (j < d && r < n) ? (double)xr[j] : 0.0;
        xx[t] = r < n ? (xx_in ? xx_in[r]
                               : np_pw_sum([&](long long i) { double v = (double)xr[i]; return dmul(v, v); }, 0, d))
                      : 0.0;
        best[t] = __longlong_as_double(0x7ff0000000000000ULL);
        bk[t] = 0x7fffffff;
    }
    for (int k0 = 0; k0 < K; k0 += 4) {
        double a[AS_SMALL_R][4];
#pragma unroll
        for (int t = 0; t < AS_SMALL_R; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u) a[t][u] = 0.0;
#pragma unroll
        for (int j = 0; j < AS_SMALL_D; j += 2) {
            if (j < d) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (k0 + u < K) {
                        const double2 c2 = *reinterpret_cast<const double2*>(sC + (size_t)(k0 + u) * dp + j);
#pragma unroll
                        for (int t = 0; t < AS_SMALL_R; ++t) {
                            a[t][u] = __fma_rn(x[t][j], c2.x, a[t][u]);
                            if (j + 1 < d) a[t][u] = __fma_rn(x[t][j + 1], c2.y, a[t][u]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + u;
            if (k < K) {
#pragma unroll
                for (int t = 0; t < AS_SMALL_R; ++t) {
                    double dv = dadd(dsub(xx[t], dmul(2.0, a[t][u])), scc[k]);
                    if (dv < 0.0) dv = 0.0;
                    if (dv < best[t]) { best[t] = dv; bk[t] = k; }   // k ascending: first index wins ties
                }
            }
        }
    }
    unsigned nchg = 0;
#pragma unroll
    for (int t = 0; t < AS_SMALL_R; ++t) {
        const long long r = r0 + t;
        if (r < n) {
            labels[r] = bk[t];
            if (d2) d2[r] = best[t];
            if (changed != nullptr && prev != nullptr && prev[r] != bk[t]) ++nchg;
        }
    }
    if (changed != nullptr && prev != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nchg += __shfl_xor_sync(0xffffffffu, nchg, o);
        if ((threadIdx.x & 31) == 0 && nchg) atomicAdd(changed, (unsigned long long)nchg);
    }
}

int launch_assign(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C,
                  long long ldc, int K, const double* cc, const double* xx, int32_t* labels, double* d2,
                  const int32_t* prev, unsigned long long* changed, cudaStream_t s) {
    if (n <= 0) return 0;
    // measured crossover against the tensor-core filter on B200: d <= 3
    static const int small_max = getenv("DA_ASSIGN_SMALL_D") ? atoi(getenv("DA_ASSIGN_SMALL_D")) : 3;
    if (g_assign_mode == 0 && d <= small_max && K <= 4096) {
        ProfScope ps("assign_small_d<=16", s);
        const size_t smem = sizeof(double) * ((size_t)K * ((d + 1) & ~1) + K);
        const unsigned g = grid_for((n + AS_SMALL_R - 1) / AS_SMALL_R, 256, 1LL << 31);
        if (smem > 48 * 1024) {
            // K up to 4096 at d = 3 needs up to 160 KB of codebook in shared memory
            DA_CUDA(cudaFuncSetAttribute(assign_small_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            DA_CUDA(cudaFuncSetAttribute(assign_small_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        }
        if (x_is_f32)
            assign_small_kernel<float><<<g, 256, smem, s>>>((const float*)X, n, ldx, d, C, ldc, K, cc, xx, labels, d2,
                                                            prev, changed);
        else
            assign_small_kernel<double><<<g, 256, smem, s>>>((const double*)X, n, ldx, d, C, ldc, K, cc, xx, labels,
                                                             d2, prev, changed);
        DA_CHECK_LAUNCH("assign_small_kernel");
        return 0;
    }
    if (g_assign_mode == 0) {
        int rc = launch_assign_tc(X, x_is_f32, n, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, changed, g_assign_stats, s);
        if (rc <= 0) return rc;
    }
    unsigned g = grid_for(n, AS_BM, 1LL << 31);
    ProfScope ps(d <= 8 ? "assign_d<=8" : d <= 32 ? "assign_d<=32" : d <= 128 ? "assign_d<=128" : "assign_d>128", s);
    const bool blk = d > BLAS_Q;
#define AS_LAUNCH(T, B) assign_kernel<T, B><<<g, AS_THREADS, 0, s>>>((const T*)X, n, ldx, d, C, ldc, K, cc, xx, \
                                                                  labels, d2, prev, changed)
    if (x_is_f32) { if (blk) AS_LAUNCH(float, true); else AS_LAUNCH(float, false); }
    else { if (blk) AS_LAUNCH(double, true); else AS_LAUNCH(double, false); }
#undef AS_LAUNCH
    DA_CHECK_LAUNCH("assign_kernel");
    return 0;
}

}  // namespace da

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
#include <algorithm>
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

long long assign_config_key() { return (long long)(uintptr_t)g_assign_stats * 31 + g_assign_mode; }

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

// Narrow active widths (d <= 16, K <= 4096): an fp32 filter with a rigorous
// bound, then float64 only where the bound cannot decide.  Thread per row; the
// codebook as fp32 rows (+ fp32 norms) in shared memory.  v'(k) = cc'_k - 2 x'.c'_k
// approximates v(k) = cc_k - 2 x.c_k within E = (2d + 12) u S with
// S = xx + 2 ||x|| max||c|| + max cc (float representation of x, c and cc, the
// d-term fp32 dot, the final subtraction, and the reference's own float64
// roundings, generously).  Codeword k can be the reference's choice only if
// max(xx + v'_k - E, 0) <= max(xx + min v' + E, 0) (the clip at 0 makes ties);
// when that holds for the minimum alone it is the label, otherwise the kept
// candidates are evaluated exactly like assign_small_kernel and the first
// minimum wins.  d2 (when asked for) is the exact value of the label.
// packed fp32 pair FMA (FFMA2): d = a * b + c lane-wise
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rd, {%0, %1};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rd;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0));
    (void)b1;
}

constexpr int AF_R = 2;   // rows per thread: one codeword load and one FFMA2 feed both
template <typename TX, int DM>
__global__ void __launch_bounds__(256) assign_ffma_kernel(const TX* __restrict__ X, long long n, long long ldx, int d,
                                                          const double* __restrict__ C, long long ldc, int K,
                                                          const double* __restrict__ cc,
                                                          const double* __restrict__ xx_in,
                                                          int32_t* __restrict__ labels, double* __restrict__ d2,
                                                          const int32_t* __restrict__ prev,
                                                          unsigned long long* __restrict__ changed,
                                                          unsigned long long* __restrict__ stats,
                                                          int* __restrict__ hard, int* __restrict__ nhard) {
    extern __shared__ __align__(16) float sCf[];   // [K][DM] fp32 codewords (zero padded), then [K] fp32 norms
    float* scc = sCf + (size_t)K * DM;
    __shared__ float s_cmax, s_ccmax;
    if (threadIdx.x == 0) { s_cmax = 0.f; s_ccmax = 0.f; }
    __syncthreads();
    float cm = 0.f, ccm = 0.f;
    for (int i = threadIdx.x; i < K * DM; i += blockDim.x) {
        const int k = i / DM, j = i - k * DM;
        sCf[i] = j < d ? (float)C[(long long)k * ldc + j] : 0.f;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        scc[k] = (float)cc[k];
        ccm = fmaxf(ccm, __double2float_ru(cc[k]));
        cm = fmaxf(cm, __double2float_ru(sqrt(cc[k]) * (1.0 + 1e-12)));
    }
    atomicMax(reinterpret_cast<int*>(&s_cmax), __float_as_int(cm));   // non-negative floats order like ints
    atomicMax(reinterpret_cast<int*>(&s_ccmax), __float_as_int(ccm));
    __syncthreads();
    // persistent blocks: the codebook is staged once per block, rows stream through
    for (long long rbase = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * AF_R; rbase < n;
         rbase += (long long)gridDim.x * blockDim.x * AF_R) {
    float x[AF_R][DM];
    double xxv[AF_R];
    float m1[AF_R], m2[AF_R];
    int k1[AF_R];
#pragma unroll
    for (int t = 0; t < AF_R; ++t) {
        const long long r = rbase + t < n ? rbase + t : rbase;
        const TX* xr = X + r * ldx;
#pragma unroll
        for (int j = 0; j < DM; ++j) x[t][j] = j < d ? (float)xr[j] : 0.f;
        xxv[t] = xx_in ? xx_in[r] : np_pw_sum([&](long long i) { double v = (double)xr[i]; return dmul(v, v); }, 0, d);
        m1[t] = m2[t] = __int_as_float(0x7f800000);
        k1[t] = 0;
    }
    // pass 1: fp32 filter values of both rows, two smallest + argmin per row
    for (int k = 0; k < K; ++k) {
        const float* c = sCf + (size_t)k * DM;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int j = 0; j < DM; j += 4) {
            const float4 c4 = *reinterpret_cast<const float4*>(c + j);
            ffma2(a0, a1, x[0][j], x[1][j], c4.x, c4.x);
            ffma2(a0, a1, x[0][j + 1], x[1][j + 1], c4.y, c4.y);
            ffma2(a0, a1, x[0][j + 2], x[1][j + 2], c4.z, c4.z);
            ffma2(a0, a1, x[0][j + 3], x[1][j + 3], c4.w, c4.w);
        }
        const float ck = scc[k];
        const float v0 = fmaf(-2.f, a0, ck), v1 = fmaf(-2.f, a1, ck);
        k1[0] = v0 < m1[0] ? k : k1[0]; m2[0] = fminf(m2[0], fmaxf(m1[0], v0)); m1[0] = fminf(m1[0], v0);
        k1[1] = v1 < m1[1] ? k : k1[1]; m2[1] = fminf(m2[1], fmaxf(m1[1], v1)); m1[1] = fminf(m1[1], v1);
    }
    unsigned nchg = 0;
    unsigned long long nx = 0;
#pragma unroll
    for (int t = 0; t < AF_R; ++t) {
        const long long r = rbase + t;
        if (r >= n) continue;
        const TX* xr = X + r * ldx;
        const double xx = xxv[t];
        const double S = xx + 2.0 * sqrt(xx) * (1.0 + 1e-12) * (double)s_cmax + (double)s_ccmax;
        const float E = __double2float_ru((2.0 * d + 12.0) * 5.9604644775390625e-08 * S);
        const float xxf = (float)xx;
        const float lim = fmaxf(__fadd_ru(__fadd_ru(xxf, m1[t]), E) * (1.f + 1e-6f) + 1e-30f, 0.f);
        const bool alone = fmaxf(__fsub_rd(__fadd_rd(xxf, m2[t]), E) * (1.f - 1e-6f), 0.f) > lim;
        auto exact = [&](int k) -> double {
            const double* crow = C + (long long)k * ldc;
            double a = 0.0;
            for (int j = 0; j < d; ++j) a = __fma_rn((double)xr[j], crow[j], a);
            const double v = dadd(dsub(xx, dmul(2.0, a)), cc[k]);
            return v < 0.0 ? 0.0 : v;
        };
        if (!alone) {   // rare: decided by assign_ffma_hard_kernel (a warp per row, no divergence here)
            hard[atomicAdd(nhard, 1)] = (int)r;
            continue;
        }
        const int lab = k1[t];
        double best = 0.0;
        if (d2) { best = exact(lab); ++nx; }
        labels[r] = lab;
        if (d2) d2[r] = best;
        if (prev != nullptr && prev[r] != lab) ++nchg;
    }
    // threads past the end leave the loop early: no warp-wide reduction, one atomic per changed thread
    if (changed != nullptr && prev != nullptr && nchg) atomicAdd(changed, (unsigned long long)nchg);
    if (stats && nx) atomicAdd(stats, nx);
    }
}

// Rows the fp32 filter could not decide: one warp per row, lane l takes
// codewords l, l+32, ...; every kept codeword is evaluated exactly and the
// lexicographic (value, index) minimum is the reference's first minimum.
template <typename TX>
__global__ void __launch_bounds__(256) assign_ffma_hard_kernel(const TX* __restrict__ X, long long ldx, int d,
                                                               const double* __restrict__ C, long long ldc, int K,
                                                               const double* __restrict__ cc,
                                                               const double* __restrict__ xx_in,
                                                               int32_t* __restrict__ labels, double* __restrict__ d2,
                                                               const int32_t* __restrict__ prev,
                                                               unsigned long long* __restrict__ changed,
                                                               unsigned long long* __restrict__ stats,
                                                               const int* __restrict__ hard, const int* __restrict__ nhard) {
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int nh = *nhard;
    if (w >= nh) return;                 // usually no or few undecided rows: most warps leave at once
    double cmax = 0.0, ccmax = 0.0;
    for (int k = lane; k < K; k += 32) { ccmax = fmax(ccmax, cc[k]); }
    for (int o = 16; o > 0; o >>= 1) ccmax = fmax(ccmax, __shfl_xor_sync(0xffffffffu, ccmax, o));
    cmax = sqrt(ccmax) * (1.0 + 1e-12);
    for (int h = w; h < nh; h += nw) {
        const long long r = hard[h];
        const TX* xr = X + r * ldx;
        const double xx = xx_in ? xx_in[r]
                                : np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
        const double S = xx + 2.0 * sqrt(xx) * (1.0 + 1e-12) * cmax + ccmax;
        const float E = __double2float_ru((2.0 * d + 12.0) * 5.9604644775390625e-08 * S);
        const float xxf = (float)xx;
        // same fp32 values as the filter (same operand roundings, same FMA order)
        float vmin = __int_as_float(0x7f800000);
        auto fval = [&](int k) -> float {
            const double* crow = C + (long long)k * ldc;
            float dot = 0.f;
            for (int j = 0; j < d; ++j) dot = fmaf((float)xr[j], (float)crow[j], dot);
            return fmaf(-2.f, dot, (float)cc[k]);
        };
        for (int k = lane; k < K; k += 32) vmin = fminf(vmin, fval(k));
        for (int o = 16; o > 0; o >>= 1) vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        const float lim = fmaxf(__fadd_ru(__fadd_ru(xxf, vmin), E) * (1.f + 1e-6f) + 1e-30f, 0.f);
        double best = __longlong_as_double(0x7ff0000000000000ULL);
        int lab = 0x7fffffff;
        unsigned long long nx = 0;
        for (int k = lane; k < K; k += 32) {
            if (fmaxf(__fsub_rd(__fadd_rd(xxf, fval(k)), E) * (1.f - 1e-6f), 0.f) <= lim) {
                const double* crow = C + (long long)k * ldc;
                double a = 0.0;
                for (int j = 0; j < d; ++j) a = __fma_rn((double)xr[j], crow[j], a);
                double v = dadd(dsub(xx, dmul(2.0, a)), cc[k]);
                if (v < 0.0) v = 0.0;
                ++nx;
                if (lex_less(v, k, best, lab)) { best = v; lab = k; }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int ok = __shfl_xor_sync(0xffffffffu, lab, o);
            if (lex_less(ov, ok, best, lab)) { best = ov; lab = ok; }
        }
        for (int o = 16; o > 0; o >>= 1) nx += __shfl_xor_sync(0xffffffffu, nx, o);
        if (lane == 0) {
            labels[r] = lab;
            if (d2) d2[r] = best;
            if (changed != nullptr && prev != nullptr && prev[r] != lab) atomicAdd(changed, 1ULL);
            if (stats && nx) atomicAdd(stats, nx);
        }
    }
}

int launch_assign(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C,
                  long long ldc, int K, const double* cc, const double* xx, int32_t* labels, double* d2,
                  const int32_t* prev, unsigned long long* changed, cudaStream_t s) {
    if (n <= 0) return 0;
    // fp32 filter for narrow prefixes (d <= 16), then the float64 kernels
    static const int ffma_max = getenv("DA_ASSIGN_FFMA_D") ? atoi(getenv("DA_ASSIGN_FFMA_D")) : 4;   // B200, 1M rows: d=2,3 0.14 ms; from d=5 the tcgen05 filter wins (0.18 vs 0.20 ms per call inside the anneal pass)
    if (g_assign_mode == 0 && d <= ffma_max && d <= 16 && K <= 4096) {
        ProfScope ps("assign_ffma_d<=8", s);
        const int dm = d <= 4 ? 4 : d <= 8 ? 8 : 16;
        const size_t smem = sizeof(float) * ((size_t)K * dm + K);
        int dev_ = 0, sms_ = 148;
        cudaGetDevice(&dev_);
        cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_);
        const unsigned g = (unsigned)std::min<long long>((n + AF_R * 256 - 1) / (AF_R * 256), 4LL * sms_);
        int* nhard = (int*)scratch(22, sizeof(int) * ((size_t)n + 64), s);
        if (!nhard) return fail_cuda(cudaErrorMemoryAllocation, "assign_ffma scratch");
        int* hard = nhard + 64;
        DA_CUDA(cudaMemsetAsync(nhard, 0, sizeof(int), s));
#define AF_LAUNCH(T, DMv)                                                                                            \
    do {                                                                                                             \
        if (smem > 48 * 1024)                                                                                        \
            { const int rc_ = ensure_smem((const void*)assign_ffma_kernel<T, DMv>, (int)smem); if (rc_) return rc_; } \
        assign_ffma_kernel<T, DMv><<<g, 256, smem, s>>>((const T*)X, n, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, \
                                                        changed, g_assign_stats, hard, nhard);                       \
        DA_CHECK_LAUNCH("assign_ffma_kernel");                                                                       \
        assign_ffma_hard_kernel<T><<<2 * sms_, 256, 0, s>>>((const T*)X, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, \
                                                           changed, g_assign_stats, hard, nhard);                    \
    } while (0)
        if (x_is_f32) { if (dm == 4) AF_LAUNCH(float, 4); else if (dm == 8) AF_LAUNCH(float, 8); else AF_LAUNCH(float, 16); }
        else { if (dm == 4) AF_LAUNCH(double, 4); else if (dm == 8) AF_LAUNCH(double, 8); else AF_LAUNCH(double, 16); }
#undef AF_LAUNCH
        DA_CHECK_LAUNCH("assign_ffma_hard_kernel");
        return 0;
    }
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

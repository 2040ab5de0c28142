// Float64 "dot-GEMM" used for the reference's BLAS calls on the hot path:
//   PCA covariance  Xc^T Xc        (annq/clustering.py:96)
//   PCA rotate      (X - mu) R^T   (annq/clustering.py:40)
//   un-rotate       Y R + mu       (annq/clustering.py:43)
//   cross products  C_a C_b^T      (annq/codebook.py:236, 247)
//   beam tables     ||c||^2 - 2 X C^T (annq/codebook.py:259-261)
// Every output element is one sequential FMA chain over k (plus an optional
// rounded epilogue), i.e. the association order of a dgemm micro-kernel.
//
// C[i, j] = epi( sum_k a(i,k) * b(k,j) ),  a(i,k) = A[i*sai + k*sak] - asub,
// b(k,j) = B[k*sbk + j*sbj] - bsub.  Inputs may be float32 (converted
// exactly) or float64.  gridDim.z enumerates (batch1, batch2, ksplit).
#include "common.cuh"
#include "internal.h"

namespace da {


namespace {
constexpr int GB_M = 64, GB_N = 64, GB_K = 16, G_THREADS = 256;
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(G_THREADS) gemm_kernel(GemmArgs g) {
    __shared__ __align__(16) double As[GB_K][GB_M];
    __shared__ __align__(16) double Bs[GB_K][GB_N];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int z = blockIdx.z;
    const int ks = z % g.ksplit;
    const int zb = z / g.ksplit;
    const int z1 = zb / g.nb2, z2 = zb % g.nb2;
    const TA* A = (const TA*)g.A + z1 * g.sA1 + z2 * g.sA2;
    const TB* B = (const TB*)g.B + z1 * g.sB1 + z2 * g.sB2;
    double* C = g.C + z1 * g.sC1 + z2 * g.sC2 + ks * g.sCz;
    const long long i0 = (long long)blockIdx.y * GB_M, j0 = (long long)blockIdx.x * GB_N;
    const long long kbeg = g.kstarts ? g.kstarts[ks] : ks * g.kchunk;
    const long long kend = g.kstarts ? g.kstarts[ks + 1] : min(g.K, kbeg + g.kchunk);
    const bool a_kfast = g.sak == 1;
    const bool b_jfast = g.sbj == 1;

    double acc[4][4], tot[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { acc[i][j] = 0.0; tot[i][j] = 0.0; }
    if (g.cinit && ks == 0) {
        // continue a chain another shard started (same FMA sequence as one long chain)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long gi = i0 + ty * 4 + i, gj = j0 + (j < 2 ? 2 * tx + j : 30 + 2 * tx + j);
                if (gi < g.M && gj < g.N) acc[i][j] = g.cinit[gi * g.sci + gj * g.scj];
            }
    }
    // BLAS k-blocking of this k-range (one block when the range is <= 384)
    long long blk_end = kbeg + blas_block_len(kend - kbeg);
    bool first_blk = true;
    auto fold = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                tot[i][j] = first_blk ? acc[i][j] : dadd(tot[i][j], acc[i][j]);
                acc[i][j] = 0.0;
            }
        first_blk = false;
    };

    for (long long k0 = kbeg; k0 < kend; k0 += GB_K) {
        __syncthreads();
#pragma unroll
        for (int it = 0; it < (GB_M * GB_K) / G_THREADS; ++it) {
            int e = it * G_THREADS + tid;
            int r, k;
            if (a_kfast) { r = e / GB_K; k = e % GB_K; } else { k = e / GB_M; r = e % GB_M; }
            long long gi = i0 + r, gk = k0 + k;
            double v = 0.0;
            if (gi < g.M && gk < kend) {
                v = (double)A[gi * g.sai + gk * g.sak];
                if (g.asub_mode == 1) v = dsub(v, g.asub[gi]);
                else if (g.asub_mode == 2) v = dsub(v, g.asub[gk]);
            }
            As[k][r] = v;
        }
#pragma unroll
        for (int it = 0; it < (GB_N * GB_K) / G_THREADS; ++it) {
            int e = it * G_THREADS + tid;
            int c, k;
            if (b_jfast) { k = e / GB_N; c = e % GB_N; } else { c = e / GB_K; k = e % GB_K; }
            long long gj = j0 + c, gk = k0 + k;
            double v = 0.0;
            if (gj < g.N && gk < kend) {
                v = (double)B[gk * g.sbk + gj * g.sbj];
                if (g.bsub_mode == 1) v = dsub(v, g.bsub[gk]);
                else if (g.bsub_mode == 2) v = dsub(v, g.bsub[gj]);
            }
            Bs[k][c] = v;
        }
        __syncthreads();
        const int kmax = (int)min((long long)GB_K, kend - k0);
        for (int k = 0; k < kmax; ++k) {
            if (k0 + k == blk_end) {
                fold();
                blk_end += blas_block_len(kend - blk_end);
            }
            double2 a01 = *reinterpret_cast<const double2*>(&As[k][ty * 4]);
            double2 a23 = *reinterpret_cast<const double2*>(&As[k][ty * 4 + 2]);
            double2 b01 = *reinterpret_cast<const double2*>(&Bs[k][2 * tx]);
            double2 b23 = *reinterpret_cast<const double2*>(&Bs[k][32 + 2 * tx]);
            double a[4] = {a01.x, a01.y, a23.x, a23.y};
            double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
        }
    }
    fold();
    const int cl[4] = {2 * tx, 2 * tx + 1, 32 + 2 * tx, 33 + 2 * tx};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        long long gi = i0 + ty * 4 + i;
        if (gi >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            long long gj = j0 + cl[j];
            if (gj >= g.N) continue;
            double v = tot[i][j];
            if (g.epi == 1) v = dadd(v, g.evec[gj]);
            else if (g.epi == 2) v = dsub(g.evec[gj], dmul(2.0, v));
            else if (g.epi == 3) { v = dadd(dsub(g.ivec[gi], dmul(2.0, v)), g.evec[gj]); if (v < 0.0) v = 0.0; }
            C[gi * g.sci + gj * g.scj] = v;
        }
    }
}

int launch_gemm(const GemmArgs& g, int nb1, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0) return 0;
    dim3 grid((unsigned)((g.N + GB_N - 1) / GB_N), (unsigned)((g.M + GB_M - 1) / GB_M),
              (unsigned)(nb1 * g.nb2 * g.ksplit));
    if (grid.y > 65535u) return fail_arg("gemm: M=%lld too large for one launch", g.M);
    if (g.a_f32 && g.b_f32) gemm_kernel<float, float><<<grid, G_THREADS, 0, s>>>(g);
    else if (g.a_f32) gemm_kernel<float, double><<<grid, G_THREADS, 0, s>>>(g);
    else if (g.b_f32) gemm_kernel<double, float><<<grid, G_THREADS, 0, s>>>(g);
    else gemm_kernel<double, double><<<grid, G_THREADS, 0, s>>>(g);
    DA_CHECK_LAUNCH("gemm_kernel");
    return 0;
}

// Sum ksplit partial matrices in order and scale: out = (sum_z P[z]) / scale_div.
// accumulate=1 continues a running total already in out (before any division).
__global__ void reduce_partials_kernel(const double* __restrict__ P, int nz, long long len, double scale_div,
                                       int accumulate, double* __restrict__ out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s = accumulate ? dadd(out[i], P[i]) : P[i];
    int z = 1;
    for (; z + 8 <= nz; z += 8) {  // loads run ahead of the ordered add chain
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = P[(long long)(z + u) * len + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = dadd(s, v[u]);
    }
    for (; z < nz; ++z) s = dadd(s, P[(long long)z * len + i]);
    out[i] = scale_div != 0.0 ? __ddiv_rn(s, scale_div) : s;
}

int launch_accumulate_partials(const double* P, int nz, long long len, double scale_div, int accumulate,
                               double* out, cudaStream_t s) {
    reduce_partials_kernel<<<grid_for(len, 256), 256, 0, s>>>(P, nz, len, scale_div, accumulate, out);
    DA_CHECK_LAUNCH("reduce_partials_kernel");
    return 0;
}

int launch_reduce_partials(const double* P, int nz, long long len, double scale_div, double* out,
                           cudaStream_t s) {
    reduce_partials_kernel<<<grid_for(len, 256), 256, 0, s>>>(P, nz, len, scale_div, 0, out);
    DA_CHECK_LAUNCH("reduce_partials_kernel");
    return 0;
}

// Column means of an (n, D) matrix: chunked sequential sums, chunks in order.
template <typename T>
__global__ void col_partial_kernel(const T* __restrict__ X, long long n, long long ld, int D, long long chunk,
                                   double* __restrict__ part) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    int p = blockIdx.y;
    if (c >= D) return;
    long long lo = (long long)p * chunk, hi = min(n, lo + chunk);
    double s = 0.0;
    for (long long r = lo; r < hi; ++r) s = dadd(s, (double)X[r * ld + c]);
    part[(long long)p * D + c] = s;
}

// numpy's X.mean(axis=0) on a C-contiguous array adds the rows one after the
// other (no pairwise tree along axis 0), so every column is one dependent add
// chain.  A block owns 8 columns: all 256 threads stream row chunks into shared
// memory (double-buffered, coalesced 8-column segments) while 8 threads of warp
// 0 run the chains out of shared memory.
constexpr int CM_COLS = 1, CM_ROWS = 2048, CM_T = 256;

template <typename T>
__global__ void __launch_bounds__(CM_T) col_mean_seq_kernel(const T* __restrict__ X, long long n, long long ld, int D,
                                                             double* __restrict__ mean, const double* __restrict__ init,
                                                             int raw) {
    __shared__ double buf[2][CM_ROWS][CM_COLS];
    const int c0 = blockIdx.x * CM_COLS;
    const int tid = threadIdx.x;
    auto load = [&](long long r0, int b) {
        for (int e = tid; e < CM_ROWS * CM_COLS; e += CM_T) {
            const int rr = e / CM_COLS, cc = e % CM_COLS;
            const long long r = r0 + rr;
            double v = 0.0;
            if (r < n && c0 + cc < D) v = (double)X[r * ld + c0 + cc];
            buf[b][rr][cc] = v;
        }
    };
    double s = (init && tid < CM_COLS && c0 + tid < D) ? init[c0 + tid] : 0.0;
    const long long nchunks = (n + CM_ROWS - 1) / CM_ROWS;
    load(0, 0);
    __syncthreads();
    for (long long ch = 0; ch < nchunks; ++ch) {
        const int b = (int)(ch & 1);
        if (ch + 1 < nchunks) load((ch + 1) * CM_ROWS, b ^ 1);
        if (tid < CM_COLS) {
            const int rows = (int)min((long long)CM_ROWS, n - ch * CM_ROWS);
            int rr = 0;
            for (; rr + 8 <= rows; rr += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = buf[b][rr + u][tid];
#pragma unroll
                for (int u = 0; u < 8; ++u) s = dadd(s, v[u]);
            }
            for (; rr < rows; ++rr) s = dadd(s, buf[b][rr][tid]);
        }
        __syncthreads();
    }
    if (tid < CM_COLS && c0 + tid < D) mean[c0 + tid] = raw ? s : __ddiv_rn(s, (double)n);
}

int launch_col_mean(const void* X, int x_f32, long long n, long long ld, int D, double* mean, cudaStream_t s) {
    if (n <= 0) return fail_arg("col_mean: n must be positive");
    ProfScope ps("col_mean", s);
    const unsigned g = (unsigned)((D + CM_COLS - 1) / CM_COLS);
    if (x_f32) col_mean_seq_kernel<float><<<g, CM_T, 0, s>>>((const float*)X, n, ld, D, mean, nullptr, 0);
    else col_mean_seq_kernel<double><<<g, CM_T, 0, s>>>((const double*)X, n, ld, D, mean, nullptr, 0);
    DA_CHECK_LAUNCH("col_mean_seq_kernel");
    return 0;
}

// Raw column sums continuing a running sum (init, may alias sums) another
// shard computed over the rows before these: the per-column add chains of
// X.mean(axis=0) cut at a shard boundary, bit for bit.
int launch_col_sums(const void* X, int x_f32, long long n, long long ld, int D, const double* init, double* sums,
                    cudaStream_t s) {
    if (n < 0) return fail_arg("col_sums: negative row count");
    if (n == 0) {
        if (init && init != sums) DA_CUDA(cudaMemcpyAsync(sums, init, sizeof(double) * D, cudaMemcpyDeviceToDevice, s));
        else if (!init) DA_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * D, s));
        return 0;
    }
    ProfScope ps("col_mean", s);
    const unsigned g = (unsigned)((D + CM_COLS - 1) / CM_COLS);
    if (x_f32) col_mean_seq_kernel<float><<<g, CM_T, 0, s>>>((const float*)X, n, ld, D, sums, init, 1);
    else col_mean_seq_kernel<double><<<g, CM_T, 0, s>>>((const double*)X, n, ld, D, sums, init, 1);
    DA_CHECK_LAUNCH("col_mean_seq_kernel");
    return 0;
}

// Chunked variant (used for shard-local sums where exact order is moot).
int launch_col_mean_chunked(const void* X, int x_f32, long long n, long long ld, int D, double* mean, cudaStream_t s) {
    if (n <= 0) return fail_arg("col_mean: n must be positive");
    int P = (int)min(256LL, max(1LL, n / 2048));
    long long chunk = (n + P - 1) / P;
    double* part = (double*)scratch(2, sizeof(double) * P * (size_t)D, s);
    if (!part) return fail_cuda(cudaErrorMemoryAllocation, "col_mean scratch");
    dim3 grid((D + 127) / 128, P);
    if (x_f32) col_partial_kernel<float><<<grid, 128, 0, s>>>((const float*)X, n, ld, D, chunk, part);
    else col_partial_kernel<double><<<grid, 128, 0, s>>>((const double*)X, n, ld, D, chunk, part);
    DA_CHECK_LAUNCH("col_partial_kernel");
    return launch_reduce_partials(part, P, D, (double)n, mean, s);
}

}  // namespace da

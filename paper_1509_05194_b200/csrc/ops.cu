// Memory-bound companions of the hot path: heat-up, exact per-vector errors,
// reconstruction, codeword norms (einsum order), pair sums, ADC scan, numpy
// pairwise means of 1-D arrays, and small gathers used by the Lloyd loop.
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace da {

// ---------------------------------------------------------------------------
// heat-up: annq/annealing.py:97-112
//   out = float32( (X64 - sum_{j} C64[j][codes_j]) + C64[m][codes_m] )
// the reconstruction is accumulated from zero in j order (codebook.py:181-188).
__global__ void heat_up_kernel(const float* __restrict__ X, long long n, int D, const int32_t* __restrict__ codes,
                               const float* __restrict__ cw, int M, int K, int m, float* __restrict__ out) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = n * D;
    for (; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / D;
        const int d = (int)(e % D);
        const int32_t* ci = codes + i * M;
        double r = 0.0;
        for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + ci[j]) * D + d]);
        double v = dadd(dsub((double)X[e], r), (double)cw[((long long)m * K + ci[m]) * D + d]);
        out[e] = __double2float_rn(v);
    }
}

int launch_heat_up(const float* X, long long n, int D, const int32_t* codes, const float* cw, int M, int K, int m,
                   float* out, cudaStream_t s) {
    if (n <= 0) return 0;
    heat_up_kernel<<<grid_for(n * D, 256, 148 * 64), 256, 0, s>>>(X, n, D, codes, cw, M, K, m, out);
    DA_CHECK_LAUNCH("heat_up_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// exact squared error of each vector under its code (annealing.py:135-137,
// codebook.py:297-300): diff = X64 - recon; (diff*diff).sum(axis=1) pairwise.
// One warp per vector; squared differences staged in shared memory.
template <typename TX, typename TC>
__global__ void vec_err_kernel(const TX* __restrict__ X, long long n, long long ldx, int D,
                               const TC* __restrict__ codes, long long ldc, const float* __restrict__ cw, int M,
                               int K, double* __restrict__ err) {
    extern __shared__ double sdiff[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long v = (long long)blockIdx.x * (blockDim.x >> 5) + wid;
    if (v >= n) return;
    double* dd = sdiff + (size_t)wid * D;
    const TC* cv = codes + v * ldc;
    const TX* xr = X + v * ldx;
    for (int d = lane; d < D; d += 32) {
        double r = 0.0;
        for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + (int)cv[j]) * D + d]);
        double df = dsub((double)xr[d], r);
        dd[d] = dmul(df, df);
    }
    __syncwarp();
    if (D <= 128) {
        double acc = 0.0;
        const int stop = D - (D % 8);
        if (D >= 8 && lane < 8) {
            acc = dd[lane];
            for (int i = 8 + lane; i < stop; i += 8) acc = dadd(acc, dd[i]);
        }
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __shfl_sync(0xffffffffu, acc, j);
        if (lane == 0) {
            double res;
            int i;
            if (D < 8) { res = 0.0; i = 0; }
            else {
                res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
                i = stop;
            }
            for (; i < D; ++i) res = dadd(res, dd[i]);
            err[v] = res;
        }
    } else if (lane == 0) {
        err[v] = np_pw_sum([&](long long i) { return dd[i]; }, 0, D);
    }
}

int launch_vec_err(const void* X, int x_f32, long long n, long long ldx, int D, const void* codes, int code_bytes,
                   long long ldc, const float* cw, int M, int K, double* err, cudaStream_t s) {
    if (n <= 0) return 0;
    int warps = 8;
    while (warps > 1 && (size_t)warps * D * 8 > 160 * 1024) warps >>= 1;
    size_t smem = (size_t)warps * D * 8;
    if (smem > 220 * 1024) return fail_arg("vec_err: D=%d too large", D);
    unsigned g = grid_for(n, warps, 1LL << 31);
#define VE_LAUNCH(TX, TC)                                                                                  \
    do {                                                                                                   \
        auto kf = vec_err_kernel<TX, TC>;                                                                  \
        if (smem > 48 * 1024) DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        kf<<<g, warps * 32, smem, s>>>((const TX*)X, n, ldx, D, (const TC*)codes, ldc, cw, M, K, err);   \
    } while (0)
    if (x_f32) {
        if (code_bytes == 1) VE_LAUNCH(float, uint8_t);
        else if (code_bytes == 2) VE_LAUNCH(float, uint16_t);
        else VE_LAUNCH(float, int32_t);
    } else {
        if (code_bytes == 1) VE_LAUNCH(double, uint8_t);
        else if (code_bytes == 2) VE_LAUNCH(double, uint16_t);
        else VE_LAUNCH(double, int32_t);
    }
#undef VE_LAUNCH
    DA_CHECK_LAUNCH("vec_err_kernel");
    return 0;
}

// reconstruction sum_m C64[m][codes_m] in m order (codebook.py:181-188)
template <typename TC>
__global__ void reconstruct_kernel(const TC* __restrict__ codes, long long n, long long ldc, const float* __restrict__ cw,
                                   int M, int K, int D, double* __restrict__ out) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = n * D;
    for (; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / D;
        const int d = (int)(e % D);
        double r = 0.0;
        for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + (int)codes[i * ldc + j]) * D + d]);
        out[e] = r;
    }
}

int launch_reconstruct(const void* codes, int code_bytes, long long n, long long ldc, const float* cw, int M, int K,
                       int D, double* out, cudaStream_t s) {
    if (n <= 0) return 0;
    unsigned g = grid_for(n * D, 256, 148 * 64);
    if (code_bytes == 1) reconstruct_kernel<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)codes, n, ldc, cw, M, K, D, out);
    else if (code_bytes == 2) reconstruct_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)codes, n, ldc, cw, M, K, D, out);
    else reconstruct_kernel<int32_t><<<g, 256, 0, s>>>((const int32_t*)codes, n, ldc, cw, M, K, D, out);
    DA_CHECK_LAUNCH("reconstruct_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// ||c||^2 per codeword in numpy einsum order (codebook.py:129, 237, 260)
__global__ void einsum_sq_kernel(const float* __restrict__ cw, long long rows, int D, double* __restrict__ out) {
    long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* c = cw + r * D;
    out[r] = np_einsum_sq([&](int i) { return (double)c[i]; }, D);
}

int launch_einsum_sq(const float* cw, long long rows, int D, double* out, cudaStream_t s) {
    if (rows <= 0) return 0;
    einsum_sq_kernel<<<grid_for(rows, 128), 128, 0, s>>>(cw, rows, D, out);
    DA_CHECK_LAUNCH("einsum_sq_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// query-independent ADC term 2 * sum_{a<b} P[a,b][i_a, i_b] (codebook.py:388-396)
template <typename TC>
__global__ void pair_sums_kernel(const TC* __restrict__ codes, long long n, long long ldc, const double* __restrict__ P,
                                 int M, int K, double* __restrict__ out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const TC* c = codes + i * ldc;
    double s = 0.0;
    for (int a = 0; a < M; ++a) {
        const int ca = (int)c[a];
        for (int b = a + 1; b < M; ++b)
            s = dadd(s, P[(((long long)a * M + b) * K + ca) * K + (int)c[b]]);
    }
    out[i] = dmul(2.0, s);
}

int launch_pair_sums(const void* codes, int code_bytes, long long n, long long ldc, const double* P, int M, int K,
                     double* out, cudaStream_t s) {
    if (n <= 0) return 0;
    unsigned g = grid_for(n, 256, 1LL << 31);
    if (code_bytes == 1) pair_sums_kernel<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)codes, n, ldc, P, M, K, out);
    else if (code_bytes == 2) pair_sums_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)codes, n, ldc, P, M, K, out);
    else pair_sums_kernel<int32_t><<<g, 256, 0, s>>>((const int32_t*)codes, n, ldc, P, M, K, out);
    DA_CHECK_LAUNCH("pair_sums_kernel");
    return 0;
}

// ||q||^2 per query as one FMA chain (codebook.py:366)
__global__ void qsq_kernel(const double* __restrict__ Q, long long nq, int D, double* __restrict__ out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const double* q = Q + i * D;
    double s = 0.0;
    for (int d = 0; d < D; ++d) s = __fma_rn(q[d], q[d], s);
    out[i] = s;
}

int launch_qsq(const double* Q, long long nq, int D, double* out, cudaStream_t s) {
    if (nq <= 0) return 0;
    qsq_kernel<<<grid_for(nq, 128), 128, 0, s>>>(Q, nq, D, out);
    DA_CHECK_LAUNCH("qsq_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// ADC scan + top-r (codebook.py:399-429):
//   dist(p) = ((pair[p] - (M-1)*qsq) + lut[0][c0]) + ... + lut[M-1][c_{M-1}]
//   keep the r smallest by (dist, position p).
// One CTA per query: the query's M*K table lives in shared memory; each warp
// streams a strided share of the candidates into its own sorted top-r list
// (warp-cooperative insertion); warp 0 merges the lists at the end.
// Candidates are either positions 0..n-1 (cand == nullptr) or a per-query list
// of row ids cand[q*ncand + p] (position p breaks ties; the id is returned).

struct TopList {
    double* v;
    long long* p;
};

__device__ __forceinline__ void warp_insert(TopList L, int& cnt, int cap, double cv, long long cp) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    int pos = 0;
    for (int b = 0; b < cnt; b += 32) {
        int i = b + lane;
        bool lt = (i < cnt) && lex_less(L.v[i], L.p[i], cv, cp);
        pos += __popc(__ballot_sync(FULL, lt));
    }
    const int end = min(cnt, cap - 1);
    for (int b = end - 1; b >= pos; b -= 32) {
        int i = b - lane;
        bool act = i >= pos;
        double tv = 0.0; long long tp = 0;
        if (act) { tv = L.v[i]; tp = L.p[i]; }
        __syncwarp();
        if (act) { L.v[i + 1] = tv; L.p[i + 1] = tp; }
        __syncwarp();
    }
    if (lane == 0) { L.v[pos] = cv; L.p[pos] = cp; }
    __syncwarp();
    cnt = min(cnt + 1, cap);
}

template <typename TC>
__global__ void adc_scan_kernel(const TC* __restrict__ codes, long long ldc, const double* __restrict__ pair,
                                const long long* __restrict__ cand, long long ncand, const double* __restrict__ lut,
                                const double* __restrict__ qsq, int M, int K, int r,
                                long long* __restrict__ ids_out, double* __restrict__ d_out) {
    extern __shared__ __align__(16) char smem[];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long q = blockIdx.x;
    double* slut = (double*)smem;
    const int MK = M * K;
    for (int i = threadIdx.x; i < MK; i += blockDim.x) slut[i] = lut[q * MK + i];
    double* lv_base = slut + MK;
    long long* lp_base = (long long*)(lv_base + (size_t)nw * r);
    __syncthreads();
    TopList L{lv_base + (size_t)wid * r, lp_base + (size_t)wid * r};
    int cnt = 0;
    const double shift = dmul((double)(M - 1), qsq[q]);
    const long long* qc = cand ? cand + q * ncand : nullptr;
    for (long long b = (long long)wid * 32; b < ncand; b += (long long)nw * 32) {
        const long long p = b + lane;
        const bool valid = p < ncand;
        double dist = 0.0;
        if (valid) {
            const long long row = qc ? qc[p] : p;
            const TC* c = codes + row * ldc;
            dist = dsub(pair[row], shift);
            for (int m = 0; m < M; ++m) dist = dadd(dist, slut[m * K + (int)c[m]]);
        }
        auto accept = [&](double a, long long pa) -> bool {
            if (cnt < r) return true;
            return lex_less(a, pa, L.v[r - 1], L.p[r - 1]);
        };
        unsigned mask = __ballot_sync(FULL, valid && accept(dist, p));
        while (mask) {
            const int src = __ffs(mask) - 1;
            const double cv = __shfl_sync(FULL, dist, src);
            const long long cp = __shfl_sync(FULL, p, src);
            warp_insert(L, cnt, r, cv, cp);
            mask &= ~(1u << src);
            mask &= __ballot_sync(FULL, valid && accept(dist, p));
        }
    }
    // publish counts, merge into warp 0's list
    __shared__ int cnts[32];
    if (lane == 0) cnts[wid] = cnt;
    __syncthreads();
    if (wid == 0) {
        for (int w = 1; w < nw; ++w) {
            TopList O{lv_base + (size_t)w * r, lp_base + (size_t)w * r};
            const int oc = cnts[w];
            for (int b = 0; b < oc; b += 32) {
                const int i = b + lane;
                const bool valid = i < oc;
                double cv = valid ? O.v[i] : 0.0;
                long long cp = valid ? O.p[i] : 0;
                auto accept = [&](double a, long long pa) -> bool {
                    if (cnt < r) return true;
                    return lex_less(a, pa, L.v[r - 1], L.p[r - 1]);
                };
                unsigned mask = __ballot_sync(FULL, valid && accept(cv, cp));
                while (mask) {
                    const int src = __ffs(mask) - 1;
                    const double v = __shfl_sync(FULL, cv, src);
                    const long long pp = __shfl_sync(FULL, cp, src);
                    warp_insert(L, cnt, r, v, pp);
                    mask &= ~(1u << src);
                    mask &= __ballot_sync(FULL, valid && accept(cv, cp));
                }
            }
        }
        for (int i = lane; i < cnt; i += 32) {
            const long long p = L.p[i];
            ids_out[q * r + i] = qc ? qc[p] : p;
            d_out[q * r + i] = L.v[i];
        }
    }
}

// texmex record streams (data.py:50-142): rows of a 4-byte dimension header then
// d payload values (kind 0 = fvecs: float32, kind 1 = bvecs: uint8).  The raw
// records of a chunk are uploaded as they lie in the file and unpacked here into
// (n, d) float32 rows (bytes widen exactly); non-finite fvecs values are counted
// into *bad (the caller raises).  One thread per 4 payload values.
__global__ void unpack_vecs_kernel(const uint8_t* __restrict__ raw, long long n, int d, int kind,
                                   float* __restrict__ out, long long ldo, unsigned long long* __restrict__ bad) {
    const long long rec = 4 + (long long)d * (kind ? 1 : 4);
    const int qpr = (d + 3) / 4;  // quads per row
    unsigned nbad = 0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n * qpr;
         t += (long long)gridDim.x * blockDim.x) {
        const long long i = t / qpr;
        const int j0 = (int)(t - i * qpr) * 4;
        const uint8_t* r = raw + i * rec + 4;
        float* o = out + i * ldo;
        if (kind) {
            for (int j = j0; j < min(d, j0 + 4); ++j) o[j] = (float)r[j];
        } else {
            const float* rf = reinterpret_cast<const float*>(r);
            for (int j = j0; j < min(d, j0 + 4); ++j) {
                const float v = __ldg(rf + j);
                nbad += isfinite(v) ? 0u : 1u;
                o[j] = v;
            }
        }
    }
    if (bad && nbad) atomicAdd(bad, (unsigned long long)nbad);
}

int launch_unpack_vecs(const void* raw, long long n, int d, int kind, float* out, long long ldo,
                       unsigned long long* bad, cudaStream_t s) {
    if (n <= 0) return 0;
    const long long work = n * ((d + 3) / 4);
    unpack_vecs_kernel<<<grid_for(work, 256), 256, 0, s>>>((const uint8_t*)raw, n, d, kind, out, ldo, bad);
    DA_CHECK_LAUNCH("unpack_vecs_kernel");
    return 0;
}

// Packed candidate records (M <= 8 one-byte codes): record[row] = 16 bytes,
// codes in bytes 0..7, the row's pair sum (float64) in bytes 8..15, so one
// random candidate costs one 32-byte sector plus its 8-byte id.
__global__ void adc_pack_kernel(const uint8_t* __restrict__ codes, long long n, long long ldc,
                                const double* __restrict__ pair, int M, uint4* __restrict__ rec) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t w[2] = {0u, 0u};
        for (int m = 0; m < M; ++m) w[m >> 2] |= (uint32_t)codes[i * ldc + m] << (8 * (m & 3));
        const unsigned long long pb = __double_as_longlong(pair[i]);
        rec[i] = make_uint4(w[0], w[1], (uint32_t)pb, (uint32_t)(pb >> 32));
    }
}

int launch_adc_pack(const void* codes, long long n, long long ldc, const double* pair, int M, void* records,
                    cudaStream_t s) {
    if (n <= 0) return 0;
    adc_pack_kernel<<<grid_for(n, 256), 256, 0, s>>>((const uint8_t*)codes, n, ldc, pair, M, (uint4*)records);
    DA_CHECK_LAUNCH("adc_pack_kernel");
    return 0;
}

// Same scan over packed records; every lane scores ADC_U candidates per step so
// their id and record loads are in flight together.
#ifndef DA_ADC_U
#define DA_ADC_U 4
#endif
constexpr int ADC_U = DA_ADC_U;

// one random 16-byte record: no L1 allocation; HINT 1 adds the L2::64B prefetch
// granule, HINT 0 leaves the fetch size to the device limit
template <int HINT>
__device__ __forceinline__ uint4 adc_ld_rec(const uint4* p) {
    uint4 v;
    if (HINT)
        asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
    return v;
}

__device__ __forceinline__ double adc_rec_dist(uint4 rc, const double* slut, int M, int K, double shift) {
    double dist = dsub(__hiloint2double((int)rc.w, (int)rc.z), shift);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        if (m < M) {
            const uint32_t word = m < 4 ? rc.x : rc.y;
            dist = dadd(dist, slut[m * K + (int)((word >> (8 * (m & 3))) & 0xFFu)]);
        }
    }
    return dist;
}

// order-preserving 64-bit key of a non-NaN double (for the shared threshold)
__device__ __forceinline__ unsigned long long dkey(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// Candidates stream through a two-deep software pipeline: the ids of step i+1
// are in flight while the records of step i are scored.  The warps of a CTA
// share one threshold (the smallest r-th distance of any warp's full list): a
// candidate above it cannot be in the query's top r, so it is never inserted.
template <int HINT>
__global__ void adc_scan_packed_kernel(const uint4* __restrict__ rec, const long long* __restrict__ cand,
                                       long long ncand, const double* __restrict__ lut,
                                       const double* __restrict__ qsq, int M, int K, int r,
                                       long long* __restrict__ ids_out, double* __restrict__ d_out) {
    extern __shared__ __align__(16) char smem[];
    __shared__ unsigned long long s_thr;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long q = blockIdx.x;
    double* slut = (double*)smem;
    const int MK = M * K;
    for (int i = threadIdx.x; i < MK; i += blockDim.x) slut[i] = lut[q * MK + i];
    double* lv_base = slut + MK;
    long long* lp_base = (long long*)(lv_base + (size_t)nw * r);
    if (threadIdx.x == 0) s_thr = ~0ULL;
    __syncthreads();
    TopList L{lv_base + (size_t)wid * r, lp_base + (size_t)wid * r};
    int cnt = 0;
    const double shift = dmul((double)(M - 1), qsq[q]);
    const long long* qc = cand ? cand + q * ncand : nullptr;
    const long long stride = (long long)nw * 32 * ADC_U;
    auto load_rows = [&](long long b, long long* row) {
#pragma unroll
        for (int u = 0; u < ADC_U; ++u) {
            const long long p = b + u * 32 + lane;
            row[u] = p < ncand ? (qc ? __ldg(qc + p) : p) : -1;
        }
    };
    long long row[ADC_U], nrow[ADC_U];
    long long b = (long long)wid * 32 * ADC_U;
    load_rows(b, row);
    for (; b < ncand; b += stride) {
        uint4 rc[ADC_U];
#pragma unroll
        for (int u = 0; u < ADC_U; ++u) rc[u] = row[u] >= 0 ? adc_ld_rec<HINT>(rec + row[u]) : make_uint4(0, 0, 0, 0);
        load_rows(b + stride, nrow);
        const unsigned long long thr = *(volatile unsigned long long*)&s_thr;
#pragma unroll
        for (int u = 0; u < ADC_U; ++u) {
            const bool valid = row[u] >= 0;
            const double dist = valid ? adc_rec_dist(rc[u], slut, M, K, shift) : 0.0;
            const long long p = b + u * 32 + lane;
            auto accept = [&](double a, long long pa) -> bool {
                if (dkey(a) > thr) return false;
                if (cnt < r) return true;
                return lex_less(a, pa, L.v[r - 1], L.p[r - 1]);
            };
            unsigned mask = __ballot_sync(FULL, valid && accept(dist, p));
            while (mask) {
                const int src = __ffs(mask) - 1;
                const double cv = __shfl_sync(FULL, dist, src);
                const long long cp = __shfl_sync(FULL, p, src);
                warp_insert(L, cnt, r, cv, cp);
                mask &= ~(1u << src);
                mask &= __ballot_sync(FULL, valid && accept(dist, p));
            }
        }
        if (cnt == r && lane == 0) atomicMin(&s_thr, dkey(L.v[r - 1]));
#pragma unroll
        for (int u = 0; u < ADC_U; ++u) row[u] = nrow[u];
    }
    __shared__ int cnts[32];
    if (lane == 0) cnts[wid] = cnt;
    __syncthreads();
    if (wid == 0) {
        for (int w = 1; w < nw; ++w) {
            TopList O{lv_base + (size_t)w * r, lp_base + (size_t)w * r};
            const int oc = cnts[w];
            for (int b2 = 0; b2 < oc; b2 += 32) {
                const int i = b2 + lane;
                const bool valid = i < oc;
                double cv = valid ? O.v[i] : 0.0;
                long long cp = valid ? O.p[i] : 0;
                auto accept = [&](double a, long long pa) -> bool {
                    if (cnt < r) return true;
                    return lex_less(a, pa, L.v[r - 1], L.p[r - 1]);
                };
                unsigned mask = __ballot_sync(FULL, valid && accept(cv, cp));
                while (mask) {
                    const int src = __ffs(mask) - 1;
                    const double v = __shfl_sync(FULL, cv, src);
                    const long long pp2 = __shfl_sync(FULL, cp, src);
                    warp_insert(L, cnt, r, v, pp2);
                    mask &= ~(1u << src);
                    mask &= __ballot_sync(FULL, valid && accept(cv, cp));
                }
            }
        }
        for (int i = lane; i < cnt; i += 32) {
            const long long p = L.p[i];
            ids_out[q * r + i] = qc ? qc[p] : p;
            d_out[q * r + i] = L.v[i];
        }
    }
}

int launch_adc_scan_packed(const void* records, const long long* cand, long long ncand, long long nq,
                           const double* lut, const double* qsq, int M, int K, int r, long long* ids_out,
                           double* d_out, cudaStream_t s) {
    if (nq <= 0) return 0;
    if (M < 1 || M > 8 || K > 256) return fail_arg("adc_scan_packed: needs M <= 8 one-byte codes (M=%d K=%d)", M, K);
    if (r < 1 || r > ncand) return fail_arg("r=%d must be in [1, %lld]", r, ncand);
    const size_t lut_b = sizeof(double) * (size_t)M * K;
    int warps = 8;
    while (warps > 1 && lut_b + (size_t)warps * r * 16 > 200 * 1024) warps >>= 1;
    const size_t smem = lut_b + (size_t)warps * r * 16;
    if (smem > 220 * 1024) return fail_arg("adc_scan: r=%d with M*K=%d exceeds shared memory", r, M * K);
    // DA_ADC_HINT=0 drops the L2::64B qualifier (measured: 128 B of DRAM per
    // record instead of 64; cudaLimitMaxL2FetchGranularity has no effect)
    const char* eh = getenv("DA_ADC_HINT");
    const int hint = eh ? atoi(eh) : 1;
    auto kf = hint ? adc_scan_packed_kernel<1> : adc_scan_packed_kernel<0>;
    ProfScope ps("adc_scan_packed", s);
    if (smem > 48 * 1024)
        DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kf<<<(unsigned)nq, warps * 32, smem, s>>>((const uint4*)records, cand, ncand, lut, qsq, M, K, r, ids_out, d_out);
    DA_CHECK_LAUNCH("adc_scan_packed_kernel");
    return 0;
}

int launch_adc_scan(const void* codes, int code_bytes, long long ldc, const double* pair, const long long* cand,
                    long long ncand, long long nq, const double* lut, const double* qsq, int M, int K, int r,
                    long long* ids_out, double* d_out, cudaStream_t s) {
    if (nq <= 0) return 0;
    if (r < 1 || r > ncand) return fail_arg("r=%d must be in [1, %lld]", r, ncand);
    const size_t lut_b = sizeof(double) * (size_t)M * K;
    int warps = 8;
    while (warps > 1 && lut_b + (size_t)warps * r * 16 > 200 * 1024) warps >>= 1;
    const size_t smem = lut_b + (size_t)warps * r * 16;
    if (smem > 220 * 1024) return fail_arg("adc_scan: r=%d with M*K=%d exceeds shared memory", r, M * K);
    ProfScope ps("adc_scan", s);
#define ADC_LAUNCH(TC)                                                                                       \
    do {                                                                                                     \
        auto kf = adc_scan_kernel<TC>;                                                                       \
        if (smem > 48 * 1024) DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        kf<<<(unsigned)nq, warps * 32, smem, s>>>((const TC*)codes, ldc, pair, cand, ncand, lut, qsq, M, K, r,  \
                                                  ids_out, d_out);                                         \
    } while (0)
    if (code_bytes == 1) ADC_LAUNCH(uint8_t);
    else if (code_bytes == 2) ADC_LAUNCH(uint16_t);
    else ADC_LAUNCH(int32_t);
#undef ADC_LAUNCH
    DA_CHECK_LAUNCH("adc_scan_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// numpy 1-D mean (pairwise_sum over the whole array, then / n).  The recursion
// depends only on n, so its tree is built once per n on the host: leaves are
// summed in parallel, internal nodes are folded level by level in one block.

struct PwPlan {
    int n_leaves = 0, n_nodes = 0;  // values: [leaves..., internal nodes by height]
    int n_levels = 0;
    long long* leaf_lo = nullptr;   // device
    int* leaf_n = nullptr;
    int2* kids = nullptr;           // device, per internal node (value indices)
    int* level_off = nullptr;       // device, n_levels+1 offsets into internal nodes
    std::vector<int> h_level_off;
};

static std::mutex g_plan_mu;
static std::map<std::pair<int, long long>, PwPlan> g_plans;  // (device, n)

static int build_plan(long long n, PwPlan& P) {
    struct Node { int l, r, h; };
    std::vector<long long> lo_v;
    std::vector<int> n_v;
    std::vector<Node> inner;  // temp ids: leaves >= 0 -> value id; inner encoded as -(idx+1)
    // recursive build returning encoded id and height
    struct Frame { long long lo, n; int state; int left; int lh; };
    std::vector<Frame> st;
    st.push_back({0, n, 0, 0, 0});
    int ret = 0, reth = 0;
    while (!st.empty()) {
        Frame& f = st.back();
        if (f.n <= 128 && f.state == 0) {
            lo_v.push_back(f.lo); n_v.push_back((int)f.n);
            ret = (int)lo_v.size() - 1; reth = 0;
            st.pop_back();
            continue;
        }
        long long n2 = f.n / 2; n2 -= n2 % 8;
        if (f.state == 0) { f.state = 1; st.push_back({f.lo, n2, 0, 0, 0}); continue; }
        if (f.state == 1) { f.left = ret; f.lh = reth; f.state = 2; long long lo = f.lo + n2, rn = f.n - n2; st.push_back({lo, rn, 0, 0, 0}); continue; }
        // state 2: right done
        int h = 1 + (f.lh > reth ? f.lh : reth);
        inner.push_back({f.left, ret, h});
        ret = -(int)inner.size();
        reth = h;
        st.pop_back();
    }
    const int nl = (int)lo_v.size();
    const int ni = (int)inner.size();
    int maxh = 0;
    for (auto& x : inner) maxh = x.h > maxh ? x.h : maxh;
    // order internal nodes by height (stable)
    std::vector<int> newid(ni);
    std::vector<int> off(maxh + 2, 0);
    for (auto& x : inner) off[x.h + 1]++;
    for (int h = 1; h <= maxh + 1; ++h) off[h] += off[h - 1];
    std::vector<int> fill(off.begin(), off.end());
    for (int i = 0; i < ni; ++i) newid[i] = fill[inner[i].h]++;
    auto val_id = [&](int enc) { return enc >= 0 ? enc : nl + newid[-enc - 1]; };
    std::vector<int2> kids(ni > 0 ? ni : 1);
    for (int i = 0; i < ni; ++i) kids[newid[i]] = make_int2(val_id(inner[i].l), val_id(inner[i].r));
    P.n_leaves = nl; P.n_nodes = ni; P.n_levels = maxh;
    // level offsets for heights 1..maxh (internal nodes have h >= 1)
    P.h_level_off.assign(off.begin() + 1, off.end());  // size maxh+1: start of h=1 .. end
    cudaError_t e;
    if ((e = cudaMalloc(&P.leaf_lo, sizeof(long long) * nl)) != cudaSuccess) return fail_cuda(e, "plan alloc");
    if ((e = cudaMalloc(&P.leaf_n, sizeof(int) * nl)) != cudaSuccess) return fail_cuda(e, "plan alloc");
    if ((e = cudaMalloc(&P.kids, sizeof(int2) * kids.size())) != cudaSuccess) return fail_cuda(e, "plan alloc");
    if ((e = cudaMalloc(&P.level_off, sizeof(int) * P.h_level_off.size())) != cudaSuccess) return fail_cuda(e, "plan alloc");
    cudaMemcpy(P.leaf_lo, lo_v.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice);
    cudaMemcpy(P.leaf_n, n_v.data(), sizeof(int) * nl, cudaMemcpyHostToDevice);
    cudaMemcpy(P.kids, kids.data(), sizeof(int2) * kids.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(P.level_off, P.h_level_off.data(), sizeof(int) * P.h_level_off.size(), cudaMemcpyHostToDevice);
    return 0;
}

__global__ void pw_leaves_kernel(const double* __restrict__ a, const long long* __restrict__ lo,
                                 const int* __restrict__ ln, int nl, double* __restrict__ vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    const double* base = a + lo[i];
    vals[i] = np_pw_leaf([&](long long j) { return base[j]; }, 0, ln[i]);
}

__global__ void pw_fold_kernel(double* __restrict__ vals, const int2* __restrict__ kids, const int* __restrict__ level_off,
                               int n_levels, int nl, double div, double* __restrict__ out) {
    for (int h = 0; h < n_levels; ++h) {
        for (int i = level_off[h] + threadIdx.x; i < level_off[h + 1]; i += blockDim.x) {
            int2 k = kids[i];
            vals[nl + i] = dadd(vals[k.x], vals[k.y]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double s = (n_levels > 0) ? vals[nl + level_off[n_levels] - 1] : vals[0];
        *out = (div != 0.0) ? __ddiv_rn(s, div) : s;
    }
}

// out = sum(a) (divide==0) or mean(a) (divide==1), numpy pairwise order.
int launch_np_sum(const double* a, long long n, int divide, double* out, cudaStream_t s) {
    if (n <= 0) return fail_arg("np_sum: n must be positive");
    int dev = 0;
    cudaGetDevice(&dev);
    PwPlan* P;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        auto key = std::make_pair(dev, n);
        auto it = g_plans.find(key);
        if (it == g_plans.end()) {
            PwPlan np_;
            int rc = build_plan(n, np_);
            if (rc) return rc;
            it = g_plans.emplace(key, np_).first;
        }
        P = &it->second;
    }
    const int total = P->n_leaves + P->n_nodes;
    double* vals = (double*)scratch(4, sizeof(double) * (size_t)total, s);
    if (!vals) return fail_cuda(cudaErrorMemoryAllocation, "np_sum scratch");
    pw_leaves_kernel<<<grid_for(P->n_leaves, 128), 128, 0, s>>>(a, P->leaf_lo, P->leaf_n, P->n_leaves, vals);
    DA_CHECK_LAUNCH("pw_leaves_kernel");
    pw_fold_kernel<<<1, 1024, 0, s>>>(vals, P->kids, P->level_off, P->n_levels, P->n_leaves,
                                      divide ? (double)n : 0.0, out);
    DA_CHECK_LAUNCH("pw_fold_kernel");
    return 0;
}

// ---------------------------------------------------------------------------
// small helpers for the Lloyd loop and the sweep

// C[dst[i]] = X[src[i]] (full rows), used by the empty-cluster reseed.
__global__ void gather_rows_kernel(const double* __restrict__ X, long long ldx, int D, const long long* __restrict__ src,
                                   const int* __restrict__ dst, int cnt, double* __restrict__ C, long long ldc) {
    int i = blockIdx.y;
    if (i >= cnt) return;
    for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x)
        C[(long long)dst[i] * ldc + d] = X[src[i] * ldx + d];
}

int launch_gather_rows(const double* X, long long ldx, int D, const long long* src, const int* dst, int cnt, double* C,
                       long long ldc, cudaStream_t s) {
    if (cnt <= 0) return 0;
    dim3 g((D + 127) / 128, cnt);
    gather_rows_kernel<<<g, 128, 0, s>>>(X, ldx, D, src, dst, cnt, C, ldc);
    DA_CHECK_LAUNCH("gather_rows_kernel");
    return 0;
}

// da_sweep's keep-the-better rule (annealing.py:173-176):
// take = beam_err <= inc_err; codes = take ? beam : incumbent; err = take ? beam : inc
__global__ void select_better_kernel(long long n, int M, const int32_t* __restrict__ beam_codes,
                                     const double* __restrict__ beam_err, int32_t* __restrict__ inc_codes,
                                     double* __restrict__ inc_err) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (beam_err[i] <= inc_err[i]) {
        for (int m = 0; m < M; ++m) inc_codes[i * M + m] = beam_codes[i * M + m];
        inc_err[i] = beam_err[i];
    }
}

int launch_select_better(long long n, int M, const int32_t* beam_codes, const double* beam_err, int32_t* inc_codes,
                         double* inc_err, cudaStream_t s) {
    if (n <= 0) return 0;
    select_better_kernel<<<grid_for(n, 256, 1LL << 31), 256, 0, s>>>(n, M, beam_codes, beam_err, inc_codes, inc_err);
    DA_CHECK_LAUNCH("select_better_kernel");
    return 0;
}

// codes[:, m] = labels
__global__ void set_column_kernel(int32_t* __restrict__ codes, long long n, int M, int m,
                                  const int32_t* __restrict__ labels) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) codes[i * M + m] = labels[i];
}

int launch_set_column(int32_t* codes, long long n, int M, int m, const int32_t* labels, cudaStream_t s) {
    if (n <= 0) return 0;
    set_column_kernel<<<grid_for(n, 256, 1LL << 31), 256, 0, s>>>(codes, n, M, m, labels);
    DA_CHECK_LAUNCH("set_column_kernel");
    return 0;
}

}  // namespace da

// Filtered beam encoder: fp32 fast path + exact float64 recheck.
//
// Same contract as encode.cu (annq/codebook.py:255-300, bit-exact result), but
// the full float64 score table and the float64 cross-term gathers are only
// computed for candidates that can still make the beam:
//
//   1. t'[m,k] = sq32 - 2 x.c in FP32 (SGEMM, FFMA, 128x128 tiles).
//   2. per stage and vector, v'(l,k) = s_l + t'[m,k] + 2 sum_{j<m} P32[j,m][c_lj,k]
//      for every candidate, with a rigorous bound |v' - v| <= E (fp32 rounding of
//      the dot products, of the table entries and of the additions; see
//      stage_bound below).
//   3. tau' = an upper bound of the width-th smallest v' (the width-th smallest
//      of the two smallest per lane).  No candidate with v' > tau' + 2E can be
//      among the exact top-width (proof in DESIGN.md), so only candidates with
//      v' <= tau' + 2E are recomputed in float64 exactly as the reference does
//      (BLAS-ordered x.c, einsum ||c||^2, sequential cross sum) and go through the
//      exact (value, flat index) top-width selection.
// Beam scores are always the exact float64 values, so codes and errors equal
// the reference's; only the amount of float64 work changes.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "beam_filter.cuh"

namespace da {

// ---------------------------------------------------------------------------
// SGEMM for the approximate score table: T[i, j] = sq32[j] - 2 * sum_k X[i,k] C[j,k]
namespace {
constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 8, SG_T = 256;

// FFMA table chunk length: ~sqrt(D) rounded to a multiple of SG_BK (minimises
// chunk + D/chunk), or 0 (one sequential chain).  DA_SGEMM_CHUNK
// overrides it (0 = sequential) for A/B runs.
// Chunking costs registers (one CTA per SM: the D=960 table takes 155 instead
// of 124 ms per 1M vectors) and pays where the rechecks it saves are many:
// wide beams (L=10, D=960: beam 248 -> 191 ms) and the greedy L=1 kernel,
// whose exact stages follow the band (D=960 per 200k: greedy 20 -> 6 ms,
// table 25 -> 31 ms).
int sgemm_chunk(int D, int L) {
    if (const char* e = getenv("DA_SGEMM_CHUNK")) {
        const int c = atoi(e);
        return c <= 0 ? 0 : ((c + SG_BK - 1) / SG_BK) * SG_BK;
    }
    if (D < 256 || (L > 1 && L < 8)) return 0;   // L = 1: the greedy kernel's band is the bound
    int c = (int)(sqrt((double)D) / SG_BK + 0.5) * SG_BK;
    return c < SG_BK ? SG_BK : c;
}
}

// chunk == 0: one sequential FFMA chain over D per entry.  chunk >= 8 (a multiple
// of SG_BK): the chain restarts every `chunk` terms and the partials are added
// into a second accumulator, so the rounding error grows with chunk + D/chunk
// instead of D (table_err in beam_filter.cuh); at D=960 that is 62 roundings
// instead of 960, and the exact-recheck queue shrinks with the bound.
template <bool CHUNKED>
__global__ void __launch_bounds__(SG_T) sgemm_table_kernel(const float* __restrict__ X, long long n, long long ldx,
                                                           const float* __restrict__ Cw, int N, int D,
                                                           const float* __restrict__ sq32, float* __restrict__ T,
                                                           long long ldt, int chunk) {
    __shared__ __align__(16) float As[2][SG_BK][SG_BM];
    __shared__ __align__(16) float Bs[2][SG_BK][SG_BN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const long long i0 = (long long)blockIdx.y * SG_BM;
    const int j0 = blockIdx.x * SG_BN;
    float acc[8][8], tot[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = tot[i][j] = 0.f;
    // each thread loads 4 A elements and 4 B elements per k-tile
    const int lr = tid >> 1;          // row within tile (0..127)
    const int lk = (tid & 1) * 4;     // k offset 0 or 4
    float ra[4], rb[4];
    auto load = [&](int k0) {
        long long gr = i0 + lr;
        int gc = j0 + lr;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int gk = k0 + lk + u;
            ra[u] = (gr < n && gk < D) ? X[gr * ldx + gk] : 0.f;
            rb[u] = (gc < N && gk < D) ? Cw[(long long)gc * D + gk] : 0.f;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            As[buf][lk + u][lr] = ra[u];
            Bs[buf][lk + u][lr] = rb[u];
        }
    };
    load(0);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < D; k0 += SG_BK) {
        const bool more = k0 + SG_BK < D;
        if (more) load(k0 + SG_BK);
#pragma unroll
        for (int k = 0; k < SG_BK; ++k) {
            float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
            float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
            float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
            float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
            float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (CHUNKED && (!more || (k0 + SG_BK) % chunk == 0)) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    tot[i][j] += acc[i][j];
                    acc[i][j] = 0.f;
                }
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        long long gr = i0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (gr >= n) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int gc = j0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (gc < N) T[gr * ldt + gc] = sq32[gc] - 2.f * (CHUNKED ? tot[i][j] : acc[i][j]);
        }
    }
}

// per-dictionary bound inputs: cmax[m] = max_k ||c_mk||, crossb[m] = sum_{j<m} max|P[j,m]|
__global__ void bound_prep_kernel(const float* __restrict__ cw, const double* __restrict__ P, int M, int K, int D,
                                  const double* __restrict__ sq, float* __restrict__ P32, float* __restrict__ sq32,
                                  double* __restrict__ cmax, double* __restrict__ pabs, double* __restrict__ cw64) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)M * K * D;
         e += (long long)gridDim.x * blockDim.x)
        cw64[e] = (double)cw[e];
    // grid: (M*M) blocks for the table conversion + maxima; block 0..M-1 also do norms
    const int pair = blockIdx.x;
    const int a = pair / M, b = pair % M;
    __shared__ double red[256];
    double mx = 0.0;
    const long long base = (long long)pair * K * K;
    for (long long e = threadIdx.x; e < (long long)K * K; e += blockDim.x) {
        double v = P[base + e];
        P32[base + e] = (float)v;
        mx = fmax(mx, fabs(v));
    }
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) pabs[a * M + b] = red[0];
    __syncthreads();
    if (b == 0) {
        // norms of dictionary a
        double cm = 0.0;
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            double s = sq[a * K + k];
            sq32[a * K + k] = (float)s;
            cm = fmax(cm, sqrt(s));
        }
        red[threadIdx.x] = cm;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
            __syncthreads();
        }
        if (threadIdx.x == 0) cmax[a] = red[0] * (1.0 + 1e-12);
    }
}

// LEAN: no shared-memory copy of the candidate values (the few lanes that hold
// two or more candidates under the limit recompute theirs), groups of two beams:
// ~5 KB of shared memory and <= 80 registers per warp, so 24 warps fit an SM
// instead of 16.  Same values, same codes.
#ifndef DA_LEAN_MINB
#define DA_LEAN_MINB 3
#endif
#ifndef DA_LEAN_G
#define DA_LEAN_G 2
#endif
// cbm[m] = (1 + 1e-12) * sum_{j<m} max|P[j,m]|: the cross-term bound of stage m
__global__ void cb_prep_kernel(const double* __restrict__ pabs, int M, double* __restrict__ cbm) {
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        double c = 0.0;
        for (int j = 0; j < m; ++j) c += pabs[j * M + m];
        cbm[m] = c * (1.0 + 1e-12);
    }
}

// Exact float64 value of candidate `flat` of stage m, in the reference's order
// (BLAS-ordered x.c, einsum ||c||^2, sequential cross sum).  Out of line: it is
// called from the queue pass and from the overflow path, and the kernel's hot
// loops must stay within the instruction cache.
template <bool INL>
__device__ __forceinline__ double beam_exact_value_t(const double* __restrict__ x64, const double* __restrict__ cw64,
                                                const float* __restrict__ cw32, int D, const double* __restrict__ sq,
                                                const double* __restrict__ P, const int32_t* __restrict__ pc,
                                                const double* __restrict__ ps, int M, int K, int m, int flat, int k_sh,
                                                const long long* __restrict__ roff = nullptr) {
    const int l = k_sh >= 0 ? flat >> k_sh : flat / K;
    const int k = flat - l * K;
    const double xc = exact_dot(x64, cw64 + ((long long)m * K + k) * D, D, cw32 ? cw32 + ((long long)m * K + k) * D : nullptr);
    const double t = dsub(sq[m * K + k], dmul(2.0, xc));
    double cross = 0.0;
    if (roff) {   // this stage's row offsets (same layout as the float table)
#pragma unroll 1
        for (int j = 0; j < m; ++j) cross = dadd(cross, P[roff[l * M + j] + k]);
    } else {
#pragma unroll 1
        for (int j = 0; j < m; ++j) cross = dadd(cross, P[(((long long)j * M + m) * K + pc[l * M + j]) * K + k]);
    }
    return dadd(dadd(ps[l], t), dmul(2.0, cross));
}
__device__ __noinline__ double beam_exact_value(const double* __restrict__ x64, const double* __restrict__ cw64,
                                                const float* __restrict__ cw32, int D, const double* __restrict__ sq,
                                                const double* __restrict__ P, const int32_t* __restrict__ pc,
                                                const double* __restrict__ ps, int M, int K, int m, int flat, int k_sh) {
    return beam_exact_value_t<false>(x64, cw64, cw32, D, sq, P, pc, ps, M, K, m, flat, k_sh);
}

// Rare path: more near-boundary candidates than the queue holds -> exact
// streaming selection over every candidate of the stage (warp-collective).
__device__ __noinline__ void beam_overflow_select(FastSmem S, int total, int width, const double* __restrict__ x64,
                                                  const double* __restrict__ cw64, const float* __restrict__ cw32,
                                                  int D, const double* __restrict__ sq, const double* __restrict__ P,
                                                  const int32_t* __restrict__ pc, const double* __restrict__ ps, int M,
                                                  int K, int m, int k_sh, unsigned long long& n_exact) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    int cnt = 0;
    auto accept = [&](double a, int fa) -> bool {
        if (cnt < width) return true;
        return lex_less(a, fa, S.lv[width - 1], S.lf[width - 1]);
    };
    for (int b = 0; b < total; b += 32) {
        const int flat = b + lane;
        const bool has = flat < total;
        const double val = has ? beam_exact_value(x64, cw64, cw32, D, sq, P, pc, ps, M, K, m, flat, k_sh) : 0.0;
        n_exact += has ? 1 : 0;
        unsigned mask = __ballot_sync(FULL, has && accept(val, flat));
        while (mask) {
            const int src = __ffs(mask) - 1;
            const double cv = __shfl_sync(FULL, val, src);
            const int cf = __shfl_sync(FULL, flat, src);
            int pos = 0;
            for (int bb = 0; bb < cnt; bb += 32) {
                int i = bb + lane;
                bool lt = (i < cnt) && lex_less(S.lv[i], S.lf[i], cv, cf);
                pos += __popc(__ballot_sync(FULL, lt));
            }
            const int endp = min(cnt, width - 1);
            for (int bb = endp - 1; bb >= pos; bb -= 32) {
                int i = bb - lane;
                bool act = i >= pos;
                double tv = 0.0;
                int tf = 0;
                if (act) { tv = S.lv[i]; tf = S.lf[i]; }
                __syncwarp();
                if (act) { S.lv[i + 1] = tv; S.lf[i + 1] = tf; }
                __syncwarp();
            }
            if (lane == 0) { S.lv[pos] = cv; S.lf[pos] = cf; }
            __syncwarp();
            cnt = min(cnt + 1, width);
            mask &= ~(1u << src);
            mask &= __ballot_sync(FULL, has && accept(val, flat));
        }
    }
    __syncwarp();
}

// Exact error of the chosen code (reconstruction in m order, numpy pairwise
// over d; diff^2 staged in dd).  Out of line: once per vector, off the hot path.
__device__ __noinline__ void beam_final_error(const double* __restrict__ x64, double* __restrict__ dd,
                                              const float* __restrict__ cw, const int32_t* __restrict__ best, int M,
                                              int K, int D, double* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    for (int d = lane; d < D; d += 32) {
        double r = 0.0;
        for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + best[j]) * D + d]);
        double df = dsub(x64[d], r);
        dd[d] = dmul(df, df);
    }
    __syncwarp();
    if (lane == 0) *err = np_pw_sum([&](long long i) { return dd[i]; }, 0, D);
}

template <typename TX, bool LEAN, bool VEC>
__global__ void __launch_bounds__(256, LEAN ? DA_LEAN_MINB : 2) beam_fast_kernel(
    const TX* __restrict__ X, long long n, long long ldx, int D, const float* __restrict__ cw, int M, int K, int L,
    int cap, const float* __restrict__ tab32, const double* __restrict__ sq, const double* __restrict__ P,
    const float* __restrict__ P32, const double* __restrict__ cmax, const double* __restrict__ cbm,
    const double* __restrict__ cw64, void* codes_out,
    int code_bytes, long long ldcodes, double* __restrict__ err_out, unsigned long long* __restrict__ stats, int tab_tc) {
    extern __shared__ __align__(16) char smem_raw[];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const long long v = (long long)blockIdx.x * nwarps + wid;
    if (v >= n) return;
    FastSmem S = carve_fast(smem_raw + (size_t)wid * fast_smem_bytes(cap, M, K, D, LEAN), cap, M, K, D, LEAN);
    // 16-byte aligned fp32 codeword rows (D % 4 == 0): vector loads in the exact dot
    const int nkb = (K + 31) / 32;
    const int nkb_sh = (nkb & (nkb - 1)) == 0 ? __ffs(nkb) - 1 : -1;
    const bool c32ok = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(cw) & 15) == 0);
    // power-of-two shapes index with shifts instead of integer division
    const int k_sh = (K & (K - 1)) == 0 ? __ffs(K) - 1 : -1;
    const float* trow = tab32 + v * (long long)M * K;
    const TX* xr = X + v * ldx;
    // x in float64 (exact widening) and ||x||
    double xx_part = 0.0;
#pragma unroll 1
    for (int d = lane; d < D; d += 32) {
        double t = (double)xr[d];
        S.x64[d] = t;
        xx_part = __fma_rn(t, t, xx_part);
    }
    for (int off = 16; off >= 1; off >>= 1) xx_part += __shfl_xor_sync(FULL, xx_part, off);
    const double xnorm = sqrt(xx_part) * (1.0 + 1e-12);
    if (lane == 0) S.score[0] = 0.0;
    __syncwarp();
    const double u = 5.9604644775390625e-08;  // 2^-24
    unsigned long long n_exact = 0;

    // the score-independent part of every stage's bound, lane m holding stage m's
    double a_stage = 0.0;
    for (int mm = lane; mm < M; mm += 32) {
        const double cb = cbm[mm], cm = cmax[mm];
        const double tmax = cm * cm + 2.0 * xnorm * cm;
        const double a = 2.0 * (table_err(tab_tc, D, u, xnorm, cm) + 2.0 * ((mm + 2.0) * u * cb) +
                                4.0 * u * (tmax + 2.0 * cb));
        if (mm == lane) a_stage = a;
    }
    int cur = 0, live = 1;
    for (int m = 0; m < M; ++m) {
        const int total = live * K;
        const int width = min(L, total);
        const int32_t* pc = S.codes + cur * cap * M;
        const double* ps = S.score + cur * cap;
        // ---- rigorous bound of |v' - v| for this stage
        // max |score| rounded up to float (non-negative floats order like their bits)
        unsigned sbits = lane < live ? __float_as_uint(__double2float_ru(fabs(ps[lane]))) : 0u;
#pragma unroll 1
        for (int l = lane + 32; l < live; l += 32) sbits = max(sbits, __float_as_uint(__double2float_ru(fabs(ps[l]))));
        const double smax = (double)__uint_as_float(__reduce_max_sync(FULL, sbits));
        double a_m = __shfl_sync(FULL, a_stage, m & 31);
        if (M > 32) {   // more stages than lanes: this stage's constant directly
            const double cb = cbm[m], cm = cmax[m];
            a_m = 2.0 * (table_err(tab_tc, D, u, xnorm, cm) + 2.0 * ((m + 2.0) * u * cb) +
                         4.0 * u * (cm * cm + 2.0 * xnorm * cm + 2.0 * cb));
        }
        const double E = a_m + 10.0 * u * smax + 1e-300;

        for (int e = lane; e < live * m; e += 32) {
            const int l = e / m, j = e % m;
            S.roff[l * M + j] = (((long long)j * M + m) * K + pc[l * M + j]) * K;
        }
        __syncwarp();
        // ---- pass A: approximate candidate values; per lane the two smallest
        // (and the index of the smallest).  With K % 256 == 0 a lane owns
        // k = kb + 4*lane + {0..3} and kb + 128 + 4*lane + {0..3} (16-B gathers),
        // otherwise k = kb + 32q + lane.  Four beams are processed together.
        const bool vec = VEC;   // K % 256 == 0: 16-byte gathers (compile-time, keeps the code small)
        auto kof = [&](int kb, int q) -> int {
            return vec ? kb + (q >> 2) * 128 + 4 * lane + (q & 3) : kb + 32 * q + lane;
        };
        float m1 = __int_as_float(0x7f800000), m2 = m1;
        int i1 = -1;
        for (int kb = 0; kb < K; kb += 256) {
            float tk[8];
            if (vec) {
                const float4 a = ld_stream_f4(trow + m * K + kb + 4 * lane);
                const float4 b = ld_stream_f4(trow + m * K + kb + 128 + 4 * lane);
                tk[0] = a.x; tk[1] = a.y; tk[2] = a.z; tk[3] = a.w; tk[4] = b.x; tk[5] = b.y; tk[6] = b.z; tk[7] = b.w;
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k = kof(kb, q);
                    tk[q] = (k < K) ? trow[m * K + k] : 0.f;
                }
            }
            // A group of G consecutive beams (flat-index order = lexicographic order
            // of the code prefixes) shares its first gl codes, so the rows j < gl
            // are gathered once and the running sum is copied to every beam; the
            // additions stay in j order, so each value is bit-identical to a
            // per-beam gather.  A tail group has exactly live - l0 beams.
            auto group = [&](auto Gc, int l0) {
                constexpr int G = decltype(Gc)::value;
                const int last = l0 + G - 1;
                const bool same = lane < m && pc[l0 * M + lane] == pc[last * M + lane];
                const unsigned neq = ~__ballot_sync(FULL, same);
                const int gl = neq ? min(m, __ffs(neq) - 1) : min(m, 32);
                float acc[G][8];
                {
                    float sh[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) sh[q] = 0.f;
                    for (int j = 0; j < gl; ++j) {
                        const float* rp = P32 + S.roff[l0 * M + j] + kb;
                        if (vec) {
                            const float4 a = __ldg(reinterpret_cast<const float4*>(rp + 4 * lane));
                            const float4 b = __ldg(reinterpret_cast<const float4*>(rp + 128 + 4 * lane));
                            add2(sh[0], sh[1], a.x, a.y); add2(sh[2], sh[3], a.z, a.w);
                            add2(sh[4], sh[5], b.x, b.y); add2(sh[6], sh[7], b.z, b.w);
                        } else {
#pragma unroll
                            for (int q = 0; q < 8; ++q) sh[q] += (kof(kb, q) < K) ? __ldg(rp + 32 * q + lane) : 0.f;
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[g][q] = sh[q];
                }
                for (int j = gl; j < m; ++j) {
                    const float* rp[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) rp[g] = P32 + S.roff[(l0 + g) * M + j] + kb;
                    float vals[G][8];
                    if (vec) {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float4 a = __ldg(reinterpret_cast<const float4*>(rp[g] + 4 * lane));
                            const float4 b = __ldg(reinterpret_cast<const float4*>(rp[g] + 128 + 4 * lane));
                            vals[g][0] = a.x; vals[g][1] = a.y; vals[g][2] = a.z; vals[g][3] = a.w;
                            vals[g][4] = b.x; vals[g][5] = b.y; vals[g][6] = b.z; vals[g][7] = b.w;
                        }
                    } else {
#pragma unroll
                        for (int g = 0; g < G; ++g)
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                vals[g][q] = (kof(kb, q) < K) ? __ldg(rp[g] + 32 * q + lane) : 0.f;
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int q = 0; q < 8; q += 2) add2(acc[g][q], acc[g][q + 1], vals[g][q], vals[g][q + 1]);
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int l = l0 + g;
                    const float sl = (float)ps[l];
                    float vv[8];
#pragma unroll
                    for (int q = 0; q < 8; q += 2) cand2(vv[q], vv[q + 1], sl, tk[q], tk[q + 1], acc[g][q], acc[g][q + 1]);
                    if (vec && !LEAN) {
                        *reinterpret_cast<float4*>(S.vbuf + l * K + kb + 4 * lane) = make_float4(vv[0], vv[1], vv[2], vv[3]);
                        *reinterpret_cast<float4*>(S.vbuf + l * K + kb + 128 + 4 * lane) =
                            make_float4(vv[4], vv[5], vv[6], vv[7]);
                    }
                    if (!vec) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int k = kof(kb, q);
                            if (k < K) {
                                if (!LEAN) S.vbuf[l * K + k] = vv[q];
                            } else {
                                vv[q] = __int_as_float(0x7f800000);
                            }
                        }
                    }
                    // batch minimum first; the per-candidate update only runs when the
                    // batch can change the lane's two smallest (rare after warm-up)
                    float bmin = fminf(fminf(fminf(vv[0], vv[1]), fminf(vv[2], vv[3])),
                                       fminf(fminf(vv[4], vv[5]), fminf(vv[6], vv[7])));
                    if (bmin < m2) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {   // branch-free two-smallest + first argmin
                            const float w = vv[q];
                            i1 = w < m1 ? l * K + kof(kb, q) : i1;
                            m2 = fminf(m2, fmaxf(m1, w));
                            m1 = fminf(m1, w);
                        }
                    }
                }
            };
            int l0 = 0;
            if (LEAN && DA_LEAN_G == 2) {
                for (; l0 + 2 <= live; l0 += 2) group(std::integral_constant<int, 2>{}, l0);
                if (l0 < live) group(std::integral_constant<int, 1>{}, l0);
            } else {
                for (; l0 + 4 <= live; l0 += 4) group(std::integral_constant<int, 4>{}, l0);
                switch (live - l0) {
                    case 3: group(std::integral_constant<int, 3>{}, l0); break;
                    case 2: group(std::integral_constant<int, 2>{}, l0); break;
                    case 1: group(std::integral_constant<int, 1>{}, l0); break;
                    default: break;
                }
            }
        }
        __syncwarp();
        // ---- threshold: width-th smallest of the 64 per-lane minima (valid upper
        // bound of the width-th smallest candidate when width <= 64)
        float thr;
        if (width >= total) {
            thr = __int_as_float(0x7f800000);
        } else if (width <= 64) {
            // multiway merge of the lanes' sorted pairs (m1 <= m2): each step takes the
            // warp minimum (redux.sync on order-preserving keys); the owner shifts
            float h0 = m1, h1 = m2;
            unsigned key = 0u;
            for (int step = 0; step < width; ++step) {
                const unsigned mk = fkey(h0);
                key = __reduce_min_sync(FULL, mk);
                const unsigned own = __ballot_sync(FULL, mk == key);
                const bool adv = lane == __ffs(own) - 1;
                h0 = adv ? h1 : h0;
                h1 = adv ? __int_as_float(0x7f800000) : h1;
            }
            thr = funkey(key);
        } else {
            thr = __int_as_float(0x7f800000);  // wide beams: recheck everything
        }
        const double lim = (double)thr + 2.0 * E;
        const float limf = (lim >= 3.0e38) ? __int_as_float(0x7f800000) : __fadd_ru((float)lim, fabsf((float)lim) * 1e-6f);

        // ---- queue every candidate with v' <= lim: a lane whose second smallest is
        // above lim contributes at most its smallest; the (few) other lanes are
        // rescanned by the whole warp.
        int* qcount = S.queue + 32;
        if (lane == 0) *qcount = 0;
        __syncwarp();
        const bool multi = m2 <= limf;
        if (m1 <= limf && !multi) {
            const int slot = atomicAdd(qcount, 1);
            if (slot < QCAP) S.queue[33 + slot] = i1;
        }
        unsigned flagged = __ballot_sync(FULL, multi);
        if (LEAN) {
            // lanes holding two or more candidates under the limit: the warp recomputes
            // their values (same gathers, same addition order as pass A), one item per
            // (flagged lane, beam, 256-column block)
            const int nflag = __popc(flagged);
            const int nkb256 = (K + 255) / 256;
            const int per_f = live * nkb256;
            for (int t = lane; t < nflag * per_f; t += 32) {
                const int fi = t / per_f, rem = t - fi * per_f;
                unsigned fm = flagged;
                for (int i = 0; i < fi; ++i) fm &= fm - 1;
                const int f = __ffs(fm) - 1;
                const int l = rem / nkb256, kb = (rem - l * nkb256) * 256;
                auto kf = [&](int q) -> int { return vec ? kb + (q >> 2) * 128 + 4 * f + (q & 3) : kb + 32 * q + f; };
                float acc[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = 0.f;
                for (int j = 0; j < m; ++j) {
                    const float* rp = P32 + S.roff[l * M + j];
                    if (vec) {
                        const float4 a = __ldg(reinterpret_cast<const float4*>(rp + kb + 4 * f));
                        const float4 b = __ldg(reinterpret_cast<const float4*>(rp + kb + 128 + 4 * f));
                        add2(acc[0], acc[1], a.x, a.y); add2(acc[2], acc[3], a.z, a.w);
                        add2(acc[4], acc[5], b.x, b.y); add2(acc[6], acc[7], b.z, b.w);
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[q] += (kf(q) < K) ? __ldg(rp + kf(q)) : 0.f;
                    }
                }
                const float sl = (float)ps[l];
                if (vec) {
                    const float4 ta = *reinterpret_cast<const float4*>(trow + m * K + kb + 4 * f);
                    const float4 tb = *reinterpret_cast<const float4*>(trow + m * K + kb + 128 + 4 * f);
                    const float tk8[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
                    unsigned hit = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) hit |= (unsigned)((sl + tk8[q]) + 2.f * acc[q] <= limf) << q;
                    while (hit) {
                        const int q = __ffs(hit) - 1;
                        hit &= hit - 1;
                        const int slot = atomicAdd(qcount, 1);
                        if (slot < QCAP) S.queue[33 + slot] = l * K + kf(q);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int k = kf(q);
                        if (k < K && (sl + trow[m * K + k]) + 2.f * acc[q] <= limf) {
                            const int slot = atomicAdd(qcount, 1);
                            if (slot < QCAP) S.queue[33 + slot] = l * K + k;
                        }
                    }
                }
            }
            flagged = 0;
        }
        const int per_lane = live * nkb;
        while (flagged) {
            const int f = __ffs(flagged) - 1;
            flagged &= flagged - 1;
            for (int t = lane; t < per_lane; t += 32) {
                // t enumerates (l, kb, q) of lane f's candidates
                const int l = nkb_sh >= 0 ? t >> nkb_sh : t / nkb;
                const int rem = t - l * nkb;
                const int kb = (rem >> 3) * 256, q = rem & 7;
                const int k = vec ? kb + (q >> 2) * 128 + 4 * f + (q & 3) : kb + 32 * q + f;
                if (k < K && S.vbuf[l * K + k] <= limf) {
                    const int slot = atomicAdd(qcount, 1);
                    if (slot < QCAP) S.queue[33 + slot] = l * K + k;
                }
            }
        }
        __syncwarp();
        const int nqueued = *qcount;
        __syncwarp();
        const float* cw32 = c32ok ? cw : nullptr;
        auto exact_value = [&](int flat) -> double {
            return beam_exact_value_t<true>(S.x64, cw64, cw32, D, sq, P, pc, ps, M, K, m, flat, k_sh, S.roff);
        };
        int cnt = 0;
        if (nqueued <= QCAP) {
            // exact values of the queued candidates, then exact top-width by
            // (value, flat) rank; queue entries are distinct
            double* ev = reinterpret_cast<double*>(S.vbuf);
            int* ef = reinterpret_cast<int*>(ev + QCAP);
            // exact values straight into shared memory (no per-lane arrays: they
            // would live in local memory)
            for (int b = 0; b < nqueued; b += 32) {
                const int i = b + lane;
                if (i < nqueued) {
                    const int flat = S.queue[33 + i];
                    ev[i] = exact_value(flat);
                    ef[i] = flat;
                    ++n_exact;
                }
            }
            __syncwarp();
            for (int b = 0; b < nqueued; b += 32) {
                const int i = b + lane;
                if (i < nqueued) {
                    const double mv = ev[i];
                    const int mf = ef[i];
                    int rank = 0;
#pragma unroll 4
                    for (int j = 0; j < nqueued; ++j) rank += lex_less(ev[j], ef[j], mv, mf);
                    if (rank < width) { S.lv[rank] = mv; S.lf[rank] = mf; }
                }
            }
            cnt = width;
            __syncwarp();
        } else {
            beam_overflow_select(S, total, width, S.x64, cw64, cw32, D, sq, P, pc, ps, M, K, m, k_sh, n_exact);
        }

        // ---- next beam in flat (lexicographic) order
        const int nxt = cur ^ 1;
        int32_t* nc = S.codes + nxt * cap * M;
        double* ns = S.score + nxt * cap;
        for (int b = 0; b < width; b += 32) {
            int i = b + lane;
            if (i < width) {
                const int fi = S.lf[i];
                int rank = 0;
#pragma unroll 4
                for (int j = 0; j < width; ++j) rank += (S.lf[j] < fi);
                const int parent = k_sh >= 0 ? fi >> k_sh : fi / K, kk = fi - parent * K;
#pragma unroll 4
                for (int j = 0; j < m; ++j) nc[rank * M + j] = pc[parent * M + j];
                nc[rank * M + m] = kk;
                ns[rank] = S.lv[i];
            }
        }
        __syncwarp();
        cur = nxt;
        live = width;
    }

    double bv = __longlong_as_double(0x7ff0000000000000ULL);
    int bi = 0x7fffffff;
    for (int i = lane; i < live; i += 32) {
        double s = S.score[cur * cap + i];
        if (lex_less(s, i, bv, bi)) { bv = s; bi = i; }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        double ov = __shfl_xor_sync(FULL, bv, off);
        int oi = __shfl_xor_sync(FULL, bi, off);
        if (lex_less(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    const int32_t* best = S.codes + cur * cap * M + (long long)bi * M;
#pragma unroll 1
    for (int j = lane; j < M; j += 32) {
        int c = best[j];
        if (code_bytes == 1) ((uint8_t*)codes_out)[v * ldcodes + j] = (uint8_t)c;
        else if (code_bytes == 2) ((uint16_t*)codes_out)[v * ldcodes + j] = (uint16_t)c;
        else ((int32_t*)codes_out)[v * ldcodes + j] = c;
    }
    if (stats) {
        for (int off = 16; off >= 1; off >>= 1) n_exact += __shfl_xor_sync(FULL, n_exact, off);
        if (lane == 0) atomicAdd(stats, n_exact);
    }
    if (err_out) beam_final_error(S.x64, reinterpret_cast<double*>(S.vbuf), cw, best, M, K, D, err_out + v);
}

int launch_encode_fast(const void* X, int x_f32, long long n, long long ldx, int D, const float* cw, int M, int K,
                       int L, const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                       double* err_out, unsigned long long* stats, cudaStream_t s) {
    if (n <= 0) return 0;
    long long capll = 1;
    for (int m = 0; m < M && capll < L; ++m) capll *= K;
    const int cap = (int)std::min((long long)L, capll);
    // measured on B200 (config B, 1M vectors): the value-buffer kernel wins for
    // narrow beams (L=4: 33.6 vs 36.4 ms), the lean one from L=8 up (L=10: 58.8 vs
    // 59.7, L=16: 100.9 vs 129.5).  DA_BEAM_VBUF=0/1 forces either (A/B runs).
    const char* ev = getenv("DA_BEAM_VBUF");
    const bool lean = ev ? atoi(ev) == 0 : L >= 8;
    const size_t per_warp = fast_smem_bytes(cap, M, K, D, lean);
    int warps = 8;
    while (warps > 1 && per_warp * warps > 200 * 1024) warps >>= 1;
    if (per_warp * warps > 220 * 1024) return 1;  // caller falls back to the plain encoder
    const size_t smem = per_warp * warps;
    // bound inputs + fp32 copies of the tables
    const size_t pe = (size_t)M * M * K * K;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t o_p32 = take(sizeof(float) * pe), o_sq32 = take(sizeof(float) * M * K);
    const size_t o_cmax = take(sizeof(double) * M), o_pabs = take(sizeof(double) * M * M);
    const size_t o_cbm = take(sizeof(double) * M);
    const size_t o_cw64 = take(sizeof(double) * (size_t)M * K * D);
    char* base = (char*)scratch(7, off, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "encode_fast scratch");
    float* P32 = (float*)(base + o_p32);
    float* sq32 = (float*)(base + o_sq32);
    double* cmax = (double*)(base + o_cmax);
    double* pabs = (double*)(base + o_pabs);
    double* cbm = (double*)(base + o_cbm);
    double* cw64 = (double*)(base + o_cw64);
    bound_prep_kernel<<<M * M, 256, 0, s>>>(cw, P, M, K, D, sq, P32, sq32, cmax, pabs, cw64);
    DA_CHECK_LAUNCH("bound_prep_kernel");
    cb_prep_kernel<<<1, 32, 0, s>>>(pabs, M, cbm);
    DA_CHECK_LAUNCH("cb_prep_kernel");

    if (!x_f32) return fail_arg("encode_fast: float32 input only");
    const bool vec = (K & 255) == 0;
    auto kf = lean ? (vec ? (const void*)beam_fast_kernel<float, true, true> : (const void*)beam_fast_kernel<float, true, false>)
                   : (vec ? (const void*)beam_fast_kernel<float, false, true> : (const void*)beam_fast_kernel<float, false, false>);
    if (smem > 48 * 1024) DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long row_bytes = (long long)M * K * sizeof(float);
    long long chunk = std::max(1024LL, (1LL << 30) / row_bytes);
    if (const char* e = getenv("DA_ENC_CHUNK")) chunk = std::max(256LL, atoll(e));   // A/B runs
    chunk = std::min(chunk, n);
    float* tab = (float*)scratch(8, (size_t)(chunk * row_bytes), s);
    if (!tab) return fail_cuda(cudaErrorMemoryAllocation, "encode_fast table scratch");
    const int N = M * K;
    for (long long c0 = 0; c0 < n; c0 += chunk) {
        const long long cn = std::min(chunk, n - c0);
        int tab_tc = 0;
        if (!x_f32) return fail_arg("encode_fast: float32 input only");
        if (getenv("DA_TABLE_FFMA") == nullptr) {
            ProfScope ps("encode_table_tc", s);
            // D too wide for the resident tile image: the D-tiled tcgen05 table
            // (looser bound than the chunked FFMA table) pays when the band is then
            // narrowed by the greedy kernel's warp-wide fp32 dots, i.e. at L = 1
            const char* est = getenv("DA_TABLE_STREAM");
            const int stream_ok = est ? atoi(est) != 0 : (L == 1 && K == 256);   // K == 256: the greedy kernel's shape
            const int rc = launch_table_tc((const float*)X + c0 * ldx, cn, ldx, D, cw, sq, M, K, tab, N, s, stream_ok);
            if (rc == 0) tab_tc = 1;
            else if (rc != kNotApplicable) return rc;
        }
        if (!tab_tc) {
            ProfScope ps("encode_table_sgemm", s);
            dim3 grid((N + SG_BN - 1) / SG_BN, (unsigned)((cn + SG_BM - 1) / SG_BM));
            const int ck = sgemm_chunk(D, L);
            if (ck) {
                sgemm_table_kernel<true><<<grid, SG_T, 0, s>>>((const float*)X + c0 * ldx, cn, ldx, cw, N, D, sq32,
                                                               tab, N, ck);
                tab_tc = -(ck + (D + ck - 1) / ck);   // rounding steps (table_err)
            } else {
                sgemm_table_kernel<false><<<grid, SG_T, 0, s>>>((const float*)X + c0 * ldx, cn, ldx, cw, N, D, sq32,
                                                                tab, N, 0);
            }
            DA_CHECK_LAUNCH("sgemm_table_kernel");
        }
        void* cout = (char*)codes_out + (size_t)c0 * ldcodes * code_bytes;
        double* eout = err_out ? err_out + c0 : nullptr;
        // two vectors per warp wins for narrow beams (B200, config B, 1M vectors: L=2
        // 21.5 vs 27.4 ms, L=6 32.1 vs 37.7), the one-vector lean kernel from L = 8
        // (L=8 39.0 vs 40.1, L=10 47.0 vs 54.3).  DA_BEAM_PAIR=0/1 forces it off/on.
        if (L == 1) {   // greedy: one live beam, lazily exact scores (encode_greedy.cu)
            ProfScope ps4("encode_greedy", s);
            const int rc = launch_greedy((const float*)X + c0 * ldx, cn, ldx, D, cw, M, K, tab, sq, P, P32, cmax, cbm,
                                         cw64, cout, code_bytes, ldcodes, eout, stats, tab_tc, s);
            if (rc == 0) continue;
            if (rc != kNotApplicable) return rc;
        }
        const char* epair = getenv("DA_BEAM_PAIR");
        const bool pair = epair ? atoi(epair) != 0 : L <= 7;
        if (pair) {
            ProfScope ps3("encode_beam_pair", s);
            const int rc = launch_beam_pair((const float*)X + c0 * ldx, cn, ldx, D, cw, M, K, L, cap, tab, sq, P, P32,
                                            cmax, cbm, cw64, cout, code_bytes, ldcodes, eout, stats, tab_tc, s);
            if (rc == 0) continue;
            if (rc != kNotApplicable) return rc;
        }
        ProfScope ps2("encode_beam_fast", s);
        const unsigned grid = (unsigned)((cn + warps - 1) / warps);
        auto* kfn = (void (*)(const float*, long long, long long, int, const float*, int, int, int, int, const float*,
                              const double*, const double*, const float*, const double*, const double*, const double*,
                              void*, int, long long, double*, unsigned long long*, int))kf;
        kfn<<<grid, warps * 32, smem, s>>>((const float*)X + c0 * ldx, cn, ldx, D, cw, M, K, L, cap, tab, sq, P, P32,
                                           cmax, cbm, cw64, cout, code_bytes, ldcodes, eout, stats, tab_tc);
        DA_CHECK_LAUNCH("beam_fast_kernel");
    }
    return 0;
}

}  // namespace da

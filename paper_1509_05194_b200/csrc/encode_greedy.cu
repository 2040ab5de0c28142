// Beam width 1 (greedy residual quantization, annq/codebook.py:264-300 with
// L = 1) with lazily exact scores.
//
// With one live beam every candidate of a stage shares the parent score s, so
// the fp32 filter values need no s at all: v'(k) = t'[m,k] + 2 sum_{j<m}
// P32[j,m][c_j,k] approximates w(k) = t[m,k] + 2 cross(k) within E1 (the same
// table / cross / rounding bound as the beam kernels), and the reference's
// value V(k) = (s + t) + 2 cross differs from s + w(k) by at most E2 (two float64
// roundings).  The exact winner therefore lies in the band v'(k) <= min v' +
// 2 (E1 + E2).  When the band holds a single candidate -- about 97 % of the
// stages on config B -- it is the reference's choice and nothing is computed in
// float64.  Otherwise the exact scores are brought up to date (the float64
// dots of every stage since the last exact one, one lane each, then the
// reference's sequential additions) and the band is decided by (V, k) like the
// reference's stable argsort.  Same codes as the beam kernels, bit for bit.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "beam_filter.cuh"

namespace da {

namespace {
constexpr int GR_WARPS = 8;
}

struct GreedySmem {
    double* x64;     // [D] (staged on the first exact stage)
    int32_t* codes;  // [M]
    int32_t* cand;   // [32] band candidates of one exact pass
};

__host__ __device__ inline size_t greedy_smem_bytes(int M, int D) {
    size_t b = sizeof(double) * (size_t)D;
    b += sizeof(int32_t) * ((size_t)M + 32);
    return (b + 15) & ~size_t(15);
}

// x.c in the reference's order with the row read from global memory as fp32
// (exact in float64): the wide-row path, where staging D doubles per warp would
// cost the kernel its occupancy.  Same FMA sequence as exact_dot.
__device__ __noinline__ double exact_dot_gx(const float* __restrict__ x, const float* __restrict__ c, int D, bool v4) {
    double tot = 0.0;
    bool first = true;
    int d = 0;
    while (d < D) {
        const int e = d + (int)blas_block_len(D - d);
        double acc = 0.0;
        if (v4 && (d & 3) == 0) {
            for (; d + 16 <= e; d += 16) {
                float4 xv[4], cv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xv[u] = __ldg(reinterpret_cast<const float4*>(x + d) + u);
                    cv[u] = __ldg(reinterpret_cast<const float4*>(c + d) + u);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc = __fma_rn((double)xv[u].x, (double)cv[u].x, acc);
                    acc = __fma_rn((double)xv[u].y, (double)cv[u].y, acc);
                    acc = __fma_rn((double)xv[u].z, (double)cv[u].z, acc);
                    acc = __fma_rn((double)xv[u].w, (double)cv[u].w, acc);
                }
            }
        }
        for (; d < e; ++d) acc = __fma_rn((double)x[d], (double)c[d], acc);
        tot = first ? acc : dadd(tot, acc);
        first = false;
    }
    return tot;
}

// Exact stage decision (warp-collective, rare): bring the exact score s from
// stage *sv up to stage m, then the band candidates' exact values (V, k) and
// their lexicographic minimum.  Out of line to keep the hot loop small.
__device__ __noinline__ int greedy_exact(GreedySmem S, const float* __restrict__ xr, int D, const float* __restrict__ cw32,
                                         const double* __restrict__ cw64, const double* __restrict__ sq,
                                         const double* __restrict__ P, int M, int K, int m, unsigned mask, int kb,
                                         double& s, int& sv, bool& staged, unsigned long long& n_exact) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool gx = S.x64 == nullptr;   // wide rows: no float64 staging, x read from global
    if (!staged && !gx) {
        for (int d = lane; d < D; d += 32) S.x64[d] = (double)xr[d];
        __syncwarp();
        staged = true;
    }
    const bool c32ok = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(cw32) & 15) == 0);
    const bool gx4 = c32ok && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
    // 1. exact scores of the stages decided without them: t64 of the chosen codes, one lane each
    while (sv < m) {
        const int nst = min(32, m - sv);
        double t = 0.0;
        if (lane < nst) {
            const int j = sv + lane, c = S.codes[j];
            const double xc = gx ? exact_dot_gx(xr, cw32 + ((long long)j * K + c) * D, D, gx4)
                                 : exact_dot(S.x64, cw64 + ((long long)j * K + c) * D, D,
                                             c32ok ? cw32 + ((long long)j * K + c) * D : nullptr);
            t = dsub(sq[j * K + c], dmul(2.0, xc));
        }
        n_exact += lane < nst ? 1 : 0;
        for (int i = 0; i < nst; ++i) {   // the reference's additions, in stage order
            const int j = sv + i, c = S.codes[j];
            const double tj = __shfl_sync(FULL, t, i);
            double cross = 0.0;
            for (int q = 0; q < j; ++q) cross = dadd(cross, P[(((long long)q * M + j) * K + S.codes[q]) * K + c]);
            s = dadd(dadd(s, tj), dmul(2.0, cross));
        }
        sv += nst;
    }
    // 2. the band: candidates with v' <= limf, compacted 32 at a time
    double bv = __longlong_as_double(0x7ff0000000000000ULL);
    int bk = 0x7fffffff;
    // enumerate (lane, q) pairs in k order: k = kb + (q >> 2) * 128 + 4 * lane + (q & 3)
    for (int half = 0; half < 2; ++half) {
        for (int sub = 0; sub < 4; ++sub) {
            const int q = half * 4 + sub;
            const bool hit = (mask >> q) & 1u;
            const unsigned hb = __ballot_sync(FULL, hit);
            if (!hb) continue;
            const int pos = __popc(hb & ((1u << lane) - 1u));
            if (hit) S.cand[pos] = kb + half * 128 + 4 * lane + sub;
            __syncwarp();
            const int nc = __popc(hb);
            if (lane < nc) {
                const int k = S.cand[lane];
                const double xc = gx ? exact_dot_gx(xr, cw32 + ((long long)m * K + k) * D, D, gx4)
                                     : exact_dot(S.x64, cw64 + ((long long)m * K + k) * D, D,
                                                 c32ok ? cw32 + ((long long)m * K + k) * D : nullptr);
                const double t = dsub(sq[m * K + k], dmul(2.0, xc));
                double cross = 0.0;
                for (int j = 0; j < m; ++j) cross = dadd(cross, P[(((long long)j * M + m) * K + S.codes[j]) * K + k]);
                const double V = dadd(dadd(s, t), dmul(2.0, cross));
                if (lex_less(V, k, bv, bk)) { bv = V; bk = k; }
            }
            n_exact += lane < nc ? 1 : 0;
            __syncwarp();
        }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, off);
        const int ok = __shfl_xor_sync(FULL, bk, off);
        if (lex_less(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    s = bv;   // the winner's exact value is the next stage's score
    sv = m + 1;
    return bk;
}

// Band narrowing (warp-collective, rare): the tensor-core table's bound grows
// with D (6 accumulation steps per 16 columns), so at D = 960 the band often
// holds a few candidates.  Their table entries are recomputed here as warp-wide
// fp32 dots -- lane l runs one FMA chain over the columns 4l..4l+3 of every
// 128-column block, then a 5-level shuffle tree: 4*ceil(D/128) + 5 roundings,
// the bound of table_err(-steps) -- and the band is rebuilt around the smallest
// recomputed value.  The winner of the wide band is in the narrow one (its
// recomputed value is within the new bound of its exact one); a single survivor
// is therefore the reference's choice, otherwise greedy_exact decides among the
// survivors.  Returns this lane's surviving candidates (bit q as in `hits`).
__device__ __noinline__ unsigned greedy_narrow(GreedySmem S, const float* __restrict__ xr, int D,
                                               const float* __restrict__ cw32, const double* __restrict__ sq,
                                               const double* __restrict__ cmax, const double* __restrict__ cbm, int K,
                                               int m, unsigned hits, float a0, float a1, float a2_, float a3, float a4,
                                               float a5, float a6, float a7, double xnorm, double e2) {
    const float acc[8] = {a0, a1, a2_, a3, a4, a5, a6, a7};   // by value: the caller's sums stay in registers
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float inf = __int_as_float(0x7f800000);
    const bool v4 = (D & 3) == 0 && ((reinterpret_cast<uintptr_t>(cw32) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
    // one list of all band candidates (k order within a lane, lanes in order)
    const int cnt = __popc(hits);
    int base = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(FULL, base, off);
        if (lane >= off) base += t;
    }
    const int total = __shfl_sync(FULL, base, 31);
    base -= cnt;
    if (total > 32) return hits;   // a very wide band: the exact pass takes it as it is
    __syncwarp();
    {
        unsigned h = hits;
        for (int i = 0; h; ++i, h &= h - 1) {
            const int q = __ffs(h) - 1;
            S.cand[base + i] = (q >> 2) * 128 + 4 * lane + (q & 3);
        }
    }
    __syncwarp();
#pragma unroll 1
    for (int c0 = 0; c0 < total; c0 += 4) {
        const int nb = min(4, total - c0);   // warp-uniform
        const float* cr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cr[i] = cw32 + ((long long)m * K + S.cand[min(c0 + i, total - 1)]) * D;
        float dot[4] = {0.f, 0.f, 0.f, 0.f};
        if (v4) {
#pragma unroll 2
            for (int d = 4 * lane; d < D; d += 128) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(xr + d));
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (i < nb) {
                        const float4 c = __ldg(reinterpret_cast<const float4*>(cr[i] + d));
                        dot[i] = fmaf(x.x, c.x, dot[i]);
                        dot[i] = fmaf(x.y, c.y, dot[i]);
                        dot[i] = fmaf(x.z, c.z, dot[i]);
                        dot[i] = fmaf(x.w, c.w, dot[i]);
                    }
                }
            }
        } else {
#pragma unroll 1
            for (int d0 = 4 * lane; d0 < D; d0 += 128) {
                for (int d = d0; d < min(d0 + 4, D); ++d) {
                    const float x = xr[d];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (i < nb) dot[i] = fmaf(x, cr[i][d], dot[i]);
                }
            }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dot[i] += __shfl_xor_sync(FULL, dot[i], off);
        }
        __syncwarp();   // every lane has read this batch's candidates: the slots now carry the dots
        if (lane < nb) {
            const float dsel = lane == 0 ? dot[0] : (lane == 1 ? dot[1] : (lane == 2 ? dot[2] : dot[3]));
            S.cand[c0 + lane] = __float_as_int(dsel);
        }
    }
    __syncwarp();
    float v2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v2[q] = inf;
    {
        unsigned h = hits;
        for (int i = 0; h; ++i, h &= h - 1) {
            const int q = __ffs(h) - 1;
            const int k = (q >> 2) * 128 + 4 * lane + (q & 3);
            const float t2 = fmaf(-2.f, __int_as_float(S.cand[base + i]), (float)sq[m * K + k]);
            const float val = fmaf(2.f, acc[q], t2);
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) v2[qq] = qq == q ? val : v2[qq];
        }
    }
    const double u = 5.9604644775390625e-08;  // 2^-24
    const double cb = cbm[m], cm = cmax[m];
    const int steps = 4 * ((D + 127) / 128) + 5;
    const double a2 = 2.0 * (table_err(-steps, D, u, xnorm, cm) + 2.0 * ((m + 2.0) * u * cb) +
                             4.0 * u * (cm * cm + 2.0 * xnorm * cm + 2.0 * cb));
    const double E = a2 + e2 + 1e-300;
    float lm = fminf(fminf(fminf(v2[0], v2[1]), fminf(v2[2], v2[3])), fminf(fminf(v2[4], v2[5]), fminf(v2[6], v2[7])));
    const float vmin = funkey(__reduce_min_sync(FULL, fkey(lm)));
    const double lim = (double)vmin + 2.0 * E;
    const float limf = (lim >= 3.0e38) ? inf : __fadd_ru((float)lim, fabsf((float)lim) * 1e-6f);
    unsigned keep = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) keep |= (unsigned)(((hits >> q) & 1u) && v2[q] <= limf) << q;
    return keep;
}

// One warp per vector, K == 256 (lane owns k = 4 lane + {0..3} and 128 + 4 lane + {0..3}).
#ifndef DA_GR_MINB
#define DA_GR_MINB 7   // 40 registers: 56 warps per SM hide the gathers (L=1 per 1M: 11.8 -> 9.1 ms)
#endif
template <bool WIDE>   // WIDE: band narrowing + vector norm loads + optional staging (wide rows / forced)
__global__ void __launch_bounds__(32 * GR_WARPS, DA_GR_MINB) greedy_kernel(
    const float* __restrict__ X, long long n, long long ldx, int D, const float* __restrict__ cw, int M, int K,
    const float* __restrict__ tab32, const double* __restrict__ sq, const double* __restrict__ P,
    const float* __restrict__ P32, const double* __restrict__ cmax, const double* __restrict__ cbm,
    const double* __restrict__ cw64, void* codes_out, int code_bytes, long long ldcodes, double* __restrict__ err_out,
    unsigned long long* __restrict__ stats, int tab_tc, int narrow, int stage_d) {
    extern __shared__ __align__(16) char smem_raw[];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const long long v = (long long)blockIdx.x * GR_WARPS + wid;
    if (v >= n) return;
    // stage_d = D: room for the float64 row (staged when an exact stage needs it, and for
    // the error); 0: wide rows without errors -- exact dots read x from global memory
    const int sd = WIDE ? stage_d : D;   // the narrow-row instance always stages
    char* p = smem_raw + (size_t)wid * greedy_smem_bytes(M, sd);
    GreedySmem S;
    S.x64 = (!WIDE || sd) ? (double*)p : nullptr;
    S.codes = (int32_t*)(p + sizeof(double) * sd);
    S.cand = S.codes + M;
    const float* xr = X + v * ldx;
    const float* trow = tab32 + v * (long long)M * K;
    // ||x|| (rounded up) for the bound: all of a lane's loads in flight at once
    double xx_part = 0.0;
    if (WIDE && (D & 3) == 0 && (ldx & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15) == 0)) {
#pragma unroll 4
        for (int d = 4 * lane; d < D; d += 128) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(xr + d));
            xx_part = __fma_rn((double)t.x, (double)t.x, xx_part);
            xx_part = __fma_rn((double)t.y, (double)t.y, xx_part);
            xx_part = __fma_rn((double)t.z, (double)t.z, xx_part);
            xx_part = __fma_rn((double)t.w, (double)t.w, xx_part);
        }
    } else {
#pragma unroll 1
        for (int d = lane; d < D; d += 32) {
            const double t = (double)xr[d];
            xx_part = __fma_rn(t, t, xx_part);
        }
    }
    for (int off = 16; off >= 1; off >>= 1) xx_part += __shfl_xor_sync(FULL, xx_part, off);
    const double xnorm = sqrt(xx_part) * (1.0 + 1e-12);
    const double u = 5.9604644775390625e-08;  // 2^-24
    // per-stage filter bound E1 (lane m holds stage m's), and |s| <= (||x|| + sum ||c||max)^2
    double a_stage = 0.0, csum = 0.0;
    for (int mm = lane; mm < M; mm += 32) {
        const double cb = cbm[mm], cm = cmax[mm];
        const double tmax = cm * cm + 2.0 * xnorm * cm;
        const double a = 2.0 * (table_err(tab_tc, D, u, xnorm, cm) + 2.0 * ((mm + 2.0) * u * cb) +
                                4.0 * u * (tmax + 2.0 * cb));
        if (mm == lane) a_stage = a;
        csum += cm;
    }
    for (int off = 16; off >= 1; off >>= 1) csum += __shfl_xor_sync(FULL, csum, off);
    const double sb = (xnorm + csum) * (xnorm + csum) * (1.0 + 1e-12);
    // E2: the reference's two float64 roundings of (s + t) + 2 cross, generously
    const double e2 = 4.0 * 1.1102230246251565e-16 * (sb + 2.0 * (xnorm + csum) * (xnorm + csum));
    double s = 0.0;
    int sv = 0;
    bool staged = false;
    unsigned long long n_exact = 0;

#pragma unroll 1
    for (int m = 0; m < M; ++m) {
        double a_m = __shfl_sync(FULL, a_stage, m & 31);
        if (M > 32) {
            const double cb = cbm[m], cm = cmax[m];
            a_m = 2.0 * (table_err(tab_tc, D, u, xnorm, cm) + 2.0 * ((m + 2.0) * u * cb) +
                         4.0 * u * (cm * cm + 2.0 * xnorm * cm + 2.0 * cb));
        }
        const double E = a_m + e2 + 1e-300;
        // K == 256: one column block
        const float4 ta = ld_stream_f4(trow + m * K + 4 * lane);
        const float4 tb = ld_stream_f4(trow + m * K + 128 + 4 * lane);
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (int j = 0; j < m; ++j) {
            const float* rp = P32 + (((long long)j * M + m) * K + S.codes[j]) * K;
            const float4 a = __ldg(reinterpret_cast<const float4*>(rp + 4 * lane));
            const float4 b = __ldg(reinterpret_cast<const float4*>(rp + 128 + 4 * lane));
            add2(acc[0], acc[1], a.x, a.y); add2(acc[2], acc[3], a.z, a.w);
            add2(acc[4], acc[5], b.x, b.y); add2(acc[6], acc[7], b.z, b.w);
        }
        float vv[8];
        const float tk[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) vv[q] = fmaf(2.f, acc[q], tk[q]);
        float lm = fminf(fminf(fminf(vv[0], vv[1]), fminf(vv[2], vv[3])), fminf(fminf(vv[4], vv[5]), fminf(vv[6], vv[7])));
        const float vmin = funkey(__reduce_min_sync(FULL, fkey(lm)));
        const double lim = (double)vmin + 2.0 * E;
        const float limf = (lim >= 3.0e38) ? __int_as_float(0x7f800000) : __fadd_ru((float)lim, fabsf((float)lim) * 1e-6f);
        unsigned hits = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) hits |= (unsigned)(vv[q] <= limf) << q;
        int cnt = __popc(hits);
        int first_q = __ffs(hits) - 1;
        int total = __reduce_add_sync(FULL, cnt);
        int code;
        if (WIDE && total > 1 && narrow) {   // tensor-core table at wide D: tighten the band first
            hits = greedy_narrow(S, xr, D, cw, sq, cmax, cbm, K, m, hits, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5],
                                 acc[6], acc[7], xnorm, e2);
            cnt = __popc(hits);
            first_q = __ffs(hits) - 1;
            total = __reduce_add_sync(FULL, cnt);
        }
        if (total == 1) {
            const unsigned own = __ballot_sync(FULL, cnt != 0);
            const int src = __ffs(own) - 1;
            const int q = __shfl_sync(FULL, first_q, src);
            code = (q >> 2) * 128 + 4 * src + (q & 3);
        } else {
            code = greedy_exact(S, xr, D, cw, cw64, sq, P, M, K, m, hits, 0, s, sv, staged, n_exact);
        }
        if (lane == 0) S.codes[m] = code;
        __syncwarp();
    }

    for (int j = lane; j < M; j += 32) {
        const int c = S.codes[j];
        if (code_bytes == 1) ((uint8_t*)codes_out)[v * ldcodes + j] = (uint8_t)c;
        else if (code_bytes == 2) ((uint16_t*)codes_out)[v * ldcodes + j] = (uint16_t)c;
        else ((int32_t*)codes_out)[v * ldcodes + j] = c;
    }
    if (stats) {
        for (int off = 16; off >= 1; off >>= 1) n_exact += __shfl_xor_sync(FULL, n_exact, off);
        if (lane == 0) atomicAdd(stats, n_exact);
    }
    if (err_out) {
        if (!staged) {
            for (int d = lane; d < D; d += 32) S.x64[d] = (double)xr[d];
            __syncwarp();
        }
        // exact error of the chosen code (needs D doubles of scratch: reuse x64 after reading it)
        double* dd = reinterpret_cast<double*>(S.x64);
        for (int d = lane; d < D; d += 32) {
            double r = 0.0;
            for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + S.codes[j]) * D + d]);
            const double df = dsub(S.x64[d], r);
            dd[d] = dmul(df, df);
        }
        __syncwarp();
        if (lane == 0) err_out[v] = np_pw_sum([&](long long i) { return dd[i]; }, 0, D);
    }
}

int launch_greedy(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, const float* tab,
                  const double* sq, const double* P, const float* P32, const double* cmax, const double* cbm,
                  const double* cw64, void* codes_out, int code_bytes, long long ldcodes, double* err_out,
                  unsigned long long* stats, int tab_tc, cudaStream_t s) {
    if (K != 256) return kNotApplicable;
    if (const char* e = getenv("DA_GREEDY"))
        if (atoi(e) == 0) return kNotApplicable;
    // wide rows without errors: no float64 staging (7.7 KB per warp at D = 960 would leave 24 warps per SM)
    const int stage_d = (err_out != nullptr || D <= 384) ? D : 0;
    const size_t smem = greedy_smem_bytes(M, stage_d) * GR_WARPS;
    if (smem > 200 * 1024) return kNotApplicable;

    const unsigned grid = (unsigned)((n + GR_WARPS - 1) / GR_WARPS);
    // band narrowing pays where the tensor-core bound is loose (wide D); DA_GREEDY_NARROW=0/1 forces it
    int narrow = tab_tc == 1 && D >= 256;
    if (const char* e = getenv("DA_GREEDY_NARROW")) narrow = atoi(e) != 0;
    const bool wide = narrow || stage_d == 0;
    auto kfn = wide ? greedy_kernel<true> : greedy_kernel<false>;
    if (smem > 48 * 1024) DA_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kfn<<<grid, 32 * GR_WARPS, smem, s>>>(X, n, ldx, D, cw, M, K, tab, sq, P, P32, cmax, cbm, cw64, codes_out, code_bytes,
                                          ldcodes, err_out, stats, tab_tc, narrow, stage_d);
    DA_CHECK_LAUNCH("greedy_kernel");
    return 0;
}

}  // namespace da

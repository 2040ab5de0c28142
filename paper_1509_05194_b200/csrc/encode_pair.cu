// Filtered beam encoder, two vectors per warp (the default gather filter for
// K = 256, L <= 32, D % 4 == 0).
//
// Same filter, bound and exact selection as beam_fast_kernel (encode_fast.cu;
// reference annq/codebook.py:264-300), so codes and float64 errors are
// identical.  Each half-warp owns one vector: in the gather pass every warp
// instruction advances both vectors, and in the per-stage bookkeeping (exact
// float64 rechecks, ranks, next beam, stage bound) the two vectors share one
// pass over the warp's 32 lanes, where one vector alone left half of the lanes
// idle (~15 rechecks and 10 beams per stage at L = 10).
//
// Lane mapping: h = lane / 16 selects the vector, hl = lane % 16.  In the
// gather pass a lane owns 16 of the 256 columns: k = {0, 64, 128, 192} +
// 4*hl + {0..3} (four 16-byte gathers per cross-table row).
#include <cstdlib>

#include "beam_filter.cuh"
#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int PK = 256;     // codewords per dictionary
#ifndef DA_PQCAP
#define DA_PQCAP 160
#endif
#ifndef DA_PAIR_MINB
#define DA_PAIR_MINB 2
#endif
constexpr int PQCAP = DA_PQCAP;   // per-vector recheck queue (overflow: exact streaming selection)
constexpr int PCAPMAX = 32; // beam width handled here (32 per-lane minima per vector)
}

struct PairSmem {
    double* x64;     // [D]
    double* score;   // [2][cap]
    double* lv;      // [cap]
    long long* roff; // [cap*M]
    double* ev;      // [max(PQCAP, D)] exact values; error staging at the end
    int32_t* ef;     // [PQCAP]
    int32_t* codes;  // [2][cap*M]
    int32_t* lf;     // [cap]
    int32_t* queue;  // [1 + PQCAP]: [0] = count
};

__host__ __device__ inline size_t pair_vec_bytes(int cap, int M, int D) {
    const int evn = D > PQCAP ? D : PQCAP;
    size_t b = sizeof(double) * ((size_t)D + 3 * cap + evn) + sizeof(long long) * (size_t)cap * M;
    b += sizeof(int32_t) * (PQCAP + 2 * (size_t)cap * M + cap + 1 + PQCAP);
    return (b + 15) & ~size_t(15);
}

__device__ inline PairSmem carve_pair(char* p, int cap, int M, int D) {
    PairSmem s;
    const int evn = D > PQCAP ? D : PQCAP;
    s.x64 = (double*)p; p += sizeof(double) * D;
    s.score = (double*)p; p += 2 * sizeof(double) * cap;
    s.lv = (double*)p; p += sizeof(double) * cap;
    s.roff = (long long*)p; p += sizeof(long long) * cap * M;
    s.ev = (double*)p; p += sizeof(double) * evn;
    s.ef = (int32_t*)p; p += sizeof(int32_t) * PQCAP;
    s.codes = (int32_t*)p; p += 2 * sizeof(int32_t) * cap * M;
    s.lf = (int32_t*)p; p += sizeof(int32_t) * cap;
    s.queue = (int32_t*)p;
    return s;
}

// min / max / sum within a 16-lane half (the other half runs the same steps)
__device__ __forceinline__ unsigned half_min_u32(unsigned v) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double half_max(double v) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double half_sum(double v) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double pair_exact(const PairSmem& S, const double* __restrict__ cw64,
                                             const float* __restrict__ cw, int D, const double* __restrict__ sq,
                                             const double* __restrict__ P, const int32_t* __restrict__ pc,
                                             const double* __restrict__ ps, int M, int m, int flat) {
    const int l = flat >> 8, k = flat & (PK - 1);
    const double xc = exact_dot(S.x64, cw64 + ((long long)m * PK + k) * D, D, cw + ((long long)m * PK + k) * D);
    const double t = dsub(sq[m * PK + k], dmul(2.0, xc));
    double cross = 0.0;
#pragma unroll 4
    for (int j = 0; j < m; ++j) cross = dadd(cross, P[(((long long)j * M + m) * PK + pc[l * M + j]) * PK + k]);
    return dadd(dadd(ps[l], t), dmul(2.0, cross));
}

// Rare path (one vector at a time, whole warp): more candidates under the limit
// than the queue holds -> exact streaming selection over every candidate.
__device__ __noinline__ void pair_overflow_select(PairSmem S, int total, int width, const double* __restrict__ cw64,
                                                  const float* __restrict__ cw, int D, const double* __restrict__ sq,
                                                  const double* __restrict__ P, const int32_t* __restrict__ pc,
                                                  const double* __restrict__ ps, int M, int m,
                                                  unsigned long long& n_exact) {
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
        const double val = has ? pair_exact(S, cw64, cw, D, sq, P, pc, ps, M, m, flat) : 0.0;
        n_exact += has ? 1 : 0;
        unsigned mask = __ballot_sync(FULL, has && accept(val, flat));
        while (mask) {
            const int src = __ffs(mask) - 1;
            const double cv = __shfl_sync(FULL, val, src);
            const int cf = __shfl_sync(FULL, flat, src);
            int pos = 0;
            for (int bb = 0; bb < cnt; bb += 32) {
                const int i = bb + lane;
                const bool lt = (i < cnt) && lex_less(S.lv[i], S.lf[i], cv, cf);
                pos += __popc(__ballot_sync(FULL, lt));
            }
            const int endp = min(cnt, width - 1);
            for (int bb = endp - 1; bb >= pos; bb -= 32) {
                const int i = bb - lane;
                const bool act = i >= pos;
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

__global__ void __launch_bounds__(256, DA_PAIR_MINB) beam_pair_kernel(
    const float* __restrict__ X, long long n, long long ldx, int D, const float* __restrict__ cw, int M, int L,
    int cap, const float* __restrict__ tab32, const double* __restrict__ sq, const double* __restrict__ P,
    const float* __restrict__ P32, const double* __restrict__ cmax, const double* __restrict__ cbm,
    const double* __restrict__ cw64, void* codes_out, int code_bytes, long long ldcodes, double* __restrict__ err_out,
    unsigned long long* __restrict__ stats, int tab_tc) {
    extern __shared__ __align__(16) char smem_raw[];
    const unsigned FULL = 0xffffffffu;
    const int K = PK;
    const int lane = threadIdx.x & 31, h = lane >> 4, hl = lane & 15;
    const unsigned hmask = 0xFFFFu << (16 * h);
    const int wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const long long v0 = ((long long)blockIdx.x * nwarps + wid) * 2;
    if (v0 >= n) return;
    const bool real = v0 + h < n;               // a missing second vector repeats the first (no output)
    const long long v = real ? v0 + h : v0;
    const size_t vb = pair_vec_bytes(cap, M, D);
    char* wbase = smem_raw + (size_t)wid * 2 * vb;
    const PairSmem SA = carve_pair(wbase, cap, M, D), SB = carve_pair(wbase + vb, cap, M, D);
    const PairSmem S = h ? SB : SA;             // this lane's vector
    const float* trow = tab32 + v * (long long)M * K;
    const float* xr = X + v * ldx;
    double xx_part = 0.0;
    for (int d = hl; d < D; d += 16) {
        const double t = (double)xr[d];
        S.x64[d] = t;
        xx_part = __fma_rn(t, t, xx_part);
    }
    const double xnorm = sqrt(half_sum(xx_part)) * (1.0 + 1e-12);
    if (hl == 0) S.score[0] = 0.0;
    __syncwarp();
    const double u = 5.9604644775390625e-08;  // 2^-24
    unsigned long long n_exact = 0;

    int cur = 0, live = 1;
    for (int m = 0; m < M; ++m) {
        const int total = live * K;
        const int width = min(L, total);
        const int32_t* pc = S.codes + cur * cap * M;
        const double* ps = S.score + cur * cap;
        // ---- rigorous bound of |v' - v| for this stage (as beam_fast_kernel)
        double smax = hl < live ? fabs(ps[hl]) : 0.0;
        for (int l = hl + 16; l < live; l += 16) smax = fmax(smax, fabs(ps[l]));
        smax = half_max(smax);
        const double cb = cbm[m];
        const double cm = cmax[m];
        const double tmax = cm * cm + 2.0 * xnorm * cm;
        const double e_t = table_err(tab_tc, D, u, xnorm, cm);
        const double e_cross = (m + 2.0) * u * cb;
        const double E = 2.0 * (e_t + 2.0 * e_cross + 4.0 * u * (smax + tmax + 2.0 * cb) + u * smax) + 1e-300;

        for (int e = hl; e < live * m; e += 16) {
            const int l = e / m, j = e - l * m;
            S.roff[l * M + j] = (((long long)j * M + m) * K + pc[l * M + j]) * K;
        }
        __syncwarp();
        // ---- pass A: both halves walk the same (group, level) structure; a lane
        // owns 16 columns k = {0, 64, 128, 192} + 4*hl + {0..3}
        float m1 = __int_as_float(0x7f800000), m2 = m1;
        int i1 = -1;
        {
            const int cbase = 4 * hl;
            float tk[16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                const float4 a = ld_stream_f4(trow + m * K + cbase + 64 * c4);
                tk[4 * c4] = a.x; tk[4 * c4 + 1] = a.y; tk[4 * c4 + 2] = a.z; tk[4 * c4 + 3] = a.w;
            }
            auto group = [&](auto Gc, int l0) {
                constexpr int G = decltype(Gc)::value;
                const int last = l0 + G - 1;
                // shared code prefix of the group, common to both vectors
                const bool same = hl < m && pc[l0 * M + hl] == pc[last * M + hl];
                const unsigned neq = ~__ballot_sync(FULL, same | (hl >= m));
                const unsigned nA = neq & 0xFFFFu, nB = neq >> 16;
                const int glA = nA ? min(m, __ffs(nA) - 1) : min(m, 16);
                const int glB = nB ? min(m, __ffs(nB) - 1) : min(m, 16);
                const int gl = min(glA, glB);
                float acc[G][16];
                {
                    float sh[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) sh[q] = 0.f;
                    for (int j = 0; j < gl; ++j) {
                        const float* rp = P32 + S.roff[l0 * M + j] + cbase;
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            const float4 a = __ldg(reinterpret_cast<const float4*>(rp + 64 * c4));
                            add2(sh[4 * c4], sh[4 * c4 + 1], a.x, a.y);
                            add2(sh[4 * c4 + 2], sh[4 * c4 + 3], a.z, a.w);
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int q = 0; q < 16; ++q) acc[g][q] = sh[q];
                }
                for (int j = gl; j < m; ++j) {
                    float4 va[G][4];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float* rp = P32 + S.roff[(l0 + g) * M + j] + cbase;
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) va[g][c4] = __ldg(reinterpret_cast<const float4*>(rp + 64 * c4));
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            add2(acc[g][4 * c4], acc[g][4 * c4 + 1], va[g][c4].x, va[g][c4].y);
                            add2(acc[g][4 * c4 + 2], acc[g][4 * c4 + 3], va[g][c4].z, va[g][c4].w);
                        }
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int l = l0 + g;
                    const float sl = (float)ps[l];
                    float vv[16];
#pragma unroll
                    for (int q = 0; q < 16; q += 2) cand2(vv[q], vv[q + 1], sl, tk[q], tk[q + 1], acc[g][q], acc[g][q + 1]);
                    float bmin = vv[0];
#pragma unroll
                    for (int q = 1; q < 16; ++q) bmin = fminf(bmin, vv[q]);
                    if (bmin < m2) {
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const float w = vv[q];
                            i1 = w < m1 ? l * K + cbase + (q >> 2) * 64 + (q & 3) : i1;
                            m2 = fminf(m2, fmaxf(m1, w));
                            m1 = fminf(m1, w);
                        }
                    }
                }
            };
            int l0 = 0;
            for (; l0 + 2 <= live; l0 += 2) group(std::integral_constant<int, 2>{}, l0);
            if (l0 < live) group(std::integral_constant<int, 1>{}, l0);
        }
        __syncwarp();
        // ---- threshold: width-th smallest of the half's 32 per-lane minima (distinct
        // candidates: an upper bound of the width-th smallest, width <= 32)
        float thr;
        if (width >= total) {
            thr = __int_as_float(0x7f800000);
        } else {
            float h0 = m1, h1 = m2;
            unsigned key = 0u;
            for (int step = 0; step < width; ++step) {
                const unsigned mk = fkey(h0);
                key = half_min_u32(mk);
                const unsigned own = __ballot_sync(FULL, mk == key) & hmask;
                const bool adv = lane == __ffs(own) - 1;
                h0 = adv ? h1 : h0;
                h1 = adv ? __int_as_float(0x7f800000) : h1;
            }
            thr = funkey(key);
        }
        const double lim = (double)thr + 2.0 * E;
        const float limf = (lim >= 3.0e38) ? __int_as_float(0x7f800000) : __fadd_ru((float)lim, fabsf((float)lim) * 1e-6f);

        // ---- queue every candidate with v' <= lim; lanes holding two or more are
        // recomputed by the whole warp (items over both vectors)
        int* qcount = S.queue;
        if (hl == 0) *qcount = 0;
        __syncwarp();
        const bool multi = m2 <= limf;
        if (m1 <= limf && !multi) {
            const int slot = atomicAdd(qcount, 1);
            if (slot < PQCAP) S.queue[1 + slot] = i1;
        }
        const unsigned flagged = __ballot_sync(FULL, multi);
        const float limA = __shfl_sync(FULL, limf, 0), limB = __shfl_sync(FULL, limf, 16);
        if (flagged) {
            const int per_f = live;          // one item per (flagged lane, beam)
            const int items = __popc(flagged) * per_f;
            for (int t = lane; t < items; t += 32) {
                const int fi = t / per_f, l = t - fi * per_f;
                const int f = __fns(flagged, 0, fi + 1);   // lane that owns these columns
                const int fh = f >> 4, fhl = f & 15;
                const PairSmem T = fh ? SB : SA;
                const double* tps = T.score + cur * cap;
                const long long vf = v0 + fh < n ? v0 + fh : v0;
                const float* ttrow = tab32 + vf * (long long)M * K;
                const float tlim = fh ? limB : limA;
                const int cbase = 4 * fhl;
                float acc[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] = 0.f;
                for (int j = 0; j < m; ++j) {
                    const float* rp = P32 + T.roff[l * M + j] + cbase;
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) {
                        const float4 a = __ldg(reinterpret_cast<const float4*>(rp + 64 * c4));
                        add2(acc[4 * c4], acc[4 * c4 + 1], a.x, a.y);
                        add2(acc[4 * c4 + 2], acc[4 * c4 + 3], a.z, a.w);
                    }
                }
                const float sl = (float)tps[l];
                unsigned hit = 0;
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    const float4 ta = *reinterpret_cast<const float4*>(ttrow + m * K + cbase + 64 * c4);
                    float vv[4];
                    cand2(vv[0], vv[1], sl, ta.x, ta.y, acc[4 * c4], acc[4 * c4 + 1]);
                    cand2(vv[2], vv[3], sl, ta.z, ta.w, acc[4 * c4 + 2], acc[4 * c4 + 3]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) hit |= (unsigned)(vv[q] <= tlim) << (4 * c4 + q);
                }
                while (hit) {
                    const int q = __ffs(hit) - 1;
                    hit &= hit - 1;
                    const int slot = atomicAdd(T.queue, 1);
                    if (slot < PQCAP) T.queue[1 + slot] = l * K + cbase + (q >> 2) * 64 + (q & 3);
                }
            }
        }
        __syncwarp();
        const int nqA = *SA.queue, nqB = *SB.queue;
        __syncwarp();
        const bool ovA = nqA > PQCAP, ovB = nqB > PQCAP;
        // ---- exact values of both queues in one pass over the warp's lanes
        {
            const int qa = ovA ? 0 : nqA, qb = ovB ? 0 : nqB;
            for (int i = lane; i < qa + qb; i += 32) {
                const int th = i < qa ? 0 : 1;
                const int ii = th ? i - qa : i;
                const PairSmem T = th ? SB : SA;
                const int flat = T.queue[1 + ii];
                T.ev[ii] = pair_exact(T, cw64, cw, D, sq, P, T.codes + cur * cap * M, T.score + cur * cap, M, m, flat);
                T.ef[ii] = flat;
                ++n_exact;
            }
            __syncwarp();
            // exact top-width by (value, flat) rank within each vector
            for (int i = lane; i < qa + qb; i += 32) {
                const int th = i < qa ? 0 : 1;
                const int ii = th ? i - qa : i;
                const int nq = th ? qb : qa;
                const PairSmem T = th ? SB : SA;
                const double mv = T.ev[ii];
                const int mf = T.ef[ii];
                int rank = 0;
#pragma unroll 4
                for (int j = 0; j < nq; ++j) rank += lex_less(T.ev[j], T.ef[j], mv, mf);
                if (rank < width) { T.lv[rank] = mv; T.lf[rank] = mf; }
            }
            __syncwarp();
        }
        if (ovA) pair_overflow_select(SA, total, width, cw64, cw, D, sq, P, SA.codes + cur * cap * M,
                                      SA.score + cur * cap, M, m, n_exact);
        if (ovB) pair_overflow_select(SB, total, width, cw64, cw, D, sq, P, SB.codes + cur * cap * M,
                                      SB.score + cur * cap, M, m, n_exact);

        // ---- next beam in flat (lexicographic) order
        const int nxt = cur ^ 1;
        int32_t* nc = S.codes + nxt * cap * M;
        double* ns = S.score + nxt * cap;
        for (int i = hl; i < width; i += 16) {
            const int fi = S.lf[i];
            int rank = 0;
#pragma unroll 4
            for (int j = 0; j < width; ++j) rank += (S.lf[j] < fi);
            const int parent = fi >> 8, kk = fi & (PK - 1);
#pragma unroll 4
            for (int j = 0; j < m; ++j) nc[rank * M + j] = pc[parent * M + j];
            nc[rank * M + m] = kk;
            ns[rank] = S.lv[i];
        }
        __syncwarp();
        cur = nxt;
        live = width;
    }

    double bv = __longlong_as_double(0x7ff0000000000000ULL);
    int bi = 0x7fffffff;
    for (int i = hl; i < live; i += 16) {
        const double s = S.score[cur * cap + i];
        if (lex_less(s, i, bv, bi)) { bv = s; bi = i; }
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const int oi = __shfl_xor_sync(FULL, bi, o);
        if (lex_less(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    const int32_t* best = S.codes + cur * cap * M + bi * M;
    if (real) {
        for (int j = hl; j < M; j += 16) {
            const int c = best[j];
            if (code_bytes == 1) ((uint8_t*)codes_out)[v * ldcodes + j] = (uint8_t)c;
            else if (code_bytes == 2) ((uint16_t*)codes_out)[v * ldcodes + j] = (uint16_t)c;
            else ((int32_t*)codes_out)[v * ldcodes + j] = c;
        }
    }
    if (stats) {
        for (int o = 16; o >= 1; o >>= 1) n_exact += __shfl_xor_sync(FULL, n_exact, o);
        if (lane == 0) atomicAdd(stats, n_exact);
    }
    if (err_out) {
        double* dd = S.ev;
        __syncwarp();
        for (int d = hl; d < D; d += 16) {
            double r = 0.0;
            for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + best[j]) * D + d]);
            const double df = dsub(S.x64[d], r);
            dd[d] = dmul(df, df);
        }
        __syncwarp();
        if (hl == 0 && real) err_out[v] = np_pw_sum([&](long long i) { return dd[i]; }, 0, D);
    }
}

// Beam pass over one chunk whose fp32 score table is built; kNotApplicable
// outside the specialisation (K = 256, L <= 32, D % 4 == 0, 16-byte rows).
int launch_beam_pair(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, int L, int cap,
                     const float* tab, const double* sq, const double* P, const float* P32, const double* cmax,
                     const double* cbm, const double* cw64, void* codes_out, int code_bytes, long long ldcodes,
                     double* err_out, unsigned long long* stats, int tab_tc, cudaStream_t s) {
    if (K != PK || L > PCAPMAX || (D & 3) || (reinterpret_cast<uintptr_t>(cw) & 15)) return kNotApplicable;
    const size_t per_warp = 2 * pair_vec_bytes(cap, M, D);
    int warps = 8;
    while (warps > 1 && per_warp * warps > 72 * 1024) warps >>= 1;
    if (per_warp * warps > 200 * 1024) return kNotApplicable;
    const size_t smem = per_warp * warps;
    if (smem > 48 * 1024)
        DA_CUDA(cudaFuncSetAttribute(beam_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long pairs = (n + 1) / 2;
    const unsigned grid = (unsigned)((pairs + warps - 1) / warps);
    beam_pair_kernel<<<grid, warps * 32, smem, s>>>(X, n, ldx, D, cw, M, L, cap, tab, sq, P, P32, cmax, cbm, cw64,
                                                    codes_out, code_bytes, ldcodes, err_out, stats, tab_tc);
    DA_CHECK_LAUNCH("beam_pair_kernel");
    return 0;
}

}  // namespace da

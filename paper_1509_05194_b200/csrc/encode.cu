// Beam-search encoder (multi-path encoding).
//
// Follows annq/codebook.py:255-300 (`_beam_tables`, `_beam_encode_chunk`):
//   t[m, k]  = ||c_mk||^2 - 2 x.c_mk                         (float64 table)
//   stage 0  : keep the min(L, K) smallest t[0, :] (stable: ties -> lower k)
//   stage m  : ext[l, k] = (score_l + t[m, k]) + 2 * sum_{j<m} P[j, m][code_lj, k]
//              keep the min(L, live*K) smallest by (value, flat index l*K+k),
//              re-sorted by flat index (= lexicographic code order)
//   final    : first minimum of the scores; exact error ||x - sum_m c||^2 with
//              the reconstruction added in m order and numpy pairwise row sum.
// The table is produced by the float64 dot-GEMM (gemm.cu, epilogue 2) one chunk
// of vectors at a time; this kernel runs one warp per vector with the beam state
// in shared memory and the cross tables read from L2.
#include "common.cuh"
#include "internal.h"

namespace da {


struct BeamSmem {
    int32_t* codes[2];   // [cap][M]
    double* score[2];    // [cap]
    double* lv;          // [cap] selection list values
    int32_t* lf;         // [cap] selection list flat indices
    double* diff;        // [D]
};

__host__ __device__ inline size_t beam_smem_bytes(int cap, int M, int D) {
    size_t b = 0;
    b += 2 * sizeof(int32_t) * (size_t)cap * M;
    b += 2 * sizeof(double) * (size_t)cap;
    b += sizeof(double) * (size_t)cap + sizeof(int32_t) * (size_t)cap;
    b += sizeof(double) * (size_t)D;
    return (b + 15) & ~size_t(15);
}

__device__ inline BeamSmem carve(char* p, int cap, int M, int D) {
    BeamSmem s;
    // doubles first for alignment
    s.score[0] = (double*)p; p += sizeof(double) * cap;
    s.score[1] = (double*)p; p += sizeof(double) * cap;
    s.lv = (double*)p; p += sizeof(double) * cap;
    s.diff = (double*)p; p += sizeof(double) * D;
    s.codes[0] = (int32_t*)p; p += sizeof(int32_t) * cap * M;
    s.codes[1] = (int32_t*)p; p += sizeof(int32_t) * cap * M;
    s.lf = (int32_t*)p;
    return s;
}

template <typename TX>
__global__ void beam_kernel(const TX* __restrict__ X, long long n, long long ldx, int D,
                            const float* __restrict__ cw, int M, int K, int L, int cap,
                            const double* __restrict__ tab,     // [n][M*K]
                            const double* __restrict__ P,       // [M][M][K][K]
                            void* __restrict__ codes_out, int code_bytes, long long ldcodes,
                            double* __restrict__ err_out) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const long long v = (long long)blockIdx.x * nwarps + wid;
    if (v >= n) return;
    BeamSmem S = carve(smem_raw + (size_t)wid * beam_smem_bytes(cap, M, D), cap, M, D);
    const double* trow = tab + v * (long long)M * K;
    const unsigned FULL = 0xffffffffu;

    int cur = 0;
    int live = 1;
    if (lane == 0) S.score[0][0] = 0.0;
    __syncwarp();

    for (int m = 0; m < M; ++m) {
        const long long cand_total = (long long)live * K;
        const int width = (int)min((long long)L, cand_total);
        int cnt = 0;
        const int32_t* pc = S.codes[cur];
        const double* ps = S.score[cur];
        for (int l = 0; l < live; ++l) {
            const double sl = ps[l];
            for (int k0 = 0; k0 < K; k0 += 32) {
                const int k = k0 + lane;
                double val = 0.0;
                int flat = l * K + k;
                bool valid = k < K;
                if (valid) {
                    double cross = 0.0;
                    for (int j = 0; j < m; ++j) {
                        int cj = pc[l * M + j];
                        cross = dadd(cross, P[(((long long)j * M + m) * K + cj) * K + k]);
                    }
                    val = dadd(dadd(sl, trow[(long long)m * K + k]), dmul(2.0, cross));
                }
                // threshold test against the current list
                auto accept = [&](double a, int fa) -> bool {
                    if (cnt < width) return true;
                    return lex_less(a, fa, S.lv[width - 1], S.lf[width - 1]);
                };
                unsigned mask = __ballot_sync(FULL, valid && accept(val, flat));
                while (mask) {
                    const int src = __ffs(mask) - 1;
                    const double cv = __shfl_sync(FULL, val, src);
                    const int cf = __shfl_sync(FULL, flat, src);
                    // position = number of list entries < (cv, cf)
                    int pos = 0;
                    for (int b = 0; b < cnt; b += 32) {
                        int i = b + lane;
                        bool lt = (i < cnt) && lex_less(S.lv[i], S.lf[i], cv, cf);
                        pos += __popc(__ballot_sync(FULL, lt));
                    }
                    const int end = min(cnt, width - 1);  // last index that survives the shift
                    // shift [pos, end) right by one, high to low in chunks of 32
                    for (int b = end - 1; b >= pos; b -= 32) {
                        int i = b - lane;
                        double tv = 0.0; int tf = 0;
                        bool act = i >= pos;
                        if (act) { tv = S.lv[i]; tf = S.lf[i]; }
                        __syncwarp();
                        if (act) { S.lv[i + 1] = tv; S.lf[i + 1] = tf; }
                        __syncwarp();
                    }
                    if (lane == 0) { S.lv[pos] = cv; S.lf[pos] = cf; }
                    __syncwarp();
                    cnt = min(cnt + 1, width);
                    mask &= ~(1u << src);
                    mask &= __ballot_sync(FULL, valid && accept(val, flat));
                }
            }
        }
        // re-sort the kept entries by flat index and build the next beam
        const int nxt = cur ^ 1;
        int32_t* nc = S.codes[nxt];
        double* ns = S.score[nxt];
        for (int b = 0; b < width; b += 32) {
            int i = b + lane;
            if (i < width) {
                const int fi = S.lf[i];
                int rank = 0;
                for (int j = 0; j < width; ++j) rank += (S.lf[j] < fi);
                const int parent = fi / K, kk = fi % K;
                for (int j = 0; j < m; ++j) nc[rank * M + j] = pc[parent * M + j];
                nc[rank * M + m] = kk;
                ns[rank] = S.lv[i];
            }
        }
        __syncwarp();
        cur = nxt;
        live = width;
    }

    // final pick: first minimum in code order
    double bv = __longlong_as_double(0x7ff0000000000000ULL);
    int bi = 0x7fffffff;
    for (int i = lane; i < live; i += 32) {
        double s = S.score[cur][i];
        if (lex_less(s, i, bv, bi)) { bv = s; bi = i; }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        double ov = __shfl_xor_sync(FULL, bv, off);
        int oi = __shfl_xor_sync(FULL, bi, off);
        if (lex_less(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    const int32_t* best = S.codes[cur] + (long long)bi * M;
    // codes out
    for (int j = lane; j < M; j += 32) {
        int c = best[j];
        if (code_bytes == 1) ((uint8_t*)codes_out)[v * ldcodes + j] = (uint8_t)c;
        else if (code_bytes == 2) ((uint16_t*)codes_out)[v * ldcodes + j] = (uint16_t)c;
        else ((int32_t*)codes_out)[v * ldcodes + j] = c;
    }
    if (err_out) {
        const TX* xr = X + v * ldx;
        for (int d = lane; d < D; d += 32) {
            double r = 0.0;
            for (int j = 0; j < M; ++j) r = dadd(r, (double)cw[((long long)j * K + best[j]) * D + d]);
            double df = dsub((double)xr[d], r);
            S.diff[d] = dmul(df, df);
        }
        __syncwarp();
        if (D <= 128) {
            // numpy pairwise leaf: lanes 0..7 own the 8 interleaved accumulators
            double acc = 0.0;
            const int stop = D - (D % 8);
            if (D >= 8 && lane < 8) {
                acc = S.diff[lane];
                for (int i = 8 + lane; i < stop; i += 8) acc = dadd(acc, S.diff[i]);
            }
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __shfl_sync(FULL, acc, j);
            if (lane == 0) {
                double res;
                int i;
                if (D < 8) {
                    res = 0.0;
                    i = 0;
                } else {
                    res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
                    i = stop;
                }
                for (; i < D; ++i) res = dadd(res, S.diff[i]);
                err_out[v] = res;
            }
        } else if (lane == 0) {
            const double* dd = S.diff;
            err_out[v] = np_pw_sum([&](long long i) { return dd[i]; }, 0, D);
        }
    }
}

// Host driver: X (n, D) f32/f64, cw (M, K, D) f32, sq (M*K) f64 einsum norms,
// P (M, M, K, K) f64.  Tables are built chunk by chunk in scratch slot 3.
int launch_encode(const void* X, int x_f32, long long n, long long ldx, int D, const float* cw, int M, int K,
                  int L, const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                  double* err_out, cudaStream_t s) {
    if (n <= 0) return 0;
    if (L < 1) return fail_arg("beam_width must be >= 1");
    // beam capacity never exceeds K^M
    long long capll = 1;
    for (int m = 0; m < M && capll < L; ++m) capll *= K;
    const int cap = (int)min((long long)L, capll);
    const size_t per_warp = beam_smem_bytes(cap, M, D);
    int warps = 8;
    while (warps > 1 && per_warp * warps > 200 * 1024) warps >>= 1;
    if (per_warp * warps > 220 * 1024) return fail_arg("beam state for L=%d, M=%d, D=%d exceeds shared memory", L, M, D);
    const size_t smem = per_warp * warps;
    auto kx = x_f32 ? (const void*)beam_kernel<float> : (const void*)beam_kernel<double>;
    if (smem > 48 * 1024) DA_CUDA(cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

    const long long row_bytes = (long long)M * K * sizeof(double);
    long long chunk = max(1024LL, (1LL << 30) / row_bytes);
    chunk = min(chunk, n);
    chunk = min(chunk, 65535LL * 64);
    double* tab = (double*)scratch(3, (size_t)(chunk * row_bytes), s);
    if (!tab) return fail_cuda(cudaErrorMemoryAllocation, "encode table scratch");
    for (long long c0 = 0; c0 < n; c0 += chunk) {
        const long long cn = min(chunk, n - c0);
        GemmArgs g{};
        g.A = x_f32 ? (const void*)((const float*)X + c0 * ldx) : (const void*)((const double*)X + c0 * ldx);
        g.a_f32 = x_f32; g.sai = ldx; g.sak = 1;
        g.B = cw; g.b_f32 = 1; g.sbk = 1; g.sbj = D;
        g.C = tab; g.sci = (long long)M * K; g.scj = 1;
        g.M = cn; g.N = (long long)M * K; g.K = D;
        g.nb2 = 1; g.ksplit = 1; g.kchunk = D;
        g.epi = 2; g.evec = sq;
        int rc;
        {
            ProfScope ps("encode_table_gemm", s);
            rc = launch_gemm(g, 1, s);
        }
        if (rc) return rc;
        ProfScope ps2("encode_beam_select", s);
        const unsigned grid = (unsigned)((cn + warps - 1) / warps);
        void* cout = (char*)codes_out + (size_t)c0 * ldcodes * code_bytes;
        double* eout = err_out ? err_out + c0 : nullptr;
        if (x_f32)
            beam_kernel<float><<<grid, warps * 32, smem, s>>>((const float*)X + c0 * ldx, cn, ldx, D, cw, M, K,
                                                              L, cap, tab, P, cout, code_bytes, ldcodes, eout);
        else
            beam_kernel<double><<<grid, warps * 32, smem, s>>>((const double*)X + c0 * ldx, cn, ldx, D, cw, M,
                                                               K, L, cap, tab, P, cout, code_bytes, ldcodes, eout);
        DA_CHECK_LAUNCH("beam_kernel");
    }
    return 0;
}

}  // namespace da

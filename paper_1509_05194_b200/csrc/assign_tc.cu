// Nearest-codeword assign on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same result as assign.cu (annq/clustering.py:139-148), bit for bit:
//   1. approximate dot products x.c for a 128-row x K (<= 256) tile with
//      tcgen05.mma kind::tf32, 3xTF32 split (hi*hi + hi*lo + lo*hi), fp32
//      accumulator in TMEM (256 columns);
//   2. per row (one thread per TMEM lane) a rigorous bound E on |approx - exact|
//      selects every codeword that could still be the (clipped, first-index)
//      minimum;
//   3. those candidates are recomputed in float64 exactly like the reference
//      ((||x||^2 - 2 x.c) + ||c||^2 with BLAS-ordered FMA dot, clip at 0) and the
//      lexicographic (d2, k) minimum is written.
// Operands are staged to shared memory by the CTA's threads (f64 -> tf32 hi/lo
// split) in the canonical K-major no-swizzle UMMA layout; one elected thread
// issues the MMAs and commits them to an mbarrier.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int TC_M = 128;     // rows per CTA (= TMEM lanes)
constexpr int TC_NMAX = 256;  // codewords per MMA (TMEM columns)
constexpr int TC_BK = 32;     // tf32 elements of K staged per round (4 MMA k-steps)
constexpr int TC_THREADS = 128;
constexpr int TC_CMAX = 8;    // candidates kept per row before falling back to a full exact scan
}  // namespace

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// K-major, no-swizzle canonical layout: 8x(16 B) core matrices; chunk c of
// 4 elements along K for row r lives at ((r/8)*(BK/4) + c)*128 + (r%8)*16.
__device__ __forceinline__ uint32_t kmajor_off(int r, int k) {
    return (uint32_t)((((r >> 3) * (TC_BK / 4) + (k >> 2)) << 7) + ((r & 7) << 4) + ((k & 3) << 2));
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);              // start address
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;           // LBO: next 16-B chunk along K
    d |= (uint64_t)(((TC_BK / 4) * 128 >> 4) & 0x3FFF) << 32;  // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                               // version (sm_100)
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
    return d;
}

__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N) {
    uint32_t d = 0;
    d |= 1u << 4;                   // D format F32
    d |= 2u << 7;                   // A format TF32
    d |= 2u << 10;                  // B format TF32
    // a_major = b_major = K (0), no negate
    d |= (uint32_t)(N >> 3) << 17;  // N
    d |= (uint32_t)(M >> 4) << 24;  // M
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :
        : "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <typename TX, bool BLK>
__device__ __forceinline__ double exact_xc(const TX* __restrict__ xr, const double* __restrict__ cr, int d) {
    if (!BLK) {
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc = __fma_rn((double)xr[k], cr[k], acc);
        return acc;
    }
    double tot = 0.0;
    bool first = true;
    int k = 0;
    while (k < d) {
        const int e = k + (int)blas_block_len(d - k);
        double acc = 0.0;
        for (; k < e; ++k) acc = __fma_rn((double)xr[k], cr[k], acc);
        tot = first ? acc : dadd(tot, acc);
        first = false;
    }
    return tot;
}

template <typename TX>
__global__ void __launch_bounds__(TC_THREADS) assign_tc_kernel(
    const TX* __restrict__ X, long long n, long long ldx, int d, const double* __restrict__ C, long long ldc, int K,
    const double* __restrict__ cc, int32_t* __restrict__ labels, double* __restrict__ d2_out,
    const int32_t* __restrict__ prev, unsigned long long* __restrict__ changed,
    unsigned long long* __restrict__ stats) {
    extern __shared__ __align__(1024) unsigned char smem[];
    float* a_hi = reinterpret_cast<float*>(smem);
    float* a_lo = a_hi + TC_M * TC_BK;
    float* b_hi = a_lo + TC_M * TC_BK;
    float* b_lo = b_hi + TC_NMAX * TC_BK;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double ccmax_sh;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const long long row0 = (long long)blockIdx.x * TC_M;
    const int N = (K + 7) & ~7;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(TC_NMAX));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // max codeword norm for the bound
    double cm = 0.0;
    for (int k = tid; k < K; k += TC_THREADS) cm = fmax(cm, cc[k]);
    for (int off = 16; off >= 1; off >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, off));
    __shared__ double red[4];
    if ((tid & 31) == 0) red[warp] = cm;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) ccmax_sh = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    const uint32_t tmem = tmem_base_sh;
    const uint32_t idesc = make_idesc_tf32(TC_M, N);

    uint32_t phase = 0;
    const int nchunks = (d + TC_BK - 1) / TC_BK;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int k0 = ch * TC_BK;
        if (ch > 0) {
            mbar_wait(&mbar, phase);  // previous MMAs done reading smem
            phase ^= 1;
        }
        // stage A: row tid
        {
            const long long r = row0 + tid;
            const TX* xr = X + r * ldx;
#pragma unroll 4
            for (int k = 0; k < TC_BK; ++k) {
                float h = 0.f, l = 0.f;
                const int gk = k0 + k;
                if (r < n && gk < d) {
                    const double v = (double)xr[gk];
                    h = to_tf32((float)v);
                    l = to_tf32((float)(v - (double)h));
                }
                const uint32_t o = kmajor_off(tid, k) >> 2;
                a_hi[o] = h;
                a_lo[o] = l;
            }
        }
        // stage B: codeword rows tid, tid+128
        for (int rr = tid; rr < TC_NMAX; rr += TC_THREADS) {
            const double* crow = C + (long long)rr * ldc;
#pragma unroll 4
            for (int k = 0; k < TC_BK; ++k) {
                float h = 0.f, l = 0.f;
                const int gk = k0 + k;
                if (rr < K && gk < d) {
                    const double v = crow[gk];
                    h = to_tf32((float)v);
                    l = to_tf32((float)(v - (double)h));
                }
                const uint32_t o = kmajor_off(rr, k) >> 2;
                b_hi[o] = h;
                b_lo[o] = l;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
            const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
#pragma unroll
            for (int s = 0; s < TC_BK / 8; ++s) {
                const uint32_t off = (uint32_t)s * 256;  // two 16-B chunks = 8 tf32 of K
                const uint32_t acc0 = (ch > 0 || s > 0) ? 1u : 0u;
                mma_tf32(tmem, make_desc(sa_hi + off), make_desc(sb_hi + off), idesc, acc0);
                mma_tf32(tmem, make_desc(sa_hi + off), make_desc(sb_lo + off), idesc, 1u);
                mma_tf32(tmem, make_desc(sa_lo + off), make_desc(sb_hi + off), idesc, 1u);
            }
            mma_commit(&mbar);
        }
    }
    mbar_wait(&mbar, phase);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- epilogue: thread tid owns row row0+tid (TMEM lane tid)
    const long long r = row0 + tid;
    const bool valid = r < n;
    const TX* xr = X + (valid ? r : 0) * ldx;
    double xx = 0.0;
    if (valid) xx = np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
    const double u22 = 2.384185791015625e-07;  // 2^-22
    const double sx = sqrt(xx), sc = sqrt(ccmax_sh);
    // 3xTF32 representation + fp32 accumulation error of 2 x.c, plus float64
    // rounding of the window arithmetic
    const double E = 2.0 * (4.0 * d + 16.0) * u22 * sx * sc * (1.0 + 1e-9) +
                     8.8817841970012523e-16 * (xx + ccmax_sh + 2.0 * sx * sc) + 1e-300;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    float v[32];
    // pass 1: smallest approximate (cc - 2 x.c)
    double wmin = __longlong_as_double(0x7ff0000000000000ULL);
    for (int c0 = 0; c0 < N; c0 += 32) {
        tmem_ld32(lane_addr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int k = c0 + i;
            if (k < K) wmin = fmin(wmin, cc[k] - 2.0 * (double)v[i]);
        }
    }
    const double ub = fmax(xx + wmin + E, 0.0);  // >= the exact clipped minimum
    // pass 2: candidates whose exact clipped distance can still be <= ub
    int cand[TC_CMAX];
    int nc = 0;
    bool overflow = false;
    for (int c0 = 0; c0 < N; c0 += 32) {
        tmem_ld32(lane_addr + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int k = c0 + i;
            if (k < K && fmax(xx + (cc[k] - 2.0 * (double)v[i]) - E, 0.0) <= ub) {
                if (nc < TC_CMAX) cand[nc] = k;
                ++nc;
            }
        }
    }
    overflow = nc > TC_CMAX;
    if (valid) {
        double best = __longlong_as_double(0x7ff0000000000000ULL);
        int bk = 0x7fffffff;
        const bool blk = d > (int)BLAS_Q;
        auto consider = [&](int k) {
            const double* crow = C + (long long)k * ldc;
            const double xc = blk ? exact_xc<TX, true>(xr, crow, d) : exact_xc<TX, false>(xr, crow, d);
            double dv = dadd(dsub(xx, dmul(2.0, xc)), cc[k]);
            if (dv < 0.0) dv = 0.0;
            if (lex_less(dv, k, best, bk)) { best = dv; bk = k; }
        };
        if (!overflow) {
            for (int i = 0; i < nc; ++i) consider(cand[i]);
        } else {
            for (int k = 0; k < K; ++k) consider(k);
        }
        labels[r] = bk;
        d2_out[r] = best;
        if (stats) atomicAdd(stats, (unsigned long long)(overflow ? K : nc));
        if (changed != nullptr && prev != nullptr && prev[r] != bk) atomicAdd(changed, 1ULL);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_NMAX));
    }
}

// Returns 1 (without launching) when the shape is outside the tensor-core path.
int launch_assign_tc(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C, long long ldc,
                     int K, const double* cc, int32_t* labels, double* d2, const int32_t* prev,
                     unsigned long long* changed, unsigned long long* stats, cudaStream_t s) {
    if (K > TC_NMAX || K < 1 || d < 1) return 1;
    if (n <= 0) return 0;
    const size_t smem = sizeof(float) * (2 * TC_M + 2 * TC_NMAX) * TC_BK;
    const unsigned grid = (unsigned)((n + TC_M - 1) / TC_M);
    ProfScope ps(d <= 8 ? "assign_tc_d<=8" : d <= 32 ? "assign_tc_d<=32" : d <= 128 ? "assign_tc_d<=128" : "assign_tc_d>128",
                 s);
    if (x_is_f32) {
        auto kf = assign_tc_kernel<float>;
        DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kf<<<grid, TC_THREADS, smem, s>>>((const float*)X, n, ldx, d, C, ldc, K, cc, labels, d2, prev, changed, stats);
    } else {
        auto kf = assign_tc_kernel<double>;
        DA_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kf<<<grid, TC_THREADS, smem, s>>>((const double*)X, n, ldx, d, C, ldc, K, cc, labels, d2, prev, changed,
                                          stats);
    }
    DA_CHECK_LAUNCH("assign_tc_kernel");
    return 0;
}

}  // namespace da

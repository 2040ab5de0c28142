// Beam encoder on the tensor cores (tcgen05), one CTA per group of vectors.
//
// Same contract as encode.cu / encode_fast.cu (annq/codebook.py:255-300, the
// result is bit-identical), different arithmetic for the FILTER:
//   the reference's stage score  (s_l + t[m,k]) + 2 sum_{j<m} P[j,m][c_lj,k]
//   equals                        s_l + ||c_mk||^2 - 2 r_l . c_mk
// with r_l = x - sum_{j<m} c_j(c_lj) the beam's residual.  So one GEMM per
// stage -- rows = (vector, beam) residuals, columns = the K codewords of
// dictionary m -- gives every candidate's approximate score: tcgen05.mma
// kind::tf32 with a 3xTF32 split, fp32 accumulators in TMEM (128 x 256).
// No score table and no cross-table gathers are needed for the filter.
// A rigorous bound E (residual rounding, 3xTF32 + fp32 accumulation, fp32
// score arithmetic) selects the candidates that can still make the exact
// top-width; those are recomputed in float64 exactly as the reference does
// (BLAS-ordered x.c, einsum ||c||^2, sequential cross sum) and the beam keeps
// exact float64 scores.
//
// Layout per CTA (128 threads = 128 TMEM lanes = 128 rows): V = 128 / cap
// vectors; row v*cap + l holds beam l of vector v.  Operands are extended by one
// k column so the MMA returns the whole approximate term directly:
//   A row = [ r_l , 1 ]          (tf32 hi/lo image of the fp32 residual)
//   B row = [ -2 c_mk , ||c_mk||^2 ]   (rows k >= K carry a 1e30 sentinel)
// Residual images live in a per-CTA global slab (L2-resident) already in the
// canonical no-swizzle K-major shared-memory layout, so both operands arrive by
// bulk copy (cp.async.bulk) into a 3-deep ring; one thread issues copies and MMAs.
//
// Per stage, thread = row: one pass over the 256 TMEM columns keeps, for each of
// 16 contiguous 16-column slices, the smallest and second smallest value (the
// column index is embedded in the 4 low mantissa bits, covered by the bound).
// A warp per vector selects the width-th smallest slice minimum (redux.sync),
// which bounds the vector's width-th smallest candidate from above.  Slices whose
// minimum is under the limit queue that one candidate; the rare slices whose
// second minimum is also under it are rescanned.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
#ifndef BT_BIG
#define BT_BIG 0
#endif
#ifndef BT_THREADS
#define BT_THREADS 256
#endif
constexpr int BT_ROWS = BT_BIG ? 256 : 128;   // rows (vector beams) per CTA
constexpr int BT_RB = BT_ROWS / 128;          // 128-row MMA blocks, one TMEM accumulator each
constexpr int BT_N = 256;
constexpr int BT_T = BT_THREADS;
constexpr int BT_H = BT_T / BT_ROWS;          // threads per row (1, or 2 = column halves)
constexpr int BT_CPT = 8 / BT_H;     // 32-column TMEM chunks per thread
constexpr int BT_SW = 2 * BT_CPT;    // contiguous slice width (16 slices per thread)
constexpr int BT_COLS = 256 / BT_H;  // columns per thread
constexpr int BT_BK = BT_H == 1 ? 8 : 16;   // k per ring chunk
constexpr int BT_NST = BT_RB == 2 ? 4 : 3;  // shared-memory ring depth (k-chunks in flight)

#ifndef BT_PREFETCH
#define BT_PREFETCH 1
#endif
constexpr int BT_S = 16;  // column slices per half row for the beam threshold (32 per row)
}  // namespace

__device__ __forceinline__ uint32_t bt_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float bt_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t bt_off(int r, int k) {
    return (uint32_t)((((r >> 3) * (BT_BK / 4) + (k >> 2)) << 7) + ((r & 7) << 4) + ((k & 3) << 2));
}
__device__ __forceinline__ uint64_t bt_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(((BT_BK / 4) * 128 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void bt_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool bt_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(bt_smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
// bounded spin: a lost arrival traps (with a message) instead of hanging the GPU
__device__ __forceinline__ void bt_wait(uint64_t* bar, uint32_t phase) {
    long long spins = 0;
    while (!bt_try_wait(bar, phase)) {
        if (++spins > (1ll << 26)) {
            printf("[da] beam_tc: mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
            __trap();
        }
    }
}
__device__ __forceinline__ void bt_ld32(uint32_t taddr, float* v) {
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


// exact x.c in the reference's order (FMA chain, OpenBLAS k-blocks above 384);
// both operands fp32 in memory (exact in float64)
__device__ __forceinline__ double bt_exact_dot(const float* __restrict__ x, const float* __restrict__ c, int D, bool v4) {
    double tot = 0.0;
    bool first = true;
    int d = 0;
    while (d < D) {
        const int e = d + (int)blas_block_len(D - d);
        double acc = 0.0;
        if (v4 && (d & 3) == 0) {   // a BLAS block may start off a 16-byte boundary
            for (; d + 8 <= e; d += 8) {
                const float4 x0 = __ldg(reinterpret_cast<const float4*>(x + d));
                const float4 x1 = __ldg(reinterpret_cast<const float4*>(x + d + 4));
                const float4 c0 = __ldg(reinterpret_cast<const float4*>(c + d));
                const float4 c1 = __ldg(reinterpret_cast<const float4*>(c + d + 4));
                acc = __fma_rn((double)x0.x, (double)c0.x, acc);
                acc = __fma_rn((double)x0.y, (double)c0.y, acc);
                acc = __fma_rn((double)x0.z, (double)c0.z, acc);
                acc = __fma_rn((double)x0.w, (double)c0.w, acc);
                acc = __fma_rn((double)x1.x, (double)c1.x, acc);
                acc = __fma_rn((double)x1.y, (double)c1.y, acc);
                acc = __fma_rn((double)x1.z, (double)c1.z, acc);
                acc = __fma_rn((double)x1.w, (double)c1.w, acc);
            }
        }
        for (; d < e; ++d) acc = __fma_rn((double)x[d], (double)c[d], acc);
        tot = first ? acc : dadd(tot, acc);
        first = false;
    }
    return tot;
}

// Same value for D <= 384 (one BLAS k-block) with x already in float64 (shared
// memory) and the codeword row streamed from fp32 global memory in prefetched
// 32-wide batches, so the FMA chain is not serialised behind each load.
__device__ __forceinline__ double bt_exact_dot_s(const double* __restrict__ xs, const float* __restrict__ c, int D) {
    double acc = 0.0;
    float4 cur[8], nxt[8];
    const int D32 = D & ~31;
    if (D32 > 0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = __ldg(reinterpret_cast<const float4*>(c) + u);
    }
    for (int d0 = 0; d0 < D32; d0 += 32) {
        if (d0 + 32 < D32) {
#pragma unroll
            for (int u = 0; u < 8; ++u) nxt[u] = __ldg(reinterpret_cast<const float4*>(c + d0 + 32) + u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 x01 = *reinterpret_cast<const double2*>(xs + d0 + 4 * u);
            const double2 x23 = *reinterpret_cast<const double2*>(xs + d0 + 4 * u + 2);
            acc = __fma_rn(x01.x, (double)cur[u].x, acc);
            acc = __fma_rn(x01.y, (double)cur[u].y, acc);
            acc = __fma_rn(x23.x, (double)cur[u].z, acc);
            acc = __fma_rn(x23.y, (double)cur[u].w, acc);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
    }
    for (int d = D32; d < D; ++d) acc = __fma_rn(xs[d], (double)c[d], acc);
    return acc;
}

// Codebook -> per (dictionary, k-chunk) tf32 hi/lo images of B = [-2c, ||c||^2],
// sentinel 1e30 in the norm column of the padding rows k >= K.
__global__ void cb_tf32_prep_kernel(const float* __restrict__ cw, const double* __restrict__ sq, int M, int K, int D,
                                    int nch, float* __restrict__ out) {
    const long long per = (long long)BT_N * BT_BK;
    const long long total = (long long)M * nch * per;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int mc = (int)(e / per);
        const int m = mc / nch, ch = mc % nch;
        const int rem = (int)(e % per);
        const int r = rem / BT_BK, k = rem % BT_BK;
        const int gk = ch * BT_BK + k;
        float v = 0.f;
        if (gk < D) v = r < K ? -2.f * cw[((long long)m * K + r) * D + gk] : 0.f;
        else if (gk == D) v = r < K ? (float)sq[(long long)m * K + r] : 1e30f;
        const float h = bt_tf32(v), l = bt_tf32(v - h);
        float* base = out + (size_t)mc * 2 * per;
        const uint32_t o = bt_off(r, k) >> 2;
        base[o] = h;
        base[per + o] = l;
    }
}

// x -> tf32 hi (at o) and lo = tf32(x - hi) (at o + A_EL), one 16-B core-matrix row each
__device__ __forceinline__ void bt_store_split(float* chunk, uint32_t o, const float* x4) {
    float4 h, lo;
    h.x = bt_tf32(x4[0]); lo.x = bt_tf32(x4[0] - h.x);
    h.y = bt_tf32(x4[1]); lo.y = bt_tf32(x4[1] - h.y);
    h.z = bt_tf32(x4[2]); lo.z = bt_tf32(x4[2] - h.z);
    h.w = bt_tf32(x4[3]); lo.w = bt_tf32(x4[3] - h.w);
    *reinterpret_cast<float4*>(chunk + o) = h;
    *reinterpret_cast<float4*>(chunk + BT_ROWS * BT_BK + o) = lo;
}

__device__ __forceinline__ void bt_bulk(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     bt_smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(bt_smem_u32(bar))
                 : "memory");
}

// float -> unsigned key with the same order (for redux.sync.min)
__device__ __forceinline__ unsigned bt_key(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float bt_unkey(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}


// One half row's pass over 128 TMEM columns: per slice the smallest (s1) and
// second smallest (s2) value, the slice-local position embedded in the 4 low
// mantissa bits.  CONTIG: slice = column / 8 (position = column % 8); else
// slice = column % 16 (position = column / 16).  Loads are warp-collective.
template <bool CONTIG>
__device__ __forceinline__ void bt_row_pass(uint32_t taddr_row, bool row_live, float* s1, float* s2) {
#pragma unroll
    for (int c = 0; c < BT_CPT; ++c) {
        float v[32];
        bt_ld32(taddr_row + 32 * c, v);
        if (row_live) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int sl = CONTIG ? c * (32 / BT_SW) + i / BT_SW : (i & 15);
                const uint32_t pos = CONTIG ? (uint32_t)(i % BT_SW) : (uint32_t)(2 * c + (i >> 4));
                const float w = __uint_as_float((__float_as_uint(v[i]) & ~15u) | pos);
                s2[sl] = fminf(s2[sl], fmaxf(s1[sl], w));
                s1[sl] = fminf(s1[sl], w);
            }
        }
    }
}

// phase timing (DA_DEBUG): thread 0 accumulates clock deltas between phase marks
#define BT_MARK(i)                                                   \
    do {                                                             \
        if (a.prof && tid == 0) {                                    \
            const long long _t = clock64();                          \
            prof_acc[i] += _t - prof_t;                              \
            prof_t = _t;                                             \
        }                                                            \
    } while (0)

struct BeamTcArgs {
    const float* X; long long n; long long ldx; int D;
    const float* cw; int M; int K; int L; int cap;
    const double* sq;      // (M*K) einsum norms (exact)
    const double* P;       // (M,M,K,K) cross tables (exact)
    const float* Bg;       // codeword images [M][nch][hi,lo][256*BK]
    const double* cmax;    // per dictionary: [max ||c||, max ||c||^2]
    float* img;            // residual images [grid][2][nch][hi,lo][128*BK]
    void* codes_out; int code_bytes; long long ldcodes;
    double* err_out;
    unsigned long long* stats;
    int nch;
    int qv;                // exact-recheck queue capacity per vector
    int* bad;              // [n] set to 1 when a vector overflowed its queue (host re-encodes it)
    int xs_smem;           // 1: the group's vectors are staged in shared memory as float64
    unsigned long long* prof;  // [12] per-phase clock sums (debug) or null
};

__global__ void __launch_bounds__(BT_T, (BT_H == 1 && BT_RB == 1) ? 2 : 1) beam_tc_kernel(BeamTcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int A_EL = BT_ROWS * BT_BK, B_EL = BT_N * BT_BK;
    float* Abuf = reinterpret_cast<float*>(smem);        // [NST][hi,lo][A_EL]
    float* Bbuf = Abuf + BT_NST * 2 * A_EL;               // [NST][hi,lo][B_EL]
    unsigned char* p = reinterpret_cast<unsigned char*>(Bbuf + BT_NST * 2 * B_EL);
    const int V = BT_ROWS / a.cap;
    const int M = a.M, K = a.K, D = a.D, cap = a.cap, L = a.L;
    const int QV = a.qv;
    double* score = reinterpret_cast<double*>(p); p += sizeof(double) * 2 * BT_ROWS;     // [2][rows]
    double* qval = reinterpret_cast<double*>(p); p += sizeof(double) * V * QV;          // [V][QV]
    double* vlim = reinterpret_cast<double*>(p); p += sizeof(double) * V;               // [V]
    double* xnorm = reinterpret_cast<double*>(p); p += sizeof(double) * V;              // [V]
    p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    float* slist = reinterpret_cast<float*>(p); p += sizeof(float) * BT_H * BT_S * BT_ROWS;   // [rows][H*S] slice minima
    int* rarg = reinterpret_cast<int*>(p); p += sizeof(int) * BT_ROWS;                  // (parent, k) per child
    int* qflat = reinterpret_cast<int*>(p); p += sizeof(int) * V * QV;                  // [V][QV]
    int* qcnt = reinterpret_cast<int*>(p); p += sizeof(int) * V;                        // [V]
    int* sel = reinterpret_cast<int*>(p); p += sizeof(int) * BT_ROWS;                   // selected entry per child slot
    int* vbad = reinterpret_cast<int*>(p); p += sizeof(int) * V;                       // [V] overflow flags
    float* erow = reinterpret_cast<float*>(p); p += sizeof(float) * BT_ROWS;           // per-row bound E_l
    uint8_t* codes = p; p += 2 * BT_ROWS * M;                                           // [2][rows][M] (K <= 256)
    p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    int* qoff = reinterpret_cast<int*>(p); p += sizeof(int) * (V + 1);                 // queue prefix offsets
    p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    double* xs = reinterpret_cast<double*>(p);                                          // [V][D] when xs_smem
    __shared__ uint64_t full_bar[BT_NST], empty_bar[BT_NST], acc_bar;
    __shared__ uint32_t tmem_sh;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nch = a.nch;
    float* img = a.img + (size_t)blockIdx.x * 2 * nch * 2 * A_EL;
    const double u24 = 5.9604644775390625e-08, u22 = 2.384185791015625e-07, u19 = 1.9073486328125e-06;
    const float INF = __int_as_float(0x7f800000);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BT_N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const bool xv4 = ((D & 3) == 0) && ((a.ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.cw) & 15) == 0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bt_smem_u32(&tmem_sh)),
                     "r"(BT_N * BT_RB));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < BT_NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&full_bar[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&empty_bar[i])));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&acc_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_sh;
    // TMEM: warp w reads lanes 32*(w%4)..; w / 4 selects the column half (BT_H == 2)
    // or the 128-row block's accumulator (BT_RB == 2)
    const int half = BT_H == 2 ? tid >> 7 : 0;
    const int blk = BT_RB == 2 ? tid >> 7 : 0;
    const uint32_t taddr_row = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * BT_COLS + blk * BT_N);
    double cmax_all = 0.0;
    for (int j = 0; j < M; ++j) cmax_all = fmax(cmax_all, a.cmax[2 * j]);
    const double steps = 3.0 * nch * (BT_BK / 8) + 7.0;   // fp32 accumulations per TMEM value (+ slack)
    // slices: contiguous 8-column blocks when K fills the row, else column mod 16
    const bool contig = K > 128;

    long long prof_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long prof_t = clock64();
    long long q = 0;        // k-chunks streamed (ring phases persist across groups)
    int bpre = 0;           // chunks of the coming stage whose codeword copy already started (tid 32)
    uint32_t acc_phase = 0;
    unsigned long long n_exact = 0;
    const long long ngroups = (a.n + V - 1) / V;
    for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const long long v0 = grp * V;
    // initial residual image: rows v*cap = [x, 1, 0...]; scores 0; ||x||
    for (int e = tid; e < V * nch * (BT_BK / 4); e += BT_T) {
        const int v = e / (nch * (BT_BK / 4)), rem = e % (nch * (BT_BK / 4));
        const int ch = rem / (BT_BK / 4), c4 = rem % (BT_BK / 4);
        const long long gv = v0 + v;
        const int k = ch * BT_BK + 4 * c4;
        float x4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int kk = k + u;
            x4[u] = kk < D ? (gv < a.n ? a.X[gv * a.ldx + kk] : 0.f) : (kk == D ? 1.f : 0.f);
        }
        bt_store_split(img + (size_t)ch * 2 * A_EL, bt_off(v * cap, 4 * c4) >> 2, x4);
    }
    if (tid < V) {
        const long long gv = v0 + tid;
        double s2 = 0.0;
        if (gv < a.n)
            for (int d = 0; d < D; ++d) { const double t = a.X[gv * a.ldx + d]; s2 = __fma_rn(t, t, s2); }
        xnorm[tid] = sqrt(s2) * (1.0 + 1e-12);
        vbad[tid] = 0;
    }
    for (int r = tid; r < BT_ROWS; r += BT_T) score[r] = 0.0;
    if (a.xs_smem)
        for (int e = tid; e < V * D; e += BT_T) {
            const int v = e / D, d = e % D;
            xs[e] = v0 + v < a.n ? (double)a.X[(v0 + v) * a.ldx + d] : 0.0;
        }

    int cur = 0, live = 1;
    for (int m = 0; m < M; ++m) {
        const long long tot_ll = (long long)live * K;
        const int width = (int)std::min((long long)L, tot_ll);
        // residual images written by threads (generic proxy) are read by bulk copies (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
        BT_MARK(0);
        // ---- GEMM: TMEM[row][k] = ||c_k||^2 - 2 r_row . c_k  (3xTF32, fp32 accumulate)
        // warp-specialised: thread 32 streams operand chunks into the ring (running up
        // to NST chunks ahead), thread 0 issues the MMAs as chunks land
        if (tid == 32) {
            const float* Ag = img + (size_t)cur * nch * 2 * A_EL;
            const float* Bm = a.Bg + (size_t)m * nch * 2 * B_EL;
            constexpr uint32_t bytes_a = 2 * A_EL * sizeof(float), bytes_b = 2 * B_EL * sizeof(float);
            // slot for chunk ch of a stage starting at q0: wait until its previous MMAs
            // retired, announce A+B bytes, start the codeword (B) copy
            auto issue_b = [&](long long q0, const float* Bsrc, int ch) {
                const long long qq = q0 + ch;
                const int st = (int)(qq % BT_NST);
                const long long lap = qq / BT_NST;
                if (lap >= 1) bt_wait(&empty_bar[st], (uint32_t)((lap - 1) & 1));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bt_smem_u32(&full_bar[st])),
                             "r"(bytes_a + bytes_b)
                             : "memory");
                bt_bulk(Bbuf + st * 2 * B_EL, Bsrc + (size_t)ch * 2 * B_EL, bytes_b, &full_bar[st]);
            };
            for (int ch = 0; ch < nch; ++ch) {
                if (ch >= bpre) issue_b(q, Bm, ch);   // the first chunks' B copies may already be in flight
                const int st = (int)((q + ch) % BT_NST);
                bt_bulk(Abuf + st * 2 * A_EL, Ag + (size_t)ch * 2 * A_EL, bytes_a, &full_bar[st]);
            }
            // start the next stage's first codeword copies now (they do not depend on
            // the epilogue); only when a next stage exists on this CTA
            bpre = 0;
            if (BT_PREFETCH && ((m + 1 < M) || (grp + gridDim.x < ngroups))) {
                const float* Bn = a.Bg + (size_t)((m + 1) % M) * nch * 2 * B_EL;
                const int first = BT_NST < nch ? BT_NST : nch;
                for (int ch = 0; ch < first; ++ch) issue_b(q + nch, Bn, ch);
                bpre = first;
            }
        }
        if (tid == 0) {
            for (int ch = 0; ch < nch; ++ch) {
                const long long qq = q + ch;
                const int st = (int)(qq % BT_NST);
                bt_wait(&full_bar[st], (uint32_t)((qq / BT_NST) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t ah = bt_smem_u32(Abuf + st * 2 * A_EL), al = ah + A_EL * 4;
                const uint32_t bh = bt_smem_u32(Bbuf + st * 2 * B_EL), bl = bh + B_EL * 4;
#pragma unroll
                for (int b = 0; b < BT_RB; ++b) {
                    // row block b: A rows 128b.. (contiguous in the image), accumulator columns 256b..
                    const uint32_t ab = (uint32_t)b * 128 * BT_BK * 4;
                    const uint32_t tb = tmem + (uint32_t)b * BT_N;
#pragma unroll
                    for (int s2 = 0; s2 < BT_BK / 8; ++s2) {
                        const uint32_t off = (uint32_t)s2 * 256;
                        const uint32_t acc0 = (ch > 0 || s2 > 0) ? 1u : 0u;
                        bt_mma(tb, bt_desc(ah + ab + off), bt_desc(bh + off), idesc, acc0);
                        bt_mma(tb, bt_desc(ah + ab + off), bt_desc(bl + off), idesc, 1u);
                        bt_mma(tb, bt_desc(al + ab + off), bt_desc(bh + off), idesc, 1u);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 bt_smem_u32(&empty_bar[st]))
                             : "memory");
                if (ch == nch - 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     bt_smem_u32(&acc_bar))
                                 : "memory");
            }
        }
        __syncwarp();   // warps 0/1 reconverge before the warp-collective TMEM loads
        q += nch;
        bt_wait(&acc_bar, acc_phase);
        BT_MARK(1);
        acc_phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");

        // ---- row pass: per 16-column slice the smallest / second smallest value
        // (column index in the 4 low mantissa bits), branch-free
        const int r = tid & (BT_ROWS - 1);
        const int rv = r / cap, rl = r % cap;
        const bool row_live = rv < V && rl < live && (v0 + rv) < a.n && !vbad[rv];
        const float s32 = row_live ? (float)score[cur * BT_ROWS + r] : 0.f;
        float s1[BT_S], s2v[BT_S];
#pragma unroll
        for (int i = 0; i < BT_S; ++i) { s1[i] = INF; s2v[i] = INF; }
        if (contig) bt_row_pass<true>(taddr_row, row_live, s1, s2v);
        else bt_row_pass<false>(taddr_row, row_live, s1, s2v);
        {
            // this half row's slice minima, sorted ascending (bitonic network), as one
            // list of the vector's 2*live lists: slist[(r * 2 + half) * S + i]
            float srt[BT_S];
#pragma unroll
            for (int i = 0; i < BT_S; ++i) srt[i] = row_live ? s32 + s1[i] : INF;
#pragma unroll
            for (int k2 = 2; k2 <= BT_S; k2 <<= 1) {
#pragma unroll
                for (int j = k2 >> 1; j > 0; j >>= 1) {
#pragma unroll
                    for (int i = 0; i < BT_S; ++i) {
                        const int l = i ^ j;
                        if (l > i) {
                            const float lo = fminf(srt[i], srt[l]), hi = fmaxf(srt[i], srt[l]);
                            if ((i & k2) == 0) { srt[i] = lo; srt[l] = hi; } else { srt[i] = hi; srt[l] = lo; }
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < BT_S; i += 4)
                *reinterpret_cast<float4*>(slist + (r * BT_H + half) * BT_S + i) = make_float4(srt[i], srt[i + 1], srt[i + 2], srt[i + 3]);
        }
        // rigorous |w' - v| for this row (v = the exact float64 score):
        //   3xTF32 (B rounding, lo*lo dropped): 2^-21 sum|a||b|; fp32 accumulation
        //   (steps * 2^-22 of the running sum); residual drift dlt (fp32 difference
        //   u24 + hi/lo truncation 2^-22 per stage); embedded index (16 ulp) and the
        //   fp32 score arithmetic; doubled for safety
        if (row_live && half == 0) {
            const double xx = xnorm[rv] * xnorm[rv];
            const double sl = score[cur * BT_ROWS + r];
            const double rn = sqrt(fmax(sl + xx, 0.0) * (1.0 + 1e-9)) + 1e-30;
            const double cm = a.cmax[2 * m], cm2 = a.cmax[2 * m + 1];
            const double dlt = (m + 1) * (u24 + u22) * (xnorm[rv] + m * cmax_all);
            const double mag = 2.0 * (rn + dlt) * cm + cm2;
            const double E = 2.0 * ((2.0 * u22 + steps * u22) * mag + 2.0 * dlt * cm +
                                    (u19 + 2.0 * u24) * (fabs(sl) + mag)) + 1e-30;
            erow[r] = (float)(E * (1.0 + 1e-6));
        } else if (half == 0) {
            erow[r] = 0.f;
        }
        if (tid < V) qcnt[tid] = 0;
        __syncthreads();
        BT_MARK(2);
        // ---- per vector (warp each): tau' = width-th smallest slice minimum
        for (int vv = warp; vv < V; vv += BT_T / 32) {
            if (v0 + vv >= a.n || vbad[vv]) continue;
            float thr = INF;
            const int nl = BT_H * live;    // sorted lists of the vector (BT_H per live row)
            if (width < tot_ll && nl * BT_S >= width) {
                const float* L0 = slist + (size_t)vv * cap * BT_H * BT_S;
                if (nl <= 32) {
                    // one sorted list per lane, held in registers; the winner shifts its list
                    float it[BT_S];
#pragma unroll
                    for (int i = 0; i < BT_S; i += 4) {
                        float4 t4 = make_float4(INF, INF, INF, INF);
                        if (lane < nl) t4 = *reinterpret_cast<const float4*>(L0 + lane * BT_S + i);
                        it[i] = t4.x; it[i + 1] = t4.y; it[i + 2] = t4.z; it[i + 3] = t4.w;
                    }
                    for (int step = 0; step < width; ++step) {
                        const unsigned mk = bt_key(it[0]);
                        const unsigned key = __reduce_min_sync(0xffffffffu, mk);
                        const unsigned own = __ballot_sync(0xffffffffu, mk == key);
                        const bool adv = lane == __ffs(own) - 1;
#pragma unroll
                        for (int i = 0; i < BT_S - 1; ++i) it[i] = adv ? it[i + 1] : it[i];
                        it[BT_S - 1] = adv ? INF : it[BT_S - 1];
                        if (step == width - 1) thr = bt_unkey(key);
                    }
                } else {
                    // lane j merges lists j, j+32, ...: head pointers in registers
                    int ptr[BT_ROWS * BT_H / 32];
                    float head[BT_ROWS * BT_H / 32];
#pragma unroll
                    for (int j = 0; j < BT_ROWS * BT_H / 32; ++j) {
                        ptr[j] = 0;
                        head[j] = lane + 32 * j < nl ? L0[(lane + 32 * j) * BT_S] : INF;
                    }
                    const int nj = (nl + 31) / 32;
                    for (int step = 0; step < width; ++step) {
                        float best = head[0];
#pragma unroll
                        for (int j = 1; j < BT_ROWS * BT_H / 32; ++j)
                            if (j < nj) best = fminf(best, head[j]);
                        const unsigned key = __reduce_min_sync(0xffffffffu, bt_key(best));
                        thr = bt_unkey(key);
                        const unsigned own = __ballot_sync(0xffffffffu, bt_key(best) == key);
                        bool adv = lane == __ffs(own) - 1;
#pragma unroll
                        for (int j = 0; j < BT_ROWS * BT_H / 32; ++j) {
                            const bool hit = adv && j < nj && head[j] == best;
                            adv = adv && !hit;
                            const int pj = ptr[j] + (hit ? 1 : 0);
                            const float nx = (hit && pj < BT_S) ? L0[(lane + 32 * j) * BT_S + pj] : INF;
                            ptr[j] = pj;
                            head[j] = hit ? nx : head[j];
                        }
                    }
                }
            }
            float emax = 0.f;
            for (int l = lane; l < live; l += 32) emax = fmaxf(emax, erow[vv * cap + l]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            // row l keeps candidates with w' <= tau' + E_max + E_l
            if (lane == 0) vlim[vv] = (double)thr + (double)emax;
        }
        __syncthreads();
        BT_MARK(3);
        // ---- queue: slice minima under the limit; slices with two or more rescan
        {
            const double lim = row_live ? vlim[rv] + (double)erow[r] : -1.0;
            const float limf = (lim >= 3.0e38) ? INF : __fadd_ru((float)lim, fabsf((float)lim) * 1e-6f);
            uint32_t flag = 0;
            if (row_live) {
#pragma unroll
                for (int i = 0; i < BT_S; ++i) {
                    if (s32 + s1[i] <= limf) {
                        if (s32 + s2v[i] <= limf) {
                            flag |= 1u << i;
                        } else {
                            const int e = (int)(__float_as_uint(s1[i]) & 15u);
                            const int k = BT_COLS * half + (contig ? BT_SW * i + e : 16 * e + i);
                            if (k < K) {
                                const int slot = atomicAdd(&qcnt[rv], 1);
                                if (slot < QV) qflat[rv * QV + slot] = rl * K + k;
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < BT_CPT; ++c) {
                // contiguous slices 4c..4c+3 live in chunk c; interleaved slices in every chunk < K
                const uint32_t fc = contig ? (flag >> (c * (32 / BT_SW))) & ((1u << (32 / BT_SW)) - 1u)
                                          : (BT_COLS * half + 32 * c < K ? flag : 0u);
                if (__any_sync(0xffffffffu, fc != 0)) {
                    float v[32];
                    bt_ld32(taddr_row + 32 * c, v);
                    if (fc) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int k = BT_COLS * half + 32 * c + i;
                            const uint32_t bit = contig ? (fc >> (i / BT_SW)) & 1u : (fc >> (i & 15)) & 1u;
                            if (bit && k < K && s32 + v[i] <= limf) {
                                const int slot = atomicAdd(&qcnt[rv], 1);
                                if (slot < QV) qflat[rv * QV + slot] = rl * K + k;
                            }
                        }
                    }
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        BT_MARK(4);
        // a queue that overflowed, or that holds fewer than width entries (cannot
        // happen with a valid bound; kept as a guard), sends the vector to the exact
        // path; the kept queues are compacted into one work list (thread 0)
        if (tid == 0) {
            int o = 0;
            for (int vv = 0; vv < V; ++vv) {
                qoff[vv] = o;
                if (v0 + vv >= a.n || vbad[vv]) continue;
                if (qcnt[vv] > QV || qcnt[vv] < width) {
                    vbad[vv] = 1;
                    a.bad[v0 + vv] = 1;
                    continue;
                }
                o += qcnt[vv];
            }
            qoff[V] = o;
        }
        __syncthreads();
        BT_MARK(5);
        BT_MARK(6);
        {
            const uint8_t* pcodes = codes + cur * BT_ROWS * M;
            const int total_q = qoff[V];
            for (int e = tid; e < total_q; e += BT_T) {
                int vv = 0;
                while (qoff[vv + 1] <= e) ++vv;
                const int idx = vv * QV + (e - qoff[vv]);
                const int flat = qflat[idx];
                const int l = flat / K, k = flat % K;
                const long long gv = v0 + vv;
                const uint8_t* pcv = pcodes + (vv * cap + l) * M;
                // cross-table terms first (independent loads), summed in order below
                double pc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    pc[j] = j < m ? a.P[(((long long)j * M + m) * K + pcv[j]) * K + k] : 0.0;
                const float* crow = a.cw + ((long long)m * K + k) * D;
                const double dot = a.xs_smem ? bt_exact_dot_s(xs + vv * D, crow, D)
                                             : bt_exact_dot(a.X + gv * a.ldx, crow, D, xv4);
                const double t = dsub(a.sq[m * K + k], dmul(2.0, dot));
                double cross = 0.0;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < m) cross = dadd(cross, pc[j]);
                for (int j = 8; j < m; ++j) cross = dadd(cross, a.P[(((long long)j * M + m) * K + pcv[j]) * K + k]);
                qval[idx] = dadd(dadd(score[cur * BT_ROWS + vv * cap + l], t), dmul(2.0, cross));
            }
            n_exact += (tid == 0) ? (unsigned long long)total_q : 0ULL;
        }
        __syncthreads();
        BT_MARK(7);
        // ---- exact top-width per vector by (value, flat) rank
        for (int idx = tid; idx < V * QV; idx += BT_T) {
            const int vv = idx / QV, slot = idx % QV;
            const int nq = qcnt[vv];
            if (v0 + vv >= a.n || vbad[vv] || slot >= nq) continue;
            const double x = qval[idx];
            const int f = qflat[idx];
            int rank = 0;
            for (int j = 0; j < nq; ++j) rank += lex_less(qval[vv * QV + j], qflat[vv * QV + j], x, f);
            if (rank < width) sel[vv * cap + rank] = idx;
        }
        __syncthreads();
        BT_MARK(8);
        // ---- children in flat order (thread per child row)
        {
            const int vv = r / cap, slotv = r % cap;
            const int nxt = cur ^ 1;
            if (half == 0 && vv < V && slotv < width && v0 + vv < a.n && !vbad[vv]) {
                const int idx = sel[vv * cap + slotv];
                const int f = qflat[idx];
                int pos = 0;
                for (int j = 0; j < width; ++j) pos += qflat[sel[vv * cap + j]] < f;
                const int parent = f / K, kk = f % K;
                uint8_t* cc = codes + (nxt * BT_ROWS + vv * cap + pos) * M;
                const uint8_t* pp = codes + (cur * BT_ROWS + vv * cap + parent) * M;
                for (int j = 0; j < m; ++j) cc[j] = pp[j];
                cc[m] = (uint8_t)kk;
                score[nxt * BT_ROWS + vv * cap + pos] = qval[idx];
                rarg[vv * cap + pos] = (parent << 16) | kk;
            }
        }
        __syncthreads();
        BT_MARK(9);
        // ---- child residual images r = (hi + lo)_parent - c_m(k), split again
        // (fp32; the bound covers both roundings); column D stays 1
        if (m + 1 < M) {
            const int nxt = cur ^ 1;
            const int vv = r / cap, slotv = r % cap;
            if (vv < V && slotv < width && v0 + vv < a.n && !vbad[vv]) {
                const int pk = rarg[r];
                const int parent = pk >> 16, kk = pk & 0xFFFF;
                // parent and child images are different buffers: no aliasing, so the
                // loads of later chunks may be issued ahead of earlier stores
                const float* __restrict__ src = img + (size_t)cur * nch * 2 * A_EL;
                float* __restrict__ dst = img + (size_t)nxt * nch * 2 * A_EL;
                const float* __restrict__ cwr = a.cw + ((long long)m * K + kk) * D;
                const int pr = vv * cap + parent;
                // the BT_H threads of a row split the k-chunks
#pragma unroll 2
                for (int ch = half; ch < nch; ch += BT_H) {
                    float4 hb[BT_BK / 4], lb[BT_BK / 4], cb[BT_BK / 4];
#pragma unroll
                    for (int c4 = 0; c4 < BT_BK / 4; ++c4) {
                        const int k = ch * BT_BK + 4 * c4;
                        const uint32_t po = bt_off(pr, 4 * c4) >> 2;
                        hb[c4] = *reinterpret_cast<const float4*>(src + (size_t)ch * 2 * A_EL + po);
                        lb[c4] = *reinterpret_cast<const float4*>(src + (size_t)ch * 2 * A_EL + A_EL + po);
                        if (xv4 && k + 3 < D) {
                            cb[c4] = __ldg(reinterpret_cast<const float4*>(cwr + k));
                        } else {
                            cb[c4].x = k + 0 < D ? cwr[k + 0] : 0.f;
                            cb[c4].y = k + 1 < D ? cwr[k + 1] : 0.f;
                            cb[c4].z = k + 2 < D ? cwr[k + 2] : 0.f;
                            cb[c4].w = k + 3 < D ? cwr[k + 3] : 0.f;
                        }
                    }
#pragma unroll
                    for (int c4 = 0; c4 < BT_BK / 4; ++c4) {
                        const float4 hh = hb[c4], ll = lb[c4], cc = cb[c4];
                        float x4[4] = {(hh.x + ll.x) - cc.x, (hh.y + ll.y) - cc.y, (hh.z + ll.z) - cc.z, (hh.w + ll.w) - cc.w};
                        bt_store_split(dst + (size_t)ch * 2 * A_EL, bt_off(r, 4 * c4) >> 2, x4);
                    }
                }
            }
        }
        __syncthreads();
        BT_MARK(10);
        cur ^= 1;
        live = width;
    }

    // final pick: first minimum among the beams in code order
    if (tid < V && v0 + tid < a.n && !vbad[tid]) {
        const int vv = tid;
        const long long gv = v0 + vv;
        double bv = __longlong_as_double(0x7ff0000000000000ULL);
        int bi = 0;
        for (int l = 0; l < live; ++l) {
            const double sc = score[cur * BT_ROWS + vv * cap + l];
            if (sc < bv) { bv = sc; bi = l; }
        }
        const uint8_t* best = codes + (cur * BT_ROWS + vv * cap + bi) * M;
        for (int j = 0; j < M; ++j) {
            const int c = best[j];
            if (a.code_bytes == 1) ((uint8_t*)a.codes_out)[gv * a.ldcodes + j] = (uint8_t)c;
            else if (a.code_bytes == 2) ((uint16_t*)a.codes_out)[gv * a.ldcodes + j] = (uint16_t)c;
            else ((int32_t*)a.codes_out)[gv * a.ldcodes + j] = c;
        }
        if (a.err_out) {
            const float* xr = a.X + gv * a.ldx;
            a.err_out[gv] = np_pw_sum(
                [&](long long d) {
                    double rr = 0.0;
                    for (int j = 0; j < M; ++j) rr = dadd(rr, (double)a.cw[((long long)j * K + best[j]) * D + d]);
                    const double df = dsub((double)xr[d], rr);
                    return dmul(df, df);
                },
                0, D);
        }
    }
    __syncthreads();
    }  // groups
    if (a.stats && tid == 0) atomicAdd(a.stats, n_exact);
    if (a.prof && tid == 0)
        for (int i = 0; i < 12; ++i) atomicAdd(a.prof + i, (unsigned long long)prof_acc[i]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BT_N * BT_RB));
    }
}

// per dictionary: max ||c|| and max ||c||^2 (from the exact einsum norms)
__global__ void tc_side_prep_kernel(const double* __restrict__ sq, int M, int K, double* __restrict__ cmax) {
    __shared__ double red[256];
    for (int m = 0; m < M; ++m) {
        double c = 0.0;
        for (int k = threadIdx.x; k < K; k += blockDim.x) c = fmax(c, sq[m * K + k]);
        red[threadIdx.x] = c;
        __syncthreads();
        for (int s2 = blockDim.x / 2; s2 > 0; s2 >>= 1) {
            if (threadIdx.x < s2) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s2]);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            cmax[2 * m] = sqrt(red[0]) * (1.0 + 1e-12);
            cmax[2 * m + 1] = red[0] * (1.0 + 1e-12);
        }
        __syncthreads();
    }
}

__global__ void gather_f32_rows_kernel(const float* __restrict__ X, long long ldx, int D, const int* __restrict__ idx,
                                       int cnt, float* __restrict__ out) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)cnt * D;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = X[(long long)idx[e / D] * ldx + e % D];
}

__global__ void scatter_codes_kernel(const void* __restrict__ src, int code_bytes, int M, const int* __restrict__ idx,
                                     int cnt, const double* __restrict__ esrc, void* __restrict__ dst, long long ldc,
                                     double* __restrict__ edst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const long long r = idx[i];
    for (int j = 0; j < M; ++j) {
        if (code_bytes == 1) ((uint8_t*)dst)[r * ldc + j] = ((const uint8_t*)src)[(long long)i * M + j];
        else if (code_bytes == 2) ((uint16_t*)dst)[r * ldc + j] = ((const uint16_t*)src)[(long long)i * M + j];
        else ((int32_t*)dst)[r * ldc + j] = ((const int32_t*)src)[(long long)i * M + j];
    }
    if (edst) edst[r] = esrc[i];
}

__global__ void list_bad_kernel(const int* __restrict__ bad, long long n, int* __restrict__ idx, int* __restrict__ cnt) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (bad[i]) idx[atomicAdd(cnt, 1)] = (int)i;
}

// Returns kNotApplicable (without launching) when the shape is outside the
// tensor-core encoder; CUDA failures are returned as their (positive) status.
int launch_encode_tc(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, int L,
                     const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                     double* err_out, unsigned long long* stats, cudaStream_t s) {
    if (K > BT_N || K < 1) return kNotApplicable;
    long long capll = 1;
    for (int m = 0; m < M && capll < L; ++m) capll *= K;
    const int cap = (int)std::min((long long)L, capll);
    if (cap > BT_ROWS || n <= 0) return n <= 0 ? 0 : kNotApplicable;
    const int V = BT_ROWS / cap;
    const int nch = (D + 1 + BT_BK - 1) / BT_BK;   // + the norm column
    // a single first-stage row cannot cover beams wider than 16: then all K go to the exact pass
    const int qv = cap > BT_H * BT_S ? std::max(3 * cap + 8, K) : 3 * cap + 8;
    size_t smem = sizeof(float) * (BT_NST * 2 * BT_ROWS * BT_BK + BT_NST * 2 * BT_N * BT_BK);
    smem += sizeof(double) * (2 * BT_ROWS + (size_t)V * qv + 2 * V);
    smem += 16 + sizeof(float) * BT_H * (size_t)BT_S * BT_ROWS + sizeof(int) * BT_ROWS + 2 * BT_ROWS * (size_t)M;
    smem += sizeof(int) * ((size_t)V * qv + V + BT_ROWS) + sizeof(int) * V +
            sizeof(float) * BT_ROWS;
    smem += 32 + sizeof(int) * (V + 1);   // alignment + qoff
    // stage the vectors as float64 when D fits one BLAS k-block and two CTAs still fit per SM
    int xs_smem = 0;
    const size_t xs_bytes = sizeof(double) * (size_t)V * D;
    if (D <= 384 && smem + xs_bytes <= 200 * 1024) { xs_smem = 1; smem += xs_bytes; }
    if (smem > 227 * 1024) return kNotApplicable;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long ngroups = (n + V - 1) / V;
    // two CTAs per SM when the shared-memory image allows it (TMEM: 2 x 256 columns):
    // one CTA's epilogue overlaps the other's MMAs
    DA_CUDA(cudaFuncSetAttribute(beam_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DA_CUDA(cudaFuncSetAttribute(beam_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 1, smem_sm = 0;
    cudaFuncAttributes fa{};
    DA_CUDA(cudaFuncGetAttributes(&fa, beam_tc_kernel));
    DA_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    const int regs_cta = ((fa.numRegs + 7) & ~7) * BT_T;
    if (2 * (smem + fa.sharedSizeBytes + 1024) <= (size_t)smem_sm && 2 * regs_cta <= 65536) per_sm = 2;
    const int grid = (int)std::min<long long>(ngroups, (long long)sms * per_sm);
    // scratch
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t o_bg = take(sizeof(float) * (size_t)M * nch * 2 * BT_N * BT_BK);
    const size_t o_cmax = take(sizeof(double) * 2 * M);
    const size_t o_rb = take(sizeof(float) * (size_t)grid * 2 * nch * 2 * BT_ROWS * BT_BK);
    const size_t o_bad = take(sizeof(int) * (size_t)n);
    const size_t o_lst = take(sizeof(int) * (size_t)n);
    const size_t o_cnt = take(sizeof(int) * 4);
    char* base = (char*)scratch(10, off, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "encode_tc scratch");
    float* Bg = (float*)(base + o_bg);
    double* cmax = (double*)(base + o_cmax);
    int* bad = (int*)(base + o_bad);
    int* cnt = (int*)(base + o_cnt);
    {
        ProfScope ps0("encode_tc_prep", s);
        cb_tf32_prep_kernel<<<grid_for((long long)M * nch * BT_N * BT_BK, 256, 4096), 256, 0, s>>>(cw, sq, M, K, D, nch, Bg);
        DA_CHECK_LAUNCH("cb_tf32_prep_kernel");
        tc_side_prep_kernel<<<1, 256, 0, s>>>(sq, M, K, cmax);
        DA_CHECK_LAUNCH("tc_side_prep_kernel");
        DA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int) * (size_t)n + 16, s));
    }
    BeamTcArgs a{};
    a.X = X; a.n = n; a.ldx = ldx; a.D = D; a.cw = cw; a.M = M; a.K = K; a.L = L; a.cap = cap;
    a.sq = sq; a.P = P; a.Bg = Bg; a.cmax = cmax; a.img = (float*)(base + o_rb);
    a.codes_out = codes_out; a.code_bytes = code_bytes; a.ldcodes = ldcodes; a.err_out = err_out; a.stats = stats;
    a.nch = nch; a.qv = qv; a.bad = bad; a.xs_smem = xs_smem;
    unsigned long long* dprof = nullptr;
    const bool dbg = getenv("DA_DEBUG") != nullptr;
    if (dbg) {
        DA_CUDA(cudaMallocAsync((void**)&dprof, sizeof(unsigned long long) * 12, s));
        DA_CUDA(cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * 12, s));
        a.prof = dprof;
    }
    {
        ProfScope ps1("encode_beam_tc", s);
        beam_tc_kernel<<<grid, BT_T, smem, s>>>(a);
        DA_CHECK_LAUNCH("beam_tc_kernel");
    }
    // vectors that overflowed their recheck queue (many near-ties) are re-encoded exactly
    int* lst = (int*)(base + o_lst);
    DA_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    list_bad_kernel<<<grid_for(n, 256, 4096), 256, 0, s>>>(bad, n, lst, cnt);
    DA_CHECK_LAUNCH("list_bad_kernel");
    int h_cnt = 0;
    DA_CUDA(cudaMemcpyAsync(&h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    DA_CUDA(cudaStreamSynchronize(s));
    if (dbg) {
        fprintf(stderr, "[da] encode_tc: n=%lld V=%d cap=%d grid=%d per_sm=%d smem=%zu overflowed=%d\n", n, V, cap, grid, per_sm, smem, h_cnt);
        unsigned long long hp[12];
        DA_CUDA(cudaMemcpy(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost));
        unsigned long long tot = 0;
        for (int i = 0; i < 11; ++i) tot += hp[i];
        const char* names[11] = {"init/sync", "gemm", "rowpass", "select", "queue", "ovf", "qoff", "recheck", "rank", "child", "update"};
        fprintf(stderr, "[da] encode_tc phases (%% of CTA clocks):");
        for (int i = 0; i < 11; ++i) fprintf(stderr, " %s %.1f", names[i], tot ? 100.0 * hp[i] / tot : 0.0);
        fprintf(stderr, "\n");
        cudaFree(dprof);
    }
    if (h_cnt > 0) {
        float* xg = nullptr;
        void* cg = nullptr;
        double* eg = nullptr;
        int* lcopy = nullptr;
        DA_CUDA(cudaMallocAsync((void**)&xg, sizeof(float) * (size_t)h_cnt * D, s));
        DA_CUDA(cudaMallocAsync(&cg, (size_t)code_bytes * h_cnt * M, s));
        DA_CUDA(cudaMallocAsync((void**)&eg, sizeof(double) * (size_t)h_cnt, s));
        DA_CUDA(cudaMallocAsync((void**)&lcopy, sizeof(int) * (size_t)h_cnt, s));
        DA_CUDA(cudaMemcpyAsync(lcopy, lst, sizeof(int) * (size_t)h_cnt, cudaMemcpyDeviceToDevice, s));
        gather_f32_rows_kernel<<<grid_for((long long)h_cnt * D, 256, 4096), 256, 0, s>>>(X, ldx, D, lcopy, h_cnt, xg);
        DA_CHECK_LAUNCH("gather_f32_rows_kernel");
        int rc = launch_encode_fast(xg, 1, h_cnt, D, D, cw, M, K, L, sq, P, cg, code_bytes, M, eg, stats, s);
        if (rc > 0) rc = launch_encode(xg, 1, h_cnt, D, D, cw, M, K, L, sq, P, cg, code_bytes, M, eg, s);
        if (rc) return rc;
        scatter_codes_kernel<<<grid_for(h_cnt, 128), 128, 0, s>>>(cg, code_bytes, M, lcopy, h_cnt, eg, codes_out, ldcodes,
                                                                  err_out);
        DA_CHECK_LAUNCH("scatter_codes_kernel");
        cudaFreeAsync(xg, s);
        cudaFreeAsync(cg, s);
        cudaFreeAsync(eg, s);
        cudaFreeAsync(lcopy, s);
    }
    return 0;
}

}  // namespace da

namespace da {

// ---------------------------------------------------------------------------
// Score table on the tensor cores: T[v][m*K + k] = ||c_mk||^2 - 2 x_v . c_mk (fp32,
// 3xTF32 on tcgen05, or two MMAs per k step for tf32-exact rows; the gather
// filter's input, encode_fast.cu / encode_greedy.cu / encode_pair.cu).
//
// Both operands stream: a pre-pass writes the [x, 1, 0..] rows of every 128-row
// tile as tf32 hi/lo images in the canonical K-major layout, one 16-KB block per
// (tile, 16-wide k chunk), and flags rows that are not tf32-exact; the table
// kernel then moves (row chunk, codeword chunk) pairs through a shared-memory
// ring by bulk copy -- nothing is staged by threads -- and accumulates over all
// chunks in TMEM.  Warp roles: warp 8 loads, warp 9 issues the MMAs (so a slot
// refill never delays the next chunk's MMAs), warps 0-7 drain accumulators into
// the table through a swizzled transpose (full 128-byte row segments).  A work
// item is (row tile, group of dictionaries); the `msplit` items of a tile run on
// neighbouring CTAs at the same time, so the tile's image is read from HBM about
// once and from L2 after that (148 whole-tile images would not fit L2 at D = 960).
// Round 2 replaced two resident-image kernels (whole tile image in shared memory,
// 2-slot codeword ring, tensor pipe 28 % busy) with this one at every D.
__global__ void a_tf32_img_kernel(const float* __restrict__ X, long long n, long long ldx, int D, int nch,
                                  long long ntiles, float* __restrict__ out, int* __restrict__ inexact) {
    // *inexact (optional) is set when some x differs from its tf32 rounding (a nonzero lo
    // part): the two-MMA table kernel then leaves the call to the three-MMA one
    bool bad = false;
    constexpr int A_EL = BT_ROWS * BT_BK;
    const bool v4 = (D & 3) == 0 && (ldx & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const long long total = ntiles * nch * (long long)(BT_ROWS * (BT_BK / 4));
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        // (tile, chunk, 8-row group, 4-wide k group, row in group): a warp writes 512
        // contiguous bytes of each image and reads 64-byte row segments
        const int r7 = (int)(e & 7), c4 = (int)((e >> 3) & (BT_BK / 4 - 1));
        const long long rest = e / (8 * (BT_BK / 4));
        const int r8 = (int)(rest % (BT_ROWS / 8));
        const long long tc = rest / (BT_ROWS / 8);
        const int ch = (int)(tc % nch);
        const long long tile = tc / nch;
        const int rr = r8 * 8 + r7;
        const long long gr = tile * BT_ROWS + rr;
        const int k = ch * BT_BK + 4 * c4;
        float x4[4];
        if (v4 && k + 3 < D) {
            const float4 t = gr < n ? __ldg(reinterpret_cast<const float4*>(X + gr * ldx + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
            x4[0] = t.x; x4[1] = t.y; x4[2] = t.z; x4[3] = t.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kk = k + u;
                x4[u] = kk < D ? (gr < n ? X[gr * ldx + kk] : 0.f) : (kk == D ? 1.f : 0.f);
            }
        }
        bt_store_split(out + (size_t)tc * 2 * A_EL, bt_off(rr, 4 * c4) >> 2, x4);
        bad |= (bt_tf32(x4[0]) != x4[0]) | (bt_tf32(x4[1]) != x4[1]) | (bt_tf32(x4[2]) != x4[2]) |
               (bt_tf32(x4[3]) != x4[3]);
    }
    if (inexact != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 &&
        *reinterpret_cast<volatile int*>(inexact) == 0)
        atomicOr(inexact, 1);
}

constexpr int TS_EPI = 256;            // epilogue threads (warps 0-7)
constexpr int TS_T = TS_EPI + 64;      // + loader warp + MMA warp
constexpr int TS_NS = 4;               // ring slots of one (A chunk, B chunk) pair: 48 KB each (40 KB when EXACT)
// EXACT: tf32-exact rows (integer data such as configs B/D/E): x_lo = 0, so the slots carry
// only the hi image and a k step is two MMAs (x.c_hi + x.c_lo) instead of three.  *flag is the
// image kernel's inexactness flag: each instance runs only when the rows are its kind.
// CL = 2: launched as clusters of two CTAs that work on two row tiles with the same dictionary
// group in lockstep.  Each CTA fetches half of every codeword chunk and multicasts it into both
// CTAs' rings (the chunk crosses L2 -> SM once per pair); a slot is refilled only after both
// CTAs' MMAs on it retire (multicast commit onto both `empty` barriers, count 2).
// Q = threads per row in the epilogue (2 or 4: 8 or 16 epilogue warps; 16 measured no faster).
__device__ __forceinline__ void bt_bulk_mc(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
            bt_smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(bt_smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void bt_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool EXACT, int CL, int Q>
__global__ void __launch_bounds__(128 * Q + 64, 1) table_tc_stream_kernel(const float* __restrict__ Ag, long long n, int M,
                                                                        int K, int nch, const float* __restrict__ Bg,
                                                                        float* __restrict__ T, long long ldt, int msplit,
                                                                        const int* __restrict__ flag) {
    if (flag != nullptr && (*flag != 0) == EXACT) return;   // uniform over the grid (and over a cluster)
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int A_EL = BT_ROWS * BT_BK, B_EL = BT_N * BT_BK;
    constexpr int A_PART = EXACT ? A_EL : 2 * A_EL;            // floats of the row image per slot
    constexpr int SLOT = A_PART + 2 * B_EL;                    // floats per ring slot: A hi (, A lo), B hi, B lo
    constexpr int TS_EPI = 128 * Q;                            // epilogue threads (shadows the 8-warp constant)
    constexpr int QC = BT_N / Q;                               // table columns per epilogue thread
    float* ring = reinterpret_cast<float*>(smem);
    float* Xpose = ring + (size_t)TS_NS * SLOT;                 // [4 Q warps][32 x 32] store transpose
    __shared__ uint64_t full_bar[TS_NS], empty_bar[TS_NS], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_sh;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bt_smem_u32(&tmem_sh)),
                     "r"(2 * BT_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < TS_NS; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&full_bar[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bt_smem_u32(&empty_bar[i])), "r"(CL));
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&acc_full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bt_smem_u32(&acc_empty[i])), "r"(TS_EPI));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CL > 1) bt_cluster_sync();   // the peer's barriers exist before anything is multicast at them
    const uint32_t tmem = tmem_sh;
    const long long ntiles = (n + BT_ROWS - 1) / BT_ROWS;
    const int mper = (M + msplit - 1) / msplit;               // dictionaries per item
    // work items: (row tile, dictionary group); a cluster takes CL consecutive tiles of one group
    uint32_t crank = 0;
    if (CL > 1) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const long long unit = blockIdx.x / CL, nunits = gridDim.x / CL;
    const long long nitems = ((ntiles + CL - 1) / CL) * msplit;
    long long my_items = 0;
    for (long long t = unit; t < nitems; t += nunits) ++my_items;
    auto item_tile = [&](long long item) -> long long { return (item / msplit) * CL + crank; };   // may be >= ntiles (CL = 2)

    if (warp == TS_EPI / 32) {
        // ---------------- loader: (A chunk, B chunk) pairs into the ring
        if ((tid & 31) == 0) {
            constexpr uint32_t bytes_a = A_PART * sizeof(float), bytes_b = 2 * B_EL * sizeof(float);
            long long q = 0;
            for (long long it = 0; it < my_items; ++it) {
                const long long item = unit + it * nunits;
                const long long tile = min(item_tile(item), ntiles - 1);   // a pair's odd tile past the end re-reads the last one
                const int m0 = (int)(item % msplit) * mper, m1 = min(M, m0 + mper);
                for (int m = m0; m < m1; ++m) {
                    for (int ch = 0; ch < nch; ++ch, ++q) {
                        const int st = (int)(q % TS_NS);
                        if (q >= TS_NS) bt_wait(&empty_bar[st], (uint32_t)(((q / TS_NS) - 1) & 1));
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                         bt_smem_u32(&full_bar[st])),
                                     "r"(bytes_a + bytes_b)
                                     : "memory");
                        float* slot = ring + (size_t)st * SLOT;
                        bt_bulk(slot, Ag + ((size_t)tile * nch + ch) * 2 * A_EL, bytes_a, &full_bar[st]);
                        const float* bsrc = Bg + ((size_t)m * nch + ch) * 2 * B_EL;
                        if (CL == 1) {
                            bt_bulk(slot + A_PART, bsrc, bytes_b, &full_bar[st]);
                        } else {   // this CTA's half (rank 0: hi image, rank 1: lo image) into both rings
                            bt_bulk_mc(slot + A_PART + crank * B_EL, bsrc + crank * B_EL, bytes_b / 2, &full_bar[st],
                                       (uint16_t)((1u << CL) - 1u));
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == TS_EPI / 32 + 1) {
        // ---------------- MMA issuer
        if ((tid & 31) == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BT_N >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            long long q = 0, nacc = 0;
            for (long long it = 0; it < my_items; ++it) {
                const long long item = unit + it * nunits;
                const int m0 = (int)(item % msplit) * mper, m1 = min(M, m0 + mper);
                for (int m = m0; m < m1; ++m, ++nacc) {
                    const int b = (int)(nacc & 1);
                    if (nacc >= 2) bt_wait(&acc_empty[b], (uint32_t)(((nacc >> 1) - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t dacc = tmem + (uint32_t)(b * BT_N);
                    for (int ch = 0; ch < nch; ++ch, ++q) {
                        const int st = (int)(q % TS_NS);
                        bt_wait(&full_bar[st], (uint32_t)((q / TS_NS) & 1));
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        const uint32_t ah = bt_smem_u32(ring + (size_t)st * SLOT), al = ah + A_EL * 4;
                        const uint32_t bh = ah + A_PART * 4, bl = bh + B_EL * 4;
#pragma unroll
                        for (int s2 = 0; s2 < BT_BK / 8; ++s2) {
                            const uint32_t off = (uint32_t)s2 * 256;
                            const uint32_t acc0 = (ch > 0 || s2 > 0) ? 1u : 0u;
                            bt_mma(dacc, bt_desc(ah + off), bt_desc(bh + off), idesc, acc0);
                            bt_mma(dacc, bt_desc(ah + off), bt_desc(bl + off), idesc, 1u);
                            if (!EXACT) bt_mma(dacc, bt_desc(al + off), bt_desc(bh + off), idesc, 1u);
                        }
                        if (CL == 1) {
                            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                             bt_smem_u32(&empty_bar[st]))
                                         : "memory");
                        } else {   // the slot is free once both CTAs' MMAs on it have retired
                            asm volatile(
                                "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                                    bt_smem_u32(&empty_bar[st])),
                                "h"((uint16_t)((1u << CL) - 1u))
                                : "memory");
                        }
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     bt_smem_u32(&acc_full[b]))
                                 : "memory");
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: TMEM -> 32 x 32 transposes -> full 128-byte row segments
        const int half = tid >> 7, lane = tid & 31;   // column group of this thread: [half * QC, (half + 1) * QC)
        const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * QC);
        float* xp = Xpose + (size_t)warp * 1024;
        long long nacc = 0;
        for (long long it = 0; it < my_items; ++it) {
            const long long item = unit + it * nunits;
            const long long tile = item_tile(item);   // rows past n are not stored (g < n below)
            const int m0 = (int)(item % msplit) * mper, m1 = min(M, m0 + mper);
            const long long wrow0 = tile * BT_ROWS + (warp & 3) * 32;
            for (int m = m0; m < m1; ++m, ++nacc) {
                const int b = (int)(nacc & 1);
                bt_wait(&acc_full[b], (uint32_t)((nacc >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
                for (int c0 = 0; c0 < QC; c0 += 32) {
                    float v[32];
                    bt_ld32(taddr + (uint32_t)(b * BT_N) + c0, v);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<float4*>(xp + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    __syncwarp();
                    const int cj = lane & 7, col = half * QC + c0 + 4 * cj;
#pragma unroll
                    for (int rb = 0; rb < 32; rb += 4) {
                        const int r = rb + (lane >> 3);
                        const float4 w = *reinterpret_cast<const float4*>(xp + r * 32 + ((cj ^ (r & 7)) << 2));
                        const long long g = wrow0 + r;
                        if (g < n) {
                            float* dst = T + g * ldt + (long long)m * K + col;
                            if ((K & 3) == 0 && col + 3 < K) __stcs(reinterpret_cast<float4*>(dst), w);
                            else {
                                if (col < K) dst[0] = w.x;
                                if (col + 1 < K) dst[1] = w.y;
                                if (col + 2 < K) dst[2] = w.z;
                                if (col + 3 < K) dst[3] = w.w;
                            }
                        }
                    }
                    __syncwarp();
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bt_smem_u32(&acc_empty[b])) : "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (CL > 1) bt_cluster_sync();   // no CTA leaves while its peer may still multicast into it
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BT_N));
    }
}

static int launch_table_tc_stream(const float* X, long long n, long long ldx, int D, const float* cw, const double* sq,
                                  int M, int K, int nch, float* T, long long ldt, cudaStream_t s, bool try_exact) {
    constexpr size_t A_EL = (size_t)BT_ROWS * BT_BK, B_EL = (size_t)BT_N * BT_BK;
    const long long ntiles = (n + BT_ROWS - 1) / BT_ROWS;
    float* Bg = (float*)scratch(14, sizeof(float) * (size_t)M * nch * 2 * B_EL, s);
    float* Ag = (float*)scratch(16, sizeof(float) * (size_t)ntiles * nch * 2 * A_EL, s);
    if (!Bg || !Ag) return fail_cuda(cudaErrorMemoryAllocation, "table_tc_stream scratch");
    cb_tf32_prep_kernel<<<grid_for((long long)M * nch * BT_N * BT_BK, 256, 4096), 256, 0, s>>>(cw, sq, M, K, D, nch, Bg);
    DA_CHECK_LAUNCH("cb_tf32_prep_kernel(stream)");
    int* flag = nullptr;
    if (try_exact) {
        flag = (int*)scratch(15, sizeof(int), s);
        if (!flag) return fail_cuda(cudaErrorMemoryAllocation, "table_tc flag");
        DA_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    }
    // a few thousand blocks with grid-stride loops: one flag check per warp at the end of its loop
    a_tf32_img_kernel<<<grid_for(ntiles * nch * (long long)(BT_ROWS * (BT_BK / 4)), 256, 148 * 32), 256, 0, s>>>(
        X, n, ldx, D, nch, ntiles, Ag, flag);
    DA_CHECK_LAUNCH("a_tf32_img_kernel");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int msplit = M % 4 == 0 ? 4 : (M % 2 == 0 ? 2 : 1);
    if (const char* e = getenv("DA_TABLE_MSPLIT")) msplit = std::max(1, std::min(M, atoi(e)));   // A/B runs
    // 3xTF32 instance: 4 slots of 48 KB + 8 transpose tiles; exact instances: 4 slots of 40 KB + 8 tiles
    // (16 epilogue warps, Q = 4, measured no faster than 8 at D = 128)
    const size_t smem = sizeof(float) * ((size_t)TS_NS * (2 * A_EL + 2 * B_EL) + 8 * 1024);
    const size_t smem_x = sizeof(float) * ((size_t)TS_NS * (A_EL + 2 * B_EL) + 8 * 1024);
    static bool attr_set_dev[64] = {};   // per device (one process per GPU is the usual case)
    bool& attr_set = attr_set_dev[dev & 63];
    if (!attr_set) {
        DA_CUDA(cudaFuncSetAttribute(table_tc_stream_kernel<false, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DA_CUDA(cudaFuncSetAttribute(table_tc_stream_kernel<true, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x));
        DA_CUDA(cudaFuncSetAttribute(table_tc_stream_kernel<true, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_x));
        attr_set = true;
    }
    const int grid = (int)std::min<long long>(ntiles * msplit, sms);
    if (try_exact) {   // both instances are launched; the image kernel's flag picks one (no host sync)
        // pairs of CTAs sharing the codeword stream (DA_TABLE_CLUSTER=1/2 forces one CTA / pairs)
        static const int cl_env = getenv("DA_TABLE_CLUSTER") ? atoi(getenv("DA_TABLE_CLUSTER")) : -1;
        const bool pair = cl_env >= 0 ? cl_env == 2 : (nch <= 9 && ntiles >= 4);
        if (pair) {
            const long long units = ((ntiles + 1) / 2) * msplit;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)(2 * std::min<long long>(units, sms / 2)));
            cfg.blockDim = dim3(TS_T);
            cfg.dynamicSmemBytes = smem_x;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            DA_CUDA(cudaLaunchKernelEx(&cfg, table_tc_stream_kernel<true, 2, 2>, (const float*)Ag, n, M, K, nch,
                                       (const float*)Bg, T, ldt, msplit, (const int*)flag));
        } else {
            table_tc_stream_kernel<true, 1, 2><<<grid, TS_T, smem_x, s>>>(Ag, n, M, K, nch, Bg, T, ldt, msplit, flag);
        }
        DA_CHECK_LAUNCH("table_tc_stream_kernel<exact>");
    }
    table_tc_stream_kernel<false, 1, 2><<<grid, TS_T, smem, s>>>(Ag, n, M, K, nch, Bg, T, ldt, msplit, flag);
    DA_CHECK_LAUNCH("table_tc_stream_kernel");
    return 0;
}

// Returns kNotApplicable when the shape does not fit (K > 256) or, for rows too wide
// for the tight bound (D > ~143: 6 accumulation steps per 16 columns), when the caller
// prefers the chunked FFMA table (`stream_ok` = 0; the caller's beam kernel then sees
// fewer exact rechecks).
int launch_table_tc(const float* X, long long n, long long ldx, int D, const float* cw, const double* sq, int M, int K,
                    float* T, long long ldt, cudaStream_t s, int stream_ok) {
    if (K > BT_N || K < 1 || n <= 0) return n <= 0 ? 0 : kNotApplicable;
    const int nch = (D + 1 + BT_BK - 1) / BT_BK;
    if (nch > 9 && !stream_ok) return kNotApplicable;
    return launch_table_tc_stream(X, n, ldx, D, cw, sq, M, K, nch, T, ldt, s, true);
}

}  // namespace da

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
// Both operands are pre-split f64 -> tf32 hi/lo into the canonical K-major
// no-swizzle UMMA layout (x_tf32_prep_kernel, cw_tf32_prep_kernel) and fetched
// with bulk copies by a producer warp, which also issues the MMAs; the exact
// rechecks run in a separate kernel with coalesced row staging.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int TC_M = 128;     // rows per CTA (= TMEM lanes)
constexpr int TC_NMAX = 256;  // codewords per MMA (TMEM columns)
constexpr int TC_BK = 32;     // tf32 elements of K staged per round (4 MMA k-steps)
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

// packed fp32 pairs (sm_100 f32x2): one FMA-pipe instruction for two elements,
// each rounded exactly like the scalar operation
__device__ __forceinline__ void tc_fma2(float& d0, float& d1, float a, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void tc_add2(float& d0, float& d1, float a0, float a1, float b) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b));
}

template <typename TX>
__device__ __forceinline__ double fma_chain(const TX* __restrict__ xr, const double* __restrict__ cr, int k, int e,
                                            double acc) {
    // loads are issued 24 ahead of the (strictly sequential) FMA chain; 16-byte
    // loads when both rows are float64 and 16-byte aligned at k
    if (sizeof(TX) == 8 && ((reinterpret_cast<uintptr_t>(xr + k) | reinterpret_cast<uintptr_t>(cr + k)) & 15) == 0) {
        for (; k + 24 <= e; k += 24) {
            double2 xv[12], cv[12];
#pragma unroll
            for (int u = 0; u < 12; ++u) {
                xv[u] = *reinterpret_cast<const double2*>(reinterpret_cast<const double*>(xr) + k + 2 * u);
                cv[u] = *reinterpret_cast<const double2*>(cr + k + 2 * u);
            }
#pragma unroll
            for (int u = 0; u < 12; ++u) {
                acc = __fma_rn(xv[u].x, cv[u].x, acc);
                acc = __fma_rn(xv[u].y, cv[u].y, acc);
            }
        }
        for (; k + 8 <= e; k += 8) {
            double2 xv[4], cv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xv[u] = *reinterpret_cast<const double2*>(reinterpret_cast<const double*>(xr) + k + 2 * u);
                cv[u] = *reinterpret_cast<const double2*>(cr + k + 2 * u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc = __fma_rn(xv[u].x, cv[u].x, acc);
                acc = __fma_rn(xv[u].y, cv[u].y, acc);
            }
        }
    }
    for (; k + 24 <= e; k += 24) {
        double xv[24], cv[24];
#pragma unroll
        for (int u = 0; u < 24; ++u) { xv[u] = (double)xr[k + u]; cv[u] = cr[k + u]; }
#pragma unroll
        for (int u = 0; u < 24; ++u) acc = __fma_rn(xv[u], cv[u], acc);
    }
    for (; k + 8 <= e; k += 8) {
        double xv[8], cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { xv[u] = (double)xr[k + u]; cv[u] = cr[k + u]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __fma_rn(xv[u], cv[u], acc);
    }
    for (; k < e; ++k) acc = __fma_rn((double)xr[k], cr[k], acc);
    return acc;
}

template <typename TX, bool BLK>
__device__ __forceinline__ double exact_xc(const TX* __restrict__ xr, const double* __restrict__ cr, int d) {
    if (!BLK) return fma_chain(xr, cr, 0, d, 0.0);
    double tot = 0.0;
    bool first = true;
    int k = 0;
    while (k < d) {
        const int e = k + (int)blas_block_len(d - k);
        const double acc = fma_chain(xr, cr, k, e, 0.0);
        k = e;
        tot = first ? acc : dadd(tot, acc);
        first = false;
    }
    return tot;
}

// Codewords (K x d, float64) -> per-chunk tf32 hi/lo tiles in the exact shared
// memory image the MMA reads (zero padded to 256 rows / 32 columns), so CTAs
// fetch each chunk with one bulk copy.
__global__ void cw_tf32_prep_kernel(const double* __restrict__ C, long long ldc, int K, int d, int nch,
                                    float* __restrict__ out) {
    const long long total = (long long)nch * TC_NMAX * TC_BK;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(e / (TC_NMAX * TC_BK));
        const int rem = (int)(e % (TC_NMAX * TC_BK));
        const int r = rem / TC_BK, k = rem % TC_BK;
        const int gk = ch * TC_BK + k;
        float h = 0.f, l = 0.f;
        if (r < K && gk < d) {
            const double v = C[(long long)r * ldc + gk];
            h = to_tf32((float)v);
            l = to_tf32((float)(v - (double)h));
        }
        float* base = out + (size_t)ch * 2 * TC_NMAX * TC_BK;
        const uint32_t o = kmajor_off(r, k) >> 2;
        base[o] = h;
        base[TC_NMAX * TC_BK + o] = l;
    }
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Rows (n x d, float32 or float64) -> per-(tile, chunk) tf32 hi/lo images in the
// exact shared-memory layout the MMA reads (128 rows x 32 k, zero padded), so the
// assign kernel fetches each chunk with one bulk copy.  Built once per Lloyd call
// (the rotated rows do not change between iterations) or per unbound assign.
template <typename TX>
__global__ void x_tf32_prep_kernel(const TX* __restrict__ X, long long n, long long ldx, int d, int nch,
                                   float* __restrict__ out) {
    // one thread per (row, 4-k group); consecutive threads take the 8 rows of one
    // core matrix, so each group of 8 writes 128 contiguous bytes per image and
    // reads 8 full 32-B row segments
    constexpr int A_ELEMS = TC_M * TC_BK, KG = TC_BK / 4;
    const long long ntiles = (n + TC_M - 1) / TC_M;
    const long long total = ntiles * nch * (A_ELEMS / 4);
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long blk = e / (A_ELEMS / 4);       // (tile, chunk)
        const int rem = (int)(e - blk * (A_ELEMS / 4));
        const int rl = rem & 7, kg = (rem >> 3) % KG, r8 = (rem >> 3) / KG;
        const int r = r8 * 8 + rl;
        const long long tile = blk / nch;
        const int ch = (int)(blk - tile * nch);
        const long long gr = tile * TC_M + r;
        const int gk0 = ch * TC_BK + kg * 4;
        float h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            h[u] = 0.f;
            l[u] = 0.f;
            if (gr < n && gk0 + u < d) {
                const double v = (double)X[gr * ldx + gk0 + u];
                h[u] = to_tf32((float)v);
                l[u] = to_tf32((float)(v - (double)h[u]));
            }
        }
        float* base = out + blk * 2 * A_ELEMS;
        const uint32_t o = kmajor_off(r, kg * 4) >> 2;
        *reinterpret_cast<float4*>(base + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(base + A_ELEMS + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

// Persistent warp-specialised kernel: one CTA per SM walks 128-row tiles.
// Warp 8 (one lane) is the producer: per (tile, 32-k chunk) it bulk-copies the
// row image and the codeword image (kept resident when d <= 32) into a 2-stage
// ring and issues 3 x (<= 4) tcgen05.mma into one of two TMEM accumulators.
// Warps 0-7 run the epilogue of each finished tile (two threads per row, one
// per half of the codewords): window, candidate list to global memory.  The
// exact float64 rechecks follow in assign_recheck_kernel.
constexpr int TC_T2 = 256;        // epilogue threads
constexpr int TC_TP = TC_T2 + 32; // + producer warp

__device__ unsigned long long g_at_prof[8];
#define AT_MARK(i)                                                   \
    do {                                                             \
        if (tid == 0) {                                              \
            const long long _t = clock64();                          \
            at_acc[i] += _t - at_t;                                  \
            at_t = _t;                                               \
        }                                                            \
    } while (0)

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 2, 256;" ::: "memory"); }
// the two warps that own the same 32 rows (column halves): named barrier 3 + quadrant, 64 threads
__device__ __forceinline__ void pair_sync(int quad) { asm volatile("bar.sync %0, 64;" ::"r"(3 + quad) : "memory"); }

template <typename TX>
__global__ void __launch_bounds__(TC_TP, 1) assign_tc_kernel(
    const TX* __restrict__ X, long long n, long long ldx, int d, int K, const double* __restrict__ cc,
    const double* __restrict__ xx_in, const float* __restrict__ Ag, const float* __restrict__ Bg,
    unsigned long long* __restrict__ stats, int* __restrict__ ovf_rows, int* __restrict__ ovf_cnt,
    uint8_t* __restrict__ gcand, uint8_t* __restrict__ gcnt, int32_t* __restrict__ lo_labels,
    const int32_t* __restrict__ lo_prev, unsigned long long* __restrict__ lo_changed, int* __restrict__ multi_rows) {
    // lo_labels != nullptr: labels-only mode (the Lloyd loop inside DA).  A row with a single
    // candidate gets its label here; rows with 2..8 candidates go to a compact list for
    // assign_multi_kernel (ovf_cnt[1] counts them) -- no pass over all rows after this kernel.
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int A_ELEMS = TC_M * TC_BK, B_ELEMS = TC_NMAX * TC_BK;
    float* Abuf = reinterpret_cast<float*>(smem);                    // [2 stages][hi, lo][A_ELEMS]
    float* Bbuf = Abuf + 2 * 2 * A_ELEMS;                             // [2 stages][hi, lo][B_ELEMS]
    double* ccs = reinterpret_cast<double*>(Bbuf + 2 * 2 * B_ELEMS);  // [TC_NMAX]
    float* ccf = reinterpret_cast<float*>(ccs + TC_NMAX);            // [TC_NMAX], +inf beyond K
    // per-tile exchange buffers, double-buffered by tile parity (no barrier between tiles)
    double* wmin_h = reinterpret_cast<double*>(ccf + TC_NMAX);        // [2 tiles][2 halves][TC_M]
    unsigned long long* cand64 = reinterpret_cast<unsigned long long*>(wmin_h + 4 * TC_M);   // [2][2][TC_M] packed lists
    int* ncand = reinterpret_cast<int*>(cand64 + 4 * TC_M);           // [2][2][TC_M]
    __shared__ uint64_t full_bar[2], empty_bar[2], acc_full[2], acc_empty[2], b_bar;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double red[8];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int N = (K + 7) & ~7;
    const int nch = (d + TC_BK - 1) / TC_BK;
    const bool b_resident = nch == 1;
    const long long ntiles = (n + TC_M - 1) / TC_M;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(2 * TC_NMAX));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], 1);
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], TC_T2 / 32);   // one arrival per epilogue warp
        }
        mbar_init(&b_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    double cm = 0.0;
    if (tid < TC_T2) {
        for (int k = tid; k < TC_NMAX; k += TC_T2) {
            const double v = k < K ? cc[k] : 0.0;
            ccs[k] = v;
            ccf[k] = k < K ? (float)v : __int_as_float(0x7f800000);
            cm = fmax(cm, v);
        }
        for (int off = 16; off >= 1; off >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, off));
        if (lane == 0) red[warp] = cm;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;

    if (warp == 8) {
        // ---------------- producer: bulk copies + MMA issue (one lane)
        if (lane == 0) {
            const uint32_t idesc = make_idesc_tf32(TC_M, N);
            if (b_resident) {
                mbar_arrive_expect_tx(&b_bar, (uint32_t)(2 * B_ELEMS * sizeof(float)));
                bulk_g2s(Bbuf, Bg, (uint32_t)(2 * B_ELEMS * sizeof(float)), &b_bar);
                mbar_wait(&b_bar, 0);
            }
            // chunks are issued one ahead of the MMAs (the next chunk's copy overlaps
            // this chunk's wait and MMAs; before, every chunk waited for its own
            // freshly issued copy)
            const uint32_t abytes = (uint32_t)(2 * A_ELEMS * sizeof(float));
            const uint32_t bbytes = b_resident ? 0u : (uint32_t)(2 * B_ELEMS * sizeof(float));
            long long iss_tile = blockIdx.x, iss_q = 0;
            int iss_ch = 0;
            auto issue_next = [&]() {
                if (iss_tile >= ntiles) return;
                const int st = (int)(iss_q & 1);
                if (iss_q >= 2) mbar_wait(&empty_bar[st], (uint32_t)(((iss_q >> 1) - 1) & 1));
                float* Ah = Abuf + st * 2 * A_ELEMS;
                float* Bs = b_resident ? Bbuf : Bbuf + st * 2 * B_ELEMS;
                mbar_arrive_expect_tx(&full_bar[st], abytes + bbytes);
                bulk_g2s(Ah, Ag + ((size_t)iss_tile * nch + iss_ch) * 2 * A_ELEMS, abytes, &full_bar[st]);
                if (!b_resident) bulk_g2s(Bs, Bg + (size_t)iss_ch * 2 * B_ELEMS, bbytes, &full_bar[st]);
                ++iss_q;
                if (++iss_ch == nch) { iss_ch = 0; iss_tile += gridDim.x; }
            };
            issue_next();
            long long q = 0, it = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                const int accb = (int)(it & 1);
                if (it >= 2) mbar_wait(&acc_empty[accb], (uint32_t)(((it - 2) >> 1) & 1));
                for (int ch = 0; ch < nch; ++ch, ++q) {
                    const int st = (int)(q & 1);
                    issue_next();                       // chunk q+1 (waits for its slot's MMAs of q-1)
                    float* Ah = Abuf + st * 2 * A_ELEMS;
                    float* Bs = b_resident ? Bbuf : Bbuf + st * 2 * B_ELEMS;
                    mbar_wait(&full_bar[st], (uint32_t)((q >> 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa_hi = smem_u32(Ah), sa_lo = smem_u32(Ah + A_ELEMS);
                    const uint32_t sb_hi = smem_u32(Bs), sb_lo = smem_u32(Bs + B_ELEMS);
                    const uint32_t dacc = tmem + (uint32_t)(accb * TC_NMAX);
                    const int ks = min(TC_BK / 8, (d - ch * TC_BK + 7) / 8);
                    for (int s2 = 0; s2 < ks; ++s2) {
                        const uint32_t off = (uint32_t)s2 * 256;
                        const uint32_t acc0 = (ch > 0 || s2 > 0) ? 1u : 0u;
                        mma_tf32(dacc, make_desc(sa_hi + off), make_desc(sb_hi + off), idesc, acc0);
                        mma_tf32(dacc, make_desc(sa_hi + off), make_desc(sb_lo + off), idesc, 1u);
                        mma_tf32(dacc, make_desc(sa_lo + off), make_desc(sb_hi + off), idesc, 1u);
                    }
                    mma_commit(&empty_bar[st]);
                    if (ch == nch - 1) mma_commit(&acc_full[accb]);
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue warps
        double ccmax = 0.0;
        for (int w = 0; w < 8; ++w) ccmax = fmax(ccmax, red[w]);
        const double sc = sqrt(ccmax);
        const double u22 = 2.384185791015625e-07;  // 2^-22
        long long at_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // phase clocks (thread 0, DA_DEBUG)
        long long at_t = clock64();
        const int erow = tid & (TC_M - 1);   // TMEM lane / tile row owned in the epilogue
        const int ehalf = tid >> 7;          // 0: codewords [0,128), 1: [128,256)
        long long it = 0;
        unsigned lo_nchg = 0;   // labels-only: rows of this thread whose label changed
        // the row norm of the next tile is loaded one tile ahead: waiting on it at the
        // top of every tile was the epilogue's largest stall
        double xx_next = 0.0;
        if (xx_in && (long long)blockIdx.x * TC_M + erow < n) xx_next = xx_in[(long long)blockIdx.x * TC_M + erow];
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int accb = (int)(it & 1);
            const long long r = tile * TC_M + erow;
            const bool valid = r < n;
            double xx = 0.0;
            if (xx_in) {
                xx = valid ? xx_next : 0.0;
                const long long rn = r + (long long)gridDim.x * TC_M;
                if (rn < n) xx_next = xx_in[rn];
            }
            if (valid && !xx_in) {
                const TX* xr = X + r * ldx;
                xx = np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
            }
            const double sx = sqrt(xx);
            // bound on |w' - (cc - 2 x.c)| for w' = fmaf(-2, dot', (float)cc): 3xTF32 + fp32
            // accumulation of the dot, fp32 rounding of cc and of the fma, float64
            // rounding of the window arithmetic
            const double E = 2.0 * (4.0 * d + 16.0) * u22 * sx * sc * (1.0 + 1e-9) +
                             2.384185791015625e-07 * (ccmax + 2.0 * sx * sc) +
                             8.8817841970012523e-16 * (xx + ccmax + 2.0 * sx * sc) + 1e-300;
            mbar_wait(&acc_full[accb], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            AT_MARK(2);
            const int cbeg = ehalf * 128, cend = min(N, cbeg + 128);
            const uint32_t taddr = tmem + (uint32_t)(accb * TC_NMAX) + ((uint32_t)((warp & 3) * 32) << 16);
            float v[32];
            float wminf = __int_as_float(0x7f800000);
            // Both passes are bound by instruction issue: the FMA and the ALU pipe each take one
            // warp instruction per two clocks.  Packed f32x2 operations halve the FMA-pipe
            // count (w' = cc - 2 v for two codewords per instruction); the minimum keeps its
            // three-input ALU form.
            {
                // four independent minimum chains (two epilogue warps per scheduler cannot
                // hide a 16-long dependent chain per load)
                float wm1 = wminf, wm2 = wminf, wm3 = wminf;
                for (int c0 = cbeg; c0 < cend; c0 += 32) {
                    tmem_ld32(taddr + c0, v);
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        float w0, w1, w2, w3, w4, w5, w6, w7;
                        tc_fma2(w0, w1, -2.f, v[i], v[i + 1], ccf[c0 + i], ccf[c0 + i + 1]);
                        tc_fma2(w2, w3, -2.f, v[i + 2], v[i + 3], ccf[c0 + i + 2], ccf[c0 + i + 3]);
                        tc_fma2(w4, w5, -2.f, v[i + 4], v[i + 5], ccf[c0 + i + 4], ccf[c0 + i + 5]);
                        tc_fma2(w6, w7, -2.f, v[i + 6], v[i + 7], ccf[c0 + i + 6], ccf[c0 + i + 7]);
                        wminf = fminf(fminf(wminf, w0), w1);
                        wm1 = fminf(fminf(wm1, w2), w3);
                        wm2 = fminf(fminf(wm2, w4), w5);
                        wm3 = fminf(fminf(wm3, w6), w7);
                    }
                }
                wminf = fminf(fminf(wminf, wm1), fminf(wm2, wm3));
            }
            double* wm = wmin_h + accb * 2 * TC_M;
            wm[ehalf * TC_M + erow] = (double)wminf;
            pair_sync(warp & 3);   // only the row's other half has to be there
            AT_MARK(3);
            const double wmin = fmin(wm[erow], wm[TC_M + erow]);
            const double ub = fmax(xx + wmin + E, 0.0);
            // candidate k iff max(xx + w'_k - E, 0) <= ub  <=>  w'_k <= ub - xx + E (ub >= 0)
            const double tlim = ub - xx + E;
            const float tf = (tlim >= 3.0e38) ? __int_as_float(0x7f800000)
                                              : __fadd_ru((float)tlim, fabsf((float)tlim) * 1e-6f + 1e-30f);
            // -tf2 with tf2 just above tf (tf = +inf: every finite w' is a candidate, as before)
            const float ntf2 = (tlim >= 3.0e38) ? -tf : -__fadd_ru(tf, fabsf(tf) * 1.1920929e-07f + 1e-37f);
            int nc = 0;
            unsigned long long pk = 0ULL;   // this half row's candidates, one byte each, ascending
            for (int c0 = cbeg; c0 < cend; c0 += 32) {
                tmem_ld32(taddr + c0, v);
                // Branch-free test: e = w' - tf2 is negative for every w' <= tf (tf2 lies above
                // tf; a difference of two distinct floats is never zero), and one funnel shift per
                // element moves its sign bit into the mask (compare + select + add cost 2.5 ALU
                // instructions per element before).  Column c0 + i ends at bit 31 - i.  Padding
                // columns (w' = +inf) give +inf or NaN: sign clear.
                uint32_t h4[4] = {0u, 0u, 0u, 0u};   // four independent shift chains of 8 columns each
#pragma unroll
                for (int i = 0; i < 8; i += 2) {
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        float w0, w1, e0, e1;
                        tc_fma2(w0, w1, -2.f, v[8 * g + i], v[8 * g + i + 1], ccf[c0 + 8 * g + i], ccf[c0 + 8 * g + i + 1]);
                        tc_add2(e0, e1, w0, w1, ntf2);
                        h4[g] = __funnelshift_l(__float_as_uint(e0), h4[g], 1);
                        h4[g] = __funnelshift_l(__float_as_uint(e1), h4[g], 1);
                    }
                }
                uint32_t hit = (h4[0] << 24) | (h4[1] << 16) | (h4[2] << 8) | h4[3];   // then walk the (rare) set bits, ascending column
                while (hit) {
                    const int i = __clz(hit);
                    hit &= ~(0x80000000u >> i);
                    if (nc < TC_CMAX) pk |= (unsigned long long)(c0 + i) << (8 * nc);
                    ++nc;
                }
            }
            cand64[(accb * 2 + ehalf) * TC_M + erow] = pk;
            ncand[(accb * 2 + ehalf) * TC_M + erow] = nc;
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[accb]);   // this warp is done with the TMEM buffer (free for tile it + 2 after all 8)
            pair_sync(warp & 3);
            AT_MARK(4);
            if (ehalf == 0 && valid) {
                // the row's candidates (both halves, ascending k) go to global memory; the
                // exact float64 rechecks run in assign_recheck_kernel with coalesced rows
                const int n0 = ncand[accb * 2 * TC_M + erow], n1 = ncand[(accb * 2 + 1) * TC_M + erow];
                if (n0 + n1 > TC_CMAX) {
                    // too many near-ties for this row: a warp-parallel exact scan over
                    // all K runs after the kernel (assign_overflow_kernel)
                    ovf_rows[atomicAdd(ovf_cnt, 1)] = (int)r;
                    gcnt[r] = 0xFF;
                    if (stats) atomicAdd(stats, (unsigned long long)K);
                } else {
                    unsigned long long mg = cand64[accb * 2 * TC_M + erow];
                    if (n1 > 0) mg |= cand64[(accb * 2 + 1) * TC_M + erow] << (8 * n0);   // n0 < 8 here
                    if (lo_labels != nullptr && n0 + n1 == 1) {
                        const int k0 = (int)(mg & 0xFFu);
                        lo_labels[r] = k0;
                        if (lo_prev != nullptr && lo_prev[r] != k0) ++lo_nchg;
                    } else {
                        *reinterpret_cast<uint2*>(gcand + r * 8) = make_uint2((uint32_t)mg, (uint32_t)(mg >> 32));
                        gcnt[r] = (uint8_t)(n0 + n1);
                        if (lo_labels != nullptr) multi_rows[atomicAdd(ovf_cnt + 1, 1)] = (int)r;
                    }
                }
            }
            AT_MARK(5);   // no barrier here: the exchange buffers alternate with the tile parity
        }
        if (lo_changed != nullptr && lo_prev != nullptr) {
            lo_nchg = __reduce_add_sync(0xffffffffu, lo_nchg);
            if (lane == 0 && lo_nchg) atomicAdd(lo_changed, (unsigned long long)lo_nchg);
        }
        if (tid == 0)
            for (int i = 0; i < 8; ++i) atomicAdd(&g_at_prof[i], (unsigned long long)at_acc[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_NMAX));
    }
}

// Rows whose candidate lists overflowed: one warp per row, lanes split the K
// codewords (each an exact BLAS-ordered dot), lexicographic (d2, k) warp minimum.
template <typename TX>
__global__ void assign_overflow_kernel(const TX* __restrict__ X, long long ldx, int d, const double* __restrict__ C,
                                       long long ldc, int K, const double* __restrict__ cc,
                                       const double* __restrict__ xx_in, const int* __restrict__ rows,
                                       const int* __restrict__ cnt, int32_t* __restrict__ labels,
                                       double* __restrict__ d2_out, const int32_t* __restrict__ prev,
                                       unsigned long long* __restrict__ changed) {
    const int lane = threadIdx.x & 31;
    const int nrows = *cnt;
    const bool blk = d > (int)BLAS_Q;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long r = rows[w];
        const TX* xr = X + r * ldx;
        const double xx = xx_in ? xx_in[r]
                                : np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
        double best = __longlong_as_double(0x7ff0000000000000ULL);
        int bk = 0x7fffffff;
        for (int k = lane; k < K; k += 32) {
            const double* crow = C + (long long)k * ldc;
            const double xc = blk ? exact_xc<TX, true>(xr, crow, d) : exact_xc<TX, false>(xr, crow, d);
            double dv = dadd(dsub(xx, dmul(2.0, xc)), cc[k]);
            if (dv < 0.0) dv = 0.0;
            if (lex_less(dv, k, best, bk)) { best = dv; bk = k; }
        }
        for (int off = 16; off >= 1; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int ok = __shfl_xor_sync(0xffffffffu, bk, off);
            if (lex_less(ob, ok, best, bk)) { best = ob; bk = ok; }
        }
        if (lane == 0) {
            labels[r] = bk;
            if (d2_out) d2_out[r] = best;
            if (changed != nullptr && prev != nullptr && prev[r] != bk) atomicAdd(changed, 1ULL);
        }
    }
}

// Exact float64 rechecks of the tensor-core candidates.  One warp per 32
// consecutive rows (lane = row).  The rows' x values and each round's candidate
// codeword rows are staged through shared memory 32 columns at a time with
// coalesced 256-B row reads, then every lane runs its own BLAS-ordered FMA chain
// from a padded (conflict-free) row.  Same value per candidate as assign.cu:
// ((xx - 2 x.c) + cc) clipped at 0, lexicographic (d2, k) minimum.
constexpr int RC_WARPS = 1;

// 4- or 8-byte global -> shared copy that bypasses the registers (LDGSTS)
template <int BYTES>
__device__ __forceinline__ void cp_async(void* sdst, const void* gsrc) {
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
    else if (BYTES == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename TX>
__global__ void __launch_bounds__(32 * RC_WARPS) assign_recheck_kernel(
    const TX* __restrict__ X, long long n, long long ldx, int d, const double* __restrict__ C, long long ldc,
    const double* __restrict__ cc, const double* __restrict__ xx_in, const uint8_t* __restrict__ gcand,
    const uint8_t* __restrict__ gcnt, int32_t* __restrict__ labels, double* __restrict__ d2_out,
    const int32_t* __restrict__ prev, unsigned long long* __restrict__ changed, unsigned long long* __restrict__ stats) {
    // row stride 34 (272 B): 16-byte aligned for the paired copies, and a quarter
    // warp's 16-byte reads of its 8 rows hit 8 disjoint bank groups
    __shared__ __align__(16) TX sx[RC_WARPS][2][32][34];   // the rows' 32-column chunk, double-buffered
    __shared__ __align__(16) double sc[RC_WARPS][32][34];  // one candidate round's codeword rows
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool blk = d > (int)BLAS_Q;
    unsigned long long nstat = 0, nchg = 0;
    for (long long r0 = ((long long)blockIdx.x * RC_WARPS + w) * 32; r0 < n; r0 += (long long)gridDim.x * RC_WARPS * 32) {
        const long long r = r0 + lane;
        const int rows = (int)min(32LL, n - r0);
        int cnt = r < n ? gcnt[r] : 0;
        if (cnt > TC_CMAX) cnt = 0;   // overflow row: assign_overflow_kernel owns it
        uint2 cw2 = make_uint2(0u, 0u);
        if (cnt) cw2 = *reinterpret_cast<const uint2*>(gcand + r * 8);
        if (d2_out == nullptr && cnt == 1) {
            // labels only: a single candidate is the nearest codeword, no float64 work
            const int k0 = (int)(cw2.x & 0xFFu);
            labels[r] = k0;
            if (prev != nullptr && prev[r] != k0) ++nchg;
            cnt = 0;
        }
        int maxc = cnt;
        for (int o = 16; o > 0; o >>= 1) maxc = max(maxc, __shfl_xor_sync(FULL, maxc, o));
        if (maxc == 0) continue;   // warp-uniform: no row of this group needs a recheck
        const unsigned need = __ballot_sync(FULL, cnt > 0);
        double acc[TC_CMAX], tot[TC_CMAX];
#pragma unroll
        for (int j = 0; j < TC_CMAX; ++j) { acc[j] = 0.0; tot[j] = 0.0; }
        // chunks: 32-column pieces that never straddle a BLAS k-block; [bs, be) is
        // the block holding column kc (one block of d columns when d <= BLAS_Q)
        auto block_of = [&](int kc, int& bs, int& be) {
            bs = 0;
            be = d;
            if (blk) {
                while (true) {
                    be = bs + (int)blas_block_len(d - bs);
                    if (kc < be) break;
                    bs = be;
                }
            }
        };
        auto chunk_end = [&](int kc) -> int {
            int bs, be;
            block_of(kc, bs, be);
            return min(be, kc + 32);
        };
        // float64 rows with even strides: 16-byte copies, two rows per instruction
        const bool wide = sizeof(TX) == 8 && ((ldx | ldc) & 1) == 0 &&
                          ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(C)) & 15) == 0;
        const int pc2 = lane & 15, rsub = lane >> 4;
        auto stage_x = [&](int kc, int wd, int buf) {
            if (wide && (wd & 1) == 0) {
                if (2 * pc2 < wd)
                    for (int i = 0; i < 16; ++i) {
                        const int rr = 2 * i + rsub;
                        if (rr < rows && ((need >> rr) & 1u))
                            cp_async<16>(&sx[w][buf][rr][2 * pc2], X + (r0 + rr) * ldx + kc + 2 * pc2);
                    }
            } else if (lane < wd) {
                for (int rr = 0; rr < rows; ++rr)
                    if ((need >> rr) & 1u) cp_async<sizeof(TX)>(&sx[w][buf][rr][lane], X + (r0 + rr) * ldx + kc + lane);
            }
            cp_async_commit();
        };
        __syncwarp();
        int kc = 0, ce = chunk_end(0), buf = 0;
        stage_x(0, ce, 0);
        while (kc < d) {
            const int wd = ce - kc;
            const int nkc = ce, nce = ce < d ? chunk_end(ce) : d;
#pragma unroll
            for (int j = 0; j < TC_CMAX; ++j) {
                if (j < maxc) {
                    const int kj = (int)(((j < 4 ? cw2.x : cw2.y) >> (8 * (j & 3))) & 0xFFu);
                    const bool has = j < cnt;
                    const unsigned hm = __ballot_sync(FULL, has);
                    const bool wchunk = wide && (wd & 1) == 0;
                    __syncwarp();
                    if (wchunk) {
                        for (int i = 0; i < 16; ++i) {
                            const int rr = 2 * i + rsub;
                            const int krr = __shfl_sync(FULL, kj, rr);
                            if (((hm >> rr) & 1u) && 2 * pc2 < wd)
                                cp_async<16>(&sc[w][rr][2 * pc2], C + (long long)krr * ldc + kc + 2 * pc2);
                        }
                    } else {
                        for (int rr = 0; rr < rows; ++rr) {
                            const int krr = __shfl_sync(FULL, kj, rr);
                            if (((hm >> rr) & 1u) && lane < wd) cp_async<8>(&sc[w][rr][lane], C + (long long)krr * ldc + kc + lane);
                        }
                    }
                    cp_async_commit();
                    if (j == 0 && nkc < d) {
                        stage_x(nkc, nce - nkc, buf ^ 1);   // next chunk's rows in flight meanwhile
                        cp_async_wait_group<1>();
                    } else {
                        cp_async_wait_group<0>();
                    }
                    __syncwarp();
                    if (has) {
                        double a = acc[j];
                        if (wchunk) {
                            for (int t = 0; t < wd; t += 2) {
                                const double2 xv = *reinterpret_cast<const double2*>(&sx[w][buf][lane][t]);
                                const double2 cv = *reinterpret_cast<const double2*>(&sc[w][lane][t]);
                                a = __fma_rn(xv.x, cv.x, a);
                                a = __fma_rn(xv.y, cv.y, a);
                            }
                        } else {
                            for (int t = 0; t < wd; ++t) a = __fma_rn((double)sx[w][buf][lane][t], sc[w][lane][t], a);
                        }
                        acc[j] = a;
                    }
                }
            }
            int bs, be;
            block_of(kc, bs, be);
            if (ce == be) {   // end of a BLAS block: fold its chain into the total
#pragma unroll
                for (int j = 0; j < TC_CMAX; ++j) {
                    tot[j] = bs == 0 ? acc[j] : dadd(tot[j], acc[j]);
                    acc[j] = 0.0;
                }
            }
            kc = nkc;
            ce = nce;
            buf ^= 1;
        }
        cp_async_wait_group<0>();
        if (cnt) {
            double xx;
            if (xx_in) {
                xx = xx_in[r];
            } else {
                const TX* xr = X + r * ldx;
                xx = np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
            }
            double best = __longlong_as_double(0x7ff0000000000000ULL);
            int bk = 0x7fffffff;
#pragma unroll
            for (int j = 0; j < TC_CMAX; ++j) {
                if (j < cnt) {
                    const int kj = (int)(((j < 4 ? cw2.x : cw2.y) >> (8 * (j & 3))) & 0xFFu);
                    double dv = dadd(dsub(xx, dmul(2.0, tot[j])), cc[kj]);
                    if (dv < 0.0) dv = 0.0;
                    if (lex_less(dv, kj, best, bk)) { best = dv; bk = kj; }
                }
            }
            labels[r] = bk;
            if (d2_out) d2_out[r] = best;
            nstat += cnt;
            if (prev != nullptr && prev[r] != bk) ++nchg;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        nstat += __shfl_xor_sync(FULL, nstat, o);
        nchg += __shfl_xor_sync(FULL, nchg, o);
    }
    if (lane == 0) {
        if (stats && nstat) atomicAdd(stats, nstat);
        if (changed != nullptr && prev != nullptr && nchg) atomicAdd(changed, nchg);
    }
}

// Labels-only mode: the rows that kept 2..8 candidates (a compact list written by
// assign_tc_kernel).  One warp per row, lane j evaluates candidate j exactly (same
// BLAS-ordered value as assign_recheck_kernel), first minimum by (value, index).
template <typename TX>
__global__ void __launch_bounds__(256) assign_multi_kernel(const TX* __restrict__ X, long long ldx, int d,
                                                           const double* __restrict__ C, long long ldc, int K,
                                                           const double* __restrict__ cc,
                                                           const double* __restrict__ xx_in,
                                                           const uint8_t* __restrict__ gcand,
                                                           const uint8_t* __restrict__ gcnt,
                                                           const int* __restrict__ rows, const int* __restrict__ cnt_p,
                                                           int32_t* __restrict__ labels,
                                                           const int32_t* __restrict__ prev,
                                                           unsigned long long* __restrict__ changed,
                                                           unsigned long long* __restrict__ stats) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int nrows = *cnt_p;
    const bool blk = d > (int)BLAS_Q;
    unsigned long long nchg = 0, nstat = 0;
    if ((((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) >= nrows) return;
    double cc_max = 0.0;
    for (int k = lane; k < K; k += 32) cc_max = fmax(cc_max, cc[k]);
    for (int off = 16; off >= 1; off >>= 1) cc_max = fmax(cc_max, __shfl_xor_sync(FULL, cc_max, off));
    const double sc_max = sqrt(cc_max) * (1.0 + 1e-12);
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long r = rows[w];
        const int cnt = gcnt[r];
        const TX* xr = X + r * ldx;
        double dv = __longlong_as_double(0x7ff0000000000000ULL);
        int kj = 0x7fffffff;
        const double xx = xx_in ? xx_in[r]
                                : np_pw_sum([&](long long i) { double t = (double)xr[i]; return dmul(t, t); }, 0, d);
        // Wide rows: the tensor-core bound grows with d ((4 d + 16) 2^-22), so many rows keep a
        // few candidates whose exact d-long float64 chains are the cost of this kernel.  The
        // candidates' values are first recomputed as warp-wide fp32 dots (ceil(d/32) FMAs per
        // lane + a 5-level shuffle tree: bound E2 below) and the keep rule of the filter is
        // applied again; a single survivor is the nearest codeword, no float64 dot at all.
        unsigned keep = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
        if (d >= 96 && cnt >= 2) {
            float w2[TC_CMAX];
            float w2min = __int_as_float(0x7f800000);
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                const int k = gcand[r * 8 + j];
                const double* crow = C + (long long)k * ldc;
                float dot = 0.f;
                for (int i = lane; i < d; i += 32) dot = fmaf((float)xr[i], (float)crow[i], dot);
                for (int off = 16; off >= 1; off >>= 1) dot += __shfl_xor_sync(FULL, dot, off);
                const float wv = fmaf(-2.f, dot, (float)cc[k]);
#pragma unroll
                for (int q = 0; q < TC_CMAX; ++q) w2[q] = q == j ? wv : w2[q];
                w2min = fminf(w2min, wv);
            }
            const double sx = sqrt(xx) * (1.0 + 1e-12);
            const double u24 = 5.9604644775390625e-08;
            const double steps = (double)((d + 31) / 32 + 5);
            // operand roundings (2 u), the fp32 dot (steps u), cc and the final fma (2 u), the
            // reference's float64 roundings; sc_max >= max ||c||, cc_max >= max ||c||^2
            const double E2 = 2.0 * (steps + 4.0) * u24 * sx * sc_max * (1.0 + 1e-9) +
                              2.0 * u24 * (cc_max + 2.0 * sx * sc_max) +
                              8.8817841970012523e-16 * (xx + cc_max + 2.0 * sx * sc_max) + 1e-30;
            const double ub = fmax(xx + (double)w2min + E2, 0.0);
            unsigned kept = 0;
#pragma unroll
            for (int q = 0; q < TC_CMAX; ++q)
                if (q < cnt && fmax(xx + (double)w2[q] - E2, 0.0) <= ub) kept |= 1u << q;
            keep = kept;
        }
        if (__popc(keep) == 1) {   // decided without float64 work (warp-uniform)
            kj = gcand[r * 8 + (__ffs(keep) - 1)];
            if (lane == 0) {
                labels[r] = kj;
                if (prev != nullptr && prev[r] != kj) ++nchg;
            }
            continue;
        }
        if (lane < cnt && ((keep >> lane) & 1u)) {
            kj = gcand[r * 8 + lane];
            const double* crow = C + (long long)kj * ldc;
            const double xc = blk ? exact_xc<TX, true>(xr, crow, d) : exact_xc<TX, false>(xr, crow, d);
            dv = dadd(dsub(xx, dmul(2.0, xc)), cc[kj]);
            if (dv < 0.0) dv = 0.0;
        }
        for (int off = 4; off >= 1; off >>= 1) {   // candidates live in lanes 0..7
            const double ob = __shfl_xor_sync(FULL, dv, off);
            const int ok = __shfl_xor_sync(FULL, kj, off);
            if (lex_less(ob, ok, dv, kj)) { dv = ob; kj = ok; }
        }
        if (lane == 0) {
            labels[r] = kj;
            nstat += __popc(keep);
            if (prev != nullptr && prev[r] != kj) ++nchg;
        }
    }
    if (lane == 0) {
        if (stats && nstat) atomicAdd(stats, nstat);
        if (changed != nullptr && prev != nullptr && nchg) atomicAdd(changed, nchg);
    }
}

// Row image bound by the host for the duration of one Lloyd call (the rotated
// rows are fixed while the centroids move): assigns on exactly this (X, n, ldx,
// d) read it instead of rebuilding it.
static struct {
    const void* X = nullptr;
    long long n = 0, ldx = 0;
    int d = 0;
    const float* img = nullptr;
} g_img;

long long assign_config_key();
// identity of the bound row image and of the assign configuration (lloyd.cu's graph keys)
int assign_image_key(const void** img, long long* mode) {
    *img = g_img.img;
    *mode = (long long)(uintptr_t)g_img.X * 1315423911LL + (long long)g_img.d * 2654435761LL + g_img.n +
            assign_config_key();
    return 0;
}

size_t assign_image_bytes(long long n, int d) {
    const long long ntiles = (n + TC_M - 1) / TC_M;
    const int nch = (d + TC_BK - 1) / TC_BK;
    return sizeof(float) * (size_t)ntiles * nch * 2 * TC_M * TC_BK;
}

static void build_image(const void* X, int x_is_f32, long long n, long long ldx, int d, float* img, cudaStream_t s) {
    const int nch = (d + TC_BK - 1) / TC_BK;
    const long long total = ((n + TC_M - 1) / TC_M) * nch * TC_M * TC_BK / 4;
    if (x_is_f32)
        x_tf32_prep_kernel<float><<<grid_for(total, 256), 256, 0, s>>>((const float*)X, n, ldx, d, nch, img);
    else
        x_tf32_prep_kernel<double><<<grid_for(total, 256), 256, 0, s>>>((const double*)X, n, ldx, d, nch, img);
}

int assign_bind_image(const void* X, int x_is_f32, long long n, long long ldx, int d, float* img, cudaStream_t s) {
    g_img.X = nullptr;
    g_img.img = nullptr;
    if (X == nullptr || img == nullptr || n <= 0 || d < 1) return 0;   // unbind
    {
        ProfScope ps("assign_image", s);
        build_image(X, x_is_f32, n, ldx, d, img, s);
    }
    DA_CHECK_LAUNCH("x_tf32_prep_kernel");
    g_img.X = X;
    g_img.n = n;
    g_img.ldx = ldx;
    g_img.d = d;
    g_img.img = img;
    return 0;
}

// Returns 1 (without launching) when the shape is outside the tensor-core path.
int launch_assign_tc(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C, long long ldc,
                     int K, const double* cc, const double* xx, int32_t* labels, double* d2, const int32_t* prev,
                     unsigned long long* changed, unsigned long long* stats, cudaStream_t s) {
    if (K > TC_NMAX || K < 1 || d < 1) return 1;
    if (n <= 0) return 0;
    const int nch = (d + TC_BK - 1) / TC_BK;
    const bool bound = g_img.img != nullptr && g_img.X == X && g_img.n == n && g_img.ldx == ldx && g_img.d == d;
    const size_t bg_bytes = (sizeof(float) * (size_t)nch * 2 * TC_NMAX * TC_BK + 255) & ~size_t(255);
    const size_t ovf_bytes = (sizeof(int) * ((size_t)n + 64) + 255) & ~size_t(255);
    const size_t cand_bytes = (9 * (size_t)n + 255) & ~size_t(255);
    const size_t img_bytes = bound ? 0 : assign_image_bytes(n, d);
    const bool labels_only = d2 == nullptr;
    char* base = (char*)scratch(9, bg_bytes + 2 * ovf_bytes + cand_bytes + img_bytes, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "assign_tc scratch");
    float* Bg = (float*)base;
    int* ovf_cnt = (int*)(base + bg_bytes);
    int* ovf_rows = ovf_cnt + 64;
    uint8_t* gcand = (uint8_t*)(base + bg_bytes + ovf_bytes);   // [n][8] candidate codewords
    uint8_t* gcnt = gcand + 8 * (size_t)n;                        // [n] counts (0xFF = overflow)
    int* multi_rows = (int*)(base + bg_bytes + ovf_bytes + cand_bytes);   // [n] rows with 2..8 candidates (labels-only)
    const float* Ag = bound ? g_img.img : (const float*)(base + bg_bytes + 2 * ovf_bytes + cand_bytes);
    DA_CUDA(cudaMemsetAsync(ovf_cnt, 0, 2 * sizeof(int), s));   // [0] overflow rows, [1] multi-candidate rows
    ProfScope ps(d <= 8 ? "assign_tc_d<=8" : d <= 32 ? "assign_tc_d<=32" : d <= 128 ? "assign_tc_d<=128" : "assign_tc_d>128",
                 s);
    if (!bound) {
        build_image(X, x_is_f32, n, ldx, d, (float*)Ag, s);
        DA_CHECK_LAUNCH("x_tf32_prep_kernel");
    }
    cw_tf32_prep_kernel<<<grid_for((long long)nch * TC_NMAX * TC_BK, 256, 4096), 256, 0, s>>>(C, ldc, K, d, nch, Bg);
    DA_CHECK_LAUNCH("cw_tf32_prep_kernel");
    const size_t smem = sizeof(float) * (2 * 2 * TC_M * TC_BK + 2 * 2 * TC_NMAX * TC_BK) + sizeof(double) * TC_NMAX +
                        sizeof(float) * TC_NMAX +
                        sizeof(double) * 4 * TC_M + sizeof(unsigned long long) * 4 * TC_M + sizeof(int) * 4 * TC_M;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long ntiles = (n + TC_M - 1) / TC_M;
    const unsigned grid = (unsigned)std::min<long long>(ntiles, sms);
    const unsigned rgrid = grid_for((n + 31) / 32, RC_WARPS, 1LL << 31);
    if (x_is_f32) {
        auto kf = assign_tc_kernel<float>;
        { const int rc_ = ensure_smem((const void*)kf, (int)smem); if (rc_) return rc_; }
        kf<<<grid, TC_TP, smem, s>>>((const float*)X, n, ldx, d, K, cc, xx, Ag, Bg, stats, ovf_rows, ovf_cnt, gcand,
                                     gcnt, labels_only ? labels : nullptr, prev, changed, multi_rows);
        DA_CHECK_LAUNCH("assign_tc_kernel");
        if (labels_only)
            assign_multi_kernel<float><<<sms, 256, 0, s>>>((const float*)X, ldx, d, C, ldc, K, cc, xx, gcand, gcnt,
                                                           multi_rows, ovf_cnt + 1, labels, prev, changed, stats);
        else
            assign_recheck_kernel<float><<<rgrid, 32 * RC_WARPS, 0, s>>>((const float*)X, n, ldx, d, C, ldc, cc, xx,
                                                                         gcand, gcnt, labels, d2, prev, changed, stats);
        DA_CHECK_LAUNCH("assign_recheck_kernel");
        assign_overflow_kernel<float><<<sms, 256, 0, s>>>((const float*)X, ldx, d, C, ldc, K, cc, xx, ovf_rows, ovf_cnt,
                                                          labels, d2, prev, changed);
    } else {
        auto kf = assign_tc_kernel<double>;
        { const int rc_ = ensure_smem((const void*)kf, (int)smem); if (rc_) return rc_; }
        kf<<<grid, TC_TP, smem, s>>>((const double*)X, n, ldx, d, K, cc, xx, Ag, Bg, stats, ovf_rows, ovf_cnt, gcand,
                                     gcnt, labels_only ? labels : nullptr, prev, changed, multi_rows);
        DA_CHECK_LAUNCH("assign_tc_kernel");
        if (labels_only)
            assign_multi_kernel<double><<<sms, 256, 0, s>>>((const double*)X, ldx, d, C, ldc, K, cc, xx, gcand, gcnt,
                                                            multi_rows, ovf_cnt + 1, labels, prev, changed, stats);
        else
            assign_recheck_kernel<double><<<rgrid, 32 * RC_WARPS, 0, s>>>((const double*)X, n, ldx, d, C, ldc, cc, xx,
                                                                          gcand, gcnt, labels, d2, prev, changed, stats);
        DA_CHECK_LAUNCH("assign_recheck_kernel");
        assign_overflow_kernel<double><<<sms, 256, 0, s>>>((const double*)X, ldx, d, C, ldc, K, cc, xx, ovf_rows,
                                                           ovf_cnt, labels, d2, prev, changed);
    }
    DA_CHECK_LAUNCH("assign_overflow_kernel");
    if (getenv("DA_DEBUG")) {
        unsigned long long hp[8];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(hp, g_at_prof, sizeof(hp));
        unsigned long long tot = 0;
        for (int i = 2; i < 6; ++i) tot += hp[i];
        const char* nm[6] = {"", "", "acc_wait", "pass1", "pass2", "cand_write"};
        fprintf(stderr, "[da] assign_tc d=%d epilogue thread phases:", d);
        for (int i = 2; i < 6; ++i) fprintf(stderr, " %s %.1f%%", nm[i], tot ? 100.0 * hp[i] / tot : 0.0);
        int hc = 0;
        cudaMemcpy(&hc, ovf_cnt, sizeof(int), cudaMemcpyDeviceToHost);
        fprintf(stderr, " overflow_rows %d\n", hc);
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_at_prof, z, sizeof(z));
    }
    return 0;
}

}  // namespace da

// Pieces of the fp32 gather-filter beam encoder (encode_fast.cu): per-warp
// shared-memory carving, the exact float64 dot in the reference's BLAS order,
// and order-preserving float keys for redux.sync.
#pragma once
#include "common.cuh"

namespace da {

constexpr int QCAP = 224;  // per-warp recheck queue

// The double-buffered beam state is addressed as base + cur * stride (a
// two-element pointer array indexed by the stage parity would live in local
// memory and turn every shared access into a generic one).
struct FastSmem {
    int32_t* codes;  // [2][cap*M]
    double* score;   // [2][cap]
    double* lv;
    int32_t* lf;
    double* x64;     // [D]
    float* vbuf;     // [cap*K] approximate values; reused as D doubles for the error
    int32_t* queue;  // [33 + QCAP]: [32] = count, [33..] = queued flat indices
    long long* roff; // [cap*M] cross-table row offsets of the current stage
};

// lean: no per-candidate value buffer (rescans recompute), only the exact-phase
// (value, flat) arrays and the float64 error staging share the region
__host__ __device__ inline size_t fast_vbuf_bytes(int cap, int K, int D, bool lean = false) {
    size_t a = lean ? 0 : sizeof(float) * (size_t)cap * K, b = sizeof(double) * (size_t)D;
    size_t c = (sizeof(double) + sizeof(int)) * (size_t)QCAP;  // exact (value, flat) of queued candidates
    size_t m = a > b ? a : b;
    m = m > c ? m : c;
    return (m + 15) & ~size_t(15);
}

__host__ __device__ inline size_t fast_smem_bytes(int cap, int M, int K, int D, bool lean = false) {
    size_t b = sizeof(double) * (3 * (size_t)cap + D) + sizeof(long long) * (size_t)cap * M;
    b = (b + 15) & ~size_t(15);
    b += fast_vbuf_bytes(cap, K, D, lean);
    b += sizeof(int32_t) * (2 * (size_t)cap * M + cap + 33 + QCAP);
    return (b + 15) & ~size_t(15);
}

__device__ inline FastSmem carve_fast(char* p, int cap, int M, int K, int D, bool lean = false) {
    FastSmem s;
    char* p0 = p;
    s.x64 = (double*)p; p += sizeof(double) * D;  // first: 16-byte aligned for double2 reads
    s.score = (double*)p; p += 2 * sizeof(double) * cap;
    s.lv = (double*)p; p += sizeof(double) * cap;
    s.roff = (long long*)p; p += sizeof(long long) * cap * M;
    p = p0 + (((size_t)(p - p0) + 15) & ~size_t(15));
    s.vbuf = (float*)p; p += fast_vbuf_bytes(cap, K, D, lean);
    s.codes = (int32_t*)p; p += 2 * sizeof(int32_t) * cap * M;
    s.lf = (int32_t*)p; p += sizeof(int32_t) * cap;
    s.queue = (int32_t*)p;
    return s;
}

// exact x.c (reference order: FMA chain over d, OpenBLAS k-blocks above 384).
// Bound by the codeword-row load latency (32 values in flight per lane), not by
// the FMA chain: interleaving the independent k-block chains with fewer loads in
// flight per chain measured 2x slower at D=960.
static __device__ __noinline__ double exact_dot_general(const double* __restrict__ x64, const double* __restrict__ c, int D,
                                                const float* __restrict__ c32 = nullptr) {
    double tot = 0.0;
    bool first = true;
    int d = 0;
    while (d < D) {
        const int len = (int)blas_block_len(D - d);
        double acc = 0.0;
        const int e = d + len;
        // loads run ahead of the (strictly sequential) FMA chain: 16 codeword values
        // per batch, fp32 in memory (exact in float64) so a batch is 4 vector loads
#ifdef DA_DOT64
        // float64 rows read as pairs (no F2F conversions; 2x the bytes)
        if (c32 && (d & 1) == 0) {
            for (; d + 16 <= e; d += 16) {
                double2 cv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) cv[u] = __ldg(reinterpret_cast<const double2*>(c + d) + u);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 xv = *reinterpret_cast<const double2*>(x64 + d + 2 * u);
                    acc = __fma_rn(xv.x, cv[u].x, acc);
                    acc = __fma_rn(xv.y, cv[u].y, acc);
                }
            }
        }
#else
        if (c32 && (d & 3) == 0) {   // a BLAS block may start off a 16-byte boundary (D = 500: blocks of 250)
            for (; d + 32 <= e; d += 32) {
                float4 cv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) cv[u] = __ldg(reinterpret_cast<const float4*>(c32 + d) + u);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __fma_rn(x64[d + 4 * u + 0], (double)cv[u].x, acc);
                    acc = __fma_rn(x64[d + 4 * u + 1], (double)cv[u].y, acc);
                    acc = __fma_rn(x64[d + 4 * u + 2], (double)cv[u].z, acc);
                    acc = __fma_rn(x64[d + 4 * u + 3], (double)cv[u].w, acc);
                }
            }
        }
#endif
        for (; d + 8 <= e; d += 8) {
            double cv[8];
            double xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { cv[u] = __ldg(c + d + u); xv[u] = x64[d + u]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __fma_rn(xv[u], cv[u], acc);
        }
        for (; d < e; ++d) acc = __fma_rn(x64[d], c[d], acc);
        tot = first ? acc : dadd(tot, acc);
        first = false;
    }
    return tot;
}

// Hot path of exact_dot for the common shape (D % 32 == 0, D <= 384: one BLAS
// block, 16-byte aligned fp32 rows): a rolled loop of 32-value batches keeps
// the kernels' hot code small (the beam kernels are instruction-fetch bound
// when their stage loop exceeds the instruction cache); anything else goes out
// of line.  Same FMA sequence either way.
__device__ __forceinline__ double exact_dot(const double* __restrict__ x64, const double* __restrict__ c, int D,
                                            const float* __restrict__ c32 = nullptr) {
    if (c32 == nullptr || (D & 31) != 0 || D > 384) return exact_dot_general(x64, c, D, c32);
    double acc = 0.0;
#pragma unroll 1
    for (int d = 0; d < D; d += 32) {
        float4 cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = __ldg(reinterpret_cast<const float4*>(c32 + d) + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc = __fma_rn(x64[d + 4 * u + 0], (double)cv[u].x, acc);
            acc = __fma_rn(x64[d + 4 * u + 1], (double)cv[u].y, acc);
            acc = __fma_rn(x64[d + 4 * u + 2], (double)cv[u].z, acc);
            acc = __fma_rn(x64[d + 4 * u + 3], (double)cv[u].w, acc);
        }
    }
    return acc;
}

// Packed fp32 pair add (FADD2, sm_100): each lane's result is rounded exactly
// like two scalar adds.
// Rigorous bound of |t' - t| for one fp32 score-table entry t' = sq32 - 2 x.c,
// by how the table was computed (`tab`):
//   0   FFMA dot accumulated sequentially over D (D roundings);
//   1   3xTF32 tensor-core dot (2^-21 representation + 2^-22 per accumulation
//       step, 6 steps per 16 of D+1);
//   -s  FFMA dot in chunks whose partials are added sequentially, s = chunk +
//       ceil(D/chunk) roundings (gamma_c + gamma_{D/c} <= gamma_{c + D/c}),
//       computed on the host: the kernels only select, no division.
// The -2 factor and the norm entry double the dot bound (+8 roundings of slack).
__device__ __forceinline__ double table_err(int tab, int D, double u, double xnorm, double cm) {
    return tab == 1 ? (2.0 * (6.0 * ((D + 16) / 16) + 7.0) * 2.384185791015625e-07 + 9.5367431640625e-07 + 2.0 * u) *
                          (2.0 * xnorm * cm + cm * cm)
                    : (2.0 * (tab < 0 ? (double)(-tab) : (double)D) + 8.0) * u * (xnorm * cm + cm * cm);
}

__device__ __forceinline__ void add2(float& a0, float& a1, float b0, float b1) {
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%0, %1};\n\t"
        "mov.b64 rb, {%2, %3};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1));
}

// (s + t) + 2 * a for a pair, packed (FADD2 + FFMA2).  2 * a is exact, so the
// fused form rounds exactly like the separate multiply and add.
__device__ __forceinline__ void cand2(float& v0, float& v1, float s, float t0, float t1, float a0, float a1) {
    asm("{\n\t.reg .b64 rs, rt, ra, r2, rd;\n\t"
        "mov.b64 rs, {%2, %2};\n\t"
        "mov.b64 rt, {%3, %4};\n\t"
        "mov.b64 ra, {%5, %6};\n\t"
        "mov.b64 r2, {%7, %7};\n\t"
        "add.rn.f32x2 rs, rs, rt;\n\t"
        "fma.rn.f32x2 rd, ra, r2, rs;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(v0), "=f"(v1)
        : "f"(s), "f"(t0), "f"(t1), "f"(a0), "f"(a1), "f"(2.0f));
}

// One streamed 16-byte read (the score table row, read once per stage): L2
// evict-first, so it does not push the cross tables out of L2.
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 v;
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(p));
    return v;
}

// float <-> unsigned key with the same order (for redux.sync.min)
__device__ __forceinline__ unsigned fkey(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funkey(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

}  // namespace da

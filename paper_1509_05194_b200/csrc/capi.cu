// C-ABI of the DA hot path (declared in include/da_b200.h).
//
// Conventions: every pointer is a device pointer allocated by the caller
// (the library never frees caller memory); `stream` is a cudaStream_t passed
// as void*; calls are asynchronous on that stream.  Return value 0 = OK,
// < 0 = invalid argument (Python raises ValueError), > 0 = CUDA error
// (RuntimeError); da_last_error() returns the thread's last message.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/da_b200.h"
#include "common.cuh"
#include "internal.h"

namespace da {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
// 0 auto (by beam width), 1 plain float64, 2 fp32 gather filter, 3 tcgen05 residual-GEMM filter
static int g_encode_mode = 0;
static unsigned long long* g_encode_stats = nullptr;  // device counter of exact rechecks

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, size):
// repeated calls inside a CUDA-graph capture (lloyd.cu) invalidate it.
int ensure_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    int& cur = done[{dev, func}];
    if (bytes <= cur) return 0;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return fail_cuda(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    cur = bytes;
    return 0;
}

void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
long long launch_total() { return g_launches.load(std::memory_order_relaxed); }
// bumped whenever a scratch buffer is freed: captured CUDA graphs that point
// into scratch memory are dropped (lloyd.cu)
std::atomic<long long> g_scratch_gen{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail_arg(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    set_error(buf);
    return -1;
}

int fail_cuda(cudaError_t e, const char* where) {
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return (int)e > 0 ? (int)e : 1;
}

static std::mutex g_scratch_mu;
static std::map<std::pair<int, int>, Scratch> g_scratch;

void* scratch(int slot, size_t bytes, cudaStream_t stream) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_scratch_mu);
    Scratch& s = g_scratch[{dev, slot}];
    if (s.bytes >= bytes && s.ptr) return s.ptr;
    if (s.ptr) {
        cudaStreamSynchronize(stream);
        cudaFree(s.ptr);
        s.ptr = nullptr;
        s.bytes = 0;
        g_scratch_gen.fetch_add(1);
    }
    size_t want = bytes < 256 ? 256 : bytes;
    want = want + want / 8;  // headroom so slightly larger calls do not reallocate
    if (cudaMalloc(&s.ptr, want) != cudaSuccess) {
        cudaGetLastError();
        s.ptr = nullptr;
        return nullptr;
    }
    s.bytes = want;
    return s.ptr;
}

}  // namespace da

using namespace da;

#define STREAM(s) ((cudaStream_t)(s))

extern "C" {

const char* da_last_error(void) { return g_last_error.c_str(); }

int da_version(void) { return DA_B200_ABI_VERSION; }

long long da_launch_count(void) { return g_launches.load(); }

int da_encode_config(int mode, unsigned long long* recheck_counter) {
    if (mode < 0 || mode > 3)
        return fail_arg("encode mode must be 0 (auto), 1 (plain float64), 2 (fp32 gather filter) or 3 (tcgen05 filter)");
    g_encode_mode = mode;
    g_encode_stats = recheck_counter;
    return 0;
}

int64_t da_assign_image_bytes(int64_t n, int d) {
    if (n < 0 || d < 1) return 0;
    return (int64_t)assign_image_bytes(n, d);
}

int da_assign_bind_image(const void* X, int x_f32, int64_t n, int64_t ldx, int d, float* image, void* stream) {
    if (X != nullptr && image != nullptr && (n < 0 || d < 1 || ldx < d))
        return fail_arg("assign_bind_image: bad shape n=%lld d=%d ldx=%lld", (long long)n, d, (long long)ldx);
    return assign_bind_image(X, x_f32, n, ldx, d, image, STREAM(stream));
}

int da_assign_config(int mode, unsigned long long* candidate_counter) {
    if (mode != 0 && mode != 1) return fail_arg("assign mode must be 0 (auto) or 1 (plain float64)");
    return set_assign_config(mode, candidate_counter);
}

int da_release_scratch(void) {
    std::lock_guard<std::mutex> g(g_scratch_mu);
    for (auto& kv : g_scratch)
        if (kv.second.ptr) cudaFree(kv.second.ptr);
    g_scratch.clear();
    g_scratch_gen.fetch_add(1);
    return 0;
}

int da_row_sqnorms(const void* A, int a_f32, int64_t rows, int64_t lda, int d, double* out, void* stream) {
    if (rows < 0 || d < 0 || lda < d) return fail_arg("row_sqnorms: bad shape rows=%lld d=%d lda=%lld", (long long)rows, d, (long long)lda);
    return launch_row_sqnorms(A, a_f32, rows, lda, d, out, STREAM(stream));
}

int da_assign(const void* X, int x_f32, int64_t n, int64_t ldx, int d, const double* C, int64_t ldc, int K,
              const double* cc, const double* xx, int32_t* labels, double* d2, const int32_t* prev,
              unsigned long long* changed, void* stream) {
    if (n < 0 || K < 1 || d < 1 || ldx < d || ldc < d)
        return fail_arg("assign: bad shape n=%lld K=%d d=%d", (long long)n, K, d);
    return launch_assign(X, x_f32, n, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, changed, STREAM(stream));
}

int da_group_sums(const double* X, int64_t n, int64_t ldx, int D, const int32_t* labels, int K, int mode,
                  double* out, int64_t ldo, int32_t* counts, void* stream) {
    if (n < 0 || K < 1 || D < 1 || ldx < D || ldo < D || (mode != 0 && mode != 1))
        return fail_arg("group_sums: bad arguments n=%lld K=%d D=%d mode=%d", (long long)n, K, D, mode);
    if (n >= (1LL << 31)) return fail_arg("group_sums: n=%lld exceeds int32 row ids", (long long)n);
    if (n == 0) {
        if (counts) cudaMemsetAsync(counts, 0, sizeof(int32_t) * K, STREAM(stream));
        return 0;
    }
    return launch_group_sums(X, n, ldx, D, labels, K, mode, out, ldo, counts, STREAM(stream));
}

int da_gs_shard_sort(const double* X, int64_t n, int64_t ldx, int d, const int32_t* labels, int K,
                     int32_t* counts_local, void* stream) {
    if (n < 0 || K < 1 || d < 1 || (n > 0 && ldx < d)) return fail_arg("gs_shard_sort: bad arguments");
    if (n >= (1LL << 31)) return fail_arg("gs_shard_sort: n=%lld exceeds int32 row ids", (long long)n);
    return launch_gs_shard_sort(X, n, ldx, d, labels, K, counts_local, STREAM(stream));
}

int da_gs_shard_plan(const double* X, int64_t n, int64_t ldx, int d, int K, const int32_t* counts_all, int world,
                     int rank, int64_t cap_leaves, double* red, double* send_state, int32_t* counts_global,
                     int rounds, double* overflow, void* stream) {
    if (world < 1 || rank < 0 || rank >= world || cap_leaves < 1 || d < 1)
        return fail_arg("gs_shard_plan: bad arguments world=%d rank=%d cap=%lld", world, rank, (long long)cap_leaves);
    return launch_gs_shard_plan(X, n, ldx, d, K, counts_all, world, rank, cap_leaves, red, send_state, counts_global,
                                rounds, overflow, STREAM(stream));
}

int da_gs_shard_round(const double* X, int64_t ldx, int d, int K, const double* recv_state, double* send_state,
                      double* red, void* stream) {
    return launch_gs_shard_round(X, ldx, d, K, recv_state, send_state, red, STREAM(stream));
}

int da_gs_shard_fold(int d, int K, const double* red, int64_t cap_leaves, const int32_t* counts_global, int mode,
                     double* out, int64_t ldo, void* stream) {
    if (mode != 0 && mode != 1) return fail_arg("gs_shard_fold: mode must be 0 or 1");
    if (ldo < d) return fail_arg("gs_shard_fold: ldo < d");
    return launch_gs_shard_fold(d, K, red, cap_leaves, counts_global, mode, out, ldo, STREAM(stream));
}

int da_label_order(const int32_t* labels, int64_t n, int K, int32_t* order, int32_t* counts, void* stream) {
    if (n < 0 || K < 1) return fail_arg("label_order: bad arguments");
    if (n >= (1LL << 31)) return fail_arg("label_order: n too large");
    return launch_label_order(labels, n, K, order, counts, STREAM(stream));
}

int da_gather_rows(const double* X, int64_t ldx, int D, const int64_t* src, const int32_t* dst, int cnt, double* C,
                   int64_t ldc, void* stream) {
    return launch_gather_rows(X, ldx, D, (const long long*)src, dst, cnt, C, ldc, STREAM(stream));
}

int da_heat_up(const float* X, int64_t n, int D, const int32_t* codes, const float* cw, int M, int K, int m,
               float* out, void* stream) {
    if (m < 0 || m >= M) return fail_arg("dictionary index %d out of range [0, %d)", m, M);
    return launch_heat_up(X, n, D, codes, cw, M, K, m, out, STREAM(stream));
}

int da_vec_err(const void* X, int x_f32, int64_t n, int64_t ldx, int D, const void* codes, int code_bytes,
               int64_t ldc, const float* cw, int M, int K, double* err, void* stream) {
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return fail_arg("code_bytes must be 1, 2 or 4");
    return launch_vec_err(X, x_f32, n, ldx, D, codes, code_bytes, ldc, cw, M, K, err, STREAM(stream));
}

int da_reconstruct(const void* codes, int code_bytes, int64_t n, int64_t ldc, const float* cw, int M, int K, int D,
                   double* out, void* stream) {
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return fail_arg("code_bytes must be 1, 2 or 4");
    return launch_reconstruct(codes, code_bytes, n, ldc, cw, M, K, D, out, STREAM(stream));
}

int da_col_mean(const void* X, int x_f32, int64_t n, int64_t ld, int D, double* mean, void* stream) {
    return launch_col_mean(X, x_f32, n, ld, D, mean, STREAM(stream));
}

int da_pca_cov(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* mean, double* cov, int divide,
               void* stream) {
    if (divide && n < 2) return fail_arg("PCA needs at least 2 vectors, got %lld", (long long)n);
    if (n < 1) return fail_arg("pca_cov: no rows");
    cudaStream_t s = STREAM(stream);
    ProfScope ps("pca_cov", s);
    // numpy evaluates Xc.T @ Xc with OpenBLAS dsyrk: the n-long contraction is cut
    // into GEMM_Q blocks (balanced tail), each an FMA chain from zero, and the block
    // results are added to C in order.  Blocks are computed in parallel here (one
    // gemm z-slice each) and folded in order, wave by wave.
    std::vector<long long> starts{0};
    for (long long ls = 0; ls < (long long)n;) {
        ls += blas_block_len((long long)n - ls);
        starts.push_back(ls);
    }
    const long long nb = (long long)starts.size() - 1;
    const long long dd = (long long)D * D;
    long long wave = std::max(1LL, std::min(nb, (256LL << 20) / (dd * 8)));
    double* part = (double*)scratch(5, sizeof(double) * (size_t)(wave * dd), s);
    long long* kst = (long long*)scratch(6, sizeof(long long) * (size_t)(nb + 1), s);
    if (!part || !kst) return fail_cuda(cudaErrorMemoryAllocation, "pca_cov scratch");
    DA_CUDA(cudaMemcpyAsync(kst, starts.data(), sizeof(long long) * (nb + 1), cudaMemcpyHostToDevice, s));
    for (long long w0 = 0; w0 < nb; w0 += wave) {
        const long long wn = std::min(wave, nb - w0);
        GemmArgs g{};
        g.A = X; g.a_f32 = x_f32; g.sai = 1; g.sak = ld; g.asub = mean; g.asub_mode = 1;
        g.B = X; g.b_f32 = x_f32; g.sbk = ld; g.sbj = 1; g.bsub = mean; g.bsub_mode = 2;
        g.C = part; g.sci = D; g.scj = 1; g.sCz = dd;
        g.M = D; g.N = D; g.K = n; g.nb2 = 1; g.ksplit = (int)wn; g.kstarts = kst + w0; g.epi = 0;
        int rc;
        {
            ProfScope p1("pca_cov_gemm", s);
            rc = launch_gemm(g, 1, s);
        }
        if (rc) return rc;
        ProfScope p2("pca_cov_fold", s);
        const bool last = w0 + wn == nb;
        rc = launch_accumulate_partials(part, (int)wn, dd, (last && divide) ? (double)(n - 1) : 0.0, w0 > 0 ? 1 : 0,
                                        cov, s);
        if (rc) return rc;
    }
    // the pinned starts vector must outlive the async copy
    DA_CUDA(cudaStreamSynchronize(s));
    return 0;
}

// Sharded PCA pieces (the reference's reductions cut at shard boundaries,
// continued bit for bit by the next shard; distributed.py runs the ring).
int da_col_sums(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* init, double* sums,
                void* stream) {
    if (D < 1) return fail_arg("col_sums: D must be positive");
    return launch_col_sums(X, x_f32, n, ld, D, init, sums, STREAM(stream));
}

int da_cov_chains(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* mean,
                  const int64_t* seg_starts, int nseg, const double* init, double* out, void* stream) {
    if (nseg < 1 || !seg_starts) return fail_arg("cov_chains: need at least one segment");
    if (nseg > 65535) return fail_arg("cov_chains: at most 65535 segments per call");
    if (seg_starts[0] < 0 || seg_starts[nseg] > n) return fail_arg("cov_chains: segments outside the rows");
    for (int i = 0; i < nseg; ++i) {
        const long long len = seg_starts[i + 1] - seg_starts[i];
        if (len < 1 || len > BLAS_Q) return fail_arg("cov_chains: segment %d has %lld rows (1..384)", i, len);
    }
    cudaStream_t s = STREAM(stream);
    ProfScope ps("pca_cov", s);
    long long* kst = (long long*)scratch(6, sizeof(long long) * (size_t)(nseg + 1), s);
    if (!kst) return fail_cuda(cudaErrorMemoryAllocation, "cov_chains scratch");
    DA_CUDA(cudaMemcpyAsync(kst, seg_starts, sizeof(long long) * (nseg + 1), cudaMemcpyHostToDevice, s));
    GemmArgs g{};
    g.A = X; g.a_f32 = x_f32; g.sai = 1; g.sak = ld; g.asub = mean; g.asub_mode = 1;
    g.B = X; g.b_f32 = x_f32; g.sbk = ld; g.sbj = 1; g.bsub = mean; g.bsub_mode = 2;
    g.C = out; g.sci = D; g.scj = 1; g.sCz = (long long)D * D;
    g.M = D; g.N = D; g.K = n; g.nb2 = 1; g.ksplit = nseg; g.kstarts = kst; g.epi = 0; g.cinit = init;
    int rc;
    {
        ProfScope p1("pca_cov_gemm", s);
        rc = launch_gemm(g, 1, s);
    }
    if (rc) return rc;
    // the host starts array may be released by the caller on return
    DA_CUDA(cudaStreamSynchronize(s));
    return 0;
}

int da_fold(const double* parts, int nz, int64_t len, int accumulate, double* out, void* stream) {
    if (nz < 1 || len < 1) return fail_arg("fold: nothing to fold");
    cudaStream_t s = STREAM(stream);
    ProfScope p2("pca_cov_fold", s);
    return launch_accumulate_partials(parts, nz, len, 0.0, accumulate, out, s);
}

int da_rotate(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* R, const double* mean,
              double* out, int inverse, void* stream) {
    GemmArgs g{};
    g.A = X; g.a_f32 = x_f32; g.sai = ld; g.sak = 1;
    g.B = R; g.b_f32 = 0;
    g.C = out; g.sci = D; g.scj = 1;
    g.M = n; g.N = D; g.K = D; g.nb2 = 1; g.ksplit = 1; g.kchunk = D;
    if (!inverse) {
        // (X - mean) @ R^T : b(k, j) = R[j, k]
        g.asub = mean; g.asub_mode = 2; g.sbk = 1; g.sbj = D; g.epi = 0;
    } else {
        // Y @ R + mean : b(k, j) = R[k, j]
        g.sbk = D; g.sbj = 1; g.epi = 1; g.evec = mean;
    }
    // chunk rows to respect the grid.y limit
    const long long rows_per = 65535LL * 64;
    for (long long r0 = 0; r0 < n; r0 += rows_per) {
        GemmArgs h = g;
        h.M = std::min(rows_per, (long long)n - r0);
        h.A = x_f32 ? (const void*)((const float*)X + r0 * ld) : (const void*)((const double*)X + r0 * ld);
        h.C = out + r0 * D;
        int rc = launch_gemm(h, 1, STREAM(stream));
        if (rc) return rc;
    }
    return 0;
}

int da_gemm_strided(const void* A, int a_f32, int64_t sai, int64_t sak, const void* B, int b_f32, int64_t sbk,
                    int64_t sbj, double* C, int64_t sci, int64_t scj, int64_t M, int64_t N, int64_t K, void* stream) {
    if (M < 0 || N < 0 || K < 0) return fail_arg("gemm: negative shape");
    if (K == 0) {
        // empty contraction: zeros
        for (long long i = 0; i < M; ++i)
            for (long long j = 0; j < N; ++j) cudaMemsetAsync(C + i * sci + j * scj, 0, sizeof(double), STREAM(stream));
        return 0;
    }
    GemmArgs g{};
    g.A = A; g.a_f32 = a_f32; g.sai = sai; g.sak = sak;
    g.B = B; g.b_f32 = b_f32; g.sbk = sbk; g.sbj = sbj;
    g.C = C; g.sci = sci; g.scj = scj;
    g.M = M; g.N = N; g.K = K; g.nb2 = 1; g.ksplit = 1; g.kchunk = K; g.epi = 0;
    return launch_gemm(g, 1, STREAM(stream));
}

int da_einsum_sq(const float* cw, int64_t rows, int D, double* out, void* stream) {
    return launch_einsum_sq(cw, rows, D, out, STREAM(stream));
}

int da_cross_products(const float* cw, int M, int K, int D, int only_m, double* P, double* sq, void* stream) {
    if (M < 1 || K < 1 || D < 1) return fail_arg("cross_products: bad shape");
    cudaStream_t s = STREAM(stream);
    // P[a][b][i][j] = c_a(i) . c_b(j)
    GemmArgs g{};
    g.A = cw; g.a_f32 = 1; g.sai = D; g.sak = 1;
    g.B = cw; g.b_f32 = 1; g.sbk = 1; g.sbj = D;
    g.C = P; g.sci = K; g.scj = 1;
    g.M = K; g.N = K; g.K = D; g.ksplit = 1; g.kchunk = D; g.epi = 0;
    if (only_m < 0) {
        g.sA1 = (long long)K * D; g.sA2 = 0;
        g.sB1 = 0; g.sB2 = (long long)K * D;
        g.sC1 = (long long)M * K * K; g.sC2 = (long long)K * K;
        g.nb2 = M;
        int rc = launch_gemm(g, M, s);
        if (rc) return rc;
        return sq ? launch_einsum_sq(cw, (long long)M * K, D, sq, s) : 0;
    }
    if (only_m >= M) return fail_arg("refresh index %d out of range", only_m);
    // rows a = m (all b) and columns b = m (all a)
    GemmArgs r = g;
    r.A = cw + (size_t)only_m * K * D; r.sA1 = 0; r.sA2 = 0;
    r.sB1 = 0; r.sB2 = (long long)K * D;
    r.C = P + (size_t)only_m * M * K * K; r.sC1 = 0; r.sC2 = (long long)K * K;
    r.nb2 = M;
    int rc = launch_gemm(r, 1, s);
    if (rc) return rc;
    GemmArgs c = g;
    c.sA1 = 0; c.sA2 = (long long)K * D;
    c.B = cw + (size_t)only_m * K * D; c.sB1 = 0; c.sB2 = 0;
    c.C = P + (size_t)only_m * K * K; c.sC1 = 0; c.sC2 = (long long)M * K * K;
    c.nb2 = M;
    rc = launch_gemm(c, 1, s);
    if (rc) return rc;
    // refresh_cross_products rebuilds sq[m] as a pairwise row sum (codebook.py:251)
    return sq ? launch_row_sqnorms(cw + (size_t)only_m * K * D, 1, K, D, D, sq + (size_t)only_m * K, s) : 0;
}

int da_encode(const void* X, int x_f32, int64_t n, int64_t ldx, int D, const float* cw, int M, int K, int L,
              const double* sq, const double* P, void* codes, int code_bytes, int64_t ldcodes, double* err,
              void* stream) {
    if (L < 1) return fail_arg("beam_width must be >= 1");
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return fail_arg("code_bytes must be 1, 2 or 4");
    if (M < 1 || K < 1 || D < 1) return fail_arg("encode: bad codebook shape");
    // auto (0): the fp32 gather filter, which measured faster than the tcgen05
    // residual-GEMM filter at every beam width on B200 once the two-vector and lean
    // kernels landed (config B, 1M vectors, L=1: 17.5 vs 20.1 ms); mode 3 forces it
    const bool tc_auto = false;
    if (x_f32 && (g_encode_mode == 3 || tc_auto)) {
        int rc = launch_encode_tc((const float*)X, n, ldx, D, cw, M, K, L, sq, P, codes, code_bytes, ldcodes, err,
                                  g_encode_stats, STREAM(stream));
        if (rc != kNotApplicable) return rc;  // done, or a real failure
        cudaGetLastError();
    }
    if (x_f32 && g_encode_mode != 1) {
        int rc = launch_encode_fast(X, x_f32, n, ldx, D, cw, M, K, L, sq, P, codes, code_bytes, ldcodes, err,
                                    g_encode_stats, STREAM(stream));
        if (rc <= 0) return rc;  // > 0 only for "does not fit": fall through to the plain encoder
        cudaGetLastError();
    }
    return launch_encode(X, x_f32, n, ldx, D, cw, M, K, L, sq, P, codes, code_bytes, ldcodes, err, STREAM(stream));
}

int da_pair_sums(const void* codes, int code_bytes, int64_t n, int64_t ldc, const double* P, int M, int K, double* out,
                 void* stream) {
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return fail_arg("code_bytes must be 1, 2 or 4");
    return launch_pair_sums(codes, code_bytes, n, ldc, P, M, K, out, STREAM(stream));
}

int da_adc_lut(const double* Q, int64_t nq, int D, const float* cw, int M, int K, const double* sq, double* lut,
               double* qsq, void* stream) {
    cudaStream_t s = STREAM(stream);
    int rc = launch_qsq(Q, nq, D, qsq, s);
    if (rc) return rc;
    GemmArgs g{};
    g.A = Q; g.a_f32 = 0; g.sai = D; g.sak = 1;
    g.B = cw; g.b_f32 = 1; g.sbk = 1; g.sbj = D;
    g.C = lut; g.sci = (long long)M * K; g.scj = 1;
    g.M = nq; g.N = (long long)M * K; g.K = D; g.nb2 = 1; g.ksplit = 1; g.kchunk = D;
    g.epi = 3; g.evec = sq; g.ivec = qsq;
    return launch_gemm(g, 1, s);
}

int da_adc_scan(const void* codes, int code_bytes, int64_t ldc, const double* pair, const int64_t* cand,
                int64_t ncand, int64_t nq, const double* lut, const double* qsq, int M, int K, int r, int64_t* ids,
                double* dists, void* stream) {
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return fail_arg("code_bytes must be 1, 2 or 4");
    return launch_adc_scan(codes, code_bytes, ldc, pair, (const long long*)cand, ncand, nq, lut, qsq, M, K, r,
                           (long long*)ids, dists, STREAM(stream));
}

int da_unpack_vecs(const void* raw, int64_t n, int d, int kind, float* out, int64_t ldo, unsigned long long* bad,
                   void* stream) {
    if (n < 0 || d < 1 || (kind != 0 && kind != 1) || ldo < d)
        return fail_arg("unpack_vecs: bad arguments n=%lld d=%d kind=%d", (long long)n, d, kind);
    return launch_unpack_vecs(raw, n, d, kind, out, ldo, bad, STREAM(stream));
}

int da_adc_pack(const void* codes, int code_bytes, int64_t n, int64_t ldc, const double* pair, int M,
                void* records, void* stream) {
    if (code_bytes != 1 || M < 1 || M > 8) return fail_arg("adc_pack: needs one-byte codes and M <= 8 (M=%d)", M);
    if (n < 0 || ldc < M) return fail_arg("adc_pack: bad shape");
    return launch_adc_pack(codes, n, ldc, pair, M, records, STREAM(stream));
}

int da_adc_scan_packed(const void* records, const int64_t* cand, int64_t ncand, int64_t nq, const double* lut,
                       const double* qsq, int M, int K, int r, int64_t* ids, double* dists, void* stream) {
    return launch_adc_scan_packed(records, (const long long*)cand, ncand, nq, lut, qsq, M, K, r, (long long*)ids,
                                  dists, STREAM(stream));
}

int da_atree_search(const double* lut, const double* qsq, int64_t nq, int M, int K, const int32_t* code,
                    const float* eps, const int64_t* child_lo, const int64_t* child_hi, const int64_t* leaf_ref,
                    const int64_t* suffix_lo, const int32_t* suffix_code, const float* suffix_eps,
                    const int64_t* ids_lo, const int64_t* ids_hi, const int64_t* leaf_ids, int64_t n_nodes,
                    int64_t n_leaves, int64_t n_root, int64_t max_children, const int64_t* budgets, int r,
                    int64_t* ids, double* dists, int64_t* counts, int64_t* stats, void* stream) {
    if (M < 1 || K < 1 || r < 1) return fail_arg("atree_search: bad shape M=%d K=%d r=%d", M, K, r);
    for (int m = 0; m < M; ++m)
        if (budgets[m] < 1) return fail_arg("atree_search: budgets must be positive");
    if (n_nodes <= 0 || n_root <= 0) return fail_arg("atree_search: empty tree");
    return launch_atree_search(lut, qsq, nq, M, K, code, eps, (const long long*)child_lo, (const long long*)child_hi,
                               (const long long*)leaf_ref, (const long long*)suffix_lo, suffix_code, suffix_eps,
                               (const long long*)ids_lo, (const long long*)ids_hi, (const long long*)leaf_ids,
                               n_nodes, n_leaves, n_root, max_children, (const long long*)budgets, r,
                               (long long*)ids, dists, (long long*)counts, (long long*)stats, STREAM(stream));
}

int da_knn(const void* base, int base_f32, int64_t n, int64_t ldb, int D, const double* base_sq, const double* Q,
           int64_t nq, const double* qsq, int r, int64_t* ids, double* dists, void* stream) {
    if (n < 1 || nq < 0 || D < 1 || ldb < D) return fail_arg("knn: bad shape n=%lld nq=%lld D=%d", (long long)n,
                                                             (long long)nq, D);
    if (r < 1 || r > n) return fail_arg("r=%d must be in [1, %lld]", r, (long long)n);
    cudaStream_t s = STREAM(stream);
    ProfScope ps("knn", s);
    // distance blocks of <= 2^27 entries (1 GB): rows of max(0, (||q||^2 - 2 q.x) + ||x||^2)
    // with the dot in OpenBLAS dgemm order, then the per-row top-r
    const long long block = std::max(1LL, std::min((long long)nq, (1LL << 27) / n));
    double* d2 = (double*)scratch(13, sizeof(double) * (size_t)(block * n), s);
    if (!d2) return fail_cuda(cudaErrorMemoryAllocation, "knn distance block");
    for (long long q0 = 0; q0 < nq; q0 += block) {
        const long long rows = std::min(block, (long long)nq - q0);
        GemmArgs g{};
        g.A = Q + q0 * D; g.a_f32 = 0; g.sai = D; g.sak = 1;
        g.B = base; g.b_f32 = base_f32; g.sbk = 1; g.sbj = ldb;
        g.C = d2; g.sci = n; g.scj = 1;
        g.M = rows; g.N = n; g.K = D; g.nb2 = 1; g.ksplit = 1; g.kchunk = D;
        g.epi = 3; g.evec = base_sq; g.ivec = qsq + q0;
        int rc = launch_gemm(g, 1, s);
        if (rc) return rc;
        rc = launch_topr_rows(d2, rows, n, r, (long long*)ids + q0 * r, dists + q0 * r, s);
        if (rc) return rc;
    }
    return 0;
}

int da_np_sum(const double* a, int64_t n, int divide, double* out, void* stream) {
    return launch_np_sum(a, n, divide, out, STREAM(stream));
}

int da_select_better(int64_t n, int M, const int32_t* beam_codes, const double* beam_err, int32_t* inc_codes,
                     double* inc_err, void* stream) {
    return launch_select_better(n, M, beam_codes, beam_err, inc_codes, inc_err, STREAM(stream));
}

int da_set_column(int32_t* codes, int64_t n, int M, int m, const int32_t* labels, void* stream) {
    return launch_set_column(codes, n, M, m, labels, STREAM(stream));
}

}  // extern "C"

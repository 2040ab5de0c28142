// Internal launch prototypes shared by the .cu files and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace da {

// RAII timing scope (prof.cu): records a CUDA event pair on stream s when
// profiling is enabled through da_prof_enable().
struct ProfScope {
    ProfScope(const char* name, cudaStream_t s);
    ~ProfScope();
    const char* name_;
    cudaStream_t s_;
    void* a_;
};

struct GemmArgs {
    const void* A; int a_f32; long long sai, sak, sA1, sA2; const double* asub; int asub_mode;  // 1: by i, 2: by k
    const void* B; int b_f32; long long sbk, sbj, sB1, sB2; const double* bsub; int bsub_mode;  // 1: by k, 2: by j
    double* C; long long sci, scj, sC1, sC2, sCz;
    long long M, N, K;
    int nb2, ksplit; long long kchunk; const long long* kstarts;  // kstarts[ksplit+1] overrides kchunk
    // epi 0: acc; 1: acc + evec[j]; 2: evec[j] - 2*acc; 3: max(0, (ivec[i] - 2*acc) + evec[j])
    int epi; const double* evec; const double* ivec;
    // optional D x D accumulator the chain of k-slice 0 continues from (sharded PCA)
    const double* cinit;
};

int launch_gemm(const GemmArgs& g, int nb1, cudaStream_t s);
int launch_reduce_partials(const double* P, int nz, long long len, double scale_div, double* out, cudaStream_t s);
int launch_col_mean(const void* X, int x_f32, long long n, long long ld, int D, double* mean, cudaStream_t s);
int launch_col_sums(const void* X, int x_f32, long long n, long long ld, int D, const double* init, double* sums,
                    cudaStream_t s);
int launch_col_mean_chunked(const void* X, int x_f32, long long n, long long ld, int D, double* mean, cudaStream_t s);
int launch_accumulate_partials(const double* P, int nz, long long len, double scale_div, int accumulate,
                               double* out, cudaStream_t s);

int launch_row_sqnorms(const void* A, int a_is_f32, long long rows, long long lda, int d, double* out,
                       cudaStream_t s);
int launch_assign(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C, long long ldc,
                  int K, const double* cc, const double* xx, int32_t* labels, double* d2, const int32_t* prev,
                  unsigned long long* changed, cudaStream_t s);

int launch_group_sums(const double* X, long long n, long long ldx, int D, const int32_t* labels, int K, int mode,
                      double* out, long long ldo, int32_t* counts, cudaStream_t s);
int launch_gs_shard_sort(const double* X, long long n, long long ldx, int d, const int32_t* labels, int K,
                         int32_t* counts_local, cudaStream_t s);
int launch_gs_shard_plan(const double* X, long long n, long long ldx, int d, int K, const int32_t* cnt_all, int W,
                         int rank, long long cap, double* red, double* send, int32_t* gcount, int rounds,
                         double* overflow, cudaStream_t s);
int launch_gs_shard_round(const double* X, long long ldx, int d, int K, const double* recv, double* send, double* red,
                          cudaStream_t s);
int launch_gs_shard_fold(int d, int K, const double* red, long long cap, const int32_t* gcount, int mode, double* out,
                         long long ldo, cudaStream_t s);
int launch_label_order(const int32_t* labels, long long n, int K, int32_t* order_out, int32_t* counts,
                       cudaStream_t s);

int launch_encode(const void* X, int x_f32, long long n, long long ldx, int D, const float* cw, int M, int K,
                  int L, const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                  double* err_out, cudaStream_t s);

}  // namespace da

namespace da {
int launch_heat_up(const float* X, long long n, int D, const int32_t* codes, const float* cw, int M, int K, int m,
                   float* out, cudaStream_t s);
int launch_vec_err(const void* X, int x_f32, long long n, long long ldx, int D, const void* codes, int code_bytes,
                   long long ldc, const float* cw, int M, int K, double* err, cudaStream_t s);
int launch_reconstruct(const void* codes, int code_bytes, long long n, long long ldc, const float* cw, int M, int K,
                       int D, double* out, cudaStream_t s);
int launch_einsum_sq(const float* cw, long long rows, int D, double* out, cudaStream_t s);
int launch_pair_sums(const void* codes, int code_bytes, long long n, long long ldc, const double* P, int M, int K,
                     double* out, cudaStream_t s);
int launch_qsq(const double* Q, long long nq, int D, double* out, cudaStream_t s);
int launch_atree_search(const double* lut, const double* qsq, long long nq, int M, int K, const int32_t* code,
                        const float* eps, const long long* child_lo, const long long* child_hi,
                        const long long* leaf_ref, const long long* suffix_lo, const int32_t* suffix_code,
                        const float* suffix_eps, const long long* ids_lo, const long long* ids_hi,
                        const long long* leaf_ids, long long n_nodes, long long n_leaves, long long n_root,
                        long long max_children, const long long* budgets_host, int r, long long* ids_out,
                        double* d_out, long long* cnt_out, long long* stats_out, cudaStream_t s);
int launch_topr_rows(const double* d2, long long rows, long long n, int r, long long* ids_out, double* d_out,
                     cudaStream_t s);
int launch_unpack_vecs(const void* raw, long long n, int d, int kind, float* out, long long ldo,
                       unsigned long long* bad, cudaStream_t s);
int launch_adc_pack(const void* codes, long long n, long long ldc, const double* pair, int M, void* records,
                    cudaStream_t s);
int launch_adc_scan_packed(const void* records, const long long* cand, long long ncand, long long nq,
                           const double* lut, const double* qsq, int M, int K, int r, long long* ids_out,
                           double* d_out, cudaStream_t s);
int launch_adc_scan(const void* codes, int code_bytes, long long ldc, const double* pair, const long long* cand,
                    long long ncand, long long nq, const double* lut, const double* qsq, int M, int K, int r,
                    long long* ids_out, double* d_out, cudaStream_t s);
int launch_np_sum(const double* a, long long n, int divide, double* out, cudaStream_t s);
int launch_gather_rows(const double* X, long long ldx, int D, const long long* src, const int* dst, int cnt, double* C,
                       long long ldc, cudaStream_t s);
int launch_select_better(long long n, int M, const int32_t* beam_codes, const double* beam_err, int32_t* inc_codes,
                         double* inc_err, cudaStream_t s);
int launch_encode_fast(const void* X, int x_f32, long long n, long long ldx, int D, const float* cw, int M, int K,
                       int L, const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                       double* err_out, unsigned long long* stats, cudaStream_t s);
int launch_beam_pair(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, int L, int cap,
                     const float* tab, const double* sq, const double* P, const float* P32, const double* cmax,
                     const double* cbm, const double* cw64, void* codes_out, int code_bytes, long long ldcodes,
                     double* err_out, unsigned long long* stats, int tab_tc, cudaStream_t s);
int launch_assign_tc(const void* X, int x_is_f32, long long n, long long ldx, int d, const double* C, long long ldc,
                     int K, const double* cc, const double* xx, int32_t* labels, double* d2, const int32_t* prev,
                     unsigned long long* changed, unsigned long long* stats, cudaStream_t s);
int set_assign_config(int mode, unsigned long long* stats);
size_t assign_image_bytes(long long n, int d);
int assign_bind_image(const void* X, int x_is_f32, long long n, long long ldx, int d, float* img, cudaStream_t s);
// launcher result meaning "this path does not take the shape" (caller falls through)
constexpr int kNotApplicable = 1 << 30;
int launch_greedy(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, const float* tab,
                  const double* sq, const double* P, const float* P32, const double* cmax, const double* cbm,
                  const double* cw64, void* codes_out, int code_bytes, long long ldcodes, double* err_out,
                  unsigned long long* stats, int tab_tc, cudaStream_t s);
int launch_table_tc(const float* X, long long n, long long ldx, int D, const float* cw, const double* sq, int M, int K,
                    float* T, long long ldt, cudaStream_t s, int stream_ok = 0);
int launch_encode_tc(const float* X, long long n, long long ldx, int D, const float* cw, int M, int K, int L,
                     const double* sq, const double* P, void* codes_out, int code_bytes, long long ldcodes,
                     double* err_out, unsigned long long* stats, cudaStream_t s);
int launch_set_column(int32_t* codes, long long n, int M, int m, const int32_t* labels, cudaStream_t s);
}  // namespace da

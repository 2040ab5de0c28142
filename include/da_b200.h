/*
 * da_b200.h - C-ABI of the B200 Dictionary-Annealing hot path.
 *
 * The reference (annq, pure Python/numpy, /root/reference/pkg/src/annq) has no
 * FFI; its "operator API" is a set of Python functions.  Each export below is
 * the device half of one of those functions; the Python host package
 * paper_1509_05194_b200 binds them with ctypes and keeps the reference's
 * signatures.  The reference site each entry replaces is
 * cited as file:line relative to pkg/src/annq/.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller; the library
 *     never frees caller memory.  Row-major layouts with explicit leading dims.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it (host-side plan caches aside).
 *   - Return: 0 ok; < 0 invalid argument (ValueError); > 0 CUDA error
 *     (RuntimeError).  da_last_error() gives the calling thread's message.
 *   - x_f32 / a_f32 flags select float32 (1) or float64 (0) inputs; float32
 *     inputs are widened exactly, as numpy's astype(float64) does.
 *   - code_bytes is 1 (uint8), 2 (uint16) or 4 (int32) for code matrices.
 */
#ifndef DA_B200_H
#define DA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DA_B200_ABI_VERSION 1

const char* da_last_error(void);
int da_version(void);
/* Number of kernels this library has launched in the process (all devices). */
long long da_launch_count(void);
/* Per-kernel CUDA-event timing (off by default).  da_prof_collect writes
 * "name count total_ms" lines into buf and clears the log. */
int da_prof_enable(int on);
int da_prof_collect(char* buf, int cap);
/* Free every library-owned scratch buffer (all devices). */
int da_release_scratch(void);

/* ||a_r||^2 over the first d columns, numpy pairwise order.
 * replaces (C_active * C_active).sum(axis=1)   clustering.py:144 */
int da_row_sqnorms(const void* A, int a_f32, int64_t rows, int64_t lda, int d, double* out, void* stream);

/* Nearest codeword over the active prefix d with first-min ties; d2 clipped at 0.
 * replaces _assign                              clustering.py:139-148
 * xx optional: precomputed ||x||^2 over the prefix (da_row_sqnorms), reused across Lloyd iterations.
 * prev/changed optional: counts rows whose label differs from prev (clustering.py:199).
 * d2 optional: NULL = labels only (the Lloyd loop inside DA, whose objective trace
 * nobody reads); rows whose nearest codeword the tensor-core bound decides alone
 * then skip the float64 recheck.  Labels and changed are the same either way. */
int da_assign(const void* X, int x_f32, int64_t n, int64_t ldx, int d, const double* C, int64_t ldc, int K,
              const double* cc, const double* xx, int32_t* labels, double* d2, const int32_t* prev,
              unsigned long long* changed, void* stream);

/* Bytes of the tf32 hi/lo row image da_assign_bind_image builds for (n, d). */
int64_t da_assign_image_bytes(int64_t n, int d);

/* Build the tf32 hi/lo image of the first d columns of X (n rows, leading dim
 * ldx) into the caller's buffer `image` (da_assign_image_bytes) and bind it:
 * every following da_assign on exactly (X, n, ldx, d) reads the image instead
 * of re-splitting the rows.  X = NULL unbinds.  The caller keeps X and image
 * unchanged while bound (one Lloyd call: the rotated rows are fixed).
 * part of lloyd_kmeans' per-stage setup  clustering.py:165-203 */
int da_assign_bind_image(const void* X, int x_f32, int64_t n, int64_t ldx, int d, float* image, void* stream);

/* Assign selection: mode 0 (default) = tcgen05 3xTF32 distance tiles in TMEM +
 * rigorous bound + exact float64 recheck (K <= 256; same labels/d2 as mode 1);
 * mode 1 = plain float64 FMA kernel.  candidate_counter (device, optional)
 * accumulates the number of exactly rechecked (row, codeword) pairs. */
int da_assign_config(int mode, unsigned long long* candidate_counter);

/* Per-label sums (mode 1) or means written into the non-empty rows of out (mode 0),
 * over all D columns, bit-identical to argsort(stable)+add.reduceat.
 * replaces _group_means                         clustering.py:151-162 */
int da_group_sums(const double* X, int64_t n, int64_t ldx, int D, const int32_t* labels, int K, int mode,
                  double* out, int64_t ldo, int32_t* counts, void* stream);

/* Stable argsort of labels in [0,K) plus bincount.
 * replaces np.argsort(assign, kind="stable") / np.bincount   clustering.py:154-155 */
int da_label_order(const int32_t* labels, int64_t n, int K, int32_t* order, int32_t* counts, void* stream);

/* C[dst[i], :] = X[src[i], :]  (empty-cluster reseed, clustering.py:192-196) */
int da_gather_rows(const double* X, int64_t ldx, int D, const int64_t* src, const int32_t* dst, int cnt, double* C,
                   int64_t ldc, void* stream);

/* Intermediate set for dictionary m, computed in float64, stored float32.
 * replaces heat_up                              annealing.py:97-112 */
int da_heat_up(const float* X, int64_t n, int D, const int32_t* codes, const float* cw, int M, int K, int m,
               float* out, void* stream);

/* Exact per-vector squared error ||x - sum_m c_m||^2 (reconstruction in m order).
 * replaces _per_vector_errors / distortion rows annealing.py:135-137, codebook.py:206-208 */
int da_vec_err(const void* X, int x_f32, int64_t n, int64_t ldx, int D, const void* codes, int code_bytes,
               int64_t ldc, const float* cw, int M, int K, double* err, void* stream);

/* float64 reconstruction sum_m C[m][codes_m].
 * replaces _reconstruct_batch                   codebook.py:181-188 */
int da_reconstruct(const void* codes, int code_bytes, int64_t n, int64_t ldc, const float* cw, int M, int K, int D,
                   double* out, void* stream);

/* Row-sharded Lloyd update, bit-identical to da_group_sums over the
 * concatenated shards (rank order) -- the reduceat order of
 * clustering.py:151-162 cut at shard boundaries.  Per update:
 *   da_gs_shard_sort   local stable sort; counts_local (K int32) -> allgather
 *                      into counts_all (world x K, rank-major);
 *   da_gs_shard_plan   global pairwise leaves; fills red (cap_leaves*d leaf sums
 *                      | K*d segment first rows) with -0.0 and this shard's leaves
 *                      and first rows; the states of leaves cut at the right
 *                      boundary go to send_state (K*8*d); counts_global = n_k;
 *   `rounds` (<= world-1) rounds of { send send_state right, receive recv_state
 *                      from the left; da_gs_shard_round } (a cut leaf's state
 *                      crosses one boundary per round); the plan adds 1.0 to
 *                      *overflow (when non-NULL) for every cut leaf that spans
 *                      more than `rounds` boundaries -- the caller then redoes
 *                      the update with world-1 rounds;
 *   allreduce(sum) of red, then da_gs_shard_fold: mode 0 = means into the
 *                      filled rows of out, mode 1 = raw sums.
 * cap_leaves >= K + N/64 + 2 (N = global rows).  One shard per process. */
int da_gs_shard_sort(const double* X, int64_t n, int64_t ldx, int d, const int32_t* labels, int K,
                     int32_t* counts_local, void* stream);
int da_gs_shard_plan(const double* X, int64_t n, int64_t ldx, int d, int K, const int32_t* counts_all, int world,
                     int rank, int64_t cap_leaves, double* red, double* send_state, int32_t* counts_global,
                     int rounds, double* overflow, void* stream);
int da_gs_shard_round(const double* X, int64_t ldx, int d, int K, const double* recv_state, double* send_state,
                      double* red, void* stream);
int da_gs_shard_fold(int d, int K, const double* red, int64_t cap_leaves, const int32_t* counts_global, int mode,
                     double* out, int64_t ldo, void* stream);

/* One Lloyd iteration in one call (clustering.py:185-202, one GPU): C_out =
 * C_prev (snap = C_prev too when non-NULL), C_out[k, :d] = reduceat-order mean
 * of the rows labelled k by labels_prev (empty clusters keep C_prev's row),
 * counts (K), then the assign of X[:, :d] against C_out into labels_out
 * (d2_out optional: NULL = labels-only) counting rows whose label changed.
 * flags_dev (2 uint64) = [rows changed, #empty clusters], copied to the pinned
 * flags_host and followed by cudaEventRecord(event) when those are non-NULL.
 * xx = row_sqnorms(X, d) of the rows (reused across iterations). */
int da_lloyd_step(const double* X, int64_t n, int64_t ldx, int d, int K, const double* C_prev, double* C_out,
                  int64_t ldc, double* snap, const int32_t* labels_prev, int32_t* labels_out, double* d2_out,
                  const double* xx, int32_t* counts, unsigned long long* flags_dev, void* flags_host, void* event,
                  void* stream);

/* Context: the devices, one library-owned non-blocking stream per
 * device, and optionally an NCCL communicator for a row shard (NCCL is bound at
 * run time from libnccl.so.2).  A stream argument of NULL in the da_ctx_*
 * collectives means the context's stream of its first device.
 *   da_nccl_unique_id: 128 bytes for ncclCommInitRank, made on one rank and
 *                      shared with the others by the caller;
 *   da_ctx_allreduce_f64 (in place, sum), da_ctx_allgather_i32, da_ctx_shift_f64
 *                      (send to rank+1, receive from rank-1): the exchange steps
 *                      of the sharded Lloyd update (da_gs_shard_*, da_lloyd_*). */
int da_ctx_create(int n_devices, const int* device_ids, void** ctx);
int da_ctx_stream(void* ctx, int i, void** stream);
int da_nccl_unique_id(void* out128);
int da_ctx_nccl_init(void* ctx, int rank, int world, const void* id128);
int da_ctx_allreduce_f64(void* ctx, double* buf, int64_t count, void* stream);
int da_ctx_allgather_i32(void* ctx, const int32_t* send, int32_t* recv, int64_t count, void* stream);
int da_ctx_shift_f64(void* ctx, const double* send, double* recv, int64_t count, void* stream);
int da_ctx_destroy(void* ctx);

/* CUDA graphs for da_lloyd_step (default on; DA_LLOYD_GRAPHS=0 disables): an
 * argument set is run eagerly once, captured the second time and replayed
 * after that; any library scratch reallocation drops the captured graphs, and
 * the per-kernel profiler bypasses them.  on = 0 disables and frees them. */
int da_lloyd_graphs(int on);
/* out[4] = iterations run eagerly, graphs captured, graph replays, failed captures */
int da_lloyd_graph_stats(long long* out);

/* Sharded Lloyd iteration around the collective:
 *   da_lloyd_prepare: C_out = C_prev (and snap), stats[0:3] = [*changed_prev, 0, 0]
 *                     (the previous assign's stats ride this update's allreduce);
 *   da_lloyd_finish:  after the allreduce.  fast=1: red = [sums K*d | counts K |
 *                     ..], C[k, :d] = sums / counts where counts > 0; fast=0: the
 *                     means are already in C (da_gs_shard_fold) and counts are
 *                     the global counts.  flags_dev (4 f64) = [#empty, stats[0],
 *                     stats[1], stats[2]] -> flags_host + event, *changed = 0, then (if
 *                     labels_out) the assign of X against C like da_lloyd_step. */
int da_lloyd_prepare(const double* C_prev, double* C_out, double* snap, int64_t elems,
                     const unsigned long long* changed_prev, double* stats, void* stream);
int da_lloyd_finish(int fast, const double* red, const int32_t* counts, int K, int d, double* C, int64_t ldc,
                    const double* stats, double* flags_dev, void* flags_host, void* event, const double* X,
                    int64_t n, int64_t ldx, const double* xx, const int32_t* labels_prev, int32_t* labels_out,
                    double* d2_out, unsigned long long* changed, void* stream);

/* Column means (PCA centre).  replaces X.mean(axis=0)   clustering.py:93 */
int da_col_mean(const void* X, int x_f32, int64_t n, int64_t ld, int D, double* mean, void* stream);

/* Sample covariance (X - mean)^T (X - mean) / (n - 1)  (divide=1), or the raw
 * centred scatter (divide=0, for sharded PCA).  replaces clustering.py:94-96 */
int da_pca_cov(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* mean, double* cov, int divide,
               void* stream);

/* Sharded PCA, bit-identical to the unsharded reductions (distributed.py runs
 * the rank-ordered ring; the reference is unsharded: clustering.py:93-96).
 *   da_col_sums:   sums = init + X[0] + X[1] + ... per column, one sequential
 *                  add chain (X.mean(axis=0)'s order) continued from the running
 *                  sums of the rows before this shard (init may alias sums;
 *                  init = NULL starts a new chain).
 *   da_cov_chains: out[s] (D x D) = the FMA chain of (x - mean)^T (x - mean) over
 *                  rows [seg_starts[s], seg_starts[s+1]) (1..384 rows: one
 *                  OpenBLAS GEMM_Q block or the part of one inside this shard),
 *                  segment 0 continuing the accumulator `init` when non-NULL.
 *   da_fold:       out = (accumulate ? out : parts[0]) + parts[..] in order (the
 *                  dsyrk block sums added into C). */
int da_col_sums(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* init, double* sums,
                void* stream);
int da_cov_chains(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* mean,
                  const int64_t* seg_starts, int nseg, const double* init, double* out, void* stream);
int da_fold(const double* parts, int nz, int64_t len, int accumulate, double* out, void* stream);

/* inverse=0: out = (X - mean) @ R^T;  inverse=1: out = X @ R + mean.
 * replaces PcaModel.transform / inverse_transform   clustering.py:39-43 */
int da_rotate(const void* X, int x_f32, int64_t n, int64_t ld, int D, const double* R, const double* mean,
              double* out, int inverse, void* stream);

/* Generic strided float64 product C[i,j] = sum_k A[i*sai+k*sak] * B[k*sbk+j*sbj]
 * (sequential FMA over k).  Used for the PCA Gram route   clustering.py:101-110 */
int da_gemm_strided(const void* A, int a_f32, int64_t sai, int64_t sak, const void* B, int b_f32, int64_t sbk,
                    int64_t sbj, double* C, int64_t sci, int64_t scj, int64_t M, int64_t N, int64_t K, void* stream);

/* ||c||^2 per codeword in numpy einsum order.  replaces codebook.py:129, 237, 260 */
int da_einsum_sq(const float* cw, int64_t rows, int D, double* out, void* stream);

/* Cross-product table P[a][b][i][j] = c_a(i).c_b(j), (M,M,K,K) float64, and sq (M,K).
 * only_m < 0: full table (cross_products, codebook.py:231-238);
 * only_m = m: rows/cols of m (refresh_cross_products, codebook.py:241-252). */
int da_cross_products(const float* cw, int M, int K, int D, int only_m, double* P, double* sq, void* stream);

/* Beam-search encode of n vectors with width L; codes (n, M) and exact errors.
 * replaces _beam_tables + _beam_encode_chunk    codebook.py:255-300
 * (encode_dataset codebook.py:319-358, encode_multipath codebook.py:303-316) */
int da_encode(const void* X, int x_f32, int64_t n, int64_t ldx, int D, const float* cw, int M, int K, int L,
              const double* sq, const double* P, void* codes, int code_bytes, int64_t ldcodes, double* err,
              void* stream);

/* Encoder selection (all modes return identical codes/errors):
 *   0 (default) = mode 2 at every beam width (it measured faster than mode 3 from L = 1 to
 *       L = 32 on B200, config B); 1 = plain float64 score tables;
 *   2 = fp32 score table on tcgen05 (tf32-exact rows: two MMAs per k step; otherwise 3xTF32;
 *       rows wider than ~180 columns: the D-tiled streaming table at L = 1, a chunked FFMA
 *       table at L >= 2) + fp32 cross-table gathers as a filter with a rigorous error bound
 *       (greedy kernel at L = 1, two vectors per warp for 2 <= L <= 7, one per warp from
 *       L = 8), exact float64 recheck of the candidates that can still make the beam;
 *   3 = tcgen05 filter: per stage one 3xTF32 GEMM of the beams' residuals against the
 *       dictionary (score = s + ||c||^2 - 2 r.c), same bound + exact recheck.
 * recheck_counter (device, optional) accumulates the number of exactly rechecked candidates. */
int da_encode_config(int mode, unsigned long long* recheck_counter);

/* Query-independent ADC term 2 sum_{a<b} P[a,b][i_a,i_b].  replaces code_pair_sums codebook.py:388-396 */
int da_pair_sums(const void* codes, int code_bytes, int64_t n, int64_t ldc, const double* P, int M, int K,
                 double* out, void* stream);

/* Per-query ADC tables ||q - c_mk||^2 clipped at 0, plus ||q||^2.
 * replaces adc_table                            codebook.py:361-369 */
int da_adc_lut(const double* Q, int64_t nq, int D, const float* cw, int M, int K, const double* sq, double* lut,
               double* qsq, void* stream);

/* ADC distances of candidate codes and top-r by (distance, position) per query.
 * cand == NULL: candidates are rows 0..ncand-1 (exhaustive); else cand is (nq, ncand)
 * row ids, position p breaks ties and ids[...] = cand[q, p].
 * replaces exhaustive_adc_search                codebook.py:399-429 */
int da_adc_scan(const void* codes, int code_bytes, int64_t ldc, const double* pair, const int64_t* cand,
                int64_t ncand, int64_t nq, const double* lut, const double* qsq, int M, int K, int r, int64_t* ids,
                double* dists, void* stream);

/* A-Tree search (one CTA per query): layered walk with per-layer budgets, boundary ties
 * kept in enumeration order, early suffix resolution, r best (distance, id) per query.
 * lut/qsq from da_adc_lut (device); tree arrays as in the reference's ATree (device);
 * budgets: M positive int64 on the HOST.  Outputs (device): ids (nq, r) padded with -1,
 * dists (nq, r) padded with NaN, counts (nq), stats (nq, 2 + M) = nodes_visited,
 * table_lookups, per-layer sizes.
 * replaces atree_search / _traverse.traverse      atree.py:336-475, _traverse.py:52-255 */
int da_atree_search(const double* lut, const double* qsq, int64_t nq, int M, int K, const int32_t* code,
                    const float* eps, const int64_t* child_lo, const int64_t* child_hi, const int64_t* leaf_ref,
                    const int64_t* suffix_lo, const int32_t* suffix_code, const float* suffix_eps,
                    const int64_t* ids_lo, const int64_t* ids_hi, const int64_t* leaf_ids, int64_t n_nodes,
                    int64_t n_leaves, int64_t n_root, int64_t max_children, const int64_t* budgets, int r,
                    int64_t* ids, double* dists, int64_t* counts, int64_t* stats, void* stream);

/* Exact squared-L2 top-r neighbours (ground truth): d2 = max((||q||^2 - 2 q.x) + ||x||^2, 0)
 * with the dot in OpenBLAS dgemm order, ties to the lower id.  base (n x D, f32 or f64, row
 * stride ldb), base_sq (n) and qsq (nq) pairwise row norms, Q (nq x D) float64; device.
 * replaces brute_force_knn / _knn_block        data.py:167-215 */
int da_knn(const void* base, int base_f32, int64_t n, int64_t ldb, int D, const double* base_sq, const double* Q,
           int64_t nq, const double* qsq, int r, int64_t* ids, double* dists, void* stream);

/* Packed candidate records for the scan (one-byte codes, M <= 8): records is n x 16 bytes,
 * codes in bytes 0..7 and the row's pair sum (float64) in bytes 8..15, so one random
 * candidate reads one 32-byte sector.  Built once per encoded set.
 * replaces the (codes, code_pair_sums) inputs of exhaustive_adc_search  codebook.py:388-429 */
int da_adc_pack(const void* codes, int code_bytes, int64_t n, int64_t ldc, const double* pair, int M,
                void* records, void* stream);

/* Unpack n raw texmex records (4-byte dimension header + d values; kind 0 =
 * fvecs float32, kind 1 = bvecs uint8), uploaded as they lie in the file, into
 * (n, d) float32 rows (leading dim ldo).  Non-finite fvecs values add to *bad.
 * replaces the payload decoding of read_fvecs / read_bvecs  data.py:94-127 */
int da_unpack_vecs(const void* raw, int64_t n, int d, int kind, float* out, int64_t ldo, unsigned long long* bad,
                   void* stream);

/* da_adc_scan over packed records (same results, same tie rule).
 * replaces exhaustive_adc_search / A-Tree candidate re-ranking  codebook.py:399-429 */
int da_adc_scan_packed(const void* records, const int64_t* cand, int64_t ncand, int64_t nq, const double* lut,
                       const double* qsq, int M, int K, int r, int64_t* ids, double* dists, void* stream);

/* numpy pairwise sum (divide=0) or mean (divide=1) of a float64 vector, result on device.
 * replaces errs.mean() / .mean() of per-vector errors   clustering.py:187, annealing.py:176 */
int da_np_sum(const double* a, int64_t n, int divide, double* out, void* stream);

/* Keep-the-better rule of da_sweep: where beam_err <= inc_err take the beam code.
 * replaces annealing.py:173-176 */
int da_select_better(int64_t n, int M, const int32_t* beam_codes, const double* beam_err, int32_t* inc_codes,
                     double* inc_err, void* stream);

/* codes[:, m] = labels  (annealing.py:169, 201) */
int da_set_column(int32_t* codes, int64_t n, int M, int m, const int32_t* labels, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DA_B200_H */

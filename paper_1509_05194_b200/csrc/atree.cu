// A-Tree search on the GPU: the layered, budget-truncated
// walk of atree_search (annq/atree.py:336-475; compiled form _traverse.py:52-255),
// one CTA per query, results identical to the reference for the same table.
//
// Per layer the CTA
//   * expands the surviving internal nodes into their children (contiguous id
//     ranges; offsets by a block scan, slot -> parent by binary search),
//     d_child = (d_parent + ts[layer][code]) + 2*eps;
//   * advances in-suffix leaves one step, d += ts[layer][suffix_code] + 2*suffix_eps;
//   * keeps the layer budget: the budget-th smallest distance by a block radix
//     select over order-preserving 64-bit keys, then every strictly smaller entry
//     and the earliest entries equal to it (fresh children before carried leaves),
//     order preserved (_traverse.py:26-48);
//   * splits the kept children into internals and entering leaves (entering
//     leaves first, then carried ones).
// When only leaves remain and no later budget can prune, the remaining suffix
// steps are resolved in one pass.  Finally the r best (distance, id) pairs over
// the surviving leaves' id lists are selected (weighted radix select on the
// distance, radix select on the ids at the boundary) and sorted.
// Scratch: per CTA, sized on the host from the budgets and the widest node.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int AT_T = 256;
}

__device__ __forceinline__ unsigned long long at_key(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// Block-wide exclusive scan of one int per thread; returns the exclusive prefix
// and writes the block total to *total (all threads).
__device__ __forceinline__ int at_block_scan(int v, int* s_w, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < nw ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) s_w[lane] = s;   // inclusive warp prefix
    }
    __syncthreads();
    const int before = (w > 0 ? s_w[w - 1] : 0) + x - v;
    *total = s_w[nw - 1];
    __syncthreads();
    return before;
}

// k-th smallest (0-based, counting weights) of keys[i], i < n.
template <typename KeyF, typename WF>
__device__ unsigned long long at_select(long long n, unsigned long long k, KeyF key, WF weight,
                                        unsigned long long* hist, unsigned long long* s_bcast) {
    unsigned long long prefix = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        for (long long i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned long long kk = key(i);
            if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> shift) & 255], weight(i));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long cum = 0;
            int b = 0;
            for (; b < 255; ++b) {
                if (cum + hist[b] > k) break;
                cum += hist[b];
            }
            s_bcast[0] = k - cum;
            s_bcast[1] = prefix | ((unsigned long long)b << shift);
        }
        __syncthreads();
        k = s_bcast[0];
        prefix = s_bcast[1];
        mask |= 255ULL << shift;
        __syncthreads();
    }
    return prefix;
}

struct AtArgs {
    const double* lut; const double* qsq; long long nq; int M; int K;
    const int32_t* code; const float* eps; const long long* child_lo; const long long* child_hi;
    const long long* leaf_ref; const long long* suffix_lo; const int32_t* suffix_code; const float* suffix_eps;
    const long long* ids_lo; const long long* ids_hi; const long long* leaf_ids;
    long long n_root; const long long* budgets; int r;
    long long cap_new, cap_b;
    char* scratch; size_t scratch_per_cta;
    long long* ids_out; double* d_out; long long* cnt_out; long long* stats_out;
};

__global__ void __launch_bounds__(AT_T) atree_search_kernel(AtArgs a) {
    __shared__ int s_w[32];
    __shared__ unsigned long long hist[256];
    __shared__ unsigned long long s_b[4];
    __shared__ long long s_ll[8];
    const int tid = threadIdx.x;
    const int M = a.M, K = a.K;
    char* base = a.scratch + (size_t)blockIdx.x * a.scratch_per_cta;
    auto carve = [&](size_t bytes) { char* p = base; base += (bytes + 255) & ~size_t(255); return p; };
    long long* nn = (long long*)carve(sizeof(long long) * a.cap_new);
    double* nd = (double*)carve(sizeof(double) * a.cap_new);
    long long* tn = (long long*)carve(sizeof(long long) * a.cap_new);
    double* td = (double*)carve(sizeof(double) * a.cap_new);
    long long* in_ = (long long*)carve(sizeof(long long) * a.cap_b);
    double* id_ = (double*)carve(sizeof(double) * a.cap_b);
    long long* ioff = (long long*)carve(sizeof(long long) * (a.cap_b + 1));
    long long* lr = (long long*)carve(sizeof(long long) * a.cap_b);
    long long* lp = (long long*)carve(sizeof(long long) * a.cap_b);
    double* ld = (double*)carve(sizeof(double) * a.cap_b);
    long long* tlr = (long long*)carve(sizeof(long long) * a.cap_b);
    long long* tlp = (long long*)carve(sizeof(long long) * a.cap_b);
    double* tld = (double*)carve(sizeof(double) * a.cap_b);
    long long* oid = (long long*)carve(sizeof(long long) * a.r);
    double* odd = (double*)carve(sizeof(double) * a.r);

    for (long long q = blockIdx.x; q < a.nq; q += gridDim.x) {
        const double* lut = a.lut + q * (long long)M * K;
        const double qsq = a.qsq[q];
        auto ts = [&](int m, int k) -> double { return dsub(lut[(long long)m * K + k], qsq); };
        long long visited = 0, lookups = 0;
        long long n_new = a.n_root, n_int = 0, n_leaf = 0;
        for (long long v = tid; v < n_new; v += AT_T) {
            nn[v] = v;
            nd[v] = dadd(dadd(qsq, ts(0, a.code[v])), dmul(2.0, (double)a.eps[v]));
        }
        __syncthreads();
        int layer = 0;
        bool resolved = false;
        for (; layer < M; ++layer) {
            if (layer > 0) {
                long long minb = a.budgets[layer];
                for (int t = layer; t < M; ++t) minb = min(minb, a.budgets[t]);
                if (n_int == 0 && n_leaf <= minb) {
                    const int rem = M - layer;
                    for (long long j = tid; j < n_leaf; j += AT_T) {
                        double acc = ld[j];
                        const long long p = lp[j];
                        for (int t = 0; t < rem; ++t)
                            acc = dadd(acc, dadd(ts(layer + t, a.suffix_code[p + t]),
                                                 dmul(2.0, (double)a.suffix_eps[p + t])));
                        ld[j] = acc;
                    }
                    lookups += n_leaf * rem;
                    if (tid == 0)
                        for (int t = layer; t < M; ++t) a.stats_out[q * (2 + M) + 2 + t] = n_leaf;
                    resolved = true;
                    __syncthreads();
                    break;
                }
                // expand internal survivors: child counts -> offsets (block scan)
                long long total = 0;
                for (long long b0 = 0; b0 < n_int; b0 += AT_T) {
                    const long long j = b0 + tid;
                    const int cnt = j < n_int ? (int)(a.child_hi[in_[j]] - a.child_lo[in_[j]]) : 0;
                    int tot;
                    const int ex = at_block_scan(cnt, s_w, &tot);
                    if (j < n_int) ioff[j] = total + ex;
                    total += tot;
                }
                if (tid == 0) ioff[n_int] = total;
                __syncthreads();
                for (long long s = tid; s < total; s += AT_T) {
                    long long lo = 0, hi = n_int - 1;   // last j with ioff[j] <= s
                    while (lo < hi) {
                        const long long mid = (lo + hi + 1) >> 1;
                        if (ioff[mid] <= s) lo = mid; else hi = mid - 1;
                    }
                    const long long c = a.child_lo[in_[lo]] + (s - ioff[lo]);
                    nn[s] = c;
                    nd[s] = dadd(dadd(id_[lo], ts(layer, a.code[c])), dmul(2.0, (double)a.eps[c]));
                }
                n_new = total;
                // advance in-suffix leaves one step
                for (long long j = tid; j < n_leaf; j += AT_T) {
                    const long long p = lp[j];
                    ld[j] = dadd(ld[j], dadd(ts(layer, a.suffix_code[p]), dmul(2.0, (double)a.suffix_eps[p])));
                    lp[j] = p + 1;
                }
                lookups += n_leaf;
                __syncthreads();
            }
            visited += n_new;
            lookups += n_new;
            const long long budget = a.budgets[layer];
            const long long size = n_new + n_leaf;
            if (tid == 0) a.stats_out[q * (2 + M) + 2 + layer] = min(size, budget);
            if (size > budget) {
                // budget-th smallest over (fresh children, then carried leaves)
                auto keyf = [&](long long i) { return at_key(i < n_new ? nd[i] : ld[i - n_new]); };
                const unsigned long long kth =
                    at_select(size, (unsigned long long)(budget - 1), keyf, [](long long) { return 1ULL; }, hist, s_b);
                // strict count, then the earliest equals fill the rest
                long long strict = 0;
                for (long long b0 = 0; b0 < size; b0 += AT_T) {
                    const long long i = b0 + tid;
                    int tot;
                    at_block_scan(i < size && keyf(i) < kth ? 1 : 0, s_w, &tot);
                    strict += tot;
                }
                const long long need = budget - strict;
                long long eq_seen = 0, wn = 0, wl = 0;
                for (long long b0 = 0; b0 < size; b0 += AT_T) {
                    const long long i = b0 + tid;
                    const unsigned long long kk = i < size ? keyf(i) : ~0ULL;
                    const int is_eq = (i < size && kk == kth) ? 1 : 0;
                    int teq;
                    const int eq_before = at_block_scan(is_eq, s_w, &teq);
                    const bool keep = i < size && (kk < kth || (is_eq && eq_seen + eq_before < need));
                    const bool is_new = i < n_new;
                    int tn_;
                    const int pn = at_block_scan(keep && is_new ? 1 : 0, s_w, &tn_);
                    int tl_;
                    const int pl = at_block_scan(keep && !is_new ? 1 : 0, s_w, &tl_);
                    if (keep && is_new) { tn[wn + pn] = nn[i]; td[wn + pn] = nd[i]; }
                    if (keep && !is_new) {
                        const long long j = i - n_new;
                        tlr[wl + pl] = lr[j]; tlp[wl + pl] = lp[j]; tld[wl + pl] = ld[j];
                    }
                    eq_seen += teq;
                    wn += tn_;
                    wl += tl_;
                }
                __syncthreads();
                for (long long i = tid; i < wn; i += AT_T) { nn[i] = tn[i]; nd[i] = td[i]; }
                for (long long j = tid; j < wl; j += AT_T) { lr[j] = tlr[j]; lp[j] = tlp[j]; ld[j] = tld[j]; }
                n_new = wn;
                n_leaf = wl;
                __syncthreads();
            }
            // split kept children: entering leaves first, then the carried leaves
            long long we = 0, wi = 0;
            for (long long b0 = 0; b0 < n_new; b0 += AT_T) {
                const long long i = b0 + tid;
                const bool valid = i < n_new;
                const long long ref = valid ? a.leaf_ref[nn[i]] : -1;
                int te, ti;
                const int pe = at_block_scan(valid && ref >= 0 ? 1 : 0, s_w, &te);
                const int pi = at_block_scan(valid && ref < 0 ? 1 : 0, s_w, &ti);
                if (valid && ref >= 0) { tlr[we + pe] = ref; tlp[we + pe] = a.suffix_lo[ref]; tld[we + pe] = nd[i]; }
                if (valid && ref < 0) { in_[wi + pi] = nn[i]; id_[wi + pi] = nd[i]; }
                we += te;
                wi += ti;
            }
            __syncthreads();
            for (long long j = tid; j < n_leaf; j += AT_T) {
                tlr[we + j] = lr[j]; tlp[we + j] = lp[j]; tld[we + j] = ld[j];
            }
            __syncthreads();
            n_leaf += we;
            for (long long j = tid; j < n_leaf; j += AT_T) { lr[j] = tlr[j]; lp[j] = tlp[j]; ld[j] = tld[j]; }
            n_int = wi;
            __syncthreads();
        }
        (void)resolved;
        // ---- r best (distance, id) over the surviving leaves' id lists
        long long total_ids = 0;
        for (long long b0 = 0; b0 < n_leaf; b0 += AT_T) {
            const long long j = b0 + tid;
            int tot;
            at_block_scan(j < n_leaf ? (int)min(a.ids_hi[lr[j]] - a.ids_lo[lr[j]], (long long)0x3fffffff) : 0, s_w,
                          &tot);
            total_ids += tot;
        }
        const long long take = min((long long)a.r, total_ids);
        if (tid == 0) s_ll[0] = 0;
        __syncthreads();
        if (take > 0) {
            auto lkey = [&](long long j) { return at_key(ld[j]); };
            auto lw = [&](long long j) { return (unsigned long long)(a.ids_hi[lr[j]] - a.ids_lo[lr[j]]); };
            const unsigned long long kth = at_select(n_leaf, (unsigned long long)(take - 1), lkey, lw, hist, s_b);
            // ids of leaves strictly below kth all qualify
            long long strict = 0;
            for (long long b0 = 0; b0 < n_leaf; b0 += AT_T) {
                const long long j = b0 + tid;
                int tot;
                at_block_scan(j < n_leaf && lkey(j) < kth ? (int)lw(j) : 0, s_w, &tot);
                strict += tot;
            }
            const long long need = take - strict;
            // boundary leaves (distance == kth): the `need` smallest ids among them
            // (a leaf's ids are ascending; every id is unique)
            unsigned long long id_cut = 0;
            if (need > 0) {
                // enumerate boundary ids by a flat index over all leaves' id ranges
                // (non-boundary leaves contribute zero weight)
                long long bcount = 0;
                for (long long b0 = 0; b0 < n_leaf; b0 += AT_T) {
                    const long long j = b0 + tid;
                    const int c = (j < n_leaf && lkey(j) == kth) ? (int)lw(j) : 0;
                    int tot;
                    const int ex = at_block_scan(c, s_w, &tot);
                    if (j < n_leaf) ioff[j] = bcount + ex;
                    bcount += tot;
                }
                if (tid == 0) ioff[n_leaf] = bcount;
                __syncthreads();
                auto bid = [&](long long s) -> unsigned long long {
                    long long lo = 0, hi = n_leaf - 1;
                    while (lo < hi) {
                        const long long mid = (lo + hi + 1) >> 1;
                        if (ioff[mid] <= s) lo = mid; else hi = mid - 1;
                    }
                    return (unsigned long long)a.leaf_ids[a.ids_lo[lr[lo]] + (s - ioff[lo])];
                };
                id_cut = at_select(bcount, (unsigned long long)(need - 1), bid, [](long long) { return 1ULL; },
                                   hist, s_b);
            }
            // collect the kept (id, distance) pairs, then place each by its rank
            for (long long j = tid; j < n_leaf; j += AT_T) {
                const unsigned long long kk = lkey(j);
                if (kk > kth) continue;
                for (long long p = a.ids_lo[lr[j]]; p < a.ids_hi[lr[j]]; ++p) {
                    const long long idv = a.leaf_ids[p];
                    if (kk < kth || (need > 0 && (unsigned long long)idv <= id_cut)) {
                        const long long slot = atomicAdd((unsigned long long*)&s_ll[0], 1ULL);
                        if (slot < take) { oid[slot] = idv; odd[slot] = ld[j]; }
                    }
                }
            }
            __syncthreads();
            for (long long t = tid; t < take; t += AT_T) {
                const double dv = odd[t];
                const long long iv = oid[t];
                long long rank = 0;
                for (long long u = 0; u < take; ++u)
                    rank += (odd[u] < dv) || (odd[u] == dv && oid[u] < iv);
                a.ids_out[q * a.r + rank] = iv;
                a.d_out[q * a.r + rank] = dv;
            }
        }
        for (long long t = take + tid; t < a.r; t += AT_T) {
            a.ids_out[q * a.r + t] = -1;
            a.d_out[q * a.r + t] = __longlong_as_double(0x7ff8000000000000ULL);
        }
        if (tid == 0) {
            a.cnt_out[q] = take;
            a.stats_out[q * (2 + M) + 0] = visited;
            a.stats_out[q * (2 + M) + 1] = lookups;
        }
        __syncthreads();
    }
}

int launch_atree_search(const double* lut, const double* qsq, long long nq, int M, int K, const int32_t* code,
                        const float* eps, const long long* child_lo, const long long* child_hi,
                        const long long* leaf_ref, const long long* suffix_lo, const int32_t* suffix_code,
                        const float* suffix_eps, const long long* ids_lo, const long long* ids_hi,
                        const long long* leaf_ids, long long n_nodes, long long n_leaves, long long n_root,
                        long long max_children, const long long* budgets_host, int r, long long* ids_out,
                        double* d_out, long long* cnt_out, long long* stats_out, cudaStream_t s) {
    if (nq <= 0) return 0;
    long long bmax = 1;
    for (int m = 0; m < M; ++m) bmax = std::max(bmax, budgets_host[m]);
    // entries never exceed the layer budget after truncation; fresh children of
    // one layer are at most (kept internals) x (widest node), or the root fan-out
    const long long cap_b = std::min(bmax, std::max(n_nodes, 1LL)) + 1;
    const long long cap_new = std::max(n_root, std::min(bmax, std::max(n_nodes, 1LL)) * std::max(max_children, 1LL)) + 1;
    const size_t per = 4 * (sizeof(long long) * (size_t)cap_new + 256) + 12 * (sizeof(long long) * (size_t)cap_b + 256) +
                       2 * (sizeof(long long) * (size_t)r + 256) + 1024;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // per-CTA scratch; at most ~4 GB in flight
    const long long by_mem = std::max(1LL, (long long)((4ULL << 30) / per));
    const int grid = (int)std::min<long long>(std::min<long long>(nq, (long long)sms * 4), by_mem);
    char* scr = (char*)scratch(11, per * (size_t)grid + 256 + sizeof(long long) * (size_t)M, s);
    if (!scr) return fail_cuda(cudaErrorMemoryAllocation, "atree scratch");
    long long* budgets_dev = (long long*)(scr + per * (size_t)grid);
    DA_CUDA(cudaMemcpyAsync(budgets_dev, budgets_host, sizeof(long long) * M, cudaMemcpyHostToDevice, s));
    AtArgs a{};
    a.lut = lut; a.qsq = qsq; a.nq = nq; a.M = M; a.K = K;
    a.code = code; a.eps = eps; a.child_lo = child_lo; a.child_hi = child_hi; a.leaf_ref = leaf_ref;
    a.suffix_lo = suffix_lo; a.suffix_code = suffix_code; a.suffix_eps = suffix_eps;
    a.ids_lo = ids_lo; a.ids_hi = ids_hi; a.leaf_ids = leaf_ids;
    a.n_root = n_root; a.budgets = budgets_dev; a.r = r;
    a.cap_new = cap_new; a.cap_b = cap_b; a.scratch = scr; a.scratch_per_cta = per;
    a.ids_out = ids_out; a.d_out = d_out; a.cnt_out = cnt_out; a.stats_out = stats_out;
    (void)n_leaves;
    ProfScope ps("atree_search", s);
    atree_search_kernel<<<grid, AT_T, 0, s>>>(a);
    DA_CHECK_LAUNCH("atree_search_kernel");
    return 0;
}

}  // namespace da

namespace da {

// ---------------------------------------------------------------------------
// Exact k-NN ground truth (data.py:167-215): one CTA per query row of a float64
// distance block d2 (rows x n, produced by the ordered GEMM), top-r by
// (distance, lower id): radix-select the r-th distance, keep everything below
// it plus the lowest ids equal to it, then place each kept pair by its rank.
__global__ void __launch_bounds__(AT_T) topr_rows_kernel(const double* __restrict__ d2, long long rows, long long n,
                                                         int r, long long* __restrict__ ids_out,
                                                         double* __restrict__ d_out, long long* __restrict__ scratch) {
    __shared__ int s_w[32];
    __shared__ unsigned long long hist[256];
    __shared__ unsigned long long s_b[4];
    const int tid = threadIdx.x;
    long long* kid = scratch + (long long)blockIdx.x * r;
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const double* drow = d2 + row * n;
        auto key = [&](long long i) { return at_key(drow[i]); };
        const unsigned long long kth = at_select(n, (unsigned long long)(r - 1), key, [](long long) { return 1ULL; },
                                                 hist, s_b);
        long long strict = 0;
        for (long long b0 = 0; b0 < n; b0 += AT_T) {
            const long long i = b0 + tid;
            int tot;
            at_block_scan(i < n && key(i) < kth ? 1 : 0, s_w, &tot);
            strict += tot;
        }
        const long long need = r - strict;
        long long eq_seen = 0, w = 0;
        for (long long b0 = 0; b0 < n; b0 += AT_T) {
            const long long i = b0 + tid;
            const unsigned long long kk = i < n ? key(i) : ~0ULL;
            const int is_eq = (i < n && kk == kth) ? 1 : 0;
            int teq;
            const int eb = at_block_scan(is_eq, s_w, &teq);
            const bool keep = i < n && (kk < kth || (is_eq && eq_seen + eb < need));
            int tk;
            const int pk = at_block_scan(keep ? 1 : 0, s_w, &tk);
            if (keep) kid[w + pk] = i;
            eq_seen += teq;
            w += tk;
        }
        __syncthreads();
        for (int t = tid; t < r; t += AT_T) {
            const long long it = kid[t];
            const double dv = drow[it];
            int rank = 0;
            for (int u = 0; u < r; ++u) {
                const long long iu = kid[u];
                const double du = drow[iu];
                rank += (du < dv) || (du == dv && iu < it);
            }
            ids_out[row * r + rank] = it;
            d_out[row * r + rank] = dv;
        }
        __syncthreads();
    }
}

int launch_topr_rows(const double* d2, long long rows, long long n, int r, long long* ids_out, double* d_out,
                     cudaStream_t s) {
    if (rows <= 0) return 0;
    if (r < 1 || r > n) return fail_arg("knn: r=%d must be in [1, %lld]", r, n);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<long long>(rows, (long long)sms * 4);
    long long* scr = (long long*)scratch(12, sizeof(long long) * (size_t)grid * r, s);
    if (!scr) return fail_cuda(cudaErrorMemoryAllocation, "knn scratch");
    topr_rows_kernel<<<grid, AT_T, 0, s>>>(d2, rows, n, r, ids_out, d_out, scr);
    DA_CHECK_LAUNCH("topr_rows_kernel");
    return 0;
}

}  // namespace da

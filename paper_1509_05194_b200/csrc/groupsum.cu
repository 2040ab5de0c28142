// Lloyd update: per-codeword sums / means over ALL coordinates.
//
// Follows annq/clustering.py:151-162 (`_group_means`):
//   order = argsort(labels, stable); counts = bincount(labels)
//   sums  = add.reduceat(X[order], segment starts, axis=0)
//   means = sums / max(counts, 1)
// numpy's reduceat along axis 0 evaluates each segment as
//   row[first] + pairwise_sum(rows[first+1 : end])       (per column)
// so this file reproduces it bit-for-bit:
//   1. stable counting sort of the labels (tile histograms -> exclusive scan
//      -> one warp per tile scatters row ids with __match_any_sync ranks);
//   2. the pairwise recursion of every segment is expanded into its <=128-row
//      leaves, one warp per (leaf, 128-column chunk) sums its rows with the
//      8-accumulator leaf rule, rows gathered through the sorted order with
//      fully coalesced 1 KB row reads;
//   3. one warp per (codeword, column chunk) folds the leaf sums back up the
//      same recursion, adds the first row, and divides by the count.
// The result is deterministic (no float atomics) and equal to the reference.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace da {

namespace {
constexpr int GS_TILE = 1024;      // rows per sort tile
constexpr int GS_SMEM_HIST = 12288; // labels that fit a shared-memory histogram
constexpr int GS_COLS = 128;       // columns per warp task (4 per lane)
}  // namespace

__global__ void tile_hist_kernel(const int32_t* __restrict__ labels, long long n, int K, int T,
                                 int32_t* __restrict__ hist) {
    extern __shared__ int32_t sh[];
    const int t = blockIdx.x;
    const long long lo = (long long)t * GS_TILE;
    const long long hi = min(n, lo + GS_TILE);
    const bool use_smem = K <= GS_SMEM_HIST;
    if (use_smem) {
        for (int k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0;
        __syncthreads();
        for (long long r = lo + threadIdx.x; r < hi; r += blockDim.x) atomicAdd(&sh[labels[r]], 1);
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += blockDim.x) hist[(long long)k * T + t] = sh[k];
    } else {
        for (long long r = lo + threadIdx.x; r < hi; r += blockDim.x)
            atomicAdd(&hist[(long long)labels[r] * T + t], 1);
    }
}

// Single-block exclusive scan of len int32 values (in place); out_total gets the sum.
__global__ void exclusive_scan_kernel(int32_t* __restrict__ a, long long len, int32_t* __restrict__ out_total) {
    __shared__ long long warp_sums[32];
    const int nt = blockDim.x;
    const long long chunk = (len + nt - 1) / nt;
    const long long lo = min(len, (long long)threadIdx.x * chunk);
    const long long hi = min(len, lo + chunk);
    long long s = 0;
    for (long long i = lo; i < hi; ++i) s += a[i];
    // block exclusive scan of s
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long incl = s;
    for (int off = 1; off < 32; off <<= 1) {
        long long v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long w = (lane < (nt >> 5)) ? warp_sums[lane] : 0;
        long long wi = w;
        for (int off = 1; off < 32; off <<= 1) {
            long long v = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += v;
        }
        if (lane < (nt >> 5)) warp_sums[lane] = wi - w;
        if (lane == (nt >> 5) - 1 && out_total) *out_total = (int32_t)wi;
    }
    __syncthreads();
    long long run = warp_sums[wid] + incl - s;
    for (long long i = lo; i < hi; ++i) {
        long long v = a[i];
        a[i] = (int32_t)run;
        run += v;
    }
}

__global__ void seg_counts_kernel(const int32_t* __restrict__ offs, int K, int T, long long n,
                                  int32_t* __restrict__ seg_start, int32_t* __restrict__ counts) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    int s = offs[(long long)k * T];
    int e = (k + 1 < K) ? offs[(long long)(k + 1) * T] : (int)n;
    seg_start[k] = s;
    counts[k] = e - s;
}

// One warp per label: exclusive scan of hist[k][0..T) in place; counts[k] = total.
// The last block to finish (threadfence + counter) also writes the segment
// starts seg = exclusive_scan(counts) and *total -- one launch instead of three.
__global__ void label_tile_scan_kernel(int32_t* __restrict__ hist, int K, int T, int32_t* __restrict__ counts,
                                       int32_t* __restrict__ seg, int32_t* __restrict__ total,
                                       unsigned* __restrict__ done) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k < K) {
        int32_t* row = hist + (long long)k * T;
        int carry = 0;
        // 16 chunks of 32 tiles in flight per batch (the loads were the latency chain)
        for (int b0 = 0; b0 < T; b0 += 32 * 16) {
            int v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int t = b0 + 32 * q + lane;
                v[q] = t < T ? row[t] : 0;
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int t = b0 + 32 * q + lane;
                int incl = v[q];
                for (int off = 1; off < 32; off <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += o;
                }
                if (t < T) row[t] = carry + incl - v[q];
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        if (lane == 0) counts[k] = carry;
    }
    if (seg == nullptr) return;
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // block-wide exclusive scan of the K counts (K / blockDim per thread, in order)
    __shared__ int wsum[32];
    const int nt = blockDim.x, per = (K + nt - 1) / nt;
    const int lo = min(K, threadIdx.x * per), hi = min(K, lo + per);
    int sum = 0;
    for (int i = lo; i < hi; ++i) sum += __ldcg(counts + i);
    int incl = sum;
    for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) wsum[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int w = threadIdx.x < (nt >> 5) ? wsum[threadIdx.x] : 0;
        int wi = w;
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += o;
        }
        wsum[threadIdx.x] = wi - w;
        if (threadIdx.x == 31) *total = wi;
    }
    __syncthreads();
    int run = wsum[threadIdx.x >> 5] + incl - sum;
    for (int i = lo; i < hi; ++i) {
        const int v = __ldcg(counts + i);
        seg[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) *done = 0u;   // ready for the next call on this stream
}

// hist[k][t] += seg_start[k] (turns within-label offsets into global cursors)
__global__ void add_seg_start_kernel(int32_t* __restrict__ hist, int K, int T, const int32_t* __restrict__ seg_start) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)K * T) return;
    hist[e] += seg_start[e / T];
}

// One warp per tile: stable scatter of row ids into their label segment.
// Cursors live in shared memory when K fits (GS_SMEM_HIST), else in the
// tile's column of the scanned histogram in global memory.
__global__ void stable_scatter_kernel(const int32_t* __restrict__ labels, long long n, int K, int T,
                                      int32_t* __restrict__ cursor, int32_t* __restrict__ order) {
    extern __shared__ int32_t scur[];
    const int t = blockIdx.x;
    const int lane = threadIdx.x;
    const long long lo = (long long)t * GS_TILE;
    const long long hi = min(n, lo + GS_TILE);
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool sm = K <= GS_SMEM_HIST;
    if (sm) {
        for (int k = lane; k < K; k += 32) scur[k] = cursor[(long long)k * T + t];
        __syncwarp();
    }
    int lab_next = (lo + lane < hi) ? labels[lo + lane] : 0;
    for (long long base = lo; base < hi; base += 32) {
        const long long r = base + lane;
        const bool valid = r < hi;
        const int lab = lab_next;
        lab_next = (r + 32 < hi) ? labels[r + 32] : 0;  // prefetch the next group
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(active, lab);
            const int leader = __ffs(peers) - 1;
            const int rank = __popc(peers & lt_mask);
            int b = 0;
            if (lane == leader) b = sm ? scur[lab] : cursor[(long long)lab * T + t];
            b = __shfl_sync(peers, b, leader);
            order[b + rank] = (int32_t)r;
            if (lane == leader) {
                if (sm) scur[lab] = b + __popc(peers);
                else cursor[(long long)lab * T + t] = b + __popc(peers);
            }
        }
        __syncwarp();
    }
}

// Same stable scatter with four warps per tile: warp w takes rows
// [lo + 256w, lo + 256w + 256); per-warp label counts (shared memory) turn the
// tile cursor into per-warp cursors, so the rows still land in row order.
constexpr int GS_SW = 4;
// Lanes holding the same label (what __match_any_sync returns), built from one
// ballot per label bit: ballots are single cheap instructions, while match.any
// serialises over the distinct values of the warp (the stable scatter issued
// 16 of them per warp per tile and was the slowest bookkeeping kernel).
__device__ __forceinline__ unsigned gs_match(unsigned active, int lab, int nbits) {
    unsigned peers = active;
    for (int b = 0; b < nbits; ++b) {
        const unsigned on = __ballot_sync(active, (lab >> b) & 1);
        peers &= ((lab >> b) & 1) ? on : ~on;
    }
    return peers;
}

__global__ void __launch_bounds__(32 * GS_SW) stable_scatter4_kernel(const int32_t* __restrict__ labels, long long n,
                                                                    int K, int T, const int32_t* __restrict__ cursor,
                                                                    int32_t* __restrict__ order,
                                                                    const int32_t* __restrict__ seg) {
    extern __shared__ int32_t wc[];   // [GS_SW][K]
    const int nbits = 32 - __clz(max(K - 1, 1));
    const int t = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long lo = (long long)t * GS_TILE + (long long)w * (GS_TILE / GS_SW);
    const long long hi = min(n, lo + GS_TILE / GS_SW);
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int k = threadIdx.x; k < GS_SW * K; k += blockDim.x) wc[k] = 0;
    __syncthreads();
    int* my = wc + w * K;
    for (long long base = lo; base < hi; base += 32) {
        const long long r = base + lane;
        const bool valid = r < hi;
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int lab = labels[r];
            const unsigned peers = gs_match(active, lab, nbits);
            if (lane == __ffs(peers) - 1) my[lab] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        int c = cursor[(long long)k * T + t] + (seg ? seg[k] : 0);
#pragma unroll
        for (int q = 0; q < GS_SW; ++q) {
            const int v = wc[q * K + k];
            wc[q * K + k] = c;
            c += v;
        }
    }
    __syncthreads();
    int lab_next = (lo + lane < hi) ? labels[lo + lane] : 0;
    for (long long base = lo; base < hi; base += 32) {
        const long long r = base + lane;
        const bool valid = r < hi;
        const int lab = lab_next;
        lab_next = (r + 32 < hi) ? labels[r + 32] : 0;
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const unsigned peers = gs_match(active, lab, nbits);
            const int leader = __ffs(peers) - 1;
            const int rank = __popc(peers & lt_mask);
            int b = 0;
            if (lane == leader) b = my[lab];
            b = __shfl_sync(peers, b, leader);
            order[b + rank] = (int32_t)r;
            if (lane == leader) my[lab] = b + __popc(peers);
        }
        __syncwarp();
    }
}

// ---- pairwise recursion bookkeeping ----------------------------------------

// The walks below keep their recursion stacks in shared memory (one column per
// thread, conflict-free): in local memory every push and pop was an L1/L2
// round trip, and these kernels are latency chains (13-55 us per call before).
// Depth: the right child of x is at most x/2 + 8, so x < 2^31 reaches a leaf
// (<= 128) within 25 levels.
constexpr int GS_DMAX = 32;
constexpr int GS_RING = 8;       // leaves in flight per seg_finish warp

// 8-byte global -> shared copy (LDGSTS), for the seg_finish leaf ring
__device__ __forceinline__ void gs_cp8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc) : "memory");
}
__device__ __forceinline__ void gs_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void gs_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
constexpr int GS_WALK_T = 128;   // threads per block of the per-codeword walks

__global__ void __launch_bounds__(GS_WALK_T) leaf_count_kernel(const int32_t* __restrict__ counts, int K,
                                                                int32_t* __restrict__ nleaf) {
    __shared__ int st[GS_DMAX][GS_WALK_T];
    const int t = threadIdx.x;
    const int k = blockIdx.x * GS_WALK_T + t;
    if (k >= K) return;
    const int c = counts[k];
    const int m = c >= 2 ? c - 1 : 0;
    int leaves = 0;
    if (m > 0) {
        int sp = 0;
        st[sp++][t] = m;
        while (sp) {
            const int x = st[--sp][t];
            if (x <= 128) { ++leaves; continue; }
            int n2 = x / 2; n2 -= n2 % 8;
            st[sp++][t] = x - n2;
            st[sp++][t] = n2;
        }
    }
    nleaf[k] = leaves;
}

// leaf_count + exclusive scan + leaf_enum in one single-block launch (K <= 512,
// one thread per codeword): count the leaves of pairwise(rest), block scan,
// then enumerate them in left-to-right order.  The second walk needs no offset
// stack: leaves come out contiguous, so a leaf starts where the previous ended.
constexpr int GS_PLAN_MAXK = 512;
__global__ void __launch_bounds__(GS_PLAN_MAXK) leaf_plan_kernel(const int32_t* __restrict__ counts,
                                                                  const int32_t* __restrict__ seg_start, int K,
                                                                  int32_t* __restrict__ leaf_base,
                                                                  int32_t* __restrict__ total_leaves,
                                                                  int4* __restrict__ leaves) {
    extern __shared__ int gs_plan_sh[];
    const int T = blockDim.x;
    int* scan = gs_plan_sh;   // [T]
    int* st = scan + T;       // [GS_DMAX][T]
    const int t = threadIdx.x;
    const int c = t < K ? counts[t] : 0;
    const int m = c >= 2 ? c - 1 : 0;
    int nl = 0;
    if (m > 0) {
        int sp = 0;
        st[(sp++) * T + t] = m;
        while (sp) {
            const int x = st[(--sp) * T + t];
            if (x <= 128) { ++nl; continue; }
            int n2 = x / 2; n2 -= n2 % 8;
            st[(sp++) * T + t] = x - n2;
            st[(sp++) * T + t] = n2;
        }
    }
    scan[t] = nl;
    __syncthreads();
    for (int off = 1; off < T; off <<= 1) {
        const int v = t >= off ? scan[t - off] : 0;
        __syncthreads();
        scan[t] += v;
        __syncthreads();
    }
    const int excl = scan[t] - nl;
    if (t < K) leaf_base[t] = excl;
    if (t == T - 1) *total_leaves = scan[t];
    if (m > 0) {
        int out = excl, lo = 0, sp = 0;
        const int rest0 = seg_start[t] + 1;
        st[(sp++) * T + t] = m;
        while (sp) {
            const int x = st[(--sp) * T + t];
            if (x <= 128) {
                leaves[out] = make_int4(t, rest0 + lo, x, out);
                ++out;
                lo += x;
                continue;
            }
            int n2 = x / 2; n2 -= n2 % 8;
            st[(sp++) * T + t] = x - n2;   // right first, so the left subtree is emitted first
            st[(sp++) * T + t] = n2;
        }
    }
}

// Per codeword: enumerate the leaves of pairwise(rest) in left-to-right order.
__global__ void __launch_bounds__(GS_WALK_T) leaf_enum_kernel(const int32_t* __restrict__ counts,
                                                               const int32_t* __restrict__ seg_start,
                                                               const int32_t* __restrict__ leaf_base, int K,
                                                               int4* __restrict__ leaves) {
    __shared__ int st_lo[GS_DMAX][GS_WALK_T];
    __shared__ int st_n[GS_DMAX][GS_WALK_T];
    const int t = threadIdx.x;
    const int k = blockIdx.x * GS_WALK_T + t;
    if (k >= K) return;
    const int c = counts[k];
    if (c < 2) return;
    int out = leaf_base[k];
    const int rest0 = seg_start[k] + 1;
    int sp = 0;
    st_lo[sp][t] = 0; st_n[sp][t] = c - 1; ++sp;
    while (sp) {
        --sp;
        const int lo = st_lo[sp][t], x = st_n[sp][t];
        if (x <= 128) {
            leaves[out] = make_int4(k, rest0 + lo, x, out);
            ++out;
            continue;
        }
        int n2 = x / 2; n2 -= n2 % 8;
        // push right first so the left leaf is emitted first
        st_lo[sp][t] = lo + n2; st_n[sp][t] = x - n2; ++sp;
        st_lo[sp][t] = lo; st_n[sp][t] = n2; ++sp;
    }
}

// One warp per (leaf, 128-column chunk): numpy pairwise leaf over gathered rows.
// Lane l owns columns {2l, 2l+1, 64+2l, 65+2l} of the chunk (two 16-B loads per
// row); the 8 interleaved accumulators follow the row index mod 8.
__global__ void __launch_bounds__(256, 2) leaf_sum_kernel(const double* __restrict__ X, long long ldx, int D,
                                const int32_t* __restrict__ order, const int4* __restrict__ leaves,
                                const int32_t* __restrict__ n_leaves_total, int n_chunks,
                                double* __restrict__ leaf_sums) {
    const int lane = threadIdx.x & 31;
    const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long total = (long long)(*n_leaves_total) * n_chunks;
    if (task >= total) return;
    const long long leaf = task / n_chunks;
    const int chunk = (int)(task % n_chunks);
    const int4 L = leaves[leaf];
    const int start = L.y, n = L.z;
    const int cbase = chunk * GS_COLS;
    const int cols[4] = {cbase + 2 * lane, cbase + 2 * lane + 1, cbase + 64 + 2 * lane, cbase + 65 + 2 * lane};
    const bool vec = ((ldx & 1) == 0) && (cbase + GS_COLS <= D);  // aligned full chunk: 16-B loads
    auto load_row = [&](long long r, double* out4) {
        const double* p = X + r * ldx;
        if (vec) {
            const double2 a = *reinterpret_cast<const double2*>(p + cols[0]);
            const double2 b = *reinterpret_cast<const double2*>(p + cols[2]);
            out4[0] = a.x; out4[1] = a.y; out4[2] = b.x; out4[3] = b.y;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) out4[q] = cols[q] < D ? p[cols[q]] : 0.0;
        }
    };
    double res[4];
    if (n < 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) res[q] = 0.0;
        for (int i = 0; i < n; ++i) {
            double v[4];
            load_row(order[start + i], v);
#pragma unroll
            for (int q = 0; q < 4; ++q) res[q] = dadd(res[q], v[q]);
        }
    } else {
        double acc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) load_row(order[start + j], acc[j]);
        int i = 8;
        const int stop = n - (n % 8);
        for (; i < stop; i += 8) {
#pragma unroll
            for (int h = 0; h < 8; h += 4) {
                double v[4][4];
#pragma unroll
                for (int j = 0; j < 4; ++j) load_row(order[start + i + h + j], v[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[h + j][q] = dadd(acc[h + j][q], v[j][q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            res[q] = dadd(dadd(dadd(acc[0][q], acc[1][q]), dadd(acc[2][q], acc[3][q])),
                          dadd(dadd(acc[4][q], acc[5][q]), dadd(acc[6][q], acc[7][q])));
        for (; i < n; ++i) {
            double v[4];
            load_row(order[start + i], v);
#pragma unroll
            for (int q = 0; q < 4; ++q) res[q] = dadd(res[q], v[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (cols[q] < D) leaf_sums[(long long)L.w * D + cols[q]] = res[q];
}

// Rows up to D = 128 (DA_GS_NARROW_MAX; wider rows use leaf_sum_kernel): one
// warp per (leaf, 8-column chunk).  The leaf rule's
// 8 interleaved accumulators are independent chains, so each gets its own
// lane: lane = 4*j + p owns accumulator j (rows j, j+8, ... of the leaf) for
// the column pair p.  A lane first loads its <= 16 row ids, then its <= 16
// rows (all independent: the whole leaf is in flight at once instead of one
// 8-row batch per round trip), then runs its chain in row order.  Lane j = 0
// gathers the 8 accumulators with shuffles, combines them in numpy's
// ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) order and adds the n % 8 tail rows in
// sequence: the same per-column operations as the one-lane-per-leaf loop.
constexpr int GS_NARROW_ROWS = 16;   // rows per accumulator chain of a <= 128-row leaf
__global__ void __launch_bounds__(256) leaf_sum_narrow_kernel(const double* __restrict__ X, long long ldx, int D,
                                                              const int32_t* __restrict__ order,
                                                              const int4* __restrict__ leaves,
                                                              const int32_t* __restrict__ n_leaves_total,
                                                              double* __restrict__ leaf_sums) {
    const int lane = threadIdx.x & 31;
    const int n_chunks = (D + 7) >> 3;
    const long long task = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (task >= (long long)(*n_leaves_total) * n_chunks) return;
    const long long leaf = task / n_chunks;
    const int chunk = (int)(task - leaf * n_chunks);
    const int j = lane >> 2, p = lane & 3;
    const int c0 = chunk * 8 + 2 * p, c1 = c0 + 1;
    const int4 L = leaves[leaf];
    const int start = L.y, n = L.z;
    const bool vec = ((ldx & 1) == 0) && (c1 < D) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    auto load_row = [&](long long r, double& v0, double& v1) {
        const double* q = X + r * ldx;
        if (vec) {
            const double2 a = *reinterpret_cast<const double2*>(q + c0);
            v0 = a.x; v1 = a.y;
        } else {
            v0 = c0 < D ? q[c0] : 0.0;
            v1 = c1 < D ? q[c1] : 0.0;
        }
    };
    double r0 = 0.0, r1 = 0.0;
    const int stop = n >= 8 ? n - (n % 8) : 0;
    if (n >= 8) {
        const int cnt = (stop - j + 7) >> 3;   // rows j, j+8, ... < stop (>= 1)
        int ids[GS_NARROW_ROWS];
#pragma unroll
        for (int t = 0; t < GS_NARROW_ROWS; ++t) ids[t] = t < cnt ? order[start + j + 8 * t] : 0;
        double v0[GS_NARROW_ROWS], v1[GS_NARROW_ROWS];
#pragma unroll
        for (int t = 0; t < GS_NARROW_ROWS; ++t) {
            if (t < cnt) load_row(ids[t], v0[t], v1[t]);
            else v0[t] = v1[t] = 0.0;
        }
        double a0 = v0[0], a1 = v1[0];
#pragma unroll
        for (int t = 1; t < GS_NARROW_ROWS; ++t)
            if (t < cnt) { a0 = dadd(a0, v0[t]); a1 = dadd(a1, v1[t]); }
        double g0[8], g1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            g0[q] = __shfl_sync(0xffffffffu, a0, 4 * q + p);
            g1[q] = __shfl_sync(0xffffffffu, a1, 4 * q + p);
        }
        r0 = dadd(dadd(dadd(g0[0], g0[1]), dadd(g0[2], g0[3])), dadd(dadd(g0[4], g0[5]), dadd(g0[6], g0[7])));
        r1 = dadd(dadd(dadd(g1[0], g1[1]), dadd(g1[2], g1[3])), dadd(dadd(g1[4], g1[5]), dadd(g1[6], g1[7])));
    }
    if (j != 0) return;
    // tail (n % 8 rows, or the whole leaf when n < 8): sequential, loads first
    const int tn = n - stop;
    double w0[8], w1[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        if (t < tn) load_row(order[start + stop + t], w0[t], w1[t]);
        else w0[t] = w1[t] = 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (t < tn) { r0 = dadd(r0, w0[t]); r1 = dadd(r1, w1[t]); }
    if (c0 < D) leaf_sums[(long long)L.w * D + c0] = r0;
    if (c1 < D) leaf_sums[(long long)L.w * D + c1] = r1;
}

// One warp (one block) per (codeword, column chunk): fold leaves up the
// recursion tree, prepend the first row, divide by the count.  mode 0 = write
// means into the filled rows of C (empties untouched); mode 1 = write raw sums
// (all rows).  The walk's shape (sizes, states) is warp-uniform and lives in
// shared memory, written by lane 0; each lane's pending left sums live in its
// own shared column.  Leaves are consumed in order, so their sums stream
// through a GS_RING-deep cp.async ring (each lane copies and reads only its
// own columns: no warp barrier needed for the ring).
__global__ void __launch_bounds__(32) seg_finish_kernel(const double* __restrict__ X, long long ldx, int D,
                                                        const int32_t* __restrict__ order,
                                                        const int32_t* __restrict__ counts,
                                                        const int32_t* __restrict__ seg_start,
                                                        const int32_t* __restrict__ leaf_base,
                                                        const int32_t* __restrict__ n_leaves_total,
                                                        const double* __restrict__ leaf_sums, int K, int n_chunks,
                                                        int mode, double* __restrict__ out, long long ldo,
                                                        const double* __restrict__ first_rows = nullptr) {
    __shared__ int s_n[GS_DMAX + 1];
    __shared__ int s_state[GS_DMAX + 1];
    __shared__ double s_left[GS_DMAX][4][32];
    __shared__ double s_ring[GS_RING][4][32];
    const int lane = threadIdx.x & 31;
    const long long task = blockIdx.x;
    if (task >= (long long)K * n_chunks) return;
    const int k = (int)(task / n_chunks);
    const int chunk = (int)(task % n_chunks);
    const int c = counts[k];
    if (c == 0) {
        if (mode == 1) {
            for (int q = 0; q < 4; ++q) {
                int col = chunk * GS_COLS + lane + 32 * q;
                if (col < D) out[(long long)k * ldo + col] = 0.0;
            }
        }
        return;
    }
    double tot[4];
    if (first_rows) {   // sharded: the segment's first row, gathered from the shard holding it
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int col = chunk * GS_COLS + lane + 32 * q;
            tot[q] = (col < D) ? first_rows[(long long)k * D + col] : 0.0;
        }
    } else {
        const long long first = order[seg_start[k]];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int col = chunk * GS_COLS + lane + 32 * q;
            tot[q] = (col < D) ? X[first * ldx + col] : 0.0;
        }
    }
    if (c >= 2) {
        const long long lf0 = leaf_base[k];
        const long long nk = (k + 1 < K ? (long long)leaf_base[k + 1] : (long long)*n_leaves_total) - lf0;
        auto issue = [&](long long j) {
            if (j < nk) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = chunk * GS_COLS + lane + 32 * q;
                    if (col < D) gs_cp8(&s_ring[j % GS_RING][q][lane], leaf_sums + (lf0 + j) * D + col);
                }
            }
            gs_cp_commit();   // one group per leaf, empty past the end: the wait count stays uniform
        };
#pragma unroll
        for (int j = 0; j < GS_RING; ++j) issue(j);
        long long leaf = 0;
        // post-order walk; all lanes follow the same shape
        int sp = 0;
        if (lane == 0) { s_n[0] = c - 1; s_state[0] = 0; }
        __syncwarp();
        double ret[4] = {0.0, 0.0, 0.0, 0.0};
        while (sp >= 0) {
            const int x = s_n[sp];
            if (x <= 128) {
                gs_cp_wait<GS_RING - 1>();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = chunk * GS_COLS + lane + 32 * q;
                    ret[q] = col < D ? s_ring[leaf % GS_RING][q][lane] : 0.0;
                }
                issue(leaf + GS_RING);
                ++leaf;
                --sp;
                while (sp >= 0) {
                    if (s_state[sp] == 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) s_left[sp][q][lane] = ret[q];
                        __syncwarp();
                        if (lane == 0) {
                            int n2 = s_n[sp] / 2; n2 -= n2 % 8;
                            s_state[sp] = 2;
                            s_n[sp + 1] = s_n[sp] - n2;
                            s_state[sp + 1] = 0;
                        }
                        __syncwarp();
                        ++sp;
                        break;
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) ret[q] = dadd(s_left[sp][q][lane], ret[q]);
                        --sp;
                    }
                }
                continue;
            }
            __syncwarp();
            if (lane == 0) {
                int n2 = x / 2; n2 -= n2 % 8;
                s_state[sp] = 1;
                s_n[sp + 1] = n2;
                s_state[sp + 1] = 0;
            }
            __syncwarp();
            ++sp;
        }
        gs_cp_wait<0>();
#pragma unroll
        for (int q = 0; q < 4; ++q) tot[q] = dadd(tot[q], ret[q]);
    }
    const double cnt = (double)c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int col = chunk * GS_COLS + lane + 32 * q;
        if (col < D) out[(long long)k * ldo + col] = (mode == 0) ? __ddiv_rn(tot[q], cnt) : tot[q];
    }
}

// Stable counting sort of the labels: counts[K], seg[K] (segment starts),
// order[n] (row ids in label order, rows in increasing order within a label).
static int gs_stable_sort(const int32_t* labels, long long n, int K, int T, int32_t* hist, int32_t* counts,
                          int32_t* seg, int32_t* total, int32_t* order, cudaStream_t s) {
    const long long KT = (long long)K * T;
    const bool smem_hist = K <= GS_SMEM_HIST;   // tiles write their whole histogram column: no memset
    const bool fast = (size_t)GS_SW * K * sizeof(int32_t) <= 48 * 1024 && K <= 1024;
    if (!smem_hist) DA_CUDA(cudaMemsetAsync(hist, 0, sizeof(int32_t) * (KT + 1), s));
    size_t sh = smem_hist ? sizeof(int32_t) * K : 0;
    tile_hist_kernel<<<T, 256, sh, s>>>(labels, n, K, T, hist);
    DA_CHECK_LAUNCH("tile_hist_kernel");
    if (fast) {
        // tile scan + segment starts in one launch; the scatter adds seg to the tile cursors
        unsigned* done = (unsigned*)scratch(23, 256, s);
        static thread_local void* zeroed = nullptr;   // the kernel leaves the counter at 0 for the next call
        if (!done) return fail_cuda(cudaErrorMemoryAllocation, "label scan counter");
        if (zeroed != done) { DA_CUDA(cudaMemsetAsync(done, 0, 256, s)); zeroed = done; }
        label_tile_scan_kernel<<<grid_for(K, 8), 256, 0, s>>>(hist, K, T, counts, seg, total, done);
        DA_CHECK_LAUNCH("label_tile_scan_kernel");
        stable_scatter4_kernel<<<T, 32 * GS_SW, sizeof(int32_t) * GS_SW * K, s>>>(labels, n, K, T, hist, order, seg);
        DA_CHECK_LAUNCH("stable_scatter4_kernel");
        return 0;
    }
    label_tile_scan_kernel<<<grid_for(K, 8), 256, 0, s>>>(hist, K, T, counts, nullptr, nullptr, nullptr);
    DA_CHECK_LAUNCH("label_tile_scan_kernel");
    DA_CUDA(cudaMemcpyAsync(seg, counts, sizeof(int32_t) * K, cudaMemcpyDeviceToDevice, s));
    exclusive_scan_kernel<<<1, 1024, 0, s>>>(seg, K, total);
    DA_CHECK_LAUNCH("exclusive_scan_kernel(counts)");
    add_seg_start_kernel<<<grid_for(KT, 256, 1LL << 31), 256, 0, s>>>(hist, K, T, seg);
    DA_CHECK_LAUNCH("add_seg_start_kernel");
    if ((size_t)GS_SW * K * sizeof(int32_t) <= 48 * 1024) {
        stable_scatter4_kernel<<<T, 32 * GS_SW, sizeof(int32_t) * GS_SW * K, s>>>(labels, n, K, T, hist, order,
                                                                                   nullptr);
        DA_CHECK_LAUNCH("stable_scatter4_kernel");
    } else {
        stable_scatter_kernel<<<T, 32, sh, s>>>(labels, n, K, T, hist, order);
        DA_CHECK_LAUNCH("stable_scatter_kernel");
    }
    return 0;
}

// Host driver.  X: (n, D) float64 rows (leading dim ldx); labels int32 in [0,K).
// Writes counts[K]; mode 0: out[k] = mean for non-empty k (empty rows untouched);
// mode 1: out[k] = raw sum (0 for empty).
int launch_group_sums(const double* X, long long n, long long ldx, int D, const int32_t* labels, int K,
                      int mode, double* out, long long ldo, int32_t* counts, cudaStream_t s) {
    if (n <= 0 || K <= 0) return 0;
    const int T = (int)((n + GS_TILE - 1) / GS_TILE);
    const long long KT = (long long)K * T;
    const long long max_leaves = K + n / 64 + 2;
    const int n_chunks = (D + GS_COLS - 1) / GS_COLS;
    // scratch layout
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    size_t o_hist = take(sizeof(int32_t) * (KT + 1));
    size_t o_order = take(sizeof(int32_t) * n);
    size_t o_seg = take(sizeof(int32_t) * K);
    size_t o_nleaf = take(sizeof(int32_t) * (K + 1));
    size_t o_total = take(sizeof(int32_t) * 4);
    size_t o_leaves = take(sizeof(int4) * max_leaves);
    size_t o_lsum = take(sizeof(double) * max_leaves * D);
    char* base = (char*)scratch(0, off, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "group_sums scratch");
    int32_t* hist = (int32_t*)(base + o_hist);
    int32_t* order = (int32_t*)(base + o_order);
    int32_t* seg = (int32_t*)(base + o_seg);
    int32_t* nleaf = (int32_t*)(base + o_nleaf);
    int32_t* total = (int32_t*)(base + o_total);
    int4* leaves = (int4*)(base + o_leaves);
    double* lsum = (double*)(base + o_lsum);

    ProfScope ps("group_sums", s);
    {
        const int rc = gs_stable_sort(labels, n, K, T, hist, counts, seg, total, order, s);
        if (rc) return rc;
    }
    if (K <= GS_PLAN_MAXK) {
        int T = 32;
        while (T < K) T <<= 1;
        const size_t psh = sizeof(int) * (size_t)T * (GS_DMAX + 1);
        if (psh > 48 * 1024)
            { const int rc_ = ensure_smem((const void*)leaf_plan_kernel, (int)psh); if (rc_) return rc_; }
        leaf_plan_kernel<<<1, T, psh, s>>>(counts, seg, K, nleaf, total + 1, leaves);
        DA_CHECK_LAUNCH("leaf_plan_kernel");
    } else {
        leaf_count_kernel<<<grid_for(K, GS_WALK_T), GS_WALK_T, 0, s>>>(counts, K, nleaf);
        DA_CHECK_LAUNCH("leaf_count_kernel");
        exclusive_scan_kernel<<<1, 1024, 0, s>>>(nleaf, K, total + 1);
        DA_CHECK_LAUNCH("exclusive_scan_kernel(leaves)");
        leaf_enum_kernel<<<grid_for(K, GS_WALK_T), GS_WALK_T, 0, s>>>(counts, seg, nleaf, K, leaves);
        DA_CHECK_LAUNCH("leaf_enum_kernel");
    }
    {
        long long tasks = max_leaves * n_chunks;
        ProfScope ps3("group_sums_leaf", s);
        static const int narrow_max = getenv("DA_GS_NARROW_MAX") ? atoi(getenv("DA_GS_NARROW_MAX")) : 128;
        if (D <= narrow_max) {
            const long long ntask = max_leaves * ((D + 7) / 8);
            leaf_sum_narrow_kernel<<<grid_for(ntask, 8, 1LL << 31), 256, 0, s>>>(X, ldx, D, order, leaves, total + 1,
                                                                                 lsum);
            DA_CHECK_LAUNCH("leaf_sum_narrow_kernel");
        } else {
            leaf_sum_kernel<<<grid_for(tasks, 8, 1LL << 31), 256, 0, s>>>(X, ldx, D, order, leaves, total + 1,
                                                                          n_chunks, lsum);
            DA_CHECK_LAUNCH("leaf_sum_kernel");
        }
    }
    {
        long long tasks = (long long)K * n_chunks;
        seg_finish_kernel<<<(unsigned)tasks, 32, 0, s>>>(X, ldx, D, order, counts, seg, nleaf, total + 1, lsum, K,
                                                         n_chunks, mode, out, ldo);
        DA_CHECK_LAUNCH("seg_finish_kernel");
    }
    return 0;
}

// Stable argsort of labels only (tests, the reseed path, the A-Tree build's
// LSD radix passes): the same tile-scan counting sort as the Lloyd update.
int launch_label_order(const int32_t* labels, long long n, int K, int32_t* order_out, int32_t* counts,
                       cudaStream_t s) {
    if (n <= 0) return 0;
    const int T = (int)((n + GS_TILE - 1) / GS_TILE);
    const long long KT = (long long)K * T;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    size_t o_hist = take(sizeof(int32_t) * (KT + 1));
    size_t o_seg = take(sizeof(int32_t) * K);
    size_t o_total = take(sizeof(int32_t) * 4);
    char* base = (char*)scratch(1, off, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "label_order scratch");
    return gs_stable_sort(labels, n, K, T, (int32_t*)(base + o_hist), counts, (int32_t*)(base + o_seg),
                          (int32_t*)(base + o_total), order_out, s);
}


// ============================================================================
// Row-sharded Lloyd update with the reference's summation order (bit-identical
// to the one-GPU launch_group_sums over the concatenated shards).
//
// Label k's global segment is the concatenation of every shard's label-k rows
// (shards are rank-ordered, rows in order within a shard), so shard r owns the
// positions [off_k, off_k + c_k) of it, off_k = sum of the counts of shards
// < r.  The pairwise recursion over the segment's rest is a function of the
// global count n_k alone, so every shard enumerates the same leaves.  Leaves
// inside a shard are summed locally with the normal leaf kernels; a leaf cut by
// a shard boundary is a chain of partial leaf states (the 8 interleaved
// accumulators, or the combined sum once the accumulator rows are done) handed
// from shard to shard, W - 1 neighbour rounds (a leaf can cross every shard).
// Leaf sums land in a global leaf-indexed buffer that is -0.0 everywhere this
// shard does not own a leaf (x + -0.0 == x for every x, signed zeros included),
// together with the segments' first rows; one allreduce completes it and every
// shard folds the same tree.  The host side is distributed.py / _engine.py.

namespace {
constexpr int GSS_SLOT = 20;   // scratch slot holding the shard's sort + plan between calls
struct ShardState {
    int32_t* hist; int32_t* order; int32_t* seg; int32_t* total; int32_t* cnt;
    int32_t* goff; int32_t* nleaf; int32_t* leaf_base; int32_t* nlocal; int4* local_leaves;
    int4* itemL; int4* itemR; int32_t* first_pos;
    long long n, cap; int K, T;
};
ShardState g_shard;   // one shard per process and device (the loops call in sequence)

__device__ int gs_count_leaves(int m) {
    if (m <= 0) return 0;
    int st[GS_DMAX], sp = 0, leaves = 0;
    st[sp++] = m;
    while (sp) {
        const int x = st[--sp];
        if (x <= 128) { ++leaves; continue; }
        int n2 = x / 2; n2 -= n2 % 8;
        st[sp++] = x - n2;
        st[sp++] = n2;
    }
    return leaves;
}
}  // namespace

// per label: global count, this shard's offset in the segment, global leaf count
__global__ void shard_label_kernel(const int32_t* __restrict__ cnt_all, int W, int rank, int K,
                                   int32_t* __restrict__ gcount, int32_t* __restrict__ goff,
                                   int32_t* __restrict__ nleaf) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    int n = 0, off = 0;
    for (int r = 0; r < W; ++r) {
        const int c = cnt_all[(long long)r * K + k];
        if (r < rank) off += c;
        n += c;
    }
    gcount[k] = n;
    goff[k] = off;
    nleaf[k] = gs_count_leaves(n >= 2 ? n - 1 : 0);
}

// per label: walk the global leaves of pairwise(rest) left to right and
// classify each against this shard's rest range [ra, rb):
//   inside        -> local leaf (k, local sorted position, length, global index)
//   cut, s > 0    -> itemL[k]: continues a state received from the left
//   cut, s == 0   -> itemR[k]: starts here, its state goes right
// items: (global leaf index, local sorted position of leaf row s, s + 256 e, x);
// a label with no rows here gets itemL = (-2, ...): forward the state as is.
__global__ void shard_enum_kernel(const int32_t* __restrict__ gcount, const int32_t* __restrict__ goff,
                                  const int32_t* __restrict__ cnt, const int32_t* __restrict__ seg,
                                  const int32_t* __restrict__ leaf_base, int K, int4* __restrict__ local_leaves,
                                  int32_t* __restrict__ nlocal, int4* __restrict__ itemL, int4* __restrict__ itemR,
                                  int32_t* __restrict__ first_pos, const int32_t* __restrict__ cnt_all, int rank,
                                  int rounds, double* __restrict__ overflow) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const int n = gcount[k], off = goff[k], c = cnt[k];
    itemL[k] = make_int4(c == 0 ? -2 : -1, 0, 0, 0);
    itemR[k] = make_int4(-1, 0, 0, 0);
    first_pos[k] = (off == 0 && c > 0) ? seg[k] : -1;
    if (c == 0 || n < 2) return;
    // rest index q <-> segment position q + 1
    const int ra = off > 0 ? off - 1 : 0, rb = off - 1 + c;
    if (rb <= ra) return;
    auto lpos = [&](int q) { return seg[k] + (q + 1 - off); };
    int st_lo[GS_DMAX], st_n[GS_DMAX], sp = 0;
    st_lo[sp] = 0; st_n[sp] = n - 1; ++sp;
    int idx = leaf_base[k];
    while (sp) {
        --sp;
        const int lo = st_lo[sp], x = st_n[sp];
        if (x <= 128) {
            const int gi = idx++;
            if (lo + x <= ra || lo >= rb) continue;
            if (lo >= ra && lo + x <= rb) {
                const int slot = atomicAdd(nlocal, 1);
                local_leaves[slot] = make_int4(k, lpos(lo), x, gi);
            } else {
                const int s = max(ra, lo) - lo, e = min(rb, lo + x) - lo;
                const int4 it = make_int4(gi, lpos(lo + s), s + 256 * e, x);
                if (s > 0) {
                    itemL[k] = it;
                    // shards this leaf's state crosses before reaching us: more than `rounds`
                    // neighbour exchanges -> the update is redone with world - 1 rounds
                    if (overflow) {
                        int r = rank, o = off;                  // segment position of our first row
                        while (r > 0 && o > lo + 1) { --r; o -= cnt_all[(long long)r * K + k]; }
                        if (rank - r > rounds) atomicAdd(overflow, 1.0);
                    }
                } else {
                    itemR[k] = it;
                }
            }
            continue;
        }
        int n2 = x / 2; n2 -= n2 % 8;
        st_lo[sp] = lo + n2; st_n[sp] = x - n2; ++sp;
        st_lo[sp] = lo; st_n[sp] = n2; ++sp;
    }
}

__global__ void fill_neg_zero_kernel(double* __restrict__ a, long long len) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
        a[i] = -0.0;
}

__global__ void shard_first_rows_kernel(const double* __restrict__ X, long long ldx, int d, int K,
                                        const int32_t* __restrict__ order, const int32_t* __restrict__ first_pos,
                                        double* __restrict__ out) {
    const int k = blockIdx.x;
    const int fp = first_pos[k];
    if (fp < 0) return;
    const long long row = order[fp];
    for (int c = threadIdx.x; c < d; c += blockDim.x) out[(long long)k * d + c] = X[row * ldx + c];
}

// One warp per label: run the leaf rule over this shard's rows [s, e) of a cut
// leaf, continuing the received state when s > 0.  State layout [K][8][d]:
// the 8 accumulators while e < x8 (rows of the 8-way part), else the combined
// running sum in slot 0.  e == x: the finished leaf sum goes to red.
__global__ void shard_edge_kernel(const double* __restrict__ X, long long ldx, int d, int K,
                                  const int32_t* __restrict__ order, const int4* __restrict__ items, int want_cont,
                                  const double* __restrict__ recv, double* __restrict__ send,
                                  double* __restrict__ red) {
    const int lane = threadIdx.x & 31;
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= K) return;
    const int4 it = items[k];
    const long long sb = (long long)k * 8 * d;
    if (it.x == -2) {                        // no rows of this label here: forward the state
        if (want_cont)
            for (int e = lane; e < 8 * d; e += 32) send[sb + e] = recv[sb + e];
        return;
    }
    if (it.x < 0) return;
    const int s = it.z & 255, e = it.z >> 8, x = it.w;
    if ((s > 0) != (want_cont != 0)) return;
    const int x8 = x >= 8 ? x - (x % 8) : 0;
    for (int c = lane; c < d; c += 32) {
        double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double res = 0.0;
        if (s > 0) {
            if (s < x8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = recv[sb + (long long)j * d + c];
            } else {
                res = recv[sb + c];
            }
        }
        for (int i = s; i < e; ++i) {
            const double v = X[(long long)order[it.y + (i - s)] * ldx + c];
            if (i < x8) {
                acc[i & 7] = i < 8 ? v : dadd(acc[i & 7], v);
                if (i == x8 - 1)
                    res = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])),
                               dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
            } else {
                res = dadd(res, v);
            }
        }
        if (e == x) {
            red[(long long)it.x * d + c] = res;
        } else if (e < x8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) send[sb + (long long)j * d + c] = acc[j];
        } else {
            send[sb + c] = res;
        }
    }
}

int launch_gs_shard_sort(const double* X, long long n, long long ldx, int d, const int32_t* labels, int K,
                         int32_t* counts_local, cudaStream_t s) {
    (void)X; (void)ldx; (void)d;
    ShardState& S = g_shard;
    S.n = n; S.K = K;
    S.T = (int)std::max(1LL, (n + GS_TILE - 1) / GS_TILE);
    const long long KT = (long long)K * S.T;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    const size_t o_hist = take(sizeof(int32_t) * (KT + 1)), o_order = take(sizeof(int32_t) * std::max(1LL, n));
    const size_t o_seg = take(sizeof(int32_t) * K), o_total = take(sizeof(int32_t) * 4);
    const size_t o_cnt = take(sizeof(int32_t) * K), o_goff = take(sizeof(int32_t) * K);
    const size_t o_nleaf = take(sizeof(int32_t) * (K + 1)), o_base = take(sizeof(int32_t) * (K + 1));
    const size_t o_il = take(sizeof(int4) * K), o_ir = take(sizeof(int4) * K), o_fp = take(sizeof(int32_t) * K);
    const size_t o_ll = take(0);   // local leaves: sized in the plan (needs the global row count)
    char* base = (char*)scratch(GSS_SLOT, off, s);
    if (!base) return fail_cuda(cudaErrorMemoryAllocation, "shard group sums scratch");
    S.hist = (int32_t*)(base + o_hist); S.order = (int32_t*)(base + o_order); S.seg = (int32_t*)(base + o_seg);
    S.total = (int32_t*)(base + o_total); S.cnt = (int32_t*)(base + o_cnt); S.goff = (int32_t*)(base + o_goff);
    S.nleaf = (int32_t*)(base + o_nleaf); S.leaf_base = (int32_t*)(base + o_base);
    S.itemL = (int4*)(base + o_il); S.itemR = (int4*)(base + o_ir); S.first_pos = (int32_t*)(base + o_fp);
    S.nlocal = S.total + 2;
    (void)o_ll;
    ProfScope ps("group_sums", s);
    if (n == 0) {
        DA_CUDA(cudaMemsetAsync(S.cnt, 0, sizeof(int32_t) * K, s));
        DA_CUDA(cudaMemsetAsync(S.seg, 0, sizeof(int32_t) * K, s));
    } else {
        const int rc = gs_stable_sort(labels, n, K, S.T, S.hist, S.cnt, S.seg, S.total, S.order, s);
        if (rc) return rc;
    }
    if (counts_local != S.cnt)
        DA_CUDA(cudaMemcpyAsync(counts_local, S.cnt, sizeof(int32_t) * K, cudaMemcpyDeviceToDevice, s));
    return 0;
}

int launch_gs_shard_plan(const double* X, long long n, long long ldx, int d, int K, const int32_t* cnt_all, int W,
                         int rank, long long cap, double* red, double* send, int32_t* gcount, int rounds,
                         double* overflow, cudaStream_t s) {
    ShardState& S = g_shard;
    if (S.K != K || S.n != n) return fail_arg("shard plan: call da_gs_shard_sort on the same rows first");
    S.cap = cap;
    int4* ll = (int4*)scratch(GSS_SLOT + 1, sizeof(int4) * (size_t)cap, s);
    if (!ll) return fail_cuda(cudaErrorMemoryAllocation, "shard leaf list");
    S.local_leaves = ll;
    ProfScope ps("group_sums", s);
    shard_label_kernel<<<grid_for(K, 128), 128, 0, s>>>(cnt_all, W, rank, K, gcount, S.goff, S.nleaf);
    DA_CHECK_LAUNCH("shard_label_kernel");
    DA_CUDA(cudaMemcpyAsync(S.leaf_base, S.nleaf, sizeof(int32_t) * K, cudaMemcpyDeviceToDevice, s));
    exclusive_scan_kernel<<<1, 1024, 0, s>>>(S.leaf_base, K, S.total + 1);
    DA_CHECK_LAUNCH("exclusive_scan_kernel(shard leaves)");
    DA_CUDA(cudaMemsetAsync(S.nlocal, 0, sizeof(int32_t), s));
    shard_enum_kernel<<<grid_for(K, 128), 128, 0, s>>>(gcount, S.goff, S.cnt, S.seg, S.leaf_base, K, ll, S.nlocal,
                                                       S.itemL, S.itemR, S.first_pos, cnt_all, rank, rounds, overflow);
    DA_CHECK_LAUNCH("shard_enum_kernel");
    const long long len = cap * d + (long long)K * d;
    fill_neg_zero_kernel<<<grid_for(len, 256, 4096), 256, 0, s>>>(red, len);
    DA_CHECK_LAUNCH("fill_neg_zero_kernel");
    if (n > 0) {
        ProfScope ps3("group_sums_leaf", s);
        static const int narrow_max = getenv("DA_GS_NARROW_MAX") ? atoi(getenv("DA_GS_NARROW_MAX")) : 128;
        const long long maxl = std::min(cap, n / 1 + 1);
        if (d <= narrow_max) {
            const long long ntask = maxl * ((d + 7) / 8);
            leaf_sum_narrow_kernel<<<grid_for(ntask, 8, 1LL << 31), 256, 0, s>>>(X, ldx, d, S.order, ll, S.nlocal, red);
            DA_CHECK_LAUNCH("leaf_sum_narrow_kernel");
        } else {
            const int n_chunks = (d + GS_COLS - 1) / GS_COLS;
            leaf_sum_kernel<<<grid_for(maxl * n_chunks, 8, 1LL << 31), 256, 0, s>>>(X, ldx, d, S.order, ll, S.nlocal,
                                                                                   n_chunks, red);
            DA_CHECK_LAUNCH("leaf_sum_kernel");
        }
        shard_first_rows_kernel<<<K, 128, 0, s>>>(X, ldx, d, K, S.order, S.first_pos, red + cap * d);
        DA_CHECK_LAUNCH("shard_first_rows_kernel");
        // round 0: the cut leaves that start here
        shard_edge_kernel<<<grid_for(K, 8), 256, 0, s>>>(X, ldx, d, K, S.order, S.itemR, 0, nullptr, send, red);
        DA_CHECK_LAUNCH("shard_edge_kernel(start)");
    }
    return 0;
}

int launch_gs_shard_round(const double* X, long long ldx, int d, int K, const double* recv, double* send, double* red,
                          cudaStream_t s) {
    ShardState& S = g_shard;
    if (S.K != K) return fail_arg("shard round: no plan for K=%d", K);
    ProfScope ps("group_sums", s);
    shard_edge_kernel<<<grid_for(K, 8), 256, 0, s>>>(X, ldx, d, K, S.order, S.itemL, 1, recv, send, red);
    DA_CHECK_LAUNCH("shard_edge_kernel(continue)");
    return 0;
}

int launch_gs_shard_fold(int d, int K, const double* red, long long cap, const int32_t* gcount, int mode, double* out,
                         long long ldo, cudaStream_t s) {
    ShardState& S = g_shard;
    if (S.K != K || S.cap != cap) return fail_arg("shard fold: no plan for K=%d cap=%lld", K, cap);
    ProfScope ps("group_sums", s);
    const int n_chunks = (d + GS_COLS - 1) / GS_COLS;
    seg_finish_kernel<<<(unsigned)((long long)K * n_chunks), 32, 0, s>>>(
        nullptr, 0, d, nullptr, gcount, nullptr, S.leaf_base, S.total + 1, red, K, n_chunks, mode, out, ldo,
        red + cap * d);
    DA_CHECK_LAUNCH("seg_finish_kernel(shard)");
    return 0;
}

}  // namespace da

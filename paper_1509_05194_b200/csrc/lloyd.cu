// One Lloyd iteration as few host calls (annq/clustering.py:185-202): the loop
// bodies of _engine._lloyd / _lloyd_sharded issued from C++ instead of a dozen
// Python-side tensor ops, so the host stays ahead of the device even when a
// shard's iteration is short (a 1/8 shard of config B: ~150 us on the GPU).
//
//   da_lloyd_step     one GPU: C_out = C_prev, group means (reduceat order),
//                     #empty clusters, assign against C_out (labels, changed,
//                     optional d2), flags -> pinned host memory, event;
//   da_lloyd_prepare  shards, before the sums: C_out = C_prev (+ snapshot), the
//                     previous assign's [rows changed, 0] into the reduced
//                     buffer's stats slot;
//   da_lloyd_finish   shards, after the allreduce: means of the fast mode
//                     (sums / counts, IEEE division, empties untouched), flags
//                     [#empty, rows changed, error sum, exchange overflow] -> pinned host + event,
//                     then the assign against the new centroids.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/da_b200.h"
#include "common.cuh"
#include "internal.h"

namespace da {

// flags[0] = 0 (the assign counts changed rows into it), flags[1] = #empty clusters
__global__ void lloyd_empty_kernel(const int32_t* __restrict__ counts, int K, unsigned long long* __restrict__ flags) {
    __shared__ int tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    int e = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) e += counts[k] == 0;
    for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, e);
    __syncthreads();
    if (threadIdx.x == 0) {
        flags[0] = 0ULL;
        flags[1] = (unsigned long long)tot;
    }
}

// red stats slot <- [rows changed by the previous assign, 0 (error sum), 0 (exchange overflow)]
__global__ void lloyd_stats_kernel(const unsigned long long* __restrict__ changed, double* __restrict__ stats) {
    stats[0] = changed ? (double)*changed : 0.0;
    stats[1] = 0.0;
    stats[2] = 0.0;
}

// fast sharded mode: red = [sums (K, d) | counts (K) | ...]: C[k, :d] = sums / counts where counts > 0
__global__ void lloyd_means_kernel(const double* __restrict__ red, int K, int d, double* __restrict__ C, long long ldc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)K * d) return;
    const int k = (int)(e / d), c = (int)(e - (long long)k * d);
    const double cnt = red[(long long)K * d + k];
    if (cnt > 0.0) C[(long long)k * ldc + c] = __ddiv_rn(red[e], cnt);
}

// flags = [#empty, stats[0], stats[1]]; counts either int32 (exact) or the f64 slot of red (fast)
__global__ void lloyd_shard_flags_kernel(const int32_t* __restrict__ counts_i, const double* __restrict__ counts_d,
                                         int K, const double* __restrict__ stats, double* __restrict__ flags,
                                         unsigned long long* __restrict__ changed) {
    __shared__ int tot;
    if (threadIdx.x == 0) tot = 0;
    __syncthreads();
    int e = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) e += counts_i ? counts_i[k] == 0 : counts_d[k] == 0.0;
    for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(&tot, e);
    __syncthreads();
    if (threadIdx.x == 0) {
        flags[0] = (double)tot;
        flags[1] = stats[0];
        flags[2] = stats[1];
        flags[3] = stats[2];
        if (changed) *changed = 0ULL;
    }
}

static int assign_against(const double* X, long long n, long long ldx, int d, int K, const double* C, long long ldc,
                          const double* xx, const int32_t* prev, int32_t* labels, double* d2,
                          unsigned long long* changed, cudaStream_t s) {
    if (n <= 0) return 0;
    double* cc = (double*)scratch(21, sizeof(double) * (size_t)K, s);
    if (!cc) return fail_cuda(cudaErrorMemoryAllocation, "lloyd cc scratch");
    int rc = launch_row_sqnorms(C, 0, K, ldc, d, cc, s);
    if (rc) return rc;
    return launch_assign(X, 0, n, ldx, d, C, ldc, K, cc, xx, labels, d2, prev, changed, s);
}

// ---------------------------------------------------------------------------
// CUDA graphs of one Lloyd iteration.  A 1/8 shard's iteration is ~20 launches
// of a few microseconds each; issued one by one the host falls behind the
// device (29 % idle at 125k rows).  Every distinct argument set of
// da_lloyd_step runs eagerly the first time (scratch warm-up), is captured the
// second time and replayed from then on.  Graphs point into library scratch,
// so any scratch reallocation drops them all (g_scratch_gen).  Off while the
// per-kernel profiler runs (its events would be captured).
extern std::atomic<long long> g_scratch_gen;
int assign_image_key(const void** img, long long* mode);

namespace {
struct GKey {
    uintptr_t v[20];
    bool operator==(const GKey& o) const { return std::memcmp(v, o.v, sizeof(v)) == 0; }
};
struct GKeyHash {
    size_t operator()(const GKey& k) const {
        size_t h = 1469598103934665603ull;
        for (uintptr_t x : k.v) { h ^= (size_t)x; h *= 1099511628211ull; }
        return h;
    }
};
struct GEntry {
    cudaGraphExec_t exec = nullptr;
    int seen = 0;
    long long kernels = 0;
    long long gen = -1;
};
std::unordered_map<GKey, GEntry, GKeyHash> g_graphs;
long long g_gstat[4] = {0, 0, 0, 0};   // eager, captured, replayed, capture failures
std::mutex g_graph_mu;
int g_graph_mode = -1;   // -1: from DA_LLOYD_GRAPHS (default on)

bool graphs_on() {
    if (g_graph_mode < 0) {
        const char* e = getenv("DA_LLOYD_GRAPHS");
        g_graph_mode = e ? (atoi(e) != 0) : 1;
    }
    return g_graph_mode == 1 && !prof_enabled();
}

void drop_graphs_locked() {
    for (auto& kv : g_graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    g_graphs.clear();
}
}  // namespace

int drop_lloyd_graphs() {
    std::lock_guard<std::mutex> g(g_graph_mu);
    drop_graphs_locked();
    return 0;
}

}  // namespace da

using namespace da;

extern "C" {

int da_lloyd_graph_stats(long long* out) {
    for (int i = 0; i < 4; ++i) out[i] = g_gstat[i];
    return 0;
}

int da_lloyd_graphs(int on) {
    std::lock_guard<std::mutex> g(g_graph_mu);
    g_graph_mode = on ? 1 : 0;
    if (!on) drop_graphs_locked();
    return 0;
}

static int lloyd_step_body(const double* X, int64_t n, int64_t ldx, int d, int K, const double* C_prev, double* C_out,
                           int64_t ldc, double* snap, const int32_t* labels_prev, int32_t* labels_out, double* d2_out,
                           const double* xx, int32_t* counts, unsigned long long* flags_dev, void* flags_host,
                           cudaStream_t s) {
    const size_t cbytes = sizeof(double) * (size_t)K * (size_t)ldc;
    if (snap) DA_CUDA(cudaMemcpyAsync(snap, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (C_out != C_prev) DA_CUDA(cudaMemcpyAsync(C_out, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    int rc = launch_group_sums(X, n, ldx, d, labels_prev, K, 0, C_out, ldc, counts, s);
    if (rc) return rc;
    lloyd_empty_kernel<<<1, 256, 0, s>>>(counts, K, flags_dev);
    DA_CHECK_LAUNCH("lloyd_empty_kernel");
    rc = assign_against(X, n, ldx, d, K, C_out, ldc, xx, labels_prev, labels_out, d2_out, flags_dev, s);
    if (rc) return rc;
    if (flags_host)
        DA_CUDA(cudaMemcpyAsync(flags_host, flags_dev, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    return 0;
}

int da_lloyd_step(const double* X, int64_t n, int64_t ldx, int d, int K, const double* C_prev, double* C_out,
                  int64_t ldc, double* snap, const int32_t* labels_prev, int32_t* labels_out, double* d2_out,
                  const double* xx, int32_t* counts, unsigned long long* flags_dev, void* flags_host, void* event,
                  void* stream) {
    if (n < 1 || K < 1 || d < 1 || ldx < d || ldc < d || !counts || !flags_dev)
        return fail_arg("lloyd_step: bad arguments n=%lld K=%d d=%d", (long long)n, K, d);
    cudaStream_t s = (cudaStream_t)stream;
    auto body = [&]() {
        return lloyd_step_body(X, n, ldx, d, K, C_prev, C_out, ldc, snap, labels_prev, labels_out, d2_out, xx, counts,
                               flags_dev, flags_host, s);
    };
    // captures are recorded on a private stream (the caller's may be the legacy
    // default stream, which cannot capture); the graph is then launched on `s`
    auto body_cap = [&](cudaStream_t cs) {
        return lloyd_step_body(X, n, ldx, d, K, C_prev, C_out, ldc, snap, labels_prev, labels_out, d2_out, xx, counts,
                               flags_dev, flags_host, cs);
    };
    int rc = 0;
    if (graphs_on()) {
        const void* img = nullptr;
        long long amode = 0;
        assign_image_key(&img, &amode);
        GKey key{{(uintptr_t)X, (uintptr_t)n, (uintptr_t)ldx, (uintptr_t)d, (uintptr_t)K, (uintptr_t)C_prev,
                  (uintptr_t)C_out, (uintptr_t)ldc, (uintptr_t)snap, (uintptr_t)labels_prev, (uintptr_t)labels_out,
                  (uintptr_t)d2_out, (uintptr_t)xx, (uintptr_t)counts, (uintptr_t)flags_dev, (uintptr_t)flags_host,
                  (uintptr_t)s, (uintptr_t)img, (uintptr_t)amode, 0}};
        std::unique_lock<std::mutex> g(g_graph_mu);
        const long long gen = g_scratch_gen.load();
        GEntry& e = g_graphs[key];
        if (e.gen != gen) {               // scratch moved since this graph was captured
            if (e.exec) cudaGraphExecDestroy(e.exec);
            e = GEntry{};
            e.gen = gen;
        }
        if (e.exec) {
            ++g_gstat[2];
            DA_CUDA(cudaGraphLaunch(e.exec, s));
            count_launches(e.kernels);
        } else if (e.seen >= 1) {
            if (g_graphs.size() > 4096) drop_graphs_locked();
            GEntry& f = g_graphs[key];
            f.gen = gen;
            const long long k0 = launch_total();
            cudaGraph_t graph = nullptr;
            static thread_local cudaStream_t cap = nullptr;
            if (!cap) cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
            cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
            const cudaError_t be = cap ? cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal)
                                       : cudaErrorStreamCaptureUnsupported;
            int brc = 0;
            cudaError_t ce = be;
            if (be == cudaSuccess) {
                brc = body_cap(cap);
                ce = cudaStreamEndCapture(cap, &graph);
            }
            if (cap && cudaStreamIsCapturing(cap, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
                cudaGraph_t g2 = nullptr;           // never leave the capture stream capturing
                cudaStreamEndCapture(cap, &g2);
                if (g2) cudaGraphDestroy(g2);
                ce = cudaErrorStreamCaptureInvalidated;
            }
            if (brc == 0 && ce == cudaSuccess && graph && g_scratch_gen.load() == gen &&
                cudaGraphInstantiate(&f.exec, graph, 0) == cudaSuccess) {
                f.kernels = launch_total() - k0;
                ++g_gstat[1];
                cudaGraphDestroy(graph);
                DA_CUDA(cudaGraphLaunch(f.exec, s));
            } else {
                // capture failed (or scratch moved inside it): run eagerly, never capture this key again
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();
                if (getenv("DA_DEBUG"))
                    fprintf(stderr, "[da] lloyd graph capture failed (begin %d, body %d, end %d, d %d, n %lld, last %s): eager\n",
                            (int)be, brc, (int)ce, d, (long long)n, da_last_error());
                f.exec = nullptr;
                f.seen = -1000000;
                ++g_gstat[3];
                rc = body();
            }
        } else {
            ++e.seen;
            ++g_gstat[0];
            g.unlock();
            rc = body();
        }
    } else {
        rc = body();
    }
    if (rc) return rc;
    if (event) DA_CUDA(cudaEventRecord((cudaEvent_t)event, s));
    return 0;
}

int da_lloyd_prepare(const double* C_prev, double* C_out, double* snap, int64_t elems,
                     const unsigned long long* changed_prev, double* stats, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const size_t cbytes = sizeof(double) * (size_t)elems;
    if (snap) DA_CUDA(cudaMemcpyAsync(snap, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (C_out != C_prev) DA_CUDA(cudaMemcpyAsync(C_out, C_prev, cbytes, cudaMemcpyDeviceToDevice, s));
    if (stats) {
        lloyd_stats_kernel<<<1, 1, 0, s>>>(changed_prev, stats);
        DA_CHECK_LAUNCH("lloyd_stats_kernel");
    }
    return 0;
}

int da_lloyd_finish(int fast, const double* red, const int32_t* counts, int K, int d, double* C, int64_t ldc,
                    const double* stats, double* flags_dev, void* flags_host, void* event, const double* X,
                    int64_t n, int64_t ldx, const double* xx, const int32_t* labels_prev, int32_t* labels_out,
                    double* d2_out, unsigned long long* changed, void* stream) {
    if (K < 1 || d < 1 || ldc < d || !flags_dev || !stats) return fail_arg("lloyd_finish: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (fast) {
        lloyd_means_kernel<<<grid_for((long long)K * d, 256), 256, 0, s>>>(red, K, d, C, ldc);
        DA_CHECK_LAUNCH("lloyd_means_kernel");
    }
    lloyd_shard_flags_kernel<<<1, 256, 0, s>>>(fast ? nullptr : counts, fast ? red + (long long)K * d : nullptr, K,
                                               stats, flags_dev, changed);
    DA_CHECK_LAUNCH("lloyd_shard_flags_kernel");
    if (flags_host) DA_CUDA(cudaMemcpyAsync(flags_host, flags_dev, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (event) DA_CUDA(cudaEventRecord((cudaEvent_t)event, s));
    if (labels_out)
        return assign_against(X, n, ldx, d, K, C, ldc, xx, labels_prev, labels_out, d2_out, changed, s);
    return 0;
}

}  // extern "C"

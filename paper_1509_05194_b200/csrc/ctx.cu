// Library context (SURVEY 8(b) minimum ABI): the devices a caller works on,
// one library-owned stream per device, and -- for a row shard -- an NCCL
// communicator, so a non-Python host can run the sharded reductions through
// the C ABI alone (the Python engine uses torch.distributed instead).
//
// NCCL is bound at run time (dlopen of libnccl.so.2, the library torch already
// loads): libda_b200.so keeps no link-time NCCL dependency, and a context
// without a communicator never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/da_b200.h"
#include "common.cuh"
#include "internal.h"

namespace da {

int drop_lloyd_graphs();

namespace {
// the slice of nccl.h this file uses (values from NCCL 2.x: stable ABI)
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclSum = 0;
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(void*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, const void* /* by value, 128 B */, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    if (g_nccl.h) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))sym("ncclGetUniqueId");
    // ncclCommInitRank takes the 128-byte id by value: call through a matching signature
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))sym("ncclCommInitRank");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))sym("ncclCommDestroy");
    g_nccl.allReduce = (decltype(g_nccl.allReduce))sym("ncclAllReduce");
    g_nccl.allGather = (decltype(g_nccl.allGather))sym("ncclAllGather");
    g_nccl.send = (decltype(g_nccl.send))sym("ncclSend");
    g_nccl.recv = (decltype(g_nccl.recv))sym("ncclRecv");
    g_nccl.groupStart = (decltype(g_nccl.groupStart))sym("ncclGroupStart");
    g_nccl.groupEnd = (decltype(g_nccl.groupEnd))sym("ncclGroupEnd");
    g_nccl.errorString = (decltype(g_nccl.errorString))sym("ncclGetErrorString");
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.commDestroy || !g_nccl.allReduce ||
        !g_nccl.allGather || !g_nccl.send || !g_nccl.recv || !g_nccl.groupStart || !g_nccl.groupEnd)
        return false;
    g_nccl.h = h;
    return true;
}

struct UniqueId { char b[128]; };
typedef ncclResult_t (*InitByValue)(ncclComm_t*, int, UniqueId, int);

int nccl_fail(ncclResult_t r, const char* where) {
    return fail_arg("%s: NCCL error %d (%s)", where, r, g_nccl.errorString ? g_nccl.errorString(r) : "?");
}
}  // namespace

struct Ctx {
    std::vector<int> devices;
    std::vector<cudaStream_t> streams;
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

}  // namespace da

using namespace da;

extern "C" {

int da_ctx_create(int n_devices, const int* device_ids, void** ctx) {
    if (!ctx || n_devices < 1 || !device_ids) return fail_arg("ctx_create: need at least one device");
    int count = 0;
    DA_CUDA(cudaGetDeviceCount(&count));
    Ctx* c = new Ctx();
    int prev = 0;
    cudaGetDevice(&prev);
    for (int i = 0; i < n_devices; ++i) {
        if (device_ids[i] < 0 || device_ids[i] >= count) {
            delete c;
            return fail_arg("ctx_create: device %d of %d", device_ids[i], count);
        }
        cudaStream_t s = nullptr;
        cudaSetDevice(device_ids[i]);
        const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            for (cudaStream_t t : c->streams) cudaStreamDestroy(t);
            delete c;
            cudaSetDevice(prev);
            return fail_cuda(e, "ctx_create: cudaStreamCreate");
        }
        c->devices.push_back(device_ids[i]);
        c->streams.push_back(s);
    }
    cudaSetDevice(prev);
    *ctx = c;
    return 0;
}

int da_ctx_stream(void* ctx, int i, void** stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || i < 0 || i >= (int)c->streams.size() || !stream) return fail_arg("ctx_stream: bad index %d", i);
    *stream = c->streams[i];
    return 0;
}

int da_nccl_unique_id(void* out128) {
    if (!out128) return fail_arg("nccl_unique_id: null buffer");
    if (!load_nccl()) return fail_arg("nccl_unique_id: libnccl.so.2 not loadable");
    const ncclResult_t r = g_nccl.getUniqueId(out128);
    return r ? nccl_fail(r, "ncclGetUniqueId") : 0;
}

int da_ctx_nccl_init(void* ctx, int rank, int world, const void* id128) {
    Ctx* c = (Ctx*)ctx;
    if (!c || world < 1 || rank < 0 || rank >= world || !id128) return fail_arg("ctx_nccl_init: bad arguments");
    if (c->comm) return fail_arg("ctx_nccl_init: the context already has a communicator");
    if (!load_nccl()) return fail_arg("ctx_nccl_init: libnccl.so.2 not loadable");
    UniqueId id;
    std::memcpy(id.b, id128, 128);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->devices[0]);
    const ncclResult_t r = ((InitByValue)g_nccl.commInitRank)(&c->comm, world, id, rank);
    cudaSetDevice(prev);
    if (r) {
        c->comm = nullptr;
        return nccl_fail(r, "ncclCommInitRank");
    }
    c->rank = rank;
    c->world = world;
    return 0;
}

// In-place sums over the context's communicator (the Lloyd update's reduced
// buffer), an allgather of int32 counts, and the right shift of the exact
// shard exchange (send to rank + 1, receive from rank - 1).
int da_ctx_allreduce_f64(void* ctx, double* buf, int64_t count, void* stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !c->comm) return fail_arg("ctx_allreduce: no communicator (da_ctx_nccl_init)");
    const ncclResult_t r = g_nccl.allReduce(buf, buf, (size_t)count, kNcclFloat64, kNcclSum, c->comm,
                                            stream ? (cudaStream_t)stream : c->streams[0]);
    return r ? nccl_fail(r, "ncclAllReduce") : 0;
}

int da_ctx_allgather_i32(void* ctx, const int32_t* send, int32_t* recv, int64_t count, void* stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !c->comm) return fail_arg("ctx_allgather: no communicator (da_ctx_nccl_init)");
    const ncclResult_t r = g_nccl.allGather(send, recv, (size_t)count, kNcclInt32, c->comm,
                                            stream ? (cudaStream_t)stream : c->streams[0]);
    return r ? nccl_fail(r, "ncclAllGather") : 0;
}

int da_ctx_shift_f64(void* ctx, const double* send, double* recv, int64_t count, void* stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !c->comm) return fail_arg("ctx_shift: no communicator (da_ctx_nccl_init)");
    cudaStream_t s = stream ? (cudaStream_t)stream : c->streams[0];
    ncclResult_t r = g_nccl.groupStart();
    if (!r && c->rank + 1 < c->world) r = g_nccl.send(send, (size_t)count, kNcclFloat64, c->rank + 1, c->comm, s);
    if (!r && c->rank > 0) r = g_nccl.recv(recv, (size_t)count, kNcclFloat64, c->rank - 1, c->comm, s);
    const ncclResult_t r2 = g_nccl.groupEnd();
    if (r) return nccl_fail(r, "ncclSend/ncclRecv");
    return r2 ? nccl_fail(r2, "ncclGroupEnd") : 0;
}

int da_ctx_destroy(void* ctx) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return 0;
    int prev = 0;
    cudaGetDevice(&prev);
    for (size_t i = 0; i < c->streams.size(); ++i) {
        cudaSetDevice(c->devices[i]);
        cudaStreamSynchronize(c->streams[i]);
        cudaStreamDestroy(c->streams[i]);
    }
    cudaSetDevice(prev);
    if (c->comm) g_nccl.commDestroy(c->comm);
    delete c;
    drop_lloyd_graphs();   // graphs may reference the context's work; scratch stays for reuse
    return 0;
}

}  // extern "C"

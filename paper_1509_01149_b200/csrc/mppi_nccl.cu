// mppi_nccl.cu — the cross-rank reductions of the K-sharded step (SURVEY §8.5, row e) driven by
// the library: MIN of the int64 (cost, k) key after the rollouts, SUM of [eta, A] after the local
// weighted-noise sums, both ncclAllReduce on the context stream between the kernels -- or, with
// the one-collective combine (default), one ncclAllGather of every rank's [key, eta, A] record.
//
// NCCL is resolved at run time from the libnccl.so.2 the process already loaded (torch's copy,
// 2.28) so the library never links a second NCCL; nccl.h is used for the types only.
#include <dlfcn.h>
#include <string.h>

#include <cstdarg>
#include <cstdio>

#include "mppi_internal.h"
#include "nccl.h"

namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclCommGetAsyncError) async_error = nullptr;   // optional
    bool ok = false;
};

const NcclApi& api() {
    static NcclApi a = [] {
        NcclApi r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.get_unique_id = (decltype(r.get_unique_id))dlsym(h, "ncclGetUniqueId");
        r.comm_init_rank = (decltype(r.comm_init_rank))dlsym(h, "ncclCommInitRank");
        r.all_reduce = (decltype(r.all_reduce))dlsym(h, "ncclAllReduce");
        r.all_gather = (decltype(r.all_gather))dlsym(h, "ncclAllGather");
        r.comm_destroy = (decltype(r.comm_destroy))dlsym(h, "ncclCommDestroy");
        r.error_string = (decltype(r.error_string))dlsym(h, "ncclGetErrorString");
        r.async_error = (decltype(r.async_error))dlsym(h, "ncclCommGetAsyncError");
        r.ok = r.get_unique_id && r.comm_init_rank && r.all_reduce && r.all_gather && r.comm_destroy && r.error_string;
        return r;
    }();
    return a;
}

}  // namespace

namespace mppi {

bool nccl_available() { return api().ok; }

int nccl_unique_id(unsigned char* out) {
    if (!api().ok) return -1;
    ncclUniqueId id;
    const ncclResult_t r = api().get_unique_id(&id);
    if (r != ncclSuccess) return (int)r;
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return 0;
}

int nccl_attach(Ctx& c, const unsigned char* id_bytes) {
    if (!api().ok) return -1;
    ncclUniqueId id;
    memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = api().comm_init_rank(&comm, c.world, id, c.rank);
    if (r != ncclSuccess) return (int)r;
    c.nccl = comm;
    return 0;
}

void nccl_detach(Ctx& c) {
    if (c.nccl && api().ok) api().comm_destroy((ncclComm_t)c.nccl);
    c.nccl = nullptr;
}

// an asynchronous communicator error (a failed peer, a network fault) as an NCCL result code; 0
// while the communicator is healthy or when the symbol is unavailable
int nccl_async_error(Ctx& c) {
    if (!c.nccl || !api().ok || !api().async_error) return 0;
    ncclResult_t r = ncclSuccess;
    if (api().async_error((ncclComm_t)c.nccl, &r) != ncclSuccess) return 0;
    return (r == ncclSuccess || r == ncclInProgress) ? 0 : (int)r;
}

const char* nccl_error(int r) { return api().ok && r > 0 ? api().error_string((ncclResult_t)r) : "NCCL unavailable"; }

// global minimum of the int64 (ord32(S) << 32 | k) key, in place
int nccl_min_key(Ctx& c, long long* key) {
    return (int)api().all_reduce(key, key, 1, ncclInt64, ncclMin, (ncclComm_t)c.nccl, c.stream);
}

// element-wise minimum of fp32 values over ranks, in place (per-t cost-to-go minima)
int nccl_min_f32(Ctx& c, float* buf, size_t count) {
    return (int)api().all_reduce(buf, buf, count, ncclFloat32, ncclMin, (ncclComm_t)c.nccl, c.stream);
}

// sum of [eta, A[0..T*m)] over ranks, in place
int nccl_sum_buf(Ctx& c, float* buf, size_t count) {
    return (int)api().all_reduce(buf, buf, count, ncclFloat32, ncclSum, (ncclComm_t)c.nccl, c.stream);
}

// every rank's record, concatenated in rank order (the one-collective combine)
int nccl_all_gather(Ctx& c, const float* send, float* recv, size_t count) {
    return (int)api().all_gather(send, recv, count, ncclFloat32, (ncclComm_t)c.nccl, c.stream);
}

int nccl_sum_f64(Ctx& c, double* buf, size_t count) {
    return (int)api().all_reduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)c.nccl, c.stream);
}

}  // namespace mppi

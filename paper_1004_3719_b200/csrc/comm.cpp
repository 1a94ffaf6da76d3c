// Communicators of the distributed sequence (SURVEY §8 rows b, e):
// NCCL over NVLink / NVSwitch for one process per GPU, and an in-process
// "local" group (ranks = host threads sharing one device) whose collectives
// are device copies, so the multi-rank path can be exercised on one GPU.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy a process such
// as PyTorch already loaded if any, else the system one), so the library has
// no link-time NCCL dependency and FFSPMV_ERR_NCCL reports a missing or
// failing NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ffspmv.h"
#include "comm.hpp"

namespace ffspmv {

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char *n) { return dlsym(h, n); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommSplit = (decltype(api.CommSplit))sym("ncclCommSplit");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommSplit && api.AllGather && api.CommDestroy &&
                 api.GetErrorString;
        if (!api.ok) api.err = "libnccl.so.2 lacks ncclCommSplit / ncclAllGather (NCCL >= 2.18 needed)";
    });
    return api;
}

// ------------------------------------------------------------ local group --
// Ranks are host threads on one device.  Every collective is synchronous:
// each rank drains its stream, the ranks meet at a barrier, each copies the
// peers' chunks into its own buffer, and they meet again.
struct LocalGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<const void *> send;
    std::vector<int> colors;
    std::map<int, std::shared_ptr<LocalGroup>> children;

    explicit LocalGroup(int size) : n(size), send(size, nullptr), colors(size, 0) {}

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t gen = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

}  // namespace

struct CommImpl {
    int kind = 0;                          // 1 NCCL, 2 local
    int nranks = 1, rank = 0;
    ncclComm_t nccl_comm = nullptr;
    std::shared_ptr<LocalGroup> local;
};

int comm_size(const CommImpl *c) { return c->nranks; }
int comm_rank(const CommImpl *c) { return c->rank; }

int comm_allgather(CommImpl *c, const void *send, void *recv, size_t bytes, void *stream,
                   std::string &err) {
    cudaStream_t st = (cudaStream_t)stream;
    if (c->kind == 1) {
        const NcclApi &api = nccl();
        ncclResult_t r = api.AllGather(send, recv, bytes, ncclUint8, c->nccl_comm, st);
        if (r != ncclSuccess) {
            err = std::string("ncclAllGather: ") + api.GetErrorString(r);
            return -1;
        }
        return 0;
    }
    LocalGroup &g = *c->local;
    int e = (int)cudaStreamSynchronize(st);
    if (e) { err = "local all-gather: stream"; return e; }
    {
        std::lock_guard<std::mutex> lk(g.mu);
        g.send[c->rank] = send;
    }
    g.barrier();
    // the copies run on the rank's own stream and are drained before the
    // second barrier: a device-to-device cudaMemcpy may return before the
    // copy completes, and neither this rank's next kernel (on `st`) nor a
    // peer overwriting its send buffer may overlap it
    for (int q = 0; q < g.n; ++q) {
        char *dst = (char *)recv + (size_t)q * bytes;
        if (g.send[q] == dst || !bytes) continue;
        if ((e = (int)cudaMemcpyAsync(dst, g.send[q], bytes, cudaMemcpyDeviceToDevice, st))) {
            err = "local all-gather: copy";
            break;
        }
    }
    if (!e && (e = (int)cudaStreamSynchronize(st))) err = "local all-gather: copy";
    g.barrier();
    return e;
}

CommImpl *comm_split(CommImpl *c, int color, int key, int nranks, int rank, std::string &err) {
    auto *out = new CommImpl();
    out->nranks = nranks;
    out->rank = rank;
    if (c->kind == 1) {
        const NcclApi &api = nccl();
        ncclResult_t r = api.CommSplit(c->nccl_comm, color, key, &out->nccl_comm, nullptr);
        if (r != ncclSuccess) {
            err = std::string("ncclCommSplit: ") + api.GetErrorString(r);
            delete out;
            return nullptr;
        }
        out->kind = 1;
        return out;
    }
    // local: the members of a color share one child group, created by the
    // first of them to arrive and kept alive by the members' references
    LocalGroup &g = *c->local;
    {
        std::lock_guard<std::mutex> lk(g.mu);
        g.colors[c->rank] = color;
    }
    g.barrier();
    {
        std::lock_guard<std::mutex> lk(g.mu);
        auto &child = g.children[color];
        if (!child) child = std::make_shared<LocalGroup>(nranks);
        out->kind = 2;
        out->local = child;
    }
    g.barrier();
    {
        std::lock_guard<std::mutex> lk(g.mu);
        g.children.erase(color);
    }
    (void)key;
    return out;
}

void comm_free(CommImpl *c) {
    if (!c) return;
    if (c->kind == 1 && c->nccl_comm) nccl().CommDestroy(c->nccl_comm);
    delete c;
}

}  // namespace ffspmv

using namespace ffspmv;

struct ffspmv_comm_s {
    CommImpl *impl;
};

namespace ffspmv {
CommImpl *comm_impl(ffspmv_comm c) { return c ? c->impl : nullptr; }
}  // namespace ffspmv

extern "C" {

ffspmv_status ffspmv_comm_unique_id(void *id_out) {
    if (!id_out) return set_error(FFSPMV_ERR_INVALID_ARG, "NULL id");
    const NcclApi &api = nccl();
    if (!api.ok) return set_error(FFSPMV_ERR_NCCL, api.err);
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return set_error(FFSPMV_ERR_NCCL, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
    std::memcpy(id_out, &id, sizeof(id));
    return FFSPMV_OK;
}

ffspmv_status ffspmv_comm_create(ffspmv_comm *out, const void *id, int nranks, int rank) {
    if (!out || !id) return set_error(FFSPMV_ERR_INVALID_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(FFSPMV_ERR_INVALID_ARG, "bad nranks / rank");
    const NcclApi &api = nccl();
    if (!api.ok) return set_error(FFSPMV_ERR_NCCL, api.err);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto *impl = new CommImpl();
    impl->kind = 1;
    impl->nranks = nranks;
    impl->rank = rank;
    ncclResult_t r = api.CommInitRank(&impl->nccl_comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete impl;
        return set_error(FFSPMV_ERR_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
    }
    *out = new ffspmv_comm_s{impl};
    return FFSPMV_OK;
}

ffspmv_status ffspmv_comm_create_local(ffspmv_comm *out, int nranks) {
    if (!out || nranks < 1) return set_error(FFSPMV_ERR_INVALID_ARG, "NULL out or nranks < 1");
    auto g = std::make_shared<LocalGroup>(nranks);
    for (int r = 0; r < nranks; ++r) {
        auto *impl = new CommImpl();
        impl->kind = 2;
        impl->nranks = nranks;
        impl->rank = r;
        impl->local = g;
        out[r] = new ffspmv_comm_s{impl};
    }
    return FFSPMV_OK;
}

ffspmv_status ffspmv_comm_destroy(ffspmv_comm c) {
    if (!c) return set_error(FFSPMV_ERR_INVALID_ARG, "NULL communicator");
    comm_free(c->impl);
    delete c;
    return FFSPMV_OK;
}

}  // extern "C"

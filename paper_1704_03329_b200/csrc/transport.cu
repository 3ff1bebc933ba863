// transport.cu -- NCCL (dlopen) and in-process loopback transports for the z-slab ranks.
#include "transport.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

namespace ljmd {

// ------------------------------------------------------------------------------- NCCL
namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api(std::string& err) {
    static NcclApi api;
    static std::once_flag once;
    static std::string load_err;
    std::call_once(once, [] {
        // reuse the libnccl torch already mapped (one NCCL per process), else load one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = getenv("LJMD_NCCL_LIB");
            if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            load_err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
#define LJMD_SYM(field, name)                                                      \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));            \
    if (!api.field) {                                                              \
        load_err = std::string("dlsym ") + name + " failed";                       \
        return;                                                                    \
    }
        LJMD_SYM(CommInitRank, "ncclCommInitRank");
        LJMD_SYM(CommDestroy, "ncclCommDestroy");
        LJMD_SYM(GroupStart, "ncclGroupStart");
        LJMD_SYM(GroupEnd, "ncclGroupEnd");
        LJMD_SYM(Send, "ncclSend");
        LJMD_SYM(Recv, "ncclRecv");
        LJMD_SYM(AllReduce, "ncclAllReduce");
        LJMD_SYM(GetErrorString, "ncclGetErrorString");
#undef LJMD_SYM
        api.ok = true;
    });
    if (!api.ok) err = load_err;
    return api;
}

class NcclTransport : public Transport {
public:
    NcclTransport(NcclApi& api, ncclComm_t comm) : api_(api), comm_(comm) {}
    ~NcclTransport() override {
        if (comm_) api_.CommDestroy(comm_);
    }
    bool exchange(cudaStream_t stream, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                  std::string& err) override {
        ncclResult_t r = api_.GroupStart();
        for (const Xfer& x : sends)
            if (r == ncclSuccess && x.bytes) r = api_.Send(x.ptr, x.bytes, ncclUint8, x.peer, comm_, stream);
        for (const Xfer& x : recvs)
            if (r == ncclSuccess && x.bytes) r = api_.Recv(x.ptr, x.bytes, ncclUint8, x.peer, comm_, stream);
        ncclResult_t r2 = api_.GroupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) err = std::string("NCCL p2p: ") + api_.GetErrorString(r);
        return r == ncclSuccess;
    }
    bool allreduce(cudaStream_t stream, double* dbuf, int n, bool max, std::string& err) override {
        ncclResult_t r = api_.AllReduce(dbuf, dbuf, (size_t)n, ncclFloat64, max ? ncclMax : ncclSum, comm_, stream);
        if (r != ncclSuccess) err = std::string("ncclAllReduce: ") + api_.GetErrorString(r);
        return r == ncclSuccess;
    }
    const char* name() const override { return "nccl"; }

private:
    NcclApi& api_;
    ncclComm_t comm_;
};

// ------------------------------------------------------------------------------- local loopback
struct LocalGroup {
    std::mutex m;
    std::condition_variable cv;
    int n = 0, arrived = 0;
    long long gen = 0;
    std::vector<std::vector<Xfer>> posts;
    std::vector<cudaEvent_t> ready;    // per rank: its send buffers are filled
    std::vector<cudaEvent_t> done;     // per rank: its receive copies are complete
    std::vector<std::vector<double>> red;
    int members = 0;

    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

std::mutex g_groups_m;
std::map<std::string, std::shared_ptr<LocalGroup>> g_groups;

class LocalTransport : public Transport {
public:
    LocalTransport(std::shared_ptr<LocalGroup> g, std::string key, int rank) : g_(g), key_(key), rank_(rank) {
        cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done_, cudaEventDisableTiming);
        std::lock_guard<std::mutex> lk(g_->m);
        g_->ready[rank] = ready_;
        g_->done[rank] = done_;
    }
    ~LocalTransport() override {
        cudaEventDestroy(ready_);
        cudaEventDestroy(done_);
        std::lock_guard<std::mutex> lk(g_groups_m);
        if (--g_->members == 0) g_groups.erase(key_);
    }
    bool exchange(cudaStream_t stream, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                  std::string& err) override {
        cudaEventRecord(ready_, stream);
        {
            std::lock_guard<std::mutex> lk(g_->m);
            g_->posts[rank_] = sends;
        }
        g_->barrier();
        std::map<int, int> seen;   // k-th recv from peer q matches q's k-th send to me
        bool ok = true;
        for (const Xfer& r : recvs) {
            const int k = seen[r.peer]++;
            const Xfer* s = nullptr;
            int c = 0;
            for (const Xfer& x : g_->posts[r.peer])
                if (x.peer == rank_ && c++ == k) {
                    s = &x;
                    break;
                }
            if (!s || s->bytes != r.bytes) {
                err = "local transport: unmatched or size-mismatched transfer";
                ok = false;
                continue;
            }
            if (!r.bytes) continue;
            cudaStreamWaitEvent(stream, g_->ready[r.peer], 0);
            if (cudaMemcpyAsync(r.ptr, s->ptr, r.bytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess) {
                err = "local transport: cudaMemcpyAsync failed";
                ok = false;
            }
        }
        cudaEventRecord(done_, stream);
        g_->barrier();
        for (const Xfer& s : sends) cudaStreamWaitEvent(stream, g_->done[s.peer], 0);
        g_->barrier();
        return ok;
    }
    bool allreduce(cudaStream_t stream, double* dbuf, int n, bool max, std::string& err) override {
        std::vector<double> h(n);
        if (cudaMemcpyAsync(h.data(), dbuf, sizeof(double) * n, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
            cudaStreamSynchronize(stream) != cudaSuccess) {
            err = "local transport: allreduce copy failed";
            return false;
        }
        {
            std::lock_guard<std::mutex> lk(g_->m);
            g_->red[rank_] = h;
        }
        g_->barrier();
        std::vector<double> acc = g_->red[0];   // fixed rank order: deterministic
        for (int r = 1; r < g_->n; ++r)
            for (int i = 0; i < n; ++i) acc[i] = max ? std::max(acc[i], g_->red[r][i]) : acc[i] + g_->red[r][i];
        g_->barrier();
        if (cudaMemcpyAsync(dbuf, acc.data(), sizeof(double) * n, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
            cudaStreamSynchronize(stream) != cudaSuccess) {
            err = "local transport: allreduce write-back failed";
            return false;
        }
        return true;
    }
    const char* name() const override { return "local"; }

private:
    std::shared_ptr<LocalGroup> g_;
    std::string key_;
    int rank_;
    cudaEvent_t ready_ = nullptr, done_ = nullptr;
};

}  // namespace

Transport* make_transport(const void* nccl_id, int rank, int nranks, int device, std::string& err) {
    (void)device;
    if (!nccl_id) {
        err = "nranks > 1 needs options.nccl_id (128-byte ncclUniqueId, or an LJMDLOCAL id)";
        return nullptr;
    }
    const char* id = static_cast<const char*>(nccl_id);
    if (std::strncmp(id, "LJMDLOCAL", 9) == 0) {
        std::string key(id, strnlen(id, 128));
        std::shared_ptr<LocalGroup> g;
        {
            std::lock_guard<std::mutex> lk(g_groups_m);
            auto it = g_groups.find(key);
            if (it == g_groups.end()) {
                g = std::make_shared<LocalGroup>();
                g->n = nranks;
                g->posts.resize(nranks);
                g->ready.resize(nranks);
                g->done.resize(nranks);
                g->red.resize(nranks);
                g_groups[key] = g;
            } else {
                g = it->second;
                if (g->n != nranks) {
                    err = "local transport: nranks mismatch within a group";
                    return nullptr;
                }
            }
            ++g->members;
        }
        return new LocalTransport(g, key, rank);
    }
    NcclApi& api = nccl_api(err);
    if (!api.ok) return nullptr;
    ncclUniqueId uid;
    std::memcpy(&uid, nccl_id, sizeof uid);
    ncclComm_t comm = nullptr;
    ncclResult_t r = api.CommInitRank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
        return nullptr;
    }
    return new NcclTransport(api, comm);
}

bool nccl_unique_id(void* out, std::string& err) {
    NcclApi& api = nccl_api(err);
    if (!api.ok) return false;
    static ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
    if (!get_id) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) get_id = reinterpret_cast<ncclResult_t (*)(ncclUniqueId*)>(dlsym(h, "ncclGetUniqueId"));
    }
    if (!get_id) {
        err = "ncclGetUniqueId not found";
        return false;
    }
    ncclUniqueId id;
    ncclResult_t r = get_id(&id);
    if (r != ncclSuccess) {
        err = std::string("ncclGetUniqueId: ") + api.GetErrorString(r);
        return false;
    }
    std::memcpy(out, &id, sizeof id);
    return true;
}

}  // namespace ljmd

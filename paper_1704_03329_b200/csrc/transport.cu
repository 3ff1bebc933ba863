// transport.cu -- NCCL (dlopen) and in-process loopback transports for the z-slab ranks.
#include "transport.h"

#include <dlfcn.h>
#include <nccl.h>

#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cctype>
#include <cstring>
#include <thread>
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


// ------------------------------------------------------------------------------- host-staged files
// Several PROCESSES on one GPU (NCCL refuses two ranks on one device): every transfer is
// staged through host memory as a file in a directory under /dev/shm shared by the ranks,
// named (call sequence, src, dst, index) and unlinked by its reader; an all-reduce is an
// all-to-all of the vectors reduced in rank order on every rank (deterministic, equal
// everywhere).  Synchronous on the host: a correctness path for the multi-process flow
// (bench.py under torchrun with LJMD_BENCH_DEVICE), not a fast one.
class ShmTransport : public Transport {
public:
    ShmTransport(std::string dir, int rank, int nranks) : dir_(std::move(dir)), rank_(rank), n_(nranks) {
        mkdir(dir_.c_str(), 0700);
    }
    ~ShmTransport() override { rmdir(dir_.c_str()); }   // the last rank out removes it
    bool exchange(cudaStream_t stream, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                  std::string& err) override {
        const long long seq = ++seq_;
        if (cudaStreamSynchronize(stream) != cudaSuccess) return fail(err, "stream sync");
        std::map<int, int> ks;
        for (const Xfer& x : sends)
            if (!post(stream, 'x', seq, rank_, x.peer, ks[x.peer]++, x.ptr, x.bytes, err)) return false;
        std::map<int, int> kr;
        for (const Xfer& x : recvs)
            if (!take(stream, 'x', seq, x.peer, rank_, kr[x.peer]++, x.ptr, x.bytes, err)) return false;
        return true;
    }
    bool allreduce(cudaStream_t stream, double* dbuf, int n, bool max, std::string& err) override {
        const long long seq = ++seq_;
        std::vector<double> mine(n), acc, other(n);
        if (cudaMemcpyAsync(mine.data(), dbuf, sizeof(double) * n, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
            cudaStreamSynchronize(stream) != cudaSuccess)
            return fail(err, "allreduce D2H");
        for (int q = 0; q < n_; ++q)
            if (q != rank_ && !write_file(name('r', seq, rank_, q, 0), mine.data(), sizeof(double) * n, err))
                return false;
        for (int q = 0; q < n_; ++q) {   // rank order: every rank sums in the same order
            const double* v = mine.data();
            if (q != rank_) {
                if (!read_file(name('r', seq, q, rank_, 0), other.data(), sizeof(double) * n, err)) return false;
                v = other.data();
            }
            if (q == 0) acc.assign(v, v + n);
            else
                for (int i = 0; i < n; ++i) acc[i] = max ? std::max(acc[i], v[i]) : acc[i] + v[i];
        }
        if (cudaMemcpyAsync(dbuf, acc.data(), sizeof(double) * n, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
            cudaStreamSynchronize(stream) != cudaSuccess)
            return fail(err, "allreduce H2D");
        return true;
    }
    const char* name() const override { return "shm"; }

private:
    static bool fail(std::string& err, const char* what) {
        err = std::string("shm transport: ") + what + " failed";
        return false;
    }
    std::string name(char ch, long long seq, int src, int dst, int k) const {
        char b[96];
        std::snprintf(b, sizeof b, "/%c%lld_%d_%d_%d", ch, seq, src, dst, k);
        return dir_ + b;
    }
    bool write_file(const std::string& path, const void* p, size_t bytes, std::string& err) {
        const std::string tmp = path + ".tmp";
        FILE* f = std::fopen(tmp.c_str(), "wb");
        if (!f || (bytes && std::fwrite(p, 1, bytes, f) != bytes) || std::fclose(f) != 0 ||
            std::rename(tmp.c_str(), path.c_str()) != 0) {
            err = "shm transport: cannot write " + path;
            return false;
        }
        return true;
    }
    bool read_file(const std::string& path, void* p, size_t bytes, std::string& err) {
        const auto t0 = std::chrono::steady_clock::now();
        struct stat st;
        while (stat(path.c_str(), &st) != 0) {   // the writer renames a complete file into place
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
                err = "shm transport: timed out waiting for " + path;
                return false;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
        if ((size_t)st.st_size != bytes) {
            err = "shm transport: size mismatch on " + path;
            return false;
        }
        FILE* f = std::fopen(path.c_str(), "rb");
        const bool ok = f && (!bytes || std::fread(p, 1, bytes, f) == bytes);
        if (f) std::fclose(f);
        std::remove(path.c_str());
        if (!ok) err = "shm transport: cannot read " + path;
        return ok;
    }
    bool post(cudaStream_t stream, char ch, long long seq, int src, int dst, int k, const void* dptr, size_t bytes,
              std::string& err) {
        buf_.resize(bytes);
        if (bytes && (cudaMemcpyAsync(buf_.data(), dptr, bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
                      cudaStreamSynchronize(stream) != cudaSuccess))
            return fail(err, "D2H");
        return write_file(name(ch, seq, src, dst, k), buf_.data(), bytes, err);
    }
    bool take(cudaStream_t stream, char ch, long long seq, int src, int dst, int k, void* dptr, size_t bytes,
              std::string& err) {
        buf_.resize(bytes);
        if (!read_file(name(ch, seq, src, dst, k), buf_.data(), bytes, err)) return false;
        if (bytes && (cudaMemcpyAsync(dptr, buf_.data(), bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
                      cudaStreamSynchronize(stream) != cudaSuccess))
            return fail(err, "H2D");
        return true;
    }
    std::string dir_;
    int rank_, n_;
    long long seq_ = 0;
    std::vector<unsigned char> buf_;
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
    if (std::strncmp(id, "LJMDSHM:", 8) == 0) {   // processes on one device (tests, bench debug)
        std::string key(id + 8, strnlen(id + 8, 120));
        for (char& ch : key)
            if (!std::isalnum((unsigned char)ch)) ch = '_';
        struct stat st;
        const std::string root = stat("/dev/shm", &st) == 0 ? "/dev/shm" : "/tmp";
        return new ShmTransport(root + "/ljmd_" + key, rank, nranks);
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

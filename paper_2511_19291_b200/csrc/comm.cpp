// comm.cpp -- NCCL transport and the in-process loopback transport (comm.h).
#include "comm.h"

#include <nccl.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace tqd {

static const char kLoopMagic[8] = {'T', 'Q', 'D', 'L', 'O', 'O', 'P', '1'};

bool comm_is_loopback_id(const void *id128) { return id128 && memcmp(id128, kLoopMagic, 8) == 0; }

void comm_make_loopback_id(void *id128) {
    static std::atomic<uint64_t> counter{1};
    const uint64_t t = (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
    const uint64_t key = (counter++ << 40) ^ ((uint64_t)getpid() << 20) ^ t;
    memset(id128, 0, 128);
    memcpy(id128, kLoopMagic, 8);
    memcpy((char *)id128 + 8, &key, 8);
}

// ---------------------------------------------------------------- NCCL
class NcclComm : public Comm {
  public:
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (flag) cudaFree(flag);
        if (c) ncclCommDestroy(c);
    }
    int check(ncclResult_t r, const char *what) {
        if (r == ncclSuccess) return 0;
        err = std::string(what) + ": " + ncclGetErrorString(r);
        return 1;
    }
    int group_start() override { return check(ncclGroupStart(), "ncclGroupStart"); }
    int send(const void *buf, size_t bytes, int peer, cudaStream_t s) override {
        return check(ncclSend(buf, bytes, ncclUint8, peer, c, s), "ncclSend");
    }
    int recv(void *buf, size_t bytes, int peer, cudaStream_t s) override {
        return check(ncclRecv(buf, bytes, ncclUint8, peer, c, s), "ncclRecv");
    }
    int group_end(cudaStream_t) override { return check(ncclGroupEnd(), "ncclGroupEnd"); }
    int allreduce_sum(void *buf, size_t count, CommElem t, cudaStream_t s) override {
        return check(ncclAllReduce(buf, buf, count, t == CE_F64 ? ncclDouble : ncclFloat, ncclSum, c, s),
                     "ncclAllReduce");
    }
    int cuda(cudaError_t e, const char *what) {
        if (e == cudaSuccess) return 0;
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return 1;
    }
    // Collective.  Returns 0 (table filled), 1 (communication error) or 2 (CUDA IPC
    // is unavailable on some rank: every rank gets 2 and the caller falls back to
    // pack -> all-to-all -> unpack).  IPC failures never skip a collective.
    int share_buffers(void *const *local, int nbuf, std::vector<void *> &table, cudaStream_t s) override {
        const size_t hs = sizeof(cudaIpcMemHandle_t);
        std::vector<char> mine(nbuf * hs, 0), all((size_t)world * nbuf * hs);
        int ok = 1;
        for (int i = 0; i < nbuf && ok; i++)
            if (cudaIpcGetMemHandle((cudaIpcMemHandle_t *)(mine.data() + i * hs), local[i]) != cudaSuccess) {
                cudaGetLastError();
                ok = 0;
            }
        char *d = nullptr;
        if (cuda(cudaMalloc(&d, all.size() + mine.size() + sizeof(int)), "cudaMalloc")) return 1;
        int rc = cuda(cudaMemcpyAsync(d, mine.data(), mine.size(), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
        if (!rc) rc = check(ncclAllGather(d, d + mine.size(), mine.size(), ncclUint8, c, s), "ncclAllGather");
        if (!rc) rc = cuda(cudaMemcpyAsync(all.data(), d + mine.size(), all.size(), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
        if (!rc) rc = cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        table.assign((size_t)world * nbuf, nullptr);
        for (int r = 0; r < world && !rc; r++)
            for (int i = 0; i < nbuf; i++) {
                if (r == rank) { table[r * nbuf + i] = local[i]; continue; }
                if (!ok) continue;
                cudaIpcMemHandle_t hdl;
                memcpy(&hdl, all.data() + ((size_t)r * nbuf + i) * hs, hs);
                if (cudaIpcOpenMemHandle(&table[r * nbuf + i], hdl, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    table[r * nbuf + i] = nullptr;
                    ok = 0;
                }
            }
        // every rank learns whether all ranks opened every peer buffer
        int *dok = reinterpret_cast<int *>(d + all.size() + mine.size());
        if (!rc) rc = cuda(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
        if (!rc) rc = check(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c, s), "ncclAllReduce");
        if (!rc) rc = cuda(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
        if (!rc) rc = cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        cudaFree(d);
        if (rc) return rc;
        if (!ok) {
            release_buffers(table, nbuf);
            return 2;
        }
        return 0;
    }
    void release_buffers(std::vector<void *> &table, int nbuf) override {
        for (int r = 0; r < world; r++)
            for (int i = 0; i < nbuf && (size_t)(r * nbuf + i) < table.size(); i++)
                if (r != rank && table[r * nbuf + i]) cudaIpcCloseMemHandle(table[r * nbuf + i]);
        table.clear();
    }
    int barrier(cudaStream_t s) override {
        if (!flag && cuda(cudaMalloc(&flag, sizeof(int)), "cudaMalloc")) return 1;
        if (check(ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, c, s), "ncclAllReduce")) return 1;
        return cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    int *flag = nullptr;
};

// ---------------------------------------------------------------- loopback
struct Hub {
    int world = 0, refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    struct Post {
        int dst;
        const void *ptr;
        size_t bytes;
    };
    std::vector<std::vector<Post>> sends;  // per source rank, current group
    std::vector<void *> bufs;              // per rank, current reduction
    std::vector<std::vector<void *>> shared;  // per rank, share_buffers
    // all ranks arrive; false on timeout (a rank died or diverged)
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return true;
        }
        return cv.wait_for(lk, std::chrono::seconds(60), [&] { return gen != g; });
    }
};

static std::mutex g_hubs_mu;
static std::map<uint64_t, Hub *> g_hubs;

class LoopComm : public Comm {
  public:
    Hub *hub = nullptr;
    uint64_t key = 0;
    struct Req {
        void *ptr;
        size_t bytes;
        int peer;
    };
    std::vector<Hub::Post> psend;
    std::vector<Req> precv;

    ~LoopComm() override {
        std::lock_guard<std::mutex> g(g_hubs_mu);
        if (hub && --hub->refs == 0) {
            g_hubs.erase(key);
            delete hub;
        }
    }
    int cuda(cudaError_t e, const char *what) {
        if (e == cudaSuccess) return 0;
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return 1;
    }
    int sync_all(const char *what) {
        if (hub->barrier()) return 0;
        err = std::string("loopback barrier timed out in ") + what;
        return 1;
    }
    int group_start() override {
        psend.clear();
        precv.clear();
        return 0;
    }
    int send(const void *buf, size_t bytes, int peer, cudaStream_t) override {
        psend.push_back({peer, buf, bytes});
        return 0;
    }
    int recv(void *buf, size_t bytes, int peer, cudaStream_t) override {
        precv.push_back({buf, bytes, peer});
        return 0;
    }
    int group_end(cudaStream_t s) override {
        // the send buffers are valid once the work queued before the group is done
        if (cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize")) return 1;
        {
            std::lock_guard<std::mutex> g(hub->mu);
            hub->sends[rank] = psend;
        }
        if (sync_all("group_end (post)")) return 1;
        std::vector<int> used(world, 0);
        for (const Req &r : precv) {
            const std::vector<Hub::Post> &ps = hub->sends[r.peer];
            int k = 0, found = -1;
            for (size_t i = 0; i < ps.size(); i++) {
                if (ps[i].dst != rank) continue;
                if (k++ == used[r.peer]) { found = (int)i; break; }
            }
            if (found < 0 || ps[found].bytes != r.bytes) {
                err = "loopback: unmatched recv from rank " + std::to_string(r.peer);
                hub->barrier();
                return 1;
            }
            used[r.peer]++;
            if (cuda(cudaMemcpyAsync(r.ptr, ps[found].ptr, r.bytes, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync")) {
                hub->barrier();
                return 1;
            }
        }
        if (cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize")) { hub->barrier(); return 1; }
        // every rank finished reading its peers' send buffers
        return sync_all("group_end (copies)");
    }
    int share_buffers(void *const *local, int nbuf, std::vector<void *> &table, cudaStream_t) override {
        {
            std::lock_guard<std::mutex> g(hub->mu);
            hub->shared[rank].assign(local, local + nbuf);
        }
        if (sync_all("share_buffers (post)")) return 1;
        table.assign((size_t)world * nbuf, nullptr);
        for (int r = 0; r < world; r++)
            for (int i = 0; i < nbuf; i++) table[r * nbuf + i] = hub->shared[r][i];
        return sync_all("share_buffers (read)");
    }
    int barrier(cudaStream_t s) override {
        if (cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize")) return 1;
        return sync_all("barrier");
    }
    int allreduce_sum(void *buf, size_t count, CommElem t, cudaStream_t s) override {
        if (cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize")) return 1;
        {
            std::lock_guard<std::mutex> g(hub->mu);
            hub->bufs[rank] = buf;
        }
        if (sync_all("allreduce (post)")) return 1;
        const size_t es = t == CE_F64 ? 8 : 4;
        std::vector<double> acc(count, 0.0);
        std::vector<char> tmp(count * es);
        for (int r = 0; r < world; r++) {  // rank order: identical sums on every rank
            if (cuda(cudaMemcpyAsync(tmp.data(), hub->bufs[r], count * es, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync") ||
                cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize")) {
                hub->barrier();
                return 1;
            }
            for (size_t i = 0; i < count; i++)
                acc[i] += t == CE_F64 ? ((const double *)tmp.data())[i] : (double)((const float *)tmp.data())[i];
        }
        if (sync_all("allreduce (read)")) return 1;
        for (size_t i = 0; i < count; i++) {
            if (t == CE_F64) ((double *)tmp.data())[i] = acc[i];
            else ((float *)tmp.data())[i] = (float)acc[i];
        }
        if (cuda(cudaMemcpyAsync(buf, tmp.data(), count * es, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync")) return 1;
        return cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
};

Comm *comm_create(const void *id128, int world, int rank, std::string &err) {
    if (comm_is_loopback_id(id128)) {
        LoopComm *c = new LoopComm();
        memcpy(&c->key, (const char *)id128 + 8, 8);
        c->world = world;
        c->rank = rank;
        std::lock_guard<std::mutex> g(g_hubs_mu);
        Hub *&h = g_hubs[c->key];
        if (!h) {
            h = new Hub();
            h->world = world;
            h->sends.resize(world);
            h->bufs.resize(world, nullptr);
            h->shared.resize(world);
        }
        if (h->world != world) {
            err = "loopback id reused with another world size";
            delete c;
            return nullptr;
        }
        h->refs++;
        c->hub = h;
        return c;
    }
    NcclComm *c = new NcclComm();
    c->world = world;
    c->rank = rank;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->c, world, id, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        c->c = nullptr;
        delete c;
        return nullptr;
    }
    return c;
}

}  // namespace tqd

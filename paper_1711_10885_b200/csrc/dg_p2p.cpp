// Direct (fused) face-trace halo (dg_p2p.h): peer receive buffers as pack destinations, with a
// per-apply event protocol ordered by host-side counters (in-process or POSIX shared memory).
#include "dg_p2p.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace dg {

namespace {
constexpr auto kTimeout = std::chrono::seconds(120);

struct LocalRank {
    bool joined = false;
    double* recv[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_packed = nullptr, ev_consumed = nullptr;
    uint64_t packed = 0, consumed = 0;
};
struct LocalGroup {
    int nranks = 0, refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<LocalRank> r;
};
std::mutex g_mu;
std::map<uint64_t, LocalGroup*> g_local;

// the export blob of one rank (multi-process)
struct Blob {
    int rank;
    int pad;
    cudaIpcMemHandle_t recv[6];
    cudaIpcEventHandle_t ev_packed, ev_consumed;
    int has[6];
};
constexpr uint64_t kShmMagic = 0x44475032505348ull;   // "DGP2PSH"
}  // namespace

struct P2P {
    int rank = 0, nranks = 1;
    int nbr[6] = {-1, -1, -1, -1, -1, -1};
    double* recv[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double* remote[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_packed = nullptr, ev_consumed = nullptr;         // mine
    cudaEvent_t peer_packed[6] = {}, peer_consumed[6] = {};         // the neighbour across each face
    uint64_t t = 0;                                                 // applies packed so far
    bool ready = false;
    // in-process backend
    uint64_t key = 0;
    LocalGroup* g = nullptr;
    // multi-process backend
    bool ipc = false;
    uint64_t* shm = nullptr;        // [0] magic, [1 .. n] packed, [n+1 .. 2n] consumed
    size_t shm_bytes = 0;
    std::string shm_name;
    std::vector<void*> opened;      // IPC-mapped peer buffers
    std::vector<cudaEvent_t> opened_ev;
};

// ---------------------------------------------------------------------------------- counters
static void post(P2P* p, int which, uint64_t v)
{
    if (p->ipc) {
        __atomic_store_n(p->shm + 1 + which * p->nranks + p->rank, v, __ATOMIC_RELEASE);
        return;
    }
    std::lock_guard<std::mutex> lk(p->g->mu);
    (which == 0 ? p->g->r[p->rank].packed : p->g->r[p->rank].consumed) = v;
    p->g->cv.notify_all();
}
static bool wait_for(P2P* p, int which, int peer, uint64_t v)
{
    if (p->ipc) {
        const auto t0 = std::chrono::steady_clock::now();
        uint64_t* c = p->shm + 1 + which * p->nranks + peer;
        int spins = 0;
        while (__atomic_load_n(c, __ATOMIC_ACQUIRE) < v) {
            if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(2));
            if (std::chrono::steady_clock::now() - t0 > kTimeout) return false;
        }
        return true;
    }
    std::unique_lock<std::mutex> lk(p->g->mu);
    return p->g->cv.wait_for(lk, kTimeout, [&] {
        return (which == 0 ? p->g->r[peer].packed : p->g->r[peer].consumed) >= v;
    });
}

static int make_events(P2P* p, bool interprocess)
{
    const unsigned fl = cudaEventDisableTiming | (interprocess ? cudaEventInterprocess : 0);
    if (cudaEventCreateWithFlags(&p->ev_packed, fl) != cudaSuccess) return -1;
    if (cudaEventCreateWithFlags(&p->ev_consumed, fl) != cudaSuccess) return -1;
    return 0;
}

// ---------------------------------------------------------------------------------- in-process
int p2p_local_join(uint64_t key, int rank, int nranks, const int nbr[6], double* const recv[6], P2P** out)
{
    if (rank < 0 || rank >= nranks) return -1;
    P2P* p = new P2P();
    p->rank = rank;
    p->nranks = nranks;
    p->key = key;
    for (int f = 0; f < 6; ++f) { p->nbr[f] = nbr[f]; p->recv[f] = recv[f]; }
    if (make_events(p, false) != 0) { p2p_destroy(p); return -1; }
    std::lock_guard<std::mutex> lk(g_mu);
    LocalGroup*& g = g_local[key];
    if (!g) {
        g = new LocalGroup();
        g->nranks = nranks;
        g->r.resize(nranks);
    }
    if (g->nranks != nranks || g->r[rank].joined) {
        if (g->refs == 0) { delete g; g_local.erase(key); }
        p2p_destroy(p);
        return -1;
    }
    {
        std::lock_guard<std::mutex> lk2(g->mu);
        LocalRank& me = g->r[rank];
        me.joined = true;
        for (int f = 0; f < 6; ++f) me.recv[f] = recv[f];
        me.ev_packed = p->ev_packed;
        me.ev_consumed = p->ev_consumed;
        me.packed = me.consumed = 0;
        g->cv.notify_all();
    }
    ++g->refs;
    p->g = g;
    *out = p;
    return 0;
}

// resolve the neighbours' buffers and events once they have joined (threads join in any order)
static int local_resolve(P2P* p)
{
    std::unique_lock<std::mutex> lk(p->g->mu);
    for (int f = 0; f < 6; ++f) {
        const int q = p->nbr[f];
        if (q < 0) continue;
        if (!p->g->cv.wait_for(lk, kTimeout, [&] { return p->g->r[q].joined; })) return -1;
        p->remote[f] = p->g->r[q].recv[f ^ 1];
        p->peer_packed[f] = p->g->r[q].ev_packed;
        p->peer_consumed[f] = p->g->r[q].ev_consumed;
        if (!p->remote[f]) return -1;
    }
    p->ready = true;
    return 0;
}

// ---------------------------------------------------------------------------------- multi-process
size_t p2p_blob_bytes() { return sizeof(Blob); }

int p2p_ipc_create(int rank, int nranks, const int nbr[6], double* const recv[6], P2P** out)
{
    if (rank < 0 || rank >= nranks) return -1;
    P2P* p = new P2P();
    p->rank = rank;
    p->nranks = nranks;
    p->ipc = true;
    for (int f = 0; f < 6; ++f) { p->nbr[f] = nbr[f]; p->recv[f] = recv[f]; }
    if (make_events(p, true) != 0) { p2p_destroy(p); return -1; }
    *out = p;
    return 0;
}

int p2p_ipc_export(const P2P* p, void* blob)
{
    Blob b;
    std::memset(&b, 0, sizeof(b));
    b.rank = p->rank;
    for (int f = 0; f < 6; ++f) {
        b.has[f] = p->recv[f] != nullptr;
        if (b.has[f] && cudaIpcGetMemHandle(&b.recv[f], p->recv[f]) != cudaSuccess) return -2;
    }
    if (cudaIpcGetEventHandle(&b.ev_packed, p->ev_packed) != cudaSuccess ||
        cudaIpcGetEventHandle(&b.ev_consumed, p->ev_consumed) != cudaSuccess)
        return -2;
    std::memcpy(blob, &b, sizeof(b));
    return 0;
}

int p2p_ipc_import(P2P* p, const void* blobs, const char* shm_name)
{
    if (!p->ipc || !shm_name || shm_name[0] != '/') return -1;
    const Blob* all = static_cast<const Blob*>(blobs);
    // shared counters: rank 0 creates and zeroes the segment, then publishes the magic word
    p->shm_bytes = (size_t)(1 + 2 * p->nranks) * sizeof(uint64_t);
    p->shm_name = shm_name;
    int fd = -1;
    const auto t0 = std::chrono::steady_clock::now();
    if (p->rank == 0) {
        fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
        if (fd < 0 || ftruncate(fd, (off_t)p->shm_bytes) != 0) { if (fd >= 0) close(fd); return -1; }
    } else {
        while ((fd = shm_open(shm_name, O_RDWR, 0600)) < 0) {
            if (std::chrono::steady_clock::now() - t0 > kTimeout) return -1;
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
    }
    void* m = nullptr;
    while (true) {   // rank > 0 may open before rank 0 sized the segment
        struct stat st;
        if (fstat(fd, &st) == 0 && (size_t)st.st_size >= p->shm_bytes) break;
        if (std::chrono::steady_clock::now() - t0 > kTimeout) { close(fd); return -1; }
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    m = mmap(nullptr, p->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return -1;
    p->shm = static_cast<uint64_t*>(m);
    if (p->rank == 0) {
        for (int i = 1; i < 1 + 2 * p->nranks; ++i) __atomic_store_n(p->shm + i, 0ull, __ATOMIC_RELAXED);
        __atomic_store_n(p->shm, kShmMagic, __ATOMIC_RELEASE);
    } else {
        while (__atomic_load_n(p->shm, __ATOMIC_ACQUIRE) != kShmMagic) {
            if (std::chrono::steady_clock::now() - t0 > kTimeout) return -1;
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
    }
    // the neighbours' receive buffers and events (each peer opened once per distinct handle)
    std::map<int, std::pair<cudaEvent_t, cudaEvent_t>> evs;
    for (int f = 0; f < 6; ++f) {
        const int q = p->nbr[f];
        if (q < 0) continue;
        const Blob& b = all[q];
        if (b.rank != q || !b.has[f ^ 1]) return -1;
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, b.recv[f ^ 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return -2;
        p->opened.push_back(ptr);
        p->remote[f] = static_cast<double*>(ptr);
        if (!evs.count(q)) {
            cudaEvent_t a = nullptr, c = nullptr;
            if (cudaIpcOpenEventHandle(&a, b.ev_packed) != cudaSuccess ||
                cudaIpcOpenEventHandle(&c, b.ev_consumed) != cudaSuccess)
                return -2;
            p->opened_ev.push_back(a);
            p->opened_ev.push_back(c);
            evs[q] = {a, c};
        }
        p->peer_packed[f] = evs[q].first;
        p->peer_consumed[f] = evs[q].second;
    }
    p->ready = true;
    return 0;
}

void p2p_destroy(P2P* p)
{
    if (!p) return;
    for (void* ptr : p->opened) cudaIpcCloseMemHandle(ptr);
    for (cudaEvent_t e : p->opened_ev) cudaEventDestroy(e);
    if (p->shm) {
        munmap(p->shm, p->shm_bytes);
        if (p->rank == 0) shm_unlink(p->shm_name.c_str());
    }
    if (p->g) {
        std::lock_guard<std::mutex> lk(g_mu);
        {
            std::lock_guard<std::mutex> lk2(p->g->mu);
            p->g->r[p->rank] = LocalRank();
        }
        if (--p->g->refs == 0) {
            g_local.erase(p->key);
            delete p->g;
        }
    }
    if (p->ev_packed) cudaEventDestroy(p->ev_packed);
    if (p->ev_consumed) cudaEventDestroy(p->ev_consumed);
    delete p;
}

double* p2p_remote(const P2P* p, int face) { return p->remote[face]; }
bool p2p_ready(const P2P* p) { return p->ready; }

// ---------------------------------------------------------------------------------- protocol
int p2p_before_pack(P2P* p, cudaStream_t comm)
{
    if (!p->ready && (p->ipc || local_resolve(p) != 0)) return -1;
    if (p->t == 0) return 0;
    for (int f = 0; f < 6; ++f) {
        const int q = p->nbr[f];
        if (q < 0) continue;
        if (!wait_for(p, 1, q, p->t)) return -1;                 // q finished reading apply t
        if (cudaStreamWaitEvent(comm, p->peer_consumed[f], 0) != cudaSuccess) return -2;
    }
    return 0;
}

int p2p_after_pack(P2P* p, cudaStream_t comm)
{
    if (cudaEventRecord(p->ev_packed, comm) != cudaSuccess) return -2;
    ++p->t;
    post(p, 0, p->t);
    return 0;
}

int p2p_before_shell(P2P* p, cudaStream_t s)
{
    for (int f = 0; f < 6; ++f) {
        const int q = p->nbr[f];
        if (q < 0) continue;
        if (!wait_for(p, 0, q, p->t)) return -1;                 // q packed apply t into my buffers
        if (cudaStreamWaitEvent(s, p->peer_packed[f], 0) != cudaSuccess) return -2;
    }
    return 0;
}

int p2p_after_shell(P2P* p, cudaStream_t s)
{
    if (cudaEventRecord(p->ev_consumed, s) != cudaSuccess) return -2;
    post(p, 1, p->t);
    return 0;
}

}  // namespace dg

// In-process halo fabric (dg_fabric.h): ranks as threads of one process.
#include "dg_fabric.h"

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <vector>

namespace dg {

namespace {

constexpr char kMagic[8] = {'D', 'G', 'F', 'A', 'B', 'R', 'I', 'C'};
constexpr auto kTimeout = std::chrono::seconds(120);

struct Send {
    int dst;
    const double* ptr;
    size_t cnt;
};

struct RankState {
    bool joined = false;
    uint64_t round = 0;         // exchanges whose send buffers are posted (packed)
    uint64_t copied = 0;        // exchanges whose receive copies are enqueued
    cudaEvent_t ev_packed = nullptr, ev_copied = nullptr;
    std::vector<Send> sends;    // the sends of round `round`, in issue order
};

}  // namespace

struct Fabric {
    uint64_t key = 0;
    int nranks = 0, refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<RankState> r;
};

static std::mutex g_mu;
static std::map<uint64_t, Fabric*> g_groups;

bool fabric_id_is(const void* id128)
{
    return id128 && std::memcmp(id128, kMagic, sizeof(kMagic)) == 0;
}

void fabric_make_id(void* out128)
{
    static std::mutex mu;
    static std::mt19937_64 gen(std::random_device{}());
    std::lock_guard<std::mutex> lk(mu);
    unsigned char* o = static_cast<unsigned char*>(out128);
    std::memset(o, 0, 128);
    std::memcpy(o, kMagic, sizeof(kMagic));
    const uint64_t key = gen();
    std::memcpy(o + 8, &key, sizeof(key));
}

int fabric_join(const void* id128, int rank, int nranks, Fabric** out)
{
    if (!fabric_id_is(id128) || rank < 0 || rank >= nranks) return -1;
    uint64_t key;
    std::memcpy(&key, static_cast<const unsigned char*>(id128) + 8, sizeof(key));
    std::lock_guard<std::mutex> lk(g_mu);
    Fabric*& f = g_groups[key];
    if (!f) {
        f = new Fabric();
        f->key = key;
        f->nranks = nranks;
        f->r.resize(nranks);
    }
    if (f->nranks != nranks || f->r[rank].joined) {
        if (f->refs == 0) { delete f; g_groups.erase(key); }
        return -1;
    }
    RankState& st = f->r[rank];
    if (cudaEventCreateWithFlags(&st.ev_packed, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&st.ev_copied, cudaEventDisableTiming) != cudaSuccess) {
        if (st.ev_packed) cudaEventDestroy(st.ev_packed);
        st.ev_packed = nullptr;
        if (f->refs == 0) { delete f; g_groups.erase(key); }
        return -1;
    }
    st.joined = true;
    st.round = st.copied = 0;
    st.sends.clear();
    ++f->refs;
    *out = f;
    return 0;
}

void fabric_leave(Fabric* f, int rank)
{
    if (!f) return;
    std::lock_guard<std::mutex> lk(g_mu);
    {
        std::lock_guard<std::mutex> lk2(f->mu);
        RankState& st = f->r[rank];
        if (st.ev_packed) cudaEventDestroy(st.ev_packed);
        if (st.ev_copied) cudaEventDestroy(st.ev_copied);
        st = RankState();
    }
    if (--f->refs == 0) {
        g_groups.erase(f->key);
        delete f;
    }
}

int fabric_prepare(Fabric* f, int rank, const int nbr[6], cudaStream_t s)
{
    std::vector<cudaEvent_t> waits;
    {
        std::unique_lock<std::mutex> lk(f->mu);
        const uint64_t R = f->r[rank].round;
        if (R == 0) return 0;
        for (int fc = 0; fc < 6; ++fc) {
            const int p = nbr[fc];
            if (p < 0) continue;
            if (!f->cv.wait_for(lk, kTimeout, [&] { return f->r[p].copied >= R; })) return -1;
            waits.push_back(f->r[p].ev_copied);
        }
    }
    // the peers cannot re-record ev_copied before this rank posts its next round
    for (cudaEvent_t e : waits)
        if (cudaStreamWaitEvent(s, e, 0) != cudaSuccess) return -2;
    return 0;
}

int fabric_exchange(Fabric* f, int rank, const int nbr[6], double* const send[6], double* const recv[6],
                    const size_t cnt[6], cudaStream_t s)
{
    RankState& me = f->r[rank];
    if (cudaEventRecord(me.ev_packed, s) != cudaSuccess) return -2;
    struct Copy {
        double* dst;
        const double* src;
        size_t cnt;
        cudaEvent_t after;
    };
    std::vector<Copy> copies;
    {
        std::unique_lock<std::mutex> lk(f->mu);
        me.sends.clear();
        for (int fc = 0; fc < 6; ++fc)
            if (nbr[fc] >= 0) me.sends.push_back({nbr[fc], send[fc], cnt[fc]});
        const uint64_t R = ++me.round;
        f->cv.notify_all();
        int taken[64] = {0};   // receives matched so far per source rank (first 64 ranks)
        std::vector<int> taken_big(f->nranks > 64 ? f->nranks : 0, 0);
        for (int fc = 0; fc < 6; ++fc) {
            const int fr = fc ^ 1, p = nbr[fr];
            if (p < 0) continue;
            if (!f->cv.wait_for(lk, kTimeout, [&] { return f->r[p].round >= R; })) return -1;
            if (f->r[p].round != R) return -1;          // out of lockstep: not collective
            int& t = p < 64 ? taken[p] : taken_big[p];
            int seen = 0;
            const Send* match = nullptr;
            for (const Send& sd : f->r[p].sends)
                if (sd.dst == rank && seen++ == t) { match = &sd; break; }
            if (!match || match->cnt != cnt[fr]) return -1;
            ++t;
            copies.push_back({recv[fr], match->ptr, match->cnt, f->r[p].ev_packed});
        }
    }
    for (const Copy& c : copies) {
        if (cudaStreamWaitEvent(s, c.after, 0) != cudaSuccess) return -2;
        if (c.cnt && cudaMemcpyAsync(c.dst, c.src, c.cnt * sizeof(double), cudaMemcpyDefault, s) != cudaSuccess)
            return -2;
    }
    if (cudaEventRecord(me.ev_copied, s) != cudaSuccess) return -2;
    {
        std::lock_guard<std::mutex> lk(f->mu);
        ++me.copied;
        f->cv.notify_all();
    }
    return 0;
}

}  // namespace dg

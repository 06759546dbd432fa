// NCCL point-to-point for the face-layer halo, resolved at run time with dlopen so the
// library loads (and its symbols can be checked) on hosts without NCCL, and so it binds
// to the NCCL copy torch already loaded into the process (same SONAME libnccl.so.2).
#include "dg_nccl.h"

#include <dlfcn.h>
#include <mutex>

namespace dg {

static std::mutex g_mu;
static NcclApi g_api;
static int g_state = 0;   // 0 untried, 1 ok, -1 failed

const NcclApi* nccl_api()
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_state) return g_state > 0 ? &g_api : nullptr;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { g_state = -1; return nullptr; }
#define DG_SYM(name) g_api.name = (decltype(g_api.name))dlsym(h, #name)
    DG_SYM(ncclGetUniqueId);
    DG_SYM(ncclCommInitRank);
    DG_SYM(ncclCommDestroy);
    DG_SYM(ncclCommGetAsyncError);
    DG_SYM(ncclGetErrorString);
    DG_SYM(ncclSend);
    DG_SYM(ncclRecv);
    DG_SYM(ncclGroupStart);
    DG_SYM(ncclGroupEnd);
    DG_SYM(ncclCommCount);
#undef DG_SYM
    if (!g_api.ncclGetUniqueId || !g_api.ncclCommInitRank || !g_api.ncclSend || !g_api.ncclRecv ||
        !g_api.ncclGroupStart || !g_api.ncclGroupEnd || !g_api.ncclCommDestroy) {
        g_state = -1;
        return nullptr;
    }
    g_state = 1;
    return &g_api;
}

}  // namespace dg

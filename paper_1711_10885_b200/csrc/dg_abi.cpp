// C ABI of libdg_b200.so (declared and documented in include/dg.h).
#include "../../include/dg.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <array>
#include <mutex>
#include <new>
#include <vector>

#include "dg_internal.h"
#include <nvtx3/nvToolsExt.h>   // header-only; ranges are no-ops unless a profiler (nsys) injects

#include "dg_fabric.h"
#include "dg_p2p.h"
#include "dg_nccl.h"

using namespace dg;

struct dg_ctx {
    int device = 0, rank = 0, nranks = 1, k = 1, n = 2, n3 = 8;
    int parts[3] = {1, 1, 1}, pc[3] = {0, 0, 0};
    int per[3] = {0, 0, 0};
    int64_t nloc[3] = {0, 0, 0}, gofs[3] = {0, 0, 0}, gcells[3] = {0, 0, 0};
    int64_t ndofs = 0;
    int nbr[6] = {-1, -1, -1, -1, -1, -1};
    int64_t halo_count[6] = {0, 0, 0, 0, 0, 0};   // doubles of face f's traces (layer cells x 2 n^2)
    int64_t layer_cells[6] = {0, 0, 0, 0, 0, 0};  // cells of face f's layer
    double* sendbuf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double* recvbuf[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    bool partitioned = false;        // some face has a neighbour rank
    int64_t inner_lo[3] = {0, 0, 0}, inner_cnt[3] = {0, 0, 0};   // cells needing no remote data
    int64_t* shell = nullptr;        // device list of the partition-layer cells
    int64_t nshell = 0;
    cudaStream_t comm_stream = nullptr, host_stream = nullptr, h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t ev_slab[2] = {nullptr, nullptr}, ev_done = nullptr;   // dg_apply_host pipeline
    cudaEvent_t ev_z = nullptr, ev_recv = nullptr;   // z ready on the caller's stream; halo received
    cudaEvent_t ev_shell = nullptr;                  // shell cells done (on the comm stream)
    // DG_SHELL_STREAM=1: the shell cells on the comm stream, concurrent with the inner box (measured
    // with 2 / 4 ranks sharing one GPU: -1.7 % / +-0; the serial shell's only cost is its partial
    // last wave, ~10 us of a 6 ms apply), else after the inner box on the caller's stream
    bool shell_on_comm = false;
    // dg_timeline: timing events around the launches of the next partitioned apply (armed once)
    bool tl_armed = false, tl_done = false;
    cudaEvent_t tl_ev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    ncclComm_t comm = nullptr;       // the halo transport: NCCL (one process per GPU) ...
    Fabric* fabric = nullptr;        // ... or the in-process fabric (ranks as threads; dg_fabric.h)
    TraceArgs targs;                 // trace pack of the partition faces (dg_aux.cu)
    P2P* p2p = nullptr;              // direct (fused) halo: the pack stores into the peers' receive buffers
    bool p2p_active = false;         // ... and applies use it (fabric-direct at setup, IPC after dg_p2p_import)
    double* hz = nullptr;            // device staging for dg_apply_host
    double* hy = nullptr;
    // general-coefficient path (full / per-cell D, dg_gen.cuh)
    bool general = false;            // launch dg_gen_kernel instead of dg_cell_kernel
    bool dfield_const = false;       // the field is the constant tensor of dg_setup (not the caller's)
    double Dconst[9] = {0};          // the tensor given to dg_setup
    double* dfield = nullptr;        // [local cell][6]
    double* dsend[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double* drecv[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double* dfield_next = nullptr;   // dg_set_diffusion builds here, then swaps (validate first)
    double* drecv_next[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int* dbad = nullptr;             // validation flag of dg_set_diffusion
    // variable-velocity / over-integrated path (dg_vb.cuh)
    int m = 0;                       // Gauss points per direction (k+1 or k+3)
    bool vb = false;                 // launch dg_vb_kernel
    // physical coefficients (dg_setup) and the affine map of the mesh (dg_set_affine; NEXT-3)
    double Dphys[9] = {0}, bphys[3] = {0}, cphys = 0.0, sigma = 0.0;
    double J[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double Jinv[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double detJ = 1.0;
    bool affine = false;
    // TMA tensor maps of the last z / y pointers (n = 8 fast kernel)
    bool no_tma = false;             // DG_NO_TMA=1: per-thread global loads / stores instead
    const double* tma_z = nullptr;
    const double* tma_y = nullptr;
    bool tma_z_ok = false, tma_y_ok = false;
    CUtensorMap tmz, tmy;
    // multilinear geometry (dg_set_geometry; NEXT-3): library copy of the padded vertex grid
    bool geo = false;
    double* vert = nullptr;
    double* vtab = nullptr;          // velocity tables of the variable-velocity kernel (update_vb)
    int vtab_m = 0;
    double* mscratch = nullptr;      // dg_matrix_apply slot-split partial sums
    int64_t mscratch_n = 0;
    KParams base;
};

static cudaError_t launch_any(const dg_ctx* ctx, const KParams& p, cudaStream_t s)
{
    if (ctx->geo) return launch_geo(ctx->k, ctx->m, p, s);
    if (ctx->vb) return launch_vb(ctx->k, ctx->m, p, s);
    return ctx->general ? launch_gen(ctx->k, p, s) : launch_cell(ctx->k, p, s);
}

static std::mutex g_tab_mu;
static bool g_tab_done[64][KMAX + 1];

static int cuda_rc(cudaError_t e) { return e == cudaSuccess ? DG_OK : DG_ECUDA; }

// The kernels move x-lines with 16-byte vector loads / stores (and TMA): every vector the
// library reads or writes must be 16-byte aligned (include/dg.h); a misaligned view would
// raise a sticky misaligned-address fault that poisons the whole CUDA context.
static bool misaligned(const void* p) { return p && ((uintptr_t)p & 15u) != 0; }

#define DG_CUDA(x)                                   \
    do {                                             \
        cudaError_t e__ = (x);                       \
        if (e__ != cudaSuccess) return DG_ECUDA;     \
    } while (0)

extern "C" const char* dg_strerror(int code)
{
    switch (code) {
    case DG_OK: return "ok";
    case DG_EINVAL: return "invalid argument";
    case DG_ENOMEM: return "out of device memory";
    case DG_ECUDA: return "CUDA error";
    case DG_ENCCL: return "NCCL error (or NCCL unavailable)";
    case DG_EUNSUPPORTED: return "unsupported configuration";
    default: return "unknown error";
    }
}

static void free_ctx(dg_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    for (int f = 0; f < 6; ++f) {
        if (c->sendbuf[f]) cudaFree(c->sendbuf[f]);
        if (c->recvbuf[f]) cudaFree(c->recvbuf[f]);
    }
    if (c->shell) cudaFree(c->shell);
    if (c->dfield) cudaFree(c->dfield);
    if (c->dfield_next) cudaFree(c->dfield_next);
    for (int f = 0; f < 6; ++f)
        if (c->drecv_next[f]) cudaFree(c->drecv_next[f]);
    if (c->dbad) cudaFree(c->dbad);
    for (int f = 0; f < 6; ++f) {
        if (c->dsend[f]) cudaFree(c->dsend[f]);
        if (c->drecv[f]) cudaFree(c->drecv[f]);
    }
    if (c->hz) cudaFree(c->hz);
    if (c->hy) cudaFree(c->hy);
    if (c->mscratch) cudaFree(c->mscratch);
    if (c->vert) cudaFree(c->vert);
    if (c->vtab) cudaFree(c->vtab);
    if (c->comm) {
        const NcclApi* api = nccl_api();
        if (api) api->ncclCommDestroy(c->comm);
    }
    if (c->fabric) fabric_leave(c->fabric, c->rank);
    if (c->p2p) p2p_destroy(c->p2p);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->host_stream) cudaStreamDestroy(c->host_stream);
    if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    for (int i = 0; i < 2; ++i)
        if (c->ev_slab[i]) cudaEventDestroy(c->ev_slab[i]);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    for (cudaEvent_t e : c->tl_ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_shell) cudaEventDestroy(c->ev_shell);
    if (c->ev_z) cudaEventDestroy(c->ev_z);
    if (c->ev_recv) cudaEventDestroy(c->ev_recv);
    delete c;
}

extern "C" int dg_nccl_unique_id(void* out128)
{
    if (!out128) return DG_EINVAL;
    const NcclApi* api = nccl_api();
    if (!api) return DG_ENCCL;
    ncclUniqueId id;
    if (api->ncclGetUniqueId(&id) != 0) return DG_ENCCL;
    std::memcpy(out128, &id, sizeof(id));
    return DG_OK;
}

extern "C" int dg_fabric_id(void* out128)
{
    if (!out128) return DG_EINVAL;
    fabric_make_id(out128);
    return DG_OK;
}

extern "C" int dg_fabric_id_direct(void* out128)
{
    if (!out128) return DG_EINVAL;
    fabric_make_id(out128);
    static_cast<unsigned char*>(out128)[16] = 1;   // applies use the direct (fused) halo
    return DG_OK;
}

extern "C" size_t dg_p2p_blob_bytes(void) { return p2p_blob_bytes(); }

extern "C" int dg_p2p_export(dg_ctx* ctx, void* blob)
{
    if (!ctx || !blob || !ctx->partitioned || ctx->fabric) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->p2p && p2p_ipc_create(ctx->rank, ctx->nranks, ctx->nbr, ctx->recvbuf, &ctx->p2p) != 0) {
        ctx->p2p = nullptr;
        return DG_ECUDA;
    }
    const int r = p2p_ipc_export(ctx->p2p, blob);
    return r == 0 ? DG_OK : DG_ECUDA;
}

extern "C" int dg_p2p_import(dg_ctx* ctx, const void* blobs, const char* shm_name)
{
    if (!ctx || !blobs || !shm_name || !ctx->p2p || ctx->p2p_active) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    DG_CUDA(cudaDeviceSynchronize());                // no apply in flight across the switch
    const int r = p2p_ipc_import(ctx->p2p, blobs, shm_name);
    if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
    ctx->p2p_active = true;
    return DG_OK;
}

// ---- halo transport: one exchange = every partition face's send buffer to the
// neighbour rank across it, every receive buffer from that rank; enqueued on stream s after
// the producer of the send buffers. NCCL: one group of point-to-point calls. Per peer, NCCL
// matches sends and receives in issue order; my buffer of face fc lands in the peer's receive
// buffer of face fc^1, so receives are issued in the order fc^1: with two ranks along a
// periodic direction both faces talk to the same peer and this keeps them paired. The
// in-process fabric (dg_fabric.h) implements the same matching rule.
static int exchange(dg_ctx* ctx, double* const send[6], double* const recv[6], const size_t cnt[6], cudaStream_t s)
{
    if (ctx->fabric) {
        const int r = fabric_exchange(ctx->fabric, ctx->rank, ctx->nbr, send, recv, cnt, s);
        return r == 0 ? DG_OK : (r == -2 ? DG_ECUDA : DG_ENCCL);
    }
    if (!ctx->comm) return DG_ENCCL;
    const NcclApi* api = nccl_api();
    if (!api) return DG_ENCCL;
    if (api->ncclGroupStart() != 0) return DG_ENCCL;
    for (int fc = 0; fc < 6; ++fc) {
        const int fr = fc ^ 1;
        if (ctx->nbr[fc] >= 0 && api->ncclSend(send[fc], cnt[fc], dgNcclFloat64, ctx->nbr[fc], ctx->comm, s) != 0) {
            api->ncclGroupEnd();
            return DG_ENCCL;
        }
        if (ctx->nbr[fr] >= 0 && api->ncclRecv(recv[fr], cnt[fr], dgNcclFloat64, ctx->nbr[fr], ctx->comm, s) != 0) {
            api->ncclGroupEnd();
            return DG_ENCCL;
        }
    }
    return api->ncclGroupEnd() == 0 ? DG_OK : DG_ENCCL;
}
// Before the send buffers are overwritten (stream s): NCCL orders its sends on the comm stream
// itself; the fabric waits for the peers' copies of the previous round.
static int exchange_prepare(dg_ctx* ctx, cudaStream_t s)
{
    if (!ctx->fabric) return DG_OK;
    const int r = fabric_prepare(ctx->fabric, ctx->rank, ctx->nbr, s);
    return r == 0 ? DG_OK : (r == -2 ? DG_ECUDA : DG_ENCCL);
}

// Kernel coefficients from the physical D, b, c, sigma and the affine map x = lo + J (xhat - lo)
// of the mesh (identity unless dg_set_affine): the kernels integrate on the axis-aligned
// reference mesh, and for a constant J the weak form there is the same with
//   Dhat = |J| J^-1 D J^-T,  bhat = |J| J^-1 b,  chat = |J| c,  sigma_q = sigma / |J^-T e_q|
// (volume element |J| dxhat; face element |cof(J) e_q| dShat with nu = cof(J) e_q / |cof(J) e_q|,
// cof(J) = |J| J^-T; delta = nu^T D nu = (|J| / |cof(J) e_q|^2) e_q^T Dhat e_q, so the weights
// w+- are unchanged and the harmonic-mean penalty scales by |J| / |cof(J) e_q|).
static void transform_D(const dg_ctx* ctx, const double* D, double* Dh)
{
    double T[9];                       // J^-1 D
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) {
            double a = 0.0;
            for (int t = 0; t < 3; ++t) a += ctx->Jinv[3 * r + t] * D[3 * t + s];
            T[3 * r + s] = a;
        }
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) {
            double a = 0.0;
            for (int t = 0; t < 3; ++t) a += T[3 * r + t] * ctx->Jinv[3 * s + t];
            Dh[3 * r + s] = ctx->detJ * a;
        }
    for (int r = 0; r < 3; ++r)        // exact symmetry
        for (int s = r + 1; s < 3; ++s) Dh[3 * s + r] = Dh[3 * r + s];
}

static void set_coefficients(dg_ctx* ctx)
{
    KParams& p = ctx->base;
    double Dh[9], bh[3];
    if (ctx->affine) {
        transform_D(ctx, ctx->Dphys, Dh);
        for (int r = 0; r < 3; ++r) {
            double a = 0.0;
            for (int t = 0; t < 3; ++t) a += ctx->Jinv[3 * r + t] * ctx->bphys[t];
            bh[r] = ctx->detJ * a;
        }
    } else {
        for (int i = 0; i < 9; ++i) Dh[i] = ctx->Dphys[i];
        for (int r = 0; r < 3; ++r) bh[r] = ctx->bphys[r];
    }
    for (int q = 0; q < 3; ++q) {
        double nrm = 0.0;              // |J^-T e_q| = norm of row q of J^-1 ... column q of J^-T
        for (int t = 0; t < 3; ++t) nrm += ctx->Jinv[3 * q + t] * ctx->Jinv[3 * q + t];
        p.sigq[q] = ctx->affine ? ctx->sigma / std::sqrt(nrm) : ctx->sigma;
        p.kb[q] = bh[q] * p.hinv[q];
        p.bq[q] = bh[q];
        p.Dqq_h[q] = Dh[4 * q] * p.hinv[q];
        p.gam[q] = Dh[4 * q] * p.sigq[q];  // <delta, delta> = delta for constant D
    }
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s) p.Dhat[3 * r + s] = Dh[3 * r + s] * p.hinv[r] * p.hinv[s];
    p.sigma = ctx->sigma;
    p.c = ctx->detJ * ctx->cphys;
    for (int i = 0; i < 9; ++i) ctx->Dconst[i] = Dh[i];
}

extern "C" int dg_setup(dg_ctx** out, const dg_mesh_desc* mesh, int k, const double D[9], const double b[3],
                        double c, double sigma, int device, int rank, int nranks, const void* nccl_unique_id)
{
    if (!out || !mesh || !D || !b) return DG_EINVAL;
    *out = nullptr;
    if (k < 1 || k > KMAX) return DG_EINVAL;
    if (nranks < 1 || rank < 0 || rank >= nranks) return DG_EINVAL;
    for (int q = 0; q < 3; ++q) {
        if (mesh->ncells[q] < 1 || !(mesh->hi[q] > mesh->lo[q])) return DG_EINVAL;
        if (!std::isfinite(mesh->lo[q]) || !std::isfinite(mesh->hi[q])) return DG_EINVAL;
        if (mesh->parts[q] < 1 || mesh->ncells[q] % mesh->parts[q] != 0) return DG_EINVAL;
    }
    if ((int64_t)mesh->parts[0] * mesh->parts[1] * mesh->parts[2] != nranks) return DG_EINVAL;
    if (!psd3(D)) return DG_EINVAL;                            // symmetric PSD
    for (int r = 0; r < 3; ++r)
        if (!std::isfinite(b[r])) return DG_EINVAL;
    if (!std::isfinite(c) || !std::isfinite(sigma) || sigma < 0.0) return DG_EINVAL;
    for (int f = 0; f < 6; ++f)
        if (mesh->bc[f] != DG_BC_DIRICHLET && mesh->bc[f] != DG_BC_PERIODIC) return DG_EUNSUPPORTED;
    for (int q = 0; q < 3; ++q)   // periodic glues the two sides of a direction: both or neither
        if ((mesh->bc[2 * q] == DG_BC_PERIODIC) != (mesh->bc[2 * q + 1] == DG_BC_PERIODIC)) return DG_EINVAL;

    dg_ctx* ctx = new (std::nothrow) dg_ctx();
    if (!ctx) return DG_ENOMEM;
    ctx->device = device;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->k = k;
    ctx->n = k + 1;
    ctx->n3 = ctx->n * ctx->n * ctx->n;
    if (cudaSetDevice(device) != cudaSuccess) { free_ctx(ctx); return DG_ECUDA; }

    // tables -> this device's constant bank (once per device and degree)
    {
        std::lock_guard<std::mutex> lk(g_tab_mu);
        if (device < 0 || device >= 64) { free_ctx(ctx); return DG_EINVAL; }
        if (!g_tab_done[device][k]) {
            HostTables t;
            if (build_tables(k, &t) != 0) { free_ctx(ctx); return DG_EINVAL; }
            if (upload_tables(k, t) != 0) { free_ctx(ctx); return DG_ECUDA; }
            g_tab_done[device][k] = true;
        }
    }

    // block partition: rank = px + Px (py + Py pz)
    for (int q = 0; q < 3; ++q) ctx->parts[q] = mesh->parts[q];
    ctx->pc[0] = rank % ctx->parts[0];
    ctx->pc[1] = (rank / ctx->parts[0]) % ctx->parts[1];
    ctx->pc[2] = rank / (ctx->parts[0] * ctx->parts[1]);
    for (int q = 0; q < 3; ++q) {
        ctx->gcells[q] = mesh->ncells[q];
        ctx->nloc[q] = mesh->ncells[q] / ctx->parts[q];
        ctx->gofs[q] = ctx->nloc[q] * ctx->pc[q];
    }
    ctx->ndofs = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2] * (int64_t)ctx->n3;
    for (int q = 0; q < 3; ++q) ctx->per[q] = mesh->bc[2 * q] == DG_BC_PERIODIC;
    for (int q = 0; q < 3; ++q)
        for (int s = 0; s < 2; ++s) {
            int pcn[3] = {ctx->pc[0], ctx->pc[1], ctx->pc[2]};
            pcn[q] += s ? 1 : -1;
            const int f = 2 * q + s;
            // periodic and split along q: the wrap neighbour is the rank at the other end;
            // periodic and not split: the wrap is local to this rank (KParams::wrap)
            if (ctx->per[q] && ctx->parts[q] > 1) pcn[q] = (pcn[q] + ctx->parts[q]) % ctx->parts[q];
            if (pcn[q] >= 0 && pcn[q] < ctx->parts[q] && !(ctx->per[q] && ctx->parts[q] == 1)) {
                ctx->nbr[f] = pcn[0] + ctx->parts[0] * (pcn[1] + ctx->parts[1] * pcn[2]);
                ctx->partitioned = true;
            }
            const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
            ctx->layer_cells[f] = ctx->nloc[t1] * ctx->nloc[t2];
            ctx->halo_count[f] = ctx->layer_cells[f] * 2 * ctx->n * ctx->n;   // face traces
        }

    // kernel constants (eq:gauss_points; penalty reading C-4)
    KParams& p = ctx->base;
    std::memset(&p, 0, sizeof(p));
    double h[3];
    for (int q = 0; q < 3; ++q) {
        h[q] = (mesh->hi[q] - mesh->lo[q]) / (double)mesh->ncells[q];
        p.hinv[q] = 1.0 / h[q];
        p.nloc[q] = ctx->nloc[q];
        p.gofs[q] = ctx->gofs[q];
        p.gcells[q] = ctx->gcells[q];
        p.per[q] = ctx->per[q];
        p.wrap[q] = ctx->per[q] && ctx->parts[q] == 1;
        p.h[q] = h[q];
        p.lo[q] = mesh->lo[q];
        p.bamp[q] = 1.0;
    }
    p.bkind = 0;
    p.tma = 0;
    ctx->m = k + 1;
    if (const char* e = std::getenv("DG_NO_TMA")) ctx->no_tma = std::atoi(e) != 0;
    p.dT = h[0] * h[1] * h[2];
    for (int q = 0; q < 3; ++q) p.dF[q] = p.dT / h[q];
    for (int i = 0; i < 9; ++i) ctx->Dphys[i] = D[i];
    for (int q = 0; q < 3; ++q) ctx->bphys[q] = b[q];
    ctx->cphys = c;
    ctx->sigma = sigma;
    set_coefficients(ctx);
    // Traversal order (L2 reuse of neighbour cells): z fastest inside columns, columns
    // grouped in 4 x 16 tiles, so a cell's neighbours are touched within ~4096 tasks.


    if (ctx->partitioned) {
        for (int f = 0; f < 6; ++f) {
            if (ctx->nbr[f] < 0) continue;
            const size_t bytes = (size_t)ctx->halo_count[f] * sizeof(double);
            if (cudaMalloc(&ctx->sendbuf[f], bytes) != cudaSuccess || cudaMalloc(&ctx->recvbuf[f], bytes) != cudaSuccess) {
                free_ctx(ctx);
                return DG_ENOMEM;
            }
            cudaMemset(ctx->recvbuf[f], 0, bytes);
        }
        // interior box: cells whose faces touch no partition face
        std::vector<int64_t> shell;
        for (int q = 0; q < 3; ++q) {
            const int64_t lo = ctx->nbr[2 * q] >= 0 ? 1 : 0;
            const int64_t hi = ctx->nloc[q] - (ctx->nbr[2 * q + 1] >= 0 ? 1 : 0);
            ctx->inner_lo[q] = lo;
            ctx->inner_cnt[q] = hi > lo ? hi - lo : 0;
        }
        for (int64_t z = 0; z < ctx->nloc[2]; ++z)
            for (int64_t y = 0; y < ctx->nloc[1]; ++y)
                for (int64_t x = 0; x < ctx->nloc[0]; ++x) {
                    const int64_t l[3] = {x, y, z};
                    bool inner = true;
                    for (int q = 0; q < 3; ++q)
                        if (l[q] < ctx->inner_lo[q] || l[q] >= ctx->inner_lo[q] + ctx->inner_cnt[q]) inner = false;
                    if (!inner) shell.push_back(x + ctx->nloc[0] * (y + ctx->nloc[1] * z));
                }
        ctx->nshell = (int64_t)shell.size();
        if (ctx->nshell) {
            if (cudaMalloc(&ctx->shell, shell.size() * sizeof(int64_t)) != cudaSuccess) { free_ctx(ctx); return DG_ENOMEM; }
            if (cudaMemcpy(ctx->shell, shell.data(), shell.size() * sizeof(int64_t), cudaMemcpyHostToDevice) !=
                cudaSuccess) { free_ctx(ctx); return DG_ECUDA; }
        }
        // the comm stream at the highest priority: the trace pack's few CTAs are dispatched ahead of
        // the inner-box kernel's pending CTAs (launched right after it on the caller's stream), so
        // the pack and the transfer run under the inner kernel instead of after its last wave
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        if (cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_z, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_recv, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_shell, cudaEventDisableTiming) != cudaSuccess) {
            free_ctx(ctx);
            return DG_ECUDA;
        }
        if (const char* e = std::getenv("DG_SHELL_STREAM")) ctx->shell_on_comm = std::atoi(e) != 0;
        {   // trace pack arguments: send buffers, work prefix sums, theta(s), theta'(s)
            HostTables t;
            if (build_tables(k, &t) != 0) { free_ctx(ctx); return DG_EINVAL; }
            TraceArgs& a = ctx->targs;
            std::memset(&a, 0, sizeof(a));
            a.start[0] = 0;
            for (int f = 0; f < 6; ++f) {
                a.dst[f] = ctx->sendbuf[f];
                a.start[f + 1] = a.start[f] + (ctx->nbr[f] >= 0 ? ctx->halo_count[f] / 2 : 0);
            }
            for (int j = 0; j < ctx->n; ++j) {
                a.th[0][j] = t.th0[j]; a.th[1][j] = t.th1[j];
                a.dth[0][j] = t.dth0[j]; a.dth[1][j] = t.dth1[j];
            }
        }
        if (nccl_unique_id && fabric_id_is(nccl_unique_id)) {
            if (fabric_join(nccl_unique_id, rank, nranks, &ctx->fabric) != 0) { ctx->fabric = nullptr; free_ctx(ctx); return DG_ENCCL; }
            if (static_cast<const unsigned char*>(nccl_unique_id)[16] == 1) {   // fabric-direct (dg_fabric_id_direct)
                uint64_t key;
                std::memcpy(&key, static_cast<const unsigned char*>(nccl_unique_id) + 8, sizeof(key));
                if (p2p_local_join(key, rank, nranks, ctx->nbr, ctx->recvbuf, &ctx->p2p) != 0) {
                    ctx->p2p = nullptr;
                    free_ctx(ctx);
                    return DG_ENCCL;
                }
                ctx->p2p_active = true;
            }
        } else if (nccl_unique_id) {
            const NcclApi* api = nccl_api();
            if (!api) { free_ctx(ctx); return DG_ENCCL; }
            ncclUniqueId id;
            std::memcpy(&id, nccl_unique_id, sizeof(id));
            if (api->ncclCommInitRank(&ctx->comm, nranks, id, rank) != 0) { ctx->comm = nullptr; free_ctx(ctx); return DG_ENCCL; }
        }
    } else {
        for (int q = 0; q < 3; ++q) { ctx->inner_lo[q] = 0; ctx->inner_cnt[q] = ctx->nloc[q]; }
    }
    for (int f = 0; f < 6; ++f) p.ghost[f] = ctx->recvbuf[f];
    // a full (off-diagonal) constant tensor runs on the general-coefficient kernel with a
    // constant per-cell field; a diagonal one on the fast kernel
    bool offdiag = false;
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s)
            if (r != s && D[3 * r + s] != 0.0) offdiag = true;
    if (offdiag) {
        int rc = dg_set_diffusion(ctx, nullptr, 0, nullptr);
        if (rc == DG_OK) rc = cuda_rc(cudaStreamSynchronize(nullptr));
        if (rc != DG_OK) { free_ctx(ctx); return rc; }
    }
    *out = ctx;
    return DG_OK;
}

static int alloc_dfield(dg_ctx* ctx)
{
    const int64_t ncell = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2];
    const size_t fb = (size_t)ncell * 6 * sizeof(double);
    if (!ctx->dfield && cudaMalloc(&ctx->dfield, fb) != cudaSuccess) return DG_ENOMEM;
    if (!ctx->dfield_next && cudaMalloc(&ctx->dfield_next, fb) != cudaSuccess) return DG_ENOMEM;
    if (!ctx->dbad && cudaMalloc(&ctx->dbad, sizeof(int)) != cudaSuccess) return DG_ENOMEM;
    for (int f = 0; f < 6; ++f) {
        if (ctx->nbr[f] < 0 || ctx->dsend[f]) continue;
        const size_t bytes = (size_t)ctx->layer_cells[f] * 6 * sizeof(double);
        if (cudaMalloc(&ctx->dsend[f], bytes) != cudaSuccess || cudaMalloc(&ctx->drecv[f], bytes) != cudaSuccess ||
            cudaMalloc(&ctx->drecv_next[f], bytes) != cudaSuccess)
            return DG_ENOMEM;
    }
    return DG_OK;
}

static void bind_dfield(dg_ctx* ctx)
{
    KParams& p = ctx->base;
    p.Dfield = ctx->dfield;
    for (int f = 0; f < 6; ++f) p.Dghost[f] = ctx->drecv[f];
}

static std::mutex g_vb_mu;
static bool g_vb_done[64][KMAX + 1][MMAX + 1];

// switch between the fast kernels and the variable-velocity / over-integrated kernel
static int update_vb(dg_ctx* ctx)
{
    const bool want = ctx->base.bkind != 0 || ctx->m != ctx->k + 1;
    if (!want) { ctx->vb = false; return DG_OK; }
    if (ctx->general || ctx->affine) return DG_EUNSUPPORTED;  // per-cell / full D / affine with b(x): not built
    if (!vb_available(ctx->k, ctx->m)) return DG_EUNSUPPORTED;
    std::lock_guard<std::mutex> lk(g_vb_mu);
    if (!g_vb_done[ctx->device][ctx->k][ctx->m]) {
        HostTables t;
        if (build_tables_m(ctx->k, ctx->m, &t) != 0) return DG_EINVAL;
        if (upload_tables_vb(ctx->k, ctx->m, t) != 0) return DG_ECUDA;
        g_vb_done[ctx->device][ctx->k][ctx->m] = true;
    }
    if (ctx->base.bkind != 0 && ctx->vtab_m != ctx->m) {   // the 1D velocity tables of this rank's cells
        if (ctx->vtab) cudaFree(ctx->vtab);
        ctx->vtab = nullptr;
        ctx->vtab_m = 0;
        const int64_t cnt = (ctx->nloc[0] + ctx->nloc[1] + ctx->nloc[2]) * 4 * (ctx->m + 2);
        if (cudaMalloc(&ctx->vtab, (size_t)cnt * sizeof(double)) != cudaSuccess) { ctx->vtab = nullptr; return DG_ENOMEM; }
        HostTables t;
        if (build_tables_m(ctx->k, ctx->m, &t) != 0) return DG_EINVAL;
        GeoPts g;
        g.m = ctx->m;
        for (int i = 0; i < ctx->m; ++i) g.xi[i] = t.xi[i];
        KParams& p = ctx->base;
        if (launch_vel_tables(ctx->vtab, ctx->nloc, ctx->gofs, p.lo, p.h, g, nullptr) != cudaSuccess ||
            cudaStreamSynchronize(nullptr) != cudaSuccess)
            return DG_ECUDA;
        p.vtab = ctx->vtab;
        p.vtoff[0] = 0;
        p.vtoff[1] = ctx->nloc[0] * 4 * (ctx->m + 2);
        p.vtoff[2] = p.vtoff[1] + ctx->nloc[1] * 4 * (ctx->m + 2);
        ctx->vtab_m = ctx->m;
    }
    ctx->vb = true;
    return DG_OK;
}

extern "C" int dg_set_affine(dg_ctx* ctx, const double J[9])
{
    if (!ctx || !J) return DG_EINVAL;
    for (int i = 0; i < 9; ++i)
        if (!std::isfinite(J[i])) return DG_EINVAL;
    const double det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                       J[2] * (J[3] * J[7] - J[4] * J[6]);
    if (!(det > 0.0)) return DG_EINVAL;                   // orientation preserving, non-degenerate
    if (ctx->vb || ctx->geo) return DG_EUNSUPPORTED;                  // b(x) / over-integration: axis-aligned only
    if (ctx->general && !ctx->dfield_const) return DG_EUNSUPPORTED;   // set the map before per-cell tensors
    DG_CUDA(cudaSetDevice(ctx->device));
    for (int i = 0; i < 9; ++i) ctx->J[i] = J[i];
    ctx->detJ = det;
    // J^-1 = adj(J) / det
    ctx->Jinv[0] = (J[4] * J[8] - J[5] * J[7]) / det;
    ctx->Jinv[1] = (J[2] * J[7] - J[1] * J[8]) / det;
    ctx->Jinv[2] = (J[1] * J[5] - J[2] * J[4]) / det;
    ctx->Jinv[3] = (J[5] * J[6] - J[3] * J[8]) / det;
    ctx->Jinv[4] = (J[0] * J[8] - J[2] * J[6]) / det;
    ctx->Jinv[5] = (J[2] * J[3] - J[0] * J[5]) / det;
    ctx->Jinv[6] = (J[3] * J[7] - J[4] * J[6]) / det;
    ctx->Jinv[7] = (J[1] * J[6] - J[0] * J[7]) / det;
    ctx->Jinv[8] = (J[0] * J[4] - J[1] * J[3]) / det;
    bool ident = true;
    for (int i = 0; i < 9; ++i) ident = ident && J[i] == ((i % 4 == 0) ? 1.0 : 0.0);
    ctx->affine = !ident;
    set_coefficients(ctx);
    // the transformed tensor may be full: the general kernel with a constant field, else the fast kernel
    ctx->general = false;
    return dg_set_diffusion(ctx, nullptr, 0, nullptr) == DG_OK ? cuda_rc(cudaStreamSynchronize(nullptr)) : DG_ECUDA;
}

static std::mutex g_geo_mu;
static bool g_geo_done[64][KMAX + 1][MMAX + 1];

extern "C" int dg_set_geometry(dg_ctx* ctx, const double* vert, int m, void* stream)
{
    if (!ctx) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (!vert) {                                        // back to the axis-aligned box mesh
        ctx->geo = false;
        ctx->m = ctx->k + 1;
        return DG_OK;
    }
    if (m < ctx->k + 1 || m > MMAX) return DG_EINVAL;
    if (!geo_available(ctx->k, m)) return DG_EUNSUPPORTED;
    if (ctx->vb || ctx->affine || (ctx->general && !ctx->dfield_const)) return DG_EUNSUPPORTED;
    {
        std::lock_guard<std::mutex> lk(g_geo_mu);
        if (!g_geo_done[ctx->device][ctx->k][m]) {
            HostTables t;
            if (build_tables_m(ctx->k, m, &t) != 0) return DG_EINVAL;
            if (upload_tables_geo(ctx->k, m, t) != 0) return DG_ECUDA;
            g_geo_done[ctx->device][ctx->k][m] = true;
        }
    }
    const int64_t nv = (ctx->nloc[0] + 3) * (ctx->nloc[1] + 3) * (ctx->nloc[2] + 3) * 3;
    double* buf = nullptr;
    if (cudaMalloc(&buf, (size_t)nv * sizeof(double)) != cudaSuccess) return DG_ENOMEM;
    if (!ctx->dbad && cudaMalloc(&ctx->dbad, sizeof(int)) != cudaSuccess) { cudaFree(buf); return DG_ENOMEM; }
    int bad = 0;
    HostTables t;
    build_tables_m(ctx->k, m, &t);
    GeoPts g;
    g.m = m;
    for (int i = 0; i < m; ++i) g.xi[i] = t.xi[i];
    if (cudaMemcpyAsync(buf, vert, (size_t)nv * sizeof(double), cudaMemcpyDefault, s) != cudaSuccess ||
        cudaMemsetAsync(ctx->dbad, 0, sizeof(int), s) != cudaSuccess ||
        launch_geo_check(buf, ctx->nloc, g, ctx->dbad, s) != cudaSuccess ||
        cudaMemcpyAsync(&bad, ctx->dbad, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaFree(buf);
        return DG_ECUDA;
    }
    if (bad) { cudaFree(buf); return DG_EINVAL; }      // an inverted or degenerate cell: nothing changes
    if (ctx->vert) cudaFree(ctx->vert);
    ctx->vert = buf;
    KParams& p = ctx->base;
    p.vert = buf;
    for (int i = 0; i < 9; ++i) p.Dp[i] = ctx->Dphys[i];
    for (int r = 0; r < 3; ++r) p.bp[r] = ctx->bphys[r];
    ctx->m = m;
    ctx->geo = true;
    return DG_OK;
}

extern "C" int dg_set_velocity(dg_ctx* ctx, int kind, const double amp[3])
{
    if (!ctx || kind < 0 || kind > 2 || (kind != 0 && !amp)) return DG_EINVAL;
    if (ctx->geo && kind != 0) return DG_EUNSUPPORTED;
    for (int r = 0; r < 3 && kind; ++r)
        if (!std::isfinite(amp[r])) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    const int old_kind = ctx->base.bkind;
    double old_amp[3] = {ctx->base.bamp[0], ctx->base.bamp[1], ctx->base.bamp[2]};
    ctx->base.bkind = kind;
    for (int r = 0; r < 3; ++r) ctx->base.bamp[r] = kind ? amp[r] : 1.0;
    const int rc = update_vb(ctx);
    if (rc != DG_OK) {
        ctx->base.bkind = old_kind;
        for (int r = 0; r < 3; ++r) ctx->base.bamp[r] = old_amp[r];
        update_vb(ctx);
    }
    return rc;
}

extern "C" int dg_set_quadrature(dg_ctx* ctx, int m)
{
    if (!ctx || m < ctx->k + 1 || m > MMAX) return DG_EINVAL;
    if (ctx->geo) return DG_EUNSUPPORTED;                 // the geometry kernel's m is dg_set_geometry's
    DG_CUDA(cudaSetDevice(ctx->device));
    const int old = ctx->m;
    ctx->m = m;
    const int rc = update_vb(ctx);
    if (rc != DG_OK) {
        ctx->m = old;
        update_vb(ctx);
    }
    return rc;
}

extern "C" int dg_set_diffusion(dg_ctx* ctx, const double* Dcell, unsigned flags, void* stream)
{
    if (!ctx || (flags & ~(unsigned)DG_HALO_EXTERNAL)) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ncell = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2];
    bool offdiag = false;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            if (r != c && ctx->Dconst[3 * r + c] != 0.0) offdiag = true;
    if (!Dcell && !offdiag) {          // back to the constant diagonal tensor of dg_setup
        ctx->general = false;
        return DG_OK;
    }
    if (ctx->vb) return DG_EUNSUPPORTED;   // b(x) / over-integration run on constant diagonal D only
    if (ctx->geo && Dcell) return DG_EUNSUPPORTED;   // multilinear meshes: one constant tensor
    int rc = alloc_dfield(ctx);
    if (rc != DG_OK) return rc;
    // Everything is built in the *_next buffers and committed (pointer swap) only when it is
    // complete: a rejected field or a failed exchange leaves the previous operator intact.
    if (!Dcell) {
        // constant tensor: field and neighbour layers are the same constant (no exchange)
        DG_CUDA(launch_dfield_const(ctx->dfield_next, ctx->Dconst, ncell, s));
        for (int f = 0; f < 6; ++f)
            if (ctx->drecv_next[f])
                DG_CUDA(launch_dfield_const(ctx->drecv_next[f], ctx->Dconst, ctx->layer_cells[f], s));
    } else {
        DG_CUDA(cudaMemsetAsync(ctx->dbad, 0, sizeof(int), s));
        // physical tensors; on an affine mesh each is mapped to |J| J^-1 D J^-T on the fly
        DG_CUDA(launch_dfield_pack(Dcell, ctx->dfield_next, ctx->dbad, ncell, ctx->affine ? ctx->Jinv : nullptr,
                                   ctx->detJ, s));
        int bad = 0;
        DG_CUDA(cudaMemcpyAsync(&bad, ctx->dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
        DG_CUDA(cudaStreamSynchronize(s));
        if (bad) return DG_EINVAL;
        if (ctx->partitioned) {
            // the neighbour ranks' boundary layers of the field (setup-time, synchronous)
            if (!(flags & DG_HALO_EXTERNAL)) {
                rc = exchange_prepare(ctx, s);
                if (rc != DG_OK) return rc;
            }
            for (int f = 0; f < 6; ++f)
                if (ctx->nbr[f] >= 0) DG_CUDA(launch_pack(ctx->dfield_next, ctx->dsend[f], 6, ctx->nloc, f, s));
            if (!(flags & DG_HALO_EXTERNAL)) {
                size_t cnt[6];
                for (int f = 0; f < 6; ++f) cnt[f] = (size_t)ctx->layer_cells[f] * 6;
                rc = exchange(ctx, ctx->dsend, ctx->drecv_next, cnt, s);
                if (rc != DG_OK) return rc;
            }
            // with DG_HALO_EXTERNAL the caller fills the committed receive layers
            // (dg_halo_buffer which = 3) after this call
            DG_CUDA(cudaStreamSynchronize(s));
        }
    }
    std::swap(ctx->dfield, ctx->dfield_next);
    for (int f = 0; f < 6; ++f) std::swap(ctx->drecv[f], ctx->drecv_next[f]);
    bind_dfield(ctx);
    ctx->dfield_const = Dcell == nullptr;
    ctx->general = true;
    return DG_OK;
}

extern "C" int dg_partition(const dg_mesh_desc* mesh, int rank, int nranks, int64_t cell_lo[3], int64_t cell_cnt[3],
                            int nbr[6])
{
    if (!mesh || nranks < 1 || rank < 0 || rank >= nranks) return DG_EINVAL;
    for (int q = 0; q < 3; ++q)
        if (mesh->ncells[q] < 1 || mesh->parts[q] < 1 || mesh->ncells[q] % mesh->parts[q] != 0) return DG_EINVAL;
    if ((int64_t)mesh->parts[0] * mesh->parts[1] * mesh->parts[2] != nranks) return DG_EINVAL;
    int pc[3];
    pc[0] = rank % mesh->parts[0];
    pc[1] = (rank / mesh->parts[0]) % mesh->parts[1];
    pc[2] = rank / (mesh->parts[0] * mesh->parts[1]);
    for (int q = 0; q < 3; ++q) {
        const int64_t nl = mesh->ncells[q] / mesh->parts[q];
        if (cell_lo) cell_lo[q] = nl * pc[q];
        if (cell_cnt) cell_cnt[q] = nl;
        const bool per = mesh->bc[2 * q] == DG_BC_PERIODIC;
        for (int s = 0; s < 2; ++s) {
            int pn[3] = {pc[0], pc[1], pc[2]};
            pn[q] += s ? 1 : -1;
            if (per && mesh->parts[q] > 1) pn[q] = (pn[q] + mesh->parts[q]) % mesh->parts[q];
            if (nbr) nbr[2 * q + s] = (pn[q] >= 0 && pn[q] < mesh->parts[q] && !(per && mesh->parts[q] == 1))
                                          ? pn[0] + mesh->parts[0] * (pn[1] + mesh->parts[1] * pn[2]) : -1;
        }
    }
    return DG_OK;
}

extern "C" int dg_local_layout(const dg_ctx* ctx, int64_t cell_lo[3], int64_t cell_cnt[3], int64_t* ndofs)
{
    if (!ctx) return DG_EINVAL;
    for (int q = 0; q < 3; ++q) {
        if (cell_lo) cell_lo[q] = ctx->gofs[q];
        if (cell_cnt) cell_cnt[q] = ctx->nloc[q];
    }
    if (ndofs) *ndofs = ctx->ndofs;
    return DG_OK;
}

// TMA staging for the n = 8 fast kernel (dg_cell.cuh): tensor maps over z and y, cached by pointer
static void set_tma(dg_ctx* ctx, KParams& p, const double* z, double* y)
{
    p.tma = 0;
    if (ctx->geo || ctx->no_tma) return;
    if (ctx->k != 7 || ctx->vb) {   // bulk copies of whole cell blocks (dg_cell.cuh, namespace bulk)
        p.tma = 2;
        return;
    }
    const int64_t rows = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2] * 64;
    if (z != ctx->tma_z) {
        ctx->tma_z_ok = make_row_map(&ctx->tmz, z, rows);
        ctx->tma_z = z;
    }
    if (y != ctx->tma_y) {
        ctx->tma_y_ok = make_row_map(&ctx->tmy, y, rows);
        ctx->tma_y = y;
    }
    if (!ctx->tma_z_ok) return;
    p.tmz = ctx->tmz;
    p.tma = 1;
    if (ctx->tma_y_ok) {
        p.tmy = ctx->tmy;
        p.tma = 2;
    }
}

// Magic numbers of decode_task (dg_cell.cuh): q = (umulhi(a, m) + a) >> l equals a / d for
// every a < 2^31 with l = ceil(log2 d), m = ceil(2^(32+l) / d) - 2^32.
static void magic_div(uint64_t d, unsigned* m, unsigned* l)
{
    if (d < 1) d = 1;
    unsigned s = 0;
    while ((1ull << s) < d) ++s;
    const unsigned __int128 num = ((unsigned __int128)1 << (32 + s));
    const uint64_t mm = (uint64_t)((num + d - 1) / d) - (1ull << 32);
    *m = (unsigned)mm;
    *l = s;
}
// the task box of a launch (cells lo .. lo + cnt - 1, traversal order of decode_task)
static void set_box(KParams& p, const int64_t lo[3], const int64_t cnt[3])
{
    p.task_list = nullptr;
    for (int q = 0; q < 3; ++q) { p.task_lo[q] = lo[q]; p.task_cnt[q] = cnt[q]; }
    p.ntasks = cnt[0] * cnt[1] * cnt[2];
    magic_div((uint64_t)cnt[2], &p.dmag[0], &p.dsh[0]);
    magic_div((uint64_t)cnt[0] * 16u, &p.dmag[1], &p.dsh[1]);
}

struct Epi {             // store epilogue (KParams::epi)
    int mode = 0;
    const double* f = nullptr;
    const double* w = nullptr;
    double a = 0.0, b = 1.0, s = 0.0;
};

// NVTX range of the enclosing scope (nsys timelines of the halo overlap)
struct NvtxRange {
    explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
    ~NvtxRange() { nvtxRangePop(); }
};

static int apply_impl(dg_ctx* ctx, const double* z, const double* f, double* y, unsigned terms, cudaStream_t s,
                      const Epi* epi = nullptr, const int64_t* tasks = nullptr, int64_t ntasks = 0)
{
    if (!ctx || !z || !y) return DG_EINVAL;
    if ((const double*)y == z || (f && f == z)) return DG_EINVAL;
    if (misaligned(z) || misaligned(y) || misaligned(f)) return DG_EINVAL;
    if (epi && (misaligned(epi->f) || misaligned(epi->w))) return DG_EINVAL;
    if (terms & ~(unsigned)(DG_ALL | DG_HALO_EXTERNAL)) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    KParams p = ctx->base;
    p.z = z;
    p.y = y;
    p.f = f;
    p.epi = f ? 1 : 0;
    if (epi) {
        p.epi = epi->mode;
        p.f = epi->f;
        p.w = epi->w;
        p.ea = epi->a;
        p.eb = epi->b;
        p.es = epi->s;
    }
    p.mask = terms & DG_ALL;
    set_tma(ctx, p, z, y);
    const bool external = (terms & DG_HALO_EXTERNAL) != 0;
    if (!ctx->partitioned) {
        const int64_t zero[3] = {0, 0, 0};
        set_box(p, zero, ctx->nloc);
        if (tasks) {                 // only the listed local cells (dg_assemble's probes)
            if (ntasks == 0) return DG_OK;
            p.task_list = tasks;
            p.ntasks = ntasks;
        }
        return cuda_rc(launch_any(ctx, p, s));
    }
    NvtxRange r_apply("dg_apply (partitioned)");
    // dg_timeline (armed): 0 start on s, 1 / 2 pack (+ exchange) begin / end on the comm stream,
    // 3 / 4 inner kernel begin / end, 5 shell launch (after its wait), 6 shell end, on s
    const bool tl = ctx->tl_armed;
    ctx->tl_armed = false;
    auto mark = [&](int i, cudaStream_t st) { return tl ? cudaEventRecord(ctx->tl_ev[i], st) : cudaSuccess; };
    DG_CUDA(mark(0, s));
    // (iv) of SURVEY.md 3 / 8(e): the partition faces' traces are packed and exchanged on the comm
    // stream while the inner-box cells (no remote data) run on s; the shell cells follow the
    // receive. The pack is off s: it is launched first, so its few CTAs start ahead of the
    // inner kernel's wave, and nothing on s waits for it.
    const bool need_comm = !external && (p.mask & DG_INTERIOR_FACES);
    if (need_comm) {
        NvtxRange r_comm("trace pack + exchange (comm stream)");
        DG_CUDA(cudaEventRecord(ctx->ev_z, s));
        DG_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_z, 0));
        if (ctx->p2p_active) {
            DG_CUDA(mark(1, ctx->comm_stream));   // (before the waits on the neighbours' consumed events)
            // fused: the pack kernel stores the traces straight into the neighbours' receive
            // buffers (NVLink peer stores through the IPC mapping, or the same device's memory
            // for ranks as threads); no send buffer, no collective (dg_p2p.h)
            int r = p2p_before_pack(ctx->p2p, ctx->comm_stream);
            if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
            TraceArgs a = ctx->targs;
            for (int f = 0; f < 6; ++f) a.dst[f] = ctx->nbr[f] >= 0 ? p2p_remote(ctx->p2p, f) : nullptr;
            DG_CUDA(launch_trace_pack(z, a, ctx->n, ctx->nloc, ctx->comm_stream));
            DG_CUDA(mark(2, ctx->comm_stream));
            r = p2p_after_pack(ctx->p2p, ctx->comm_stream);
            if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
        } else {
            DG_CUDA(mark(1, ctx->comm_stream));
            int rc = exchange_prepare(ctx, ctx->comm_stream);
            if (rc != DG_OK) return rc;
            DG_CUDA(launch_trace_pack(z, ctx->targs, ctx->n, ctx->nloc, ctx->comm_stream));
            size_t cnt[6];
            for (int f = 0; f < 6; ++f) cnt[f] = (size_t)ctx->halo_count[f];
            rc = exchange(ctx, ctx->sendbuf, ctx->recvbuf, cnt, ctx->comm_stream);
            if (rc != DG_OK) return rc;
            DG_CUDA(mark(2, ctx->comm_stream));
            DG_CUDA(cudaEventRecord(ctx->ev_recv, ctx->comm_stream));
        }
    } else if (tl) {
        DG_CUDA(mark(1, s));
        DG_CUDA(mark(2, s));
    }
    // inner cells: no remote data
    set_box(p, ctx->inner_lo, ctx->inner_cnt);
    auto launch = [&](const KParams& kp) { return launch_any(ctx, kp, s); };
    {
        NvtxRange r_inner("inner-box cells");
        DG_CUDA(mark(3, s));
        DG_CUDA(launch(p));
        DG_CUDA(mark(4, s));
    }
    NvtxRange r_shell("shell cells (after the receive)");
    if (need_comm && ctx->shell_on_comm) {
        // the shell cells on the (high-priority) comm stream right after the receive: they run
        // under the inner kernel's waves instead of after its tail; the caller's stream then waits
        // for them (y complete when the apply's work on s is)
        cudaStream_t cs = ctx->comm_stream;
        if (ctx->p2p_active) {
            const int r = p2p_before_shell(ctx->p2p, cs);
            if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
        }
        p.task_list = ctx->shell;
        p.ntasks = ctx->nshell;
        p.ghosts = 1;
        DG_CUDA(mark(5, cs));
        DG_CUDA(launch_any(ctx, p, cs));
        DG_CUDA(mark(6, cs));
        if (ctx->p2p_active) {
            const int r = p2p_after_shell(ctx->p2p, cs);
            if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
        }
        DG_CUDA(cudaEventRecord(ctx->ev_shell, cs));
        DG_CUDA(cudaStreamWaitEvent(s, ctx->ev_shell, 0));
        if (tl) ctx->tl_done = true;
        return DG_OK;
    }
    if (need_comm) {
        if (ctx->p2p_active) {
            const int r = p2p_before_shell(ctx->p2p, s);
            if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
        } else {
            DG_CUDA(cudaStreamWaitEvent(s, ctx->ev_recv, 0));
        }
    }
    p.task_list = ctx->shell;
    p.ntasks = ctx->nshell;
    p.ghosts = 1;
    DG_CUDA(mark(5, s));
    DG_CUDA(launch(p));
    DG_CUDA(mark(6, s));
    if (tl) ctx->tl_done = true;
    if (need_comm && ctx->p2p_active) {
        const int r = p2p_after_shell(ctx->p2p, s);
        if (r != 0) return r == -2 ? DG_ECUDA : DG_ENCCL;
    }
    return DG_OK;
}

extern "C" int dg_timeline(dg_ctx* ctx, int arm, double* ms, int n)
{
    if (!ctx) return DG_EINVAL;
    if (!ctx->partitioned) return DG_EUNSUPPORTED;
    DG_CUDA(cudaSetDevice(ctx->device));
    if (arm) {
        for (cudaEvent_t& e : ctx->tl_ev)
            if (!e && cudaEventCreate(&e) != cudaSuccess) return DG_ECUDA;
        ctx->tl_armed = true;
        ctx->tl_done = false;
        return DG_OK;
    }
    if (!ms || n < 6 || !ctx->tl_done) return DG_EINVAL;
    DG_CUDA(cudaEventSynchronize(ctx->tl_ev[4]));   // (the shell may run on the comm stream)
    DG_CUDA(cudaEventSynchronize(ctx->tl_ev[6]));
    for (int i = 1; i <= 6; ++i) {
        float t = 0.0f;
        DG_CUDA(cudaEventElapsedTime(&t, ctx->tl_ev[0], ctx->tl_ev[i]));
        ms[i - 1] = (double)t;
    }
    return DG_OK;
}

extern "C" int dg_apply(dg_ctx* ctx, const double* z, double* y, void* stream)
{
    return apply_impl(ctx, z, nullptr, y, DG_ALL, (cudaStream_t)stream);
}

extern "C" int dg_apply_ex(dg_ctx* ctx, const double* z, double* y, unsigned terms, void* stream)
{
    return apply_impl(ctx, z, nullptr, y, terms, (cudaStream_t)stream);
}

extern "C" int dg_residual(dg_ctx* ctx, const double* z, const double* f, double* r, void* stream)
{
    if (!f || f == r) return DG_EINVAL;
    return apply_impl(ctx, z, f, r, DG_ALL, (cudaStream_t)stream);
}

// Slab pipeline of dg_apply_host (single-rank contexts): the cell box is cut into z-slabs
// (z is the slowest index, so a slab is one contiguous chunk of every vector). Slab i's
// H2D copy (stream h2d), the kernel over slab i-1 (stream host_stream; its upper z-neighbours
// live in slab i) and the D2H copy of slab i-2's y (stream d2h) overlap, so the host <-> device
// transfers in both directions (separate copy engines) hide each other and the kernel.
static int apply_host_pipelined(dg_ctx* ctx, const double* z_host, double* y_host)
{
    const int64_t nz = ctx->nloc[2];
    const int64_t layer = ctx->nloc[0] * ctx->nloc[1] * (int64_t)ctx->n3;   // doubles per z-layer
    int64_t want = 32;                                                        // slabs (pipeline depth)
    if (const char* e = std::getenv("DG_HOST_SLABS")) want = std::max(1L, std::atol(e));
    int64_t S = (nz + want - 1) / want;
    if (S < 1) S = 1;
    const int64_t nslab = (nz + S - 1) / S;
    cudaStream_t sc = ctx->host_stream, sh = ctx->h2d_stream, sd = ctx->d2h_stream;
    for (int64_t i = 0; i <= nslab; ++i) {
        if (i < nslab) {   // H2D of slab i
            const int64_t z0 = i * S, cnt = std::min(S, nz - z0);
            DG_CUDA(cudaMemcpyAsync(ctx->hz + z0 * layer, z_host + z0 * layer, (size_t)(cnt * layer) * sizeof(double),
                                    cudaMemcpyHostToDevice, sh));
            DG_CUDA(cudaEventRecord(ctx->ev_slab[i & 1], sh));
            DG_CUDA(cudaStreamWaitEvent(sc, ctx->ev_slab[i & 1], 0));
        }
        if (i >= 1) {      // kernel over slab i-1 (all of its neighbours are resident now)
            const int64_t z0 = (i - 1) * S, cnt = std::min(S, nz - z0);
            KParams p = ctx->base;
            p.z = ctx->hz;
            p.y = ctx->hy;
            p.f = nullptr;
            p.epi = 0;
            p.mask = DG_ALL;
            set_tma(ctx, p, ctx->hz, ctx->hy);
            const int64_t blo[3] = {0, 0, z0}, bcnt[3] = {ctx->nloc[0], ctx->nloc[1], cnt};
            set_box(p, blo, bcnt);
            DG_CUDA(launch_any(ctx, p, sc));
            DG_CUDA(cudaEventRecord(ctx->ev_done, sc));
            DG_CUDA(cudaStreamWaitEvent(sd, ctx->ev_done, 0));
            DG_CUDA(cudaMemcpyAsync(y_host + z0 * layer, ctx->hy + z0 * layer, (size_t)(cnt * layer) * sizeof(double),
                                    cudaMemcpyDeviceToHost, sd));
        }
    }
    DG_CUDA(cudaStreamSynchronize(sd));
    DG_CUDA(cudaStreamSynchronize(sc));
    return DG_OK;
}

extern "C" int dg_ssp_stage(dg_ctx* ctx, const double* z, const double* f, const double* w, double a, double b,
                            double dt, double* out, void* stream)
{
    if (!ctx || !z || !out || out == z || (f && f == out)) return DG_EINVAL;
    if (!std::isfinite(a) || !std::isfinite(b) || !std::isfinite(dt)) return DG_EINVAL;
    if (ctx->geo) return DG_EUNSUPPORTED;   // the mass matrix of a multilinear cell is not Delta_T I
    Epi e;
    e.mode = 2;
    e.f = f;
    e.w = (a != 0.0) ? w : nullptr;
    if (a != 0.0 && !w) return DG_EINVAL;
    e.a = a;
    e.b = b;
    e.s = dt / (ctx->base.dT * ctx->detJ);   // M^-1 = 1/(|J| Delta_T) (orthonormal basis)
    return apply_impl(ctx, z, nullptr, out, DG_ALL, (cudaStream_t)stream, &e);
}

extern "C" int dg_apply_host(dg_ctx* ctx, const double* z_host, double* y_host)
{
    if (!ctx || !z_host || !y_host) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    const size_t bytes = (size_t)ctx->ndofs * sizeof(double);
    if (!ctx->host_stream) {
        if (cudaStreamCreateWithFlags(&ctx->host_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_slab[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_slab[1], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming) != cudaSuccess)
            return DG_ECUDA;
    }
    if (!ctx->hz) {
        if (cudaMalloc(&ctx->hz, bytes) != cudaSuccess) return DG_ENOMEM;
        if (cudaMalloc(&ctx->hy, bytes) != cudaSuccess) { cudaFree(ctx->hz); ctx->hz = nullptr; return DG_ENOMEM; }
    }
    if (!ctx->partitioned && !ctx->per[2]) return apply_host_pipelined(ctx, z_host, y_host);
    // partitioned (halo exchange needs the whole local z) or z-periodic (slab 0 needs the last
    // slab): copy in, apply, copy out
    DG_CUDA(cudaMemcpyAsync(ctx->hz, z_host, bytes, cudaMemcpyHostToDevice, ctx->host_stream));
    int rc = apply_impl(ctx, ctx->hz, nullptr, ctx->hy, DG_ALL, ctx->host_stream);
    if (rc != DG_OK) return rc;
    DG_CUDA(cudaMemcpyAsync(y_host, ctx->hy, bytes, cudaMemcpyDeviceToHost, ctx->host_stream));
    DG_CUDA(cudaStreamSynchronize(ctx->host_stream));
    return DG_OK;
}

// ---- matrix-based comparison (NEXT-4; dg_matrix.cu) ----
extern "C" int dg_matrix_size(const dg_ctx* ctx, int64_t* ndoubles)
{
    if (!ctx || !ndoubles) return DG_EINVAL;
    const int64_t ncell = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2];
    *ndoubles = ncell * 7 * (int64_t)ctx->n3 * (ctx->n3 + (ctx->n3 & 1));
    return DG_OK;
}

// Probes of different colours are independent (separate z / y, disjoint matrix columns): they
// run on up to 8 streams ("lanes"), each with its own probe vectors, so the small per-probe
// launches (a task list of ~7/27 of the cells) overlap and fill the GPU.
extern "C" int dg_assemble(dg_ctx* ctx, double* A, void* stream)
{
    if (!ctx || !A || misaligned(A)) return DG_EINVAL;
    if (ctx->nranks != 1) return DG_EUNSUPPORTED;
    DG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    int64_t nA = 0;
    dg_matrix_size(ctx, &nA);
    const size_t vbytes = (size_t)ctx->ndofs * sizeof(double);
    const int64_t ncell = ctx->nloc[0] * ctx->nloc[1] * ctx->nloc[2];
    const int n3 = ctx->n3;
    int ncol[3];
    bool present[3][5];
    matrix_colours(ctx->nloc, ctx->per, ncol, present);
    std::vector<std::array<int, 3>> cols;
    for (int c2 = 0; c2 < ncol[2]; ++c2)
        for (int c1 = 0; c1 < ncol[1]; ++c1)
            for (int c0 = 0; c0 < ncol[0]; ++c0)
                if (present[0][c0] && present[1][c1] && present[2][c2]) cols.push_back({c0, c1, c2});
    // task lists of all colours, back to back (a cell is next to at most 7 colour classes)
    int64_t* tasks = nullptr;
    unsigned long long* count = nullptr;
    if (cudaMalloc(&tasks, (size_t)(7 * ncell + 1) * sizeof(int64_t)) != cudaSuccess) return DG_ENOMEM;
    if (cudaMalloc(&count, sizeof(unsigned long long)) != cudaSuccess) { cudaFree(tasks); return DG_ENOMEM; }
    int rc = DG_OK;
    std::vector<int64_t> off(cols.size() + 1, 0);
    for (size_t ci = 0; ci < cols.size() && rc == DG_OK; ++ci) {
        unsigned long long nt = 0;
        if (launch_probe_tasks(ctx->nloc, ctx->per, cols[ci].data(), tasks + off[ci], count, s) != cudaSuccess ||
            cudaMemcpyAsync(&nt, count, sizeof(nt), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            rc = DG_ECUDA;
        off[ci + 1] = off[ci] + (int64_t)nt;
    }
    struct Lane {
        cudaStream_t st = nullptr;
        cudaEvent_t ev = nullptr;
        double* z = nullptr;
        double* y = nullptr;
    };
    std::vector<Lane> lanes;
    const int want = (int)std::min<size_t>(8, cols.size());
    for (int l = 0; l < want && rc == DG_OK; ++l) {
        Lane ln;
        if (cudaMalloc(&ln.z, vbytes) != cudaSuccess) break;
        if (cudaMalloc(&ln.y, vbytes) != cudaSuccess) { cudaFree(ln.z); break; }
        if (cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming) != cudaSuccess) {
            rc = DG_ECUDA;
            lanes.push_back(ln);
            break;
        }
        lanes.push_back(ln);
    }
    cudaGetLastError();                       // a failed optional lane allocation is not an error
    if (rc == DG_OK && lanes.empty() && !cols.empty()) rc = DG_ENOMEM;
    cudaEvent_t ev0 = nullptr;
    if (rc == DG_OK && (cudaMemsetAsync(A, 0, (size_t)nA * sizeof(double), s) != cudaSuccess ||
                        cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming) != cudaSuccess ||
                        cudaEventRecord(ev0, s) != cudaSuccess))
        rc = DG_ECUDA;
    for (auto& ln : lanes)
        if (rc == DG_OK && (cudaStreamWaitEvent(ln.st, ev0, 0) != cudaSuccess ||
                            cudaMemsetAsync(ln.z, 0, vbytes, ln.st) != cudaSuccess))
            rc = DG_ECUDA;
    for (size_t ci = 0; ci < cols.size() && rc == DG_OK; ++ci) {
        Lane& ln = lanes[ci % lanes.size()];
        const int* col = cols[ci].data();
        const int64_t* tl = tasks + off[ci];
        const int64_t nt = off[ci + 1] - off[ci];
        if (launch_probe_set(ln.z, n3, ctx->nloc, ctx->per, col, 0, 1.0, ln.st) != cudaSuccess) {
            rc = DG_ECUDA;
            break;
        }
        // probe (col, j): z = sum of e_(T, j) over the cells T of colour col; y on the cells next to
        // them (the task list); the scatter also moves the probe to (col, j + 1) and, after the
        // last j, leaves z zero for the lane's next colour
        for (int j = 0; j < n3 && rc == DG_OK; ++j) {
            rc = apply_impl(ctx, ln.z, nullptr, ln.y, DG_ALL, ln.st, nullptr, tl, nt);
            if (rc != DG_OK) break;
            if (launch_probe_scatter(A, ln.y, ln.z, tl, nt, n3, ctx->nloc, ctx->per, col, j, j + 1 < n3 ? j + 1 : -1,
                                     ln.st) != cudaSuccess)
                rc = DG_ECUDA;
        }
    }
    for (auto& ln : lanes) {
        if (ln.ev && ln.st && (cudaEventRecord(ln.ev, ln.st) != cudaSuccess || cudaStreamWaitEvent(s, ln.ev, 0) != cudaSuccess))
            rc = rc == DG_OK ? DG_ECUDA : rc;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == DG_OK) rc = DG_ECUDA;
    for (auto& ln : lanes) {
        if (ln.st) { cudaStreamSynchronize(ln.st); cudaStreamDestroy(ln.st); }
        if (ln.ev) cudaEventDestroy(ln.ev);
        cudaFree(ln.z);
        cudaFree(ln.y);
    }
    if (ev0) cudaEventDestroy(ev0);
    cudaFree(tasks);
    cudaFree(count);
    return rc;
}

extern "C" int dg_matrix_apply(dg_ctx* ctx, const double* A, const double* z, double* y, void* stream)
{
    if (!ctx || !A || !z || !y || (const double*)y == z) return DG_EINVAL;
    if (misaligned(A) || misaligned(z) || misaligned(y)) return DG_EINVAL;
    if (ctx->nranks != 1) return DG_EUNSUPPORTED;
    DG_CUDA(cudaSetDevice(ctx->device));
    const int64_t ns = matrix_scratch_doubles(ctx->n3, ctx->ndofs / ctx->n3);
    if (ns > ctx->mscratch_n) {
        if (ctx->mscratch) cudaFree(ctx->mscratch);
        ctx->mscratch = nullptr;
        ctx->mscratch_n = 0;
        if (cudaMalloc(&ctx->mscratch, (size_t)ns * sizeof(double)) != cudaSuccess) return DG_ENOMEM;
        ctx->mscratch_n = ns;
    }
    return cuda_rc(launch_matrix_apply(A, z, y, ns ? ctx->mscratch : nullptr, ctx->n3, ctx->nloc, ctx->per,
                                       (cudaStream_t)stream));
}

extern "C" int dg_sync(dg_ctx* ctx)
{
    if (!ctx) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    DG_CUDA(cudaDeviceSynchronize());
    if (ctx->comm) {
        const NcclApi* api = nccl_api();
        ncclResult_t r = 0;
        if (api && api->ncclCommGetAsyncError && api->ncclCommGetAsyncError(ctx->comm, &r) == 0 && r != 0)
            return DG_ENCCL;
    }
    return DG_OK;
}

extern "C" int dg_destroy(dg_ctx* ctx)
{
    if (!ctx) return DG_EINVAL;
    int rc = DG_OK;
    cudaSetDevice(ctx->device);
    if (cudaDeviceSynchronize() != cudaSuccess) rc = DG_ECUDA;
    free_ctx(ctx);
    return rc;
}

extern "C" int dg_halo_info(const dg_ctx* ctx, int face, int* neighbor_rank, int64_t* count)
{
    if (!ctx || face < 0 || face > 5) return DG_EINVAL;
    if (neighbor_rank) *neighbor_rank = ctx->nbr[face];
    if (count) *count = ctx->halo_count[face];
    return DG_OK;
}

extern "C" int dg_halo_buffer(dg_ctx* ctx, int face, int which, double** ptr)
{
    if (!ctx || face < 0 || face > 5 || which < 0 || which > 3 || !ptr) return DG_EINVAL;
    *ptr = which == 0 ? ctx->sendbuf[face] : which == 1 ? ctx->recvbuf[face]
         : which == 2 ? ctx->dsend[face] : ctx->drecv[face];
    return DG_OK;
}

extern "C" int dg_halo_pack(dg_ctx* ctx, const double* z, void* stream)
{
    if (!ctx || !z || misaligned(z)) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    return cuda_rc(launch_trace_pack(z, ctx->targs, ctx->n, ctx->nloc, (cudaStream_t)stream));
}

extern "C" int dg_fill_uniform(double* dst, int64_t count, uint64_t seed, int64_t offset, void* stream)
{
    if ((!dst && count > 0) || count < 0 || offset < 0) return DG_EINVAL;
    return cuda_rc(launch_fill_uniform(dst, count, seed, offset, (cudaStream_t)stream));
}

extern "C" int dg_fill_uniform_local(dg_ctx* ctx, double* dst, uint64_t seed, void* stream)
{
    if (!ctx || !dst) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    return cuda_rc(launch_fill_uniform_local(dst, ctx->n3, ctx->nloc, ctx->gofs, ctx->gcells, seed, (cudaStream_t)stream));
}

extern "C" int dg_fill_uniform_cells(dg_ctx* ctx, double* dst, int per_cell, uint64_t seed, void* stream)
{
    if (!ctx || !dst || per_cell < 1) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    return cuda_rc(launch_fill_uniform_local(dst, per_cell, ctx->nloc, ctx->gofs, ctx->gcells, seed, (cudaStream_t)stream));
}

extern "C" int dg_comm_info(const dg_ctx* ctx, int* transport, int* nranks)
{
    if (!ctx) return DG_EINVAL;
    int t = 0, n = ctx->nranks;
    if (ctx->fabric) {
        t = ctx->p2p_active ? 3 : 2;
    } else if (ctx->comm) {
        t = 1;
        const NcclApi* api = nccl_api();
        int c = 0;
        if (api && api->ncclCommCount) {
            if (api->ncclCommCount(ctx->comm, &c) != 0) return DG_ENCCL;
            n = c;
        }
    }
    if (ctx->p2p_active && !ctx->fabric) t = 4;
    if (transport) *transport = t;
    if (nranks) *nranks = n;
    return DG_OK;
}

extern "C" int dg_get_kernel_info(const dg_ctx* ctx, dg_kernel_info* info)
{
    if (!ctx || !info) return DG_EINVAL;
    DG_CUDA(cudaSetDevice(ctx->device));
    LaunchInfo li;
    const int rc = ctx->geo ? geo_launch_info(ctx->k, ctx->m, &li) : ctx->vb ? vb_launch_info(ctx->k, ctx->m, &li)
                           : (ctx->general ? gen_launch_info(ctx->k, &li) : cell_launch_info(ctx->k, &li));
    if (rc != 0) return DG_ECUDA;
    info->launches_per_apply = ctx->partitioned ? 3 : 1;   // trace pack, inner box, shell
    info->cells_per_cta = li.cells_per_cta;
    info->threads_per_cta = li.threads;
    info->smem_bytes = li.smem;
    info->regs_per_thread = li.regs;
    info->ctas_per_sm = li.ctas_per_sm;
    return DG_OK;
}

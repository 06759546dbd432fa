/*
 * dg.h -- C ABI of the B200-native (sm_100a, FP64) matrix-free SIPG/WSIPG
 * operator of arXiv 1711.10885.
 *
 * The operation: for the convection-diffusion-reaction problem
 *     -div(D grad u) + div(b u) + c u = f          (eq:modelproblem, stationary)
 * discretized by the weighted symmetric interior penalty DG method with
 * tensor-product orthonormal Legendre bases of degree k and (k+1)^3 Gauss
 * points, the library computes
 *     y = A z,   (A)_ij = a_h(phi_j, phi_i)           (eq:blf)
 * matrix-free by sum factorization, and the residual
 *     r = f - A z.
 *
 * Readings of the paper the ABI fixes:
 *   - reference cell [0,1]^3, theta_j(x) = sqrt(2j+1) P_j(2x-1)        (C-2)
 *   - DOF order: cell e = ix + Nx(iy + Ny iz) (of THIS RANK's local box),
 *     local j = jx + n(jy + n jz), n = k+1; block e occupies
 *     [e n^3, (e+1) n^3) of every vector                               (C-3)
 *   - weighted average {v}_w = w- v- + w+ v+ (PAPER.md:271 garbled)   (C-1)
 *   - penalty gamma_F = <delta-, delta+> * sigma, delta = nu^T D nu;
 *     on the boundary gamma = delta * sigma                            (C-4, C-6)
 *   - all six box sides weak Dirichlet with g = 0 inside A             (C-9, C-10)
 *
 * Vectors are caller-owned DEVICE pointers to FP64 arrays of dg_local_layout()
 * ndofs entries (unless stated otherwise), 16-byte aligned (the kernels move x-lines with
 * 16-byte vector accesses and TMA; a misaligned pointer returns DG_EINVAL). The library never
 * allocates or frees them. z must not alias y, r or f. y / r are fully overwritten.
 *
 * Every call returns an int status (DG_OK = 0 or a negative DG_E* code); no
 * C++ exception crosses the ABI. dg_apply* / dg_residual are enqueued on the
 * caller's CUDA stream and return immediately; device faults surface at
 * dg_sync or dg_destroy. With nranks > 1 every apply is collective (all ranks
 * call it in the same order). A context is not thread-safe; distinct contexts
 * are independent.
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg_ctx dg_ctx;  /* opaque: tables, halo buffers, NCCL communicator, streams */

typedef struct {
    int64_t ncells[3];   /* GLOBAL structured box mesh: cells per direction (>= 1) */
    double  lo[3], hi[3];/* box corners, hi > lo; uniform cuboid cells h_q = (hi-lo)/ncells */
    int     bc[6];       /* per side (x-,x+,y-,y+,z-,z+): DG_BC_DIRICHLET or DG_BC_PERIODIC
                            (periodic must be set on both sides of a direction) */
    int     parts[3];    /* rank grid Px,Py,Pz; product == nranks; each must divide ncells */
} dg_mesh_desc;

enum { DG_OK = 0, DG_EINVAL = -1, DG_ENOMEM = -2, DG_ECUDA = -3, DG_ENCCL = -4, DG_EUNSUPPORTED = -5 };

/* Term masks (PAPER.md:342-347 split a_h into volume, interior-face, boundary-face parts). */
enum { DG_VOLUME = 1, DG_INTERIOR_FACES = 2, DG_BOUNDARY_FACES = 4, DG_ALL = 7,
       /* halo already placed in the receive buffers by the caller (dg_halo_buffer);
          skip the pack + NCCL exchange. Used by single-process loopback tests. */
       DG_HALO_EXTERNAL = 0x100 };

/* Boundary conditions per box side.
 *   DG_BC_DIRICHLET: weak Dirichlet with g = 0 inside A (reading C-9; g enters only f).
 *   DG_BC_PERIODIC : the two sides of a direction are glued; the wrap face between the last
 *                    and the first cell layer is an interior face with nu = +e_q, treated like
 *                    a processor boundary (the paper's benchmark setting;
 *                    DESIGN.md reading N-1). Split over ranks, the wrap neighbour is the rank
 *                    at the other end of the rank grid. */
enum { DG_BC_DIRICHLET = 0, DG_BC_PERIODIC = 1 };

/*
 * Create a context on CUDA device `device` for rank `rank` of `nranks`.
 *   k      polynomial degree, 1 <= k <= 10 (n = k+1 basis functions and Gauss points per direction)
 *   D      3x3 row-major diffusion tensor, symmetric positive semi-definite
 *          (D = 0 is accepted: the mass-matrix invariant). A diagonal D runs on the fused
 *          constant-coefficient kernel; a full D (off-diagonal entries, PAPER.md:202-205, :436;
 *          reading C-16) on the general-coefficient kernel (dg_set_diffusion)
 *   b      constant velocity (div b = 0), c reaction coefficient, sigma >= 0 penalty factor
 *   nccl_unique_id  128-byte ncclUniqueId broadcast by the caller (halo over NCCL, one process
 *                   per GPU), or an id from dg_fabric_id shared by the ranks as THREADS of one
 *                   process (the in-process fabric: same exchange semantics, stream-ordered
 *                   copies; single-GPU tests of the partitioned path); NULL iff nranks == 1 or
 *                   iff the caller drives the halo itself (DG_HALO_EXTERNAL)
 * Errors: DG_EINVAL (k, mesh, D not symmetric positive semi-definite -- all principal minors of
 *         D / max|D_ij| >= -1e-13 --, sigma < 0, parts, periodic on one side of a direction
 *         only), DG_EUNSUPPORTED (unknown bc),
 *         DG_ECUDA, DG_ENCCL, DG_ENOMEM.
 * Not timed; uploads tables and allocates the halo buffers.
 */
int dg_setup(dg_ctx** out, const dg_mesh_desc* mesh, int k, const double D[9], const double b[3],
             double c, double sigma, int device, int rank, int nranks, const void* nccl_unique_id);

/* Host-only block partition (no device access): rank = px + Px (py + Py pz); this rank's
   global cell offset / counts and the neighbour rank across each face 2q+s (-1: domain
   boundary). dg_setup uses the same rule. */
int dg_partition(const dg_mesh_desc* mesh, int rank, int nranks, int64_t cell_lo[3], int64_t cell_cnt[3],
                 int nbr[6]);

/* This rank's cell box (global cell offset and counts) and its vector length. */
int dg_local_layout(const dg_ctx* ctx, int64_t cell_lo[3], int64_t cell_cnt[3], int64_t* ndofs);

/* y = A z on stream (a cudaStream_t; NULL = legacy default stream). */
int dg_apply(dg_ctx* ctx, const double* z, double* y, void* stream);

/* y = (the parts of A selected by `terms`) z; terms = OR of DG_VOLUME / DG_INTERIOR_FACES /
   DG_BOUNDARY_FACES, optionally | DG_HALO_EXTERNAL. */
int dg_apply_ex(dg_ctx* ctx, const double* z, double* y, unsigned terms, void* stream);

/* r = f - A z, fused into the final store (f: assembled l_h(phi_i)). */
int dg_residual(dg_ctx* ctx, const double* z, const double* f, double* r, void* stream);

/* One stage of an explicit strong-stability-preserving Runge-Kutta method in Shu-Osher form
 * (NEXT-2; M z^(k+1) = M z^(k) + dt (f - A z^(k)), "higher-order Runge-Kutta
 * methods involve basically the same computations per stage"; Heun = SSP-RK2):
 *     out = a w + b (z + dt M^-1 (f - A z)),    M = Delta_T I  (orthonormal basis)
 * fused into the kernel's single store. f == NULL means f = 0; w is read only when a != 0.
 * Forward Euler: (a, b) = (0, 1). Heun: stage 1 z1 = stage(z = u, a = 0, b = 1);
 * stage 2 u' = stage(z = z1, w = u, a = 1/2, b = 1/2). out must not alias z or f (it may alias w).
 * Collective like dg_apply. Errors: DG_EINVAL (aliasing, non-finite a, b, dt, a != 0 without w). */
int dg_ssp_stage(dg_ctx* ctx, const double* z, const double* f, const double* w, double a, double b, double dt,
                 double* out, void* stream);

/* End-to-end variant with HOST buffers: z_host, y_host are host pointers (pinned for speed)
   of ndofs doubles; synchronous. Single-rank contexts without z-periodicity run a slab
   pipeline: z-slabs are copied in, applied and copied out on three internal streams, so
   both transfer directions and the kernel overlap; otherwise copy in, apply, copy out. */
int dg_apply_host(dg_ctx* ctx, const double* z_host, double* y_host);

/* Wait for all work of the context; surfaces asynchronous CUDA / NCCL errors. */
int dg_sync(dg_ctx* ctx);
int dg_destroy(dg_ctx* ctx);
const char* dg_strerror(int code);

/* Per-cell diffusion tensors (NEXT-1: the paper's Problem A, "tensor-valued diffusion
 * coefficients ... constant per cell ... weighted averaging across cell boundaries for
 * discontinuous coefficients"). Dcell: caller-owned DEVICE array of this
 * rank's local cells x 9 doubles (row-major 3x3, symmetric PSD), local cell order (C-3);
 * the library copies it (6 unique entries per cell) and, with nranks > 1, exchanges the
 * partition-layer tensors with the neighbour ranks (collective; skipped with
 * flags = DG_HALO_EXTERNAL: the caller then fills the receive layers, dg_halo_buffer
 * which = 3). On a face the tensors D-, D+ of its two cells give delta = nu^T D nu per side,
 * the weights w- = d+/(d- + d+), w+ = d-/(d- + d+) and the penalty
 * gamma = <d-, d+> sigma. Subsequent applies use the
 * general-coefficient kernel. Dcell = NULL reverts to the constant D of dg_setup.
 * Synchronous on `stream`. Errors: DG_EINVAL (non-symmetric / non-finite / negative diagonal
 * entry, bad flags), DG_ENOMEM, DG_ECUDA, DG_ENCCL. Not timed. */
int dg_set_diffusion(dg_ctx* ctx, const double* Dcell, unsigned flags, void* stream);

/* Affine geometry (NEXT-3: the paper's Problem B has "affine geometries"): the
 * physical mesh is the image x = lo + J (xhat - lo) of the axis-aligned box mesh of dg_setup
 * (J row-major 3x3, det J > 0); D, b, c, sigma (dg_setup) and per-cell tensors (dg_set_diffusion)
 * are physical. The kernels integrate on the reference mesh with Dhat = |J| J^-1 D J^-T,
 * bhat = |J| J^-1 b, chat = |J| c and the penalty sigma / |J^-T e_q| per face direction (the
 * exact change of variables of eq:blf for a constant J: volume element |J|, face element
 * |cof(J) e_q|, normal cof(J) e_q / |cof(J) e_q|); the SSP mass is |J| Delta_T. J = I restores the
 * axis-aligned mesh. Call before dg_set_diffusion with per-cell tensors.
 * Errors: DG_EINVAL (det J <= 0, non-finite), DG_EUNSUPPORTED (velocity field / over-integration
 * set, or per-cell tensors already set). */
int dg_set_affine(dg_ctx* ctx, const double J[9]);

/* Multilinear (Q1) geometry (NEXT-3: the paper's Problem C has "multilinear geometries",
 * PAPER.md:957-961; "the transformation x = mu_T(xhat) ... is a d-valued Q_1 finite element
 * function and sum-factorization can be used to evaluate its values and derivatives at quadrature
 * points"). Cell (i, j, k) of this rank's box is the image of [0,1]^3 under the
 * trilinear map of its 8 vertices; every integral of eq:blf is evaluated with the map's Jacobian
 * at each of the m^3 volume / m^2 face Gauss points (gradients J^-T grad_hat, dx = det J dxi,
 * face normal cof(J) e_q / |cof(J) e_q|, dS = |cof(J) e_q| dxi; each side of a face with its own
 * Jacobian; penalty <delta-, delta+> sigma with delta = nu^T D nu, sigma as given).
 *   vert  caller-owned array (device or host) of the PADDED vertex grid of this rank's box:
 *         (nloc[0]+3) x (nloc[1]+3) x (nloc[2]+3) vertices x 3 doubles (x, y, z), x fastest;
 *         local vertex (i, j, k), -1 <= i <= nloc[0] + 1, at index
 *         ((k+1) (nloc[1]+3) + (j+1)) (nloc[0]+3) + (i+1). The outer layer holds the vertices of
 *         the neighbour cells across the box faces: on a partition face the neighbour rank's, on
 *         a periodic side the periodic continuation (the far side's vertices shifted by the
 *         period); unused on Dirichlet sides. The library copies it (not timed). NULL reverts to
 *         the axis-aligned box mesh of dg_setup.
 *   m     Gauss points per direction: k+1 (q = 2p), k+3 (q = 2p+4) or ceil((3k+5)/2) (Problem
 *         C's q = 3p+4) while m <= 16.
 * D (full symmetric PSD), b and c are the constants of dg_setup. Not combined with per-cell
 * tensors, velocity fields, dg_set_affine or dg_ssp_stage (the mass of a multilinear cell is not
 * Delta_T I).
 * Errors: DG_EINVAL (m < k+1; a cell with det J <= 0 at a quadrature point or corner: the
 * operator is then unchanged), DG_EUNSUPPORTED (uncompiled (k, m), the combinations above),
 * DG_ENOMEM, DG_ECUDA. */
int dg_set_geometry(dg_ctx* ctx, const double* vert, int m, void* stream);

/* Velocity field b(x) evaluated at every quadrature point (NEXT-2: the paper's Taylor-Green
 * transport run):
 *   kind 0: the constant b of dg_setup (default);
 *   kind 1: Taylor-Green, b = (cos x1 sin(-x2) sin(-x3), 1/2 sin x1 cos(-x2) sin(-x3),
 *           1/2 sin x1 sin(-x2) cos(-x3)) (eq:2), x the physical coordinates;
 *   kind 2: the linear divergence-free test field b = (x2, x3, x1);
 * each component times amp[r]. b is continuous, so b.nu is evaluated once per face point
 * (reading N-4); a periodic box needs a box-periodic field (Taylor-Green on (-pi, pi)^3).
 * Runs on the variable-velocity kernel (constant diagonal D).
 * Errors: DG_EINVAL (kind, non-finite amp), DG_EUNSUPPORTED (per-cell / full D set, multilinear
 * geometry set, an uncompiled (k, m)). */
int dg_set_velocity(dg_ctx* ctx, int kind, const double amp[3]);

/* Gauss points per direction m (NEXT-3 over-integration; q = 2p + 4 is m = k + 3, PAPER.md:950-956,
 * :1102-1104; Problem C's q = 3p + 4 is m = ceil((3k + 5) / 2)) on the
 * variable-velocity kernel: m = k + 1 (default), k + 3 or ceil((3k + 5) / 2), each while m <= 16.
 * Errors: DG_EINVAL (m < k + 1), DG_EUNSUPPORTED (other m, per-cell / full D set, multilinear
 * geometry set: its m is dg_set_geometry's). */
int dg_set_quadrature(dg_ctx* ctx, int m);

/* ---- matrix-based comparison (the paper's "matrix-based" columns of
 * Table 1: "we also assemble the matrix of the operator (again using our sum-factorized
 * implementation) and apply the resulting matrix to a vector") ----
 * Single-rank contexts only (DG_EUNSUPPORTED otherwise).
 *
 * Layout (block stencil, caller-owned DEVICE array of dg_matrix_size doubles): for every local
 * cell S in cell-major order 7 blocks of n^3 x n^3 doubles; slot 0 = A_{S,S}, slot 1 + f =
 * A_{S,T_f}, T_f the face-f neighbour (f = 2q + s as for the halo faces, wrapped on periodic
 * directions); each block COLUMN-major with leading dimension ld = n^3 rounded up to even:
 * A[((S * 7 + slot) * n^3 + j) * ld + i] is the entry of row (S, i) and column (T_slot, j); for
 * odd n^3 row i = n^3 is a zero pad (16-byte aligned columns). Slots with no neighbour (Dirichlet
 * side) and slots whose neighbour already occurs in an earlier slot (1 or 2 cells along a
 * periodic direction) are zero. 7 n^3 ld doubles per cell: 14.7 MB at k = 7. */
int dg_matrix_size(const dg_ctx* ctx, int64_t* ndoubles);
/* Assemble the operator the next dg_apply would apply (constant or per-cell D, velocity field,
 * quadrature, affine map) into A: every column is a probe of the fused sum-factorized kernel
 * with unit vectors on a colour class of cells whose closed face neighbourhoods are disjoint
 * (27 to 125 classes x n^3 probes). Allocates two ndofs scratch vectors; synchronous on stream.
 * Errors: DG_EINVAL, DG_ENOMEM, DG_ECUDA, DG_EUNSUPPORTED (nranks > 1). */
int dg_assemble(dg_ctx* ctx, double* A, void* stream);
/* y = A z with an assembled A (the matrix-based operator application): per cell
 * y_S = sum_slot A_{S,T_slot} z_{T_slot}; enqueued on stream (meshes with few row blocks use a
 * library-owned scratch of 7 x rows doubles, allocated at the first call). Errors: DG_EINVAL
 * (null, y == z), DG_ENOMEM, DG_ECUDA, DG_EUNSUPPORTED (nranks > 1). */
int dg_matrix_apply(dg_ctx* ctx, const double* A, const double* z, double* y, void* stream);

/* ---- halo plumbing (multi-rank; also used by the single-process loopback test) ----
 * face f = 2q + s (q = direction, s = 0 low / 1 high side of this rank's box).
 * neighbor_rank = -1 when the face lies on the domain boundary. The halo is the face traces of
 * for every cell of the face layer, the normal-first
 * contraction of its block u(a,b) = sum_e theta_e(s) z(e; a,b) and
 * d(a,b) = sum_e theta'_e(s) z(e; a,b) over the tangential modal indices (a along the lower
 * tangential direction t1, b along t2): [cell t1 + N_t1 t2][u | d][a + n b], 2 n^2 doubles per
 * cell (1/4 of the block at k = 7); the receiving rank runs the tangential stages.
 * count = doubles per face = cells of the face layer x 2 n^2. */
int dg_halo_info(const dg_ctx* ctx, int face, int* neighbor_rank, int64_t* count);
/* which = 0: send buffer (this rank's own boundary layer, filled by dg_halo_pack),
   which = 1: receive buffer (the neighbour's layer adjacent to this face, read by the kernel),
   which = 2 / 3: the same for the per-cell diffusion field (6 doubles per layer cell;
   count / n^3 * 6 doubles; allocated by dg_set_diffusion, NULL before). */
int dg_halo_buffer(dg_ctx* ctx, int face, int which, double** ptr);
/* Fill the send buffers (which = 0) with the face traces of z (the kernel dg_apply runs on its
   comm stream before the exchange). */
int dg_halo_pack(dg_ctx* ctx, const double* z, void* stream);

/* ---- seeded inputs (reading C-13; identical to paper_1711_10885_b200/inputs.py) ----
 * dst[i] = U(seed, offset + i), i < count, on device memory. */
int dg_fill_uniform(double* dst, int64_t count, uint64_t seed, int64_t offset, void* stream);
/* Fill this rank's local vector with the values of the GLOBAL DOF indices it owns. */
int dg_fill_uniform_local(dg_ctx* ctx, double* dst, uint64_t seed, void* stream);

/* Per-cell inputs of this rank's cells: dst[per_cell * l + i] = U(seed, per_cell * e + i) for
   local cell l with GLOBAL cell index e (e.g. per_cell = 6 for the Problem A tensor field,
   paper_1711_10885_b200/inputs.py). */
int dg_fill_uniform_cells(dg_ctx* ctx, double* dst, int per_cell, uint64_t seed, void* stream);

/* Create a 128-byte ncclUniqueId (rank 0 calls this and broadcasts it). */
int dg_nccl_unique_id(void* out128);
/* Create a 128-byte id of an in-process fabric group: pass the same id to dg_setup of every
   rank (threads of this process, one context each; each rank's applies on its own thread).
   A rank's exchange blocks its thread until its neighbours reach the same exchange (120 s
   timeout -> DG_ENCCL). */
int dg_fabric_id(void* out128);
/* The same, but the group's applies use the DIRECT (fused) halo: each rank's trace pack kernel
   stores the partition faces' traces straight into the neighbour's receive buffer (no send buffer,
   no copy), ordered by events (see dg_p2p_import). Setup-time exchanges still copy. */
int dg_fabric_id_direct(void* out128);

/* ---- direct (fused) halo between PROCESSES (one per GPU): the trace pack kernel stores every
 * partition face's traces straight into the neighbour rank's receive buffer over NVLink, through a
 * CUDA IPC mapping of that buffer: the compute step and the transfer are one kernel, with no send
 * buffer and no collective (SURVEY 8(e) "fused collective"). Per apply: the pack waits on the
 * neighbours' "consumed" events of the previous apply (write-after-read), records "packed"; the
 * shell cells wait on the neighbours' "packed" events and record "consumed"; counters in a POSIX
 * shared-memory segment order every record before the peers' waits (no kernel waits on another).
 * Setup-time exchanges (dg_set_diffusion) keep NCCL. Usage, after dg_setup on every rank (with an
 * ncclUniqueId): blob = dg_p2p_blob_bytes() bytes from dg_p2p_export; all-gather the blobs in rank
 * order; dg_p2p_import(ctx, all_blobs, shm_name) with a name common to the ranks ("/..."; rank 0
 * creates the segment). Collective; synchronous.
 * Errors: DG_EINVAL (not partitioned, in-process fabric, import before export or twice),
 * DG_ECUDA (IPC handles / events), DG_ENCCL (shared memory, timeout). */
size_t dg_p2p_blob_bytes(void);
int dg_p2p_export(dg_ctx* ctx, void* blob);
int dg_p2p_import(dg_ctx* ctx, const void* blobs, const char* shm_name);

/* The halo transport of this context: transport 0 = none (single rank or DG_HALO_EXTERNAL only),
   1 = NCCL, 2 = in-process fabric (copies), 3 = in-process fabric, direct (fused pack into the
   peers' buffers), 4 = direct over CUDA IPC (fused pack storing over NVLink; NCCL for setup-time
   exchanges); nranks = the communicator's rank count as NCCL reports it (ncclCommCount), else the
   dg_setup nranks. */
int dg_comm_info(const dg_ctx* ctx, int* transport, int* nranks);

/* Overlap evidence for the partitioned apply (the face-trace exchange concurrent with
   the inner-box cells). arm = 1: the next dg_apply / dg_residual of this
   (partitioned) context records timing events around its launches. arm = 0: waits for that apply
   and writes n >= 6 times in ms, relative to the apply's start on the caller's stream:
   ms[0] / ms[1] the trace pack (+ exchange) begin / end on the comm stream (begin before the waits
   on the neighbours' buffers), ms[2] / ms[3] the inner-box kernel begin / end, ms[4] the shell
   kernel's start (after its wait for the received traces; after the inner box on the caller's
   stream, or concurrent with it on the comm stream with DG_SHELL_STREAM=1), ms[5] its end.
   DG_EUNSUPPORTED for a
   single-rank context, DG_EINVAL when no armed apply has run or n < 6. */
int dg_timeline(dg_ctx* ctx, int arm, double* ms, int n);

/* Library / kernel facts for the harness: kernel launches per dg_apply, threads and
   cells per CTA, dynamic shared memory per CTA, registers per thread, of the kernel the
   next apply launches (the general-coefficient kernel after dg_set_diffusion / full D). */
typedef struct {
    int launches_per_apply;
    int cells_per_cta;
    int threads_per_cta;
    int smem_bytes;
    int regs_per_thread;
    int ctas_per_sm;
} dg_kernel_info;
int dg_get_kernel_info(const dg_ctx* ctx, dg_kernel_info* info);

#ifdef __cplusplus
}
#endif
#endif /* DG_B200_H */

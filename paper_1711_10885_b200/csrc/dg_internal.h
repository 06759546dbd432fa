// Internal declarations shared by the CUDA translation units of libdg_b200.so.
// (Product path only; nothing here is shared with oracle/.)
#pragma once
#include <cstdint>
#include <cuda.h>            // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>

namespace dg {

// Device-side bounds checks of the debug build (-DDG_CHECK; tools/check_build.py): a violated
// index traps the kernel, so the GPU test suite run against that build is a memcheck of the
// cell / neighbour / ghost / TMA indexing (compute-sanitizer is unavailable on the GPU pool).
#ifdef DG_CHECK
#define DG_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define DG_ASSERT(c) do { } while (0)
#endif

constexpr int KMAX = 10;
constexpr int NMAX = KMAX + 1;
constexpr int MMAX = 18;          // Gauss points per direction: up to q = 3p + 4 at p = 10

// Symmetric positive SEMI-definite test of a row-major 3x3 tensor (the diffusion tensor of
// eq:modelproblem; D = 0 is admitted): finite, exactly
// symmetric, and all seven principal minors of D / max|D_ij| >= -1e-13 (a symmetric matrix is
// PSD iff every principal minor is >= 0; the tolerance admits rounding in semi-definite inputs).
__host__ __device__ inline bool psd3(const double* d)
{
    double s = 0.0;
    for (int i = 0; i < 9; ++i) {
        if (!(d[i] - d[i] == 0.0)) return false;              // NaN / inf
        s = fmax(s, fabs(d[i]));
    }
    if (d[1] != d[3] || d[2] != d[6] || d[5] != d[7]) return false;
    if (s == 0.0) return true;
    const double a = d[0] / s, b = d[4] / s, c = d[8] / s, x = d[1] / s, y = d[2] / s, z = d[5] / s;
    const double tol = -1e-13;
    if (a < tol || b < tol || c < tol) return false;
    if (a * b - x * x < tol || a * c - y * y < tol || b * c - z * z < tol) return false;
    const double det = a * (b * c - z * z) - x * (x * c - z * y) + y * (x * z - b * y);
    return det >= tol;
}

// 1D tables for one degree (host side, double). Built by tables.cpp.
struct HostTables {
    int n, m;                // basis size n = k+1, Gauss points per direction m (>= n)
    double xi[MMAX], w[MMAX];
    double V[MMAX][NMAX];    // V[i][j]  = theta_j(xi_i)                    (A^(q) of eq:evalfe)
    double Dc[MMAX][MMAX];   // Dc[i][l] = L'_l(xi_i): collocation derivative at the Gauss points
    double L0[MMAX], L1[MMAX];    // L_l(0), L_l(1): Lagrange basis at the Gauss points, at the endpoints
    double LD0[MMAX], LD1[MMAX];  // L'_l(0), L'_l(1)
    double th0[NMAX], th1[NMAX];  // theta_j(0), theta_j(1)       (B^(d) of PAPER.md:528-545)
    double dth0[NMAX], dth1[NMAX];// theta'_j(0), theta'_j(1)
    double G[MMAX][NMAX];    // G[i][j]  = theta'_j(xi_i)   (reference derivative, modal -> Gauss points)
};
int build_tables(int k, HostTables* t);
int build_tables_m(int k, int m, HostTables* t);

// Per-launch parameters (passed by value; lands in the kernel parameter constant bank).
struct KParams {
    const double* z;
    double* y;
    const double* f;          // epi 1: y = f - A z; epi 2: the f of the SSP stage (nullptr = 0)
    const double* w;          // epi 2: the a w term (nullptr = 0)
    double ea, eb, es;        // epi 2: y = ea w + eb (z + es (f - A z)), es = dt / Delta_T
    int epi;                  // store epilogue: 0 y = A z, 1 residual, 2 SSP-RK stage
    const double* ghost[6];   // neighbour-rank face traces per face 2q+s: [layer cell][u | d][n^2] (nullptr: none)
    const int64_t* task_list; // local linear cell ids (nullptr -> task box)
    int64_t ntasks;
    int64_t task_lo[3], task_cnt[3];
    unsigned dmag[2], dsh[2]; // magic division by task_cnt[2] and by TRAV_TY * task_cnt[0] (decode_task)
    int64_t nloc[3];          // local cell counts
    int64_t gofs[3];          // global index of local cell (0,0,0)
    int64_t gcells[3];        // global cell counts
    double hinv[3];
    double Dhat[9];           // D_rs / (h_r h_s)
    double kb[3];             // b_r / h_r
    double c;
    double dT;                // Delta_T = h1 h2 h3
    double dF[3];             // Delta_F,q = prod_{r != q} h_r
    double Dqq_h[3];          // D_qq / h_q   (normal flux scale)
    double gam[3];            // gamma = <D_qq, D_qq> sigma = D_qq sigma
    double bq[3];             // b_q
    unsigned mask;
    int per[3];               // direction q periodic (every cell has both q-neighbours; NEXT-1)
    int wrap[3];              // periodic AND unpartitioned along q: the wrap neighbour is local
    // general-coefficient kernel (full / per-cell D; NEXT-1):
    const double* Dfield;     // [local cell][6] = D00 D11 D22 D01 D02 D12
    const double* Dghost[6];  // neighbour-rank layers of Dfield per face (nullptr: none)
    double sigma;
    double sigq[3];           // penalty factor per face direction (sigma / |J^-T e_q| on an affine mesh)
    double h[3];
    // variable-velocity kernel (NEXT-2/3):
    int bkind;                // 0 constant b, 1 Taylor-Green field, 2 linear (x2, x3, x1)
    double bamp[3];           // per-component amplitude of the field
    double lo[3];             // physical coordinates of the global box's low corner
    // TMA staging of the x-direction cell blocks (n = 8 fast kernel): z and y viewed as
    // [cells * 64 rows][8 doubles] with the 64-byte swizzle
    int tma;                  // n = 8: 1 tmz (loads) valid, 2 tmy (store) valid too; other n: 2 = bulk copies
    CUtensorMap tmz, tmy;
    // multilinear-geometry kernel (NEXT-3, dg_geo.cuh): the padded vertex grid of this rank's box
    // ((nloc+3)^3 x 3 doubles, local vertex -1 .. nloc+1) and the physical D, b
    const double* vert;
    double Dp[9];
    double bp[3];
    int ghosts;               // this launch covers cells with a neighbour on another rank (the shell launch)
    // variable-velocity kernel: the 1D velocity tables (fields at the end keep the offsets above)
    const double* vtab;       // per direction d, local cell i: [x | sin x | cos x | 1][m + 2 points] (vel_table_kernel)
    int64_t vtoff[3];         // offset of direction d's tables in vtab
};

struct LaunchInfo {
    int cells_per_cta, threads, smem, regs, ctas_per_sm;
};

// Per-degree launchers (one translation unit per n, dg_cell_n<N>.cu).
int upload_tables(int k, const HostTables& t);          // to this device's __constant__ bank
cudaError_t launch_cell(int k, const KParams& p, cudaStream_t s);
cudaError_t launch_gen(int k, const KParams& p, cudaStream_t s);      // general-coefficient kernel
// variable-velocity / over-integrated kernel for (k, m), m in {k+1, k+3}, k <= 8 (dg_vb.cuh)
bool vb_available(int k, int m);
int upload_tables_vb(int k, int m, const HostTables& t);
cudaError_t launch_vb(int k, int m, const KParams& p, cudaStream_t s);
int vb_launch_info(int k, int m, LaunchInfo* info);
int cell_launch_info(int k, LaunchInfo* info);
// 2D tensor map [rows][8 doubles] (64-byte rows, box 64 x 8, 64-byte swizzle) over ptr; false if unavailable
bool make_row_map(CUtensorMap* map, const double* ptr, int64_t rows);
int gen_launch_info(int k, LaunchInfo* info);
// multilinear-geometry kernel for (k, m) (dg_geo.cuh; pairs in dg_dispatch.cpp)
bool geo_available(int k, int m);
int upload_tables_geo(int k, int m, const HostTables& t);
cudaError_t launch_geo(int k, int m, const KParams& p, cudaStream_t s);
int geo_launch_info(int k, int m, LaunchInfo* info);

// Halo / inputs kernels (dg_aux.cu).
struct TraceArgs {              // face-trace halo of the partition faces (trace_pack_kernel)
    double* dst[6];             // send buffer of face f (nullptr: no neighbour rank)
    int64_t start[7];           // prefix sums of the work items (layer cells x n^2) per face
    double th[2][NMAX], dth[2][NMAX];   // theta_j(s), theta'_j(s), s = 0, 1
};
struct GeoPts { int m; double xi[MMAX]; };
// 1D velocity tables of the variable-velocity kernel: for every direction d and local cell index i,
// x, sin x, cos x, 1 at the m Gauss coordinates and the two endpoints (x = lo + (gofs + i + xr) h)
cudaError_t launch_vel_tables(double* out, const int64_t nloc[3], const int64_t gofs[3], const double lo[3],
                              const double h[3], const GeoPts& g, cudaStream_t s);   // the m-point Gauss rule of dg_set_geometry's check
cudaError_t launch_geo_check(const double* vert, const int64_t nloc[3], const GeoPts& g, int* bad, cudaStream_t s);
cudaError_t launch_trace_pack(const double* z, const TraceArgs& a, int n, const int64_t nloc[3], cudaStream_t s);
cudaError_t launch_pack(const double* z, double* dst, int n3, const int64_t nloc[3], int face, cudaStream_t s);
cudaError_t launch_dfield_pack(const double* D9, double* D6, int* bad, int64_t ncell, const double* Jinv,
                               double det, cudaStream_t s);
cudaError_t launch_dfield_const(double* D6, const double D9[9], int64_t ncell, cudaStream_t s);
// matrix-based comparison (dg_matrix.cu, NEXT-4)
void matrix_colours(const int64_t nloc[3], const int per[3], int ncol[3], bool present[3][5]);
cudaError_t launch_probe_set(double* z, int n3, const int64_t nloc[3], const int per[3], const int col[3], int j,
                             double val, cudaStream_t s);
cudaError_t launch_probe_tasks(const int64_t nloc[3], const int per[3], const int col[3], int64_t* list,
                               unsigned long long* count, cudaStream_t s);
cudaError_t launch_probe_scatter(double* A, const double* y, double* z, const int64_t* tasks, int64_t ntask, int n3,
                                 const int64_t nloc[3], const int per[3], const int col[3], int j, int nj,
                                 cudaStream_t s);
int64_t matrix_scratch_doubles(int n3, int64_t ncell);
cudaError_t launch_matrix_apply(const double* A, const double* z, double* y, double* scratch, int n3,
                                const int64_t nloc[3], const int per[3], cudaStream_t s);
cudaError_t launch_fill_uniform(double* dst, int64_t count, uint64_t seed, int64_t offset, cudaStream_t s);
cudaError_t launch_fill_uniform_local(double* dst, int n3, const int64_t nloc[3], const int64_t gofs[3],
                                      const int64_t gcells[3], uint64_t seed, cudaStream_t s);

}  // namespace dg

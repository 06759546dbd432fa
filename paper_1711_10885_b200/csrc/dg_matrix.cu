// Matrix-based comparison (Table 1 "matrix-based"
// columns): assembly of A by probing the matrix-free operator, and the block-stencil matvec.
//
// Layout of the assembled matrix (include/dg.h, dg_matrix_size): for every local cell S
// (cell-major order, C-3) 7 blocks of n^3 x n^3, slot 0 = A_{S,S}, slot 1 + f = A_{S,T_f} with
// T_f the face-f neighbour of S (f = 2q + s, s = 0 low, 1 high; wrapped on periodic
// directions). Each block is stored COLUMN-major with the leading dimension ld = n^3 rounded up
// to even, A[((S * 7 + slot) * n3 + j) * ld + i] = A_{(S,i),(T,j)} (row i = n^3 of an odd n^3 is
// a zero pad): the probe of column j writes a contiguous run, the matvec thread of rows i, i + 1
// reads 16 aligned bytes and a warp's reads are contiguous. A slot without a neighbour (domain
// boundary) or whose neighbour already appears in an earlier slot (1 or 2 cells along a
// periodic direction) holds zeros.
//
// Assembly: a_h is linear in its trial argument and the support of column (T, j) is T and its
// six face neighbours, so every cell of a colour class whose closed neighbourhoods are
// disjoint can be probed at once: z = sum_{T of colour c} e_(T,j), y = A z by the fused
// kernel (launched over the cells next to colour c only, a task list), and y_S is column j of
// the block (S, T) for the one T of colour c next to S. The
// colouring is i mod 3 per direction, the r = N mod 3 trailing cells of a periodic direction
// getting colours 3, 4 of their own (a wrap neighbour pair would otherwise share a colour).
#include "dg_internal.h"

#ifndef DG_MU
#define DG_MU 8      // matrix copies per thread and ring stage (16 with 8-byte copies)
#endif
#ifndef DG_MNS
#define DG_MNS 2     // stages of the cp.async ring (measured at U = 8: 2 > 3 > 4 > 6)
#endif

namespace dg {

struct MatGeom {
    int64_t nloc[3];
    int per[3];
    int64_t tail[3];     // first cell of the periodic tail (nloc when there is none)
};

__device__ __forceinline__ int mcolour(const MatGeom& g, int q, int64_t i)
{
    return i < g.tail[q] ? (int)(i % 3) : 3 + (int)(i - g.tail[q]);
}

__device__ __forceinline__ int64_t mstep(int64_t c, int64_t N, int per, int d, bool* ok)
{
    c += d;
    if (c < 0 || c >= N) {
        if (!per) *ok = false;
        c = c < 0 ? c + N : c - N;
    }
    return c;
}

// the cell in slot `slot` of S (-1: no neighbour); its coordinates in cc (optional)
__device__ __forceinline__ int64_t mneighbour(const MatGeom& g, int64_t S, int slot, int64_t* cc)
{
    int64_t x = S % g.nloc[0];
    int64_t y = (S / g.nloc[0]) % g.nloc[1];
    int64_t z = S / (g.nloc[0] * g.nloc[1]);
    bool ok = true;
    const int d = (slot & 1) ? -1 : 1;         // slot 1 + f: f even (low side) -> -1
    if (slot == 1 || slot == 2) x = mstep(x, g.nloc[0], g.per[0], d, &ok);
    else if (slot == 3 || slot == 4) y = mstep(y, g.nloc[1], g.per[1], d, &ok);
    else if (slot == 5 || slot == 6) z = mstep(z, g.nloc[2], g.per[2], d, &ok);
    if (!ok) return -1;
    if (cc) { cc[0] = x; cc[1] = y; cc[2] = z; }
    return x + g.nloc[0] * (y + g.nloc[1] * z);
}

__device__ __forceinline__ bool has_colour(const MatGeom& g, const int64_t c[3], const int col[3])
{
    return mcolour(g, 0, c[0]) == col[0] && mcolour(g, 1, c[1]) == col[1] && mcolour(g, 2, c[2]) == col[2];
}

// z[(T, j)] = val for every cell T of colour col
__global__ void probe_set_kernel(double* z, int n3, MatGeom g, int c0, int c1, int c2, int j, double val)
{
    const int64_t ncell = g.nloc[0] * g.nloc[1] * g.nloc[2];
    const int col[3] = {c0, c1, c2};
    for (int64_t T = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; T < ncell; T += (int64_t)gridDim.x * blockDim.x) {
        int64_t c[3];
        mneighbour(g, T, 0, c);
        if (has_colour(g, c, col)) z[T * n3 + j] = val;
    }
}

// The cells whose closed face neighbourhood holds a cell of colour col (the only cells whose y
// a probe of that colour changes): appended to list (order irrelevant: cells are independent).
__global__ void probe_tasks_kernel(MatGeom g, int c0, int c1, int c2, int64_t* __restrict__ list,
                                   unsigned long long* __restrict__ count)
{
    const int64_t ncell = g.nloc[0] * g.nloc[1] * g.nloc[2];
    const int col[3] = {c0, c1, c2};
    for (int64_t S = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; S < ncell; S += (int64_t)gridDim.x * blockDim.x) {
        int64_t c[3];
        bool hit = false;
        for (int s = 0; s < 7 && !hit; ++s)
            if (mneighbour(g, S, s, c) >= 0 && has_colour(g, c, col)) hit = true;
        if (hit) list[atomicAdd(count, 1ull)] = S;
    }
}

// Column j of the blocks (S, T), T of colour col, from y = A z, over the task-list cells
// (those next to colour col); threads of row 0 also clear the probe entries of (col, j) in z
// and set (col, nj) (nj < 0: none).
__global__ void probe_scatter_kernel(double* __restrict__ A, const double* __restrict__ y, double* __restrict__ z,
                                     const int64_t* __restrict__ tasks, int64_t ntask, int n3, MatGeom g, int c0,
                                     int c1, int c2, int j, int nj)
{
    const int ld = n3 + (n3 & 1);
    const int col[3] = {c0, c1, c2};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntask * n3; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = t / n3;
        const int i = (int)(t - q * n3);
        const int64_t S = tasks[q];
        int64_t c[3];
        int slot = -1;
        for (int s = 0; s < 7 && slot < 0; ++s) {
            if (mneighbour(g, S, s, c) < 0) continue;
            if (has_colour(g, c, col)) slot = s;
        }
        if (slot >= 0) A[((S * 7 + slot) * n3 + j) * (int64_t)ld + i] = y[S * n3 + i];
        if (i == 0 && slot == 0) {
            z[S * n3 + j] = 0.0;
            if (nj >= 0) z[S * n3 + nj] = 1.0;
        }
    }
}

// y_S = sum_slot A_{S, T_slot} z_{T_slot}: two consecutive (padded) rows (S, i), (S, i + 1)
// per thread, so a warp's matrix reads are 512-byte contiguous runs of the column-major blocks.
// The matrix is streamed once from HBM by per-thread 16-byte asynchronous copies (LDGSTS,
// cp.async.cg) through an NS-stage shared-memory ring: every thread keeps NS - 1 chunks of U
// copies in flight however the compiler schedules (with plain loads ptxas interleaved each
// load with its FMA: 2 in flight, 4.2 TB/s; 8-byte copies of an unpadded odd n^3 reached
// 4.2 TB/s too). The (slot, column-chunk) sequence runs through the slots without draining the
// pipeline; a slot without a neighbour copies nothing (zero fill) and multiplies the cell's own
// z. z comes through L1 (the lanes of a warp read the same entry of the same neighbour block).
__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes, int src_bytes)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ int64_t pick7(const int64_t (&T)[7], int s)
{
    int64_t v = T[0];
#pragma unroll
    for (int q = 1; q < 7; ++q) v = (s == q) ? T[q] : v;
    return v;
}

constexpr int MTHREADS = 128;

// Slot split (small grids): CTA (b, p) handles the slots [p * 7 / nsplit, (p + 1) * 7 / nsplit)
// of row block b and writes its partial sums to part + p * nrow (scratch, padded rows);
// matrix_reduce_kernel adds the nsplit partials in a fixed order (deterministic).
template <int U, int NS>
__global__ void __launch_bounds__(MTHREADS) matrix_apply_async_kernel(const double* __restrict__ A,
                                                                      const double* __restrict__ z,
                                                                      double* __restrict__ y, double* __restrict__ part,
                                                                      int n3, MatGeom g, int64_t nrow, int nsplit)
{
    extern __shared__ __align__(16) double sbuf[];
    const int tid = threadIdx.x;
    const int ld = n3 + (n3 & 1);
    const int p = blockIdx.y;
    const int s0 = p * 7 / nsplit, s1 = (p + 1) * 7 / nsplit;
    const int64_t r = (blockIdx.x * (int64_t)MTHREADS + tid) * 2;     // padded row index
    if (r >= nrow) return;
    const int64_t S = r / ld;
    const int i = (int)(r - S * ld);
    int64_t T[7];
    unsigned has = 0;
#pragma unroll
    for (int s = 0; s < 7; ++s) {
        T[s] = mneighbour(g, S, s, nullptr);
        if (T[s] >= 0) has |= 1u << s; else T[s] = S;
    }
    const int CPS = (n3 + U - 1) / U;
    const int K = (s1 - s0) * CPS;
    const double* arow = A + S * 7 * (int64_t)n3 * ld + i;
    double* my = sbuf + tid * 2;
    auto issue = [&](int k) {
        const int s = s0 + k / CPS, j0 = (k % CPS) * U;
        const bool hs = (has >> s) & 1u;
        const double* a = arow + ((int64_t)s * n3 + j0) * ld;
        double* dst = my + (k % NS) * U * MTHREADS * 2;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = hs && (j0 + u < n3);
            cp_async(dst + u * MTHREADS * 2, ok ? (const void*)(a + (int64_t)u * ld) : (const void*)A, 16, ok ? 16 : 0);
        }
        cp_commit();
    };
    double acc[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
#pragma unroll
    for (int k = 0; k < NS - 1; ++k) {
        if (k < K) issue(k);
        else cp_commit();
    }
    for (int k = 0; k < K; ++k) {
        if (k + NS - 1 < K) issue(k + NS - 1);
        else cp_commit();
        cp_wait<NS - 1>();
        const int s = s0 + k / CPS, j0 = (k % CPS) * U;
        const double* zt = z + pick7(T, s) * n3 + j0;
        const double2* src = reinterpret_cast<const double2*>(my + (k % NS) * U * MTHREADS * 2);
        if (j0 + U <= n3) {
            double zj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) zj[u] = __ldg(zt + u);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double2 v = src[u * MTHREADS];
                acc[0][u & 3] = fma(v.x, zj[u], acc[0][u & 3]);
                acc[1][u & 3] = fma(v.y, zj[u], acc[1][u & 3]);
            }
        } else {
            for (int u = 0; u < n3 - j0; ++u) {
                const double zj = __ldg(zt + u);
                const double2 v = src[u * MTHREADS];
                acc[0][0] = fma(v.x, zj, acc[0][0]);
                acc[1][0] = fma(v.y, zj, acc[1][0]);
            }
        }
    }
    const double y0 = (acc[0][0] + acc[0][1]) + (acc[0][2] + acc[0][3]);
    const double y1 = (acc[1][0] + acc[1][1]) + (acc[1][2] + acc[1][3]);
    if (part) {
        *reinterpret_cast<double2*>(part + p * nrow + r) = make_double2(y0, y1);
    } else {
        y[S * n3 + i] = y0;
        if (i + 1 < n3) y[S * n3 + i + 1] = y1;
    }
}

static MatGeom make_geom(const int64_t nloc[3], const int per[3])
{
    MatGeom g;
    for (int q = 0; q < 3; ++q) {
        g.nloc[q] = nloc[q];
        g.per[q] = per[q];
        g.tail[q] = (per[q] && nloc[q] % 3) ? 3 * (nloc[q] / 3) : nloc[q];
    }
    return g;
}

void matrix_colours(const int64_t nloc[3], const int per[3], int ncol[3], bool present[3][5])
{
    const MatGeom g = make_geom(nloc, per);
    for (int q = 0; q < 3; ++q) {
        ncol[q] = 5;
        for (int v = 0; v < 5; ++v)
            present[q][v] = v < 3 ? (v < g.tail[q]) : (v - 3 < g.nloc[q] - g.tail[q]);
    }
}

static int grid_for(int64_t work, int threads)
{
    int64_t b = (work + threads - 1) / threads;
    if (b > 148 * 64) b = 148 * 64;
    return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_probe_set(double* z, int n3, const int64_t nloc[3], const int per[3], const int col[3], int j,
                             double val, cudaStream_t s)
{
    const MatGeom g = make_geom(nloc, per);
    const int64_t ncell = nloc[0] * nloc[1] * nloc[2];
    probe_set_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(z, n3, g, col[0], col[1], col[2], j, val);
    return cudaGetLastError();
}

cudaError_t launch_probe_tasks(const int64_t nloc[3], const int per[3], const int col[3], int64_t* list,
                               unsigned long long* count, cudaStream_t s)
{
    const MatGeom g = make_geom(nloc, per);
    const int64_t ncell = nloc[0] * nloc[1] * nloc[2];
    const cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    probe_tasks_kernel<<<grid_for(ncell, 256), 256, 0, s>>>(g, col[0], col[1], col[2], list, count);
    return cudaGetLastError();
}

cudaError_t launch_probe_scatter(double* A, const double* y, double* z, const int64_t* tasks, int64_t ntask, int n3,
                                 const int64_t nloc[3], const int per[3], const int col[3], int j, int nj,
                                 cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    const MatGeom g = make_geom(nloc, per);
    probe_scatter_kernel<<<grid_for(ntask * n3, 256), 256, 0, s>>>(A, y, z, tasks, ntask, n3, g, col[0], col[1], col[2],
                                                                   j, nj);
    return cudaGetLastError();
}

__global__ void matrix_reduce_kernel(const double* __restrict__ part, double* __restrict__ y, int n3, int64_t nrow,
                                     int nsplit)
{
    const int ld = n3 + (n3 & 1);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrow; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t S = r / ld;
        const int i = (int)(r - S * ld);
        if (i >= n3) continue;
        double v = part[r];
        for (int p = 1; p < nsplit; ++p) v += part[p * nrow + r];
        y[S * n3 + i] = v;
    }
}

template <int U, int NS>
static cudaError_t launch_async(const double* A, const double* z, double* y, double* scratch, int n3,
                                const MatGeom& g, int64_t nrow, cudaStream_t s)
{
    const int64_t blocks = (nrow / 2 + MTHREADS - 1) / MTHREADS;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    const int smem = NS * U * MTHREADS * 2 * (int)sizeof(double);
    auto kern = matrix_apply_async_kernel<U, NS>;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int nsplit = scratch ? 7 : 1;
    kern<<<dim3((unsigned)blocks, nsplit), MTHREADS, smem, s>>>(A, z, y, scratch, n3, g, nrow, nsplit);
    if (scratch) {
        int64_t rb = (nrow + 255) / 256;
        if (rb > 148 * 16) rb = 148 * 16;
        matrix_reduce_kernel<<<(unsigned)rb, 256, 0, s>>>(scratch, y, n3, nrow, nsplit);
    }
    return cudaGetLastError();
}

// Split the slots over 7 CTAs when the row blocks alone fill fewer than ~8 waves of the GPU
// (few large cells: each row block streams 7 n^3 x 256 doubles, 14 MB at k = 10).
int64_t matrix_scratch_doubles(int n3, int64_t ncell)
{
    const int64_t nrow = ncell * (n3 + (n3 & 1));
    const int64_t blocks = (nrow / 2 + MTHREADS - 1) / MTHREADS;
    const int64_t resident = 148 * 6;
    return blocks < 8 * resident ? 7 * nrow : 0;
}

cudaError_t launch_matrix_apply(const double* A, const double* z, double* y, double* scratch, int n3,
                                const int64_t nloc[3], const int per[3], cudaStream_t s)
{
    const MatGeom g = make_geom(nloc, per);
    const int64_t nrow = nloc[0] * nloc[1] * nloc[2] * (n3 + (n3 & 1));
    if (nrow == 0) return cudaSuccess;
    return launch_async<DG_MU, DG_MNS>(A, z, y, scratch, n3, g, nrow, s);
}

}  // namespace dg

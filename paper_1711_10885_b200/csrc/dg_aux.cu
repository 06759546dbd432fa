// Auxiliary kernels: halo packing (face traces of the partition layers; per-cell field layers)
// and the counter-based input generator (reading C-13; identical to inputs.py).
#include "dg_internal.h"

namespace dg {

// Per-cell data of a boundary layer (the diffusion-tensor field, n3 = 6 doubles per cell):
// face f = 2q + s: the layer lc[q] = (s ? nloc[q]-1 : 0); cells ordered by the two
// tangential local coordinates (t1 fastest), t1 < t2, each a contiguous n3-block.
__global__ void pack_kernel(const double* __restrict__ z, double* __restrict__ dst, int n3, int64_t n0, int64_t n1,
                            int64_t n2, int q, int s, int64_t total)
{
    const int64_t nl[3] = {n0, n1, n2};
    const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cellk = i / n3, j = i - cellk * n3;
        int64_t lc[3];
        lc[t1] = cellk % nl[t1];
        lc[t2] = cellk / nl[t1];
        lc[q] = s ? nl[q] - 1 : 0;
        const int64_t e = lc[0] + n0 * (lc[1] + n1 * lc[2]);
        dst[i] = z[e * n3 + j];
    }
}

cudaError_t launch_pack(const double* z, double* dst, int n3, const int64_t nloc[3], int face, cudaStream_t s)
{
    const int q = face >> 1, sd = face & 1;
    const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
    const int64_t total = nloc[t1] * nloc[t2] * n3;
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pack_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, dst, n3, nloc[0], nloc[1], nloc[2], q, sd, total);
    return cudaGetLastError();
}

// Face-trace halo: for every partition face f = 2q + s with a
// neighbour rank, the normal-first contraction of this rank's boundary layer
//     u(a, b) = sum_e theta_e(s) z(e along q; a, b),   d(a, b) = sum_e theta'_e(s) z(...)
// for each layer cell (ordered t1 fastest, t1 < t2 the tangential directions) and tangential
// modal pair (a along t1, b along t2): 2 n^2 doubles per cell, [u | d] at a + n b, 1/4 of the
// block at k = 7. The receiving rank sees this cell across its face f^1 at x_q = s and runs the
// tangential stages itself (nb_load / nb_traces in dg_cell.cuh). The chain order (e = 0..n-1,
// fma) is the kernels' own, so a partitioned apply equals the single-rank one bit for bit.
__global__ void trace_pack_kernel(const double* __restrict__ z, TraceArgs a, int n, int64_t n0, int64_t n1, int64_t n2)
{
    const int64_t nl[3] = {n0, n1, n2};
    const int nn = n * n;
    const int64_t n3 = (int64_t)nn * n;
    const int64_t total = a.start[6];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int f = 0;
        while (i >= a.start[f + 1]) ++f;
        const int q = f >> 1, s = f & 1;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        const int64_t li = i - a.start[f];
        const int64_t cellk = li / nn;
        const int t = (int)(li - cellk * nn);
        const int ta = t % n, tb = t / n;
        int64_t lc[3];
        lc[t1] = cellk % nl[t1];
        lc[t2] = cellk / nl[t1];
        lc[q] = s ? nl[q] - 1 : 0;
        const double* blk = z + (lc[0] + n0 * (lc[1] + n1 * lc[2])) * n3;
        const int se = (q == 0) ? 1 : (q == 1) ? n : nn;
        const int base = (q == 0) ? n * ta + nn * tb : (q == 1) ? ta + nn * tb : ta + n * tb;
        double u = 0.0, d = 0.0;
        for (int e = 0; e < n; ++e) {
            const double v = __ldg(blk + base + e * se);
            u = fma(a.th[s][e], v, u);
            d = fma(a.dth[s][e], v, d);
        }
        double* o = a.dst[f] + cellk * 2 * nn;
        o[t] = u;
        o[nn + t] = d;
    }
}

cudaError_t launch_trace_pack(const double* z, const TraceArgs& a, int n, const int64_t nloc[3], cudaStream_t s)
{
    const int64_t total = a.start[6];
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    trace_pack_kernel<<<(unsigned)blocks, 256, 0, s>>>(z, a, n, nloc[0], nloc[1], nloc[2]);
    return cudaGetLastError();
}

__global__ void vel_table_kernel(double* __restrict__ out, int64_t n0, int64_t n1, int64_t n2, int64_t g0, int64_t g1,
                                 int64_t g2, double l0, double l1, double l2, double h0, double h1, double h2, GeoPts g)
{
    const int M2 = g.m + 2;
    const int64_t nl[3] = {n0, n1, n2}, go[3] = {g0, g1, g2};
    const double lo[3] = {l0, l1, l2}, h[3] = {h0, h1, h2};
    const int64_t total = (n0 + n1 + n2) * M2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int d = 0;
        int64_t r = t, off = 0;
        while (r >= nl[d] * M2) { r -= nl[d] * M2; off += nl[d] * 4 * M2; ++d; }
        const int64_t i = r / M2;
        const int e = (int)(r - i * M2);
        const double xr = (e < g.m) ? g.xi[e] : (double)(e - g.m);   // reference coordinate
        const double x = lo[d] + ((double)(go[d] + i) + xr) * h[d];
        double sn, cs;
        sincos(x, &sn, &cs);
        double* o = out + off + i * 4 * M2;
        o[0 * M2 + e] = x;
        o[1 * M2 + e] = sn;
        o[2 * M2 + e] = cs;
        o[3 * M2 + e] = 1.0;
    }
}

cudaError_t launch_vel_tables(double* out, const int64_t nloc[3], const int64_t gofs[3], const double lo[3],
                              const double h[3], const GeoPts& g, cudaStream_t s)
{
    const int64_t total = (nloc[0] + nloc[1] + nloc[2]) * (g.m + 2);
    if (total == 0) return cudaSuccess;
    vel_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(out, nloc[0], nloc[1], nloc[2], gofs[0], gofs[1],
                                                                     gofs[2], lo[0], lo[1], lo[2], h[0], h[1], h[2], g);
    return cudaGetLastError();
}

// Multilinear mesh check (dg_set_geometry): every local cell's Q1 map must be orientation
// preserving at all m^3 quadrature points and its 8 corners (det J > 0); *bad != 0 otherwise.
__global__ void geo_check_kernel(const double* __restrict__ vert, int64_t n0, int64_t n1, int64_t n2, GeoPts g,
                                 int* bad)
{
    const int64_t ncell = n0 * n1 * n2, PX = n0 + 3, PY = n1 + 3;
    const int npts = g.m * g.m * g.m + 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncell * npts;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i / npts;
        const int t = (int)(i - e * npts);
        const int64_t ix = e % n0, iy = (e / n0) % n1, iz = e / (n0 * n1);
        double xi[3];
        if (t < g.m * g.m * g.m) {
            xi[0] = g.xi[t % g.m];
            xi[1] = g.xi[(t / g.m) % g.m];
            xi[2] = g.xi[t / (g.m * g.m)];
        } else {
            const int c = t - g.m * g.m * g.m;
            xi[0] = c & 1; xi[1] = (c >> 1) & 1; xi[2] = c >> 2;
        }
        // vertex (i, j, k) of the cell's corner cube: padded index (ix + 1 + i, ...)
        auto X = [&](int a, int b, int c, int r) {
            return vert[(((iz + 1 + c) * PY + (iy + 1 + b)) * PX + (ix + 1 + a)) * 3 + r];
        };
        double J[3][3];
        for (int r = 0; r < 3; ++r) {
            double j0 = 0.0, j1 = 0.0, j2 = 0.0;
            for (int u = 0; u < 2; ++u)
                for (int v = 0; v < 2; ++v) {
                    const double bu1 = u ? xi[1] : 1.0 - xi[1], bv2 = v ? xi[2] : 1.0 - xi[2];
                    const double bu0 = u ? xi[0] : 1.0 - xi[0], bv1 = v ? xi[1] : 1.0 - xi[1];
                    j0 += bu1 * bv2 * (X(1, u, v, r) - X(0, u, v, r));
                    j1 += bu0 * bv2 * (X(u, 1, v, r) - X(u, 0, v, r));
                    j2 += bu0 * bv1 * (X(u, v, 1, r) - X(u, v, 0, r));
                }
            J[r][0] = j0; J[r][1] = j1; J[r][2] = j2;
        }
        const double det = J[0][0] * (J[1][1] * J[2][2] - J[2][1] * J[1][2]) -
                           J[0][1] * (J[1][0] * J[2][2] - J[2][0] * J[1][2]) +
                           J[0][2] * (J[1][0] * J[2][1] - J[2][0] * J[1][1]);
        if (!(det > 0.0)) atomicOr(bad, 1);
    }
}

cudaError_t launch_geo_check(const double* vert, const int64_t nloc[3], const GeoPts& g, int* bad, cudaStream_t s)
{
    const int64_t total = nloc[0] * nloc[1] * nloc[2] * (int64_t)(g.m * g.m * g.m + 8);
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    geo_check_kernel<<<(unsigned)blocks, 256, 0, s>>>(vert, nloc[0], nloc[1], nloc[2], g, bad);
    return cudaGetLastError();
}

__device__ __forceinline__ double splitmix_uniform(uint64_t g, uint64_t seed)
{
    uint64_t x = (seed << 40) + g + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (double)(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

__global__ void fill_kernel(double* dst, int64_t count, uint64_t seed, int64_t offset)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = splitmix_uniform((uint64_t)(offset + i), seed);
}

cudaError_t launch_fill_uniform(double* dst, int64_t count, uint64_t seed, int64_t offset, cudaStream_t s)
{
    if (count <= 0) return cudaSuccess;
    fill_kernel<<<148 * 8, 256, 0, s>>>(dst, count, seed, offset);
    return cudaGetLastError();
}

__global__ void fill_local_kernel(double* dst, int n3, int64_t n0, int64_t n1, int64_t n2, int64_t o0, int64_t o1,
                                  int64_t o2, int64_t g0, int64_t g1, uint64_t seed, int64_t total)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i / n3, j = i - e * n3;
        const int64_t lx = e % n0, ly = (e / n0) % n1, lz = e / (n0 * n1);
        const int64_t ge = (o0 + lx) + g0 * ((o1 + ly) + g1 * (o2 + lz));
        dst[i] = splitmix_uniform((uint64_t)(ge * n3 + j), seed);
    }
}

cudaError_t launch_fill_uniform_local(double* dst, int n3, const int64_t nloc[3], const int64_t gofs[3],
                                      const int64_t gcells[3], uint64_t seed, cudaStream_t s)
{
    const int64_t total = nloc[0] * nloc[1] * nloc[2] * n3;
    if (total <= 0) return cudaSuccess;
    fill_local_kernel<<<148 * 8, 256, 0, s>>>(dst, n3, nloc[0], nloc[1], nloc[2], gofs[0], gofs[1], gofs[2],
                                              gcells[0], gcells[1], seed, total);
    return cudaGetLastError();
}

}  // namespace dg

namespace dg {

// Per-cell tensors [cell][9] (row-major) -> [cell][6] = D00 D11 D22 D01 D02 D12 with
// validation: symmetric, finite, nonnegative diagonal (PSD necessary conditions); *bad != 0
// on violation (dg_set_diffusion returns DG_EINVAL).
struct Mat3 { double a[9]; };

__global__ void dfield_pack_kernel(const double* __restrict__ D9, double* __restrict__ D6, int* bad, int64_t ncell,
                                   int affine, Mat3 Ji, double det)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncell; e += (int64_t)gridDim.x * blockDim.x) {
        const double* d = D9 + 9 * e;
        if (!psd3(d)) atomicOr(bad, 1);   // symmetric PSD
        double m[9];
        for (int i = 0; i < 9; ++i) m[i] = d[i];
        if (affine) {                  // Dhat = |J| J^-1 D J^-T (reference-mesh tensor of an affine mesh)
            double t[9];
            for (int r = 0; r < 3; ++r)
                for (int s = 0; s < 3; ++s)
                    t[3 * r + s] = Ji.a[3 * r] * d[s] + Ji.a[3 * r + 1] * d[3 + s] + Ji.a[3 * r + 2] * d[6 + s];
            for (int r = 0; r < 3; ++r)
                for (int s = 0; s < 3; ++s)
                    m[3 * r + s] = det * (t[3 * r] * Ji.a[3 * s] + t[3 * r + 1] * Ji.a[3 * s + 1] +
                                          t[3 * r + 2] * Ji.a[3 * s + 2]);
        }
        double* o = D6 + 6 * e;
        o[0] = m[0]; o[1] = m[4]; o[2] = m[8]; o[3] = m[1]; o[4] = m[2]; o[5] = m[5];
    }
}

__global__ void dfield_const_kernel(double* __restrict__ D6, double d0, double d1, double d2, double d3, double d4,
                                    double d5, int64_t ncell)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncell; e += (int64_t)gridDim.x * blockDim.x) {
        double* o = D6 + 6 * e;
        o[0] = d0; o[1] = d1; o[2] = d2; o[3] = d3; o[4] = d4; o[5] = d5;
    }
}

static unsigned blocks_for(int64_t n)
{
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)(b > 0 ? b : 1);
}

cudaError_t launch_dfield_pack(const double* D9, double* D6, int* bad, int64_t ncell, const double* Jinv,
                               double det, cudaStream_t s)
{
    if (ncell == 0) return cudaSuccess;
    Mat3 Ji;
    for (int i = 0; i < 9; ++i) Ji.a[i] = Jinv ? Jinv[i] : (i % 4 == 0 ? 1.0 : 0.0);
    dfield_pack_kernel<<<blocks_for(ncell), 256, 0, s>>>(D9, D6, bad, ncell, Jinv ? 1 : 0, Ji, det);
    return cudaGetLastError();
}

cudaError_t launch_dfield_const(double* D6, const double D[9], int64_t ncell, cudaStream_t s)
{
    if (ncell == 0) return cudaSuccess;
    dfield_const_kernel<<<blocks_for(ncell), 256, 0, s>>>(D6, D[0], D[4], D[8], D[1], D[2], D[5], ncell);
    return cudaGetLastError();
}

}  // namespace dg

namespace dg {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)f;
    }
    return fn;
}

bool make_row_map(CUtensorMap* map, const double* ptr, int64_t rows)
{
    EncodeTiledFn fn = encoder();
    if (!fn || !ptr || rows <= 0 || rows > (int64_t)0xffffffffLL || ((uintptr_t)ptr & 15)) return false;
    cuuint64_t dims[2] = {8, (cuuint64_t)rows};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {8, 64};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)ptr, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace dg

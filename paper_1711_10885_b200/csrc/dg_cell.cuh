// Fused cell kernel: y = A z for the SIPG/WSIPG operator of arXiv 1711.10885,
// FP64, sm_100a.
//
// Work decomposition (Cfg<N>, measured per degree): a cell is processed by TPC threads
// (a fraction of a warp for small n, with several cells per CTA; 1-4 warps for n >= 5, one
// cell per CTA; k = 7: two warps, one pencil per thread); each thread owns P "pencils" (lines
// of n points along one direction) in each of the three roles (x-, y- and z-pencil). Phases
// synchronise with __syncwarp when a cell fits a warp, else with CTA barriers. The 1D
// matrices live in __constant__ memory (one copy per use site so the compiler reloads per
// stage instead of hoisting whole matrices into registers). At n = 8 the own and x-neighbour
// blocks arrive by TMA and y leaves by a TMA store (namespace tma below).
//
// Per cell (Algorithm 1, reorganised owner-computes):
//   (1) u at the n^3 Gauss points by sum factorization u_q = (V x V x V) z
//       (eq:evalfe; kernel eq:sum_fact_kernel :590-595), each stage
//       by the even-odd decomposition of V (V_{n-1-i,j} = (-1)^j V_ij); the reference
//       gradient by collocation derivatives Dc = G V^{-1} along each pencil (exact on
//       Q_k; Dc is centro-antisymmetric, also applied even-odd)
//   (2) quadrature-point data x^(r) (eq:gauss_points), x^(0) = c u W
//   (3) y = (V^T x V^T x V^T)(x^(0) + sum_r Dc_r^T x^(r) + face lifts)   (eq:evalblf :425-444)
//   (4-10) faces: own traces are 1D extrapolations of u_q along the normal (L_l(s), L'_l(s));
//       neighbour traces are the paper's face sum factorization with the normal direction
//       FIRST: theta(s)/theta'(s) contraction of the neighbour's
//       coefficients, then V along the two tangential directions. Consistency, symmetry,
//       penalty and upwind terms (eq:blf :301-315, Phi :334-341) are evaluated pointwise
//       and lifted with the normal direction LAST into the quadrature-space array before
//       the transposed stages. Each cell writes only its own y block once: no atomics.
#pragma once
#include "dg_internal.h"

namespace dg {

template <int N>
struct EO {                        // even-odd form of a centro-antisymmetric matrix A
    static constexpr int H = N / 2;
    double p[H > 0 ? H : 1][H > 0 ? H : 1];   // (A_ij + A_i,N-1-j) / 2
    double m[H > 0 ? H : 1][H > 0 ? H : 1];   // (A_ij - A_i,N-1-j) / 2
    double col[H > 0 ? H : 1];                // A_iH            (odd N)
    double row[H > 0 ? H : 1];                // A_Hj            (odd N)
};

// Leading pad of the table block: the constant-bank placement of the per-stage tables changes
// the fast kernel's speed by a few per cent (C3, one box, A/B: shifts of 0 / 16 / 32 / 48 / 64 /
// 80 / 96 / 192 / 320 / 384 / 512 / 1024 bytes gave 82.5 / 83.3 / 83.4 / 83.4 / 84.0 / 83.7 / 83.6
// / 83.6 / 83.5 / 82.7 / 82.3 / 81.4 GDOF/s, an 8-byte shift 78.1; Problem A k = 7 lost 0.9 %
// with it), so n = 8 keeps the best one
// (one table per translation unit: DG_PADX doubles, per degree below, overridable for sweeps)
#ifndef DG_PADX
#define DG_PADX ((DG_N) == 8 ? 8 : 0)
#endif
template <int P> struct TabHead { double head[P]; };
template <> struct TabHead<0> {};

template <int N>
struct Tab : TabHead<DG_PADX> {
    static constexpr int HC = (N + 1) / 2;
    double Vh[12][HC][N];    // V_ij = theta_j(xi_i), rows i < ceil(n/2); one copy per use site
    // pad0..pad3: unused. They keep the constant-bank offsets of the tables below where an
    // earlier table set put them; the packed layout measured 0.9 % slower at C3 (82.5 -> 81.8
    // GDOF/s, A/B on one box), i.e. the placement of each stage's tables in constant-cache lines
    // matters at this level.
    EO<N> pad0[12];
    double w[N];
    double pad1[6][4][N];
    double th0[N], th1[N], dth0[N], dth1[N];
    double pad2[HC][N];
    // sigma/delta form (below): doubled forward V, doubled even-odd Dc and Dc^T diag(w), one copy
    // per use site (the middle row of an odd n plain)
    double Vs[9][HC][N];
    EO<N> Dcs[5], DcTws[3];
    // sigma/delta form of the general kernel (dg_gen.cuh): doubled Dc^T, doubled G (its odd rows
    // first), trace rows acting on sigma/delta arrays (value / derivative at 0, 1), lift rows
    // adding a plain vector to a sigma/delta array
    EO<N> DcTs[5];
    double Gs[HC][N];
    double Ls[2][4][N];
    double Lsl[4][N];
    EO<N> pad3[3];
    // the roles' own traces from the even/odd sums (one copy per direction):
    double Le[3][4][(N / 2) > 0 ? N / 2 : 1];  // (L0_i +- L0_{n-1-i})/2, (L'0_i +- L'0_{n-1-i})/2, i < n/2
    double Lmid[3][2];                     // L0_H, L'0_H (odd n)
};

#ifndef DG_N
#error "dg_cell.cuh is compiled once per degree with -DDG_N=<k+1>"
#endif
__constant__ Tab<DG_N> g_tab;

// TPC threads per cell, P pencils per thread (TPC * P >= n^2), C cells per CTA.
template <int N> struct Cfg;
// Build-time override of this TU's configuration (variant sweeps: tools/tune_cfg.py).
#ifdef DG_TPC
#define DG_OVR(n, ov, d) ((DG_N) == (n) ? (ov) : (d))
#else
#define DG_OVR(n, ov, d) (d)
#endif
template <> struct Cfg<2> { static constexpr int TPC = DG_OVR(2, DG_TPC, 8), P = DG_OVR(2, DG_P, 1), C = DG_OVR(2, DG_C, 16), MINB = DG_OVR(2, DG_MINB, 8); };
template <> struct Cfg<3> { static constexpr int TPC = DG_OVR(3, DG_TPC, 16), P = DG_OVR(3, DG_P, 1), C = DG_OVR(3, DG_C, 8), MINB = DG_OVR(3, DG_MINB, 8); };
template <> struct Cfg<4> { static constexpr int TPC = DG_OVR(4, DG_TPC, 16), P = DG_OVR(4, DG_P, 1), C = DG_OVR(4, DG_C, 4), MINB = DG_OVR(4, DG_MINB, 12); };
template <> struct Cfg<5> { static constexpr int TPC = DG_OVR(5, DG_TPC, 32), P = DG_OVR(5, DG_P, 1), C = DG_OVR(5, DG_C, 1), MINB = DG_OVR(5, DG_MINB, 16); };
template <> struct Cfg<6> { static constexpr int TPC = DG_OVR(6, DG_TPC, 36), P = DG_OVR(6, DG_P, 1), C = DG_OVR(6, DG_C, 3), MINB = DG_OVR(6, DG_MINB, 7); };
template <> struct Cfg<7> { static constexpr int TPC = DG_OVR(7, DG_TPC, 64), P = DG_OVR(7, DG_P, 1), C = DG_OVR(7, DG_C, 1), MINB = DG_OVR(7, DG_MINB, 12); };
template <> struct Cfg<8> { static constexpr int TPC = DG_OVR(8, DG_TPC, 64), P = DG_OVR(8, DG_P, 1), C = DG_OVR(8, DG_C, 1), MINB = DG_OVR(8, DG_MINB, 10); };
template <> struct Cfg<9> { static constexpr int TPC = DG_OVR(9, DG_TPC, 96), P = DG_OVR(9, DG_P, 1), C = DG_OVR(9, DG_C, 1), MINB = DG_OVR(9, DG_MINB, 8); };
template <> struct Cfg<10> { static constexpr int TPC = DG_OVR(10, DG_TPC, 128), P = DG_OVR(10, DG_P, 1), C = DG_OVR(10, DG_C, 1), MINB = DG_OVR(10, DG_MINB, 6); };
template <> struct Cfg<11> { static constexpr int TPC = DG_OVR(11, DG_TPC, 128), P = DG_OVR(11, DG_P, 1), C = DG_OVR(11, DG_C, 1), MINB = DG_OVR(11, DG_MINB, 6); };

// Shared-memory layout of one n^3 cell array: x-, y- and z-pencil accesses of a warp are
// (nearly) bank-conflict free (searched offline; n = 8 uses an XOR swizzle that is conflict
// free for all three access patterns).
// Padded linear layouts for the other n, chosen with the bank-conflict model of
// tools/smem_layout.py (validated against ncu: 55 % / 26 % conflicts predicted for the old n = 4
// / n = 6 layouts, 53 % / 28 % measured) over SY, SZ and index rotations.
template <int N> struct Lay {
    static constexpr int SY = (N == 6) ? 9 : N;
    static constexpr int SZ = (N == 2) ? 5 : (N == 3) ? 9 : (N == 5) ? 25 : (N == 6) ? 54
                            : (N == 7) ? 55 : (N == 9) ? 89 : (N == 10) ? 106 : 123;
    static constexpr int SLOT = SZ * (N - 1) + SY * (N - 1) + N;
    __device__ __forceinline__ static int at(int x, int y, int z) { return x + SY * y + SZ * z; }
};
// n = 4: a half-warp (16 lanes, one 8-byte phase) holds one cell's 16 pencils; the residue mod 16
// (x ^ z) + 4 (y ^ z) is a bijection on every axis-aligned plane, so x-, y- and z-pencil accesses
// are all conflict free (a padded linear layout cannot be: it left 53 % of the wavefronts as
// bank conflicts, ncu C4-k3).
template <> struct Lay<4> {
    static constexpr int SLOT = 64;
    __device__ __forceinline__ static int at(int x, int y, int z) { return (x ^ z) + 4 * (y ^ z) + 16 * z; }
};
template <> struct Lay<8> {
    static constexpr int SLOT = 512;
    __device__ __forceinline__ static int at(int x, int y, int z)
    {
        return (x ^ ((y >> 1) | ((z & 1) << 2))) + 8 * (y ^ (z & 1)) + 64 * z;
    }
};

// Face arrays: 6 faces x 2 quantities x n^2 points, row padded. Slot 2f holds the
// neighbour trace u+, then the lift coefficient cv; slot 2f+1 the neighbour normal
// derivative, then cg.
template <int N> struct FLay {
    static constexpr int RS = (N >= 5) ? N : N + 1;
    static constexpr int ARR = (N == 5) ? 25 : (N == 6) ? 41 : (N == 7) ? 56 : (N == 9) ? 81 : (N == 10) ? 101
                             : (N == 11) ? 121 : N * RS + 1;
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return arr * ARR + i1 + RS * i2; }
};
// n = 4: 16 doubles per array, swizzled by the array index so that the tangential-stage lines of
// 4 consecutive arrays (one lane per line) and the per-point accesses are conflict free.
template <> struct FLay<4> {
    static constexpr int SLOT = 12 * 16;
    __device__ __forceinline__ static int at(int arr, int i1, int i2)
    {
        const int s = arr & 3;
        return 16 * arr + (i1 ^ s) + 4 * (i2 ^ s);
    }
};
// n = 8 (round 1; kept for the variable-velocity kernel): 64 doubles per array, XOR swizzle.
struct FLaySwz8 {
    static constexpr int SLOT = 12 * 64;
    __device__ __forceinline__ static int at(int arr, int i1, int i2)
    {
        return 64 * arr + 8 * (i2 ^ (arr & 1)) + (i1 ^ ((i2 >> 1) | ((arr & 1) << 2)));
    }
};
// n = 8: the low three bits of the word index are i1 ^ i2 (a Latin square: a bijection along i1 and
// along i2), bit 3 is i2 & 1, and the array stride 72 = 8 mod 16 puts arrays a and a + 1 on
// complementary banks: conflict free for points (a, b) per lane and for the tangential stages'
// lines along i1 or i2 of two consecutive arrays per half-warp, with less index arithmetic than
// the XOR swizzle (DG_FLAY_SWZ=1 restores it).
#ifndef DG_FLAY_SWZ
#define DG_FLAY_SWZ 0
#endif
#if DG_FLAY_SWZ
template <> struct FLay<8> : FLaySwz8 {};
#else
template <> struct FLay<8> {
    static constexpr int ARR = 72;
    static constexpr int SLOT = 12 * ARR;
    __device__ __forceinline__ static int at(int arr, int i1, int i2) { return ARR * arr + 8 * i2 + (i1 ^ i2); }
};
#endif
// n = 8: the high x-neighbour block is TMA-staged in the face slots 4.. (free in phase 1) at a
// 512-byte aligned offset past arrays 0..3 (written in phase 1)
constexpr int XH8 = DG_FLAY_SWZ ? 256 : 320;
static_assert(XH8 >= 4 * (FLay<8>::SLOT / 12) && XH8 + 512 <= FLay<8>::SLOT, "x-neighbour staging inside face slots 4..11");

template <int N>
struct Smem {
    static constexpr int PER_CELL = 2 * Lay<N>::SLOT + FLay<N>::SLOT;
    // n = 8: TMA staging of the own block (4 KB, 128-byte aligned) plus the mbarrier; the two
    // x-neighbour blocks are staged in A1 and face slots 4..11, free during phase 1
    // n = 7, 9, 10, 11: the own block is staged by a bulk copy in A1 (free in phase 1) and y
    // leaves from A1 by a bulk copy (namespace bulk); only the mbarrier is extra
    static constexpr int STAGE = (N == 8) ? 512 + 16 + 16 : (N >= 7 ? 2 : 0);
    static constexpr int BYTES = Cfg<N>::C * PER_CELL * 8 + STAGE * 8;
};

// ---------------------------------------------------------------------------------- TMA (n = 8)
// The cell block (64 x-lines of 64 B) moves between HBM and shared memory by the tensor memory
// accelerator with the 64-byte swizzle: 16-byte chunk c of row L lands at chunk c ^ ((addr >> 7) & 3)
// of its row, so the LDS.128 / STS.128 of one x-line per thread are bank-conflict free, and the
// global side is read / written as whole 4 KB blocks (no 4x sector over-fetch of per-thread
// x-line loads, no load/store instructions on the LSU pipe).
namespace tma {
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void load_rows(double* dst, const CUtensorMap* m, int row, uint64_t* b)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(saddr(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(row), "r"(saddr(b))
                 : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t phase)
{
    asm volatile("{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}\n"
                 ::"r"(saddr(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void store_rows(const CUtensorMap* m, int row, const double* src)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                 ::"l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(row), "r"(saddr(src)) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// double index of element e of row L in a TMA-swizzled block at S
__device__ __forceinline__ int at(const double* S, int L, int e)
{
    const uint32_t row = saddr(S) + 64u * (uint32_t)L;
    return 8 * L + 2 * ((e >> 1) ^ (int)((row >> 7) & 3u)) + (e & 1);
}
// Issue the TMA loads of a cell's own block (into STG) and of its local x-neighbours' blocks
// (into XL, XH) and wait for them; returns whether both x-neighbours are TMA-staged (a ghost
// neighbour on another rank is read by per-thread loads instead). One cell per CTA.
__device__ __forceinline__ bool stage_x(const KParams& p, double* STG, double* XL, double* XH, int tid,
                                       const int (&lc)[3], int64_t cell, unsigned nbi, uint64_t* mbar = nullptr)
{
    if (!mbar) mbar = reinterpret_cast<uint64_t*>(STG + 512);   // (default: right after the staging block)
    const int nq = (int)p.nloc[0];
    const bool hl = (nbi & 1u) != 0, hh = (nbi & 2u) != 0;
    const bool ll = hl && (lc[0] > 0 || p.wrap[0]), lh = hh && (lc[0] + 1 < nq || p.wrap[0]);
    const bool tma_x = (ll || !hl) && (lh || !hh);
    if (tid == 0) mbar_init(mbar);
    __syncthreads();
    if (tid == 0) {
        const int64_t clo = (lc[0] > 0) ? cell - 1 : cell + (nq - 1);
        const int64_t chi = (lc[0] + 1 < nq) ? cell + 1 : cell - (nq - 1);
        const int64_t ncell = p.nloc[0] * p.nloc[1] * p.nloc[2];
        DG_ASSERT(cell >= 0 && cell < ncell && clo >= 0 && clo < ncell && chi >= 0 && chi < ncell);
        const bool xl = tma_x && ll, xh = tma_x && lh;
        expect_tx(mbar, 4096u * (1u + (xl ? 1u : 0u) + (xh ? 1u : 0u)));
        load_rows(STG, &p.tmz, (int)(cell * 64), mbar);
        if (xl) load_rows(XL, &p.tmz, (int)(clo * 64), mbar);
        if (xh) load_rows(XH, &p.tmz, (int)(chi * 64), mbar);
    }
    wait(mbar, 0);
    return tma_x;
}
__device__ __forceinline__ void mbar_init_n(uint64_t* b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// x-line L (elements e, e+1) of a staged block
__device__ __forceinline__ double2 line2(const double* S, int L, int e)
{
    return *reinterpret_cast<const double2*>(S + at(S, L, e));
}
// write the y x-line of row L into the staging block, then (tid 0) one TMA store of the block
__device__ __forceinline__ void put2(double* S, int L, int e, double a, double b)
{
    *reinterpret_cast<double2*>(S + at(S, L, e)) = make_double2(a, b);
}
__device__ __forceinline__ void store_block(const KParams& p, const double* S, int tid, int64_t cell)
{
    fence_async();
    __syncthreads();
    if (tid == 0) store_rows(&p.tmy, (int)(cell * 64), S);
}
}  // namespace tma

// ---------------------------------------------------------------------------------- bulk copies (n != 8)
// A cell block (n^3 doubles, x-lines of n) moves between HBM and a LINEAR shared-memory image by
// one non-tensor bulk copy (cp.async.bulk, 16-byte granules): the image S is placed so that
// S == the block start (mod 16 bytes); the 16-byte-aligned interior is copied, a leading and / or
// trailing odd double (a block start 8 mod 16, an odd remainder) goes by plain loads / stores.
// Each thread reads / writes its x-lines at N L + e of the image: bank-conflict free (odd n: N L
// mod 16 is a bijection on 16 lanes; even n: 16-byte accesses, N L / 2 mod 8 a bijection on 8).
// It replaces the per-thread line loads (a lane's n doubles at an n-double lane stride, n sectors
// per warp instruction) and the per-thread stores that held the CTA until they drained.
namespace bulk {
struct Span {
    int sh;          // image offset in doubles (0, 1): S = base + sh
    int hd, tl;      // leading / trailing plain doubles
    uint32_t bytes;  // bulk-copied bytes
};
template <int N>
__device__ __forceinline__ Span span(const double* g, const double* base)
{
    constexpr int n3 = N * N * N;
    Span o;
    const uint32_t gp = (uint32_t)(reinterpret_cast<uintptr_t>(g) >> 3) & 1u;
    o.sh = (int)((gp ^ (tma::saddr(base) >> 3)) & 1u);
    o.hd = (int)gp;
    o.tl = (n3 - o.hd) & 1;
    o.bytes = (uint32_t)(n3 - o.hd - o.tl) * 8u;
    return o;
}
__device__ __forceinline__ void load(double* s, const double* g, uint32_t bytes, uint64_t* mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(tma::saddr(s)), "l"(reinterpret_cast<uint64_t>(g)), "r"(bytes), "r"(tma::saddr(mbar))
                 : "memory");
}
__device__ __forceinline__ void store(double* g, const double* s, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                 ::"l"(reinterpret_cast<uint64_t>(g)), "r"(tma::saddr(s)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
}  // namespace bulk

// ---------------------------------------------------------------------------------- 1D stages
// t[k][i] = sum_j V_ij r[k][j]  (even-odd: V_{n-1-i,j} = (-1)^j V_ij)
template <int N, int P>
__device__ __forceinline__ void c_apply(const EO<N>& A, const double (&r)[P][N], double (&t)[P][N])
{
    constexpr int H = N / 2;
    double s[P][H > 0 ? H : 1], d[P][H > 0 ? H : 1];
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int j = 0; j < H; ++j) {
            s[k][j] = r[k][j] + r[k][N - 1 - j];
            d[k][j] = r[k][j] - r[k][N - 1 - j];
        }
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double Pp[P], Q[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            Pp[k] = (N & 1) ? A.col[i] * r[k][H] : 0.0;
            Q[k] = 0.0;
        }
#pragma unroll
        for (int j = 0; j < H; ++j)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                Pp[k] = fma(A.p[i][j], s[k][j], Pp[k]);
                Q[k] = fma(A.m[i][j], d[k][j], Q[k]);
            }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            t[k][i] = Pp[k] + Q[k];
            t[k][N - 1 - i] = Q[k] - Pp[k];
        }
    }
    if (N & 1) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < H; ++j) acc = fma(A.row[j], d[k][j], acc);
            t[k][H] = acc;
        }
    }
}

template <int N>
__device__ __forceinline__ double dot(const double* a, const double* v)
{
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = fma(a[i], v[i], s);
    return s;
}

// ---------------------------------------------------------------------------------- sigma/delta form
// Every array of the pencil kernels is kept in "sigma/delta form" along each of its three
// directions: position i < n/2 holds t_i + t_(n-1-i), position n-1-i holds t_i - t_(n-1-i)
// (odd n: the middle entry plain). All pointwise operations (Gauss weights w_i = w_(n-1-i), constant
// coefficients, the face fluxes, the traces and lifts) are linear with symmetric weights, so
// they commute with this change of basis along every direction, and the 1D stages consume and
// produce it directly with doubled even-odd tables: no sum / difference instructions around
// the forward stages, the Dc and Dc^T diag(w) stages, or before the backward stages.

template <int N, int P>
__device__ __forceinline__ void v_fwd_sd(const double (&Vs)[(N + 1) / 2][N], const double (&r)[P][N], double (&t)[P][N])
{
    // Vs: rows i < n/2 doubled; for odd n the middle row is the plain V_Hj (the middle entry
    // of the sigma/delta form is the plain value t_H)
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double E[P], O[P];
#pragma unroll
        for (int k = 0; k < P; ++k) { E[k] = 0.0; O[k] = 0.0; }
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (j & 1) O[k] = fma(Vs[i][j], r[k][j], O[k]);
                else E[k] = fma(Vs[i][j], r[k][j], E[k]);
            }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            t[k][i] = E[k];
            t[k][N - 1 - i] = O[k];
        }
    }
    if (N & 1) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double E = 0.0;
#pragma unroll
            for (int j = 0; j < N; j += 2) E = fma(Vs[H][j], r[k][j], E);
            t[k][H] = E;
        }
    }
}

template <int N, int P>
__device__ __forceinline__ void v_bwd_sd(const double (&Vh)[(N + 1) / 2][N], const double (&r)[P][N], double (&t)[P][N])
{
    constexpr int H = N / 2;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double acc[P];
#pragma unroll
        for (int k = 0; k < P; ++k) acc[k] = ((N & 1) && !(j & 1)) ? Vh[H][j] * r[k][H] : 0.0;
#pragma unroll
        for (int i = 0; i < H; ++i)
#pragma unroll
            for (int k = 0; k < P; ++k) acc[k] = fma(Vh[i][j], (j & 1) ? r[k][N - 1 - i] : r[k][i], acc[k]);
#pragma unroll
        for (int k = 0; k < P; ++k) t[k][j] = acc[k];
    }
}

// out = A r for a centro-antisymmetric A, r and out in sigma/delta form: A2 is the even-odd form
// with p, m and (odd n) col doubled, row plain; optional addends (pairs doubled, middle plain)
template <int N, int P, bool ADD>
__device__ __forceinline__ void c_apply_s(const EO<N>& A2, const double (&r)[P][N], double (&t)[P][N],
                                          const double (&qa)[P][(N / 2) > 0 ? N / 2 : 1],
                                          const double (&pb)[P][(N / 2) > 0 ? N / 2 : 1], const double (&mid)[P])
{
    constexpr int H = N / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double Pp[P], Q[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
            Pp[k] = ADD ? pb[k][i] : 0.0;
            if (N & 1) Pp[k] = fma(A2.col[i], r[k][H], Pp[k]);
            Q[k] = ADD ? qa[k][i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < H; ++j)
#pragma unroll
            for (int k = 0; k < P; ++k) {
                Pp[k] = fma(A2.p[i][j], r[k][j], Pp[k]);
                Q[k] = fma(A2.m[i][j], r[k][N - 1 - j], Q[k]);
            }
#pragma unroll
        for (int k = 0; k < P; ++k) {
            t[k][i] = Q[k];
            t[k][N - 1 - i] = Pp[k];
        }
    }
    if (N & 1) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            double acc = ADD ? mid[k] : 0.0;
#pragma unroll
            for (int j = 0; j < H; ++j) acc = fma(A2.row[j], r[k][N - 1 - j], acc);
            t[k][H] = acc;
        }
    }
}

// ---------------------------------------------------------------------------------- rectangular stages
// (m >= n Gauss points: the over-integrated kernels dg_vb.cuh, dg_geo.cuh)
// r (n modal values) -> t (m points): t_i = sum_j V_ij r_j, even-odd over the symmetric rule
template <int N, int M>
__device__ __forceinline__ void vr_fwd(const double (&Vh)[(M + 1) / 2][N], const double (&r)[N], double (&t)[M])
{
    constexpr int H = M / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
        double E = 0.0, O = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (j & 1) O = fma(Vh[i][j], r[j], O);
            else E = fma(Vh[i][j], r[j], E);
        }
        t[i] = E + O;
        t[M - 1 - i] = E - O;
    }
    if (M & 1) {
        double E = 0.0;
#pragma unroll
        for (int j = 0; j < N; j += 2) E = fma(Vh[H][j], r[j], E);
        t[H] = E;
    }
}

// t (m points) -> r (n modal values): r_j = sum_i V_ij t_i
template <int N, int M>
__device__ __forceinline__ void vr_bwd(const double (&Vh)[(M + 1) / 2][N], const double (&t)[M], double (&r)[N])
{
    constexpr int H = M / 2;
    double s[H > 0 ? H : 1], d[H > 0 ? H : 1];
#pragma unroll
    for (int i = 0; i < H; ++i) {
        s[i] = t[i] + t[M - 1 - i];
        d[i] = t[i] - t[M - 1 - i];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double acc = ((M & 1) && !(j & 1)) ? Vh[H][j] * t[H] : 0.0;
#pragma unroll
        for (int i = 0; i < H; ++i) acc = fma(Vh[i][j], (j & 1) ? d[i] : s[i], acc);
        r[j] = acc;
    }
}

// ---------------------------------------------------------------------------------- face terms
// Contribution cv * phi_i + cg_phys * d_q phi_i of one face point, returned as
// (cv, cg = cg_phys / h_q, the coefficient of the REFERENCE normal derivative).
// own side s: s = 1 -> face x_q = 1, this cell is T- ; s = 0 -> face x_q = 0, this cell is T+.
struct FaceOut { double cv, cg; };

__device__ __forceinline__ FaceOut flux_interior(const KParams& p, int q, int s, double W, double uo, double dref,
                                                 double un, double sn)
{
    const double so = p.Dqq_h[q] * dref;                      // D_qq du/dx_q (own)
    const double um = s ? uo : un, up = s ? un : uo;
    const double sm = s ? so : sn, sp = s ? sn : so;
    const double bn = p.bq[q];
    const double Phi = (bn >= 0.0) ? bn * um : bn * up;       // upwind flux
    const double J = um - up;                                 // [[u]] = u- - u+
    const double Avg = 0.5 * (sm + sp);                       // nu.{D grad u}_w, w = 1/2 (constant D), C-1
    const double com = Phi - Avg + p.gam[q] * J;
    FaceOut o;
    o.cv = s ? W * com : -W * com;                            // [[phi]] = +phi on T-, -phi on T+
    o.cg = -W * 0.5 * J * p.Dqq_h[q];                         // -(nu.{D grad phi}_w, [[u]])
    return o;
}
__device__ __forceinline__ FaceOut flux_boundary(const KParams& p, int q, int s, double W, double uo, double dref)
{
    const double nu = s ? 1.0 : -1.0;                         // outward normal
    const double bn = nu * p.bq[q];
    const double sn = nu * p.Dqq_h[q] * dref;                 // nu . D grad u
    const double Phi = (bn >= 0.0) ? bn * uo : 0.0;           // Phi(u, 0, b_nu)
    FaceOut o;
    o.cv = W * (Phi - sn + p.gam[q] * uo);                    // [[.]] = {.} = v- on the boundary (:282-286)
    o.cg = -W * uo * nu * p.Dqq_h[q];
    return o;
}

// ---------------------------------------------------------------------------------- kernel pieces
// Load the lines of the two neighbours across direction q that this thread's pencils need
// (tangential modal indices (a, bb) fixed, normal index e = 0..n-1).
// A neighbour on another rank (the partition face of this rank's box) is not loaded as a block:
// its rank sent the normal-first contraction of its boundary layer (the face traces of SURVEY
// 8(e), dg_trace_pack in dg_aux.cu: 2 n^2 doubles per face cell, [u | d] at a + n bb). For such
// a "ghost" side the two values land in rl/rh[k][0..1] and bit 0 (low) / 1 (high) of the
// returned mask tells nb_traces to take them as they are.
template <int N, int P, bool GH = true>
__device__ __forceinline__ unsigned nb_load(const KParams& p, const double* zc, const int64_t n3, int q, const int lc[3],
                                            unsigned nbmask, const int (&pa)[P], const int (&pb)[P], const bool (&act)[P],
                                            double (&rl)[P][N], double (&rh)[P][N])
{
    constexpr int NN = N * N;
    const int lq = lc[q];
    const int nq = (int)p.nloc[q];
    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
    const int64_t gi = (q == 0) ? (lc[1] + p.nloc[1] * lc[2]) : (q == 1) ? (lc[0] + p.nloc[0] * lc[2])
                                                                        : (lc[0] + p.nloc[0] * lc[1]);
    const bool hl = (nbmask >> (2 * q)) & 1u, hh = (nbmask >> (2 * q + 1)) & 1u;
    // (GH = false: a launch over cells with no neighbour on another rank -- the inner box or a
    // single-rank operator -- compiles this away)
    const bool gl = GH && hl && lq == 0 && !p.wrap[q];     // the low neighbour lives on another rank
    const bool gh = GH && hh && lq + 1 == nq && !p.wrap[q];
    const int64_t wst = (int64_t)(nq - 1) * st * n3;   // periodic wrap inside this rank's box
    // (GH = false never reaches the third alternative -- a cell at the box edge with a neighbour
    // there is a wrap or a ghost -- but this form of the selection measured 2.2 % faster at C3
    // than selecting zc: 84.5 against 82.7 GDOF/s, A/B on one box; it is only a code-generation
    // effect, nothing is loaded through p.ghost without GH)
    const double* zl = (lq > 0) ? zc - st * n3
                     : (p.wrap[q] ? zc + wst : ((!GH && hl) ? p.ghost[2 * q] + gi * n3 : zc));
    const double* zh = (lq + 1 < nq) ? zc + st * n3
                     : (p.wrap[q] ? zc - wst : ((!GH && hh) ? p.ghost[2 * q + 1] + gi * n3 : zc));
    const double* tl = gl ? p.ghost[2 * q] + gi * 2 * NN : nullptr;
    const double* th = gh ? p.ghost[2 * q + 1] + gi * 2 * NN : nullptr;
    const bool ll = hl && !gl, lh = hh && !gh;
#ifdef DG_CHECK
    {
        const int64_t nall = p.nloc[0] * p.nloc[1] * p.nloc[2] * n3;
        const int t1 = (q == 0) ? 1 : 0, t2 = (q == 2) ? 1 : 2;
        const int64_t nlay = p.nloc[t1] * p.nloc[t2];
        DG_ASSERT(gi >= 0 && gi < nlay);
        DG_ASSERT(zl >= p.z && zl + n3 <= p.z + nall);
        DG_ASSERT(zh >= p.z && zh + n3 <= p.z + nall);
        if (gl) DG_ASSERT(p.ghost[2 * q] != nullptr);
        if (gh) DG_ASSERT(p.ghost[2 * q + 1] != nullptr);
    }
#endif
#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (q == 0 && N % 2 == 0) {
            const int base = N * pa[k] + NN * pb[k];
#pragma unroll
            for (int e = 0; e < N; e += 2) {
                const double2 vl = (act[k] && ll) ? __ldg(reinterpret_cast<const double2*>(zl + base + e))
                                                  : make_double2(0.0, 0.0);
                const double2 vh = (act[k] && lh) ? __ldg(reinterpret_cast<const double2*>(zh + base + e))
                                                  : make_double2(0.0, 0.0);
                rl[k][e] = vl.x; rl[k][e + 1] = vl.y;
                rh[k][e] = vh.x; rh[k][e + 1] = vh.y;
            }
        } else {
            const int se = (q == 0) ? 1 : (q == 1) ? N : NN;
            const int base = (q == 0) ? N * pa[k] + NN * pb[k] : (q == 1) ? pa[k] + NN * pb[k] : pa[k] + N * pb[k];
#pragma unroll
            for (int e = 0; e < N; ++e) {
                rl[k][e] = (act[k] && ll) ? __ldg(zl + base + e * se) : 0.0;
                rh[k][e] = (act[k] && lh) ? __ldg(zh + base + e * se) : 0.0;
            }
        }
        if (gl || gh) {
            const int t = pa[k] + N * pb[k];
            if (gl) {
                rl[k][0] = act[k] ? __ldg(tl + t) : 0.0;
                rl[k][1] = act[k] ? __ldg(tl + NN + t) : 0.0;
            }
            if (gh) {
                rh[k][0] = act[k] ? __ldg(th + t) : 0.0;
                rh[k][1] = act[k] ? __ldg(th + NN + t) : 0.0;
            }
        }
    }
    return (gl ? 1u : 0u) | (gh ? 2u : 0u);
}

// The neighbour traces of one pencil, normal direction FIRST: the low
// neighbour (face 2q) is seen at its x_q = 1 (theta(1), theta'(1)), the high one (face 2q+1) at
// x_q = 0; ghost sides (bit 0 / 1 of gm) arrive contracted.
template <int N>
__device__ __forceinline__ void nb_traces(const double* th0, const double* th1, const double* dth0, const double* dth1,
                                          const double (&rl)[N], const double (&rh)[N], unsigned gm, double& ul,
                                          double& dl, double& uh, double& dh)
{
    ul = 0.0; dl = 0.0; uh = 0.0; dh = 0.0;
#pragma unroll
    for (int e = 0; e < N; ++e) {
        ul = fma(th1[e], rl[e], ul);
        dl = fma(dth1[e], rl[e], dl);
        uh = fma(th0[e], rh[e], uh);
        dh = fma(dth0[e], rh[e], dh);
    }
    if (gm & 1u) { ul = rl[0]; dl = rl[1]; }
    if (gm & 2u) { uh = rh[0]; dh = rh[1]; }
}

// Normal-direction-first contraction of the loaded neighbour lines into the face arrays.
template <int N, int P, class FL = FLay<N>>
__device__ __forceinline__ void nb_contract(const Tab<N>& T, double* NT, int q, unsigned nbmask, const int (&pa)[P],
                                           const int (&pb)[P], const bool (&act)[P], const double (&rl)[P][N],
                                           const double (&rh)[P][N], unsigned gm)
{
    const bool hl = (nbmask >> (2 * q)) & 1u, hh = (nbmask >> (2 * q + 1)) & 1u;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        double ul, dl, uh, dh;
        nb_traces<N>(T.th0, T.th1, T.dth0, T.dth1, rl[k], rh[k], gm, ul, dl, uh, dh);
        if (act[k]) {
            if (hl) {
                NT[FL::at(4 * q, pa[k], pb[k])] = ul;
                NT[FL::at(4 * q + 1, pa[k], pb[k])] = dl;
            }
            if (hh) {
                NT[FL::at(4 * q + 2, pa[k], pb[k])] = uh;
                NT[FL::at(4 * q + 3, pa[k], pb[k])] = dh;
            }
        }
    }
}

// Tangential stage of the 4 neighbour-trace arrays of direction q: V along i1 (dim 0) or i2 (dim 1).
template <int N, int TPC>
__device__ __forceinline__ void nb_tangential(const double (&Vh)[(N + 1) / 2][N], double* NT, int q, int dim,
                                             unsigned nbmask, int lane)
{
    for (int tk = lane; tk < 4 * N; tk += TPC) {
        const int arr = 4 * q + tk / N, line = tk % N;
        if ((nbmask >> (arr >> 1)) & 1u) {
            double rr[1][N], tt[1][N];
#pragma unroll
            for (int e = 0; e < N; ++e) rr[0][e] = NT[dim ? FLay<N>::at(arr, line, e) : FLay<N>::at(arr, e, line)];
            v_fwd_sd<N, 1>(Vh, rr, tt);   // Vh is a doubled copy (Tab::Vs)
#pragma unroll
            for (int e = 0; e < N; ++e) NT[dim ? FLay<N>::at(arr, line, e) : FLay<N>::at(arr, e, line)] = tt[0][e];
        }
    }
}

// Role of direction q (even-odd form): traces from the even/odd sums of the Dc stage,
// Gauss weights folded into Dc^T diag(w), face lifts merged into the Dc^T accumulators.
template <int N, int P>
__device__ __forceinline__ void role_eo(const KParams& p, const Tab<N>& T, const double* NT, int q, unsigned nbmask,
                                        bool do_int, bool do_bnd, bool do_vol, bool with_reaction,
                                        const int (&pa)[P], const int (&pb)[P], const double (&r)[P][N],
                                        double (&out)[P][N])
{
    constexpr int H = N / 2;
    constexpr int HH = H > 0 ? H : 1;
    double g[P][N], s[P][HH], d[P][HH];
    {                                           // r in sigma/delta form: the sums are the input itself
        double z0[P][HH], zm[P];
        c_apply_s<N, P, false>(T.Dcs[q], r, g, z0, z0, zm);
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int j = 0; j < H; ++j) {
                s[k][j] = r[k][j];
                d[k][j] = r[k][N - 1 - j];
            }
    }
    const double* Lp = T.Le[q][0];
    const double* Lm = T.Le[q][1];
    const double* LDp = T.Le[q][2];
    const double* LDm = T.Le[q][3];
    double qa[P][HH], pbv[P][HH], mid[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double wab = T.w[pa[k]] * T.w[pb[k]];
        // own traces u(0), u(1), u'(0), u'(1) from the even/odd sums
        double A = (N & 1) ? T.Lmid[q][0] * r[k][H] : 0.0, B = 0.0;
        double Ad = (N & 1) ? T.Lmid[q][1] * r[k][H] : 0.0, Bd = 0.0;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            A = fma(Lp[i], s[k][i], A);
            B = fma(Lm[i], d[k][i], B);
            Ad = fma(LDp[i], s[k][i], Ad);
            Bd = fma(LDm[i], d[k][i], Bd);
        }
        const double tr_u[2] = {A + B, A - B}, tr_d[2] = {Ad + Bd, Bd - Ad};
        const double Wf = p.dF[q] * wab;
        FaceOut fo[2];
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            const int f = 2 * q + sd;
            fo[sd].cv = 0.0;
            fo[sd].cg = 0.0;
            if ((nbmask >> f) & 1u) {
                if (do_int) {
                    const double un = NT[FLay<N>::at(2 * f, pa[k], pb[k])];
                    const double sn = p.Dqq_h[q] * NT[FLay<N>::at(2 * f + 1, pa[k], pb[k])];
                    fo[sd] = flux_interior(p, q, sd, Wf, tr_u[sd], tr_d[sd], un, sn);
                }
            } else if (do_bnd) {
                fo[sd] = flux_boundary(p, q, sd, Wf, tr_u[sd], tr_d[sd]);
            }
        }
        // lift (normal direction LAST) as even/odd addends of the Dc^T stage: the pair addends
        // enter the sigma/delta output doubled, the middle one plain
        const double Pc = fo[0].cv + fo[1].cv, Mc = fo[0].cv - fo[1].cv;
        const double Qc = fo[0].cg - fo[1].cg, Rc = fo[0].cg + fo[1].cg;
        const double Pc2 = 2.0 * Pc, Mc2 = 2.0 * Mc, Qc2 = 2.0 * Qc, Rc2 = 2.0 * Rc;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            qa[k][i] = fma(Pc2, Lp[i], Qc2 * LDp[i]);
            pbv[k][i] = fma(Mc2, Lm[i], Rc2 * LDm[i]);
        }
        mid[k] = (N & 1) ? fma(Pc, T.Lmid[q][0], Qc * T.Lmid[q][1]) : 0.0;
        // quadrature-point data with the weights folded into Dc^T diag(w) (eq:gauss_points)
        const double sw = do_vol ? p.dT * wab : 0.0;
        const double kd = sw * p.Dhat[4 * q], kb = sw * p.kb[q];
#pragma unroll
        for (int e = 0; e < N; ++e) g[k][e] = fma(kd, g[k][e], -kb * r[k][e]);
    }
    c_apply_s<N, P, true>(T.DcTws[q], g, out, qa, pbv, mid);
    if (with_reaction && do_vol) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const double wc = p.dT * T.w[pa[k]] * T.w[pb[k]] * p.c;
#pragma unroll
            for (int e = 0; e < N; ++e) out[k][e] = fma(wc * T.w[e], r[k][e], out[k][e]);
        }
    }
}

// ---------------------------------------------------------------------------------- task -> cell
// z fastest within a column; columns in tiles of TX x TY (ragged at the box edge). The two
// runtime divisors (column height nz, tile-row size TY nx) use host-precomputed magic numbers
// (q = (umulhi(a, m) + a) >> l, exact for a < 2^31); full tiles divide by the compile-time
// TX TY, TX.
constexpr unsigned TRAV_TX = 4, TRAV_TY = 16;
__device__ __forceinline__ unsigned fdiv(unsigned a, unsigned m, unsigned l) { return (__umulhi(a, m) + a) >> l; }
__device__ __forceinline__ void decode_task(const KParams& p, unsigned task, int (&lc)[3])
{
    const unsigned nz = (unsigned)p.task_cnt[2], nx = (unsigned)p.task_cnt[0], ny = (unsigned)p.task_cnt[1];
    const unsigned col = fdiv(task, p.dmag[0], p.dsh[0]);                 // task / nz
    const unsigned ty = fdiv(col, p.dmag[1], p.dsh[1]);                   // col / (TY nx)
    const unsigned wy = min(TRAV_TY, ny - ty * TRAV_TY);
    const unsigned cr = col - ty * TRAV_TY * nx;
    unsigned tx, wx, ci;
    if (wy == TRAV_TY) {
        tx = cr / (TRAV_TX * TRAV_TY);
        wx = min(TRAV_TX, nx - tx * TRAV_TX);
        ci = cr - tx * TRAV_TX * TRAV_TY;
    } else {
        tx = cr / (TRAV_TX * wy);
        wx = min(TRAV_TX, nx - tx * TRAV_TX);
        ci = cr - tx * TRAV_TX * wy;
    }
    const unsigned cy = (wx == TRAV_TX) ? ci / TRAV_TX : ci / wx;
    const unsigned cx = ci - cy * wx;
    lc[0] = (int)(p.task_lo[0] + tx * TRAV_TX + cx);
    lc[1] = (int)(p.task_lo[1] + ty * TRAV_TY + cy);
    lc[2] = (int)(p.task_lo[2] + (task - col * nz));
}

// ---------------------------------------------------------------------------------- store epilogue
// The single store of a cell's y block, with the explicit-step arithmetic of PAPER.md:366-373
// fused in (M = Delta_T I for the orthonormal basis on cuboid cells, so M^-1 is a scalar):
//   epi 0: y = A z      epi 1: y = f - A z      epi 2: y = a w + b (z + (dt/Delta_T)(f - A z))
// (one Shu-Osher stage of an SSP Runge-Kutta method; f or w may be absent = 0). Every value
// read here belongs to this thread's own x-line of this cell.
template <int N>
__device__ __forceinline__ void epilogue(const KParams& p, int64_t off, double (&t)[N])
{
    if (p.epi == 1) {
#pragma unroll
        for (int e = 0; e < N; ++e) t[e] = __ldg(p.f + off + e) - t[e];
    } else if (p.epi == 2) {
#pragma unroll
        for (int e = 0; e < N; ++e) {
            const double r = (p.f ? __ldg(p.f + off + e) : 0.0) - t[e];
            const double v = fma(p.es, r, __ldg(p.z + off + e));
            t[e] = p.w ? fma(p.ea, __ldg(p.w + off + e), p.eb * v) : p.eb * v;
        }
    }
}

// ---------------------------------------------------------------------------------- kernel
template <int N, bool GH>
__global__ void __launch_bounds__(Cfg<N>::C * Cfg<N>::TPC, Cfg<N>::MINB)
dg_cell_kernel(const __grid_constant__ KParams p)
{
    constexpr int TPC = Cfg<N>::TPC, P = Cfg<N>::P, C = Cfg<N>::C;
    constexpr int NN = N * N;
    static_assert(N == DG_N, "one degree per translation unit");
    static_assert(TPC * P >= NN, "pencil slots");
    extern __shared__ double smem[];
    const Tab<N>& T = g_tab;

    const int tid = threadIdx.x;
    const int slot = tid / TPC;
    const int lane = tid - slot * TPC;

    double* A0 = smem + slot * Smem<N>::PER_CELL;
    double* A1 = A0 + Lay<N>::SLOT;
    double* NT = A1 + Lay<N>::SLOT;

    auto csync = [&]() {
        if (32 % TPC == 0) __syncwarp(); else __syncthreads();   // a cell within one warp, else CTA-wide
    };

    // ---- cell of this slot (32-bit index math: at most 2^31 cells per rank)
    unsigned task = blockIdx.x * (unsigned)C + (unsigned)slot;
    const bool valid = task < (unsigned)p.ntasks;
    if (!valid) task = (unsigned)p.ntasks - 1u;
    int lc[3];
    if (p.task_list) {
        const unsigned e = (unsigned)p.task_list[task];
        const unsigned nx = (unsigned)p.nloc[0], ny = (unsigned)p.nloc[1];
        lc[0] = (int)(e % nx);
        lc[1] = (int)((e / nx) % ny);
        lc[2] = (int)(e / (nx * ny));
    } else {
        decode_task(p, task, lc);
    }
    const int64_t n3 = (int64_t)NN * N;
    const int64_t cell = lc[0] + p.nloc[0] * (lc[1] + p.nloc[1] * (int64_t)lc[2]);
    DG_ASSERT(lc[0] >= 0 && lc[0] < p.nloc[0] && lc[1] >= 0 && lc[1] < p.nloc[1] && lc[2] >= 0 && lc[2] < p.nloc[2]);
    const double* zc = p.z + cell * n3;
    const bool do_int = (p.mask & 2u) != 0, do_bnd = (p.mask & 4u) != 0, do_vol = (p.mask & 1u) != 0;

    unsigned nbmask = 0;   // bit f = 2q + s: a neighbour cell (local or on another rank) exists
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int q = f >> 1, s = f & 1;
        const int64_t g = p.gofs[q] + lc[q] + (s ? 1 : -1);
        if (p.per[q] || (g >= 0 && g < p.gcells[q])) nbmask |= 1u << f;
    }
    const unsigned nbi = do_int ? nbmask : 0u;   // neighbours whose traces are needed

    // this thread's pencils: pencil index pc = lane + k TPC = a + N bb
    int pa[P], pb[P];
    bool act[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const int pc = lane + k * TPC;
        act[k] = pc < NN;
        const int pcc = act[k] ? pc : 0;
        pa[k] = pcc % N;
        pb[k] = pcc / N;
    }

    double r[P][N], t[P][N];
    // TMA staging (n = 8, one cell per CTA): own block and the local x-neighbours' blocks
    double* STG = nullptr;
    bool tma_x = false;
    if constexpr (N == 8 && C == 1) {
        if (p.tma) {
            STG = reinterpret_cast<double*>(
                (reinterpret_cast<uintptr_t>(smem + Smem<N>::PER_CELL) + 127) & ~(uintptr_t)127);
            tma_x = tma::stage_x(p, STG, A1, NT + XH8, tid, lc, cell, nbi);
        }
    }
    // bulk staging of the own block (n = 7, 9, 10, 11) in A1, free in phase 1 (C4 k = 6 / 8 / 9 / 10:
    // 58.6 -> 60.0, 51.9 -> 54.5, 51.6 -> 53.7, 50.3 -> 53.4 GDOF/s; n = 6 measured 62.8 -> 60.9: off)
    constexpr bool BULK = (N >= 7 && N != 8);
    static_assert(!BULK || Lay<N>::SLOT >= NN * N + 1, "A1 holds the shifted block image");
    double* SB = nullptr;
    bulk::Span bs{};
    if constexpr (BULK) {
        if (p.tma) {
            uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + C * Smem<N>::PER_CELL);
            bs = bulk::span<N>(zc, A1);
            SB = A1 + bs.sh;
            if (tid == 0) tma::mbar_init_n(mbar, C);
            __syncthreads();
            if (lane == 0) {
                tma::expect_tx(mbar, bs.bytes);
                bulk::load(SB + bs.hd, zc + bs.hd, bs.bytes, mbar);
            }
            tma::wait(mbar, 0);
        }
    }
    {
        double rl[P][N], rh[P][N];
        unsigned gm0 = 0;   // ghost x-neighbours (never TMA-staged)
        // ---- phase 1: x-pencils (y = a, z = bb) from global, V along x -> A0;
        //      x-neighbour lines loaded alongside and contracted (normal first)
        if (tma_x) {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int L = pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; e += 2) {
                    const double2 a = tma::line2(STG, L, e);
                    const double2 lo = tma::line2(A1, L, e);
                    const double2 hi = tma::line2(NT + XH8, L, e);
                    r[k][e] = a.x; r[k][e + 1] = a.y;
                    rl[k][e] = lo.x; rl[k][e + 1] = lo.y;
                    rh[k][e] = hi.x; rh[k][e + 1] = hi.y;
                }
            }
        } else {
        gm0 = nb_load<N, P, GH>(p, zc, n3, 0, lc, nbi, pa, pb, act, rl, rh);
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (STG) {
                const int L = pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; e += 2) {
                    const double2 a = tma::line2(STG, L, e);
                    r[k][e] = a.x; r[k][e + 1] = a.y;
                }
                continue;
            }
            if (BULK && SB) {
                const double* src = SB + N * (pa[k] + N * pb[k]);
                if (N % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < N; e += 2) {
                        const double2 v = act[k] ? *reinterpret_cast<const double2*>(src + e) : make_double2(0.0, 0.0);
                        r[k][e] = v.x;
                        r[k][e + 1] = v.y;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < N; ++e) r[k][e] = act[k] ? src[e] : 0.0;
                }
                continue;
            }
            const double* src = zc + N * (pa[k] + N * pb[k]);
            if (N % 2 == 0) {
#pragma unroll
                for (int e = 0; e < N; e += 2) {
                    const double2 v = act[k] ? __ldg(reinterpret_cast<const double2*>(src + e)) : make_double2(0.0, 0.0);
                    r[k][e] = v.x;
                    r[k][e + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < N; ++e) r[k][e] = act[k] ? __ldg(src + e) : 0.0;
            }
        }
        if (BULK && SB) {   // the plain leading / trailing doubles of the block
            if (bs.hd && lane == 0) r[0][0] = __ldg(zc);
            if (bs.tl && lane == (NN - 1) % TPC) r[(NN - 1) / TPC][N - 1] = __ldg(zc + NN * N - 1);
        }
        }
        v_fwd_sd<N, P>(T.Vs[0], r, t);
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) A0[Lay<N>::at(e, pa[k], pb[k])] = t[k][e];
        nb_contract<N, P>(T, NT, 0, nbi, pa, pb, act, rl, rh, gm0);
#ifndef DG_EARLYNB
#define DG_EARLYNB 1
#endif
        // each phase's neighbour loads issued before the previous phase's barrier, so they fly during
        // the wait (A/B on one box: C3 +0.2 %, A-k7 +0.5 %, A-k10 +0.7 %; the fast n = 11 -0.5 %: off)
        constexpr bool ENB = DG_EARLYNB && N != 11;
        unsigned gm1 = 0;
        if (ENB) gm1 = nb_load<N, P, GH>(p, zc, n3, 1, lc, nbi, pa, pb, act, rl, rh);
        csync();

        // ---- phase 2: y-pencils (x = a, z = bb): V along y -> A1; y-neighbours; x-arrays step B
        if (!ENB) gm1 = nb_load<N, P, GH>(p, zc, n3, 1, lc, nbi, pa, pb, act, rl, rh);
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
        v_fwd_sd<N, P>(T.Vs[1], r, t);
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) A1[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
        nb_tangential<N, TPC>(T.Vs[2], NT, 0, 0, nbi, (lane + TPC / 2) % TPC);
        nb_contract<N, P>(T, NT, 1, nbi, pa, pb, act, rl, rh, gm1);
        unsigned gm2 = 0;
        if (ENB) gm2 = nb_load<N, P, GH>(p, zc, n3, 2, lc, nbi, pa, pb, act, rl, rh);
        csync();

        // ---- phase 3: z-pencils (x = a, y = bb): u at the Gauss points -> A0; z-neighbours;
        //      y-arrays step B, x-arrays step C
        if (!ENB) gm2 = nb_load<N, P, GH>(p, zc, n3, 2, lc, nbi, pa, pb, act, rl, rh);
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A1[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
        v_fwd_sd<N, P>(T.Vs[3], r, t);
#pragma unroll
        for (int k = 0; k < P; ++k)
            if (act[k])
#pragma unroll
                for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = t[k][e];
        nb_tangential<N, TPC>(T.Vs[4], NT, 1, 0, nbi, lane);
        nb_tangential<N, TPC>(T.Vs[5], NT, 0, 1, nbi, (lane + TPC / 2) % TPC);
        nb_contract<N, P>(T, NT, 2, nbi, pa, pb, act, rl, rh, gm2);
        csync();
    }

    // ---- phase 4: x role -> T1 = Dc^T x^(1) + x-face lifts -> A1; z-arrays step B, y step C
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    role_eo<N, P>(p, T, NT, 0, nbmask, do_int, do_bnd, do_vol, false, pa, pb, r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A1[Lay<N>::at(e, pa[k], pb[k])] = t[k][e];
    nb_tangential<N, TPC>(T.Vs[6], NT, 2, 0, nbi, lane);
    nb_tangential<N, TPC>(T.Vs[7], NT, 1, 1, nbi, (lane + TPC / 2) % TPC);
    csync();

    // ---- phase 5: y role -> A1 += T2; z-arrays step C
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    role_eo<N, P>(p, T, NT, 1, nbmask, do_int, do_bnd, do_vol, false, pa, pb, r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) {
                const int ie = Lay<N>::at(pa[k], e, pb[k]);
                A1[ie] = A1[ie] + t[k][e];
            }
    nb_tangential<N, TPC>(T.Vs[8], NT, 2, 1, nbi, lane);
    csync();

    // ---- phase 6: z role (+ reaction) -> X = T1 + T2 + T3; V^T along z -> A0
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
    role_eo<N, P>(p, T, NT, 2, nbmask, do_int, do_bnd, do_vol, true, pa, pb, r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) t[k][e] += act[k] ? A1[Lay<N>::at(pa[k], pb[k], e)] : 0.0;
    v_bwd_sd<N, P>(T.Vh[9], t, r);   // in place: A0 z-positions of this pencil are read only by this thread
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], pb[k], e)] = r[k][e];
    csync();

    // ---- phase 7: y-pencils: V^T along y (in place)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(pa[k], e, pb[k])] : 0.0;
    v_bwd_sd<N, P>(T.Vh[10], r, t);
#pragma unroll
    for (int k = 0; k < P; ++k)
        if (act[k])
#pragma unroll
            for (int e = 0; e < N; ++e) A0[Lay<N>::at(pa[k], e, pb[k])] = t[k][e];
    csync();

    // ---- phase 8: x-pencils: V^T along x, then the single store of y (or f - y)
#pragma unroll
    for (int k = 0; k < P; ++k)
#pragma unroll
        for (int e = 0; e < N; ++e) r[k][e] = act[k] ? A0[Lay<N>::at(e, pa[k], pb[k])] : 0.0;
    v_bwd_sd<N, P>(T.Vh[11], r, t);
    if constexpr (N == 8 && C == 1) {
        if (STG && p.tma == 2 && p.epi == 0) {   // y through the staging block and one TMA store
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const int L = pa[k] + N * pb[k];
#pragma unroll
                for (int e = 0; e < N; e += 2) tma::put2(STG, L, e, t[k][e], t[k][e + 1]);
            }
            tma::store_block(p, STG, tid, cell);
            return;
        }
    }
    if constexpr (BULK) {
        if (p.tma == 2 && p.epi == 0) {   // y through the linear image in A1 (free) and one bulk store
            double* yc = p.y + cell * n3;
            const bulk::Span ys = bulk::span<N>(yc, A1);
            double* S = A1 + ys.sh;
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (!act[k]) continue;
                double* dst = S + N * (pa[k] + N * pb[k]);
                if (N % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < N; e += 2) *reinterpret_cast<double2*>(dst + e) = make_double2(t[k][e], t[k][e + 1]);
                } else {
#pragma unroll
                    for (int e = 0; e < N; ++e) dst[e] = t[k][e];
                }
            }
            if (valid) {
                if (ys.hd && lane == 0) __stcs(yc, t[0][0]);
                if (ys.tl && lane == (NN - 1) % TPC) __stcs(yc + NN * N - 1, t[(NN - 1) / TPC][N - 1]);
            }
            tma::fence_async();
            __syncthreads();
            if (valid && lane == 0) bulk::store(yc + ys.hd, S + ys.hd, ys.bytes);
            return;
        }
    }
    if (valid) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (!act[k]) continue;
            const int64_t off = cell * n3 + N * (pa[k] + N * pb[k]);
            double* yc = p.y + off;
            epilogue<N>(p, off, t[k]);
            if (N % 2 == 0) {
#pragma unroll
                for (int e = 0; e < N; e += 2)
                    __stcs(reinterpret_cast<double2*>(yc + e), make_double2(t[k][e], t[k][e + 1]));
            } else {
#pragma unroll
                for (int e = 0; e < N; ++e) __stcs(yc + e, t[k][e]);
            }
        }
    }
}

}  // namespace dg

// k = 7 (n = 8) cell kernel on the FP64 tensor cores: every 1D contraction of the sum
// factorization is a warp-level DMMA (mma.sync m8n8k4 f64; SASS DMMA.8x8x4).
//
// Why: on sm_100a the FP64 tensor path runs at the same peak as the DFMA pipe (measured
// 37.2 vs 33.7 TFLOP/s, tools/fp64_peaks.cu; tcgen05 has no f64 kind), but one DMMA issues
// 256 FMAs where the SIMT stage needs 8 DFMA + 4 uniform-constant loads per 32 FMAs. The
// SIMT kernel (dg_cell.cuh) is issue/latency bound at ~50 % of the FP64 pipe; this one
// moves ~5x fewer instructions per cell.
//
// One warp per cell (lane l: g = l >> 2, t = l & 3). A direction-q "fragment" F[nt][c] holds
// element e = 2t + c along q of the pencil (g, nt), with the pencil coordinates
//   q = x: (x, y, z) = (e, g, nt)   q = y: (nt, e, g)   q = z: (g, nt, e).
// A stage out = M in along q is D = in^T M^T in the m8n8k4 "form 2": rows = 8 pencils of
// n-tile nt, k = element index permuted as kappa(c, t) = 2t + c, so the accumulator of one
// stage (D[g][2t + u]) is directly the A operand of the next stage in the same direction
// (the role: Dc -> pointwise -> Dc^T -> lifts stays in registers). Stages that change
// direction go through shared memory with an XOR swizzle that is bank-conflict free for
// every fragment pattern (checked exhaustively offline).
//
// Mathematics as in dg_cell.cuh (Algorithm 1; eq:blf :301-315;
// sum factorization :573-604; faces normal-first / normal-last :623-627).
#pragma once

namespace dg {
namespace m8 {

// per-lane constant fragments (global memory, read once per thread)
enum { F_VF0, F_VF1, F_VB0, F_VB1, F_DC0, F_DC1, F_DT0, F_DT1, F_LT0, F_LT1, F_LL, F_WG, F_WT0, F_WT1, F_COUNT };
__device__ double g_frag[32][16];

__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// cell array swizzle (512 doubles): conflict free for the fragment patterns of all 3 directions
// (bank = low 4 bits of the double index: 16 lanes of each half-warp hit 16 distinct banks)
__device__ __forceinline__ int L(int x, int y, int z)
{
    const int f = (((y >> 1) ^ z) & 1) | (((y >> 2) & 1) << 1) | ((((z >> 1) ^ (z >> 2)) & 1) << 2);
    return (x ^ f) + 8 * (y ^ ((z ^ (z >> 1)) & 1)) + 64 * z;
}
// element e of pencil (g, nt) in direction q
__device__ __forceinline__ int Lq(int q, int e, int g, int nt)
{
    return (q == 0) ? L(e, g, nt) : (q == 1) ? L(nt, e, g) : L(g, nt, e);
}
// face arrays (12 x 64): (i1, i2) = tangential coordinates (t1 < t2)
__device__ __forceinline__ int LN(int arr, int i1, int i2)
{
    return 64 * arr + (i1 ^ ((i2 & 1) | (((i2 >> 1) & 1) << 2))) + 8 * (i2 ^ (((i2 >> 1) ^ (i2 >> 2)) & 1));
}

constexpr int PER_CELL = 512 * 2 + 12 * 64;   // A0, A1, face arrays (doubles)
constexpr int C = 1;                           // cells (warps) per CTA
constexpr int MINB = 14;

struct Frag {
    double vf[2], vb[2], dc[2], dt[2], lt[2], ll, wg, wt[2];
};

// one stage on the 8 n-tiles: out[nt] = sum_c mma(in[nt][c], m[c])
__device__ __forceinline__ void stage(const double (&in)[8][2], const double (&m)[2], double (&out)[8][2])
{
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        double d0 = 0.0, d1 = 0.0;
        mma(d0, d1, in[nt][0], m[0]);
        mma(d0, d1, in[nt][1], m[1]);
        out[nt][0] = d0;
        out[nt][1] = d1;
    }
}

__device__ __forceinline__ void load_q(const double* A, int q, int g, int t, double (&F)[8][2])
{
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        F[nt][0] = A[Lq(q, 2 * t, g, nt)];
        F[nt][1] = A[Lq(q, 2 * t + 1, g, nt)];
    }
}
__device__ __forceinline__ void store_q(double* A, int q, int g, int t, const double (&F)[8][2])
{
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        A[Lq(q, 2 * t, g, nt)] = F[nt][0];
        A[Lq(q, 2 * t + 1, g, nt)] = F[nt][1];
    }
}

// tangential stage (V along i1 when dim = 0, along i2 when dim = 1) of the 4 face arrays of
// direction qf: each 8 x 8 array is one n-tile (pencils = the other index = g)
__device__ __forceinline__ void tangential(double* NT, int qf, int dim, unsigned nbi, int g, int t, const Frag& fr)
{
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int arr = 4 * qf + j;
        if (!((nbi >> (arr >> 1)) & 1u)) continue;
        const int i00 = dim ? LN(arr, g, 2 * t) : LN(arr, 2 * t, g);
        const int i01 = dim ? LN(arr, g, 2 * t + 1) : LN(arr, 2 * t + 1, g);
        const double a0 = NT[i00], a1 = NT[i01];
        double d0 = 0.0, d1 = 0.0;
        mma(d0, d1, a0, fr.vf[0]);
        mma(d0, d1, a1, fr.vf[1]);
        NT[i00] = d0;
        NT[i01] = d1;
    }
}

// SIMT normal-first contraction of the two q-neighbours (thread: lines (a, b) and (a, b + 4))
template <int SIDE>
__device__ __forceinline__ void nb_face(const KParams& p, const Tab<8>& T, double* NT, const double* zc, int64_t n3,
                                        int q, const int (&lc)[3], unsigned nbi, int lane)
{
    const int f = 2 * q + SIDE;
    if (!((nbi >> f) & 1u)) return;
    const int lq = lc[q];
    const int64_t st = (q == 0) ? 1 : (q == 1) ? p.nloc[0] : p.nloc[0] * p.nloc[1];
    const int64_t nq = p.nloc[q];
    const double* zn;
    if (SIDE ? (lq + 1 < nq) : (lq > 0)) {
        zn = zc + (SIDE ? st : -st) * n3;
    } else {
        const int64_t gi = (q == 0) ? (lc[1] + p.nloc[1] * lc[2]) : (q == 1) ? (lc[0] + p.nloc[0] * lc[2])
                                                                            : (lc[0] + p.nloc[0] * lc[1]);
        zn = p.ghost[f] + gi * n3;   // unreachable: launch_cell runs this variant on single-rank boxes only
    }
    const int se = (q == 0) ? 1 : (q == 1) ? 8 : 64;
    const double* thv = SIDE ? T.th0 : T.th1;      // neighbour face at x_q = 1 - SIDE
    const double* dthv = SIDE ? T.dth0 : T.dth1;
    const int a = lane & 7, b0 = lane >> 3;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int b = b0 + 4 * k;
        const int base = (q == 0) ? 8 * a + 64 * b : (q == 1) ? a + 64 * b : a + 8 * b;
        double v[8];
        if (q == 0) {
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const double2 w = __ldg(reinterpret_cast<const double2*>(zn + base + e));
                v[e] = w.x;
                v[e + 1] = w.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __ldg(zn + base + e * se);
        }
        double su = 0.0, sd = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            su = fma(thv[e], v[e], su);
            sd = fma(dthv[e], v[e], sd);
        }
        NT[LN(2 * f, a, b)] = su;
        NT[LN(2 * f + 1, a, b)] = sd;
    }
}

// Face-flux coefficients of one face (uniform per cell): the SIPG + upwind terms are linear in
// (u own, d own = d u/dx_hat_q own, u neighbour, d neighbour); cv = Wf (k . v), cg = Wf (k' . v).
// This lane's coefficient: t = 0 -> cv of face s = 0, 1 -> cv(s = 1), 2 -> cg(s = 0), 3 -> cg(s = 1).
struct FaceK { double ku, kd, kn, ks; };   // ks multiplies D_qq/h_q * (neighbour d u/dx_hat_q)

__device__ __forceinline__ FaceK face_coeffs(const KParams& p, int q, int s, int kind_cg, bool interior, bool active_int,
                                            bool active_bnd)
{
    const double b = p.bq[q], g = p.gam[q], dh = p.Dqq_h[q];
    const double bp = b >= 0.0 ? b : 0.0, bm = b < 0.0 ? b : 0.0;
    FaceK k = {0.0, 0.0, 0.0, 0.0};
    if (interior) {
        if (!active_int) return k;
        // Phi, J = u- - u+, Avg = (s- + s+)/2 (C-1), gamma J (C-4); s = 1: own = T-
        if (!kind_cg) {
            if (s) { k.ku = bp + g; k.kn = bm - g; k.kd = -0.5 * dh; k.ks = -0.5; }
            else   { k.ku = g - bm; k.kn = -bp - g; k.kd = 0.5 * dh; k.ks = 0.5; }
        } else {
            const double sg = s ? -0.5 * dh : 0.5 * dh;   // -(nu.{D grad phi}_w, [[u]])
            k.ku = sg;
            k.kn = -sg;
        }
    } else {
        if (!active_bnd) return k;
        const double nu = s ? 1.0 : -1.0, bn = nu * b;   // PAPER.md:282-286, :309-313, C-6
        if (!kind_cg) { k.ku = (bn >= 0.0 ? bn : 0.0) + g; k.kd = -nu * dh; }
        else { k.ku = -nu * dh; }
    }
    return k;
}

// role of direction Q on u fragments U (element i = 2t + c of pencil (g, nt)):
// T = Dc^T [W (D_qq/h_q^2 Dc u - b_q/h_q u)] (+ W c u for Q = z) + lifts of the two Q-faces
template <int Q>
__device__ __forceinline__ void role(const KParams& p, const Tab<8>& T, const double* NT, unsigned nbmask,
                                     bool do_int, bool do_bnd, bool do_vol, int g, int t, const Frag& fr,
                                     const double (&U)[8][2], double (&Tout)[8][2])
{
    const double kd = p.Dhat[4 * Q], kb = p.kb[Q];
    const double wvol = do_vol ? p.dT * fr.wg : 0.0;
    const double wk0 = wvol * fr.wt[0] * kd, wk1 = wvol * fr.wt[1] * kd;
    const double wb0 = wvol * fr.wt[0] * kb, wb1 = wvol * fr.wt[1] * kb;
    const double wc0 = wvol * fr.wt[0] * p.c, wc1 = wvol * fr.wt[1] * p.c;
    // this lane's face coefficient (uniform per cell, no branches in the tile loop)
    const int s = t & 1, kind = t >> 1;
    const int f = 2 * Q + s;
    const bool interior = (nbmask >> f) & 1u;
    const FaceK fk = face_coeffs(p, Q, s, kind, interior, do_int, do_bnd);
    const double wf = p.dF[Q] * fr.wg;
    const double ksn = fk.ks * p.Dqq_h[Q];
    const int arr_u = 2 * f, arr_d = 2 * f + 1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        // Dc along Q, then the quadrature-point data (eq:gauss_points)
        double g0 = 0.0, g1 = 0.0;
        mma(g0, g1, U[nt][0], fr.dc[0]);
        mma(g0, g1, U[nt][1], fr.dc[1]);
        const double wn = T.w[nt];
        const double x0 = wn * (wk0 * g0 - wb0 * U[nt][0]);
        const double x1 = wn * (wk1 * g1 - wb1 * U[nt][1]);
        double o0 = 0.0, o1 = 0.0;
        if (Q == 2) { o0 = wn * wc0 * U[nt][0]; o1 = wn * wc1 * U[nt][1]; }   // reaction x^(0)
        mma(o0, o1, x0, fr.dt[0]);
        mma(o0, o1, x1, fr.dt[1]);
        // own traces (u(0), u(1), u'(0), u'(1)) of pencil g: lanes t = 0 (r 0,1), t = 1 (r 2,3)
        double r0 = 0.0, r1 = 0.0;
        mma(r0, r1, U[nt][0], fr.lt[0]);
        mma(r0, r1, U[nt][1], fr.lt[1]);
        const int src = g << 2;
        const double ua = __shfl_sync(0xffffffffu, r0, src), ub = __shfl_sync(0xffffffffu, r1, src);
        const double da = __shfl_sync(0xffffffffu, r0, src + 1), db = __shfl_sync(0xffffffffu, r1, src + 1);
        const double uo = s ? ub : ua, dref = s ? db : da;
        // neighbour trace at the face point of pencil (g, nt)
        const int i1 = (Q == 1) ? nt : g, i2 = (Q == 1) ? g : nt;
        const double un = interior ? NT[LN(arr_u, i1, i2)] : 0.0;
        const double sn = interior ? NT[LN(arr_d, i1, i2)] : 0.0;
        const double coef = wf * wn * (fk.ku * uo + fk.kd * dref + fk.kn * un + ksn * sn);
        // lift (normal direction LAST): k = t against (L0, L1, L'0, L'1)
        mma(o0, o1, coef, fr.ll);
        Tout[nt][0] = o0;
        Tout[nt][1] = o1;
    }
}

__global__ void __launch_bounds__(32 * C, MINB) dg_cell_mma8(const KParams p)
{
    extern __shared__ double smem[];
    const Tab<8>& T = g_tab;
    const int lane = threadIdx.x & 31;
    const int slot = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* A0 = smem + slot * PER_CELL;
    double* A1 = A0 + 512;
    double* NT = A1 + 512;

    Frag fr;
    {
        const double* fp = g_frag[lane];
        fr.vf[0] = fp[F_VF0]; fr.vf[1] = fp[F_VF1];
        fr.vb[0] = fp[F_VB0]; fr.vb[1] = fp[F_VB1];
        fr.dc[0] = fp[F_DC0]; fr.dc[1] = fp[F_DC1];
        fr.dt[0] = fp[F_DT0]; fr.dt[1] = fp[F_DT1];
        fr.lt[0] = fp[F_LT0]; fr.lt[1] = fp[F_LT1];
        fr.ll = fp[F_LL]; fr.wg = fp[F_WG];
        fr.wt[0] = fp[F_WT0]; fr.wt[1] = fp[F_WT1];
    }

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
    const int64_t n3 = 512;
    const int64_t cell = lc[0] + p.nloc[0] * (lc[1] + p.nloc[1] * (int64_t)lc[2]);
    DG_ASSERT(lc[0] >= 0 && lc[0] < p.nloc[0] && lc[1] >= 0 && lc[1] < p.nloc[1] && lc[2] >= 0 && lc[2] < p.nloc[2]);
    const double* zc = p.z + cell * n3;
    const bool do_int = (p.mask & 2u) != 0, do_bnd = (p.mask & 4u) != 0, do_vol = (p.mask & 1u) != 0;
    unsigned nbmask = 0;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int q = f >> 1, s = f & 1;
        const int64_t gg = p.gofs[q] + lc[q] + (s ? 1 : -1);
        if (gg >= 0 && gg < p.gcells[q]) nbmask |= 1u << f;
    }
    const unsigned nbi = do_int ? nbmask : 0u;

    double Fa[8][2], Fb[8][2];

    // ---- phase 1: x-stage from HBM (pencil (y, z) = (g, nt), x = 2t, 2t+1: one 16-byte load)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(zc + 2 * t + 8 * g + 64 * nt));
        Fa[nt][0] = v.x;
        Fa[nt][1] = v.y;
    }
    nb_face<0>(p, T, NT, zc, n3, 0, lc, nbi, lane);
    stage(Fa, fr.vf, Fb);
    store_q(A0, 0, g, t, Fb);
    nb_face<1>(p, T, NT, zc, n3, 0, lc, nbi, lane);
    __syncwarp();

    // ---- phase 2: y-stage; y-neighbours; x-face arrays along i1
    nb_face<0>(p, T, NT, zc, n3, 1, lc, nbi, lane);
    load_q(A0, 1, g, t, Fa);
    stage(Fa, fr.vf, Fb);
    store_q(A1, 1, g, t, Fb);
    tangential(NT, 0, 0, nbi, g, t, fr);
    nb_face<1>(p, T, NT, zc, n3, 1, lc, nbi, lane);
    __syncwarp();

    // ---- phase 3: z-stage -> u at the Gauss points (A0); z-neighbours; y arrays along i1, x along i2
    nb_face<0>(p, T, NT, zc, n3, 2, lc, nbi, lane);
    load_q(A1, 2, g, t, Fa);
    stage(Fa, fr.vf, Fb);
    store_q(A0, 2, g, t, Fb);
    tangential(NT, 1, 0, nbi, g, t, fr);
    tangential(NT, 0, 1, nbi, g, t, fr);
    nb_face<1>(p, T, NT, zc, n3, 2, lc, nbi, lane);
    __syncwarp();

    // ---- phase 4: x role -> A1; z arrays along i1, y arrays along i2
    tangential(NT, 2, 0, nbi, g, t, fr);
    tangential(NT, 1, 1, nbi, g, t, fr);
    load_q(A0, 0, g, t, Fa);
    role<0>(p, T, NT, nbmask, do_int, do_bnd, do_vol, g, t, fr, Fa, Fb);
    store_q(A1, 0, g, t, Fb);
    __syncwarp();

    // ---- phase 5: y role, accumulated into A1; z arrays along i2
    tangential(NT, 2, 1, nbi, g, t, fr);
    load_q(A0, 1, g, t, Fa);
    role<1>(p, T, NT, nbmask, do_int, do_bnd, do_vol, g, t, fr, Fa, Fb);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        const int i0 = Lq(1, 2 * t, g, nt), i1 = Lq(1, 2 * t + 1, g, nt);
        A1[i0] += Fb[nt][0];
        A1[i1] += Fb[nt][1];
    }
    __syncwarp();

    // ---- phase 6: z role (+ reaction) + T_x + T_y, then V^T along z -> A0
    load_q(A0, 2, g, t, Fa);
    role<2>(p, T, NT, nbmask, do_int, do_bnd, do_vol, g, t, fr, Fa, Fb);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        Fb[nt][0] += A1[Lq(2, 2 * t, g, nt)];
        Fb[nt][1] += A1[Lq(2, 2 * t + 1, g, nt)];
    }
    stage(Fb, fr.vb, Fa);
    store_q(A0, 2, g, t, Fa);
    __syncwarp();

    // ---- phase 7: V^T along y (in place)
    load_q(A0, 1, g, t, Fa);
    stage(Fa, fr.vb, Fb);
    store_q(A0, 1, g, t, Fb);
    __syncwarp();

    // ---- phase 8: V^T along x -> y (or f - y): pencil (y, z) = (g, nt), x = 2t, 2t+1
    load_q(A0, 0, g, t, Fa);
    stage(Fa, fr.vb, Fb);
    if (valid) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const int64_t off = cell * n3 + 2 * t + 8 * g + 64 * nt;
            double y0 = Fb[nt][0], y1 = Fb[nt][1];
            if (p.epi == 1) {
                const double2 fv = __ldg(reinterpret_cast<const double2*>(p.f + off));
                y0 = fv.x - y0;
                y1 = fv.y - y1;
            }
            __stcs(reinterpret_cast<double2*>(p.y + off), make_double2(y0, y1));
        }
    }
}

}  // namespace m8
}  // namespace dg
